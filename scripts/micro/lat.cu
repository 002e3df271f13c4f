// Microbenchmark: dependent-chain latency and throughput of DFMA / FFMA /
// DP rcp.approx / DSETP-select on this GPU.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void chain_d(double* out, double a, double b, int n, long long* cyc) {
  double x = threadIdx.x * 1e-3;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = fma(x, a, b); x = fma(x, a, b); x = fma(x, a, b); x = fma(x, a, b); }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[threadIdx.x + blockIdx.x * blockDim.x] = x;
}
__global__ void chain_f(float* out, float a, float b, int n, long long* cyc) {
  float x = threadIdx.x * 1e-3f;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = fmaf(x, a, b); x = fmaf(x, a, b); x = fmaf(x, a, b); x = fmaf(x, a, b); }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[threadIdx.x + blockIdx.x * blockDim.x] = x;
}
__global__ void chain_rcp(double* out, int n, long long* cyc) {
  double x = 1.5 + threadIdx.x * 1e-3;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { double r; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); x = r + 1.0; }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[threadIdx.x + blockIdx.x * blockDim.x] = x;
}
// throughput: 8 independent chains per thread
__global__ void thr_d(double* out, double a, double b, int n) {
  double x[8];
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3 + k;
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
  double s = 0; for (int k = 0; k < 8; ++k) s += x[k];
  out[threadIdx.x + blockIdx.x * blockDim.x] = s;
}
__global__ void thr_f(float* out, float a, float b, int n) {
  float x[8];
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3f + k;
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = fmaf(x[k], a, b);
  float s = 0; for (int k = 0; k < 8; ++k) s += x[k];
  out[threadIdx.x + blockIdx.x * blockDim.x] = s;
}
__global__ void rcp_err(double* out, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  double x = 1.0 + (double)i / n * 3.0;
  double r; asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double y; asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  out[2 * i] = fabs(r * x - 1.0);
  out[2 * i + 1] = fabs(y * y * x - 1.0);
}
int main() {
  double* dd; float* df; long long* cyc;
  cudaMalloc(&dd, 1 << 26); cudaMalloc(&df, 1 << 26); cudaMalloc(&cyc, 8 * 1024);
  long long h[1];
  int n = 4096;
  chain_d<<<1, 32>>>(dd, 0.999, 1e-3, n, cyc); cudaDeviceSynchronize();
  chain_d<<<1, 32>>>(dd, 0.999, 1e-3, n, cyc); cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("DFMA dependent latency: %.2f cycles\n", (double)h[0] / (4.0 * n));
  chain_f<<<1, 32>>>(df, 0.999f, 1e-3f, n, cyc); cudaDeviceSynchronize();
  chain_f<<<1, 32>>>(df, 0.999f, 1e-3f, n, cyc); cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("FFMA dependent latency: %.2f cycles\n", (double)h[0] / (4.0 * n));
  chain_rcp<<<1, 32>>>(dd, n, cyc); cudaDeviceSynchronize();
  chain_rcp<<<1, 32>>>(dd, n, cyc); cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("rcp.approx.f64 + DADD dependent latency: %.2f cycles\n", (double)h[0] / n);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int blocks = 148 * 16, threads = 256, m = 2048;
  thr_d<<<blocks, threads>>>(dd, 0.999, 1e-3, m);
  cudaEventRecord(e0); thr_d<<<blocks, threads>>>(dd, 0.999, 1e-3, m); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("DFMA throughput: %.1f TFLOP/s (FMA=2)\n", 2.0 * blocks * threads * m * 8 / (ms * 1e-3) / 1e12);
  thr_f<<<blocks, threads>>>(df, 0.999f, 1e-3f, m);
  cudaEventRecord(e0); thr_f<<<blocks, threads>>>(df, 0.999f, 1e-3f, m); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("FFMA throughput: %.1f TFLOP/s (FMA=2)\n", 2.0 * blocks * threads * m * 8 / (ms * 1e-3) / 1e12);
  int N = 1 << 20; rcp_err<<<N / 256, 256>>>(dd, N);
  double* hh = (double*)malloc(16 * N); cudaMemcpy(hh, dd, 16 * N, cudaMemcpyDeviceToHost);
  double mr = 0, ms2 = 0; for (int i = 0; i < N; ++i) { if (hh[2*i] > mr) mr = hh[2*i]; if (hh[2*i+1] > ms2) ms2 = hh[2*i+1]; }
  printf("rcp.approx.f64 max rel err %.3g (2^%.1f); rsqrt.approx.f64 max (y^2 x - 1) %.3g (2^%.1f)\n", mr, log2(mr), ms2, log2(ms2));
  return 0;
}
