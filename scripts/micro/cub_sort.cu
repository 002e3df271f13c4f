// Yardstick: CUB DeviceRadixSort::SortPairs (onesweep) on E 64-bit keys with a
// 45-bit range + uint32 values, the shape of K4.  Prints ms per sort.
#include <cub/cub.cuh>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <random>
int main(int argc, char** argv) {
  const int E = argc > 1 ? atoi(argv[1]) : 6500000;
  const int bits = argc > 2 ? atoi(argv[2]) : 45;
  std::vector<unsigned long long> hk(E);
  std::vector<unsigned> hv(E);
  std::mt19937_64 rng(1);
  for (int i = 0; i < E; ++i) {
    unsigned long long tile = rng() % 8160;
    unsigned key = 0x80000000u | (unsigned)(rng() & 0x7fffffff);
    hk[i] = (tile << 32) | key;
    hv[i] = i;
  }
  unsigned long long *k0, *k1; unsigned *v0, *v1;
  cudaMalloc(&k0, E * 8); cudaMalloc(&k1, E * 8); cudaMalloc(&v0, E * 4); cudaMalloc(&v1, E * 4);
  cudaMemcpy(k0, hk.data(), E * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(v0, hv.data(), E * 4, cudaMemcpyHostToDevice);
  size_t tmp = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp, k0, k1, v0, v1, E, 0, bits);
  void* dt; cudaMalloc(&dt, tmp);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int w = 0; w < 3; ++w) cub::DeviceRadixSort::SortPairs(dt, tmp, k0, k1, v0, v1, E, 0, bits);
  cudaEventRecord(a);
  const int R = 20;
  for (int r = 0; r < R; ++r) cub::DeviceRadixSort::SortPairs(dt, tmp, k0, k1, v0, v1, E, 0, bits);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("cub SortPairs E=%d bits=%d: %.3f ms per sort (%.1f GB/s pass-equivalent)\n", E, bits, ms / R,
         (double)E * 12 * 2 * ((bits + 7) / 8) / (ms / R * 1e-3) / 1e9);
  // K4's exact shape: one 64-bit word per entry, (tile | depth) in 40 bits
  // above a 23-bit Gaussian id, sorted on bits [23, 63) -- keys only
  for (int i = 0; i < E; ++i) {
    const unsigned long long tile = hk[i] >> 32, dk = (hk[i] & 0xffffffffull) >> 5;
    hk[i] = (((tile << 27) | dk) << 23) | (unsigned long long)(i & 0x7fffff);
  }
  cudaMemcpy(k0, hk.data(), E * 8, cudaMemcpyHostToDevice);
  size_t tmp2 = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, tmp2, k0, k1, E, 23, 63);
  void* dt2; cudaMalloc(&dt2, tmp2);
  for (int w = 0; w < 3; ++w) cub::DeviceRadixSort::SortKeys(dt2, tmp2, k0, k1, E, 23, 63);
  cudaEventRecord(a);
  for (int r = 0; r < R; ++r) cub::DeviceRadixSort::SortKeys(dt2, tmp2, k0, k1, E, 23, 63);
  cudaEventRecord(b); cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  printf("cub SortKeys E=%d u64 bits [23,63) (K4 shape): %.3f ms per sort\n", E, ms / R);
  return 0;
}
