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
  return 0;
}
