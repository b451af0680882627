// Dev micro-benchmark: CUB onesweep SortPairs<u32,u32> throughput on B200 for
// uniform keys vs. skewed (voxel-like) keys of the same size and bit width.
#include <cub/device/device_radix_sort.cuh>
#include <cstdio>
#include <vector>
#include <random>
__global__ void gen_uniform(unsigned* k, unsigned* v, size_t n, int bits, unsigned long long seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    unsigned long long z = seed + i * 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL; z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL; z ^= z >> 31;
    k[i] = (unsigned)z & ((1u << bits) - 1); v[i] = (unsigned)i;
  }
}
__global__ void gen_skew(unsigned* k, unsigned* v, size_t n, int bits, unsigned long long seed) {
  // runs of 1..128 equal keys, keys drawn from a small hot set 10% of the time
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    size_t ray = i / 100;
    unsigned long long z = seed + ray * 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL; z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL; z ^= z >> 31;
    unsigned base = (unsigned)z & ((1u << bits) - 1);
    k[i] = (base + (unsigned)(i % 100) * 17) & ((1u << bits) - 1); v[i] = (unsigned)ray;
  }
}
int main() {
  const size_t n = 243000000; const int bits = 23;
  unsigned *k0, *k1, *v0, *v1; cudaMalloc(&k0, n*4); cudaMalloc(&k1, n*4); cudaMalloc(&v0, n*4); cudaMalloc(&v1, n*4);
  size_t tb = 0; cub::DeviceRadixSort::SortPairs(nullptr, tb, k0, k1, v0, v1, (int)n, 0, bits);
  void* tmp; cudaMalloc(&tmp, tb);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int mode = 0; mode < 2; ++mode) for (int eb : {16, 21, 23, 24, 32}) {
    if (mode == 0) gen_uniform<<<4096, 256>>>(k0, v0, n, eb, 1); else gen_skew<<<4096, 256>>>(k0, v0, n, eb, 1);
    cub::DeviceRadixSort::SortPairs(tmp, tb, k0, k1, v0, v1, (int)n, 0, eb);
    cudaEventRecord(a);
    for (int r = 0; r < 3; ++r) cub::DeviceRadixSort::SortPairs(tmp, tb, k0, k1, v0, v1, (int)n, 0, eb);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); ms /= 3;
    int passes = (eb + 7) / 8;
    printf("%s bits=%d: %.3f ms  (%.2f ms/pass, %.0f GB/s per pass at 16 B/item)\n", mode ? "skew" : "uniform", eb, ms, ms / passes, n * 16.0 / (ms / passes) / 1e6);
  }
  return 0;
}
