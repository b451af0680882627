// Dev micro-benchmark: cycles per step of the fold's distance chain variants,
// one warp alone on the GPU (clock64), data in shared memory like the ring.
#include <cstdio>
struct alignas(16) R { float W, T, r1, wc; };
__device__ __forceinline__ float fq(float a, float T, float r1) {
  const float q0 = __fmul_rn(a, r1);
  return __fmaf_rn(r1, __fmaf_rn(-T, q0, a), q0);
}
template <int V>
__global__ void k(const R* g, int n, float* out, long long* cyc) {
  __shared__ R ring[32];
  ring[threadIdx.x] = g[threadIdx.x];
  __syncwarp();
  float D = 0.05f;
  bool all = true;
  long long t0 = clock64();
  for (int it = 0; it < n; ++it) {
#pragma unroll 16
    for (int u = 0; u < 32; ++u) {
      const R x = ring[u];
      const float a = __fadd_rn(__fmul_rn(x.W, D), x.wc);
      if (V == 0) {  // current: predicate on a != 0 before the quotient
        all = all & (a == 0.0f || (fabsf(a) >= 0x1p-60f && fabsf(a) <= 0x1p60f));
        D = a == 0.0f ? a : fq(a, x.T, x.r1);
      } else if (V == 1) {  // quotient always, select after
        const float q = fq(a, x.T, x.r1);
        all = all & (a == 0.0f || (fabsf(a) >= 0x1p-60f && fabsf(a) <= 0x1p60f));
        D = (a == 0.0f) ? a : q;
      } else if (V == 2) {  // bare 5-op chain
        D = fq(a, x.T, x.r1);
      } else {  // IEEE division
        D = __fdiv_rn(a, x.T);
      }
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = D + (all ? 0.f : 1.f); cyc[0] = t1 - t0; }
}
int main() {
  R h[32];
  for (int i = 0; i < 32; ++i) { h[i].W = 1e4f; h[i].T = 1e4f + 2.5f + i * 0.01f; h[i].r1 = 1.0f / h[i].T; h[i].wc = 0.25f; }
  R* g; float* o; long long* c; cudaMalloc(&g, sizeof(h)); cudaMalloc(&o, 4); cudaMalloc(&c, 8);
  cudaMemcpy(g, h, sizeof(h), cudaMemcpyHostToDevice);
  const int n = 4096;
  const char* names[4] = {"predicated (current)", "select after quotient", "bare 5-op chain", "__fdiv_rn"};
  for (int v = 0; v < 4; ++v) {
    for (int rep = 0; rep < 2; ++rep) {
      if (v == 0) k<0><<<1, 32>>>(g, n, o, c);
      if (v == 1) k<1><<<1, 32>>>(g, n, o, c);
      if (v == 2) k<2><<<1, 32>>>(g, n, o, c);
      if (v == 3) k<3><<<1, 32>>>(g, n, o, c);
    }
    long long cyc; cudaMemcpy(&cyc, c, 8, cudaMemcpyDeviceToHost);
    printf("%-24s %.1f cycles/step\n", names[v], double(cyc) / (n * 32.0));
  }
  return 0;
}
