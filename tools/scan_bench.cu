// Dev micro-benchmark: the long-run consumer's distance chain on real cfg1 hot
// chains (tools/chains_sample.bin: 64 chains >= 4096 records, (d, w) bits as
// traced by the oracle), serial vs window scan (fold_chunk_scan). One warp per
// SMSP, chunks pre-weighed into shared memory like the ring; clock64 per chunk.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -std=c++17 -I paper_1611_03631_b200/csrc -I include tools/scan_bench.cu -o tools/scan_bench
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include "vxg_kernels.cuh"
using namespace vxg;

// ---- candidate (rejected): the distance chain of one chunk as a warp scan
// Measured on B200 (this tool, 64 hot cfg1 chains): serial 26.9 cycles/record,
// scan 29.8 — one scan round costs ~730 cycles (5 SHFL+PRMT rounds, 7-way
// tabulation, escape handling), more than the 32-step serial chain it replaces.
// With the colours stationary over a chunk, its 32 records only move the
// distance: D_{i+1} = f_i(D_i) = RN(RN(RN(W_i D_i) + wc_i) / T_i), a serial
// chain of five dependent FP ops per record. On the long (hot) runs D wanders
// within a few ulps (cfg1: a chunk of 32 records visits 3-6 consecutive floats),
// so every lane tabulates its record's f_i on the window of the 7 consecutive
// floats around the chunk's entry value, as a map of window indices (7 =
// "left the window", absorbing). The maps compose by byte permutation (PRMT);
// an inclusive warp scan of the compositions gives every record's exact
// entering value in log2(32) rounds instead of 32 dependent steps. Nothing is
// reassociated: each tabulated value is the record's own fast-exact step, so
// the result is the sequential chain's bit for bit. If the trajectory leaves
// the window at record j, record j is stepped from its (known) entering value
// and the scan restarts from j+1 around the new value.

// bytes b0..b3 (each <= 7) of a map -> PRMT selector b0 | b1<<4 | b2<<8 | b3<<12
__device__ __forceinline__ uint32_t nib_sel(uint32_t m) { return __byte_perm(m | (m >> 4), 0u, 0x4420u); }

// Folds records [0, cnt) of the chunk rb into D (all records live, colours
// stationary: the caller's vote). Returns the number of leading records folded
// (cnt unless D reached a value whose window would cross zero or leave the
// finite range; the caller steps the rest serially). qr collects every
// numerator evaluated (the caller's warp-wide range check).
__device__ __forceinline__ uint32_t fold_chunk_scan(float& D, const PreRec* rb, uint32_t cnt, int lane,
                                                    QuotRange& qr) {
  const float4 x = reinterpret_cast<const float4*>(rb)[lane * static_cast<int>(sizeof(PreRec) / sizeof(float4))];
  uint32_t from = 0;
  while (from < cnt) {
    const uint32_t b0 = __float_as_uint(D);
    const uint32_t mag = b0 & 0x7fffffffu;
    if (mag < 4u || mag >= 0x7f7ffff0u) return from;  // D = (near) zero or huge: serial steps
    const bool act = static_cast<uint32_t>(lane) >= from && static_cast<uint32_t>(lane) < cnt;
    uint32_t mlo = 0x03020100u, mhi = 0x07060504u;  // identity
    if (act) {
      mlo = 0u;
      mhi = 0x07000000u;
#pragma unroll
      for (int k = 0; k < 7; ++k) {
        const float a = __fadd_rn(__fmul_rn(x.x, __uint_as_float(b0 + static_cast<uint32_t>(k) - 3u)), x.w);
        qr_add(qr, a);
        const uint32_t idx = __float_as_uint(fast_quot0(a, Recip{x.y, x.z, true})) - b0 + 3u;
        const uint32_t s = idx < 7u ? idx : 7u;
        if (k < 4) mlo |= s << (8 * k); else mhi |= s << (8 * (k - 4));
      }
    }
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {  // inclusive scan: mine o (lanes before)
      const uint32_t plo = __shfl_up_sync(0xffffffffu, mlo, off);
      const uint32_t phi = __shfl_up_sync(0xffffffffu, mhi, off);
      if (lane >= off) {
        const uint32_t nlo = __byte_perm(mlo, mhi, nib_sel(plo));
        mhi = __byte_perm(mlo, mhi, nib_sel(phi));
        mlo = nlo;
      }
    }
    const uint32_t s_after = mlo >> 24;  // window index after this record, from entry index 3
    const uint32_t esc = __ballot_sync(0xffffffffu, s_after == 7u);
    if (esc == 0u) {
      D = __uint_as_float(b0 + __shfl_sync(0xffffffffu, s_after, 31) - 3u);
      return cnt;
    }
    const int j = __ffs(esc) - 1;  // first record whose result left the window
    const uint32_t s_prev = __shfl_sync(0xffffffffu, s_after, j > 0 ? j - 1 : 0);
    const float Din = __uint_as_float(b0 + (j > 0 ? s_prev : 3u) - 3u);
    const float a = __fadd_rn(__fmul_rn(x.x, Din), x.w);
    if (lane == j) qr_add(qr, a);
    D = __shfl_sync(0xffffffffu, fast_quot0(a, Recip{x.y, x.z, true}), j);
    from = static_cast<uint32_t>(j) + 1u;
  }
  return cnt;
}


__global__ void k_prep(const uint32_t* dw, const uint64_t* off, int nch, float trunc, float wmax, PreRec* out) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nch) return;
  float W = 0.0f;
  for (uint64_t i = off[c]; i < off[c + 1]; ++i) {
    const float d = __uint_as_float(dw[2 * i]), w = __uint_as_float(dw[2 * i + 1]);
    PreRec p{};
    p.W = W;
    p.T = __fadd_rn(W, w);
    p.r1 = make_recip(p.T).r1;
    const float cl = d < -trunc ? -trunc : (trunc < d ? trunc : d);
    p.wc = __fmul_rn(w, cl);
    p.w = w;
    p.d = d;
    out[i] = p;
    W = fminf(p.T, wmax);
  }
}

template <int kMode>  // 0 serial, 1 scan
__global__ void k_run(const PreRec* recs, const uint64_t* off, int nch, float* Dout, unsigned long long* cyc) {
  __shared__ PreRec ring[4][32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int c = blockIdx.x * 4 + wid;
  if (c >= nch) return;
  float D = 0.0f;
  long long tot = 0;
  for (uint64_t b = off[c]; b < off[c + 1]; b += 32) {
    const uint32_t cnt = static_cast<uint32_t>(off[c + 1] - b < 32 ? off[c + 1] - b : 32);
    if (lane < cnt) ring[wid][lane] = recs[b + lane];
    __syncwarp();
    const long long t0 = clock64();
    QuotRange qr;
    uint32_t u0 = 0;
    if (kMode == 1) u0 = fold_chunk_scan(D, ring[wid], cnt, lane, qr);
    for (uint32_t u = u0; u < cnt; ++u) {
      const PreRec& x = ring[wid][u];
      const float a = __fadd_rn(__fmul_rn(x.W, D), x.wc);
      qr_add(qr, a);
      D = fast_quot0(a, Recip{x.T, x.r1, true});
    }
    asm volatile("" ::"f"(D));
    tot += clock64() - t0;
    __syncwarp();
  }
  if (lane == 0) {
    Dout[c] = D;
    atomicAdd(cyc, static_cast<unsigned long long>(tot));
  }
}

int main() {
  FILE* f = fopen("tools/chains_sample.bin", "rb");
  uint32_t n;
  if (!f || fread(&n, 4, 1, f) != 1) return 1;
  std::vector<uint32_t> dw;
  std::vector<uint64_t> off{0};
  for (uint32_t c = 0; c < n; ++c) {
    uint32_t L;
    if (fread(&L, 4, 1, f) != 1) return 1;
    const size_t o = dw.size();
    dw.resize(o + 2 * L);
    if (fread(dw.data() + o, 4, 2 * L, f) != 2 * L) return 1;
    off.push_back(off.back() + L);
  }
  uint32_t *d_dw;
  uint64_t* d_off;
  PreRec* d_rec;
  float* d_D;
  unsigned long long* d_cyc;
  cudaMalloc(&d_dw, dw.size() * 4);
  cudaMalloc(&d_off, off.size() * 8);
  cudaMalloc(&d_rec, off.back() * sizeof(PreRec));
  cudaMalloc(&d_D, 2 * n * 4);
  cudaMalloc(&d_cyc, 16);
  cudaMemcpy(d_dw, dw.data(), dw.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(d_off, off.data(), off.size() * 8, cudaMemcpyHostToDevice);
  cudaMemset(d_cyc, 0, 16);
  k_prep<<<(n + 63) / 64, 64>>>(d_dw, d_off, n, 0.1f, 1e4f, d_rec);
  k_run<0><<<(n + 3) / 4, 128>>>(d_rec, d_off, n, d_D, d_cyc);
  k_run<1><<<(n + 3) / 4, 128>>>(d_rec, d_off, n, d_D + n, d_cyc + 1);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("cuda error %s\n", cudaGetErrorString(e)); return 1; }
  std::vector<float> D(2 * n);
  unsigned long long cyc[2];
  cudaMemcpy(D.data(), d_D, 2 * n * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(cyc, d_cyc, 16, cudaMemcpyDeviceToHost);
  int mism = 0;
  for (uint32_t c = 0; c < n; ++c) mism += memcmp(&D[c], &D[n + c], 4) != 0;
  printf("records %llu: serial %.2f cyc/record, scan %.2f cyc/record, mismatching chains %d\n",
         (unsigned long long)off.back(), (double)cyc[0] / off.back(), (double)cyc[1] / off.back(), mism);
  return 0;
}
