// Stable LSD radix sort of the fold's (voxel key, ray id) records.
//
// The keys of one batch are dense: slot * vps^3 + local < blocks * vps^3, i.e.
// 21 bits for the 450-block cfg1 layer. One reduce-then-scan pass per digit of
// 7 bits (8 above 21 key bits): three passes at ~3.3 TB/s each on B200, where
// CUB's 8-bit onesweep runs three at ~1.9 TB/s. Wider digits (11 bits: two
// passes) fragment the scatter and cost more per bin than they save.
//   k_sort_upsweep   per super-tile digit histogram   (reads 4 B/record)
//   ExclusiveSum     digit-major [digit][super-tile]  -> global output bases
//   k_sort_downsweep per sub-tile: warp-private match_any ranking (stable),
//                    next sub-tile's keys/ids loaded during this one's scatter,
//                    smem staging in digit order, coalesced scatter
//                                                      (reads 8 B, writes 8 B)
// Records within a voxel keep their emission (= ray) order, which is what the
// ordered fold (tsdf_integrator.cpp:246, one update_tsdf_voxel per ray in
// order) needs. Invalid records (key 0xFFFFFFFF) have all-ones digits and land
// after every valid key as long as every valid key < 2^kbits - 1.
#pragma once
#include <cstdint>

namespace vxg {

constexpr int kSortThreads = 256;
constexpr int kSortWarps = kSortThreads / 32;

// kBits: largest digit of a pass; kIpt: records per thread per sub-tile.
template <int kBits, int kIpt, int kNs = 8>
struct SortCfg {
  static constexpr int kBins = 1 << kBits;
  static constexpr int kSub = kSortThreads * kIpt;                  // records per sub-tile
  static constexpr int kNsub = kNs;                                 // sub-tiles per super-tile (one CTA); 1 for small inputs (more CTAs)
  static constexpr uint32_t kSuper = static_cast<uint32_t>(kSub) * kNsub;
  static constexpr int kWcStride = kBins + 2;                       // + overflow bin for the tail, even
  static constexpr int kScanPer = (kBins + 1 + kSortThreads - 1) / kSortThreads;
  struct Smem {
    uint16_t wcnt[kSortWarps][kWcStride];  // per-warp digit counts, then cross-warp prefixes
    uint32_t tcount[kBins + 1];            // sub-tile digit counts
    uint32_t tstart[kBins + 1];            // sub-tile digit starts (exclusive scan of tcount)
    uint32_t gbase[kBins];                 // global output position of the digit's next record
    uint32_t gdelta[kBins];                // gbase - tstart: staged index -> output position
    uint32_t wsum[kSortWarps];
    uint2 stage[kSub];                     // (key, ray id) in digit order
  };
};

template <int kBits, int kIpt, int kNs = 8>
__global__ void __launch_bounds__(kSortThreads) k_sort_upsweep(const uint32_t* __restrict__ keys, uint64_t n,
                                                               int shift, uint32_t mask, uint32_t S,
                                                               uint32_t* __restrict__ counts) {
  using C = SortCfg<kBits, kIpt, kNs>;
  __shared__ uint32_t h[C::kBins];
  const uint32_t bins = mask + 1u;
  for (uint32_t d = threadIdx.x; d < bins; d += kSortThreads) h[d] = 0u;
  __syncthreads();
  const uint64_t lo = static_cast<uint64_t>(blockIdx.x) * C::kSuper;
  const uint32_t cnt = static_cast<uint32_t>(min(static_cast<uint64_t>(C::kSuper), n - lo));
  const uint4* k4 = reinterpret_cast<const uint4*>(keys + lo);  // lo % 4 == 0, buffers 256-B aligned
  const uint32_t n4 = cnt / 4u;
  for (uint32_t i = threadIdx.x; i < n4; i += kSortThreads) {  // shared-memory atomics (MATCH.ANY is slower)
    const uint4 k = k4[i];
    atomicAdd(&h[(k.x >> shift) & mask], 1u);
    atomicAdd(&h[(k.y >> shift) & mask], 1u);
    atomicAdd(&h[(k.z >> shift) & mask], 1u);
    atomicAdd(&h[(k.w >> shift) & mask], 1u);
  }
  for (uint32_t i = 4u * n4 + threadIdx.x; i < cnt; i += kSortThreads) atomicAdd(&h[(keys[lo + i] >> shift) & mask], 1u);
  __syncthreads();
  for (uint32_t d = threadIdx.x; d < bins; d += kSortThreads) counts[static_cast<uint64_t>(d) * S + blockIdx.x] = h[d];
}

// Lanes of the warp holding the same digit d (< 2^(kB+1)): one ballot per bit.
template <int kB>
__device__ __forceinline__ uint32_t digit_peers(uint32_t d) {
  uint32_t peers = 0xffffffffu;
#pragma unroll
  for (int b = 0; b <= kB; ++b) {
    const uint32_t v = __ballot_sync(0xffffffffu, (d >> b) & 1u);
    peers &= ((d >> b) & 1u) ? v : ~v;
  }
  return peers;
}

// kMarks (last pass only): instead of writing the sorted keys, mark each
// voxel's run [dense_start, dense_end) of the final order. The pass input is
// sorted by the other digits, so equal keys are contiguous inside a digit's
// staged segment; a segment's first/last record may continue a run from the
// previous / into the next sub-tile or CTA (atomicMin / atomicMax), a key
// change inside a segment is the run's global start / end (plain store).
template <int kBits, int kIpt, int kMinBlocks, bool kPrefetch = false, bool kMatch = false, bool kMarks = false,
          int kNs = 8>
__global__ void __launch_bounds__(kSortThreads, kMinBlocks)
    k_sort_downsweep(const uint32_t* __restrict__ kin, const uint32_t* __restrict__ vin, uint32_t* __restrict__ kout,
                     uint32_t* __restrict__ vout, uint64_t n, int shift, uint32_t mask, uint32_t S,
                     const uint32_t* __restrict__ offs, uint32_t K = 0, uint32_t* __restrict__ dense_start = nullptr,
                     uint32_t* __restrict__ dense_end = nullptr) {
  using C = SortCfg<kBits, kIpt, kNs>;
  extern __shared__ __align__(16) uint8_t sort_smem_raw[];
  typename C::Smem& sm = *reinterpret_cast<typename C::Smem*>(sort_smem_raw);
  const uint32_t bins = mask + 1u;
  const int tid = threadIdx.x, w = tid >> 5;
  const uint32_t lane = tid & 31u, lt = (1u << lane) - 1u;
  for (uint32_t d = tid; d < bins; d += kSortThreads) sm.gbase[d] = offs[static_cast<uint64_t>(d) * S + blockIdx.x];
  const uint64_t super0 = static_cast<uint64_t>(blockIdx.x) * C::kSuper;
  uint32_t* wc32 = reinterpret_cast<uint32_t*>(&sm.wcnt[0][0]);
  // warp w owns sub-tile items [w*IPT*32, (w+1)*IPT*32), item (j, lane) = j*32 + lane
  const uint32_t i0 = static_cast<uint32_t>(w) * (kIpt * 32) + lane;
  uint32_t key[kIpt], val[kIpt];
  auto load_sub = [&](uint64_t b, uint32_t nvv) {
#pragma unroll
    for (int j = 0; j < kIpt; ++j) {
      const uint32_t i = i0 + j * 32;
      key[j] = i < nvv ? kin[b + i] : 0u;
      if (kPrefetch) val[j] = i < nvv ? vin[b + i] : 0u;
    }
  };
  if (kPrefetch && super0 < n) load_sub(super0, static_cast<uint32_t>(min(static_cast<uint64_t>(C::kSub), n - super0)));
  for (int t = 0; t < C::kNsub; ++t) {
    const uint64_t base = super0 + static_cast<uint64_t>(t) * C::kSub;
    if (base >= n) break;  // CTA-uniform
    const uint32_t nv = static_cast<uint32_t>(min(static_cast<uint64_t>(C::kSub), n - base));
    for (int i = tid; i < kSortWarps * C::kWcStride / 2; i += kSortThreads) wc32[i] = 0u;
    if (!kPrefetch) load_sub(base, nv);
    __syncthreads();  // wcnt zeroed; previous sub-tile's gbase update visible
    // stable warp-private ranking: (j, lane) order == item order
    uint32_t rk[kIpt];
#pragma unroll
    for (int j = 0; j < kIpt; ++j) {
      const uint32_t d = i0 + j * 32 < nv ? (key[j] >> shift) & mask : bins;
      const uint32_t peers = kMatch ? __match_any_sync(0xffffffffu, d) : digit_peers<kBits>(d);
      const uint32_t pre = sm.wcnt[w][d];
      __syncwarp();
      if ((peers & lt) == 0u) sm.wcnt[w][d] = static_cast<uint16_t>(pre + __popc(peers));
      __syncwarp();
      rk[j] = pre + __popc(peers & lt);
    }
    __syncthreads();
    // cross-warp exclusive prefixes (in place) and sub-tile digit counts
    for (uint32_t d = tid; d <= bins; d += kSortThreads) {
      uint32_t run = 0;
#pragma unroll
      for (int q = 0; q < kSortWarps; ++q) {
        const uint32_t c = sm.wcnt[q][d];
        sm.wcnt[q][d] = static_cast<uint16_t>(run);
        run += c;
      }
      sm.tcount[d] = run;
    }
    __syncthreads();
    {  // exclusive scan tcount[0..bins] -> tstart
      const uint32_t nb = bins + 1u;
      uint32_t loc[C::kScanPer], sum = 0;
#pragma unroll
      for (int q = 0; q < C::kScanPer; ++q) {
        const uint32_t idx = static_cast<uint32_t>(tid) * C::kScanPer + q;
        loc[q] = idx < nb ? sm.tcount[idx] : 0u;
        sum += loc[q];
      }
      uint32_t x = sum;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, off);
        if (lane >= static_cast<uint32_t>(off)) x += y;
      }
      if (lane == 31u) sm.wsum[w] = x;
      __syncthreads();
      uint32_t run = x - sum;
      for (int q = 0; q < w; ++q) run += sm.wsum[q];
#pragma unroll
      for (int q = 0; q < C::kScanPer; ++q) {
        const uint32_t idx = static_cast<uint32_t>(tid) * C::kScanPer + q;
        if (idx < nb) sm.tstart[idx] = run;
        run += loc[q];
      }
    }
    __syncthreads();
    // fold the sub-tile digit starts into the per-warp prefixes (one lookup per
    // record below) and the global bases into per-digit deltas
    for (uint32_t e = tid; e < kSortWarps * (bins + 1u); e += kSortThreads) {
      const uint32_t q = e / (bins + 1u), d = e - q * (bins + 1u);
      sm.wcnt[q][d] = static_cast<uint16_t>(sm.wcnt[q][d] + sm.tstart[d]);
    }
    for (uint32_t d = tid; d < bins; d += kSortThreads) sm.gdelta[d] = sm.gbase[d] - sm.tstart[d];
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kIpt; ++j) {
      const uint32_t i = i0 + j * 32;
      if (i < nv) {
        const uint32_t d = (key[j] >> shift) & mask;
        sm.stage[sm.wcnt[w][d] + rk[j]] = make_uint2(key[j], kPrefetch ? val[j] : vin[base + i]);
      }
    }
    if (kPrefetch) {  // next sub-tile's loads overlap this one's scatter
      const uint64_t nb = base + C::kSub;
      if (t + 1 < C::kNsub && nb < n) load_sub(nb, static_cast<uint32_t>(min(static_cast<uint64_t>(C::kSub), n - nb)));
    }
    __syncthreads();
    if (!kMarks) {
      for (uint32_t i = tid; i < nv; i += kSortThreads) {
        const uint2 kv = sm.stage[i];
        const uint32_t d = (kv.x >> shift) & mask;
        const uint32_t p = sm.gdelta[d] + i;
        kout[p] = kv.x;
        vout[p] = kv.y;
      }
    } else {
      // consecutive staged records sit in consecutive lanes: the neighbours'
      // keys come by shuffle; a digit change between neighbours is the digit
      // segment's edge (the staged records are in digit order)
      for (uint32_t b = static_cast<uint32_t>(tid) & ~31u; b < nv; b += kSortThreads) {  // warp-uniform
        const uint32_t i = b + lane;
        const bool in = i < nv;
        const uint2 kv = in ? sm.stage[i] : make_uint2(0xFFFFFFFFu, 0u);
        uint32_t prev = __shfl_up_sync(0xffffffffu, kv.x, 1);
        uint32_t next = __shfl_down_sync(0xffffffffu, kv.x, 1);
        if (lane == 0u) prev = (in && i > 0) ? sm.stage[i - 1].x : 0xFFFFFFFFu;
        if (lane == 31u || i + 1 >= nv) next = (i + 1 < nv) ? sm.stage[i + 1].x : 0xFFFFFFFFu;
        if (in) {
          const uint32_t d = (kv.x >> shift) & mask;
          const uint32_t p = sm.gdelta[d] + i;
          vout[p] = kv.y;
          if (kv.x < K) {
            const bool seg_first = i == 0 || ((prev >> shift) & mask) != d;
            const bool seg_last = i + 1 == nv || ((next >> shift) & mask) != d;
            if (seg_first)
              atomicMin(&dense_start[kv.x], p);
            else if (prev != kv.x)
              dense_start[kv.x] = p;
            if (seg_last)
              atomicMax(&dense_end[kv.x], p + 1);
            else if (next != kv.x)
              dense_end[kv.x] = p + 1;
          }
        }
      }
    }
    __syncthreads();
    for (uint32_t d = tid; d < bins; d += kSortThreads) sm.gbase[d] += sm.tcount[d];
  }
}

// Runs of the sorted records, one per voxel with records (dense_end[k] != 0),
// compacted in key order through the scan below.
struct RunIn {
  const uint32_t* dense_end;
  __device__ __forceinline__ uint32_t operator()(uint64_t k) const { return dense_end[k] != 0u ? 1u : 0u; }
};
struct RunOut {
  uint64_t K;
  const uint32_t* dense_start;
  const uint32_t* dense_end;
  uint32_t* run_keys;
  uint32_t* run_start;
  uint32_t* run_len;
  uint32_t* nruns;
  __device__ __forceinline__ void operator()(uint64_t k, uint32_t has, uint32_t j) const {
    if (has) {
      run_keys[j] = static_cast<uint32_t>(k);
      run_start[j] = dense_start[k];
      run_len[j] = dense_end[k] - dense_start[k];
    }
    if (k == K - 1) *nruns = j + has;
  }
};

// ---- exclusive prefix sums: reduce-then-scan over tiles of kScanTile items
// (k_scan_reduce -> the tile sums scanned by the same routine -> k_scan_apply).
// in == out is allowed (every item is read before it is written, by the same
// thread).
constexpr int kScanThreads = 256;
constexpr int kScanIpt = 16;
constexpr uint32_t kScanTile = kScanThreads * kScanIpt;

// In: value of item i (uint64_t -> T). Out: (i, value, exclusive prefix) -> side effects.
template <typename T>
struct ScanLoad {
  const T* p;
  __device__ __forceinline__ T operator()(uint64_t i) const { return p[i]; }
};
template <typename T>
struct ScanStore {
  T* p;
  __device__ __forceinline__ void operator()(uint64_t i, T, T pre) const { p[i] = pre; }
};

__device__ __forceinline__ void scan_pin(uint32_t& x) { asm volatile("" : "+r"(x)); }
__device__ __forceinline__ void scan_pin(unsigned long long& x) { asm volatile("" : "+l"(x)); }

template <typename T, typename In>
__global__ void __launch_bounds__(kScanThreads) k_scan_reduce(In in, uint64_t n, T* __restrict__ tile_sums) {
  __shared__ T s_warp[kScanThreads / 32];
  const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kScanTile;
  T x = 0;
#pragma unroll
  for (int j = 0; j < kScanIpt; ++j) {
    const uint64_t i = base + static_cast<uint64_t>(j) * kScanThreads + threadIdx.x;
    if (i < n) x += in(i);
  }
  const uint32_t lane = threadIdx.x & 31u, w = threadIdx.x >> 5;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) x += __shfl_xor_sync(0xffffffffu, x, off);
  if (lane == 0u) s_warp[w] = x;
  __syncthreads();
  if (threadIdx.x == 0) {
    T tot = 0;
#pragma unroll
    for (int q = 0; q < kScanThreads / 32; ++q) tot += s_warp[q];
    tile_sums[blockIdx.x] = tot;
  }
}

// out(i, in(i), tile_offs[tile] + sum of the tile's items before i). A warp
// owns kScanIpt * 32 consecutive items, item (j, lane) = j * 32 + lane of its
// span: coalesced accesses, one shuffle scan per j, one barrier per tile.
// tile_offs == nullptr: one CTA walks `tiles` consecutive tiles alone with a
// running carry (small inputs: one launch instead of three).
template <typename T, typename In, typename Out>
__global__ void __launch_bounds__(kScanThreads) k_scan_apply(In in, uint64_t n, const T* __restrict__ tile_offs,
                                                             Out out, int tiles = 1) {
  __shared__ T s_warp[2][kScanThreads / 32];
  const uint32_t lane = threadIdx.x & 31u, w = threadIdx.x >> 5;
  T carry = tile_offs != nullptr ? tile_offs[blockIdx.x] : T(0);
  for (int t = 0; t < tiles; ++t) {
    const uint64_t i0 = (static_cast<uint64_t>(blockIdx.x) + t) * kScanTile + static_cast<uint64_t>(w) * (32 * kScanIpt) + lane;
    T v[kScanIpt], e[kScanIpt], run = 0;  // e: exclusive prefix inside the warp's span
#pragma unroll
    for (int j = 0; j < kScanIpt; ++j) v[j] = i0 + j * 32 < n ? in(i0 + j * 32) : T(0);
    // all loads in flight before the first scan (otherwise the compiler
    // re-reads in(i) per use and exposes one memory round trip per j)
#pragma unroll
    for (int j = 0; j < kScanIpt; ++j) scan_pin(v[j]);
#pragma unroll
    for (int j = 0; j < kScanIpt; ++j) {
      T x = v[j];
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const T y = __shfl_up_sync(0xffffffffu, x, off);
        if (lane >= static_cast<uint32_t>(off)) x += y;
      }
      e[j] = run + x - v[j];
      run += __shfl_sync(0xffffffffu, x, 31);
    }
    T* sw = s_warp[t & 1];  // double-buffered: one barrier per tile
    if (lane == 0u) sw[w] = run;
    __syncthreads();
    T pre = carry, tot = 0;
#pragma unroll
    for (int q = 0; q < kScanThreads / 32; ++q) {
      const T c = sw[q];
      if (q < static_cast<int>(w)) pre += c;
      tot += c;
    }
#pragma unroll
    for (int j = 0; j < kScanIpt; ++j)
      if (i0 + j * 32 < n) out(i0 + j * 32, v[j], pre + e[j]);
    carry += tot;
  }
}

// ---- bundling: one bucket per run of equal sorted keys (a compaction of the
// run heads through the scan above: the keys are read twice, nothing else)
template <typename KeyT>
struct SegHeadIn {
  const KeyT* k;
  __device__ __forceinline__ uint32_t operator()(uint64_t i) const { return (i == 0 || k[i] != k[i - 1]) ? 1u : 0u; }
};
template <typename KeyT>
struct SegHeadOut {
  const KeyT* k;
  uint64_t n;
  unsigned long long* ukeys;
  uint32_t* ustart;
  uint32_t* num_segs;
  __device__ __forceinline__ void operator()(uint64_t i, uint32_t head, uint32_t pre) const {
    if (head) {
      ukeys[pre] = static_cast<unsigned long long>(k[i]);
      ustart[pre] = static_cast<uint32_t>(i);
    }
    if (i == n - 1) *num_segs = pre + head;
  }
};

__global__ void k_seg_counts(uint32_t S, uint64_t P, const uint32_t* __restrict__ ustart, uint32_t* __restrict__ ucount) {
  for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < S; s += gridDim.x * blockDim.x)
    ucount[s] = (s + 1 < S ? ustart[s + 1] : static_cast<uint32_t>(P)) - ustart[s];
}

// ---- 64-bit keys through the 32-bit pair sort: positions sorted by the low
// word, then (stable) by the high word
__global__ void k_key_word(uint64_t n, const unsigned long long* __restrict__ keys, const uint32_t* __restrict__ perm,
                           int shift, uint32_t mask, bool complement, uint32_t* __restrict__ out_k,
                           uint32_t* __restrict__ out_v) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t src = perm != nullptr ? perm[i] : static_cast<uint32_t>(i);
    const uint32_t wv = static_cast<uint32_t>(keys[src] >> shift) & mask;
    out_k[i] = complement ? mask - wv : wv;
    if (out_v != nullptr) out_v[i] = src;
  }
}

__global__ void k_gather_sorted(uint64_t n, const uint32_t* __restrict__ perm, const unsigned long long* __restrict__ keys,
                                const uint32_t* __restrict__ vals, unsigned long long* __restrict__ out_keys,
                                uint32_t* __restrict__ out_vals) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t src = perm[i];
    if (out_keys != nullptr) out_keys[i] = keys[src];
    if (out_vals != nullptr) out_vals[i] = vals[src];
  }
}

// ---- fold order: runs by a coarse length code, longest first, key order inside a code
// Codes are monotone in the length: exact below 16, then 8 steps per octave
// (lengths within 12.5 % share a code), so a warp's 32 short runs are
// balanced while runs of one code keep their key order (neighbouring voxels
// share rays: the fold's gathers stay local). kLongRun must be a code boundary.
__device__ __host__ __forceinline__ uint32_t run_len_code(uint32_t len) {
  if (len < 16u) return len;
#ifdef __CUDA_ARCH__
  const int e = 31 - __clz(len);
#else
  int e = 31;
  while (!(len >> e)) --e;
#endif
  return 16u + static_cast<uint32_t>(e - 4) * 8u + ((len >> (e - 3)) & 7u);
}
constexpr uint32_t kRunCodeMax = 255u;

__global__ void k_run_codes(uint32_t nruns, const uint32_t* __restrict__ run_len, uint32_t* __restrict__ dcode,
                            uint32_t* __restrict__ iota, uint32_t* __restrict__ max_len) {
  uint32_t m = 0;
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < nruns; r += gridDim.x * blockDim.x) {
    const uint32_t len = run_len[r];
    dcode[r] = kRunCodeMax - run_len_code(len);
    iota[r] = r;
    m = max(m, len);
  }
  m = __reduce_max_sync(0xffffffffu, m);
  if ((threadIdx.x & 31u) == 0u && m) atomicMax(max_len, m);
}

}  // namespace vxg
