// Kernels of the B200 TSDF integration pipeline.
//
// Data layout in HBM:
//   slab       : cap_blocks x vps^3 vxg_voxel (12 B AoS, x-fastest = the VXBLX
//                voxel payload, serialization.cpp:107-114), zero = default voxel
//   block hash : open addressing, linear probing, 2^k x (u64 packed key, i32 slot)
//   records    : per candidate voxel update, u32 key (slot*vps^3 + local, or
//                0xFFFFFFFF for a skipped candidate) + u32 ray id (8 B); the fold
//                re-derives (d, w, colour) from the ray (FoldRay, one 32-B sector)
#pragma once

#include <cstdint>

#include "vxg_device.cuh"
#include "vxg_sort.cuh"

namespace vxg {

struct alignas(16) SegInfo {  // one bucket of integrate_grouped's Loop A (tsdf_integrator.h:90-95)
  float mean[3];
  float base_weight;  // float(sum w) / measurement_weight(mean)  (tsdf_integrator.cpp:236-241)
  int32_t g[3];       // terminal voxel
  uint32_t color;     // r | g<<8 | b<<16 | has_color<<31
  uint64_t hash;      // IndexHash(terminal)
  uint32_t frame;
  uint32_t pos;       // first point index within the frame (first appearance)
  uint32_t cast;      // bucket.weight > 0 (tsdf_integrator.cpp:224)
  uint32_t pad[3];
};

struct alignas(16) RayInfo {  // one cast_and_update call (tsdf_integrator.cpp:129-173), in ray order
  float p[3];        // surface point (world)
  float weight;      // merged base weight (1.0f in simple mode)
  uint32_t color;    // r | g<<8 | b<<16 | has_color<<31
  uint32_t frame;
  float depth;       // ||p - origin|| (cast_and_update :136), set by k_ray_count
  float base;        // measurement_weight base 1/depth^2 (1 in constant mode), set by k_ray_count
  int32_t term[3];   // own terminal voxel (anti-graze)
  uint32_t valid;
};

// The fields the fold's weighing needs, one 32-byte sector per ray.
struct alignas(32) FoldRay {
  float p[3];
  float weight;
  uint32_t color;
  uint32_t frame;
  float base;
  float pad;
};

// Record values: the ray index, with kFarRecord set when the emit proved the
// voxel centre more than truncation + v in front of the point along the ray
// (d >= truncation in the reference's rounded arithmetic): clamp(d) is then
// exactly +truncation and w the ray's w_front = mweight_base(d > -eps) *
// weight, so the fold reads only the ray's 8-byte FarRay {w_front, colour}
// (4 per sector, a quarter of the FoldRay table) instead of its FoldRay.
constexpr uint32_t kFarRecord = 0x80000000u;
constexpr uint32_t kRayMask = 0x7fffffffu;

struct alignas(16) Record {
  float d;
  float w;
  uint32_t color;
  uint32_t pad;
};

struct TsdfParams {
  float voxel_size;
  float truncation;
  float dropoff_epsilon;
  float max_weight;
  float min_ray;
  float max_ray;
  int weight_mode;
  int merge_mode;
  uint32_t long_code;  // fold: runs whose length code (run_len_code) is >= this go to the warp pairs
};

__device__ __forceinline__ uint32_t frame_of(const uint64_t* off, uint32_t F, uint64_t i) {
  uint32_t lo = 0, hi = F;
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (off[mid] <= i) lo = mid; else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ uint32_t pack_color(const uint8_t* c) {
  return static_cast<uint32_t>(c[0]) | (static_cast<uint32_t>(c[1]) << 8) | (static_cast<uint32_t>(c[2]) << 16) |
         0x80000000u;
}

// ---------------------------------------------------------------- simple mode
// integrate_simple (tsdf_integrator.cpp:175-190) range filter: flag[i] = in range.
__global__ void k_simple_inrange(const float* __restrict__ xyz, uint64_t P, const uint64_t* __restrict__ off,
                                 const float* __restrict__ poses, uint32_t F, TsdfParams tp,
                                 uint32_t* __restrict__ flag, unsigned long long* __restrict__ skipped) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < P;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t f = frame_of(off, F, i);
    const float* Pm = poses + 12 * f;
    float p[3];
    transform_point(Pm, xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2], p);
    const float depth = norm3(fsub(p[0], Pm[3]), fsub(p[1], Pm[7]), fsub(p[2], Pm[11]));
    const bool in = !(depth < tp.min_ray || depth > tp.max_ray);
    flag[i] = in ? 1u : 0u;
    if (!in) atomicAdd(&skipped[f], 1ull);
  }
}

__global__ void k_simple_rays(const float* __restrict__ xyz, const uint8_t* __restrict__ rgb, uint64_t P,
                              const uint64_t* __restrict__ off, const float* __restrict__ poses, uint32_t F,
                              const uint32_t* __restrict__ flag, const uint32_t* __restrict__ ray_idx,
                              RayInfo* __restrict__ rays) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < P;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    if (!flag[i]) continue;
    const uint32_t f = frame_of(off, F, i);
    const float* Pm = poses + 12 * f;
    RayInfo r;
    transform_point(Pm, xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2], r.p);
    r.weight = 1.0f;
    r.color = rgb != nullptr ? pack_color(rgb + 3 * i) : 0u;
    r.frame = f;
    r.valid = 1u;
    r.depth = 0.0f;
    r.term[0] = r.term[1] = r.term[2] = 0;
    r.base = 0.0f;
    rays[ray_idx[i]] = r;
  }
}

// ---------------------------------------------------------------- grouped mode
// Loop A key: (frame, terminal voxel relative to the origin voxel); out-of-range
// points get the frame's sentinel (all-ones voxel field) and are counted later.
template <typename KeyT>
__global__ void k_group_keys(const float* __restrict__ xyz, uint64_t P, const uint64_t* __restrict__ off,
                             const float* __restrict__ poses, uint32_t F, TsdfParams tp, int rb, int kb,
                             KeyT* __restrict__ keys, uint32_t* __restrict__ vals,
                             uint32_t* __restrict__ counters) {
  const uint64_t field_mask = (1ull << (3 * kb)) - 1ull;
  const int lim = (1 << kb) - 1;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < P;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t f = frame_of(off, F, i);
    const float* Pm = poses + 12 * f;
    float p[3];
    transform_point(Pm, xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2], p);
    const float depth = norm3(fsub(p[0], Pm[3]), fsub(p[1], Pm[7]), fsub(p[2], Pm[11]));
    uint64_t key = (static_cast<uint64_t>(f) << (3 * kb)) | field_mask;
    if (!(depth < tp.min_ray || depth > tp.max_ray)) {
      int e[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) e[k] = gidx(p[k], tp.voxel_size) - gidx(Pm[4 * k + 3], tp.voxel_size) + rb;
      if (e[0] < 0 || e[0] >= lim || e[1] < 0 || e[1] >= lim || e[2] < 0 || e[2] >= lim) {
        atomicOr(&counters[1], static_cast<uint32_t>(kErrKeyRange));
      } else {
        key = (static_cast<uint64_t>(f) << (3 * kb)) | (static_cast<uint64_t>(e[0]) << (2 * kb)) |
              (static_cast<uint64_t>(e[1]) << kb) | static_cast<uint64_t>(e[2]);
      }
    }
    keys[i] = static_cast<KeyT>(key);
    vals[i] = static_cast<uint32_t>(i);
  }
}

// Per bucket: sequential fp64 sums in scan order (tsdf_integrator.cpp:213-219),
// then the merged ray (:224-241). Points are fetched kSegChunk at a time
// (independent loads and weights ahead of the dependent fp64 sums).
constexpr int kSegChunk = 8;

// Per-point terms of the bucket sums, computed in sorted order by a fully
// parallel pass (one gather per point) so the per-bucket sequential fp64 sums
// stream contiguous memory: world point p = T_f * x and its weight 1/|p - o|^2.
template <typename KeyT>
__global__ void k_point_prep(uint64_t P, const KeyT* __restrict__ skeys, const uint32_t* __restrict__ svals,
                             const float* __restrict__ xyz, const uint8_t* __restrict__ rgb,
                             const float* __restrict__ poses, TsdfParams tp, int kb, float4* __restrict__ pw,
                             uint32_t* __restrict__ cc) {
  const uint64_t field_mask = (1ull << (3 * kb)) - 1ull;
  for (uint64_t j = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; j < P;
       j += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t key = static_cast<uint64_t>(skeys[j]);
    if ((key & field_mask) == field_mask) continue;  // out-of-range point: its bucket is skipped
    const uint32_t f = static_cast<uint32_t>(key >> (3 * kb));
    const uint32_t i = svals[j];
    const float* Pm = poses + 12 * f;
    float pp[3];
    transform_point(Pm, xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2], pp);
    const float depth = norm3(fsub(pp[0], Pm[3]), fsub(pp[1], Pm[7]), fsub(pp[2], Pm[11]));
    const float ww = tp.weight_mode == VXG_WEIGHT_CONSTANT ? 1.0f : fdiv(1.0f, fmul(depth, depth));
    pw[j] = make_float4(pp[0], pp[1], pp[2], ww);
    if (rgb != nullptr)
      cc[j] = static_cast<uint32_t>(rgb[3 * i]) | (static_cast<uint32_t>(rgb[3 * i + 1]) << 8) |
              (static_cast<uint32_t>(rgb[3 * i + 2]) << 16);
  }
}

__global__ void k_seg_reduce(const uint32_t* __restrict__ num_segs_p, const unsigned long long* __restrict__ ukeys,
                             const uint32_t* __restrict__ uoffs, const uint32_t* __restrict__ ucounts,
                             const uint32_t* __restrict__ svals, const float4* __restrict__ pw,
                             const uint32_t* __restrict__ cc, const uint8_t* __restrict__ rgb,
                             const uint64_t* __restrict__ off,
                             const float* __restrict__ poses, TsdfParams tp, int rb, int kb,
                             SegInfo* __restrict__ segs, uint32_t* __restrict__ seg_count,
                             uint32_t* __restrict__ seg_start, unsigned long long* __restrict__ skipped) {
  const uint32_t S = *num_segs_p;
  const uint64_t field_mask = (1ull << (3 * kb)) - 1ull;
  const uint64_t kmask = (1ull << kb) - 1ull;
  for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < S; s += gridDim.x * blockDim.x) {
    const uint64_t key = ukeys[s];
    const uint32_t f = static_cast<uint32_t>(key >> (3 * kb));
    const uint32_t start = uoffs[s], cnt = ucounts[s];
    const bool sentinel = (key & field_mask) == field_mask;  // out-of-range points (:204-207)
    {
      const unsigned active = __activemask();
      const unsigned peers = __match_any_sync(active, f);
      const uint32_t nb = __reduce_add_sync(peers, sentinel ? 0u : 1u);
      const uint32_t mn = __reduce_min_sync(peers, sentinel ? 0xFFFFFFFFu : s);
      if ((threadIdx.x & 31) == static_cast<unsigned>(__ffs(peers) - 1) && nb) {
        atomicAdd(&seg_count[f], nb);
        atomicMin(&seg_start[f], mn);
      }
    }
    SegInfo out;
    out.frame = f;
    if (sentinel) {
      atomicAdd(&skipped[f], static_cast<unsigned long long>(cnt));
      out.cast = 0xFFFFFFFFu;  // marks "not a bucket"
      segs[s] = out;
      continue;
    }
    const float* Pm = poses + 12 * f;
    const float o[3] = {Pm[3], Pm[7], Pm[11]};
    double wp[3] = {0.0, 0.0, 0.0}, wc[3] = {0.0, 0.0, 0.0}, W = 0.0;
    const uint32_t first = svals[start];
    // point order within the bucket (stable sort); the terms of kSegChunk
    // points are loaded before their (sequential) sums, so the loads overlap
    auto add_point = [&](const float4& q, uint32_t c) {
      const double wd = static_cast<double>(q.w);
      wp[0] = __dadd_rn(wp[0], __dmul_rn(wd, static_cast<double>(q.x)));
      wp[1] = __dadd_rn(wp[1], __dmul_rn(wd, static_cast<double>(q.y)));
      wp[2] = __dadd_rn(wp[2], __dmul_rn(wd, static_cast<double>(q.z)));
      if (rgb != nullptr) {
#pragma unroll
        for (int k = 0; k < 3; ++k) wc[k] = __dadd_rn(wc[k], __dmul_rn(wd, static_cast<double>((c >> (8 * k)) & 0xffu)));
      }
      W = __dadd_rn(W, wd);
    };
    uint32_t j = 0;
    for (; j + kSegChunk <= cnt; j += kSegChunk) {
      float4 q[kSegChunk];
      uint32_t c[kSegChunk];
#pragma unroll
      for (int u = 0; u < kSegChunk; ++u) {
        q[u] = pw[start + j + u];
        c[u] = rgb != nullptr ? cc[start + j + u] : 0u;
      }
#pragma unroll
      for (int u = 0; u < kSegChunk; ++u) add_point(q[u], c[u]);
    }
    for (; j < cnt; ++j) add_point(pw[start + j], rgb != nullptr ? cc[start + j] : 0u);
#pragma unroll
    for (int k = 0; k < 3; ++k) out.mean[k] = __double2float_rn(__ddiv_rn(wp[k], W));
    uint32_t col = 0u;
    if (rgb != nullptr) {
      col = 0x80000000u;
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        long l = lround(__ddiv_rn(wc[k], W));
        l = l < 0l ? 0l : (255l < l ? 255l : l);
        col |= static_cast<uint32_t>(l) << (8 * k);
      }
    }
    out.color = col;
    const float z = norm3(fsub(out.mean[0], o[0]), fsub(out.mean[1], o[1]), fsub(out.mean[2], o[2]));
    const float mw = tp.weight_mode == VXG_WEIGHT_CONSTANT ? 1.0f : fdiv(1.0f, fmul(z, z));
    out.base_weight = fdiv(__double2float_rn(W), mw);
    const int og[3] = {gidx(o[0], tp.voxel_size), gidx(o[1], tp.voxel_size), gidx(o[2], tp.voxel_size)};
    out.g[0] = static_cast<int32_t>((key >> (2 * kb)) & kmask) - rb + og[0];
    out.g[1] = static_cast<int32_t>((key >> kb) & kmask) - rb + og[1];
    out.g[2] = static_cast<int32_t>(key & kmask) - rb + og[2];
    out.hash = teschner_hash(out.g[0], out.g[1], out.g[2]);
    out.pos = static_cast<uint32_t>(first - off[f]);
    out.cast = W > 0.0 ? 1u : 0u;
    segs[s] = out;
  }
}

// Ray order: libstdc++ iteration order = groups by first
// occupation time of their bucket (descending), then insertion position
// (descending). fo[bucket] = min position over the bucket's keys.
__global__ void k_order_fo(uint32_t S, const SegInfo* __restrict__ segs, const uint32_t* __restrict__ pos,
                           const uint32_t* __restrict__ part, const uint64_t* __restrict__ tbl_off,
                           const uint64_t* __restrict__ bc, uint32_t* __restrict__ fo) {
  for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < S; s += gridDim.x * blockDim.x) {
    const SegInfo& g = segs[s];
    if (g.cast == 0xFFFFFFFFu) continue;
    if (part != nullptr && !part[s]) continue;
    const uint32_t ps = pos != nullptr ? pos[s] : g.pos;
    atomicMin(&fo[tbl_off[g.frame] + g.hash % bc[g.frame]], ps);
  }
}

__global__ void k_order_keys(uint32_t S, const SegInfo* __restrict__ segs, const uint32_t* __restrict__ pos,
                             const uint32_t* __restrict__ part, const uint64_t* __restrict__ tbl_off,
                             const uint64_t* __restrict__ bc, const uint32_t* __restrict__ fo, int pb,
                             unsigned long long* __restrict__ keys, uint32_t* __restrict__ vals) {
  const uint64_t M = (1ull << pb) - 1ull;
  for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < S; s += gridDim.x * blockDim.x) {
    const SegInfo& g = segs[s];
    uint64_t key = ~0ull;
    if (g.cast != 0xFFFFFFFFu) {
      const uint32_t ps = pos != nullptr ? pos[s] : g.pos;
      const bool in = part == nullptr || part[s];
      if (in) {
        const uint64_t first = fo[tbl_off[g.frame] + g.hash % bc[g.frame]];
        key = (static_cast<uint64_t>(g.frame) << (2 * pb + 1)) | ((M - first) << pb) | (M - ps);
      } else {
        key = (static_cast<uint64_t>(g.frame) << (2 * pb + 1)) | (1ull << (2 * pb)) | ps;
      }
    }
    keys[s] = key;
    vals[s] = s;
  }
}

// ---- rehash epochs of the frames whose bucketing map rehashes (SURVEY.md
// Appendix B), all such frames of a batch at once. The frames' segments are
// concatenated (frame g owns [base, base + K)); every sort key carries g in its
// high bits, so one stable sort orders every frame's segments independently.
// Inside a frame, rank = first-appearance rank of the key. Epoch e (bucket
// count bc, keys of rank < t_hi present) re-inserts the previous epoch's
// iteration order (positions 0..t_lo-1), then the keys of rank [t_lo, t_hi) in
// first-appearance order; its iteration order sorts the present keys by (first
// occupation of their bucket desc, position desc). Frames with fewer epochs sit
// out the later ones (active = 0: key 0, no writes).
struct RhFrame {
  uint32_t seg0;    // first segment of the frame in segs
  uint32_t base;    // first index in the concatenated arrays
  uint32_t K;       // segments (distinct terminal keys) of the frame
  uint32_t ray0;    // first slot of the frame in the global ray order
  uint32_t t_lo;    // keys re-inserted from the previous epoch's order
  uint32_t t_hi;    // keys present in this epoch (clamped to K)
  uint32_t active;  // this epoch exists for the frame
  uint32_t last;    // this epoch is the frame's final one
  uint64_t bc;      // bucket count
  uint64_t fo_off;  // the frame's first-occupation table in fo
};

__global__ void k_rhb_init(uint32_t n, uint32_t G, const RhFrame* __restrict__ fr, const SegInfo* __restrict__ segs,
                           int pb, uint32_t* __restrict__ rh_g, uint32_t* __restrict__ keys,
                           uint32_t* __restrict__ vals) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    uint32_t lo = 0, hi = G;  // last frame with base <= i
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (fr[mid].base <= i) lo = mid; else hi = mid;
    }
    rh_g[i] = lo;
    keys[i] = (lo << pb) | segs[fr[lo].seg0 + (i - fr[lo].base)].pos;
    vals[i] = i;
  }
}

__global__ void k_rhb_rank(uint32_t n, const RhFrame* __restrict__ fr, const uint32_t* __restrict__ rh_g,
                           const uint32_t* __restrict__ by_pos, uint32_t* __restrict__ rank) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const uint32_t i = by_pos[j];
    rank[i] = j - fr[rh_g[i]].base;
  }
}

__device__ __forceinline__ uint32_t rh_pos(uint32_t rank, const uint32_t* prev, uint32_t i, uint32_t t_lo) {
  return rank < t_lo ? prev[i] : rank;
}

__global__ void k_rhb_fo(uint32_t n, const RhFrame* __restrict__ fr, const uint32_t* __restrict__ rh_g,
                         const SegInfo* __restrict__ segs, const uint32_t* __restrict__ rank,
                         const uint32_t* __restrict__ prev, uint32_t* __restrict__ fo) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const RhFrame p = fr[rh_g[i]];
    const uint32_t r = rank[i];
    if (!p.active || r >= p.t_hi) continue;
    atomicMin(&fo[p.fo_off + segs[p.seg0 + (i - p.base)].hash % p.bc], rh_pos(r, prev, i, p.t_lo));
  }
}

// pass 1 key (secondary): position, descending
__global__ void k_rhb_pos_desc(uint32_t n, const RhFrame* __restrict__ fr, const uint32_t* __restrict__ rh_g,
                               const uint32_t* __restrict__ rank, const uint32_t* __restrict__ prev, int kb,
                               uint32_t* __restrict__ keys, uint32_t* __restrict__ vals) {
  const uint32_t M = (1u << kb) - 1u;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t g = rh_g[i];
    const RhFrame& p = fr[g];
    keys[i] = (g << (kb + 1)) | (p.active ? M - rh_pos(rank[i], prev, i, p.t_lo) : 0u);
    vals[i] = i;
  }
}

// pass 2 key (primary, stable over pass 1): first occupation of the bucket,
// descending; keys not yet present last
__global__ void k_rhb_fo_desc(uint32_t n, const RhFrame* __restrict__ fr, const uint32_t* __restrict__ rh_g,
                              const uint32_t* __restrict__ vals, const SegInfo* __restrict__ segs,
                              const uint32_t* __restrict__ rank, const uint32_t* __restrict__ fo, int kb,
                              uint32_t* __restrict__ keys) {
  const uint32_t M = (1u << kb) - 1u;
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const uint32_t i = vals[j];
    const uint32_t g = rh_g[i];
    const RhFrame p = fr[g];
    uint32_t k = 0u;
    if (p.active)
      k = rank[i] < p.t_hi ? M - fo[p.fo_off + segs[p.seg0 + (i - p.base)].hash % p.bc] : M + 1u;
    keys[j] = (g << (kb + 1)) | k;
  }
}

// prev[order[j]] = local position for the present keys; on a frame's last
// epoch also its slice of the global ray order
__global__ void k_rhb_commit(uint32_t n, const RhFrame* __restrict__ fr, const uint32_t* __restrict__ rh_g,
                             const uint32_t* __restrict__ order, uint32_t* __restrict__ prev,
                             uint32_t* __restrict__ ray_order) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const uint32_t i = order[j];
    const RhFrame p = fr[rh_g[i]];
    if (!p.active) continue;
    const uint32_t jl = j - p.base;
    if (jl >= p.t_hi) continue;  // t_hi <= K
    prev[i] = jl;
    if (p.last) ray_order[p.ray0 + jl] = p.seg0 + (i - p.base);
  }
}

__global__ void k_gather_rays(uint32_t R, const uint32_t* __restrict__ order, const SegInfo* __restrict__ segs,
                              RayInfo* __restrict__ rays) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < R; j += gridDim.x * blockDim.x) {
    const SegInfo& g = segs[order[j]];
    RayInfo r;
    r.p[0] = g.mean[0];
    r.p[1] = g.mean[1];
    r.p[2] = g.mean[2];
    r.weight = g.base_weight;
    r.color = g.color;
    r.frame = g.frame;
    r.valid = g.cast;
    r.depth = 0.0f;
    r.term[0] = g.g[0];
    r.term[1] = g.g[1];
    r.term[2] = g.g[2];
    r.base = 0.0f;
    rays[j] = r;
  }
}

// Warp-aggregated counter add: lanes with equal `key` (frames are contiguous in
// ray order, so a warp usually spans one or two) combine into one atomic.
__device__ __forceinline__ void warp_add_by_key(unsigned long long* __restrict__ arr, uint32_t key, uint32_t val) {
  const unsigned active = __activemask();
  const unsigned peers = __match_any_sync(active, key);
  const uint32_t sum = __reduce_add_sync(peers, val);
  if ((threadIdx.x & 31) == static_cast<unsigned>(__ffs(peers) - 1) && sum != 0u)
    atomicAdd(&arr[key], static_cast<unsigned long long>(sum));
}

// measurement_weight (tsdf_integrator.cpp:29-44) with base = 1/(z*z) hoisted
// per ray (same value: fdiv(1, fmul(z, z))).
__device__ __forceinline__ float mweight_base(int mode, float base, float d, float truncation, float eps) {
  if (mode == VXG_WEIGHT_CONSTANT) return 1.0f;
  if (mode == VXG_WEIGHT_INVERSE_Z2) return base;
  if (mode != VXG_WEIGHT_INVERSE_Z2_DROPOFF) return 0.0f;
  if (d > -eps) return base;
  if (d < -truncation) return 0.0f;
  return fdiv(fmul(base, fadd(d, truncation)), fsub(truncation, eps));
}

// ---------------------------------------------------------------- rays -> records
// cast_and_update's prologue (tsdf_integrator.cpp:135-143): exactly span+1
// voxels per ray, so record offsets are known before traversal. Also stores
// the ray's depth and hoisted 1/depth^2.
__global__ void k_ray_count(uint32_t R, RayInfo* __restrict__ rays, const float* __restrict__ poses,
                            TsdfParams tp, unsigned long long* __restrict__ counts,
                            unsigned long long* __restrict__ raycasts, FoldRay* __restrict__ fray,
                            uint2* __restrict__ far) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < R; j += gridDim.x * blockDim.x) {
    const RayInfo r = rays[j];
    uint64_t c = 0;
    uint32_t cast = 0;
    if (r.valid == 1u) {
      const float* Pm = poses + 12 * r.frame;
      const float ray[3] = {fsub(r.p[0], Pm[3]), fsub(r.p[1], Pm[7]), fsub(r.p[2], Pm[11])};
      const float depth = norm3(ray[0], ray[1], ray[2]);
      rays[j].depth = depth;
      const float base = tp.weight_mode == VXG_WEIGHT_CONSTANT ? 1.0f : fdiv(1.0f, fmul(depth, depth));
      rays[j].base = base;
      FoldRay fr;
      fr.p[0] = r.p[0];
      fr.p[1] = r.p[1];
      fr.p[2] = r.p[2];
      fr.weight = r.weight;
      fr.color = r.color;
      fr.frame = r.frame;
      fr.base = base;
      fr.pad = depth;
      fray[j] = fr;
      far[j] = make_uint2(
          __float_as_uint(fmul(mweight_base(tp.weight_mode, base, 0.0f, tp.truncation, tp.dropoff_epsilon), r.weight)),
          r.color);
      if (!(depth <= 0.0f)) {
        cast = 1u;
        const float s = fdiv(tp.truncation, depth);
        Dda dda;
        dda.init(Pm[3], Pm[7], Pm[11], fadd(r.p[0], fmul(ray[0], s)), fadd(r.p[1], fmul(ray[1], s)),
                 fadd(r.p[2], fmul(ray[2], s)), tp.voxel_size);
        c = static_cast<uint64_t>(dda.span) + 1ull;
      }
    }
    counts[j] = c;
    warp_add_by_key(raycasts, r.frame, cast);
  }
}

struct TermView {  // per-frame sorted terminal keys for the anti-graze probe
  const unsigned long long* keys;
  const uint32_t* start;
  const uint32_t* count;
  int rb;
  int kb;
};

__device__ __forceinline__ bool is_terminal(const TermView& tv, uint32_t f, const int* og, const int* g) {
  const int lim = (1 << tv.kb) - 1;
  int e[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    e[k] = g[k] - og[k] + tv.rb;
    if (e[k] < 0 || e[k] >= lim) return false;
  }
  const uint64_t key = (static_cast<uint64_t>(f) << (3 * tv.kb)) | (static_cast<uint64_t>(e[0]) << (2 * tv.kb)) |
                       (static_cast<uint64_t>(e[1]) << tv.kb) | static_cast<uint64_t>(e[2]);
  uint32_t lo = tv.start[f], n = tv.count[f];
  while (n > 0) {
    const uint32_t half = n >> 1;
    const uint64_t k = tv.keys[lo + half];
    if (k < key) { lo += half + 1; n -= half + 1; } else { n = half; }
  }
  return lo < tv.start[f] + tv.count[f] && tv.keys[lo] == key;
}

// Per-CTA direct-mapped cache of block slots in shared memory. An entry is one
// 64-bit word (slot << 40 | 13-bit-per-axis block key), so concurrent
// readers/writers never see a torn pair; blocks outside the 13-bit range
// bypass the cache.
constexpr int kBlockCacheSize = 1024;

__device__ __forceinline__ bool cache_key13(int bx, int by, int bz, uint64_t* k) {
  // all three in [-4096, 4096): one unsigned compare on the biased values
  const uint32_t ux = static_cast<uint32_t>(bx + 4096), uy = static_cast<uint32_t>(by + 4096),
                 uz = static_cast<uint32_t>(bz + 4096);
  if ((ux | uy | uz) >= 8192u) return false;
  *k = (static_cast<uint64_t>(bx & 0x1FFF) << 26) | (static_cast<uint64_t>(by & 0x1FFF) << 13) |
       static_cast<uint64_t>(bz & 0x1FFF);
  return true;
}

__device__ __forceinline__ int32_t cached_find_or_insert(unsigned long long* cache, const MapView& map, int bx,
                                                         int by, int bz) {
  uint64_t k13;
  const bool cacheable = cache_key13(bx, by, bz, &k13);
  uint32_t idx = 0;
  if (cacheable) {
    // the cache index only has to spread neighbouring blocks (this path runs at a few
    // active lanes per warp in the walk: every instruction counts): two 32-bit multiplies
    const uint32_t h = static_cast<uint32_t>(bx) * 0x9E3779B1u ^ static_cast<uint32_t>(by) * 0x85EBCA6Bu ^
                       static_cast<uint32_t>(bz) * 0xC2B2AE35u;
    idx = (h >> 16) & (kBlockCacheSize - 1);
    const unsigned long long e = cache[idx];
    if (e != ~0ull && (e & ((1ull << 40) - 1)) == k13) return static_cast<int32_t>(e >> 40);
  }
  const int32_t slot = map.find_or_insert(pack_block(bx, by, bz), bx, by, bz);
  if (cacheable && slot >= 0) cache[idx] = (static_cast<unsigned long long>(slot) << 40) | k13;
  return slot;
}

// cast_and_update's loop (tsdf_integrator.cpp:145-171): walk, weigh, allocate,
// emit one record per candidate voxel at offset[ray] + k: (voxel key, ray
// index). The fold recomputes (d, w) from the ray with the same arithmetic, so
// records stay 8 bytes. Skipped candidates (anti-graze, w <= 0) emit an
// invalid key (sorted past every voxel, never folded).
//  * rays are processed in order of decreasing length (perm) so a warp's lanes
//    walk similar numbers of voxels; outputs still go to offset[ray].
//  * the walk state is kept in named registers (no runtime-indexed arrays);
//    per step only the stepped axis's centre and block/local split change
//    (same integer -> same vcenter; floor-div carry), both equal to the
//    reference's from-scratch values.
struct Walk {
  int c0, c1, c2;        // current voxel
  int e0, e1, e2;        // end voxel
  int s0, s1, s2;        // steps
  float m0, m1, m2;      // t_max
  float d0, d1, d2;      // t_delta
};

__device__ __forceinline__ void walk_axis_init(float st, float en, float v, int* cur, int* end, int* step,
                                               float* tmax, float* tdelta, uint32_t* span) {
  *cur = gidx(st, v);
  *end = gidx(en, v);
  const float dir = fsub(en, st);
  *step = dir > 0.0f ? 1 : (dir < 0.0f ? -1 : 0);
  if (*step == 0) {
    *tmax = __int_as_float(0x7f800000);
    *tdelta = __int_as_float(0x7f800000);
  } else {
    const float boundary = fmul(__int2float_rn(*cur + (*step > 0 ? 1 : 0)), v);
    *tmax = fdiv(fsub(boundary, st), dir);
    *tdelta = fdiv(v, fabsf(dir));
  }
  const int dd = *end - *cur;
  *span += static_cast<uint32_t>(dd < 0 ? -dd : dd);
}

// kAnti: MergeMode::kGroupedAntiGraze probe; kPow2: vps = 2^lg (block/local
// split by shift and mask, the floor division of core.h:34-40 for a power of
// two), else the incremental carry of the stepped axis.
// A warp walks its 32 rays in lockstep (step k of every lane, inactive past a
// ray's end); each lane stages its keys in a shared-memory row of 32, and every
// 32 steps the warp writes row after row as 128-byte runs (a ray's records are
// contiguous at offset[ray]): coalesced stores instead of 32 scattered ones.
#ifndef VXG_EMIT_THREADS
#define VXG_EMIT_THREADS 256
#endif
constexpr int kEmitThreads = VXG_EMIT_THREADS;
template <bool kAnti, bool kPow2>
__global__ void __launch_bounds__(kEmitThreads) k_emit(uint32_t R0, uint32_t R1, const uint32_t* __restrict__ perm,
                       const RayInfo* __restrict__ rays, const unsigned long long* __restrict__ roff, uint64_t base,
                       const float* __restrict__ poses, TsdfParams tp, MapView map, TermView tv,
                       uint32_t* __restrict__ rkeys, uint32_t* __restrict__ rvals,
                       unsigned long long* __restrict__ updates) {
  constexpr int kWarps = kEmitThreads / 32;
  __shared__ unsigned long long bcache[kBlockCacheSize];
  __shared__ uint32_t kstage[kWarps][32 * 33];  // one padded row per lane: conflict-free both ways
  __shared__ uint4 kmeta[kWarps][32];           // per lane: (count, first record, ray id)
  for (int i = threadIdx.x; i < kBlockCacheSize; i += blockDim.x) bcache[i] = ~0ull;
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31u, wib = threadIdx.x >> 5;
  uint32_t* row = &kstage[wib][lane * 33];
  const uint32_t* wrows = kstage[wib];
  const uint4* wmeta = kmeta[wib];
  const int vps = map.vps;
  const int lg = kPow2 ? __ffs(vps) - 1 : 0;
  const float v = tp.voxel_size;
  const uint32_t wstride = gridDim.x * kWarps * 32u;
  for (uint32_t t0 = R0 + (blockIdx.x * kWarps + wib) * 32u; t0 < R1; t0 += wstride) {
    const uint32_t t = t0 + lane;
    const bool has = t < R1;
    const uint32_t j = has ? perm[t] : 0u;
    RayInfo r;
    if (has) {
      r = rays[j];
    } else {
      r = RayInfo{};
      r.valid = 0u;
      r.frame = 0u;
    }
    const float* Pm = poses + 12 * r.frame;
    const float o0 = Pm[3], o1 = Pm[7], o2 = Pm[11];
    const float depth = r.depth;
    uint32_t valid = 0, count = 0, out0 = 0;
    const bool live = has && r.valid == 1u && !(depth <= 0.0f);
    float ray0 = 0.0f, ray1 = 0.0f, ray2 = 0.0f, w_front = 0.0f, t_safe = -1.0f, t_far = -1.0f;
    Walk wk{};
    if (live) {
      ray0 = fsub(r.p[0], o0), ray1 = fsub(r.p[1], o1), ray2 = fsub(r.p[2], o2);
      const float s = fdiv(tp.truncation, depth);
      // mweight_base for any d >= 0 (d > -eps in the drop-off mode), times the ray weight
      w_front = fmul(mweight_base(tp.weight_mode, r.base, 0.0f, tp.truncation, tp.dropoff_epsilon), r.weight);
      uint32_t span = 0;
      walk_axis_init(o0, fadd(r.p[0], fmul(ray0, s)), v, &wk.c0, &wk.e0, &wk.s0, &wk.m0, &wk.d0, &span);
      walk_axis_init(o1, fadd(r.p[1], fmul(ray1, s)), v, &wk.c1, &wk.e1, &wk.s1, &wk.m1, &wk.d1, &span);
      walk_axis_init(o2, fadd(r.p[2], fmul(ray2, s)), v, &wk.c2, &wk.e2, &wk.s2, &wk.m2, &wk.d2, &span);
      count = span + 1u;
      // walk parameter (0 at the origin, 1 at the end point p + ray * s) below
      // which every voxel centre is provably in front of the point: a voxel
      // left at t_exit * |end - o| < depth - 3 v has its centre at least
      // 1.1 v before the point along the ray (half diagonal 0.87 v, plus one
      // voxel for the DDA's rounded axis choices), where the reference's
      // rounded `along` cannot be negative, so d >= 0 and w = w_front
      t_safe = (depth - 3.0f * v) / (fadd(depth, tp.truncation) + v);
      // likewise a voxel left before t_far has its centre more than
      // truncation + 1.1 v before the point: d >= truncation (kFarRecord).
      // t_exit grows along the walk, so the far records are a prefix of the ray's.
      t_far = (depth - tp.truncation - 3.0f * v) / (fadd(depth, tp.truncation) + v);
      // record offsets inside one chunk are 32-bit (chunks stay below 2^29 records)
      out0 = static_cast<uint32_t>(roff[j] - base);
    }
    kmeta[wib][lane] = make_uint4(count, out0, j, 0u);
    int og0 = 0, og1 = 0, og2 = 0;
    if (kAnti) {
      og0 = gidx(o0, v);
      og1 = gidx(o1, v);
      og2 = gidx(o2, v);
    }
    int b0, b1, b2, l0, l1, l2;
    if (kPow2) {
      b0 = wk.c0 >> lg, b1 = wk.c1 >> lg, b2 = wk.c2 >> lg;
      l0 = wk.c0 & (vps - 1), l1 = wk.c1 & (vps - 1), l2 = wk.c2 & (vps - 1);
    } else {
      b0 = floor_div(wk.c0, vps), b1 = floor_div(wk.c1, vps), b2 = floor_div(wk.c2, vps);
      l0 = wk.c0 - b0 * vps, l1 = wk.c1 - b1 * vps, l2 = wk.c2 - b2 * vps;
    }
    int cb0 = 0x7fffffff, cb1 = 0, cb2 = 0;
    int32_t cslot = -1;
    const uint32_t maxc = __reduce_max_sync(0xffffffffu, count);
    __syncwarp();  // kmeta visible to the warp
    uint32_t nfar = 0;  // leading records of this ray proven far (kFarRecord)
    for (uint32_t k = 0; k < maxc; ++k) {
      if (k < count) {
        nfar += fminf(fminf(wk.m0, wk.m1), wk.m2) < t_far ? 1u : 0u;
        uint32_t key = kInvalidRecord;
        bool skip = false;
        if (kAnti) {
          const int g[3] = {wk.c0, wk.c1, wk.c2};
          const int og[3] = {og0, og1, og2};
          skip = !(wk.c0 == r.term[0] && wk.c1 == r.term[1] && wk.c2 == r.term[2]) && is_terminal(tv, r.frame, og, g);
        }
        if (!skip) {
          // projective_distance(x, p, s) (tsdf_integrator.cpp:22-27); p - s == ray.
          // In front of the point (along >= 0) d = +|t| >= 0, where every weight
          // mode gives the ray's constant w_front: the norm is needed only behind it.
          float w = w_front;
          const float t_exit = fminf(fminf(wk.m0, wk.m1), wk.m2);
          if (!(t_exit < t_safe)) {  // the last voxels of the walk: evaluate along (and d behind the point)
            const float x0 = vcenter(wk.c0, v), x1 = vcenter(wk.c1, v), x2 = vcenter(wk.c2, v);
            const float t0f = fsub(r.p[0], x0), t1f = fsub(r.p[1], x1), t2f = fsub(r.p[2], x2);
            const float along = dot3(t0f, t1f, t2f, ray0, ray1, ray2);
            if (!(along >= 0.0f)) {
              const float magnitude = norm3(t0f, t1f, t2f);
              const float d = along < 0.0f ? -magnitude : magnitude;
              w = fmul(mweight_base(tp.weight_mode, r.base, d, tp.truncation, tp.dropoff_epsilon), r.weight);
            }
          }
          if (!(w <= 0.0f)) {
            if (b0 != cb0 || b1 != cb1 || b2 != cb2) {
              cb0 = b0;
              cb1 = b1;
              cb2 = b2;
              if (block_in_range(b0, b1, b2)) {
                cslot = cached_find_or_insert(bcache, map, b0, b1, b2);
              } else {
                atomicOr(&map.counters[1], static_cast<uint32_t>(kErrKeyRange));
                cslot = -1;
              }
            }
            if (cslot >= 0) {
              const uint32_t lin = kPow2 ? static_cast<uint32_t>(l0 | (l1 << lg) | (l2 << (2 * lg)))
                                         : static_cast<uint32_t>(l0 + vps * (l1 + vps * l2));
              key = static_cast<uint32_t>(cslot) * static_cast<uint32_t>(map.nvox) + lin;
            }
            ++valid;
          }
        }
        row[k & 31u] = key;
        // RayCaster::next tail (the walk stops after count voxels, which is
        // where the reference's end-voxel test stops it): axis = argmin t_max,
        // ties to the lowest axis. Straight-line selects: the lanes of a warp
        // step different axes.
        const bool a1 = wk.m1 < wk.m0;
        const float mlo = a1 ? wk.m1 : wk.m0;
        const bool a2 = wk.m2 < mlo;
        const bool st2 = a2, st1 = !a2 & a1, st0 = !a2 & !a1;
        wk.c0 += st0 ? wk.s0 : 0;
        wk.c1 += st1 ? wk.s1 : 0;
        wk.c2 += st2 ? wk.s2 : 0;
        wk.m0 = st0 ? fadd(wk.m0, wk.d0) : wk.m0;
        wk.m1 = st1 ? fadd(wk.m1, wk.d1) : wk.m1;
        wk.m2 = st2 ? fadd(wk.m2, wk.d2) : wk.m2;
        if (kPow2) {
          b0 = wk.c0 >> lg, b1 = wk.c1 >> lg, b2 = wk.c2 >> lg;
          l0 = wk.c0 & (vps - 1), l1 = wk.c1 & (vps - 1), l2 = wk.c2 & (vps - 1);
        } else {
          l0 += st0 ? wk.s0 : 0;
          l1 += st1 ? wk.s1 : 0;
          l2 += st2 ? wk.s2 : 0;
          b0 += (l0 == vps) - (l0 < 0);
          b1 += (l1 == vps) - (l1 < 0);
          b2 += (l2 == vps) - (l2 < 0);
          l0 = l0 == vps ? 0 : (l0 < 0 ? vps - 1 : l0);
          l1 = l1 == vps ? 0 : (l1 < 0 ? vps - 1 : l1);
          l2 = l2 == vps ? 0 : (l2 < 0 ? vps - 1 : l2);
        }
      }
      if ((k & 31u) == 31u || k + 1u == maxc) {  // warp-uniform: write the staged rows
        kmeta[wib][lane].w = nfar;  // far records are a prefix: those below nfar so far
        __syncwarp();
        const uint32_t k0 = k & ~31u, nrow = (k & 31u) + 1u;
        for (uint32_t l = 0; l < 32u; ++l) {
          const uint4 ml = wmeta[l];  // broadcast
          if (ml.x > k0) {
            const uint32_t m = min(nrow, ml.x - k0);
            if (lane < m) {
              const uint32_t o = ml.y + k0 + lane;
              rkeys[o] = wrows[l * 33u + lane];
              rvals[o] = ml.z | (k0 + lane < ml.w ? kFarRecord : 0u);  // ray index (+ far flag): the sort value
            }
          }
        }
        __syncwarp();
      }
    }
    warp_add_by_key(updates, r.frame, valid);
  }
}

// ---------------------------------------------------------------- sharded map (multi-GPU)
// Update records travelling between shards carry a global voxel key:
// (bx + 2^14) << 49 | (by + 2^14) << 34 | (bz + 2^14) << 19 | local linear
// index (vps <= 64). The owner of a block is mix64(packed block) % world.
constexpr int32_t kGBias = 1 << 14;

__device__ __host__ __forceinline__ bool gkey_encode(int b0, int b1, int b2, uint32_t lin, uint64_t* out) {
  if (b0 < -kGBias || b0 >= kGBias || b1 < -kGBias || b1 >= kGBias || b2 < -kGBias || b2 >= kGBias) return false;
  *out = (static_cast<uint64_t>(b0 + kGBias) << 49) | (static_cast<uint64_t>(b1 + kGBias) << 34) |
         (static_cast<uint64_t>(b2 + kGBias) << 19) | static_cast<uint64_t>(lin);
  return true;
}

__device__ __host__ __forceinline__ void gkey_decode(uint64_t k, int* b, uint32_t* lin) {
  b[0] = static_cast<int>((k >> 49) & 0x7FFF) - kGBias;
  b[1] = static_cast<int>((k >> 34) & 0x7FFF) - kGBias;
  b[2] = static_cast<int>((k >> 19) & 0x7FFF) - kGBias;
  *lin = static_cast<uint32_t>(k & 0x7FFFF);
}

__device__ __host__ __forceinline__ uint32_t block_owner(int b0, int b1, int b2, uint32_t world) {
  return static_cast<uint32_t>(mix64(pack_block(b0, b1, b2)) % world);
}

// Sharded emit, second half: the walk itself is the single-GPU k_emit run
// against a DICTIONARY (a block hash without a slab: the blocks this rank's ray
// slice touches, in first-touch order), so its records carry 32-bit keys
// dict_slot * nvox + local. This pass turns them into what travels: the global
// voxel key and the owner of its block (world = dropped: skipped candidates,
// zero-weight updates, blocks outside the +-2^14 key range, and in the
// replicated traversal the other owners' records). The values (ray id + far
// flag) are used as they are.
__global__ void k_globalize(uint64_t n, const uint32_t* __restrict__ keys, const int32_t* __restrict__ dict_bidx,
                            uint32_t nvox, uint32_t world, int keep_owner, unsigned long long* __restrict__ gkeys,
                            uint32_t* __restrict__ owner, uint32_t* __restrict__ counters) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t k = keys[i];
    unsigned long long gk = ~0ull;
    uint32_t own = world;
    if (k != kInvalidRecord) {
      const uint32_t slot = k / nvox, lin = k - slot * nvox;
      const int b0 = dict_bidx[3 * slot], b1 = dict_bidx[3 * slot + 1], b2 = dict_bidx[3 * slot + 2];
      uint64_t e;
      if (gkey_encode(b0, b1, b2, lin, &e)) {
        gk = e;
        own = block_owner(b0, b1, b2, world);
        if (keep_owner >= 0 && own != static_cast<uint32_t>(keep_owner)) own = world;
      } else {
        atomicOr(&counters[1], static_cast<uint32_t>(kErrKeyRange));
      }
    }
    gkeys[i] = gk;
    owner[i] = own;
  }
}

// bounds[o] = first position of owner o in the owner-sorted records (o <= world).
__global__ void k_owner_bounds(uint64_t n, const uint32_t* __restrict__ sorted_owner, uint32_t world,
                               unsigned long long* __restrict__ bounds) {
  const uint32_t o = blockIdx.x * blockDim.x + threadIdx.x;
  if (o > world) return;
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (sorted_owner[mid] < o) lo = mid + 1; else hi = mid;
  }
  bounds[o] = lo;
}

// Ray range of a record range: first ray whose record offset is >= lo / >= hi.
__global__ void k_ray_bounds(uint32_t R, const unsigned long long* __restrict__ roff, uint64_t lo_rec, uint64_t hi_rec,
                             unsigned long long* __restrict__ out) {
  const uint32_t t = threadIdx.x;
  if (t > 1) return;
  const uint64_t target = t == 0 ? lo_rec : hi_rec;
  uint32_t lo = 0, hi = R;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (roff[mid] < target) lo = mid + 1; else hi = mid;
  }
  out[t] = lo;
}

// Packs the owner-sorted records into 16-byte messages {key lo, key hi, ray, 0}.
__global__ void k_gather_send(uint64_t n, const uint32_t* __restrict__ perm, const unsigned long long* __restrict__ gkeys,
                              const uint32_t* __restrict__ gvals, uint4* __restrict__ send) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t p = perm[i];
    const unsigned long long k = gkeys[p];
    send[i] = make_uint4(static_cast<uint32_t>(k), static_cast<uint32_t>(k >> 32), gvals[p], 0u);
  }
}

// Owner side: global voxel key -> this shard's slot (allocating on first
// update, like get_or_allocate_block) -> u32 record key; counts updates per frame.
__global__ void k_localize(uint64_t n, const uint4* __restrict__ recv, MapView map, const FoldRay* __restrict__ rays,
                           uint32_t* __restrict__ rkeys, uint32_t* __restrict__ rvals,
                           unsigned long long* __restrict__ updates) {
  // Records arrive in ray order, so a warp's 32 consecutive records are a few
  // segments of one ray inside one block each: the first lane of a block
  // segment looks the block up (shared-memory cache, then the hash) and hands
  // the slot to its segment, the first lane of a ray segment reads the ray's
  // frame and adds the segment's length to the frame's update count.
  __shared__ unsigned long long bcache[kBlockCacheSize];
  for (int i = threadIdx.x; i < kBlockCacheSize; i += blockDim.x) bcache[i] = ~0ull;
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31u;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i0 = blockIdx.x * static_cast<uint64_t>(blockDim.x) + (threadIdx.x & ~31u); i0 < n; i0 += stride) {
    const uint64_t i = i0 + lane;  // warp-uniform trip count (full-warp shuffles)
    const bool in = i < n;
    const uint4 m = in ? recv[i] : make_uint4(0u, 0u, 0u, 0u);
    const uint64_t k = static_cast<uint64_t>(m.x) | (static_cast<uint64_t>(m.y) << 32);
    const uint64_t blk = k >> 19;  // the block part of the global key
    const uint32_t ray = m.z & kRayMask;
    const uint64_t pblk = __shfl_up_sync(0xffffffffu, blk, 1);
    const uint32_t pray = __shfl_up_sync(0xffffffffu, ray, 1);
    const uint32_t inm = __ballot_sync(0xffffffffu, in);
    const bool bhead = in && (lane == 0u || pblk != blk);
    const bool rhead = in && (lane == 0u || pray != ray);
    const uint32_t bheads = __ballot_sync(0xffffffffu, bhead), rheads = __ballot_sync(0xffffffffu, rhead);
    int32_t slot = -1;
    if (bhead) {
      int b[3];
      uint32_t l;
      gkey_decode(k, b, &l);
      slot = cached_find_or_insert(bcache, map, b[0], b[1], b[2]);
    }
    const uint32_t upto = (2u << lane) - 1u;  // lanes 0..lane
    const int bsrc = 31 - __clz(bheads & upto);
    slot = __shfl_sync(0xffffffffu, slot, bsrc < 0 ? 0 : bsrc);
    if (in) {
      const uint32_t lin = static_cast<uint32_t>(k & ((1ull << 19) - 1ull));
      rkeys[i] = slot >= 0 ? static_cast<uint32_t>(slot) * static_cast<uint32_t>(map.nvox) + lin : kInvalidRecord;
      rvals[i] = m.z;  // ray id + far flag
    }
    if (rhead) {  // this ray segment: [lane, next ray head or the end of the valid lanes)
      const uint32_t after = rheads & ~upto;
      const uint32_t end = after ? static_cast<uint32_t>(__ffs(after) - 1) : static_cast<uint32_t>(__popc(inm));
      atomicAdd(&updates[rays[ray].frame], static_cast<unsigned long long>(end - lane));
    }
  }
}

// update_tsdf_voxel applied per voxel in (frame, ray-order) order. Records are
// stably sorted by voxel key into runs (one per voxel), handed out longest
// first. A run's fold is an inherently serial chain, so the kernel keeps
// everything that does not depend on the voxel state OFF that chain:
//  * runs >= kLongRun (the critical path, a few thousand runs): one warp per run. The 32 lanes gather 32 records
//    (coalesced ray ids, parallel ray reads) and evaluate (d, w) in parallel,
//    two chunks ahead of the fold; every lane then folds the chunk from shared
//    memory (redundantly, so no lane idles on a branch).
//  * shorter runs: one thread per run, 32 runs per warp, (d, w) for
//    kFoldChunk records evaluated ahead of each folded chunk.
// The fold step itself is update_voxel_fast (shared reciprocal, stationary
// colour skip), bit-identical to update_tsdf_voxel.
#ifndef VXG_LONG_RUN
#define VXG_LONG_RUN 4096
#endif
constexpr uint32_t kLongRun = VXG_LONG_RUN;
constexpr int kFoldChunk = 8;

struct alignas(16) Upd {
  float d;
  float w;
  uint32_t c;
  uint32_t pad;
};

// org: sensor origins, 3 floats per frame (the fold kernels stage them in
// shared memory so the only global latency per record is the ray gather).
// mweight_base with the dropoff division by the constant (truncation - eps)
// through its precomputed reciprocal (exact inside the fast range, else the
// IEEE division itself).
__device__ __forceinline__ float mweight_base_r(int mode, float base, float d, float truncation, float eps,
                                                const Recip& den) {
  if (mode == VXG_WEIGHT_CONSTANT) return 1.0f;
  if (mode == VXG_WEIGHT_INVERSE_Z2) return base;
  if (mode != VXG_WEIGHT_INVERSE_Z2_DROPOFF) return 0.0f;
  if (d > -eps) return base;
  if (d < -truncation) return 0.0f;
  const float n = fmul(base, fadd(d, truncation));
  if (den.ok && fast_range(n)) return fast_quot(n, den);
  return fdiv(n, den.b);
}

__device__ __forceinline__ Upd weigh(const FoldRay& ry, const float* org, float x0, float x1, float x2,
                                     const TsdfParams& tp) {
  const float* O = org + 3 * ry.frame;
  Upd u;
  u.d = projective_distance(x0, x1, x2, ry.p[0], ry.p[1], ry.p[2], O[0], O[1], O[2]);
  const Recip den = make_recip(fsub(tp.truncation, tp.dropoff_epsilon));  // loop-invariant
  u.w = fmul(mweight_base_r(tp.weight_mode, ry.base, u.d, tp.truncation, tp.dropoff_epsilon, den), ry.weight);
  u.c = ry.color;
  u.pad = 0u;
  return u;
}

// A record's ray for the fold: far records (kFarRecord) read only the
// FarRay (no FoldRay load); the weighing then runs branch-free on a zero ray
// and weigh_far selects the far values, so a warp whose lanes mix far and near
// records does not diverge.
struct FoldIn {
  FoldRay ry;
  uint2 fr;  // {w_front bits, colour}; .x = 0xFFFFFFFF marks a near record
};
__device__ __forceinline__ FoldIn load_fold_in(const FoldRay* __restrict__ rays, const uint2* __restrict__ far,
                                               uint32_t v) {
  FoldIn in;
  const uint32_t r = v & kRayMask;
  if (v & kFarRecord) {
    in.ry = FoldRay{};
    in.fr = far[r];
  } else {
    in.ry = rays[r];
    in.fr = make_uint2(0xFFFFFFFFu, 0u);
  }
  return in;
}
__device__ __forceinline__ Upd weigh_in(const FoldIn& in, const float* org, float x0, float x1, float x2,
                                        const TsdfParams& tp) {
  Upd u = weigh(in.ry, org, x0, x1, x2, tp);
  const bool far = in.fr.x != 0xFFFFFFFFu;
  u.d = far ? tp.truncation : u.d;
  u.w = far ? __uint_as_float(in.fr.x) : u.w;
  u.c = far ? in.fr.y : u.c;
  return u;
}
// Warp-cooperative form (every lane weighs its own record, all lanes call):
// when no lane holds a near record the projective distance is skipped.
__device__ __forceinline__ Upd weigh_in_warp(const FoldIn& in, bool live, const float* org, float x0, float x1,
                                             float x2, const TsdfParams& tp) {
  const bool far = in.fr.x != 0xFFFFFFFFu;
  if (__all_sync(0xffffffffu, far || !live)) {
    Upd u;
    u.d = tp.truncation;
    u.w = __uint_as_float(in.fr.x);
    u.c = in.fr.y;
    u.pad = 0u;
    return u;
  }
  return weigh_in(in, org, x0, x1, x2, tp);
}

constexpr uint32_t kOrgCache = 1024;  // frames whose origins fit the fold kernels' smem table

__global__ void k_origins(uint32_t F, const float* __restrict__ poses, float* __restrict__ org) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < 3 * F; i += gridDim.x * blockDim.x)
    org[i] = poses[12 * (i / 3) + 3 + 4 * (i % 3)];
}

// Stages the origin table in shared memory (kSmem: the host launched the
// variant only when F <= kOrgCache, so the loads compile to LDS).
template <bool kSmem>
__device__ __forceinline__ const float* stage_origins(float* s_org, const float* __restrict__ g_org, uint32_t F) {
  if (!kSmem) return g_org;
  for (uint32_t i = threadIdx.x; i < 3 * F; i += blockDim.x) s_org[i] = g_org[i];
  __syncthreads();
  return s_org;
}

struct RunCtx {
  uint32_t key, start, len;
  float x0, x1, x2;
};

__device__ __forceinline__ RunCtx run_ctx(const MapView& map, const TsdfParams& tp, const uint32_t* ukeys,
                                          const uint32_t* ustart, const uint32_t* ulen, uint32_t run) {
  RunCtx c;
  c.key = ukeys[run];
  c.start = ustart[run];
  c.len = ulen[run];
  c.x0 = c.x1 = c.x2 = 0.0f;
  if (c.key == kInvalidRecord) return c;  // run of skipped candidates: never folded
  const int vps = map.vps;
  const uint32_t slot = c.key / static_cast<uint32_t>(map.nvox);
  const uint32_t lin = c.key - slot * static_cast<uint32_t>(map.nvox);
  const int l0 = static_cast<int>(lin % vps), l1 = static_cast<int>((lin / vps) % vps),
            l2 = static_cast<int>(lin / (vps * vps));
  c.x0 = vcenter(map.block_idx[3 * slot + 0] * vps + l0, tp.voxel_size);
  c.x1 = vcenter(map.block_idx[3 * slot + 1] * vps + l1, tp.voxel_size);
  c.x2 = vcenter(map.block_idx[3 * slot + 2] * vps + l2, tp.voxel_size);
  return c;
}

struct VoxState {
  float D, W, cr, cg, cb;
};

__device__ __forceinline__ VoxState load_vox(const vxg_voxel* vp) {
  VoxState s;
  s.D = vp->distance;
  s.W = vp->weight;
  s.cr = static_cast<float>(vp->r);
  s.cg = static_cast<float>(vp->g);
  s.cb = static_cast<float>(vp->b);
  return s;
}

__device__ __forceinline__ void store_vox(vxg_voxel* vp, const VoxState& s) {
  vp->distance = s.D;
  vp->weight = s.W;
  vp->r = static_cast<uint8_t>(s.cr);
  vp->g = static_cast<uint8_t>(s.cg);
  vp->b = static_cast<uint8_t>(s.cb);
}

constexpr int floor_log2_c(uint32_t x) { return x <= 1u ? 0 : 1 + floor_log2_c(x >> 1); }
static_assert(kLongRun >= 16u && (kLongRun & ((1u << (floor_log2_c(kLongRun) - 3)) - 1u)) == 0u,
              "kLongRun must be the first length of its run-length code (run_len_code)");

// Long runs come first in the fold order: sorted_code holds kRunCodeMax -
// run_len_code(length) in ascending order; a run is long when its code is >=
// long_code. The host picks long_code per fold (vxg_handle::long_code_for):
// code(kLongRun) for full batches (kLongRun starts a code, so that is len >=
// kLongRun), lower for small ones, where the thread-per-run path would leave
// one thread folding a thousand-record run while the GPU idles.
__device__ __forceinline__ uint32_t count_long_runs(const uint32_t* __restrict__ sorted_code, uint32_t nruns,
                                                    uint32_t long_code) {
  const uint32_t thr = kRunCodeMax - long_code;
  uint32_t lo = 0, hi = nruns;  // first index whose run is short
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (sorted_code[mid] <= thr) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// ---- warp-specialised long-run fold (phase 1)
// Each long run is processed by a PAIR of warps: the producer gathers and
// weighs 32 records per chunk (ids two chunks ahead, rays one chunk ahead)
// into a kRingStages-deep shared-memory ring; the consumer only folds. mbarrier
// full/empty per stage hand chunks over, so the consumer's serial chain never
// waits on global memory or on the weighing arithmetic.
#ifndef VXG_RING_STAGES
#define VXG_RING_STAGES 4
#endif
constexpr int kRingStages = VXG_RING_STAGES;

struct alignas(32) PreRec {  // one record as handed to the long-run consumer (one 32-byte sector)
  float W;   // weight before this update (the producer's W scan)
  float T;   // RN(W + w)
  float r1;  // refined reciprocal of T
  float wc;  // RN(w * clamp(d))
  uint32_t c;   // colour word (has_color << 31); the consumer forms RN(w * channel) itself when it needs it
  float w, d;   // raw (for the colour chains and the exact fallback)
  uint32_t ok;  // w in (0, 2^100) and T in the fast-division range
};

// Per-chunk summary the producer publishes with the chunk: the weight after
// it, whether every record is in the fast range, and per colour channel the
// interval of current colours o for which every record of the chunk is
// stationary: RN(|n - o| w) < RN(0.499 T) <=> |n - o| <= k with
// k = max{k : RN(k w) < RN(0.499 T)} (RN(k w) is monotone in k).
struct alignas(16) ChunkHdr {
  float W_end;
  uint32_t ok;
  int lo[3];
  int hi[3];
};

// Some k in [0, 255] with RN(k w) < thr, for w > 0 and thr > 0 (RN(k w) is
// monotone in k, so every smaller k qualifies too): the estimate thr / w,
// shaved by 1e-4 and verified by the one multiplication that defines it. It
// is the maximal k except within 1e-4 of an integer quotient; a smaller
// radius only sends a few more chunks down the colour chains (same results).
__device__ __forceinline__ int stationary_radius(float w, float thr) {
  const int k = static_cast<int>(fminf(__fdividef(thr, w) * 0.9999f, 255.0f));
  return (k > 0 && __fmul_rn(static_cast<float>(k), w) < thr) ? k : 0;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "VXG_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra VXG_WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// Non-blocking look at a phase (acquire, like try_wait): 1 when it has completed.
// The result is an ordinary register, so the instruction's latency overlaps
// whatever the warp does before it reads the flag.
__device__ __forceinline__ uint32_t mbar_test(unsigned long long* bar, uint32_t parity) {
  uint32_t r;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(r)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return r;
}

// Run marks of the sorted records: voxel k's records are [dense_start[k],
// dense_end[k]) (dense_end[k] stays 0 for a voxel without records).
__global__ void k_run_marks(uint64_t T, const uint32_t* __restrict__ skeys, uint32_t* __restrict__ dense_start,
                            uint32_t* __restrict__ dense_end) {
  // 4 keys per thread (16-byte loads); neighbours across threads by shuffle
  const uint64_t n4 = (T + 3) / 4;
  const uint32_t lane = threadIdx.x & 31u;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t q0 = blockIdx.x * static_cast<uint64_t>(blockDim.x); q0 < n4; q0 += stride) {
    const uint64_t q = q0 + threadIdx.x;  // warp-uniform trip count (full-warp shuffles)
    uint32_t k[4];
    if (4 * q + 3 < T) {
      const uint4 v = reinterpret_cast<const uint4*>(skeys)[q];
      k[0] = v.x; k[1] = v.y; k[2] = v.z; k[3] = v.w;
    } else {
#pragma unroll
      for (int u = 0; u < 4; ++u) k[u] = 4 * q + u < T ? skeys[4 * q + u] : kInvalidRecord;
    }
    uint32_t prev = __shfl_up_sync(0xffffffffu, k[3], 1);
    uint32_t next = __shfl_down_sync(0xffffffffu, k[0], 1);
    if (lane == 0u) prev = q > 0 && 4 * q - 1 < T ? skeys[4 * q - 1] : kInvalidRecord;
    if (lane == 31u) next = 4 * q + 4 < T ? skeys[4 * q + 4] : kInvalidRecord;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint64_t i = 4 * q + u;
      const uint32_t key = k[u];
      if (i >= T || key == kInvalidRecord) continue;  // invalid keys sort after every run; never folded
      const uint32_t before = u == 0 ? prev : k[u - 1];
      const uint32_t after = u == 3 ? next : k[u + 1];
      if (i == 0 || before != key) dense_start[key] = static_cast<uint32_t>(i);
      if (i + 1 == T || after != key) dense_end[key] = static_cast<uint32_t>(i + 1);
    }
  }
}

// Shared state of kP long-run producer/consumer pairs.
template <int kP>
struct LongSmem {
  PreRec ring[kP][kRingStages][32];
  unsigned long long ring_full[kP][kRingStages];
  unsigned long long ring_empty[kP][kRingStages];
  uint32_t pair_run[kP];
  float4 wscan[kP][8];  // the chunk's 32 weights, broadcast to the producer lanes
  ChunkHdr ring_hdr[kP][kRingStages];
  uint2 spec_tab[kP][2][32];  // per record: its step as a map over 7 candidate distances (+ dead), one byte each
  // two producers per run (kProd = 2) alternate chunks: chunk c's producer hands the weight after it to
  // chunk c+1's through wbox[c & 1] / wfull[c & 1]
  float wbox[kP][2];
  unsigned long long wfull[kP][2];
};

template <int kP>
__device__ __forceinline__ void long_smem_init(LongSmem<kP>& S) {
  if (threadIdx.x < kP * kRingStages) {
    // one arrival per hand-over: lane 0, after a __syncwarp that orders the warp's ring accesses before it
    mbar_init(&S.ring_full[threadIdx.x / kRingStages][threadIdx.x % kRingStages], 1);
    mbar_init(&S.ring_empty[threadIdx.x / kRingStages][threadIdx.x % kRingStages], 1);
  }
  if (threadIdx.x < kP * 2) mbar_init(&S.wfull[threadIdx.x / 2][threadIdx.x % 2], 1);
}

// Long runs (>= kLongRun records), one producer/consumer warp pair per run,
// handed out longest first through work[0]. wid: this warp's index among the
// 2 kP pair warps (named barriers 1..kP). kSep: consumers only on
// sub-partitions 0 and 1 (warp & 3 < 2), producers on 2 and 3, so no consumer
// shares its scheduler with a producer.
template <int kP, bool kSep, int kProd = 1, bool kDbg = true>
__device__ __forceinline__ void fold_long_pairs(
    LongSmem<kP>& S, const int wid, const float* poses, const uint32_t nruns, const uint32_t n_long,
    const uint32_t* __restrict__ order, const uint32_t* __restrict__ ukeys, const uint32_t* __restrict__ ustart,
    const uint32_t* __restrict__ ulen, const uint32_t* __restrict__ svals, const FoldRay* __restrict__ rays, const uint2* __restrict__ far,
    const MapView& map, const TsdfParams& tp, uint8_t* __restrict__ touched, uint32_t* __restrict__ work,
    unsigned long long* __restrict__ dbg_arg) {
  // kDbg = false: the trace hooks below (22 per chunk) compile away
  unsigned long long* const dbg = kDbg ? dbg_arg : nullptr;
  auto& ring = S.ring;
  auto& ring_full = S.ring_full;
  auto& ring_empty = S.ring_empty;
  auto& pair_run = S.pair_run;
  auto& wscan = S.wscan;
  auto& ring_hdr = S.ring_hdr;
  const uint32_t n_all = nruns;
  const int lane = threadIdx.x & 31;
  const float Wmax = tp.max_weight;
  {
    // default (kP = 4): consumers are warps 4..7 (highest ids: the warp
    // arbiter favours them); pair p = consumer 4+p (sub-partition p) +
    // producer (p+1)&3 (another one)
    // kProd = 2 (kP = 4, the merged grid): warps 0..7 are producers, 8..11 consumers; producer h of pair p
    // is warp 4 h + ((p + 1 + h) & 3): never on its consumer's sub-partition
    static_assert(kProd == 1 || (kProd == 2 && kP == 4 && !kSep), "two producers: the kP = 4 merged layout only");
    const bool producer = kProd == 2 ? wid < 2 * kP : (kSep ? (wid & 3) >= 2 : wid < kP);
    const int ph = kProd == 2 ? (wid >> 2) : 0;  // which of the run's producers this warp is
    const int pair = kProd == 2 ? (producer ? (((wid & 3) + 3 - ph) & 3) : (wid - 2 * kP))
                                : (kSep ? ((wid >> 2) * 2 + (wid & 1)) : (producer ? ((wid + kP - 1) % kP) : (wid - kP)));
    constexpr int kPairThreads = 32 * (1 + kProd);
    uint32_t kk0 = 0;  // chunks of this pair's earlier runs (ring position / phase of chunk k: kk0 + k)
    while (true) {
      if (!producer && lane == 0) pair_run[pair] = atomicAdd(&work[0], 1u);
      asm volatile("bar.sync %0, %1;" ::"r"(1 + pair), "n"(kPairThreads) : "memory");
      const uint32_t r = pair_run[pair];
      asm volatile("bar.sync %0, %1;" ::"r"(1 + pair), "n"(kPairThreads) : "memory");  // pair_run is rewritten next run
      if (r >= n_long) break;
      const RunCtx c = run_ctx(map, tp, ukeys, ustart, ulen, order[r]);
      if (c.key == kInvalidRecord) continue;
      const uint32_t nchunks = (c.len + 31) >> 5;
      vxg_voxel* vp = map.slab + c.key;
      if (producer) {
        // The weight chain W_{i+1} = min(W_i + w_i, Wmax) does not depend on
        // the distance or the colours: run it here and hand each record its
        // W_i, T_i = RN(W_i + w_i), reciprocal, RN(w clamp(d)), RN(w n_c).
        long long pwait = 0, pbusy0 = dbg != nullptr ? clock64() : 0, pt_weigh = 0, pt_scan = 0, pt_top = 0, pt_pre = 0,
                  pt_store = 0;
        float W = vp->weight;
        // pipeline (gather latency ~ a whole chunk of the consumer's chain):
        // rays three chunks ahead, their ids five chunks ahead
        const FoldIn zr{FoldRay{}, make_uint2(0xFFFFFFFFu, 0u)};
        const uint32_t* ids = svals + c.start;
        auto id_at = [&](uint32_t jj) { return jj < c.len ? ids[jj] : 0u; };
        auto ray_at = [&](uint32_t jj, uint32_t v) { return jj < c.len ? load_fold_in(rays, far, v) : zr; };
        auto weigh_at = [&](uint32_t jj, const FoldIn& r) {
          Upd x = weigh_in_warp(r, jj < c.len, poses, c.x0, c.x1, c.x2, tp);
          if (jj >= c.len) {
            x.d = 0.0f;
            x.w = 0.0f;
            x.c = 0u;
            x.pad = 0u;
          }
          return x;
        };
        // this producer's chunks: ph, ph + kProd, ...; pos(i) = its lane's record of own chunk i
        auto pos = [&](uint32_t i) { return ((static_cast<uint32_t>(ph) + kProd * i) << 5) + lane; };
        FoldIn ry1 = ray_at(pos(1), id_at(pos(1)));
        FoldIn ry2 = ray_at(pos(2), id_at(pos(2)));
        uint32_t v3 = id_at(pos(3)), v4 = id_at(pos(4));
        // records are weighed one chunk ahead of their hand-over
        Upd u_next = weigh_at(pos(0), ray_at(pos(0), id_at(pos(0))));
        for (uint32_t i = 0, k = ph; k < nchunks; ++i, k += kProd) {
          const uint32_t kk = kk0 + k;
          const long long tt0 = dbg != nullptr ? clock64() : 0;
          const FoldIn ry3 = ray_at(pos(i + 3), v3);
          v3 = v4;
          v4 = id_at(pos(i + 5));
          const uint32_t cnt = min(32u, c.len - k * 32);
          const Upd u = u_next;
          const long long tp0 = dbg != nullptr ? clock64() : 0;
          pt_top += tp0 - tt0;
          u_next = weigh_at(pos(i + 1), ry1);
          if (dbg != nullptr) {  // force the weighing to complete before the timestamp
            asm volatile("" ::"f"(u_next.d), "f"(u_next.w));
            pt_weigh += clock64() - tp0;
          }
          const long long tp1 = dbg != nullptr ? clock64() : 0;
          // The weight chain W_{i+1} = min(RN(W_i + w_i), Wmax) (w_i > 0) does
          // not depend on the distance or the colours: run it here and hand
          // each record its W_i, T_i = RN(W_i + w_i) and reciprocal. The clamp
          // commutes out of the chain: with S_0 = W_0, S_{i+1} = RN(S_i + w+_i)
          // (w+ = w > 0 ? w : 0, and RN(S + 0) = S), W_i = min(S_i, Wmax) —
          // before saturation S_i = W_i, and once S_k >= Wmax every later
          // S >= Wmax while W stays Wmax. The serial part is one FADD per record.
          if (kProd == 2 && k > 0) {  // the weight after chunk k - 1, from the run's other producer
            const uint32_t cp = kk - 1u;
            mbar_wait(&S.wfull[pair][cp & 1u], (cp >> 1) & 1u);
            W = S.wbox[pair][cp & 1u];
          }
          const float w = u.w;
          float Wmine = W;
          if (W != Wmax) {  // W is warp-uniform (replicated scan)
            const float wp = w > 0.0f ? w : 0.0f;
            float S = W, Smine = W;
            reinterpret_cast<float*>(wscan[pair])[lane] = wp;
            __syncwarp();
            float4 wq[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) wq[q] = wscan[pair][q];
            if (__float_as_uint(W) != 0x80000000u) {
#pragma unroll
              for (int q = 0; q < 32; ++q) {  // records >= cnt carry w+ = 0: RN(S + 0) = S
                const float4 v = wq[q >> 2];
                const float wu = (q & 3) == 0 ? v.x : ((q & 3) == 1 ? v.y : ((q & 3) == 2 ? v.z : v.w));
                Smine = lane == q ? S : Smine;
                S = __fadd_rn(S, wu);
              }
            } else {  // W = -0 (imported layer): RN(-0 + 0) = +0, so skip the zero terms explicitly
#pragma unroll
              for (int q = 0; q < 32; ++q) {
                const float4 v = wq[q >> 2];
                const float wu = (q & 3) == 0 ? v.x : ((q & 3) == 1 ? v.y : ((q & 3) == 2 ? v.z : v.w));
                Smine = lane == q ? S : Smine;
                S = wu > 0.0f ? __fadd_rn(S, wu) : S;
              }
            }
            __syncwarp();
            Wmine = fminf(Smine, Wmax);
            W = fminf(S, Wmax);
          }
          // else saturated: W_i = min(RN(Wmax + w), Wmax) = Wmax for w > 0 and
          // unchanged for w <= 0, so every record sees Wmax and W stays Wmax
          if (kProd == 2) {  // hand the weight after this chunk on (every chunk arrives once: phase = kk / 2)
            if (lane == 0) S.wbox[pair][kk & 1u] = W;
            __syncwarp();
            if (lane == 0) mbar_arrive(&S.wfull[pair][kk & 1u]);
          }
          if (dbg != nullptr) {
            asm volatile("" ::"f"(W), "f"(Wmine));
            pt_scan += clock64() - tp1;
          }
          const long long tp2 = dbg != nullptr ? clock64() : 0;
          PreRec pr;
          const float clamped = u.d < -tp.truncation ? -tp.truncation : (tp.truncation < u.d ? tp.truncation : u.d);
          pr.W = Wmine;
          pr.T = __fadd_rn(Wmine, w);
          const Recip rt = make_recip(pr.T);
          pr.r1 = rt.r1;
          pr.wc = __fmul_rn(w, clamped);
          pr.c = u.c;
          pr.w = w;
          pr.d = u.d;
          pr.ok = ((w > 0.0f) & (w < 0x1p100f) & rt.ok) ? 1u : 0u;
          // chunk summary (records >= cnt do not constrain it)
          int lo0 = -1024, lo1 = -1024, lo2 = -1024, hi0 = 1024, hi1 = 1024, hi2 = 1024;
          const bool in_chunk = static_cast<uint32_t>(lane) < cnt;
          if (in_chunk && pr.ok && (u.c >> 31)) {
            const int kr = stationary_radius(w, __fmul_rn(0.499f, pr.T));
            const int n0 = static_cast<int>(u.c & 0xffu), n1 = static_cast<int>((u.c >> 8) & 0xffu),
                      n2 = static_cast<int>((u.c >> 16) & 0xffu);
            lo0 = n0 - kr;
            hi0 = n0 + kr;
            lo1 = n1 - kr;
            hi1 = n1 + kr;
            lo2 = n2 - kr;
            hi2 = n2 + kr;
          }
          ChunkHdr hd;
          hd.W_end = W;
          hd.ok = __all_sync(0xffffffffu, !in_chunk || pr.ok) ? 1u : 0u;
          // bit 1: every record pulls towards +truncation (clamped d = truncation:
          // free space in front of the surface) — the consumer's cue to try the
          // speculative walk
          hd.ok |= __all_sync(0xffffffffu, !in_chunk || clamped == tp.truncation) ? 2u : 0u;
          hd.lo[0] = __reduce_max_sync(0xffffffffu, lo0);
          hd.lo[1] = __reduce_max_sync(0xffffffffu, lo1);
          hd.lo[2] = __reduce_max_sync(0xffffffffu, lo2);
          hd.hi[0] = __reduce_min_sync(0xffffffffu, hi0);
          hd.hi[1] = __reduce_min_sync(0xffffffffu, hi1);
          hd.hi[2] = __reduce_min_sync(0xffffffffu, hi2);
          const int s = static_cast<int>(kk % kRingStages);
          if (dbg != nullptr) asm volatile("" ::"r"(hd.hi[2]), "r"(hd.lo[0]), "f"(pr.r1));
          const long long tw0 = dbg != nullptr ? clock64() : 0;
          pt_pre += tw0 - tp2;
          if (kk >= kRingStages) mbar_wait(&ring_empty[pair][s], ((kk / kRingStages) - 1) & 1u);
          const long long tw1 = dbg != nullptr ? clock64() : 0;
          pwait += tw1 - tw0;
          ring[pair][s][lane] = pr;
          if (lane == 0) ring_hdr[pair][s] = hd;
          __syncwarp();
          if (lane == 0) mbar_arrive(&ring_full[pair][s]);
          ry1 = ry2;
          ry2 = ry3;
          if (dbg != nullptr) pt_store += clock64() - tw1;
        }
        if (dbg != nullptr && lane == 0) {
          atomicAdd(&dbg[4 * n_all + 4], static_cast<unsigned long long>(pwait));
          atomicAdd(&dbg[4 * n_all + 5], static_cast<unsigned long long>(clock64() - pbusy0));
          atomicAdd(&dbg[4 * n_all + 6], static_cast<unsigned long long>(pt_weigh));
          atomicAdd(&dbg[4 * n_all + 7], static_cast<unsigned long long>(pt_scan));
          atomicAdd(&dbg[4 * n_all + 14], static_cast<unsigned long long>(pt_top));
          atomicAdd(&dbg[4 * n_all + 15], static_cast<unsigned long long>(pt_pre));
          atomicAdd(&dbg[4 * n_all + 16], static_cast<unsigned long long>(pt_store));
        }
      } else {
        VoxState st = load_vox(vp);
        unsigned long long t_start = 0, n_sat = 0, n_spec = 0, n_fail = 0, n_skip = 0;
        uint32_t spec_skip = 0u, spec_back = 0u;  // back-off after a walk left its window
        long long cwait = 0, cbusy0 = dbg != nullptr ? clock64() : 0, ct_vote = 0, ct_chain = 0, ct_spec = 0, nc_spec = 0,
                  ct_serial = 0, nc_serial = 0;
        if (dbg != nullptr) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
        // The chain's critical path is D -> candidates -> table exchange -> walk -> D. What does not depend
        // on D is taken off it: a chunk's header and this lane's record are loaded at the end of the previous
        // iteration, and whether the NEXT chunk has arrived is asked (mbar_test) before this chunk's walk and
        // read after it — the blocking wait (90 cycles even when complete) only runs when it has not.
        ChunkHdr hd;
        float4 xrec;
        {
          const int s0 = static_cast<int>(kk0 % kRingStages);
          const long long tw0 = dbg != nullptr ? clock64() : 0;
          mbar_wait(&ring_full[pair][s0], (kk0 / kRingStages) & 1u);
          if (dbg != nullptr) cwait += clock64() - tw0;
          hd = ring_hdr[pair][s0];
          xrec = reinterpret_cast<const float4*>(ring[pair][s0] + lane)[0];
        }
        for (uint32_t k = 0; k < nchunks; ++k) {
          const uint32_t kk = kk0 + k;
          const int s = static_cast<int>(kk % kRingStages);
          const int sn = static_cast<int>((kk + 1u) % kRingStages);
          const uint32_t pn = ((kk + 1u) / kRingStages) & 1u;
          const bool more = k + 1 < nchunks;
          const uint32_t next_ready = more ? mbar_test(&ring_full[pair][sn], pn) : 0u;
          const long long tc0 = dbg != nullptr ? clock64() : 0;
          const PreRec* rb = ring[pair][s];
          const uint32_t cnt = min(32u, c.len - k * 32);
          const float W_end = hd.W_end;
          // colours provably unchanged over the whole chunk? (intervals from the producer)
          const int o0 = static_cast<int>(st.cr), o1 = static_cast<int>(st.cg), o2 = static_cast<int>(st.cb);
          const bool vote = (hd.ok & 1u) != 0u && hd.lo[0] <= o0 && o0 <= hd.hi[0] && hd.lo[1] <= o1 && o1 <= hd.hi[1] &&
                            hd.lo[2] <= o2 && o2 <= hd.hi[2];
          const bool stationary = vote;  // warp-uniform
          const long long tc1 = dbg != nullptr ? clock64() : 0;
          bool done = false, spec_done = false;
          // Speculative walk. In free space every record pulls D towards
          // +truncation, where D already sits: a step moves it by 0 or +-1 ulp
          // (rounding), so over a chunk D stays within a few ulps of where it
          // started. Each lane evaluates ITS record's step — the same
          // instructions as the serial chain below — on the 7 floats D0-3ulp ..
          // D0+3ulp and publishes the results as a byte map over candidate
          // indices (7 = left the window, absorbing); the chain is then one PRMT
          // per record, composing the 32 maps in order from index 3. Exact by
          // construction; a walk that leaves the window (or a failed range
          // check) re-runs the chunk serially and backs off.
          if (stationary && cnt == 32 && (hd.ok & 2u) != 0u) {
            const uint32_t b0 = __float_as_uint(st.D);
            if (spec_skip != 0u) {
              --spec_skip;
              ++n_skip;
            } else if (b0 - 0x00800004u < 0x7e000000u) {  // D0 and its neighbours positive, normal, finite
              const float4 x = xrec;  // this lane's record: W, T, r1, wc
              const Recip rt{x.y, x.z, true};
              const uint32_t base = b0 - 3u;
              uint32_t tlo = 0u, thi = 0x07000000u;
              bool rng = true;
#pragma unroll
              for (int cnd = 0; cnd < 7; ++cnd) {
                const float a = __fadd_rn(__fmul_rn(x.x, __uint_as_float(base + cnd)), x.w);
                const float q = fast_quot0(a, rt);
                rng &= fast_range(a);
                const uint32_t code = min(__float_as_uint(q) - base, 7u);
                if (cnd < 4) tlo |= code << (8 * cnd); else thi |= code << (8 * (cnd - 4));
              }
              if (!rng) tlo = thi = 0x07070707u;
              uint2* tb = S.spec_tab[pair][kk & 1u];
              tb[lane] = make_uint2(tlo, thi);
              __syncwarp();
              const uint4* t4 = reinterpret_cast<const uint4*>(tb);
              uint32_t sel = 3u;
#pragma unroll
              for (int u = 0; u < 16; ++u) {
                const uint4 t = t4[u];
                // prmt's own selector semantics (bit 3 of a nibble = sign
                // replication) never trigger: every table byte is <= 7
                asm("prmt.b32 %0, %1, %2, %0;" : "+r"(sel) : "r"(t.x), "r"(t.y));
                asm("prmt.b32 %0, %1, %2, %0;" : "+r"(sel) : "r"(t.z), "r"(t.w));
              }
              sel &= 7u;
              if (sel != 7u) {
                st.D = __uint_as_float(base + sel);
                st.W = W_end;
                done = true;
                spec_done = true;
                n_sat += cnt;
                n_spec += cnt;
                spec_back = 0u;
              } else {
                ++n_fail;
                // a failed walk costs about a third of the serial chunk it falls
                // back to: only a streak of failures (D is on the move) backs off
                spec_back = min(spec_back + 1u, 8u);
                spec_skip = spec_back >= 3u ? 1u << (spec_back - 3u) : 0u;
              }
            }
          }
          if (done) {
          } else if (stationary) {  // distance chain only: FMUL, FADD, 3-FMA quotient per step
            float D = st.D;
            // range of |a| off the chain (two FMNMX per step): every a in
            // [2^-60, 2^60] is quot_ok; a = +-0 fails conservatively (exact re-run)
            float amin = 0x1p100f, amax = 0.0f;
            const float4* rq = reinterpret_cast<const float4*>(rb);
            constexpr int kStride = sizeof(PreRec) / sizeof(float4);
            if (cnt == 32) {
              constexpr int kAhead = 6;  // (W, T, r1, wc) loaded kAhead steps before use
              float4 buf[kAhead];
#pragma unroll
              for (int u = 0; u < kAhead; ++u) buf[u] = rq[u * kStride];
#pragma unroll
              for (int u = 0; u < 32; ++u) {
                const float4 x = buf[u % kAhead];
                if (u + kAhead < 32) buf[u % kAhead] = rq[(u + kAhead) * kStride];
                const float a = __fadd_rn(__fmul_rn(x.x, D), x.w);
                amin = fminf(amin, fabsf(a));
                amax = fmaxf(amax, fabsf(a));
                D = fast_quot0(a, Recip{x.y, x.z, true});
              }
            } else {
              for (uint32_t u = 0; u < cnt; ++u) {
                const float4 x = rq[u * kStride];
                const float a = __fadd_rn(__fmul_rn(x.x, D), x.w);
                amin = fminf(amin, fabsf(a));
                amax = fmaxf(amax, fabsf(a));
                D = fast_quot0(a, Recip{x.y, x.z, true});
              }
            }
            if (amin >= 0x1p-60f && amax <= 0x1p60f && D == D) {  // (FMNMX drops NaN: test D itself)
              st.D = D;
              st.W = W_end;
              done = true;
              n_sat += cnt;
            }
          } else {  // one chain per lane: ch = lane & 3 (distance, r, g, b), W precomputed
            const int ch = lane & 3;
            const bool colour = ch != 0;
            float qs = ch == 0 ? st.D : (ch == 1 ? st.cr : (ch == 2 ? st.cg : st.cb));
            QuotRange qr;
            float qmax = 0.0f;
            bool bad = false;
            for (uint32_t u = 0; u < cnt; ++u) {
              const PreRec& x = rb[u];
              const bool live = x.w > 0.0f;
              const bool active = !colour || (x.c >> 31) != 0u;
              const float add = ch == 0 ? x.wc : __fmul_rn(x.w, __uint2float_rn((x.c >> (colour ? 8 * ch - 8 : 0)) & 0xffu));
              const float a = __fadd_rn(__fmul_rn(x.W, qs), add);
              const float q = fast_quot0(a, Recip{x.T, x.r1, true});
              if (live & active) {
                bad |= x.ok == 0u;
                qr_add(qr, a);
                if (colour) qmax = fmaxf(qmax, q);
              }
              const float sn = colour ? fminf(round_half_away_pos(q), 255.0f) : q;
              qs = (live & active) ? sn : qs;
            }
            // q < 2^22 for colours (round_half_away_pos); NaN q fails the range check of a
            const bool ok = !bad & qr_ok(qr) & (qmax < 0x1p22f);
            if (__all_sync(0xffffffffu, ok)) {
              st.D = __shfl_sync(0xffffffffu, qs, 0);
              st.cr = __shfl_sync(0xffffffffu, qs, 1);
              st.cg = __shfl_sync(0xffffffffu, qs, 2);
              st.cb = __shfl_sync(0xffffffffu, qs, 3);
              st.W = W_end;
              done = true;
            }
          }
          if (!done) {  // rare: exact re-run of the chunk from its start state
            for (uint32_t u = 0; u < cnt; ++u)
              step_exact(st.D, st.W, st.cr, st.cg, st.cb, rb[u].d, rb[u].w, rb[u].c, tp.truncation, Wmax);
          }
          if (dbg != nullptr) {
            asm volatile("" ::"f"(st.D));
            const long long tc2 = clock64();
            ct_chain += tc2 - tc1;
            ct_vote += tc1 - tc0;
            if (spec_done) {
              ct_spec += tc2 - tc1;
              ++nc_spec;
            } else {
              ct_serial += tc2 - tc1;
              ++nc_serial;
            }
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&ring_empty[pair][s]);
          if (more) {  // the next chunk's header and this lane's record of it
            if (!next_ready) {
              const long long tw0 = dbg != nullptr ? clock64() : 0;
              mbar_wait(&ring_full[pair][sn], pn);
              if (dbg != nullptr) cwait += clock64() - tw0;
            }
            hd = ring_hdr[pair][sn];
            xrec = reinterpret_cast<const float4*>(ring[pair][sn] + lane)[0];
          }
        }
        if (dbg != nullptr && lane == 0) {
          atomicAdd(&dbg[4 * n_all + 2], static_cast<unsigned long long>(cwait));
          atomicAdd(&dbg[4 * n_all + 3], static_cast<unsigned long long>(clock64() - cbusy0));
          atomicAdd(&dbg[4 * n_all + 8], static_cast<unsigned long long>(ct_vote));
          atomicAdd(&dbg[4 * n_all + 9], static_cast<unsigned long long>(ct_chain));
          atomicAdd(&dbg[4 * n_all + 10], static_cast<unsigned long long>(ct_spec));
          atomicAdd(&dbg[4 * n_all + 11], static_cast<unsigned long long>(nc_spec));
          atomicAdd(&dbg[4 * n_all + 12], static_cast<unsigned long long>(ct_serial));
          atomicAdd(&dbg[4 * n_all + 13], static_cast<unsigned long long>(nc_serial));
        }
        if (lane == 0) {
          store_vox(vp, st);
          if (touched != nullptr) touched[c.key / static_cast<uint32_t>(map.nvox)] = 1u;
          if (dbg != nullptr) {
            unsigned long long t_end;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
            dbg[4 * r + 0] = t_start;
            dbg[4 * r + 1] = t_end;
            dbg[4 * r + 2] = c.len | (min(n_fail, 0xFFFFull) << 32) | (min(n_skip, 0xFFFFull) << 48);
            dbg[4 * r + 3] = n_sat | (n_spec << 32);
          }
        }
      }
      kk0 += nchunks;
    }
  }

  if (dbg != nullptr && lane == 0) {  // when this warp ran out of work
    unsigned long long t_end;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
    atomicMax(&dbg[4 * nruns], t_end);
    atomicMin(&dbg[4 * nruns + 1], t_end);
  }
}

// Long runs alone: kP pairs per CTA (64 kP threads), one CTA per SM; the
// short-run grid (k_fold_short) is its programmatic dependent.
template <int kP, bool kSep, bool kSmemOrg>
__global__ void __launch_bounds__(64 * kP, 1) k_fold_runs(
    const uint32_t* __restrict__ num_runs_p, const uint32_t* __restrict__ order,
    const uint32_t* __restrict__ sorted_len, const uint32_t* __restrict__ ukeys, const uint32_t* __restrict__ ustart,
    const uint32_t* __restrict__ ulen, const uint32_t* __restrict__ svals, const FoldRay* __restrict__ rays, const uint2* __restrict__ far,
    const float* __restrict__ g_org, uint32_t F, MapView map, TsdfParams tp, uint8_t* __restrict__ touched,
    uint32_t* __restrict__ work, unsigned long long* __restrict__ dbg) {
  __shared__ LongSmem<kP> S;
  __shared__ float s_org[3 * kOrgCache];
  const float* poses = stage_origins<kSmemOrg>(s_org, g_org, F);
  asm volatile("griddepcontrol.launch_dependents;");  // k_fold_short may start once every CTA is here
  // (no check of map.counters here: the host launches a fold only after its
  // records' emission succeeded, and a later batch's emission may already be
  // setting flags while this fold waits for its turn)
  long_smem_init(S);
  __syncthreads();
  const uint32_t nruns = *num_runs_p;
  uint32_t n_long = 0;
  if ((threadIdx.x & 31) == 0) n_long = count_long_runs(sorted_len, nruns, tp.long_code);
  n_long = __shfl_sync(0xffffffffu, n_long, 0);
  fold_long_pairs<kP, kSep>(S, static_cast<int>(threadIdx.x >> 5), poses, nruns, n_long, order, ukeys, ustart, ulen,
                            svals, rays, far, map, tp, touched, work, dbg);
}

// Short runs (< kLongRun records): one thread per run, launched on a second
// stream next to k_fold_runs (disjoint voxels), with its own register budget
// so more warps hide the ray-id -> ray gather latency.
template <int kC>
__device__ __forceinline__ void fold_short_loop(
    const float* poses, const uint32_t nruns, const uint32_t n_long, const uint32_t* __restrict__ order,
    const uint32_t* __restrict__ ukeys, const uint32_t* __restrict__ ustart, const uint32_t* __restrict__ ulen,
    const uint32_t* __restrict__ svals, const FoldRay* __restrict__ rays, const uint2* __restrict__ far, const MapView& map, const TsdfParams& tp,
    uint8_t* __restrict__ touched, uint32_t* __restrict__ work) {
  const int lane = threadIdx.x & 31;
  while (true) {
    uint32_t base = 0;
    if (lane == 0) base = atomicAdd(&work[1], 32u);
    base = __shfl_sync(0xffffffffu, base, 0);
    if (n_long + base >= nruns) break;
    const uint32_t r = n_long + base + lane;
    // The warp's 32 runs walk in lockstep to the longest of them (runs of one
    // length code, at most 12.5 % apart: the fold order), so the lanes can
    // vote: runs are neighbouring voxels (key order inside a code), and in free
    // space ALL their records are far — then nobody weighs (no projective
    // distance, no square root: most of a record's instructions). A lane
    // without a run (grid tail, skipped candidates) walks an empty one.
    RunCtx c{kInvalidRecord, 0u, 0u, 0.0f, 0.0f, 0.0f};
    if (r < nruns) c = run_ctx(map, tp, ukeys, ustart, ulen, order[r]);
    const bool act = c.key != kInvalidRecord;
    if (!act) c.start = c.len = 0u;
    vxg_voxel* vp = map.slab + (act ? c.key : 0u);
    VoxState st{};
    if (act) st = load_vox(vp);
    // software pipeline over chunks of kC records: rays gathered two chunks
    // ahead, weighed one chunk ahead of their fold steps. Positions past the
    // run re-read its last record (an empty run: record 0 of the batch) and
    // carry w = 0 (a no-op step), so the loop body has no per-record guards.
    const uint32_t* ids = svals + c.start;
    const uint32_t last = c.len ? c.len - 1u : 0u;
    const uint32_t wlen = __reduce_max_sync(0xffffffffu, c.len);
    FoldIn rn[kC];
    Upd xn[kC], xs[kC];
    auto weigh_chunk = [&](uint32_t idx0, const FoldIn* ry, Upd* x) {  // all 32 lanes call
#pragma unroll
      for (int u = 0; u < kC; ++u) {  // one vote per record position of the chunk
        const bool in = idx0 + u < c.len;
        if (__all_sync(0xffffffffu, ry[u].fr.x != 0xFFFFFFFFu || !in)) {
          x[u].d = tp.truncation;
          x[u].w = in ? __uint_as_float(ry[u].fr.x) : 0.0f;
          x[u].c = ry[u].fr.y;
          x[u].pad = 0u;
        } else {
          x[u] = weigh_in(ry[u], poses, c.x0, c.x1, c.x2, tp);
          x[u].w = in ? x[u].w : 0.0f;
        }
      }
    };
    // Gathers run ahead of their use: a far record's 8-byte FarRay two chunks
    // ahead (most records, and the only gather of an all-far warp: an L2 / DRAM
    // round trip is longer than one chunk's work), a near record's 32-byte ray
    // one chunk ahead (it would cost 8 more registers per chunk position), the
    // ids one chunk ahead of the first gather that needs them.
    auto far_part = [&](uint32_t v) {
      return (v & kFarRecord) ? far[v & kRayMask] : make_uint2(0xFFFFFFFFu, 0u);
    };
    auto near_part = [&](uint32_t v) { return (v & kFarRecord) ? FoldRay{} : rays[v & kRayMask]; };
    uint32_t idq[kC], idn[kC];  // ids of chunk c+3 (far part in flight) and c+4
    uint2 fq[kC];               // far parts of chunk c+3
#pragma unroll
    for (int u = 0; u < kC; ++u) rn[u] = load_fold_in(rays, far, ids[min(static_cast<uint32_t>(u), last)]);
    weigh_chunk(0u, rn, xn);
#pragma unroll
    for (int u = 0; u < kC; ++u) rn[u] = load_fold_in(rays, far, ids[min(static_cast<uint32_t>(kC + u), last)]);
#pragma unroll
    for (int u = 0; u < kC; ++u) {
      idq[u] = ids[min(static_cast<uint32_t>(2 * kC + u), last)];
      fq[u] = far_part(idq[u]);
      idn[u] = ids[min(static_cast<uint32_t>(3 * kC + u), last)];
    }
    for (uint32_t j = 0; j < wlen; j += kC) {
#pragma unroll
      for (int u = 0; u < kC; ++u) xs[u] = xn[u];
      // weigh chunk j+kC; complete chunk j+2kC (its far parts were loaded last
      // iteration, its near rays now); far parts of chunk j+3kC; ids of j+4kC
      weigh_chunk(j + kC, rn, xn);
#pragma unroll
      for (int u = 0; u < kC; ++u) {
        rn[u].ry = near_part(idq[u]);
        rn[u].fr = fq[u];
      }
#pragma unroll
      for (int u = 0; u < kC; ++u) {
        idq[u] = idn[u];
        fq[u] = far_part(idq[u]);
        idn[u] = ids[min(j + 4 * kC + u, last)];
      }
      const VoxState s0 = st;
      bool ok = true;
#pragma unroll
      for (int u = 0; u < kC; ++u)
        step_fast_skip(st.D, st.W, st.cr, st.cg, st.cb, xs[u].d, xs[u].w, xs[u].c, tp.truncation, tp.max_weight, ok);
      if (!ok) {  // rare: exact re-run of the chunk from its start state
        st = s0;
        for (int u = 0; u < kC; ++u)
          step_exact(st.D, st.W, st.cr, st.cg, st.cb, xs[u].d, xs[u].w, xs[u].c, tp.truncation, tp.max_weight);
      }
    }
    if (act) {
      store_vox(vp, st);
      if (touched != nullptr) touched[c.key / static_cast<uint32_t>(map.nvox)] = 1u;
    }
  }
}

// Short runs, launched behind k_fold_runs in the same stream as a programmatic
// dependent (PDL): it starts once every long-run CTA is resident (each triggers
// at entry), so the persistent short-run CTAs never delay the longest chains;
// it completes only after k_fold_runs (griddepcontrol.wait on the way out).
template <int kMinBlocks, int kC, bool kSmemOrg>
__global__ void __launch_bounds__(256, kMinBlocks) k_fold_short(
    const uint32_t* __restrict__ num_runs_p, const uint32_t* __restrict__ order,
    const uint32_t* __restrict__ sorted_len, const uint32_t* __restrict__ ukeys, const uint32_t* __restrict__ ustart,
    const uint32_t* __restrict__ ulen, const uint32_t* __restrict__ svals, const FoldRay* __restrict__ rays, const uint2* __restrict__ far,
    const float* __restrict__ g_org, uint32_t F, MapView map, TsdfParams tp, uint8_t* __restrict__ touched,
    uint32_t* __restrict__ work) {
  __shared__ float s_org[3 * kOrgCache];
  const float* poses = stage_origins<kSmemOrg>(s_org, g_org, F);
  {
    const uint32_t nruns = *num_runs_p;
    uint32_t n_long = 0;
    if ((threadIdx.x & 31) == 0) n_long = count_long_runs(sorted_len, nruns, tp.long_code);
    n_long = __shfl_sync(0xffffffffu, n_long, 0);
    fold_short_loop<kC>(poses, nruns, n_long, order, ukeys, ustart, ulen, svals, rays, far, map, tp, touched, work);
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

// Long and short runs in ONE persistent grid, one 512-thread CTA per SM.
// kProd = 1: warps 8..15 are four long-run producer/consumer pairs, warps 0..7
// fold short runs from the start. kProd = 2: warps 4..15 are four teams of
// TWO producers and a consumer (a run's producers take alternate chunks and
// hand the running weight to each other), warps 0..3 fold short runs — the
// consumer, not the producer, then bounds a chain (faster chains, fewer
// short-run warps beside them: the host picks it for small folds, where the
// longest chain is the whole fold). Consumers are the highest warp ids, one per
// sub-partition, so the arbiter favours the serial chains; every team warp
// joins the short runs once the long runs are handed out.
// VXG_FOLD_MAXREG (dev A/B): cap the fold's registers so that the next batch's
// bundling kernels find room beside the persistent fold CTAs.
#ifdef VXG_FOLD_MAXREG
#define VXG_FOLD_BOUNDS __maxnreg__(VXG_FOLD_MAXREG)
#else
#define VXG_FOLD_BOUNDS __launch_bounds__(512, 1)
#endif
template <bool kSmemOrg, int kC = 2, int kProd = 1, bool kDbg = false>
__global__ void VXG_FOLD_BOUNDS k_fold_all(
    const uint32_t* __restrict__ num_runs_p, const uint32_t* __restrict__ order,
    const uint32_t* __restrict__ sorted_len, const uint32_t* __restrict__ ukeys, const uint32_t* __restrict__ ustart,
    const uint32_t* __restrict__ ulen, const uint32_t* __restrict__ svals, const FoldRay* __restrict__ rays, const uint2* __restrict__ far,
    const float* __restrict__ g_org, uint32_t F, MapView map, TsdfParams tp, uint8_t* __restrict__ touched,
    uint32_t* __restrict__ work, unsigned long long* __restrict__ dbg) {
  __shared__ LongSmem<4> S;
  __shared__ float s_org[3 * kOrgCache];
  const float* poses = stage_origins<kSmemOrg>(s_org, g_org, F);
  long_smem_init(S);
  __syncthreads();
  const uint32_t nruns = *num_runs_p;
  uint32_t n_long = 0;
  if ((threadIdx.x & 31) == 0) n_long = count_long_runs(sorted_len, nruns, tp.long_code);
  n_long = __shfl_sync(0xffffffffu, n_long, 0);
  const int wid = static_cast<int>(threadIdx.x >> 5);
  constexpr int kShortWarps = 16 - 4 * (1 + kProd);  // 8 beside pairs, 4 beside two-producer teams
  if (wid >= kShortWarps)
    fold_long_pairs<4, false, kProd, kDbg>(S, wid - kShortWarps, poses, nruns, n_long, order, ukeys, ustart, ulen,
                                           svals, rays, far, map, tp, touched, work, dbg);
  fold_short_loop<kC>(poses, nruns, n_long, order, ukeys, ustart, ulen, svals, rays, far, map, tp, touched, work);
}

// Self-tests of the fast fold arithmetic against the reference-order path.
__global__ void k_selftest_div(uint64_t n, uint64_t seed, unsigned long long* __restrict__ mismatches,
                               float* __restrict__ example) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t h1 = mix64(seed ^ (i * 0x9e3779b97f4a7c15ULL)), h2 = mix64(h1 + 0x632be59bd9b4e019ULL);
    // random sign/mantissa, exponents spanning [-70, 70] (includes out-of-range -> fallback)
    const uint32_t ea = 127 + static_cast<int>((h1 >> 32) % 141) - 70, eb = 127 + static_cast<int>((h2 >> 32) % 141) - 70;
    const float a = __uint_as_float((static_cast<uint32_t>(h1 >> 63) << 31) | (ea << 23) | (static_cast<uint32_t>(h1) & 0x7fffff));
    const float b = __uint_as_float((eb << 23) | (static_cast<uint32_t>(h2) & 0x7fffff));
    const Recip r = make_recip(b);
    const float q = div_by(a, r);
    const float ref = __fdiv_rn(a, b);
    if (__float_as_uint(q) != __float_as_uint(ref)) {
      if (atomicAdd(mismatches, 1ull) == 0ull) {
        example[0] = a;
        example[1] = b;
      }
    }
  }
}

__global__ void k_selftest_fold(uint64_t n_seq, uint32_t len, uint64_t seed, float trunc, float wmax,
                                unsigned long long* __restrict__ mismatches) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n_seq;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    float D0 = 0.f, W0 = 0.f, D1 = 0.f, W1 = 0.f, cr = 0.f, cg = 0.f, cb = 0.f;
    uint32_t rgb = 0u;
    uint64_t h = mix64(seed + i);
    const float wscale = (h & 1) ? 0.01f : 50.0f;
    for (uint32_t k = 0; k < len; ++k) {
      h = mix64(h + k + 1);
      const float d = (static_cast<float>(h & 0xffffff) / 16777216.0f - 0.5f) * 4.0f * trunc;
      const float w = (static_cast<float>((h >> 24) & 0xffffff) / 16777216.0f) * wscale + 1e-6f;
      const uint32_t col = static_cast<uint32_t>((h >> 40) & 0xffffffu) | (((h >> 12) & 3u) ? 0x80000000u : 0u);
      update_voxel(D0, W0, rgb, d, w, col, (col >> 31) != 0u, trunc, wmax);
      update_voxel_fast(D1, W1, cr, cg, cb, d, w, col, trunc, wmax);
      const uint32_t rgb1 = static_cast<uint32_t>(cr) | (static_cast<uint32_t>(cg) << 8) | (static_cast<uint32_t>(cb) << 16);
      if (__float_as_uint(D0) != __float_as_uint(D1) || __float_as_uint(W0) != __float_as_uint(W1) || rgb != rgb1) {
        atomicAdd(mismatches, 1ull);
        break;
      }
    }
  }
}

__global__ void k_add_u64(uint32_t n, unsigned long long* __restrict__ dst, const unsigned long long* __restrict__ src) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) dst[i] += src[i];
}

// Pipeline chunk bounds: out[c] = first ray of chunk c (c <= n, out[n] = R),
// out[n + 1 + c] = its first record; chunk c starts at the first ray whose
// record offset reaches c * total / n.
__global__ void k_chunk_bounds(uint32_t R, const unsigned long long* __restrict__ roff, unsigned long long total,
                               uint32_t n, unsigned long long* __restrict__ out) {
  for (uint32_t c = threadIdx.x; c <= n; c += blockDim.x) {
    const unsigned long long target = total / n * c + (total % n) * c / n;
    uint32_t lo = 0, hi = R;  // smallest r with roff(r) >= target, roff(R) = total
    while (lo < hi) {
      const uint32_t mid = lo + (hi - lo) / 2;
      if (roff[mid] >= target) hi = mid; else lo = mid + 1;
    }
    if (c == n) lo = R;
    out[c] = lo;
    out[n + 1 + c] = lo < R ? roff[lo] : total;
  }
}

// Emission order key of ray r: chunk first (descending sort puts chunk 0
// first), then the record count (longest first inside a chunk).
__global__ void k_chunk_keys(uint32_t R, const unsigned long long* __restrict__ rcount,
                             const unsigned long long* __restrict__ bounds, uint32_t n,
                             unsigned long long* __restrict__ keys) {
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < R; r += gridDim.x * blockDim.x) {
    uint32_t lo = 0, hi = n - 1;  // largest c with bounds[c] <= r
    while (lo < hi) {
      const uint32_t mid = (lo + hi + 1) / 2;
      if (bounds[mid] <= r) lo = mid; else hi = mid - 1;
    }
    keys[r] = (static_cast<unsigned long long>(n - 1 - lo) << 16) | min(rcount[r], 65535ull);
  }
}

__global__ void k_iota(uint32_t n, uint32_t* __restrict__ out) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = i;
}

// ---------------------------------------------------------------- map maintenance
__global__ void k_fix_block_idx(uint64_t hcap, const unsigned long long* __restrict__ hkeys,
                                const int32_t* __restrict__ hvals, uint32_t lo, uint32_t hi,
                                int32_t* __restrict__ block_idx) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < hcap;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t k = hkeys[i];
    const int32_t s = hvals[i];
    if (k == kEmptyKey || s < 0) continue;
    if (static_cast<uint32_t>(s) >= lo && static_cast<uint32_t>(s) < hi) {
      int b[3];
      unpack_block(k, b);
      block_idx[3 * s + 0] = b[0];
      block_idx[3 * s + 1] = b[1];
      block_idx[3 * s + 2] = b[2];
    }
  }
}

__global__ void k_rehash(uint64_t old_cap, const unsigned long long* __restrict__ okeys,
                         const int32_t* __restrict__ ovals, MapView map) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < old_cap;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const unsigned long long k = okeys[i];
    if (k == kEmptyKey) continue;
    uint64_t j = mix64(k) & map.hmask;
    while (true) {
      const unsigned long long prev = atomicCAS(&map.hkeys[j], kEmptyKey, k);
      if (prev == kEmptyKey) {
        map.hvals[j] = ovals[i];
        break;
      }
      j = (j + 1) & map.hmask;
    }
  }
}

__global__ void k_import_slots(uint64_t n, const int32_t* __restrict__ idx, MapView map, int32_t* __restrict__ slots) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const int b0 = idx[3 * i], b1 = idx[3 * i + 1], b2 = idx[3 * i + 2];
    if (!block_in_range(b0, b1, b2)) {
      atomicOr(&map.counters[1], static_cast<uint32_t>(kErrKeyRange));
      slots[i] = -1;
      continue;
    }
    slots[i] = map.find_or_insert(pack_block(b0, b1, b2), b0, b1, b2);
  }
}

__global__ void k_scatter_blocks(uint64_t n, const int32_t* __restrict__ slots, const vxg_voxel* __restrict__ src,
                                 MapView map) {
  const uint64_t nv = static_cast<uint64_t>(map.nvox);
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n * nv;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t b = i / nv;
    const int32_t s = slots[b];
    if (s < 0) continue;
    map.slab[static_cast<uint64_t>(s) * nv + (i - b * nv)] = src[i];
  }
}

// Export: blocks slots[0..n) gathered into one contiguous AoS buffer (the
// VXBLX payload order), pad bytes zeroed; 4-byte words, coalesced both ways.
__global__ void k_gather_blocks(uint64_t n, const uint32_t* __restrict__ slots, const vxg_voxel* __restrict__ slab,
                                uint32_t nvox, vxg_voxel* __restrict__ dst) {
  const uint64_t wpb = 3ull * nvox;  // 4-byte words per block
  const uint32_t* src = reinterpret_cast<const uint32_t*>(slab);
  uint32_t* out = reinterpret_cast<uint32_t*>(dst);
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n * wpb;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t b = i / wpb, w = i - b * wpb;
    const uint32_t sl = slots[b];
    uint32_t v = sl == 0xFFFFFFFFu ? 0u : __ldg(src + static_cast<uint64_t>(sl) * wpb + w);  // absent: zeros
    if (w % 3 == 2) v &= 0x00FFFFFFu;  // r, g, b, pad=0
    out[i] = v;
  }
}

// Layer::block_ptr (layer.h:89-97) for n block indices: slot, or ~0u when absent.
__global__ void k_block_slots(uint64_t n, const int32_t* __restrict__ idx, MapView map, uint32_t* __restrict__ slots) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const int b0 = idx[3 * i], b1 = idx[3 * i + 1], b2 = idx[3 * i + 2];
    int32_t s = -1;
    if (block_in_range(b0, b1, b2)) s = map.find(pack_block(b0, b1, b2));
    slots[i] = (s < 0 || static_cast<uint32_t>(s) >= map.cap_blocks) ? 0xFFFFFFFFu : static_cast<uint32_t>(s);
  }
}

__global__ void k_query(uint64_t n, const int32_t* __restrict__ g, MapView map, vxg_voxel* __restrict__ out,
                        uint8_t* __restrict__ found) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    int b[3], l[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      b[a] = floor_div(g[3 * i + a], map.vps);
      l[a] = g[3 * i + a] - b[a] * map.vps;
    }
    int32_t s = -1;
    if (block_in_range(b[0], b[1], b[2])) s = map.find(pack_block(b[0], b[1], b[2]));
    if (s < 0 || static_cast<uint32_t>(s) >= map.cap_blocks) {
      found[i] = 0u;
      out[i] = vxg_voxel{0.0f, 0.0f, 0, 0, 0, 0};
    } else {
      found[i] = 1u;
      out[i] = map.slab[static_cast<uint64_t>(s) * map.nvox + l[0] + map.vps * (l[1] + map.vps * l[2])];
    }
  }
}

// interpolate_distance (interpolation.h:28-60): trilinear over the 8 voxel
// centres around p, absent when any corner is unallocated or unobserved
// (weight <= kTsdfObservedWeight, voxel.h:17). One thread per point; the 8
// corners share at most 8 blocks, looked up through the device hash.
__device__ __forceinline__ bool corner_distance(const MapView& map, int gx, int gy, int gz, float* d) {
  const int b0 = floor_div(gx, map.vps), b1 = floor_div(gy, map.vps), b2 = floor_div(gz, map.vps);
  if (!block_in_range(b0, b1, b2)) return false;
  const int32_t s = map.find(pack_block(b0, b1, b2));
  if (s < 0 || static_cast<uint32_t>(s) >= map.cap_blocks) return false;
  const vxg_voxel& v = map.slab[static_cast<uint64_t>(s) * map.nvox + (gx - b0 * map.vps) +
                               map.vps * ((gy - b1 * map.vps) + map.vps * (gz - b2 * map.vps))];
  if (!(v.weight > 1e-4f)) return false;
  *d = v.distance;
  return true;
}

// interpolate_distance at one point; false when absent.
__device__ __forceinline__ bool interp_distance(const MapView& map, float voxel_size, const float* p, float* out) {
  float q[3], frac[3];
  int base[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {  // q = p / v - 0.5 (Eigen: per-component quotient, then difference)
    q[a] = fsub(fdiv(p[a], voxel_size), 0.5f);
    base[a] = static_cast<int>(floorf(q[a]));
    frac[a] = fsub(q[a], static_cast<float>(base[a]));
  }
  float c[2][2][2];
  bool ok = true;
#pragma unroll
  for (int dz = 0; dz < 2; ++dz)
#pragma unroll
    for (int dy = 0; dy < 2; ++dy)
#pragma unroll
      for (int dx = 0; dx < 2; ++dx)
        ok = ok && corner_distance(map, base[0] + dx, base[1] + dy, base[2] + dz, &c[dx][dy][dz]);
  if (!ok) return false;
  float plane[2][2], line[2];
#pragma unroll
  for (int dy = 0; dy < 2; ++dy)
#pragma unroll
    for (int dz = 0; dz < 2; ++dz) plane[dy][dz] = fadd(c[0][dy][dz], fmul(frac[0], fsub(c[1][dy][dz], c[0][dy][dz])));
#pragma unroll
  for (int dz = 0; dz < 2; ++dz) line[dz] = fadd(plane[0][dz], fmul(frac[1], fsub(plane[1][dz], plane[0][dz])));
  *out = fadd(line[0], fmul(frac[2], fsub(line[1], line[0])));
  return true;
}

__global__ void k_interpolate(uint64_t n, const float* __restrict__ pts, MapView map, float voxel_size,
                              float* __restrict__ out, uint8_t* __restrict__ found) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    float r = 0.0f;
    const bool ok = interp_distance(map, voxel_size, pts + 3 * i, &r);
    out[i] = ok ? r : 0.0f;
    found[i] = ok ? 1u : 0u;
  }
}

// ---------------------------------------------------------------- meshing (MeshExtractor)
// Marching cubes per block (mesh_extractor.cpp:85-151) on the slab. One thread
// per cube of the requested blocks (cube = voxel (x, y, z) of the block and its
// +1 neighbours, which may lie in adjacent blocks). Pass 1 counts each cube's
// triangles; an exclusive scan over (block, cube) in the reference's loop
// order (z, y, x) gives every cube its output position; pass 2 writes the
// triangles. The case tables come from the caller (vxg_mc_tables) and are
// staged in shared memory.
struct McSmem {
  int32_t coff[8][3];
  int32_t ecorner[12][2];
  uint16_t edge[256];
  int8_t tri[256][16];
  uint8_t ntri[256];
};

__device__ __forceinline__ void mc_stage(McSmem& sm, const vxg_mc_tables* __restrict__ t) {
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    sm.edge[i] = t->edge_table[i];
    int n = 0;
    for (int k = 0; k < 16; ++k) {
      sm.tri[i][k] = t->tri_table[i][k];
    }
    while (n < 16 && t->tri_table[i][n] != -1) ++n;
    sm.ntri[i] = static_cast<uint8_t>(n / 3);
  }
  if (threadIdx.x < 24) sm.coff[threadIdx.x / 3][threadIdx.x % 3] = t->corner_offsets[threadIdx.x / 3][threadIdx.x % 3];
  if (threadIdx.x < 24) sm.ecorner[threadIdx.x / 2][threadIdx.x % 2] = t->edge_corners[threadIdx.x / 2][threadIdx.x % 2];
  __syncthreads();
}

// Layer::voxel_ptr + observed() for a voxel of the cube; the cube's own block
// is `slot` (the common case), others go through the block hash.
__device__ __forceinline__ const vxg_voxel* mc_voxel(const MapView& map, int32_t slot, int bx, int by, int bz, int gx,
                                                     int gy, int gz) {
  const int vps = map.vps;
  const int b0 = floor_div(gx, vps), b1 = floor_div(gy, vps), b2 = floor_div(gz, vps);
  int32_t s = slot;
  if (b0 != bx || b1 != by || b2 != bz) {
    if (!block_in_range(b0, b1, b2)) return nullptr;
    s = map.find(pack_block(b0, b1, b2));
    if (s < 0 || static_cast<uint32_t>(s) >= map.cap_blocks) return nullptr;
  }
  const vxg_voxel* v = &map.slab[static_cast<uint64_t>(s) * map.nvox + (gx - b0 * vps) +
                                 vps * ((gy - b1 * vps) + vps * (gz - b2 * vps))];
  return v->weight > 1e-4f ? v : nullptr;  // TsdfVoxel::observed (voxel.h:17)
}

struct McCube {
  int g[8][3];
  float d[8];
  uint8_t rgb[8][3];
  int config;
};

// Corners of cube (x, y, z) of block slot; false when a corner is missing or
// unobserved (mesh_extractor.cpp:96-108).
__device__ __forceinline__ bool mc_cube(const MapView& map, const McSmem& sm, int32_t slot, const int* bidx, int lin,
                                        McCube& c) {
  const int vps = map.vps;
  const int x = lin % vps, y = (lin / vps) % vps, z = lin / (vps * vps);
  c.config = 0;
  for (int k = 0; k < 8; ++k) {
    const int gx = bidx[0] * vps + x + sm.coff[k][0], gy = bidx[1] * vps + y + sm.coff[k][1],
              gz = bidx[2] * vps + z + sm.coff[k][2];
    const vxg_voxel* v = mc_voxel(map, slot, bidx[0], bidx[1], bidx[2], gx, gy, gz);
    if (v == nullptr) return false;
    c.g[k][0] = gx;
    c.g[k][1] = gy;
    c.g[k][2] = gz;
    c.d[k] = v->distance;
    c.rgb[k][0] = v->r;
    c.rgb[k][1] = v->g;
    c.rgb[k][2] = v->b;
    if (v->distance < 0.0f) c.config |= 1 << k;
  }
  return true;
}

__global__ void k_mc_count(uint64_t n_cubes, const int32_t* __restrict__ slots, MapView map,
                           const vxg_mc_tables* __restrict__ tables, uint32_t* __restrict__ ntri) {
  __shared__ McSmem sm;
  mc_stage(sm, tables);
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n_cubes;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t b = i / static_cast<uint64_t>(map.nvox);
    const int lin = static_cast<int>(i - b * static_cast<uint64_t>(map.nvox));
    const int32_t slot = slots[b];
    const int bidx[3] = {map.block_idx[3 * slot], map.block_idx[3 * slot + 1], map.block_idx[3 * slot + 2]};
    McCube c;
    uint32_t n = 0;
    if (mc_cube(map, sm, slot, bidx, lin, c) && sm.edge[c.config] != 0) n = sm.ntri[c.config];
    ntri[i] = n;
  }
}

__global__ void k_gather_stride(uint64_t n, const uint32_t* __restrict__ src, uint64_t stride, uint32_t* __restrict__ dst) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    dst[i] = src[i * stride];
}

// vertex_normal (mesh_extractor.cpp:69-83): central differences of
// interpolate_distance at +-h per axis; the face normal when any sample is
// absent or the gradient vanishes.
__device__ __forceinline__ void mc_vertex_normal(const MapView& map, float v, const float* p, const float* face,
                                                 float* out) {
  float grad[3];
  for (int i = 0; i < 3; ++i) {
    float lo[3] = {p[0], p[1], p[2]}, hi[3] = {p[0], p[1], p[2]};
    lo[i] = fsub(lo[i], v);
    hi[i] = fadd(hi[i], v);
    float dlo, dhi;
    if (!interp_distance(map, v, lo, &dlo) || !interp_distance(map, v, hi, &dhi)) {
      out[0] = face[0];
      out[1] = face[1];
      out[2] = face[2];
      return;
    }
    grad[i] = fdiv(fsub(dhi, dlo), fmul(2.0f, v));
  }
  const float norm = __fsqrt_rn(fadd(fmul(grad[0], grad[0]), fadd(fmul(grad[1], grad[1]), fmul(grad[2], grad[2]))));
  if (norm < 1e-10f) {
    out[0] = face[0];
    out[1] = face[1];
    out[2] = face[2];
    return;
  }
  out[0] = fdiv(grad[0], norm);
  out[1] = fdiv(grad[1], norm);
  out[2] = fdiv(grad[2], norm);
}

__global__ void k_mc_emit(uint64_t n_cubes, const int32_t* __restrict__ slots, MapView map, float voxel_size,
                          const vxg_mc_tables* __restrict__ tables, const uint32_t* __restrict__ ntri,
                          const uint32_t* __restrict__ tri_off, int with_colors, float* __restrict__ verts,
                          float* __restrict__ normals, uint8_t* __restrict__ colors) {
  __shared__ McSmem sm;
  mc_stage(sm, tables);
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n_cubes;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    if (ntri[i] == 0u) continue;
    const uint64_t b = i / static_cast<uint64_t>(map.nvox);
    const int lin = static_cast<int>(i - b * static_cast<uint64_t>(map.nvox));
    const int32_t slot = slots[b];
    const int bidx[3] = {map.block_idx[3 * slot], map.block_idx[3 * slot + 1], map.block_idx[3 * slot + 2]};
    McCube c;
    mc_cube(map, sm, slot, bidx, lin, c);
    // edge vertices (edge_vertex, mesh_extractor.cpp:21-39): from the corner
    // with the lower (x, y, z) global index
    float ep[12][3];
    uint8_t ec[12][3];
    const uint16_t emask = sm.edge[c.config];
    for (int e = 0; e < 12; ++e) {
      if (!(emask & (1u << e))) continue;
      int lo = sm.ecorner[e][0], hi = sm.ecorner[e][1];
      const int* A = c.g[lo];
      const int* B = c.g[hi];
      const bool swap = B[0] != A[0] ? B[0] < A[0] : (B[1] != A[1] ? B[1] < A[1] : B[2] < A[2]);
      if (swap) {
        const int t = lo;
        lo = hi;
        hi = t;
      }
      const float t = fdiv(c.d[lo], fsub(c.d[lo], c.d[hi]));
      for (int a = 0; a < 3; ++a) {
        const float plo = vcenter(c.g[lo][a], voxel_size), phi = vcenter(c.g[hi][a], voxel_size);
        ep[e][a] = fadd(plo, fmul(t, fsub(phi, plo)));
        const float clo = static_cast<float>(c.rgb[lo][a]);
        const long r = lroundf(fadd(clo, fmul(t, fsub(static_cast<float>(c.rgb[hi][a]), clo))));
        ec[e][a] = static_cast<uint8_t>(r < 0 ? 0 : (r > 255 ? 255 : r));
      }
    }
    uint64_t o = tri_off[i];
    const int8_t* tt = sm.tri[c.config];
    for (int t = 0; t < 16 && tt[t] != -1; t += 3, ++o) {
      // the table winding faces the negative side: (e0, e2, e1) (:117-122)
      const int es[3] = {tt[t], tt[t + 2], tt[t + 1]};
      const float* p0 = ep[es[0]];
      const float* p1 = ep[es[1]];
      const float* p2 = ep[es[2]];
      const float u[3] = {fsub(p1[0], p0[0]), fsub(p1[1], p0[1]), fsub(p1[2], p0[2])};
      const float w[3] = {fsub(p2[0], p0[0]), fsub(p2[1], p0[1]), fsub(p2[2], p0[2])};
      float fnv[3] = {fsub(fmul(u[1], w[2]), fmul(u[2], w[1])), fsub(fmul(u[2], w[0]), fmul(u[0], w[2])),
                      fsub(fmul(u[0], w[1]), fmul(u[1], w[0]))};
      const float fn = __fsqrt_rn(fadd(fmul(fnv[0], fnv[0]), fadd(fmul(fnv[1], fnv[1]), fmul(fnv[2], fnv[2]))));
      if (fn > 1e-12f) {
        fnv[0] = fdiv(fnv[0], fn);
        fnv[1] = fdiv(fnv[1], fn);
        fnv[2] = fdiv(fnv[2], fn);
      } else {
        fnv[0] = 0.0f;
        fnv[1] = 0.0f;
        fnv[2] = 1.0f;
      }
      for (int k = 0; k < 3; ++k) {
        const float* p = ep[es[k]];
        float nrm[3];
        mc_vertex_normal(map, voxel_size, p, fnv, nrm);
        for (int a = 0; a < 3; ++a) {
          verts[9 * o + 3 * k + a] = p[a];
          normals[9 * o + 3 * k + a] = nrm[a];
          if (with_colors) colors[9 * o + 3 * k + a] = ec[es[k]][a];
        }
      }
    }
  }
}

// ---------------------------------------------------------------- free-function evaluation
__global__ void k_eval_pd(uint64_t n, const float* x, const float* p, const float* s, float* out) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    out[i] = projective_distance(x[3 * i], x[3 * i + 1], x[3 * i + 2], p[3 * i], p[3 * i + 1], p[3 * i + 2],
                                 s[3 * i], s[3 * i + 1], s[3 * i + 2]);
  }
}

__global__ void k_eval_mw(uint64_t n, int mode, const float* z, const float* d, float trunc, float eps, float* out) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    out[i] = measurement_weight(mode, z[i], d[i], trunc, eps);
  }
}

__global__ void k_eval_update(uint64_t nv, vxg_voxel* voxels, const uint64_t* starts, const float* d, const float* w,
                              const uint8_t* rgb, float trunc, float wmax) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < nv;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    float D = voxels[i].distance, W = voxels[i].weight;
    uint32_t c = static_cast<uint32_t>(voxels[i].r) | (static_cast<uint32_t>(voxels[i].g) << 8) |
                 (static_cast<uint32_t>(voxels[i].b) << 16);
    for (uint64_t j = starts[i]; j < starts[i + 1]; ++j) {
      const uint32_t col = rgb != nullptr ? pack_color(rgb + 3 * j) : 0u;
      update_voxel(D, W, c, d[j], w[j], col, rgb != nullptr, trunc, wmax);
    }
    voxels[i].distance = D;
    voxels[i].weight = W;
    voxels[i].r = static_cast<uint8_t>(c & 0xffu);
    voxels[i].g = static_cast<uint8_t>((c >> 8) & 0xffu);
    voxels[i].b = static_cast<uint8_t>((c >> 16) & 0xffu);
  }
}

__global__ void k_eval_raycast(uint64_t n, const float* start, const float* end, float v, uint32_t* counts,
                               const uint64_t* offsets, int32_t* out) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    Dda dda;
    dda.init(start[3 * i], start[3 * i + 1], start[3 * i + 2], end[3 * i], end[3 * i + 1], end[3 * i + 2], v);
    const uint32_t count = dda.span + 1u;
    counts[i] = count;
    if (out == nullptr) continue;
    int32_t* o = out + 3 * offsets[i];
    for (uint32_t k = 0; k < count; ++k) {
      o[3 * k + 0] = dda.cur[0];
      o[3 * k + 1] = dda.cur[1];
      o[3 * k + 2] = dda.cur[2];
      if (k + 1 < count && !dda.at_end()) dda.advance();
    }
  }
}

}  // namespace vxg
