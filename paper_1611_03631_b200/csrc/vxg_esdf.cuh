// ESDF on the device slab: the occupancy-seeded baseline
// vxf::EsdfIntegrator::build_from_occupancy (esdf_integrator.cpp:303-330) with
// the quasi-Euclidean metric.
//
// The reference drains a wavefront queue; with the quasi-Euclidean metric and
// only non-negative, only-lowering values the result does not depend on the
// queue order: every final distance is the minimum over 26-connected paths of
// observed voxels from a seed (observed, TSDF distance < 0, fixed at 0) of the
// path's left-to-right fp32 sum RN(RN(0 + s1) + s2)... of the step lengths
// v*sqrt(1|2|3) (relax_neighbors :258-292), capped at d_max. (Each value is a
// path value, and by monotonicity of RN(x + s) it is <= every path's value.)
// So a parallel relaxation to the fixed point d(u) = min(d(u), min_v RN(d(v) +
// s_uv)) reproduces the reference's distances and flags bit for bit. Parents
// record which neighbour a voxel was last lowered from: order-dependent under
// ties, so the GPU picks the first minimising neighbour in the reference's
// neighbour order (dz, dy, dx), a valid parent that may differ from the
// reference's on ties (the Euclidean metric feeds parents back into distances
// and is not offered here: tools/esdf_order_probe).
//
// Layout: one ESDF block per TSDF slot (same slot numbering), 8-byte voxels =
// the ESDF VXBLX payload (f32 distance, u8 flags, 3 x i8 parent).
#pragma once

#include "vxg_kernels.cuh"

namespace vxg {

constexpr uint8_t kEsdfObserved = 1, kEsdfFixed = 2;  // voxel.h:24-25

// Neighbour block slots: nbr[27 * s + (dz+1)*9 + (dy+1)*3 + (dx+1)], -1 if absent.
__global__ void k_esdf_neighbors(uint32_t nb, const int32_t* __restrict__ block_idx, MapView map,
                                 int32_t* __restrict__ nbr) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < 27u * nb; i += gridDim.x * blockDim.x) {
    const uint32_t s = i / 27u, d = i % 27u;
    const int dx = static_cast<int>(d % 3u) - 1, dy = static_cast<int>((d / 3u) % 3u) - 1,
              dz = static_cast<int>(d / 9u) - 1;
    const int bx = block_idx[3 * s] + dx, by = block_idx[3 * s + 1] + dy, bz = block_idx[3 * s + 2] + dz;
    int32_t t = -1;
    if (block_in_range(bx, by, bz)) t = map.find(pack_block(bx, by, bz));
    if (t >= static_cast<int32_t>(nb)) t = -1;
    nbr[i] = t;
  }
}

// Seeding (:310-326): observed voxels with TSDF distance < 0 are fixed at 0,
// other observed ones start at d_max; unobserved voxels keep the default voxel
// (d_max, no flags; :81-83).
__global__ void k_esdf_init(uint64_t n, const vxg_voxel* __restrict__ tsdf, vxg_esdf_voxel* __restrict__ esdf,
                            float d_max) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const vxg_voxel t = tsdf[i];
    vxg_esdf_voxel e;
    e.distance = d_max;
    e.flags = 0;
    e.parent[0] = e.parent[1] = e.parent[2] = 0;
    if (t.weight > 1e-4f) {  // TsdfVoxel::observed (voxel.h:17)
      e.flags = kEsdfObserved;
      if (t.distance < 0.0f) {
        e.distance = 0.0f;
        e.flags |= kEsdfFixed;
      }
    }
    esdf[i] = e;
  }
}

constexpr int kEsdfThreads = 512;  // 8 voxels of a 16^3 block per thread: latency-bound sweeps want warps

struct EsdfSteps {
  float s[4];  // v * sqrt(k) for k = |offset|^2 in 1..3 (constructor :75), s[0] unused
};

// The neighbour of local voxel (x, y, z) of slot `slot` at offset (dx, dy, dz):
// pointer into the ESDF slab, or nullptr when its block is unallocated.
__device__ __forceinline__ const vxg_esdf_voxel* esdf_neighbor(const vxg_esdf_voxel* esdf, const int32_t* nbr27,
                                                              int vps, int x, int y, int z, int dx, int dy, int dz) {
  int nx = x + dx, ny = y + dy, nz = z + dz;
  const int bx = nx < 0 ? -1 : (nx >= vps ? 1 : 0);
  const int by = ny < 0 ? -1 : (ny >= vps ? 1 : 0);
  const int bz = nz < 0 ? -1 : (nz >= vps ? 1 : 0);
  const int32_t t = nbr27[(bz + 1) * 9 + (by + 1) * 3 + (bx + 1)];
  if (t < 0) return nullptr;
  nx -= bx * vps;
  ny -= by * vps;
  nz -= bz * vps;
  return esdf + static_cast<uint64_t>(t) * vps * vps * vps + nx + vps * (ny + vps * nz);
}

// One CTA per active block: Gauss-Seidel sweeps of the pull relaxation over
// the block's voxels until the block is stable; a block that changed marks
// itself and its 26 neighbours active for the next round (their voxels read
// its new values). Values only decrease and stay path values, so concurrent
// CTAs reading each other's blocks mid-update (possibly stale: L1 is not
// coherent across SMs within a launch) converge to the same fixed point; the
// barrier between sweeps makes the block's own updates visible.
__global__ void __launch_bounds__(kEsdfThreads) k_esdf_relax(uint32_t nb, vxg_esdf_voxel* __restrict__ esdf,
                                                    const int32_t* __restrict__ nbr, int vps, EsdfSteps steps,
                                                    const uint8_t* __restrict__ active_in,
                                                    uint8_t* __restrict__ active_out, uint32_t* __restrict__ changed) {
  __shared__ int32_t s_nbr[27];
  for (uint32_t s = blockIdx.x; s < nb; s += gridDim.x) {
    if (!active_in[s]) continue;
    __syncthreads();
    if (threadIdx.x < 27) s_nbr[threadIdx.x] = nbr[27 * s + threadIdx.x];
    __syncthreads();
    const int nvox = vps * vps * vps;
    vxg_esdf_voxel* blk = esdf + static_cast<uint64_t>(s) * nvox;
    bool block_changed = false;
    for (int sweep = 0;; ++sweep) {
      bool any = false;
      for (int i = threadIdx.x; i < nvox; i += blockDim.x) {
        const vxg_esdf_voxel u = blk[i];
        if ((u.flags & (kEsdfObserved | kEsdfFixed)) != kEsdfObserved) continue;
        const int x = i % vps, y = (i / vps) % vps, z = i / (vps * vps);
        float best = u.distance;
#pragma unroll
        for (int dz = -1; dz <= 1; ++dz)
#pragma unroll
          for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
            for (int dx = -1; dx <= 1; ++dx) {
              if (dx == 0 && dy == 0 && dz == 0) continue;
              const vxg_esdf_voxel* p = esdf_neighbor(esdf, s_nbr, vps, x, y, z, dx, dy, dz);
              if (p == nullptr) continue;
              const uint2 v = *reinterpret_cast<const uint2*>(p);  // {distance, flags | parent << 8}
              if (!(v.y & kEsdfObserved)) continue;
              const float cand = __fadd_rn(__uint_as_float(v.x), steps.s[dx * dx + dy * dy + dz * dz]);
              if (cand < best) best = cand;
            }
        if (best < u.distance) {
          blk[i].distance = best;
          any = true;
        }
      }
      if (!__syncthreads_or(any)) break;
      block_changed = true;
    }
    if (block_changed && threadIdx.x < 27) {
      const int32_t t = s_nbr[threadIdx.x];
      if (t >= 0) active_out[t] = 1u;
      if (threadIdx.x == 0) atomicAdd(changed, 1u);
    }
  }
}

// Parents (relax_neighbors :268-290): the first neighbour in the reference's
// order (dz, dy, dx) whose candidate equals the voxel's final distance; none
// for fixed voxels, unobserved ones and voxels still at d_max (never lowered).
__global__ void k_esdf_parents(uint32_t nb, vxg_esdf_voxel* __restrict__ esdf, const int32_t* __restrict__ nbr,
                               int vps, EsdfSteps steps, float d_max) {
  const int nvox = vps * vps * vps;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < static_cast<uint64_t>(nb) * nvox;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t s = static_cast<uint32_t>(i / nvox);
    const int l = static_cast<int>(i % nvox);
    vxg_esdf_voxel u = esdf[i];
    if ((u.flags & (kEsdfObserved | kEsdfFixed)) != kEsdfObserved || !(u.distance < d_max)) continue;
    const int x = l % vps, y = (l / vps) % vps, z = l / (vps * vps);
    const int32_t* nbr27 = nbr + 27 * s;
    bool done = false;
    for (int dz = -1; dz <= 1 && !done; ++dz)
      for (int dy = -1; dy <= 1 && !done; ++dy)
        for (int dx = -1; dx <= 1 && !done; ++dx) {
          if (dx == 0 && dy == 0 && dz == 0) continue;
          const vxg_esdf_voxel* p = esdf_neighbor(esdf, nbr27, vps, x, y, z, dx, dy, dz);
          if (p == nullptr || !(p->flags & kEsdfObserved)) continue;
          if (__fadd_rn(p->distance, steps.s[dx * dx + dy * dy + dz * dz]) == u.distance) {
            esdf[i].parent[0] = static_cast<int8_t>(dx);
            esdf[i].parent[1] = static_cast<int8_t>(dy);
            esdf[i].parent[2] = static_cast<int8_t>(dz);
            done = true;
          }
        }
  }
}

}  // namespace vxg
