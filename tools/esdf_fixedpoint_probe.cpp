// Dev probe (not product, not a test): how close is an ORDER-INDEPENDENT fixed
// point of the reference's lower-wavefront rule (relax_neighbors,
// esdf_integrator.cpp:232-294, quasi-Euclidean) to the reference's own
// build_batch under its three queue orders? The fixed point freezes every
// non-fixed voxel's sign to its TSDF sign: a positive voxel takes the minimum of
// d(v) + step over observed neighbours v whose candidate is positive, a negative
// voxel the maximum of d(v) - step over those whose candidate is negative
// (sweeps to convergence; the result does not depend on the sweep order because
// values only move monotonically towards 0 and every value is a path value).
// Prints, per band mode, voxels that differ between the fixed point and each
// queue mode next to the modes' differences among themselves.
#include "vxf/esdf_integrator.h"
#include "vxf/serialization.h"
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
using namespace vxf;
int main(int argc, char** argv) {
  std::ifstream in(argv[1], std::ios::binary);
  TsdfLayer t = load_tsdf_layer(in);
  const float trunc = atof(argv[2]);
  const int vps = t.voxels_per_side();
  const float v = t.voxel_size();
  for (int band = 0; band < 2; ++band) {
    EsdfConfig c;
    c.d_max = 4.0f;
    c.truncation = trunc;
    c.metric = DistanceMetric::kQuasiEuclidean;
    c.band_mode = band ? FixedBandMode::kHalfTruncation : FixedBandMode::kOneVoxel;
    EsdfLayer* L[3];
    for (int q = 0; q < 3; ++q) {
      c.queue_mode = (QueueMode)q;
      L[q] = new EsdfLayer(EsdfIntegrator::build_batch(t, c));
    }
    const float gamma = c.band_radius(v);
    // fixed point on a copy of mode 0's block set
    EsdfLayer F(v, vps);
    EsdfVoxel dv; dv.distance = c.d_max; F.set_default_voxel(dv);
    for (auto& kv : t.blocks()) {
      auto& fb = F.get_or_allocate_block(kv.first);
      for (size_t i = 0; i < kv.second->num_voxels(); ++i) {
        const TsdfVoxel& tv = kv.second->voxel(i);
        if (!tv.observed()) continue;
        EsdfVoxel& e = fb.voxel(i);
        e.set_observed(true);
        if (is_fixed(tv.distance, gamma)) { e.set_fixed(true); e.distance = tv.distance; }
        else e.distance = tv.distance < 0.0f ? -c.d_max : c.d_max;
      }
    }
    long sweeps = 0;
    for (bool any = true; any; ++sweeps) {
      any = false;
      for (auto& kv : F.blocks()) {
        for (size_t i = 0; i < kv.second->num_voxels(); ++i) {
          EsdfVoxel& u = kv.second->voxel(i);
          if (!u.observed() || u.fixed()) continue;
          const GlobalVoxelIndex g = combine_indices(kv.first, kv.second->local_from_linear(i), vps);
          for (int dz = -1; dz <= 1; ++dz) for (int dy = -1; dy <= 1; ++dy) for (int dx = -1; dx <= 1; ++dx) {
            if (!dx && !dy && !dz) continue;
            BlockIndex b; LocalVoxelIndex l;
            split_global_index(g + GlobalVoxelIndex(dx, dy, dz), vps, &b, &l);
            auto* nb = F.block_ptr(b);
            if (!nb) continue;
            const EsdfVoxel& n = nb->voxel(l);
            if (!n.observed()) continue;
            const float step = v * std::sqrt(static_cast<float>(dx * dx + dy * dy + dz * dz));
            if (u.distance > 0.0f) {
              const float cand = n.distance + step;
              if (cand > 0.0f && cand < u.distance) { u.distance = cand; any = true; }
            } else if (u.distance < 0.0f) {
              const float cand = n.distance - step;
              if (cand < 0.0f && cand > u.distance) { u.distance = cand; any = true; }
            }
          }
        }
      }
    }
    long nobs = 0, dm[3][3] = {}, df[3] = {}, agree = 0, agree_diff = 0, outside = 0;
    double agree_max = 0;
    double maxabs[3] = {}, maxmm = 0;
    for (auto& kv : L[0]->blocks()) {
      auto* fb = F.block_ptr(kv.first);
      for (size_t i = 0; i < kv.second->num_voxels(); ++i) {
        if (kv.second->voxel(i).observed()) ++nobs;
        float d[3];
        for (int q = 0; q < 3; ++q) d[q] = L[q]->block_ptr(kv.first)->voxel(i).distance;
        for (int a = 0; a < 3; ++a) for (int b = a + 1; b < 3; ++b) if (memcmp(&d[a], &d[b], 4)) { ++dm[a][b]; maxmm = std::max(maxmm, (double)std::fabs(d[a] - d[b])); }
        const float f = fb->voxel(i).distance;
        if (kv.second->voxel(i).observed()) {
          if (!memcmp(&d[0], &d[1], 4) && !memcmp(&d[0], &d[2], 4)) { ++agree; if (memcmp(&f, &d[0], 4)) { ++agree_diff; agree_max = std::max(agree_max, (double)std::fabs(f - d[0])); } }
          else { const float lo = std::min(d[0], std::min(d[1], d[2])), hi = std::max(d[0], std::max(d[1], d[2])); if (f < lo || f > hi) ++outside; }
        }
        for (int q = 0; q < 3; ++q) if (memcmp(&f, &d[q], 4)) { ++df[q]; maxabs[q] = std::max(maxabs[q], (double)std::fabs(f - d[q])); }
      }
    }
    printf("band %d: modes agree on %ld voxels, fixed point differs on %ld of them (max %.3f); where they disagree the fixed point is outside [min, max] of the modes on %ld\n", band, agree, agree_diff, agree_max, outside);
    printf("band %d: observed %ld, sweeps %ld | modes differ: fifo/single %ld fifo/multi %ld single/multi %ld (max |diff| %.3f) | fixed point vs fifo %ld single %ld multi %ld (max |diff| %.3f %.3f %.3f)\n",
           band, nobs, sweeps, dm[0][1], dm[0][2], dm[1][2], maxmm, df[0], df[1], df[2], maxabs[0], maxabs[1], maxabs[2]);
  }
}
