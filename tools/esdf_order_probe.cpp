// Dev probe (not product, not a test): is the reference's ESDF propagation
// (src/esdf_integrator.cpp) independent of the wavefront queue order? Builds
// EsdfIntegrator::build_batch over a VXBLX TSDF layer with the three queue
// modes (esdf_integrator.h:22-26) for both metrics and both band modes, and
// counts voxels whose distance / parent differ between modes. Compiled from the
// UNMODIFIED reference sources against oracle/eigen_shim by
// tools/esdf_order_probe.sh; the layers come from the oracle (cfg1/2/3 frames).
// Result: thousands to hundreds of thousands of voxels differ,
// so no parallel propagation can be bit-exact with the reference's sequential
// queue order — the reason ESDF stays off the GPU path.
#include "vxf/esdf_integrator.h"
#include "vxf/serialization.h"
#include <fstream>
#include <cstdio>
#include <cstring>
using namespace vxf;
int main(int argc, char** argv) {
  std::ifstream in(argv[1], std::ios::binary);
  TsdfLayer t = load_tsdf_layer(in);
  float trunc = atof(argv[2]);
  for (int metric = 0; metric < 2; ++metric) for (int band = 0; band < 2; ++band) {
    EsdfLayer* L[3];
    for (int q = 0; q < 3; ++q) {
      EsdfConfig c; c.d_max = 4.0f; c.truncation = trunc;
      c.metric = metric ? DistanceMetric::kEuclidean : DistanceMetric::kQuasiEuclidean;
      c.band_mode = band ? FixedBandMode::kHalfTruncation : FixedBandMode::kOneVoxel;
      c.queue_mode = (QueueMode)q;
      L[q] = new EsdfLayer(EsdfIntegrator::build_batch(t, c));
    }
    long nd[3] = {0,0,0}, np[3] = {0,0,0}, nobs = 0, nflip = 0;
    for (auto& kv : L[0]->blocks()) {
      for (int q = 1; q < 3; ++q) {
        auto* b = L[q]->block_ptr(kv.first);
        for (size_t i = 0; i < kv.second->num_voxels(); ++i) {
          auto& a = kv.second->voxel(i); auto& o = b->voxel(i);
          if (q == 1 && a.observed()) ++nobs;
          if (memcmp(&a.distance, &o.distance, 4)) ++nd[q];
          if (a.parent != o.parent) ++np[q];
        }
      }
      const auto* tb = t.block_ptr(kv.first);
      for (size_t i = 0; i < kv.second->num_voxels(); ++i) {
        auto& a = kv.second->voxel(i);
        if (a.observed() && !a.fixed() && ((a.distance < 0) != (tb->voxel(i).distance < 0))) ++nflip;
      }
    }
    printf("metric %d band %d: observed %ld, sign flips vs tsdf %ld | fifo vs single: dist %ld parent %ld | fifo vs multi: dist %ld parent %ld\n",
           metric, band, nobs, nflip, nd[1], np[1], nd[2], np[2]);
  }
}
