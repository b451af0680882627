// Test infrastructure (not product): per-scan insert timing of a caller of the
// reference's C++ API, the way `vxf integrate` measures it (cli.cpp:168-186:
// steady_clock around each TsdfIntegrator::integrate call, median reported).
// Built twice by oracle/Makefile from the same source against the reference's
// headers: _ref/bench_insert_ref links the reference's own tsdf_integrator.cpp,
// _ref/bench_insert_vxg links the B200 drop-in
// (paper_1611_03631_b200/dropin/vxf_tsdf_integrator_vxg.cpp + libvxg.so), which
// also writes the updated blocks back into the caller's host TsdfLayer.
// Input: a scan file written by tests/dropin_insert_timing.py — u32 F, then per scan
// u32 n, 12 floats (row-major 3x4 sensor-to-world), n x 3 floats, n x 3 bytes.
// Args: <scan file> <voxel_size> <truncation> <epsilon> <max_ray> <merge 0|1|2> <weight 0|1|2> <min_ray> <max_weight>
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <vector>

#include "vxf/layer.h"
#include "vxf/scan.h"
#include "vxf/tsdf_integrator.h"

using namespace vxf;

int main(int argc, char** argv) {
  if (argc < 10) return 2;
  std::ifstream in(argv[1], std::ios::binary);
  uint32_t F = 0;
  in.read(reinterpret_cast<char*>(&F), 4);
  std::vector<Scan> scans(F);
  for (uint32_t f = 0; f < F; ++f) {
    uint32_t n = 0;
    float P[12];
    in.read(reinterpret_cast<char*>(&n), 4);
    in.read(reinterpret_cast<char*>(P), sizeof(P));
    std::vector<float> xyz(3 * static_cast<size_t>(n));
    std::vector<uint8_t> rgb(3 * static_cast<size_t>(n));
    in.read(reinterpret_cast<char*>(xyz.data()), xyz.size() * 4);
    in.read(reinterpret_cast<char*>(rgb.data()), rgb.size());
    Scan& s = scans[f];
    s.points.resize(n);
    s.colors.resize(n);
    for (uint32_t i = 0; i < n; ++i) {
      s.points[i] = Point(xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]);
      s.colors[i] = Color{rgb[3 * i], rgb[3 * i + 1], rgb[3 * i + 2]};
    }
    Eigen::Matrix3f R;
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) R(r, c) = P[4 * r + c];
    s.pose = Transform::Identity();
    s.pose.linear() = R;
    s.pose.translation() = Point(P[3], P[7], P[11]);
  }
  TsdfConfig cfg;
  const float v = static_cast<float>(atof(argv[2]));
  cfg.truncation = static_cast<float>(atof(argv[3]));
  cfg.dropoff_epsilon = static_cast<float>(atof(argv[4]));
  cfg.max_ray_length = static_cast<float>(atof(argv[5]));
  cfg.merge_mode = static_cast<MergeMode>(atoi(argv[6]));
  cfg.weight_mode = static_cast<WeightMode>(atoi(argv[7]));
  cfg.min_ray_length = static_cast<float>(atof(argv[8]));
  cfg.max_weight = static_cast<float>(atof(argv[9]));
  TsdfLayer layer(v, 16);
  TsdfIntegrator integ(cfg, &layer);
  std::vector<double> ms;
  size_t updates = 0;
  for (uint32_t f = 0; f < F; ++f) {
    const auto t0 = std::chrono::steady_clock::now();
    updates += integ.integrate(scans[f]);
    ms.push_back(1e3 * std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
  }
  std::vector<double> s = ms;
  std::sort(s.begin(), s.end());
  double mean = 0;
  for (double x : ms) mean += x / ms.size();
  printf("{\"scans\": %u, \"updates\": %zu, \"blocks\": %zu, \"median_ms\": %.4f, \"p90_ms\": %.4f, \"mean_ms\": %.4f, "
         "\"first_ms\": %.4f}\n",
         F, updates, layer.block_count(), s[s.size() / 2], s[std::min(s.size() - 1, s.size() * 9 / 10)], mean, ms[0]);
  return 0;
}
