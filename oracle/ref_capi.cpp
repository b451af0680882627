// TEST INFRASTRUCTURE ONLY: a C ABI over the UNMODIFIED reference sources
// (/root/reference/proj/src/tsdf_integrator.cpp, src/serialization.cpp and the
// vxf headers), compiled against oracle/eigen_shim by oracle/Makefile into
// oracle/_ref/libvxfref.so. Used to pin the oracle restatement
// (tests/test_oracle_pin.py), to generate tests/golden/ fixtures, and as the
// timed CPU baseline (bench.py cpu_baseline kind "reference", --impl reference).
// No reference source is copied into this repository.
#include <cstring>
#include <sstream>
#include <stdexcept>
#include <string>

#include "vxf/analysis.h"
#include "vxf/interpolation.h"
#include "vxf/layer.h"
#include "vxf/serialization.h"
#include "vxf/tsdf_integrator.h"

#include "../include/vxg_types.h"

namespace {

thread_local std::string g_last_error;

vxf::TsdfConfig to_config(const vxg_tsdf_config* c) {
  vxf::TsdfConfig t;
  t.truncation = c->truncation;
  t.dropoff_epsilon = c->dropoff_epsilon;
  t.max_weight = c->max_weight;
  t.weight_mode = static_cast<vxf::WeightMode>(c->weight_mode);
  t.merge_mode = static_cast<vxf::MergeMode>(c->merge_mode);
  t.min_ray_length = c->min_ray_length;
  t.max_ray_length = c->max_ray_length;
  return t;
}

struct RefHandle {
  vxf::TsdfLayer layer;
  vxf::TsdfIntegrator integrator;
  RefHandle(float v, int vps, const vxf::TsdfConfig& c) : layer(v, vps), integrator(c, &layer) {}
};

}  // namespace

extern "C" {

const char* vxr_last_error(void) { return g_last_error.c_str(); }

void* vxr_create(const vxg_tsdf_config* c, float voxel_size, int vps) {
  try {
    return new RefHandle(voxel_size, vps, to_config(c));
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return nullptr;
  }
}

void vxr_destroy(void* h) { delete static_cast<RefHandle*>(h); }

// Scan{points, colors, pose} -> TsdfIntegrator::integrate (tsdf_integrator.cpp:111).
int vxr_integrate(void* hp, const float* xyz, const uint8_t* rgb, size_t n, const float pose[12],
                  vxg_stats* out) {
  auto* h = static_cast<RefHandle*>(hp);
  vxf::Scan scan;
  scan.points.resize(n);
  for (size_t i = 0; i < n; ++i) scan.points[i] = vxf::Point(xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]);
  if (rgb != nullptr) {
    scan.colors.resize(n);
    for (size_t i = 0; i < n; ++i) scan.colors[i] = vxf::Color{rgb[3 * i], rgb[3 * i + 1], rgb[3 * i + 2]};
  }
  vxf::Transform pose_t = vxf::Transform::Identity();
  for (int r = 0; r < 3; ++r) {
    for (int k = 0; k < 3; ++k) pose_t.linear()(r, k) = pose[4 * r + k];
    pose_t.translation()[r] = pose[4 * r + 3];
  }
  scan.pose = pose_t;
  try {
    const size_t updates = h->integrator.integrate(scan);
    if (out != nullptr) {
      out->updates = updates;
      out->raycasts = h->integrator.raycasts_last_scan();
      out->skipped = h->integrator.skipped_points_last_scan();
    }
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return VXG_EINVAL;
  }
  return VXG_OK;
}

size_t vxr_block_count(void* hp) { return static_cast<RefHandle*>(hp)->layer.block_count(); }

// vxf::save_layer (serialization.cpp:141-168,216-218) into a caller buffer.
size_t vxr_save_vxblx(void* hp, uint8_t* buf, size_t cap) {
  std::ostringstream os(std::ios::binary);
  vxf::save_layer(static_cast<RefHandle*>(hp)->layer, os);
  const std::string s = os.str();
  if (buf != nullptr && cap >= s.size()) std::memcpy(buf, s.data(), s.size());
  return s.size();
}

int vxr_config_validate(const vxg_tsdf_config* c, char* err, size_t err_len) {
  try {
    to_config(c).validate();
  } catch (const std::exception& e) {
    if (err != nullptr && err_len > 0) {
      std::strncpy(err, e.what(), err_len - 1);
      err[err_len - 1] = '\0';
    }
    return VXG_EINVAL;
  }
  return VXG_OK;
}

float vxr_projective_distance(const float x[3], const float p[3], const float s[3]) {
  return vxf::projective_distance(vxf::Point(x[0], x[1], x[2]), vxf::Point(p[0], p[1], p[2]),
                                  vxf::Point(s[0], s[1], s[2]));
}

float vxr_measurement_weight(int mode, float z, float d, float truncation, float eps) {
  return vxf::measurement_weight(static_cast<vxf::WeightMode>(mode), z, d, truncation, eps);
}

void vxr_update_voxel(vxg_voxel* v, float d, float w, float truncation, float max_weight, const uint8_t* color) {
  vxf::TsdfVoxel t;
  t.distance = v->distance;
  t.weight = v->weight;
  t.color = vxf::Color{v->r, v->g, v->b};
  if (color != nullptr) {
    vxf::update_tsdf_voxel(&t, d, w, truncation, max_weight, vxf::Color{color[0], color[1], color[2]}, true);
  } else {
    vxf::update_tsdf_voxel(&t, d, w, truncation, max_weight);
  }
  v->distance = t.distance;
  v->weight = t.weight;
  v->r = t.color.r;
  v->g = t.color.g;
  v->b = t.color.b;
}

size_t vxr_raycast(const float start[3], const float end[3], float voxel_size, int32_t* out, size_t cap) {
  vxf::RayCaster caster(vxf::Point(start[0], start[1], start[2]), vxf::Point(end[0], end[1], end[2]), voxel_size);
  vxf::GlobalVoxelIndex g;
  size_t k = 0;
  while (caster.next(&g)) {
    if (k < cap) {
      out[3 * k + 0] = g.x();
      out[3 * k + 1] = g.y();
      out[3 * k + 2] = g.z();
    }
    ++k;
  }
  return k;
}

uint64_t vxr_index_hash(int32_t x, int32_t y, int32_t z) {
  return static_cast<uint64_t>(vxf::IndexHash()(Eigen::Vector3i(x, y, z)));
}

// interpolate_distance (interpolation.h:28-60) per point: found[i] = 0 when absent.
void vxr_interpolate(void* hp, const float* pts, size_t n, float* d, uint8_t* found) {
  const auto& layer = static_cast<RefHandle*>(hp)->layer;
  for (size_t i = 0; i < n; ++i) {
    const auto r = vxf::interpolate_distance(layer, vxf::Point(pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]));
    found[i] = r.has_value() ? 1 : 0;
    d[i] = r.has_value() ? *r : 0.0f;
  }
}

// surface_error (analysis.cpp:41-59): out = {rms, mean, max, count, unknown_fraction}.
void vxr_surface_error(void* hp, const float* pts, size_t n, float truncation, double out[5]) {
  std::vector<vxf::Point> p(n);
  for (size_t i = 0; i < n; ++i) p[i] = vxf::Point(pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]);
  const vxf::ErrorStats s = vxf::surface_error(static_cast<RefHandle*>(hp)->layer, p, truncation);
  out[0] = s.rms;
  out[1] = s.mean;
  out[2] = s.max;
  out[3] = static_cast<double>(s.count);
  out[4] = s.unknown_fraction;
}

}  // extern "C"
