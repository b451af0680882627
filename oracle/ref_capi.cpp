// TEST INFRASTRUCTURE ONLY: a C ABI over the UNMODIFIED reference sources
// (/root/reference/proj/src/tsdf_integrator.cpp, src/serialization.cpp and the
// vxf headers), compiled against oracle/eigen_shim by oracle/Makefile into
// oracle/_ref/libvxfref.so. Used to pin the oracle restatement
// (tests/test_oracle_pin.py), to generate tests/golden/ fixtures, and as the
// timed CPU baseline (bench.py cpu_baseline kind "reference", --impl reference).
// No reference source is copied into this repository.
#include <chrono>
#include <cstring>
#include <sstream>
#include <stdexcept>
#include <string>

#include "vxf/analysis.h"
#include "vxf/esdf_integrator.h"
#include "vxf/interpolation.h"
#include "vxf/layer.h"
#include "vxf/marching_cubes_tables.h"
#include "vxf/mesh_extractor.h"
#include "vxf/scan.h"
#include "vxf/serialization.h"
#include "vxf/tsdf_integrator.h"

#include "../include/vxg_types.h"

namespace {

thread_local std::string g_last_error;
thread_local double g_last_seconds = 0.0;

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

// Seconds the last vxr_integrate spent inside TsdfIntegrator::integrate.
double vxr_last_integrate_seconds(void) { return g_last_seconds; }

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
    // timed exactly as the reference times an insert (benchmark.cpp:93-95,
    // cli.cpp:171-174): steady_clock around integrate() only
    const auto t0 = std::chrono::steady_clock::now();
    const size_t updates = h->integrator.integrate(scan);
    g_last_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
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

// vxf::EsdfIntegrator::build_from_occupancy (esdf_integrator.cpp:303-330) over
// the handle's layer, saved with vxf::save_layer (ESDF payload) into a caller
// buffer. Returns the byte size, or 0 with vxr_last_error() on an exception.
size_t vxr_esdf_occupancy(void* hp, const vxg_esdf_config* c, uint8_t* buf, size_t cap) {
  try {
    vxf::EsdfConfig e;
    e.d_max = c->d_max;
    e.band_mode = static_cast<vxf::FixedBandMode>(c->band_mode);
    e.truncation = c->truncation;
    e.metric = static_cast<vxf::DistanceMetric>(c->metric);
    e.queue_mode = static_cast<vxf::QueueMode>(c->queue_mode);
    e.bucket_width = c->bucket_width;
    const vxf::EsdfLayer esdf = vxf::EsdfIntegrator::build_from_occupancy(static_cast<RefHandle*>(hp)->layer, e);
    std::ostringstream os(std::ios::binary);
    vxf::save_layer(esdf, os);
    const std::string s = os.str();
    if (buf != nullptr && cap >= s.size()) std::memcpy(buf, s.data(), s.size());
    return s.size();
  } catch (const std::exception& ex) {
    g_last_error = ex.what();
    return 0;
  }
}

// vxf::save_layer (serialization.cpp:141-168,216-218) into a caller buffer.
size_t vxr_save_vxblx(void* hp, uint8_t* buf, size_t cap) {
  std::ostringstream os(std::ios::binary);
  vxf::save_layer(static_cast<RefHandle*>(hp)->layer, os);
  const std::string s = os.str();
  if (buf != nullptr && cap >= s.size()) std::memcpy(buf, s.data(), s.size());
  return s.size();
}

// vxf::load_tsdf_layer (serialization.cpp:193-212) of a VXBLX image, then
// vxf::save_layer of the loaded layer into a caller buffer. Returns the byte
// size, or 0 with vxr_last_error() on a ParseError.
size_t vxr_load_resave(const uint8_t* in, size_t len, uint8_t* buf, size_t cap) {
  try {
    std::istringstream is(std::string(reinterpret_cast<const char*>(in), len), std::ios::binary);
    const vxf::TsdfLayer layer = vxf::load_tsdf_layer(is);
    std::ostringstream os(std::ios::binary);
    vxf::save_layer(layer, os);
    const std::string s = os.str();
    if (buf != nullptr && cap >= s.size()) std::memcpy(buf, s.data(), s.size());
    return s.size();
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return 0;
  }
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

// Layer block overwrite (for analytic fields in the meshing parity tests).
void vxr_set_block(void* hp, const int32_t idx[3], const vxg_voxel* voxels) {
  auto& layer = static_cast<RefHandle*>(hp)->layer;
  auto& blk = layer.get_or_allocate_block(vxf::BlockIndex(idx[0], idx[1], idx[2]));
  const int n = layer.voxels_per_side() * layer.voxels_per_side() * layer.voxels_per_side();
  for (int i = 0; i < n; ++i) {
    vxf::TsdfVoxel& v = blk.voxel(i);
    v.distance = voxels[i].distance;
    v.weight = voxels[i].weight;
    v.color = vxf::Color{voxels[i].r, voxels[i].g, voxels[i].b};
  }
}

// The reference build's marching-cubes case tables (marching_cubes_tables.h),
// handed to the B200 path (vxg_mesh_extract takes them from its caller).
void vxr_mc_tables(vxg_mc_tables* t) {
  namespace mc = vxf::mc_tables;
  for (int c = 0; c < 8; ++c)
    for (int a = 0; a < 3; ++a) t->corner_offsets[c][a] = mc::kCornerOffsets[c][a];
  for (int e = 0; e < 12; ++e)
    for (int a = 0; a < 2; ++a) t->edge_corners[e][a] = mc::kEdgeCorners[e][a];
  for (int i = 0; i < 256; ++i) {
    t->edge_table[i] = mc::kEdgeTable[i];
    for (int k = 0; k < 16; ++k) t->tri_table[i][k] = static_cast<int8_t>(mc::kTriTable[i][k]);
  }
}

// MeshExtractor::extract_all / extract_blocks, then fragments() in (x,y,z)
// block order; same output contract as vxo_mesh_extract. Returns n_frag, or
// (size_t)-1 when a fragment's triangles are not (3t, 3t+1, 3t+2).
size_t vxr_mesh_extract(void* hp, int with_colors, const int32_t* blocks, size_t n_req, int32_t* bidx,
                        uint64_t* frag_tri, float* verts, float* normals, uint8_t* colors, size_t cap_frag,
                        size_t cap_tri, uint64_t* n_tri) {
  const auto& layer = static_cast<RefHandle*>(hp)->layer;
  vxf::MeshExtractor ex(&layer, with_colors != 0);
  if (blocks == nullptr) {
    ex.extract_all();
  } else {
    vxf::IndexSet req;
    for (size_t i = 0; i < n_req; ++i) req.insert(vxf::BlockIndex(blocks[3 * i], blocks[3 * i + 1], blocks[3 * i + 2]));
    ex.extract_blocks(req);
  }
  std::vector<vxf::BlockIndex> order;
  for (const auto& kv : ex.fragments()) order.push_back(kv.first);
  std::sort(order.begin(), order.end(), [](const vxf::BlockIndex& a, const vxf::BlockIndex& b) {
    return std::tie(a.x(), a.y(), a.z()) < std::tie(b.x(), b.y(), b.z());
  });
  uint64_t T = 0;
  for (const auto& b : order) T += ex.fragments().at(b).triangles.size();
  *n_tri = T;
  if (cap_frag < order.size() || cap_tri < T) return order.size();
  uint64_t o = 0;
  for (size_t j = 0; j < order.size(); ++j) {
    const vxf::Mesh& m = ex.fragments().at(order[j]);
    if (bidx) {
      bidx[3 * j] = order[j].x();
      bidx[3 * j + 1] = order[j].y();
      bidx[3 * j + 2] = order[j].z();
    }
    if (frag_tri) frag_tri[j] = o;
    for (size_t k = 0; k < m.triangles.size(); ++k)
      if (m.triangles[k][0] != 3 * k || m.triangles[k][1] != 3 * k + 1 || m.triangles[k][2] != 3 * k + 2)
        return static_cast<size_t>(-1);
    for (size_t q = 0; q < m.vertices.size(); ++q)
      for (int a = 0; a < 3; ++a) {
        if (verts) verts[9 * o + 3 * q + a] = m.vertices[q][a];
        if (normals) normals[9 * o + 3 * q + a] = m.normals[q][a];
        if (colors && with_colors) {
          const vxf::Color& c = m.colors[q];
          colors[9 * o + 3 * q + a] = a == 0 ? c.r : (a == 1 ? c.g : c.b);
        }
      }
    o += m.triangles.size();
  }
  if (frag_tri) frag_tri[order.size()] = o;
  return order.size();
}

// vxf::load_ply_points: two calls (xyz == NULL: count + has_color). Returns 0,
// or 1 with the exception text in vxr_last_error().
int vxr_load_ply(const char* path, float* xyz, uint8_t* rgb, uint64_t* n, int* has_color) {
  try {
    const vxf::Scan s = vxf::load_ply_points(path);
    *n = s.points.size();
    *has_color = s.has_colors() ? 1 : 0;
    if (xyz)
      for (size_t i = 0; i < s.points.size(); ++i)
        for (int a = 0; a < 3; ++a) xyz[3 * i + a] = s.points[i][a];
    if (rgb && s.has_colors())
      for (size_t i = 0; i < s.colors.size(); ++i) {
        rgb[3 * i] = s.colors[i].r;
        rgb[3 * i + 1] = s.colors[i].g;
        rgb[3 * i + 2] = s.colors[i].b;
      }
    return 0;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return 1;
  }
}

// vxf::load_tum_trajectory: poses as row-major [R | t].
int vxr_load_tum(const char* path, double* ts, float* poses, uint64_t* n) {
  try {
    const auto tr = vxf::load_tum_trajectory(path);
    *n = tr.size();
    for (size_t i = 0; i < tr.size(); ++i) {
      if (ts) ts[i] = tr[i].timestamp;
      if (poses)
        for (int r = 0; r < 3; ++r) {
          for (int c = 0; c < 3; ++c) poses[12 * i + 4 * r + c] = tr[i].pose.linear()(r, c);
          poses[12 * i + 4 * r + 3] = tr[i].pose.translation()[r];
        }
    }
    return 0;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return 1;
  }
}

// vxf::save_ply_mesh of a mesh given as flat arrays.
int vxr_save_ply_mesh(const char* path, const float* v, const float* nrm, const uint8_t* c, uint64_t nv,
                      const uint32_t* tri, uint64_t nt) {
  try {
    vxf::Mesh m;
    for (uint64_t i = 0; i < nv; ++i) {
      m.vertices.emplace_back(v[3 * i], v[3 * i + 1], v[3 * i + 2]);
      m.normals.emplace_back(nrm[3 * i], nrm[3 * i + 1], nrm[3 * i + 2]);
      if (c) m.colors.push_back(vxf::Color{c[3 * i], c[3 * i + 1], c[3 * i + 2]});
    }
    for (uint64_t t = 0; t < nt; ++t) m.triangles.push_back({tri[3 * t], tri[3 * t + 1], tri[3 * t + 2]});
    vxf::save_ply_mesh(m, path);
    return 0;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return 1;
  }
}

}  // extern "C"
