// CPU ORACLE — TEST INFRASTRUCTURE ONLY (see vxf_oracle.h).
//
// Restatement of the reference hot path with explicit arithmetic. Every
// function cites the reference file:line it follows (paths relative to
// /root/reference/proj). Build flags (oracle/Makefile): g++ -O3 -DNDEBUG
// -ffp-contract=off, default -march: the reference's CMake Release flags
// (CMakeLists.txt:7-9) plus an explicit no-FMA guard.
//
// Eigen evaluation order assumed at the boundary:
//   Isometry3f * v  : p_i = t_i + (R_i0 x + (R_i1 y + R_i2 z))
//   norm / dot      : a0 + (a1 + a2)
#include "vxf_oracle.h"

#include <algorithm>
#include <array>
#include <cmath>
#include <cstring>
#include <limits>
#include <string>
#include <unordered_map>
#include <vector>

namespace {

using Key3 = std::array<int32_t, 3>;

// IndexHash (core.h:68-74): int arithmetic (wrapping), sign-extended to size_t.
struct TeschnerHash {
  size_t operator()(const Key3& k) const {
    const uint32_t h = (static_cast<uint32_t>(k[0]) * 73856093u) ^
                       (static_cast<uint32_t>(k[1]) * 19349669u) ^
                       (static_cast<uint32_t>(k[2]) * 83492791u);
    return static_cast<size_t>(static_cast<int64_t>(static_cast<int32_t>(h)));
  }
};

struct BlockKeyHash {
  size_t operator()(const Key3& k) const {
    uint64_t z = (static_cast<uint64_t>(static_cast<uint32_t>(k[0])) << 42) ^
                 (static_cast<uint64_t>(static_cast<uint32_t>(k[1])) << 21) ^
                 static_cast<uint64_t>(static_cast<uint32_t>(k[2]));
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return static_cast<size_t>(z ^ (z >> 31));
  }
};

inline float sq_norm3(float a, float b, float c) { return a * a + (b * b + c * c); }
inline float norm3(float a, float b, float c) { return std::sqrt(sq_norm3(a, b, c)); }
inline float dot3(const float* a, const float* b) { return a[0] * b[0] + (a[1] * b[1] + a[2] * b[2]); }

// Isometry3f * Vector3f (scan.pose * scan.points[i], tsdf_integrator.cpp:180,202).
inline void transform_point(const float pose[12], const float* x, float* p) {
  for (int i = 0; i < 3; ++i) {
    p[i] = pose[4 * i + 3] + (pose[4 * i + 0] * x[0] + (pose[4 * i + 1] * x[1] + pose[4 * i + 2] * x[2]));
  }
}

// global_index_from_point (core.h:43-47).
inline Key3 global_index(const float* p, float v) {
  return {static_cast<int32_t>(std::floor(p[0] / v)), static_cast<int32_t>(std::floor(p[1] / v)),
          static_cast<int32_t>(std::floor(p[2] / v))};
}

// floor_div (core.h:34-40).
inline int floor_div(int a, int b) {
  int q = a / b;
  if ((a % b != 0) && ((a < 0) != (b < 0))) --q;
  return q;
}

// projective_distance (tsdf_integrator.cpp:22-27).
float projective_distance(const float* x, const float* p, const float* s) {
  const float to_point[3] = {p[0] - x[0], p[1] - x[1], p[2] - x[2]};
  const float magnitude = norm3(to_point[0], to_point[1], to_point[2]);
  const float ps[3] = {p[0] - s[0], p[1] - s[1], p[2] - s[2]};
  const float along = dot3(to_point, ps);
  return along < 0.0f ? -magnitude : magnitude;
}

// measurement_weight (tsdf_integrator.cpp:29-44).
float measurement_weight(int mode, float z, float d, float truncation, float eps) {
  switch (mode) {
    case VXG_WEIGHT_CONSTANT:
      return 1.0f;
    case VXG_WEIGHT_INVERSE_Z2:
      return 1.0f / (z * z);
    case VXG_WEIGHT_INVERSE_Z2_DROPOFF: {
      const float base = 1.0f / (z * z);
      if (d > -eps) return base;
      if (d < -truncation) return 0.0f;
      return base * (d + truncation) / (truncation - eps);
    }
  }
  return 0.0f;
}

// update_tsdf_voxel (tsdf_integrator.cpp:51-67).
void update_voxel(vxg_voxel* v, float d, float w, float truncation, float max_weight,
                  const uint8_t* color) {
  if (w <= 0.0f) return;
  const float clamped = std::clamp(d, -truncation, truncation);
  const float total = v->weight + w;
  v->distance = (v->weight * v->distance + w * clamped) / total;
  if (color != nullptr) {
    auto blend = [&](uint8_t old_c, uint8_t new_c) {
      const float mixed = (v->weight * static_cast<float>(old_c) + w * static_cast<float>(new_c)) / total;
      return static_cast<uint8_t>(std::clamp(std::lround(mixed), 0l, 255l));
    };
    const uint8_t r = blend(v->r, color[0]);
    const uint8_t g = blend(v->g, color[1]);
    const uint8_t b = blend(v->b, color[2]);
    v->r = r;
    v->g = g;
    v->b = b;
  }
  v->weight = std::min(total, max_weight);
}

// RayCaster (tsdf_integrator.cpp:69-104).
struct RayCaster {
  Key3 cur{}, end{};
  int step[3]{};
  float t_max[3]{}, t_delta[3]{};
  size_t remaining = 0;
  bool done = false;

  RayCaster(const float* start, const float* end_pt, float v) {
    cur = global_index(start, v);
    end = global_index(end_pt, v);
    const float dir[3] = {end_pt[0] - start[0], end_pt[1] - start[1], end_pt[2] - start[2]};
    size_t span = 0;
    for (int i = 0; i < 3; ++i) {
      step[i] = dir[i] > 0.0f ? 1 : (dir[i] < 0.0f ? -1 : 0);
      if (step[i] == 0) {
        t_max[i] = std::numeric_limits<float>::infinity();
        t_delta[i] = std::numeric_limits<float>::infinity();
      } else {
        const float boundary = static_cast<float>(cur[i] + (step[i] > 0 ? 1 : 0)) * v;
        t_max[i] = (boundary - start[i]) / dir[i];
        t_delta[i] = v / std::fabs(dir[i]);
      }
      span += static_cast<size_t>(std::abs(end[i] - cur[i]));
    }
    remaining = span + 1;
  }

  bool next(Key3* out) {
    if (done || remaining == 0) return false;
    *out = cur;
    --remaining;
    if (cur == end) {
      done = true;
      return true;
    }
    int axis = 0;
    if (t_max[1] < t_max[axis]) axis = 1;
    if (t_max[2] < t_max[axis]) axis = 2;
    cur[axis] += step[axis];
    t_max[axis] += t_delta[axis];
    return true;
  }
};

struct PointBucket {  // tsdf_integrator.h:90-95
  double wp[3] = {0.0, 0.0, 0.0};
  double wc[3] = {0.0, 0.0, 0.0};
  double weight = 0.0;
  size_t count = 0;
};

using BucketMap = std::unordered_map<Key3, PointBucket, TeschnerHash>;

}  // namespace

struct vxo_layer {
  float voxel_size;
  int vps;
  std::unordered_map<Key3, std::vector<vxg_voxel>, BlockKeyHash> blocks;
  std::vector<Key3> alloc_order;  // allocation sequence: rebuilds the reference's BlockMap iteration order

  // get_or_allocate_block (layer.h:79-87); default voxel all-zero (voxel.h:13-15).
  std::vector<vxg_voxel>& block(const Key3& b) {
    auto it = blocks.find(b);
    if (it == blocks.end()) {
      it = blocks.emplace(b, std::vector<vxg_voxel>(static_cast<size_t>(vps) * vps * vps, vxg_voxel{0.f, 0.f, 0, 0, 0, 0})).first;
      alloc_order.push_back(b);
    }
    return it->second;
  }
};

namespace {

struct TraceRec {  // one update_tsdf_voxel call, in reference order
  int32_t ray;
  int32_t g[3];
  float d;
  float w;
  uint32_t color;  // r | g<<8 | b<<16 | has_color<<31
};

struct Integrator {
  const vxg_tsdf_config& c;
  vxo_layer* layer;
  uint64_t raycasts = 0;
  std::vector<TraceRec>* trace = nullptr;  // test hook: record the update sequence
  Key3 cached_index{0, 0, 0};
  std::vector<vxg_voxel>* cached_block = nullptr;

  // cast_and_update (tsdf_integrator.cpp:129-173).
  uint64_t cast_and_update(const float* origin, const float* sp, float weight, const uint8_t* color,
                           const BucketMap* terminals, const Key3* own_terminal) {
    const float v = layer->voxel_size;
    const int vps = layer->vps;
    const float ray[3] = {sp[0] - origin[0], sp[1] - origin[1], sp[2] - origin[2]};
    const float depth = norm3(ray[0], ray[1], ray[2]);
    if (depth <= 0.0f) return 0;
    const float s = c.truncation / depth;
    const float ray_end[3] = {sp[0] + ray[0] * s, sp[1] + ray[1] * s, sp[2] + ray[2] * s};
    ++raycasts;
    uint64_t updates = 0;
    RayCaster caster(origin, ray_end, v);
    Key3 g;
    while (caster.next(&g)) {
      if (terminals != nullptr && g != *own_terminal && terminals->count(g) > 0) continue;
      // voxel_center (core.h:50-52)
      const float x[3] = {(static_cast<float>(g[0]) + 0.5f) * v, (static_cast<float>(g[1]) + 0.5f) * v,
                          (static_cast<float>(g[2]) + 0.5f) * v};
      const float d = projective_distance(x, sp, origin);
      const float w = measurement_weight(c.weight_mode, depth, d, c.truncation, c.dropoff_epsilon) * weight;
      if (w <= 0.0f) continue;
      // split_global_index (core.h:55-61)
      Key3 b, local;
      for (int i = 0; i < 3; ++i) {
        b[i] = floor_div(g[i], vps);
        local[i] = g[i] - b[i] * vps;
      }
      if (cached_block == nullptr || b != cached_index) {
        cached_block = &layer->block(b);
        cached_index = b;
      }
      const size_t lin = static_cast<size_t>(local[0]) +
                         static_cast<size_t>(vps) * (static_cast<size_t>(local[1]) + static_cast<size_t>(vps) * static_cast<size_t>(local[2]));
      update_voxel(&(*cached_block)[lin], d, w, c.truncation, c.max_weight, color);
      if (trace != nullptr) {
        const uint32_t col = color != nullptr ? (static_cast<uint32_t>(color[0]) | (static_cast<uint32_t>(color[1]) << 8) |
                                                 (static_cast<uint32_t>(color[2]) << 16) | 0x80000000u)
                                              : 0u;
        trace->push_back(TraceRec{static_cast<int32_t>(raycasts - 1), {g[0], g[1], g[2]}, d, w, col});
      }
      ++updates;
    }
    return updates;
  }
};

// Loop A of integrate_grouped (tsdf_integrator.cpp:196-220).
void build_buckets(const vxg_tsdf_config& c, float v, const float* xyz, const uint8_t* rgb, size_t n,
                   const float pose[12], BucketMap* buckets, uint64_t* skipped) {
  const float origin[3] = {pose[3], pose[7], pose[11]};
  buckets->reserve(n / 4 + 1);
  const int bucket_mode = c.weight_mode == VXG_WEIGHT_CONSTANT ? VXG_WEIGHT_CONSTANT : VXG_WEIGHT_INVERSE_Z2;
  for (size_t i = 0; i < n; ++i) {
    float p[3];
    transform_point(pose, xyz + 3 * i, p);
    const float depth = norm3(p[0] - origin[0], p[1] - origin[1], p[2] - origin[2]);
    if (depth < c.min_ray_length || depth > c.max_ray_length) {
      ++*skipped;
      continue;
    }
    const float w = measurement_weight(bucket_mode, depth, 0.0f, c.truncation, c.dropoff_epsilon);
    PointBucket& b = (*buckets)[global_index(p, v)];
    for (int k = 0; k < 3; ++k) b.wp[k] += static_cast<double>(w) * static_cast<double>(p[k]);
    if (rgb != nullptr) {
      for (int k = 0; k < 3; ++k) b.wc[k] += static_cast<double>(w) * static_cast<double>(rgb[3 * i + k]);
    }
    b.weight += w;
    ++b.count;
  }
}

}  // namespace

extern "C" {

void vxo_config_default(vxg_tsdf_config* c) {
  c->truncation = 0.4f;
  c->dropoff_epsilon = 0.1f;
  c->max_weight = 1e4f;
  c->weight_mode = VXG_WEIGHT_INVERSE_Z2_DROPOFF;
  c->merge_mode = VXG_MERGE_GROUPED;
  c->min_ray_length = 0.05f;
  c->max_ray_length = 10.0f;
}

void vxo_config_for_voxel_size(vxg_tsdf_config* c, float v) {
  vxo_config_default(c);
  c->truncation = 4.0f * v;
  c->dropoff_epsilon = v;
}

int vxo_config_validate(const vxg_tsdf_config* c, char* err, size_t err_len) {
  const char* msg = nullptr;
  if (!(c->dropoff_epsilon > 0.0f) || !(c->dropoff_epsilon < c->truncation)) {
    msg = "tsdf config requires 0 < dropoff_epsilon < truncation";
  } else if (!(c->min_ray_length >= 0.0f) || !(c->min_ray_length < c->max_ray_length)) {
    msg = "tsdf config requires 0 <= min_ray_length < max_ray_length";
  } else if (!(c->max_weight > 0.0f)) {
    msg = "tsdf config requires max_weight > 0";
  } else if (c->weight_mode < 0 || c->weight_mode > 2 || c->merge_mode < 0 || c->merge_mode > 2) {
    msg = "tsdf config has an unknown weight or merge mode";
  }
  if (msg == nullptr) return VXG_OK;
  if (err != nullptr && err_len > 0) {
    std::strncpy(err, msg, err_len - 1);
    err[err_len - 1] = '\0';
  }
  return VXG_EINVAL;
}

vxo_layer* vxo_layer_create(float voxel_size, int vps) {
  if (voxel_size <= 0.0f || vps < 1) return nullptr;  // layer.h:62-67
  auto* l = new vxo_layer;
  l->voxel_size = voxel_size;
  l->vps = vps;
  return l;
}

void vxo_layer_destroy(vxo_layer* l) { delete l; }

size_t vxo_block_count(const vxo_layer* l) { return l->blocks.size(); }

static std::vector<TraceRec>* g_trace = nullptr;

int vxo_integrate(vxo_layer* l, const vxg_tsdf_config* c, const float* xyz, const uint8_t* rgb, size_t n,
                  const float pose[12], vxg_stats* out) {
  if (vxo_config_validate(c, nullptr, 0) != VXG_OK) return VXG_EINVAL;
  Integrator it{*c, l};
  it.trace = g_trace;
  const float origin[3] = {pose[3], pose[7], pose[11]};
  uint64_t updates = 0, skipped = 0;
  if (c->merge_mode == VXG_MERGE_SIMPLE) {
    // integrate_simple (tsdf_integrator.cpp:175-190)
    for (size_t i = 0; i < n; ++i) {
      float p[3];
      transform_point(pose, xyz + 3 * i, p);
      const float depth = norm3(p[0] - origin[0], p[1] - origin[1], p[2] - origin[2]);
      if (depth < c->min_ray_length || depth > c->max_ray_length) {
        ++skipped;
        continue;
      }
      updates += it.cast_and_update(origin, p, 1.0f, rgb != nullptr ? rgb + 3 * i : nullptr, nullptr, nullptr);
    }
  } else {
    // integrate_grouped (tsdf_integrator.cpp:192-246)
    const bool anti_graze = c->merge_mode == VXG_MERGE_GROUPED_ANTI_GRAZE;
    BucketMap buckets;
    build_buckets(*c, l->voxel_size, xyz, rgb, n, pose, &buckets, &skipped);
    const int bucket_mode = c->weight_mode == VXG_WEIGHT_CONSTANT ? VXG_WEIGHT_CONSTANT : VXG_WEIGHT_INVERSE_Z2;
    for (const auto& [terminal, b] : buckets) {  // Loop B, map iteration order
      if (b.weight <= 0.0) continue;
      const float mean[3] = {static_cast<float>(b.wp[0] / b.weight), static_cast<float>(b.wp[1] / b.weight),
                             static_cast<float>(b.wp[2] / b.weight)};
      uint8_t color[3] = {0, 0, 0};
      if (rgb != nullptr) {
        for (int k = 0; k < 3; ++k) {
          const double cc = b.wc[k] / b.weight;
          color[k] = static_cast<uint8_t>(std::clamp(std::lround(cc), 0l, 255l));
        }
      }
      const float z = norm3(mean[0] - origin[0], mean[1] - origin[1], mean[2] - origin[2]);
      const float base_weight = static_cast<float>(b.weight) /
                                measurement_weight(bucket_mode, z, 0.0f, c->truncation, c->dropoff_epsilon);
      updates += it.cast_and_update(origin, mean, base_weight, rgb != nullptr ? color : nullptr,
                                    anti_graze ? &buckets : nullptr, &terminal);
    }
  }
  if (out != nullptr) {
    out->updates = updates;
    out->raycasts = it.raycasts;
    out->skipped = skipped;
  }
  return VXG_OK;
}

// Test hook: integrates one scan like vxo_integrate and returns the ordered
// sequence of update_tsdf_voxel calls as records of 7 x 32-bit words
// (ray index in ray order, gx, gy, gz, d (f32 bits), w (f32 bits), colour).
size_t vxo_trace_updates(vxo_layer* l, const vxg_tsdf_config* c, const float* xyz, const uint8_t* rgb, size_t n,
                         const float pose[12], uint32_t* out, size_t cap) {
  std::vector<TraceRec> tr;
  g_trace = &tr;
  vxg_stats st;
  vxo_integrate(l, c, xyz, rgb, n, pose, &st);
  g_trace = nullptr;
  for (size_t i = 0; i < tr.size() && i < cap; ++i) {
    uint32_t* o = out + 7 * i;
    o[0] = static_cast<uint32_t>(tr[i].ray);
    o[1] = static_cast<uint32_t>(tr[i].g[0]);
    o[2] = static_cast<uint32_t>(tr[i].g[1]);
    o[3] = static_cast<uint32_t>(tr[i].g[2]);
    std::memcpy(&o[4], &tr[i].d, 4);
    std::memcpy(&o[5], &tr[i].w, 4);
    o[6] = tr[i].color;
  }
  return tr.size();
}

size_t vxo_export_blocks(const vxo_layer* l, int32_t* idx, vxg_voxel* voxels, size_t cap) {
  std::vector<Key3> order;
  order.reserve(l->blocks.size());
  for (const auto& kv : l->blocks) order.push_back(kv.first);
  std::sort(order.begin(), order.end());  // (x,y,z) lexicographic, serialization.cpp:150-156
  const size_t nv = static_cast<size_t>(l->vps) * l->vps * l->vps;
  size_t k = 0;
  for (; k < order.size() && k < cap; ++k) {
    if (idx != nullptr) {
      idx[3 * k + 0] = order[k][0];
      idx[3 * k + 1] = order[k][1];
      idx[3 * k + 2] = order[k][2];
    }
    if (voxels != nullptr) std::memcpy(voxels + k * nv, l->blocks.at(order[k]).data(), nv * sizeof(vxg_voxel));
  }
  return k;
}

int vxo_voxel(const vxo_layer* l, int32_t gx, int32_t gy, int32_t gz, vxg_voxel* out) {
  const int vps = l->vps;
  const Key3 g{gx, gy, gz};
  Key3 b, local;
  for (int i = 0; i < 3; ++i) {
    b[i] = floor_div(g[i], vps);
    local[i] = g[i] - b[i] * vps;
  }
  auto it = l->blocks.find(b);
  if (it == l->blocks.end()) return 0;
  *out = it->second[static_cast<size_t>(local[0]) + vps * (static_cast<size_t>(local[1]) + vps * static_cast<size_t>(local[2]))];
  return 1;
}

int vxo_set_block(vxo_layer* l, const int32_t idx[3], const vxg_voxel* voxels) {
  auto& blk = l->block(Key3{idx[0], idx[1], idx[2]});
  std::memcpy(blk.data(), voxels, blk.size() * sizeof(vxg_voxel));
  return VXG_OK;
}

size_t vxo_save_vxblx(const vxo_layer* l, uint8_t* buf, size_t cap) {
  const size_t nv = static_cast<size_t>(l->vps) * l->vps * l->vps;
  const size_t need = 6 + 4 + 8 + 4 + 1 + 8 + l->blocks.size() * (24 + nv * 12);
  if (buf == nullptr || cap < need) return need;
  uint8_t* o = buf;
  auto put = [&](const void* src, size_t len) {  // little-endian host (x86-64)
    std::memcpy(o, src, len);
    o += len;
  };
  const char magic[6] = {'V', 'X', 'B', 'L', 'X', '\0'};
  const uint32_t version = 1;
  const double vs = static_cast<double>(l->voxel_size);
  const uint32_t vps = static_cast<uint32_t>(l->vps);
  const uint8_t kind = 0;
  const uint64_t count = l->blocks.size();
  put(magic, 6);
  put(&version, 4);
  put(&vs, 8);
  put(&vps, 4);
  put(&kind, 1);
  put(&count, 8);
  std::vector<Key3> order;
  for (const auto& kv : l->blocks) order.push_back(kv.first);
  std::sort(order.begin(), order.end());
  for (const Key3& k : order) {
    for (int i = 0; i < 3; ++i) {
      const int64_t v = k[i];
      put(&v, 8);
    }
    for (const vxg_voxel& vx : l->blocks.at(k)) {
      put(&vx.distance, 4);
      put(&vx.weight, 4);
      const uint8_t rgbp[4] = {vx.r, vx.g, vx.b, 0};
      put(rgbp, 4);
    }
  }
  return need;
}

float vxo_projective_distance(const float x[3], const float p[3], const float s[3]) {
  return projective_distance(x, p, s);
}

float vxo_measurement_weight(int mode, float z, float d, float truncation, float eps) {
  return measurement_weight(mode, z, d, truncation, eps);
}

void vxo_update_voxel(vxg_voxel* v, float d, float w, float truncation, float max_weight, const uint8_t* color) {
  update_voxel(v, d, w, truncation, max_weight, color);
}

size_t vxo_raycast(const float start[3], const float end[3], float voxel_size, int32_t* out, size_t cap) {
  RayCaster caster(start, end, voxel_size);
  Key3 g;
  size_t k = 0;
  while (caster.next(&g)) {
    if (k < cap) {
      out[3 * k + 0] = g[0];
      out[3 * k + 1] = g[1];
      out[3 * k + 2] = g[2];
    }
    ++k;
  }
  return k;
}

void vxo_global_index(const float p[3], float voxel_size, int32_t out[3]) {
  const Key3 g = global_index(p, voxel_size);
  out[0] = g[0];
  out[1] = g[1];
  out[2] = g[2];
}

uint64_t vxo_index_hash(int32_t x, int32_t y, int32_t z) { return TeschnerHash()(Key3{x, y, z}); }

size_t vxo_grouped_ray_order(const vxg_tsdf_config* c, float voxel_size, const float* xyz, size_t n,
                             const float pose[12], int32_t* keys, size_t cap) {
  BucketMap buckets;
  uint64_t skipped = 0;
  build_buckets(*c, voxel_size, xyz, nullptr, n, pose, &buckets, &skipped);
  size_t k = 0;
  for (const auto& kv : buckets) {
    if (k < cap) {
      keys[3 * k + 0] = kv.first[0];
      keys[3 * k + 1] = kv.first[1];
      keys[3 * k + 2] = kv.first[2];
    }
    ++k;
  }
  return k;
}

size_t vxo_bucket_schedule(size_t n_points, size_t max_keys, uint64_t* out, size_t cap) {
  struct Ident {
    size_t operator()(uint64_t k) const { return static_cast<size_t>(k); }
  };
  std::unordered_map<uint64_t, char, Ident> m;
  m.reserve(n_points / 4 + 1);
  size_t e = 0;
  auto emit = [&](uint64_t before, uint64_t bc) {
    if (e < cap) {
      out[2 * e] = before;
      out[2 * e + 1] = bc;
    }
    ++e;
  };
  emit(0, m.bucket_count());
  for (size_t k = 0; k < max_keys; ++k) {
    const size_t before = m.bucket_count();
    m.emplace(k, 0);
    if (m.bucket_count() != before) emit(k, m.bucket_count());
  }
  return e;
}

}  // extern "C"

// ---------------------------------------------------------------- read-side consumers
// interpolate_distance (interpolation.h:28-60): q = p/v - 0.5 per axis (Eigen
// Vector3f / scalar then - Constant), base = floor(q), frac = q - base; absent
// when any of the 8 corners is unallocated or unobserved (weight <= 1e-4,
// voxel.h:17, core.h:32); lerp along x, then y, then z, no FMA.
static int oracle_interp(const vxo_layer* l, const float* p, float* out) {
  const float v = l->voxel_size;
  float q[3], frac[3];
  int32_t base[3];
  for (int i = 0; i < 3; ++i) {
    q[i] = p[i] / v - 0.5f;
    base[i] = static_cast<int32_t>(std::floor(q[i]));
    frac[i] = q[i] - static_cast<float>(base[i]);
  }
  float corner[2][2][2];
  for (int dz = 0; dz < 2; ++dz)
    for (int dy = 0; dy < 2; ++dy)
      for (int dx = 0; dx < 2; ++dx) {
        vxg_voxel vx;
        if (!vxo_voxel(l, base[0] + dx, base[1] + dy, base[2] + dz, &vx) || !(vx.weight > 1e-4f)) return 0;
        corner[dx][dy][dz] = vx.distance;
      }
  float plane[2][2];
  for (int dy = 0; dy < 2; ++dy)
    for (int dz = 0; dz < 2; ++dz) {
      const float diff = corner[1][dy][dz] - corner[0][dy][dz];
      const float prod = frac[0] * diff;
      plane[dy][dz] = corner[0][dy][dz] + prod;
    }
  float line[2];
  for (int dz = 0; dz < 2; ++dz) {
    const float diff = plane[1][dz] - plane[0][dz];
    const float prod = frac[1] * diff;
    line[dz] = plane[0][dz] + prod;
  }
  const float diff = line[1] - line[0];
  const float prod = frac[2] * diff;
  *out = line[0] + prod;
  return 1;
}

extern "C" void vxo_interpolate(const vxo_layer* l, const float* pts, size_t n, float* d, uint8_t* found) {
  for (size_t i = 0; i < n; ++i) {
    float r = 0.0f;
    found[i] = static_cast<uint8_t>(oracle_interp(l, pts + 3 * i, &r));
    d[i] = found[i] ? r : 0.0f;
  }
}

// surface_error (analysis.cpp:41-59, Accumulator :16-37): fp64 sequential sums
// in point order of clamp(d, -truncation, truncation).
extern "C" void vxo_surface_error(const vxo_layer* l, const float* pts, size_t n, float truncation, double out[5]) {
  double sum = 0.0, sum_sq = 0.0, max_abs = 0.0;
  size_t count = 0, unknown = 0;
  for (size_t i = 0; i < n; ++i) {
    float r;
    if (!oracle_interp(l, pts + 3 * i, &r)) {
      ++unknown;
      continue;
    }
    const float c = r < -truncation ? -truncation : (truncation < r ? truncation : r);
    const double e = static_cast<double>(c);
    sum += e;
    sum_sq += e * e;
    max_abs = std::max(max_abs, std::abs(e));
    ++count;
  }
  out[0] = count ? std::sqrt(sum_sq / static_cast<double>(count)) : 0.0;
  out[1] = count ? sum / static_cast<double>(count) : 0.0;
  out[2] = count ? max_abs : 0.0;
  out[3] = static_cast<double>(count);
  out[4] = n ? static_cast<double>(unknown) / static_cast<double>(n) : 0.0;
}

// ---------------------------------------------------------------- meshing
// MeshExtractor::extract_block (mesh_extractor.cpp:85-151), restated with plain
// floats (the Eigen operations it uses are per-component; cross and norm in the
// shim's order), case tables from the caller.
namespace {

struct McCorner {
  int32_t g[3];
  float d;
  uint8_t rgb[3];
};

// edge_vertex (mesh_extractor.cpp:21-39): interpolate from the corner with the
// lower (x, y, z) global index so shared edges agree bitwise.
void mc_edge_vertex(const McCorner& a, const McCorner& b, float v, float* pos, uint8_t* col) {
  const McCorner* lo = &a;
  const McCorner* hi = &b;
  if (std::lexicographical_compare(hi->g, hi->g + 3, lo->g, lo->g + 3)) std::swap(lo, hi);
  const float t = lo->d / (lo->d - hi->d);
  for (int i = 0; i < 3; ++i) {
    const float plo = (static_cast<float>(lo->g[i]) + 0.5f) * v;  // voxel_center (core.h:50-52)
    const float phi = (static_cast<float>(hi->g[i]) + 0.5f) * v;
    const float diff = phi - plo;
    const float step = t * diff;
    pos[i] = plo + step;
    const float clo = static_cast<float>(lo->rgb[i]);
    const float span = static_cast<float>(hi->rgb[i]) - clo;
    const float blend = clo + t * span;
    const long r = std::lround(blend);
    col[i] = static_cast<uint8_t>(std::clamp(r, 0l, 255l));
  }
}

float mc_norm(const float* a) {
  const float s12 = a[1] * a[1] + a[2] * a[2];
  return std::sqrt(a[0] * a[0] + s12);
}

// vertex_normal (mesh_extractor.cpp:69-83)
void mc_vertex_normal(const vxo_layer* l, const float* p, const float* face, float* out) {
  const float h = l->voxel_size;
  float grad[3];
  for (int i = 0; i < 3; ++i) {
    float lo[3] = {p[0], p[1], p[2]}, hi[3] = {p[0], p[1], p[2]};
    lo[i] -= h;
    hi[i] += h;
    float dlo, dhi;
    const int flo = oracle_interp(l, lo, &dlo);
    const int fhi = oracle_interp(l, hi, &dhi);
    if (!flo || !fhi) {
      std::memcpy(out, face, 3 * sizeof(float));
      return;
    }
    grad[i] = (dhi - dlo) / (2.0f * h);
  }
  const float n = mc_norm(grad);
  if (n < 1e-10f) {
    std::memcpy(out, face, 3 * sizeof(float));
    return;
  }
  for (int i = 0; i < 3; ++i) out[i] = grad[i] / n;
}

struct McOut {
  std::vector<float> v, n;
  std::vector<uint8_t> c;
};

void mc_extract_block(const vxo_layer* l, const vxg_mc_tables* t, bool with_colors, const Key3& b, McOut* out) {
  const int vps = l->vps;
  const float v = l->voxel_size;
  McCorner corners[8];
  for (int z = 0; z < vps; ++z)
    for (int y = 0; y < vps; ++y)
      for (int x = 0; x < vps; ++x) {
        int config = 0;
        bool complete = true;
        for (int c = 0; c < 8 && complete; ++c) {
          const int32_t g[3] = {b[0] * vps + x + t->corner_offsets[c][0], b[1] * vps + y + t->corner_offsets[c][1],
                                b[2] * vps + z + t->corner_offsets[c][2]};
          vxg_voxel vx;
          if (!vxo_voxel(l, g[0], g[1], g[2], &vx) || !(vx.weight > 1e-4f)) {  // voxel_ptr / observed()
            complete = false;
            break;
          }
          corners[c] = McCorner{{g[0], g[1], g[2]}, vx.distance, {vx.r, vx.g, vx.b}};
          if (vx.distance < 0.0f) config |= 1 << c;
        }
        if (!complete || t->edge_table[config] == 0) continue;
        float ep[12][3];
        uint8_t ec[12][3];
        for (int e = 0; e < 12; ++e)
          if (t->edge_table[config] & (1 << e))
            mc_edge_vertex(corners[t->edge_corners[e][0]], corners[t->edge_corners[e][1]], v, ep[e], ec[e]);
        for (int k = 0; t->tri_table[config][k] != -1; k += 3) {
          // table winding faces the negative side: (e0, e2, e1) (:116-122)
          const int es[3] = {t->tri_table[config][k], t->tri_table[config][k + 2], t->tri_table[config][k + 1]};
          const float* p0 = ep[es[0]];
          const float* p1 = ep[es[1]];
          const float* p2 = ep[es[2]];
          const float a[3] = {p1[0] - p0[0], p1[1] - p0[1], p1[2] - p0[2]};
          const float c[3] = {p2[0] - p0[0], p2[1] - p0[1], p2[2] - p0[2]};
          float fnv[3];
          for (int i = 0; i < 3; ++i) {  // cross product, component i = a_j c_k - a_k c_j
            const int j = (i + 1) % 3, kk = (i + 2) % 3;
            const float m1 = a[j] * c[kk];
            const float m2 = a[kk] * c[j];
            fnv[i] = m1 - m2;
          }
          const float fn = mc_norm(fnv);
          if (fn > 1e-12f) {
            for (int i = 0; i < 3; ++i) fnv[i] = fnv[i] / fn;
          } else {
            fnv[0] = 0.0f;
            fnv[1] = 0.0f;
            fnv[2] = 1.0f;
          }
          for (int q = 0; q < 3; ++q) {
            const float* p = ep[es[q]];
            float nrm[3];
            mc_vertex_normal(l, p, fnv, nrm);
            out->v.insert(out->v.end(), p, p + 3);
            out->n.insert(out->n.end(), nrm, nrm + 3);
            if (with_colors) out->c.insert(out->c.end(), ec[es[q]], ec[es[q]] + 3);
          }
        }
      }
}

}  // namespace

extern "C" size_t vxo_mesh_extract(const vxo_layer* l, const vxg_mc_tables* t, int with_colors, const int32_t* blocks,
                                   size_t n_req, int32_t* bidx, uint64_t* frag_tri, float* verts, float* normals,
                                   uint8_t* colors, size_t cap_frag, size_t cap_tri, uint64_t* n_tri) {
  std::vector<Key3> order;
  if (blocks == nullptr) {
    for (const auto& kv : l->blocks) order.push_back(kv.first);
  } else {
    for (size_t i = 0; i < n_req; ++i) {
      const Key3 k{blocks[3 * i], blocks[3 * i + 1], blocks[3 * i + 2]};
      if (l->blocks.count(k)) order.push_back(k);
    }
  }
  std::sort(order.begin(), order.end());
  order.erase(std::unique(order.begin(), order.end()), order.end());
  McOut out;
  std::vector<uint64_t> frag(order.size() + 1, 0);
  for (size_t j = 0; j < order.size(); ++j) {
    mc_extract_block(l, t, with_colors != 0, order[j], &out);
    frag[j + 1] = out.v.size() / 9;
  }
  const uint64_t T = frag.back();
  *n_tri = T;
  if (cap_frag >= order.size() && cap_tri >= T) {
    for (size_t j = 0; j < order.size(); ++j)
      for (int a = 0; a < 3; ++a)
        if (bidx) bidx[3 * j + a] = order[j][a];
    if (frag_tri) std::memcpy(frag_tri, frag.data(), frag.size() * sizeof(uint64_t));
    if (verts && T) std::memcpy(verts, out.v.data(), 9 * T * sizeof(float));
    if (normals && T) std::memcpy(normals, out.n.data(), 9 * T * sizeof(float));
    if (colors && with_colors && T) std::memcpy(colors, out.c.data(), 9 * T);
  }
  return order.size();
}

// ---------------------------------------------------------------- ESDF (occupancy-seeded baseline)
// Restatement of EsdfIntegrator::build_from_occupancy (esdf_integrator.cpp:303-330)
// with the reference's queue semantics, so parents (order-dependent under ties)
// come out exactly as the reference's.
namespace {

constexpr uint8_t kEsdfObserved = 1, kEsdfFixed = 2, kEsdfInLower = 8;  // voxel.h:24-27

struct EsdfVox {  // voxel.h:22-48 (parent kept as int16 like the reference)
  float distance;
  int16_t parent[3];
  uint8_t flags;
};

struct EsdfWave {  // WavefrontQueue (esdf_integrator.cpp:20-52)
  int mode;
  float bucket_width;
  std::vector<std::vector<Key3>> buckets;  // FIFO per bucket: vector + read head
  std::vector<size_t> heads;
  std::vector<Key3> fifo;
  size_t fifo_head = 0;
  size_t cursor = 0, size = 0;
  EsdfWave(int m, float bw, float d_max) : mode(m), bucket_width(bw) {
    if (mode != VXG_QUEUE_FIFO) {
      const size_t n = static_cast<size_t>(std::ceil(d_max / bucket_width)) + 1;
      buckets.resize(n);
      heads.assign(n, 0);
    }
  }
  void push(const Key3& g, float priority) {
    if (mode == VXG_QUEUE_FIFO) {
      fifo.push_back(g);
    } else {
      size_t b = static_cast<size_t>(std::fabs(priority) / bucket_width);
      if (b >= buckets.size()) b = buckets.size() - 1;
      buckets[b].push_back(g);
      if (b < cursor) cursor = b;
    }
    ++size;
  }
  bool pop(Key3* g) {
    if (size == 0) return false;
    if (mode == VXG_QUEUE_FIFO) {
      *g = fifo[fifo_head++];
    } else {
      while (heads[cursor] == buckets[cursor].size()) ++cursor;
      *g = buckets[cursor][heads[cursor]++];
    }
    --size;
    return true;
  }
};

}  // namespace

extern "C" size_t vxo_esdf_occupancy(const vxo_layer* l, const vxg_esdf_config* c, uint8_t* buf, size_t cap,
                                     char* err, size_t err_len) {
  auto fail = [&](const char* m) -> size_t {
    if (err && err_len) {
      std::strncpy(err, m, err_len - 1);
      err[err_len - 1] = 0;
    }
    return 0;
  };
  const float v = l->voxel_size;
  const int vps = l->vps;
  // EsdfConfig::band_radius (esdf_integrator.h:36-38) + validate (:10-18)
  const float gamma = c->band_mode == VXG_BAND_ONE_VOXEL ? v : 0.5f * c->truncation;
  if (!(gamma > 0.0f) || !(gamma <= c->truncation)) return fail("esdf config requires 0 < band radius <= truncation");
  if (!(c->d_max > gamma)) return fail("esdf config requires d_max > band radius");
  // neighbours in the constructor's order (:69-79): dz, dy, dx in -1..1
  struct Nb {
    int dx, dy, dz;
    float step;
  };
  std::vector<Nb> nbs;
  for (int dz = -1; dz <= 1; ++dz)
    for (int dy = -1; dy <= 1; ++dy)
      for (int dx = -1; dx <= 1; ++dx) {
        if (dx == 0 && dy == 0 && dz == 0) continue;
        nbs.push_back({dx, dy, dz, v * std::sqrt(static_cast<float>(dx * dx + dy * dy + dz * dz))});
      }
  const size_t nv = static_cast<size_t>(vps) * vps * vps;
  std::unordered_map<Key3, std::vector<EsdfVox>, BlockKeyHash> esdf;
  const EsdfVox def{c->d_max, {0, 0, 0}, 0};  // default voxel (:81-83)
  auto vox = [&](const Key3& g) -> EsdfVox* {  // esdf_voxel (:86-97)
    const Key3 b{floor_div(g[0], vps), floor_div(g[1], vps), floor_div(g[2], vps)};
    auto it = esdf.find(b);
    if (it == esdf.end()) return nullptr;
    const int lx = g[0] - b[0] * vps, ly = g[1] - b[1] * vps, lz = g[2] - b[2] * vps;
    return &it->second[static_cast<size_t>(lx + vps * (ly + vps * lz))];
  };
  const float bw = c->bucket_width > 0.0f ? c->bucket_width : v;
  EsdfWave lower(c->queue_mode, bw, c->d_max);
  auto push_lower = [&](const Key3& g, EsdfVox* e) {  // :99-105
    if (c->queue_mode != VXG_QUEUE_PRIORITY_MULTI) {
      if (e->flags & kEsdfInLower) return;
      e->flags |= kEsdfInLower;
    }
    lower.push(g, std::fabs(e->distance));
  };
  // seeding (:310-326), in the reference TSDF layer's block iteration order:
  // IndexMap = unordered_map with IndexHash (core.h:68-85) filled in allocation order
  std::unordered_map<Key3, int, TeschnerHash> ref_order;
  for (const Key3& b : l->alloc_order) ref_order.emplace(b, 0);
  for (const auto& kv : ref_order) esdf.emplace(kv.first, std::vector<EsdfVox>(nv, def));
  for (const auto& kr : ref_order) {
    const auto& kv = *l->blocks.find(kr.first);
    std::vector<EsdfVox>& eb = esdf.at(kv.first);
    for (size_t lin = 0; lin < nv; ++lin) {
      const vxg_voxel& tv = kv.second[lin];
      if (!(tv.weight > 1e-4f)) continue;  // observed (core.h:32)
      EsdfVox& ev = eb[lin];
      ev.flags |= kEsdfObserved;
      if (tv.distance < 0.0f) {
        ev.distance = 0.0f;
        ev.flags |= kEsdfFixed;
        const int lx = static_cast<int>(lin % vps), ly = static_cast<int>((lin / vps) % vps),
                  lz = static_cast<int>(lin / (static_cast<size_t>(vps) * vps));
        push_lower(Key3{kv.first[0] * vps + lx, kv.first[1] * vps + ly, kv.first[2] * vps + lz}, &ev);
      } else {
        ev.distance = c->d_max;
      }
    }
  }
  // process_lower_queue (:220-230) + relax_neighbors (:232-294)
  Key3 g;
  while (lower.pop(&g)) {
    EsdfVox* e = vox(g);
    e->flags &= static_cast<uint8_t>(~kEsdfInLower);
    if (!(e->flags & kEsdfObserved)) continue;
    const EsdfVox cur = *e;
    float seed_value = 0.0f;
    const bool euclid = c->metric == VXG_METRIC_EUCLIDEAN;
    if (euclid) {
      const bool has_parent = cur.parent[0] != 0 || cur.parent[1] != 0 || cur.parent[2] != 0;
      if (has_parent) {
        const EsdfVox* seed = vox(Key3{g[0] + cur.parent[0], g[1] + cur.parent[1], g[2] + cur.parent[2]});
        if (seed != nullptr && (seed->flags & kEsdfFixed)) {
          seed_value = seed->distance;
        } else {
          const float len = v * std::sqrt(static_cast<float>(cur.parent[0] * cur.parent[0] +
                                                             cur.parent[1] * cur.parent[1] +
                                                             cur.parent[2] * cur.parent[2]));
          seed_value = cur.distance > 0.0f ? cur.distance - len : cur.distance + len;
        }
      } else {
        seed_value = cur.distance;
      }
    }
    for (const Nb& n : nbs) {
      const Key3 ng{g[0] + n.dx, g[1] + n.dy, g[2] + n.dz};
      EsdfVox* nv_ = vox(ng);
      if (nv_ == nullptr || !(nv_->flags & kEsdfObserved) || (nv_->flags & kEsdfFixed)) continue;
      float cpos, cneg;
      int16_t np[3];
      if (!euclid) {
        cpos = cur.distance + n.step;
        cneg = cur.distance - n.step;
        np[0] = static_cast<int16_t>(-n.dx);
        np[1] = static_cast<int16_t>(-n.dy);
        np[2] = static_cast<int16_t>(-n.dz);
      } else {
        np[0] = static_cast<int16_t>(cur.parent[0] - n.dx);
        np[1] = static_cast<int16_t>(cur.parent[1] - n.dy);
        np[2] = static_cast<int16_t>(cur.parent[2] - n.dz);
        const float sd = v * std::sqrt(static_cast<float>(np[0] * np[0] + np[1] * np[1] + np[2] * np[2]));
        cpos = seed_value + sd;
        cneg = seed_value - sd;
      }
      if (nv_->distance > 0.0f && cpos < nv_->distance) {
        nv_->distance = cpos;
        std::memcpy(nv_->parent, np, sizeof(np));
        push_lower(ng, nv_);
      } else if (nv_->distance < 0.0f && cneg > nv_->distance) {
        nv_->distance = cneg;
        std::memcpy(nv_->parent, np, sizeof(np));
        push_lower(ng, nv_);
      }
    }
  }
  // save_layer (serialization.cpp:141-168) with the ESDF payload (:116-122)
  const size_t need = 6 + 4 + 8 + 4 + 1 + 8 + esdf.size() * (24 + nv * 8);
  if (buf == nullptr || cap < need) return need;
  uint8_t* o = buf;
  auto put = [&](const void* src, size_t len) {
    std::memcpy(o, src, len);
    o += len;
  };
  const char magic[6] = {'V', 'X', 'B', 'L', 'X', '\0'};
  const uint32_t version = 1;
  const double vs = static_cast<double>(v);
  const uint32_t vps32 = static_cast<uint32_t>(vps);
  const uint8_t kind = 1;
  const uint64_t count = esdf.size();
  put(magic, 6);
  put(&version, 4);
  put(&vs, 8);
  put(&vps32, 4);
  put(&kind, 1);
  put(&count, 8);
  std::vector<Key3> order;
  for (const auto& kv : esdf) order.push_back(kv.first);
  std::sort(order.begin(), order.end());
  for (const Key3& k : order) {
    for (int i = 0; i < 3; ++i) {
      const int64_t x = k[i];
      put(&x, 8);
    }
    for (const EsdfVox& e : esdf.at(k)) {
      put(&e.distance, 4);
      uint8_t fp[4] = {e.flags, 0, 0, 0};
      for (int i = 0; i < 3; ++i) fp[1 + i] = static_cast<uint8_t>(static_cast<int8_t>(std::clamp<int>(e.parent[i], -128, 127)));
      put(fp, 4);
    }
  }
  return need;
}
