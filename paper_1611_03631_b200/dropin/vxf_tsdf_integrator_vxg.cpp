// Link-level drop-in for the reference's vxf::TsdfIntegrator
// (/root/reference/proj/include/vxf/tsdf_integrator.h), backed by the B200
// C ABI (include/vxg.h). Compile this file INSTEAD of the reference's
// src/tsdf_integrator.cpp and link libvxg.so: callers (cmd_integrate,
// run_sim_benchmark, the reference's tests) keep using vxf::TsdfIntegrator and
// vxf::TsdfLayer unchanged.
//
// Behaviour:
//  * the constructor validates the config with the reference's messages
//    (tsdf_integrator.cpp:10-20, :106-109);
//  * integrate() throws std::invalid_argument on a colour-size mismatch
//    (:115-117), integrates the scan on the GPU, then writes every block the
//    scan updated back into the caller's host TsdfLayer (allocating new blocks
//    through get_or_allocate_block and calling mark_updated, so host-side
//    consumers see the same updated-block sets, layer.h:124-130), and returns
//    the update count; raycasts_last_scan()/skipped_points_last_scan() match;
//  * the host layer is the source of truth between calls: if it was replaced
//    or gained blocks the device does not hold, it is re-uploaded (the
//    single-writer contract, layer.h:53-55, means it is otherwise unchanged).
//  * the free functions projective_distance / measurement_weight /
//    update_tsdf_voxel evaluate on the device (vxg_eval_*); RayCaster iterates
//    over the device walk (vxg_eval_raycast; not on the integration path).
#include <cmath>
#include <cstring>
#include <limits>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "vxf/tsdf_integrator.h"
#include "vxg.h"

namespace vxf {

namespace {

[[noreturn]] void fail(int rc) {
  const std::string msg = vxg_last_error();
  if (rc == VXG_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error("vxg: " + msg);
}

void check(int rc) {
  if (rc != VXG_OK) fail(rc);
}

vxg_tsdf_config to_c(const TsdfConfig& c) {
  vxg_tsdf_config o;
  o.truncation = c.truncation;
  o.dropoff_epsilon = c.dropoff_epsilon;
  o.max_weight = c.max_weight;
  o.weight_mode = static_cast<int32_t>(c.weight_mode);
  o.merge_mode = static_cast<int32_t>(c.merge_mode);
  o.min_ray_length = c.min_ray_length;
  o.max_ray_length = c.max_ray_length;
  return o;
}

constexpr const char* kConsumer = "__vxg_dropin";

struct Mirror {
  vxg_handle* h = nullptr;
  const TsdfLayer* layer = nullptr;
  float voxel_size = 0.f;
  int vps = 0;
  std::map<std::tuple<int, int, int>, const void*> fingerprint;  // block index -> Block* after last sync
  std::vector<int32_t> wb_idx;     // writeback scratch, kept across scans (no 10-20 MB
  std::vector<vxg_voxel> wb_vox;   // allocation + zero fill per scan)
  ~Mirror() {
    if (h) vxg_destroy(h);
  }
};

std::mutex g_mu;
std::map<const TsdfIntegrator*, std::unique_ptr<Mirror>> g_mirrors;

std::tuple<int, int, int> key3(const BlockIndex& b) { return {b.x(), b.y(), b.z()}; }

bool layer_matches(const Mirror& m, const TsdfLayer& layer) {
  if (m.layer != &layer || m.voxel_size != layer.voxel_size() || m.vps != layer.voxels_per_side()) return false;
  if (layer.block_count() != m.fingerprint.size()) return false;
  for (const auto& [idx, block] : layer.blocks()) {
    auto it = m.fingerprint.find(key3(idx));
    if (it == m.fingerprint.end() || it->second != block.get()) return false;
  }
  return true;
}

// Uploads the whole host layer (fresh handle).
void upload(Mirror& m, TsdfLayer& layer, const TsdfConfig& cfg) {
  if (m.h) vxg_destroy(m.h);
  m.h = nullptr;
  const vxg_tsdf_config c = to_c(cfg);
  check(vxg_create(&c, layer.voxel_size(), layer.voxels_per_side(), 0, 64, &m.h));
  check(vxg_register_consumer(m.h, kConsumer));
  m.layer = &layer;
  m.voxel_size = layer.voxel_size();
  m.vps = layer.voxels_per_side();
  m.fingerprint.clear();
  const size_t nv = static_cast<size_t>(m.vps) * m.vps * m.vps;
  std::vector<int32_t> idx;
  std::vector<vxg_voxel> vox;
  for (const auto& [bidx, block] : layer.blocks()) {
    idx.insert(idx.end(), {bidx.x(), bidx.y(), bidx.z()});
    for (size_t i = 0; i < nv; ++i) {
      const TsdfVoxel& v = block->voxel(i);
      vox.push_back(vxg_voxel{v.distance, v.weight, v.color.r, v.color.g, v.color.b, 0});
    }
    m.fingerprint[key3(bidx)] = block.get();
  }
  if (!idx.empty()) check(vxg_import_blocks(m.h, idx.data(), vox.data(), idx.size() / 3));
  uint64_t n = 0;  // imports count as updates for the device-side consumer; start clean
  check(vxg_drain_updated(m.h, kConsumer, nullptr, 0, &n));
  std::vector<int32_t> sink(3 * (n + 1));
  check(vxg_drain_updated(m.h, kConsumer, sink.data(), n, &n));
}

// Writes the blocks updated by the last scan back into the host layer: the
// drained block indices, then their payloads in one device gather + D2H
// (vxg_fetch_blocks), copied into the host blocks.
void download(Mirror& m, TsdfLayer& layer) {
  uint64_t n = 0;
  check(vxg_drain_updated(m.h, kConsumer, nullptr, 0, &n));
  std::vector<int32_t>& idx = m.wb_idx;
  if (idx.size() < 3 * (n + 1)) idx.resize(3 * (n + 1));
  check(vxg_drain_updated(m.h, kConsumer, idx.data(), n, &n));
  if (n == 0) return;
  const size_t nv = static_cast<size_t>(m.vps) * m.vps * m.vps;
  std::vector<vxg_voxel>& out = m.wb_vox;
  if (out.size() < nv * n) out.resize(nv * n);
  check(vxg_fetch_blocks(m.h, idx.data(), n, out.data(), nullptr));
  for (uint64_t b = 0; b < n; ++b) {
    const BlockIndex bidx(idx[3 * b], idx[3 * b + 1], idx[3 * b + 2]);
    Block<TsdfVoxel>& block = layer.get_or_allocate_block(bidx);
    layer.mark_updated(bidx);
    const vxg_voxel* src = out.data() + b * nv;
    for (size_t i = 0; i < nv; ++i) {
      TsdfVoxel& t = block.voxel(i);
      t.distance = src[i].distance;
      t.weight = src[i].weight;
      t.color = Color{src[i].r, src[i].g, src[i].b};
    }
    m.fingerprint[key3(bidx)] = &block;
  }
}

// The voxels of one walk, computed by the device DDA (vxg_eval_raycast); the
// last walk is cached per thread so RayCaster::next is a lookup.
struct Walk {
  float start[3] = {}, end[3] = {}, v = 0.f;
  bool valid = false;
  std::vector<int32_t> voxels;  // 3 per voxel, traversal order
};
thread_local Walk g_walk;

const Walk& device_walk(const float s[3], const float e[3], float v) {
  Walk& w = g_walk;
  if (w.valid && std::memcmp(w.start, s, sizeof(w.start)) == 0 && std::memcmp(w.end, e, sizeof(w.end)) == 0 &&
      std::memcmp(&w.v, &v, sizeof(v)) == 0)
    return w;
  uint32_t count = 0;
  check(vxg_eval_raycast(0, s, e, 1, v, &count, nullptr, nullptr));
  const uint64_t off = 0;
  w.voxels.assign(3 * static_cast<size_t>(count), 0);
  if (count > 0) check(vxg_eval_raycast(0, s, e, 1, v, &count, &off, w.voxels.data()));
  std::memcpy(w.start, s, sizeof(w.start));
  std::memcpy(w.end, e, sizeof(w.end));
  w.v = v;
  w.valid = true;
  return w;
}

}  // namespace

void TsdfConfig::validate() const {  // tsdf_integrator.cpp:10-20
  if (!(dropoff_epsilon > 0.0f) || !(dropoff_epsilon < truncation))
    throw std::invalid_argument("tsdf config requires 0 < dropoff_epsilon < truncation");
  if (!(min_ray_length >= 0.0f) || !(min_ray_length < max_ray_length))
    throw std::invalid_argument("tsdf config requires 0 <= min_ray_length < max_ray_length");
  if (!(max_weight > 0.0f)) throw std::invalid_argument("tsdf config requires max_weight > 0");
}

FloatingPoint projective_distance(const Point& x, const Point& p, const Point& s) {
  const float xs[3] = {x.x(), x.y(), x.z()}, ps[3] = {p.x(), p.y(), p.z()}, ss[3] = {s.x(), s.y(), s.z()};
  float out = 0.f;
  check(vxg_eval_projective_distance(0, xs, ps, ss, 1, &out));
  return out;
}

FloatingPoint measurement_weight(WeightMode mode, FloatingPoint z, FloatingPoint d, FloatingPoint truncation,
                                 FloatingPoint dropoff_epsilon) {
  float out = 0.f;
  check(vxg_eval_measurement_weight(0, static_cast<int>(mode), &z, &d, 1, truncation, dropoff_epsilon, &out));
  return out;
}

void update_tsdf_voxel(TsdfVoxel* voxel, FloatingPoint d, FloatingPoint w, FloatingPoint truncation,
                       FloatingPoint max_weight, const Color& color, bool has_color) {
  vxg_voxel v{voxel->distance, voxel->weight, voxel->color.r, voxel->color.g, voxel->color.b, 0};
  const uint64_t starts[2] = {0, 1};
  const uint8_t rgb[3] = {color.r, color.g, color.b};
  check(vxg_eval_update_voxels(0, &v, 1, starts, &d, &w, has_color ? rgb : nullptr, truncation, max_weight));
  voxel->distance = v.distance;
  voxel->weight = v.weight;
  voxel->color = Color{v.r, v.g, v.b};
}

void update_tsdf_voxel(TsdfVoxel* voxel, FloatingPoint d, FloatingPoint w, FloatingPoint truncation,
                       FloatingPoint max_weight) {
  update_tsdf_voxel(voxel, d, w, truncation, max_weight, Color{}, false);
}

// RayCaster (tsdf_integrator.cpp:69-104) as an adapter over the device walk:
// the members keep the segment (t_max_ = start, t_delta_ = end, step_[0] =
// the voxel size's bits), current_/end_ the first/terminal voxel and
// remaining_ the voxels still to visit; next() reads the walk the device
// computed for this segment (same voxels, same order, span + 1 of them).
RayCaster::RayCaster(const Point& start, const Point& end, FloatingPoint voxel_size) {
  const float s[3] = {start.x(), start.y(), start.z()}, e[3] = {end.x(), end.y(), end.z()};
  const Walk& w = device_walk(s, e, voxel_size);
  t_max_ = start;
  t_delta_ = end;
  int32_t vbits = 0;
  std::memcpy(&vbits, &voxel_size, sizeof(vbits));
  step_ = Eigen::Vector3i(vbits, 0, 0);
  remaining_ = w.voxels.size() / 3;
  if (remaining_ > 0) {
    current_ = GlobalVoxelIndex(w.voxels[0], w.voxels[1], w.voxels[2]);
    const size_t l = 3 * (remaining_ - 1);
    end_ = GlobalVoxelIndex(w.voxels[l], w.voxels[l + 1], w.voxels[l + 2]);
  }
}

bool RayCaster::next(GlobalVoxelIndex* index) {
  if (done_ || remaining_ == 0) return false;
  const float s[3] = {t_max_.x(), t_max_.y(), t_max_.z()}, e[3] = {t_delta_.x(), t_delta_.y(), t_delta_.z()};
  float v = 0.f;
  const int32_t vbits = step_[0];
  std::memcpy(&v, &vbits, sizeof(v));
  const Walk& w = device_walk(s, e, v);
  const size_t k = w.voxels.size() / 3 - remaining_;
  current_ = GlobalVoxelIndex(w.voxels[3 * k], w.voxels[3 * k + 1], w.voxels[3 * k + 2]);
  *index = current_;
  if (--remaining_ == 0) done_ = true;
  return true;
}

TsdfIntegrator::TsdfIntegrator(const TsdfConfig& config, TsdfLayer* layer) : config_(config), layer_(layer) {
  config_.validate();
  std::lock_guard<std::mutex> lock(g_mu);
  g_mirrors.erase(this);  // a previous integrator at this address is gone
}

size_t TsdfIntegrator::integrate(const Scan& scan) {
  raycasts_last_scan_ = 0;
  skipped_last_scan_ = 0;
  cached_block_ = nullptr;
  if (!scan.colors.empty() && scan.colors.size() != scan.points.size()) {
    throw std::invalid_argument("scan colors must parallel points");
  }
  std::lock_guard<std::mutex> lock(g_mu);
  std::unique_ptr<Mirror>& mp = g_mirrors[this];
  if (!mp) mp = std::make_unique<Mirror>();
  Mirror& m = *mp;
  if (m.h == nullptr || !layer_matches(m, *layer_)) upload(m, *layer_, config_);
  const vxg_tsdf_config c = to_c(config_);
  check(vxg_set_config(m.h, &c));
  const size_t n = scan.points.size();
  std::vector<float> xyz(3 * n);
  for (size_t i = 0; i < n; ++i) {
    xyz[3 * i + 0] = scan.points[i].x();
    xyz[3 * i + 1] = scan.points[i].y();
    xyz[3 * i + 2] = scan.points[i].z();
  }
  std::vector<uint8_t> rgb;
  if (scan.has_colors()) {
    rgb.resize(3 * n);
    for (size_t i = 0; i < n; ++i) {
      rgb[3 * i + 0] = scan.colors[i].r;
      rgb[3 * i + 1] = scan.colors[i].g;
      rgb[3 * i + 2] = scan.colors[i].b;
    }
  }
  float pose[12];
  for (int r = 0; r < 3; ++r) {
    for (int k = 0; k < 3; ++k) pose[4 * r + k] = scan.pose.linear()(r, k);
    pose[4 * r + 3] = scan.pose.translation()[r];
  }
  vxg_stats st{0, 0, 0};
  check(vxg_integrate(m.h, xyz.data(), rgb.empty() ? nullptr : rgb.data(), n, pose, &st));
  download(m, *layer_);
  raycasts_last_scan_ = st.raycasts;
  skipped_last_scan_ = st.skipped;
  return st.updates;
}

}  // namespace vxf
