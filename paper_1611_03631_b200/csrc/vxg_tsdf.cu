// Host orchestration of the B200 TSDF pipeline behind the C ABI (include/vxg.h).
//
// Per batch of frames (results identical to sequential per-frame integrate()):
//   simple : K1 range filter -> scan -> rays (point order)
//   grouped: K1 keys -> radix sort -> run-length -> K2 fp64 bucket reduce
//            -> K3 libstdc++ ray order (fo[bucket] atomicMin + sort) -> rays
//   common : ray span count -> scan -> K4 emit records (+ K6 block alloc)
//            -> K5 stable radix sort by voxel -> K7 ordered fold
// Sorting/scans use CUB (CCCL 2.8, header-only, compiled into this library).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <array>
#include <mutex>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <set>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <utility>
#include <vector>


#include "../../include/vxg.h"
#include "vxg_esdf.cuh"
#include "vxg_kernels.cuh"
#include "vxg_sort.cuh"

namespace vxg {
using Schedule = std::vector<std::pair<uint64_t, uint64_t>>;
Schedule bucket_schedule(uint64_t n_points, uint64_t max_keys);
}  // namespace vxg

using namespace vxg;

namespace {

thread_local std::string g_err;

}  // namespace

// vxg_last_error() for the other translation units of the library (scan I/O).
namespace vxg {
void set_last_error(const std::string& msg) { g_err = msg; }
}  // namespace vxg

namespace {

struct Status {
  int code;
  std::string msg;
};

struct VxgError : std::runtime_error {
  int code;
  VxgError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define CU(x)                                                                                   \
  do {                                                                                          \
    cudaError_t e_ = (x);                                                                       \
    if (e_ != cudaSuccess) {                                                                    \
      throw VxgError(VXG_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_));               \
    }                                                                                           \
  } while (0)

template <typename T>
struct DBuf {
  T* p = nullptr;
  size_t cap = 0;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() { release(); }
  void swap(DBuf& o) {
    std::swap(p, o.p);
    std::swap(cap, o.cap);
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
  // Grow-only; contents are NOT preserved.
  T* ensure(size_t n) {
    if (n <= cap && p) return p;
    release();
    size_t want = std::max<size_t>(n + n / 4, 256);
    CU(cudaMalloc(&p, want * sizeof(T)));
    cap = want;
    return p;
  }
};

constexpr int kStages = 9;
const char* kStageNames[kStages] = {"h2d",         "bundle", "ray_order", "ray_setup", "emit",
                                    "record_sort", "runs",   "apply",     "d2h"};
enum Stage { ST_H2D = 0, ST_BUNDLE, ST_ORDER, ST_RAYS, ST_EMIT, ST_SORT, ST_RUNS, ST_APPLY, ST_D2H };

int bits_for(uint64_t v) {  // smallest b with v < 2^b
  int b = 0;
  while (b < 64 && (v >> b) != 0) ++b;
  return b;
}

unsigned grid_for(uint64_t n, unsigned block = 256) {
  uint64_t g = (n + block - 1) / block;
  if (g < 1) g = 1;
  if (g > 148ull * 16) g = 148ull * 16;
  return static_cast<unsigned>(g);
}

std::string validate_config(const vxg_tsdf_config* c) {  // TsdfConfig::validate, tsdf_integrator.cpp:10-20
  if (!(c->dropoff_epsilon > 0.0f) || !(c->dropoff_epsilon < c->truncation))
    return "tsdf config requires 0 < dropoff_epsilon < truncation";
  if (!(c->min_ray_length >= 0.0f) || !(c->min_ray_length < c->max_ray_length))
    return "tsdf config requires 0 <= min_ray_length < max_ray_length";
  if (!(c->max_weight > 0.0f)) return "tsdf config requires max_weight > 0";
  if (c->weight_mode < 0 || c->weight_mode > 2 || c->merge_mode < 0 || c->merge_mode > 2)
    return "tsdf config has an unknown weight or merge mode";
  return "";
}

}  // namespace

struct vxg_handle {
  vxg_tsdf_config cfg{};
  float voxel_size = 0.f;
  int vps = 16;
  int nvox = 4096;
  int device = 0;
  cudaStream_t own = nullptr;
  cudaStream_t st = nullptr;
  cudaStream_t copy_st = nullptr;         // H2D staging of host inputs (overlaps compute)
  cudaStream_t fold_st = nullptr;         // short-run fold beside the long-run fold
  cudaEvent_t fold_fork = nullptr, fold_join = nullptr;
  // ---- chunk pipeline: chunk c's fold (fold_long_st + fold_st) runs while
  // chunk c+1 is emitted and sorted on st. Two buffer sets (records + runs)
  // alternate between chunks; set_done[s] marks the end of the last fold that
  // read set s. Folds of consecutive chunks are ordered (same voxels).
  cudaStream_t fold_long_st = nullptr;
  cudaEvent_t fold_long_done = nullptr, fold_origins = nullptr;
  cudaEvent_t set_done[2] = {nullptr, nullptr};
  bool set_busy[2] = {false, false};
  int cur_set = 0;
  bool fold_inflight = false;  // a fold was launched that st has not joined yet
  // ---- across calls: a batch's fold may still run when vxg_integrate_* returns
  // (its stats do not depend on it); the next batch's bundling and ray order
  // overlap it, and every entry point that reads or writes the map, or ends a
  // timed region, joins it first (settle / vxg_flush). vxg_reset is deferred
  // the same way: applied (after the fold) just before the next batch's first
  // map access, or by settle().
  bool async_fold = true;
  bool pending_reset = false;
  uint32_t* top_pinned = nullptr;  // longest run per chunk (read back at the batch end)
  uint32_t n_top = 0;
  static constexpr uint32_t kTopCap = 256;
  uint64_t top_T[256] = {};      // records of the fold each top_pinned entry belongs to
  double chain_ratio = -1.0;     // longest run / records of the most recent folds read back (-1: none yet)
  std::vector<cudaEvent_t> copy_events;
  // ---- streaming ingestion: two staging slots (vxg_stage_packed / vxg_integrate_staged)
  struct StageSlot {
    DBuf<float> xyz;
    DBuf<uint8_t> rgb;
    std::vector<uint64_t> off;  // rebased: off[0] = 0
    bool has_rgb = false;
    bool full = false;          // staged, not yet integrated
    bool used = false;          // `released` has been recorded once
    cudaEvent_t copied = nullptr, released = nullptr;
  } stage_slot[2];
  int next_stage = 0;
  // ---- meshing results (vxg_mesh_extract / vxg_mesh_fetch)
  DBuf<vxg_mc_tables> mesh_tab;
  DBuf<int32_t> mesh_slots;
  DBuf<uint32_t> mesh_ntri, mesh_off, mesh_frag_dev;
  DBuf<float> mesh_v, mesh_n;
  DBuf<uint8_t> mesh_c;
  std::vector<int32_t> mesh_bidx;
  std::vector<uint64_t> mesh_frag;
  uint64_t mesh_T = 0;
  bool mesh_colors = false, mesh_ready = false;

  // ---- map (slab + block hash)
  DBuf<vxg_voxel> slab;
  DBuf<int32_t> block_idx;
  DBuf<unsigned long long> hkeys;
  DBuf<int32_t> hvals;
  DBuf<uint32_t> counters;  // [0] blocks, [1] error bits
  uint64_t cap_blocks = 0;
  uint64_t hcap = 0;
  uint64_t n_blocks = 0;  // host mirror after each call
  std::vector<int32_t> host_idx;  // block index per slot (host mirror, grows with n_blocks)

  // ---- ESDF (vxg_esdf_build_occupancy): one ESDF block per TSDF slot < esdf_blocks
  DBuf<vxg_esdf_voxel> esdf;
  DBuf<int32_t> esdf_nbr;
  DBuf<uint8_t> esdf_act, esdf_act2;
  DBuf<uint32_t> esdf_changed;
  uint64_t esdf_blocks = 0;
  bool esdf_ready = false;

  // ---- updated-block consumers (layer.h:124-148)
  std::map<std::string, std::set<uint32_t>> consumers;
  DBuf<uint8_t> touched;

  // ---- scratch
  DBuf<float> in_xyz;
  DBuf<uint8_t> in_rgb;
  DBuf<uint64_t> d_off;
  DBuf<float> d_poses;
  DBuf<unsigned long long> d_stats;  // 3F: updates, raycasts, skipped
  DBuf<unsigned long long> d_upd;    // F: chunk-local updates
  DBuf<unsigned long long> pkeys, pkeys2, okeys, okeys2;
  DBuf<uint32_t> pvals, pvals2, ovals, ovals2;
  DBuf<uint32_t> flags, ray_idx, ucounts, uoffs, seg_count, seg_start, num_runs, fo, pos, part;
  DBuf<unsigned long long> ukeys;
  DBuf<SegInfo> segs;
  DBuf<RayInfo> rays;
  DBuf<unsigned long long> rcount, roff, rcount2;
  DBuf<uint32_t> ray_perm, ray_iota;
  DBuf<uint32_t> rh_k0, rh_k1, rh_v0, rh_v1, rh_rank, rh_prev, rh_g;  // rehash epochs (order_rehash_frames)
  DBuf<RhFrame> rh_frames;
  DBuf<uint64_t> tbl_off, bcs;
  DBuf<uint32_t> rkeys, rkeys2, rvals, rvals2;
  DBuf<uint32_t> run_keys, run_len, run_start, run_len2, run_order, run_iota, run_code, run_max, work;
  struct FoldSet {  // the other buffer set of the chunk pipeline (swapped with the members above)
    DBuf<uint32_t> rkeys, rkeys2, rvals, rvals2, run_keys, run_len, run_start, run_len2, run_order, num_runs, work;
    DBuf<float> d_org;
  } alt;
  DBuf<unsigned long long> ckeys;       // emission order keys: (chunk, ray length)
  DBuf<unsigned long long> chunk_base;  // per chunk: first ray, first record
  DBuf<uint32_t> sort_counts, sort_offs, dense_start, dense_end, run_flag, run_pos;
  DBuf<FoldRay> fold_rays;
  DBuf<uint2> far_rays;  // {w_front, colour} per ray: what a far record's fold step reads
  DBuf<uint32_t> num_segs;  // bundling: bucket count (RLE output)
  DBuf<float4> pt_w;    // bundling: per sorted point (world point, weight)
  DBuf<uint32_t> pt_c;  // bundling: per sorted point colour
  DBuf<float> d_org;  // sensor origins, 3 floats per frame
  bool debug_fold = false;  // globaltimer trace of the fold (vxg_debug_fold)
  DBuf<unsigned long long> fold_dbg;
  uint32_t fold_dbg_n = 0;
  uint64_t info_records = 0, info_runs = 0, info_max_run = 0;  // since the last vxg_batch_info reset
  uint64_t info_sort_passes = 0;

  // ---- profiling
  bool profile = false;
  double stage_ms[kStages] = {};
  uint64_t stage_launch[kStages] = {};
  uint64_t stage_units[kStages] = {};
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> pending;
  std::vector<cudaEvent_t> event_pool;
  uint64_t launches = 0;

  MapView view() {
    MapView m;
    m.hkeys = hkeys.p;
    m.hvals = hvals.p;
    m.hmask = hcap - 1;
    m.slab = slab.p;
    m.block_idx = block_idx.p;
    m.counters = counters.p;
    m.cap_blocks = static_cast<uint32_t>(cap_blocks);
    m.vps = vps;
    m.nvox = nvox;
    return m;
  }

  TsdfParams params() const {
    TsdfParams t;
    t.voxel_size = voxel_size;
    t.truncation = cfg.truncation;
    t.dropoff_epsilon = cfg.dropoff_epsilon;
    t.max_weight = cfg.max_weight;
    t.min_ray = cfg.min_ray_length;
    t.max_ray = cfg.max_ray_length;
    t.weight_mode = cfg.weight_mode;
    t.merge_mode = cfg.merge_mode;
    t.long_code = run_len_code(kLongRun);
    return t;
  }
  // Length code from which a run of a fold over T records goes to the warp
  // pairs (~21 ns per record, one run per pair) instead of one thread (~250 ns
  // per record, 32 runs per warp). The thread path has ~3x the throughput per
  // issue slot, the pair path 12x less latency per run: a run should take the
  // pair path when folding it in one thread would outlast the rest of the fold,
  // i.e. when its length exceeds a fixed fraction of T. The fraction is
  // 6144 / 2.4e8 (kLongFrac): on the cfg1 batch 4096 gives the shortest apply
  // STAGE (2.09 ms) but 6144 the shortest STEP (9.67 vs 9.95 ms) — fewer runs on
  // the instruction-hungry pair path, and the few threads still folding 4-6 k
  // records leave the SMs to the next batch's bundling (apply 2.28 ms, mostly
  // overlapped). Floor 64 (a single 640x480 frame, 2 M records: its longest
  // chain is the whole fold), ceiling 8192 (larger folds are chunked at 5e8
  // records and hidden behind the next chunk's emit and sort: a higher ceiling
  // only stretches their thin tail — cfg3 apply 18 / 33 ms at 4096 / 13.7 k
  // with the same step).
  static constexpr double kLongFrac = 6144.0 / 2.4e8;
  static uint32_t long_code_for(uint64_t T) {
    static const bool fixed = getenv("VXG_FIXED_LONG_RUN") != nullptr;  // dev A/B: kLongRun whatever T
    if (fixed) return run_len_code(kLongRun);
    static const double scale = [] {  // dev A/B: VXG_LONG_SCALE multiplies the fraction
      const char* e = getenv("VXG_LONG_SCALE");
      return e ? atof(e) : 1.0;
    }();
    static const double cap = [] {  // dev A/B: VXG_LONG_CAP
      const char* e = getenv("VXG_LONG_CAP");
      return e ? atof(e) : 8192.0;
    }();
    const double want = scale * static_cast<double>(T) * kLongFrac;
    const uint32_t len = static_cast<uint32_t>(std::min<double>(cap, std::max(64.0, want)));
    return run_len_code(len);
  }

  cudaEvent_t ev() {
    if (!event_pool.empty()) {
      cudaEvent_t e = event_pool.back();
      event_pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    CU(cudaEventCreate(&e));
    return e;
  }
  // Stage timer: begin() records on the stream; end() records and queues the pair.
  int cur_stage = -1;
  cudaEvent_t cur_begin = nullptr;
  void begin(int s, cudaStream_t on = nullptr) {
    if (!profile) return;
    cur_stage = s;
    cur_begin = ev();
    CU(cudaEventRecord(cur_begin, on ? on : st));
  }
  void end(uint64_t units = 0, uint64_t n_launch = 0, cudaStream_t on = nullptr) {
    if (!profile || cur_stage < 0) return;
    cudaEvent_t e = ev();
    CU(cudaEventRecord(e, on ? on : st));
    pending.push_back({cur_stage, {cur_begin, e}});
    stage_units[cur_stage] += units;
    stage_launch[cur_stage] += n_launch;
    cur_stage = -1;
  }
  void collect() {  // after a stream sync; stages still running (a fold that outlives the call) stay queued
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> keep;
    for (auto& pe : pending) {
      const cudaError_t q = cudaEventQuery(pe.second.second);
      if (q == cudaErrorNotReady) {
        (void)cudaGetLastError();
        keep.push_back(pe);
        continue;
      }
      CU(q);
      float ms = 0.f;
      CU(cudaEventElapsedTime(&ms, pe.second.first, pe.second.second));
      stage_ms[pe.first] += ms;
      event_pool.push_back(pe.second.first);
      event_pool.push_back(pe.second.second);
    }
    pending.swap(keep);
  }

  // Exclusive prefix sums on st (vxg_sort.cuh); in == out is allowed.
  DBuf<unsigned long long> scan_tmp[3];
  static constexpr uint64_t kScanSoloTiles = 2;  // up to 8 K items: one CTA, one launch
  template <typename T, typename In, typename Out>
  void scan_with(In in, Out out, uint64_t n) {
    if (n == 0) return;
    const uint64_t tiles = (n + kScanTile - 1) / kScanTile;
    if (tiles <= kScanSoloTiles) {
      k_scan_apply<T, In, Out><<<1, kScanThreads, 0, st>>>(in, n, nullptr, out, static_cast<int>(tiles));
      ++launches;
      CU(cudaGetLastError());
      return;
    }
    T* sums = reinterpret_cast<T*>(scan_tmp[0].ensure(tiles));
    k_scan_reduce<T, In><<<static_cast<unsigned>(tiles), kScanThreads, 0, st>>>(in, n, sums);
    scan_level<T>(sums, tiles, 1);
    k_scan_apply<T, In, Out><<<static_cast<unsigned>(tiles), kScanThreads, 0, st>>>(in, n, sums, out);
    launches += 2;
    CU(cudaGetLastError());
  }
  template <typename T>
  void scan_level(T* sums, uint64_t n, int level) {  // in place
    const uint64_t tiles = (n + kScanTile - 1) / kScanTile;
    using L = ScanLoad<T>;
    using S = ScanStore<T>;
    if (tiles <= kScanSoloTiles) {
      k_scan_apply<T, L, S><<<1, kScanThreads, 0, st>>>(L{sums}, n, nullptr, S{sums}, static_cast<int>(tiles));
      ++launches;
      return;
    }
    if (level > 2) throw VxgError(VXG_EINVAL, "prefix sum too large");
    T* up = reinterpret_cast<T*>(scan_tmp[level].ensure(tiles));
    k_scan_reduce<T, L><<<static_cast<unsigned>(tiles), kScanThreads, 0, st>>>(L{sums}, n, up);
    scan_level<T>(up, tiles, level + 1);
    k_scan_apply<T, L, S><<<static_cast<unsigned>(tiles), kScanThreads, 0, st>>>(L{sums}, n, up, S{sums});
    launches += 2;
  }
  template <typename T>
  void scan_exclusive(const T* in, T* out, uint64_t n) {
    scan_with<T>(ScanLoad<T>{in}, ScanStore<T>{out}, n);
  }
  // Stable sort of n (64-bit key, value) pairs by the low `bits` key bits
  // through the 32-bit pair sort: positions by the low word, then by the high
  // word; out_keys / out_vals (either may be null) receive the sorted pairs.
  DBuf<uint32_t> s64_k0, s64_k1, s64_v0, s64_v1;
  void sort_pairs64(const unsigned long long* keys, const uint32_t* vals, uint64_t n, int bits, bool descending,
                    unsigned long long* out_keys, uint32_t* out_vals);

  // ---------------------------------------------------------------- map
  // (Re)allocates an empty map of `cap` blocks of new_vps^3 voxels. Every
  // check and allocation happens before any handle state changes: on failure
  // the handle keeps its previous map (and geometry) intact.
  void alloc_map(uint64_t cap, int new_vps = 0) {
    if (new_vps <= 0) new_vps = vps;
    const uint64_t nv = static_cast<uint64_t>(new_vps) * new_vps * new_vps;
    cap = std::max<uint64_t>(cap, 1);
    if (cap * nv >= 0xFFFFFFFFull)  // voxel keys slot * vps^3 + local are 32-bit (kInvalidRecord = ~0u)
      throw VxgError(VXG_ENOMEM, "block slab would exceed the 32-bit voxel key range");
    sync_folds();  // the slab about to be freed may still be folded into
    uint64_t hc = 1;
    while (hc < 2 * cap) hc <<= 1;
    vxg_voxel* ns = nullptr;
    int32_t* ni = nullptr;
    unsigned long long* nk = nullptr;
    int32_t* nh = nullptr;
    auto fail = [&](const char* what) {
      cudaGetLastError();
      if (ns) cudaFree(ns);
      if (ni) cudaFree(ni);
      if (nk) cudaFree(nk);
      if (nh) cudaFree(nh);
      throw VxgError(VXG_ENOMEM, std::string("cannot allocate the ") + what + " for " + std::to_string(cap) +
                                     " blocks");
    };
    if (cudaMalloc(&ns, cap * nv * sizeof(vxg_voxel)) != cudaSuccess) fail("block slab");
    if (cudaMalloc(&ni, cap * 3 * sizeof(int32_t)) != cudaSuccess) fail("block index table");
    if (cudaMalloc(&nk, hc * sizeof(unsigned long long)) != cudaSuccess) fail("block hash");
    if (cudaMalloc(&nh, hc * sizeof(int32_t)) != cudaSuccess) fail("block hash");
    counters.ensure(4);
    slab.release();
    block_idx.release();
    hkeys.release();
    hvals.release();
    slab.p = ns;
    slab.cap = cap * nv;
    block_idx.p = ni;
    block_idx.cap = cap * 3;
    hkeys.p = nk;
    hkeys.cap = hc;
    hvals.p = nh;
    hvals.cap = hc;
    hcap = hc;
    cap_blocks = cap;
    vps = new_vps;
    nvox = static_cast<int>(nv);
    CU(cudaMemsetAsync(slab.p, 0, cap * nv * sizeof(vxg_voxel), st));
    CU(cudaMemsetAsync(hkeys.p, 0xFF, hcap * sizeof(unsigned long long), st));
    CU(cudaMemsetAsync(hvals.p, 0xFF, hcap * sizeof(int32_t), st));
    CU(cudaMemsetAsync(counters.p, 0, 4 * sizeof(uint32_t), st));
    n_blocks = 0;
    host_idx.clear();
    touched.release();  // per-slot flags of the old map
    CU(cudaStreamSynchronize(st));
  }

  // Grows slab (preserving the first `used` blocks) and the hash.
  void grow_map(uint64_t need_blocks) {
    uint64_t used = std::min<uint64_t>(need_blocks, cap_blocks);
    uint64_t new_cap = std::max<uint64_t>(cap_blocks * 2, need_blocks + need_blocks / 4 + 64);
    if (new_cap * static_cast<uint64_t>(nvox) >= 0xFFFFFFFFull)
      throw VxgError(VXG_ENOMEM, "block slab would exceed the 32-bit voxel key range");
    vxg_voxel* ns = nullptr;
    int32_t* ni = nullptr;
    if (cudaMalloc(&ns, new_cap * nvox * sizeof(vxg_voxel)) != cudaSuccess) {
      cudaGetLastError();
      throw VxgError(VXG_ENOMEM, "cannot grow the block slab to " + std::to_string(new_cap) + " blocks");
    }
    CU(cudaMalloc(&ni, new_cap * 3 * sizeof(int32_t)));
    CU(cudaMemsetAsync(ns, 0, new_cap * nvox * sizeof(vxg_voxel), st));
    CU(cudaMemcpyAsync(ns, slab.p, used * nvox * sizeof(vxg_voxel), cudaMemcpyDeviceToDevice, st));
    CU(cudaMemcpyAsync(ni, block_idx.p, used * 3 * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
    CU(cudaStreamSynchronize(st));
    cudaFree(slab.p);
    cudaFree(block_idx.p);
    slab.p = ns;
    slab.cap = new_cap * nvox;
    block_idx.p = ni;
    block_idx.cap = new_cap * 3;
    const uint64_t old_cap = cap_blocks;
    cap_blocks = new_cap;
    // hash: keep load <= 1/2
    uint64_t new_h = hcap;
    while (new_h < 2 * new_cap) new_h <<= 1;
    if (new_h != hcap) rehash(new_h);
    // slots handed out beyond the old capacity got no block index yet
    k_fix_block_idx<<<grid_for(hcap), 256, 0, st>>>(hcap, hkeys.p, hvals.p, static_cast<uint32_t>(old_cap),
                                                   static_cast<uint32_t>(new_cap), block_idx.p);
    ++launches;
    CU(cudaGetLastError());
  }

  void rehash(uint64_t new_h) {
    unsigned long long* nk = nullptr;
    int32_t* nv = nullptr;
    CU(cudaMalloc(&nk, new_h * sizeof(unsigned long long)));
    CU(cudaMalloc(&nv, new_h * sizeof(int32_t)));
    CU(cudaMemsetAsync(nk, 0xFF, new_h * sizeof(unsigned long long), st));
    CU(cudaMemsetAsync(nv, 0xFF, new_h * sizeof(int32_t), st));
    MapView m = view();
    m.hkeys = nk;
    m.hvals = nv;
    m.hmask = new_h - 1;
    k_rehash<<<grid_for(hcap), 256, 0, st>>>(hcap, hkeys.p, hvals.p, m);
    ++launches;
    CU(cudaGetLastError());
    CU(cudaStreamSynchronize(st));
    cudaFree(hkeys.p);
    cudaFree(hvals.p);
    hkeys.p = nk;
    hkeys.cap = new_h;
    hvals.p = nv;
    hvals.cap = new_h;
    hcap = new_h;
  }

  // touched[slot] flags for updated-block consumers: sized to the slab, zeroed
  // whenever (re)allocated; the old flags are kept across growth.
  void ensure_touched() {
    if (consumers.empty()) return;
    if (touched.p != nullptr && touched.cap >= cap_blocks) return;
    uint8_t* n = nullptr;
    CU(cudaMalloc(&n, cap_blocks));
    CU(cudaMemsetAsync(n, 0, cap_blocks, st));
    if (touched.p != nullptr) CU(cudaMemcpyAsync(n, touched.p, touched.cap, cudaMemcpyDeviceToDevice, st));
    CU(cudaStreamSynchronize(st));
    touched.release();
    touched.p = n;
    touched.cap = cap_blocks;
  }

  // ---------------------------------------------------------------- chunk pipeline
  void ensure_fold_streams() {
    if (fold_long_st != nullptr) return;
    CU(cudaStreamCreateWithFlags(&fold_st, cudaStreamNonBlocking));
    // the long-run CTAs must become resident before the short-run grid fills
    // the SMs (the longest chain bounds the fold): highest priority
    int lo_prio = 0, hi_prio = 0;
    CU(cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio));
    CU(cudaStreamCreateWithPriority(&fold_long_st, cudaStreamNonBlocking, hi_prio));
    CU(cudaEventCreateWithFlags(&fold_fork, cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&fold_join, cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&fold_long_done, cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&fold_origins, cudaEventDisableTiming));
    for (auto& e : set_done) CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    CU(cudaHostAlloc(&top_pinned, kTopCap * sizeof(uint32_t), cudaHostAllocDefault));
  }
  // Switch to the other buffer set; st waits until the fold that last read it is done.
  void swap_fold_set() {
    rkeys.swap(alt.rkeys);
    rkeys2.swap(alt.rkeys2);
    rvals.swap(alt.rvals);
    rvals2.swap(alt.rvals2);
    run_keys.swap(alt.run_keys);
    run_len.swap(alt.run_len);
    run_start.swap(alt.run_start);
    run_len2.swap(alt.run_len2);
    run_order.swap(alt.run_order);
    num_runs.swap(alt.num_runs);
    work.swap(alt.work);
    d_org.swap(alt.d_org);
    cur_set ^= 1;
    if (set_busy[cur_set]) CU(cudaStreamWaitEvent(st, set_done[cur_set], 0));
  }
  // Host wait for every launched fold (before the slab moves or buffers are freed).
  void sync_folds() {
    if (fold_st != nullptr) CU(cudaStreamSynchronize(fold_st));
    if (fold_long_st != nullptr) CU(cudaStreamSynchronize(fold_long_st));
    set_busy[0] = set_busy[1] = false;
  }
  // Record buffers of the current set; reallocation waits for in-flight folds.
  void ensure_records(uint64_t T) {
    if (T > rkeys.cap || T > rkeys2.cap || T > rvals.cap || T > rvals2.cap) sync_folds();
    rkeys.ensure(T);
    rkeys2.ensure(T);
    rvals.ensure(T);
    rvals2.ensure(T);
  }
  // st waits for the last launched fold (end of a batch / before the slab is read).
  void join_folds() {
    if (!fold_inflight) return;
    CU(cudaStreamWaitEvent(st, fold_join, 0));
    fold_inflight = false;
  }
  // A deferred vxg_reset: clear the slab's used blocks, the hash and the
  // counters once every fold that writes them is done.
  void apply_pending_reset() {
    if (!pending_reset) return;
    join_folds();
    uint32_t c[2];
    read_counters(c);
    const uint64_t used = std::min<uint64_t>(std::max<uint64_t>(std::max<uint64_t>(c[0], reset_used), last_blocks),
                                             cap_blocks);
    CU(cudaMemsetAsync(slab.p, 0, used * nvox * sizeof(vxg_voxel), st));
    CU(cudaMemsetAsync(hkeys.p, 0xFF, hcap * sizeof(unsigned long long), st));
    CU(cudaMemsetAsync(hvals.p, 0xFF, hcap * sizeof(int32_t), st));
    CU(cudaMemsetAsync(counters.p, 0, 2 * sizeof(uint32_t), st));
    last_blocks = 0;
    reset_used = 0;
    pending_reset = false;
  }
  // Before any entry point that reads or writes the map: st ordered after
  // every launched fold, deferred reset applied.
  void settle() {
    apply_pending_reset();
    join_folds();
  }
  // Folds may outlive the call only on a plain single-GPU handle without
  // updated-block consumers (the fold marks the touched blocks they drain).
  bool sharded() const { return shard_world > 1 || nccl_comm != nullptr; }
  bool fold_may_outlive_call() const { return async_fold && consumers.empty() && !sharded() && !debug_fold; }
  uint64_t reset_used = 0;  // blocks in use when vxg_reset was called (deferred)
  // After a host sync of st that followed join_folds(): longest runs of the batch.
  void drain_tops() {
    double ratio = -1.0;
    for (uint32_t i = 0; i < n_top; ++i) {
      info_max_run = std::max<uint64_t>(info_max_run, top_pinned[i]);
      if (top_T[i]) ratio = std::max(ratio, static_cast<double>(top_pinned[i]) / static_cast<double>(top_T[i]));
    }
    if (n_top) chain_ratio = ratio;
    n_top = 0;
  }

  // Small device->host reads go through a pinned mailbox: a pageable
  // destination makes the driver stage the copy, and such a copy can queue
  // behind a large H2D in flight on the copy stream (the next batch's
  // staging), stalling the call for the whole transfer.
  struct D2H {
    void* host;
    const void* dev;
    size_t bytes;
  };
  uint8_t* mailbox = nullptr;
  size_t mailbox_cap = 0;
  void fetch(std::initializer_list<D2H> list) {
    size_t total = 0;
    for (const D2H& d : list) total += (d.bytes + 15) & ~size_t(15);
    if (total > mailbox_cap) {
      if (mailbox) CU(cudaFreeHost(mailbox));
      mailbox = nullptr;
      mailbox_cap = std::max<size_t>(total + total / 2, 4096);
      CU(cudaHostAlloc(reinterpret_cast<void**>(&mailbox), mailbox_cap, cudaHostAllocDefault));
    }
    size_t o = 0;
    for (const D2H& d : list) {
      if (d.bytes) CU(cudaMemcpyAsync(mailbox + o, d.dev, d.bytes, cudaMemcpyDeviceToHost, st));
      o += (d.bytes + 15) & ~size_t(15);
    }
    CU(cudaStreamSynchronize(st));
    o = 0;
    for (const D2H& d : list) {
      if (d.bytes) std::memcpy(d.host, mailbox + o, d.bytes);
      o += (d.bytes + 15) & ~size_t(15);
    }
  }

  void read_counters(uint32_t* c) { fetch({{c, counters.p, 2 * sizeof(uint32_t)}}); }

  // Refresh host_idx for slots appended since the last call.
  void sync_block_mirror(uint64_t nb) {
    if (nb > cap_blocks) nb = cap_blocks;
    if (nb <= n_blocks && host_idx.size() == 3 * n_blocks) {
      n_blocks = nb;
      host_idx.resize(3 * nb);
      return;
    }
    const uint64_t have = host_idx.size() / 3;
    host_idx.resize(3 * nb);
    if (nb > have) {
      fetch({{host_idx.data() + 3 * have, block_idx.p + 3 * have, (nb - have) * 3 * sizeof(int32_t)}});
    }
    n_blocks = nb;
  }

  // ---------------------------------------------------------------- pipeline
  void run_sub(const float* xyz, const uint8_t* rgb, const uint64_t* offsets, const float* poses, uint64_t F,
               bool device_input, vxg_stats* out);
  void build_rays_simple(const float* dxyz, const uint8_t* drgb, uint64_t P, uint32_t F, uint32_t* R_out);
  void build_rays_grouped(const float* dxyz, const uint8_t* drgb, uint64_t P, const uint64_t* h_off, uint32_t F,
                          uint32_t* R_out, TermView* tv);
  void order_rehash_frames(const std::vector<uint32_t>& frames, const std::vector<uint32_t>& K,
                           const std::vector<uint32_t>& start, const std::vector<Schedule>& sched,
                           const std::vector<uint32_t>& ray0, int pb);
  void emit_and_apply(uint32_t R, uint32_t F, const TermView& tv);
  uint64_t count_rays(uint32_t R, uint32_t F);
  void sort_fold(uint64_t T, uint64_t nslots, uint32_t F);
  void sort_records(uint64_t T, int kbits, uint32_t** sk, uint32_t** sv, uint32_t K);
  template <int kBits, int kIpt, int kMB, int kNs = 8>
  void lsd_sort(uint64_t T, int kbits, uint32_t* k0, uint32_t* v0, uint32_t* k1, uint32_t* v1, uint32_t** sk,
                uint32_t** sv, bool grouped, uint32_t K = 0);
  // the plain pair sort: small inputs take one sub-tile per CTA (8x the CTAs)
  void sort_pairs32(uint64_t n, int kbits, uint32_t* k0, uint32_t* v0, uint32_t* k1, uint32_t* v1, uint32_t** sk,
                    uint32_t** sv) {
    if (n < (16u << 20))
      lsd_sort<8, 12, 4, 1>(n, kbits, k0, v0, k1, v1, sk, sv, false);
    else
      lsd_sort<8, 12, 4>(n, kbits, k0, v0, k1, v1, sk, sv, false);
  }
  bool marks_fused = false;  // the last sort pass wrote dense_start / dense_end (no sorted keys)
  int last_lsd_passes = 0;
  uint64_t last_blocks = 0;  // blocks allocated after the last produce attempt
  bool grew_after_attempt(int attempt);
  void begin_batch(const float* xyz, const uint8_t* rgb, const uint64_t* offsets, const float* poses, uint64_t F,
                   uint32_t* R_out, TermView* tv);
  void end_batch(uint64_t F, vxg_stats* out);
  // ---- sharded map (multi-GPU / loopback group)
  int shard_rank = 0;
  int shard_world = 1;
  bool shard_replicated = false;  // replicated traversal, no record exchange
  // records this rank folds: received (exchange) or its own partition (replicated)
  const uint4* owned_records() const {
    return shard_replicated ? send_buf.p + send_offsets[shard_rank] : recv_buf.p;
  }
  uint64_t owned_count() const {
    return shard_replicated ? (send_counts.empty() ? 0 : send_counts[shard_rank]) : recv_total;
  }
  void* nccl_comm = nullptr;
  std::vector<uint64_t> send_counts, send_offsets, recv_counts;
  uint64_t recv_total = 0;
  DBuf<unsigned long long> gkeys, sbounds, obounds, dev_counts;
  DBuf<uint32_t> gowner, gowner2, giota, gperm;
  DBuf<uint4> send_buf, recv_buf;
  // sharded emit: dictionary of the blocks this rank's ray slice touches (hash + block index table, no
  // slab) for the single-GPU k_emit to write 32-bit keys against; k_globalize turns them into global keys
  DBuf<unsigned long long> dict_hkeys, sh_upd;
  DBuf<int32_t> dict_hvals, dict_bidx;
  DBuf<uint32_t> dict_counters, sh_keys, sh_vals;
  uint64_t dict_cap = 0;
  void shard_front(uint32_t R, uint32_t F, const TermView& tv);
  void shard_back(const uint4* recv, uint64_t n, uint32_t F);
  void nccl_exchange();
  void nccl_reduce_updates(uint32_t F);
};

void vxg_handle::sort_pairs64(const unsigned long long* keys, const uint32_t* vals, uint64_t n, int bits,
                              bool descending, unsigned long long* out_keys, uint32_t* out_vals) {
  if (n == 0) return;
  if (n > 0xFFFFFFFFull) throw VxgError(VXG_EINVAL, "sort too large (32-bit positions)");
  bits = std::max(bits, 1);
  s64_k0.ensure(n);
  s64_k1.ensure(n);
  s64_v0.ensure(n);
  s64_v1.ensure(n);
  const int lo_bits = std::min(bits, 32), hi_bits = bits - lo_bits;
  const uint32_t lo_mask = lo_bits == 32 ? 0xFFFFFFFFu : (1u << lo_bits) - 1u;
  uint32_t *sk = nullptr, *sv = nullptr;
  k_key_word<<<grid_for(n), 256, 0, st>>>(n, keys, nullptr, 0, lo_mask, descending, s64_k0.p, s64_v0.p);
  ++launches;
  sort_pairs32(n, lo_bits, s64_k0.p, s64_v0.p, s64_k1.p, s64_v1.p, &sk, &sv);
  if (hi_bits > 0) {
    uint32_t* kf = sk == s64_k0.p ? s64_k1.p : s64_k0.p;  // free key buffer
    uint32_t* vf = sv == s64_v0.p ? s64_v1.p : s64_v0.p;  // free value buffer
    k_key_word<<<grid_for(n), 256, 0, st>>>(n, keys, sv, 32, hi_bits == 32 ? 0xFFFFFFFFu : (1u << hi_bits) - 1u, descending,
                                            kf, nullptr);
    ++launches;
    uint32_t *sk2 = nullptr, *sv2 = nullptr;
    sort_pairs32(n, hi_bits, kf, sv, sk, vf, &sk2, &sv2);
    sv = sv2;
  }
  k_gather_sorted<<<grid_for(n), 256, 0, st>>>(n, sv, keys, vals, out_keys, out_vals);
  ++launches;
  CU(cudaGetLastError());
}

void vxg_handle::build_rays_simple(const float* dxyz, const uint8_t* drgb, uint64_t P, uint32_t F, uint32_t* R_out) {
  const TsdfParams tp = params();
  begin(ST_BUNDLE);
  flags.ensure(P);
  ray_idx.ensure(P);
  k_simple_inrange<<<grid_for(P), 256, 0, st>>>(dxyz, P, d_off.p, d_poses.p, F, tp, flags.p, d_stats.p + 2 * F);
  ++launches;
  CU(cudaGetLastError());
  scan_exclusive<uint32_t>(flags.p, ray_idx.p, P);
  uint32_t last_idx = 0, last_flag = 0;
  fetch({{&last_idx, ray_idx.p + (P - 1), sizeof(uint32_t)}, {&last_flag, flags.p + (P - 1), sizeof(uint32_t)}});
  const uint32_t R = last_idx + last_flag;
  rays.ensure(std::max<uint32_t>(R, 1));
  k_simple_rays<<<grid_for(P), 256, 0, st>>>(dxyz, drgb, P, d_off.p, d_poses.p, F, flags.p, ray_idx.p, rays.p);
  ++launches;
  CU(cudaGetLastError());
  end(P, 4);
  *R_out = R;
}

// Reorders the buckets of every frame whose map rehashes while they are
// inserted, on the device and for all such frames at
// once: epoch e re-inserts the previous iteration order, then appends the next
// keys by first appearance, under bucket count bc_e (k_rhb_*). Each epoch
// level is two stable 32-bit sorts over the concatenated frames (frame in the
// high key bits; position desc, then first bucket occupation desc), so the
// launch count grows with the epoch count, not with the frame count. Frames
// are processed in groups whose index fits the key.
void vxg_handle::order_rehash_frames(const std::vector<uint32_t>& frames, const std::vector<uint32_t>& K,
                                     const std::vector<uint32_t>& start, const std::vector<Schedule>& sched,
                                     const std::vector<uint32_t>& ray0, int pb) {
  uint32_t maxK = 1;
  for (uint32_t f : frames) maxK = std::max(maxK, K[f]);
  const int kb = bits_for(maxK);  // positions < K <= 2^kb - 1
  const int key_bits = std::max(pb, kb + 1);
  if (key_bits >= 32) throw VxgError(VXG_EINVAL, "scan too large for the rehash ray-order key");
  const size_t group = size_t(1) << std::min(16, 32 - key_bits);  // frames per group: g < 2^(32 - key_bits)
  for (size_t g0 = 0; g0 < frames.size(); g0 += group) {
    const size_t G = std::min(group, frames.size() - g0);
    const int gb = bits_for(G - 1);
    // epochs per frame and the per-(epoch, frame) parameters
    std::vector<uint32_t> n_ep(G);
    uint32_t E = 0, n = 0;
    for (size_t g = 0; g < G; ++g) {
      const uint32_t f = frames[g0 + g];
      const Schedule& sch = sched[f];
      uint32_t e = 0;
      while (e < sch.size()) {
        if (e > 0 && sch[e].first >= K[f]) break;
        ++e;
        const uint64_t t_hi = e < sch.size() ? sch[e].first : UINT64_MAX;
        if (t_hi >= K[f]) break;
      }
      n_ep[g] = e;
      E = std::max(E, e);
      n += K[f];
    }
    std::vector<RhFrame> P(static_cast<size_t>(E) * G);
    std::vector<uint64_t> fo_total(E, 0);
    uint32_t base = 0;
    for (size_t g = 0; g < G; ++g) {
      const uint32_t f = frames[g0 + g];
      const Schedule& sch = sched[f];
      for (uint32_t e = 0; e < E; ++e) {
        RhFrame& q = P[e * G + g];
        q = RhFrame{};
        q.seg0 = start[f];
        q.base = base;
        q.K = K[f];
        q.ray0 = ray0[f];
        if (e < n_ep[g]) {
          const uint64_t t_hi = e + 1 < sch.size() ? sch[e + 1].first : UINT64_MAX;
          q.t_lo = static_cast<uint32_t>(sch[e].first);
          q.t_hi = static_cast<uint32_t>(std::min<uint64_t>(t_hi, K[f]));
          q.active = 1u;
          q.last = e + 1 == n_ep[g] ? 1u : 0u;
          q.bc = sch[e].second;
          q.fo_off = fo_total[e];
          fo_total[e] += q.bc;
        }
      }
      base += K[f];
    }
    RhFrame* dP = rh_frames.ensure(P.size());
    CU(cudaMemcpyAsync(dP, P.data(), P.size() * sizeof(RhFrame), cudaMemcpyHostToDevice, st));
    uint32_t* k0 = rh_k0.ensure(n);
    uint32_t* k1 = rh_k1.ensure(n);
    uint32_t* v0 = rh_v0.ensure(n);
    uint32_t* v1 = rh_v1.ensure(n);
    uint32_t* rank = rh_rank.ensure(n);
    uint32_t* prev = rh_prev.ensure(n);
    uint32_t* rg = rh_g.ensure(n);
    uint32_t *sk = nullptr, *sv = nullptr;
    // rank = first-appearance rank inside the frame
    k_rhb_init<<<grid_for(n), 256, 0, st>>>(n, static_cast<uint32_t>(G), dP, segs.p, pb, rg, k0, v0);
    sort_pairs32(n, gb + pb, k0, v0, k1, v1, &sk, &sv);
    k_rhb_rank<<<grid_for(n), 256, 0, st>>>(n, dP, rg, sv, rank);
    launches += 2;
    for (uint32_t e = 0; e < E; ++e) {
      const RhFrame* dPe = dP + static_cast<size_t>(e) * G;
      fo.ensure(std::max<uint64_t>(fo_total[e], 1));
      CU(cudaMemsetAsync(fo.p, 0xFF, fo_total[e] * sizeof(uint32_t), st));
      k_rhb_fo<<<grid_for(n), 256, 0, st>>>(n, dPe, rg, segs.p, rank, prev, fo.p);
      k_rhb_pos_desc<<<grid_for(n), 256, 0, st>>>(n, dPe, rg, rank, prev, kb, k0, v0);
      sort_pairs32(n, gb + kb + 1, k0, v0, k1, v1, &sk, &sv);
      uint32_t* kf = sk == k0 ? k1 : k0;  // free key buffer
      uint32_t* vf = sv == v0 ? v1 : v0;  // free value buffer
      k_rhb_fo_desc<<<grid_for(n), 256, 0, st>>>(n, dPe, rg, sv, segs.p, rank, fo.p, kb, kf);
      uint32_t *sk2 = nullptr, *sv2 = nullptr;
      sort_pairs32(n, gb + kb + 1, kf, sv, sk, vf, &sk2, &sv2);
      k_rhb_commit<<<grid_for(n), 256, 0, st>>>(n, dPe, rg, sv2, prev, ovals.p);
      launches += 4;
      CU(cudaGetLastError());
    }
  }
}

void vxg_handle::build_rays_grouped(const float* dxyz, const uint8_t* drgb, uint64_t P, const uint64_t* h_off,
                                    uint32_t F, uint32_t* R_out, TermView* tv) {
  const TsdfParams tp = params();
  // key geometry: every in-range terminal voxel lies within rb voxels of the
  // origin voxel on each axis; kb bits hold [0, 2 rb] plus an all-ones sentinel.
  const int rb = static_cast<int>(std::ceil((static_cast<double>(cfg.max_ray_length) + cfg.truncation) / voxel_size)) + 3;
  int kb = bits_for(static_cast<uint64_t>(2 * rb + 2));
  const int fb = bits_for(F > 1 ? F - 1 : 0);
  if (3 * kb + fb > 64) throw VxgError(VXG_EINVAL, "max_ray_length / voxel_size too large for the bundling key");
  begin(ST_BUNDLE);
  pvals.ensure(P);
  pvals2.ensure(P);
  const int end_bit = 3 * kb + fb;
  ukeys.ensure(P);
  ucounts.ensure(P);
  num_segs.ensure(1);  // its own count: num_runs belongs to the fold sets (a fold may still read it)
  if (end_bit <= 32) {  // 32-bit keys: half the sort traffic
    uint32_t* k32 = reinterpret_cast<uint32_t*>(pkeys.ensure((P + 1) / 2));
    uint32_t* k32b = reinterpret_cast<uint32_t*>(pkeys2.ensure((P + 1) / 2));
    k_group_keys<uint32_t><<<grid_for(P), 256, 0, st>>>(dxyz, P, d_off.p, d_poses.p, F, tp, rb, kb, k32, pvals.p,
                                                        counters.p);
    ++launches;
    CU(cudaGetLastError());
    // stable sort by (frame, terminal voxel): the custom LSD sort, 8-bit digits
    uint32_t *sk = nullptr, *sv = nullptr;
    sort_pairs32(P, end_bit, k32, pvals.p, k32b, pvals2.p, &sk, &sv);  // frames stay contiguous
    if (sk != k32b) {  // even pass count: the result is in the first buffers
      pkeys.swap(pkeys2);
      pvals.swap(pvals2);
      k32 = reinterpret_cast<uint32_t*>(pkeys.p);
      k32b = reinterpret_cast<uint32_t*>(pkeys2.p);
    }
    // one bucket per run of equal keys: heads, their ranks, (key, start) per bucket
    uoffs.ensure(P);
    scan_with<uint32_t>(SegHeadIn<uint32_t>{k32b}, SegHeadOut<uint32_t>{k32b, P, ukeys.p, uoffs.p, num_segs.p}, P);
    pt_w.ensure(P);
    pt_c.ensure(P);
    k_point_prep<uint32_t><<<grid_for(P), 256, 0, st>>>(P, k32b, pvals2.p, dxyz, drgb, d_poses.p, tp, kb, pt_w.p,
                                                        pt_c.p);
    ++launches;
    CU(cudaGetLastError());
  } else {
    pkeys.ensure(P);
    pkeys2.ensure(P);
    k_group_keys<unsigned long long><<<grid_for(P), 256, 0, st>>>(dxyz, P, d_off.p, d_poses.p, F, tp, rb, kb,
                                                                  pkeys.p, pvals.p, counters.p);
    ++launches;
    CU(cudaGetLastError());
    sort_pairs64(pkeys.p, pvals.p, P, end_bit, false, pkeys2.p, pvals2.p);
    uoffs.ensure(P);
    scan_with<uint32_t>(SegHeadIn<unsigned long long>{pkeys2.p},
                        SegHeadOut<unsigned long long>{pkeys2.p, P, ukeys.p, uoffs.p, num_segs.p}, P);
    pt_w.ensure(P);
    pt_c.ensure(P);
    k_point_prep<unsigned long long><<<grid_for(P), 256, 0, st>>>(P, pkeys2.p, pvals2.p, dxyz, drgb, d_poses.p, tp, kb,
                                                                  pt_w.p, pt_c.p);
    ++launches;
    CU(cudaGetLastError());
  }
  uint32_t S = 0;
  fetch({{&S, num_segs.p, sizeof(uint32_t)}});
  if (S) {
    k_seg_counts<<<grid_for(S), 256, 0, st>>>(S, P, uoffs.p, ucounts.p);
    ++launches;
  }
  segs.ensure(std::max<uint32_t>(S, 1));
  seg_count.ensure(F);
  seg_start.ensure(F);
  CU(cudaMemsetAsync(seg_count.p, 0, F * sizeof(uint32_t), st));
  CU(cudaMemsetAsync(seg_start.p, 0xFF, F * sizeof(uint32_t), st));
  k_seg_reduce<<<grid_for(S), 256, 0, st>>>(num_segs.p, ukeys.p, uoffs.p, ucounts.p, pvals2.p, pt_w.p, pt_c.p, drgb,
                                            d_off.p,
                                            d_poses.p, tp, rb, kb, segs.p, seg_count.p, seg_start.p, d_stats.p + 2 * F);
  ++launches;
  CU(cudaGetLastError());
  std::vector<uint32_t> K(F), start(F);
  fetch({{K.data(), seg_count.p, F * sizeof(uint32_t)}, {start.data(), seg_start.p, F * sizeof(uint32_t)}});
  end(P, 7);

  // ---- K3 ray order
  begin(ST_ORDER);
  uint64_t maxN = 1;
  for (uint32_t f = 0; f < F; ++f) maxN = std::max<uint64_t>(maxN, h_off[f + 1] - h_off[f]);
  const int pb = bits_for(maxN);
  if (2 * pb + 1 + fb > 64) throw VxgError(VXG_EINVAL, "scan too large for the ray-order key");
  std::vector<uint64_t> h_tbl(F), h_bc(F);
  std::vector<Schedule> sched(F);
  uint64_t tbl_total = 0;
  uint32_t R = 0;
  std::vector<uint32_t> ray0(F);
  for (uint32_t f = 0; f < F; ++f) {
    const uint64_t N = h_off[f + 1] - h_off[f];
    sched[f] = bucket_schedule(N, K[f]);
    h_bc[f] = sched[f][0].second;
    h_tbl[f] = tbl_total;
    tbl_total += h_bc[f];
    ray0[f] = R;
    R += K[f];
  }
  tbl_off.ensure(F);
  bcs.ensure(F);
  CU(cudaMemcpyAsync(tbl_off.p, h_tbl.data(), F * sizeof(uint64_t), cudaMemcpyHostToDevice, st));
  CU(cudaMemcpyAsync(bcs.p, h_bc.data(), F * sizeof(uint64_t), cudaMemcpyHostToDevice, st));
  fo.ensure(std::max<uint64_t>(tbl_total, 1));
  CU(cudaMemsetAsync(fo.p, 0xFF, tbl_total * sizeof(uint32_t), st));
  k_order_fo<<<grid_for(S), 256, 0, st>>>(S, segs.p, nullptr, nullptr, tbl_off.p, bcs.p, fo.p);
  okeys.ensure(std::max<uint32_t>(S, 1));
  okeys2.ensure(std::max<uint32_t>(S, 1));
  ovals.ensure(std::max<uint32_t>(S, 1));
  ovals2.ensure(std::max<uint32_t>(S, 1));
  k_order_keys<<<grid_for(S), 256, 0, st>>>(S, segs.p, nullptr, nullptr, tbl_off.p, bcs.p, fo.p, pb, okeys.p, ovals.p);
  launches += 2;
  CU(cudaGetLastError());
  const int obits = std::min(64, fb + 2 * pb + 1);
  sort_pairs64(okeys.p, ovals.p, S, obits, false, nullptr, ovals2.p);
  std::swap(ovals.p, ovals2.p);
  std::swap(ovals.cap, ovals2.cap);
  std::vector<uint32_t> rehashing;
  for (uint32_t f = 0; f < F; ++f)
    if (sched[f].size() > 1 && K[f] > sched[f][1].first) rehashing.push_back(f);
  if (!rehashing.empty()) order_rehash_frames(rehashing, K, start, sched, ray0, pb);
  rays.ensure(std::max<uint32_t>(R, 1));
  k_gather_rays<<<grid_for(R), 256, 0, st>>>(R, ovals.p, segs.p, rays.p);
  ++launches;
  CU(cudaGetLastError());
  end(S, 3);
  tv->keys = ukeys.p;
  tv->start = seg_start.p;
  tv->count = seg_count.p;
  tv->rb = rb;
  tv->kb = kb;
  *R_out = R;
}

uint64_t vxg_handle::count_rays(uint32_t R, uint32_t F) {
  const TsdfParams tp = params();
  begin(ST_RAYS);
  rcount.ensure(R);
  roff.ensure(R);
  join_folds();  // the previous batch's fold reads fold_rays
  if (R > fold_rays.cap || R > far_rays.cap) sync_folds();  // (and the host may free them only after that fold)
  fold_rays.ensure(R);
  far_rays.ensure(R);
  k_ray_count<<<grid_for(R), 256, 0, st>>>(R, rays.p, d_poses.p, tp, rcount.p, d_stats.p + F, fold_rays.p,
                                           far_rays.p);
  ++launches;
  CU(cudaGetLastError());
  scan_exclusive<unsigned long long>(rcount.p, roff.p, R);
  unsigned long long tail[2] = {0, 0};
  fetch({{&tail[0], roff.p + (R - 1), sizeof(unsigned long long)},
         {&tail[1], rcount.p + (R - 1), sizeof(unsigned long long)}});
  end(R, 3);
  return tail[0] + tail[1];
}

// Stable LSD radix sort of the T records by voxel key (vxg_sort.cuh): digits
// of up to kBits bits (3 passes for the <= 21-bit keys of a 512-block layer
// of 16^3 voxels); returns the buffers holding the sorted keys / ray ids.
// grouped = true: only equal keys need to end up adjacent (ray order kept
// inside each group), not in key order. The digits are then applied top digit
// first — in emission (ray) order the top digit (block slot bits) is the most
// clustered, so that pass scatters long coalesced segments and ranks few
// distinct values — then the others from the bottom: groups come out ordered
// by a bit-permuted key (measured 3.57 vs 4.14 ms on cfg1). Other plans
// (VXG_DIGITS, B200, cfg1): 14:7,7:7,0:7 3.81; 12:9,0:6,6:6 3.97; 14:7,0:6,6:8
// 3.88; 12:9,0:4,4:8 4.15; plain LSD 4.29 vs 3.77 ms for the default.
std::vector<std::pair<int, int>> grouped_digit_plan(int kbits);

template <int kBits, int kIpt, int kMB, int kNs>
void vxg_handle::lsd_sort(uint64_t T, int kbits, uint32_t* k0, uint32_t* v0, uint32_t* k1, uint32_t* v1,
                          uint32_t** sk, uint32_t** sv, bool grouped, uint32_t K) {
  using C = SortCfg<kBits, kIpt, kNs>;
  static bool attr = false;
  if (!attr) {
    CU(cudaFuncSetAttribute(k_sort_downsweep<kBits, kIpt, kMB, true, true, false, kNs>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sizeof(typename C::Smem))));
    CU(cudaFuncSetAttribute(k_sort_downsweep<kBits, kIpt, kMB, true, true, true, kNs>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sizeof(typename C::Smem))));
    attr = true;
  }
  // K > 0: the last pass marks the runs (dense_start / dense_end over K keys)
  static const bool no_fuse = getenv("VXG_NO_FUSED_MARKS") != nullptr;  // dev A/B
  marks_fused = K > 0 && !no_fuse;
  if (marks_fused) {
    dense_start.ensure(K);
    dense_end.ensure(K);
    CU(cudaMemsetAsync(dense_start.p, 0xFF, K * sizeof(uint32_t), st));
    CU(cudaMemsetAsync(dense_end.p, 0, K * sizeof(uint32_t), st));
  }
  std::vector<std::pair<int, int>> plan = grouped ? grouped_digit_plan(kbits) : std::vector<std::pair<int, int>>{};
  if (plan.empty()) {
    const int np = std::max(1, (kbits + kBits - 1) / kBits);
    int dshift[8], dbits[8];  // natural digits, least significant first
    for (int p = 0, sh = 0; p < np; ++p) {
      dbits[p] = (kbits - sh + (np - p) - 1) / (np - p);
      dshift[p] = sh;
      sh += dbits[p];
    }
    for (int q = 0; q < np; ++q) {
      const int p = !grouped ? q : (q == 0 ? np - 1 : q - 1);
      plan.emplace_back(dshift[p], dbits[p]);
    }
  }
  const int passes = static_cast<int>(plan.size());
  last_lsd_passes = passes;
  const uint32_t S = static_cast<uint32_t>((T + C::kSuper - 1) / C::kSuper);
  uint32_t *ki = k0, *vi = v0, *ko = k1, *vo = v1;
  for (int q = 0; q < passes; ++q) {
    const int shift = plan[q].first, bits = plan[q].second;
    const uint32_t mask = bits ? (1u << bits) - 1u : 0u;
    const uint64_t nc = static_cast<uint64_t>(mask + 1u) * S;
    sort_counts.ensure(nc);
    sort_offs.ensure(nc);
    k_sort_upsweep<kBits, kIpt, kNs><<<S, kSortThreads, 0, st>>>(ki, T, shift, mask, S, sort_counts.p);
    scan_exclusive<uint32_t>(sort_counts.p, sort_offs.p, nc);
    if (marks_fused && q + 1 == passes)
      k_sort_downsweep<kBits, kIpt, kMB, true, true, true, kNs><<<S, kSortThreads, sizeof(typename C::Smem), st>>>(
          ki, vi, ko, vo, T, shift, mask, S, sort_offs.p, K, dense_start.p, dense_end.p);
    else
      k_sort_downsweep<kBits, kIpt, kMB, true, true, false, kNs><<<S, kSortThreads, sizeof(typename C::Smem), st>>>(
          ki, vi, ko, vo, T, shift, mask, S, sort_offs.p);
    launches += 2;  // (+ the prefix-sum kernels, counted by scan_exclusive)
    CU(cudaGetLastError());
    std::swap(ki, ko);
    std::swap(vi, vo);
  }
  *sk = ki;
  *sv = vi;
}

// Digit plan of the grouped record sort, (shift, bits) per pass in pass order
// (dev A/B: VXG_DIGITS="14:7,0:7,7:7"; the fields must tile [0, kbits)).
// Empty: the default (top digit first, then the others from the bottom).
std::vector<std::pair<int, int>> grouped_digit_plan(int kbits) {
  std::vector<std::pair<int, int>> plan;
  const char* e = getenv("VXG_DIGITS");
  if (e == nullptr) return plan;
  uint64_t cover = 0;
  for (const char* c = e; *c;) {
    int sh = 0, b = 0, n = 0;
    if (sscanf(c, "%d:%d%n", &sh, &b, &n) != 2) return {};
    plan.emplace_back(sh, b);
    cover |= ((1ull << b) - 1ull) << sh;
    c += n;
    if (*c == ',') ++c;
  }
  if (cover != (1ull << kbits) - 1ull) return {};
  return plan;
}

void vxg_handle::sort_records(uint64_t T, int kbits, uint32_t** sk, uint32_t** sv, uint32_t K) {
  int maxb = 0;
  for (const auto& d : grouped_digit_plan(kbits)) maxb = std::max(maxb, d.second);
  if (maxb > 8)
    lsd_sort<9, 12, 4>(T, kbits, rkeys.p, rvals.p, rkeys2.p, rvals2.p, sk, sv, true, K);
  else if (maxb == 8 || (maxb == 0 && kbits > 21))
    lsd_sort<8, 12, 4>(T, kbits, rkeys.p, rvals.p, rkeys2.p, rvals2.p, sk, sv, true, K);
  else
    lsd_sort<7, 12, 4>(T, kbits, rkeys.p, rvals.p, rkeys2.p, rvals2.p, sk, sv, true, K);
  info_sort_passes = static_cast<uint64_t>(last_lsd_passes);
}

// Sorts the T records of one attempt (keys < nslots * vps^3, or invalid) and
// folds every voxel's run in ray order.
void vxg_handle::sort_fold(uint64_t T, uint64_t nslots, uint32_t F) {
  TsdfParams tp = params();
  tp.long_code = long_code_for(T);
  begin(ST_SORT);
  const uint64_t K = std::max<uint64_t>(1, std::min<uint64_t>(nslots, cap_blocks) * static_cast<uint64_t>(nvox));
  const int kbits = bits_for(K);  // every valid key < K <= 2^kbits - 1: the invalid key sorts last
  if (const char* dump = getenv("VXG_DUMP_RECORDS")) {  // dev hook: unsorted records for tools/sort_lab.cu
    std::vector<uint32_t> hk(T), hv(T);
    CU(cudaMemcpyAsync(hk.data(), rkeys.p, T * 4, cudaMemcpyDeviceToHost, st));
    CU(cudaMemcpyAsync(hv.data(), rvals.p, T * 4, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    if (FILE* f = fopen(dump, "wb")) {
      const uint64_t hdr[2] = {T, static_cast<uint64_t>(kbits)};
      fwrite(hdr, sizeof(hdr), 1, f);
      fwrite(hk.data(), 4, T, f);
      fwrite(hv.data(), 4, T, f);
      fclose(f);
    }
  }
  uint32_t *skeys = nullptr, *svals = nullptr;
  sort_records(T, kbits, &skeys, &svals, static_cast<uint32_t>(K));
  end(T, 0);
  begin(ST_RUNS);
  if (!marks_fused) {  // mark each voxel's run [start, end) (dense by key) from the sorted keys
    dense_start.ensure(K);
    dense_end.ensure(K);
    CU(cudaMemsetAsync(dense_end.p, 0, K * sizeof(uint32_t), st));
    k_run_marks<<<grid_for((T + 3) / 4), 256, 0, st>>>(T, skeys, dense_start.p, dense_end.p);
    ++launches;
  }
  // compact the runs in key order
  if (K > run_keys.cap || K > run_len.cap || K > run_start.cap || !num_runs.p || !work.p) sync_folds();
  run_keys.ensure(K);
  run_len.ensure(K);
  run_start.ensure(K);
  num_runs.ensure(1);
  work.ensure(2);
  scan_with<uint32_t>(RunIn{dense_end.p},
                      RunOut{K, dense_start.p, dense_end.p, run_keys.p, run_start.p, run_len.p, num_runs.p}, K);
  uint32_t nruns = 0;
  fetch({{&nruns, num_runs.p, sizeof(uint32_t)}});
  if (std::max<uint32_t>(nruns, 1) > std::min(run_len2.cap, run_order.cap)) sync_folds();
  run_len2.ensure(std::max<uint32_t>(nruns, 1));
  run_order.ensure(std::max<uint32_t>(nruns, 1));
  run_iota.ensure(std::max<uint32_t>(nruns, 1));
  run_code.ensure(std::max<uint32_t>(nruns, 1));
  run_max.ensure(1);
  if (nruns) {
    // fold order: one stable counting pass over a coarse length code, longest
    // runs first (they bound the fold's critical path), key order inside a
    // code (run_len_code); run_len2 receives the sorted codes
    CU(cudaMemsetAsync(run_max.p, 0, sizeof(uint32_t), st));
    k_run_codes<<<grid_for(nruns), 256, 0, st>>>(nruns, run_len.p, run_code.p, run_iota.p, run_max.p);
    ++launches;
    uint32_t *sk = nullptr, *sv = nullptr;
    const bool mf = marks_fused;
    const int lp = last_lsd_passes;
    sort_pairs32(nruns, 8, run_code.p, run_iota.p, run_len2.p, run_order.p, &sk, &sv);
    marks_fused = mf;
    last_lsd_passes = lp;
    if (sk != run_len2.p) throw VxgError(VXG_ECUDA, "run order sort: unexpected pass count");
  }
  end(T, 0);
  ensure_fold_streams();
  // longest run of this chunk, read back at the batch end
  if (nruns) {
    if (n_top == kTopCap) {
      CU(cudaStreamSynchronize(st));
      drain_tops();
    }
    top_T[n_top] = T;
    CU(cudaMemcpyAsync(top_pinned + n_top++, run_max.p, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
  }
  uint8_t* tch = consumers.empty() ? nullptr : touched.p;
  CU(cudaMemsetAsync(work.p, 0, 2 * sizeof(uint32_t), st));
  int dev_sms = 148;
  cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, device);
  // long runs: one CTA (4 producer/consumer pairs) per SM on fold_long_st;
  // short runs: k_fold_short on fold_st beside it (disjoint voxels). Both run
  // after this chunk's runs are ready (fold_fork) and after the previous
  // chunk's fold (fold_join); st goes on with the next chunk meanwhile.
  const unsigned long_grid = static_cast<unsigned>(std::max<uint64_t>(
      1, std::min<uint64_t>(static_cast<uint64_t>(dev_sms), (nruns + 3) / 4)));
  unsigned long long* dbg = nullptr;
  if (debug_fold) {
    fold_dbg.ensure(4 * nruns + 20);
    CU(cudaMemsetAsync(fold_dbg.p, 0, (4 * nruns + 20) * sizeof(unsigned long long), st));
    CU(cudaMemsetAsync(fold_dbg.p + 4 * nruns + 1, 0xFF, sizeof(unsigned long long), st));
    dbg = fold_dbg.p;
    fold_dbg_n = nruns;
  }
  if (nruns) {
    // origins of this set on st (d_poses is rewritten by the next batch
    // while this fold may still wait for the previous one)
    if (3ull * std::max<uint32_t>(F, 1) > d_org.cap) sync_folds();  // the set's old table may still be read
    d_org.ensure(3 * std::max<uint32_t>(F, 1));
    k_origins<<<grid_for(3 * F), 256, 0, st>>>(F, d_poses.p, d_org.p);
    ++launches;
    CU(cudaEventRecord(fold_fork, st));
    CU(cudaStreamWaitEvent(fold_long_st, fold_fork, 0));  // after the previous chunk's fold: same stream
    // The long-run grid must be resident before the short-run grid (persistent
    // CTAs) fills the SMs, or the longest chain starts only after every short
    // run is done (measured 3.7 vs 2.6 ms on cfg1): the short grid is its
    // programmatic dependent in the same stream (see k_fold_short).
    static const int long_layout = [] {
      const char* e = getenv("VXG_LONG_LAYOUT");
      return e ? atoi(e) : 0;
    }();
    static const int long_smem = [] {
      const char* e = getenv("VXG_LONG_SMEM");
      return e ? atoi(e) : 0;
    }();
    static const int long_ctas = [] {
      const char* e = getenv("VXG_LONG_CTAS");
      return e ? atoi(e) : 0;
    }();
    const unsigned lg = long_ctas > 0 ? static_cast<unsigned>(long_ctas) : long_grid;
    const bool smem_org = F <= kOrgCache;
    static const int fold_merged = [] {  // dev A/B: VXG_FOLD_MERGED=0 -> two grids (long + PDL short)
      const char* e = getenv("VXG_FOLD_MERGED");
      return e ? atoi(e) : 1;
    }();
    begin(ST_APPLY, fold_long_st);
    if (fold_merged) {
      static const int fold_kc = [] {  // dev A/B: records per short-run chunk (VXG_FOLD_KC = 1 | 2 | 3 | 4)
        const char* e = getenv("VXG_FOLD_KC");
        return e ? atoi(e) : 2;  // measured apply 2.74 / 2.34 / 2.38 / 2.57 ms for 1 / 2 / 3 / 4 (cfg1)
      }();
      // two producers per long run for small folds (their longest chain IS the fold: a single scan, the
      // simple integrator's one-frame batches); pairs + 8 short-run warps for full batches (issue-bound)
      static const int fold_prod = [] {  // dev A/B: VXG_FOLD_PROD = 1 | 2 forces a layout
        const char* e = getenv("VXG_FOLD_PROD");
        return e ? atoi(e) : 0;
      }();
      // Teams when the fold is chain-bound: its longest run, at ~20 ns per record, outlasts the rest of
      // the fold at ~1.1e11 records/s. Measured: cfg4 (longest run 9e-4 of the chunk's records) gains
      // 11 % with teams, cfg2 (~5e-4) loses 2 %, cfg1 (3e-4) loses 0.3 ms of apply: threshold 7e-4. The
      // longest run of THIS fold is only on the device; the ratio of the handle's most recent folds
      // stands in for it, and a small fold is one scan (its longest chain is all its rays).
      const bool teams = fold_prod ? fold_prod == 2
                                   : (chain_ratio >= 0.0 ? chain_ratio > 7e-4 || T < 20000000ull : T < 100000000ull);
      if (!smem_org) dbg = nullptr;  // the trace build stages the origins in shared memory (F <= kOrgCache)
      auto kern = dbg != nullptr ? (teams ? k_fold_all<true, 2, 2, true> : k_fold_all<true, 2, 1, true>)  // (trace: smem origins)
                  : !smem_org ? (teams ? k_fold_all<false, 2, 2> : k_fold_all<false, 2, 1>)
                            : (fold_kc == 1 ? k_fold_all<true, 1>
                                : (fold_kc == 3 ? k_fold_all<true, 3>
                                                : (fold_kc == 4 ? k_fold_all<true, 4>
                                                                : (teams ? k_fold_all<true, 2, 2> : k_fold_all<true, 2, 1>))));
      kern<<<static_cast<unsigned>(dev_sms), 512, 0, fold_long_st>>>(num_runs.p, run_order.p, run_len2.p, run_keys.p,
                                                                     run_start.p, run_len.p, svals, fold_rays.p,
                                                                     far_rays.p, d_org.p, F, view(), tp, tch, work.p,
                                                                     dbg);
      CU(cudaGetLastError());
      end(T, 2, fold_long_st);
      CU(cudaEventRecord(fold_join, fold_long_st));
      CU(cudaEventRecord(set_done[cur_set], fold_long_st));
      set_busy[cur_set] = true;
      fold_inflight = true;
      launches += 1;
      info_records += T;
      info_runs += nruns;
      static const bool no_pipe_m = getenv("VXG_NO_PIPELINE") != nullptr;
      if (no_pipe_m) join_folds();
      return;
    }
#define VXG_FOLD_LONG(P, SEP, THREADS)                                                                              \
  do {                                                                                                           \
    auto kern = smem_org ? k_fold_runs<P, SEP, true> : k_fold_runs<P, SEP, false>;                              \
    if (long_smem) CU(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, long_smem));      \
    kern<<<lg, THREADS, long_smem, fold_long_st>>>(num_runs.p, run_order.p, run_len2.p, run_keys.p, run_start.p,  \
                                                   run_len.p, svals, fold_rays.p, far_rays.p, d_org.p, F, view(), tp, tch, \
                                                   work.p, dbg);                                                 \
  } while (0)
    if (long_layout == 2)
      VXG_FOLD_LONG(2, true, 128);
    else
      VXG_FOLD_LONG(4, false, 256);
#undef VXG_FOLD_LONG
    static const int short_blocks = [] {
      const char* e = getenv("VXG_FOLD_SHORT_BLOCKS");
      return e ? atoi(e) : 5;
    }();
    static const bool serial = getenv("VXG_FOLD_SERIAL") != nullptr;  // dev: long runs uncontended
    const unsigned short_grid = static_cast<unsigned>(std::max<uint64_t>(
        1, std::min<uint64_t>(static_cast<uint64_t>(dev_sms) * 4, (nruns + 255) / 256)));
    cudaLaunchAttribute pdl[1];
    pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    pdl[0].val.programmaticStreamSerializationAllowed = serial ? 0 : 1;
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(short_grid);
    lc.blockDim = dim3(256);
    lc.dynamicSmemBytes = 0;
    lc.stream = fold_long_st;
    lc.attrs = pdl;
    lc.numAttrs = 1;
    MapView mv = view();
    const uint32_t* cnum = num_runs.p;
    const uint32_t* cord = run_order.p;
    const uint32_t* clen2 = run_len2.p;
    const uint32_t* ckey = run_keys.p;
    const uint32_t* cst = run_start.p;
    const uint32_t* clen = run_len.p;
    const uint32_t* csv = svals;
    const FoldRay* crays = fold_rays.p;
    const uint2* cfar = far_rays.p;
    const float* corg = d_org.p;
#define VXG_FOLD_SHORT(MB, C)                                                                                 \
  do {                                                                                                        \
    auto kern = smem_org ? k_fold_short<MB, C, true> : k_fold_short<MB, C, false>;                           \
    CU(cudaLaunchKernelEx(&lc, kern, cnum, cord, clen2, ckey, cst, clen, csv, crays, cfar, corg, F, mv, tp, tch, \
                          work.p));                                                                          \
  } while (0)
    if (short_blocks == 1)
      VXG_FOLD_SHORT(3, 4);
    else if (short_blocks == 3)
      VXG_FOLD_SHORT(2, 2);
    else if (short_blocks == 4)
      VXG_FOLD_SHORT(3, 2);
    else if (short_blocks == 6)
      VXG_FOLD_SHORT(4, 2);
    else
      VXG_FOLD_SHORT(2, 4);
#undef VXG_FOLD_SHORT
    end(T, 2, fold_long_st);
    CU(cudaEventRecord(fold_join, fold_long_st));
    CU(cudaEventRecord(set_done[cur_set], fold_long_st));
    set_busy[cur_set] = true;
    fold_inflight = true;
    launches += 2;
  }
  CU(cudaGetLastError());
  static const bool no_pipe = getenv("VXG_NO_PIPELINE") != nullptr;  // dev A/B: fold before the next chunk
  if (no_pipe) join_folds();
  info_records += T;
  info_runs += nruns;
}

// After a produce+sort_fold attempt: true if the map had to grow (the caller
// re-produces the records; the slab was not modified by the failed attempt).
bool vxg_handle::grew_after_attempt(int attempt) {
  uint32_t c[2];
  read_counters(c);
  last_blocks = c[0];
  if (c[1] & kErrKeyRange) throw VxgError(VXG_ERANGE, "voxel block index outside the supported range");
  if (c[1] & (kErrSlabFull | kErrHashFull)) {
    if (attempt > 64) throw VxgError(VXG_ENOMEM, "block allocation did not converge");
    sync_folds();  // earlier chunks' folds still read/write the slab that is about to move
    if (c[1] & kErrHashFull) rehash(hcap * 2);
    grow_map(std::max<uint64_t>(c[0], cap_blocks + 1));
    ensure_touched();
    return true;
  }
  return false;
}

// Pipeline chunks: records are produced, sorted and folded in chunks of
// consecutive rays (ray order), so every voxel still folds its updates in the
// reference's order (chunk by chunk). Chunk c's fold overlaps chunk c+1's emit
// and sort. Batches are chunked only when their records exceed kMaxRecords:
// measured on cfg1 (2.4e8 records), 4 chunks cost 14.4 vs 12.6 ms/step — a
// hot voxel's chain sits inside one chunk (its rays come from a few adjacent
// frames), so every chunk's fold is still bound by a full-length chain and
// the folds, which must run in chunk order, add up (VXG_CHUNK_RECORDS: A/B).
uint32_t pipeline_chunks(uint64_t total) {
  const uint64_t kMaxRecords = (1ull << 29) - (1ull << 20);  // keeps every chunk 32-bit addressable
  static const uint64_t per = [kMaxRecords] {
    const char* e = getenv("VXG_CHUNK_RECORDS");
    return e ? std::max<uint64_t>(1, strtoull(e, nullptr, 10)) : kMaxRecords;
  }();
  uint64_t n = std::max<uint64_t>((total + per - 1) / per, (total + kMaxRecords - 1) / kMaxRecords);
  return static_cast<uint32_t>(std::min<uint64_t>(std::max<uint64_t>(n, 1), 64));
}

void vxg_handle::emit_and_apply(uint32_t R, uint32_t F, const TermView& tv) {
  const TsdfParams tp = params();
  if (R > kRayMask) throw VxgError(VXG_EINVAL, "too many rays in one batch (record values hold 31-bit ray ids)");
  apply_pending_reset();
  const uint64_t total = count_rays(R, F);
  const uint32_t nch = pipeline_chunks(total);
  // chunk bounds (first ray, first record) by record count, on the device
  chunk_base.ensure(2 * (nch + 1));
  std::vector<unsigned long long> hb(2 * (nch + 1));
  k_chunk_bounds<<<1, 64, 0, st>>>(R, roff.p, total, nch, chunk_base.p);
  ++launches;
  // emission order: rays by decreasing record count inside each chunk (balanced
  // warps); the records still land at their ray-order offsets.
  ray_perm.ensure(R);
  ray_iota.ensure(R);
  ckeys.ensure(R);
  k_iota<<<grid_for(R), 256, 0, st>>>(R, ray_iota.p);
  k_chunk_keys<<<grid_for(R), 256, 0, st>>>(R, rcount.p, chunk_base.p, nch, ckeys.p);
  launches += 2;
  const int cbits = 16 + bits_for(nch - 1);
  sort_pairs64(ckeys.p, ray_iota.p, R, cbits, true, nullptr, ray_perm.p);
  ensure_touched();
  fetch({{hb.data(), chunk_base.p, hb.size() * sizeof(unsigned long long)}});
  d_upd.ensure(F);
  for (uint32_t c = 0; c < nch; ++c) {
    const uint32_t r0 = static_cast<uint32_t>(hb[c]), r1 = static_cast<uint32_t>(hb[c + 1]);
    const uint64_t base = hb[nch + 1 + c];
    const uint64_t T = hb[nch + 2 + c] - base;
    if (T == 0 || r1 <= r0) continue;
    swap_fold_set();
    ensure_records(T);
    for (int attempt = 0;; ++attempt) {
      CU(cudaMemsetAsync(counters.p + 1, 0, sizeof(uint32_t), st));
      CU(cudaMemsetAsync(d_upd.p, 0, F * sizeof(unsigned long long), st));
      begin(ST_EMIT);
      {
        const bool anti = tp.merge_mode == VXG_MERGE_GROUPED_ANTI_GRAZE;
        const bool pow2 = (vps & (vps - 1)) == 0;
        auto kern = anti ? (pow2 ? k_emit<true, true> : k_emit<true, false>)
                         : (pow2 ? k_emit<false, true> : k_emit<false, false>);
        kern<<<grid_for(r1 - r0, kEmitThreads), kEmitThreads, 0, st>>>(r0, r1, ray_perm.p, rays.p, roff.p, base, d_poses.p, tp, view(),
                                                     tv, rkeys.p, rvals.p, d_upd.p);
      }
      ++launches;
      CU(cudaGetLastError());
      end(T, 1);
      if (grew_after_attempt(attempt)) continue;
      sort_fold(T, last_blocks, F);
      break;
    }
    // fold this chunk's per-frame update counts into the stats
    k_add_u64<<<grid_for(F), 256, 0, st>>>(F, d_stats.p, d_upd.p);
    ++launches;
    CU(cudaGetLastError());
  }
  if (!fold_may_outlive_call()) join_folds();
}

// Stages the batch metadata and builds the rays (bundling + ray order).
void vxg_handle::begin_batch(const float* xyz, const uint8_t* rgb, const uint64_t* offsets, const float* poses,
                             uint64_t F, uint32_t* R_out, TermView* tv) {
  const uint64_t P = offsets[F] - offsets[0];
  std::vector<uint64_t> h_off(F + 1);
  for (uint64_t f = 0; f <= F; ++f) h_off[f] = offsets[f] - offsets[0];
  begin(ST_H2D);
  d_off.ensure(F + 1);
  d_poses.ensure(12 * F);
  d_stats.ensure(3 * F);
  CU(cudaMemcpyAsync(d_off.p, h_off.data(), (F + 1) * sizeof(uint64_t), cudaMemcpyHostToDevice, st));
  CU(cudaMemcpyAsync(d_poses.p, poses, 12 * F * sizeof(float), cudaMemcpyHostToDevice, st));
  CU(cudaMemsetAsync(d_stats.p, 0, 3 * F * sizeof(unsigned long long), st));
  CU(cudaMemsetAsync(counters.p + 1, 0, sizeof(uint32_t), st));
  const float* dxyz = xyz + 3 * offsets[0];
  const uint8_t* drgb = rgb != nullptr ? rgb + 3 * offsets[0] : nullptr;
  end(P * (drgb ? 15 : 12), 0);
  *R_out = 0;
  *tv = TermView{nullptr, nullptr, nullptr, 0, 0};
  if (P == 0) return;
  if (cfg.merge_mode == VXG_MERGE_SIMPLE) {
    build_rays_simple(dxyz, drgb, P, static_cast<uint32_t>(F), R_out);
  } else {
    build_rays_grouped(dxyz, drgb, P, h_off.data(), static_cast<uint32_t>(F), R_out, tv);
  }
  uint32_t c[2];
  read_counters(c);
  last_blocks = c[0];
  if (c[1] & kErrKeyRange) throw VxgError(VXG_ERANGE, "terminal voxel outside the bundling key range");
}

// Reads the per-frame stats back and feeds the updated-block consumers.
void vxg_handle::end_batch(uint64_t F, vxg_stats* out) {
  apply_pending_reset();  // a batch without rays never reached the map: the reset still applies
  if (!fold_may_outlive_call()) join_folds();
  begin(ST_D2H);
  std::vector<unsigned long long> s(3 * F);
  uint32_t c[2];
  end(0, 0);
  fetch({{s.data(), d_stats.p, 3 * F * sizeof(unsigned long long)}, {c, counters.p, 2 * sizeof(uint32_t)}});
  collect();
  drain_tops();
  if (out != nullptr) {
    for (uint64_t f = 0; f < F; ++f) {
      out[f].updates = s[f];
      out[f].raycasts = s[F + f];
      out[f].skipped = s[2 * F + f];
    }
  }
  // consumers: blocks touched by this batch
  const uint64_t nb = std::min<uint64_t>(c[0], cap_blocks);
  sync_block_mirror(nb);
  if (!consumers.empty() && nb > 0 && touched.p != nullptr) {
    std::vector<uint8_t> t(nb);
    fetch({{t.data(), touched.p, nb}});
    CU(cudaMemsetAsync(touched.p, 0, touched.cap, st));
    for (auto& kv : consumers)
      for (uint32_t i = 0; i < nb; ++i)
        if (t[i]) kv.second.insert(i);
  }
}

void vxg_handle::run_sub(const float* xyz, const uint8_t* rgb, const uint64_t* offsets, const float* poses,
                         uint64_t F, bool device_input, vxg_stats* out) {
  if (!device_input) throw VxgError(VXG_EINVAL, "internal: run_sub expects staged device inputs");
  uint32_t R = 0;
  TermView tv;
  begin_batch(xyz, rgb, offsets, poses, F, &R, &tv);
  if (sharded()) {
    if (nccl_comm == nullptr) throw VxgError(VXG_EINVAL, "sharded handle without a communicator (vxg_shard_init)");
    settle();
    shard_front(R, static_cast<uint32_t>(F), tv);
    if (!shard_replicated) nccl_exchange();
    shard_back(owned_records(), owned_count(), static_cast<uint32_t>(F));
    nccl_reduce_updates(static_cast<uint32_t>(F));
  } else if (R > 0) {
    emit_and_apply(R, static_cast<uint32_t>(F), tv);
  }
  end_batch(F, out);
}

// ---------------------------------------------------------------- sharded map
// Every shard bundles the whole batch (identical rays and ray order), walks a
// record-balanced contiguous slice of the global ray order, and partitions the
// slice's update records by block owner. Concatenating what an owner receives
// in source-rank order preserves ray order, so the owner's stable sort + fold
// reproduce the single-GPU result for its blocks exactly.
void vxg_handle::shard_front(uint32_t R, uint32_t F, const TermView& tv) {
  send_counts.assign(shard_world, 0);
  send_offsets.assign(shard_world, 0);
  if (R == 0) return;
  const TsdfParams tp = params();
  const uint64_t total = count_rays(R, F);
  uint32_t R0 = 0, R1 = R;
  unsigned long long base = 0, endrec = total;
  if (!shard_replicated) {
    // this rank's ray slice: records [rank*total/world, (rank+1)*total/world)
    sbounds.ensure(2);
    const uint64_t lo_rec = total * static_cast<uint64_t>(shard_rank) / shard_world;
    const uint64_t hi_rec = total * static_cast<uint64_t>(shard_rank + 1) / shard_world;
    k_ray_bounds<<<1, 32, 0, st>>>(R, roff.p, lo_rec, hi_rec, sbounds.p);
    ++launches;
    unsigned long long hb[2];
    CU(cudaMemcpyAsync(hb, sbounds.p, sizeof(hb), cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    R0 = static_cast<uint32_t>(hb[0]);
    R1 = static_cast<uint32_t>(hb[1]);
    if (R0 < R) CU(cudaMemcpy(&base, roff.p + R0, sizeof(base), cudaMemcpyDeviceToHost));
    else base = total;
    if (R1 < R) CU(cudaMemcpy(&endrec, roff.p + R1, sizeof(endrec), cudaMemcpyDeviceToHost));
  }  // replicated traversal (SURVEY.md 8e fallback): every rank walks all rays, keeps its own blocks
  const uint64_t T = endrec - base;
  if (T == 0) return;
  if (T >= 0xFFFFFFFFull) throw VxgError(VXG_EINVAL, "too many records in one sharded batch slice (32-bit offsets)");
  begin(ST_EMIT);
  gkeys.ensure(T);
  gowner.ensure(T);
  gowner2.ensure(T);
  giota.ensure(T);
  gperm.ensure(T);
  sh_keys.ensure(T);
  sh_vals.ensure(T);
  sh_upd.ensure(std::max<uint32_t>(F, 1));
  ray_iota.ensure(R);
  k_iota<<<grid_for(R), 256, 0, st>>>(R, ray_iota.p);  // the slice is walked in ray order
  ++launches;
  if (dict_cap == 0) dict_cap = std::max<uint64_t>(cap_blocks, 1024);
  for (;;) {
    if (dict_cap * static_cast<uint64_t>(nvox) >= 0xFFFFFFFFull)
      throw VxgError(VXG_ENOMEM, "sharded emit: block dictionary would exceed the 32-bit voxel key range");
    uint64_t hc = 1;
    while (hc < 2 * dict_cap) hc <<= 1;
    dict_hkeys.ensure(hc);
    dict_hvals.ensure(hc);
    dict_bidx.ensure(3 * dict_cap);
    dict_counters.ensure(2);
    CU(cudaMemsetAsync(dict_hkeys.p, 0xFF, hc * sizeof(unsigned long long), st));  // kEmptyKey
    CU(cudaMemsetAsync(dict_hvals.p, 0xFF, hc * sizeof(int32_t), st));             // kEmptySlot
    CU(cudaMemsetAsync(dict_counters.p, 0, 2 * sizeof(uint32_t), st));
    CU(cudaMemsetAsync(sh_upd.p, 0, std::max<uint32_t>(F, 1) * sizeof(unsigned long long), st));
    MapView dv = view();
    dv.hkeys = dict_hkeys.p;
    dv.hvals = dict_hvals.p;
    dv.hmask = hc - 1;
    dv.slab = nullptr;
    dv.block_idx = dict_bidx.p;
    dv.counters = dict_counters.p;
    dv.cap_blocks = static_cast<uint32_t>(dict_cap);
    const bool anti = tp.merge_mode == VXG_MERGE_GROUPED_ANTI_GRAZE;
    const bool pow2 = (vps & (vps - 1)) == 0;
    auto kern = anti ? (pow2 ? k_emit<true, true> : k_emit<true, false>)
                     : (pow2 ? k_emit<false, true> : k_emit<false, false>);
    kern<<<grid_for(R1 - R0, kEmitThreads), kEmitThreads, 0, st>>>(R0, R1, ray_iota.p, rays.p, roff.p, base, d_poses.p,
                                                                   tp, dv, tv, sh_keys.p, sh_vals.p, sh_upd.p);
    ++launches;
    CU(cudaGetLastError());
    uint32_t dc[2];
    fetch({{dc, dict_counters.p, sizeof(dc)}});
    if (dc[1] & kErrKeyRange) throw VxgError(VXG_ERANGE, "voxel block index outside the packed key range");
    if (dc[1] & (kErrSlabFull | kErrHashFull)) {  // dictionary too small: grow and walk again
      dict_cap = std::max<uint64_t>(2 * dict_cap, static_cast<uint64_t>(dc[0]) + dc[0] / 4);
      continue;
    }
    break;
  }
  k_globalize<<<grid_for(T), 256, 0, st>>>(T, sh_keys.p, dict_bidx.p, static_cast<uint32_t>(nvox),
                                           static_cast<uint32_t>(shard_world), shard_replicated ? shard_rank : -1,
                                           gkeys.p, gowner.p, counters.p);
  k_iota<<<grid_for(T), 256, 0, st>>>(static_cast<uint32_t>(T), giota.p);
  launches += 2;
  CU(cudaGetLastError());
  const int obits = bits_for(static_cast<uint64_t>(shard_world));
  uint32_t *so = nullptr, *sp = nullptr;  // stable partition by owner (invalid records: owner == world, last)
  sort_pairs32(T, obits, gowner.p, giota.p, gowner2.p, gperm.p, &so, &sp);
  obounds.ensure(shard_world + 1);
  k_owner_bounds<<<1, 64, 0, st>>>(T, so, static_cast<uint32_t>(shard_world), obounds.p);
  ++launches;
  std::vector<unsigned long long> bnd(shard_world + 1);
  CU(cudaMemcpyAsync(bnd.data(), obounds.p, (shard_world + 1) * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  uint32_t c[2];
  read_counters(c);
  last_blocks = c[0];
  if (c[1] & kErrKeyRange) throw VxgError(VXG_ERANGE, "voxel block index outside the sharded key range (+-2^14 blocks)");
  const uint64_t n_valid = bnd[shard_world];
  send_buf.ensure(std::max<uint64_t>(n_valid, 1));
  if (n_valid) {
    k_gather_send<<<grid_for(n_valid), 256, 0, st>>>(n_valid, sp, gkeys.p, sh_vals.p, send_buf.p);
    ++launches;
    CU(cudaGetLastError());
  }
  for (int o = 0; o < shard_world; ++o) {
    send_offsets[o] = bnd[o];
    send_counts[o] = bnd[o + 1] - bnd[o];
  }
  end(T, 0);
}

// Owner side: localize the received records (allocating owned blocks), then
// the same stable sort + ordered fold as one GPU; updates counted per frame.
void vxg_handle::shard_back(const uint4* recv, uint64_t n, uint32_t F) {
  d_upd.ensure(F);
  CU(cudaMemsetAsync(d_upd.p, 0, F * sizeof(unsigned long long), st));
  if (n > 0) {
    ensure_touched();
    ensure_records(n);
    for (int attempt = 0;; ++attempt) {
      CU(cudaMemsetAsync(counters.p + 1, 0, sizeof(uint32_t), st));
      CU(cudaMemsetAsync(d_upd.p, 0, F * sizeof(unsigned long long), st));
      k_localize<<<grid_for(n), 256, 0, st>>>(n, recv, view(), fold_rays.p, rkeys.p, rvals.p, d_upd.p);
      ++launches;
      CU(cudaGetLastError());
      if (grew_after_attempt(attempt)) continue;
      sort_fold(n, last_blocks, F);
      break;
    }
  }
  k_add_u64<<<grid_for(F), 256, 0, st>>>(F, d_stats.p, d_upd.p);
  ++launches;
  CU(cudaGetLastError());
}

// ---------------------------------------------------------------- NCCL (dlopen)
// NCCL is loaded at run time (libnccl.so.2: torch's or the system's) so the
// library has no link-time dependency on it; only sharded multi-GPU handles use it.
namespace {

struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi* nccl() {
  static NcclApi api;
  static bool loaded = false;
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  if (loaded) return &api;
  void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (lib == nullptr) lib = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (lib == nullptr) throw VxgError(VXG_ECUDA, "cannot load libnccl.so.2 for the sharded path");
  auto sym = [&](const char* n) {
    void* p = dlsym(lib, n);
    if (p == nullptr) throw VxgError(VXG_ECUDA, std::string("libnccl lacks ") + n);
    return p;
  };
  api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
  api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
  api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
  api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
  api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
  api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
  api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
  api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
  api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
  loaded = true;
  return &api;
}

#define NC(x)                                                                                   \
  do {                                                                                          \
    ncclResult_t r_ = (x);                                                                      \
    if (r_ != ncclSuccess) throw VxgError(VXG_ECUDA, std::string("NCCL: ") + nccl()->GetErrorString(r_)); \
  } while (0)

}  // namespace

// All-to-all of the per-owner record buffers over NVLink (ncclSend/ncclRecv
// group): counts first, then the 16-byte records, received in source-rank
// order into one contiguous buffer.
void vxg_handle::nccl_exchange() {
  NcclApi* nc = nccl();
  auto comm = static_cast<ncclComm_t>(nccl_comm);
  const int W = shard_world;
  dev_counts.ensure(2 * W);
  std::vector<unsigned long long> sc(W);
  for (int p = 0; p < W; ++p) sc[p] = send_counts[p];
  CU(cudaMemcpyAsync(dev_counts.p, sc.data(), W * sizeof(unsigned long long), cudaMemcpyHostToDevice, st));
  NC(nc->GroupStart());
  for (int p = 0; p < W; ++p) {
    NC(nc->Send(dev_counts.p + p, 1, ncclUint64, p, comm, st));
    NC(nc->Recv(dev_counts.p + W + p, 1, ncclUint64, p, comm, st));
  }
  NC(nc->GroupEnd());
  std::vector<unsigned long long> rc(W);
  CU(cudaMemcpyAsync(rc.data(), dev_counts.p + W, W * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  recv_counts.assign(W, 0);
  recv_total = 0;
  std::vector<uint64_t> roffs(W);
  for (int p = 0; p < W; ++p) {
    recv_counts[p] = rc[p];
    roffs[p] = recv_total;
    recv_total += rc[p];
  }
  recv_buf.ensure(std::max<uint64_t>(recv_total, 1));
  send_buf.ensure(1);
  NC(nc->GroupStart());
  for (int p = 0; p < W; ++p) {
    if (send_counts[p]) NC(nc->Send(send_buf.p + send_offsets[p], send_counts[p] * sizeof(uint4), ncclUint8, p, comm, st));
    if (recv_counts[p]) NC(nc->Recv(recv_buf.p + roffs[p], recv_counts[p] * sizeof(uint4), ncclUint8, p, comm, st));
  }
  NC(nc->GroupEnd());
}

// Per-frame update counts are partial per owner: sum them over the shards.
void vxg_handle::nccl_reduce_updates(uint32_t F) {
  NC(nccl()->AllReduce(d_stats.p, d_stats.p, F, ncclUint64, ncclSum, static_cast<ncclComm_t>(nccl_comm), st));
}

// Loopback exchange for a group of shards on ONE device (all on one stream):
// the same sharded kernels, with device-to-device copies standing in for NVLink.
struct vxg_group {
  std::vector<vxg_handle*> shards;
};

namespace {

void group_exchange(vxg_group* g) {
  const int W = static_cast<int>(g->shards.size());
  cudaStream_t st = g->shards[0]->st;
  for (int dst = 0; dst < W; ++dst) {
    vxg_handle* d = g->shards[dst];
    uint64_t total = 0;
    for (int src = 0; src < W; ++src) total += g->shards[src]->send_counts.empty() ? 0 : g->shards[src]->send_counts[dst];
    d->recv_buf.ensure(std::max<uint64_t>(total, 1));
    d->recv_total = total;
    uint64_t at = 0;
    for (int src = 0; src < W; ++src) {
      vxg_handle* s = g->shards[src];
      if (s->send_counts.empty() || s->send_counts[dst] == 0) continue;
      CU(cudaMemcpyAsync(d->recv_buf.p + at, s->send_buf.p + s->send_offsets[dst], s->send_counts[dst] * sizeof(uint4),
                         cudaMemcpyDeviceToDevice, st));
      at += s->send_counts[dst];
    }
  }
}

}  // namespace

// ============================================================================ C ABI
namespace {

template <typename Fn>
int guarded(Fn fn) {
  cudaGetLastError();  // do not inherit a stale, non-sticky error from an unrelated earlier call
  try {
    fn();
    return VXG_OK;
  } catch (const VxgError& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "host allocation failed";
    return VXG_ENOMEM;
  } catch (const std::exception& e) {
    g_err = e.what();
    return VXG_EINVAL;
  }
}

void set_device(const vxg_handle* h) { CU(cudaSetDevice(h->device)); }

template <typename T>
T* to_dev(const T* src, size_t n, DBuf<T>* buf) {
  buf->ensure(std::max<size_t>(n, 1));
  if (n) CU(cudaMemcpy(buf->p, src, n * sizeof(T), cudaMemcpyHostToDevice));
  return buf->p;
}

void export_sorted(vxg_handle* h, std::vector<uint32_t>* order) {
  uint32_t c[2];
  h->read_counters(c);
  h->sync_block_mirror(std::min<uint64_t>(c[0], h->cap_blocks));
  order->resize(h->n_blocks);
  for (uint32_t i = 0; i < h->n_blocks; ++i) (*order)[i] = i;
  const int32_t* idx = h->host_idx.data();
  std::sort(order->begin(), order->end(), [&](uint32_t a, uint32_t b) {
    const int32_t* A = idx + 3 * a;
    const int32_t* B = idx + 3 * b;
    if (A[0] != B[0]) return A[0] < B[0];
    if (A[1] != B[1]) return A[1] < B[1];
    return A[2] < B[2];
  });
}

// Copies the blocks at slots[0..n) (host array) into `dst` (host memory,
// n * vps^3 voxels, pads zeroed): a device gather into contiguous scratch,
// then one D2H per piece of at most 256 MB.
void gather_to_host(vxg_handle* h, const uint32_t* slots, uint64_t n, vxg_voxel* dst) {
  const uint64_t nv = static_cast<uint64_t>(h->nvox);
  const uint64_t per = std::max<uint64_t>(1, (256ull << 20) / (nv * sizeof(vxg_voxel)));
  DBuf<uint32_t> dslots;
  DBuf<vxg_voxel> buf;
  dslots.ensure(std::min(per, n));
  buf.ensure(std::min(per, n) * nv);
  for (uint64_t k0 = 0; k0 < n; k0 += per) {
    const uint64_t m = std::min(per, n - k0);
    CU(cudaMemcpyAsync(dslots.p, slots + k0, m * sizeof(uint32_t), cudaMemcpyHostToDevice, h->st));
    k_gather_blocks<<<grid_for(m * nv * 3), 256, 0, h->st>>>(m, dslots.p, h->slab.p, static_cast<uint32_t>(nv), buf.p);
    CU(cudaGetLastError());
    CU(cudaMemcpyAsync(dst + k0 * nv, buf.p, m * nv * sizeof(vxg_voxel), cudaMemcpyDeviceToHost, h->st));
    CU(cudaStreamSynchronize(h->st));
  }
}

}  // namespace

extern "C" {

const char* vxg_last_error(void) { return g_err.c_str(); }

int vxg_device_info(int device, char* buf, size_t buf_len) {
  return guarded([&] {
    cudaDeviceProp p;
    CU(cudaGetDeviceProperties(&p, device));
    std::snprintf(buf, buf_len, "%s sm_%d%d SMs=%d HBM=%.1fGB L2=%.0fMB", p.name, p.major, p.minor,
                  p.multiProcessorCount, p.totalGlobalMem / 1e9, p.l2CacheSize / 1e6);
  });
}

int vxg_create(const vxg_tsdf_config* config, float voxel_size, int vps, int device, uint64_t block_capacity,
               vxg_handle** out) {
  return guarded([&] {
    if (config == nullptr || out == nullptr) throw VxgError(VXG_EINVAL, "null argument");
    if (voxel_size <= 0.0f || vps < 1)  // layer.h:62-67
      throw VxgError(VXG_EINVAL, "layer requires voxel_size > 0 and voxels_per_side >= 1");
    if (vps > 64) throw VxgError(VXG_EINVAL, "voxels_per_side > 64 is not supported on the device slab");
    const std::string msg = validate_config(config);
    if (!msg.empty()) throw VxgError(VXG_EINVAL, msg);
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
      cudaGetLastError();
      throw VxgError(VXG_ECUDA, "no CUDA device available (vxg has no CPU fallback)");
    }
    if (device < 0 || device >= ndev) throw VxgError(VXG_EINVAL, "device index out of range");
    cudaDeviceProp prop;
    CU(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10) throw VxgError(VXG_ECUDA, std::string("vxg is built for sm_100a; device is ") + prop.name);
    auto* h = new vxg_handle;
    try {
      h->cfg = *config;
      h->voxel_size = voxel_size;
      h->vps = vps;
      h->nvox = vps * vps * vps;
      h->device = device;
      CU(cudaSetDevice(device));
      CU(cudaStreamCreateWithFlags(&h->own, cudaStreamNonBlocking));
      h->st = h->own;
      h->async_fold = getenv("VXG_SYNC_FOLD") == nullptr;  // dev A/B: every call joins its fold
      h->alloc_map(block_capacity ? block_capacity : 4096);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

int vxg_destroy(vxg_handle* h) {
  if (h == nullptr) return VXG_OK;
  return guarded([&] {
    cudaSetDevice(h->device);
    h->sync_folds();
    if (h->st != nullptr && h->st == h->own) cudaStreamSynchronize(h->st);
    if (h->own) cudaStreamSynchronize(h->own);
    for (auto& pe : h->pending) {
      cudaEventDestroy(pe.second.first);
      cudaEventDestroy(pe.second.second);
    }
    for (cudaEvent_t e : h->event_pool) cudaEventDestroy(e);
    if (h->copy_st) {
      cudaStreamSynchronize(h->copy_st);
      cudaStreamDestroy(h->copy_st);
    }
    for (cudaEvent_t e : h->copy_events) cudaEventDestroy(e);
    for (auto& ss : h->stage_slot) {
      if (ss.copied) cudaEventDestroy(ss.copied);
      if (ss.released) cudaEventDestroy(ss.released);
    }
    if (h->fold_st) {
      cudaStreamSynchronize(h->fold_st);
      cudaStreamSynchronize(h->fold_long_st);
      cudaStreamDestroy(h->fold_st);
      cudaStreamDestroy(h->fold_long_st);
      cudaEventDestroy(h->fold_fork);
      cudaEventDestroy(h->fold_join);
      cudaEventDestroy(h->fold_long_done);
      cudaEventDestroy(h->fold_origins);
      for (cudaEvent_t e : h->set_done) cudaEventDestroy(e);
      cudaFreeHost(h->top_pinned);
    }
    if (h->mailbox) cudaFreeHost(h->mailbox);
    if (h->nccl_comm) nccl()->CommDestroy(static_cast<ncclComm_t>(h->nccl_comm));
    if (h->own) cudaStreamDestroy(h->own);
    delete h;
  });
}

int vxg_get_config(const vxg_handle* h, vxg_tsdf_config* out) {
  if (h == nullptr || out == nullptr) return VXG_EINVAL;
  *out = h->cfg;
  return VXG_OK;
}

// Orders the handle's stream after every fold launched so far (a batch's fold
// may outlive vxg_integrate_*), and applies a deferred reset. No host sync:
// work queued on the stream afterwards (an event, a copy) sees the final map.
int vxg_flush(vxg_handle* h) {
  return guarded([&] {
    if (h == nullptr) throw VxgError(VXG_EINVAL, "null argument");
    set_device(h);
    h->settle();
  });
}

int vxg_set_config(vxg_handle* h, const vxg_tsdf_config* config) {
  return guarded([&] {
    const std::string msg = validate_config(config);
    if (!msg.empty()) throw VxgError(VXG_EINVAL, msg);
    h->cfg = *config;
  });
}

int vxg_set_stream(vxg_handle* h, void* stream) {
  return guarded([&] {
    set_device(h);
    h->settle();
    CU(cudaStreamSynchronize(h->st));
    h->st = stream != nullptr ? static_cast<cudaStream_t>(stream) : h->own;
  });
}

namespace {

struct Copy {
  uint64_t dst_pt;  // destination point offset in the staging buffer
  const float* xyz;
  const uint8_t* rgb;
  uint64_t n;
};

// Frame-aligned sub-batches: <= 2^30 points each (32-bit point indices).
std::vector<std::pair<uint64_t, uint64_t>> plan_subbatches(const uint64_t* off, uint64_t F, bool host_input) {
  const uint64_t P = off[F] - off[0];
  // Device input: one sub-batch whenever it fits. Host input: split so the H2D
  // copy of part k+1 overlaps the compute of part k.
  // Two parts for large host batches: measured on B200 (cfg1, 100 frames,
  // 460 MB over PCIe) 20.1 ms vs 21.7 ms for one part; more parts lose more in
  // the fold (fewer records per voxel per launch) than they hide.
  static const int env_parts = [] {
    const char* e = getenv("VXG_H2D_PARTS");
    return e ? std::max(1, atoi(e)) : 0;
  }();
  const uint64_t h2d_parts = env_parts > 0 ? static_cast<uint64_t>(env_parts) : (P >= (1ull << 24) ? 2ull : 1ull);
  uint64_t target = 1ull << 30;
  if (host_input && h2d_parts > 1) target = std::max<uint64_t>(1, (P + h2d_parts - 1) / h2d_parts);
  std::vector<std::pair<uint64_t, uint64_t>> parts;
  uint64_t f0 = 0;
  while (f0 < F) {
    uint64_t f1 = f0 + 1;
    while (f1 < F && off[f1 + 1] - off[f0] <= target && f1 - f0 < 65535) ++f1;
    if (off[f1] - off[f0] >= (1ull << 31)) throw VxgError(VXG_EINVAL, "a single scan exceeds 2^31 points");
    parts.emplace_back(f0, f1);
    f0 = f1;
  }
  return parts;
}

// Device-resident inputs: run the sub-batches directly. Host inputs: stage them
// into device memory on the copy stream (one event per sub-batch) and let each
// sub-batch's compute wait only for its own copy.
void integrate_staged(vxg_handle* h, const std::vector<Copy>& copies, const float* dev_xyz, const uint8_t* dev_rgb,
                      bool any_rgb, const uint64_t* off, const float* poses, uint64_t F, bool device_input,
                      vxg_stats* out) {
  const auto parts = plan_subbatches(off, F, !device_input);
  const float* bx = dev_xyz;
  const uint8_t* bc = dev_rgb;
  if (!device_input) {
    const uint64_t P = off[F] - off[0];
    float* sx = h->in_xyz.ensure(std::max<uint64_t>(3 * P, 3));
    uint8_t* sc = any_rgb ? h->in_rgb.ensure(std::max<uint64_t>(3 * P, 3)) : nullptr;
    if (h->copy_st == nullptr) CU(cudaStreamCreateWithFlags(&h->copy_st, cudaStreamNonBlocking));
    while (h->copy_events.size() < parts.size()) {
      cudaEvent_t e;
      CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      h->copy_events.push_back(e);
    }
    // the staging buffers may still be read by the previous call's kernels
    cudaEvent_t prev_done = h->ev();
    CU(cudaEventRecord(prev_done, h->st));
    CU(cudaStreamWaitEvent(h->copy_st, prev_done, 0));
    size_t ci = 0;
    for (size_t p = 0; p < parts.size(); ++p) {
      const uint64_t end_pt = off[parts[p].second] - off[0];
      while (ci < copies.size() && copies[ci].dst_pt < end_pt) {
        const Copy& c = copies[ci++];
        if (c.n == 0) continue;
        CU(cudaMemcpyAsync(sx + 3 * c.dst_pt, c.xyz, 3 * c.n * sizeof(float), cudaMemcpyHostToDevice, h->copy_st));
        if (sc != nullptr && c.rgb != nullptr)
          CU(cudaMemcpyAsync(sc + 3 * c.dst_pt, c.rgb, 3 * c.n, cudaMemcpyHostToDevice, h->copy_st));
      }
      CU(cudaEventRecord(h->copy_events[p], h->copy_st));
    }
    h->event_pool.push_back(prev_done);
    bx = sx;
    bc = sc;
  }
  // rebase: staging buffers start at point off[0]
  std::vector<uint64_t> roff(F + 1);
  for (uint64_t f = 0; f <= F; ++f) roff[f] = off[f] - off[0];
  for (size_t p = 0; p < parts.size(); ++p) {
    if (!device_input) CU(cudaStreamWaitEvent(h->st, h->copy_events[p], 0));
    const uint64_t f0 = parts[p].first, f1 = parts[p].second;
    h->run_sub(device_input ? dev_xyz : bx, device_input ? dev_rgb : bc, (device_input ? off : roff.data()) + f0,
               poses + 12 * f0, f1 - f0, true, out ? out + f0 : nullptr);
  }
}

}  // namespace

int vxg_integrate_packed(vxg_handle* h, const float* xyz, const uint8_t* rgb, const uint64_t* offsets,
                         const float* poses, uint64_t F, int flags, vxg_stats* out) {
  return guarded([&] {
    if (h == nullptr || offsets == nullptr || poses == nullptr) throw VxgError(VXG_EINVAL, "null argument");
    if (F == 0) return;
    for (uint64_t f = 0; f < F; ++f)
      if (offsets[f + 1] < offsets[f]) throw VxgError(VXG_EINVAL, "frame offsets must be non-decreasing");
    if (offsets[F] > offsets[0] && xyz == nullptr) throw VxgError(VXG_EINVAL, "null point buffer");
    set_device(h);
    const bool dev = (flags & VXG_INPUT_DEVICE) != 0;
    std::vector<Copy> copies;
    if (!dev) {
      // one copy per frame keeps the sub-batch events frame-aligned
      for (uint64_t f = 0; f < F; ++f)
        copies.push_back({offsets[f] - offsets[0], xyz + 3 * offsets[f], rgb ? rgb + 3 * offsets[f] : nullptr,
                          offsets[f + 1] - offsets[f]});
    }
    integrate_staged(h, copies, xyz, rgb, rgb != nullptr, offsets, poses, F, dev, out);
  });
}

int vxg_stage_packed(vxg_handle* h, const float* xyz, const uint8_t* rgb, const uint64_t* offsets, uint64_t F,
                     int* slot) {
  return guarded([&] {
    if (h == nullptr || offsets == nullptr || slot == nullptr) throw VxgError(VXG_EINVAL, "null argument");
    for (uint64_t f = 0; f < F; ++f)
      if (offsets[f + 1] < offsets[f]) throw VxgError(VXG_EINVAL, "frame offsets must be non-decreasing");
    const uint64_t P = F ? offsets[F] - offsets[0] : 0;
    if (P > 0 && xyz == nullptr) throw VxgError(VXG_EINVAL, "null point buffer");
    const int k = h->next_stage;
    vxg_handle::StageSlot& ss = h->stage_slot[k];
    if (ss.full) throw VxgError(VXG_EINVAL, "both staging slots hold batches not yet integrated");
    set_device(h);
    if (h->copy_st == nullptr) CU(cudaStreamCreateWithFlags(&h->copy_st, cudaStreamNonBlocking));
    if (ss.copied == nullptr) {
      CU(cudaEventCreateWithFlags(&ss.copied, cudaEventDisableTiming));
      CU(cudaEventCreateWithFlags(&ss.released, cudaEventDisableTiming));
    }
    // the slot's buffers may still be read by the batch integrated from it last
    if (ss.used) CU(cudaStreamWaitEvent(h->copy_st, ss.released, 0));
    float* dx = ss.xyz.ensure(std::max<uint64_t>(3 * P, 3));
    uint8_t* dc = rgb != nullptr ? ss.rgb.ensure(std::max<uint64_t>(3 * P, 3)) : nullptr;
    if (P > 0) {
      CU(cudaMemcpyAsync(dx, xyz + 3 * offsets[0], 3 * P * sizeof(float), cudaMemcpyHostToDevice, h->copy_st));
      if (dc != nullptr)
        CU(cudaMemcpyAsync(dc, rgb + 3 * offsets[0], 3 * P, cudaMemcpyHostToDevice, h->copy_st));
    }
    CU(cudaEventRecord(ss.copied, h->copy_st));
    ss.off.assign(F + 1, 0);
    for (uint64_t f = 0; f <= F; ++f) ss.off[f] = offsets[f] - offsets[0];
    ss.has_rgb = rgb != nullptr;
    ss.full = true;
    h->next_stage = k ^ 1;
    *slot = k;
  });
}

int vxg_integrate_staged(vxg_handle* h, int slot, const float* poses, vxg_stats* out) {
  return guarded([&] {
    if (h == nullptr) throw VxgError(VXG_EINVAL, "null argument");
    if (slot < 0 || slot > 1 || !h->stage_slot[slot].full) throw VxgError(VXG_EINVAL, "no batch staged in this slot");
    vxg_handle::StageSlot& ss = h->stage_slot[slot];
    const uint64_t F = ss.off.size() - 1;
    if (F > 0 && poses == nullptr) throw VxgError(VXG_EINVAL, "null argument");
    set_device(h);
    ss.full = false;  // consumed even if the integration throws (the copy is complete or abandoned)
    CU(cudaStreamWaitEvent(h->st, ss.copied, 0));
    if (F > 0)
      integrate_staged(h, {}, ss.xyz.p, ss.has_rgb ? ss.rgb.p : nullptr, ss.has_rgb, ss.off.data(), poses, F, true,
                       out);
    CU(cudaEventRecord(ss.released, h->st));
    ss.used = true;
  });
}

int vxg_integrate_batch(vxg_handle* h, const vxg_frame* frames, uint64_t F, int flags, vxg_stats* out) {
  return guarded([&] {
    if (h == nullptr || (frames == nullptr && F > 0)) throw VxgError(VXG_EINVAL, "null argument");
    if (F == 0) return;
    set_device(h);
    const bool dev = (flags & VXG_INPUT_DEVICE) != 0;
    uint64_t P = 0;
    bool any_rgb = false, mixed_rgb = false;
    for (uint64_t f = 0; f < F; ++f) {
      P += frames[f].n;
      any_rgb = any_rgb || frames[f].rgb != nullptr;
    }
    for (uint64_t f = 0; f < F; ++f)
      if (any_rgb && frames[f].rgb == nullptr && frames[f].n > 0) mixed_rgb = true;
    if (mixed_rgb) {  // colour presence differs per scan: integrate scan by scan
      for (uint64_t f = 0; f < F; ++f) {
        const uint64_t o2[2] = {0, frames[f].n};
        std::vector<Copy> c{{0, frames[f].xyz, frames[f].rgb, frames[f].n}};
        integrate_staged(h, dev ? std::vector<Copy>{} : c, frames[f].xyz, frames[f].rgb, frames[f].rgb != nullptr,
                         o2, frames[f].pose, 1, dev, out ? out + f : nullptr);
      }
      return;
    }
    std::vector<uint64_t> off(F + 1, 0);
    std::vector<float> poses(12 * F);
    std::vector<Copy> copies;
    for (uint64_t f = 0; f < F; ++f) {
      off[f + 1] = off[f] + frames[f].n;
      std::memcpy(&poses[12 * f], frames[f].pose, 12 * sizeof(float));
      copies.push_back({off[f], frames[f].xyz, frames[f].rgb, frames[f].n});
    }
    if (!dev) {
      integrate_staged(h, copies, nullptr, nullptr, any_rgb, off.data(), poses.data(), F, false, out);
      return;
    }
    // device frames in separate allocations: gather into the packed staging buffer
    float* sx = h->in_xyz.ensure(std::max<uint64_t>(3 * P, 3));
    uint8_t* sc = any_rgb ? h->in_rgb.ensure(std::max<uint64_t>(3 * P, 3)) : nullptr;
    for (const Copy& c : copies) {
      if (c.n == 0) continue;
      CU(cudaMemcpyAsync(sx + 3 * c.dst_pt, c.xyz, 3 * c.n * sizeof(float), cudaMemcpyDeviceToDevice, h->st));
      if (sc) CU(cudaMemcpyAsync(sc + 3 * c.dst_pt, c.rgb, 3 * c.n, cudaMemcpyDeviceToDevice, h->st));
    }
    integrate_staged(h, {}, sx, sc, any_rgb, off.data(), poses.data(), F, true, out);
  });
}

int vxg_integrate(vxg_handle* h, const float* xyz, const uint8_t* rgb, uint64_t n, const float pose[12],
                  vxg_stats* out) {
  vxg_frame fr;
  fr.xyz = xyz;
  fr.rgb = rgb;
  fr.n = n;
  if (pose == nullptr) {
    g_err = "null pose";
    return VXG_EINVAL;
  }
  std::memcpy(fr.pose, pose, sizeof(fr.pose));
  vxg_stats s{0, 0, 0};
  const int rc = vxg_integrate_batch(h, &fr, 1, VXG_INPUT_HOST, &s);
  if (rc == VXG_OK && out != nullptr) *out = s;
  return rc;
}

int vxg_block_count(vxg_handle* h, uint64_t* out) {
  return guarded([&] {
    set_device(h);
    h->settle();
    uint32_t c[2];
    h->read_counters(c);
    *out = std::min<uint64_t>(c[0], h->cap_blocks);
  });
}

int vxg_export_blocks(vxg_handle* h, int32_t* idx, vxg_voxel* voxels, uint64_t cap, uint64_t* n_out) {
  return guarded([&] {
    set_device(h);
    h->settle();
    std::vector<uint32_t> order;
    export_sorted(h, &order);
    const uint64_t n = std::min<uint64_t>(cap, order.size());
    if (idx != nullptr) {
      for (uint64_t k = 0; k < n; ++k)
        for (int a = 0; a < 3; ++a) idx[3 * k + a] = h->host_idx[3 * order[k] + a];
    }
    if (voxels != nullptr && n > 0) gather_to_host(h, order.data(), n, voxels);
    if (n_out) *n_out = n;
  });
}

int vxg_fetch_blocks(vxg_handle* h, const int32_t* idx, uint64_t n, vxg_voxel* voxels, uint8_t* found) {
  return guarded([&] {
    set_device(h);
    h->settle();
    if (n == 0) return;
    if (idx == nullptr) throw VxgError(VXG_EINVAL, "null argument");
    const uint64_t nv = static_cast<uint64_t>(h->nvox);
    const uint64_t per = std::max<uint64_t>(1, (256ull << 20) / (nv * sizeof(vxg_voxel)));
    DBuf<int32_t> didx;
    DBuf<uint32_t> dslots;
    DBuf<vxg_voxel> buf;
    std::vector<uint32_t> hs;
    didx.ensure(3 * std::min(per, n));
    dslots.ensure(std::min(per, n));
    if (voxels != nullptr) buf.ensure(std::min(per, n) * nv);
    for (uint64_t k0 = 0; k0 < n; k0 += per) {
      const uint64_t m = std::min(per, n - k0);
      CU(cudaMemcpyAsync(didx.p, idx + 3 * k0, 3 * m * sizeof(int32_t), cudaMemcpyHostToDevice, h->st));
      k_block_slots<<<grid_for(m), 256, 0, h->st>>>(m, didx.p, h->view(), dslots.p);
      CU(cudaGetLastError());
      if (voxels != nullptr) {
        k_gather_blocks<<<grid_for(m * nv * 3), 256, 0, h->st>>>(m, dslots.p, h->slab.p, static_cast<uint32_t>(nv),
                                                                 buf.p);
        CU(cudaGetLastError());
        CU(cudaMemcpyAsync(voxels + k0 * nv, buf.p, m * nv * sizeof(vxg_voxel), cudaMemcpyDeviceToHost, h->st));
      }
      if (found != nullptr) {
        hs.resize(m);
        CU(cudaMemcpyAsync(hs.data(), dslots.p, m * sizeof(uint32_t), cudaMemcpyDeviceToHost, h->st));
      }
      CU(cudaStreamSynchronize(h->st));
      if (found != nullptr)
        for (uint64_t k = 0; k < m; ++k) found[k0 + k] = hs[k] != 0xFFFFFFFFu ? 1 : 0;
    }
  });
}

int vxg_import_blocks(vxg_handle* h, const int32_t* idx, const vxg_voxel* voxels, uint64_t n) {
  return guarded([&] {
    set_device(h);
    h->settle();
    if (n == 0) return;
    // A block index given more than once: the last copy wins whole, as in the
    // reference's load (get_or_allocate_block + read_voxel per block,
    // serialization.cpp:193-212). Earlier copies are dropped before upload.
    std::vector<int32_t> uidx;
    std::vector<vxg_voxel> uvox;
    {
      std::map<std::array<int32_t, 3>, uint64_t> last;
      for (uint64_t b = 0; b < n; ++b) last[{idx[3 * b], idx[3 * b + 1], idx[3 * b + 2]}] = b;
      if (last.size() != n) {
        const uint64_t nv = static_cast<uint64_t>(h->nvox);
        std::vector<uint64_t> keep;
        keep.reserve(last.size());
        for (uint64_t b = 0; b < n; ++b)
          if (last[{idx[3 * b], idx[3 * b + 1], idx[3 * b + 2]}] == b) keep.push_back(b);
        uidx.resize(3 * keep.size());
        uvox.resize(keep.size() * nv);
        for (size_t k = 0; k < keep.size(); ++k) {
          std::memcpy(uidx.data() + 3 * k, idx + 3 * keep[k], 3 * sizeof(int32_t));
          std::memcpy(uvox.data() + k * nv, voxels + keep[k] * nv, nv * sizeof(vxg_voxel));
        }
        idx = uidx.data();
        voxels = uvox.data();
        n = keep.size();
      }
    }
    DBuf<int32_t> didx, slots;
    DBuf<vxg_voxel> dv;
    didx.ensure(3 * n);
    slots.ensure(n);
    dv.ensure(n * h->nvox);
    CU(cudaMemcpyAsync(didx.p, idx, 3 * n * sizeof(int32_t), cudaMemcpyHostToDevice, h->st));
    CU(cudaMemcpyAsync(dv.p, voxels, n * h->nvox * sizeof(vxg_voxel), cudaMemcpyHostToDevice, h->st));
    for (int attempt = 0;; ++attempt) {
      CU(cudaMemsetAsync(h->counters.p + 1, 0, sizeof(uint32_t), h->st));
      k_import_slots<<<grid_for(n), 256, 0, h->st>>>(n, didx.p, h->view(), slots.p);
      CU(cudaGetLastError());
      uint32_t c[2];
      h->read_counters(c);
      if (c[1] & kErrKeyRange) throw VxgError(VXG_ERANGE, "block index outside the supported range");
      if (c[1] & (kErrSlabFull | kErrHashFull)) {
        if (attempt > 64) throw VxgError(VXG_ENOMEM, "block allocation did not converge");
        if (c[1] & kErrHashFull) h->rehash(h->hcap * 2);
        h->grow_map(std::max<uint64_t>(c[0], h->cap_blocks + 1));
        continue;
      }
      break;
    }
    k_scatter_blocks<<<grid_for(n * h->nvox), 256, 0, h->st>>>(n, slots.p, dv.p, h->view());
    CU(cudaGetLastError());
    uint32_t c[2];
    h->read_counters(c);
    h->sync_block_mirror(std::min<uint64_t>(c[0], h->cap_blocks));
  });
}

int vxg_query_voxels(vxg_handle* h, const int32_t* g, uint64_t n, vxg_voxel* out, uint8_t* found) {
  return guarded([&] {
    set_device(h);
    h->settle();
    if (n == 0) return;
    DBuf<int32_t> dg;
    DBuf<vxg_voxel> dout;
    DBuf<uint8_t> dfound;
    dg.ensure(3 * n);
    dout.ensure(n);
    dfound.ensure(n);
    CU(cudaMemcpyAsync(dg.p, g, 3 * n * sizeof(int32_t), cudaMemcpyHostToDevice, h->st));
    k_query<<<grid_for(n), 256, 0, h->st>>>(n, dg.p, h->view(), dout.p, dfound.p);
    CU(cudaGetLastError());
    CU(cudaMemcpyAsync(out, dout.p, n * sizeof(vxg_voxel), cudaMemcpyDeviceToHost, h->st));
    CU(cudaMemcpyAsync(found, dfound.p, n, cudaMemcpyDeviceToHost, h->st));
    CU(cudaStreamSynchronize(h->st));
  });
}

int vxg_interpolate_distance(vxg_handle* h, const float* pts, uint64_t n, float* d, uint8_t* found, int flags) {
  return guarded([&] {
    set_device(h);
    h->settle();
    if (n == 0) return;
    if (pts == nullptr || d == nullptr || found == nullptr) throw VxgError(VXG_EINVAL, "null argument");
    if (flags & VXG_INPUT_DEVICE) {
      k_interpolate<<<grid_for(n), 256, 0, h->st>>>(n, pts, h->view(), h->voxel_size, d, found);
      ++h->launches;
      CU(cudaGetLastError());
      CU(cudaStreamSynchronize(h->st));
      return;
    }
    DBuf<float> dp, dd;
    DBuf<uint8_t> df;
    dp.ensure(3 * n);
    dd.ensure(n);
    df.ensure(n);
    CU(cudaMemcpyAsync(dp.p, pts, 3 * n * sizeof(float), cudaMemcpyHostToDevice, h->st));
    k_interpolate<<<grid_for(n), 256, 0, h->st>>>(n, dp.p, h->view(), h->voxel_size, dd.p, df.p);
    ++h->launches;
    CU(cudaGetLastError());
    CU(cudaMemcpyAsync(d, dd.p, n * sizeof(float), cudaMemcpyDeviceToHost, h->st));
    CU(cudaMemcpyAsync(found, df.p, n, cudaMemcpyDeviceToHost, h->st));
    CU(cudaStreamSynchronize(h->st));
  });
}

int vxg_mesh_extract(vxg_handle* h, const vxg_mc_tables* tables, const int32_t* blocks, uint64_t n_req,
                     int with_colors, uint64_t* n_frag, uint64_t* n_tri) {
  return guarded([&] {
    if (h == nullptr || tables == nullptr || n_frag == nullptr || n_tri == nullptr)
      throw VxgError(VXG_EINVAL, "null argument");
    if (blocks == nullptr && n_req > 0) throw VxgError(VXG_EINVAL, "null block list");
    set_device(h);
    h->settle();
    h->mesh_ready = false;
    std::vector<uint32_t> order;
    export_sorted(h, &order);  // every allocated block, sorted by (x, y, z)
    std::vector<int32_t> slots;
    if (blocks == nullptr) {
      slots.assign(order.begin(), order.end());
    } else {  // extract_blocks: the requested blocks that are allocated (block_ptr != nullptr)
      std::unordered_map<uint64_t, uint32_t> rank;
      rank.reserve(order.size());
      for (uint32_t r = 0; r < order.size(); ++r) {
        const int32_t* b = h->host_idx.data() + 3 * order[r];
        rank.emplace(pack_block(b[0], b[1], b[2]), r);
      }
      std::vector<uint32_t> ranks;
      for (uint64_t i = 0; i < n_req; ++i) {
        const int32_t* b = blocks + 3 * i;
        if (!block_in_range(b[0], b[1], b[2])) continue;
        const auto it = rank.find(pack_block(b[0], b[1], b[2]));
        if (it != rank.end()) ranks.push_back(it->second);
      }
      std::sort(ranks.begin(), ranks.end());
      ranks.erase(std::unique(ranks.begin(), ranks.end()), ranks.end());
      for (uint32_t r : ranks) slots.push_back(static_cast<int32_t>(order[r]));
    }
    const uint64_t B = slots.size();
    h->mesh_bidx.resize(3 * B);
    for (uint64_t j = 0; j < B; ++j)
      for (int a = 0; a < 3; ++a) h->mesh_bidx[3 * j + a] = h->host_idx[3 * static_cast<uint64_t>(slots[j]) + a];
    h->mesh_frag.assign(B + 1, 0);
    h->mesh_T = 0;
    h->mesh_colors = with_colors != 0;
    if (B > 0) {
      const uint64_t nc = B * static_cast<uint64_t>(h->nvox);
      if (nc >= (1ull << 31)) throw VxgError(VXG_EINVAL, "too many blocks for one extraction");
      CU(cudaMemcpyAsync(h->mesh_tab.ensure(1), tables, sizeof(vxg_mc_tables), cudaMemcpyHostToDevice, h->st));
      CU(cudaMemcpyAsync(h->mesh_slots.ensure(B), slots.data(), B * sizeof(int32_t), cudaMemcpyHostToDevice, h->st));
      h->mesh_ntri.ensure(nc + 1);
      h->mesh_off.ensure(nc + 1);
      const unsigned grid = grid_for(nc);
      k_mc_count<<<grid, 256, 0, h->st>>>(nc, h->mesh_slots.p, h->view(), h->mesh_tab.p, h->mesh_ntri.p);
      CU(cudaMemsetAsync(h->mesh_ntri.p + nc, 0, sizeof(uint32_t), h->st));
      ++h->launches;
      h->scan_exclusive<uint32_t>(h->mesh_ntri.p, h->mesh_off.p, nc + 1);
      // fragment boundaries: the scan at every block's first cube (+ the total)
      h->mesh_frag_dev.ensure(B + 1);
      k_gather_stride<<<grid_for(B + 1), 256, 0, h->st>>>(B + 1, h->mesh_off.p, static_cast<uint64_t>(h->nvox),
                                                          h->mesh_frag_dev.p);
      ++h->launches;
      std::vector<uint32_t> fr(B + 1);
      CU(cudaMemcpyAsync(fr.data(), h->mesh_frag_dev.p, (B + 1) * sizeof(uint32_t), cudaMemcpyDeviceToHost, h->st));
      CU(cudaStreamSynchronize(h->st));
      for (uint64_t j = 0; j <= B; ++j) h->mesh_frag[j] = fr[j];
      h->mesh_T = fr[B];
      if (h->mesh_T > 0) {
        h->mesh_v.ensure(9 * h->mesh_T);
        h->mesh_n.ensure(9 * h->mesh_T);
        if (h->mesh_colors) h->mesh_c.ensure(9 * h->mesh_T);
        k_mc_emit<<<grid, 256, 0, h->st>>>(nc, h->mesh_slots.p, h->view(), h->voxel_size, h->mesh_tab.p,
                                           h->mesh_ntri.p, h->mesh_off.p, with_colors, h->mesh_v.p, h->mesh_n.p,
                                           h->mesh_colors ? h->mesh_c.p : nullptr);
        ++h->launches;
      }
      CU(cudaGetLastError());
      CU(cudaStreamSynchronize(h->st));
    }
    h->mesh_ready = true;
    *n_frag = B;
    *n_tri = h->mesh_T;
  });
}

int vxg_mesh_fetch(vxg_handle* h, int32_t* block_idx, uint64_t* frag_tri, float* vertices, float* normals,
                   uint8_t* colors) {
  return guarded([&] {
    if (h == nullptr) throw VxgError(VXG_EINVAL, "null argument");
    if (!h->mesh_ready) throw VxgError(VXG_EINVAL, "no extracted mesh (call vxg_mesh_extract first)");
    set_device(h);
    h->settle();
    const uint64_t B = h->mesh_bidx.size() / 3, T = h->mesh_T;
    if (block_idx) std::memcpy(block_idx, h->mesh_bidx.data(), 3 * B * sizeof(int32_t));
    if (frag_tri) std::memcpy(frag_tri, h->mesh_frag.data(), (B + 1) * sizeof(uint64_t));
    if (T > 0) {
      if (vertices) CU(cudaMemcpyAsync(vertices, h->mesh_v.p, 9 * T * sizeof(float), cudaMemcpyDeviceToHost, h->st));
      if (normals) CU(cudaMemcpyAsync(normals, h->mesh_n.p, 9 * T * sizeof(float), cudaMemcpyDeviceToHost, h->st));
      if (colors && h->mesh_colors) CU(cudaMemcpyAsync(colors, h->mesh_c.p, 9 * T, cudaMemcpyDeviceToHost, h->st));
    }
    CU(cudaStreamSynchronize(h->st));
  });
}

int vxg_surface_error(vxg_handle* h, const float* pts, uint64_t n, float truncation, double* out) {
  return guarded([&] {
    if (out == nullptr) throw VxgError(VXG_EINVAL, "null argument");
    std::vector<float> d(n);
    std::vector<uint8_t> found(n);
    if (n) {
      const int rc = vxg_interpolate_distance(h, pts, n, d.data(), found.data(), 0);
      if (rc != VXG_OK) throw VxgError(rc, vxg_last_error());
    }
    // Accumulator (analysis.cpp:16-37): fp64 sums in point order over the
    // interpolated distances the GPU returned, clamped to the truncation.
    double sum = 0.0, sum_sq = 0.0, max_abs = 0.0;
    uint64_t count = 0, unknown = 0;
    for (uint64_t i = 0; i < n; ++i) {
      if (!found[i]) {
        ++unknown;
        continue;
      }
      const float c = d[i] < -truncation ? -truncation : (truncation < d[i] ? truncation : d[i]);
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
  });
}

// EsdfConfig::band_radius + validate (esdf_integrator.h:36-40, .cpp:10-18).
static std::string validate_esdf(const vxg_esdf_config* c, float voxel_size) {
  const float gamma = c->band_mode == VXG_BAND_ONE_VOXEL ? voxel_size : 0.5f * c->truncation;
  if (!(gamma > 0.0f) || !(gamma <= c->truncation)) return "esdf config requires 0 < band radius <= truncation";
  if (!(c->d_max > gamma)) return "esdf config requires d_max > band radius";
  return "";
}

int vxg_esdf_build_occupancy(vxg_handle* h, const vxg_esdf_config* config, uint64_t* rounds) {
  return guarded([&] {
    if (config == nullptr) throw VxgError(VXG_EINVAL, "null esdf config");
    const std::string msg = validate_esdf(config, h->voxel_size);
    if (!msg.empty()) throw VxgError(VXG_EINVAL, msg);
    if (config->metric != VXG_METRIC_QUASI_EUCLIDEAN)
      throw VxgError(VXG_EINVAL,
                     "the device ESDF supports the quasi-Euclidean metric only (Euclidean results depend on the "
                     "wavefront order)");
    if (config->band_mode != VXG_BAND_ONE_VOXEL && config->band_mode != VXG_BAND_HALF_TRUNCATION)
      throw VxgError(VXG_EINVAL, "esdf config has an unknown band mode");
    set_device(h);
    h->settle();
    uint32_t c[2];
    h->read_counters(c);
    const uint64_t nb = std::min<uint64_t>(c[0], h->cap_blocks);
    h->sync_block_mirror(nb);
    h->esdf_ready = false;
    h->esdf_blocks = nb;
    uint64_t nr = 0;
    if (nb > 0) {
      const uint64_t nv = nb * static_cast<uint64_t>(h->nvox);
      h->esdf.ensure(nv);
      h->esdf_nbr.ensure(27 * nb);
      h->esdf_act.ensure(nb);
      h->esdf_act2.ensure(nb);
      h->esdf_changed.ensure(1);
      cudaStream_t st = h->st;
      const MapView m = h->view();
      k_esdf_neighbors<<<grid_for(27 * nb), 256, 0, st>>>(static_cast<uint32_t>(nb), h->block_idx.p, m,
                                                          h->esdf_nbr.p);
      k_esdf_init<<<grid_for(nv), 256, 0, st>>>(nv, h->slab.p, h->esdf.p, config->d_max);
      h->launches += 2;
      EsdfSteps steps;  // v * sqrt(|offset|^2) in fp32 (esdf_integrator.cpp:75)
      steps.s[0] = 0.0f;
      for (int k = 1; k <= 3; ++k) steps.s[k] = h->voxel_size * std::sqrt(static_cast<float>(k));
      CU(cudaMemsetAsync(h->esdf_act.p, 1, nb, st));
      const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(nb, 148ull * 8));
      for (;;) {
        CU(cudaMemsetAsync(h->esdf_act2.p, 0, nb, st));
        CU(cudaMemsetAsync(h->esdf_changed.p, 0, sizeof(uint32_t), st));
        k_esdf_relax<<<grid, kEsdfThreads, 0, st>>>(static_cast<uint32_t>(nb), h->esdf.p, h->esdf_nbr.p, h->vps, steps,
                                           h->esdf_act.p, h->esdf_act2.p, h->esdf_changed.p);
        ++h->launches;
        ++nr;
        uint32_t changed = 0;
        CU(cudaMemcpyAsync(&changed, h->esdf_changed.p, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
        CU(cudaStreamSynchronize(st));
        h->esdf_act.swap(h->esdf_act2);
        if (changed == 0) break;
      }
      k_esdf_parents<<<grid_for(nv), 256, 0, st>>>(static_cast<uint32_t>(nb), h->esdf.p, h->esdf_nbr.p, h->vps,
                                                   steps, config->d_max);
      ++h->launches;
      CU(cudaGetLastError());
      CU(cudaStreamSynchronize(st));
    }
    h->esdf_ready = true;
    if (rounds) *rounds = nr;
  });
}

// save_layer(EsdfLayer) (serialization.cpp:141-168, payload :116-122) of the
// last vxg_esdf_build_occupancy result.
int vxg_esdf_serialize_vxblx(vxg_handle* h, uint8_t* buf, uint64_t cap, uint64_t* need) {
  return guarded([&] {
    if (!h->esdf_ready) throw VxgError(VXG_EINVAL, "no ESDF layer: call vxg_esdf_build_occupancy first");
    set_device(h);
    h->settle();
    const uint64_t nb = h->esdf_blocks;
    std::vector<uint32_t> order(nb);
    for (uint32_t i = 0; i < nb; ++i) order[i] = i;
    const int32_t* idx = h->host_idx.data();
    std::sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) {
      const int32_t* A = idx + 3 * a;
      const int32_t* B = idx + 3 * b;
      if (A[0] != B[0]) return A[0] < B[0];
      if (A[1] != B[1]) return A[1] < B[1];
      return A[2] < B[2];
    });
    const uint64_t total = 31 + nb * (24 + static_cast<uint64_t>(h->nvox) * 8);
    if (need) *need = total;
    if (buf == nullptr || cap < total) return;
    uint8_t* o = buf;
    auto put = [&](const void* src, size_t len) {
      std::memcpy(o, src, len);
      o += len;
    };
    const char magic[6] = {'V', 'X', 'B', 'L', 'X', '\0'};
    const uint32_t version = 1;
    const double vs = static_cast<double>(h->voxel_size);
    const uint32_t vps = static_cast<uint32_t>(h->vps);
    const uint8_t kind = 1;
    put(magic, 6);
    put(&version, 4);
    put(&vs, 8);
    put(&vps, 4);
    put(&kind, 1);
    put(&nb, 8);
    const size_t bb = static_cast<size_t>(h->nvox) * sizeof(vxg_esdf_voxel);
    std::vector<uint8_t> all(nb * bb);
    if (nb) CU(cudaMemcpyAsync(all.data(), h->esdf.p, nb * bb, cudaMemcpyDeviceToHost, h->st));
    CU(cudaStreamSynchronize(h->st));
    for (uint64_t k = 0; k < nb; ++k) {
      for (int a = 0; a < 3; ++a) {
        const int64_t v = h->host_idx[3 * order[k] + a];
        put(&v, 8);
      }
      put(all.data() + static_cast<size_t>(order[k]) * bb, bb);  // payload layout == vxg_esdf_voxel
    }
  });
}

int vxg_serialize_vxblx(vxg_handle* h, uint8_t* buf, uint64_t cap, uint64_t* need) {
  return guarded([&] {
    set_device(h);
    h->settle();
    std::vector<uint32_t> order;
    export_sorted(h, &order);
    const uint64_t nb = order.size();
    const uint64_t total = 31 + nb * (24 + static_cast<uint64_t>(h->nvox) * 12);
    if (need) *need = total;
    if (buf == nullptr || cap < total) return;
    uint8_t* o = buf;
    auto put = [&](const void* src, size_t len) {
      std::memcpy(o, src, len);
      o += len;
    };
    const char magic[6] = {'V', 'X', 'B', 'L', 'X', '\0'};
    const uint32_t version = 1;
    const double vs = static_cast<double>(h->voxel_size);
    const uint32_t vps = static_cast<uint32_t>(h->vps);
    const uint8_t kind = 0;
    put(magic, 6);
    put(&version, 4);
    put(&vs, 8);
    put(&vps, 4);
    put(&kind, 1);
    put(&nb, 8);
    const size_t bb = static_cast<size_t>(h->nvox) * sizeof(vxg_voxel);
    // the blocks' payloads in sorted order: one gather + one D2H per 4096 blocks,
    // written into place behind each block's 24-byte index
    const uint64_t kStep = 4096;
    std::vector<vxg_voxel> tmp;
    for (uint64_t k0 = 0; k0 < nb; k0 += kStep) {
      const uint64_t m = std::min<uint64_t>(kStep, nb - k0);
      tmp.resize(m * static_cast<uint64_t>(h->nvox));
      gather_to_host(h, order.data() + k0, m, tmp.data());
      for (uint64_t k = 0; k < m; ++k) {
        for (int a = 0; a < 3; ++a) {
          const int64_t v = h->host_idx[3 * order[k0 + k] + a];
          put(&v, 8);
        }
        put(tmp.data() + k * h->nvox, bb);  // payload layout == vxg_voxel (f32, f32, u8 x3, u8 pad)
      }
    }
  });
}

int vxg_save_vxblx(vxg_handle* h, const char* path) {
  uint64_t need = 0;
  int rc = vxg_serialize_vxblx(h, nullptr, 0, &need);
  if (rc != VXG_OK) return rc;
  std::vector<uint8_t> buf(need);
  rc = vxg_serialize_vxblx(h, buf.data(), need, &need);
  if (rc != VXG_OK) return rc;
  std::ofstream f(path, std::ios::binary);
  if (!f) {
    g_err = std::string("cannot write layer file: ") + path;
    return VXG_EIO;
  }
  f.write(reinterpret_cast<const char*>(buf.data()), static_cast<std::streamsize>(buf.size()));
  if (!f) {
    g_err = "failed writing layer stream";
    return VXG_EIO;
  }
  return VXG_OK;
}

// Deferred: the slab, hash and counters are cleared once the folds still in
// flight are done, before the next batch's first map access (or by any entry
// point that reads the map). The host mirror is empty from here on.
int vxg_reset(vxg_handle* h) {
  return guarded([&] {
    set_device(h);
    h->reset_used = std::max<uint64_t>(h->reset_used, std::min<uint64_t>(h->n_blocks, h->cap_blocks));
    h->pending_reset = true;
    if (!h->async_fold) h->settle();
    h->n_blocks = 0;
    h->host_idx.clear();
    for (auto& kv : h->consumers) kv.second.clear();
  });
}

int vxg_load_vxblx(vxg_handle* h, const uint8_t* buf, uint64_t len) {
  return guarded([&] {
    // read_header / load_layer_impl (serialization.cpp:170-212), same ParseError texts.
    uint64_t at = 0;
    auto get = [&](void* dst, size_t n, const char* what) {
      if (at + n > len) throw VxgError(VXG_EPARSE, std::string("truncated layer file while reading ") + what);
      std::memcpy(dst, buf + at, n);
      at += n;
    };
    char magic[6];
    get(magic, 6, "magic");
    if (std::memcmp(magic, "VXBLX\0", 6) != 0) throw VxgError(VXG_EPARSE, "bad magic bytes; not a layer file");
    uint32_t version;
    get(&version, 4, "version");
    if (version != 1) throw VxgError(VXG_EPARSE, "unsupported layer file version " + std::to_string(version));
    double vs;
    get(&vs, 8, "voxel_size");
    uint32_t vps;
    get(&vps, 4, "voxels_per_side");
    uint8_t kind;
    get(&kind, 1, "layer_kind");
    if (kind > 1) throw VxgError(VXG_EPARSE, "unknown layer kind " + std::to_string(kind));
    uint64_t count;
    get(&count, 8, "block_count");
    if (vs <= 0.0 || vps == 0) throw VxgError(VXG_EPARSE, "invalid layer geometry in header");
    if (kind != 0) throw VxgError(VXG_EPARSE, "layer kind mismatch: file holds a different voxel type");
    if (vps > 64) throw VxgError(VXG_EINVAL, "voxels_per_side > 64 is not supported on the device slab");
    const uint64_t nvox = static_cast<uint64_t>(vps) * vps * vps;
    std::vector<int32_t> idx;
    std::vector<vxg_voxel> vox;
    idx.reserve(3 * std::min<uint64_t>(count, 1 << 20));
    for (uint64_t b = 0; b < count; ++b) {
      for (int a = 0; a < 3; ++a) {
        int64_t v;
        get(&v, 8, "block index");
        idx.push_back(static_cast<int32_t>(v));
      }
      const size_t base = vox.size();
      vox.resize(base + nvox);
      for (uint64_t i = 0; i < nvox; ++i) {
        float d, w;
        uint8_t c[4];
        get(&d, 4, "tsdf voxel distance");
        get(&w, 4, "tsdf voxel weight");
        get(c, 3, "tsdf voxel color");
        get(c + 3, 1, "tsdf voxel pad");
        vox[base + i] = vxg_voxel{d, w, c[0], c[1], c[2], 0};
      }
    }
    set_device(h);
    h->settle();
    if (static_cast<int>(vps) != h->vps) {
      // the new geometry's key range is checked before the handle changes
      uint64_t cap = h->cap_blocks;
      while (cap > 1 && cap * nvox >= 0xFFFFFFFFull) cap /= 2;
      h->alloc_map(std::max<uint64_t>(cap, count + 64), static_cast<int>(vps));
    } else {
      if (vxg_reset(h) != VXG_OK) throw VxgError(VXG_ECUDA, g_err);
    }
    h->voxel_size = static_cast<float>(vs);
    // duplicate indices: later blocks overwrite earlier ones (get_or_allocate_block)
    const int rc = vxg_import_blocks(h, idx.data(), vox.data(), count);
    if (rc != VXG_OK) throw VxgError(rc, g_err);
  });
}

int vxg_register_consumer(vxg_handle* h, const char* name) {
  return guarded([&] {
    if (name == nullptr) throw VxgError(VXG_EINVAL, "null consumer name");
    set_device(h);
    h->settle();
    h->consumers[name];
    h->ensure_touched();
  });
}

int vxg_drain_updated(vxg_handle* h, const char* name, int32_t* idx, uint64_t cap, uint64_t* n_out) {
  return guarded([&] {
    auto it = h->consumers.find(name ? name : "");
    if (it == h->consumers.end())
      throw VxgError(VXG_EINVAL, std::string("unknown updated-block consumer: ") + (name ? name : ""));
    uint64_t k = 0;
    for (uint32_t slot : it->second) {
      if (idx != nullptr && k < cap)
        for (int a = 0; a < 3; ++a) idx[3 * k + a] = h->host_idx[3 * slot + a];
      ++k;
    }
    if (n_out) *n_out = k;
    if (idx != nullptr) it->second.clear();
  });
}

int vxg_profile(vxg_handle* h, int enable) {
  h->profile = enable != 0;
  return VXG_OK;
}

int vxg_stage_count(void) { return kStages; }

const char* vxg_stage_name(int s) { return (s >= 0 && s < kStages) ? kStageNames[s] : ""; }

int vxg_stage_times(vxg_handle* h, double* ms, uint64_t* launches, uint64_t* units, int reset) {
  if (h == nullptr) return VXG_EINVAL;
  const int rc = guarded([&] {  // every stage of the calls so far, including a fold still running
    set_device(h);
    h->join_folds();
    CU(cudaStreamSynchronize(h->st));
    h->collect();
  });
  if (rc != VXG_OK) return rc;
  for (int s = 0; s < kStages; ++s) {
    if (ms) ms[s] = h->stage_ms[s];
    if (launches) launches[s] = h->stage_launch[s];
    if (units) units[s] = h->stage_units[s];
    if (reset) {
      h->stage_ms[s] = 0;
      h->stage_launch[s] = 0;
      h->stage_units[s] = 0;
    }
  }
  return VXG_OK;
}

int vxg_batch_info(vxg_handle* h, uint64_t* out, int reset) {
  if (h == nullptr || out == nullptr) return VXG_EINVAL;
  out[0] = h->info_records;
  out[1] = h->info_runs;
  out[2] = h->info_max_run;
  out[3] = h->n_blocks;
  out[4] = h->info_sort_passes;
  if (reset) h->info_records = h->info_runs = h->info_max_run = 0;
  return VXG_OK;
}

// Self-test of the fast exact fold arithmetic: n random divisions and n_seq
// random update sequences of length len, compared bit-for-bit with the
// reference-order path (__fdiv_rn / update_voxel). out[0] = division
// mismatches, out[1] = sequence mismatches.
extern "C" int vxg_selftest_fold(int device, uint64_t n, uint64_t n_seq, uint32_t len, uint64_t seed, uint64_t* out) {
  return guarded([&] {
    CU(cudaSetDevice(device));
    DBuf<unsigned long long> mm;
    DBuf<float> ex;
    mm.ensure(2);
    ex.ensure(2);
    CU(cudaMemset(mm.p, 0, 2 * sizeof(unsigned long long)));
    k_selftest_div<<<148 * 16, 256>>>(n, seed, mm.p, ex.p);
    k_selftest_fold<<<148 * 4, 128>>>(n_seq, len, seed, 0.1f, 1e4f, mm.p + 1);
    CU(cudaGetLastError());
    unsigned long long h[2];
    CU(cudaMemcpy(h, mm.p, sizeof(h), cudaMemcpyDeviceToHost));
    out[0] = h[0];
    out[1] = h[1];
  });
}

// Self-test of the in-house device primitives behind the pipeline (vxg_sort.cuh:
// prefix sums, the 32-bit pair sort in both tile shapes, 64-bit-key sorts)
// against the host: n random items, keys of `bits` bits. out[0] / out[1] =
// mismatches of the 32- / 64-bit exclusive prefix sums, out[2] = of
// sort_pairs64 (keys or values, stable order), out[3] = of sort_pairs32.
extern "C" int vxg_selftest_prims(vxg_handle* h, uint64_t n, int bits, int descending, uint64_t seed,
                                  uint64_t* out) {
  return guarded([&] {
    if (h == nullptr || out == nullptr || bits < 1 || bits > 64) throw VxgError(VXG_EINVAL, "bad argument");
    set_device(h);
    h->settle();
    auto rnd = [&seed]() {  // splitmix64
      uint64_t z = (seed += 0x9E3779B97F4A7C15ull);
      z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
      z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
      return z ^ (z >> 31);
    };
    out[0] = out[1] = out[2] = out[3] = 0;
    if (n == 0) return;
    // ---- prefix sums
    std::vector<uint32_t> a32(n), r32(n);
    std::vector<unsigned long long> a64(n), r64(n);
    for (uint64_t i = 0; i < n; ++i) {
      a32[i] = static_cast<uint32_t>(rnd() & 15u);
      a64[i] = rnd() & 0xFFFFFFFFFFull;
    }
    DBuf<uint32_t> d32, o32;
    DBuf<unsigned long long> d64, o64;
    d32.ensure(n), o32.ensure(n), d64.ensure(n), o64.ensure(n);
    CU(cudaMemcpyAsync(d32.p, a32.data(), n * 4, cudaMemcpyHostToDevice, h->st));
    CU(cudaMemcpyAsync(d64.p, a64.data(), n * 8, cudaMemcpyHostToDevice, h->st));
    h->scan_exclusive<uint32_t>(d32.p, o32.p, n);
    h->scan_exclusive<unsigned long long>(d64.p, d64.p, n);  // in place
    CU(cudaMemcpyAsync(r32.data(), o32.p, n * 4, cudaMemcpyDeviceToHost, h->st));
    CU(cudaMemcpyAsync(r64.data(), d64.p, n * 8, cudaMemcpyDeviceToHost, h->st));
    CU(cudaStreamSynchronize(h->st));
    uint32_t s32 = 0;
    unsigned long long s64 = 0;
    for (uint64_t i = 0; i < n; ++i) {
      out[0] += r32[i] != s32;
      out[1] += r64[i] != s64;
      s32 += a32[i];
      s64 += a64[i];
    }
    // ---- pair sorts
    const unsigned long long mask = bits == 64 ? ~0ull : (1ull << bits) - 1ull;
    std::vector<unsigned long long> k64(n), rk(n);
    std::vector<uint32_t> v(n), rv(n), idx(n);
    for (uint64_t i = 0; i < n; ++i) {
      // few distinct values in the low byte: plenty of ties for the stability check
      k64[i] = ((rnd() & ~0xFFull) | (rnd() & 3u)) & mask;
      v[i] = static_cast<uint32_t>(rnd());
      idx[i] = static_cast<uint32_t>(i);
    }
    std::stable_sort(idx.begin(), idx.end(), [&](uint32_t x, uint32_t y) {
      return descending ? k64[x] > k64[y] : k64[x] < k64[y];
    });
    DBuf<unsigned long long> dk, dko;
    DBuf<uint32_t> dv, dvo;
    dk.ensure(n), dko.ensure(n), dv.ensure(n), dvo.ensure(n);
    CU(cudaMemcpyAsync(dk.p, k64.data(), n * 8, cudaMemcpyHostToDevice, h->st));
    CU(cudaMemcpyAsync(dv.p, v.data(), n * 4, cudaMemcpyHostToDevice, h->st));
    h->sort_pairs64(dk.p, dv.p, n, bits, descending != 0, dko.p, dvo.p);
    CU(cudaMemcpyAsync(rk.data(), dko.p, n * 8, cudaMemcpyDeviceToHost, h->st));
    CU(cudaMemcpyAsync(rv.data(), dvo.p, n * 4, cudaMemcpyDeviceToHost, h->st));
    CU(cudaStreamSynchronize(h->st));
    for (uint64_t i = 0; i < n; ++i) out[2] += rk[i] != k64[idx[i]] || rv[i] != v[idx[i]];
    if (bits <= 32 && !descending) {
      std::vector<uint32_t> k32(n), rk32(n);
      for (uint64_t i = 0; i < n; ++i) k32[i] = static_cast<uint32_t>(k64[i]);
      DBuf<uint32_t> a, b, c;
      a.ensure(n), b.ensure(n), c.ensure(n);
      CU(cudaMemcpyAsync(a.p, k32.data(), n * 4, cudaMemcpyHostToDevice, h->st));
      CU(cudaMemcpyAsync(dv.p, v.data(), n * 4, cudaMemcpyHostToDevice, h->st));
      uint32_t *sk = nullptr, *sv = nullptr;
      h->sort_pairs32(n, bits, a.p, dv.p, b.p, c.p, &sk, &sv);
      CU(cudaMemcpyAsync(rk32.data(), sk, n * 4, cudaMemcpyDeviceToHost, h->st));
      CU(cudaMemcpyAsync(rv.data(), sv, n * 4, cudaMemcpyDeviceToHost, h->st));
      CU(cudaStreamSynchronize(h->st));
      for (uint64_t i = 0; i < n; ++i) out[3] += rk32[i] != k32[idx[i]] || rv[i] != v[idx[i]];
    }
  });
}

// Debug: enable the fold trace / read it: out = 4*nruns+2 u64 (per long run:
// start ns, end ns, length, records folded on the saturated lane; then the
// latest and earliest warp exit time). Returns nruns in *n.
extern "C" int vxg_debug_fold(vxg_handle* h, int enable, unsigned long long* out, uint64_t cap, uint64_t* n) {
  return guarded([&] {
    h->debug_fold = enable != 0;
    if (n) *n = h->fold_dbg_n;
    if (out && h->fold_dbg.p) {
      const uint64_t m = std::min<uint64_t>(cap, 4ull * h->fold_dbg_n + 20);
      CU(cudaMemcpy(out, h->fold_dbg.p, m * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    }
  });
}

// Debug: the n longest fold chains of the last chunk (length, voxel key).
extern "C" int vxg_debug_top_runs(vxg_handle* h, uint32_t* len, uint32_t* keys, uint32_t n) {
  return guarded([&] {
    set_device(h);
    h->settle();
    // (the fold order is by length code, key order inside a code: the first n
    // runs are among the longest, not exactly the n longest)
    uint32_t nruns = 0;
    CU(cudaMemcpy(&nruns, h->num_runs.p, sizeof(uint32_t), cudaMemcpyDeviceToHost));
    const uint32_t m = std::min(n, nruns);
    std::vector<uint32_t> ord(m), rl(nruns), rk(nruns);
    CU(cudaMemcpy(ord.data(), h->run_order.p, m * sizeof(uint32_t), cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(rl.data(), h->run_len.p, nruns * sizeof(uint32_t), cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(rk.data(), h->run_keys.p, nruns * sizeof(uint32_t), cudaMemcpyDeviceToHost));
    for (uint32_t i = 0; i < n; ++i) {
      keys[i] = i < m ? rk[ord[i]] : 0xFFFFFFFFu;
      len[i] = i < m ? rl[ord[i]] : 0u;
    }
  });
}

int vxg_kernel_launches(vxg_handle* h, uint64_t* out, int reset) {
  if (out) *out = h->launches;
  if (reset) h->launches = 0;
  return VXG_OK;
}

int vxg_nccl_unique_id(uint8_t* out) {
  return guarded([&] {
    ncclUniqueId id;
    NC(nccl()->GetUniqueId(&id));
    std::memcpy(out, id.internal, NCCL_UNIQUE_ID_BYTES);
  });
}

int vxg_shard_set_replicated(vxg_handle* h, int on) {
  if (h == nullptr) return VXG_EINVAL;
  h->shard_replicated = on != 0;
  return VXG_OK;
}

int vxg_group_set_replicated(vxg_group* g, int on) {
  if (g == nullptr) return VXG_EINVAL;
  for (vxg_handle* h : g->shards) h->shard_replicated = on != 0;
  return VXG_OK;
}

int vxg_shard_init(vxg_handle* h, int rank, int world, const uint8_t* id_bytes) {
  return guarded([&] {
    if (world < 1 || rank < 0 || rank >= world) throw VxgError(VXG_EINVAL, "invalid shard rank / world");
    set_device(h);
    h->settle();
    if (world > 1 || id_bytes != nullptr) {  // world 1 with an id: the NCCL path over a 1-rank communicator
      ncclUniqueId id;
      std::memcpy(id.internal, id_bytes, NCCL_UNIQUE_ID_BYTES);
      ncclComm_t comm;
      NC(nccl()->CommInitRank(&comm, world, id, rank));
      h->nccl_comm = comm;
    }
    h->shard_rank = rank;
    h->shard_world = world;
  });
}

int vxg_group_create(const vxg_tsdf_config* config, float voxel_size, int vps, int device, int world,
                     uint64_t block_capacity, vxg_group** out) {
  return guarded([&] {
    if (world < 1) throw VxgError(VXG_EINVAL, "group needs world >= 1");
    auto* g = new vxg_group;
    for (int r = 0; r < world; ++r) {
      vxg_handle* h = nullptr;
      const int rc = vxg_create(config, voxel_size, vps, device, block_capacity, &h);
      if (rc != VXG_OK) {
        for (vxg_handle* x : g->shards) vxg_destroy(x);
        delete g;
        throw VxgError(rc, g_err);
      }
      h->shard_rank = r;
      h->shard_world = world;
      if (r > 0) h->st = g->shards[0]->st;  // one stream: phases run in order
      g->shards.push_back(h);
    }
    *out = g;
  });
}

int vxg_group_destroy(vxg_group* g) {
  if (g == nullptr) return VXG_OK;
  // shards 1.. run on shard 0's stream: destroy them before shard 0
  for (size_t i = g->shards.size(); i-- > 0;) vxg_destroy(g->shards[i]);
  delete g;
  return VXG_OK;
}

int vxg_group_shard(vxg_group* g, int i, vxg_handle** out) {
  if (g == nullptr || i < 0 || i >= static_cast<int>(g->shards.size())) return VXG_EINVAL;
  *out = g->shards[i];
  return VXG_OK;
}

int vxg_group_set_config(vxg_group* g, const vxg_tsdf_config* config) {
  for (vxg_handle* h : g->shards) {
    const int rc = vxg_set_config(h, config);
    if (rc != VXG_OK) return rc;
  }
  return VXG_OK;
}

int vxg_group_integrate_packed(vxg_group* g, const float* xyz, const uint8_t* rgb, const uint64_t* offsets,
                               const float* poses, uint64_t F, int flags, vxg_stats* out) {
  return guarded([&] {
    if (g == nullptr || offsets == nullptr || poses == nullptr) throw VxgError(VXG_EINVAL, "null argument");
    if (F == 0) return;
    vxg_handle* h0 = g->shards[0];
    set_device(h0);
    const uint64_t P = offsets[F] - offsets[0];
    const float* dx = xyz;
    const uint8_t* dc = rgb;
    std::vector<uint64_t> off(offsets, offsets + F + 1);
    if (!(flags & VXG_INPUT_DEVICE) && P > 0) {
      float* sx = h0->in_xyz.ensure(3 * P);
      CU(cudaMemcpyAsync(sx, xyz + 3 * offsets[0], 3 * P * sizeof(float), cudaMemcpyHostToDevice, h0->st));
      uint8_t* sc = nullptr;
      if (rgb) {
        sc = h0->in_rgb.ensure(3 * P);
        CU(cudaMemcpyAsync(sc, rgb + 3 * offsets[0], 3 * P, cudaMemcpyHostToDevice, h0->st));
      }
      dx = sx;
      dc = sc;
      for (auto& o : off) o -= offsets[0];
    }
    const auto parts = plan_subbatches(off.data(), F, false);
    const int W = static_cast<int>(g->shards.size());
    std::vector<std::vector<vxg_stats>> st(W);
    for (const auto& part : parts) {
      const uint64_t f0 = part.first, f1 = part.second, nF = f1 - f0;
      std::vector<uint32_t> R(W);
      std::vector<TermView> tv(W);
      for (int r = 0; r < W; ++r) g->shards[r]->begin_batch(dx, dc, off.data() + f0, poses + 12 * f0, nF, &R[r], &tv[r]);
      for (int r = 0; r < W; ++r) g->shards[r]->shard_front(R[r], static_cast<uint32_t>(nF), tv[r]);
      if (!g->shards[0]->shard_replicated) group_exchange(g);
      for (int r = 0; r < W; ++r) g->shards[r]->shard_back(g->shards[r]->owned_records(), g->shards[r]->owned_count(),
                                                           static_cast<uint32_t>(nF));
      for (int r = 0; r < W; ++r) {
        st[r].assign(nF, vxg_stats{0, 0, 0});
        g->shards[r]->end_batch(nF, st[r].data());
      }
      if (out) {
        for (uint64_t f = 0; f < nF; ++f) {
          vxg_stats s = st[0][f];  // raycasts / skipped: identical on every shard
          s.updates = 0;
          for (int r = 0; r < W; ++r) s.updates += st[r][f].updates;
          out[f0 + f] = s;
        }
      }
    }
  });
}

// VXBLX of the union of the shards (ownership is disjoint).
int vxg_group_serialize_vxblx(vxg_group* g, uint8_t* buf, uint64_t cap, uint64_t* need) {
  return guarded([&] {
    vxg_handle* h0 = g->shards[0];
    const uint64_t nv = static_cast<uint64_t>(h0->nvox);
    std::vector<std::pair<std::array<int32_t, 3>, std::pair<int, uint64_t>>> all;
    std::vector<std::vector<vxg_voxel>> vox(g->shards.size());
    for (size_t s = 0; s < g->shards.size(); ++s) {
      uint64_t nb = 0;
      if (vxg_block_count(g->shards[s], &nb) != VXG_OK) throw VxgError(VXG_ECUDA, g_err);
      std::vector<int32_t> idx(3 * nb + 3);
      vox[s].resize(nb * nv + 1);
      uint64_t got = 0;
      if (vxg_export_blocks(g->shards[s], idx.data(), vox[s].data(), nb, &got) != VXG_OK) throw VxgError(VXG_ECUDA, g_err);
      for (uint64_t k = 0; k < got; ++k) all.push_back({{idx[3 * k], idx[3 * k + 1], idx[3 * k + 2]}, {static_cast<int>(s), k}});
    }
    std::sort(all.begin(), all.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
    const uint64_t total = 31 + all.size() * (24 + nv * 12);
    if (need) *need = total;
    if (buf == nullptr || cap < total) return;
    uint8_t* o = buf;
    auto put = [&](const void* src, size_t len) {
      std::memcpy(o, src, len);
      o += len;
    };
    const char magic[6] = {'V', 'X', 'B', 'L', 'X', '\0'};
    const uint32_t version = 1;
    const double vs = static_cast<double>(h0->voxel_size);
    const uint32_t vps = static_cast<uint32_t>(h0->vps);
    const uint8_t kind = 0;
    const uint64_t nb = all.size();
    put(magic, 6);
    put(&version, 4);
    put(&vs, 8);
    put(&vps, 4);
    put(&kind, 1);
    put(&nb, 8);
    for (const auto& e : all) {
      for (int a = 0; a < 3; ++a) {
        const int64_t v = e.first[a];
        put(&v, 8);
      }
      vxg_voxel* src = vox[e.second.first].data() + e.second.second * nv;
      for (uint64_t i = 0; i < nv; ++i) src[i].pad = 0;
      put(src, nv * sizeof(vxg_voxel));
    }
  });
}

// ---------------------------------------------------------------- free functions on device

int vxg_eval_projective_distance(int device, const float* x, const float* p, const float* s, uint64_t n, float* out) {
  return guarded([&] {
    CU(cudaSetDevice(device));
    DBuf<float> a, b, c, o;
    float* dx = to_dev(x, 3 * n, &a);
    float* dp = to_dev(p, 3 * n, &b);
    float* ds = to_dev(s, 3 * n, &c);
    o.ensure(std::max<uint64_t>(n, 1));
    k_eval_pd<<<grid_for(n), 256>>>(n, dx, dp, ds, o.p);
    CU(cudaGetLastError());
    CU(cudaMemcpy(out, o.p, n * sizeof(float), cudaMemcpyDeviceToHost));
  });
}

int vxg_eval_measurement_weight(int device, int mode, const float* z, const float* d, uint64_t n, float trunc,
                                float eps, float* out) {
  return guarded([&] {
    CU(cudaSetDevice(device));
    DBuf<float> a, b, o;
    float* dz = to_dev(z, n, &a);
    float* dd = to_dev(d, n, &b);
    o.ensure(std::max<uint64_t>(n, 1));
    k_eval_mw<<<grid_for(n), 256>>>(n, mode, dz, dd, trunc, eps, o.p);
    CU(cudaGetLastError());
    CU(cudaMemcpy(out, o.p, n * sizeof(float), cudaMemcpyDeviceToHost));
  });
}

int vxg_eval_update_voxels(int device, vxg_voxel* voxels, uint64_t nv, const uint64_t* starts, const float* d,
                           const float* w, const uint8_t* rgb, float trunc, float wmax) {
  return guarded([&] {
    CU(cudaSetDevice(device));
    const uint64_t nr = starts[nv];
    DBuf<vxg_voxel> dv;
    DBuf<uint64_t> ds;
    DBuf<float> dd, dw;
    DBuf<uint8_t> dc;
    vxg_voxel* pv = to_dev(voxels, nv, &dv);
    uint64_t* ps = to_dev(starts, nv + 1, &ds);
    float* pd = to_dev(d, nr, &dd);
    float* pw = to_dev(w, nr, &dw);
    uint8_t* pc = rgb != nullptr ? to_dev(rgb, 3 * nr, &dc) : nullptr;
    k_eval_update<<<grid_for(nv), 256>>>(nv, pv, ps, pd, pw, pc, trunc, wmax);
    CU(cudaGetLastError());
    CU(cudaMemcpy(voxels, pv, nv * sizeof(vxg_voxel), cudaMemcpyDeviceToHost));
  });
}

int vxg_eval_raycast(int device, const float* start, const float* end, uint64_t n, float v, uint32_t* counts,
                     const uint64_t* offsets, int32_t* out) {
  return guarded([&] {
    CU(cudaSetDevice(device));
    DBuf<float> a, b;
    DBuf<uint32_t> dc;
    DBuf<uint64_t> doff;
    DBuf<int32_t> dout;
    float* ds = to_dev(start, 3 * n, &a);
    float* de = to_dev(end, 3 * n, &b);
    dc.ensure(std::max<uint64_t>(n, 1));
    uint64_t* po = nullptr;
    int32_t* pout = nullptr;
    uint64_t total = 0;
    if (out != nullptr && n > 0) {
      po = to_dev(offsets, n, &doff);
      std::vector<uint32_t> tmp(1);
      total = offsets[n - 1];
      // caller-provided counts give the last ray's length
      total += counts[n - 1];
      dout.ensure(3 * total);
      pout = dout.p;
    }
    k_eval_raycast<<<grid_for(n), 256>>>(n, ds, de, v, dc.p, po, pout);
    CU(cudaGetLastError());
    CU(cudaMemcpy(counts, dc.p, n * sizeof(uint32_t), cudaMemcpyDeviceToHost));
    if (pout) CU(cudaMemcpy(out, pout, 3 * total * sizeof(int32_t), cudaMemcpyDeviceToHost));
  });
}

}  // extern "C"
