// Bucket-count schedule of the reference's per-scan bucketing map.
//
// integrate_grouped (reference src/tsdf_integrator.cpp:199-200) builds an
// IndexMap<PointBucket> (= std::unordered_map, core.h:84-85) and calls
// reserve(points.size() / 4 + 1); its iteration order (the merged-mode ray
// order, :223) depends on the bucket count in force at each insertion. The
// counts and rehash points are a property of the libstdc++ rehash policy, so
// they are PROBED from the same libstdc++ here instead of re-deriving its prime
// table: the result lists (elements already inserted when a rehash fires, new
// bucket count), entry 0 being (0, bucket count after reserve).
#include <cstdint>
#include <map>
#include <mutex>
#include <unordered_map>
#include <utility>
#include <vector>

namespace vxg {

using Schedule = std::vector<std::pair<uint64_t, uint64_t>>;

namespace {

struct Cached {
  Schedule schedule;
  uint64_t covered = 0;  // schedule exact for up to this many distinct keys
};

std::mutex g_mu;
std::map<uint64_t, Cached> g_cache;

Schedule probe(uint64_t n_points, uint64_t max_keys) {
  struct Ident {
    size_t operator()(uint64_t k) const noexcept { return static_cast<size_t>(k); }
  };
  std::unordered_map<uint64_t, char, Ident> m;
  m.reserve(n_points / 4 + 1);
  Schedule s;
  s.emplace_back(0, m.bucket_count());
  for (uint64_t k = 0; k < max_keys; ++k) {
    const size_t before = m.bucket_count();
    m.emplace(k, 0);
    if (m.bucket_count() != before) s.emplace_back(k, m.bucket_count());
  }
  return s;
}

}  // namespace

// Bucket count right after reserve(n_points / 4 + 1) on an empty map.
uint64_t initial_buckets(uint64_t n_points) {
  static std::map<uint64_t, uint64_t> memo;  // under g_mu
  auto it = memo.find(n_points);
  if (it != memo.end()) return it->second;
  std::unordered_map<uint64_t, char> m;
  m.reserve(n_points / 4 + 1);
  return memo[n_points] = m.bucket_count();
}

// Schedule valid for any scan of n_points points with at most max_keys
// distinct terminal voxels. The growth after reserve depends only on the
// bucket count reserve picked (the rehash policy's next-resize threshold is a
// function of the bucket count), so the probe is cached per initial bucket
// count: scans whose point counts differ (LiDAR) share it.
Schedule bucket_schedule(uint64_t n_points, uint64_t max_keys) {
  std::lock_guard<std::mutex> lock(g_mu);
  const uint64_t bc0 = initial_buckets(n_points);
  Cached& c = g_cache[bc0];
  if (c.schedule.empty() || c.covered < max_keys) {
    uint64_t want = max_keys;
    if (c.covered > 0 && want < 2 * c.covered) want = 2 * c.covered;
    if (want < max_keys) want = max_keys;
    c.schedule = probe(n_points, want);
    c.covered = want;
  }
  return c.schedule;
}

}  // namespace vxg
