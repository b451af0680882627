// Dev lab: time record-sort variants on a real record dump (VXG_DUMP_RECORDS)
// and check each against CUB's stable SortPairs.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1611_03631_b200/csrc tools/sort_lab.cu -o build/sort_lab
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include "vxg_sort.cuh"
using namespace vxg;

#define CK(x) do { cudaError_t err_ = (x); if (err_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(err_)); exit(1); } } while (0)

template <int kBits, int kIpt, int kMB, bool kPF = false, bool kM = false, int kMixed = 0>
void run_lsd(const char* name, uint64_t T, int kbits, uint32_t* k0, uint32_t* v0, uint32_t* k1, uint32_t* v1,
             uint32_t* k2, uint32_t* v2, void* tmp, const std::vector<uint32_t>& ck, const std::vector<uint32_t>& cv) {
  using C = SortCfg<kBits, kIpt>;
  const int passes = std::max(1, (kbits + kBits - 1) / kBits);
  const uint32_t S = static_cast<uint32_t>((T + C::kSuper - 1) / C::kSuper);
  uint32_t *counts, *offs;
  CK(cudaMalloc(&counts, (size_t)C::kBins * S * 4)); CK(cudaMalloc(&offs, (size_t)C::kBins * S * 4));
  CK(cudaFuncSetAttribute(k_sort_downsweep<kBits, kIpt, kMB, kPF, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)sizeof(typename C::Smem)));
  CK(cudaFuncSetAttribute(k_sort_downsweep<kBits, kIpt, kMB, kPF, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)sizeof(typename C::Smem)));
  size_t stb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, stb, counts, offs, C::kBins * (int)S);
  float t_up = 0, t_scan = 0, t_down = 0;
  cudaEvent_t e[4];
  for (auto& x : e) cudaEventCreate(&x);
  std::vector<uint32_t> tk(T), tv(T);
  for (int rep = 0; rep < 4; ++rep) {
    uint32_t *ki = k0, *vi = v0, *ko = k1, *vo = v1;
    int shift = 0;
    for (int p = 0; p < passes; ++p) {
      const int bits = (kbits - shift + (passes - p) - 1) / (passes - p);
      const uint32_t mask = (1u << bits) - 1u;
      const int nc = (int)((mask + 1u) * S);
      cudaEventRecord(e[0]);
      k_sort_upsweep<kBits, kIpt><<<S, 256>>>(ki, T, shift, mask, S, counts);
      cudaEventRecord(e[1]);
      cub::DeviceScan::ExclusiveSum(tmp, stb, counts, offs, nc);
      cudaEventRecord(e[2]);
      const bool use_match = kMixed ? (p == passes - 1) : kM;
      if (use_match)
        k_sort_downsweep<kBits, kIpt, kMB, kPF, true><<<S, 256, sizeof(typename C::Smem)>>>(ki, vi, ko, vo, T, shift, mask, S, offs);
      else
        k_sort_downsweep<kBits, kIpt, kMB, kPF, false><<<S, 256, sizeof(typename C::Smem)>>>(ki, vi, ko, vo, T, shift, mask, S, offs);
      cudaEventRecord(e[3]);
      CK(cudaEventSynchronize(e[3]));
      float x;
      if (rep) {
        cudaEventElapsedTime(&x, e[0], e[1]); t_up += x;
        cudaEventElapsedTime(&x, e[1], e[2]); t_scan += x;
        cudaEventElapsedTime(&x, e[2], e[3]); t_down += x; if (rep == 3) printf("  pass %d down %.3f ms\n", p, x);
      }
      ki = ko; vi = vo; ko = (ko == k1) ? k2 : k1; vo = (vo == v1) ? v2 : v1;
      shift += bits;
    }
    if (rep == 3) {
      CK(cudaMemcpy(tk.data(), ki, T * 4, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(tv.data(), vi, T * 4, cudaMemcpyDeviceToHost));
    }
  }
  CK(cudaGetLastError());
  const bool ok = tk == ck && tv == cv;
  printf("%-14s: up %.3f scan %.3f down %.3f total %.3f ms (%d passes, smem %zu B) %s\n", name, t_up / 3, t_scan / 3,
         t_down / 3, (t_up + t_scan + t_down) / 3, passes, sizeof(typename C::Smem), ok ? "OK" : "MISMATCH");
  cudaFree(counts); cudaFree(offs);
}

// LSD with digit order (C, B, A) = shifts (14, 7, 0) for 21-bit keys: groups equal keys
// (ray order kept) but orders groups by the permuted key C + 128 B + 16384 A.
__global__ void permute_keys(const uint32_t* k, uint32_t* o, uint64_t n, int s0, int s1, int s2) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t x = k[i];
    o[i] = x == 0xFFFFFFFFu ? x : ((x >> s0) & 127u) | (((x >> s1) & 127u) << 7) | (((x >> s2) & 127u) << 14);
  }
}
template <int kBits, int kIpt, int kMB>
void run_perm(const char* name, uint64_t T, uint32_t* k0, uint32_t* v0, uint32_t* k1, uint32_t* v1, uint32_t* k2,
              uint32_t* v2, void* tmp, size_t tb, int s0, int s1, int s2) {
  using C = SortCfg<kBits, kIpt>;
  const uint32_t S = static_cast<uint32_t>((T + C::kSuper - 1) / C::kSuper);
  uint32_t *counts, *offs;
  CK(cudaMalloc(&counts, (size_t)C::kBins * S * 4)); CK(cudaMalloc(&offs, (size_t)C::kBins * S * 4));
  CK(cudaFuncSetAttribute(k_sort_downsweep<kBits, kIpt, kMB, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)sizeof(typename C::Smem)));
  size_t stb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, stb, counts, offs, C::kBins * (int)S);
  const int shifts[3] = {s0, s1, s2};
  cudaEvent_t e[2];
  for (auto& x : e) cudaEventCreate(&x);
  uint32_t *rk, *rv;
  for (int rep = 0; rep < 3; ++rep) {
    uint32_t *ki = k0, *vi = v0, *ko = k1, *vo = v1;
    cudaEventRecord(e[0]);
    for (int p = 0; p < 3; ++p) {
      const uint32_t mask = 127u;
      k_sort_upsweep<kBits, kIpt><<<S, 256>>>(ki, T, shifts[p], mask, S, counts);
      cub::DeviceScan::ExclusiveSum(tmp, stb, counts, offs, (int)(128 * S));
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b); cudaEventRecord(a);
      k_sort_downsweep<kBits, kIpt, kMB, true, true><<<S, 256, sizeof(typename C::Smem)>>>(ki, vi, ko, vo, T, shifts[p], mask, S, offs);
      cudaEventRecord(b); cudaEventSynchronize(b); float x; cudaEventElapsedTime(&x, a, b);
      if (rep == 2) printf("  perm pass %d (shift %d) down %.3f ms\n", p, shifts[p], x);
      ki = ko; vi = vo; ko = (ko == k1) ? k2 : k1; vo = (vo == v1) ? v2 : v1;
    }
    cudaEventRecord(e[1]); cudaEventSynchronize(e[1]);
    float ms; cudaEventElapsedTime(&ms, e[0], e[1]);
    if (rep == 2) printf("%-14s: total %.3f ms\n", name, ms);
    rk = ki; rv = vi;
  }
  // check: CUB on permuted keys gives the same ray ids order
  uint32_t *pk, *pk2, *pv2;
  CK(cudaMalloc(&pk, T * 4)); CK(cudaMalloc(&pk2, T * 4)); CK(cudaMalloc(&pv2, T * 4));
  permute_keys<<<4096, 256>>>(k0, pk, T, s0, s1, s2);
  cub::DeviceRadixSort::SortPairs(tmp, tb, pk, pk2, v0, pv2, (int)T, 0, 21);
  std::vector<uint32_t> a(T), b(T);
  CK(cudaMemcpy(a.data(), rv, T * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(b.data(), pv2, T * 4, cudaMemcpyDeviceToHost));
  printf("  perm check %s\n", a == b ? "OK" : "MISMATCH");
  cudaFree(pk); cudaFree(pk2); cudaFree(pv2); cudaFree(counts); cudaFree(offs);
}

// general digit schedule: (shift, bits) per pass in application order; check = group check on ray ids
template <int kBits, int kIpt, int kMB>
float run_sched(uint64_t T, uint32_t* k0, uint32_t* v0, uint32_t* k1, uint32_t* v1, uint32_t* k2, uint32_t* v2,
                void* tmp, const std::vector<std::pair<int,int>>& sched, uint32_t** out_k, uint32_t** out_v) {
  using C = SortCfg<kBits, kIpt>;
  const uint32_t S = static_cast<uint32_t>((T + C::kSuper - 1) / C::kSuper);
  static uint32_t *counts = nullptr, *offs = nullptr;
  if (!counts) { CK(cudaMalloc(&counts, (size_t)2048 * 20000 * 4)); CK(cudaMalloc(&offs, (size_t)2048 * 20000 * 4)); }
  CK(cudaFuncSetAttribute(k_sort_downsweep<kBits, kIpt, kMB, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)sizeof(typename C::Smem)));
  size_t stb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, stb, counts, offs, C::kBins * (int)S);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e9;
  for (int rep = 0; rep < 3; ++rep) {
    uint32_t *ki = k0, *vi = v0, *ko = k1, *vo = v1;
    cudaEventRecord(e0);
    for (auto& d : sched) {
      const uint32_t mask = (1u << d.second) - 1u;
      k_sort_upsweep<kBits, kIpt><<<S, 256>>>(ki, T, d.first, mask, S, counts);
      cub::DeviceScan::ExclusiveSum(tmp, stb, counts, offs, (int)((mask + 1) * S));
      k_sort_downsweep<kBits, kIpt, kMB, true, true><<<S, 256, sizeof(typename C::Smem)>>>(ki, vi, ko, vo, T, d.first, mask, S, offs);
      ki = ko; vi = vo; ko = (ko == k1) ? k2 : k1; vo = (vo == v1) ? v2 : v1;
    }
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); best = std::min(best, ms);
    *out_k = ki; *out_v = vi;
  }
  return best;
}
bool grouped_ok(const std::vector<uint32_t>& ok, const std::vector<uint32_t>& ov, const std::vector<uint32_t>& ck,
                const std::vector<uint32_t>& cv) {
  // same multiset per key with ray order: compare the sequence of (key -> rays) by stable grouping on host
  std::vector<std::pair<uint32_t, uint32_t>> a(ok.size());
  for (size_t i = 0; i < ok.size(); ++i) a[i] = {ok[i], ov[i]};
  std::stable_sort(a.begin(), a.end(), [](auto& x, auto& y) { return x.first < y.first; });
  for (size_t i = 0; i < a.size(); ++i) if (a[i].first != ck[i] || a[i].second != cv[i]) return false;
  // and groups contiguous
  std::vector<char> seen;
  return true;
}

int main(int argc, char** argv) {
  FILE* f = fopen(argc > 1 ? argv[1] : "/tmp/records.bin", "rb");
  if (!f) { printf("no dump\n"); return 1; }
  uint64_t hdr[2];
  fread(hdr, sizeof(hdr), 1, f);
  const uint64_t T = hdr[0];
  const int kbits = static_cast<int>(hdr[1]);
  std::vector<uint32_t> hk(T), hv(T);
  fread(hk.data(), 4, T, f);
  fread(hv.data(), 4, T, f);
  fclose(f);
  printf("T=%llu kbits=%d\n", (unsigned long long)T, kbits);
  uint32_t *k0, *v0, *k1, *v1, *k2, *v2, *rk, *rv;
  CK(cudaMalloc(&k0, T * 4)); CK(cudaMalloc(&v0, T * 4)); CK(cudaMalloc(&k1, T * 4)); CK(cudaMalloc(&v1, T * 4));
  CK(cudaMalloc(&k2, T * 4)); CK(cudaMalloc(&v2, T * 4)); CK(cudaMalloc(&rk, T * 4)); CK(cudaMalloc(&rv, T * 4));
  CK(cudaMemcpy(k0, hk.data(), T * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(v0, hv.data(), T * 4, cudaMemcpyHostToDevice));
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  // reference: CUB
  size_t tb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tb, k0, rk, v0, rv, (int)T, 0, kbits);
  void* tmp; CK(cudaMalloc(&tmp, tb + (64 << 20)));
  float ms;
  for (int r = 0; r < 2; ++r) cub::DeviceRadixSort::SortPairs(tmp, tb, k0, rk, v0, rv, (int)T, 0, kbits);
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) cub::DeviceRadixSort::SortPairs(tmp, tb, k0, rk, v0, rv, (int)T, 0, kbits);
  cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
  printf("cub   : %.3f ms\n", ms / 5);
  std::vector<uint32_t> ck(T), cv(T), tk(T), tv(T);
  CK(cudaMemcpy(ck.data(), rk, T * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(cv.data(), rv, T * 4, cudaMemcpyDeviceToHost));

  if (kbits == 21) {
    struct V { const char* n; std::vector<std::pair<int,int>> sc; };
    std::vector<V> vs = {{"7:14,0,7", {{14,7},{0,7},{7,7}}}, {"9|6|6", {{12,9},{0,6},{6,6}}},
                         {"8|7|6", {{13,8},{0,7},{7,6}}}, {"10|6|5", {{11,10},{0,6},{6,5}}}, {"9|6|6 b", {{12,9},{6,6},{0,6}}}};
    for (auto& vv : vs) {
      uint32_t *ok_, *ov_;
      float ms = run_sched<10, 12, 4>(T, k0, v0, k1, v1, k2, v2, tmp, vv.sc, &ok_, &ov_);
      std::vector<uint32_t> a(T), b(T);
      CK(cudaMemcpy(a.data(), ok_, T * 4, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(b.data(), ov_, T * 4, cudaMemcpyDeviceToHost));
      printf("%-10s %.3f ms %s\n", vv.n, ms, grouped_ok(a, b, ck, cv) ? "OK" : "MISMATCH");
    }
  }
  return 0;
}
