// lsa.cuh -- the multi-GPU exchange fused into the pass ("fused version"):
// the warp that completes a rank's octant subtree stores the rank's statistic vector
// straight into every peer's symmetric window over NVLink (NCCL 2.28 device API,
// load/store-accessible "LSA" pointers), fences at system scope and raises a per-rank
// sequence flag in each peer; the tail kernel of every rank waits on the world's flags
// and reads the partials from its own memory.  No NCCL kernel, no extra launch: the
// 96-byte exchange is a handful of remote stores issued while the last CTA finishes.
//
// Window layout (identical on every rank, registered NCCL_WIN_COLL_SYMMETRIC):
//   data  [2 parities][kMaxRanks][kMaxNS] doubles   (sweep s writes parity s & 1)
//   flags [2 parities][kMaxRanks] uint64            (flag = sequence number s)
// Double buffering is enough: rank A can only start pass s+2 after its tail s+1 saw every
// rank's pass s+1, i.e. after every rank's tail s finished reading parity s & 1.
// Every wait is bounded: a stalled peer ends the fit with an error, never a hung GPU.
#pragma once

#include <nccl.h>
#include <nccl_device.h>
#include <stdint.h>

namespace cavi {

constexpr int kMaxRanks = 8;
constexpr int kMaxNS = 15 + 15 * 16 / 2 + 3;  // n_stats(15)

struct LsaLink {
  ncclWindow_t win;           // null: exchange through NCCL (or single GPU)
  unsigned long long* seq;    // [1] sweeps exchanged so far (this rank's device memory)
  int world, rank;            // LSA team == world (single NVLink domain)
};

constexpr size_t lsa_data_off(int parity, int rank) {
  return ((size_t)(parity * kMaxRanks + rank) * kMaxNS) * sizeof(double);
}
constexpr size_t lsa_flag_off(int parity, int rank) {
  return (size_t)2 * kMaxRanks * kMaxNS * sizeof(double) + (size_t)(parity * kMaxRanks + rank) * sizeof(uint64_t);
}
constexpr size_t kLsaWindowBytes = (size_t)2 * kMaxRanks * kMaxNS * sizeof(double) + 2 * kMaxRanks * sizeof(uint64_t);

__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ double ld_relaxed_sys(const double* p) {
  double v;
  asm volatile("ld.relaxed.sys.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}

// One warp: publish this rank's ns statistics `val(st)` for sequence s to every peer.
template <typename F>
__device__ __forceinline__ void lsa_publish(const LsaLink& L, uint64_t s, int ns, F val, int lane) {
  const int par = (int)(s & 1);
  for (int st = lane; st < ns; st += 32) {
    const double v = val(st);
    for (int p = 0; p < L.world; ++p)
      static_cast<double*>(ncclGetLsaPointer(L.win, lsa_data_off(par, L.rank), p))[st] = v;
  }
  asm volatile("fence.acq_rel.sys;" ::: "memory");  // every lane's remote stores before any flag
  __syncwarp();
  if (lane < L.world)
    st_release_sys(static_cast<uint64_t*>(ncclGetLsaPointer(L.win, lsa_flag_off(par, L.rank), lane)), s);
}

// One warp: wait until every rank published sequence s (bounded).  Every lane acquires
// every flag itself (and sees it reach s) before it reads any data the flags guard.
// Returns false on timeout (uniformly across the warp).
__device__ __forceinline__ bool lsa_wait(const LsaLink& L, uint64_t s, int lane, long long max_cycles) {
  const int par = (int)(s & 1);
  bool ok = true;
  const long long t0 = clock64();
  for (int r = 0; r < L.world && ok; ++r) {
    const uint64_t* f = static_cast<const uint64_t*>(ncclGetLocalPointer(L.win, lsa_flag_off(par, r)));
    while (ld_acquire_sys(f) < s) {
      if (clock64() - t0 > max_cycles) {
        ok = false;
        break;
      }
    }
  }
  return __all_sync(0xffffffffu, ok);
}

__device__ __forceinline__ double lsa_read(const LsaLink& L, uint64_t s, int rank, int st) {
  return ld_relaxed_sys(static_cast<const double*>(ncclGetLocalPointer(L.win, lsa_data_off((int)(s & 1), rank))) + st);
}

// A rank without genes still takes part in every exchange: publish zeros (unless the fit
// is done, in which case no rank publishes: `done` is identical on every rank).
static __global__ void lsa_publish_zeros_kernel(LsaLink L, int ns, const int* done) {
  if (*(volatile const int*)done) return;
  const uint64_t s = *L.seq + 1;
  lsa_publish(L, s, ns, [](int) { return 0.0; }, threadIdx.x);
}

// Start-up check of the path (all ranks, collectively): publish a rank pattern for sequence
// `s`, wait (bounded), verify every peer's pattern.  ok[0] = 1 on success.
static __global__ void lsa_selftest_kernel(LsaLink L, uint64_t s, int* ok) {
  const int lane = threadIdx.x;
  lsa_publish(L, s, 4, [&](int st) { return 1000.0 * L.rank + st + 0.25 * (double)s; }, lane);
  bool good = lsa_wait(L, s, lane, 1ll << 31);
  if (good && lane < 4)
    for (int r = 0; r < L.world; ++r) good = good && lsa_read(L, s, r, lane) == 1000.0 * r + lane + 0.25 * (double)s;
  good = __all_sync(0xffffffffu, good);
  if (lane == 0) *ok = good ? 1 : 0;
}

}  // namespace cavi
