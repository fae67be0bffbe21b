// lsa.cuh -- the multi-GPU exchange fused into the pass ("fused version"):
// the warp that completes a rank's octant subtree stores the rank's statistic vector
// straight into every peer's symmetric window over NVLink (NCCL 2.28 device API,
// load/store-accessible "LSA" pointers); the tail kernel of every rank polls its own window
// until every rank's words for this sweep have landed, and reduces them.  No NCCL kernel,
// no extra launch, and no fence: like NCCL's LL protocol, every 8-byte word carries its own
// flag -- (sequence << 32 | 32 data bits), two words per double -- so a word is valid
// exactly when its flag equals the sweep's sequence number (8-byte stores are single-copy
// atomic over NVLink).
//
// Window layout (identical on every rank, registered NCCL_WIN_COLL_SYMMETRIC):
//   words [2 parities][kMaxRanks][kMaxNS][2] uint64   (sweep s writes parity s & 1)
// Double buffering is enough: rank A can only start pass s+2 after its tail s+1 saw every
// rank's pass s+1, i.e. after every rank's tail s finished reading parity s & 1; stale
// words of that parity carry sequence s-2, never s.
// Every wait is bounded (globaltimer deadline, CAVI_PEER_TIMEOUT_S, default 10 s): a
// stalled peer ends the fit with CV_ERR_PEER, never a hung GPU.  After a timeout the ranks'
// counters may disagree and the failed sweep's words stay in the windows; every shard call
// therefore starts with a collective resync (cavi.cu shard_entry): seq := max over ranks + 2,
// a tag no stale word can carry.
#pragma once

#include <nccl.h>
#include <nccl_device.h>
#include <stdint.h>

namespace cavi {

constexpr int kMaxRanks = 8;
constexpr int kMaxNS = 15 + 15 * 16 / 2 + 3;  // n_stats(15)

struct LsaLink {
  ncclWindow_t win;           // null: exchange through NCCL (or single GPU)
  unsigned long long* seq;    // [0] sweeps exchanged so far (this rank's device memory);
                              // [1] fault injection (tests): the sequence whose publish is dropped, 0 = none
  int world, rank;            // LSA team == world (single NVLink domain)
  unsigned long long timeout_ns;  // bound on the tail's wait for the peers' words
};

__device__ __forceinline__ unsigned long long lsa_now_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

constexpr size_t lsa_data_off(int parity, int rank) {
  return ((size_t)(parity * kMaxRanks + rank) * kMaxNS * 2) * sizeof(uint64_t);
}
constexpr size_t kLsaWindowBytes = (size_t)2 * kMaxRanks * kMaxNS * 2 * sizeof(uint64_t);

__device__ __forceinline__ void st_relaxed_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_relaxed_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// One warp: publish this rank's ns statistics `val(st)` for sequence s to every peer.
template <typename F>
__device__ __forceinline__ void lsa_publish(const LsaLink& L, uint64_t s, int ns, F val, int lane) {
  if (L.seq[1] == s) return;  // injected fault: this rank never publishes sweep s
  const int par = (int)(s & 1);
  const uint64_t tag = (uint64_t)(uint32_t)s << 32;
  for (int st = lane; st < ns; st += 32) {
    const uint64_t u = (uint64_t)__double_as_longlong(val(st));
    const uint64_t w0 = tag | (u & 0xffffffffull), w1 = tag | (u >> 32);
    for (int p = 0; p < L.world; ++p) {
      uint64_t* dst = static_cast<uint64_t*>(ncclGetLsaPointer(L.win, lsa_data_off(par, L.rank), p)) + 2 * st;
      st_relaxed_sys(dst, w0);
      st_relaxed_sys(dst + 1, w1);
    }
  }
}

// One statistic of this rank for sequence s into every peer (the pass's final warp, lane-wise)
__device__ __forceinline__ void lsa_publish_stat(const LsaLink& L, uint64_t s, int st, double v) {
  if (L.seq[1] == s) return;  // injected fault: this rank never publishes sweep s
  const int par = (int)(s & 1);
  const uint64_t tag = (uint64_t)(uint32_t)s << 32;
  const uint64_t u = (uint64_t)__double_as_longlong(v);
  const uint64_t w0 = tag | (u & 0xffffffffull), w1 = tag | (u >> 32);
  for (int p = 0; p < L.world; ++p) {
    uint64_t* dst = static_cast<uint64_t*>(ncclGetLsaPointer(L.win, lsa_data_off(par, L.rank), p)) + 2 * st;
    st_relaxed_sys(dst, w0);
    st_relaxed_sys(dst + 1, w1);
  }
}

// Value of statistic st from rank r for sequence s, polled from this rank's window
// (bounded by the globaltimer deadline; *ok = false on timeout).
__device__ __forceinline__ double lsa_take(const LsaLink& L, uint64_t s, int r, int st, unsigned long long deadline,
                                           bool* ok) {
  const uint32_t want = (uint32_t)s;
  const uint64_t* w = static_cast<const uint64_t*>(ncclGetLocalPointer(L.win, lsa_data_off((int)(s & 1), r))) + 2 * st;
  uint64_t a = ld_relaxed_sys(w), b = ld_relaxed_sys(w + 1);
  while ((uint32_t)(a >> 32) != want || (uint32_t)(b >> 32) != want) {
    if (lsa_now_ns() > deadline) {
      *ok = false;
      return 0.0;
    }
    a = ld_relaxed_sys(w);
    b = ld_relaxed_sys(w + 1);
  }
  return __longlong_as_double((long long)((b << 32) | (a & 0xffffffffull)));
}

// A rank without genes still takes part in every exchange: publish zeros (unless the fit
// is done, in which case no rank publishes: `done` is identical on every rank).
static __global__ void lsa_publish_zeros_kernel(LsaLink L, int ns, const int* done) {
  if (*(volatile const int*)done) return;
  const uint64_t s = *L.seq + 1;
  lsa_publish(L, s, ns, [](int) { return 0.0; }, threadIdx.x);
}

// Start-up check of the path (all ranks, collectively): publish a rank pattern for sequence
// `s`, poll (bounded), verify every peer's pattern.  ok[0] = 1 on success.
static __global__ void lsa_selftest_kernel(LsaLink L, uint64_t s, int* ok) {
  const int lane = threadIdx.x;
  lsa_publish(L, s, 32, [&](int st) { return 1000.0 * L.rank + st + 0.25 * (double)s; }, lane);
  bool good = true;
  const unsigned long long deadline = lsa_now_ns() + L.timeout_ns;
  for (int r = 0; r < L.world; ++r) {
    const double v = lsa_take(L, s, r, lane, deadline, &good);
    good = good && v == 1000.0 * r + lane + 0.25 * (double)s;
  }
  good = __all_sync(0xffffffffu, good);
  if (lane == 0) *ok = good ? 1 : 0;
}

// seq := (max over ranks, already in *m) + 2 -- the entry resync of every shard call
static __global__ void lsa_resync_kernel(const unsigned long long* m, unsigned long long* seq) {
  seq[0] = m[0] + 2ull;
  seq[1] = 0ull;
}

}  // namespace cavi
