// devcommon.cuh -- device helpers shared by the binning kernels of
// kernels.cu and warp_tiles.cu (private to librafi).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <mutex>
#include <utility>

#include "internal.h"

#include <cstdio>

// Debug builds (build.py --variants "debug"): device-side bounds checks that
// trap with a message (compute-sanitizer is not available on the GPU pool).
#ifdef RAFI_DEBUG_BOUNDS
#define RAFI_DCHECK(cond, what)                                                        \
  do {                                                                                 \
    if (!(cond)) {                                                                     \
      printf("RAFI_DCHECK failed: %s (%s:%d) block %d thread %d\n", what, __FILE__, __LINE__, \
             (int)blockIdx.x, (int)threadIdx.x);                                        \
      __trap();                                                                        \
    }                                                                                  \
  } while (0)
#else
#define RAFI_DCHECK(cond, what) \
  do {                          \
  } while (0)
#endif

namespace rafi_impl {

constexpr int kHistTilesPerCta = 8;  // tiles per "block" of the two-level tile scan (H granularity)

constexpr uint32_t kFull = 0xffffffffu;

// x / d for x < 2^32 / d (checked by the callers' bounds), d >= 1.
struct FastDiv {
  uint32_t d, m;
  __host__ explicit FastDiv(uint32_t dd) : d(dd), m(dd <= 1 ? 0u : (uint32_t)((((uint64_t)1 << 32) + dd - 1) / dd)) {}
  __device__ __forceinline__ uint32_t div(uint32_t x) const { return d <= 1 ? x : __umulhi(x, m); }
};

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm volatile("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}


__device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }
__device__ __forceinline__ uint64_t umax64(uint64_t a, uint64_t b) { return a > b ? a : b; }

__device__ __forceinline__ uint64_t n_items(const CtrlDev& c, uint64_t cap) {
  return c.ctr < cap ? c.ctr : cap;
}


// "Last block done" detection for single-launch epilogues: every block
// publishes its writes and counts itself in *done; the last one returns true
// (and re-arms the counter for the next launch).
__device__ __forceinline__ bool last_block(unsigned* done) {
  __shared__ bool s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned total = gridDim.x * gridDim.y * gridDim.z;
    s_last = atomicAdd(done, 1u) == total - 1;
    if (s_last) { *done = 0; __threadfence(); }
  }
  __syncthreads();
  return s_last;
}

// ---------------------------------------------------------------- a5/a8 peer control

// The count exchange and the completion barrier of a FUSED/CE
// forward without NCCL: every process owns a mailbox (mbox_words), CUDA-IPC
// mapped by every peer.  A round's epoch is the local counter mbox[0], bumped
// in lockstep by every process.  Writers order their data before a flag with
// one system-scope fence and relaxed flag stores; readers poll with
// ld.acquire.sys.
struct PeerCtl {
  unsigned long long* const* mbox;  // [P] mailboxes (local or IPC-mapped), nullptr = off
  int proc, P;
  unsigned long long timeout_ns;    // give up a wait after this long (0 = never)
  unsigned long long* err;          // set to 1 when a wait gave up (CtrlDev::status of local rank 0)
};

__device__ __forceinline__ void st_relaxed_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// Wait until *flag >= e.  A peer that never arrives would be a hang: after
// pc.timeout_ns (0 = never) give up, flag the error for the host and return
// false -- no trap, so the CUDA context stays usable for cleanup.
static __device__ bool spin_until(const PeerCtl& pc, const unsigned long long* flag, unsigned long long e) {
  const unsigned long long t0 = globaltimer_ns();
  for (uint32_t i = 1; ld_acquire_sys(flag) < e; ++i) {
    if (pc.timeout_ns && (i & 1023) == 0 && globaltimer_ns() - t0 > pc.timeout_ns) {
      atomicExch(pc.err, 1ull);
      return false;
    }
  }
  return true;
}

// Completion barrier by one whole block: this process's pushes of the round
// (made visible system-wide before the call) precede its flag in every
// mailbox; return once every process's flag is up (or a wait timed out,
// which sets *pc.err).
static __device__ void ctl_barrier_block(const PeerCtl& pc) {
  unsigned long long* mine = pc.mbox[pc.proc];
  const unsigned long long e = *reinterpret_cast<volatile unsigned long long*>(&mine[0]);
  if (threadIdx.x == 0) {
    __threadfence_system();
    for (int p = 0; p < pc.P; ++p) st_relaxed_sys(&pc.mbox[p][8 + pc.P + pc.proc], e);
  }
  for (int p = threadIdx.x; p < pc.P; p += blockDim.x) spin_until(pc, &mine[8 + pc.P + p], e);
  __syncthreads();
  asm volatile("fence.acq_rel.sys;" ::: "memory");
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// 1-D bulk copy global -> shared through the TMA unit (cp.async.bulk, UBLKCP)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}

// Dynamic shared memory above 48 KiB is opted into per kernel AND per device
// (every device has its own context): remember the largest grant per pair.
inline cudaError_t ensure_smem(const void* fn, int bytes, int device) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> granted;
  std::lock_guard<std::mutex> lock(mu);
  int& have = granted[{fn, device}];
  if (bytes <= have) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) have = bytes;
  return e;
}

// ---------------------------------------------------------------- warp-tile path (warp_tiles.cu)

// The warp-tile histogram serves any 128/256-item tiling with R <= 8.
inline bool hist_w_ok(uint32_t tile, int R) { return (tile == 128 || tile == 256) && R <= 8; }
int launch_hist_w(Ctx* c, int nsm);
int launch_scatter_w(Ctx* c, bool fused, bool wrap, PeerCtl pc, int nsm);

}  // namespace rafi_impl
