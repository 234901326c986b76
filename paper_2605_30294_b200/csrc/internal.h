// internal.h -- private declarations of librafi (not part of the ABI).
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdint>
#include <string>
#include <vector>

#include "rafi.h"

namespace rafi_impl {

void set_error(const std::string& msg);

#define RAFI_CK_CUDA(expr)                                                              \
  do {                                                                                  \
    cudaError_t e_ = (expr);                                                            \
    if (e_ != cudaSuccess) {                                                            \
      ::rafi_impl::set_error(std::string(#expr) + ": " + cudaGetErrorString(e_));       \
      return e_ == cudaErrorMemoryAllocation ? RAFI_ERR_NOMEM : RAFI_ERR_CUDA;           \
    }                                                                                   \
  } while (0)

#define RAFI_CK_NCCL(expr)                                                              \
  do {                                                                                  \
    ncclResult_t r_ = (expr);                                                           \
    if (r_ != ncclSuccess) {                                                            \
      ::rafi_impl::set_error(std::string(#expr) + ": " + ncclGetErrorString(r_));       \
      return RAFI_ERR_NCCL;                                                             \
    }                                                                                   \
  } while (0)

#define RAFI_CK(expr)          \
  do {                         \
    int s_ = (expr);           \
    if (s_ != RAFI_OK) return s_; \
  } while (0)

// Device-resident per-local-rank control block.  ctr/invalid are the
// counters emitOutgoing bumps; the rest is written by the binning kernels.
struct alignas(64) CtrlDev {
  unsigned long long ctr;       // emit counter (not clamped)
  unsigned long long invalid;   // rejected emits
  unsigned long long num_in;    // numIncoming, device copy
  unsigned long long n_out;     // min(ctr, cap) seen by the last forward
  unsigned long long dropped;   // ctr - n_out of the last forward
  unsigned long long invalid_last;
  unsigned long long status;    // local rank 0 only: nonzero = a peer-control wait timed out (RAFI_ERR_TIMEOUT)
  unsigned long long pad;
};

// Device table of one local rank's buffers (kernel argument array).
struct RankDev {
  uint8_t* out;
  int32_t* dest;
  uint8_t* binned[2];
  uint8_t* in;
  uint32_t* H;
  uint32_t* O;
};

// Per-source run of one destination's incoming queue, for the copy kernel.
struct CopyRun {
  const uint8_t* src;      // first byte of the run (source batch + src_off * B)
  unsigned long long dst;  // first item in the destination incoming queue (recv_off)
  unsigned long long count;  // items
};

// Peer control mailbox (one per process, CUDA-IPC mapped by every peer), u64
// words: [0] epoch (local), [8, 8+P) count flags, [8+P, 8+2P) completion
// flags, [8+2P, 8+2P+R*R) the count matrix as the peers push their rows.
inline size_t mbox_words(int P, int R) { return 8 + 2 * (size_t)P + (size_t)R * R; }

struct LocalRank {
  uint8_t* out = nullptr;     // outgoing queue (emit target)
  unsigned long long* mbox = nullptr;  // peer control mailbox (used for local rank 0)
  int32_t* dest = nullptr;    // destination per slot
  uint8_t* binned[2] = {nullptr, nullptr};  // send batches (double-buffered for PEER)
  uint8_t* in = nullptr;      // incoming queue
  uint32_t* H = nullptr;      // [R][tiles] per-tile per-destination counts
  uint32_t* O = nullptr;      // [R][tiles] items per destination in earlier tiles
  uint64_t num_in = 0;        // host copy of numIncoming
  uint64_t n_out = 0, dropped = 0, invalid = 0;  // last forward
  uint64_t sent_remote = 0, recv_remote = 0;
};

struct Ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  ncclComm_t comm = nullptr;  // borrowed; null for a single process
  int nprocs = 1, proc = 0;   // NCCL size / rank
  int L = 1;                  // local ranks
  int R = 1;                  // global ranks = nprocs * L
  uint64_t B = 0;             // item bytes
  uint64_t cap = 0;           // capacity per queue
  uint32_t tile = 0;          // binning tile (items)
  uint64_t max_tiles = 0;     // ceil(cap / tile)
  int exchange = RAFI_EXCHANGE_AUTO;
  int exchange_eff = RAFI_EXCHANGE_FUSED;
  int scatter = RAFI_SCATTER_AUTO;     // requested scatter write path (RAFI_OPT_SCATTER)
  int scatter_eff = RAFI_SCATTER_THREADS;
  bool tile_user = false;              // RAFI_OPT_TILE pinned the tile
  bool timing = false;
  bool broken = false;
  uint64_t round = 0;
  int cur = 0;       // which binned buffer this round writes
  int last_cur = 0;  // which one the last forward wrote
  bool last_fused = false;
  bool host_stale = false;  // rafi_forward_async ran since the last host refresh
  int64_t last_G = 0;

  std::vector<LocalRank> lr;
  RankDev* rank_dev = nullptr;        // [L] device copy of the buffer table
  CtrlDev* ctrl = nullptr;            // [L] device
  uint64_t* Cdev = nullptr;           // [R*R] count matrix, device (row s = source)
  uint64_t* Chost = nullptr;          // [R*R] pinned host mirror
  CtrlDev* ctrl_host = nullptr;       // [L] pinned host mirror
  CopyRun* runs_dev = nullptr;        // [L*R] copy plan, device
  CopyRun* runs_host = nullptr;       // [L*R] pinned
  uint64_t* plan_dev = nullptr;       // [L] per local dest: num_in (for wrap-up)
  uint64_t* off_dev = nullptr;        // [L][R] per-destination base: send_off (staged) / recv_off (FUSED)
  int* ovf_dev = nullptr;             // [1] FUSED: collective receive-overflow flag
  unsigned* done_dev = nullptr;       // [2] last-block counters (scan+plan, scatter+wrap-up)
  uint8_t** in_table_dev = nullptr;   // [R] every global rank's incoming queue (local or IPC-mapped)
  std::vector<uint8_t*> peer_in;      // host copy of in_table
  std::vector<unsigned long long*> peer_mbox;  // [R] every global rank's mailbox (local or IPC-mapped)
  unsigned long long** mbox_table_dev = nullptr;  // [P] mailbox of each process's local rank 0
  int control = RAFI_CONTROL_AUTO;     // RAFI_OPT_CONTROL (requested)
  int ctl_eff = RAFI_CONTROL_AUTO;     // effective control of a multi-process forward (NCCL / PEER / HOST)
  bool ctl_peer = false;               // count exchange + completion barrier over peer mailboxes
  rafi_bootstrap boot{};               // host all-gather of the process group (rafi_create_boot), or empty
  bool shared_gpu = false;             // two processes of the group share one device (no cross-process spin waits)
  uint64_t peer_timeout_ns = 20000000000ull;  // RAFI_OPT_PEER_TIMEOUT_MS (0 = wait forever)
  bool scatter_barrier = false;        // the next scatter launch ends with the peer completion barrier
  uint64_t* plan_host = nullptr;      // [L] pinned
  // peer pointers to every global rank's binned buffers ([R][2]); local ones
  // are our own allocations, remote ones are CUDA-IPC mappings
  std::vector<uint8_t*> peer_binned;
  std::vector<void*> ipc_opened;      // mappings to close
  bool peer_ok = false;

  const void* cls_ptr[2] = {nullptr, nullptr};  // rafi_emit_bulk pointer-type cache
  bool cls_dev[2] = {false, false};
  // host I/O: staging for rafi_emit_bulk from host memory (double-buffered,
  // filled on io_in) and asynchronous read-back (io_out)
  cudaStream_t io_in = nullptr, io_out = nullptr;
  uint8_t* stage2[2] = {nullptr, nullptr};
  size_t stage_cap[2] = {0, 0};
  bool stage_used[2] = {false, false};
  int stage_slot = 1;
  cudaEvent_t ev_stage_ready[2] = {}, ev_stage_free[2] = {}, ev_in_ready = nullptr, ev_out_done = nullptr;
  bool out_pending = false;

  // blocking FUSED forward replayed as one cached CUDA graph (RAFI_OPT_FORWARD_GRAPH)
  bool fwd_graph = true;
  bool fwd_dirty = true;            // options / buffers changed since the graph was captured
  bool fwd_T = false;               // the cached graph records the timing events
  cudaStream_t cap_stream = nullptr;
  cudaGraphExec_t fwd_exec = nullptr;
  uint64_t fwd_graph_launches = 0;  // kernels in the cached graph
  cudaEvent_t ev[8] = {};
  static constexpr int kEmitEv = 32;     // ring of (start, end) event pairs for timed bulk emits
  cudaEvent_t ev_emit[kEmitEv][2] = {};
  int emit_head = 0, emit_tail = 0, emit_mark = 0;  // unread pairs [head, mark) are complete
  bool timing_unread = false, unread_fused = false;  // last forward's events not read yet
  rafi_stats st{};
  uint64_t launches = 0;
  uint64_t fwd_launches = 0;
};

inline RankDev* rank_table(Ctx* c) { return c->rank_dev; }
// bytes of the control blocks [L] followed by the count matrix [R*R] (one allocation)
inline size_t ctrl_c_bytes(const Ctx* c) { return sizeof(CtrlDev) * c->L + sizeof(uint64_t) * c->R * c->R; }

// kernels.cu
uint32_t choose_tile(uint64_t item_bytes, int R, int L);
// warp_tiles.cu: binning tiles of the warp-tile path (one warp owns one
// tile): 128 or 256 items, R <= 8, item_bytes % 8 == 0, and at least two warp
// regions fit; warp_tile_for = the tile the automatic choice takes (0: the
// path does not apply).
bool warp_tiles_ok(uint32_t tile, uint64_t item_bytes, int R, int L);
uint32_t warp_tile_for(uint64_t item_bytes, int R, int L);
uint32_t choose_tile_perm(uint64_t item_bytes, int R);
bool perm_supported(uint64_t item_bytes);
size_t perm_smem_bytes(uint32_t tile, uint64_t item_bytes, int R);
int launch_emit_bulk(Ctx* c, int local, const uint8_t* items, const int32_t* dests, uint64_t n);
// a2 + a3: histogram, then scan (+ plan, + peer count exchange).  On small
// warp-tile forwards launch_hist also scans (and launch_scan is a no-op), so
// both take the scan's arguments.
int launch_hist(Ctx* c, int plan_mode, unsigned long long* G_out = nullptr, bool ctl = false);
int launch_scan(Ctx* c, int plan_mode, unsigned long long* G_out = nullptr, bool ctl = false);
int launch_scatter(Ctx* c, bool fused, bool wrap);
int launch_plan(Ctx* c, bool fused, unsigned long long* G_out = nullptr);
int launch_copy(Ctx* c, int nruns_per_dest);
int launch_wrapup(Ctx* c);
int launch_ctl_selftest(unsigned long long* const* mbox, uint64_t* Cs, int P, int L, int rounds, int absent,
                        unsigned long long timeout_ns, unsigned long long* err, unsigned long long* bad);
size_t scatter_smem_bytes(uint32_t tile, uint64_t item_bytes, int R);

}  // namespace rafi_impl
