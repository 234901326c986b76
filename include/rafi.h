/*
 * rafi.h -- C ABI of the B200-native RaFI work-item forwarding library.
 *
 * RaFI ("Ray Forwarding Infrastructure", arXiv 2605.30294) lets GPU kernels
 * emit trivially copyable work items ("rays") addressed to ranks, and moves
 * them to those ranks once per round.  This header is the host side; the
 * device side is include/rafi_device.cuh.  Citations: PAPER:<line> (section)
 * of the paper's LaTeX source.
 *
 * Conventions (all functions):
 *   - Host-callable only.  Return a rafi_status (0 = OK, < 0 = error) unless
 *     stated otherwise.  No C++ exception crosses this boundary.  The text of
 *     the most recent error of the calling thread is rafi_last_error().
 *   - Pointers are plain host or device addresses; no torch types.
 *   - Sizes and counts are 64-bit.  Item counts per rank per round must be
 *     < 2^32 (the paper's 32-bit index in the sort key).
 *   - A context OWNS its queues (cudaMalloc'd).  The NCCL communicator and
 *     the CUDA stream passed at creation are BORROWED: the caller keeps them
 *     alive until rafi_destroy and destroys them afterwards.
 *   - All device work of a context is ordered on its stream.
 *   - Collective calls (rafi_create* with a communicator, rafi_resize,
 *     rafi_forward) must be made by every process of the communicator in the
 *     same order, across all contexts on that communicator.
 *   - After a collective error (e.g. RAFI_ERR_RECV_OVERFLOW) the context is
 *     unusable except for the read-only getters and rafi_destroy; such an
 *     error is returned identically on every rank.
 */
#ifndef RAFI_H
#define RAFI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RAFI_ABI_VERSION 2

typedef enum {
  RAFI_OK = 0,
  RAFI_ERR_INVALID_ARG = -1,   /* bad argument; nothing was done */
  RAFI_ERR_CUDA = -2,          /* a CUDA runtime call failed (see rafi_last_error) */
  RAFI_ERR_NCCL = -3,          /* an NCCL call failed */
  RAFI_ERR_NOMEM = -4,         /* device or pinned-host allocation failed */
  RAFI_ERR_RECV_OVERFLOW = -5, /* some rank would receive more than its capacity (collective) */
  RAFI_ERR_STATE = -6,         /* context is unusable after an earlier collective error */
  RAFI_ERR_UNSUPPORTED = -7,   /* valid request this build/configuration does not support */
  RAFI_ERR_TIMEOUT = -8,       /* a peer-control wait exceeded RAFI_OPT_PEER_TIMEOUT_MS (context unusable) */
  RAFI_ERR_BOOTSTRAP = -9      /* the host all-gather callback of rafi_create_boot reported failure */
} rafi_status;

typedef struct rafi_ctx rafi_ctx; /* opaque; owns all queues */

/*
 * The device interface ("DeviceInterface<T>"): a trivially
 * copyable view assembled on the host and passed BY VALUE as a kernel
 * parameter.  It holds the paper's "four pointers":
 * the input array, the output array, the destination array and the atomic
 * emit counter.  Re-fetch it after every rafi_forward / rafi_resize (the
 * incoming pointer and count change).
 */
typedef struct {
  const void* in;                 /* incoming items, dense, num_in * item_bytes bytes */
  uint64_t num_in;                /* numIncoming() */
  const uint64_t* num_in_dev;     /* the same count, device-resident */
  void* out;                      /* outgoing queue, capacity * item_bytes bytes */
  int32_t* dest;                  /* destination rank per outgoing slot */
  unsigned long long* ctr;        /* atomic emit counter; NOT clamped at capacity */
  unsigned long long* invalid;    /* emits rejected for an invalid destination */
  uint64_t capacity;              /* items (resizeRayQueues) */
  uint32_t item_bytes;            /* sizeof(T) */
  int32_t num_ranks;              /* R: valid destinations are [0, R) */
  int32_t my_rank;                /* this queue's rank in [0, R) */
  int32_t reserved;
} rafi_device_view;

typedef struct {
  size_t item_bytes;   /* sizeof(T) >= 1; items are packed at this stride, no padding */
  size_t capacity;     /* max items per queue, per local rank */
  void* nccl_comm;     /* ncclComm_t spanning all processes (BORROWED), or NULL for one process */
  void* stream;        /* cudaStream_t (BORROWED); NULL = the legacy default stream */
  int local_ranks;     /* logical ranks this process hosts on its device (>= 1); R = procs * local_ranks */
  int device;          /* CUDA device ordinal, or -1 for the calling thread's current device */
} rafi_create_params;

/* Per-round statistics of one local rank (last completed rafi_forward). */
typedef struct {
  uint64_t round;             /* rafi_forward calls completed on this context */
  uint64_t n_out;             /* items that entered the last forward: min(ctr, capacity) */
  uint64_t dropped;           /* emits beyond capacity in that round */
  uint64_t invalid;           /* emits with a destination outside [0, R) */
  uint64_t num_in;            /* items received (= numIncoming now) */
  uint64_t bytes_sent_remote; /* payload bytes this rank sent to other ranks */
  uint64_t bytes_recv_remote; /* payload bytes this rank received from other ranks */
  int64_t G;                  /* the last forward's return value */
  int32_t num_ranks;
  int32_t my_rank;
  /* device time of each phase of the last forward, ms (CUDA events on the
     context stream); 0 unless RAFI_OPT_TIMING is on.  Whole-context values:
     one launch covers all local ranks. */
  float ms_hist, ms_scan, ms_scatter, ms_count_exchange, ms_payload_exchange, ms_wrapup, ms_total;
  float ms_reserved;
  uint64_t kernel_launches;   /* cumulative kernels this context has launched */
  uint64_t forward_launches;  /* kernels launched by the last forward */
  /* sums of the phase times over the forwards (and bulk emits) timed since
     RAFI_OPT_TIMING was last set; acc_forwards / acc_emits count them */
  double acc_ms_emit, acc_ms_hist, acc_ms_scan, acc_ms_scatter, acc_ms_count_exchange, acc_ms_payload_exchange,
      acc_ms_wrapup, acc_ms_total;
  uint64_t acc_forwards, acc_emits;
} rafi_stats;

/* ---- options (rafi_set_option / rafi_get_option) --------------------------- */
#define RAFI_OPT_EXCHANGE 1        /* payload exchange: RAFI_EXCHANGE_* (default AUTO) */
#define RAFI_OPT_TIMING 2          /* 1 = record per-phase CUDA events (forward: adds one event sync;
                                      bulk emit: events around the kernel); setting it resets the
                                      accumulated sums in rafi_stats; default 0 */
#define RAFI_OPT_TILE 3            /* binning tile in items: 256 * 2^k (k <= 4), or 128 on the warp-tile path
                                      (THREADS, R <= 8, item_bytes % 4 == 0; RAFI_ERR_INVALID_ARG
                                      otherwise); 0 = auto from item size and R (warp tiles of 256 or 128
                                      items at R <= 8, block tiles otherwise) */
#define RAFI_OPT_SELF_DIRECT 4     /* reserved (self run placement); 0 */
#define RAFI_OPT_CONTROL 7         /* count exchange and completion barrier of FUSED forwards:
                                      RAFI_CONTROL_* (default AUTO).  Every rank must use the same setting */
#define RAFI_OPT_PEER_TIMEOUT_MS 9 /* RAFI_CONTROL_PEER: how long a kernel waits for a peer's mailbox flag
                                      before giving up, ms (default 20000; 0 = wait forever).  A wait that
                                      times out moves nothing, leaves the kernel normally and makes the
                                      forward (or the next rafi_sync_host) return RAFI_ERR_TIMEOUT; the
                                      context is then unusable.  No trap: the CUDA context stays healthy */
#define RAFI_OPT_FORWARD_GRAPH 8   /* 1 (default) = a blocking FUSED rafi_forward launches its kernels, the
                                      collectives and the read-back of the counts as one cached CUDA graph
                                      (re-captured after any option change or resize); 0 = one launch each.
                                      Forwards timed by RAFI_OPT_TIMING always launch one by one */
#define RAFI_OPT_SCATTER 5         /* how the binning scatter writes destination runs:
                                      RAFI_SCATTER_* (default AUTO).  Same result bytes either way.
                                      Only between rounds; re-chooses the tile unless RAFI_OPT_TILE
                                      pinned it.  RAFI_ERR_UNSUPPORTED if BULK is asked for an item size
                                      that is not a multiple of 4 or a tile that does not fit */

#define RAFI_SCATTER_AUTO 0        /* BULK when the scatter pushes runs of items of >= 24 B to NVLink peers
                                      (FUSED over several processes), the queues hold >= 2^19 items and
                                      BULK is supported, else THREADS (measured winners) */
#define RAFI_SCATTER_THREADS 1     /* threads store every run with coalesced stores.  R <= 8 and
                                      item_bytes % 4 == 0: one warp per 128/256-item tile, 16/8/4-B item
                                      units.  Otherwise block tiles: 16/8/4/2/1-B item units, or, for 4-B
                                      units (item_bytes % 8 == 4, >= 16), 16-B-aligned chunks gathered
                                      from the (at most two) items they cover */
#define RAFI_SCATTER_BULK 2        /* runs are permuted in shared memory and written by TMA bulk stores
                                      (cp.async.bulk shared->global, local or NVLink peer); threads write
                                      only the unaligned < 16-B heads and tails; item_bytes % 4 == 0 */

#define RAFI_CONTROL_AUTO 0        /* PEER when every rank's queues are mapped and no two processes share a
                                      device, else NCCL when there is a communicator, else HOST */
#define RAFI_CONTROL_NCCL 1        /* ncclAllGather of the count rows, ncclAllReduce as the completion barrier */
#define RAFI_CONTROL_PEER 2        /* the scan kernel's last block pushes this process's count rows into
                                      every peer's CUDA-IPC mailbox over NVLink, fences once and raises a
                                      flag in each; the scatter kernel's last block runs the completion
                                      barrier the same way; both spin on ld.acquire.sys (bounded by
                                      RAFI_OPT_PEER_TIMEOUT_MS).  Refused (RAFI_ERR_UNSUPPORTED) when two
                                      processes share a device: nothing makes their kernels co-resident */
#define RAFI_CONTROL_HOST 3        /* the paper's host-side count exchange: each process copies
                                      its count rows to the host, the bootstrap's all-gather callback
                                      (rafi_create_boot) exchanges them, the plan runs on the device, and
                                      after the scatter a host all-gather is the completion barrier.  No
                                      kernel ever waits on another process.  Needs a bootstrap; blocking
                                      forwards only (rafi_forward_async: RAFI_ERR_UNSUPPORTED) */

#define RAFI_EXCHANGE_AUTO 0       /* FUSED when every rank's queues are addressable, else NCCL */
#define RAFI_EXCHANGE_NCCL 1       /* stage the sorted batch, grouped ncclSend/ncclRecv (one local rank per process) */
#define RAFI_EXCHANGE_PEER 2       /* stage the sorted batch, receivers pull it with a copy kernel over
                                      local / CUDA-IPC peer pointers (NVLink) */
#define RAFI_EXCHANGE_FUSED 3      /* the scatter writes every destination run straight into the destination
                                      rank's incoming queue (local HBM or NVLink peer memory); the count
                                      matrix is exchanged first (RAFI_OPT_CONTROL); no send batch, no
                                      separate copy */

/* ---- lifecycle ------------------------------------------------------------ */

/* HostContext<T>(gpu, comm) + resizeRayQueues(capacity).
 * One local rank on the current device.  nccl_comm may be NULL (R = 1).
 * COLLECTIVE when nccl_comm spans several processes. */
int rafi_create(rafi_ctx** out, size_t item_bytes, size_t capacity, void* nccl_comm, void* stream);

/* General form; see rafi_create_params.  COLLECTIVE over nccl_comm. */
int rafi_create_ex(rafi_ctx** out, const rafi_create_params* params);

/* Host all-gather over the process group: every process calls it with the
 * same `bytes`; on return recv[p*bytes, (p+1)*bytes) holds process p's send.
 * Blocking and collective; returns 0 on success.  Any host transport works
 * (MPI_Allgather, a torch.distributed gloo group, ...): the paper exchanges
 * counts over MPI on the host. */
typedef int (*rafi_allgather_fn)(void* user, const void* send, void* recv, size_t bytes);

typedef struct {
  int nprocs;                  /* processes in the group (>= 1) */
  int proc;                    /* this process's index in [0, nprocs) */
  rafi_allgather_fn allgather; /* required when nprocs > 1 */
  void* user;                  /* passed through to allgather */
} rafi_bootstrap;

/* rafi_create_ex with a host bootstrap instead of (or besides) an NCCL
 * communicator: the process group is `boot` (params->nccl_comm may be NULL;
 * if given it must span the same processes in the same order).  The bootstrap
 * carries the CUDA-IPC handles of every queue, so without NCCL the FUSED and
 * PEER exchanges run under RAFI_CONTROL_PEER or RAFI_CONTROL_HOST (the NCCL
 * exchange and control need params->nccl_comm).  Processes may share a device
 * (e.g. tests on one GPU): AUTO control is then HOST.  Creation fails on every
 * process with RAFI_ERR_INVALID_ARG if item_bytes, capacity or local_ranks
 * differ between processes.  COLLECTIVE over the group. */
int rafi_create_boot(rafi_ctx** out, const rafi_create_params* params, const rafi_bootstrap* boot);

/* resizeRayQueues(N): reallocates every queue of every local
 * rank to `capacity` items.  Incoming items are kept up to the new capacity;
 * the outgoing queue must be empty (no emits since the last forward), else
 * RAFI_ERR_INVALID_ARG.  Not concurrent with emits or forwards.  COLLECTIVE:
 * every process must pass the same capacity (checked); the old queues are
 * freed only after every process has closed its CUDA-IPC mappings of them. */
int rafi_resize(rafi_ctx* ctx, size_t capacity);

/* Frees all queues.  Does NOT destroy the communicator or the stream.  Waits
 * for the context's outstanding device work.  NULL is a no-op. */
void rafi_destroy(rafi_ctx* ctx);

/* ---- device interface ------------------------------------------------------- */

/* getDeviceInterface() for local rank `local` in [0, local_ranks). */
int rafi_get_device_view(const rafi_ctx* ctx, int local, rafi_device_view* out);

/* numIncoming() on the host; 0 for a bad argument. */
uint64_t rafi_num_incoming(const rafi_ctx* ctx, int local);

/* Bulk emitOutgoing from the host (PAPER:70-71 semantics, one launch):
 * appends items[i] (item_bytes each, packed) addressed to dests[i] to local
 * rank `local`'s outgoing queue.  `items`/`dests` may be device pointers or
 * host pointers (pinned or pageable; copied through a staging buffer on the
 * context stream).  Invalid destinations are rejected and counted; emits past
 * capacity are dropped and counted.  Within one call accepted items keep their
 * relative order in the queue except across 2048-item blocks, whose order
 * follows the atomic counter.  Asynchronous w.r.t. the host for device and
 * pinned host pointers: host inputs are copied on a separate copy-in stream
 * into one of two staging buffers (so the copy of the next batch overlaps
 * this batch's forward and read-back); the caller must keep a host buffer
 * unchanged until the context stream has passed this call. */
int rafi_emit_bulk(rafi_ctx* ctx, int local, const void* items, const int32_t* dests, uint64_t n);

/* ---- forwarding -------------------------------------------------------------- */

/* forwardRays().  COLLECTIVE.  Bins every local rank's
 * outgoing queue by destination (stable in slot order), exchanges counts and
 * payloads so that each item lands in the incoming queue of the rank its emit
 * named -- per destination, sources in rank order, each source's items in
 * slot order -- resets the emit counters, and returns G >= 0, the total
 * number of items received by all ranks (identical on every rank; 0 means
 * distributed termination).  Returns a negative rafi_status on
 * error; RAFI_ERR_RECV_OVERFLOW (some rank would receive > capacity) is
 * detected before any payload moves and leaves all queues unchanged.
 * The payload copy may still be in flight on the stream when this returns;
 * anything ordered after it on the stream sees the new incoming queues. */
int64_t rafi_forward(rafi_ctx* ctx);

/* ---- device-side termination and CUDA graphs --------- */

/* The FUSED forward without any host synchronisation: enqueues the complete
 * forward on the context stream (so it can be captured into a CUDA graph,
 * NCCL collectives included) and, when the work runs, writes G -- the same
 * value rafi_forward returns -- to *G_dev (device-visible u64;
 * it may be mapped pinned host memory).  On a receive overflow (or a peer
 * control timeout) nothing moves and *G_dev = ~0ull; the context becomes
 * unusable and the next rafi_sync_host returns the error.  Host-side counters (rafi_num_incoming, rafi_get_stats and
 * the num_in field of views) are NOT refreshed: device code must read
 * numIncoming through num_in_dev (rafi::Queue does), and launches sized on
 * the host should cover the capacity.  COLLECTIVE.  Needs the FUSED exchange
 * (RAFI_ERR_UNSUPPORTED otherwise) and NCCL or PEER control.  A pending
 * rafi_read_incoming_async is waited for in stream order first. */
int rafi_forward_async(rafi_ctx* ctx, unsigned long long* G_dev);

/* Blocks until the context stream is idle and refreshes the host-side
 * counters from the device (after rafi_forward_async / graph launches). */
int rafi_sync_host(rafi_ctx* ctx);

/* Capture work issued on the context stream (app kernels, rafi_forward_async)
 * into an executable CUDA graph (*exec, cudaGraphExec_t), and replay it.  The
 * context stream must not be the legacy default stream.  rafi_capture_begin
 * and rafi_graph_launch first make the context stream wait (stream-ordered)
 * for any pending rafi_read_incoming_async, so a replayed forward never
 * rewrites an incoming queue that is still being copied out. */
int rafi_capture_begin(rafi_ctx* ctx);
int rafi_capture_end(rafi_ctx* ctx, void** exec);
int rafi_graph_launch(rafi_ctx* ctx, void* exec);
int rafi_graph_destroy(void* exec);

/* ---- introspection (host copies; ordered on the context stream, blocking) --- */

int rafi_num_ranks(const rafi_ctx* ctx);                 /* R, or < 0 on error */
int rafi_local_ranks(const rafi_ctx* ctx);               /* local ranks, or < 0 */
int rafi_rank_of(const rafi_ctx* ctx, int local);        /* global rank of local rank, or < 0 */
uint64_t rafi_capacity(const rafi_ctx* ctx);
uint64_t rafi_item_bytes(const rafi_ctx* ctx);

/* Copies incoming items [first, first+count) of local rank `local` to dst
 * (host or device pointer). */
int rafi_read_incoming(const rafi_ctx* ctx, int local, void* dst, uint64_t first, uint64_t count);

/* Asynchronous rafi_read_incoming (dst should be pinned host memory or
 * device memory): the copy runs on the context's copy-out stream after the
 * work already enqueued on the context stream, and overlaps later work -- in
 * particular the next rafi_emit_bulk's host-to-device copy, which runs on a
 * separate copy-in stream.  The next forward waits for it before rewriting
 * the incoming queue.  dst must stay valid until rafi_read_wait returns.
 * Not while the context stream is being captured (RAFI_ERR_UNSUPPORTED). */
int rafi_read_incoming_async(rafi_ctx* ctx, int local, void* dst, uint64_t first, uint64_t count);

/* Blocks until every rafi_read_incoming_async of the context has landed. */
int rafi_read_wait(rafi_ctx* ctx);

/* Snapshot of the outgoing queue before forwarding: *ctr and *invalid receive
 * the raw counters; items_dst / dests_dst (may be NULL) receive
 * min(ctr, capacity) items / dests. */
int rafi_read_outgoing(const rafi_ctx* ctx, int local, void* items_dst, int32_t* dests_dst,
                       uint64_t* ctr, uint64_t* invalid);

/* The destination-sorted send batch of the last forward (n_out items).
 * RAFI_ERR_UNSUPPORTED after a FUSED forward, which writes no send batch. */
int rafi_read_binned(const rafi_ctx* ctx, int local, void* dst, uint64_t count);

/* The last forward's R x R count matrix, row = source rank, column = destination. */
int rafi_get_matrix(const rafi_ctx* ctx, uint64_t* C);

int rafi_get_stats(const rafi_ctx* ctx, int local, rafi_stats* out);

int rafi_set_option(rafi_ctx* ctx, int key, long long value);
int rafi_get_option(const rafi_ctx* ctx, int key, long long* value);

const char* rafi_status_str(int status);
const char* rafi_last_error(void);
int rafi_abi_version(void);

/* ---- NCCL communicator helpers (the library's own NCCL, linked once) -------- */

/* ncclGetUniqueId into id[128]. */
int rafi_nccl_unique_id(void* id128);
/* ncclCommInitRank on `device` (-1 = current); *comm receives an ncclComm_t. */
int rafi_nccl_comm_init(void** comm, int nranks, int rank, const void* id128, int device);
int rafi_nccl_comm_destroy(void* comm);

/* ---- diagnostics ------------------------------------------------------------ */

/* Self-test of the peer-control protocol (RAFI_CONTROL_PEER: the count
 * exchange of a5, and the completion barrier) on ONE device, where
 * processes cannot be co-scheduled: P blocks of one cooperative launch each
 * play a process with its own mailbox and L local ranks, for `rounds` rounds
 * of [write own count rows, count exchange, check the whole R x R matrix,
 * completion barrier].  Block `absent` (>= 0) never arrives, so the others must
 * give up after timeout_ms (0 = never: only with absent < 0).  *bad = matrix
 * entries that arrived wrong; *timed_out = processes whose wait gave up. */
int rafi_selftest_peer_control(int device, int P, int L, int rounds, int absent, long long timeout_ms,
                               uint64_t* bad, uint64_t* timed_out);

/* Diagnostic (measurement only): make the FUSED scatter write global rank
 * `grank`'s incoming queue (a local rank of this process) into `queue`
 * instead of the context's own buffer -- a device pointer of at least
 * capacity * item_bytes bytes, 16-byte aligned, owned by the caller and valid
 * until it is restored.  It may live on ANOTHER device: peer access to that
 * device is enabled here.  With it one process can drive the NVLink push of a
 * FUSED forward (rank me's block for rank d written straight
 * into d's queue) on its own, e.g. under a single-process ncu NVLink counter
 * capture.  The redirected rank's num_incoming stays correct, but reads of
 * its incoming queue through this API (rafi_read_incoming, the device view)
 * see the context's own, stale buffer.  queue = NULL restores the default.
 * RAFI_ERR_INVALID_ARG (grank not local, misaligned), RAFI_ERR_CUDA. */
int rafi_diag_redirect_incoming(rafi_ctx* ctx, int grank, void* queue);

/* ---- host-side planning (pure host code; no GPU needed) --------------------- */

/* From the R x R count matrix C (row-major, C[s*R+d] = items s sends to d)
 * computes what destination rank `d` receives: recv_count[s] = C[s][d],
 * recv_off[s] = sum_{s'<s} C[s'][d] (prefix sums), and for each
 * source the offset of its block for d inside its sorted batch,
 * src_off[s] = sum_{d'<d} C[s][d'].  *total = sum_s C[s][d];
 * *G = sum of all entries; *overflow = 1 if ANY column sum
 * exceeds capacity (so every rank decides alike), else 0.
 * Any output pointer may be NULL. */
int rafi_plan(int R, const uint64_t* C, uint64_t capacity, int d, uint64_t* recv_count,
              uint64_t* recv_off, uint64_t* src_off, uint64_t* total, uint64_t* G, int* overflow);

#ifdef __cplusplus
}
#endif

#endif /* RAFI_H */
