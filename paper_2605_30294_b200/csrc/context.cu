// context.cu -- host context of librafi: lifecycle, arena, the forward()
// state machine and the C ABI entry points.
//
// Per local rank the arena holds (all cudaMalloc'd, so CUDA IPC works):
//   out[cap*B]   outgoing queue, the emit target
//   dest[cap]    int32 destination per slot
//   binned[2]    destination-sorted send batch; two of them when peers pull
//                over NVLink, so round k+1's scatter never overwrites what a
//                peer may still be reading from round k (double buffer)
//   in[cap*B]    incoming queue
//   H, O         per-tile per-destination counts and their scan
// plus a 64-byte control block (counters) per local rank.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "internal.h"

namespace rafi_impl {

static thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }

static constexpr size_t kPad = 256;  // slack after each item buffer (vector over-reads)

static int alloc_dev(void** p, size_t bytes) {
  *p = nullptr;
  if (bytes == 0) bytes = 16;
  cudaError_t e = cudaMalloc(p, bytes);
  if (e != cudaSuccess) {
    set_error(std::string("cudaMalloc(") + std::to_string(bytes) + "): " + cudaGetErrorString(e));
    cudaGetLastError();
    return e == cudaErrorMemoryAllocation ? RAFI_ERR_NOMEM : RAFI_ERR_CUDA;
  }
  return RAFI_OK;
}

static void free_rank(LocalRank& r) {
  cudaFree(r.out); cudaFree(r.dest); cudaFree(r.binned[0]); cudaFree(r.binned[1]);
  cudaFree(r.in); cudaFree(r.H); cudaFree(r.O); cudaFree(r.mbox);
  r.mbox = nullptr;
  r.out = nullptr; r.dest = nullptr; r.binned[0] = r.binned[1] = nullptr; r.in = nullptr;
  r.H = nullptr; r.O = nullptr;
}

static void close_ipc(Ctx* c) {
  for (void* p : c->ipc_opened) cudaIpcCloseMemHandle(p);
  c->ipc_opened.clear();
  c->peer_binned.clear();
  c->peer_in.clear();
  c->peer_mbox.clear();
  c->peer_ok = false;
}

static bool double_buffered(const Ctx* c) { return c->nprocs > 1; }

static int alloc_rank(Ctx* c, LocalRank& r, uint64_t cap) {
  const size_t ib = (size_t)cap * c->B + kPad;
  RAFI_CK(alloc_dev((void**)&r.out, ib));
  RAFI_CK(alloc_dev((void**)&r.dest, (size_t)cap * 4 + kPad));
  RAFI_CK(alloc_dev((void**)&r.binned[0], ib));
  if (double_buffered(c)) RAFI_CK(alloc_dev((void**)&r.binned[1], ib));
  RAFI_CK(alloc_dev((void**)&r.in, ib));
  const size_t hb = (size_t)std::max<uint64_t>(c->max_tiles, 1) * c->R * 4 + kPad;
  RAFI_CK(alloc_dev((void**)&r.H, hb));
  RAFI_CK(alloc_dev((void**)&r.O, hb));
  const size_t mb = mbox_words(c->nprocs, c->R) * sizeof(unsigned long long);
  RAFI_CK(alloc_dev((void**)&r.mbox, mb));
  RAFI_CK_CUDA(cudaMemset(r.mbox, 0, mb));
  return RAFI_OK;
}

static int upload_rank_table(Ctx* c) {
  std::vector<RankDev> t(c->L);
  for (int l = 0; l < c->L; ++l) {
    LocalRank& r = c->lr[l];
    t[l] = RankDev{r.out, r.dest, {r.binned[0], r.binned[1] ? r.binned[1] : r.binned[0]}, r.in, r.H, r.O};
  }
  RAFI_CK_CUDA(cudaMemcpyAsync(c->rank_dev, t.data(), sizeof(RankDev) * c->L, cudaMemcpyHostToDevice, c->stream));
  RAFI_CK_CUDA(cudaStreamSynchronize(c->stream));
  return RAFI_OK;
}

// Host all-gather over the process group (collective, blocking): the
// bootstrap's callback when there is one, else NCCL through a small device
// buffer on the context stream.  recv[p * bytes ..] = process p's send.
static int proc_allgather(Ctx* c, const void* send, void* recv, size_t bytes) {
  if (c->nprocs == 1) {
    std::memcpy(recv, send, bytes);
    return RAFI_OK;
  }
  if (c->boot.allgather) {
    if (c->boot.allgather(c->boot.user, send, recv, bytes) != 0) {
      set_error("bootstrap all-gather callback failed");
      return RAFI_ERR_BOOTSTRAP;
    }
    return RAFI_OK;
  }
  uint8_t* dbuf = nullptr;
  RAFI_CK(alloc_dev((void**)&dbuf, bytes * c->nprocs));
  int rc = RAFI_OK;
  do {
    if (cudaMemcpyAsync(dbuf + bytes * c->proc, send, bytes, cudaMemcpyHostToDevice, c->stream) != cudaSuccess) { rc = RAFI_ERR_CUDA; break; }
    const ncclResult_t nr = ncclAllGather(dbuf + bytes * c->proc, dbuf, bytes, ncclUint8, c->comm, c->stream);
    if (nr != ncclSuccess) { set_error(std::string("ncclAllGather: ") + ncclGetErrorString(nr)); rc = RAFI_ERR_NCCL; break; }
    if (cudaMemcpyAsync(recv, dbuf, bytes * c->nprocs, cudaMemcpyDeviceToHost, c->stream) != cudaSuccess) { rc = RAFI_ERR_CUDA; break; }
    if (cudaStreamSynchronize(c->stream) != cudaSuccess) { rc = RAFI_ERR_CUDA; break; }
  } while (0);
  if (rc == RAFI_ERR_CUDA) { cudaGetLastError(); set_error("proc_allgather: CUDA copy failed"); }
  cudaFree(dbuf);
  return rc;
}

// Host barrier over the process group.
static int proc_barrier(Ctx* c) {
  int one = 1;
  std::vector<int> all(c->nprocs);
  return proc_allgather(c, &one, all.data(), sizeof(int));
}

// Every rank learns every rank's binned[0..1], in and mailbox pointers:
// local ones directly, other processes' through CUDA IPC handles all-gathered
// over the process group.  The same exchange checks that every process
// agrees on (item_bytes, capacity, local_ranks) and notes whether two
// processes share a device.  Collective; peer_ok, shared_gpu and any
// disagreement are decided identically on all ranks.
static constexpr int kMapped = 4;  // binned[0], binned[1], in, mbox

static uint8_t* mapped_buf(LocalRank& r, int b) {
  return b < 2 ? (r.binned[b] ? r.binned[b] : r.binned[0]) : b == 2 ? r.in : reinterpret_cast<uint8_t*>(r.mbox);
}

static int upload_in_table(Ctx* c) {
  std::vector<uint8_t*> t(c->R, nullptr);
  for (int g = 0; g < c->R; ++g) t[g] = c->peer_in.empty() ? nullptr : c->peer_in[g];
  RAFI_CK_CUDA(cudaMemcpyAsync(c->in_table_dev, t.data(), sizeof(uint8_t*) * c->R, cudaMemcpyHostToDevice, c->stream));
  std::vector<unsigned long long*> m(c->nprocs, nullptr);
  for (int p = 0; p < c->nprocs; ++p) m[p] = c->peer_mbox.empty() ? nullptr : c->peer_mbox[(size_t)p * c->L];
  RAFI_CK_CUDA(cudaMemcpyAsync(c->mbox_table_dev, m.data(), sizeof(void*) * c->nprocs, cudaMemcpyHostToDevice,
                               c->stream));
  RAFI_CK_CUDA(cudaStreamSynchronize(c->stream));
  return RAFI_OK;
}

struct ProcRecord {  // what every process publishes at create / resize
  uint64_t item_bytes, capacity;
  int32_t local_ranks, ipc_ok;
  uint8_t uuid[16];  // device UUID
};

static int exchange_peer_pointers(Ctx* c) {
  close_ipc(c);
  c->peer_binned.assign((size_t)c->R * 2, nullptr);
  c->peer_in.assign((size_t)c->R, nullptr);
  c->peer_mbox.assign((size_t)c->R, nullptr);
  auto place = [&](int g, int b, uint8_t* p) {
    if (b < 2) c->peer_binned[(size_t)g * 2 + b] = p;
    else if (b == 2) c->peer_in[g] = p;
    else c->peer_mbox[g] = reinterpret_cast<unsigned long long*>(p);
  };
  for (int l = 0; l < c->L; ++l)
    for (int b = 0; b < kMapped; ++b) place(c->proc * c->L + l, b, mapped_buf(c->lr[l], b));
  if (c->nprocs == 1) { c->peer_ok = true; c->shared_gpu = false; return upload_in_table(c); }
  const size_t nh = (size_t)kMapped * c->L;
  const size_t per = sizeof(ProcRecord) + sizeof(cudaIpcMemHandle_t) * nh;
  std::vector<uint8_t> mine(per, 0), all(per * c->nprocs);
  ProcRecord me{};
  me.item_bytes = c->B;
  me.capacity = c->cap;
  me.local_ranks = c->L;
  me.ipc_ok = 1;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, c->device) == cudaSuccess) std::memcpy(me.uuid, &prop.uuid, 16);
  else cudaGetLastError();
  for (int l = 0; l < c->L; ++l)
    for (int b = 0; b < kMapped; ++b) {
      cudaIpcMemHandle_t h;
      std::memset(&h, 0, sizeof(h));
      if (cudaIpcGetMemHandle(&h, mapped_buf(c->lr[l], b)) != cudaSuccess) { me.ipc_ok = 0; cudaGetLastError(); }
      std::memcpy(mine.data() + sizeof(ProcRecord) + sizeof(h) * (kMapped * l + b), &h, sizeof(h));
    }
  std::memcpy(mine.data(), &me, sizeof(me));
  RAFI_CK(proc_allgather(c, mine.data(), all.data(), per));
  auto rec = [&](int p) {
    ProcRecord r;
    std::memcpy(&r, all.data() + per * p, sizeof(r));
    return r;
  };
  bool agree = true;
  c->shared_gpu = false;
  for (int p = 0; p < c->nprocs; ++p) {
    const ProcRecord r = rec(p);
    if (r.item_bytes != c->B || r.capacity != c->cap || r.local_ranks != c->L) agree = false;
    for (int q = 0; q < p; ++q)
      if (std::memcmp(rec(q).uuid, r.uuid, 16) == 0) c->shared_gpu = true;
  }
  if (!agree) {
    set_error("processes disagree on item_bytes, capacity or local_ranks");
    return RAFI_ERR_INVALID_ARG;
  }
  int ok = 1;
  for (int p = 0; p < c->nprocs; ++p) ok &= rec(p).ipc_ok;
  for (int p = 0; p < c->nprocs && ok; ++p) {
    if (p == c->proc) continue;
    for (int l = 0; l < c->L && ok; ++l)
      for (int b = 0; b < kMapped && ok; ++b) {
        cudaIpcMemHandle_t h;
        std::memcpy(&h, all.data() + per * p + sizeof(ProcRecord) + sizeof(h) * (kMapped * l + b), sizeof(h));
        void* ptr = nullptr;
        if (cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
          ok = 0; cudaGetLastError(); break;
        }
        c->ipc_opened.push_back(ptr);
        place(p * c->L + l, b, (uint8_t*)ptr);
      }
  }
  // agree: peer modes only if every process mapped every peer
  std::vector<int> oks(c->nprocs);
  RAFI_CK(proc_allgather(c, &ok, oks.data(), sizeof(int)));
  c->peer_ok = true;
  for (int v : oks) c->peer_ok = c->peer_ok && v;
  if (!c->peer_ok) {
    close_ipc(c);
    c->peer_binned.assign((size_t)c->R * 2, nullptr);
    c->peer_in.assign((size_t)c->R, nullptr);
    c->peer_mbox.assign((size_t)c->R, nullptr);
  }
  return upload_in_table(c);
}

static void drop_fwd_graph(Ctx* c);

// Effective control of a multi-process forward (RAFI_OPT_CONTROL): who
// exchanges the counts (a5) and runs the completion barrier.
static int resolve_control(Ctx* c, int want) {
  int x = want;
  const bool peer_possible = c->peer_ok && !c->shared_gpu;
  if (c->nprocs == 1) {
    x = RAFI_CONTROL_AUTO;  // one process: nothing to exchange
  } else if (x == RAFI_CONTROL_AUTO) {
    x = peer_possible ? RAFI_CONTROL_PEER : c->comm ? RAFI_CONTROL_NCCL : RAFI_CONTROL_HOST;
  }
  if (x == RAFI_CONTROL_PEER && !peer_possible) {
    set_error(c->shared_gpu ? "PEER control spins on flags other processes raise: refused when processes share a "
                              "device (no co-residency guarantee); use HOST control"
                            : "PEER control needs every rank's mailbox mapped (CUDA IPC failed)");
    return RAFI_ERR_UNSUPPORTED;
  }
  if (x == RAFI_CONTROL_NCCL && !c->comm) {
    set_error("NCCL control needs an NCCL communicator");
    return RAFI_ERR_UNSUPPORTED;
  }
  if (x == RAFI_CONTROL_HOST && !c->boot.allgather) {
    set_error("HOST control needs a bootstrap all-gather (rafi_create_boot)");
    return RAFI_ERR_UNSUPPORTED;
  }
  c->control = want;
  c->ctl_eff = x;
  c->ctl_peer = x == RAFI_CONTROL_PEER;
  return RAFI_OK;
}

static int resolve_exchange(Ctx* c) {
  int x = c->exchange;
  if (x == RAFI_EXCHANGE_AUTO) x = (c->nprocs == 1 || c->peer_ok) ? RAFI_EXCHANGE_FUSED : RAFI_EXCHANGE_NCCL;
  if ((x == RAFI_EXCHANGE_PEER || x == RAFI_EXCHANGE_FUSED) && !(c->nprocs == 1 || c->peer_ok)) {
    set_error("PEER exchange needs every rank's buffers mapped (CUDA IPC failed)");
    return RAFI_ERR_UNSUPPORTED;
  }
  if (x == RAFI_EXCHANGE_NCCL && c->L != 1) {
    set_error("NCCL exchange supports one local rank per process");
    return RAFI_ERR_UNSUPPORTED;
  }
  if (x == RAFI_EXCHANGE_NCCL && c->nprocs > 1 && !c->comm) {
    set_error("NCCL exchange needs an NCCL communicator");
    return RAFI_ERR_UNSUPPORTED;
  }
  RAFI_CK(resolve_control(c, c->control));
  c->exchange_eff = x;
  return RAFI_OK;
}

// Effective scatter write path (RAFI_OPT_SCATTER).
static constexpr size_t kMaxSmem = 227u * 1024u;  // opt-in shared memory per CTA on sm_100a

static int resolve_scatter(Ctx* c) {
  int x = c->scatter;
  if (x == RAFI_SCATTER_AUTO) {
    // BULK where the scatter pushes runs of 24 B and larger items to NVLink
    // peers in large rounds (measured faster there at N=2 and N=4 by 0-13%,
    // DESIGN.md section 6); THREADS for local HBM (faster at every item size),
    // for 16-B items (N=2: 87 vs 66 G items/s; N=4: 130 vs 133), and for
    // queues below 2^19 items, where the warp tiles' two-kernel forward wins
    // on latency (N=2, 4096 items: 61 vs 66 us blocking, 41 vs 43 us graph)
    const bool remote_push = c->nprocs > 1 && c->exchange_eff == RAFI_EXCHANGE_FUSED;
    x = remote_push && c->B >= 24 && c->cap >= (1ull << 19) && perm_supported(c->B) &&
                perm_smem_bytes(256, c->B, c->R) <= kMaxSmem
            ? RAFI_SCATTER_BULK
            : RAFI_SCATTER_THREADS;
  }
  if (x == RAFI_SCATTER_BULK && !(perm_supported(c->B) && perm_smem_bytes(256, c->B, c->R) <= kMaxSmem)) {
    set_error("permuting scatter needs item_bytes % 4 == 0 and a 256-item tile that fits in shared memory");
    return RAFI_ERR_UNSUPPORTED;
  }
  c->scatter_eff = x;
  return RAFI_OK;
}

static uint32_t auto_tile(const Ctx* c) {
  return c->scatter_eff == RAFI_SCATTER_BULK ? choose_tile_perm(c->B, c->R) : choose_tile(c->B, c->R, c->L);
}

// Binning tile (between rounds); grows H/O when the tile count grows.
static int set_tile(Ctx* c, uint32_t t) {
  if ((uint64_t)(c->cap + t - 1) / t > c->max_tiles) {
    for (auto& r : c->lr) {
      cudaFree(r.H); cudaFree(r.O); r.H = r.O = nullptr;
      const size_t hb = (size_t)((c->cap + t - 1) / t) * c->R * 4 + kPad;
      RAFI_CK(alloc_dev((void**)&r.H, hb));
      RAFI_CK(alloc_dev((void**)&r.O, hb));
    }
    c->max_tiles = (c->cap + t - 1) / t;
    RAFI_CK(upload_rank_table(c));
  }
  c->tile = t;
  return RAFI_OK;
}

// Re-resolve the scatter path (AUTO depends on the exchange) and its tile.
static int refresh_scatter(Ctx* c) {
  RAFI_CK(resolve_scatter(c));
  if (!c->tile_user) RAFI_CK(set_tile(c, auto_tile(c)));
  return RAFI_OK;
}

static int alloc_all(Ctx* c) {
  c->max_tiles = (c->cap + c->tile - 1) / c->tile;
  c->lr.assign(c->L, LocalRank{});
  for (int l = 0; l < c->L; ++l) RAFI_CK(alloc_rank(c, c->lr[l], c->cap));
  RAFI_CK(upload_rank_table(c));
  return RAFI_OK;
}

static void destroy_ctx(Ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  drop_fwd_graph(c);
  if (c->cap_stream) { cudaStreamDestroy(c->cap_stream); c->cap_stream = nullptr; }
  close_ipc(c);
  for (auto& r : c->lr) free_rank(r);
  cudaFree(c->rank_dev); cudaFree(c->ctrl); cudaFree(c->runs_dev); cudaFree(c->plan_dev);
  cudaFree(c->off_dev); cudaFree(c->ovf_dev); cudaFree(c->in_table_dev); cudaFree(c->done_dev);
  cudaFree(c->mbox_table_dev);
  if (c->io_in) {
    cudaStreamSynchronize(c->io_in); cudaStreamSynchronize(c->io_out);
    cudaStreamDestroy(c->io_in); cudaStreamDestroy(c->io_out);
    for (int s = 0; s < 2; ++s) {
      cudaFree(c->stage2[s]); cudaEventDestroy(c->ev_stage_ready[s]); cudaEventDestroy(c->ev_stage_free[s]);
    }
    cudaEventDestroy(c->ev_in_ready); cudaEventDestroy(c->ev_out_done);
  }
  cudaFreeHost(c->ctrl_host); cudaFreeHost(c->runs_host); cudaFreeHost(c->plan_host);
  for (auto& e : c->ev) if (e) cudaEventDestroy(e);
  for (auto& pr : c->ev_emit)
    for (auto& e : pr) if (e) cudaEventDestroy(e);
  cudaGetLastError();
  delete c;
}

static int create(Ctx** out, const rafi_create_params* p, const rafi_bootstrap* boot) {
  *out = nullptr;
  if (!p || p->item_bytes < 1 || p->local_ranks < 1 || p->item_bytes > (1u << 30)) {
    set_error("rafi_create: item_bytes >= 1 and local_ranks >= 1 required");
    return RAFI_ERR_INVALID_ARG;
  }
  if (p->capacity >= (1ull << 32)) {
    set_error("rafi_create: capacity must be < 2^32 items (32-bit index in the sort key, PAPER:109)");
    return RAFI_ERR_INVALID_ARG;
  }
  if (boot && (boot->nprocs < 1 || boot->proc < 0 || boot->proc >= boot->nprocs ||
               (boot->nprocs > 1 && !boot->allgather))) {
    set_error("rafi_create_boot: 0 <= proc < nprocs and an all-gather callback (nprocs > 1) required");
    return RAFI_ERR_INVALID_ARG;
  }
  Ctx* c = new (std::nothrow) Ctx();
  if (!c) return RAFI_ERR_NOMEM;
  int dev = p->device;
  if (dev < 0) {
    if (cudaGetDevice(&dev) != cudaSuccess) { cudaGetLastError(); set_error("no CUDA device"); delete c; return RAFI_ERR_CUDA; }
  }
  c->device = dev;
  int rc = RAFI_OK;
  auto fail = [&](int r) { destroy_ctx(c); return r; };
  if (cudaSetDevice(dev) != cudaSuccess) { cudaGetLastError(); set_error("cudaSetDevice failed"); return fail(RAFI_ERR_CUDA); }
  c->stream = (cudaStream_t)p->stream;
  c->comm = (ncclComm_t)p->nccl_comm;
  if (c->comm) {
    int n = 1, r = 0;
    if (ncclCommCount(c->comm, &n) != ncclSuccess || ncclCommUserRank(c->comm, &r) != ncclSuccess) {
      set_error("ncclCommCount/UserRank failed");
      return fail(RAFI_ERR_NCCL);
    }
    c->nprocs = n; c->proc = r;
  }
  if (boot) {
    if (c->comm && (boot->nprocs != c->nprocs || boot->proc != c->proc)) {
      set_error("rafi_create_boot: the bootstrap and the NCCL communicator describe different groups");
      return fail(RAFI_ERR_INVALID_ARG);
    }
    c->boot = *boot;
    c->nprocs = boot->nprocs;
    c->proc = boot->proc;
  }
  c->L = p->local_ranks;
  c->R = c->nprocs * c->L;
  c->B = p->item_bytes;
  c->cap = p->capacity;
  if ((rc = resolve_scatter(c))) return fail(rc);
  c->tile = auto_tile(c);
  if ((rc = alloc_dev((void**)&c->rank_dev, sizeof(RankDev) * c->L))) return fail(rc);
  if ((rc = alloc_dev((void**)&c->ctrl, ctrl_c_bytes(c)))) return fail(rc);
  c->Cdev = reinterpret_cast<uint64_t*>(c->ctrl + c->L);  // count matrix right after the control blocks
  if ((rc = alloc_dev((void**)&c->runs_dev, sizeof(CopyRun) * c->L * c->R))) return fail(rc);
  if ((rc = alloc_dev((void**)&c->plan_dev, sizeof(uint64_t) * c->L))) return fail(rc);
  if ((rc = alloc_dev((void**)&c->off_dev, sizeof(uint64_t) * c->L * c->R))) return fail(rc);
  if ((rc = alloc_dev((void**)&c->ovf_dev, 2 * sizeof(int)))) return fail(rc);
  if ((rc = alloc_dev((void**)&c->done_dev, 2 * sizeof(unsigned)))) return fail(rc);
  if ((rc = alloc_dev((void**)&c->in_table_dev, sizeof(uint8_t*) * c->R))) return fail(rc);
  if ((rc = alloc_dev((void**)&c->mbox_table_dev, sizeof(void*) * c->nprocs))) return fail(rc);
  if (cudaMallocHost((void**)&c->ctrl_host, ctrl_c_bytes(c)) != cudaSuccess ||
      cudaMallocHost((void**)&c->runs_host, sizeof(CopyRun) * c->L * c->R) != cudaSuccess ||
      cudaMallocHost((void**)&c->plan_host, sizeof(uint64_t) * c->L) != cudaSuccess) {
    cudaGetLastError();
    set_error("cudaMallocHost failed");
    return fail(RAFI_ERR_NOMEM);
  }
  c->Chost = reinterpret_cast<uint64_t*>(c->ctrl_host + c->L);
  if (cudaMemsetAsync(c->ctrl, 0, ctrl_c_bytes(c), c->stream) != cudaSuccess ||
      cudaMemsetAsync(c->ovf_dev, 0, 2 * sizeof(int), c->stream) != cudaSuccess ||
      cudaMemsetAsync(c->done_dev, 0, 2 * sizeof(unsigned), c->stream) != cudaSuccess ||
      false) {
    cudaGetLastError(); set_error("cudaMemsetAsync failed"); return fail(RAFI_ERR_CUDA);
  }
  for (auto& e : c->ev)
    if (cudaEventCreate(&e) != cudaSuccess) { cudaGetLastError(); set_error("cudaEventCreate"); return fail(RAFI_ERR_CUDA); }
  for (auto& pr : c->ev_emit)
    for (auto& e : pr)
      if (cudaEventCreate(&e) != cudaSuccess) { cudaGetLastError(); set_error("cudaEventCreate"); return fail(RAFI_ERR_CUDA); }
  if ((rc = alloc_all(c))) return fail(rc);
  if ((rc = exchange_peer_pointers(c))) return fail(rc);
  if ((rc = resolve_exchange(c))) return fail(rc);
  if ((rc = refresh_scatter(c))) return fail(rc);
  if (cudaStreamSynchronize(c->stream) != cudaSuccess) { cudaGetLastError(); set_error("sync"); return fail(RAFI_ERR_CUDA); }
  *out = c;
  return RAFI_OK;
}

// ------------------------------------------------------------------ forward

static float ev_ms(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0.f;
  if (cudaEventElapsedTime(&ms, a, b) != cudaSuccess) { cudaGetLastError(); return 0.f; }
  return ms;
}

// Host bookkeeping from the mirrored count matrix and control blocks.
// Returns 1 if some rank would receive more than its capacity (Z3).
static int book_keep(Ctx* c, uint64_t* G_out) {
  const int R = c->R, L = c->L;
  uint64_t G = 0;
  int overflow = 0;
  for (int e = 0; e < R; ++e) {
    uint64_t col = 0;
    for (int s = 0; s < R; ++s) col += c->Chost[(size_t)s * R + e];
    if (col > c->cap) overflow = 1;
    G += col;
  }
  *G_out = G;
  if (overflow) return 1;
  for (int l = 0; l < L; ++l) {
    const int g = c->proc * L + l;
    LocalRank& r = c->lr[l];
    uint64_t tot = 0, sent = 0, recv = 0;
    for (int s = 0; s < R; ++s) {
      const uint64_t in_c = c->Chost[(size_t)s * R + g];
      tot += in_c;
      if (s != g) { recv += in_c * c->B; sent += c->Chost[(size_t)g * R + s] * c->B; }
    }
    r.num_in = tot;
    r.n_out = c->ctrl_host[l].n_out;
    r.dropped = c->ctrl_host[l].dropped;
    r.invalid = c->ctrl_host[l].invalid_last;
    r.sent_remote = sent;
    r.recv_remote = recv;
  }
  return 0;
}

// FUSED forward: counts first, then one kernel bins and pushes every run
// straight into its destination's incoming queue (NEXT-1 of SURVEY §8(f)).
//   hist -> scan -> [all-gather counts] -> plan -> scatter+push -> [barrier] -> wrap-up
// Phase event i on the context stream (timed forwards launch directly, not
// from the cached graph: event record nodes inside a graph cost ~4 us each).
static cudaError_t record_ev(Ctx* c, int i) { return cudaEventRecord(c->ev[i], c->stream); }

static int enqueue_fused(Ctx* c, unsigned long long* G_dev, bool T) {
  const int R = c->R, L = c->L;
  c->fwd_launches = 0;
  if (T) RAFI_CK_CUDA(record_ev(c, 0));
  // a3 (+ a5's plan when this process holds every rank: the scan's last block
  // plans; with peer control it first exchanges the counts through the
  // mailboxes, so one kernel does scan + count exchange + plan -- on small
  // warp-tile forwards the histogram's last CTA does all of it)
  const bool peer = c->nprocs > 1 && c->ctl_peer;
  const int pm = (c->nprocs == 1 || peer) ? 2 : 0;
  RAFI_CK(launch_hist(c, pm, G_dev, peer));
  if (T) RAFI_CK_CUDA(record_ev(c, 1));
  RAFI_CK(launch_scan(c, pm, G_dev, peer));
  if (T) RAFI_CK_CUDA(record_ev(c, 2));
  if (c->nprocs > 1 && !peer) {
    // a5: the whole R x R matrix on every rank; offsets + overflow on device
    RAFI_CK_NCCL(ncclAllGather(c->Cdev + (size_t)c->proc * L * R, c->Cdev, (size_t)L * R, ncclUint64, c->comm,
                               c->stream));
    RAFI_CK(launch_plan(c, true, G_dev));
  }
  if (T) RAFI_CK_CUDA(record_ev(c, 3));
  // a4 + a6: stable scatter, each destination run written into its receiver's
  // queue; a7 wrap-up by its last block (skipped on overflow), and with peer
  // control the completion barrier after it
  c->scatter_barrier = peer;
  const int rc = launch_scatter(c, true, true);
  c->scatter_barrier = false;
  RAFI_CK(rc);
  if (T) RAFI_CK_CUDA(record_ev(c, 4));
  // every push has landed before any rank's next app kernel reads its queue:
  // the all-reduce completes only after every rank's scatter kernel completed
  if (c->nprocs > 1 && !peer)
    RAFI_CK_NCCL(ncclAllReduce(c->ovf_dev + 1, c->ovf_dev + 1, 1, ncclInt32, ncclMax, c->comm, c->stream));
  if (T) RAFI_CK_CUDA(record_ev(c, 5));
  if (T) RAFI_CK_CUDA(record_ev(c, 6));
  return RAFI_OK;
}

static void mark_timing(Ctx* c, bool fused);

// After the mirrored control blocks and count matrix reached the host: a
// peer-control timeout (flagged by the kernels), else the bookkeeping and the
// collective receive-overflow decision (Z3).
static int finish_host(Ctx* c, uint64_t* G) {
  c->host_stale = false;
  if (c->ctrl_host[0].status) {
    c->broken = true;
    set_error("peer control: a mailbox wait exceeded RAFI_OPT_PEER_TIMEOUT_MS (some process never arrived)");
    return RAFI_ERR_TIMEOUT;
  }
  if (book_keep(c, G)) {
    c->broken = true;
    set_error("receive overflow: some rank would receive more than its capacity");
    return RAFI_ERR_RECV_OVERFLOW;
  }
  return RAFI_OK;
}

// Host refresh after device work: count matrix + counters -> host bookkeeping.
static int refresh_host(Ctx* c, uint64_t* G) {
  // control blocks and count matrix are one allocation: one copy back
  RAFI_CK_CUDA(cudaMemcpyAsync(c->ctrl_host, c->ctrl, ctrl_c_bytes(c), cudaMemcpyDeviceToHost, c->stream));
  RAFI_CK_CUDA(cudaStreamSynchronize(c->stream));
  return finish_host(c, G);
}

// Count exchange on the host (a5 as the paper does it): after the
// scan, copy this process's L count rows to the host, all-gather them over
// the process group into the mirrored R x R matrix, and (to_dev) upload the
// whole matrix for the device-side plan.  Blocking.
static int host_count_exchange(Ctx* c, bool to_dev) {
  const size_t rows = (size_t)c->L * c->R;
  RAFI_CK_CUDA(cudaMemcpyAsync(c->ctrl_host, c->ctrl, ctrl_c_bytes(c), cudaMemcpyDeviceToHost, c->stream));
  RAFI_CK_CUDA(cudaStreamSynchronize(c->stream));
  std::vector<uint64_t> mine(c->Chost + c->proc * rows, c->Chost + (c->proc + 1) * rows);
  RAFI_CK(proc_allgather(c, mine.data(), c->Chost, rows * sizeof(uint64_t)));  // process-major = rank-major
  if (to_dev)
    RAFI_CK_CUDA(cudaMemcpyAsync(c->Cdev, c->Chost, sizeof(uint64_t) * c->R * c->R, cudaMemcpyHostToDevice,
                                 c->stream));
  return RAFI_OK;
}

// FUSED forward under HOST control: no kernel waits on another process.
//   hist -> scan -> D2H rows, host all-gather, H2D matrix -> plan ->
//   scatter+push -> stream sync -> host barrier
static int64_t forward_fused_host(Ctx* c) {
  const bool T = c->timing;
  c->fwd_launches = 0;
  if (T) RAFI_CK_CUDA(record_ev(c, 0));
  RAFI_CK(launch_hist(c, 0, nullptr, false));
  if (T) RAFI_CK_CUDA(record_ev(c, 1));
  RAFI_CK(launch_scan(c, 0, nullptr, false));
  if (T) RAFI_CK_CUDA(record_ev(c, 2));
  RAFI_CK(host_count_exchange(c, true));
  RAFI_CK(launch_plan(c, true, nullptr));  // offsets, num_in, and ovf (identical on every rank)
  if (T) RAFI_CK_CUDA(record_ev(c, 3));
  uint64_t G = 0;
  int rc = finish_host(c, &G);  // overflow: the scatter below moves nothing (ovf), every rank errs alike
  RAFI_CK(launch_scatter(c, true, true));
  if (T) RAFI_CK_CUDA(record_ev(c, 4));
  RAFI_CK_CUDA(cudaStreamSynchronize(c->stream));
  // completion barrier: every process's pushes have landed once all arrive
  RAFI_CK(proc_barrier(c));
  if (T) {
    RAFI_CK_CUDA(record_ev(c, 5));
    RAFI_CK_CUDA(record_ev(c, 6));
  }
  if (rc != RAFI_OK) return rc;
  if (T) mark_timing(c, true);
  c->last_fused = true;
  c->round += 1;
  c->last_G = (int64_t)G;
  return (int64_t)G;
}

// Phase timings are read lazily -- at the next forward or stats read, off the
// critical path -- and summed over every timed forward / bulk emit since
// RAFI_OPT_TIMING was set.
static void collect_timing(Ctx* c) {
  if (!c->timing_unread) return;
  c->timing_unread = false;
  cudaEventSynchronize(c->ev[6]);
  rafi_stats& s = c->st;
  if (c->unread_fused) {
    s.ms_hist = ev_ms(c->ev[0], c->ev[1]);
    s.ms_scan = ev_ms(c->ev[1], c->ev[2]);
    s.ms_count_exchange = ev_ms(c->ev[2], c->ev[3]);
    s.ms_scatter = ev_ms(c->ev[3], c->ev[4]);
    s.ms_payload_exchange = ev_ms(c->ev[4], c->ev[5]);  // the completion barrier
    s.ms_wrapup = ev_ms(c->ev[5], c->ev[6]);
  } else {
    s.ms_hist = ev_ms(c->ev[0], c->ev[1]);
    s.ms_scan = ev_ms(c->ev[1], c->ev[2]);
    s.ms_scatter = ev_ms(c->ev[2], c->ev[3]);
    s.ms_count_exchange = ev_ms(c->ev[3], c->ev[4]);
    s.ms_payload_exchange = ev_ms(c->ev[7], c->ev[5]);
    s.ms_wrapup = ev_ms(c->ev[5], c->ev[6]);
  }
  s.ms_total = ev_ms(c->ev[0], c->ev[6]);
  s.acc_ms_hist += s.ms_hist;
  s.acc_ms_scan += s.ms_scan;
  s.acc_ms_scatter += s.ms_scatter;
  s.acc_ms_count_exchange += s.ms_count_exchange;
  s.acc_ms_payload_exchange += s.ms_payload_exchange;
  s.acc_ms_wrapup += s.ms_wrapup;
  s.acc_ms_total += s.ms_total;
  s.acc_forwards += 1;
  while (c->emit_head != c->emit_mark) {  // emits enqueued before that forward: complete
    s.acc_ms_emit += ev_ms(c->ev_emit[c->emit_head][0], c->ev_emit[c->emit_head][1]);
    s.acc_emits += 1;
    c->emit_head = (c->emit_head + 1) % Ctx::kEmitEv;
  }
}

static void mark_timing(Ctx* c, bool fused) {
  c->timing_unread = true;
  c->unread_fused = fused;
  c->emit_mark = c->emit_tail;
}

static void drop_fwd_graph(Ctx* c) {
  if (c->fwd_exec) { cudaGraphExecDestroy(c->fwd_exec); c->fwd_exec = nullptr; }
  c->fwd_dirty = true;
}

// Capture [enqueue_fused + read-back of counters and count matrix] on a
// private stream into a graph; its kernels are counted at every replay.
static int build_fwd_graph(Ctx* c, bool T) {
  drop_fwd_graph(c);
  if (!c->cap_stream) RAFI_CK_CUDA(cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking));
  cudaStream_t user = c->stream;
  const uint64_t l0 = c->launches;
  RAFI_CK_CUDA(cudaStreamBeginCapture(c->cap_stream, cudaStreamCaptureModeRelaxed));
  c->stream = c->cap_stream;
  int rc = enqueue_fused(c, nullptr, T);
  if (rc == RAFI_OK &&
      cudaMemcpyAsync(c->ctrl_host, c->ctrl, ctrl_c_bytes(c), cudaMemcpyDeviceToHost, c->stream) != cudaSuccess) {
    set_error("cudaMemcpyAsync (capture)");
    rc = RAFI_ERR_CUDA;
  }
  c->stream = user;
  cudaGraph_t g = nullptr;
  const cudaError_t e = cudaStreamEndCapture(c->cap_stream, &g);
  if (rc == RAFI_OK && e != cudaSuccess) { set_error(std::string("cudaStreamEndCapture: ") + cudaGetErrorString(e)); rc = RAFI_ERR_CUDA; }
  if (rc == RAFI_OK && cudaGraphInstantiate(&c->fwd_exec, g, 0) != cudaSuccess) {
    set_error("cudaGraphInstantiate (forward)");
    c->fwd_exec = nullptr;
    rc = RAFI_ERR_CUDA;
  }
  if (g) cudaGraphDestroy(g);
  cudaGetLastError();
  c->fwd_graph_launches = c->launches - l0;
  c->launches = l0;
  if (rc != RAFI_OK) return rc;
  c->fwd_dirty = false;
  c->fwd_T = T;
  return RAFI_OK;
}

static int64_t forward_fused(Ctx* c) {
  if (c->nprocs > 1 && c->ctl_eff == RAFI_CONTROL_HOST) return forward_fused_host(c);
  const bool T = c->timing;
  uint64_t G = 0;
  if (c->fwd_graph && !T) {
    // one graph launch instead of 3-6 launches and a copy: what a small,
    // latency-bound round costs on the host.  Timed forwards (RAFI_OPT_TIMING)
    // launch directly, with their events between the launches.
    if (c->fwd_dirty || !c->fwd_exec || c->fwd_T != T) RAFI_CK(build_fwd_graph(c, T));
    RAFI_CK_CUDA(cudaGraphLaunch(c->fwd_exec, c->stream));
    c->launches += c->fwd_graph_launches;
    c->fwd_launches = c->fwd_graph_launches;
    RAFI_CK_CUDA(cudaStreamSynchronize(c->stream));
    RAFI_CK(finish_host(c, &G));
  } else {
    RAFI_CK(enqueue_fused(c, nullptr, T));
    RAFI_CK(refresh_host(c, &G));
  }
  if (T) mark_timing(c, true);
  c->last_fused = true;
  c->round += 1;
  c->last_G = (int64_t)G;  // a8
  return (int64_t)G;
}

static int64_t forward_staged(Ctx* c) {
  const int R = c->R, L = c->L;
  const uint64_t B = c->B;
  c->fwd_launches = 0;
  const bool T = c->timing;
  if (T) RAFI_CK_CUDA(cudaEventRecord(c->ev[0], c->stream));
  // a2-a4: bin every local rank's outgoing batch by destination
  RAFI_CK(launch_hist(c, 1));
  if (T) RAFI_CK_CUDA(cudaEventRecord(c->ev[1], c->stream));
  RAFI_CK(launch_scan(c, 1));  // + the send offsets, by the scan's last block
  if (T) RAFI_CK_CUDA(cudaEventRecord(c->ev[2], c->stream));
  RAFI_CK(launch_scatter(c, false, false));
  if (T) RAFI_CK_CUDA(cudaEventRecord(c->ev[3], c->stream));
  // a5: every process learns the whole R x R count matrix.  The all-gather is
  // ordered after each process's scatter on its stream, so once it completes
  // every rank's send batch is final (what the PEER pull relies on).
  if (c->nprocs > 1 && c->comm) {
    RAFI_CK_NCCL(ncclAllGather(c->Cdev + (size_t)c->proc * L * R, c->Cdev, (size_t)L * R, ncclUint64, c->comm,
                               c->stream));
    RAFI_CK_CUDA(cudaMemcpyAsync(c->ctrl_host, c->ctrl, ctrl_c_bytes(c), cudaMemcpyDeviceToHost, c->stream));
  } else if (c->nprocs > 1) {
    // no communicator: the rows go through the bootstrap's host all-gather
    // (each process synchronises first, so every send batch is final)
    RAFI_CK(host_count_exchange(c, false));
  } else {
    RAFI_CK_CUDA(cudaMemcpyAsync(c->ctrl_host, c->ctrl, ctrl_c_bytes(c), cudaMemcpyDeviceToHost, c->stream));
  }
  if (T) RAFI_CK_CUDA(cudaEventRecord(c->ev[4], c->stream));
  RAFI_CK_CUDA(cudaStreamSynchronize(c->stream));
  // plan and the collective overflow decision (Z3)
  uint64_t G = 0;
  int overflow = 0;
  for (int e = 0; e < R; ++e) {
    uint64_t col = 0;
    for (int s = 0; s < R; ++s) col += c->Chost[(size_t)s * R + e];
    if (col > c->cap) overflow = 1;
    G += col;
  }
  if (overflow) {
    c->broken = true;
    set_error("receive overflow: some rank would receive more than its capacity");
    return RAFI_ERR_RECV_OVERFLOW;
  }
  std::vector<uint64_t> recv_cnt(R), recv_off(R), src_off(R);
  for (int l = 0; l < L; ++l) {
    const int g = c->proc * L + l;
    uint64_t tot = 0;
    rafi_plan(R, c->Chost, c->cap, g, recv_cnt.data(), recv_off.data(), src_off.data(), &tot, nullptr, nullptr);
    c->plan_host[l] = tot;
    LocalRank& r = c->lr[l];
    r.num_in = tot;
    r.n_out = c->ctrl_host[l].n_out;
    r.dropped = c->ctrl_host[l].dropped;
    r.invalid = c->ctrl_host[l].invalid_last;
    uint64_t sent = 0, recv = 0;
    for (int s = 0; s < R; ++s) {
      if (s != g) {
        sent += c->Chost[(size_t)g * R + s] * B;
        recv += recv_cnt[s] * B;
      }
      CopyRun& run = c->runs_host[(size_t)l * R + s];
      run.src = c->peer_binned.empty() ? nullptr : c->peer_binned[(size_t)s * 2 + c->cur] + src_off[s] * B;
      run.dst = recv_off[s];
      run.count = recv_cnt[s];
    }
    r.sent_remote = sent;
    r.recv_remote = recv;
  }
  RAFI_CK_CUDA(cudaMemcpyAsync(c->plan_dev, c->plan_host, sizeof(uint64_t) * L, cudaMemcpyHostToDevice, c->stream));
  // a6: payload exchange
  if (T) RAFI_CK_CUDA(cudaEventRecord(c->ev[7], c->stream));
  if (c->exchange_eff == RAFI_EXCHANGE_PEER) {
    RAFI_CK_CUDA(cudaMemcpyAsync(c->runs_dev, c->runs_host, sizeof(CopyRun) * L * R, cudaMemcpyHostToDevice,
                                 c->stream));
    uint64_t maxb = 0;
    for (int l = 0; l < L; ++l) maxb = std::max<uint64_t>(maxb, c->plan_host[l] * B);
    const int chunks = (int)std::min<uint64_t>((maxb + 65535) / 65536, 1u << 30);
    if (maxb) RAFI_CK(launch_copy(c, chunks));
  } else {  // NCCL grouped send/recv (one local rank per process)
    const int me = c->proc;
    uint8_t* sb = c->lr[0].binned[c->cur];
    uint8_t* ib = c->lr[0].in;
    rafi_plan(R, c->Chost, c->cap, me, recv_cnt.data(), recv_off.data(), nullptr, nullptr, nullptr, nullptr);
    uint64_t soff = 0;
    RAFI_CK_NCCL(ncclGroupStart());
    for (int p = 0; p < R; ++p) {
      const uint64_t sc = c->Chost[(size_t)me * R + p];
      if (p == me) {
        if (sc) {
          cudaError_t e = cudaMemcpyAsync(ib + recv_off[me] * B, sb + soff * B, sc * B, cudaMemcpyDeviceToDevice, c->stream);
          if (e != cudaSuccess) { ncclGroupEnd(); RAFI_CK_CUDA(e); }
        }
      } else {
        if (sc) RAFI_CK_NCCL(ncclSend(sb + soff * B, sc * B, ncclUint8, p, c->comm, c->stream));
        if (recv_cnt[p]) RAFI_CK_NCCL(ncclRecv(ib + recv_off[p] * B, recv_cnt[p] * B, ncclUint8, p, c->comm, c->stream));
      }
      soff += sc;
    }
    RAFI_CK_NCCL(ncclGroupEnd());
  }
  if (T) RAFI_CK_CUDA(cudaEventRecord(c->ev[5], c->stream));
  // a7: wrap-up: counters to 0, numIncoming = received
  RAFI_CK(launch_wrapup(c));
  if (T) {
    RAFI_CK_CUDA(cudaEventRecord(c->ev[6], c->stream));
    mark_timing(c, false);
  }
  c->last_cur = c->cur;
  c->last_fused = false;
  if (double_buffered(c)) c->cur ^= 1;
  c->round += 1;
  c->last_G = (int64_t)G;  // a8: sum of all received counts, same on every rank
  return (int64_t)G;
}

static bool capturing(cudaStream_t s) {
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &st) != cudaSuccess) { cudaGetLastError(); return false; }
  return st != cudaStreamCaptureStatusNone;
}

// An asynchronous read of the incoming queue (rafi_read_incoming_async) must
// land before a forward rewrites the queue: the context stream waits for it
// in stream order.  While the stream is being captured (a user-level capture
// that did not go through rafi_capture_begin) an event recorded outside the
// capture cannot be waited on, so the host waits instead.
static int wait_pending_reads(Ctx* c) {
  if (!c->out_pending) return RAFI_OK;
  if (capturing(c->stream)) RAFI_CK_CUDA(cudaStreamSynchronize(c->io_out));
  else RAFI_CK_CUDA(cudaStreamWaitEvent(c->stream, c->ev_out_done, 0));
  c->out_pending = false;
  return RAFI_OK;
}

static int64_t forward(Ctx* c) {
  if (c->broken) { set_error("context unusable after an earlier collective error"); return RAFI_ERR_STATE; }
  RAFI_CK_CUDA(cudaSetDevice(c->device));
  collect_timing(c);  // the previous forward's events, before they are re-recorded
  RAFI_CK(wait_pending_reads(c));
  return c->exchange_eff == RAFI_EXCHANGE_FUSED ? forward_fused(c) : forward_staged(c);
}

// Copy streams for host I/O (rafi_emit_bulk from host memory, asynchronous
// read-back), created on first use.
static int ensure_io(Ctx* c) {
  if (c->io_in) return RAFI_OK;
  RAFI_CK_CUDA(cudaStreamCreateWithFlags(&c->io_in, cudaStreamNonBlocking));
  RAFI_CK_CUDA(cudaStreamCreateWithFlags(&c->io_out, cudaStreamNonBlocking));
  for (int s = 0; s < 2; ++s) {
    RAFI_CK_CUDA(cudaEventCreateWithFlags(&c->ev_stage_ready[s], cudaEventDisableTiming));
    RAFI_CK_CUDA(cudaEventCreateWithFlags(&c->ev_stage_free[s], cudaEventDisableTiming));
  }
  RAFI_CK_CUDA(cudaEventCreateWithFlags(&c->ev_in_ready, cudaEventDisableTiming));
  RAFI_CK_CUDA(cudaEventCreateWithFlags(&c->ev_out_done, cudaEventDisableTiming));
  return RAFI_OK;
}

static bool bad_local(const Ctx* c, int local) { return !c || local < 0 || local >= c->L; }

static bool is_device_ptr(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) { cudaGetLastError(); return false; }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

}  // namespace rafi_impl

using namespace rafi_impl;

extern "C" {

int rafi_abi_version(void) { return RAFI_ABI_VERSION; }

const char* rafi_last_error(void) { return g_last_error.c_str(); }

const char* rafi_status_str(int s) {
  switch (s) {
    case RAFI_OK: return "RAFI_OK";
    case RAFI_ERR_INVALID_ARG: return "RAFI_ERR_INVALID_ARG";
    case RAFI_ERR_CUDA: return "RAFI_ERR_CUDA";
    case RAFI_ERR_NCCL: return "RAFI_ERR_NCCL";
    case RAFI_ERR_NOMEM: return "RAFI_ERR_NOMEM";
    case RAFI_ERR_RECV_OVERFLOW: return "RAFI_ERR_RECV_OVERFLOW";
    case RAFI_ERR_STATE: return "RAFI_ERR_STATE";
    case RAFI_ERR_UNSUPPORTED: return "RAFI_ERR_UNSUPPORTED";
    default: return "RAFI_ERR_UNKNOWN";
  }
}

int rafi_create_ex(rafi_ctx** out, const rafi_create_params* p) { return rafi_create_boot(out, p, nullptr); }

int rafi_create_boot(rafi_ctx** out, const rafi_create_params* p, const rafi_bootstrap* boot) {
  if (!out) return RAFI_ERR_INVALID_ARG;
  Ctx* c = nullptr;
  int rc = create(&c, p, boot);
  if (rc != RAFI_OK) return rc;
  // rafi_ctx is never defined: the opaque handle is the Ctx address
  *out = reinterpret_cast<rafi_ctx*>(c);
  return RAFI_OK;
}

int rafi_create(rafi_ctx** out, size_t item_bytes, size_t capacity, void* nccl_comm, void* stream) {
  rafi_create_params p;
  p.item_bytes = item_bytes;
  p.capacity = capacity;
  p.nccl_comm = nccl_comm;
  p.stream = stream;
  p.local_ranks = 1;
  p.device = -1;
  return rafi_create_ex(out, &p);
}

void rafi_destroy(rafi_ctx* ctx) { destroy_ctx(reinterpret_cast<Ctx*>(ctx)); }

int rafi_resize(rafi_ctx* ctx, size_t capacity) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c) return RAFI_ERR_INVALID_ARG;
  if (c->broken) return RAFI_ERR_STATE;
  if (capacity >= (1ull << 32)) { set_error("capacity must be < 2^32"); return RAFI_ERR_INVALID_ARG; }
  RAFI_CK_CUDA(cudaSetDevice(c->device));
  if (c->io_out) RAFI_CK_CUDA(cudaStreamSynchronize(c->io_out));  // pending async reads of the old queues
  RAFI_CK_CUDA(cudaMemcpyAsync(c->ctrl_host, c->ctrl, sizeof(CtrlDev) * c->L, cudaMemcpyDeviceToHost, c->stream));
  RAFI_CK_CUDA(cudaStreamSynchronize(c->stream));
  uint64_t mine[2] = {capacity, 1};
  for (int l = 0; l < c->L; ++l)
    if (c->ctrl_host[l].ctr != 0 || c->ctrl_host[l].invalid != 0) mine[1] = 0;
  // collective decision before anything changes: same capacity everywhere,
  // every outgoing queue empty
  std::vector<uint64_t> all(2 * (size_t)c->nprocs);
  RAFI_CK(proc_allgather(c, mine, all.data(), sizeof(mine)));
  for (int p = 0; p < c->nprocs; ++p) {
    if (!all[2 * p + 1]) {
      set_error("rafi_resize: an outgoing queue is not empty (emits since the last forward)");
      return RAFI_ERR_INVALID_ARG;
    }
    if (all[2 * p] != capacity) {
      set_error("rafi_resize: processes passed different capacities");
      return RAFI_ERR_INVALID_ARG;
    }
  }
  std::vector<LocalRank> old = c->lr;
  const uint64_t keep_cap = c->cap;
  c->cap = capacity;
  c->max_tiles = (c->cap + c->tile - 1) / c->tile;
  c->lr.assign(c->L, LocalRank{});
  int rc = RAFI_OK;
  for (int l = 0; l < c->L && rc == RAFI_OK; ++l) rc = alloc_rank(c, c->lr[l], capacity);
  if (rc != RAFI_OK) {
    for (auto& r : c->lr) free_rank(r);
    c->lr = old; c->cap = keep_cap; c->max_tiles = (c->cap + c->tile - 1) / c->tile;
    return rc;
  }
  for (int l = 0; l < c->L; ++l) {
    const uint64_t keep = std::min<uint64_t>(old[l].num_in, capacity);
    if (keep) RAFI_CK_CUDA(cudaMemcpyAsync(c->lr[l].in, old[l].in, keep * c->B, cudaMemcpyDeviceToDevice, c->stream));
    c->lr[l].num_in = keep;
    c->plan_host[l] = keep;
  }
  RAFI_CK_CUDA(cudaMemcpyAsync(c->plan_dev, c->plan_host, sizeof(uint64_t) * c->L, cudaMemcpyHostToDevice, c->stream));
  RAFI_CK(launch_wrapup(c));
  RAFI_CK_CUDA(cudaStreamSynchronize(c->stream));
  close_ipc(c);
  // peers may still hold CUDA-IPC mappings of the old queues: free them only
  // after every process has closed its own
  RAFI_CK(proc_barrier(c));
  for (auto& r : old) free_rank(r);
  RAFI_CK(upload_rank_table(c));
  c->cur = 0;
  drop_fwd_graph(c);  // captured with the old buffers and grid sizes
  RAFI_CK(exchange_peer_pointers(c));
  RAFI_CK(resolve_exchange(c));
  RAFI_CK(refresh_scatter(c));
  return RAFI_OK;
}

int rafi_get_device_view(const rafi_ctx* ctx, int local, rafi_device_view* v) {
  const Ctx* c = reinterpret_cast<const Ctx*>(ctx);
  if (bad_local(c, local) || !v) return RAFI_ERR_INVALID_ARG;
  const LocalRank& r = c->lr[local];
  std::memset(v, 0, sizeof(*v));
  v->in = r.in;
  v->num_in = r.num_in;
  v->num_in_dev = reinterpret_cast<const uint64_t*>(&c->ctrl[local].num_in);
  v->out = r.out;
  v->dest = r.dest;
  v->ctr = &c->ctrl[local].ctr;
  v->invalid = &c->ctrl[local].invalid;
  v->capacity = c->cap;
  v->item_bytes = (uint32_t)c->B;
  v->num_ranks = c->R;
  v->my_rank = c->proc * c->L + local;
  return RAFI_OK;
}

uint64_t rafi_num_incoming(const rafi_ctx* ctx, int local) {
  const Ctx* c = reinterpret_cast<const Ctx*>(ctx);
  if (bad_local(c, local)) return 0;
  return c->lr[local].num_in;
}

int rafi_emit_bulk(rafi_ctx* ctx, int local, const void* items, const int32_t* dests, uint64_t n) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (bad_local(c, local) || (n && (!items || !dests))) return RAFI_ERR_INVALID_ARG;
  if (c->broken) return RAFI_ERR_STATE;
  if (n == 0) return RAFI_OK;
  RAFI_CK_CUDA(cudaSetDevice(c->device));
  const uint8_t* it = static_cast<const uint8_t*>(items);
  const int32_t* ds = dests;
  // memory type of the two pointers; UVA ranges of host and device memory are
  // disjoint, so the last answer per pointer can be reused (saves two driver
  // queries per call on the hot path)
  auto classify = [&](int k, const void* p) {
    if (c->cls_ptr[k] != p) { c->cls_ptr[k] = p; c->cls_dev[k] = is_device_ptr(p); }
    return c->cls_dev[k];
  };
  const bool dev_items = classify(0, items), dev_dests = classify(1, dests);
  int sslot = -1;
  if (!dev_items || !dev_dests) {
    // host inputs: copied on the copy-in stream into one of two staging
    // buffers, so the copy of batch k+1 overlaps the device work (and the
    // asynchronous read-back) of batch k
    RAFI_CK(ensure_io(c));
    sslot = c->stage_slot ^= 1;
    const size_t ib = (size_t)n * c->B, need = ((ib + 255) & ~(size_t)255) + (size_t)n * 4;
    if (need > c->stage_cap[sslot]) {
      RAFI_CK_CUDA(cudaStreamSynchronize(c->stream));
      RAFI_CK_CUDA(cudaStreamSynchronize(c->io_in));
      cudaFree(c->stage2[sslot]);
      c->stage2[sslot] = nullptr; c->stage_cap[sslot] = 0; c->stage_used[sslot] = false;
      RAFI_CK(alloc_dev((void**)&c->stage2[sslot], need));
      c->stage_cap[sslot] = need;
    }
    if (c->stage_used[sslot]) RAFI_CK_CUDA(cudaStreamWaitEvent(c->io_in, c->ev_stage_free[sslot], 0));
    uint8_t* si = c->stage2[sslot];
    int32_t* sd = reinterpret_cast<int32_t*>(si + ((ib + 255) & ~(size_t)255));
    if (!dev_items) { RAFI_CK_CUDA(cudaMemcpyAsync(si, items, ib, cudaMemcpyHostToDevice, c->io_in)); it = si; }
    if (!dev_dests) { RAFI_CK_CUDA(cudaMemcpyAsync(sd, dests, (size_t)n * 4, cudaMemcpyHostToDevice, c->io_in)); ds = sd; }
    RAFI_CK_CUDA(cudaEventRecord(c->ev_stage_ready[sslot], c->io_in));
    RAFI_CK_CUDA(cudaStreamWaitEvent(c->stream, c->ev_stage_ready[sslot], 0));
  }
  const int slot = c->emit_tail, next = (slot + 1) % Ctx::kEmitEv;
  const bool timed = c->timing && next != c->emit_head;  // ring full: this emit goes untimed
  if (timed) RAFI_CK_CUDA(cudaEventRecord(c->ev_emit[slot][0], c->stream));
  RAFI_CK(launch_emit_bulk(c, local, it, ds, n));
  if (timed) {
    RAFI_CK_CUDA(cudaEventRecord(c->ev_emit[slot][1], c->stream));
    c->emit_tail = next;
  }
  if (sslot >= 0) {  // the staging slot is free again once the emit kernel has read it
    RAFI_CK_CUDA(cudaEventRecord(c->ev_stage_free[sslot], c->stream));
    c->stage_used[sslot] = true;
  }
  return RAFI_OK;
}

int rafi_read_incoming_async(rafi_ctx* ctx, int local, void* dst, uint64_t first, uint64_t count) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (bad_local(c, local) || (count && !dst)) return RAFI_ERR_INVALID_ARG;
  const LocalRank& r = c->lr[local];
  if (first > r.num_in || count > r.num_in - first) return RAFI_ERR_INVALID_ARG;
  if (!count) return RAFI_OK;
  RAFI_CK_CUDA(cudaSetDevice(c->device));
  if (c->stream && capturing(c->stream)) {
    set_error("rafi_read_incoming_async is not capturable");
    return RAFI_ERR_UNSUPPORTED;
  }
  RAFI_CK(ensure_io(c));
  RAFI_CK_CUDA(cudaEventRecord(c->ev_in_ready, c->stream));  // incoming queue final in stream order
  RAFI_CK_CUDA(cudaStreamWaitEvent(c->io_out, c->ev_in_ready, 0));
  RAFI_CK_CUDA(cudaMemcpyAsync(dst, r.in + first * c->B, count * c->B, cudaMemcpyDefault, c->io_out));
  RAFI_CK_CUDA(cudaEventRecord(c->ev_out_done, c->io_out));
  c->out_pending = true;
  return RAFI_OK;
}

int rafi_read_wait(rafi_ctx* ctx) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c) return RAFI_ERR_INVALID_ARG;
  if (c->io_out) RAFI_CK_CUDA(cudaStreamSynchronize(c->io_out));
  return RAFI_OK;
}

int64_t rafi_forward(rafi_ctx* ctx) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c) return RAFI_ERR_INVALID_ARG;
  return forward(c);
}

int rafi_forward_async(rafi_ctx* ctx, unsigned long long* G_dev) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c || !G_dev) return RAFI_ERR_INVALID_ARG;
  if (c->broken) { set_error("context unusable after an earlier collective error"); return RAFI_ERR_STATE; }
  if (c->exchange_eff != RAFI_EXCHANGE_FUSED) {
    set_error("rafi_forward_async needs the FUSED exchange");
    return RAFI_ERR_UNSUPPORTED;
  }
  if (c->nprocs > 1 && c->ctl_eff == RAFI_CONTROL_HOST) {
    set_error("rafi_forward_async needs NCCL or PEER control (HOST control synchronises with the host)");
    return RAFI_ERR_UNSUPPORTED;
  }
  RAFI_CK_CUDA(cudaSetDevice(c->device));
  RAFI_CK(wait_pending_reads(c));
  RAFI_CK(enqueue_fused(c, G_dev, false));
  c->last_fused = true;
  c->host_stale = true;
  c->round += 1;
  return RAFI_OK;
}

int rafi_sync_host(rafi_ctx* ctx) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c) return RAFI_ERR_INVALID_ARG;
  RAFI_CK_CUDA(cudaSetDevice(c->device));
  uint64_t G = 0;
  RAFI_CK(refresh_host(c, &G));
  c->last_G = (int64_t)G;
  return RAFI_OK;
}

int rafi_capture_begin(rafi_ctx* ctx) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c || !c->stream) { set_error("capture needs a non-default context stream"); return RAFI_ERR_INVALID_ARG; }
  RAFI_CK_CUDA(cudaSetDevice(c->device));
  RAFI_CK(wait_pending_reads(c));  // before the capture: ordered ahead of every later replay on this stream
  RAFI_CK_CUDA(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeRelaxed));
  return RAFI_OK;
}

int rafi_capture_end(rafi_ctx* ctx, void** exec) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c || !exec) return RAFI_ERR_INVALID_ARG;
  cudaGraph_t g = nullptr;
  RAFI_CK_CUDA(cudaStreamEndCapture(c->stream, &g));
  cudaGraphExec_t e = nullptr;
  cudaError_t r = cudaGraphInstantiate(&e, g, 0);
  cudaGraphDestroy(g);
  RAFI_CK_CUDA(r);
  *exec = e;
  return RAFI_OK;
}

int rafi_graph_launch(rafi_ctx* ctx, void* exec) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c || !exec) return RAFI_ERR_INVALID_ARG;
  RAFI_CK_CUDA(cudaSetDevice(c->device));
  RAFI_CK(wait_pending_reads(c));  // a replayed forward must not rewrite a queue still being copied out
  RAFI_CK_CUDA(cudaGraphLaunch((cudaGraphExec_t)exec, c->stream));
  c->host_stale = true;
  return RAFI_OK;
}

int rafi_graph_destroy(void* exec) {
  if (exec) RAFI_CK_CUDA(cudaGraphExecDestroy((cudaGraphExec_t)exec));
  return RAFI_OK;
}

int rafi_num_ranks(const rafi_ctx* ctx) { const Ctx* c = reinterpret_cast<const Ctx*>(ctx); return c ? c->R : RAFI_ERR_INVALID_ARG; }
int rafi_local_ranks(const rafi_ctx* ctx) { const Ctx* c = reinterpret_cast<const Ctx*>(ctx); return c ? c->L : RAFI_ERR_INVALID_ARG; }
int rafi_rank_of(const rafi_ctx* ctx, int local) {
  const Ctx* c = reinterpret_cast<const Ctx*>(ctx);
  if (bad_local(c, local)) return RAFI_ERR_INVALID_ARG;
  return c->proc * c->L + local;
}
uint64_t rafi_capacity(const rafi_ctx* ctx) { const Ctx* c = reinterpret_cast<const Ctx*>(ctx); return c ? c->cap : 0; }
uint64_t rafi_item_bytes(const rafi_ctx* ctx) { const Ctx* c = reinterpret_cast<const Ctx*>(ctx); return c ? c->B : 0; }

int rafi_read_incoming(const rafi_ctx* ctx, int local, void* dst, uint64_t first, uint64_t count) {
  const Ctx* c = reinterpret_cast<const Ctx*>(ctx);
  if (bad_local(c, local) || (count && !dst)) return RAFI_ERR_INVALID_ARG;
  const LocalRank& r = c->lr[local];
  if (first > r.num_in || count > r.num_in - first) return RAFI_ERR_INVALID_ARG;
  if (!count) return RAFI_OK;
  RAFI_CK_CUDA(cudaSetDevice(c->device));
  RAFI_CK_CUDA(cudaMemcpyAsync(dst, r.in + first * c->B, count * c->B, cudaMemcpyDefault, c->stream));
  RAFI_CK_CUDA(cudaStreamSynchronize(c->stream));
  return RAFI_OK;
}

int rafi_read_outgoing(const rafi_ctx* ctx, int local, void* items_dst, int32_t* dests_dst, uint64_t* ctr,
                       uint64_t* invalid) {
  const Ctx* c = reinterpret_cast<const Ctx*>(ctx);
  if (bad_local(c, local)) return RAFI_ERR_INVALID_ARG;
  RAFI_CK_CUDA(cudaSetDevice(c->device));
  CtrlDev h;
  RAFI_CK_CUDA(cudaMemcpyAsync(&h, &c->ctrl[local], sizeof(h), cudaMemcpyDeviceToHost, c->stream));
  RAFI_CK_CUDA(cudaStreamSynchronize(c->stream));
  const uint64_t n = std::min<uint64_t>(h.ctr, c->cap);
  if (ctr) *ctr = h.ctr;
  if (invalid) *invalid = h.invalid;
  if (n && items_dst)
    RAFI_CK_CUDA(cudaMemcpyAsync(items_dst, c->lr[local].out, n * c->B, cudaMemcpyDefault, c->stream));
  if (n && dests_dst)
    RAFI_CK_CUDA(cudaMemcpyAsync(dests_dst, c->lr[local].dest, n * 4, cudaMemcpyDefault, c->stream));
  RAFI_CK_CUDA(cudaStreamSynchronize(c->stream));
  return RAFI_OK;
}

int rafi_read_binned(const rafi_ctx* ctx, int local, void* dst, uint64_t count) {
  const Ctx* c = reinterpret_cast<const Ctx*>(ctx);
  if (bad_local(c, local) || (count && !dst)) return RAFI_ERR_INVALID_ARG;
  if (c->last_fused) { set_error("the FUSED exchange writes no send batch"); return RAFI_ERR_UNSUPPORTED; }
  const LocalRank& r = c->lr[local];
  if (count > r.n_out) return RAFI_ERR_INVALID_ARG;
  if (!count) return RAFI_OK;
  RAFI_CK_CUDA(cudaSetDevice(c->device));
  const uint8_t* b = r.binned[c->last_cur] ? r.binned[c->last_cur] : r.binned[0];
  RAFI_CK_CUDA(cudaMemcpyAsync(dst, b, count * c->B, cudaMemcpyDefault, c->stream));
  RAFI_CK_CUDA(cudaStreamSynchronize(c->stream));
  return RAFI_OK;
}

int rafi_get_matrix(const rafi_ctx* ctx, uint64_t* Cm) {
  const Ctx* c = reinterpret_cast<const Ctx*>(ctx);
  if (!c || !Cm) return RAFI_ERR_INVALID_ARG;
  std::memcpy(Cm, c->Chost, sizeof(uint64_t) * c->R * c->R);
  return RAFI_OK;
}

int rafi_get_stats(const rafi_ctx* ctx, int local, rafi_stats* out) {
  const Ctx* c = reinterpret_cast<const Ctx*>(ctx);
  if (bad_local(c, local) || !out) return RAFI_ERR_INVALID_ARG;
  collect_timing(const_cast<Ctx*>(c));  // lazily read the last timed forward (logically const)
  *out = c->st;
  const LocalRank& r = c->lr[local];
  out->round = c->round;
  out->n_out = r.n_out;
  out->dropped = r.dropped;
  out->invalid = r.invalid;
  out->num_in = r.num_in;
  out->bytes_sent_remote = r.sent_remote;
  out->bytes_recv_remote = r.recv_remote;
  out->G = c->last_G;
  out->num_ranks = c->R;
  out->my_rank = c->proc * c->L + local;
  out->kernel_launches = c->launches;
  out->forward_launches = c->fwd_launches;
  return RAFI_OK;
}

int rafi_set_option(rafi_ctx* ctx, int key, long long v) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c) return RAFI_ERR_INVALID_ARG;
  // any option but the timing switch may change what the cached forward graph
  // launches (the graph is only used untimed)
  if (key != RAFI_OPT_TIMING) c->fwd_dirty = true;
  switch (key) {
    case RAFI_OPT_EXCHANGE: {
      if (v < RAFI_EXCHANGE_AUTO || v > RAFI_EXCHANGE_FUSED) return RAFI_ERR_INVALID_ARG;
      const int old = c->exchange;
      c->exchange = (int)v;
      int rc = resolve_exchange(c);
      if (rc != RAFI_OK) { c->exchange = old; resolve_exchange(c); return rc; }
      return refresh_scatter(c);
    }
    case RAFI_OPT_TIMING:
      c->timing = v != 0;
      c->st.acc_ms_emit = c->st.acc_ms_hist = c->st.acc_ms_scan = c->st.acc_ms_scatter = 0;
      c->st.acc_ms_count_exchange = c->st.acc_ms_payload_exchange = c->st.acc_ms_wrapup = c->st.acc_ms_total = 0;
      c->st.acc_forwards = c->st.acc_emits = 0;
      c->emit_head = c->emit_tail = c->emit_mark = 0;
      c->timing_unread = false;
      return RAFI_OK;
    case RAFI_OPT_TILE: {
      // only between rounds with an empty outgoing queue; re-sizes H/O
      // 256 * 2^k; or 128 on the warp-tile path (THREADS, R <= 8, item_bytes % 8 == 0)
      if (v != 0 && (v < 128 || v > 4096 || (v & (v - 1)) != 0)) return RAFI_ERR_INVALID_ARG;
      if (v == 128 && !(c->scatter_eff == RAFI_SCATTER_THREADS && warp_tiles_ok(128, c->B, c->R, c->L)))
        return RAFI_ERR_INVALID_ARG;
      const uint32_t t = v ? (uint32_t)v : auto_tile(c);
      if (c->scatter_eff == RAFI_SCATTER_BULK && perm_smem_bytes(t, c->B, c->R) > kMaxSmem) {
        set_error("tile too large for the permuting scatter's shared memory");
        return RAFI_ERR_UNSUPPORTED;
      }
      RAFI_CK(set_tile(c, t));
      c->tile_user = v != 0;
      return RAFI_OK;
    }
    case RAFI_OPT_SCATTER: {
      if (v < RAFI_SCATTER_AUTO || v > RAFI_SCATTER_BULK) return RAFI_ERR_INVALID_ARG;
      const int old = c->scatter;
      c->scatter = (int)v;
      int rc = resolve_scatter(c);
      if (rc != RAFI_OK) { c->scatter = old; resolve_scatter(c); return rc; }
      if (!c->tile_user) RAFI_CK(set_tile(c, auto_tile(c)));
      return RAFI_OK;
    }
    case RAFI_OPT_SELF_DIRECT: return v == 0 ? RAFI_OK : RAFI_ERR_UNSUPPORTED;
    case RAFI_OPT_FORWARD_GRAPH:
      if (v != 0 && v != 1) return RAFI_ERR_INVALID_ARG;
      c->fwd_graph = v != 0;
      return RAFI_OK;
    case RAFI_OPT_CONTROL: {
      if (v < RAFI_CONTROL_AUTO || v > RAFI_CONTROL_HOST) return RAFI_ERR_INVALID_ARG;
      const int old = c->control;
      const int rc = resolve_control(c, (int)v);
      if (rc != RAFI_OK) { resolve_control(c, old); return rc; }
      return RAFI_OK;
    }
    case RAFI_OPT_PEER_TIMEOUT_MS:
      if (v < 0 || v > 3600000000ll) return RAFI_ERR_INVALID_ARG;
      c->peer_timeout_ns = (uint64_t)v * 1000000ull;
      return RAFI_OK;
    default: return RAFI_ERR_INVALID_ARG;
  }
}

int rafi_get_option(const rafi_ctx* ctx, int key, long long* v) {
  const Ctx* c = reinterpret_cast<const Ctx*>(ctx);
  if (!c || !v) return RAFI_ERR_INVALID_ARG;
  switch (key) {
    case RAFI_OPT_EXCHANGE: *v = c->exchange_eff; return RAFI_OK;
    case RAFI_OPT_TIMING: *v = c->timing; return RAFI_OK;
    case RAFI_OPT_TILE: *v = c->tile; return RAFI_OK;
    case RAFI_OPT_SCATTER: *v = c->scatter_eff; return RAFI_OK;
    case RAFI_OPT_CONTROL: *v = c->ctl_eff; return RAFI_OK;
    case RAFI_OPT_PEER_TIMEOUT_MS: *v = (long long)(c->peer_timeout_ns / 1000000ull); return RAFI_OK;
    case RAFI_OPT_FORWARD_GRAPH: *v = c->fwd_graph; return RAFI_OK;
    case RAFI_OPT_SELF_DIRECT: *v = 0; return RAFI_OK;
    default: return RAFI_ERR_INVALID_ARG;
  }
}

int rafi_selftest_peer_control(int device, int P, int L, int rounds, int absent, long long timeout_ms,
                               uint64_t* bad, uint64_t* timed_out) {
  if (P < 1 || P > 128 || L < 1 || P * L > 1024 || rounds < 1 || absent >= P || timeout_ms < 0 ||
      (absent >= 0 && timeout_ms == 0) || !bad || !timed_out)
    return RAFI_ERR_INVALID_ARG;
  if (device >= 0) RAFI_CK_CUDA(cudaSetDevice(device));
  const int R = P * L;
  const size_t mw = mbox_words(P, R);
  std::vector<unsigned long long*> boxes(P, nullptr);
  unsigned long long** table = nullptr;
  uint64_t* Cs = nullptr;
  unsigned long long* flags = nullptr;  // [P] err, [1] bad
  int rc = RAFI_OK;
  for (int p = 0; p < P && rc == RAFI_OK; ++p) {
    rc = alloc_dev((void**)&boxes[p], mw * sizeof(unsigned long long));
    if (rc == RAFI_OK && cudaMemset(boxes[p], 0, mw * sizeof(unsigned long long)) != cudaSuccess) rc = RAFI_ERR_CUDA;
  }
  if (rc == RAFI_OK) rc = alloc_dev((void**)&table, sizeof(void*) * P);
  if (rc == RAFI_OK) rc = alloc_dev((void**)&Cs, sizeof(uint64_t) * (size_t)P * R * R);
  if (rc == RAFI_OK) rc = alloc_dev((void**)&flags, sizeof(unsigned long long) * (P + 1));
  if (rc == RAFI_OK && (cudaMemcpy(table, boxes.data(), sizeof(void*) * P, cudaMemcpyHostToDevice) != cudaSuccess ||
                        cudaMemset(flags, 0, sizeof(unsigned long long) * (P + 1)) != cudaSuccess))
    rc = RAFI_ERR_CUDA;
  if (rc == RAFI_OK)
    rc = launch_ctl_selftest(table, Cs, P, L, rounds, absent, (unsigned long long)timeout_ms * 1000000ull, flags,
                             flags + P);
  if (rc == RAFI_OK && cudaDeviceSynchronize() != cudaSuccess) { set_error("selftest kernel failed"); rc = RAFI_ERR_CUDA; }
  if (rc == RAFI_OK) {
    std::vector<unsigned long long> h(P + 1);
    if (cudaMemcpy(h.data(), flags, sizeof(unsigned long long) * (P + 1), cudaMemcpyDeviceToHost) != cudaSuccess) {
      rc = RAFI_ERR_CUDA;
    } else {
      *bad = h[P];
      *timed_out = 0;
      for (int p = 0; p < P; ++p) *timed_out += h[p] != 0;
    }
  }
  if (rc == RAFI_ERR_CUDA) cudaGetLastError();
  for (auto* b : boxes) cudaFree(b);
  cudaFree(table); cudaFree(Cs); cudaFree(flags);
  return rc;
}

int rafi_diag_redirect_incoming(rafi_ctx* ctx, int grank, void* queue) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c) return RAFI_ERR_INVALID_ARG;
  const int l = grank - c->proc * c->L;
  if (l < 0 || l >= c->L || ((uintptr_t)queue & 15)) return RAFI_ERR_INVALID_ARG;
  if ((int)c->peer_in.size() != c->R) return RAFI_ERR_UNSUPPORTED;
  RAFI_CK_CUDA(cudaSetDevice(c->device));
  if (queue) {
    cudaPointerAttributes a{};
    RAFI_CK_CUDA(cudaPointerGetAttributes(&a, queue));
    if (a.type != cudaMemoryTypeDevice) return RAFI_ERR_INVALID_ARG;
    if (a.device != c->device) {
      const cudaError_t e = cudaDeviceEnablePeerAccess(a.device, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
      else RAFI_CK_CUDA(e);
    }
  }
  c->peer_in[grank] = queue ? static_cast<uint8_t*>(queue) : c->lr[l].in;
  drop_fwd_graph(c);
  return upload_in_table(c);
}

int rafi_nccl_unique_id(void* id128) {
  if (!id128) return RAFI_ERR_INVALID_ARG;
  ncclUniqueId id;
  RAFI_CK_NCCL(ncclGetUniqueId(&id));
  static_assert(sizeof(id) == 128, "ncclUniqueId size");
  std::memcpy(id128, &id, sizeof(id));
  return RAFI_OK;
}

int rafi_nccl_comm_init(void** comm, int nranks, int rank, const void* id128, int device) {
  if (!comm || !id128 || nranks < 1 || rank < 0 || rank >= nranks) return RAFI_ERR_INVALID_ARG;
  if (device >= 0) RAFI_CK_CUDA(cudaSetDevice(device));
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof(id));
  ncclComm_t c = nullptr;
  RAFI_CK_NCCL(ncclCommInitRank(&c, nranks, id, rank));
  *comm = c;
  return RAFI_OK;
}

int rafi_nccl_comm_destroy(void* comm) {
  if (!comm) return RAFI_OK;
  RAFI_CK_NCCL(ncclCommDestroy((ncclComm_t)comm));
  return RAFI_OK;
}

}  // extern "C"
