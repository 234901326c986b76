// kernels.cu -- the sm_100a kernels of the forwarding hot path.
//
//   k_emit_bulk   a1  bulk emitOutgoing: block-aggregated atomic append
//   k_hist        a2  per-tile per-destination counts (replaces key gen +
//                     radix-sort counting)
//   k_scan        a3  per-destination prefix over tiles and the count-matrix
//                     row (replaces the boundary kernel + D2H + host gap fill,
//                     PAPER:121-124)
//   k_plan        a5  per-destination bases from the count matrix
//   k_scatter     a4  stable scatter into one contiguous block per
//                     destination (replaces the gather), staged
//                     through shared memory so that both the read of the tile
//                     and the write of every destination run are coalesced
//   k_copy        a6  payload exchange as a copy kernel over local or CUDA-IPC
//                     peer pointers (NVLink), the PEER transport
//   k_wrapup      a7  reset counters, publish numIncoming
//
// None of this is a dense contraction: all kernels are HBM/NVLink-bound byte
// movers (no tensor cores).  See DESIGN.md for the rooflines.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "devcommon.cuh"
#include "internal.h"

namespace rafi_impl {

// Scatter tuning: units in flight per thread (build-time; see
// paper_2605_30294_b200/build.py variants).  Resident CTAs per SM and the
// per-CTA shared-memory budget depend on the item size (scatter_minb).
#ifndef RAFI_SCATTER_ILP
#define RAFI_SCATTER_ILP 4
#endif



constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxK = 16;          // items per thread per tile (tile <= 4096)
constexpr int kEmitK = 8;          // emit tile = 2048 items
constexpr int kEmitTile = kThreads * kEmitK;

// Map a flat tile index over all local ranks to (local rank, tile).
__device__ __forceinline__ bool tile_of(uint64_t g, const CtrlDev* ctrl, int L, uint64_t cap, uint32_t T,
                                        int* l_out, uint64_t* t_out, uint64_t* n_out, uint64_t* tiles_out) {
  uint64_t acc = 0;
  for (int l = 0; l < L; ++l) {
    uint64_t n = n_items(ctrl[l], cap);
    uint64_t tl = (n + T - 1) / T;
    if (g < acc + tl) {
      *l_out = l; *t_out = g - acc; *n_out = n; *tiles_out = tl;
      return true;
    }
    acc += tl;
  }
  return false;
}

// ---------------------------------------------------------------- a1 emit

template <typename U>
__global__ void __launch_bounds__(kThreads)
k_emit_bulk(const uint8_t* __restrict__ items, const int32_t* __restrict__ dests, uint64_t n,
            uint8_t* __restrict__ out, int32_t* __restrict__ qdest, CtrlDev* ctrl, int R, uint64_t cap,
            uint32_t B, uint32_t UPI, FastDiv divU) {
  __shared__ uint16_t src_of[kEmitTile];
  __shared__ uint32_t wtot[kWarps], wbase[kWarps];
  __shared__ unsigned long long sbase;
  __shared__ uint32_t snvalid;
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const U* itemsU = reinterpret_cast<const U*>(items);
  U* outU = reinterpret_cast<U*>(out);
  // the next tile's destinations are loaded while this tile's items move
  int dnext[kEmitK];
  auto load_dests = [&](uint64_t g) {
#pragma unroll
    for (int k = 0; k < kEmitK; ++k) {
      const uint64_t i = g * kEmitTile + w * 32 * kEmitK + k * 32 + lane;
      dnext[k] = i < n ? dests[i] : -1;
    }
  };
  load_dests(blockIdx.x);
  for (uint64_t g = blockIdx.x; g * kEmitTile < n; g += gridDim.x) {
    const uint64_t t0 = g * kEmitTile;
    const uint32_t nt = (uint32_t)umin64(kEmitTile, n - t0);
    int dk[kEmitK];
    uint32_t rk[kEmitK];
    uint32_t run = 0;
#pragma unroll
    for (int k = 0; k < kEmitK; ++k) {
      const uint32_t il = w * 32 * kEmitK + k * 32 + lane;
      int d = il < nt ? dnext[k] : -1;
      const bool valid = il < nt && (unsigned)d < (unsigned)R;
      const unsigned b = __ballot_sync(kFull, valid);
      dk[k] = valid ? d : -1;
      rk[k] = run + __popc(b & lanemask_lt());
      run += __popc(b);
    }
    if (lane == 0) wtot[w] = run;
    __syncthreads();
    if (tid == 0) {
      uint32_t acc = 0;
      for (int i = 0; i < kWarps; ++i) { wbase[i] = acc; acc += wtot[i]; }
      snvalid = acc;
      sbase = acc ? atomicAdd(&ctrl->ctr, (unsigned long long)acc) : 0ull;
      if (nt > acc) atomicAdd(&ctrl->invalid, (unsigned long long)(nt - acc));
    }
    __syncthreads();
    const unsigned long long base = sbase;
    const uint32_t nvalid = snvalid;
#pragma unroll
    for (int k = 0; k < kEmitK; ++k) {
      if (dk[k] >= 0) {
        const uint32_t p = wbase[w] + rk[k];
        src_of[p] = (uint16_t)(w * 32 * kEmitK + k * 32 + lane);
        if (base + p < cap) qdest[base + p] = dk[k];
      }
    }
    __syncthreads();
    const uint32_t nkeep = base >= cap ? 0u : (uint32_t)umin64(nvalid, cap - base);
    load_dests(g + gridDim.x);
    if (nvalid == nt) {
      // every destination valid (the common case): slot order = tile order,
      // one contiguous span, 4 independent units in flight per thread
      const U* sp = itemsU + t0 * UPI;
      U* dp = outU + base * UPI;
      const uint32_t units = nkeep * UPI;
      uint32_t x = tid;
      for (; x + 3 * kThreads < units; x += 4 * kThreads) {
        const U a = sp[x], b = sp[x + kThreads], c = sp[x + 2 * kThreads], d = sp[x + 3 * kThreads];
        dp[x] = a; dp[x + kThreads] = b; dp[x + 2 * kThreads] = c; dp[x + 3 * kThreads] = d;
      }
      for (; x < units; x += kThreads) dp[x] = sp[x];
    } else if (UPI <= 64) {
      const uint32_t units = nkeep * UPI;
      for (uint32_t x = tid; x < units; x += kThreads) {
        const uint32_t p = divU.div(x), u = x - p * UPI;
        outU[(base + p) * UPI + u] = itemsU[(t0 + src_of[p]) * UPI + u];
      }
    } else {
      for (uint32_t p = w; p < nkeep; p += kWarps)
        for (uint32_t u = lane; u < UPI; u += 32)
          outU[(base + p) * UPI + u] = itemsU[(t0 + src_of[p]) * UPI + u];
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- a2 histogram

__device__ __forceinline__ uint32_t warp_sum(uint32_t x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(kFull, x, o);
  return x;
}

constexpr int kHistVec = 4;          // 16-byte dest loads per lane per tile and batch (a batch covers 512 items)

// Tiles a warp counts concurrently: two for R <= 8 (eight 16-byte loads in
// flight per lane, four warps per CTA), one otherwise (eight warps per CTA).
template <int RMAX>
struct HistShape {
  static constexpr int kTPW = (RMAX > 0 && RMAX <= 8) ? 2 : 1;
  static constexpr int kThreadsH = 32 * kHistTilesPerCta / kTPW;
};

// Per-tile per-destination counts (the counting half of the paper's radix
// sort by destination), one warp per one or two tiles, 16-byte
// loads, many small CTAs resident per SM.  CTA (b, l) covers tiles 8b..8b+7 of
// local rank l and also does the first level of the tile scan: for every
// destination d it writes O[l][d][t] = items with dest d in tiles 8b..t-1 of
// the block, and the block aggregate H[l][d][b] (scanned by k_scan).
// RMAX > 0: register counters for R <= RMAX reduced with warp shuffles;
// RMAX == 0: shared counters fed by __match_any_sync aggregation.
template <int RMAX>
__global__ void __launch_bounds__(HistShape<RMAX>::kThreadsH, 1024 / HistShape<RMAX>::kThreadsH)
k_hist(const RankDev* __restrict__ rk, const CtrlDev* __restrict__ ctrl, int R, uint64_t cap, uint32_t T) {
  constexpr int TPW = HistShape<RMAX>::kTPW;
  constexpr int NT = HistShape<RMAX>::kThreadsH;
  extern __shared__ uint32_t tc[];  // [kHistTilesPerCta][R] tile counts
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int l = blockIdx.y;
  const uint64_t n = n_items(ctrl[l], cap);
  const uint64_t tiles = (n + T - 1) / T;
  const uint64_t tb = (uint64_t)blockIdx.x * kHistTilesPerCta;
  if (tb >= tiles) return;  // uniform over the CTA
  const uint64_t nblk = (tiles + kHistTilesPerCta - 1) / kHistTilesPerCta;
  if (RMAX > 0) {
    // the warp's TPW tiles, batch by batch, all their loads issued before counting
    // packed counters: byte (d & 7) of word d >> 3 counts destination d; a
    // lane sees at most T / 32 <= 128 items of a tile, so no byte overflows
    constexpr int NW = RMAX > 0 ? (RMAX + 7) / 8 : 1;
    uint64_t c[TPW][NW];
    uint32_t nq[TPW];
    const int4* d4[TPW];
#pragma unroll
    for (int k = 0; k < TPW; ++k) {
      const uint64_t t = tb + w * TPW + k;
      const uint64_t t0 = t * T;
      const uint32_t nt = t < tiles ? (uint32_t)umin64(T, n - t0) : 0u;
      nq[k] = (nt + 3) / 4;
      d4[k] = reinterpret_cast<const int4*>(rk[l].dest + (t < tiles ? t0 : 0));  // t0*4 is a multiple of 1 KiB
#pragma unroll
      for (int x = 0; x < NW; ++x) c[k][x] = 0;
    }
    for (uint32_t q0 = 0; q0 < (T + 3) / 4; q0 += 32 * kHistVec) {
      int4 v[TPW][kHistVec];
#pragma unroll
      for (int k = 0; k < TPW; ++k)
#pragma unroll
        for (int j = 0; j < kHistVec; ++j) {
          const uint32_t q = q0 + j * 32 + lane;
          v[k][j] = q < nq[k] ? d4[k][q] : make_int4(-1, -1, -1, -1);
        }
#pragma unroll
      for (int k = 0; k < TPW; ++k) {
        const uint64_t t = tb + w * TPW + k;
        const uint32_t nt = t < tiles ? (uint32_t)umin64(T, n - t * T) : 0u;
        // every queued dest is in [0, R) (invalid ones were rejected at emit)
        auto add = [&](int d) {
          if (NW == 1) {
            c[k][0] += 1ull << ((unsigned)d << 3);
          } else {
            const uint64_t one = 1ull << ((d & 7) * 8);
#pragma unroll
            for (int x = 0; x < NW; ++x) c[k][x] += (d >> 3) == x ? one : 0ull;
          }
        };
        if ((q0 + 32 * kHistVec) * 4 <= nt) {  // the whole batch is in the tile: no bounds checks
#pragma unroll
          for (int j = 0; j < kHistVec; ++j) {
            add(v[k][j].x); add(v[k][j].y); add(v[k][j].z); add(v[k][j].w);
          }
        } else {
#pragma unroll
          for (int j = 0; j < kHistVec; ++j) {
            const uint32_t i0 = (q0 + j * 32 + lane) * 4;
            const int e[4] = {v[k][j].x, v[k][j].y, v[k][j].z, v[k][j].w};
#pragma unroll
            for (int m = 0; m < 4; ++m)
              if (i0 + m < nt) add(e[m]);
          }
        }
      }
    }
#pragma unroll
    for (int k = 0; k < TPW; ++k) {
      uint32_t* mine = tc + (w * TPW + k) * R;
#pragma unroll
      for (int r = 0; r < RMAX; ++r) {
        const uint32_t x = warp_sum((uint32_t)(c[k][r >> 3] >> ((r & 7) * 8)) & 0xffu);
        if (lane == (r & 31) && r < R) mine[r] = x;
      }
    }
  } else {
    const int ti = w;  // one tile per warp
    const uint64_t t = tb + ti;
    uint32_t* mine = tc + ti * R;
    for (int d = lane; d < R; d += 32) mine[d] = 0;
    __syncwarp();
    if (t < tiles) {
      const uint64_t t0 = t * T;
      const uint32_t nt = (uint32_t)umin64(T, n - t0);
      const int32_t* dest = rk[l].dest + t0;
      for (uint32_t i = lane; i < T; i += 32) {  // T is a multiple of 32
        const int d = i < nt ? dest[i] : -1;
        const unsigned m = __match_any_sync(kFull, d);
        if (d >= 0 && lane == __ffs(m) - 1) mine[d] += __popc(m);
        __syncwarp();
      }
    }
  }
  __syncthreads();
  // first scan level: exclusive prefix over the CTA's tiles, per destination
  uint32_t* O = rk[l].O;
  for (int d = threadIdx.x; d < R; d += NT) {
    uint32_t acc = 0;
    for (int ti = 0; ti < kHistTilesPerCta; ++ti) {
      const uint64_t t = tb + ti;
      if (t < tiles) {
        RAFI_DCHECK((uint64_t)d * tiles + t < (uint64_t)R * ((cap + T - 1) / T), "O index");
        O[(uint64_t)d * tiles + t] = acc;
      }
      acc += tc[ti * R + d];
    }
    rk[l].H[(uint64_t)d * nblk + blockIdx.x] = acc;
  }
}

// Self-test of the peer-control protocol on ONE device: the P blocks of one
// cooperative launch (co-resident by construction, so their spins cannot
// deadlock) each play one process with its own mailbox and its own copy of
// the count matrix.  Every round, block p writes its L rows, runs the count
// exchange, checks that the whole matrix arrived (a mismatch bumps *bad),
// then runs the completion barrier.  Block `absent` (or -1) never shows up:
// the others must give up after timeout_ns and flag err[p].
__device__ __forceinline__ uint64_t ctl_tag(int rnd, int row, int d) {
  return ((uint64_t)rnd << 40) ^ ((uint64_t)row << 20) ^ (uint64_t)d ^ 0x5EEDull;
}

__global__ void __launch_bounds__(256) k_ctl_selftest(unsigned long long* const* mbox, uint64_t* Cs, int P, int L,
                                                      int rounds, int absent, unsigned long long timeout_ns,
                                                      unsigned long long* err, unsigned long long* bad) {
  const int p = blockIdx.x;
  if (p == absent) return;
  const int R = P * L;
  PeerCtl pc;
  pc.mbox = mbox; pc.proc = p; pc.P = P; pc.timeout_ns = timeout_ns; pc.err = err + p;
  uint64_t* C = Cs + (size_t)p * R * R;
  for (int rnd = 1; rnd <= rounds; ++rnd) {
    for (int x = threadIdx.x; x < R * R; x += blockDim.x) {
      const int row = x / R, d = x % R;
      C[x] = row / L == p ? ctl_tag(rnd, row, d) : ~0ull;  // other processes' rows must arrive
    }
    __syncthreads();
    if (!ctl_counts_block(pc, C, L, R)) return;
    unsigned long long nbad = 0;
    for (int x = threadIdx.x; x < R * R; x += blockDim.x) nbad += C[x] != ctl_tag(rnd, x / R, x % R);
    if (nbad) atomicAdd(bad, nbad);
    __threadfence_system();
    ctl_barrier_block(pc);
    if (*reinterpret_cast<volatile unsigned long long*>(pc.err)) return;
  }
}

// ---------------------------------------------------------------- a3 scan

// One CTA per (destination d, local rank l): in place, H[l][d][b] := items
// with dest d in blocks 0..b-1 (second scan level; the tile offset is then
// O[l][d][t] + H[l][d][t/8]), and the row total send_count[d] -> count matrix
// C[g][d] (the paper's segment tally, kept on device).  The
// per-destination base (send offset, or the receiver's recv offset under
// FUSED) is added by k_plan / k_scatter.
constexpr int kScanThreads = 1024;
constexpr int kScanV = 4;

__global__ void __launch_bounds__(kScanThreads)
k_scan(const RankDev* __restrict__ rk, CtrlDev* __restrict__ ctrl, uint64_t* __restrict__ Cmat,
       int grank0, int R, uint64_t cap, uint32_t T, int L, int plan_mode, unsigned* __restrict__ done,
       uint64_t* __restrict__ dst_off, uint64_t* __restrict__ num_in, int* __restrict__ ovf,
       unsigned long long* __restrict__ G_out, PeerCtl pc) {
  __shared__ uint32_t wsum[kScanThreads / 32];
  __shared__ uint32_t carry_s;
  __shared__ uint32_t sh[kScanThreads * kScanV];
  const int d = blockIdx.x, l = blockIdx.y;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const uint64_t n = n_items(ctrl[l], cap);
  const uint64_t tiles = (n + T - 1) / T;
  const uint64_t M = (tiles + kHistTilesPerCta - 1) / kHistTilesPerCta;  // live blocks
  uint32_t* H = rk[l].H + (uint64_t)d * M;
  if (tid == 0) carry_s = 0;
  __syncthreads();
  for (uint64_t base = 0; base < M; base += (uint64_t)kScanThreads * kScanV) {
    uint32_t v[kScanV];
    uint32_t s = 0;
#pragma unroll
    for (int j = 0; j < kScanV; ++j) {  // coalesced load, transposed through shared memory
      const uint64_t i = base + (uint64_t)j * kScanThreads + tid;
      sh[j * kScanThreads + tid] = i < M ? H[i] : 0u;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kScanV; ++j) { v[j] = sh[tid * kScanV + j]; s += v[j]; }
    uint32_t x = s;  // inclusive warp scan
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    if (w == 0) {
      const uint32_t ws = wsum[lane];
      uint32_t z = ws;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, z, o);
        if (lane >= o) z += y;
      }
      wsum[lane] = z - ws;  // exclusive
    }
    __syncthreads();
    uint32_t e = carry_s + wsum[w] + x - s;
#pragma unroll
    for (int j = 0; j < kScanV; ++j) { sh[tid * kScanV + j] = e; e += v[j]; }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kScanV; ++j) {
      const uint64_t i = base + (uint64_t)j * kScanThreads + tid;
      if (i < M) H[i] = sh[j * kScanThreads + tid];
    }
    if (tid == kScanThreads - 1) carry_s = e;
    __syncthreads();
  }
  if (tid == 0) {
    Cmat[(uint64_t)(grank0 + l) * R + d] = carry_s;
    if (d == 0) {
      CtrlDev& c = ctrl[l];
      c.n_out = n;
      c.dropped = c.ctr - n;
      c.invalid_last = c.invalid;
    }
  }
  // the last block: with peer control, the count exchange (every rank's rows
  // into Cmat); then, plan_mode 1 (staged) / 2 (FUSED), every local rank's
  // plan -- one launch instead of three
  if ((plan_mode || pc.mbox) && last_block(done)) {
    if (pc.mbox && !ctl_counts_block(pc, Cmat, L, R)) {
      // a peer never arrived: move nothing this round (the host reports RAFI_ERR_TIMEOUT)
      if (threadIdx.x == 0) {
        *ovf = 2;
        if (G_out) *G_out = ~0ull;
      }
      return;
    }
    if (plan_mode) plan_all(Cmat, grank0, L, R, cap, plan_mode == 2, dst_off, num_in, ovf, G_out);
  }
}

// ---------------------------------------------------------------- a4 scatter


// Shared-memory layout of k_scatter (host mirror: scatter_layout()).
struct ScatterLayout {
  uint32_t stage_items;   // bytes of one stage's item buffer (0 if items are read from global)
  uint32_t stage_stride;  // bytes per stage (items + dests), 128-aligned
  uint32_t off_mbar, off_src, off_wcnt, off_wbase, off_rstart, off_tcnt, off_dbase, total;
};

__host__ __device__ inline ScatterLayout scatter_layout(uint32_t T, uint64_t B, int R, bool stage_items) {
  ScatterLayout s;
  auto al = [](uint64_t x, uint64_t a) { return (uint32_t)((x + a - 1) / a * a); };
  s.stage_items = stage_items ? al((uint64_t)T * B, 16) : 0u;
  s.stage_stride = al((uint64_t)s.stage_items + 4ull * T, 128);
  uint32_t o = 2 * s.stage_stride;
  s.off_mbar = o; o += 16;
  s.off_src = o; o = al(o + 2ull * T, 16);
  s.off_wcnt = o; o += 4 * kWarps * R;
  s.off_wbase = o; o += 4 * kWarps * R;
  s.off_rstart = o; o += 4 * R;
  s.off_tcnt = o; o = al(o + 4ull * R, 8);
  s.off_dbase = o; o += 8 * R;
  s.total = al(o, 16);
  return s;
}

// Phase 1 of both scatter kernels: warp w ranks items w*32*kK .. +32*kK-1 of
// the tile (slot order).  dk[k] = destination of item w*32*kK + 32k + lane
// (R past the tile end), rk_[k] = its rank among the warp's earlier items
// with the same destination (stability); wcnt[w][d] ends as
// the warp's count of destination d (zeroed by the caller).
template <int kK>
__device__ __forceinline__ void rank_chunk(const int32_t* __restrict__ dest_s, uint32_t nt, int R,
                                           uint32_t* __restrict__ wcnt, int (&dk)[kK], uint32_t (&rk_)[kK]) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 0; k < kK; ++k) {
    const uint32_t il = w * 32 * kK + k * 32 + lane;
    const int d = il < nt ? dest_s[il] : R;
    const unsigned m = __match_any_sync(kFull, d);
    uint32_t c = 0;
    if (d < R) c = wcnt[w * R + d];
    __syncwarp();
    if (d < R && lane == __ffs(m) - 1) wcnt[w * R + d] = c + __popc(m);
    __syncwarp();
    dk[k] = d;
    rk_[k] = c + __popc(m & lanemask_lt());
  }
}

// Stable scatter of each tile into one contiguous run per destination.
//   * Tile loads (items + dests) are 1-D TMA bulk copies into a two-stage
//     shared-memory ring guarded by mbarriers: tile i+1 (and i+2) stream in
//     while tile i is ranked and written.
//   * Ranking: __match_any_sync per warp chunk + per-warp running counts gives
//     each item its rank among same-destination items of the tile in slot
//     order (stability).
//   * Writing: the tile is re-ordered destination-major in shared memory
//     index space and written as consecutive 16/8/4/2/1-byte units, so every
//     destination run is stored with fully coalesced transactions.
//   * Destination: dst_table == nullptr -> the local send batch binned[cur]
//     (position = offset in the destination-major batch).  Otherwise the
//     FUSED exchange: unit goes straight to destination rank d's incoming
//     queue, dst_table[d] (local HBM or a CUDA-IPC peer mapping over NVLink).
//   Item index = O[l][d][t] (prefix over earlier tiles) + rank within the tile
//   + dst_off[l][d], the per-destination base from k_plan: send_off_me[d]
//   (staged) or recv_off_d[me] (FUSED).
template <typename U, bool kStageItems, int kK, int kMinB, bool kChunk>
__global__ void __launch_bounds__(kThreads, kMinB)
k_scatter(const RankDev* __restrict__ rk, const CtrlDev* __restrict__ ctrl, uint8_t* const* __restrict__ dst_table,
          const uint64_t* __restrict__ dst_off, const int* __restrict__ ovf, int L, int R, uint64_t cap, uint32_t T,
          int cur, uint32_t B, uint32_t UPI, FastDiv divU, FastDiv divB, ScatterLayout lay, unsigned* __restrict__ wrap_done,
          CtrlDev* __restrict__ ctrl_w, const uint64_t* __restrict__ wrap_num_in,
          PeerCtl pc) {
  if (ovf && *ovf) return;  // collective receive overflow: move nothing (Z3)
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + lay.off_mbar);
  uint16_t* src_of = reinterpret_cast<uint16_t*>(smem + lay.off_src);
  uint32_t* wcnt = reinterpret_cast<uint32_t*>(smem + lay.off_wcnt);
  uint32_t* wbase = reinterpret_cast<uint32_t*>(smem + lay.off_wbase);
  uint32_t* rstart = reinterpret_cast<uint32_t*>(smem + lay.off_rstart);
  uint32_t* tcnt = reinterpret_cast<uint32_t*>(smem + lay.off_tcnt);
  uintptr_t* dbase = reinterpret_cast<uintptr_t*>(smem + lay.off_dbase);
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  constexpr uint32_t K = kK;  // items per thread per tile (T = 256 * kK)

  auto issue = [&](uint32_t it) {  // thread 0: start loading iteration it's tile into stage it&1
    const uint64_t g = blockIdx.x + (uint64_t)it * gridDim.x;
    int l;
    uint64_t t, n, tiles;
    if (!tile_of(g, ctrl, L, cap, T, &l, &t, &n, &tiles)) return;
    const uint64_t t0 = t * T;
    const uint32_t nt = (uint32_t)umin64(T, n - t0);
    uint8_t* st = smem + (it & 1) * lay.stage_stride;
    const uint32_t bi = kStageItems ? ((nt * B + 15) & ~15u) : 0u;
    const uint32_t bd = (nt * 4 + 15) & ~15u;
    mbar_expect_tx(&mbar[it & 1], bi + bd);
    if (kStageItems) bulk_g2s(st, rk[l].out + t0 * B, bi, &mbar[it & 1]);
    bulk_g2s(st + lay.stage_items, rk[l].dest + t0, bd, &mbar[it & 1]);
  };

  if (tid == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) { issue(0); issue(1); }

  for (uint32_t it = 0;; ++it) {
    const uint64_t g = blockIdx.x + (uint64_t)it * gridDim.x;
    int l;
    uint64_t t, n, tiles;
    if (!tile_of(g, ctrl, L, cap, T, &l, &t, &n, &tiles)) break;
    const uint64_t t0 = t * T;
    const uint32_t nt = (uint32_t)umin64(T, n - t0);
    const uint8_t* st = smem + (it & 1) * lay.stage_stride;
    const int32_t* dest_s = reinterpret_cast<const int32_t*>(st + lay.stage_items);
    for (int x = tid; x < kWarps * R; x += kThreads) wcnt[x] = 0;
    // phase 2 inputs that do not depend on the tile data
    for (int d = tid; d < R; d += kThreads) {
      const uint8_t* base = dst_table ? dst_table[d] : rk[l].binned[cur];
      dbase[d] = (uintptr_t)base;
      // global base of (d, t), parked in rstart until phase 3
      const uint64_t nblk = (tiles + kHistTilesPerCta - 1) / kHistTilesPerCta;
      rstart[d] = rk[l].O[(uint64_t)d * tiles + t] + rk[l].H[(uint64_t)d * nblk + t / kHistTilesPerCta] +
                  (uint32_t)dst_off[(uint64_t)l * R + d];
    }
    mbar_wait(&mbar[it & 1], (it >> 1) & 1);
    __syncthreads();
    // phase 1: stable rank among same-destination items of the warp's chunk
    int dk[kK];
    uint32_t rk_[kK];
    rank_chunk<kK>(dest_s, nt, R, wcnt, dk, rk_);
    __syncthreads();
    // phase 2: warp bases per destination; tile-local run starts
    for (int d = tid; d < R; d += kThreads) {
      uint32_t run = 0;
      for (int i = 0; i < kWarps; ++i) { wbase[i * R + d] = run; run += wcnt[i * R + d]; }
      tcnt[d] = run;
    }
    __syncthreads();
    if (tid == 0) {
      uint32_t acc = 0;
      for (int d = 0; d < R; ++d) { const uint32_t c = tcnt[d]; tcnt[d] = acc; acc += c; }  // tcnt := tile run start
    }
    __syncthreads();
    // phase 3: destination-major order -> (source item, destination, position)
#pragma unroll
    for (int k = 0; k < kK; ++k) {
      if (dk[k] < R) {
        const int d = dk[k];
        const uint32_t r = wbase[w * R + d] + rk_[k];
        const uint32_t p = tcnt[d] + r;
        src_of[p] = (uint16_t)(w * 32 * K + k * 32 + lane);
      }
    }
    // per-run destination base, shifted so that position p of run d lands at
    // base_d + p*B (runs are contiguous in both the tile order and the output)
    for (int d = tid; d < R; d += kThreads) {
      const uint32_t cnt = (d + 1 < R ? tcnt[d + 1] : nt) - tcnt[d];
      RAFI_DCHECK((uint64_t)rstart[d] + cnt <= cap, "destination run beyond the destination queue");
      const uint32_t r0 = rstart[d];
      const uintptr_t a = dbase[d] + (uintptr_t)r0 * B;  // first byte of the run
      dbase[d] = a - (uintptr_t)tcnt[d] * B;
      // kChunk: rstart is free from here on and holds the number of
      // 16-byte-aligned chunks the run's bytes touch
      if (kChunk) rstart[d] = cnt ? (uint32_t)(((a + (uintptr_t)cnt * B + 15) >> 4) - (a >> 4)) : 0u;
    }
    __syncthreads();
    // phase 4: coalesced write of every destination run
    const U* srcU = kStageItems ? reinterpret_cast<const U*>(st) : reinterpret_cast<const U*>(rk[l].out + t0 * B);
    // A thread walks its units in increasing order, so the run it is in only
    // moves forward: one shared-memory read (src_of) per unit besides the data.
    if (kChunk) {
      // items of 4-byte granularity (20, 28, 36, 44 B ...): a thread writes one
      // 16-byte-aligned chunk of a run at a time,
      // gathering its four words from the (at most two) items it overlaps, so a
      // 44-B item costs 2.75 vector stores instead of 11 word stores
      // rstart[d] holds run d's chunk count; a thread walks the runs forward,
      // keeping [c0, c1) = the flat chunk range of the run it is in
      const uint8_t* src8 = reinterpret_cast<const uint8_t*>(srcU);
      int d = 0;
      uint32_t c0 = 0, c1 = rstart[0];
      for (uint32_t x = tid;; x += kThreads) {
        while (x >= c1 && d < R) {
          if (++d < R) { c0 = c1; c1 += rstart[d]; }
        }
        if (d >= R) break;
        const uint32_t p0 = tcnt[d], p1 = d + 1 < R ? tcnt[d + 1] : nt;
        const uintptr_t rs = dbase[d] + (uintptr_t)p0 * B, re = dbase[d] + (uintptr_t)p1 * B;
        const uintptr_t g = ((rs >> 4) + (x - c0)) << 4;
        RAFI_DCHECK(rs % 4 == 0 && g + 16 > rs && g < re, "chunk outside its run");
        if (g >= rs && g + 16 <= re) {
          const uint32_t o = (uint32_t)(g - rs), q = divB.div(o), e = o - q * B;
          RAFI_DCHECK(e < B && q * B + e == o && p0 + q < p1 && (e + 16 <= B || p0 + q + 1 < p1), "chunk items");
          const uint32_t s0 = (uint32_t)src_of[p0 + q] * B + e;
          const uint32_t s1 = e + 16 > B ? (uint32_t)src_of[p0 + q + 1] * B + e - B : s0;
          RAFI_DCHECK(s0 % 4 == 0 && s1 % 4 == 0 && ((uintptr_t)src8 & 3) == 0, "chunk source alignment");
          uint32_t v[4];
#pragma unroll
          for (int j = 0; j < 4; ++j)
            v[j] = *reinterpret_cast<const uint32_t*>(src8 + (e + 4 * j < B ? s0 : s1) + 4 * j);
          *reinterpret_cast<uint4*>(g) = make_uint4(v[0], v[1], v[2], v[3]);
        } else {  // the run's first or last chunk: word by word
          const uintptr_t w0 = g > rs ? g : rs, w1 = g + 16 < re ? g + 16 : re;
          for (uintptr_t a = w0; a < w1; a += 4) {
            const uint32_t o = (uint32_t)(a - rs), q = divB.div(o), e = o - q * B;
            *reinterpret_cast<uint32_t*>(a) =
                *reinterpret_cast<const uint32_t*>(src8 + (uint32_t)src_of[p0 + q] * B + e);
          }
        }
      }
    } else if (UPI <= 64) {
      const uint32_t units = nt * UPI;
      int d = 0;
      uint32_t nb = R > 1 ? tcnt[1] : nt;  // first position after run d
      U* dst = reinterpret_cast<U*>(dbase[0]);
      constexpr int kU = RAFI_SCATTER_ILP;  // independent units per thread in flight (ILP)
      for (uint32_t x0 = tid; x0 < units; x0 += kU * kThreads) {
        uint32_t p[kU], u[kU], s[kU];
        U v[kU];
        U* dd[kU];
#pragma unroll
        for (int j = 0; j < kU; ++j) {
          const uint32_t x = x0 + j * kThreads;
          p[j] = divU.div(x);
          u[j] = x - p[j] * UPI;
          s[j] = x < units ? (uint32_t)src_of[p[j]] : 0u;
        }
#pragma unroll
        for (int j = 0; j < kU; ++j) {
          v[j] = srcU[s[j] * UPI + u[j]];
          if (x0 + j * kThreads < units && p[j] >= nb) {
            do { ++d; nb = d + 1 < R ? tcnt[d + 1] : nt; } while (p[j] >= nb);
            dst = reinterpret_cast<U*>(dbase[d]);
          }
          dd[j] = dst;
        }
#pragma unroll
        for (int j = 0; j < kU; ++j)
          if (x0 + j * kThreads < units) {
            RAFI_DCHECK((uintptr_t)&dd[j][(uint64_t)p[j] * UPI + u[j]] >=
                            (uintptr_t)(dst_table ? dst_table[0] : rk[l].binned[cur]) ||
                            dst_table, "scatter store below the send batch");
            dd[j][(uint64_t)p[j] * UPI + u[j]] = v[j];
          }
      }
    } else {
      int d = 0;
      uint32_t nb = R > 1 ? tcnt[1] : nt;
      for (uint32_t p = w; p < nt; p += kWarps) {
        while (p >= nb) { ++d; nb = d + 1 < R ? tcnt[d + 1] : nt; }
        U* dst = reinterpret_cast<U*>(dbase[d]) + (uint64_t)p * UPI;
        const U* src = srcU + (uint64_t)src_of[p] * UPI;
        for (uint32_t u = lane; u < UPI; u += 32) dst[u] = src[u];
      }
    }
    __syncthreads();  // every thread is done with this stage
    if (tid == 0) {
      fence_proxy_async();  // order the generic-proxy reads before the async refill
      issue(it + 2);
    }
  }
  if (dst_table) __threadfence_system();  // pushes to peer memory complete before the kernel does
  // wrap-up epilogue by the last block: every block has finished
  // reading the emit counters, so they can be reset for the next round
  if (wrap_done && last_block(wrap_done)) {
    for (int l2 = threadIdx.x; l2 < L; l2 += blockDim.x) {
      ctrl_w[l2].ctr = 0;
      ctrl_w[l2].invalid = 0;
      ctrl_w[l2].num_in = wrap_num_in[l2];
    }
    // peer control: the completion barrier (every block's pushes were made
    // visible system-wide before it counted itself in last_block)
    if (pc.mbox) ctl_barrier_block(pc);
  }
}

// ---------------------------------------------------------------- a4 scatter, bulk-store variant

// 1-D bulk copy shared -> global through the TMA unit (UBLKCP.G.S), tracked in
// the issuing thread's bulk async-group.  dst may be a CUDA-IPC peer mapping.
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// Shared-memory layout of k_scatter_perm (host mirror: bulk_layout()).
struct BulkLayout {
  uint32_t stage_items;   // bytes of one stage's items, 16-aligned
  uint32_t stage_stride;  // items + dests, 128-aligned
  uint32_t obuf_stride;   // one destination-major output tile: T*B + alignment slack per run
  uint32_t nobuf;         // output tiles: 2 (store of tile i overlaps tile i+1) or 1 (large items)
  uint32_t off_obuf, off_mbar, off_wcnt, off_wbase, off_tcnt, off_ooff, off_dbase, total;
};

__host__ __device__ inline BulkLayout bulk_layout(uint32_t T, uint64_t B, int R, uint32_t nobuf) {
  BulkLayout s;
  s.nobuf = nobuf;
  auto al = [](uint64_t x, uint64_t a) { return (uint32_t)((x + a - 1) / a * a); };
  s.stage_items = al((uint64_t)T * B, 16);
  s.stage_stride = al((uint64_t)s.stage_items + 4ull * T, 128);
  s.obuf_stride = al((uint64_t)T * B + 32ull * R + 16, 128);  // <= 30 B of slack per run
  uint32_t o = 2 * s.stage_stride;
  s.off_obuf = o; o += nobuf * s.obuf_stride;
  s.off_mbar = o; o += 16;
  s.off_wcnt = o; o += 4 * kWarps * R;
  s.off_wbase = o; o += 4 * kWarps * R;
  s.off_tcnt = o; o += 4 * R;
  s.off_ooff = o; o = al(o + 4ull * R, 8);
  s.off_dbase = o; o += 8 * R;
  s.total = al(o, 16);
  return s;
}

// Same result as k_scatter (every item read once, written once,
// destination-major and stable in slot order), different data movement:
//   * tile loads: TMA bulk copies into a two-stage mbarrier ring (as k_scatter);
//   * ranking: rank_chunk (as k_scatter);
//   * permutation: each thread moves its own items (consecutive items, so
//     conflict-free reads) into a destination-major output tile in shared
//     memory.  Run d starts at an offset congruent to its global byte address
//     modulo 16, so the body of every run is one 16-byte-aligned span on both
//     sides whatever the item size;
//   * stores: one elected thread issues a TMA bulk store (cp.async.bulk
//     shared -> global) per run body, straight into the destination queue (the
//     local send batch, the local incoming queue, or a peer's incoming queue
//     over NVLink under FUSED), double-buffered output tiles when they fit;
//     threads write the unaligned heads and tails (< 16 B).
// The stage is released to the next TMA load as soon as it is permuted.
template <typename U, int kK, int kMinB>
__global__ void __launch_bounds__(kThreads, kMinB)
k_scatter_perm(const RankDev* __restrict__ rk, const CtrlDev* __restrict__ ctrl, uint8_t* const* __restrict__ dst_table,
               const uint64_t* __restrict__ dst_off, const int* __restrict__ ovf, int L, int R, uint64_t cap, uint32_t T,
               int cur, uint32_t B, uint32_t UPI, BulkLayout lay, unsigned* __restrict__ wrap_done,
               CtrlDev* __restrict__ ctrl_w, const uint64_t* __restrict__ wrap_num_in,
          PeerCtl pc) {
  if (ovf && *ovf) return;  // collective receive overflow: move nothing (Z3)
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + lay.off_mbar);
  uint32_t* wcnt = reinterpret_cast<uint32_t*>(smem + lay.off_wcnt);
  uint32_t* wbase = reinterpret_cast<uint32_t*>(smem + lay.off_wbase);
  uint32_t* tcnt = reinterpret_cast<uint32_t*>(smem + lay.off_tcnt);
  uint32_t* ooff = reinterpret_cast<uint32_t*>(smem + lay.off_ooff);
  uintptr_t* dbase = reinterpret_cast<uintptr_t*>(smem + lay.off_dbase);
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;

  auto issue = [&](uint32_t it) {  // thread 0: start loading iteration it's tile into stage it&1
    const uint64_t g = blockIdx.x + (uint64_t)it * gridDim.x;
    int l;
    uint64_t t, n, tiles;
    if (!tile_of(g, ctrl, L, cap, T, &l, &t, &n, &tiles)) return;
    const uint64_t t0 = t * T;
    const uint32_t nt = (uint32_t)umin64(T, n - t0);
    uint8_t* st = smem + (it & 1) * lay.stage_stride;
    const uint32_t bi = (nt * B + 15) & ~15u;
    const uint32_t bd = (nt * 4 + 15) & ~15u;
    mbar_expect_tx(&mbar[it & 1], bi + bd);
    bulk_g2s(st, rk[l].out + t0 * B, bi, &mbar[it & 1]);
    bulk_g2s(st + lay.stage_items, rk[l].dest + t0, bd, &mbar[it & 1]);
  };

  // byte address of item 0 of destination d's run of iteration it's tile:
  // destination base + (tile prefix O + block prefix H + per-destination
  // base) * B; 0 past the last tile
  auto run_addr = [&](uint32_t it, int d) -> uintptr_t {
    const uint64_t g = blockIdx.x + (uint64_t)it * gridDim.x;
    int l;
    uint64_t t, n, tiles;
    if (!tile_of(g, ctrl, L, cap, T, &l, &t, &n, &tiles)) return 0;
    const uint64_t nblk = (tiles + kHistTilesPerCta - 1) / kHistTilesPerCta;
    const uint64_t first = (uint64_t)rk[l].O[(uint64_t)d * tiles + t] +
                           rk[l].H[(uint64_t)d * nblk + t / kHistTilesPerCta] + dst_off[(uint64_t)l * R + d];
    return (uintptr_t)(dst_table ? dst_table[d] : rk[l].binned[cur]) + (uintptr_t)(first * B);
  };

  if (tid == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) { issue(0); issue(1); }
  uintptr_t pf_addr = (R <= kThreads && tid < R) ? run_addr(0, tid) : 0;

  for (uint32_t it = 0;; ++it) {
    const uint64_t g = blockIdx.x + (uint64_t)it * gridDim.x;
    int l;
    uint64_t t, n, tiles;
    if (!tile_of(g, ctrl, L, cap, T, &l, &t, &n, &tiles)) break;
    const uint64_t t0 = t * T;
    const uint32_t nt = (uint32_t)umin64(T, n - t0);
    const uint8_t* st = smem + (it & 1) * lay.stage_stride;
    uint8_t* ob = smem + lay.off_obuf + (lay.nobuf == 2 ? (it & 1) : 0u) * lay.obuf_stride;
    const int32_t* dest_s = reinterpret_cast<const int32_t*>(st + lay.stage_items);
    for (int x = tid; x < kWarps * R; x += kThreads) wcnt[x] = 0;
    if (R <= kThreads) {  // the addresses were loaded one tile ahead
      if (tid < R) {
        dbase[tid] = pf_addr;
        pf_addr = run_addr(it + 1, tid);
      }
    } else {
      for (int d = tid; d < R; d += kThreads) dbase[d] = run_addr(it, d);
    }
    mbar_wait(&mbar[it & 1], (it >> 1) & 1);
    __syncthreads();
    int dk[kK];
    uint32_t rk_[kK];
    rank_chunk<kK>(dest_s, nt, R, wcnt, dk, rk_);
    __syncthreads();
    // warp bases per destination, tile count per destination
    for (int d = tid; d < R; d += kThreads) {
      uint32_t run = 0;
      for (int i = 0; i < kWarps; ++i) { wbase[i * R + d] = run; run += wcnt[i * R + d]; }
      tcnt[d] = run;
    }
    __syncthreads();
    if (tid == 0) {
      // output-tile offsets: run d at the next offset congruent to its global
      // address mod 16 (tcnt stays the per-destination count)
      uint32_t o = 0;
      for (int d = 0; d < R; ++d) {
        o = ((o + 15) & ~15u) + (uint32_t)(dbase[d] & 15);
        ooff[d] = o;
        o += tcnt[d] * B;
      }
      // this output buffer's stores (two tiles ago, or the last tile's with one buffer) have read it
      if (lay.nobuf == 2) bulk_wait_read<1>(); else bulk_wait_read<0>();
    }
    __syncthreads();
    // permutation: item il (slot order) -> position rank in run d of the output
    // tile.  Lane j starts at unit j mod UPI of its item and wraps around, so
    // the lanes of one shared-memory wavefront hit different banks even when
    // B is a multiple of 128 (items at the same bank offset).
    const U* srcU = reinterpret_cast<const U*>(st);
    const uint32_t u0 = lane % UPI;
#pragma unroll
    for (int k = 0; k < kK; ++k) {
      const int d = dk[k];
      if (d < R) {
        const uint32_t il = w * 32 * kK + k * 32 + lane;
        U* dstU = reinterpret_cast<U*>(ob + ooff[d] + (wbase[w * R + d] + rk_[k]) * B);
        const U* s = srcU + (uint64_t)il * UPI;
        uint32_t u = u0;
        for (uint32_t j = 0; j < UPI; j += 4) {
          U v[4];
          uint32_t uu[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uu[q] = u;
            if (j + q < UPI) v[q] = s[u];
            u = u + 1 == UPI ? 0u : u + 1;
          }
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (j + q < UPI) dstU[uu[q]] = v[q];
        }
      }
    }
    fence_proxy_async();  // this thread's generic smem writes -> visible to the bulk stores
    __syncthreads();
    if (tid == 0) {
      issue(it + 2);  // the stage is consumed: refill it
      for (int d = 0; d < R; ++d) {
        const uint64_t len = (uint64_t)tcnt[d] * B;
        const uintptr_t a = dbase[d], e = a + len;
        const uintptr_t b0 = (a + 15) & ~(uintptr_t)15, b1 = e & ~(uintptr_t)15;
        if (b1 > b0) bulk_s2g(reinterpret_cast<void*>(b0), ob + ooff[d] + (b0 - a), (uint32_t)(b1 - b0));
      }
      bulk_commit();
    }
    // heads and tails (< 16 B each, or the whole run when it has no aligned body)
    for (int d = tid; d < R; d += kThreads) {
      const uint64_t len = (uint64_t)tcnt[d] * B;
      if (!len) continue;
      const uintptr_t a = dbase[d], e = a + len;
      uintptr_t b0 = (a + 15) & ~(uintptr_t)15, b1 = e & ~(uintptr_t)15;
      if (b1 <= b0) b0 = b1 = e;  // no body: threads write the whole run
      const uint8_t* o = ob + ooff[d];
      for (uintptr_t x = a; x < b0; x += sizeof(U))
        *reinterpret_cast<U*>(x) = *reinterpret_cast<const U*>(o + (x - a));
      for (uintptr_t x = b1; x < e; x += sizeof(U))
        *reinterpret_cast<U*>(x) = *reinterpret_cast<const U*>(o + (x - a));
    }
    __syncthreads();  // tcnt / ooff / dbase / the output tile are rewritten by the next tile
  }
  if (tid == 0) bulk_wait_all();  // every bulk store has completed its writes
  if (dst_table) __threadfence_system();
  if (wrap_done && last_block(wrap_done)) {
    for (int l2 = threadIdx.x; l2 < L; l2 += blockDim.x) {
      ctrl_w[l2].ctr = 0;
      ctrl_w[l2].invalid = 0;
      ctrl_w[l2].num_in = wrap_num_in[l2];
    }
    // peer control: the completion barrier (every block's pushes were made
    // visible system-wide before it counted itself in last_block)
    if (pc.mbox) ctl_barrier_block(pc);
  }
}

// ---------------------------------------------------------------- a5 plan

// Standalone plan (after the count all-gather when several processes share
// the communicator): one block computes every local rank's bases.
template <bool kFused>
__global__ void k_plan(const uint64_t* __restrict__ C, int grank0, int L, int R, uint64_t cap,
                       uint64_t* __restrict__ dst_off, uint64_t* __restrict__ num_in, int* __restrict__ ovf,
                       unsigned long long* __restrict__ G_out) {
  plan_all(C, grank0, L, R, cap, kFused, dst_off, num_in, ovf, G_out);
}

// ---------------------------------------------------------------- a6 copy (PEER)

constexpr uint32_t kCopyChunkBytes = 64 * 1024;

template <typename U>
__global__ void __launch_bounds__(kThreads)
k_copy(const CopyRun* __restrict__ runs, const RankDev* __restrict__ rk, int R, uint32_t UPI,
       const uint64_t* __restrict__ tot_items) {
  const int l = blockIdx.y;
  const uint64_t tot_units = tot_items[l] * UPI;
  const uint64_t CH = kCopyChunkBytes / sizeof(U);
  const uint64_t nchunks = (tot_units + CH - 1) / CH;
  U* dst = reinterpret_cast<U*>(rk[l].in);
  const CopyRun* rr = runs + (uint64_t)l * R;
  for (uint64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    const uint64_t u0 = c * CH, u1 = umin64(u0 + CH, tot_units);
    for (int s = 0; s < R; ++s) {
      const uint64_t a = rr[s].dst * UPI, b = a + rr[s].count * UPI;
      const uint64_t lo = umax64(a, u0), hi = umin64(b, u1);
      if (lo >= hi) continue;
      const U* src = reinterpret_cast<const U*>(rr[s].src);
      uint64_t u = lo + threadIdx.x;
      for (; u + 3 * kThreads < hi; u += 4 * kThreads) {
        const U v0 = src[u - a], v1 = src[u - a + kThreads], v2 = src[u - a + 2 * kThreads],
                v3 = src[u - a + 3 * kThreads];
        dst[u] = v0; dst[u + kThreads] = v1; dst[u + 2 * kThreads] = v2; dst[u + 3 * kThreads] = v3;
      }
      for (; u < hi; u += kThreads) dst[u] = src[u - a];
    }
  }
}

static PeerCtl peer_ctl(Ctx* c, bool on) {
  PeerCtl pc;
  pc.mbox = on ? c->mbox_table_dev : nullptr;
  pc.proc = c->proc;
  pc.P = c->nprocs;
  pc.timeout_ns = c->peer_timeout_ns;
  pc.err = &c->ctrl[0].status;
  return pc;
}

int launch_ctl_selftest(unsigned long long* const* mbox, uint64_t* Cs, int P, int L, int rounds, int absent,
                        unsigned long long timeout_ns, unsigned long long* err, unsigned long long* bad) {
  void* args[] = {(void*)&mbox, (void*)&Cs, (void*)&P, (void*)&L, (void*)&rounds, (void*)&absent, (void*)&timeout_ns,
                  (void*)&err, (void*)&bad};
  RAFI_CK_CUDA(cudaLaunchCooperativeKernel((const void*)k_ctl_selftest, dim3(P), dim3(256), args, 0, nullptr));
  return RAFI_OK;
}

// ---------------------------------------------------------------- a7 wrap-up

__global__ void k_wrapup(CtrlDev* ctrl, const uint64_t* num_in, int L, const int* ovf) {
  const int l = threadIdx.x;
  if (l < L && !(ovf && *ovf)) {
    ctrl[l].ctr = 0;
    ctrl[l].invalid = 0;
    ctrl[l].num_in = num_in[l];
  }
}

// ---------------------------------------------------------------- host side

static int g_num_sms = 0;

static int num_sms(int device) {
  if (!g_num_sms) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess || v <= 0) v = 148;
    g_num_sms = v;
  }
  return g_num_sms;
}

// Largest of 16/8/4/2/1 dividing the item size and every base address.
static uint32_t unit_for(uint64_t B, uintptr_t align_bits) {
  for (uint32_t u = 16; u > 1; u >>= 1)
    if (B % u == 0 && (align_bits % u) == 0) return u;
  return 1;
}

// Items up to 96 B: four 54-KiB CTAs per SM (more warps to hide the
// dependent shared-memory/index latency of many small units); larger items:
// two 110-KiB CTAs (longer tiles).  Measured with the cfg5 size sweep
// (profiles/r01_scatter_variants.md).
static int scatter_minb(uint64_t B) { return B <= 96 ? 4 : 2; }
// Up to 64 B the tile may use 62 KiB: that doubles the tile where a 54-KiB
// budget falls just short (24 B: 1024 items, 56 B: 512 items; three CTAs/SM
// then) and changes nothing else (tile sweeps, profiles/r01_suite_n1_tiles_threads.md).
static uint32_t scatter_budget(uint64_t B) {
  if (B <= 64) return 62u * 1024u;
  return scatter_minb(B) == 4 ? 54u * 1024u : 110u * 1024u;
}

uint32_t choose_tile(uint64_t item_bytes, int R, int L) {
  // R <= 8 and 8-byte units: the warp-tile path (warp_tiles.cu), 256-item tiles
  if (const uint32_t w = warp_tile_for(item_bytes, R, L)) return w;
  // two pipeline stages (items + dests) plus 2 B/item of indices in ~110 KiB,
  // so two CTAs fit on an SM
  const uint64_t t = scatter_budget(item_bytes) / (2 * item_bytes + 10);
  uint32_t k = 1;  // items per thread: a power of two (the scatter is templated on it)
  while (k < (uint32_t)kMaxK && (uint64_t)kThreads * k * 2 <= t) k *= 2;
  return kThreads * k;
}

static bool stage_items(uint32_t T, uint64_t B) { return 2ull * T * (B + 4) <= 200u * 1024u; }

size_t scatter_smem_bytes(uint32_t T, uint64_t B, int R) { return scatter_layout(T, B, R, stage_items(T, B)).total; }

int launch_emit_bulk(Ctx* c, int local, const uint8_t* items, const int32_t* dests, uint64_t n) {
  if (n == 0) return RAFI_OK;
  LocalRank& L = c->lr[local];
  const uint32_t unit = unit_for(c->B, (uintptr_t)items | (uintptr_t)L.out);
  const uint32_t UPI = (uint32_t)(c->B / unit);
  const FastDiv dv(UPI);
  const uint64_t tiles = (n + kEmitTile - 1) / kEmitTile;
  const int grid = (int)std::min<uint64_t>(tiles, (uint64_t)num_sms(c->device) * 8);
  CtrlDev* ctrl = c->ctrl + local;
#define EMIT_LAUNCH(T_)                                                                             \
  k_emit_bulk<T_><<<grid, kThreads, 0, c->stream>>>(items, dests, n, L.out, L.dest, ctrl, c->R, c->cap, \
                                                   (uint32_t)c->B, UPI, dv)
  switch (unit) {
    case 16: EMIT_LAUNCH(uint4); break;
    case 8: EMIT_LAUNCH(uint2); break;
    case 4: EMIT_LAUNCH(uint32_t); break;
    case 2: EMIT_LAUNCH(uint16_t); break;
    default: EMIT_LAUNCH(uint8_t); break;
  }
#undef EMIT_LAUNCH
  RAFI_CK_CUDA(cudaGetLastError());
  c->launches += 1;
  return RAFI_OK;
}

static int persistent_grid(Ctx* c, int per_sm) {
  const uint64_t max_tiles_all = c->max_tiles * (uint64_t)c->L;
  return (int)std::max<uint64_t>(1, std::min<uint64_t>(max_tiles_all, (uint64_t)num_sms(c->device) * per_sm));
}

int launch_hist(Ctx* c, int plan_mode, unsigned long long* G_out, bool ctl) {
  if (hist_w_ok(c->tile, c->R)) {  // one warp per scan block (same O/H layout)
    RAFI_CK(launch_hist_w(c, num_sms(c->device), plan_mode, G_out, peer_ctl(c, ctl)));
    c->launches += 1; c->fwd_launches += 1;
    return RAFI_OK;
  }
  const dim3 grid((unsigned)std::max<uint64_t>(1, (c->max_tiles + kHistTilesPerCta - 1) / kHistTilesPerCta), c->L);
  const size_t sm = sizeof(uint32_t) * kHistTilesPerCta * c->R;
#define HIST(RM)                                                                                        \
  do {                                                                                                  \
    if (sm > 48 * 1024)                                                                                 \
      RAFI_CK_CUDA(cudaFuncSetAttribute(k_hist<RM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)); \
    k_hist<RM><<<grid, HistShape<RM>::kThreadsH, sm, c->stream>>>(rank_table(c), c->ctrl, c->R, c->cap, c->tile); \
  } while (0)
  if (c->R <= 1) HIST(1);
  else if (c->R <= 2) HIST(2);
  else if (c->R <= 4) HIST(4);
  else if (c->R <= 8) HIST(8);
  else if (c->R <= 16) HIST(16);
  else if (c->R <= 32) HIST(32);
  else HIST(0);
#undef HIST
  RAFI_CK_CUDA(cudaGetLastError());
  c->launches += 1; c->fwd_launches += 1;
  return RAFI_OK;
}

int launch_scan(Ctx* c, int plan_mode, unsigned long long* G_out, bool ctl) {
  if (hist_w_ok(c->tile, c->R) && hist_w_fuses_scan(c)) return RAFI_OK;  // done by k_hist_w's last CTA
  k_scan<<<dim3(c->R, c->L), kScanThreads, 0, c->stream>>>(rank_table(c), c->ctrl, c->Cdev, c->proc * c->L, c->R,
                                                           c->cap, c->tile, c->L, plan_mode, c->done_dev, c->off_dev,
                                                           c->plan_dev, c->ovf_dev, G_out, peer_ctl(c, ctl));
  RAFI_CK_CUDA(cudaGetLastError());
  c->launches += 1; c->fwd_launches += 1;
  return RAFI_OK;
}

template <typename U, bool kSI, int kK, int kMinB, bool kChunk>
static int launch_scatter_kk(Ctx* c, bool fused, bool wrap, uint32_t UPI, int grid, const ScatterLayout& lay) {
  auto k = k_scatter<U, kSI, kK, kMinB, kChunk>;
  RAFI_CK_CUDA(ensure_smem((const void*)k, (int)lay.total, c->device));
  k<<<grid, kThreads, lay.total, c->stream>>>(rank_table(c), c->ctrl, fused ? c->in_table_dev : nullptr, c->off_dev,
                                             fused ? c->ovf_dev : nullptr, c->L, c->R, c->cap,
                                             c->tile, c->cur, (uint32_t)c->B, UPI, FastDiv(UPI),
                                             FastDiv((uint32_t)c->B), lay, wrap ? c->done_dev + 1 : nullptr, c->ctrl,
                                             c->plan_dev, peer_ctl(c, c->scatter_barrier));
  RAFI_CK_CUDA(cudaGetLastError());
  return RAFI_OK;
}

// 16-byte chunk gathering (kChunk) for 4-byte units (B % 8 == 4, B >= 16):
// 44 B goes from 4.43 to 5.41 TB/s.  8-byte units (24, 40 B) stay on unit
// stores, which measured faster there (profiles/r01_suite_n1_cfg5_chunk.md).
template <typename U, int kK, int kMinB>
static int launch_scatter_k(Ctx* c, bool fused, bool wrap, uint32_t UPI, int grid) {
  const bool si = stage_items(c->tile, c->B);
  const ScatterLayout lay = scatter_layout(c->tile, c->B, c->R, si);
  constexpr bool kCanChunk = sizeof(U) == 4;
  const bool chunk = kCanChunk && c->B >= 16 && c->B % 16 != 0;
  if (chunk)
    return si ? launch_scatter_kk<U, true, kK, kMinB, kCanChunk>(c, fused, wrap, UPI, grid, lay)
              : launch_scatter_kk<U, false, kK, kMinB, kCanChunk>(c, fused, wrap, UPI, grid, lay);
  return si ? launch_scatter_kk<U, true, kK, kMinB, false>(c, fused, wrap, UPI, grid, lay)
            : launch_scatter_kk<U, false, kK, kMinB, false>(c, fused, wrap, UPI, grid, lay);
}

template <typename U, int kMinB>
static int launch_scatter_m(Ctx* c, bool fused, bool wrap, uint32_t UPI, int grid) {
  switch (c->tile / kThreads) {
    case 1: return launch_scatter_k<U, 1, kMinB>(c, fused, wrap, UPI, grid);
    case 2: return launch_scatter_k<U, 2, kMinB>(c, fused, wrap, UPI, grid);
    case 4: return launch_scatter_k<U, 4, kMinB>(c, fused, wrap, UPI, grid);
    case 8: return launch_scatter_k<U, 8, kMinB>(c, fused, wrap, UPI, grid);
    case 16: return launch_scatter_k<U, 16, kMinB>(c, fused, wrap, UPI, grid);
    default: set_error("tile must be 256 * 2^k"); return RAFI_ERR_INVALID_ARG;
  }
}

template <typename U>
static int launch_scatter_t(Ctx* c, bool fused, bool wrap, uint32_t UPI, int grid) {
  return scatter_minb(c->B) == 4 ? launch_scatter_m<U, 4>(c, fused, wrap, UPI, grid)
                                 : launch_scatter_m<U, 2>(c, fused, wrap, UPI, grid);
}

// ---- permuting scatter (RAFI_SCATTER_BULK: TMA bulk stores)

bool perm_supported(uint64_t B) { return B % 4 == 0; }

// Output tiles: two (the store of tile i overlaps tile i+1) when that still
// leaves room for two CTAs per SM, else one.
static uint32_t perm_nobuf(uint32_t T, uint64_t B, int R) {
  return bulk_layout(T, B, R, 2).total <= 112u * 1024u ? 2u : 1u;
}

size_t perm_smem_bytes(uint32_t T, uint64_t B, int R) { return bulk_layout(T, B, R, perm_nobuf(T, B, R)).total; }

// Largest tile (256 * 2^k) whose layout fits two CTAs per SM, else one.  Its
// NVLink pushes gain 2-9% from 512-item tiles over 256-item ones at N=2 and
// N=4 (profiles/r01_bulk_tiles_multigpu.md).
uint32_t choose_tile_perm(uint64_t B, int R) {
  for (uint32_t budget : {112u * 1024u, 227u * 1024u}) {
    uint32_t best = 0;
    for (uint32_t T = kThreads; T <= kThreads * kMaxK; T *= 2)
      if (perm_smem_bytes(T, B, R) <= budget) best = T;
    if (best) return best;
  }
  return kThreads;
}

template <typename U, int kK, int kMinB>
static int launch_perm_k(Ctx* c, bool fused, bool wrap, uint32_t UPI, int grid) {
  const BulkLayout lay = bulk_layout(c->tile, c->B, c->R, perm_nobuf(c->tile, c->B, c->R));
  auto k = k_scatter_perm<U, kK, kMinB>;
  RAFI_CK_CUDA(ensure_smem((const void*)k, (int)lay.total, c->device));
  k<<<grid, kThreads, lay.total, c->stream>>>(rank_table(c), c->ctrl, fused ? c->in_table_dev : nullptr, c->off_dev,
                                             fused ? c->ovf_dev : nullptr, c->L, c->R, c->cap, c->tile, c->cur,
                                             (uint32_t)c->B, UPI, lay, wrap ? c->done_dev + 1 : nullptr, c->ctrl,
                                             c->plan_dev, peer_ctl(c, c->scatter_barrier));
  RAFI_CK_CUDA(cudaGetLastError());
  return RAFI_OK;
}

template <typename U, int kMinB>
static int launch_perm_m(Ctx* c, bool fused, bool wrap, uint32_t UPI, int grid) {
  switch (c->tile / kThreads) {
    case 1: return launch_perm_k<U, 1, kMinB>(c, fused, wrap, UPI, grid);
    case 2: return launch_perm_k<U, 2, kMinB>(c, fused, wrap, UPI, grid);
    case 4: return launch_perm_k<U, 4, kMinB>(c, fused, wrap, UPI, grid);
    case 8: return launch_perm_k<U, 8, kMinB>(c, fused, wrap, UPI, grid);
    case 16: return launch_perm_k<U, 16, kMinB>(c, fused, wrap, UPI, grid);
    default: set_error("tile must be 256 * 2^k"); return RAFI_ERR_INVALID_ARG;
  }
}

template <typename U>
static int launch_perm_t(Ctx* c, bool fused, bool wrap, uint32_t UPI, int grid, int per_sm) {
  return per_sm >= 4 ? launch_perm_m<U, 4>(c, fused, wrap, UPI, grid) : launch_perm_m<U, 2>(c, fused, wrap, UPI, grid);
}

static int launch_scatter_perm(Ctx* c, bool fused, bool wrap) {
  const uint32_t unit = unit_for(c->B, 0);
  const uint32_t UPI = (uint32_t)(c->B / unit);
  const size_t smem = perm_smem_bytes(c->tile, c->B, c->R);
  const int fit = (int)((228u * 1024u) / (smem + 1024u));
  const int per_sm = std::max(1, std::min(4, fit));
  const int grid = persistent_grid(c, per_sm);
  int rc;
  switch (unit) {
    case 16: rc = launch_perm_t<uint4>(c, fused, wrap, UPI, grid, per_sm); break;
    case 8: rc = launch_perm_t<uint2>(c, fused, wrap, UPI, grid, per_sm); break;
    case 4: rc = launch_perm_t<uint32_t>(c, fused, wrap, UPI, grid, per_sm); break;
    default: set_error("permuting scatter needs item_bytes % 4 == 0"); return RAFI_ERR_UNSUPPORTED;
  }
  if (rc == RAFI_OK) { c->launches += 1; c->fwd_launches += 1; }
  return rc;
}

int launch_scatter(Ctx* c, bool fused, bool wrap) {
  if (c->scatter_eff == RAFI_SCATTER_BULK) return launch_scatter_perm(c, fused, wrap);
  if (warp_tiles_ok(c->tile, c->B, c->R, c->L)) {
    RAFI_CK(launch_scatter_w(c, fused, wrap, peer_ctl(c, c->scatter_barrier), num_sms(c->device)));
    c->launches += 1; c->fwd_launches += 1;
    return RAFI_OK;
  }
  const uint32_t unit = unit_for(c->B, 0);
  const uint32_t UPI = (uint32_t)(c->B / unit);
  const size_t smem = scatter_smem_bytes(c->tile, c->B, c->R);
  const int fit = (int)((227u * 1024u) / (smem + 1024u));  // CTAs whose shared memory fits on an SM
  const int per_sm = std::max(1, std::min(scatter_minb(c->B), fit));
  const int grid = persistent_grid(c, per_sm);
  int rc;
  switch (unit) {
    case 16: rc = launch_scatter_t<uint4>(c, fused, wrap, UPI, grid); break;
    case 8: rc = launch_scatter_t<uint2>(c, fused, wrap, UPI, grid); break;
    case 4: rc = launch_scatter_t<uint32_t>(c, fused, wrap, UPI, grid); break;
    case 2: rc = launch_scatter_t<uint16_t>(c, fused, wrap, UPI, grid); break;
    default: rc = launch_scatter_t<uint8_t>(c, fused, wrap, UPI, grid); break;
  }
  if (rc == RAFI_OK) { c->launches += 1; c->fwd_launches += 1; }
  return rc;
}

int launch_plan(Ctx* c, bool fused, unsigned long long* G_out) {
  if (fused)
    k_plan<true><<<1, 256, 0, c->stream>>>(c->Cdev, c->proc * c->L, c->L, c->R, c->cap, c->off_dev, c->plan_dev,
                                           c->ovf_dev, G_out);
  else
    k_plan<false><<<1, 256, 0, c->stream>>>(c->Cdev, c->proc * c->L, c->L, c->R, c->cap, c->off_dev, c->plan_dev,
                                            c->ovf_dev, nullptr);
  RAFI_CK_CUDA(cudaGetLastError());
  c->launches += 1; c->fwd_launches += 1;
  return RAFI_OK;
}

int launch_copy(Ctx* c, int max_chunks) {
  const uint32_t unit = unit_for(c->B, 0);
  const uint32_t UPI = (uint32_t)(c->B / unit);
  int gx = (int)std::max<int64_t>(1, std::min<int64_t>(max_chunks, (int64_t)num_sms(c->device) * 8 / c->L));
  dim3 grid(gx, c->L);
#define COPY_LAUNCH(T_) \
  k_copy<T_><<<grid, kThreads, 0, c->stream>>>(c->runs_dev, rank_table(c), c->R, UPI, c->plan_dev)
  switch (unit) {
    case 16: COPY_LAUNCH(uint4); break;
    case 8: COPY_LAUNCH(uint2); break;
    case 4: COPY_LAUNCH(uint32_t); break;
    case 2: COPY_LAUNCH(uint16_t); break;
    default: COPY_LAUNCH(uint8_t); break;
  }
#undef COPY_LAUNCH
  RAFI_CK_CUDA(cudaGetLastError());
  c->launches += 1; c->fwd_launches += 1;
  return RAFI_OK;
}

int launch_wrapup(Ctx* c) {
  k_wrapup<<<1, 32 * ((c->L + 31) / 32), 0, c->stream>>>(c->ctrl, c->plan_dev, c->L, c->ovf_dev);
  RAFI_CK_CUDA(cudaGetLastError());
  c->launches += 1; c->fwd_launches += 1;
  return RAFI_OK;
}

}  // namespace rafi_impl
