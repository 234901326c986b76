// warp_tiles.cu -- the warp-tile binning path (a2 histogram + a4 stable
// scatter) for R <= 8 destinations and item sizes that are a multiple of 4 B.
//
// The binning tile is 256 items (128 for items of 96 B and more) and ONE WARP
// owns a whole tile, from the TMA load to the last store, so the scatter
// needs no block-level barrier at all:
//
//   k_hist_w     a2  persistent; one warp counts one scan block (8 tiles) at
//                    a time, streamed through a private three-stage ring of
//                    TMA bulk loads: per-lane 4-bit counters, a 31-shuffle
//                    butterfly reduce-scatter that leaves lane j with word j
//                    of the 8 tiles x 8 destinations count table, and the
//                    in-block prefix (O) and block total (H) -- the same
//                    two-level layout k_scan and both scatters read.
//   k_scatter_w  a4  persistent, one CTA per SM of up to 16 independent warps.
//                    Each warp streams its tiles through a private two-stage
//                    ring of 1-D TMA bulk loads (items + dests, mbarrier
//                    completion), ranks the tile's items among same-destination
//                    items in slot order (__match_any_sync and a chunk x
//                    destination table), and writes every
//                    destination run with coalesced 16/8/4-byte unit stores
//                    straight into the destination queue (the local send
//                    batch, the local incoming queue, or -- FUSED -- a peer's
//                    incoming queue over NVLink).
//
// Why (profiles/r02_binning_r8.md): the block-tile scatter of kernels.cu pays
// ~6 __syncthreads per tile; at R = 8 its warps spend a third of their time
// in barriers and the kernel reaches 0.65 of HBM.  Here a warp only ever waits
// for its own data: 0.90-0.96 of HBM for 16-B-multiple items at R = 8.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "devcommon.cuh"
#include "internal.h"

namespace rafi_impl {

// tuning (build-time; paper_2605_30294_b200/build.py variants)
#ifndef RAFI_W_UNROLL
#define RAFI_W_UNROLL 8
#endif
constexpr int kWMaxWarps = 16;
constexpr int kWUnroll = RAFI_W_UNROLL;   // independent unit moves in flight per lane
#ifndef RAFI_W_UNROLL_NARROW
#define RAFI_W_UNROLL_NARROW 8
#endif
constexpr int kWUnrollNarrow = RAFI_W_UNROLL_NARROW;  // the same for the untracked 8/4-byte-unit loop
constexpr uint32_t kWSmemMax = 227u * 1024u;

// ---------------------------------------------------------------- a2 histogram

// Warps per CTA (one CTA per SM) and TMA ring depth per warp, by tile size.
// Measured at R = 8 (fraction of the copy peak, gpurun_out/r02pp_sweep.jsonl):
// 256-item tiles 8 x 3: 0.72, 16 x 1: 0.75, 12 x 1: 0.77; 128-item tiles
// 8 x 3: 0.51, 12 x 2: 0.66, 16 x 1 or 3: 0.74 -- warps in flight, not ring
// depth, hide the load latency here.
#ifndef RAFI_H_WARPS_256
#define RAFI_H_WARPS_256 12
#endif
#ifndef RAFI_H_STAGES_256
#define RAFI_H_STAGES_256 1
#endif
#ifndef RAFI_H_WARPS_128
#define RAFI_H_WARPS_128 16
#endif
#ifndef RAFI_H_STAGES_128
#define RAFI_H_STAGES_128 1
#endif

// dests per scan block: 8 tiles (2048 = 8 KiB at 256-item tiles, 1024 at 128)
template <int kWT>
struct HistBlk {
  static constexpr uint32_t kBlk = kWT * kHistTilesPerCta;
  static constexpr int kPerTile = kWT / 128;  // int4 per lane per tile
  static constexpr int kStages = kWT == 256 ? RAFI_H_STAGES_256 : RAFI_H_STAGES_128;  // TMA ring depth per warp
  static constexpr int kWarps = kWT == 256 ? RAFI_H_WARPS_256 : RAFI_H_WARPS_128;      // warps per CTA
};

template <int kWT>
__host__ __device__ constexpr uint32_t hist_w_smem(int L) {
  return HistBlk<kWT>::kWarps * (HistBlk<kWT>::kStages * HistBlk<kWT>::kBlk * 4 + 64) + 8 * (2 * L + 1);
}

// Small forwards (at most kFuseBlocks scan blocks per rank by capacity): the
// histogram's last CTA also does k_scan's work -- the second scan level, the
// count-matrix rows, the round's counters, and (PEER control) the count
// exchange and the plan -- so a forward is two kernels instead of three.
constexpr uint64_t kFuseBlocks = 64;

struct ScanFuse {
  int on;                       // 0: k_scan runs as its own launch
  int grank0, plan_mode;        // as k_scan: plan_mode 0 none, 1 staged, 2 FUSED
  uint64_t* Cmat;
  unsigned* done;               // last-CTA counter
  uint64_t* dst_off;
  uint64_t* num_in;
  int* ovf;
  unsigned long long* G_out;
};

// Persistent: warp w of CTA x takes scan blocks gw, gw + stride, ... (flat
// over the local ranks), each streamed into its private kHStages-deep ring by
// one 8-KiB TMA bulk load.  Scan block b of local rank l = tiles 8b .. 8b+7.
template <int kWT>
__global__ void __launch_bounds__(HistBlk<kWT>::kWarps * 32, 1) k_hist_w(const RankDev* __restrict__ rk,
                                                             CtrlDev* __restrict__ ctrl, int L, int R,
                                                             uint64_t cap, ScanFuse fz, PeerCtl pc) {
  constexpr uint32_t kHBlk = HistBlk<kWT>::kBlk;
  constexpr int kHStages = HistBlk<kWT>::kStages;
  constexpr int kHWarps = HistBlk<kWT>::kWarps;
  extern __shared__ __align__(128) uint8_t smem[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* my = smem + (size_t)w * (kHStages * kHBlk * 4 + 64);
  uint64_t* mbar = reinterpret_cast<uint64_t*>(my + kHStages * kHBlk * 4);
  uint64_t* bpre = reinterpret_cast<uint64_t*>(smem + kHWarps * (kHStages * kHBlk * 4 + 64));  // [L + 1]
  uint64_t* nl = bpre + (L + 1);
  if (threadIdx.x == 0) {
    uint64_t acc = 0;
    for (int l = 0; l < L; ++l) {
      const uint64_t n = n_items(ctrl[l], cap);
      nl[l] = n;
      bpre[l] = acc;
      acc += (n + kHBlk - 1) / kHBlk;
    }
    bpre[L] = acc;
  }
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < kHStages; ++s) mbar_init(&mbar[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const uint64_t total = bpre[L];
  const uint64_t gw = (uint64_t)blockIdx.x * kHWarps + w, stride = (uint64_t)gridDim.x * kHWarps;
  auto locate = [&](uint64_t g, int* l) {
    int x = 0;
    while (g >= bpre[x + 1]) ++x;
    *l = x;
    return g - bpre[x];
  };
  auto issue = [&](uint32_t it) {
    const uint64_t g = gw + (uint64_t)it * stride;
    if (g >= total) return;
    int l;
    const uint64_t i0 = locate(g, &l) * kHBlk;
    const uint32_t bytes = ((uint32_t)umin64(kHBlk, nl[l] - i0) * 4 + 15) & ~15u;  // queues carry >= 16 B of slack
    uint64_t* bar = &mbar[it % kHStages];
    mbar_expect_tx(bar, bytes);
    bulk_g2s(my + (it % kHStages) * kHBlk * 4, rk[l].dest + i0, bytes, bar);
  };
  if (lane == 0)
    for (int s = 0; s < kHStages; ++s) issue(s);
  for (uint32_t it = 0;; ++it) {
    const uint64_t g = gw + (uint64_t)it * stride;
    if (g >= total) break;
    int l;
    const uint64_t b = locate(g, &l);
    const uint64_t n = nl[l];
    const uint64_t tiles = (n + kWT - 1) / kWT;
    const uint64_t nblk = (tiles + kHistTilesPerCta - 1) / kHistTilesPerCta;
    const uint64_t i0 = b * kHBlk;
    const bool full = i0 + kHBlk <= n;
    mbar_wait(&mbar[it % kHStages], (it / kHStages) & 1);
    const int4* d4 = reinterpret_cast<const int4*>(my + (it % kHStages) * kHBlk * 4);
    // int4 q = 32 i + lane holds dests 4q .. 4q+3, in tile 4q / kWT = i / kPerTile.
    // Per tile, nibble d of c counts destination d among this lane's
    // 4 kPerTile <= 8 dests (every queued dest is in [0, R), R <= 8: invalid
    // ones were rejected at emit) -- one shift and one add per dest -- then
    // widened to 16-bit fields:  word 4t+k holds dests k and k+4
    uint32_t a[32];
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      uint32_t c = 0;
#pragma unroll
      for (int h = 0; h < HistBlk<kWT>::kPerTile; ++h) {
        const int i = HistBlk<kWT>::kPerTile * t + h;
        const int4 v = d4[i * 32 + lane];
        const int e[4] = {v.x, v.y, v.z, v.w};
        if (full) {
#pragma unroll
          for (int m = 0; m < 4; ++m) c += 1u << ((unsigned)e[m] << 2);
        } else {
          const uint64_t e0 = i0 + (uint64_t)(i * 32 + lane) * 4;
#pragma unroll
          for (int m = 0; m < 4; ++m)
            if (e0 + m < n) c += 1u << ((unsigned)e[m] << 2);
        }
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) a[4 * t + k] = (c >> (4 * k)) & 0x000F000Fu;
    }
    __syncwarp();  // every lane has read the stage
    if (lane == 0) {
      fence_proxy_async();
      issue(it + kHStages);
    }
    // butterfly reduce-scatter: at distance s a lane keeps one half of its
    // words (the upper one if bit s of its lane id is set) and adds its
    // partner's copy of that half; after s = 16 .. 1, lane j holds the warp
    // sum of word j
#pragma unroll
    for (int s = 16; s >= 1; s >>= 1) {
      const bool up = (lane & s) != 0;
#pragma unroll
      for (int j = 0; j < s; ++j) {
        const uint32_t send = up ? a[j] : a[j + s];
        const uint32_t keep = up ? a[j + s] : a[j];
        a[j] = keep + __shfl_xor_sync(kFull, send, s);
      }
    }
    const uint32_t x = a[0];  // tile 8b + (lane >> 2), word lane & 3: two 16-bit counts (<= 256 each)
    // prefix over the block's tiles (lanes k, k+4, ..., k+28 share a word)
    uint32_t inc = x;
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, inc, o);
      if (lane >= o) inc += y;
    }
    const uint32_t excl = inc - x;  // <= 2048 per field: no carry
    const uint32_t tot = __shfl_sync(kFull, inc, 28 + (lane & 3));
    const int k = lane & 3;
    const uint64_t t = b * kHistTilesPerCta + (lane >> 2);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int d = k + 4 * h;
      if (d < R) {
        if (t < tiles) rk[l].O[(uint64_t)d * tiles + t] = (excl >> (16 * h)) & 0xffffu;
        if ((lane >> 2) == kHistTilesPerCta - 1) rk[l].H[(uint64_t)d * nblk + b] = (tot >> (16 * h)) & 0xffffu;
      }
    }
  }
  if (!fz.on || !last_block(fz.done)) return;
  // k_scan's work, by the last CTA (every CTA's O/H writes are visible:
  // last_block fences before counting itself in): per (rank, destination)
  // the exclusive prefix of H over the <= kFuseBlocks scan blocks, in place,
  // and the count-matrix row; then the round's counters
  for (int x = threadIdx.x; x < L * R; x += blockDim.x) {
    const int l = x / R, d = x - l * R;
    const uint64_t tiles = (nl[l] + kWT - 1) / kWT;
    const uint64_t nblk = (tiles + kHistTilesPerCta - 1) / kHistTilesPerCta;
    uint32_t* H = rk[l].H + (uint64_t)d * nblk;
    uint64_t acc = 0;
    for (uint64_t b = 0; b < nblk; ++b) {
      const uint32_t v = H[b];
      H[b] = (uint32_t)acc;
      acc += v;
    }
    fz.Cmat[(uint64_t)(fz.grank0 + l) * R + d] = acc;
    if (d == 0) {
      CtrlDev& c = ctrl[l];
      c.n_out = nl[l];
      c.dropped = c.ctr - nl[l];
      c.invalid_last = c.invalid;
    }
  }
  __syncthreads();
  if (fz.plan_mode || pc.mbox) {
    if (pc.mbox && !ctl_counts_block(pc, fz.Cmat, L, R)) {
      // a peer never arrived: move nothing this round (the host reports RAFI_ERR_TIMEOUT)
      if (threadIdx.x == 0) {
        *fz.ovf = 2;
        if (fz.G_out) *fz.G_out = ~0ull;
      }
      return;
    }
    if (fz.plan_mode)
      plan_all(fz.Cmat, fz.grank0, L, R, cap, fz.plan_mode == 2, fz.dst_off, fz.num_in, fz.ovf, fz.G_out);
  }
}

// ---------------------------------------------------------------- a4 scatter

// Shared memory of k_scatter_w: `warps` private warp regions, then the CTA's
// tile map.  Warp region: stages_for(B) x (items, dests), src_of[256] (u16), the
// chunk x destination table T[8][8] (u32), rs[R + 1] (u32), gb[R] (u64),
// mbarriers.
struct WarpLayout {
  uint32_t stage_items, stage_stride;
  uint32_t off_src, off_cnt, off_rs, off_gb, off_mbar, per_warp;
  uint32_t off_cta, total;
};

// TMA ring depth per warp: two stages for 16-byte-unit items up to 96 B;
// one (so twice the warps fit) for narrower units and for larger items --
// there warps in flight beat ring depth (at R = 8: 44 B 0.75 -> 0.83,
// 128 B 0.90 -> 0.94, but 48 B 0.95 -> 0.89 and 96 B 0.94 -> 0.92;
// gpurun_out/r02rr_sweep.jsonl, r02ss_sweep.jsonl).
static int stages_for(uint64_t B) { return (B % 16 == 0 && B <= 96) ? 2 : 1; }

static WarpLayout warp_layout(uint32_t kWT, uint64_t B, int R, int L, int warps) {
  const int kWStages = stages_for(B);
  auto al = [](uint64_t x, uint64_t a) { return (uint32_t)((x + a - 1) / a * a); };
  WarpLayout s;
  s.stage_items = al((uint64_t)kWT * B, 16);
  s.stage_stride = al((uint64_t)s.stage_items + 4ull * kWT, 128);
  uint32_t o = kWStages * s.stage_stride;
  s.off_src = o; o += 2 * kWT;
  s.off_cnt = o; o += 4 * (kWT / 32) * 8;
  s.off_rs = o; o = al(o + 4ull * (R + 1), 8);
  s.off_gb = o; o += 8 * R;
  s.off_mbar = o; o += 8 * kWStages;
  s.per_warp = al(o, 128);
  s.off_cta = s.per_warp * warps;
  s.total = al(s.off_cta + 8ull * (2 * L + 1), 16);
  return s;
}

static int warps_that_fit(uint32_t kWT, uint64_t B, int R, int L) {
  int w = 0;
  while (w < kWMaxWarps && warp_layout(kWT, B, R, L, w + 1).total <= kWSmemMax) ++w;
  return w;
}

// Unit stores into a destination queue (local HBM or a CUDA-IPC peer
// mapping: both in the global window), issued as STG rather than generic ST.
__device__ __forceinline__ void st_global(uint4* p, const uint4& v) {
  asm volatile("st.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ void st_global(uint2* p, const uint2& v) {
  asm volatile("st.global.v2.u32 [%0], {%1, %2};" ::"l"(p), "r"(v.x), "r"(v.y) : "memory");
}
__device__ __forceinline__ void st_global(uint32_t* p, const uint32_t& v) {
  asm volatile("st.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <typename U, int kWT, int kWStages>
__global__ void __launch_bounds__(kWMaxWarps * 32, 1)
k_scatter_w(const RankDev* __restrict__ rk, const CtrlDev* __restrict__ ctrl, uint8_t* const* __restrict__ dst_table,
            const uint64_t* __restrict__ dst_off, const int* __restrict__ ovf, int L, int R, uint64_t cap, int cur,
            uint32_t B, uint32_t UPI, FastDiv divU, WarpLayout lay, unsigned* __restrict__ wrap_done,
            CtrlDev* __restrict__ ctrl_w, const uint64_t* __restrict__ wrap_num_in, PeerCtl pc) {
  if (ovf && *ovf) return;  // collective receive overflow: move nothing (Z3)
  constexpr int kWK = kWT / 32;  // items per lane of a warp tile
  extern __shared__ __align__(128) uint8_t smem[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, W = blockDim.x >> 5;
  // tile map: tpre[l] = first flat tile of local rank l (tpre[L] = all), nl[l] = its items
  uint64_t* tpre = reinterpret_cast<uint64_t*>(smem + lay.off_cta);
  uint64_t* nl = tpre + (L + 1);
  uint8_t* my = smem + (size_t)w * lay.per_warp;
  uint64_t* mbar = reinterpret_cast<uint64_t*>(my + lay.off_mbar);
  uint16_t* src_of = reinterpret_cast<uint16_t*>(my + lay.off_src);
  uint32_t* T = reinterpret_cast<uint32_t*>(my + lay.off_cnt);  // [chunk k][destination e]
  uint32_t* rs = reinterpret_cast<uint32_t*>(my + lay.off_rs);
  uintptr_t* gb = reinterpret_cast<uintptr_t*>(my + lay.off_gb);
  if (threadIdx.x == 0) {
    uint64_t acc = 0;
    for (int l = 0; l < L; ++l) {
      const uint64_t n = n_items(ctrl[l], cap);
      nl[l] = n;
      tpre[l] = acc;
      acc += (n + kWT - 1) / kWT;
    }
    tpre[L] = acc;
  }
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < kWStages; ++s) mbar_init(&mbar[s], 1);
    fence_mbar_init();
  }
  __syncthreads();  // the only CTA barrier before the epilogue
  const uint64_t gw = (uint64_t)blockIdx.x * W + w, stride = (uint64_t)gridDim.x * W;
  // The warp's tiles are gw, gw + stride, ... (flat over the local ranks); a
  // cursor walks them with a monotone local-rank search.  Three cursors: the
  // TMA loads (kWStages ahead), the run-base fetch (one ahead), the tile.
  struct Cursor {
    uint64_t g;
    int l;
  };
  auto seek = [&](Cursor& c) {
    while (c.l < L && c.g >= tpre[c.l + 1]) ++c.l;
  };
  auto advance = [&](Cursor& c) {
    c.g += stride;
    seek(c);
  };
  Cursor ci{gw, 0}, cf{gw, 0}, ct{gw, 0};
  seek(ci);
  seek(cf);
  seek(ct);
  uint32_t n_issued = 0;
  auto issue = [&]() {  // lane 0: start loading the tile at ci into stage n_issued % kWStages
    if (ci.l < L) {
      const int l = ci.l;
      const uint64_t t0 = (ci.g - tpre[l]) * kWT;
      const uint32_t nt = (uint32_t)umin64(kWT, nl[l] - t0);
      uint8_t* st = my + (n_issued % kWStages) * lay.stage_stride;
      uint64_t* bar = &mbar[n_issued % kWStages];
      const uint32_t bi = (nt * B + 15) & ~15u, bd = (nt * 4 + 15) & ~15u;  // queues carry >= 16 B of slack
      mbar_expect_tx(bar, bi + bd);
      bulk_g2s(st, rk[l].out + t0 * B, bi, bar);
      bulk_g2s(st + lay.stage_items, rk[l].dest + t0, bd, bar);
    }
    ++n_issued;
    advance(ci);
  };
  if (lane == 0)
    for (int s = 0; s < kWStages; ++s) issue();

  // lane d < R: global start of destination d's run in the cursor's tile
  // -- prefix over earlier tiles (O within the scan block + H over blocks)
  // plus the per-destination base from the plan -- and d's queue.  Fetched one
  // tile ahead, so these dependent global loads are in flight while the
  // current tile is ranked and written.
  // (The three terms stay apart until the next iteration adds them: an add
  // here would stall the warp on the loads right away.)
  struct RunBase {
    uint32_t o, h;
    uint64_t off;
    uintptr_t db;
  };
  auto fetch = [&](RunBase* r) {
    if (cf.l < L && lane < R) {
      const int l = cf.l;
      const uint64_t t = cf.g - tpre[l];
      const uint64_t tiles = tpre[l + 1] - tpre[l];
      const uint64_t nblk = (tiles + kHistTilesPerCta - 1) / kHistTilesPerCta;
      r->o = rk[l].O[(uint64_t)lane * tiles + t];
      r->h = rk[l].H[(uint64_t)lane * nblk + t / kHistTilesPerCta];
      r->off = dst_off[(uint64_t)l * R + lane];
      r->db = reinterpret_cast<uintptr_t>(dst_table ? dst_table[lane] : rk[l].binned[cur]);
    }
    advance(cf);
  };
  RunBase nxt{0u, 0u, 0ull, 0};
  fetch(&nxt);

  for (uint32_t it = 0; ct.l < L; ++it, advance(ct)) {
    const int l = ct.l;
    const uint64_t t = ct.g - tpre[l];
    const uint32_t nt = (uint32_t)umin64(kWT, nl[l] - t * kWT);
    const RunBase cur_rb = nxt;
    fetch(&nxt);
    for (int x = lane; x < kWK * 8; x += 32) T[x] = 0;  // kWK chunks x 8 destinations
    __syncwarp();
    const uint32_t s = it % kWStages;
    mbar_wait(&mbar[s], (it / kWStages) & 1);
    const uint8_t* st = my + s * lay.stage_stride;
    const int32_t* dest_s = reinterpret_cast<const int32_t*>(st + lay.stage_items);
    // rank (stable in slot order): item 32k + lane (chunk k)
    // goes to tile position T[k][d] + (earlier lanes of chunk k with the same
    // destination d), where T[k][d] = start of run d in the tile + items with
    // destination d in chunks 0 .. k-1.  Three warp-synchronous steps, no
    // serial chain over the chunks: the chunk leaders publish their group
    // sizes, lane e (< R) scans destination e over the chunks, the run starts
    // come from a shuffle scan over the destinations.
    int dk[kWK];
    unsigned mk[kWK];
    uint32_t before[kWK];
#pragma unroll
    for (int k = 0; k < kWK; ++k) {
      const uint32_t il = k * 32 + lane;
      dk[k] = il < nt ? dest_s[il] : R;
      mk[k] = __match_any_sync(kFull, dk[k]);
      before[k] = __popc(mk[k] & lanemask_lt());
    }
#pragma unroll
    for (int k = 0; k < kWK; ++k)
      if (dk[k] < R && before[k] == 0) T[k * 8 + dk[k]] = __popc(mk[k]);
    __syncwarp();
    uint32_t pre[kWK];
    uint32_t tot = 0;
    if (lane < R) {
#pragma unroll
      for (int k = 0; k < kWK; ++k) {
        pre[k] = tot;
        tot += T[k * 8 + lane];
      }
    }
    uint32_t inc = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, inc, o);
      if (lane >= o) inc += y;
    }
    const uint32_t excl = inc - tot;  // run start of destination lane (rs[R] = nt)
    if (lane <= R) rs[lane] = excl;
    if (lane < R) {
      // position p of run d goes to gb[d] + p * B
      gb[lane] = cur_rb.db + (uintptr_t)((uint64_t)cur_rb.o + cur_rb.h + cur_rb.off - excl) * B;
#pragma unroll
      for (int k = 0; k < kWK; ++k) T[k * 8 + lane] = excl + pre[k];
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < kWK; ++k)
      if (dk[k] < R) src_of[T[k * 8 + dk[k]] + before[k]] = (uint16_t)((k * 32 + lane) | (dk[k] << 8));
    __syncwarp();
    // destination-major unit moves: lane x of 32 consecutive units, so every
    // run is written with coalesced stores.  src_of[p] carries the source
    // slot (low 8 bits) and the destination (high bits) of position p, so a
    // unit needs no run tracking: its address is gb[d] + p * B + u * |U|.
    const U* sU = reinterpret_cast<const U*>(st);
    const uint32_t units = nt * UPI;
    if (sizeof(U) == 16 || UPI <= 3) {
      // 16-byte units and items of at most three units: a lane's position
      // only grows, so it tracks its run (one compare per unit) -- cheaper
      // here than a third shared load per unit (at R = 8: 48 B 0.95 vs 0.91,
      // 24 B 0.86 vs 0.80 of HBM)
      int d = 0;
      uint32_t nb = rs[1];
      uintptr_t base = gb[0];
      for (uint32_t xb = lane; xb < units; xb += 32 * kWUnroll) {
        U v[kWUnroll];
        uint32_t p[kWUnroll], u[kWUnroll];
#pragma unroll
        for (int j = 0; j < kWUnroll; ++j) {
          const uint32_t x = xb + 32 * j;
          p[j] = divU.div(x);
          u[j] = x - p[j] * UPI;
          if (x < units) v[j] = sU[(src_of[p[j]] & 0xffu) * UPI + u[j]];
        }
#pragma unroll
        for (int j = 0; j < kWUnroll; ++j) {
          if (xb + 32 * j < units) {
            while (p[j] >= nb) {
              ++d;
              nb = rs[d + 1];
              base = gb[d];
            }
            RAFI_DCHECK(d < R, "warp scatter: position beyond the last run");
            st_global(reinterpret_cast<U*>(base + (uintptr_t)p[j] * B) + u[j], v[j]);
          }
        }
      }
    } else {
    // 8- and 4-byte units, more than three per item: no run tracking, the
    // destination comes with the source slot (at R = 8: 20 B 0.64 -> 0.87,
    // 40 B 0.78 -> 0.83, 44 B 0.50 -> 0.76 of HBM)
    uint32_t x0 = lane;
    for (; x0 + 32 * (kWUnrollNarrow - 1) < units; x0 += 32 * kWUnrollNarrow) {  // whole batches: no bounds checks
      U v[kWUnrollNarrow];
      uint32_t p[kWUnrollNarrow], u[kWUnrollNarrow], inf[kWUnrollNarrow];
#pragma unroll
      for (int j = 0; j < kWUnrollNarrow; ++j) {
        const uint32_t x = x0 + 32 * j;
        p[j] = divU.div(x);
        u[j] = x - p[j] * UPI;
        inf[j] = src_of[p[j]];
        v[j] = sU[(inf[j] & 0xffu) * UPI + u[j]];
      }
#pragma unroll
      for (int j = 0; j < kWUnrollNarrow; ++j) {
        RAFI_DCHECK((inf[j] >> 8) < (uint32_t)R && p[j] >= rs[inf[j] >> 8] && p[j] < rs[(inf[j] >> 8) + 1],
                    "warp scatter: position outside its run");
        st_global(reinterpret_cast<U*>(gb[inf[j] >> 8] + (uintptr_t)p[j] * B) + u[j], v[j]);
      }
    }
    for (; x0 < units; x0 += 32) {  // the tile's last units
      const uint32_t p = divU.div(x0), u = x0 - p * UPI, inf = src_of[p];
      RAFI_DCHECK((inf >> 8) < (uint32_t)R, "warp scatter: position beyond the last run");
      st_global(reinterpret_cast<U*>(gb[inf >> 8] + (uintptr_t)p * B) + u, sU[(inf & 0xffu) * UPI + u]);
    }
    }
    __syncwarp();  // every lane is done with this stage
    if (lane == 0) {
      fence_proxy_async();  // order the generic-proxy reads before the async refill
      issue();
    }
  }
  if (dst_table) __threadfence_system();  // pushes to peer memory complete before the kernel does
  // wrap-up epilogue by the last CTA: every CTA has finished
  // reading the emit counters, so they can be reset for the next round
  if (wrap_done && last_block(wrap_done)) {
    for (int l2 = threadIdx.x; l2 < L; l2 += blockDim.x) {
      ctrl_w[l2].ctr = 0;
      ctrl_w[l2].invalid = 0;
      ctrl_w[l2].num_in = wrap_num_in[l2];
    }
    if (pc.mbox) ctl_barrier_block(pc);
  }
}

// ---------------------------------------------------------------- host side

bool warp_tiles_ok(uint32_t tile, uint64_t B, int R, int L) {
  return (tile == 128 || tile == 256) && R <= 8 && B % 4 == 0 && warps_that_fit(tile, B, R, L) >= 2;
}

// 256-item tiles while they leave >= 6 warps per SM (with stages_for(): up to
// 128-B items), else 128 while >= 4 warps fit (up to 256 B).  Measured with
// two stages everywhere (gpurun_out/r02n_sweep.jsonl): at <= 64 B the
// 256-item tiles win, 0.93-0.95 vs 0.84-0.89, and their histogram streams
// 8-KiB blocks; with one stage, 128-B items at 256 items per tile reach 0.94
// (r02ss).  0 = the warp-tile path does not apply.
uint32_t warp_tile_for(uint64_t B, int R, int L) {
  if (!(R <= 8 && B % 4 == 0)) return 0;
  if (warps_that_fit(256, B, R, L) >= 6) return 256;
  if (warps_that_fit(128, B, R, L) >= 4) return 128;  // else (items > 256 B) block tiles
  return 0;
}

bool hist_w_fuses_scan(const Ctx* c) {
  return (c->max_tiles + kHistTilesPerCta - 1) / kHistTilesPerCta <= kFuseBlocks;
}

template <int kWT>
static int launch_hist_t(Ctx* c, int nsm, int plan_mode, unsigned long long* G_out, PeerCtl pc) {
  const uint32_t sm = hist_w_smem<kWT>(c->L);
  RAFI_CK_CUDA(ensure_smem((const void*)k_hist_w<kWT>, (int)sm, c->device));
  const uint64_t blocks = (c->max_tiles + kHistTilesPerCta - 1) / kHistTilesPerCta * (uint64_t)c->L;
  constexpr int kHWarps = HistBlk<kWT>::kWarps;
  const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)nsm, (blocks + kHWarps - 1) / kHWarps));
  ScanFuse fz;
  fz.on = hist_w_fuses_scan(c) ? 1 : 0;
  fz.grank0 = c->proc * c->L;
  fz.plan_mode = plan_mode;
  fz.Cmat = c->Cdev;
  fz.done = c->done_dev;  // k_scan's last-block counter (k_scan is not launched then)
  fz.dst_off = c->off_dev;
  fz.num_in = c->plan_dev;
  fz.ovf = c->ovf_dev;
  fz.G_out = G_out;
  k_hist_w<kWT><<<grid, kHWarps * 32, sm, c->stream>>>(c->rank_dev, c->ctrl, c->L, c->R, c->cap, fz, pc);
  RAFI_CK_CUDA(cudaGetLastError());
  return RAFI_OK;
}

int launch_hist_w(Ctx* c, int nsm, int plan_mode, unsigned long long* G_out, PeerCtl pc) {
  return c->tile == 128 ? launch_hist_t<128>(c, nsm, plan_mode, G_out, pc)
                        : launch_hist_t<256>(c, nsm, plan_mode, G_out, pc);
}

template <typename U, int kWT, int kS>
static int launch_w(Ctx* c, bool fused, bool wrap, PeerCtl pc, int nsm) {
  const int warps = warps_that_fit(kWT, c->B, c->R, c->L);
  const WarpLayout lay = warp_layout(kWT, c->B, c->R, c->L, warps);
  auto k = k_scatter_w<U, kWT, kS>;
  RAFI_CK_CUDA(ensure_smem((const void*)k, (int)lay.total, c->device));
  const uint32_t UPI = (uint32_t)(c->B / sizeof(U));
  const uint64_t tiles_all = c->max_tiles * (uint64_t)c->L;
  const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)nsm, (tiles_all + warps - 1) / warps));
  k<<<grid, 32 * warps, lay.total, c->stream>>>(c->rank_dev, c->ctrl, fused ? c->in_table_dev : nullptr, c->off_dev,
                                               fused ? c->ovf_dev : nullptr, c->L, c->R, c->cap, c->cur,
                                               (uint32_t)c->B, UPI, FastDiv(UPI), lay, wrap ? c->done_dev + 1 : nullptr,
                                               c->ctrl, c->plan_dev, pc);
  RAFI_CK_CUDA(cudaGetLastError());
  return RAFI_OK;
}

// Units: the widest of 16 / 8 / 4 bytes dividing the item size.  (A 16-byte
// chunk gather for 4-byte-unit items -- each lane assembling an aligned chunk
// from the words of the one or two items it covers -- was measured and
// dropped: 44 B at R = 8, 0.53 vs 0.76 of HBM with plain 4-byte units.)
int launch_scatter_w(Ctx* c, bool fused, bool wrap, PeerCtl pc, int nsm) {
  const bool two = stages_for(c->B) == 2;  // only for 16-byte units
  if (c->tile == 128)
    return c->B % 16 == 0  ? (two ? launch_w<uint4, 128, 2>(c, fused, wrap, pc, nsm)
                                  : launch_w<uint4, 128, 1>(c, fused, wrap, pc, nsm))
           : c->B % 8 == 0 ? launch_w<uint2, 128, 1>(c, fused, wrap, pc, nsm)
                           : launch_w<uint32_t, 128, 1>(c, fused, wrap, pc, nsm);
  return c->B % 16 == 0  ? (two ? launch_w<uint4, 256, 2>(c, fused, wrap, pc, nsm)
                                : launch_w<uint4, 256, 1>(c, fused, wrap, pc, nsm))
         : c->B % 8 == 0 ? launch_w<uint2, 256, 1>(c, fused, wrap, pc, nsm)
                         : launch_w<uint32_t, 256, 1>(c, fused, wrap, pc, nsm);
}

}  // namespace rafi_impl
