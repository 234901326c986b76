// drivers.cu -- proxy application kernels (include/rafi_drivers.h), written
// only against the public device interface include/rafi_device.cuh.
#include <cuda_runtime.h>

#include <cstdint>

#include "internal.h"
#include "rafi_device.cuh"
#include "rafi_drivers.h"

namespace {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + kGolden;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ int mulshift(uint64_t h, int R) {
  return (int)(((h >> 32) * (uint64_t)R) >> 32);
}

template <int B>
struct Item {
  uint32_t w[B / 4];
};

template <int B>
__device__ __forceinline__ void fill_item(Item<B>& it, uint32_t src, uint32_t rnd, uint64_t id) {
  it.w[0] = src;
  it.w[1] = rnd;
  it.w[2] = (uint32_t)id;
  it.w[3] = (uint32_t)(id >> 32);
#pragma unroll
  for (int k = 0; k < B / 4 - 4; ++k) it.w[4 + k] = (uint32_t)splitmix64(id ^ ((uint64_t)k * kGolden));
}

template <int B>
__global__ void k_drv_emit(rafi_device_view v, int pattern, uint64_t seed, uint32_t rnd, uint64_t n, uint64_t seq0,
                           int target, uint64_t inv_thr) {
  rafi::Queue<Item<B>> q(v);
  const int R = v.num_ranks;
  const uint32_t src = (uint32_t)v.my_rank;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t seq = seq0 + i;
    const uint64_t id = ((uint64_t)src << 40) | seq;
    Item<B> it;
    fill_item<B>(it, src, rnd, id);
    const uint64_t h = splitmix64(seed ^ ((uint64_t)src << 48) ^ ((uint64_t)rnd << 40) ^ seq);
    int d;
    switch (pattern) {
      case RAFI_DRV_UNIFORM: d = mulshift(h, R); break;
      case RAFI_DRV_SELF: d = (int)src; break;
      case RAFI_DRV_RING: d = (int)((src + 1) % R); break;
      case RAFI_DRV_ALL_TO_ONE: d = target; break;
      case RAFI_DRV_ROUND_ROBIN: d = (int)(seq % (uint64_t)R); break;
      default: {  // skewed: stay with p = 0.9, else another rank
        const bool stay = (h >> 32) < 3865470566ull;
        const int nb = R == 1 ? 0 : (int)((src + 1 + (uint32_t)((h & 0xFFFF) % (uint64_t)(R - 1))) % R);
        d = stay ? (int)src : nb;
      }
    }
    if ((h & 0xFFFFFFFFull) < inv_thr) d = (seq & 1) == 0 ? -1 : R;
    q.emitOutgoing(it, d);
  }
}

template <int B>
__global__ void k_drv_walk(rafi_device_view v, uint64_t seed, uint32_t rnd, uint32_t last_round) {
  rafi::Queue<Item<B>> q(v);
  const int R = v.num_ranks;
  const unsigned long long n = q.numIncoming();
  if (rnd > last_round) return;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    Item<B> it = q.getIncoming(i);
    it.w[1] = rnd;
    const uint64_t id = (uint64_t)it.w[2] | ((uint64_t)it.w[3] << 32);
    const uint64_t h = splitmix64(seed ^ ((uint64_t)rnd << 40) ^ id);
    q.emitOutgoing(it, mulshift(h, R));
  }
}

template <int B>
int launch_emit(rafi_impl::Ctx* c, const rafi_device_view& v, int pattern, uint64_t seed, uint32_t rnd, uint64_t n,
                uint64_t seq0, int target, uint64_t thr) {
  const int threads = 256;
  const uint64_t blocks = (n + threads - 1) / threads;
  const int grid = (int)(blocks < 148 * 16 ? (blocks ? blocks : 1) : 148 * 16);
  k_drv_emit<B><<<grid, threads, 0, c->stream>>>(v, pattern, seed, rnd, n, seq0, target, thr);
  return cudaGetLastError() == cudaSuccess ? RAFI_OK : RAFI_ERR_CUDA;
}

template <int B>
int launch_walk(rafi_impl::Ctx* c, const rafi_device_view& v, uint64_t seed, uint32_t rnd, uint32_t last) {
  const int threads = 256;
  const uint64_t n = v.num_in;
  if (!n) return RAFI_OK;
  const uint64_t blocks = (n + threads - 1) / threads;
  const int grid = (int)(blocks < 148 * 16 ? blocks : 148 * 16);
  k_drv_walk<B><<<grid, threads, 0, c->stream>>>(v, seed, rnd, last);
  return cudaGetLastError() == cudaSuccess ? RAFI_OK : RAFI_ERR_CUDA;
}

#define RAFI_DRV_SIZES(X) X(16) X(20) X(24) X(32) X(40) X(44) X(48) X(64) X(96) X(128)

}  // namespace

extern "C" int rafi_drv_emit_synthetic(rafi_ctx* ctx, int local, int pattern, uint64_t seed, uint32_t rnd, uint64_t n,
                                       uint64_t seq0, int target, uint64_t invalid_threshold) {
  auto* c = reinterpret_cast<rafi_impl::Ctx*>(ctx);
  rafi_device_view v;
  int rc = rafi_get_device_view(ctx, local, &v);
  if (rc != RAFI_OK) return rc;
  if (pattern < 0 || pattern > RAFI_DRV_SKEWED) return RAFI_ERR_INVALID_ARG;
  if (n == 0) return RAFI_OK;
  if (cudaSetDevice(c->device) != cudaSuccess) return RAFI_ERR_CUDA;
  c->launches += 1;
  switch (v.item_bytes) {
#define CASE(B) \
  case B: return launch_emit<B>(c, v, pattern, seed, rnd, n, seq0, target, invalid_threshold);
    RAFI_DRV_SIZES(CASE)
#undef CASE
    default: rafi_impl::set_error("rafi_drv_emit_synthetic: unsupported item size"); return RAFI_ERR_UNSUPPORTED;
  }
}

extern "C" int rafi_drv_random_walk(rafi_ctx* ctx, uint64_t seed, uint32_t rnd, uint32_t last_round) {
  auto* c = reinterpret_cast<rafi_impl::Ctx*>(ctx);
  if (!c) return RAFI_ERR_INVALID_ARG;
  if (cudaSetDevice(c->device) != cudaSuccess) return RAFI_ERR_CUDA;
  for (int l = 0; l < c->L; ++l) {
    rafi_device_view v;
    int rc = rafi_get_device_view(ctx, l, &v);
    if (rc != RAFI_OK) return rc;
    switch (v.item_bytes) {
#define CASE(B) \
  case B: rc = launch_walk<B>(c, v, seed, rnd, last_round); break;
      RAFI_DRV_SIZES(CASE)
#undef CASE
      default: rafi_impl::set_error("rafi_drv_random_walk: unsupported item size"); return RAFI_ERR_UNSUPPORTED;
    }
    if (rc != RAFI_OK) return rc;
    if (v.num_in) c->launches += 1;
  }
  return RAFI_OK;
}
