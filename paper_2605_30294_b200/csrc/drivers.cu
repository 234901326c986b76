// drivers.cu -- proxy application kernels (include/rafi_drivers.h), written
// only against the public device interface include/rafi_device.cuh.
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

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

// Device re-emit of a resident batch.  kBatch == 1: one emitOutgoing(item,
// dest) per item (one warp atomic per 32 items); kBatch > 1: each thread
// emits kBatch items with the batched emitOutgoing (one warp atomic per
// 32 * kBatch items).  Thread t of a block-chunk handles items t, t + blockDim,
// ... so the loads of each k are coalesced.
template <int B, int kBatch>
__global__ void __launch_bounds__(256) k_drv_emit_items(rafi_device_view v, const uint8_t* __restrict__ items,
                                                        const int32_t* __restrict__ dests, uint64_t n) {
  rafi::Queue<Item<B>> q(v);
  const uint64_t chunk = (uint64_t)blockDim.x * kBatch;
  for (uint64_t c0 = blockIdx.x * chunk; c0 < n; c0 += (uint64_t)gridDim.x * chunk) {
    if (kBatch == 1) {
      const uint64_t i = c0 + threadIdx.x;
      if (i < n) q.emitOutgoing(rafi::load_item<Item<B>>(items + i * B), dests[i]);
      continue;
    }
    Item<B> it[kBatch];
    int d[kBatch];
    int cnt = 0;
#pragma unroll
    for (int k = 0; k < kBatch; ++k) {
      const uint64_t i = c0 + (uint64_t)k * blockDim.x + threadIdx.x;
      if (i < n) {
        it[k] = rafi::load_item<Item<B>>(items + i * B);
        d[k] = dests[i];
        cnt = k + 1;
      }
    }
    q.emitOutgoing<kBatch>(it, d, cnt);
  }
}

// Threads to launch for an app step over the incoming queue: the host-known
// count, or the capacity when the count lives only on the device -- after
// rafi_forward_async / graph replays, and whenever the launch is being
// captured into a graph (a replay must cover whatever count the device holds
// then; the kernels read numIncoming from num_in_dev).
uint64_t launch_count(const rafi_impl::Ctx* c, const rafi_device_view& v) {
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  if (c->stream && cudaStreamIsCapturing(c->stream, &st) != cudaSuccess) { cudaGetLastError(); st = cudaStreamCaptureStatusNone; }
  const bool device_count = c->host_stale || st != cudaStreamCaptureStatusNone;
  return device_count ? (c->cap ? c->cap : 1) : v.num_in;
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
  const uint64_t n = launch_count(c, v);
  if (!n) return RAFI_OK;
  const uint64_t blocks = (n + threads - 1) / threads;
  const int grid = (int)(blocks < 148 * 16 ? blocks : 148 * 16);
  k_drv_walk<B><<<grid, threads, 0, c->stream>>>(v, seed, rnd, last);
  return cudaGetLastError() == cudaSuccess ? RAFI_OK : RAFI_ERR_CUDA;
}

// ------------------------------------------------------------------ proxies
// Float arithmetic below is + - * / sqrt only; this file is compiled with
// -fmad=false (IEEE-exact, no contraction) so the CPU twin matches bit for bit.

constexpr float kTwoM24 = 5.9604644775390625e-08f;  // 2^-24

__device__ __forceinline__ float u24(uint64_t h) { return (float)(uint32_t)(h >> 40) * kTwoM24; }

struct Grid3 {
  int gx, gy, gz;
  __device__ __forceinline__ int clampi(int v, int hi) const { return v < 0 ? 0 : (v > hi ? hi : v); }
  __device__ __forceinline__ int owner(float x, float y, float z) const {
    const int cx = clampi((int)(x * (float)gx), gx - 1);
    const int cy = clampi((int)(y * (float)gy), gy - 1);
    const int cz = clampi((int)(z * (float)gz), gz - 1);
    return (cz * gy + cy) * gx + cx;
  }
  __device__ __forceinline__ void cell(int r, int* cx, int* cy, int* cz) const {
    *cx = r % gx;
    *cy = (r / gx) % gy;
    *cz = r / (gx * gy);
  }
};

__device__ __forceinline__ bool inside(float x, float y, float z) {
  return x >= 0.0f && x < 1.0f && y >= 0.0f && y < 1.0f && z >= 0.0f && z < 1.0f;
}

struct Particle {
  uint32_t id;
  float x, y, z;
};
static_assert(sizeof(Particle) == 16, "particle");

struct Ray {
  float ox, oy, oz, dx, dy, dz, t;
  uint32_t id;
  float integral;
  uint32_t rng, bounces, pad;
};
static_assert(sizeof(Ray) == 48, "ray");

__device__ __forceinline__ void seed_pos(uint64_t seed, uint32_t id, const Grid3& G, int r, float* x, float* y,
                                         float* z) {
  int cx, cy, cz;
  G.cell(r, &cx, &cy, &cz);
  *x = ((float)cx + u24(splitmix64(seed ^ ((uint64_t)id << 3) ^ 0ull))) / (float)G.gx;
  *y = ((float)cy + u24(splitmix64(seed ^ ((uint64_t)id << 3) ^ 1ull))) / (float)G.gy;
  *z = ((float)cz + u24(splitmix64(seed ^ ((uint64_t)id << 3) ^ 2ull))) / (float)G.gz;
}

__device__ __forceinline__ void unit_dir(float ax, float ay, float az, float* dx, float* dy, float* dz) {
  const float len2 = ax * ax + ay * ay + az * az;
  if (len2 < 1e-6f) { *dx = 1.0f; *dy = 0.0f; *dz = 0.0f; return; }
  const float len = sqrtf(len2);
  *dx = ax / len; *dy = ay / len; *dz = az / len;
}

__global__ void k_advect_seed(rafi_device_view v, uint64_t n, uint64_t seed, Grid3 G) {
  rafi::Queue<Particle> q(v);
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    Particle p;
    p.id = (uint32_t)((uint64_t)v.my_rank * n + i);
    seed_pos(seed, p.id, G, v.my_rank, &p.x, &p.y, &p.z);
    q.emitOutgoing(p, G.owner(p.x, p.y, p.z));
  }
}

__device__ __forceinline__ void field(float omega, float eps, float x, float y, float* vx, float* vy, float* vz) {
  *vx = -(omega * (y - 0.5f));
  *vy = omega * (x - 0.5f);
  *vz = eps;
}

__global__ void k_advect_step(rafi_device_view v, uint32_t rnd, uint32_t max_rounds, float omega, float eps, float h,
                              Grid3 G) {
  rafi::Queue<Particle> q(v);
  const unsigned long long n = q.numIncoming();
  const float hh = 0.5f * h, h6 = h / 6.0f;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    Particle p = q.getIncoming(i);
    float k1x, k1y, k1z, k2x, k2y, k2z, k3x, k3y, k3z, k4x, k4y, k4z;
    field(omega, eps, p.x, p.y, &k1x, &k1y, &k1z);
    field(omega, eps, p.x + hh * k1x, p.y + hh * k1y, &k2x, &k2y, &k2z);
    field(omega, eps, p.x + hh * k2x, p.y + hh * k2y, &k3x, &k3y, &k3z);
    field(omega, eps, p.x + h * k3x, p.y + h * k3y, &k4x, &k4y, &k4z);
    p.x = p.x + h6 * (((k1x + 2.0f * k2x) + 2.0f * k3x) + k4x);
    p.y = p.y + h6 * (((k1y + 2.0f * k2y) + 2.0f * k3y) + k4y);
    p.z = p.z + h6 * (((k1z + 2.0f * k2z) + 2.0f * k3z) + k4z);
    if (!inside(p.x, p.y, p.z) || rnd >= max_rounds) continue;  // retires
    q.emitOutgoing(p, G.owner(p.x, p.y, p.z));
  }
}

__global__ void k_march_seed(rafi_device_view v, uint64_t n, uint64_t seed, Grid3 G) {
  rafi::Queue<Ray> q(v);
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    Ray r;
    r.id = (uint32_t)((uint64_t)v.my_rank * n + i);
    seed_pos(seed, r.id, G, v.my_rank, &r.ox, &r.oy, &r.oz);
    const uint64_t b = seed ^ ((uint64_t)r.id << 3);
    const float ax = 2.0f * u24(splitmix64(b ^ 3ull)) - 1.0f;
    const float ay = 2.0f * u24(splitmix64(b ^ 4ull)) - 1.0f;
    const float az = 2.0f * u24(splitmix64(b ^ 5ull)) - 1.0f;
    unit_dir(ax, ay, az, &r.dx, &r.dy, &r.dz);
    r.t = 0.0f;
    r.integral = 0.0f;
    r.rng = (uint32_t)splitmix64(b ^ 6ull);
    r.bounces = 0;
    r.pad = 0;
    q.emitOutgoing(r, G.owner(r.ox, r.oy, r.oz));
  }
}

__global__ void k_march_step(rafi_device_view v, uint64_t seed, uint32_t p_thr, uint32_t max_bounces,
                             uint32_t max_steps, Grid3 G, float* result) {
  rafi::Queue<Ray> q(v);
  const unsigned long long n = q.numIncoming();
  const int me = v.my_rank;
  const float D = 0.00390625f;  // 1/256
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    Ray r = q.getIncoming(i);
    int dest = me;
    bool retired = false;
    for (uint32_t s = 0; s < max_steps; ++s) {
      r.ox = r.ox + D * r.dx;
      r.oy = r.oy + D * r.dy;
      r.oz = r.oz + D * r.dz;
      r.t = r.t + D;
      if (!inside(r.ox, r.oy, r.oz)) { retired = true; break; }
      const int o = G.owner(r.ox, r.oy, r.oz);
      if (o != me) { dest = o; break; }
      const int ix = G.clampi((int)(r.ox * 128.0f), 127), iy = G.clampi((int)(r.oy * 128.0f), 127),
                iz = G.clampi((int)(r.oz * 128.0f), 127);
      const uint64_t hv = splitmix64(seed ^ ((uint64_t)ix << 42) ^ ((uint64_t)iy << 21) ^ (uint64_t)iz);
      r.integral = r.integral + u24(hv) * D;
      const uint64_t hr = splitmix64(((uint64_t)r.id << 32) | r.rng);
      r.rng = (uint32_t)(hr >> 32);
      if ((uint32_t)hr < p_thr) {
        r.bounces += 1;
        if (r.bounces > max_bounces) { retired = true; break; }
        const float ax = 2.0f * u24(splitmix64(hr ^ 1ull)) - 1.0f;
        const float ay = 2.0f * u24(splitmix64(hr ^ 2ull)) - 1.0f;
        const float az = 2.0f * u24(splitmix64(hr ^ 3ull)) - 1.0f;
        unit_dir(ax, ay, az, &r.dx, &r.dy, &r.dz);
      }
    }
    if (retired) result[r.id] = r.integral;
    else q.emitOutgoing(r, dest);
  }
}

template <class K, class... A>
int launch_grid(rafi_impl::Ctx* c, uint64_t n, K kernel, A... args) {
  if (!n) return RAFI_OK;
  const uint64_t blocks = (n + 255) / 256;
  const int grid = (int)(blocks < 148 * 16 ? blocks : 148 * 16);
  kernel<<<grid, 256, 0, c->stream>>>(args...);
  c->launches += 1;
  return cudaGetLastError() == cudaSuccess ? RAFI_OK : RAFI_ERR_CUDA;
}

int check_grid(rafi_impl::Ctx* c, int gx, int gy, int gz) {
  if (gx < 1 || gy < 1 || gz < 1 || gx * gy * gz != c->R) {
    rafi_impl::set_error("proxy grid gx*gy*gz must equal the number of ranks");
    return RAFI_ERR_INVALID_ARG;
  }
  return RAFI_OK;
}

#define RAFI_DRV_SIZES(X) X(16) X(20) X(24) X(32) X(40) X(44) X(48) X(64) X(96) X(128)
#define RAFI_DRV_ITEM_SIZES(X) X(4) X(8) X(12) RAFI_DRV_SIZES(X)

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

extern "C" int rafi_drv_emit_items(rafi_ctx* ctx, int local, const void* items, const int32_t* dests, uint64_t n,
                                   int batch) {
  auto* c = reinterpret_cast<rafi_impl::Ctx*>(ctx);
  rafi_device_view v;
  int rc = rafi_get_device_view(ctx, local, &v);
  if (rc != RAFI_OK) return rc;
  if (n == 0) return RAFI_OK;
  if (!items || !dests || ((uintptr_t)items & 15) || (batch != 1 && batch != 8)) return RAFI_ERR_INVALID_ARG;
  if (cudaSetDevice(c->device) != cudaSuccess) return RAFI_ERR_CUDA;
  const uint64_t blocks = (n + 256ull * batch - 1) / (256ull * batch);
  const int grid = (int)(blocks < 148 * 8 ? blocks : 148 * 8);
  const uint8_t* it = static_cast<const uint8_t*>(items);
  switch (v.item_bytes) {
#define CASE(B)                                                                                        \
  case B:                                                                                              \
    if (batch == 1) k_drv_emit_items<B, 1><<<grid, 256, 0, c->stream>>>(v, it, dests, n);            \
    else k_drv_emit_items<B, 8><<<grid, 256, 0, c->stream>>>(v, it, dests, n);                       \
    break;
    RAFI_DRV_ITEM_SIZES(CASE)
#undef CASE
    default: rafi_impl::set_error("rafi_drv_emit_items: unsupported item size"); return RAFI_ERR_UNSUPPORTED;
  }
  c->launches += 1;
  return cudaGetLastError() == cudaSuccess ? RAFI_OK : RAFI_ERR_CUDA;
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
    if (launch_count(c, v)) c->launches += 1;
  }
  return RAFI_OK;
}

extern "C" int rafi_drv_advect_seed(rafi_ctx* ctx, int local, uint64_t n, uint64_t seed, int gx, int gy, int gz) {
  auto* c = reinterpret_cast<rafi_impl::Ctx*>(ctx);
  if (!c) return RAFI_ERR_INVALID_ARG;
  rafi_device_view v;
  int rc = rafi_get_device_view(ctx, local, &v);
  if (rc != RAFI_OK) return rc;
  if (v.item_bytes != sizeof(Particle)) return RAFI_ERR_INVALID_ARG;
  if ((rc = check_grid(c, gx, gy, gz)) != RAFI_OK) return rc;
  if (cudaSetDevice(c->device) != cudaSuccess) return RAFI_ERR_CUDA;
  return launch_grid(c, n, k_advect_seed, v, n, seed, Grid3{gx, gy, gz});
}

extern "C" int rafi_drv_advect_step(rafi_ctx* ctx, uint32_t rnd, uint32_t max_rounds, float omega, float eps, float h,
                                    int gx, int gy, int gz) {
  auto* c = reinterpret_cast<rafi_impl::Ctx*>(ctx);
  if (!c) return RAFI_ERR_INVALID_ARG;
  int rc = check_grid(c, gx, gy, gz);
  if (rc != RAFI_OK) return rc;
  if (c->B != sizeof(Particle)) return RAFI_ERR_INVALID_ARG;
  if (cudaSetDevice(c->device) != cudaSuccess) return RAFI_ERR_CUDA;
  for (int l = 0; l < c->L; ++l) {
    rafi_device_view v;
    if ((rc = rafi_get_device_view(ctx, l, &v)) != RAFI_OK) return rc;
    if ((rc = launch_grid(c, launch_count(c, v), k_advect_step, v, rnd, max_rounds, omega, eps, h, Grid3{gx, gy, gz})))
      return rc;
  }
  return RAFI_OK;
}

extern "C" int rafi_drv_march_seed(rafi_ctx* ctx, int local, uint64_t n, uint64_t seed, int gx, int gy, int gz) {
  auto* c = reinterpret_cast<rafi_impl::Ctx*>(ctx);
  if (!c) return RAFI_ERR_INVALID_ARG;
  rafi_device_view v;
  int rc = rafi_get_device_view(ctx, local, &v);
  if (rc != RAFI_OK) return rc;
  if (v.item_bytes != sizeof(Ray)) return RAFI_ERR_INVALID_ARG;
  if ((rc = check_grid(c, gx, gy, gz)) != RAFI_OK) return rc;
  if (cudaSetDevice(c->device) != cudaSuccess) return RAFI_ERR_CUDA;
  return launch_grid(c, n, k_march_seed, v, n, seed, Grid3{gx, gy, gz});
}

extern "C" int rafi_drv_march_step(rafi_ctx* ctx, uint32_t rnd, uint64_t seed, uint32_t p_thr, uint32_t max_bounces,
                                   uint32_t max_steps, int gx, int gy, int gz, float* result) {
  (void)rnd;
  auto* c = reinterpret_cast<rafi_impl::Ctx*>(ctx);
  if (!c || !result) return RAFI_ERR_INVALID_ARG;
  int rc = check_grid(c, gx, gy, gz);
  if (rc != RAFI_OK) return rc;
  if (c->B != sizeof(Ray)) return RAFI_ERR_INVALID_ARG;
  if (cudaSetDevice(c->device) != cudaSuccess) return RAFI_ERR_CUDA;
  for (int l = 0; l < c->L; ++l) {
    rafi_device_view v;
    if ((rc = rafi_get_device_view(ctx, l, &v)) != RAFI_OK) return rc;
    if ((rc = launch_grid(c, launch_count(c, v), k_march_step, v, seed, p_thr, max_bounces, max_steps, Grid3{gx, gy, gz},
                          result)))
      return rc;
  }
  return RAFI_OK;
}

// ------------------------------------------------------------------ N-body exchange (NEXT-2)
// Three contexts of different item types on one communicator:
// particle migration, root-multipole broadcast, refinement requests and
// subtree responses.  Multipole statistics use exact integer sums of
// positions quantised to 2^-20, so they do not depend on summation order.

namespace {

struct NbParticle {
  float px, py, pz, vx, vy, vz, fx, fy, fz, mass;
};
struct NbVirtual {
  float cx, cy, cz, mass, smax;
  int32_t sourceRank;
};
struct NbRequest {
  int32_t senderRank;
};
static_assert(sizeof(NbParticle) == 40 && sizeof(NbVirtual) == 24 && sizeof(NbRequest) == 4, "nbody types");

constexpr int kNbStats = 10 + 8 * 4;  // count, sum[3], min[3], max[3]; 8 x (count, sum[3])
constexpr float kQ = 1048576.0f, kIQ = 9.5367431640625e-07f;  // 2^20, 2^-20

__device__ __forceinline__ uint32_t q20(float x) { return (uint32_t)(x * kQ); }

// owner by Morton order: 10 bits per axis, equal-width code intervals
__device__ __forceinline__ int morton_owner(float x, float y, float z, int R) {
  const uint32_t qx = min((uint32_t)(x * 1024.0f), 1023u), qy = min((uint32_t)(y * 1024.0f), 1023u),
                 qz = min((uint32_t)(z * 1024.0f), 1023u);
  uint64_t code = 0;
#pragma unroll
  for (int b = 0; b < 10; ++b)
    code |= ((uint64_t)((qx >> b) & 1) << (3 * b)) | ((uint64_t)((qy >> b) & 1) << (3 * b + 1)) |
            ((uint64_t)((qz >> b) & 1) << (3 * b + 2));
  return (int)((code * (uint64_t)R) >> 30);
}

__device__ __forceinline__ float wrap01(float x) {
  if (x < 0.0f) x = x + 1.0f;
  if (x >= 1.0f) x = x - 1.0f;
  return x;
}

__global__ void k_nb_seed(rafi_device_view v, uint64_t n, uint64_t seed) {
  rafi::Queue<NbParticle> q(v);
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t id = (uint64_t)v.my_rank * n + i;
    const uint64_t b = seed ^ (id << 3);
    NbParticle p;
    p.px = u24(splitmix64(b ^ 0ull));
    p.py = u24(splitmix64(b ^ 1ull));
    p.pz = u24(splitmix64(b ^ 2ull));
    p.vx = (u24(splitmix64(b ^ 3ull)) - 0.5f) * 0.25f;
    p.vy = (u24(splitmix64(b ^ 4ull)) - 0.5f) * 0.25f;
    p.vz = (u24(splitmix64(b ^ 5ull)) - 0.5f) * 0.25f;
    p.fx = p.fy = p.fz = 0.0f;
    p.mass = 1.0f;
    q.emitOutgoing(p, morton_owner(p.px, p.py, p.pz, v.num_ranks));
  }
}

__global__ void k_nb_migrate(rafi_device_view v, float dt) {
  rafi::Queue<NbParticle> q(v);
  const unsigned long long n = q.numIncoming();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    NbParticle p = q.getIncoming(i);
    p.px = wrap01(p.px + dt * p.vx);
    p.py = wrap01(p.py + dt * p.vy);
    p.pz = wrap01(p.pz + dt * p.vz);
    q.emitOutgoing(p, morton_owner(p.px, p.py, p.pz, v.num_ranks));
  }
}

__global__ void k_nb_stats_init(unsigned long long* st) {
  const int i = threadIdx.x;
  if (i < kNbStats) st[blockIdx.x * kNbStats + i] = (i >= 4 && i < 7) ? 0xFFFFFFFFull : 0ull;
}

// Statistics are reduced per thread in registers, then per block in shared
// memory, then one global atomic per value and block (integer sums: exact in
// any order).
__global__ void k_nb_stats_root(rafi_device_view v, unsigned long long* st) {
  __shared__ unsigned long long s[10];
  rafi::Queue<NbParticle> q(v);
  const unsigned long long n = q.numIncoming();
  if (threadIdx.x < 10) s[threadIdx.x] = (threadIdx.x >= 4 && threadIdx.x < 7) ? 0xFFFFFFFFull : 0ull;
  __syncthreads();
  unsigned long long c = 0, sx = 0, sy = 0, sz = 0;
  uint32_t mnx = 0xFFFFFFFFu, mny = 0xFFFFFFFFu, mnz = 0xFFFFFFFFu, mxx = 0, mxy = 0, mxz = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const NbParticle p = q.getIncoming(i);
    const uint32_t x = q20(p.px), y = q20(p.py), z = q20(p.pz);
    c += 1; sx += x; sy += y; sz += z;
    mnx = min(mnx, x); mny = min(mny, y); mnz = min(mnz, z);
    mxx = max(mxx, x); mxy = max(mxy, y); mxz = max(mxz, z);
  }
  if (c) {
    atomicAdd(&s[0], c); atomicAdd(&s[1], sx); atomicAdd(&s[2], sy); atomicAdd(&s[3], sz);
    atomicMin(&s[4], (unsigned long long)mnx); atomicMin(&s[5], (unsigned long long)mny);
    atomicMin(&s[6], (unsigned long long)mnz); atomicMax(&s[7], (unsigned long long)mxx);
    atomicMax(&s[8], (unsigned long long)mxy); atomicMax(&s[9], (unsigned long long)mxz);
  }
  __syncthreads();
  if (threadIdx.x == 0 && s[0]) {
    atomicAdd(&st[0], s[0]); atomicAdd(&st[1], s[1]); atomicAdd(&st[2], s[2]); atomicAdd(&st[3], s[3]);
    atomicMin(&st[4], s[4]); atomicMin(&st[5], s[5]); atomicMin(&st[6], s[6]);
    atomicMax(&st[7], s[7]); atomicMax(&st[8], s[8]); atomicMax(&st[9], s[9]);
  }
}

__global__ void k_nb_stats_oct(rafi_device_view v, unsigned long long* st) {
  __shared__ unsigned long long s[32];
  rafi::Queue<NbParticle> q(v);
  const unsigned long long n = q.numIncoming();
  if (st[0] == 0) return;
  if (threadIdx.x < 32) s[threadIdx.x] = 0;
  __syncthreads();
  const uint64_t cx = st[1] / st[0], cy = st[2] / st[0], cz = st[3] / st[0];
  unsigned long long a[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) a[j] = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const NbParticle p = q.getIncoming(i);
    const uint32_t x = q20(p.px), y = q20(p.py), z = q20(p.pz);
    const int o = (x >= cx) | ((y >= cy) << 1) | ((z >= cz) << 2);
#pragma unroll
    for (int j = 0; j < 8; ++j)  // register-resident per-octant sums (no dynamic indexing)
      if (j == o) { a[4 * j] += 1; a[4 * j + 1] += x; a[4 * j + 2] += y; a[4 * j + 3] += z; }
  }
#pragma unroll
  for (int j = 0; j < 32; ++j)
    if (a[j]) atomicAdd(&s[j], a[j]);
  __syncthreads();
  if (threadIdx.x < 32 && s[threadIdx.x]) atomicAdd(&st[10 + threadIdx.x], s[threadIdx.x]);
}

__device__ __forceinline__ NbVirtual nb_node(const unsigned long long* s, float smax, int me) {
  NbVirtual n;
  n.cx = (float)(s[1] / s[0]) * kIQ;
  n.cy = (float)(s[2] / s[0]) * kIQ;
  n.cz = (float)(s[3] / s[0]) * kIQ;
  n.mass = (float)s[0];
  n.smax = smax;
  n.sourceRank = me;
  return n;
}

__device__ __forceinline__ float nb_root_smax(const unsigned long long* st) {
  const uint64_t ex = st[7] - st[4], ey = st[8] - st[5], ez = st[9] - st[6];
  const uint64_t e = ex > ey ? (ex > ez ? ex : ez) : (ey > ez ? ey : ez);
  return (float)e * kIQ;
}

// root broadcast: one VirtualParticle to every other rank
__global__ void k_nb_root(rafi_device_view v, const unsigned long long* st) {
  rafi::Queue<NbVirtual> q(v);
  if (st[0] == 0) return;
  const NbVirtual root = nb_node(st, nb_root_smax(st), v.my_rank);
  for (int d = threadIdx.x; d < v.num_ranks; d += blockDim.x)
    if (d != v.my_rank) q.emitOutgoing(root, d);
}

// MAC test on each received root; request refinement from its source
__global__ void k_nb_refine(rafi_device_view vv, rafi_device_view vq, const unsigned long long* st, float theta2) {
  rafi::Queue<NbVirtual> in(vv);
  rafi::Queue<NbRequest> out(vq);
  const unsigned long long n = in.numIncoming();
  if (st[0] == 0) return;
  const float mx = (float)(st[1] / st[0]) * kIQ, my = (float)(st[2] / st[0]) * kIQ,
              mz = (float)(st[3] / st[0]) * kIQ;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const NbVirtual r = in.getIncoming(i);
    const float dx = r.cx - mx, dy = r.cy - my, dz = r.cz - mz;
    const float d2 = dx * dx + dy * dy + dz * dz;
    if (r.smax * r.smax > theta2 * d2) out.emitOutgoing(NbRequest{vq.my_rank}, r.sourceRank);
  }
}

// respond to each request with the (non-empty) octant children
__global__ void k_nb_respond(rafi_device_view vq, rafi_device_view vv, const unsigned long long* st) {
  rafi::Queue<NbRequest> in(vq);
  rafi::Queue<NbVirtual> out(vv);
  const unsigned long long n = in.numIncoming();
  if (st[0] == 0) return;
  const float half = nb_root_smax(st) * 0.5f;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n * 8; i += (uint64_t)gridDim.x * blockDim.x) {
    const NbRequest r = in.getIncoming(i / 8);
    const unsigned long long* s = st + 10 + 4 * (i % 8);
    if (s[0]) out.emitOutgoing(nb_node(s, half, vv.my_rank), r.senderRank);
  }
}

int nb_check(rafi_impl::Ctx* c, uint64_t B) {
  if (!c) return RAFI_ERR_INVALID_ARG;
  if (c->B != B) { rafi_impl::set_error("nbody driver: wrong item size for this context"); return RAFI_ERR_INVALID_ARG; }
  return cudaSetDevice(c->device) == cudaSuccess ? RAFI_OK : RAFI_ERR_CUDA;
}

}  // namespace

extern "C" int rafi_drv_nbody_seed(rafi_ctx* ctx, int local, uint64_t n, uint64_t seed) {
  auto* c = reinterpret_cast<rafi_impl::Ctx*>(ctx);
  int rc = nb_check(c, sizeof(NbParticle));
  if (rc) return rc;
  rafi_device_view v;
  if ((rc = rafi_get_device_view(ctx, local, &v))) return rc;
  return launch_grid(c, n, k_nb_seed, v, n, seed);
}

extern "C" int rafi_drv_nbody_migrate(rafi_ctx* ctx, float dt) {
  auto* c = reinterpret_cast<rafi_impl::Ctx*>(ctx);
  int rc = nb_check(c, sizeof(NbParticle));
  if (rc) return rc;
  for (int l = 0; l < c->L; ++l) {
    rafi_device_view v;
    if ((rc = rafi_get_device_view(ctx, l, &v))) return rc;
    if ((rc = launch_grid(c, launch_count(c, v), k_nb_migrate, v, dt))) return rc;
  }
  return RAFI_OK;
}

extern "C" int rafi_drv_nbody_stats(rafi_ctx* ctx, unsigned long long* stats) {
  auto* c = reinterpret_cast<rafi_impl::Ctx*>(ctx);
  int rc = nb_check(c, sizeof(NbParticle));
  if (rc) return rc;
  if (!stats) return RAFI_ERR_INVALID_ARG;
  k_nb_stats_init<<<c->L, 64, 0, c->stream>>>(stats);
  c->launches += 1;
  for (int l = 0; l < c->L; ++l) {
    rafi_device_view v;
    if ((rc = rafi_get_device_view(ctx, l, &v))) return rc;
    if ((rc = launch_grid(c, launch_count(c, v), k_nb_stats_root, v, stats + (uint64_t)l * kNbStats))) return rc;
  }
  for (int l = 0; l < c->L; ++l) {
    rafi_device_view v;
    if ((rc = rafi_get_device_view(ctx, l, &v))) return rc;
    if ((rc = launch_grid(c, launch_count(c, v), k_nb_stats_oct, v, stats + (uint64_t)l * kNbStats))) return rc;
  }
  return cudaGetLastError() == cudaSuccess ? RAFI_OK : RAFI_ERR_CUDA;
}

extern "C" int rafi_drv_nbody_root(rafi_ctx* vctx, const unsigned long long* stats) {
  auto* c = reinterpret_cast<rafi_impl::Ctx*>(vctx);
  int rc = nb_check(c, sizeof(NbVirtual));
  if (rc) return rc;
  for (int l = 0; l < c->L; ++l) {
    rafi_device_view v;
    if ((rc = rafi_get_device_view(vctx, l, &v))) return rc;
    k_nb_root<<<1, 256, 0, c->stream>>>(v, stats + (uint64_t)l * kNbStats);
    c->launches += 1;
  }
  return cudaGetLastError() == cudaSuccess ? RAFI_OK : RAFI_ERR_CUDA;
}

extern "C" int rafi_drv_nbody_refine(rafi_ctx* vctx, rafi_ctx* qctx, const unsigned long long* stats, float theta2) {
  auto* cv = reinterpret_cast<rafi_impl::Ctx*>(vctx);
  auto* cq = reinterpret_cast<rafi_impl::Ctx*>(qctx);
  int rc = nb_check(cv, sizeof(NbVirtual));
  if (rc || (rc = nb_check(cq, sizeof(NbRequest)))) return rc;
  if (cv->L != cq->L || cv->R != cq->R || cv->stream != cq->stream) return RAFI_ERR_INVALID_ARG;
  for (int l = 0; l < cv->L; ++l) {
    rafi_device_view a, b;
    if ((rc = rafi_get_device_view(vctx, l, &a)) || (rc = rafi_get_device_view(qctx, l, &b))) return rc;
    if ((rc = launch_grid(cv, launch_count(cv, a), k_nb_refine, a, b, stats + (uint64_t)l * kNbStats, theta2)))
      return rc;
  }
  return RAFI_OK;
}

extern "C" int rafi_drv_nbody_respond(rafi_ctx* qctx, rafi_ctx* vctx, const unsigned long long* stats) {
  auto* cq = reinterpret_cast<rafi_impl::Ctx*>(qctx);
  auto* cv = reinterpret_cast<rafi_impl::Ctx*>(vctx);
  int rc = nb_check(cq, sizeof(NbRequest));
  if (rc || (rc = nb_check(cv, sizeof(NbVirtual)))) return rc;
  if (cv->L != cq->L || cv->R != cq->R || cv->stream != cq->stream) return RAFI_ERR_INVALID_ARG;
  for (int l = 0; l < cq->L; ++l) {
    rafi_device_view a, b;
    if ((rc = rafi_get_device_view(qctx, l, &a)) || (rc = rafi_get_device_view(vctx, l, &b))) return rc;
    if ((rc = launch_grid(cq, 8 * launch_count(cq, a), k_nb_respond, a, b, stats + (uint64_t)l * kNbStats)))
      return rc;
  }
  return RAFI_OK;
}

// ------------------------------------------------------------------ streamlines (NEXT-4)
// Particle advection on a sampled vector field: per-rank
// field blocks with a one-vertex halo, trilinear sampling, RK4,
// owner by macrocell.  + - * / only, no contraction.

namespace {

struct SGrid {
  int nx, ny, nz, gx, gy, gz, mx, my, mz;  // vertices, macrocell grid, cells per macrocell
};

struct SBlock {
  const float* v;  // local vertices (x fastest), float3 each
  int lo[3];       // first stored vertex
  int ld[3];       // stored vertices per axis
};

__device__ __forceinline__ int s_cell(float p, int n) {
  int i = (int)(p * (float)(n - 1));
  return i > n - 2 ? n - 2 : (i < 0 ? 0 : i);
}

__device__ __forceinline__ int s_owner(const SGrid& g, float x, float y, float z) {
  return ((s_cell(z, g.nz) / g.mz) * g.gy + s_cell(y, g.ny) / g.my) * g.gx + s_cell(x, g.nx) / g.mx;
}

__device__ __forceinline__ bool s_in_closed(float x, float y, float z) {
  return x >= 0.0f && x <= 1.0f && y >= 0.0f && y <= 1.0f && z >= 0.0f && z <= 1.0f;
}

// trilinear sample; false if the stage point left the domain or the block+halo
__device__ bool s_sample(const SGrid& g, const SBlock& b, float x, float y, float z, float* out, int* halo_miss) {
  if (!s_in_closed(x, y, z)) return false;
  const float ux = x * (float)(g.nx - 1), uy = y * (float)(g.ny - 1), uz = z * (float)(g.nz - 1);
  const int i = s_cell(x, g.nx), j = s_cell(y, g.ny), k = s_cell(z, g.nz);
  const float fx = ux - (float)i, fy = uy - (float)j, fz = uz - (float)k;
  const int li = i - b.lo[0], lj = j - b.lo[1], lk = k - b.lo[2];
  if (li < 0 || lj < 0 || lk < 0 || li > b.ld[0] - 2 || lj > b.ld[1] - 2 || lk > b.ld[2] - 2) {
    atomicAdd(halo_miss, 1);
    return false;
  }
  const float gx0 = 1.0f - fx, gy0 = 1.0f - fy, gz0 = 1.0f - fz;
  const int sx = 3, sy = 3 * b.ld[0], sz = 3 * b.ld[0] * b.ld[1];
  const float* c = b.v + (size_t)lk * sz + (size_t)lj * sy + (size_t)li * sx;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const float c00 = c[a] * gx0 + c[sx + a] * fx;
    const float c10 = c[sy + a] * gx0 + c[sy + sx + a] * fx;
    const float c01 = c[sz + a] * gx0 + c[sz + sx + a] * fx;
    const float c11 = c[sz + sy + a] * gx0 + c[sz + sy + sx + a] * fx;
    const float c0 = c00 * gy0 + c10 * fy, c1 = c01 * gy0 + c11 * fy;
    out[a] = c0 * gz0 + c1 * fz;
  }
  return true;
}

__global__ void k_stream_seed(rafi_device_view v, SGrid g, const float* seeds, uint64_t n, uint32_t id0) {
  rafi::Queue<Particle> q(v);
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    Particle p;
    p.id = id0 + (uint32_t)i;
    p.x = seeds[3 * i];
    p.y = seeds[3 * i + 1];
    p.z = seeds[3 * i + 2];
    if (!inside(p.x, p.y, p.z)) continue;  // a seed outside the domain has an empty streamline
    q.emitOutgoing(p, s_owner(g, p.x, p.y, p.z));
  }
}

__global__ void k_stream_step(rafi_device_view v, SGrid g, SBlock b, uint32_t rnd, float h, float eps,
                              uint32_t max_steps, float* rpos, uint32_t* rsteps, int* halo_miss) {
  rafi::Queue<Particle> q(v);
  const unsigned long long n = q.numIncoming();
  const float hh = 0.5f * h, h6 = h / 6.0f;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    Particle p = q.getIncoming(i);
    float k1[3], k2[3], k3[3], k4[3];
    bool ok = s_sample(g, b, p.x, p.y, p.z, k1, halo_miss);
    ok = ok && s_sample(g, b, p.x + hh * k1[0], p.y + hh * k1[1], p.z + hh * k1[2], k2, halo_miss);
    ok = ok && s_sample(g, b, p.x + hh * k2[0], p.y + hh * k2[1], p.z + hh * k2[2], k3, halo_miss);
    ok = ok && s_sample(g, b, p.x + h * k3[0], p.y + h * k3[1], p.z + h * k3[2], k4, halo_miss);
    if (!ok) {  // a stage left the domain: terminated before this step
      rpos[3 * p.id] = p.x; rpos[3 * p.id + 1] = p.y; rpos[3 * p.id + 2] = p.z;
      rsteps[p.id] = rnd - 1;
      continue;
    }
    const float nx = p.x + h6 * (((k1[0] + 2.0f * k2[0]) + 2.0f * k3[0]) + k4[0]);
    const float ny = p.y + h6 * (((k1[1] + 2.0f * k2[1]) + 2.0f * k3[1]) + k4[1]);
    const float nz = p.z + h6 * (((k1[2] + 2.0f * k2[2]) + 2.0f * k3[2]) + k4[2]);
    const float dx = nx - p.x, dy = ny - p.y, dz = nz - p.z;
    p.x = nx; p.y = ny; p.z = nz;
    if (dx * dx + dy * dy + dz * dz < eps * eps || !inside(nx, ny, nz) || rnd >= max_steps) {
      rpos[3 * p.id] = nx; rpos[3 * p.id + 1] = ny; rpos[3 * p.id + 2] = nz;
      rsteps[p.id] = rnd;
      continue;
    }
    q.emitOutgoing(p, s_owner(g, nx, ny, nz));
  }
}

}  // namespace

struct rafi_stream_field {
  rafi_impl::Ctx* c = nullptr;
  SGrid g{};
  std::vector<SBlock> blocks;  // per local rank (device pointers)
  int* halo_miss = nullptr;    // device counter
};

extern "C" int rafi_drv_stream_create(rafi_ctx* ctx, const float* field, int nx, int ny, int nz, int gx, int gy,
                                      int gz, rafi_stream_field** out) {
  auto* c = reinterpret_cast<rafi_impl::Ctx*>(ctx);
  if (!c || !field || !out || nx < 2 || ny < 2 || nz < 2) return RAFI_ERR_INVALID_ARG;
  if (c->B != sizeof(Particle)) return RAFI_ERR_INVALID_ARG;
  int rc = check_grid(c, gx, gy, gz);
  if (rc) return rc;
  if ((nx - 1) % gx || (ny - 1) % gy || (nz - 1) % gz) {
    rafi_impl::set_error("stream field: cells per axis must divide evenly into the macrocell grid");
    return RAFI_ERR_INVALID_ARG;
  }
  if (cudaSetDevice(c->device) != cudaSuccess) return RAFI_ERR_CUDA;
  auto* f = new rafi_stream_field();
  f->c = c;
  f->g = SGrid{nx, ny, nz, gx, gy, gz, (nx - 1) / gx, (ny - 1) / gy, (nz - 1) / gz};
  const int n[3] = {nx, ny, nz}, m[3] = {f->g.mx, f->g.my, f->g.mz};
  for (int l = 0; l < c->L; ++l) {
    const int r = c->proc * c->L + l;
    const int cc[3] = {r % gx, (r / gx) % gy, r / (gx * gy)};
    SBlock b{};
    for (int a = 0; a < 3; ++a) {
      b.lo[a] = cc[a] * m[a] - 1 < 0 ? 0 : cc[a] * m[a] - 1;
      const int hi = (cc[a] + 1) * m[a] + 1 > n[a] - 1 ? n[a] - 1 : (cc[a] + 1) * m[a] + 1;
      b.ld[a] = hi - b.lo[a] + 1;
    }
    std::vector<float> host((size_t)b.ld[0] * b.ld[1] * b.ld[2] * 3);
    for (int k = 0; k < b.ld[2]; ++k)
      for (int j = 0; j < b.ld[1]; ++j)
        for (int i = 0; i < b.ld[0]; ++i)
          for (int a = 0; a < 3; ++a)
            host[(((size_t)k * b.ld[1] + j) * b.ld[0] + i) * 3 + a] =
                field[((((size_t)(k + b.lo[2]) * ny) + (j + b.lo[1])) * nx + (i + b.lo[0])) * 3 + a];
    float* d = nullptr;
    if (cudaMalloc(&d, host.size() * sizeof(float)) != cudaSuccess ||
        cudaMemcpy(d, host.data(), host.size() * sizeof(float), cudaMemcpyHostToDevice) != cudaSuccess) {
      cudaGetLastError();
      rafi_drv_stream_destroy(f);
      return RAFI_ERR_CUDA;
    }
    b.v = d;
    f->blocks.push_back(b);
  }
  if (cudaMalloc(&f->halo_miss, sizeof(int)) != cudaSuccess || cudaMemset(f->halo_miss, 0, sizeof(int)) != cudaSuccess) {
    cudaGetLastError();
    rafi_drv_stream_destroy(f);
    return RAFI_ERR_CUDA;
  }
  *out = f;
  return RAFI_OK;
}

extern "C" int rafi_drv_stream_seed(rafi_stream_field* f, int local, const float* seeds, uint64_t n, uint32_t id0) {
  if (!f || local < 0 || local >= f->c->L || (n && !seeds)) return RAFI_ERR_INVALID_ARG;
  if (!n) return RAFI_OK;
  rafi_device_view v;
  int rc = rafi_get_device_view(reinterpret_cast<rafi_ctx*>(f->c), local, &v);
  if (rc) return rc;
  float* d = nullptr;
  if (cudaMalloc(&d, 3 * n * sizeof(float)) != cudaSuccess) { cudaGetLastError(); return RAFI_ERR_NOMEM; }
  if (cudaMemcpyAsync(d, seeds, 3 * n * sizeof(float), cudaMemcpyDefault, f->c->stream) != cudaSuccess) {
    cudaGetLastError(); cudaFree(d); return RAFI_ERR_CUDA;
  }
  rc = launch_grid(f->c, n, k_stream_seed, v, f->g, (const float*)d, n, id0);
  cudaStreamSynchronize(f->c->stream);
  cudaFree(d);
  return rc;
}

extern "C" int rafi_drv_stream_step(rafi_stream_field* f, uint32_t rnd, float h, float eps, uint32_t max_steps,
                                    float* rpos, uint32_t* rsteps) {
  if (!f || !rpos || !rsteps) return RAFI_ERR_INVALID_ARG;
  auto* c = f->c;
  if (cudaSetDevice(c->device) != cudaSuccess) return RAFI_ERR_CUDA;
  for (int l = 0; l < c->L; ++l) {
    rafi_device_view v;
    int rc = rafi_get_device_view(reinterpret_cast<rafi_ctx*>(c), l, &v);
    if (rc) return rc;
    if ((rc = launch_grid(c, launch_count(c, v), k_stream_step, v, f->g, f->blocks[l], rnd, h, eps, max_steps, rpos,
                          rsteps, f->halo_miss)))
      return rc;
  }
  return RAFI_OK;
}

extern "C" int rafi_drv_stream_destroy(rafi_stream_field* f) {
  if (!f) return RAFI_OK;
  cudaSetDevice(f->c->device);
  cudaStreamSynchronize(f->c->stream);
  for (auto& b : f->blocks) cudaFree(const_cast<float*>(b.v));
  cudaFree(f->halo_miss);
  delete f;
  return RAFI_OK;
}

extern "C" int rafi_drv_stream_halo_misses(rafi_stream_field* f, int* count) {
  if (!f || !count) return RAFI_ERR_INVALID_ARG;
  cudaStreamSynchronize(f->c->stream);
  return cudaMemcpy(count, f->halo_miss, sizeof(int), cudaMemcpyDeviceToHost) == cudaSuccess ? RAFI_OK : RAFI_ERR_CUDA;
}
