// p2p_bw.cu -- NVLink peer-bandwidth ceilings on this box, measured the way
// the forwarding path moves bytes (the denominator for the exchange roofline).
//
// Single process, every visible GPU, peer access enabled.  Each pattern moves
// BYTES per GPU and reports GB/s per GPU per direction (max-over-GPUs time):
//   ce_uni      cudaMemcpyPeerAsync 0 -> 1 (copy engines, one direction)
//   ce_bidir    every GPU copies to its ring successor at once (copy engines)
//   sm_push     st.global.v4 into the peer (0 -> 1 only)
//   sm_pull     ld.global.v4 from the peer (1 reads 0)
//   sm_push_bi  every GPU pushes to its ring successor at once
//   tma_push_bi cp.async.bulk global->shared->peer global, every GPU at once
//   mix_F       every GPU sends to its ring successor: fraction F/10 by SM
//               stores, the rest by the copy engines, at the same time
//   a2a_pull    the same exchange done by the receivers' loads
//   a2a_push    every GPU pushes 1/N of its buffer to each GPU (itself
//               included: the FUSED exchange's traffic without the binning);
//               reported per GPU as remote bytes / time
// and the PCIe ceilings of the end-to-end path (GPU 0, pinned host memory):
//   h2d, d2h    one direction alone;  h2d_d2h   both at once (per direction)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o p2p_bw p2p_bw.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e = (x);                                                               \
    if (e != cudaSuccess) {                                                            \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); \
      exit(1);                                                                         \
    }                                                                                  \
  } while (0)

__global__ void __launch_bounds__(256) k_copy16(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n; i += 4 * stride) {
    const uint4 a = src[i], b = src[i + stride], c = src[i + 2 * stride], d = src[i + 3 * stride];
    dst[i] = a; dst[i + stride] = b; dst[i + 2 * stride] = c; dst[i + 3 * stride] = d;
  }
  for (; i < n; i += stride) dst[i] = src[i];
}

// all-to-all: part p of src goes to dst[p] + me*part.  The flat work index
// interleaves destinations, rotated by the sender (p = (me + f) mod G), so the
// GPUs do not all write to the same receiver at the same time.
struct Dsts { uint4* p[8]; };
__global__ void __launch_bounds__(256) k_a2a(const uint4* __restrict__ src, Dsts dst, int me, int G, size_t part) {
  constexpr size_t CH = 256 * 4;  // uint4 per chunk per CTA step (16 KiB)
  const size_t nch = (part + CH - 1) / CH;
  for (size_t f = blockIdx.x; f < nch * G; f += gridDim.x) {
    const int p = (int)((me + f) % G);
    const size_t c = f / G;
    const uint4* s = src + (size_t)p * part + c * CH;
    uint4* d = dst.p[p] + (size_t)me * part + c * CH;
    const size_t lim = part - c * CH < CH ? part - c * CH : CH;
    uint4 v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const size_t i = threadIdx.x + j * 256;
      if (i < lim) v[j] = s[i];
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const size_t i = threadIdx.x + j * 256;
      if (i < lim) d[i] = v[j];
    }
  }
}

// all-to-all pull: part me of every GPU p's buffer is read into dst + p*part
// (the receiver side of the same exchange), destinations rotated per reader.
struct Srcs { const uint4* p[8]; };
__global__ void __launch_bounds__(256) k_a2a_pull(Srcs src, uint4* __restrict__ dst, int me, int G, size_t part) {
  constexpr size_t CH = 256 * 4;
  const size_t nch = (part + CH - 1) / CH;
  for (size_t f = blockIdx.x; f < nch * G; f += gridDim.x) {
    const int p = (int)((me + f) % G);
    const size_t c = f / G;
    const uint4* s = src.p[p] + (size_t)me * part + c * CH;
    uint4* d = dst + (size_t)p * part + c * CH;
    const size_t lim = part - c * CH < CH ? part - c * CH : CH;
    uint4 v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const size_t i = threadIdx.x + j * 256;
      if (i < lim) v[j] = s[i];
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const size_t i = threadIdx.x + j * 256;
      if (i < lim) d[i] = v[j];
    }
  }
}

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// TMA: chunks of 32 KiB through a two-buffer shared ring, bulk load then bulk store
__global__ void __launch_bounds__(32) k_tma_copy(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst,
                                                 size_t bytes) {
  constexpr uint32_t CH = 32 * 1024;
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar[2];
  if (threadIdx.x != 0) return;
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[0])));
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[1])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const size_t nch = bytes / CH;
  uint32_t ph[2] = {0, 0};
  int k = 0;
  for (size_t c = blockIdx.x; c < nch; c += gridDim.x, k ^= 1) {
    // buffer k: wait until the store issued two chunks ago has read it
    asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[k])), "r"(CH) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     su32(sm + k * CH)),
                 "l"(src + c * CH), "r"(CH), "r"(su32(&bar[k]))
                 : "memory");
    asm volatile(
        "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
            su32(&bar[k])),
        "r"(ph[k])
        : "memory");
    ph[k] ^= 1;
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + c * CH), "r"(su32(sm + k * CH)),
                 "r"(CH)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

static int G = 0, SMS = 148;
static std::vector<cudaStream_t> st;
static std::vector<cudaEvent_t> e0, e1;

template <class F>
static double timed(F launch, const std::vector<int>& devs, int reps = 5) {
  double best = 1e30;
  for (int r = 0; r < reps + 1; ++r) {
    for (int d : devs) { CK(cudaSetDevice(d)); CK(cudaDeviceSynchronize()); }
    for (int d : devs) { CK(cudaSetDevice(d)); CK(cudaEventRecord(e0[d], st[d])); }
    for (int d : devs) { CK(cudaSetDevice(d)); launch(d); CK(cudaGetLastError()); }
    for (int d : devs) { CK(cudaSetDevice(d)); CK(cudaEventRecord(e1[d], st[d])); }
    double mx = 0;
    for (int d : devs) {
      CK(cudaSetDevice(d));
      CK(cudaEventSynchronize(e1[d]));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0[d], e1[d]));
      mx = std::max(mx, (double)ms);
    }
    if (r > 0) best = std::min(best, mx);  // first rep is warm-up
  }
  return best;
}

int main(int argc, char** argv) {
  const size_t BYTES = (argc > 1 ? strtoull(argv[1], nullptr, 10) : 1ull << 30);
  CK(cudaGetDeviceCount(&G));
  G = std::min(G, 8);
  CK(cudaDeviceGetAttribute(&SMS, cudaDevAttrMultiProcessorCount, 0));
  std::vector<uint8_t*> a(G), b(G);
  st.resize(G); e0.resize(G); e1.resize(G);
  for (int d = 0; d < G; ++d) {
    CK(cudaSetDevice(d));
    for (int p = 0; p < G && G > 1; ++p)
      if (p != d) {
        int ok = 0;
        CK(cudaDeviceCanAccessPeer(&ok, d, p));
        if (!ok) { printf("{\"error\": \"no peer access %d->%d\"}\n", d, p); return 0; }
        CK(cudaDeviceEnablePeerAccess(p, 0));
      }
    CK(cudaMalloc(&a[d], BYTES));
    CK(cudaMalloc(&b[d], BYTES));
    CK(cudaMemset(a[d], d + 1, BYTES));
    CK(cudaStreamCreateWithFlags(&st[d], cudaStreamNonBlocking));
    CK(cudaEventCreate(&e0[d]));
    CK(cudaEventCreate(&e1[d]));
    CK(cudaFuncSetAttribute(k_tma_copy, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
  }
  const size_t n16 = BYTES / 16;
  const int grid = SMS * 8;
  auto gbs = [&](double ms, double bytes) { return bytes / (ms * 1e-3) / 1e9; };
  auto line = [&](const char* name, int gpus, double ms, double bytes_per_gpu) {
    printf("{\"pattern\": \"%s\", \"gpus\": %d, \"bytes_per_gpu\": %.0f, \"ms\": %.4f, \"gbs_per_gpu\": %.1f}\n", name,
           gpus, bytes_per_gpu, ms, gbs(ms, bytes_per_gpu));
    fflush(stdout);
  };
  std::vector<int> one = {0}, all;
  for (int d = 0; d < G; ++d) all.push_back(d);

  {  // PCIe (GPU 0): pinned host <-> device, one direction and both at once
    uint8_t *h0, *h1;
    CK(cudaSetDevice(0));
    CK(cudaMallocHost(&h0, BYTES));
    CK(cudaMallocHost(&h1, BYTES));
    memset(h0, 1, BYTES);
    memset(h1, 2, BYTES);
    cudaStream_t s2;
    CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
    double ms = timed([&](int d) { CK(cudaMemcpyAsync(a[0], h0, BYTES, cudaMemcpyHostToDevice, st[d])); }, one);
    line("h2d", 1, ms, BYTES);
    ms = timed([&](int d) { CK(cudaMemcpyAsync(h1, b[0], BYTES, cudaMemcpyDeviceToHost, st[d])); }, one);
    line("d2h", 1, ms, BYTES);
    cudaEvent_t f;
    CK(cudaEventCreate(&f));
    ms = timed([&](int d) {
      CK(cudaEventRecord(f, st[d]));
      CK(cudaStreamWaitEvent(s2, f, 0));
      CK(cudaMemcpyAsync(a[0], h0, BYTES, cudaMemcpyHostToDevice, st[d]));
      CK(cudaMemcpyAsync(h1, b[0], BYTES, cudaMemcpyDeviceToHost, s2));
      CK(cudaEventRecord(f, s2));
      CK(cudaStreamWaitEvent(st[d], f, 0));
    }, one);
    line("h2d_d2h", 1, ms, BYTES);
    CK(cudaFreeHost(h0));
    CK(cudaFreeHost(h1));
  }
  if (G < 2) return 0;

  double ms = timed([&](int d) { CK(cudaMemcpyPeerAsync(b[1], 1, a[0], 0, BYTES, st[d])); }, one);
  line("ce_uni", 2, ms, BYTES);
  ms = timed([&](int d) { CK(cudaMemcpyPeerAsync(b[(d + 1) % G], (d + 1) % G, a[d], d, BYTES, st[d])); }, all);
  line("ce_bidir", G, ms, BYTES);
  ms = timed([&](int d) { k_copy16<<<grid, 256, 0, st[d]>>>((const uint4*)a[0], (uint4*)b[1], n16); }, one);
  line("sm_push", 2, ms, BYTES);
  std::vector<int> d1 = {1};
  ms = timed([&](int d) { k_copy16<<<grid, 256, 0, st[d]>>>((const uint4*)a[0], (uint4*)b[1], n16); }, d1);
  line("sm_pull", 2, ms, BYTES);
  ms = timed([&](int d) {
    k_copy16<<<grid, 256, 0, st[d]>>>((const uint4*)a[d], (uint4*)b[(d + 1) % G], n16);
  }, all);
  line("sm_push_bi", G, ms, BYTES);
  ms = timed([&](int d) {
    k_tma_copy<<<SMS * 3, 32, 64 * 1024, st[d]>>>(a[d], b[(d + 1) % G], BYTES);
  }, all);
  line("tma_push_bi", G, ms, BYTES);
  {  // SM stores and copy engines sharing the links: does their sum exceed either?
    std::vector<cudaStream_t> s2(G);
    std::vector<cudaEvent_t> f(G);
    for (int d = 0; d < G; ++d) {
      CK(cudaSetDevice(d));
      CK(cudaStreamCreateWithFlags(&s2[d], cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&f[d], cudaEventDisableTiming));
    }
    for (int F : {3, 5, 7}) {
      const size_t nsm = (n16 * F / 10) & ~(size_t)255, nce = n16 - nsm;
      ms = timed([&](int d) {
        const int q = (d + 1) % G;
        CK(cudaEventRecord(f[d], st[d]));
        CK(cudaStreamWaitEvent(s2[d], f[d], 0));
        CK(cudaMemcpyPeerAsync(b[q] + nsm * 16, q, a[d] + nsm * 16, d, nce * 16, s2[d]));
        k_copy16<<<grid, 256, 0, st[d]>>>((const uint4*)a[d], (uint4*)b[q], nsm);
        CK(cudaEventRecord(f[d], s2[d]));
        CK(cudaStreamWaitEvent(st[d], f[d], 0));
      }, all);
      char name[16];
      snprintf(name, sizeof(name), "mix_%d", F);
      line(name, G, ms, BYTES);
    }
  }
  ms = timed([&](int d) { k_copy16<<<grid, 256, 0, st[d]>>>((const uint4*)a[d], (uint4*)b[d], n16); }, one);
  line("local_copy", 1, ms, 2.0 * BYTES);  // read + write, the HBM copy figure
  Dsts ds{};
  for (int p = 0; p < G; ++p) ds.p[p] = (uint4*)b[p];
  const size_t part = n16 / G;
  ms = timed([&](int d) {
    k_a2a<<<grid, 256, 0, st[d]>>>((const uint4*)a[d], ds, d, G, part);
  }, all);
  line("a2a_push", G, ms, (double)part * 16 * (G - 1));
  Srcs ss{};
  for (int p = 0; p < G; ++p) ss.p[p] = (const uint4*)a[p];
  ms = timed([&](int d) { k_a2a_pull<<<grid, 256, 0, st[d]>>>(ss, (uint4*)b[d], d, G, part); }, all);
  line("a2a_pull", G, ms, (double)part * 16 * (G - 1));
  return 0;
}
