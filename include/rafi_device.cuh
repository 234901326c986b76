/*
 * rafi_device.cuh -- device interface of RaFI, header-only.
 *
 *   rafi::Queue<T> q(view);            // view from rafi_get_device_view()
 *   for (i = tid; i < q.numIncoming(); i += stride) {
 *     T ray = q.getIncoming(i);          // any thread, any index, any order
 *     ...
 *     q.emitOutgoing(ray, nextRank);     // any thread, any number of times
 *   }
 *
 * T is any trivially copyable type with sizeof(T) == the context's item_bytes
 * (PAPER:40).  emitOutgoing follows the paper's atomic append
 * with one change for B200: the lanes of a warp that emit together are
 * aggregated, so a warp issues ONE atomicAdd on the emit counter instead of
 * one per lane.  Slot = counter value before the add (+ the lane's rank among
 * the emitting lanes); the item is kept iff slot < capacity ("calls that would
 * exceed the output queue size will simply get dropped"); the
 * counter itself is not clamped, so the host can report drops.  A destination
 * outside [0, R) is rejected without taking a slot and counted separately.
 *
 * Item moves are vectorised by sizeof(T): 16-byte stores/loads when
 * sizeof(T) % 16 == 0, 8-byte when % 8 == 0, 4-byte when % 4 == 0, bytes
 * otherwise.  The queues are cudaMalloc'd (256-byte aligned), so slot *
 * sizeof(T) keeps that alignment.  Needs C++17 (if constexpr).
 */
#ifndef RAFI_DEVICE_CUH
#define RAFI_DEVICE_CUH

#include <cstring>
#include <type_traits>

#include "rafi.h"

namespace rafi {

/* Widest unit (16, 8, 4 or 1 bytes) that divides sizeof(T). */
template <class T>
struct ItemUnit {
  using type = std::conditional_t<
      sizeof(T) % 16 == 0, uint4,
      std::conditional_t<sizeof(T) % 8 == 0, uint2, std::conditional_t<sizeof(T) % 4 == 0, unsigned, unsigned char>>>;
  static constexpr size_t count = sizeof(T) / sizeof(type);
};

/* Store item at dst (aligned to ItemUnit<T>) in unit-wide stores. */
template <class T>
__device__ __forceinline__ void store_item(void* dst, const T& item) {
  using U = typename ItemUnit<T>::type;
  U tmp[ItemUnit<T>::count];
  memcpy(tmp, &item, sizeof(T));
  U* d = static_cast<U*>(dst);
#pragma unroll
  for (size_t k = 0; k < ItemUnit<T>::count; ++k) d[k] = tmp[k];
}

/* Load an item from src (aligned to ItemUnit<T>) in unit-wide loads. */
template <class T>
__device__ __forceinline__ T load_item(const void* src) {
  using U = typename ItemUnit<T>::type;
  U tmp[ItemUnit<T>::count];
  const U* s = static_cast<const U*>(src);
#pragma unroll
  for (size_t k = 0; k < ItemUnit<T>::count; ++k) tmp[k] = s[k];
  T item;
  memcpy(&item, tmp, sizeof(T));
  return item;
}

__device__ __forceinline__ unsigned lane_id() {
  unsigned l;
  asm volatile("mov.u32 %0, %%laneid;" : "=r"(l));
  return l;
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm volatile("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

template <class T>
struct Queue {
  static_assert(std::is_trivially_copyable<T>::value,
                "RaFI items must be trivially copyable (PAPER:40)");
  rafi_device_view v;

  __host__ __device__ explicit Queue(const rafi_device_view& view) : v(view) {}

  /* numIncoming(): valid on host and device.  Device code reads the
     device-resident count, so it stays correct across rafi_forward_async /
     graph replays; the host reads the copy in the view. */
  __host__ __device__ unsigned long long numIncoming() const {
#ifdef __CUDA_ARCH__
    return *reinterpret_cast<const unsigned long long*>(v.num_in_dev);
#else
    return v.num_in;
#endif
  }

  /* getIncoming(i). */
  __device__ T getIncoming(unsigned long long i) const {
    return load_item<T>(static_cast<const char*>(v.in) + i * sizeof(T));
  }

  /* emitOutgoing(item, dest); returns true iff stored. */
  __device__ bool emitOutgoing(const T& item, int dest) const {
    const bool valid = (unsigned)dest < (unsigned)v.num_ranks;
    const unsigned active = __activemask();
    const unsigned vmask = __ballot_sync(active, valid);
    const unsigned lane = lane_id();
    if (!valid) {
      const unsigned imask = active & ~vmask;
      if (lane == (unsigned)(__ffs(imask) - 1)) atomicAdd(v.invalid, (unsigned long long)__popc(imask));
      return false;
    }
    const unsigned leader = __ffs(vmask) - 1;
    unsigned long long base = 0;
    if (lane == leader) base = atomicAdd(v.ctr, (unsigned long long)__popc(vmask));
    base = __shfl_sync(vmask, base, leader);
    const unsigned long long slot = base + __popc(vmask & lanemask_lt());
    if (slot >= v.capacity) return false;
    store_item<T>(static_cast<char*>(v.out) + slot * sizeof(T), item);
    v.dest[slot] = dest;
    return true;
  }

  /* Batched emitOutgoing: this thread emits items[0..count) to dests[0..count)
     (count <= K), with the same accept / drop / reject rules as K single
     calls.  The warp takes ONE atomicAdd for all its lanes' items (instead of
     one per emitOutgoing call): under full-GPU load the single emit counter's
     atomic unit serialises per address, and this is what lifts emission to
     the HBM write roofline.  Slots are item-major within the warp (item k of
     every lane, then item k+1), so the stores of each k are coalesced.
     Returns how many of this thread's items were stored. */
  template <int K>
  __device__ int emitOutgoing(const T (&items)[K], const int (&dests)[K], int count = K) const {
    const unsigned active = __activemask();
    const unsigned lane = lane_id();
    unsigned vm[K];
    unsigned total = 0, ninv = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const bool in_batch = k < count;
      const bool valid = in_batch && (unsigned)dests[k] < (unsigned)v.num_ranks;
      vm[k] = __ballot_sync(active, valid);
      ninv += __popc(__ballot_sync(active, in_batch && !valid));
      total += __popc(vm[k]);
    }
    const unsigned leader = __ffs(active) - 1;
    unsigned long long base = 0;
    if (lane == leader) {
      if (total) base = atomicAdd(v.ctr, (unsigned long long)total);
      if (ninv) atomicAdd(v.invalid, (unsigned long long)ninv);
    }
    base = __shfl_sync(active, base, leader);
    const unsigned lt = lanemask_lt();
    int stored = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if (vm[k] & (1u << lane)) {
        const unsigned long long slot = base + __popc(vm[k] & lt);
        if (slot < v.capacity) {
          store_item<T>(static_cast<char*>(v.out) + slot * sizeof(T), items[k]);
          v.dest[slot] = dests[k];
          ++stored;
        }
      }
      base += __popc(vm[k]);
    }
    return stored;
  }

  __host__ __device__ int numRanks() const { return v.num_ranks; }
  __host__ __device__ int myRank() const { return v.my_rank; }
};

/* Host helper: wrap a view, checking sizeof(T) against the context. */
template <class T>
inline bool make_queue(const rafi_device_view& view, Queue<T>* out) {
  if (view.item_bytes != sizeof(T)) return false;
  *out = Queue<T>(view);
  return true;
}

}  // namespace rafi

#endif /* RAFI_DEVICE_CUH */
