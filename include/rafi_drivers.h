/*
 * rafi_drivers.h -- proxy application kernels shipped with librafi.
 *
 * These are USER kernels of the forwarding library, written only against the
 * public device header (rafi_device.cuh): they read the incoming queue with
 * getIncoming() and append with emitOutgoing(), exactly as an application
 * kernel would.  They exist to drive the hot
 * path with the paper's workload shapes and to exercise emitOutgoing from
 * device code.  Items follow the synthetic layout of DESIGN.md "Input recipe"
 * (u32 src, u32 round, u64 id, hashed u32 words); the generator is a
 * counter-based SplitMix64, implemented here and, separately, in synth/.
 *
 * Same conventions as rafi.h (status returns, borrowed context, work ordered
 * on the context stream, asynchronous).
 */
#ifndef RAFI_DRIVERS_H
#define RAFI_DRIVERS_H

#include <stdint.h>

#include "rafi.h"

#ifdef __cplusplus
extern "C" {
#endif

/* destination patterns of rafi_drv_emit_synthetic (synth.PATTERNS) */
#define RAFI_DRV_UNIFORM 0
#define RAFI_DRV_SELF 1
#define RAFI_DRV_RING 2
#define RAFI_DRV_ALL_TO_ONE 3
#define RAFI_DRV_ROUND_ROBIN 4
#define RAFI_DRV_SKEWED 5

/* Synthetic producer (cfg1/2/5 emitter): local rank `local` emits n items
 * with sequence numbers seq0..seq0+n-1 of round `rnd`, one per thread, each
 * through emitOutgoing() with the pattern's destination.  A fraction of
 * destinations (low 32 bits of the hash < invalid_threshold) is made invalid
 * (-1 or R) to exercise rejection.  item_bytes must be a multiple of 4 and
 * >= 16 (RAFI_ERR_UNSUPPORTED otherwise). */
int rafi_drv_emit_synthetic(rafi_ctx* ctx, int local, int pattern, uint64_t seed, uint32_t rnd, uint64_t n,
                            uint64_t seq0, int target, uint64_t invalid_threshold);

/* Random-walk step (cfg1 app kernel): every incoming item of every local
 * rank gets round field = rnd and is re-emitted to
 * multiply-shift(splitmix64(seed ^ (rnd << 40) ^ id), R).  Items are not
 * re-emitted once rnd > last_round (the walk ends). */
int rafi_drv_random_walk(rafi_ctx* ctx, uint64_t seed, uint32_t rnd, uint32_t last_round);

#ifdef __cplusplus
}
#endif

#endif /* RAFI_DRIVERS_H */
