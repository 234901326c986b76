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

/* Device re-emit of a resident batch (the app-facing emit path, PAPER:70-71,
 * 98): threads load items (item_bytes, packed; a device pointer aligned to 16
 * bytes) and their dests (int32, device) and emit them through
 * rafi::Queue<T> on local rank `local`'s queue, with vector item loads and
 * stores.  batch = 1: one emitOutgoing(item, dest) per item (one warp
 * atomicAdd per 32 items); batch = 8: the batched emitOutgoing<8> (one warp
 * atomicAdd per 256 items).  Same accept / drop / reject rules as every emit.
 * For item sizes of rafi_drv_emit_synthetic plus 4, 8 and 12 bytes
 * (RAFI_ERR_UNSUPPORTED otherwise).  Used to time the device emit against its
 * 2 * (item_bytes + 4) bytes-per-item roofline. */
int rafi_drv_emit_items(rafi_ctx* ctx, int local, const void* items, const int32_t* dests, uint64_t n, int batch);

/* Random-walk step (cfg1 app kernel): every incoming item of every local
 * rank gets round field = rnd and is re-emitted to
 * multiply-shift(splitmix64(seed ^ (rnd << 40) ^ id), R).  Items are not
 * re-emitted once rnd > last_round (the walk ends). */
int rafi_drv_random_walk(rafi_ctx* ctx, uint64_t seed, uint32_t rnd, uint32_t last_round);

/* ---- cfg4: particle advection proxy (§5.4) ----------------
 * Domain [0,1)^3 split into gx*gy*gz macrocells, rank = (cz*gy + cy)*gx + cx
 * (R must equal gx*gy*gz).  Item (16 B): {u32 id; float x, y, z}.
 * seed: local rank `local` creates n particles, id = rank*n + i, uniformly in
 * its own cell (u_k = top 24 bits of splitmix64(seed ^ id<<3 ^ k) * 2^-24),
 * and emits each to owner(position).
 * step: every incoming particle of every local rank takes one RK4 step of
 * v = omega*(-(y-1/2), x-1/2, 0) + (0, 0, eps) with step h; it
 * retires if it left [0,1)^3 or rnd >= max_rounds, else it is emitted to
 * owner(new position).  Float math is + - * / only, no FMA
 * contraction, so the CPU twin in oracle/ matches bit for bit. */
int rafi_drv_advect_seed(rafi_ctx* ctx, int local, uint64_t n, uint64_t seed, int gx, int gy, int gz);
int rafi_drv_advect_step(rafi_ctx* ctx, uint32_t rnd, uint32_t max_rounds, float omega, float eps, float h, int gx,
                         int gy, int gz);

/* ---- cfg3: brick-decomposed ray marcher proxy ----
 * Same brick decomposition.  Item (48 B): {float o[3], d[3], t; u32 id;
 * float integral; u32 rng, bounces, pad}.
 * seed: n rays per local rank, origin uniform in its brick, direction a
 * normalised hashed vector (sqrt and /), emitted to owner(origin).
 * step: every incoming ray marches with dt = 1/256: o += dt*d; if it left the
 * domain it retires (result[id] = integral); if it entered another brick it is
 * emitted to that brick's rank; else integral += rho(voxel)*dt with rho a
 * hash of the 1/128 voxel, and with probability p_thr/2^32 per step it
 * scatters to a new hashed direction (retiring after max_bounces).  After
 * max_steps steps in one round it is re-emitted to its own rank.
 * result: device float[R*n] indexed by id. */
int rafi_drv_march_seed(rafi_ctx* ctx, int local, uint64_t n, uint64_t seed, int gx, int gy, int gz);
int rafi_drv_march_step(rafi_ctx* ctx, uint32_t rnd, uint64_t seed, uint32_t p_thr, uint32_t max_bounces,
                        uint32_t max_steps, int gx, int gy, int gz, float* result);

/* ---- N-body exchange pattern: three contexts, three item types
 * P: Particle (40 B) {float pos[3], vel[3], force[3], mass};
 * V: VirtualParticle (24 B) {float com[3], mass, smax; int sourceRank};
 * Q: RefinementReq (4 B) {int senderRank}.
 * Owner of a position: Morton order, 10 bits per axis, R equal code
 * intervals.  Multipole statistics are exact integer sums of
 * positions quantised to 2^-20 (order independent): stats[L][42] u64 =
 * count, sum[3], min[3], max[3], then 8 octants x (count, sum[3]) about the
 * root centre of mass.  One step, with a forward of the named context after
 * each call: migrate (P) -> stats -> root (V) -> refine (V -> Q) ->
 * respond (Q -> V).  Contexts used together must share the stream and R. */
int rafi_drv_nbody_seed(rafi_ctx* P, int local, uint64_t n, uint64_t seed);
int rafi_drv_nbody_migrate(rafi_ctx* P, float dt);  /* pos += dt*vel (periodic), emit to the owner */
int rafi_drv_nbody_stats(rafi_ctx* P, unsigned long long* stats_dev);
int rafi_drv_nbody_root(rafi_ctx* V, const unsigned long long* stats_dev);  /* root VP to every other rank */
/* each received root whose smax^2 > theta2 * dist^2 to this rank's centre
 * of mass gets a RefinementReq back to its source */
int rafi_drv_nbody_refine(rafi_ctx* V, rafi_ctx* Q, const unsigned long long* stats_dev, float theta2);
/* each request is answered with this rank's non-empty octant nodes */
int rafi_drv_nbody_respond(rafi_ctx* Q, rafi_ctx* V, const unsigned long long* stats_dev);

/* ---- streamlines on a sampled vector field (§5.4; NEXT-4) --
 * A vertex lattice nx*ny*nz of float3 over [0,1]^3 (x fastest) is split into
 * gx*gy*gz macrocell blocks of (nx-1)/gx x ... cells; every rank keeps its
 * block plus a one-vertex halo, so the RK4 stages of a particle it owns
 * sample exactly the global field as long as h*|v| <= half a cell (the
 * result is then independent of the partition).  Item (16 B): {u32 id;
 * float x, y, z}.  Sampling is trilinear, evaluated as
 * a*(1-f) + b*f per axis (x, then y, then z); owner(p) = macrocell of the
 * lattice cell floor(p*(n-1)) clamped to the last cell.
 * step (round rnd): one classical RK4 step per incoming particle; it retires
 * -- result_pos[id] / result_steps[id] written -- if a stage leaves the
 * domain (steps = rnd-1, position unchanged), the step moved less than eps,
 * the new position is outside [0,1)^3, or rnd >= max_steps; otherwise it is
 * emitted to owner(new position).
 * create copies the blocks of every local rank from the host field
 * (nx*ny*nz*3 floats) to the device; the handle is freed by destroy. */
typedef struct rafi_stream_field rafi_stream_field;
int rafi_drv_stream_create(rafi_ctx* ctx, const float* field_host, int nx, int ny, int nz, int gx, int gy, int gz,
                           rafi_stream_field** out);
/* emits n seeds (positions seeds_host[3n], ids id0..id0+n-1) from local rank
 * `local` to their owners */
int rafi_drv_stream_seed(rafi_stream_field* f, int local, const float* seeds_host, uint64_t n, uint32_t id0);
int rafi_drv_stream_step(rafi_stream_field* f, uint32_t rnd, float h, float eps, uint32_t max_steps,
                         float* result_pos, uint32_t* result_steps);
int rafi_drv_stream_destroy(rafi_stream_field* f);
/* number of stage samples that fell outside a rank's block + halo (the
 * h*|v| <= half-cell condition broken); blocking */
int rafi_drv_stream_halo_misses(rafi_stream_field* f, int* count);

#ifdef __cplusplus
}
#endif

#endif /* RAFI_DRIVERS_H */
