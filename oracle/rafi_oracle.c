/*
 * rafi_oracle.c -- CPU ORACLE for RaFI work-item forwarding (arXiv 2605.30294).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load or call this code.
 * The product path (paper_2605_30294_b200/) never links, imports or executes
 * anything under oracle/, and this file shares no code, header, table or
 * constant with it.
 *
 * Plain, slow, single-threaded C11.  One process simulates all R ranks of a
 * communicator; "MPI" collectives are written out as the loops they define.
 * Citations are PAPER:<line> (section) of /root/reference/PAPER.md and
 * SPEC:<line> of SPEC.md (used for worked examples only).
 *
 * Two independent forward() implementations:
 *   orc_forward_plain    -- the plain definition of the result (filter each
 *                           destination's items in slot order, concatenate in
 *                           source-rank order).  This is what the method
 *                           computes "up to rounding order" (there is no FP).
 *   orc_forward_literal  -- the paper's pipeline step by step: 64-bit sort key
 *                           (PAPER:109), LSD radix sort, gather
 *                           (PAPER:113), boundary kernel with {-1,-1}
 *                           sentinels + host gap fill,
 *                           MPI_Alltoall of counts + prefix sums,
 *                           MPI_Alltoallv on byte counts, wrap-up
 *                           (PAPER:134), reduce-add.
 * Tests require the two to agree byte for byte, and pin both against SPEC's
 * worked examples, closed forms and brute force (tests/test_oracle*.py).
 *
 * Readings of the paper, in brief:
 *   Z1 drop rule: slot = value of the emit counter before the increment; the
 *      emit is kept iff slot < capacity; the counter is not clamped.
 *   Z2 invalid dest (not in [0,R)): rejected, counted, takes no slot.
 *   Z3 receive overflow (some rank would receive > capacity): detected after
 *      the count exchange, reported on every rank, state unchanged.
 *   Z4 forward returns the all-reduced sum of received counts.
 *   Z5 incoming order: source-rank major, then emission-slot order.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_ERR_ARG (-1)
#define ORC_ERR_NOMEM (-2)
#define ORC_ERR_RECV_OVERFLOW (-3)

typedef struct orc_world {
    int R;              /* ranks in the simulated communicator */
    uint64_t cap;       /* queue capacity in items (resizeRayQueues) */
    uint64_t B;         /* item size in bytes ("trivially copyable") */
    /* per-rank state: the paper's "four pointers" */
    uint8_t **out;      /* [R][cap*B] output queue */
    int32_t **dest;     /* [R][cap] destination ranks */
    uint64_t *emitted;  /* [R] the atomic emit counter */
    uint64_t *invalid;  /* [R] rejected emits (Z2) */
    uint8_t **in;       /* [R][cap*B] input queue */
    uint64_t *n_in;     /* [R] numIncoming() */
    /* results of the last forward (for parity tests) */
    uint8_t **binned;   /* [R][cap*B] sender-side dest-sorted batch */
    uint64_t *C;        /* [R*R] C[s*R+d] = items s sent to d */
    uint64_t *send_off; /* [R*R] send_off[s*R+d] */
    uint64_t *recv_off; /* [R*R] recv_off[d*R+s] */
    uint64_t *dropped;  /* [R] dropped at emit in the last round */
    uint64_t *invalid_last; /* [R] invalid emits in the last round */
    uint64_t G;         /* last return value */
} orc_world;

static void *xcalloc(size_t n, size_t sz) {
    if (n == 0 || sz == 0) return calloc(1, 1);
    return calloc(n, sz);
}

void orc_destroy(orc_world *w) {
    if (!w) return;
    for (int r = 0; r < w->R; ++r) {
        if (w->out) free(w->out[r]);
        if (w->dest) free(w->dest[r]);
        if (w->in) free(w->in[r]);
        if (w->binned) free(w->binned[r]);
    }
    free(w->out); free(w->dest); free(w->in); free(w->binned);
    free(w->emitted); free(w->invalid); free(w->n_in);
    free(w->C); free(w->send_off); free(w->recv_off);
    free(w->dropped); free(w->invalid_last);
    free(w);
}

/* HostContext<T> + resizeRayQueues(cap) for all R simulated ranks. */
orc_world *orc_create(int R, uint64_t cap, uint64_t B) {
    if (R < 1 || B < 1) return NULL;
    orc_world *w = (orc_world *)calloc(1, sizeof(orc_world));
    if (!w) return NULL;
    w->R = R; w->cap = cap; w->B = B;
    w->out = (uint8_t **)xcalloc((size_t)R, sizeof(uint8_t *));
    w->dest = (int32_t **)xcalloc((size_t)R, sizeof(int32_t *));
    w->in = (uint8_t **)xcalloc((size_t)R, sizeof(uint8_t *));
    w->binned = (uint8_t **)xcalloc((size_t)R, sizeof(uint8_t *));
    w->emitted = (uint64_t *)xcalloc((size_t)R, 8);
    w->invalid = (uint64_t *)xcalloc((size_t)R, 8);
    w->n_in = (uint64_t *)xcalloc((size_t)R, 8);
    w->C = (uint64_t *)xcalloc((size_t)R * R, 8);
    w->send_off = (uint64_t *)xcalloc((size_t)R * R, 8);
    w->recv_off = (uint64_t *)xcalloc((size_t)R * R, 8);
    w->dropped = (uint64_t *)xcalloc((size_t)R, 8);
    w->invalid_last = (uint64_t *)xcalloc((size_t)R, 8);
    if (!w->out || !w->dest || !w->in || !w->binned || !w->emitted || !w->invalid ||
        !w->n_in || !w->C || !w->send_off || !w->recv_off || !w->dropped || !w->invalid_last) {
        orc_destroy(w); return NULL;
    }
    for (int r = 0; r < R; ++r) {
        w->out[r] = (uint8_t *)xcalloc((size_t)cap, (size_t)B);
        w->dest[r] = (int32_t *)xcalloc((size_t)cap, 4);
        w->in[r] = (uint8_t *)xcalloc((size_t)cap, (size_t)B);
        w->binned[r] = (uint8_t *)xcalloc((size_t)cap, (size_t)B);
        if (!w->out[r] || !w->dest[r] || !w->in[r] || !w->binned[r]) { orc_destroy(w); return NULL; }
    }
    return w;
}

/* ---- device interface, simulated sequentially ---------- */

/* numIncoming() */
uint64_t orc_num_incoming(const orc_world *w, int r) { return w->n_in[r]; }

/* getIncoming(i): copies item i of rank r's input queue. */
int orc_get_incoming(const orc_world *w, int r, uint64_t i, void *item) {
    if (r < 0 || r >= w->R || i >= w->n_in[r]) return ORC_ERR_ARG;
    memcpy(item, w->in[r] + i * w->B, (size_t)w->B);
    return ORC_OK;
}

/* emitOutgoing(item, dest): "atomically appends a new ray to
 * the output queue"; "Calls ... that would exceed the output queue size will
 * simply get dropped"; dest "has to be a valid MPI rank" (Z2).  Sequential
 * model of the atomicAdd: slot = counter value before the add (Z1).
 * Returns 1 if stored, 0 if dropped or rejected. */
int orc_emit(orc_world *w, int r, const void *item, int64_t d) {
    if (d < 0 || d >= w->R) { w->invalid[r] += 1; return 0; }          /* Z2 */
    uint64_t slot = w->emitted[r];
    w->emitted[r] += 1;
    if (slot < w->cap) {
        memcpy(w->out[r] + slot * w->B, item, (size_t)w->B);
        w->dest[r][slot] = (int32_t)d;
        return 1;
    }
    return 0;                                                           /* Z1 */
}

/* n sequential emitOutgoing calls in array order (the same rule as orc_emit,
 * one call per item).  Returns the number accepted. */
uint64_t orc_emit_many(orc_world *w, int r, const void *items, const int32_t *dests, uint64_t n) {
    uint64_t acc = 0;
    const uint8_t *p = (const uint8_t *)items;
    for (uint64_t i = 0; i < n; ++i) acc += (uint64_t)orc_emit(w, r, p + i * w->B, dests[i]);
    return acc;
}

/* Load an observed queue state (items in slot order, their dests, the raw
 * counter values) into rank r -- used for snapshot parity, where the emit
 * slot order was decided by GPU atomics. */
int orc_load_snapshot(orc_world *w, int r, const void *items, const int32_t *dests,
                      uint64_t ctr, uint64_t invalid) {
    if (r < 0 || r >= w->R) return ORC_ERR_ARG;
    uint64_t n = ctr < w->cap ? ctr : w->cap;
    for (uint64_t i = 0; i < n; ++i)
        if (dests[i] < 0 || dests[i] >= w->R) return ORC_ERR_ARG;
    if (n) {
        memcpy(w->out[r], items, (size_t)(n * w->B));
        memcpy(w->dest[r], dests, (size_t)(n * 4));
    }
    w->emitted[r] = ctr;
    w->invalid[r] = invalid;
    return ORC_OK;
}

/* Seed rank r's input queue directly (tests only; the paper seeds by emitting
 * to self and forwarding once). */
int orc_set_incoming(orc_world *w, int r, const void *items, uint64_t n) {
    if (r < 0 || r >= w->R || n > w->cap) return ORC_ERR_ARG;
    if (n) memcpy(w->in[r], items, (size_t)(n * w->B));
    w->n_in[r] = n;
    return ORC_OK;
}

/* ---- forwardRays(), plain definition ----------------- */

/* Every emitted ray "ends up exactly where the corresponding emitOutgoing
 * call indicated it should go"; per destination, sources in rank
 * order (prefix-sum recv offsets) and, per source, the stable
 * (dest, slot) order of the sort key.  Returns G (the
 * all-reduced received count) or ORC_ERR_RECV_OVERFLOW (Z3). */
int64_t orc_forward_plain(orc_world *w) {
    const int R = w->R;
    const uint64_t B = w->B;
    uint64_t *n = (uint64_t *)xcalloc((size_t)R, 8);
    uint64_t *C = (uint64_t *)xcalloc((size_t)R * R, 8);
    uint64_t *T = (uint64_t *)xcalloc((size_t)R, 8);
    if (!n || !C || !T) { free(n); free(C); free(T); return ORC_ERR_NOMEM; }

    /* items actually in each queue (Z1) and the count matrix */
    for (int s = 0; s < R; ++s) {
        n[s] = w->emitted[s] < w->cap ? w->emitted[s] : w->cap;
        for (uint64_t i = 0; i < n[s]; ++i) C[(size_t)s * R + w->dest[s][i]] += 1;
    }
    for (int d = 0; d < R; ++d)
        for (int s = 0; s < R; ++s) T[d] += C[(size_t)s * R + d];
    for (int d = 0; d < R; ++d)
        if (T[d] > w->cap) { free(n); free(C); free(T); return ORC_ERR_RECV_OVERFLOW; } /* Z3 */

    /* sender side: one contiguous block per destination, slot order inside */
    for (int s = 0; s < R; ++s) {
        uint64_t pos = 0;
        for (int d = 0; d < R; ++d) {
            w->send_off[(size_t)s * R + d] = pos;
            for (uint64_t i = 0; i < n[s]; ++i)
                if (w->dest[s][i] == d) {
                    memcpy(w->binned[s] + pos * B, w->out[s] + i * B, (size_t)B);
                    pos += 1;
                }
        }
    }
    /* receiver side: concatenate the blocks addressed to d, source-major */
    uint64_t G = 0;
    for (int d = 0; d < R; ++d) {
        uint64_t pos = 0;
        for (int s = 0; s < R; ++s) {
            uint64_t c = C[(size_t)s * R + d];
            w->recv_off[(size_t)d * R + s] = pos;
            if (c) memcpy(w->in[d] + pos * B, w->binned[s] + w->send_off[(size_t)s * R + d] * B,
                          (size_t)(c * B));
            pos += c;
        }
        w->n_in[d] = pos;
        G += pos;
    }
    /* wrap-up */
    for (int s = 0; s < R; ++s) {
        w->dropped[s] = w->emitted[s] - n[s];
        w->invalid_last[s] = w->invalid[s];
        w->emitted[s] = 0;
        w->invalid[s] = 0;
    }
    memcpy(w->C, C, (size_t)R * R * 8);
    w->G = G;
    free(n); free(C); free(T);
    return (int64_t)G;
}

/* ---- forwardRays(), paper-literal pipeline --------------- */

/* "sets the upper 32 bits of the i'th element to the desired
 * destination rank, and the lower 32 bits to i". */
void orc_pack_keys(const int32_t *dest, uint64_t n, uint64_t *keys) {
    for (uint64_t i = 0; i < n; ++i) keys[i] = ((uint64_t)(uint32_t)dest[i] << 32) | (uint64_t)(uint32_t)i;
}

/* key-only radix sort of the uint64 keys.  LSD, 16-bit digits,
 * four stable counting-sort passes (the reading SPEC:253 states). */
int orc_radix_sort_keys(uint64_t *keys, uint64_t n) {
    uint64_t *tmp = (uint64_t *)xcalloc((size_t)(n ? n : 1), 8);
    uint64_t *cnt = (uint64_t *)xcalloc(65536, 8);
    if (!tmp || !cnt) { free(tmp); free(cnt); return ORC_ERR_NOMEM; }
    for (int pass = 0; pass < 4; ++pass) {
        int shift = 16 * pass;
        memset(cnt, 0, 65536 * 8);
        for (uint64_t i = 0; i < n; ++i) cnt[(keys[i] >> shift) & 0xFFFF] += 1;
        uint64_t sum = 0;
        for (int b = 0; b < 65536; ++b) { uint64_t c = cnt[b]; cnt[b] = sum; sum += c; }
        for (uint64_t i = 0; i < n; ++i) tmp[cnt[(keys[i] >> shift) & 0xFFFF]++] = keys[i];
        memcpy(keys, tmp, (size_t)(n * 8));
    }
    free(tmp); free(cnt);
    return ORC_OK;
}

/* "for each array index outIdx, reads the given 64-bit value ...
 * extracts that pair's ray index, reads the ray from the corresponding
 * location in the input array, and stores that in the outIdx position". */
void orc_gather(const uint8_t *src, const uint64_t *keys, uint64_t n, uint64_t B, uint8_t *dst,
                int32_t *sorted_dest) {
    for (uint64_t o = 0; o < n; ++o) {
        uint64_t i = keys[o] & 0xFFFFFFFFull;
        memcpy(dst + o * B, src + i * B, (size_t)B);
        if (sorted_dest) sorted_dest[o] = (int32_t)(keys[o] >> 32);
    }
}

/* PAPER:121-124, Step 1: begin/end per rank initialised to {-1,-1}; index i
 * is a beginning if dest[i-1] differs (or i == 0) and an end if dest[i+1]
 * differs (or i == n-1) -- the garbled sentence read as Z6.  Then, on the
 * host, "fill in any gaps (some ranks may not have received any rays)" and
 * count = end - begin.  Gap reading: an empty rank's offset is
 * where the next block starts, i.e. the end of the previous non-empty one. */
void orc_compute_segments(const int32_t *sorted_dest, uint64_t n, int R, uint64_t *send_count,
                          uint64_t *send_offset) {
    int64_t *begin = (int64_t *)xcalloc((size_t)R, 8);
    int64_t *end = (int64_t *)xcalloc((size_t)R, 8);
    for (int r = 0; r < R; ++r) { begin[r] = -1; end[r] = -1; }
    for (uint64_t i = 0; i < n; ++i) {       /* "one thread per index" */
        int32_t d = sorted_dest[i];
        if (i == 0 || sorted_dest[i - 1] != d) begin[d] = (int64_t)i;
        if (i == n - 1 || sorted_dest[i + 1] != d) end[d] = (int64_t)i + 1;
    }
    int64_t last_end = 0;                    /* host gap fill */
    for (int r = 0; r < R; ++r) {
        if (begin[r] == -1) { begin[r] = last_end; end[r] = last_end; }
        send_offset[r] = (uint64_t)begin[r];
        send_count[r] = (uint64_t)(end[r] - begin[r]);
        last_end = end[r];
    }
    free(begin); free(end);
}

/* MPI_Alltoall of one count per peer: rank d's recv[d][s] is
 * rank s's send[s][d].  Buffers are [R][R], row = the calling rank. */
void orc_alltoall_u64(int R, const uint64_t *send, uint64_t *recv) {
    for (int d = 0; d < R; ++d)
        for (int s = 0; s < R; ++s) recv[(size_t)d * R + s] = send[(size_t)s * R + d];
}

/* MPI_Alltoallv on bytes: for every (s,d), copy
 * send_bytes[s][d] bytes from sendbuf[s]+sdispl[s][d] to
 * recvbuf[d]+rdispl[d][s]. */
void orc_alltoallv_bytes(int R, uint8_t *const *sendbuf, const uint64_t *scount,
                         const uint64_t *sdispl, uint8_t *const *recvbuf, const uint64_t *rdispl) {
    for (int s = 0; s < R; ++s)
        for (int d = 0; d < R; ++d) {
            uint64_t c = scount[(size_t)s * R + d];
            if (c) memcpy(recvbuf[d] + rdispl[(size_t)d * R + s], sendbuf[s] + sdispl[(size_t)s * R + d],
                          (size_t)c);
        }
}

int64_t orc_forward_literal(orc_world *w) {
    const int R = w->R;
    const uint64_t B = w->B;
    const size_t RR = (size_t)R * R;
    uint64_t *send_count = (uint64_t *)xcalloc(RR, 8);  /* [s][d] */
    uint64_t *send_offset = (uint64_t *)xcalloc(RR, 8); /* [s][d] */
    uint64_t *recv_count = (uint64_t *)xcalloc(RR, 8);  /* [d][s] */
    uint64_t *recv_offset = (uint64_t *)xcalloc(RR, 8); /* [d][s] */
    uint64_t *n = (uint64_t *)xcalloc((size_t)R, 8);
    if (!send_count || !send_offset || !recv_count || !recv_offset || !n) goto nomem;

    /* per rank: swap queues, sort by destination, tally */
    for (int s = 0; s < R; ++s) {
        n[s] = w->emitted[s] < w->cap ? w->emitted[s] : w->cap;
        uint64_t *keys = (uint64_t *)xcalloc((size_t)(n[s] ? n[s] : 1), 8);
        int32_t *sdest = (int32_t *)xcalloc((size_t)(n[s] ? n[s] : 1), 4);
        if (!keys || !sdest) { free(keys); free(sdest); goto nomem; }
        orc_pack_keys(w->dest[s], n[s], keys);
        if (orc_radix_sort_keys(keys, n[s]) != ORC_OK) { free(keys); free(sdest); goto nomem; }
        orc_gather(w->out[s], keys, n[s], B, w->binned[s], sdest);
        orc_compute_segments(sdest, n[s], R, send_count + (size_t)s * R, send_offset + (size_t)s * R);
        free(keys); free(sdest);
    }
    /* Step 2: MPI_Alltoall of counts, then prefix sums */
    orc_alltoall_u64(R, send_count, recv_count);
    for (int d = 0; d < R; ++d) {
        uint64_t sum = 0;
        for (int s = 0; s < R; ++s) { recv_offset[(size_t)d * R + s] = sum; sum += recv_count[(size_t)d * R + s]; }
        if (sum > w->cap) {                  /* Z3: before any payload moves */
            free(send_count); free(send_offset); free(recv_count); free(recv_offset); free(n);
            return ORC_ERR_RECV_OVERFLOW;
        }
    }
    /* Step 3: byte counts = count * sizeof(RayT), MPI_Alltoallv */
    {
        uint64_t *sb = (uint64_t *)xcalloc(RR, 8), *sd = (uint64_t *)xcalloc(RR, 8), *rd = (uint64_t *)xcalloc(RR, 8);
        if (!sb || !sd || !rd) { free(sb); free(sd); free(rd); goto nomem; }
        for (size_t k = 0; k < RR; ++k) { sb[k] = send_count[k] * B; sd[k] = send_offset[k] * B; rd[k] = recv_offset[k] * B; }
        orc_alltoallv_bytes(R, w->binned, sb, sd, w->in, rd);
        free(sb); free(sd); free(rd);
    }
    /* wrap-up and the "reduce add" */
    uint64_t G = 0;
    for (int d = 0; d < R; ++d) {
        uint64_t tot = 0;
        for (int s = 0; s < R; ++s) tot += recv_count[(size_t)d * R + s];
        w->n_in[d] = tot;
        G += tot;
    }
    for (int s = 0; s < R; ++s) {
        w->dropped[s] = w->emitted[s] - n[s];
        w->invalid_last[s] = w->invalid[s];
        w->emitted[s] = 0;
        w->invalid[s] = 0;
    }
    memcpy(w->C, send_count, RR * 8);
    memcpy(w->send_off, send_offset, RR * 8);
    memcpy(w->recv_off, recv_offset, RR * 8);
    w->G = G;
    free(send_count); free(send_offset); free(recv_count); free(recv_offset); free(n);
    return (int64_t)G;
nomem:
    free(send_count); free(send_offset); free(recv_count); free(recv_offset); free(n);
    return ORC_ERR_NOMEM;
}

/* ---- accessors for the ctypes wrapper ------------------------------------ */
int orc_R(const orc_world *w) { return w->R; }
uint64_t orc_cap(const orc_world *w) { return w->cap; }
uint64_t orc_B(const orc_world *w) { return w->B; }
uint8_t *orc_out_ptr(orc_world *w, int r) { return w->out[r]; }
int32_t *orc_dest_ptr(orc_world *w, int r) { return w->dest[r]; }
uint8_t *orc_in_ptr(orc_world *w, int r) { return w->in[r]; }
uint8_t *orc_binned_ptr(orc_world *w, int r) { return w->binned[r]; }
uint64_t orc_emitted(const orc_world *w, int r) { return w->emitted[r]; }
uint64_t orc_invalid(const orc_world *w, int r) { return w->invalid[r]; }
uint64_t orc_dropped_last(const orc_world *w, int r) { return w->dropped[r]; }
uint64_t orc_invalid_last(const orc_world *w, int r) { return w->invalid_last[r]; }
const uint64_t *orc_C_ptr(const orc_world *w) { return w->C; }
const uint64_t *orc_send_off_ptr(const orc_world *w) { return w->send_off; }
const uint64_t *orc_recv_off_ptr(const orc_world *w) { return w->recv_off; }
uint64_t orc_G(const orc_world *w) { return w->G; }
