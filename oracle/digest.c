/*
 * digest.c -- STREAMING-DIGEST mode of the CPU oracle (TEST INFRASTRUCTURE ONLY).
 *
 * Same status as rafi_oracle.c: only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load or call this code;
 * it shares nothing with the product path (paper_2605_30294_b200/).
 *
 * What it computes: the result of orc_forward_plain (rafi_oracle.c) for
 * configurations whose materialised state does not fit the host (SURVEY.md
 * §8(c) "Streaming-digest mode"; e.g. cfg5 at R=8 x 32M x 128 B is 64 GiB).
 *
 * By the plain definition of forwardRays, the
 * incoming queue of destination d is the concatenation, over sources
 * s = 0, 1, ..., R-1, of source s's queued items whose destination is d, each
 * source's in slot order (Z5).  So if every source's outgoing queue is fed
 * once, sources in ascending rank order and each queue in slot order, and
 * every item is appended to a running digest of its destination, then digest
 * d folds exactly the item sequence of in_d -- while the count matrix C[s][d]
 * is counted exactly.  Nothing is sorted, nothing is stored.
 * The Z1 drop rule (only min(ctr, cap) items are queued) and the Z3 receive
 * overflow decision (some column sum > cap) are applied as in the plain
 * forward.
 *
 * The digest of an item sequence x_0, x_1, ... of B-byte items:
 *   word_j(x)  = the j-th 8-byte little-endian word of x (last one zero-padded)
 *   H(x)       = fmix64(B ^ sum_j fmix64(word_j(x) ^ ((j + 1) * PHI)))  (sums mod 2^64)
 *   D_0 = SEED;  D_{i+1} = fmix64(D_i + H(x_i))
 * fmix64 is MurmurHash3's 64-bit finaliser.  Chaining makes the digest
 * sensitive to item order; H is sensitive to every byte and its position.
 * orc_digest_items() applies the same fold to a materialised queue (e.g. an
 * incoming queue read back from the GPU), so the two are comparable.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_ERR_ARG (-1)
#define ORC_ERR_NOMEM (-2)
#define ORC_ERR_RECV_OVERFLOW (-3)

static const uint64_t PHI = 0x9E3779B97F4A7C15ull;
static const uint64_t DIGEST_SEED = 0x243F6A8885A308D3ull;

static uint64_t fmix64(uint64_t k) {
    k ^= k >> 33;
    k *= 0xFF51AFD7ED558CCDull;
    k ^= k >> 33;
    k *= 0xC4CEB9FE1A85EC53ull;
    k ^= k >> 33;
    return k;
}

/* H(x) for one B-byte item. */
static uint64_t item_hash(const uint8_t *x, uint64_t B) {
    uint64_t acc = 0;
    uint64_t j = 0;
    for (uint64_t o = 0; o < B; o += 8, ++j) {
        uint64_t w = 0;
        uint64_t len = B - o < 8 ? B - o : 8;
        memcpy(&w, x + o, (size_t)len);               /* little-endian host (x86-64) */
        acc += fmix64(w ^ ((j + 1) * PHI));
    }
    return fmix64(B ^ acc);
}

/* Digest of n materialised items of B bytes (e.g. an incoming queue). */
uint64_t orc_digest_items(const void *items, uint64_t n, uint64_t B) {
    const uint8_t *p = (const uint8_t *)items;
    uint64_t D = DIGEST_SEED;
    for (uint64_t i = 0; i < n; ++i) D = fmix64(D + item_hash(p + i * B, B));
    return D;
}

typedef struct orc_digest {
    int R;
    uint64_t B, cap;
    int next_src;      /* sources must be fed in ascending order */
    uint64_t *C;       /* [R*R] C[s*R+d] */
    uint64_t *D;       /* [R] running digest of in_d */
    uint64_t *fed;     /* [R] items fed per source (the slot index of the next one) */
} orc_digest;

void orc_digest_destroy(orc_digest *g) {
    if (!g) return;
    free(g->C); free(g->D); free(g->fed);
    free(g);
}

orc_digest *orc_digest_create(int R, uint64_t cap, uint64_t B) {
    if (R < 1 || B < 1) return NULL;
    orc_digest *g = (orc_digest *)calloc(1, sizeof(orc_digest));
    if (!g) return NULL;
    g->R = R; g->B = B; g->cap = cap; g->next_src = 0;
    g->C = (uint64_t *)calloc((size_t)R * R, 8);
    g->D = (uint64_t *)calloc((size_t)R, 8);
    g->fed = (uint64_t *)calloc((size_t)R, 8);
    if (!g->C || !g->D || !g->fed) { orc_digest_destroy(g); return NULL; }
    for (int d = 0; d < R; ++d) g->D[d] = DIGEST_SEED;
    return g;
}

/* Feed the next n queued items (slots fed[s] .. fed[s]+n-1, in slot order) of
 * source s.  Sources in ascending order; a source may be fed in several
 * chunks.  Items beyond capacity are not queued (Z1) and must not be fed: the
 * caller feeds exactly min(ctr, cap) items per source.  Every dest must be in
 * [0, R) (invalid emits take no slot, Z2). */
int orc_digest_feed(orc_digest *g, int s, const void *items, const int32_t *dests, uint64_t n) {
    if (s < g->next_src || s >= g->R || g->fed[s] + n > g->cap) return ORC_ERR_ARG;
    const uint8_t *p = (const uint8_t *)items;
    for (uint64_t i = 0; i < n; ++i)
        if (dests[i] < 0 || dests[i] >= g->R) return ORC_ERR_ARG;
    g->next_src = s;
    for (uint64_t i = 0; i < n; ++i) {
        const int d = dests[i];
        g->C[(size_t)s * g->R + d] += 1;
        g->D[d] = fmix64(g->D[d] + item_hash(p + i * g->B, g->B));
    }
    g->fed[s] += n;
    return ORC_OK;
}

/* After all sources were fed: G = sum of all received counts, or
 * ORC_ERR_RECV_OVERFLOW if some destination would receive more than cap (Z3). */
int64_t orc_digest_finish(const orc_digest *g) {
    uint64_t G = 0;
    for (int d = 0; d < g->R; ++d) {
        uint64_t T = 0;
        for (int s = 0; s < g->R; ++s) T += g->C[(size_t)s * g->R + d];
        if (T > g->cap) return ORC_ERR_RECV_OVERFLOW;
        G += T;
    }
    return (int64_t)G;
}

uint64_t orc_digest_value(const orc_digest *g, int d) { return g->D[d]; }
const uint64_t *orc_digest_C_ptr(const orc_digest *g) { return g->C; }
