/*
 * nbody.c -- CPU twin of the N-body exchange-pattern driver (NEXT-2):
 * three RaFI contexts with different item types on one communicator
 * (PAPER:381-410): particle migration, root-multipole broadcast, refinement
 * requests and subtree responses.
 *
 * TEST INFRASTRUCTURE ONLY.  Written separately from the GPU driver
 * (paper_2605_30294_b200/csrc/drivers.cu), following include/rafi_drivers.h.
 * Each "world" argument is one orc_world per context, all with the same R;
 * rank r's step reads r's incoming queue and emits with orc_emit, exactly
 * as the GPU kernels use getIncoming / emitOutgoing.  The physics (forces,
 * leapfrog, BVH) is out of scope; positions drift with their velocity.
 * Parity unpinned w.r.t. the paper (no printed values); pinned by the
 * invariants in tests/test_nbody.py.
 */
#include <stdint.h>
#include <string.h>

typedef struct orc_world orc_world;
uint64_t orc_num_incoming(const orc_world *w, int r);
int orc_get_incoming(const orc_world *w, int r, uint64_t i, void *item);
int orc_emit(orc_world *w, int r, const void *item, int64_t d);
int orc_R(const orc_world *w);

typedef struct { float px, py, pz, vx, vy, vz, fx, fy, fz, mass; } nb_particle;   /* 40 B */
typedef struct { float cx, cy, cz, mass, smax; int32_t source_rank; } nb_virtual; /* 24 B */
typedef struct { int32_t sender_rank; } nb_request;                               /* 4 B */

#define NB_STATS 42

static uint64_t mix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static float top24(uint64_t h) { return (float)(uint32_t)(h >> 40) * 5.9604644775390625e-08f; }

static uint32_t quant20(float x) { return (uint32_t)(x * 1048576.0f); }

/* Morton-order owner: 10 bits per axis interleaved x,y,z from bit 0; R equal
 * intervals of the 30-bit code. */
int orc_morton_owner(float x, float y, float z, int R) {
    uint32_t q[3];
    float c[3] = {x, y, z};
    for (int a = 0; a < 3; ++a) {
        uint32_t v = (uint32_t)(c[a] * 1024.0f);
        q[a] = v > 1023u ? 1023u : v;
    }
    uint64_t code = 0;
    for (int b = 0; b < 10; ++b)
        for (int a = 0; a < 3; ++a) code |= (uint64_t)((q[a] >> b) & 1u) << (3 * b + a);
    return (int)((code * (uint64_t)R) >> 30);
}

static float periodic(float x) {
    if (x < 0.0f) x = x + 1.0f;
    if (x >= 1.0f) x = x - 1.0f;
    return x;
}

void orc_nbody_seed(orc_world *P, int r, uint64_t n, uint64_t seed) {
    int R = orc_R(P);
    for (uint64_t i = 0; i < n; ++i) {
        uint64_t id = (uint64_t)r * n + i, b = seed ^ (id << 3);
        nb_particle p;
        p.px = top24(mix64(b ^ 0u));
        p.py = top24(mix64(b ^ 1u));
        p.pz = top24(mix64(b ^ 2u));
        p.vx = (top24(mix64(b ^ 3u)) - 0.5f) * 0.25f;
        p.vy = (top24(mix64(b ^ 4u)) - 0.5f) * 0.25f;
        p.vz = (top24(mix64(b ^ 5u)) - 0.5f) * 0.25f;
        p.fx = p.fy = p.fz = 0.0f;
        p.mass = 1.0f;
        orc_emit(P, r, &p, orc_morton_owner(p.px, p.py, p.pz, R));
    }
}

/* particle migration: drift, then emit to the owner rank */
void orc_nbody_migrate(orc_world *P, int r, float dt) {
    int R = orc_R(P);
    uint64_t n = orc_num_incoming(P, r);
    for (uint64_t i = 0; i < n; ++i) {
        nb_particle p;
        orc_get_incoming(P, r, i, &p);
        p.px = periodic(p.px + dt * p.vx);
        p.py = periodic(p.py + dt * p.vy);
        p.pz = periodic(p.pz + dt * p.vz);
        orc_emit(P, r, &p, orc_morton_owner(p.px, p.py, p.pz, R));
    }
}

/* root multipole and octant statistics of rank r's particles (exact integers) */
void orc_nbody_stats(const orc_world *P, int r, uint64_t *st) {
    uint64_t n = orc_num_incoming(P, r);
    memset(st, 0, sizeof(uint64_t) * NB_STATS);
    st[4] = st[5] = st[6] = 0xFFFFFFFFull;
    for (uint64_t i = 0; i < n; ++i) {
        nb_particle p;
        orc_get_incoming(P, r, i, &p);
        uint32_t q[3] = {quant20(p.px), quant20(p.py), quant20(p.pz)};
        st[0] += 1;
        for (int a = 0; a < 3; ++a) {
            st[1 + a] += q[a];
            if (q[a] < st[4 + a]) st[4 + a] = q[a];
            if (q[a] > st[7 + a]) st[7 + a] = q[a];
        }
    }
    if (st[0] == 0) return;
    uint64_t c[3] = {st[1] / st[0], st[2] / st[0], st[3] / st[0]};
    for (uint64_t i = 0; i < n; ++i) {
        nb_particle p;
        orc_get_incoming(P, r, i, &p);
        uint32_t q[3] = {quant20(p.px), quant20(p.py), quant20(p.pz)};
        int o = (q[0] >= c[0]) | ((q[1] >= c[1]) << 1) | ((q[2] >= c[2]) << 2);
        uint64_t *s = st + 10 + 4 * o;
        s[0] += 1;
        for (int a = 0; a < 3; ++a) s[1 + a] += q[a];
    }
}

static nb_virtual node_of(const uint64_t *s, float smax, int me) {
    nb_virtual v;
    v.cx = (float)(s[1] / s[0]) * 9.5367431640625e-07f;
    v.cy = (float)(s[2] / s[0]) * 9.5367431640625e-07f;
    v.cz = (float)(s[3] / s[0]) * 9.5367431640625e-07f;
    v.mass = (float)s[0];
    v.smax = smax;
    v.source_rank = me;
    return v;
}

static float root_size(const uint64_t *st) {
    uint64_t e = 0;
    for (int a = 0; a < 3; ++a) {
        uint64_t d = st[7 + a] - st[4 + a];
        if (d > e) e = d;
    }
    return (float)e * 9.5367431640625e-07f;
}

/* root broadcast: rank r's root node to every other rank */
void orc_nbody_root(orc_world *V, int r, const uint64_t *st) {
    if (st[0] == 0) return;
    nb_virtual root = node_of(st, root_size(st), r);
    for (int d = 0; d < orc_R(V); ++d)
        if (d != r) orc_emit(V, r, &root, d);
}

/* multipole acceptance test on each received root; refinement request to its
 * source when smax^2 > theta2 * dist^2 */
void orc_nbody_refine(const orc_world *V, orc_world *Q, int r, const uint64_t *st, float theta2) {
    if (st[0] == 0) return;
    float m[3] = {(float)(st[1] / st[0]) * 9.5367431640625e-07f, (float)(st[2] / st[0]) * 9.5367431640625e-07f,
                  (float)(st[3] / st[0]) * 9.5367431640625e-07f};
    uint64_t n = orc_num_incoming(V, r);
    for (uint64_t i = 0; i < n; ++i) {
        nb_virtual v;
        orc_get_incoming(V, r, i, &v);
        float dx = v.cx - m[0], dy = v.cy - m[1], dz = v.cz - m[2];
        float d2 = dx * dx + dy * dy + dz * dz;
        if (v.smax * v.smax > theta2 * d2) {
            nb_request q = {r};
            orc_emit(Q, r, &q, v.source_rank);
        }
    }
}

/* answer each request with the non-empty octant nodes */
void orc_nbody_respond(const orc_world *Q, orc_world *V, int r, const uint64_t *st) {
    if (st[0] == 0) return;
    float half = root_size(st) * 0.5f;
    uint64_t n = orc_num_incoming(Q, r);
    for (uint64_t i = 0; i < n; ++i) {
        nb_request q;
        orc_get_incoming(Q, r, i, &q);
        for (int o = 0; o < 8; ++o) {
            const uint64_t *s = st + 10 + 4 * o;
            if (s[0]) {
                nb_virtual v = node_of(s, half, r);
                orc_emit(V, r, &v, q.sender_rank);
            }
        }
    }
}
