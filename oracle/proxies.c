/*
 * proxies.c -- CPU twins of the proxy applications (cfg3 ray marcher, cfg4
 * particle advector) that drive the forwarding path in tests and benches.
 *
 * TEST INFRASTRUCTURE ONLY (see rafi_oracle.c).  Written separately from the
 * GPU drivers (paper_2605_30294_b200/csrc/drivers.cu); the two share no code.
 * They follow the same recipe, include/rafi_drivers.h, so the tests can
 * require bit-identical results.  Float math is + - * / sqrt only, compiled
 * with -ffp-contract=off (no FMA), IEEE single precision (SSE2).
 *
 * These are application steps, not the method: the paper's apps trace rays
 * through bricks (VoPaT) and advect particles with RK4 across
 * macrocells; each step reads a rank's incoming queue with
 * getIncoming() and emits with emitOutgoing() (the oracle's orc_emit).
 * PARITY UNPINNED with respect to the paper for absolute proxy values (the
 * paper prints none); pinned by closed forms in tests/test_proxies.py.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

typedef struct orc_world orc_world;
uint64_t orc_num_incoming(const orc_world *w, int r);
int orc_get_incoming(const orc_world *w, int r, uint64_t i, void *item);
int orc_emit(orc_world *w, int r, const void *item, int64_t d);

static uint64_t sm64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static float unit24(uint64_t h) { return (float)(uint32_t)(h >> 40) * 5.9604644775390625e-08f; }

static int clampi(int v, int hi) { return v < 0 ? 0 : (v > hi ? hi : v); }

/* rank = (cz*gy + cy)*gx + cx of the cell containing (x,y,z) */
int orc_grid_owner(float x, float y, float z, int gx, int gy, int gz) {
    int cx = clampi((int)(x * (float)gx), gx - 1);
    int cy = clampi((int)(y * (float)gy), gy - 1);
    int cz = clampi((int)(z * (float)gz), gz - 1);
    return (cz * gy + cy) * gx + cx;
}

static int in_domain(float x, float y, float z) {
    return x >= 0.0f && x < 1.0f && y >= 0.0f && y < 1.0f && z >= 0.0f && z < 1.0f;
}

static void seed_position(uint64_t seed, uint32_t id, int r, int gx, int gy, int gz, float *x, float *y, float *z) {
    int cx = r % gx, cy = (r / gx) % gy, cz = r / (gx * gy);
    uint64_t b = seed ^ ((uint64_t)id << 3);
    *x = ((float)cx + unit24(sm64(b ^ 0u))) / (float)gx;
    *y = ((float)cy + unit24(sm64(b ^ 1u))) / (float)gy;
    *z = ((float)cz + unit24(sm64(b ^ 2u))) / (float)gz;
}

static void normalize3(float ax, float ay, float az, float *d) {
    float len2 = ax * ax + ay * ay + az * az;
    if (len2 < 1e-6f) { d[0] = 1.0f; d[1] = 0.0f; d[2] = 0.0f; return; }
    float len = sqrtf(len2);
    d[0] = ax / len; d[1] = ay / len; d[2] = az / len;
}

/* ---- cfg4: particle {u32 id; float x, y, z} --------------------------- */

typedef struct { uint32_t id; float x, y, z; } particle_t;

void orc_advect_seed(orc_world *w, int r, uint64_t n, uint64_t seed, int gx, int gy, int gz) {
    for (uint64_t i = 0; i < n; ++i) {
        particle_t p;
        p.id = (uint32_t)((uint64_t)r * n + i);
        seed_position(seed, p.id, r, gx, gy, gz, &p.x, &p.y, &p.z);
        orc_emit(w, r, &p, orc_grid_owner(p.x, p.y, p.z, gx, gy, gz));
    }
}

static void velocity(float omega, float eps, float x, float y, float *v) {
    v[0] = -(omega * (y - 0.5f));   /* rigid rotation about the centre axis */
    v[1] = omega * (x - 0.5f);
    v[2] = eps;                     /* plus a small drift */
}

/* one classical RK4 step, then retire or emit to the owner */
void orc_advect_step(orc_world *w, int r, uint32_t rnd, uint32_t max_rounds, float omega, float eps, float h,
                     int gx, int gy, int gz) {
    const float hh = 0.5f * h, h6 = h / 6.0f;
    uint64_t n = orc_num_incoming(w, r);
    for (uint64_t i = 0; i < n; ++i) {
        particle_t p;
        float k1[3], k2[3], k3[3], k4[3];
        orc_get_incoming(w, r, i, &p);
        velocity(omega, eps, p.x, p.y, k1);
        velocity(omega, eps, p.x + hh * k1[0], p.y + hh * k1[1], k2);
        velocity(omega, eps, p.x + hh * k2[0], p.y + hh * k2[1], k3);
        velocity(omega, eps, p.x + h * k3[0], p.y + h * k3[1], k4);
        p.x = p.x + h6 * (((k1[0] + 2.0f * k2[0]) + 2.0f * k3[0]) + k4[0]);
        p.y = p.y + h6 * (((k1[1] + 2.0f * k2[1]) + 2.0f * k3[1]) + k4[1]);
        p.z = p.z + h6 * (((k1[2] + 2.0f * k2[2]) + 2.0f * k3[2]) + k4[2]);
        if (!in_domain(p.x, p.y, p.z) || rnd >= max_rounds) continue;   /* retires */
        orc_emit(w, r, &p, orc_grid_owner(p.x, p.y, p.z, gx, gy, gz));
    }
}

/* ---- cfg3: ray {float o[3], d[3], t; u32 id; float integral; u32 rng, bounces, pad} */

typedef struct {
    float ox, oy, oz, dx, dy, dz, t;
    uint32_t id;
    float integral;
    uint32_t rng, bounces, pad;
} ray_t;

void orc_march_seed(orc_world *w, int r, uint64_t n, uint64_t seed, int gx, int gy, int gz) {
    for (uint64_t i = 0; i < n; ++i) {
        ray_t y;
        float d[3];
        memset(&y, 0, sizeof(y));
        y.id = (uint32_t)((uint64_t)r * n + i);
        seed_position(seed, y.id, r, gx, gy, gz, &y.ox, &y.oy, &y.oz);
        uint64_t b = seed ^ ((uint64_t)y.id << 3);
        normalize3(2.0f * unit24(sm64(b ^ 3u)) - 1.0f, 2.0f * unit24(sm64(b ^ 4u)) - 1.0f,
                   2.0f * unit24(sm64(b ^ 5u)) - 1.0f, d);
        y.dx = d[0]; y.dy = d[1]; y.dz = d[2];
        y.rng = (uint32_t)sm64(b ^ 6u);
        orc_emit(w, r, &y, orc_grid_owner(y.ox, y.oy, y.oz, gx, gy, gz));
    }
}

void orc_march_step(orc_world *w, int me, uint64_t seed, uint32_t p_thr, uint32_t max_bounces,
                    uint32_t max_steps, int gx, int gy, int gz, float *result) {
    const float D = 0.00390625f;   /* march step 1/256 */
    uint64_t n = orc_num_incoming(w, me);
    for (uint64_t i = 0; i < n; ++i) {
        ray_t y;
        orc_get_incoming(w, me, i, &y);
        int dest = me, retired = 0;
        for (uint32_t s = 0; s < max_steps; ++s) {
            y.ox = y.ox + D * y.dx;
            y.oy = y.oy + D * y.dy;
            y.oz = y.oz + D * y.dz;
            y.t = y.t + D;
            if (!in_domain(y.ox, y.oy, y.oz)) { retired = 1; break; }       /* left the domain */
            int o = orc_grid_owner(y.ox, y.oy, y.oz, gx, gy, gz);
            if (o != me) { dest = o; break; }                              /* next brick's rank */
            int ix = clampi((int)(y.ox * 128.0f), 127), iy = clampi((int)(y.oy * 128.0f), 127),
                iz = clampi((int)(y.oz * 128.0f), 127);
            uint64_t hv = sm64(seed ^ ((uint64_t)ix << 42) ^ ((uint64_t)iy << 21) ^ (uint64_t)iz);
            y.integral = y.integral + unit24(hv) * D;                       /* density along the ray */
            uint64_t hr = sm64(((uint64_t)y.id << 32) | y.rng);
            y.rng = (uint32_t)(hr >> 32);
            if ((uint32_t)hr < p_thr) {                                     /* scatter event */
                float d[3];
                y.bounces += 1;
                if (y.bounces > max_bounces) { retired = 1; break; }
                normalize3(2.0f * unit24(sm64(hr ^ 1u)) - 1.0f, 2.0f * unit24(sm64(hr ^ 2u)) - 1.0f,
                           2.0f * unit24(sm64(hr ^ 3u)) - 1.0f, d);
                y.dx = d[0]; y.dy = d[1]; y.dz = d[2];
            }
        }
        if (retired) result[y.id] = y.integral;
        else orc_emit(w, me, &y, dest);
    }
}
