/*
 * streamlines.c -- CPU twin of the streamline driver (NEXT-4): particle
 * advection on a sampled vector field (§5.4).
 *
 * TEST INFRASTRUCTURE ONLY.  Written separately from the GPU driver
 * (paper_2605_30294_b200/csrc/drivers.cu) after include/rafi_drivers.h.
 * Unlike the GPU driver, which gives every rank its own block plus a
 * one-vertex halo, the twin samples the GLOBAL field: equality of the two is
 * the partition-independence property.  IEEE single precision,
 * -ffp-contract=off.  Pinned by tests/test_streamlines.py (RK4 exact for
 * constant fields, trilinear exact for linear fields, closure of a rigid
 * rotation within the RK4 error bound).
 */
#include <stddef.h>
#include <stdint.h>

typedef struct orc_world orc_world;
uint64_t orc_num_incoming(const orc_world *w, int r);
int orc_get_incoming(const orc_world *w, int r, uint64_t i, void *item);
int orc_emit(orc_world *w, int r, const void *item, int64_t d);

typedef struct { uint32_t id; float x, y, z; } sl_particle;

typedef struct {
    const float *v;       /* nz*ny*nx float3, x fastest */
    int nx, ny, nz;       /* vertices */
    int gx, gy, gz;       /* macrocell grid */
} sl_field;

static int cell_of(float p, int n) {
    int i = (int)(p * (float)(n - 1));
    return i > n - 2 ? n - 2 : (i < 0 ? 0 : i);
}

/* macrocell (rank) of the lattice cell containing p */
int orc_sl_owner(const float *p, int nx, int ny, int nz, int gx, int gy, int gz) {
    int mx = (nx - 1) / gx, my = (ny - 1) / gy, mz = (nz - 1) / gz;
    return ((cell_of(p[2], nz) / mz) * gy + cell_of(p[1], ny) / my) * gx + cell_of(p[0], nx) / mx;
}

static int in_closed(float x, float y, float z) {
    return x >= 0.0f && x <= 1.0f && y >= 0.0f && y <= 1.0f && z >= 0.0f && z <= 1.0f;
}

static int in_open(float x, float y, float z) {
    return x >= 0.0f && x < 1.0f && y >= 0.0f && y < 1.0f && z >= 0.0f && z < 1.0f;
}

/* trilinear interpolation of the 8 surrounding vertex vectors */
static int sample(const sl_field *f, float x, float y, float z, float *out) {
    if (!in_closed(x, y, z)) return 0;
    float ux = x * (float)(f->nx - 1), uy = y * (float)(f->ny - 1), uz = z * (float)(f->nz - 1);
    int i = cell_of(x, f->nx), j = cell_of(y, f->ny), k = cell_of(z, f->nz);
    float fx = ux - (float)i, fy = uy - (float)j, fz = uz - (float)k;
    float gx0 = 1.0f - fx, gy0 = 1.0f - fy, gz0 = 1.0f - fz;
    for (int a = 0; a < 3; ++a) {
#define V(di, dj, dk) f->v[(((size_t)(k + dk) * f->ny + (j + dj)) * f->nx + (i + di)) * 3 + a]
        float c00 = V(0, 0, 0) * gx0 + V(1, 0, 0) * fx;
        float c10 = V(0, 1, 0) * gx0 + V(1, 1, 0) * fx;
        float c01 = V(0, 0, 1) * gx0 + V(1, 0, 1) * fx;
        float c11 = V(0, 1, 1) * gx0 + V(1, 1, 1) * fx;
#undef V
        float c0 = c00 * gy0 + c10 * fy, c1 = c01 * gy0 + c11 * fy;
        out[a] = c0 * gz0 + c1 * fz;
    }
    return 1;
}

void orc_sl_seed(orc_world *w, int r, const float *field, int nx, int ny, int nz, int gx, int gy, int gz,
                 const float *seeds, uint64_t n, uint32_t id0) {
    (void)field;
    for (uint64_t i = 0; i < n; ++i) {
        sl_particle p = {id0 + (uint32_t)i, seeds[3 * i], seeds[3 * i + 1], seeds[3 * i + 2]};
        if (!in_open(p.x, p.y, p.z)) continue;     /* empty streamline */
        float q[3] = {p.x, p.y, p.z};
        orc_emit(w, r, &p, orc_sl_owner(q, nx, ny, nz, gx, gy, gz));
    }
}

/* one RK4 step for every incoming particle of rank r */
void orc_sl_step(orc_world *w, int r, const float *field, int nx, int ny, int nz, int gx, int gy, int gz,
                 uint32_t rnd, float h, float eps, uint32_t max_steps, float *rpos, uint32_t *rsteps) {
    sl_field f = {field, nx, ny, nz, gx, gy, gz};
    const float hh = 0.5f * h, h6 = h / 6.0f;
    uint64_t n = orc_num_incoming(w, r);
    for (uint64_t i = 0; i < n; ++i) {
        sl_particle p;
        float k1[3], k2[3], k3[3], k4[3];
        orc_get_incoming(w, r, i, &p);
        int ok = sample(&f, p.x, p.y, p.z, k1);
        ok = ok && sample(&f, p.x + hh * k1[0], p.y + hh * k1[1], p.z + hh * k1[2], k2);
        ok = ok && sample(&f, p.x + hh * k2[0], p.y + hh * k2[1], p.z + hh * k2[2], k3);
        ok = ok && sample(&f, p.x + h * k3[0], p.y + h * k3[1], p.z + h * k3[2], k4);
        if (!ok) {                                  /* a stage left the domain */
            rpos[3 * p.id] = p.x; rpos[3 * p.id + 1] = p.y; rpos[3 * p.id + 2] = p.z;
            rsteps[p.id] = rnd - 1;
            continue;
        }
        float nxp = p.x + h6 * (((k1[0] + 2.0f * k2[0]) + 2.0f * k3[0]) + k4[0]);
        float nyp = p.y + h6 * (((k1[1] + 2.0f * k2[1]) + 2.0f * k3[1]) + k4[1]);
        float nzp = p.z + h6 * (((k1[2] + 2.0f * k2[2]) + 2.0f * k3[2]) + k4[2]);
        float dx = nxp - p.x, dy = nyp - p.y, dz = nzp - p.z;
        p.x = nxp; p.y = nyp; p.z = nzp;
        if (dx * dx + dy * dy + dz * dz < eps * eps || !in_open(nxp, nyp, nzp) || rnd >= max_steps) {
            rpos[3 * p.id] = nxp; rpos[3 * p.id + 1] = nyp; rpos[3 * p.id + 2] = nzp;
            rsteps[p.id] = rnd;
            continue;
        }
        float q[3] = {nxp, nyp, nzp};
        orc_emit(w, r, &p, orc_sl_owner(q, nx, ny, nz, gx, gy, gz));
    }
}
