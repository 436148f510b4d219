/*
 * jacobi_oracle.c -- TEST INFRASTRUCTURE ONLY (the parity checker).
 *
 * A plain-C restatement of the reference `stencilpipe` hot path, used by
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg.  Nothing in paper_0912_4506_b200/ may link, load or call it.
 *
 * Pinning: tests/test_oracle.py checks every function here against the
 * golden vectors in tests/golden/ that tests/golden/make_golden.py produced
 * by importing the reference package itself (/root/reference/pkg/src), and
 * against the reference tests' in-test known answers.
 *
 * Reference anchors (R = /root/reference/pkg/src/stencilpipe):
 *   ONE_SIXTH, stencil_point  R/kernel.py:15-20
 *   stencil_region            R/kernel.py:27-34   fixed order ((x-+x+)+(y-+y+))+(z-+z+), then *ONE_SIXTH
 *   update_region             R/kernel.py:37-40
 *   sweep_naive               R/kernel.py:43-47
 *   _mix64, _H1.._H3          R/grid.py:54-63
 *   FillPattern.evaluate      R/grid.py:96-118
 *
 * Arithmetic: compile with -O2 -ffp-contract=off and never -ffast-math, so
 * each add and the final multiply are single IEEE-754 round-to-nearest ops,
 * exactly what numpy's ufunc loops do.  float32 grids compute in float (numpy
 * NEP 50 keeps float32 arrays float32 when multiplied by a python float, and
 * ONE_SIXTH then rounds to 0x3E2AAAAB).
 *
 * Layout (shared with the device grid, see include/stencilpipe_b200.h):
 * C order (z, y, x), x contiguous, ghost depths gx/gy/gz on both sides,
 * element (z,y,x) of the interior at  base[origin + z*pz + y*py + x].
 */
#include <stdint.h>
#include <stddef.h>
#include <string.h>
#include <pthread.h>
#include <stdlib.h>
#include <unistd.h>

/* Parallel-for over [lo, hi) on up to or_threads pthreads (static chunks). */
static int g_threads = 0;

int or_num_threads(void) {
    if (g_threads <= 0) {
        const char* e = getenv("ORACLE_THREADS");
        long n = e ? atol(e) : sysconf(_SC_NPROCESSORS_ONLN);
        g_threads = n > 0 ? (int)n : 1;
    }
    return g_threads;
}

void or_set_threads(int n) { g_threads = n; }

typedef void (*range_fn)(void* ctx, int64_t lo, int64_t hi, int chunk);
typedef struct { range_fn fn; void* ctx; int64_t lo, hi; int chunk; } par_job;

static void* par_tramp(void* p) {
    par_job* j = (par_job*)p;
    j->fn(j->ctx, j->lo, j->hi, j->chunk);
    return NULL;
}

static void par_for(int64_t lo, int64_t hi, range_fn fn, void* ctx) {
    int64_t n = hi - lo;
    int nt = or_num_threads();
    if (nt > n) nt = (int)(n > 0 ? n : 1);
    if (nt <= 1) { fn(ctx, lo, hi, 0); return; }
    pthread_t th[256];
    par_job jobs[256];
    if (nt > 256) nt = 256;
    for (int i = 0; i < nt; ++i) {
        jobs[i].fn = fn; jobs[i].ctx = ctx; jobs[i].chunk = i;
        jobs[i].lo = lo + n * i / nt; jobs[i].hi = lo + n * (i + 1) / nt;
        if (i > 0) pthread_create(&th[i], NULL, par_tramp, &jobs[i]);
    }
    par_tramp(&jobs[0]);
    for (int i = 1; i < nt; ++i) pthread_join(th[i], NULL);
}

typedef struct {
    int64_t nx, ny, nz;       /* interior extents */
    int64_t gx, gy, gz;       /* ghost depth present on each side */
    int64_t py, pz;           /* row / plane pitch in elements */
    int64_t origin;           /* element offset of interior (0,0,0) */
} or_layout;

/* ---- FillPattern (R/grid.py:54-118) -------------------------------------- */

#define H1 0x9E3779B97F4A7C15ULL
#define H2 0xBF58476D1CE4E5B9ULL
#define H3 0x94D049BB133111EBULL

static inline uint64_t mix64(uint64_t h) {           /* R/grid.py:60-63 */
    h = (h ^ (h >> 30)) * H2;
    h = (h ^ (h >> 27)) * H3;
    return h ^ (h >> 31);
}

/* R/grid.py:109-117: coordinates are int64 cast to uint64 (so -1 wraps). */
double or_random_value(int64_t z, int64_t y, int64_t x, uint64_t seed) {
    uint64_t h = ((uint64_t)z * H1) ^ ((uint64_t)y * H2) ^ ((uint64_t)x * H3);
    h += seed;
    h = mix64(mix64(h));
    return (double)(h >> 11) * 0x1.0p-53;
}

/* Pattern kinds: 0 constant, 1 linear, 2 hotplate, 3 random (R/grid.py:98-117),
 * 4 random mapped to [-1,1) as 2u-1 (BASELINE config 4).  When has_faces is
 * set, a cell whose GLOBAL coordinate lies outside [0, gn) on some axis takes
 * faces[] of the first such face in the order (z-, z+, y-, y+, x-, x+); this
 * is the duck-typed Dirichlet-box pattern the BASELINE configs describe. */
typedef struct {
    int32_t kind;
    int32_t has_faces;
    double value;
    uint64_t seed;
    int64_t gorigin[3];       /* global (z,y,x) of local interior (0,0,0) */
    int64_t gn[3];            /* global interior extents (z,y,x) */
    double faces[6];
} or_pattern;

double or_pattern_value(const or_pattern* p, int64_t z, int64_t y, int64_t x) {
    int64_t c[3] = {z + p->gorigin[0], y + p->gorigin[1], x + p->gorigin[2]};
    if (p->has_faces) {
        for (int a = 0; a < 3; ++a) {
            if (c[a] < 0) return p->faces[2 * a];
            if (c[a] >= p->gn[a]) return p->faces[2 * a + 1];
        }
    }
    switch (p->kind) {
    case 0: return p->value;
    case 1: return (double)(c[0] + c[1] + c[2]);
    case 2: return c[2] < 0 ? 1.0 : 0.0;
    case 3: return or_random_value(c[0], c[1], c[2], p->seed);
    case 4: return 2.0 * or_random_value(c[0], c[1], c[2], p->seed) - 1.0;
    default: return 0.0;
    }
}

/* Fill the whole ghosted box of a layout (TwoGrid.__init__, R/grid.py:126-134). */
typedef struct { void* base; const or_layout* L; const or_pattern* p; int f32; } fill_ctx;

static void fill_range(void* c, int64_t z0, int64_t z1, int chunk) {
    (void)chunk;
    fill_ctx* k = (fill_ctx*)c;
    const or_layout* L = k->L;
    for (int64_t z = z0; z < z1; ++z)
        for (int64_t y = -L->gy; y < L->ny + L->gy; ++y) {
            int64_t off = L->origin + z * L->pz + y * L->py;
            for (int64_t x = -L->gx; x < L->nx + L->gx; ++x) {
                double v = or_pattern_value(k->p, z, y, x);
                if (k->f32) ((float*)k->base)[off + x] = (float)v;
                else ((double*)k->base)[off + x] = v;
            }
        }
}

void or_fill_f64(double* base, const or_layout* L, const or_pattern* p) {
    fill_ctx k = {base, L, p, 0};
    par_for(-L->gz, L->nz + L->gz, fill_range, &k);
}

void or_fill_f32(float* base, const or_layout* L, const or_pattern* p) {
    fill_ctx k = {base, L, p, 1};
    par_for(-L->gz, L->nz + L->gz, fill_range, &k);
}

/* ---- stencil (R/kernel.py:15-40) ----------------------------------------- */

static const double ONE_SIXTH = 1.0 / 6.0;   /* R/kernel.py:15, 0x3FC5555555555555 */

double or_stencil_point(double xm, double xp, double ym, double yp, double zm, double zp) {
    return ((xm + xp) + (ym + yp) + (zm + zp)) * ONE_SIXTH;   /* R/kernel.py:18-20 */
}

/* update_region (R/kernel.py:37-40): dst[box] = stencil(src) over the logical
 * box [lo, hi) given in (z, y, x) order; every other cell of dst untouched.
 * Per cell: ((x- + x+) + (y- + y+)) + (z- + z+), then * ONE_SIXTH. */
typedef struct { const void* src; void* dst; const or_layout* L; const int64_t* lo; const int64_t* hi; } upd_ctx;

static void upd_range_f64(void* c, int64_t z0, int64_t z1, int chunk) {
    (void)chunk;
    upd_ctx* k = (upd_ctx*)c;
    const int64_t py = k->L->py, pz = k->L->pz;
    for (int64_t z = z0; z < z1; ++z)
        for (int64_t y = k->lo[1]; y < k->hi[1]; ++y) {
            const double* s = (const double*)k->src + k->L->origin + z * pz + y * py;
            double* d = (double*)k->dst + k->L->origin + z * pz + y * py;
            for (int64_t x = k->lo[2]; x < k->hi[2]; ++x) {
                double sx = s[x - 1] + s[x + 1];
                double sy = s[x - py] + s[x + py];
                double sz = s[x - pz] + s[x + pz];
                d[x] = ((sx + sy) + sz) * ONE_SIXTH;
            }
        }
}

static void upd_range_f32(void* c, int64_t z0, int64_t z1, int chunk) {
    (void)chunk;
    upd_ctx* k = (upd_ctx*)c;
    const int64_t py = k->L->py, pz = k->L->pz;
    const float sixth = (float)ONE_SIXTH;       /* 0x3E2AAAAB */
    for (int64_t z = z0; z < z1; ++z)
        for (int64_t y = k->lo[1]; y < k->hi[1]; ++y) {
            const float* s = (const float*)k->src + k->L->origin + z * pz + y * py;
            float* d = (float*)k->dst + k->L->origin + z * pz + y * py;
            for (int64_t x = k->lo[2]; x < k->hi[2]; ++x) {
                float sx = s[x - 1] + s[x + 1];
                float sy = s[x - py] + s[x + py];
                float sz = s[x - pz] + s[x + pz];
                d[x] = ((sx + sy) + sz) * sixth;
            }
        }
}

void or_update_region_f64(const double* src, double* dst, const or_layout* L,
                          const int64_t lo[3], const int64_t hi[3]) {
    upd_ctx k = {src, dst, L, lo, hi};
    par_for(lo[0], hi[0], upd_range_f64, &k);
}

void or_update_region_f32(const float* src, float* dst, const or_layout* L,
                          const int64_t lo[3], const int64_t hi[3]) {
    upd_ctx k = {src, dst, L, lo, hi};
    par_for(lo[0], hi[0], upd_range_f32, &k);
}

/* `levels` naive sweeps (R/kernel.py:43-47 applied `levels` times, i.e.
 * verify.oracle R/verify.py:16-21) over the full interior, ping-ponging a/b.
 * Returns 0 if the result is in a, 1 if in b (the TwoGrid.active flag). */
int or_sweeps_f64(double* a, double* b, const or_layout* L, int64_t levels) {
    const int64_t lo[3] = {0, 0, 0}, hi[3] = {L->nz, L->ny, L->nx};
    int active = 0;
    for (int64_t i = 0; i < levels; ++i) {
        if (active == 0) or_update_region_f64(a, b, L, lo, hi);
        else or_update_region_f64(b, a, L, lo, hi);
        active ^= 1;
    }
    return active;
}

int or_sweeps_f32(float* a, float* b, const or_layout* L, int64_t levels) {
    const int64_t lo[3] = {0, 0, 0}, hi[3] = {L->nz, L->ny, L->nx};
    int active = 0;
    for (int64_t i = 0; i < levels; ++i) {
        if (active == 0) or_update_region_f32(a, b, L, lo, hi);
        else or_update_region_f32(b, a, L, lo, hi);
        active ^= 1;
    }
    return active;
}

/* ---- digest of an interior (shared definition with the device digest) ----
 * Order-independent 64-bit digest: sum over interior cells of
 * mix64(bits(v) + linear_index * H1), mod 2^64, linear_index = (z*ny+y)*nx+x.
 * The device reduction uses the same definition, so a full-size grid is
 * compared bit-for-bit through one 64-bit word.  Float32 cells hash their
 * 32-bit pattern zero-extended. */
typedef struct { const void* base; const or_layout* L; int f32; uint64_t part[256]; } dig_ctx;

static void dig_range(void* c, int64_t z0, int64_t z1, int chunk) {
    dig_ctx* k = (dig_ctx*)c;
    const or_layout* L = k->L;
    uint64_t acc = 0;
    for (int64_t z = z0; z < z1; ++z)
        for (int64_t y = 0; y < L->ny; ++y) {
            int64_t off = L->origin + z * L->pz + y * L->py;
            uint64_t idx = (uint64_t)((z * L->ny + y) * L->nx);
            for (int64_t x = 0; x < L->nx; ++x) {
                uint64_t bits;
                if (k->f32) { uint32_t b; memcpy(&b, (const float*)k->base + off + x, 4); bits = b; }
                else memcpy(&bits, (const double*)k->base + off + x, 8);
                acc += mix64(bits + (idx + (uint64_t)x) * H1);
            }
        }
    k->part[chunk] = acc;   /* one slot per chunk: no race */
}

static uint64_t digest_any(const void* base, const or_layout* L, int f32) {
    dig_ctx k;
    memset(&k, 0, sizeof k);
    k.base = base; k.L = L; k.f32 = f32;
    par_for(0, L->nz, dig_range, &k);
    uint64_t total = 0;
    for (int i = 0; i < 256; ++i) total += k.part[i];
    return total;
}

uint64_t or_digest_f64(const double* base, const or_layout* L) { return digest_any(base, L, 0); }
uint64_t or_digest_f32(const float* base, const or_layout* L) { return digest_any(base, L, 1); }
