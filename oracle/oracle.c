/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle for the FP64 hot path.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library, and only as the checker. The product never links it.
 *
 * A plain-C restatement of the reference's execution path
 * (/root/reference/proj/include/tilemul/exec.hpp, plan.hpp) and of the
 * seeded input generator of its `run` command
 * (/root/reference/proj/tools/tilemul_main.cpp:236-242). Parity is pinned:
 * tests/test_oracle.py checks every function here against
 * oracle/_ref/libtilemul_ref.so (the reference headers compiled unmodified)
 * and against the committed golden vectors in tests/golden/.
 *
 * Compiled with -O2 -ffp-contract=off so a*b+c stays a rounded multiply
 * followed by a rounded add, exactly as the reference's -O2 x86-64 build.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---- mt19937_64 (the published Matsumoto–Nishimura 64-bit recurrence) ---- */
typedef struct {
    uint64_t s[312];
    int i;
} or_mt64;

void or_mt64_seed(or_mt64* g, uint64_t seed) {
    g->s[0] = seed;
    for (int i = 1; i < 312; ++i)
        g->s[i] = 6364136223846793005ULL * (g->s[i - 1] ^ (g->s[i - 1] >> 62)) + (uint64_t)i;
    g->i = 312;
}

static void or_mt64_twist(or_mt64* g) {
    const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL, A = 0xB5026F5AA96619E9ULL;
    for (int i = 0; i < 312; ++i) {
        uint64_t x = (g->s[i] & UM) | (g->s[(i + 1) % 312] & LM);
        uint64_t xa = x >> 1;
        if (x & 1ULL) xa ^= A;
        g->s[i] = g->s[(i + 156) % 312] ^ xa;
    }
    g->i = 0;
}

uint64_t or_mt64_next(or_mt64* g) {
    if (g->i >= 312) or_mt64_twist(g);
    uint64_t y = g->s[g->i++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}

/* uniform_real_distribution<double>(-1, 1) over a 64-bit engine, as
 * libstdc++ computes it: u = double(x) / 2^64 (generate_canonical with one
 * draw), clamped below 1, then v = (b - a) * u + a = 2u - 1. */
double or_uniform_pm1(uint64_t x) {
    double u = (double)x / 18446744073709551616.0;
    if (u >= 1.0) u = nextafter(1.0, 0.0);
    return 2.0 * u + -1.0;
}

void or_fill_uniform(uint64_t seed, double* a, int64_t na, double* b, int64_t nb, double* c, int64_t nc) {
    or_mt64* g = (or_mt64*)malloc(sizeof(or_mt64));
    or_mt64_seed(g, seed);
    for (int64_t i = 0; i < na; ++i) a[i] = or_uniform_pm1(or_mt64_next(g));
    for (int64_t i = 0; i < nb; ++i) b[i] = or_uniform_pm1(or_mt64_next(g));
    if (c)
        for (int64_t i = 0; i < nc; ++i) c[i] = or_uniform_pm1(or_mt64_next(g));
    free(g);
}

/* ---- reference_gemm: naive i-j-p, local sum from 0, then added to C
 * (exec.hpp:15-30). Column-major. */
void or_reference_gemm(int64_t m, int64_t n, int64_t k, const double* a, const double* b, double* c) {
    for (int64_t i = 0; i < m; ++i)
        for (int64_t j = 0; j < n; ++j) {
            double acc = 0.0;
            for (int64_t p = 0; p < k; ++p) acc += a[i + p * m] * b[p + j * k];
            c[i + j * m] += acc;
        }
}

/* ---- micro_kernel (exec.hpp:35-46): acc <- c; p, j, i: acc += a*b; c <- acc.
 * fused=1 is the oracle of the GPU DFMA kernel: acc = fma(a, b, acc), one
 * rounding per step, same ascending-p order. */
static void or_micro_kernel(const double* a, int64_t lda, const double* b, int64_t ldb, double* c, int64_t ldc,
                            int64_t mr, int64_t nr, int64_t kc, double* acc, int fused) {
    for (int64_t j = 0; j < nr; ++j)
        for (int64_t i = 0; i < mr; ++i) acc[i + j * mr] = c[i + j * ldc];
    for (int64_t p = 0; p < kc; ++p)
        for (int64_t j = 0; j < nr; ++j) {
            const double bpj = b[p + j * ldb];
            if (fused)
                for (int64_t i = 0; i < mr; ++i) acc[i + j * mr] = fma(a[i + p * lda], bpj, acc[i + j * mr]);
            else
                for (int64_t i = 0; i < mr; ++i) acc[i + j * mr] += a[i + p * lda] * bpj;
        }
    for (int64_t j = 0; j < nr; ++j)
        for (int64_t i = 0; i < mr; ++i) c[i + j * ldc] = acc[i + j * mr];
}

/* ---- LoopNest::walk (plan.hpp:61-84) over column-major buffers. loops[]
 * holds (dim 0=m 1=n 2=k, blocksize) outermost first; each leaf cell runs the
 * micro-kernel on its (i0,m,j0,n,p0,k) region. */
typedef struct {
    int64_t m, n, k;
    const double *a, *b;
    double* c;
    double* acc;
    const int* dims;
    const int64_t* bsz;
    int nloops;
    int fused;
    int64_t cells;
} or_walk_ctx;

static void or_walk(or_walk_ctx* w, int depth, int64_t o0, int64_t o1, int64_t o2, int64_t e0, int64_t e1,
                    int64_t e2) {
    if (depth == w->nloops) {
        w->cells++;
        or_micro_kernel(w->a + o0 + o2 * w->m, w->m, w->b + o2 + o1 * w->k, w->k, w->c + o0 + o1 * w->m, w->m, e0,
                        e1, e2, w->acc, w->fused);
        return;
    }
    int d = w->dims[depth];
    int64_t bs = w->bsz[depth];
    int64_t start = d == 0 ? o0 : d == 1 ? o1 : o2;
    int64_t ext = d == 0 ? e0 : d == 1 ? e1 : e2;
    int64_t chunks = (ext + bs - 1) / bs;
    for (int64_t ch = 0; ch < chunks; ++ch) {
        int64_t s = start + ch * bs;
        int64_t e = bs < start + ext - s ? bs : start + ext - s;
        if (d == 0) or_walk(w, depth + 1, s, o1, o2, e, e1, e2);
        else if (d == 1) or_walk(w, depth + 1, o0, s, o2, e0, e, e2);
        else or_walk(w, depth + 1, o0, o1, s, e0, e1, e);
    }
}

/* execute() restated (exec.hpp:94-138, single worker — worker count never
 * changes results, test_exec.cpp:223-254). Returns the cell count. */
int64_t or_execute(int64_t m, int64_t n, int64_t k, const int* dims, const int64_t* bsz, int nloops, int64_t mr,
                   int64_t nr, const double* a, const double* b, double* c, int fused) {
    or_walk_ctx w;
    w.m = m; w.n = n; w.k = k; w.a = a; w.b = b; w.c = c;
    w.acc = (double*)malloc(sizeof(double) * (size_t)(mr * nr > 0 ? mr * nr : 1));
    w.dims = dims; w.bsz = bsz; w.nloops = nloops; w.fused = fused; w.cells = 0;
    or_walk(&w, 0, 0, 0, 0, m, n, k);
    free(w.acc);
    return w.cells;
}

/* Sequential-k product for a sample of entries: c0 + sum_p a*b in ascending
 * p, one rounding per multiply and per add (fused=0) or one per fma
 * (fused=1). This is exactly what execute() leaves in C[i,j] for any nest,
 * since every nest visits the k chunks of one C entry in ascending order
 * and a store/load of a double between cells is exact. */
void or_entries(int64_t m, int64_t n, int64_t k, const double* a, int64_t lda, const double* b, int64_t ldb,
                const double* c0, int64_t ldc, const int64_t* ii, const int64_t* jj, int64_t count, int fused,
                double* out, double* absbound) {
    for (int64_t t = 0; t < count; ++t) {
        int64_t i = ii[t], j = jj[t];
        double acc = c0 ? c0[i + j * ldc] : 0.0;
        double ab = 0.0;
        for (int64_t p = 0; p < k; ++p) {
            double x = a[i + p * lda], y = b[p + j * ldb];
            if (fused) acc = fma(x, y, acc);
            else acc += x * y;
            ab += fabs(x) * fabs(y);
        }
        out[t] = acc;
        if (absbound) absbound[t] = ab;
    }
    (void)m; (void)n;
}

/* (|A||B|)_ij for every entry: the scale of the entrywise error bound
 * 4*k*u*(|A||B|)_ij (BASELINE.json north_star). */
void or_abs_product(int64_t m, int64_t n, int64_t k, const double* a, const double* b, double* out) {
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i < m; ++i) out[i + j * m] = 0.0;
    for (int64_t j = 0; j < n; ++j)
        for (int64_t p = 0; p < k; ++p) {
            double bv = fabs(b[p + j * k]);
            for (int64_t i = 0; i < m; ++i) out[i + j * m] += fabs(a[i + p * m]) * bv;
        }
}
