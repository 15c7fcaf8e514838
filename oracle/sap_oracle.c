/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle for the SaP hot path.
 *
 * A plain-C99 restatement of the reference algorithm (arXiv 1509.07919's
 * SaP dense-banded path as implemented in /root/reference/proj). It is the
 * checker the parity tests compare the CUDA path against; it is never linked
 * into, loaded by, or called from the product library. Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it.
 *
 * Parity pinning: tests/test_oracle.py checks every function here against
 * golden vectors produced by the UNMODIFIED reference (oracle/_ref, built from
 * /root/reference by oracle/Makefile; fixtures in tests/golden/ made by
 * tests/golden/make_golden.py) and against the reference's own known-answer
 * tests (proj/tests/test_banded_core.cpp:257-277 etc.).
 *
 * Arithmetic follows the reference's Release build: IEEE double, separate
 * multiply and subtract (this file is compiled with -ffp-contract=off),
 * sequential summation in the reference's loop order.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------------- */
/* std::mt19937 + libstdc++ uniform_real_distribution<double>(-1, 1)       */
/* (the generator behind testsup::random_banded, proj/tests/test_support.hpp:133-150) */

typedef struct {
    uint32_t mt[624];
    int idx;
} sapo_mt19937;

static void mt_seed(sapo_mt19937* g, uint32_t seed) {
    g->mt[0] = seed;
    for (int i = 1; i < 624; ++i) g->mt[i] = 1812433253u * (g->mt[i - 1] ^ (g->mt[i - 1] >> 30)) + (uint32_t)i;
    g->idx = 624;
}

static uint32_t mt_next(sapo_mt19937* g) {
    if (g->idx >= 624) {
        for (int i = 0; i < 624; ++i) {
            uint32_t y = (g->mt[i] & 0x80000000u) | (g->mt[(i + 1) % 624] & 0x7fffffffu);
            uint32_t v = g->mt[(i + 397) % 624] ^ (y >> 1);
            if (y & 1u) v ^= 0x9908b0dfu;
            g->mt[i] = v;
        }
        g->idx = 0;
    }
    uint32_t y = g->mt[g->idx++];
    y ^= y >> 11;
    y ^= (y << 7) & 0x9d2c5680u;
    y ^= (y << 15) & 0xefc60000u;
    y ^= y >> 18;
    return y;
}

/* generate_canonical<double, 53>: two 32-bit draws, sum / 2^64, clamp below 1. */
static double mt_canonical(sapo_mt19937* g) {
    double sum = 0.0, tmp = 1.0;
    for (int k = 0; k < 2; ++k) {
        sum += (double)mt_next(g) * tmp;
        tmp *= 4294967296.0;
    }
    double r = sum / tmp;
    if (r >= 1.0) r = nextafter(1.0, 0.0);
    return r;
}

static double mt_uniform(sapo_mt19937* g, double a, double b) { return mt_canonical(g) * (b - a) + a; }

/* random_banded (proj/tests/test_support.hpp:133-150) then random_rhs
 * (proj/tests/acceptance.cpp:48-53) from the same generator. */
int sapo_random_banded(int n, int k, double d, uint32_t seed, double* band, double* rhs) {
    sapo_mt19937* g = (sapo_mt19937*)malloc(sizeof(sapo_mt19937));
    mt_seed(g, seed);
    const int w = 2 * k + 1;
    memset(band, 0, sizeof(double) * (size_t)n * (size_t)w);
    for (int i = 0; i < n; ++i) {
        double off = 0.0;
        const int lo = i - k > 0 ? i - k : 0;
        const int hi = i + k < n - 1 ? i + k : n - 1;
        for (int j = lo; j <= hi; ++j) {
            if (j == i) continue;
            double v = mt_uniform(g, -1.0, 1.0);
            if (v == 0.0) v = 0.5;
            band[(size_t)j * w + (size_t)(i - j + k)] = v;
            off += fabs(v);
        }
        band[(size_t)i * w + (size_t)k] = off > 0.0 ? d * off : d;
    }
    if (rhs)
        for (int i = 0; i < n; ++i) rhs[i] = mt_uniform(g, -1.0, 1.0);
    free(g);
    return 0;
}

/* Raw generator stream, for pinning the generator itself. */
void sapo_uniform_stream(uint32_t seed, int count, double* out) {
    sapo_mt19937 g;
    mt_seed(&g, seed);
    for (int i = 0; i < count; ++i) out[i] = mt_uniform(&g, -1.0, 1.0);
}

/* ---------------------------------------------------------------------- */
/* Partitioning (proj/include/sap/partition.hpp:34-69)                     */

int sapo_max_feasible_partitions(int n, int k) {
    if (n <= 0) return 0;
    return k == 0 ? n : n / (2 * k);
}

/* Returns 0 on success, 1 when the reference throws std::invalid_argument. */
int sapo_partition_layout(int n, int p, int k, int* sizes, int* offsets) {
    if (n <= 0 || p <= 0 || k < 0) return 1;
    const int base = n / p, rem = n % p;
    const int required = k == 0 ? 1 : 2 * k;
    if (base < required) return 1;
    offsets[0] = 0;
    for (int i = 0; i < p; ++i) {
        sizes[i] = base + (i < rem ? 1 : 0);
        offsets[i + 1] = offsets[i] + sizes[i];
    }
    return 0;
}

/* ---------------------------------------------------------------------- */
/* Band storage: slot(i, j) = j*(2k+1) + (i-j+k) (proj/include/sap/banded_matrix.hpp:49-51) */

#define SLOT(i, j, k) ((size_t)(j) * (size_t)(2 * (k) + 1) + (size_t)((i) - (j) + (k)))

/* BandedMatrix::matvec (proj/include/sap/banded_matrix.hpp:72-80) */
void sapo_band_matvec(int n, int k, const double* a, const double* x, double* y) {
    for (int i = 0; i < n; ++i) {
        double acc = 0.0;
        const int lo = i - k > 0 ? i - k : 0;
        const int hi = i + k < n - 1 ? i + k : n - 1;
        for (int j = lo; j <= hi; ++j) acc += a[SLOT(i, j, k)] * x[j];
        y[i] = acc;
    }
}

/* SparseMatrix::matvec (proj/include/sap/sparse_matrix.hpp:24-31) */
void sapo_csr_matvec(int n, const int* rp, const int* ci, const double* v, const double* x, double* y) {
    for (int i = 0; i < n; ++i) {
        double acc = 0.0;
        for (int s = rp[i]; s < rp[i + 1]; ++s) acc += v[s] * x[ci[s]];
        y[i] = acc;
    }
}

/* band_lu_inplace (proj/include/sap/block_factors.hpp:22-44) */
int sapo_band_lu_inplace(int m, int k, double* f, double boost_eps, double scale) {
    const double bv = boost_eps * (scale > 0 ? scale : 1.0);
    int boosts = 0;
    for (int j = 0; j < m; ++j) {
        double p = f[SLOT(j, j, k)];
        if (fabs(p) < bv) {
            p = p < 0.0 ? -bv : bv;
            f[SLOT(j, j, k)] = p;
            ++boosts;
        }
        const int hi = j + k < m - 1 ? j + k : m - 1;
        for (int i = j + 1; i <= hi; ++i) f[SLOT(i, j, k)] /= p;
        for (int c = j + 1; c <= hi; ++c) {
            const double ujc = f[SLOT(j, c, k)];
            if (ujc == 0.0) continue;
            for (int i = j + 1; i <= hi; ++i) f[SLOT(i, c, k)] -= f[SLOT(i, j, k)] * ujc;
        }
    }
    return boosts;
}

/* band_ul_inplace (proj/include/sap/block_factors.hpp:49-71) */
int sapo_band_ul_inplace(int m, int k, double* f, double boost_eps, double scale) {
    const double bv = boost_eps * (scale > 0 ? scale : 1.0);
    int boosts = 0;
    for (int j = m - 1; j >= 0; --j) {
        double p = f[SLOT(j, j, k)];
        if (fabs(p) < bv) {
            p = p < 0.0 ? -bv : bv;
            f[SLOT(j, j, k)] = p;
            ++boosts;
        }
        const int lo = j - k > 0 ? j - k : 0;
        for (int i = lo; i < j; ++i) f[SLOT(i, j, k)] /= p;
        for (int c = lo; c < j; ++c) {
            const double ajc = f[SLOT(j, c, k)];
            if (ajc == 0.0) continue;
            for (int i = lo; i < j; ++i) f[SLOT(i, c, k)] -= f[SLOT(i, j, k)] * ajc;
        }
    }
    return boosts;
}

/* band_lu_solve (proj/include/sap/block_factors.hpp:74-90) */
void sapo_band_lu_solve(int m, int k, const double* f, double* x) {
    for (int i = 0; i < m; ++i) {
        double acc = x[i];
        const int lo = i - k > 0 ? i - k : 0;
        for (int j = lo; j < i; ++j) acc -= f[SLOT(i, j, k)] * x[j];
        x[i] = acc;
    }
    for (int i = m - 1; i >= 0; --i) {
        double acc = x[i];
        const int hi = i + k < m - 1 ? i + k : m - 1;
        for (int j = i + 1; j <= hi; ++j) acc -= f[SLOT(i, j, k)] * x[j];
        x[i] = acc / f[SLOT(i, i, k)];
    }
}

/* band_ul_solve (proj/include/sap/block_factors.hpp:93-109) */
void sapo_band_ul_solve(int m, int k, const double* f, double* x) {
    for (int i = m - 1; i >= 0; --i) {
        double acc = x[i];
        const int hi = i + k < m - 1 ? i + k : m - 1;
        for (int j = i + 1; j <= hi; ++j) acc -= f[SLOT(i, j, k)] * x[j];
        x[i] = acc;
    }
    for (int i = 0; i < m; ++i) {
        double acc = x[i];
        const int lo = i - k > 0 ? i - k : 0;
        for (int j = lo; j < i; ++j) acc -= f[SLOT(i, j, k)] * x[j];
        x[i] = acc / f[SLOT(i, i, k)];
    }
}

/* factor_blocks without block permutations (proj/include/sap/block_factors.hpp:138-206):
 * per block, copy the in-block band, take its infinity norm as the boost
 * scale, UL on a copy (lu_and_ul only), then LU in place. Factors are written
 * back to back in partition order, block b at offsets[b]*(2k+1). */
int sapo_factor_blocks(int n, int k, const double* a, int p, int lu_and_ul, double boost_eps, double* lu,
                       double* ul, int* boosts, int* boosts_ul, double* norms) {
    int* sizes = (int*)malloc(sizeof(int) * (size_t)p);
    int* offs = (int*)malloc(sizeof(int) * (size_t)(p + 1));
    if (sapo_partition_layout(n, p, k, sizes, offs)) {
        free(sizes);
        free(offs);
        return 1;
    }
    const int w = 2 * k + 1;
    for (int b = 0; b < p; ++b) {
        const int off = offs[b], m = sizes[b];
        double* band = lu + (size_t)off * w;
        memset(band, 0, sizeof(double) * (size_t)m * w);
        for (int r = 0; r < m; ++r) {
            const int lo = r - k > 0 ? r - k : 0;
            const int hi = r + k < m - 1 ? r + k : m - 1;
            for (int c = lo; c <= hi; ++c) band[SLOT(r, c, k)] = a[SLOT(off + r, off + c, k)];
        }
        double norm = 0.0;
        for (int r = 0; r < m; ++r) {
            double row = 0.0;
            const int lo = r - k > 0 ? r - k : 0;
            const int hi = r + k < m - 1 ? r + k : m - 1;
            for (int c = lo; c <= hi; ++c) row += fabs(band[SLOT(r, c, k)]);
            if (row > norm) norm = row;
        }
        if (norms) norms[b] = norm;
        if (lu_and_ul && ul) {
            double* u = ul + (size_t)off * w;
            memcpy(u, band, sizeof(double) * (size_t)m * w);
            const int nb = sapo_band_ul_inplace(m, k, u, boost_eps, norm);
            if (boosts_ul) boosts_ul[b] = nb;
        }
        boosts[b] = sapo_band_lu_inplace(m, k, band, boost_eps, norm);
    }
    free(sizes);
    free(offs);
    return 0;
}

/* ---------------------------------------------------------------------- */
/* Dense helpers (proj/include/sap/spike.hpp:20-76)                        */

int sapo_dense_lu_nopivot_boosted(int w, double* a, double boost_eps) {
    double norm = 0.0;
    for (int i = 0; i < w; ++i) {
        double row = 0.0;
        for (int j = 0; j < w; ++j) row += fabs(a[(size_t)i * w + j]);
        if (row > norm) norm = row;
    }
    const double bv = boost_eps * (norm > 0 ? norm : 1.0);
    int boosts = 0;
    for (int j = 0; j < w; ++j) {
        double p = a[(size_t)j * w + j];
        if (fabs(p) < bv) {
            p = p < 0.0 ? -bv : bv;
            a[(size_t)j * w + j] = p;
            ++boosts;
        }
        for (int i = j + 1; i < w; ++i) {
            const double l = a[(size_t)i * w + j] / p;
            a[(size_t)i * w + j] = l;
            if (l == 0.0) continue;
            for (int c = j + 1; c < w; ++c) a[(size_t)i * w + c] -= l * a[(size_t)j * w + c];
        }
    }
    return boosts;
}

void sapo_dense_lu_solve(int w, const double* f, double* x) {
    for (int i = 0; i < w; ++i) {
        double acc = x[i];
        for (int j = 0; j < i; ++j) acc -= f[(size_t)i * w + j] * x[j];
        x[i] = acc;
    }
    for (int i = w - 1; i >= 0; --i) {
        double acc = x[i];
        for (int j = i + 1; j < w; ++j) acc -= f[(size_t)i * w + j] * x[j];
        x[i] = acc / f[(size_t)i * w + i];
    }
}

static void dense_gemv_sub(int w, const double* a, const double* x, double* y) {
    for (int i = 0; i < w; ++i) {
        double acc = 0.0;
        for (int j = 0; j < w; ++j) acc += a[(size_t)i * w + j] * x[j];
        y[i] -= acc;
    }
}

static int all_finite(const double* v, size_t n) {
    for (size_t i = 0; i < n; ++i)
        if (!isfinite(v[i])) return 0;
    return 1;
}

/* ---------------------------------------------------------------------- */
/* Coupling + spike tips + reduced blocks (proj/include/sap/spike.hpp:95-254) */

/* extract_coupling (proj/include/sap/spike.hpp:95-116), uniform K: w = k. */
void sapo_extract_coupling(int n, int k, const double* a, int p, const int* offs, double* bblk, double* cblk) {
    const int w = k;
    for (int t = 0; t + 1 < p; ++t) {
        const int e = offs[t + 1];
        double* bb = bblk + (size_t)t * w * w;
        double* cc = cblk + (size_t)t * w * w;
        for (int r = 0; r < w; ++r)
            for (int j = 0; j < w; ++j) {
                const int bi = e - w + r, bj = e + j, ci = e + r, cj = e - w + j;
                bb[(size_t)r * w + j] = (bi >= 0 && bi < n && bj >= 0 && bj < n && abs(bi - bj) <= k) ? a[SLOT(bi, bj, k)] : 0.0;
                cc[(size_t)r * w + j] = (ci >= 0 && ci < n && cj >= 0 && cj < n && abs(ci - cj) <= k) ? a[SLOT(ci, cj, k)] : 0.0;
            }
    }
}

/* compute_spike_tips + finish_reduced_blocks (proj/include/sap/spike.hpp:143-254).
 * Returns 0, or 2 where the reference throws PreconditionerError. */
int sapo_spike_tips(int k, int p, const int* sizes, const int* offs, const double* lu, const double* ul,
                    const double* bblk, const double* cblk, double boost_eps, double* vb, double* wt,
                    double* rbar, int* rbar_boosts) {
    const int w = k, bw = 2 * k + 1;
    double* col = (double*)malloc(sizeof(double) * (size_t)(w > 0 ? w : 1));
    for (int t = 0; t + 1 < p; ++t) {
        const int m = sizes[t];
        const double* band = lu + (size_t)offs[t] * bw;
        double* tip = vb + (size_t)t * w * w;
        for (int c = 0; c < w; ++c) {
            for (int r = 0; r < w; ++r) col[r] = bblk[(size_t)t * w * w + (size_t)r * w + c];
            for (int i = 0; i < w; ++i) {
                double acc = col[i];
                for (int j = 0; j < i; ++j) {
                    const int gi = m - w + i, gj = m - w + j;
                    const double l = (gi - gj > k || gj - gi > k) ? 0.0 : band[SLOT(gi, gj, k)];
                    acc -= l * col[j];
                }
                col[i] = acc;
            }
            for (int i = w - 1; i >= 0; --i) {
                double acc = col[i];
                for (int j = i + 1; j < w; ++j) {
                    const int gi = m - w + i, gj = m - w + j;
                    const double u = (gi - gj > k || gj - gi > k) ? 0.0 : band[SLOT(gi, gj, k)];
                    acc -= u * col[j];
                }
                col[i] = acc / band[SLOT(m - w + i, m - w + i, k)];
            }
            for (int r = 0; r < w; ++r) tip[(size_t)r * w + c] = col[r];
        }
        if (!all_finite(tip, (size_t)w * w)) {
            free(col);
            return 2;
        }
        const double* uband = ul + (size_t)offs[t + 1] * bw;
        double* tip2 = wt + (size_t)t * w * w;
        for (int c = 0; c < w; ++c) {
            for (int r = 0; r < w; ++r) col[r] = cblk[(size_t)t * w * w + (size_t)r * w + c];
            for (int i = w - 1; i >= 0; --i) {
                double acc = col[i];
                for (int j = i + 1; j < w; ++j) {
                    const double u = (i - j > k || j - i > k) ? 0.0 : uband[SLOT(i, j, k)];
                    acc -= u * col[j];
                }
                col[i] = acc;
            }
            for (int i = 0; i < w; ++i) {
                double acc = col[i];
                for (int j = 0; j < i; ++j) {
                    const double l = (i - j > k || j - i > k) ? 0.0 : uband[SLOT(i, j, k)];
                    acc -= l * col[j];
                }
                col[i] = acc / uband[SLOT(i, i, k)];
            }
            for (int r = 0; r < w; ++r) tip2[(size_t)r * w + c] = col[r];
        }
        if (!all_finite(tip2, (size_t)w * w)) {
            free(col);
            return 2;
        }
    }
    free(col);
    /* finish_reduced_blocks (proj/include/sap/spike.hpp:143-170) */
    for (int t = 0; t + 1 < p; ++t) {
        const double* wtt = wt + (size_t)t * w * w;
        const double* vbt = vb + (size_t)t * w * w;
        double* r = rbar + (size_t)t * w * w;
        for (int i = 0; i < w; ++i)
            for (int j = 0; j < w; ++j) {
                double acc = 0.0;
                for (int l = 0; l < w; ++l) acc += wtt[(size_t)i * w + l] * vbt[(size_t)l * w + j];
                r[(size_t)i * w + j] = (i == j ? 1.0 : 0.0) - acc;
            }
        if (!all_finite(r, (size_t)w * w)) return 2;
        rbar_boosts[t] = sapo_dense_lu_nopivot_boosted(w, r, boost_eps);
    }
    return 0;
}

/* ---------------------------------------------------------------------- */
/* Preconditioner state + apply (proj/include/sap/spike.hpp:304-351)       */

typedef struct {
    int n, k, p, kind; /* kind: 0 coupled, 1 decoupled, 2 diagonal, 3 none */
    int *sizes, *offs;
    double *lu, *ul, *bblk, *cblk, *vb, *wt, *rbar, *diag;
    int* rbar_boosts;
} sapo_precond;

static void precond_free(sapo_precond* s) {
    free(s->sizes); free(s->offs); free(s->lu); free(s->ul); free(s->bblk); free(s->cblk);
    free(s->vb); free(s->wt); free(s->rbar); free(s->diag); free(s->rbar_boosts);
}

/* build_precond_op<double> minus the closure (proj/include/sap/pipeline.hpp:140-202). */
static int precond_build(sapo_precond* s, int n, int k, const double* a, int p, int kind, double boost_eps) {
    memset(s, 0, sizeof(*s));
    s->n = n; s->k = k; s->p = p; s->kind = kind;
    if (kind == 3) return 0;
    const int w = 2 * k + 1;
    if (kind == 2) {
        double scale = 0.0;
        for (int i = 0; i < n; ++i) {
            double row = 0.0;
            const int lo = i - k > 0 ? i - k : 0;
            const int hi = i + k < n - 1 ? i + k : n - 1;
            for (int j = lo; j <= hi; ++j) row += fabs(a[SLOT(i, j, k)]);
            if (row > scale) scale = row;
        }
        const double bv = boost_eps * (scale > 0 ? scale : 1.0);
        s->diag = (double*)malloc(sizeof(double) * (size_t)n);
        for (int i = 0; i < n; ++i) {
            double d = a[SLOT(i, i, k)];
            if (fabs(d) < bv) d = d < 0.0 ? -bv : bv;
            s->diag[i] = d;
        }
        return 0;
    }
    s->sizes = (int*)malloc(sizeof(int) * (size_t)p);
    s->offs = (int*)malloc(sizeof(int) * (size_t)(p + 1));
    if (sapo_partition_layout(n, p, k, s->sizes, s->offs)) return 1;
    const int want_ul = kind == 0 && p > 1;
    s->lu = (double*)malloc(sizeof(double) * (size_t)n * w);
    if (want_ul) s->ul = (double*)malloc(sizeof(double) * (size_t)n * w);
    int* boosts = (int*)malloc(sizeof(int) * (size_t)p);
    sapo_factor_blocks(n, k, a, p, want_ul, boost_eps, s->lu, s->ul, boosts, NULL, NULL);
    free(boosts);
    if (want_ul) {
        const size_t ww = (size_t)k * k * (size_t)(p - 1);
        s->bblk = (double*)malloc(sizeof(double) * (ww ? ww : 1));
        s->cblk = (double*)malloc(sizeof(double) * (ww ? ww : 1));
        s->vb = (double*)malloc(sizeof(double) * (ww ? ww : 1));
        s->wt = (double*)malloc(sizeof(double) * (ww ? ww : 1));
        s->rbar = (double*)malloc(sizeof(double) * (ww ? ww : 1));
        s->rbar_boosts = (int*)malloc(sizeof(int) * (size_t)p);
        sapo_extract_coupling(n, k, a, p, s->offs, s->bblk, s->cblk);
        return sapo_spike_tips(k, p, s->sizes, s->offs, s->lu, s->ul, s->bblk, s->cblk, boost_eps, s->vb, s->wt,
                               s->rbar, s->rbar_boosts);
    }
    return 0;
}

static void precond_apply(const sapo_precond* s, const double* b, double* x) {
    const int n = s->n, k = s->k, p = s->p, bw = 2 * k + 1;
    memcpy(x, b, sizeof(double) * (size_t)n);
    if (s->kind == 3) return;
    if (s->kind == 2) {
        for (int i = 0; i < n; ++i) x[i] /= s->diag[i];
        return;
    }
    for (int i = 0; i < p; ++i) sapo_band_lu_solve(s->sizes[i], k, s->lu + (size_t)s->offs[i] * bw, x + s->offs[i]);
    if (s->kind == 1 || p == 1) return;
    const int w = k, ni = p - 1;
    double* xt = (double*)malloc(sizeof(double) * (size_t)(ni * w + 1));
    double* xb = (double*)malloc(sizeof(double) * (size_t)(ni * w + 1));
    for (int t = 0; t < ni; ++t) {
        const int e = s->offs[t + 1];
        double* gb = xb + (size_t)t * w;
        double* rhs = xt + (size_t)t * w;
        memcpy(gb, x + e - w, sizeof(double) * (size_t)w);
        memcpy(rhs, x + e, sizeof(double) * (size_t)w);
        dense_gemv_sub(w, s->wt + (size_t)t * w * w, gb, rhs);
        sapo_dense_lu_solve(w, s->rbar + (size_t)t * w * w, rhs);
        dense_gemv_sub(w, s->vb + (size_t)t * w * w, rhs, gb);
    }
    memcpy(x, b, sizeof(double) * (size_t)n);
    for (int t = 0; t < ni; ++t) {
        const int e = s->offs[t + 1];
        dense_gemv_sub(w, s->bblk + (size_t)t * w * w, xt + (size_t)t * w, x + e - w);
        dense_gemv_sub(w, s->cblk + (size_t)t * w * w, xb + (size_t)t * w, x + e);
    }
    for (int i = 0; i < p; ++i) sapo_band_lu_solve(s->sizes[i], k, s->lu + (size_t)s->offs[i] * bw, x + s->offs[i]);
    free(xt);
    free(xb);
}

/* One-shot apply for tests: builds the preconditioner and applies it once. */
int sapo_apply(int n, int k, const double* a, int p, int kind, double boost_eps, const double* in, double* out) {
    sapo_precond s;
    const int rc = precond_build(&s, n, k, a, p, kind, boost_eps);
    if (rc == 0) precond_apply(&s, in, out);
    precond_free(&s);
    return rc;
}

/* ---------------------------------------------------------------------- */
/* BiCGStab(l) (proj/include/sap/krylov.hpp:45-350)                         */

typedef void (*sapo_op)(const void* ctx, const double* in, double* out);

static double dot(int n, const double* a, const double* b) {
    double acc = 0.0;
    for (int i = 0; i < n; ++i) acc += a[i] * b[i];
    return acc;
}

static int vfinite(int n, const double* a) {
    for (int i = 0; i < n; ++i)
        if (!isfinite(a[i])) return 0;
    return 1;
}

static double true_residual(int n, sapo_op A, const void* actx, const double* b, const double* x, double* scratch) {
    A(actx, x, scratch);
    double acc = 0.0;
    for (int i = 0; i < n; ++i) {
        const double d = b[i] - scratch[i];
        acc += d * d;
    }
    return sqrt(acc);
}

/* tiny_solve with partial pivoting (proj/include/sap/krylov.hpp:76-99). */
static int tiny_solve(int n, double* a, double* rhs) {
    for (int j = 0; j < n; ++j) {
        int piv = j;
        for (int i = j + 1; i < n; ++i)
            if (fabs(a[i * n + j]) > fabs(a[piv * n + j])) piv = i;
        if (a[piv * n + j] == 0.0) return 0;
        if (piv != j) {
            for (int c = 0; c < n; ++c) {
                const double t = a[j * n + c];
                a[j * n + c] = a[piv * n + c];
                a[piv * n + c] = t;
            }
            const double t = rhs[j];
            rhs[j] = rhs[piv];
            rhs[piv] = t;
        }
        for (int i = j + 1; i < n; ++i) {
            const double l = a[i * n + j] / a[j * n + j];
            if (l == 0.0) continue;
            for (int c = j; c < n; ++c) a[i * n + c] -= l * a[j * n + c];
            rhs[i] -= l * rhs[j];
        }
    }
    for (int i = n - 1; i >= 0; --i) {
        double acc = rhs[i];
        for (int j = i + 1; j < n; ++j) acc -= a[i * n + j] * rhs[j];
        rhs[i] = acc / a[i * n + i];
    }
    return 1;
}

typedef struct {
    double iterations;
    int converged;
    double final_relative_residual;
    int failure; /* KrylovFailure order: none, max_iterations, breakdown, non_finite, indefinite */
    int hist_len;
} sapo_stats;

typedef struct {
    sapo_stats* st;
    double* hist;
    int cap;
    double bnorm;
    int ell;
} rec_ctx;

static void push_hist(rec_ctx* r, double v) {
    if (r->st->hist_len < r->cap) r->hist[r->st->hist_len] = v;
    r->st->hist_len++;
}

static void record(rec_ctx* r, int sweep, int step, double res) {
    const long steps = (long)sweep * 2 * r->ell + step;
    const long quarters = (4 * steps + 2 * r->ell - 1) / (2 * r->ell);
    r->st->iterations = (double)quarters / 4.0;
    push_hist(r, res / r->bnorm);
    r->st->final_relative_residual = res / r->bnorm;
}

/* solve_krylov (proj/include/sap/krylov.hpp:110-350). */
static int bicgstab_l(int n, sapo_op A, const void* actx, sapo_op M, const void* mctx, const double* b, double* x,
                      int ell, double rel_tol, double abs_tol, int max_iterations, sapo_stats* st, double* hist,
                      int cap) {
    memset(st, 0, sizeof(*st));
    if (ell < 1) return 1;
    for (int i = 0; i < n; ++i) x[i] = 0.0;
    const double bnorm = sqrt(dot(n, b, b));
    rec_ctx rc = {st, hist, cap, bnorm, ell};
    if (bnorm == 0.0) {
        st->converged = 1;
        push_hist(&rc, 0.0);
        return 0;
    }
    const double thr = rel_tol * bnorm + abs_tol;
    double tr = bnorm;
    push_hist(&rc, tr / bnorm);
    st->final_relative_residual = tr / bnorm;
    if (tr <= thr) {
        st->converged = 1;
        return 0;
    }
    const size_t N = (size_t)n;
    double* buf = (double*)calloc((size_t)(2 * (ell + 1) + 5) * N + 1, sizeof(double));
    double** r = (double**)malloc(sizeof(double*) * (size_t)(ell + 1));
    double** u = (double**)malloc(sizeof(double*) * (size_t)(ell + 1));
    for (int i = 0; i <= ell; ++i) {
        r[i] = buf + (size_t)i * N;
        u[i] = buf + (size_t)(ell + 1 + i) * N;
    }
    double* tmp = buf + (size_t)(2 * (ell + 1)) * N;
    double* rtilde = tmp + N;
    double* scratch = rtilde + N;
    double* xc = scratch + N;
    double* gram = (double*)malloc(sizeof(double) * (size_t)(ell * ell + 1));
    double* rhs = (double*)malloc(sizeof(double) * (size_t)(ell + 1));
    double* gamma = (double*)calloc((size_t)ell + 1, sizeof(double));
    double* gamma_p = (double*)calloc((size_t)ell + 1, sizeof(double));
    double* gamma_pp = (double*)calloc((size_t)ell + 1, sizeof(double));
    double* sigma = (double*)calloc((size_t)ell + 1, sizeof(double));
    double* tau = (double*)calloc((size_t)(ell + 1) * (ell + 1), sizeof(double));

#define RESET_STATE(perturb)                                                          \
    do {                                                                              \
        A(actx, x, tmp);                                                              \
        for (int i_ = 0; i_ < n; ++i_) tmp[i_] = b[i_] - tmp[i_];                     \
        M(mctx, tmp, r[0]);                                                           \
        memcpy(rtilde, r[0], sizeof(double) * N);                                     \
        if (perturb) {                                                                \
            sapo_mt19937* g_ = (sapo_mt19937*)malloc(sizeof(sapo_mt19937));           \
            mt_seed(g_, 0x9d2c5680u);                                                 \
            const double scale_ = 1e-8 * sqrt(dot(n, r[0], r[0]));                    \
            for (int i_ = 0; i_ < n; ++i_) rtilde[i_] += scale_ * mt_uniform(g_, -1.0, 1.0); \
            free(g_);                                                                 \
        }                                                                             \
        memset(u[0], 0, sizeof(double) * N);                                          \
    } while (0)

    RESET_STATE(0);
    double rho0 = 1.0, alpha = 0.0, omega = 1.0;
    int restarted = 0, breakdown = 0, done = 0;
    for (int sweep = 0; sweep < max_iterations && !done; ++sweep) {
        breakdown = 0;
        rho0 = -omega * rho0;
        for (int j = 0; j < ell && !breakdown && !done; ++j) {
            const double rho1 = dot(n, r[j], rtilde);
            if (!isfinite(rho1)) { st->failure = 3; done = 1; break; }
            if (rho0 == 0.0 || rho1 == 0.0) { breakdown = 1; break; }
            const double beta = alpha * rho1 / rho0;
            rho0 = rho1;
            for (int i = 0; i <= j; ++i)
                for (int t = 0; t < n; ++t) u[i][t] = r[i][t] - beta * u[i][t];
            A(actx, u[j], tmp);
            M(mctx, tmp, u[j + 1]);
            const double g = dot(n, u[j + 1], rtilde);
            if (!isfinite(g)) { st->failure = 3; done = 1; break; }
            if (g == 0.0) { breakdown = 1; break; }
            alpha = rho0 / g;
            for (int i = 0; i <= j; ++i)
                for (int t = 0; t < n; ++t) r[i][t] -= alpha * u[i + 1][t];
            A(actx, r[j], tmp);
            M(mctx, tmp, r[j + 1]);
            for (int t = 0; t < n; ++t) x[t] += alpha * u[0][t];
            if (!vfinite(n, x)) { st->failure = 3; done = 1; break; }
            tr = true_residual(n, A, actx, b, x, scratch);
            if (!isfinite(tr)) { st->failure = 3; done = 1; break; }
            record(&rc, sweep, j + 1, tr);
            if (tr <= thr) { st->converged = 1; done = 1; break; }
        }
        if (done) break;
        if (!breakdown) {
            for (int d = 1; d < ell && !done; ++d) {
                for (int a_ = 1; a_ <= d; ++a_) {
                    for (int c = 1; c <= d; ++c) gram[(a_ - 1) * d + (c - 1)] = dot(n, r[a_], r[c]);
                    rhs[a_ - 1] = dot(n, r[a_], r[0]);
                }
                if (!tiny_solve(d, gram, rhs)) continue;
                int ok = 1;
                for (int c = 0; c < d; ++c) ok = ok && isfinite(rhs[c]);
                if (!ok) continue;
                memcpy(xc, x, sizeof(double) * N);
                for (int i = 1; i <= d; ++i)
                    for (int t = 0; t < n; ++t) xc[t] += rhs[i - 1] * r[i - 1][t];
                tr = true_residual(n, A, actx, b, xc, scratch);
                if (!isfinite(tr)) continue;
                record(&rc, sweep, ell + d, tr);
                if (tr <= thr) {
                    memcpy(x, xc, sizeof(double) * N);
                    st->converged = 1;
                    done = 1;
                }
            }
            if (done) break;
            for (int j = 1; j <= ell && !breakdown && !done; ++j) {
                for (int i = 1; i < j; ++i) {
                    const double tij = dot(n, r[j], r[i]) / sigma[i];
                    tau[i * (ell + 1) + j] = tij;
                    for (int t = 0; t < n; ++t) r[j][t] -= tij * r[i][t];
                }
                sigma[j] = dot(n, r[j], r[j]);
                if (!isfinite(sigma[j])) { st->failure = 3; done = 1; break; }
                if (sigma[j] == 0.0) { breakdown = 1; break; }
                gamma_p[j] = dot(n, r[0], r[j]) / sigma[j];
            }
            if (done) break;
        }
        if (!breakdown) {
            gamma[ell] = gamma_p[ell];
            omega = gamma[ell];
            for (int j = ell - 1; j >= 1; --j) {
                double acc = gamma_p[j];
                for (int i = j + 1; i <= ell; ++i) acc -= tau[j * (ell + 1) + i] * gamma[i];
                gamma[j] = acc;
            }
            for (int j = 1; j < ell; ++j) {
                double acc = gamma[j + 1];
                for (int i = j + 1; i < ell; ++i) acc += tau[j * (ell + 1) + i] * gamma[i + 1];
                gamma_pp[j] = acc;
            }
            for (int t = 0; t < n; ++t) {
                x[t] += gamma[1] * r[0][t];
                r[0][t] -= gamma_p[ell] * r[ell][t];
                u[0][t] -= gamma[ell] * u[ell][t];
            }
            for (int j = 1; j < ell; ++j)
                for (int t = 0; t < n; ++t) {
                    u[0][t] -= gamma[j] * u[j][t];
                    x[t] += gamma_pp[j] * r[j][t];
                    r[0][t] -= gamma_p[j] * r[j][t];
                }
            if (!vfinite(n, x)) { st->failure = 3; break; }
            tr = true_residual(n, A, actx, b, x, scratch);
            if (!isfinite(tr)) { st->failure = 3; break; }
            record(&rc, sweep, 2 * ell, tr);
            if (tr <= thr) { st->converged = 1; break; }
        }
        if (breakdown) {
            if (restarted) { st->failure = 2; break; }
            restarted = 1;
            RESET_STATE(1);
            rho0 = 1.0;
            alpha = 0.0;
            omega = 1.0;
        }
        if (sweep == max_iterations - 1) {
            st->iterations = (double)max_iterations;
            st->failure = 1;
        }
    }
#undef RESET_STATE
    if (!st->converged && st->failure == 0 && max_iterations <= 0) {
        st->iterations = (double)max_iterations;
        st->failure = 1;
    }
    free(buf); free(r); free(u); free(gram); free(rhs); free(gamma); free(gamma_p); free(gamma_pp);
    free(sigma); free(tau);
    return 0;
}

typedef struct { int n, k; const double* a; } band_ctx;
static void band_op(const void* c, const double* in, double* out) {
    const band_ctx* b = (const band_ctx*)c;
    sapo_band_matvec(b->n, b->k, b->a, in, out);
}
typedef struct { int n; const int* rp; const int* ci; const double* v; } csr_ctx;
static void csr_op(const void* c, const double* in, double* out) {
    const csr_ctx* s = (const csr_ctx*)c;
    sapo_csr_matvec(s->n, s->rp, s->ci, s->v, in, out);
}
static void pre_op(const void* c, const double* in, double* out) { precond_apply((const sapo_precond*)c, in, out); }
static void ident_op(const void* c, const double* in, double* out) {
    memcpy(out, in, sizeof(double) * (size_t)((const csr_ctx*)c)->n);
}

/* The dense wiring of proj/tests/acceptance.cpp:114-132 (setup =
 * build_precond_op, solve = run_krylov with the banded operator).
 * Returns 0, 1 (invalid argument) or 2 (preconditioner error). */
int sapo_solve_banded(int n, int k, const double* a, const double* rhs, int p, int kind, double boost_eps, int ell,
                      double rel_tol, double abs_tol, int max_iterations, double* x, sapo_stats* st, double* hist,
                      int cap) {
    sapo_precond s;
    int rc = precond_build(&s, n, k, a, p, kind, boost_eps);
    if (rc == 0) {
        band_ctx bc = {n, k, a};
        rc = bicgstab_l(n, band_op, &bc, pre_op, &s, rhs, x, ell, rel_tol, abs_tol, max_iterations, st, hist, cap);
    }
    precond_free(&s);
    return rc;
}

/* solve_krylov on a CSR operator with the identity preconditioner. */
int sapo_krylov_csr_identity(int n, const int* rp, const int* ci, const double* v, const double* rhs, int ell,
                             double rel_tol, int max_iterations, double* x, sapo_stats* st, double* hist, int cap) {
    csr_ctx c = {n, rp, ci, v};
    return bicgstab_l(n, csr_op, &c, ident_op, &c, rhs, x, ell, rel_tol, 0.0, max_iterations, st, hist, cap);
}
