/*
 * efta_oracle.c — TEST INFRASTRUCTURE ONLY (the parity checker, never the product).
 *
 * Plain-C restatement of the reference's hot path (arXiv 2504.02211 artifact,
 * /root/reference/proj). Every function cites the reference file:line it
 * follows. Floating-point operations are issued in the reference's order and
 * precision (fp32 accumulation, fp64 comparisons, libm expf/log) and the
 * library is built with -ffp-contract=off like the reference
 * (proj/CMakeLists.txt:12-14), so results are bit-identical to the reference
 * on the same inputs. That claim is pinned by tests/test_oracle.py against
 * (a) the reference's own known-answer tests (restated there) and
 * (b) outputs of the unmodified reference compiled into oracle/_ref.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may load it.
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "oracle_abi.h"

static _Thread_local char g_err[256];
static void set_err(const char* s) { snprintf(g_err, sizeof g_err, "%s", s); }
const char* eorc_last_error(void) { return g_err; }

/* ------------------------------------------------------------------ RNG --- */
/* std::mt19937_64 as specified by the C++ standard; wrapped exactly like
 * include/efta/rng.hpp:19-52 (uniform, below) and :55-58 (trial_seed). */
typedef struct {
    uint64_t mt[312];
    int idx;
} rng_t;

static void rng_init(rng_t* r, uint64_t seed) {
    r->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        r->mt[i] = 6364136223846793005ull * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    r->idx = 312;
}

static uint64_t rng_next(rng_t* r) {
    if (r->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            uint64_t x = (r->mt[i] & 0xFFFFFFFF80000000ull) | (r->mt[(i + 1) % 312] & 0x7FFFFFFFull);
            uint64_t xa = x >> 1;
            if (x & 1) xa ^= 0xB5026F5AA96619E9ull;
            r->mt[i] = r->mt[(i + 156) % 312] ^ xa;
        }
        r->idx = 0;
    }
    uint64_t x = r->mt[r->idx++];
    x ^= (x >> 29) & 0x5555555555555555ull;
    x ^= (x << 17) & 0x71D67FFFEDA60000ull;
    x ^= (x << 37) & 0xFFF7EEE000000000ull;
    x ^= x >> 43;
    return x;
}

/* rng.hpp:26-28 */
static double rng_uniform(rng_t* r) { return (double)(rng_next(r) >> 11) * 0x1.0p-53; }
static double rng_uniform2(rng_t* r, double lo, double hi) { return lo + (hi - lo) * rng_uniform(r); }

/* rng.hpp:31-38 */
static uint32_t rng_below(rng_t* r, uint32_t n) {
    const uint64_t span = 0x100000000ull;
    const uint64_t limit = span - span % n;
    for (;;) {
        const uint64_t x = rng_next(r) >> 32;
        if (x < limit) return (uint32_t)(x % n);
    }
}

void eorc_rng_below_seq(uint64_t seed, int n, const uint32_t* bounds, uint32_t* out) {
    rng_t r;
    rng_init(&r, seed);
    for (int i = 0; i < n; ++i) out[i] = rng_below(&r, bounds[i]);
}

/* rng.hpp:8-13 */
static uint64_t splitmix64(uint64_t* state) {
    uint64_t z = (*state += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

/* rng.hpp:55-58 */
uint64_t eorc_trial_seed(uint64_t base, uint64_t trial) {
    uint64_t s = base ^ (0xd1b54a32d192ed03ull * (trial + 1));
    return splitmix64(&s);
}

/* ----------------------------------------------------------------- half --- */
static inline uint32_t f2u(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }
static inline float u2f(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }

/* include/efta/half.hpp:15-39 */
float eorc_half_bits_to_float(uint16_t h) {
    const uint32_t sign = (uint32_t)(h >> 15) << 31;
    uint32_t exp = (h >> 10) & 0x1f, mant = h & 0x3ff, bits;
    if (exp == 0) {
        if (mant == 0) {
            bits = sign;
        } else {
            int shift = 0;
            while ((mant & 0x400) == 0) { mant <<= 1; ++shift; }
            mant &= 0x3ff;
            bits = sign | ((uint32_t)(127 - 15 + 1 - shift) << 23) | (mant << 13);
        }
    } else if (exp == 0x1f) {
        bits = sign | 0x7f800000u | (mant << 13);
    } else {
        bits = sign | ((exp - 15 + 127) << 23) | (mant << 13);
    }
    return u2f(bits);
}

/* include/efta/half.hpp:43-78 (round to nearest even, saturate to inf) */
uint16_t eorc_float_to_half_bits(float f) {
    const uint32_t bits = f2u(f);
    const uint16_t sign = (uint16_t)((bits >> 16) & 0x8000);
    const int32_t exp = (int32_t)((bits >> 23) & 0xff);
    const uint32_t mant = bits & 0x7fffff;
    if (exp == 0xff) return (uint16_t)(sign | 0x7c00 | (mant ? 0x200 | (mant >> 13) : 0));
    int32_t e = exp - 127 + 15;
    if (e >= 0x1f) return (uint16_t)(sign | 0x7c00);
    if (e <= 0) {
        if (e < -10) return sign;
        uint32_t m = mant | 0x800000;
        const int shift = 14 - e;
        uint32_t hm = m >> shift;
        const uint32_t rem = m & ((1u << shift) - 1);
        const uint32_t halfway = 1u << (shift - 1);
        if (rem > halfway || (rem == halfway && (hm & 1))) ++hm;
        return (uint16_t)(sign | hm);
    }
    uint32_t hm = mant >> 13;
    const uint32_t rem = mant & 0x1fff;
    if (rem > 0x1000 || (rem == 0x1000 && (hm & 1))) {
        ++hm;
        if (hm == 0x400) {
            hm = 0;
            ++e;
            if (e >= 0x1f) return (uint16_t)(sign | 0x7c00);
        }
    }
    return (uint16_t)(sign | ((uint32_t)e << 10) | hm);
}

static float quantize_half(float f) { return eorc_half_bits_to_float(eorc_float_to_half_bits(f)); }

/* src/fault.cpp:27-37 */
float eorc_flip_bit(float v, int width, int bit) {
    if (width == 32) return u2f(f2u(v) ^ (1u << bit));
    return eorc_half_bits_to_float((uint16_t)(eorc_float_to_half_bits(v) ^ (1u << bit)));
}

/* src/matrix.cpp:20-25 */
static void random_fill(rng_t* r, int rows, int cols, double lo, double hi, int half, float* out) {
    for (int i = 0; i < rows * cols; ++i) {
        const float v = (float)rng_uniform2(r, lo, hi);
        out[i] = half ? quantize_half(v) : v;
    }
}

void eorc_random_matrix(uint64_t seed, int rows, int cols, double lo, double hi, int half_grid,
                        float* out) {
    rng_t r;
    rng_init(&r, seed);
    random_fill(&r, rows, cols, lo, hi, half_grid, out);
}

/* ------------------------------------------------------------ counters --- */
typedef struct {
    uint64_t main_scores, cs_scores, main_output, cs_output, exp_checks, output_checks;
} counters_t;

/* ------------------------------------------------------------ fault inj --- */
/* include/efta/fault.hpp:77-103: per-spec evaluation counters; fire on the
 * trigger-th evaluation; record before/after. */
typedef struct {
    const orc_fault_spec* specs;
    int n_specs;
    int* evals;
    orc_fired* fired;
    int fired_cap, n_fired;
} injector_t;

static float tap(injector_t* inj, int site, int bi, int bj, int r, int c, float v) {
    if (!inj) return v;
    for (int k = 0; k < inj->n_specs; ++k) {
        const orc_fault_spec* f = &inj->specs[k];
        if (f->site != site || f->block_i != bi || f->block_j != bj || f->row != r || f->col != c)
            continue;
        if (++inj->evals[k] == f->trigger) {
            const float flipped = eorc_flip_bit(v, 32, f->bit);
            if (inj->n_fired < inj->fired_cap) {
                inj->fired[inj->n_fired].spec = *f;
                inj->fired[inj->n_fired].before = v;
                inj->fired[inj->n_fired].after = flipped;
            }
            ++inj->n_fired;
            return flipped;
        }
    }
    return v;
}

/* ---------------------------------------------------------------- ABFT --- */
/* src/abft.cpp:19-42 (encode_strided) and :44-63 (strided_sums): identical
 * summation order (l ascending, fp32). */
static void strided_sums(const float* t, int rows, int cols, int stride, float* s1, float* s2) {
    const int groups = cols / stride;
    for (int r = 0; r < rows; ++r)
        for (int j = 0; j < stride; ++j) {
            float a = 0.0f, b = 0.0f;
            for (int l = 0; l < groups; ++l) {
                const float v = t[(size_t)r * cols + j + stride * l];
                a += v;
                b += (float)(l + 1) * v;
            }
            s1[r * stride + j] = a;
            s2[r * stride + j] = b;
        }
}

int eorc_encode_strided(int rows, int cols, int stride, const float* t, float* c1, float* c2) {
    if (stride <= 0 || cols % stride != 0) {
        set_err("encode_strided: stride must divide tile width");
        return 1;
    }
    strided_sums(t, rows, cols, stride, c1, c2);
    return 0;
}

static int all_finite(const float* p, size_t n) {
    for (size_t i = 0; i < n; ++i)
        if (!isfinite(p[i])) return 0;
    return 1;
}

/* src/abft.cpp:65-187 */
static void verify_locate_correct(float* t, int rows, int cols, int stride, const float* c1,
                                  const float* c2, double eps_abs, const double* row_eps_mult,
                                  orc_verify_report* rep) {
    memset(rep, 0, sizeof(*rep));
    rep->row = -1;
    rep->col = -1;
    const int groups = cols / stride;
    if (!all_finite(c1, (size_t)rows * stride) || !all_finite(c2, (size_t)rows * stride)) {
        rep->status = ORC_NONFINITE;
        rep->residual = INFINITY;
        return;
    }
    /* :83-111 erasure restore of non-finite data cells */
    if (!all_finite(t, (size_t)rows * cols)) {
        for (int r = 0; r < rows; ++r)
            for (int j = 0; j < stride; ++j) {
                int bad = -1, bad_count = 0;
                for (int l = 0; l < groups; ++l)
                    if (!isfinite(t[(size_t)r * cols + j + stride * l])) { bad = l; ++bad_count; }
                if (bad_count == 0) continue;
                ++rep->violations;
                if (bad_count > 1) {
                    rep->status = ORC_NONFINITE;
                    rep->residual = INFINITY;
                    return;
                }
                float rest = 0.0f;
                for (int l = 0; l < groups; ++l)
                    if (l != bad) rest += t[(size_t)r * cols + j + stride * l];
                const int col = j + stride * bad;
                t[(size_t)r * cols + col] = c1[r * stride + j] - rest;
                ++rep->corrections;
                rep->row = r;
                rep->col = col;
                rep->delta = INFINITY;
            }
    }
    float* s1 = (float*)malloc(sizeof(float) * rows * stride);
    float* s2 = (float*)malloc(sizeof(float) * rows * stride);
    strided_sums(t, rows, cols, stride, s1, s2);
    int any_uncorrectable = 0;
    for (int r = 0; r < rows; ++r) {
        const double eps_row = row_eps_mult ? eps_abs * row_eps_mult[r] : eps_abs;
        for (int j = 0; j < stride; ++j) {
            double s1d = s1[r * stride + j], s2d = s2[r * stride + j];
            if (!isfinite(s1d) || !isfinite(s2d)) { /* :124-131 redo group in double */
                s1d = 0.0;
                s2d = 0.0;
                for (int l = 0; l < groups; ++l) {
                    const double vv = t[(size_t)r * cols + j + stride * l];
                    s1d += vv;
                    s2d += (l + 1.0) * vv;
                }
            }
            const double d1 = (double)c1[r * stride + j] - s1d;
            const double d2 = (double)c2[r * stride + j] - s2d;
            const double res = fmax(fabs(d1), fabs(d2) / groups);
            if (res > rep->residual) rep->residual = res;
            const int v1 = fabs(d1) > eps_row;
            const int v2 = fabs(d2) > eps_row * groups;
            if (!v1 && !v2) continue;
            ++rep->violations;
            if (!v1) { rep->checksum_repair = 1; continue; }
            const double ratio = d2 / d1;
            const double nearest = round(ratio);
            if (nearest == 0.0 && fabs(ratio) <= 0.25) { rep->checksum_repair = 1; continue; }
            const int g = (int)nearest - 1;
            if (g < 0 || g >= groups || fabs(ratio - nearest) > 0.25) {
                if (fmax(fabs(d1), fabs(d2) / groups) > eps_row * 16.0 /* kLocateNoiseBand */)
                    any_uncorrectable = 1;
                continue;
            }
            const int col = j + stride * g;
            float rest = 0.0f;
            for (int l = 0; l < groups; ++l)
                if (l != g) rest += t[(size_t)r * cols + j + stride * l];
            const float old_val = t[(size_t)r * cols + col];
            const float new_val = c1[r * stride + j] - rest;
            t[(size_t)r * cols + col] = new_val;
            ++rep->corrections;
            const double applied = (double)new_val - (double)old_val;
            if (fabs(applied) > fabs(rep->delta)) {
                rep->delta = applied;
                rep->row = r;
                rep->col = col;
            }
        }
    }
    free(s1);
    free(s2);
    if (any_uncorrectable) rep->status = ORC_DETECTED_UNCORRECTABLE;
    else if (rep->corrections > 0 || rep->checksum_repair) rep->status = ORC_CORRECTED;
}

int eorc_verify_locate_correct(int rows, int cols, int stride, float* t, const float* c1,
                               const float* c2, double eps, const double* row_eps_mult,
                               orc_verify_report* rep) {
    if (stride <= 0 || cols % stride != 0) {
        set_err("verify_locate_correct: checksum/tile shape mismatch");
        return 1;
    }
    verify_locate_correct(t, rows, cols, stride, c1, c2, eps, row_eps_mult, rep);
    return 0;
}

/* src/gemm.cpp:7-21: C = C_init + A*B, fp32 products, fixed k order. */
static void gemm_mixed(const float* a, const float* b, const float* c_init, float* c, int m, int k,
                       int n) {
    for (int i = 0; i < m; ++i)
        for (int j = 0; j < n; ++j) {
            float acc = c_init ? c_init[(size_t)i * n + j] : 0.0f;
            for (int p = 0; p < k; ++p) acc += a[(size_t)i * k + p] * b[(size_t)p * n + j];
            c[(size_t)i * n + j] = acc;
        }
}

/* src/abft.cpp:322-369: one pass over [bt | c1(bt) | c2(bt)], optional
 * initial value c_init with its checksums. cp_* are m x stride. */
static void checksummed_gemm(const float* a, const float* bt, int m, int kd, int w, int stride,
                             const float* c_init, const float* cp1_init, const float* cp2_init,
                             float* c, float* cp1, float* cp2) {
    const int wa = w + 2 * stride;
    float* e1 = (float*)malloc(sizeof(float) * kd * stride);
    float* e2 = (float*)malloc(sizeof(float) * kd * stride);
    strided_sums(bt, kd, w, stride, e1, e2);
    float* aug = (float*)malloc(sizeof(float) * (size_t)kd * wa);
    for (int r = 0; r < kd; ++r) {
        for (int cc = 0; cc < w; ++cc) aug[(size_t)r * wa + cc] = bt[(size_t)r * w + cc];
        for (int j = 0; j < stride; ++j) {
            aug[(size_t)r * wa + w + j] = e1[r * stride + j];
            aug[(size_t)r * wa + w + stride + j] = e2[r * stride + j];
        }
    }
    float* init = NULL;
    if (c_init) {
        init = (float*)malloc(sizeof(float) * (size_t)m * wa);
        for (int r = 0; r < m; ++r) {
            for (int cc = 0; cc < w; ++cc) init[(size_t)r * wa + cc] = c_init[(size_t)r * w + cc];
            for (int j = 0; j < stride; ++j) {
                init[(size_t)r * wa + w + j] = cp1_init[r * stride + j];
                init[(size_t)r * wa + w + stride + j] = cp2_init[r * stride + j];
            }
        }
    }
    float* caug = (float*)malloc(sizeof(float) * (size_t)m * wa);
    gemm_mixed(a, aug, init, caug, m, kd, wa);
    for (int r = 0; r < m; ++r) {
        for (int cc = 0; cc < w; ++cc) c[(size_t)r * w + cc] = caug[(size_t)r * wa + cc];
        for (int j = 0; j < stride; ++j) {
            cp1[r * stride + j] = caug[(size_t)r * wa + w + j];
            cp2[r * stride + j] = caug[(size_t)r * wa + w + stride + j];
        }
    }
    free(e1); free(e2); free(aug); free(init); free(caug);
}

int eorc_checksummed_gemm(int m, int kd, int w, int stride, const float* a, const float* bt,
                          float* c, float* c1, float* c2) {
    if (stride <= 0 || w % stride != 0) {
        set_err("checksummed_gemm: stride must divide width");
        return 1;
    }
    checksummed_gemm(a, bt, m, kd, w, stride, NULL, NULL, NULL, c, c1, c2);
    return 0;
}

/* ---------------------------------------------------------------- SNVR --- */
static inline int usable(float p) { return isfinite(p) && p > 0.0f; }

/* src/snvr.cpp:52-83 (scan). Returns any-violation; updates rep. */
static int exp_scan(const float* p, const float* pc1, const float* m, int rows, int w, int stride,
                    double eps1, char* affected, orc_verify_report* rep) {
    const int groups = w / stride;
    int any = 0;
    for (int r = 0; r < rows; ++r) {
        int degenerate = !isfinite(m[r]);
        for (int c = 0; c < w && !degenerate; ++c)
            if (!usable(p[(size_t)r * w + c])) degenerate = 1;
        for (int j = 0; j < stride && !degenerate; ++j)
            if (!usable(pc1[r * stride + j])) degenerate = 1;
        if (degenerate) {
            affected[r] = 1;
            any = 1;
            rep->residual = INFINITY;
            ++rep->violations;
            continue;
        }
        for (int j = 0; j < stride; ++j) {
            double lhs = 0.0;
            for (int l = 0; l < groups; ++l) lhs += log((double)p[(size_t)r * w + j + stride * l]);
            const double rhs = log((double)pc1[r * stride + j]);
            const double diff = fabs(lhs - rhs);
            if (diff > rep->residual) rep->residual = diff;
            if (diff > eps1) {
                affected[r] = 1;
                any = 1;
                ++rep->violations;
            }
        }
    }
    return any;
}

/* std::max(a,b) semantics: returns a unless a < b (NaN-propagation as in the reference) */
static inline float smax(float a, float b) { return (a < b) ? b : a; }

static float row_max_ref(const float* t, int cols) { /* src/matrix.cpp:90-94 */
    float v = t[0];
    for (int c = 1; c < cols; ++c) v = smax(v, t[c]);
    return v;
}

static float row_sum(const float* t, int cols) { /* src/matrix.cpp:96-100 */
    float s = 0.0f;
    for (int c = 0; c < cols; ++c) s += t[c];
    return s;
}

/* src/snvr.cpp:43-159 */
static void verify_exp_stage(float* p, float* pc1, float* s, const float* cs1, const float* cs2,
                             float* m, const float* m_old, float* block_max, int rows, int w,
                             int stride, double eps1, double eps_lin, injector_t* inj, int bi,
                             int bj, orc_verify_report* rep, int* recomputed) {
    const int groups = w / stride;
    memset(rep, 0, sizeof(*rep));
    rep->row = -1;
    rep->col = -1;
    *recomputed = 0;
    char* affected = (char*)calloc(rows, 1);
    if (!exp_scan(p, pc1, m, rows, w, stride, eps1, affected, rep)) {
        free(affected);
        return;
    }
    /* :89-98 linear repair of the score tile */
    orc_verify_report lin;
    verify_locate_correct(s, rows, w, stride, cs1, cs2, eps_lin, NULL, &lin);
    if (lin.corrections > 0) {
        rep->corrections += lin.corrections;
        if (lin.row >= 0) affected[lin.row] = 1;
        rep->row = lin.row;
        rep->col = lin.col;
        rep->delta = lin.delta;
    }
    /* :102-139 recompute affected rows from held state */
    float* before = (float*)malloc(sizeof(float) * (w + stride));
    for (int r = 0; r < rows; ++r) {
        if (!affected[r]) continue;
        memcpy(before, p + (size_t)r * w, sizeof(float) * w);
        memcpy(before + w, pc1 + r * stride, sizeof(float) * stride);
        const float bm = row_max_ref(s + (size_t)r * w, w);
        block_max[r] = bm;
        float mm = smax(m_old[r], bm);
        mm = tap(inj, ORC_REDUCE_MAX, bi, bj, r, 0, mm);
        m[r] = mm;
        for (int c = 0; c < w; ++c) {
            float a = s[(size_t)r * w + c] - mm;
            a = tap(inj, ORC_SUB_MAX, bi, bj, r, c, a);
            float e = expf(a);
            e = tap(inj, ORC_EXP_OUT, bi, bj, r, c, e);
            p[(size_t)r * w + c] = e;
        }
        for (int j = 0; j < stride; ++j) pc1[r * stride + j] = expf(cs1[r * stride + j] - (float)groups * mm);
        int changed = 0;
        for (int c = 0; c < w && !changed; ++c)
            if (f2u(before[c]) != f2u(p[(size_t)r * w + c])) changed = 1;
        for (int j = 0; j < stride && !changed; ++j)
            if (f2u(before[w + j]) != f2u(pc1[r * stride + j])) changed = 1;
        if (changed) {
            *recomputed = 1;
            ++rep->corrections;
            if (rep->row < 0) rep->row = r;
        }
    }
    free(before);
    /* :141-157 re-scan */
    const orc_verify_report first = *rep;
    rep->residual = 0.0;
    char* still = (char*)calloc(rows, 1);
    const int bad = exp_scan(p, pc1, m, rows, w, stride, eps1, still, rep);
    rep->violations = first.violations;
    rep->residual = fmax(first.residual, bad ? rep->residual : 0.0);
    if (bad || lin.status == ORC_DETECTED_UNCORRECTABLE) rep->status = ORC_DETECTED_UNCORRECTABLE;
    else if (rep->corrections > 0) rep->status = ORC_CORRECTED;
    else rep->status = ORC_CLEAN;
    free(still);
    free(affected);
}

/* ------------------------------------------------------------- report --- */
typedef struct {
    orc_event* events;
    int cap, n;
    int detections, corrections, recomputes, range_replacements, failed;
} report_t;

/* src/efta.cpp:49-55 */
static void push_event(report_t* R, int kind, int bi, int bj, const orc_verify_report* r) {
    if (R->n < R->cap) {
        orc_event* e = &R->events[R->n];
        memset(e, 0, sizeof(*e));
        e->kind = kind;
        e->block_i = bi;
        e->block_j = bj;
        e->status = r->status;
        e->row = r->row;
        e->col = r->col;
        e->violations = r->violations;
        e->corrections = r->corrections;
        e->checksum_repair = r->checksum_repair;
        e->residual = r->residual;
        e->delta = r->delta;
    }
    ++R->n;
    if (r->status != ORC_CLEAN) ++R->detections;
    R->corrections += r->corrections;
    if (r->status == ORC_DETECTED_UNCORRECTABLE || r->status == ORC_NONFINITE) R->failed = 1;
}

static int validate_cfg(int n, int d, int block, int stride, float* scale) {
    /* include/efta/config.hpp:30-41 */
    if (n <= 0 || d <= 0 || block <= 0 || stride <= 0) { set_err("config: dimensions must be positive"); return 1; }
    if (n % block != 0) { set_err("config: block must divide seq_len"); return 1; }
    if (block % stride != 0) { set_err("config: stride must divide block"); return 1; }
    if (d % stride != 0) { set_err("config: stride must divide head_dim"); return 1; }
    if (*scale == 0.0f) *scale = 1.0f / sqrtf((float)d);
    return 0;
}

/* -------------------------------------------------------- efta_forward --- */
/* src/efta.cpp:72-351 (modes NONE / EFTA / EFTA_OPTIMIZED) */
int eorc_efta_forward(int N, int d, int B, int s, float scale, int mode, double eps1, double eps2,
                      double eps_lin, int observe_linear, float bias, const float* q,
                      const float* k, const float* v, float* o, float* m_out, float* l_out,
                      const orc_fault_spec* specs, int n_specs, orc_event* events, int ev_cap,
                      orc_fired* fired, int fired_cap, orc_summary* sum) {
    if (validate_cfg(N, d, B, s, &scale)) return 1;
    if (mode < 0 || mode > 2) { set_err("efta_forward: unsupported mode"); return 1; }
    const int n = N / B;
    const int protect = mode == ORC_MODE_EFTA || mode == ORC_MODE_EFTA_OPT;
    const int GB = B / s; /* cfg.groups(B), efta.cpp:164 */
    counters_t cnt;
    memset(&cnt, 0, sizeof cnt);
    report_t R;
    memset(&R, 0, sizeof R);
    R.events = events;
    R.cap = ev_cap;
    injector_t injs, *inj = NULL;
    if (n_specs > 0) {
        injs.specs = specs;
        injs.n_specs = n_specs;
        injs.evals = (int*)calloc(n_specs, sizeof(int));
        injs.fired = fired;
        injs.fired_cap = fired_cap;
        injs.n_fired = 0;
        inj = &injs;
    }

    /* per-block scratch */
    float* kt = (float*)malloc(sizeof(float) * d * B);       /* K_j^T, d x B */
    float* sc = (float*)malloc(sizeof(float) * B * B);
    float* scp1 = (float*)malloc(sizeof(float) * B * s);
    float* scp2 = (float*)malloc(sizeof(float) * B * s);
    float* p = (float*)malloc(sizeof(float) * B * B);
    float* pc1 = (float*)malloc(sizeof(float) * B * s);
    float* oacc = (float*)malloc(sizeof(float) * B * d);
    float* onew = (float*)malloc(sizeof(float) * B * d);
    float* ocp1 = (float*)malloc(sizeof(float) * B * s);
    float* ocp2 = (float*)malloc(sizeof(float) * B * s);
    float* ncp1 = (float*)malloc(sizeof(float) * B * s);
    float* ncp2 = (float*)malloc(sizeof(float) * B * s);
    float *m = (float*)malloc(sizeof(float) * B), *l = (float*)malloc(sizeof(float) * B);
    float *m_old = (float*)malloc(sizeof(float) * B), *bmax = (float*)malloc(sizeof(float) * B);
    float* factor = (float*)malloc(sizeof(float) * B);
    float* hist = (float*)malloc(sizeof(float) * B * n); /* RowmaxHistory::block_max */
    float* hglob = (float*)malloc(sizeof(float) * B);
    double* eps_mult = (double*)malloc(sizeof(double) * B);

    for (int i = 0; i < n; ++i) {
        const float* qi = q + (size_t)i * B * d;
        memset(oacc, 0, sizeof(float) * B * d);
        if (protect) {
            memset(ocp1, 0, sizeof(float) * B * s);
            memset(ocp2, 0, sizeof(float) * B * s);
        }
        for (int r = 0; r < B; ++r) { m[r] = -INFINITY; l[r] = 0.0f; hglob[r] = -INFINITY; }

        for (int j = 0; j < n; ++j) {
            const float* kj = k + (size_t)j * B * d;
            const float* vj = v + (size_t)j * B * d;
            for (int r = 0; r < B; ++r)
                for (int c = 0; c < d; ++c) kt[(size_t)c * B + r] = kj[(size_t)r * d + c];

            /* scores (efta.cpp:125-148) */
            if (protect) {
                checksummed_gemm(qi, kt, B, d, B, s, NULL, NULL, NULL, sc, scp1, scp2);
                cnt.cs_scores += 2ull * B * (2 * s) * d;
            } else {
                gemm_mixed(qi, kt, NULL, sc, B, d, B);
            }
            cnt.main_scores += 2ull * B * B * d;
            for (int x = 0; x < B * B; ++x) sc[x] *= scale;
            cnt.main_scores += (uint64_t)B * B;
            if (protect) {
                for (int x = 0; x < B * s; ++x) { scp1[x] *= scale; scp2[x] *= scale; }
                cnt.cs_scores += 2ull * B * s;
            }
            if (inj)
                for (int r = 0; r < B; ++r)
                    for (int c = 0; c < B; ++c)
                        sc[r * B + c] = tap(inj, ORC_GEMM1_OUT, i, j, r, c, sc[r * B + c]);

            /* running max (efta.cpp:150-159) */
            for (int r = 0; r < B; ++r) {
                m_old[r] = m[r];
                float bm = row_max_ref(sc + (size_t)r * B, B);
                bm += bias;
                bmax[r] = bm;
                float mm = smax(m_old[r], bm);
                mm = tap(inj, ORC_REDUCE_MAX, i, j, r, 0, mm);
                m[r] = mm;
            }

            /* exp stage (efta.cpp:161-178) */
            for (int r = 0; r < B; ++r) {
                for (int c = 0; c < B; ++c) {
                    float a = sc[r * B + c] - m[r];
                    a = tap(inj, ORC_SUB_MAX, i, j, r, c, a);
                    float e = expf(a);
                    e = tap(inj, ORC_EXP_OUT, i, j, r, c, e);
                    p[r * B + c] = e;
                }
                if (protect)
                    for (int jj = 0; jj < s; ++jj)
                        pc1[r * s + jj] = expf(scp1[r * s + jj] - (float)GB * m[r]);
            }

            if (protect) {
                if (observe_linear) { /* efta.cpp:181-185 */
                    orc_verify_report lrep;
                    verify_locate_correct(sc, B, B, s, scp1, scp2, INFINITY, NULL, &lrep);
                    push_event(&R, ORC_SCORE_CHECKSUM, i, j, &lrep);
                }
                orc_verify_report erep;
                int recomputed = 0;
                ++cnt.exp_checks;
                verify_exp_stage(p, pc1, sc, scp1, scp2, m, m_old, bmax, B, B, s, eps1, eps_lin,
                                 inj, i, j, &erep, &recomputed);
                if (recomputed) ++R.recomputes;
                push_event(&R, ORC_EXP_CHECKSUM, i, j, &erep);
            }

            /* rescale factor guard (efta.cpp:192-230) */
            for (int r = 0; r < B; ++r) {
                float f = expf(m_old[r] - m[r]);
                if (protect && j > 0 && !(isfinite(f) && f > 0.0f && f <= 1.0f)) {
                    orc_verify_report g;
                    memset(&g, 0, sizeof g);
                    g.row = r;
                    g.col = -1;
                    g.residual = isfinite(f) ? (double)f - 1.0 : INFINITY;
                    float bm = row_max_ref(sc + (size_t)r * B, B) + bias;
                    bmax[r] = bm;
                    float mm = smax(m_old[r], bm);
                    mm = tap(inj, ORC_REDUCE_MAX, i, j, r, 0, mm);
                    m[r] = mm;
                    for (int c = 0; c < B; ++c) {
                        float a = sc[r * B + c] - mm;
                        a = tap(inj, ORC_SUB_MAX, i, j, r, c, a);
                        float e = expf(a);
                        e = tap(inj, ORC_EXP_OUT, i, j, r, c, e);
                        p[r * B + c] = e;
                    }
                    for (int jj = 0; jj < s; ++jj)
                        pc1[r * s + jj] = expf(scp1[r * s + jj] - (float)GB * mm);
                    f = expf(m_old[r] - m[r]);
                    ++R.recomputes;
                    if (isfinite(f) && f > 0.0f && f <= 1.0f) {
                        g.status = ORC_CORRECTED;
                        g.corrections = 1;
                    } else {
                        g.status = ORC_DETECTED_UNCORRECTABLE;
                    }
                    push_event(&R, ORC_FACTOR_RANGE, i, j, &g);
                }
                factor[r] = f;
            }

            for (int r = 0; r < B; ++r) { hist[r * n + j] = bmax[r]; hglob[r] = m[r]; }

            /* denominator (efta.cpp:238-242) */
            for (int r = 0; r < B; ++r) {
                float lv = factor[r] * l[r] + row_sum(p + (size_t)r * B, B);
                lv = tap(inj, ORC_REDUCE_SUM, i, j, r, 0, lv);
                l[r] = lv;
            }

            /* rescale accumulator (efta.cpp:246-260) */
            for (int r = 0; r < B; ++r)
                for (int c = 0; c < d; ++c) {
                    float ov = oacc[r * d + c] * factor[r];
                    ov = tap(inj, ORC_RESCALE_FACTOR, i, j, r, c, ov);
                    oacc[r * d + c] = ov;
                }
            cnt.main_output += (uint64_t)B * d;
            if (protect) {
                for (int r = 0; r < B; ++r)
                    for (int jj = 0; jj < s; ++jj) {
                        ocp1[r * s + jj] *= factor[r];
                        ocp2[r * s + jj] *= factor[r];
                    }
                cnt.cs_output += 2ull * B * s;
            }

            /* O += P V_j (efta.cpp:270-280) */
            if (protect) {
                checksummed_gemm(p, vj, B, B, d, s, oacc, ocp1, ocp2, onew, ncp1, ncp2);
                memcpy(ocp1, ncp1, sizeof(float) * B * s);
                memcpy(ocp2, ncp2, sizeof(float) * B * s);
                cnt.cs_output += 2ull * B * (2 * s) * B;
            } else {
                gemm_mixed(p, vj, oacc, onew, B, B, d);
            }
            cnt.main_output += 2ull * B * d * B;
            memcpy(oacc, onew, sizeof(float) * B * d);
            if (inj)
                for (int r = 0; r < B; ++r)
                    for (int c = 0; c < d; ++c)
                        oacc[r * d + c] = tap(inj, ORC_GEMM2_ACC, i, j, r, c, oacc[r * d + c]);

            if (mode == ORC_MODE_EFTA) { /* efta.cpp:282-286 */
                ++cnt.output_checks;
                orc_verify_report orep;
                verify_locate_correct(oacc, B, d, s, ocp1, ocp2, eps2, NULL, &orep);
                push_event(&R, ORC_OUTPUT_CHECKSUM, i, j, &orep);
            }
        }

        /* range restriction (efta.cpp:289-310, snvr.cpp:161-182) */
        int have_mult = 0;
        if (protect) {
            int n_repl = 0, first = -1;
            double maxv = 0.0;
            for (int r = 0; r < B; ++r) eps_mult[r] = 1.0;
            for (int r = 0; r < B; ++r) {
                float lower = 0.0f;
                for (int jb = 0; jb < n; ++jb) lower += expf(hist[r * n + jb] - hglob[r]);
                const int bad = !isfinite(l[r]) || l[r] < lower || l[r] > (float)N;
                if (!bad) continue;
                double viol;
                if (!isfinite(l[r])) viol = INFINITY;
                else viol = l[r] < lower ? (double)lower - l[r] : (double)l[r] - (float)N;
                if (viol > maxv) maxv = viol;
                l[r] = lower;
                if (first < 0) first = r;
                ++n_repl;
                /* efta.cpp:306-308: replaced rows get eps multiplier N / l */
                eps_mult[r] = (double)N / (double)l[r];
            }
            if (n_repl > 0) {
                orc_verify_report g;
                memset(&g, 0, sizeof g);
                g.status = ORC_CORRECTED;
                g.corrections = n_repl;
                g.residual = maxv;
                g.row = first;
                g.col = -1;
                push_event(&R, ORC_ROWSUM_RANGE, i, n, &g);
                R.range_replacements += n_repl;
                have_mult = 1;
            }
        }

        /* normalization (efta.cpp:312-327) */
        for (int r = 0; r < B; ++r)
            for (int c = 0; c < d; ++c) {
                float ov = oacc[r * d + c] / l[r];
                ov = tap(inj, ORC_NORMALIZE_OUT, i, 0, r, c, ov);
                oacc[r * d + c] = ov;
            }
        cnt.main_output += (uint64_t)B * d;
        if (protect) {
            for (int r = 0; r < B; ++r)
                for (int jj = 0; jj < s; ++jj) {
                    ocp1[r * s + jj] /= l[r];
                    ocp2[r * s + jj] /= l[r];
                }
            cnt.cs_output += 2ull * B * s;
        }

        if (protect) { /* efta.cpp:329-336 */
            ++cnt.output_checks;
            orc_verify_report orep;
            verify_locate_correct(oacc, B, d, s, ocp1, ocp2, eps2, have_mult ? eps_mult : NULL,
                                  &orep);
            push_event(&R, ORC_OUTPUT_CHECKSUM, i, n, &orep);
        }

        for (int r = 0; r < B; ++r) {
            memcpy(o + (size_t)(i * B + r) * d, oacc + (size_t)r * d, sizeof(float) * d);
            if (m_out) m_out[i * B + r] = m[r];
            if (l_out) l_out[i * B + r] = l[r];
        }
    }

    if (sum) {
        memset(sum, 0, sizeof(*sum));
        sum->detections = R.detections;
        sum->corrections = R.corrections;
        sum->recomputes = R.recomputes;
        sum->range_replacements = R.range_replacements;
        sum->failed = R.failed;
        sum->n_events = R.n;
        sum->n_fired = inj ? inj->n_fired : 0;
        sum->flops_main_gemm_scores = cnt.main_scores;
        sum->flops_cs_gemm_scores = cnt.cs_scores;
        sum->flops_main_gemm_output = cnt.main_output;
        sum->flops_cs_gemm_output = cnt.cs_output;
        sum->exp_checks = cnt.exp_checks;
        sum->output_checks = cnt.output_checks;
    }
    free(kt); free(sc); free(scp1); free(scp2); free(p); free(pc1); free(oacc); free(onew);
    free(ocp1); free(ocp2); free(ncp1); free(ncp2); free(m); free(l); free(m_old); free(bmax);
    free(factor); free(hist); free(hglob); free(eps_mult);
    if (inj) free(injs.evals);
    return 0;
}

/* ------------------------------------------------------------ campaign --- */
/* src/fault.cpp:81-96 column bound per site */
static int site_col_bound(int site, int block, int d) {
    switch (site) {
        case ORC_GEMM1_OUT: case ORC_SUB_MAX: case ORC_EXP_OUT: return block;
        case ORC_REDUCE_MAX: case ORC_REDUCE_SUM: return 1;
        default: return d;
    }
}

/* src/campaign.cpp:177-185 + src/fault.cpp:143-164 (sample_random_plan,
 * non-decoupled layout) */
int eorc_gen_trial(uint64_t seed, int n, int d, int block, int stride, const int* sites,
                   int n_sites, float* q, float* k, float* v, orc_fault_spec* spec_out) {
    float scale = 0.0f;
    if (validate_cfg(n, d, block, stride, &scale)) return 1;
    rng_t r;
    rng_init(&r, seed);
    random_fill(&r, n, d, -1.0, 1.0, 1, q);
    random_fill(&r, n, d, -1.0, 1.0, 1, k);
    random_fill(&r, n, d, -1.0, 1.0, 1, v);
    if (n_sites > 0) {
        orc_fault_spec f;
        f.site = sites[rng_below(&r, (uint32_t)n_sites)];
        const int nb = n / block;
        f.block_i = (int)rng_below(&r, (uint32_t)nb);
        f.block_j = f.site == ORC_NORMALIZE_OUT ? 0 : (int)rng_below(&r, (uint32_t)nb);
        f.row = (int)rng_below(&r, (uint32_t)block);
        f.col = (int)rng_below(&r, (uint32_t)site_col_bound(f.site, block, d));
        f.bit = (int)rng_below(&r, 32);
        f.trigger = 1;
        *spec_out = f;
    }
    return 0;
}

/* src/attention.cpp:20-57: two-pass attention with full S and P */
int eorc_standard_attention(int n, int d, int block, int stride, float scale, const float* q,
                            const float* k, const float* v, float* o) {
    if (validate_cfg(n, d, block, stride, &scale)) return 1;
    float* kt = (float*)calloc((size_t)d * n, sizeof(float));
    float* s = (float*)malloc(sizeof(float) * (size_t)n * n);
    for (int r = 0; r < n; ++r)
        for (int c = 0; c < d; ++c) kt[(size_t)c * n + r] = k[(size_t)r * d + c];
    gemm_mixed(q, kt, NULL, s, n, d, n);
    for (size_t x = 0; x < (size_t)n * n; ++x) s[x] *= scale;
    float* l = (float*)malloc(sizeof(float) * n);
    for (int r = 0; r < n; ++r) {
        const float mr = row_max_ref(s + (size_t)r * n, n);
        for (int c = 0; c < n; ++c) s[(size_t)r * n + c] = expf(s[(size_t)r * n + c] - mr);
        l[r] = row_sum(s + (size_t)r * n, n);
    }
    gemm_mixed(s, v, NULL, o, n, n, d);
    for (int r = 0; r < n; ++r)
        for (int c = 0; c < d; ++c) o[(size_t)r * d + c] /= l[r];
    free(kt); free(s); free(l);
    return 0;
}
