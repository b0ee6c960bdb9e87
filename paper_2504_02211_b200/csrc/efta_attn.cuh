// efta_attn.cuh — fused end-to-end fault-tolerant attention forward for sm_100a.
//
// Replaces the reference's efta_forward (src/efta.cpp:72-351) for one
// [batch*heads, seq, d] fp16 problem. One CTA owns one (head, 128-row query
// block) = the reference's row-block i; it streams the key/value blocks j
// (B_c = 128) with the reference's online-softmax recurrence (rescale every
// iteration, src/efta.cpp:192-260).
//
// Warp roles (256 threads):
//   warp 0      TMA producer for K_j (+ its strided checksum rows KC_j)
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer
//   warp 3      TMA producer for V_j (+ VC_j) and Q
//   warps 4..7  "row warpgroup": thread t owns query row t == TMEM lane t.
//               Softmax, exp-stage check, factor guard, O rescale (correction),
//               epilogue normalisation + final output check + store.
//
// TMEM columns (512 allocated):
//   S[b] = b*160 (b = j&1): 128 score cols | 16 hi | 16 lo checksum cols
//          (P_j as fp16x2 is written over its first 64 cols)
//   O    = 320: D cols | 16 hi | 16 lo checksum cols
//
// Checksum operands (hi/lo fp16 split of the fp32 strided sums, produced by
// efta_encode_kv in efta_encode.cuh) ride alongside every K/V tile:
//   KC_j  [32 x D]   rows 0-7 c1_hi, 8-15 c2_hi, 16-23 c1_lo, 24-31 c2_lo
//   VC_j  [128 x 64] per key: cols 0-7 c1_hi, 8-15 c2_hi, 16-23 c1_lo, 24-31 c2_lo, 32-63 zero
// They are appended to the B operands so a single tcgen05.mma per k-step computes
// the scores plus their checksums (N = 160) and P.V plus the output checksums
// (N = D + 32): every operand is read from SMEM/TMEM exactly once.
#pragma once
#include <cuda.h>
#include <cuda_fp16.h>
#include <cstdint>
#include <math_constants.h>

#include "efta_types.h"
#include "sm100_ptx.cuh"

namespace efta_sm100 {

constexpr int kBlock = 128;   // B_r = B_c (reference AttnConfig::block)
constexpr int kStride = 8;    // s   (reference AttnConfig::stride)
constexpr int kCsCols = 2 * kStride;  // c1 | c2
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

struct AttnParams {
    int seq_len, nblk, n_heads_flat;
    float scale, scale_log2, rowmax_bias;
    double eps1, eps2, eps_lin;
    float* o;        // [BH, S, D] fp32
    float* m_out;    // [BH, S]
    float* l_out;    // [BH, S]
    efta_event* events;
    int ev_cap;
    efta_counters* counters;
    const efta_fault_spec* faults;
    int n_faults;
    efta_fired* fired;
    int fired_cap;
    int observe_linear;
    // exp-stage bracket: |ln(prod/pc1)| > eps1  <=>  prod outside [pc1*exp_lo, pc1*exp_hi]
    float exp_lo, exp_hi;
    float* scratch;  // workspace scratch: the persistent pair kernel's tile counter (int at [0])
    unsigned long long* prof;  // EFTA_PROF builds only: phase timestamps of one CTA
    const __half* q;           // [BH, S, D]: the pair kernel's rare path recomputes score c2 from Q . KC2
    const __half* kc;          // [BH_kv*n, 32, D] checksum rows (workspace)
    int heads_q;               // query heads per batch entry (H)
    int kv_group;              // query heads per K/V head (GQA; 1 = multi-head attention)
    int causal;                // causal build of the pair kernel was selected (key k visible to query q iff k <= q)
    int o_tok;                 // 1: o holds fp16 [B, S, H, D] (token-major, the next linear layer's input)
};

// Pair-kernel tile u -> (head, query pair, key blocks to visit). Causal: a query pair (2i, 2i+1)
// needs key blocks 0..2i+1; a head's pairs are handed out longest first (head-major, so the
// head's K / V stay in L2 while its tiles run).
struct PairTile {
    int head, pair, nblk;
};
template <bool CAUSAL>
__device__ __forceinline__ PairTile pair_tile(const AttnParams& p, int u) {
    const int npq = p.nblk / 2;
    PairTile t;
    t.head = u / npq;
    t.pair = CAUSAL ? npq - 1 - u % npq : u % npq;
    t.nblk = CAUSAL ? 2 * t.pair + 2 : p.nblk;
    return t;
}

// Grouped-query attention: flat query head (b*H + h) -> flat K/V head (b*H_kv + h / group)
__device__ __forceinline__ int kv_head(const AttnParams& p, int head) {
    return p.kv_group == 1 ? head : (head / p.heads_q) * (p.heads_q / p.kv_group) + (head % p.heads_q) / p.kv_group;
}

#ifdef EFTA_PROF
// phase timestamps (clock64) of CTA (2,5) (a pair leader): lane 0 of the stamping warp;
// EFTA_TSQ stamps all four warps of a row warpgroup at slots 16 + base + warp quarter
#define EFTA_TS(slot, j)                                                                       \
    do {                                                                                       \
        if (p.prof && blockIdx.x == 2 && blockIdx.y == (gridDim.y > 1 ? 5 : 0) &&             \
            (threadIdx.x & 31) == 0 && (j) >= 0 && (j) < 64)                                   \
            p.prof[(j) * 64 + (slot)] = clock64();                                             \
    } while (0)
#define EFTA_TSQ(base, j)                                                                      \
    do {                                                                                       \
        if (p.prof && blockIdx.x == 2 && blockIdx.y == (gridDim.y > 1 ? 5 : 0) &&             \
            (threadIdx.x & 31) == 0 && (j) >= 0 && (j) < 64)                                   \
            p.prof[(j) * 64 + 16 + (base) + ((threadIdx.x >> 5) & 3)] = clock64();              \
    } while (0)
// per warp quarter of the calling warpgroup (lane 0 of each warp): slots base .. base + 3
#define EFTA_TSW(base, j)                                                                      \
    do {                                                                                       \
        if (p.prof && blockIdx.x == 2 && blockIdx.y == (gridDim.y > 1 ? 5 : 0) &&             \
            (threadIdx.x & 31) == 0 && (j) >= 0 && (j) < 64)                                   \
            p.prof[(j) * 64 + (base) + ((threadIdx.x >> 5) & 3)] = clock64();                  \
    } while (0)
#else
#define EFTA_TS(slot, j) do { } while (0)
#define EFTA_TSQ(base, j) do { } while (0)
#define EFTA_TSW(base, j) do { } while (0)
#endif


// fast variants rescale O lazily (only when the running max grows by > kLazyTau)
__host__ __device__ constexpr bool attn_lazy(int mode, bool dbg) { return !dbg && mode != 1; }
constexpr float kLazyTau = 5.545177444479562f;  // 8 * ln 2: P <= 2^8 between rescales

template <int D>
struct AttnLayout {
    static constexpr int NSUB = D / 64;
    static constexpr int KS = (D == 64) ? 3 : 2;  // K ring stages
    static constexpr int VS = (D == 64) ? 3 : 2;  // V ring stages
    // K stage: per 64-column chunk [K_j rows 0..127 | KC rows 0..31] so that one
    // K-major B descriptor spans N = 128 (+32 checksum rows) = 160
    static constexpr uint32_t K_SUB = 16384 + 4096;
    static constexpr uint32_t K_STAGE = NSUB * K_SUB;
    // V stage: MN-major [V chunk 0 | V chunk 1 | VC (32 used of 64 cols)], 16 KB each,
    // so one MN-major B descriptor spans N = D (+32 checksum columns)
    static constexpr uint32_t V_STAGE = (NSUB + 1) * 16384;
    static constexpr uint32_t Q_BYTES = NSUB * 16384;
    static constexpr uint32_t K_BYTES = NSUB * 16384;
    static constexpr uint32_t KC_BYTES = NSUB * 4096;
    static constexpr uint32_t V_BYTES = NSUB * 16384;
    static constexpr uint32_t VC_BYTES = 16384;
    static constexpr uint32_t OFF_Q = 0;
    static constexpr uint32_t OFF_K = OFF_Q + Q_BYTES;
    static constexpr uint32_t OFF_V = OFF_K + KS * K_STAGE;
    static constexpr uint32_t OFF_BAR = OFF_V + VS * V_STAGE;
    // barriers: q_full, k_full[KS], k_empty[KS], v_full[VS], v_empty[VS], s_full[2],
    //           p_ready, o_done  -> then tmem slot + scratch for tile reductions
    static constexpr int NBAR = 1 + 2 * KS + 2 * VS + 2 + 2;
    static constexpr uint32_t OFF_TMEM = OFF_BAR + NBAR * 8;
    static constexpr uint32_t OFF_RED = (OFF_TMEM + 16 + 15) & ~15u;
    static constexpr uint32_t RED_BYTES = 128 * 24 + 256;  // RowSlot[128] + ints + doubles
    static constexpr uint32_t SMEM_BYTES = OFF_RED + RED_BYTES + 1024;  // + alignment slack
    // TMEM: S[b] = b*160: cols 0..127 scores (P aliased over 0..63), 128..143 checksum
    // hi-products, 144..159 lo-products; O at 320: D cols + 16 hi + 16 lo checksum cols.
    static constexpr uint32_t S_STRIDE = 160;
    static constexpr uint32_t COL_S0 = 0, COL_O = 320;
    static constexpr uint32_t TMEM_COLS = 512;
};

// ---------------------------------------------------------------- fault taps
// Per-thread injector state. The reference allows at most one spec per
// row-block (src/fault.cpp:117-119), so a (head, block_i) CTA has <= 1 spec
// and only the thread owning spec.row evaluates it. Evaluation counting and
// trigger semantics mirror FaultInjector::tap (include/efta/fault.hpp:82-95).
struct ThreadTap {
    int active, site, bj, col, bit, trigger, count, idx;
    int logged;  // the fired record is written once even if a block is re-evaluated (pair kernel chain redo)
    __device__ __forceinline__ float fire(const AttnParams& p, float v) {
        const float flipped = __uint_as_float(__float_as_uint(v) ^ (1u << bit));
        if (!logged) {
            logged = 1;
            const int slot = atomicAdd(&p.counters->n_fired, 1);
            if (slot < p.fired_cap) {
                p.fired[slot].spec = p.faults[idx];
                p.fired[slot].before = v;
                p.fired[slot].after = flipped;
            }
        }
        return flipped;
    }
    __device__ __forceinline__ float operator()(const AttnParams& p, int s, int j, int c,
                                                float v) {
        if (!active || s != site || j != bj || c != col) return v;
        if (++count != trigger) return v;
        return fire(p, v);
    }
    // One evaluation of cell `col` of site s at key block j: counts it and returns true
    // when this evaluation is the trigger-th (the caller then flips that cell with fire()).
    // Lets an unrolled register row be tapped without dynamic indexing.
    __device__ __forceinline__ bool hit(int s, int j) {
        if (!active || s != site || j != bj) return false;
        return ++count == trigger;
    }
    // set up from the device fault table for (head, row-block bi, row); at most one spec
    // per row-block (src/fault.cpp:117-119), the last match wins like the linear scan
    __device__ __forceinline__ void load(const AttnParams& p, int head, int bi, int row) {
        active = 0;
        count = 0;
        logged = 0;
        for (int i = 0; i < p.n_faults; ++i) {
            const efta_fault_spec f = p.faults[i];
            if (f.head == head && f.block_i == bi && f.row == row) {
                active = 1;
                site = f.site;
                bj = f.block_j;
                col = f.col;
                bit = f.bit;
                trigger = f.trigger;
                idx = i;
            }
        }
    }
};

// value of / store into element `col` of a register row without dynamic indexing (selects;
// rare-path and tap-build helpers)
template <int N>
__device__ __forceinline__ float sel_get(const float* x, int col) {
    float v = 0.0f;
#pragma unroll
    for (int c = 0; c < N; ++c) v = (c == col) ? x[c] : v;
    return v;
}
template <int N>
__device__ __forceinline__ void sel_set(float* x, int col, float v) {
#pragma unroll
    for (int c = 0; c < N; ++c) x[c] = (c == col) ? v : x[c];
}
// tap one cell of a register row: counts the evaluation of (site, j, tap.col), flips on trigger
template <int N>
__device__ __forceinline__ void tap_row(ThreadTap& tap, const AttnParams& p, int site, int j, float* x) {
    if (tap.hit(site, j) && tap.col < N) sel_set<N>(x, tap.col, tap.fire(p, sel_get<N>(x, tap.col)));
}

__device__ __forceinline__ void atomic_max_nonneg(float* addr, float v) {
    if (!(v >= 0.0f)) return;
    if (isinf(v)) return;  // the reference's calibration ignores non-finite residuals
    atomicMax(reinterpret_cast<int*>(addr), __float_as_int(v));
}

__device__ __forceinline__ void push_event(const AttnParams& p, int kind, int head, int bi,
                                           int bj, int status, int row, int col, int violations,
                                           int corrections, int checksum_repair, double residual,
                                           double delta) {
    // reference FTReport::push_event (src/efta.cpp:49-55): only non-CLEAN
    // events are logged on the device; detections / corrections / failed
    // aggregate exactly like the reference's counters.
    efta_counters* c = p.counters;
    if (status != EFTA_CLEAN) atomicAdd(&c->detections, 1);
    if (corrections) atomicAdd(&c->corrections, corrections);
    if (status == EFTA_DETECTED_UNCORRECTABLE || status == EFTA_NONFINITE) atomicExch(&c->failed, 1);
    if (status == EFTA_CLEAN) return;
    const int slot = atomicAdd(&c->n_events, 1);
    if (slot >= p.ev_cap) return;
    efta_event& e = p.events[slot];
    e.kind = kind;
    e.head = head;
    e.block_i = bi;
    e.block_j = bj;
    e.status = status;
    e.row = row;
    e.col = col;
    e.violations = violations;
    e.corrections = corrections;
    e.checksum_repair = checksum_repair;
    e.residual = residual;
    e.delta = delta;
}

// ------------------------------------------------- strided verify of one row
// Row-local restatement of verify_locate_correct (src/abft.cpp:65-187) for
// the G = W/8 groups of one thread-owned row (no shuffles: the whole row and
// its 2x8 checksums live in this thread). Operates on a local array (only used
// on the slow path). The caller handles the tile-wide "checksum non-finite"
// early return (abft.cpp:74-78).
// The strided group check of one row against its checksums with the reference's double
// residuals (|c1 - s1| > eps or |c2 - s2| > eps * G flags the row; residual max(|d1|, |d2| / G)),
// behind an fp32 screen: when every difference is finite and below both thresholds by a 2^-12
// margin, the double test passes too, and the fp32 residual equals the double one rounded once
// (fsub is the correctly rounded exact difference, G a power of two), so a clean row skips the
// double arithmetic (measured ~1200-1700 clk per d=64 tile epilogue, on the max chain). Any other
// row runs the double path unchanged. FIN_ON_D: a non-finite sum is judged on the difference (the
// GEMM epilogue) rather than on the sums (attention); both flag the row.
template <int NG, int G, bool FIN_ON_D>
__device__ __forceinline__ void group_check(const float (&c1)[NG], const float (&c2)[NG], const float (&s1)[NG],
                                            const float (&s2)[NG], double eps, bool& viol, bool& cs_bad,
                                            double& res) {
    static_assert((G & (G - 1)) == 0, "G must be a power of two (exact residual scaling)");
    const float e1 = static_cast<float>(eps * (1.0 - 0x1p-12));
    const float e2 = static_cast<float>(eps * G * (1.0 - 0x1p-12));
    bool fast = true;
    float rf = 0.0f;
#pragma unroll
    for (int x = 0; x < NG; ++x) {
        const float a = fabsf(__fsub_rn(c1[x], s1[x])), b = fabsf(__fsub_rn(c2[x], s2[x]));
        fast = fast && a <= e1 && b <= e2;  // false for NaN / inf differences
        rf = fmaxf(rf, fmaxf(a, b * (1.0f / G)));
    }
    if (fast) {
        res = fmax(res, static_cast<double>(rf));
        return;
    }
#pragma unroll
    for (int x = 0; x < NG; ++x) {
        cs_bad |= !isfinite(c1[x]) || !isfinite(c2[x]);
        if (!FIN_ON_D && (!isfinite(s1[x]) || !isfinite(s2[x]))) { viol = true; continue; }
        const double d1 = static_cast<double>(c1[x]) - s1[x];
        const double d2 = static_cast<double>(c2[x]) - s2[x];
        if (FIN_ON_D && (!isfinite(d1) || !isfinite(d2))) { viol = true; continue; }
        res = fmax(res, fmax(fabs(d1), fabs(d2) / G));
        viol |= (fabs(d1) > eps) || (fabs(d2) > eps * G);
    }
}

struct RowVerify {
    int violations, corrections, checksum_repair, uncorrectable, nonfinite;
    int restored_col;      // last erasure-restored column (-1 none)
    double residual;
    double best_abs;       // largest |applied| correction (strict >, first wins)
    double best_delta;     // signed value of that correction
    int best_col;
};

template <int W>
__device__ __noinline__ void verify_row(float* t, const float* c1, const float* c2, double eps_row,
                                        RowVerify& rv) {
    constexpr int G = W / kStride;
    rv.violations = rv.corrections = rv.checksum_repair = rv.uncorrectable = rv.nonfinite = 0;
    rv.restored_col = -1;
    rv.residual = 0.0;
    rv.best_abs = 0.0;
    rv.best_delta = 0.0;
    rv.best_col = -1;
    bool any_nonfinite = false;
    for (int c = 0; c < W; ++c) any_nonfinite |= !isfinite(t[c]);
    if (any_nonfinite) {  // abft.cpp:83-111 erasure restore
        for (int j = 0; j < kStride; ++j) {
            int bad = -1, bad_count = 0;
            for (int l = 0; l < G; ++l)
                if (!isfinite(t[j + kStride * l])) { bad = l; ++bad_count; }
            if (bad_count == 0) continue;
            ++rv.violations;
            if (bad_count > 1) { rv.nonfinite = 1; rv.residual = CUDART_INF; return; }
            float rest = 0.0f;
            for (int l = 0; l < G; ++l)
                if (l != bad) rest = __fadd_rn(rest, t[j + kStride * l]);
            const int col = j + kStride * bad;
            t[col] = __fsub_rn(c1[j], rest);
            ++rv.corrections;
            rv.restored_col = col;
        }
    }
    for (int j = 0; j < kStride; ++j) {
        float a = 0.0f, b = 0.0f;
        for (int l = 0; l < G; ++l) {
            const float v = t[j + kStride * l];
            a = __fadd_rn(a, v);
            b = __fadd_rn(b, __fmul_rn(static_cast<float>(l + 1), v));
        }
        double s1d = a, s2d = b;
        if (!isfinite(s1d) || !isfinite(s2d)) {  // abft.cpp:120-131
            s1d = 0.0;
            s2d = 0.0;
            for (int l = 0; l < G; ++l) {
                const double vv = t[j + kStride * l];
                s1d += vv;
                s2d += (l + 1.0) * vv;
            }
        }
        const double d1 = static_cast<double>(c1[j]) - s1d;
        const double d2 = static_cast<double>(c2[j]) - s2d;
        rv.residual = fmax(rv.residual, fmax(fabs(d1), fabs(d2) / G));
        const bool v1 = fabs(d1) > eps_row;
        const bool v2 = fabs(d2) > eps_row * G;
        if (!v1 && !v2) continue;
        ++rv.violations;
        if (!v1) { rv.checksum_repair = 1; continue; }
        const double ratio = d2 / d1;
        const double nearest = round(ratio);
        if (nearest == 0.0 && fabs(ratio) <= 0.25) { rv.checksum_repair = 1; continue; }
        const int g = static_cast<int>(nearest) - 1;
        if (g < 0 || g >= G || fabs(ratio - nearest) > 0.25) {
            if (fmax(fabs(d1), fabs(d2) / G) > eps_row * 16.0) rv.uncorrectable = 1;
            continue;
        }
        const int col = j + kStride * g;
        float rest = 0.0f;
        for (int l = 0; l < G; ++l)
            if (l != g) rest = __fadd_rn(rest, t[j + kStride * l]);
        const float old_val = t[col];
        const float new_val = __fsub_rn(c1[j], rest);
        t[col] = new_val;
        ++rv.corrections;
        const double applied = static_cast<double>(new_val) - static_cast<double>(old_val);
        if (fabs(applied) > rv.best_abs) {
            rv.best_abs = fabs(applied);
            rv.best_delta = applied;
            rv.best_col = col;
        }
    }
}

// Tile-level aggregation of per-row RowVerify records into one reference
// VerificationReport (rows visited in order, abft.cpp:116-186). `red` is
// shared scratch: 128 x {best_abs(double), best_col, restored_col}.
struct TileReport {
    int status, row, col, violations, corrections, checksum_repair;
    double residual, delta;
};

struct RowSlot {
    double best_abs, best_delta;
    int best_col, restored_col;
};

// bo: barrier-id offset of the calling row warpgroup (0, or kBarAltOfs for the second
// warpgroup of the alternating schedule, efta_attn_alt.cuh)
__device__ __forceinline__ void wg_sync(uint32_t bo = 0) { named_bar_sync(1 + bo, 128); }

// All 128 row threads call this; returns the tile report on thread 0 (row 0).
static __device__ __noinline__ TileReport reduce_tile_report(const RowVerify& rv, bool tile_nonfinite,
                                                     int row, RowSlot* slots, int* ints,
                                                     double* dbl, uint32_t bo = 0) {
    // ints: [0] violations [1] corrections [2] checksum_repair [3] uncorrectable [4] nonfinite
    if (row == 0) {
        for (int i = 0; i < 5; ++i) ints[i] = 0;
        dbl[0] = 0.0;
    }
    wg_sync(bo);
    atomicAdd(&ints[0], rv.violations);
    atomicAdd(&ints[1], rv.corrections);
    if (rv.checksum_repair) atomicOr(&ints[2], 1);
    if (rv.uncorrectable) atomicOr(&ints[3], 1);
    if (rv.nonfinite) atomicOr(&ints[4], 1);
    slots[row].best_abs = rv.best_abs;
    slots[row].best_delta = rv.best_delta;
    slots[row].best_col = rv.best_col;
    slots[row].restored_col = rv.restored_col;
    // residual max through a CAS loop on doubles (rare path)
    {
        unsigned long long* a = reinterpret_cast<unsigned long long*>(&dbl[0]);
        unsigned long long old = *a, assumed;
        do {
            assumed = old;
            if (__longlong_as_double(assumed) >= rv.residual || isnan(rv.residual)) break;
            old = atomicCAS(a, assumed, __double_as_longlong(rv.residual));
        } while (old != assumed);
    }
    wg_sync(bo);
    TileReport tr{};
    if (row == 0) {
        tr.violations = ints[0];
        tr.corrections = ints[1];
        tr.checksum_repair = ints[2];
        tr.residual = dbl[0];
        tr.row = -1;
        tr.col = -1;
        tr.delta = 0.0;
        if (tile_nonfinite || ints[4]) {
            tr.status = EFTA_NONFINITE;
            tr.residual = CUDART_INF;
        } else {
            double best = 0.0, best_signed = 0.0;
            int last_restored_row = -1, last_restored_col = -1;
            for (int r = 0; r < 128; ++r) {
                if (slots[r].restored_col >= 0) {
                    last_restored_row = r;
                    last_restored_col = slots[r].restored_col;
                }
                if (slots[r].best_col >= 0 && slots[r].best_abs > best) {
                    best = slots[r].best_abs;
                    best_signed = slots[r].best_delta;
                    tr.row = r;
                    tr.col = slots[r].best_col;
                }
            }
            if (last_restored_row >= 0) {  // erasure restore sets delta = inf (abft.cpp:105-107)
                tr.row = last_restored_row;
                tr.col = last_restored_col;
                tr.delta = CUDART_INF;
            } else {
                tr.delta = best_signed;
            }
            if (ints[3]) tr.status = EFTA_DETECTED_UNCORRECTABLE;
            else if (tr.corrections > 0 || tr.checksum_repair) tr.status = EFTA_CORRECTED;
            else tr.status = EFTA_CLEAN;
        }
    }
    wg_sync(bo);
    return tr;
}

}  // namespace efta_sm100
