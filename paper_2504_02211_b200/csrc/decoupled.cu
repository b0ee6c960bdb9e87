// decoupled.cu — GPU decoupled fault-tolerant attention (the paper's comparison baseline).
//
// Replaces the reference's decoupled_ft_forward (src/decoupled.cpp:98-282): the attention
// pipeline split into three kernels that exchange full N x N intermediates through HBM,
// each protected on its own:
//   1. S = Q K^T with traditional two-sided checksums per 128 x 128 block
//      (with_check_rows / with_check_cols, decoupled.cpp:66-94; verify_two_sided :46-63),
//   2. P = softmax(S * scale) per row with duplicated evaluation (DMR) and the
//      rowsum-vs-1 check (:149-250),
//   3. O = P V with two-sided checksums per 128-row block (:254-279).
//
// B200 layout (per head, fp16 operands, fp32 accumulation on the tensor cores):
//   Q_aug, K_aug  [n*132, d]       every 128-row tile followed by its column checksums
//                                  s1 = sum_r T[r][c], s2 = sum_r (r+1) T[r][c] as hi/lo fp16
//                                  rows (s1_hi, s2_hi, s1_lo, s2_lo): the checksum operand then
//                                  carries ~22 mantissa bits (the reference's checksums are fp32)
//   S_aug         [n*132, n*132]   fp32 = Q_aug K_aug^T (one cuBLAS GEMM per head): block (i, j)
//                                  holds S_ij, its column checks (rows 128..131) and its row
//                                  checks (cols 128..131) — the reference's caug
//   P_aug         [n*132, N]       fp16 normalised P, per tile followed by its column checksums
//   V_aug         [N, d+8]         [V | s1_hi s2_hi s1_lo s2_lo | 0 0 0 0] (row checks of V)
//   (grouped-query attention: K_aug / V_aug are built per query head from its group's K / V)
//   O_aug         [n*132, d+8]     fp32 = P_aug V_aug
// The GEMMs are plain library GEMMs (cuBLAS, fp16 in / fp32 out): the decoupled design is
// "library GEMMs + separate checking kernels" by construction. The checking kernels
// (encode, block verification, DMR softmax) are hand-written below. S_aug and P_aug are the
// 4 N^2 intermediate traffic the fused kernel avoids (tests/acceptance.cpp:364-385).
#include <cublas_v2.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <string>

#include "efta_attn.cuh"

using namespace efta_sm100;

namespace {

constexpr int TB = 128;          // data rows / cols of a block (reference AttnConfig::block)
constexpr int TA = TB + 4;       // augmented tile: + s1_hi, s2_hi, s1_lo, s2_lo
constexpr double kNoiseBand = 16.0;  // kLocateNoiseBand (include/efta/abft.hpp:49)

struct DecParams {
    AttnParams p;    // eps, events, counters, faults, fired (flat head indices)
    int n, N, D, DP; // blocks, seq_len, head_dim, padded V_aug / O_aug width (D + 8)
    int head0;       // flat index of this chunk's first head
    int n_chunk;     // heads of this chunk
    long long s_ld;  // n * TA
    float* s_aug;    // [heads][n*TA][n*TA]
    __half* p_aug;   // [heads][n*TA][N]
    float* o_aug;    // [heads][n*TA][DP]
};

// -------------------------------------------------------------------- fault taps
// FaultInjector::tap (include/efta/fault.hpp:82-95) for the decoupled layout: a spec fires on
// its trigger-th evaluation of (site, block_i, block_j, row, col). Each value is evaluated by
// exactly one thread, which counts its own evaluations (eval = 1, 2, ... passed in).
__device__ __noinline__ float dec_tap(const AttnParams& p, int head, int site, int bi, int bj, int row, int col,
                                      int eval, float v) {
    for (int f = 0; f < p.n_faults; ++f) {
        const efta_fault_spec& s = p.faults[f];
        if (s.head != head || s.site != site || s.block_i != bi || s.block_j != bj || s.row != row ||
            s.col != col || s.trigger != eval)
            continue;
        const float flipped = __uint_as_float(__float_as_uint(v) ^ (1u << s.bit));
        const int slot = atomicAdd(&p.counters->n_fired, 1);
        if (slot < p.fired_cap) {
            p.fired[slot].spec = s;
            p.fired[slot].before = v;
            p.fired[slot].after = flipped;
        }
        return flipped;
    }
    return v;
}

// -------------------------------------------------------------------- encode
// Q_aug / K_aug tiles: data rows copied, column checksums in fp32 ascending row order
// (encode_traditional, src/abft.cpp:189-203; with_check_cols of K^T, decoupled.cpp:79-94, is the
// same sum over the key rows), split hi/lo. grid (n, heads, 2 = {Q, K}), 128 threads.
// K / V head of flat query head `head` (grouped-query attention; group 1 = itself)
__device__ __forceinline__ int dec_kv_head(int head, int heads_q, int group) {
    return group == 1 ? head : (head / heads_q) * (heads_q / group) + (head % heads_q) / group;
}

// q: this chunk's query heads; k: all K heads (row block of query head head0 + h's K/V head)
__global__ void __launch_bounds__(128) dec_encode_qk_kernel(const __half* __restrict__ q,
                                                            const __half* __restrict__ k,
                                                            __half* __restrict__ qa, __half* __restrict__ ka,
                                                            int N, int D, int n, int head0, int heads_q,
                                                            int group) {
    const int i = blockIdx.x, h = blockIdx.y;
    const int src_head = blockIdx.z ? dec_kv_head(head0 + h, heads_q, group) : h;
    const __half* src = (blockIdx.z ? k : q) + (static_cast<size_t>(src_head) * N + static_cast<size_t>(i) * TB) * D;
    __half* dst = (blockIdx.z ? ka : qa) + (static_cast<size_t>(h) * n + i) * TA * D;
    for (int idx = threadIdx.x; idx < TB * D / 8; idx += blockDim.x)
        reinterpret_cast<uint4*>(dst)[idx] = reinterpret_cast<const uint4*>(src)[idx];
    for (int c = threadIdx.x; c < D; c += blockDim.x) {
        float s1 = 0.0f, s2 = 0.0f;
        for (int r = 0; r < TB; ++r) {
            const float v = __half2float(src[static_cast<size_t>(r) * D + c]);
            s1 = __fadd_rn(s1, v);
            s2 = __fadd_rn(s2, __fmul_rn(static_cast<float>(r + 1), v));
        }
        const __half h1 = __float2half_rn(s1), h2 = __float2half_rn(s2);
        dst[(TB + 0) * D + c] = h1;
        dst[(TB + 1) * D + c] = h2;
        dst[(TB + 2) * D + c] = __float2half_rn(__fsub_rn(s1, __half2float(h1)));
        dst[(TB + 3) * D + c] = __float2half_rn(__fsub_rn(s2, __half2float(h2)));
    }
}

// V_aug rows: [V | row checksums hi/lo | 0] (with_check_cols(v), decoupled.cpp:79-94: s1 = sum_c V,
// s2 = sum_c (c+1) V in ascending column order). grid (n, heads), 128 threads = rows.
__global__ void __launch_bounds__(128) dec_encode_v_kernel(const __half* __restrict__ v, __half* __restrict__ va,
                                                           int N, int D, int DP, int head0, int heads_q, int group) {
    const int i = blockIdx.x, h = blockIdx.y;
    const size_t row = static_cast<size_t>(h) * N + static_cast<size_t>(i) * TB + threadIdx.x;
    const size_t src_row = static_cast<size_t>(dec_kv_head(head0 + h, heads_q, group)) * N +
                           static_cast<size_t>(i) * TB + threadIdx.x;
    const __half* src = v + src_row * D;
    __half* dst = va + row * DP;
    float s1 = 0.0f, s2 = 0.0f;
    for (int c = 0; c < D; c += 8) {
        const uint4 raw = *reinterpret_cast<const uint4*>(src + c);
        *reinterpret_cast<uint4*>(dst + c) = raw;
        const __half* hv = reinterpret_cast<const __half*>(&raw);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const float x = __half2float(hv[e]);
            s1 = __fadd_rn(s1, x);
            s2 = __fadd_rn(s2, __fmul_rn(static_cast<float>(c + e + 1), x));
        }
    }
    const __half h1 = __float2half_rn(s1), h2 = __float2half_rn(s2);
    __align__(16) __half tail[8] = {h1, h2, __float2half_rn(__fsub_rn(s1, __half2float(h1))),
                                    __float2half_rn(__fsub_rn(s2, __half2float(h2))),
                                    __float2half_rn(0.0f), __float2half_rn(0.0f), __float2half_rn(0.0f),
                                    __float2half_rn(0.0f)};
    *reinterpret_cast<uint4*>(dst + D) = *reinterpret_cast<const uint4*>(tail);
}

// -------------------------------------------------------------------- traditional verification
// verify_traditional (src/abft.cpp:205-320) on an m x ncols block held in memory with element
// (r, c) at base[r * si + c * sj] (si / sj swap for the transposed pass), one thread per column
// c < ncols (blockDim >= ncols). ck1 / ck2: the propagated column checks (shared memory). The
// per-column work is the reference's; the report fields combine across columns exactly as its
// sequential column loop would (counts summed, residual max, location of the largest applied
// repair with the first column winning ties, early NONFINITE exit after the first column with
// two non-finite cells).
struct VRep {
    int status, row, col, violations, corrections, checksum_repair;
    double residual, delta;
};

struct VScratch {  // shared scratch of one CTA
    int i[8];
    double d[4];
    unsigned long long u[2];
};

__device__ __forceinline__ bool finitef(float x) { return isfinite(x); }

__device__ void verify_trad(float* base, long long si, long long sj, int m, int ncols, const float* ck1,
                            const float* ck2, double eps, VRep& out, VScratch& sh) {
    const int c = threadIdx.x;
    const bool mine = c < ncols;
    if (threadIdx.x == 0) {
        sh.i[0] = 0; sh.i[1] = 0x7fffffff; sh.i[2] = 0; sh.i[3] = 0; sh.i[4] = 0; sh.i[5] = -1; sh.i[6] = 0;
        sh.i[7] = 0;
        sh.d[0] = 0.0;
        sh.u[0] = 0ull; sh.u[1] = ~0ull;
    }
    __syncthreads();
    // checksums not finite -> NONFINITE, residual inf (abft.cpp:210-214)
    if (mine && !(finitef(ck1[c]) && finitef(ck2[c]))) atomicOr(&sh.i[0], 1);
    __syncthreads();
    if (sh.i[0]) {
        out = VRep{EFTA_NONFINITE, -1, -1, 0, 0, 0, CUDART_INF, 0.0};
        __syncthreads();
        return;
    }
    // non-finite data cells: restore from the unit checksum (abft.cpp:221-245)
    int bad = -1, bad_count = 0;
    if (mine)
        for (int r = 0; r < m; ++r)
            if (!finitef(base[r * si + c * sj])) { bad = r; ++bad_count; }
    if (mine && bad_count > 1) atomicMin(&sh.i[1], c);  // first column with two bad cells
    __syncthreads();
    const int first_multi = sh.i[1];
    int viol = 0, corr = 0;
    bool restored = false;
    if (mine && bad_count == 1 && c < first_multi) {
        float rest = 0.0f;
        for (int r = 0; r < m; ++r)
            if (r != bad) rest = __fadd_rn(rest, base[r * si + c * sj]);
        base[bad * si + c * sj] = __fsub_rn(ck1[c], rest);
        ++viol;
        ++corr;
        restored = true;
        atomicMax(&sh.i[5], c);  // the last restored column reports row / col
    }
    if (mine && bad_count > 0 && c == first_multi) ++viol;
    __syncthreads();
    if (first_multi != 0x7fffffff) {
        // NONFINITE exit: counts of the columns the sequential loop visited
        atomicAdd(&sh.i[2], viol);
        atomicAdd(&sh.i[3], corr);
        __syncthreads();
        const int lc = sh.i[5];
        int lrow = -1;
        if (lc >= 0 && c == lc) sh.i[6] = bad;
        __syncthreads();
        if (lc >= 0) lrow = sh.i[6];
        out = VRep{EFTA_NONFINITE, lrow, lc, sh.i[2], sh.i[3], 0, CUDART_INF, lc >= 0 ? CUDART_INF : 0.0};
        __syncthreads();
        return;
    }
    const int restored_col = sh.i[5];
    if (restored && c == restored_col) sh.i[6] = bad;
    __syncthreads();
    const int restored_row = restored_col >= 0 ? sh.i[6] : -1;
    // main pass (abft.cpp:247-312)
    double residual = 0.0;
    bool uncorr = false, cs_rep = false;
    double applied = 0.0;
    int arow = -1;
    if (mine) {
        float s1 = 0.0f, s2 = 0.0f;
        for (int r = 0; r < m; ++r) {
            const float v = base[r * si + c * sj];
            s1 = __fadd_rn(s1, v);
            s2 = __fadd_rn(s2, __fmul_rn(static_cast<float>(r + 1), v));
        }
        double s1d = s1, s2d = s2;
        if (!isfinite(s1d) || !isfinite(s2d)) {
            s1d = 0.0;
            s2d = 0.0;
            for (int r = 0; r < m; ++r) {
                const double vv = base[r * si + c * sj];
                s1d += vv;
                s2d += (r + 1.0) * vv;
            }
        }
        const double d1 = static_cast<double>(ck1[c]) - s1d;
        const double d2 = static_cast<double>(ck2[c]) - s2d;
        residual = fmax(fabs(d1), fabs(d2) / m);
        const bool v1 = fabs(d1) > eps, v2 = fabs(d2) > eps * m;
        if (v1 || v2) {
            ++viol;
            if (!v1) {
                cs_rep = true;
            } else {
                const double ratio = d2 / d1;
                const double nr = round(ratio);  // std::round: halves away from zero
                if (nr == 0.0 && fabs(ratio) <= 0.25) {
                    cs_rep = true;
                } else {
                    const int row = static_cast<int>(nr) - 1;
                    if (row < 0 || row >= m || fabs(ratio - nr) > 0.25) {
                        if (fmax(fabs(d1), fabs(d2) / m) > eps * kNoiseBand) uncorr = true;
                    } else {
                        float rest = 0.0f;
                        for (int r = 0; r < m; ++r)
                            if (r != row) rest = __fadd_rn(rest, base[r * si + c * sj]);
                        const float old_val = base[row * si + c * sj];
                        const float new_val = __fsub_rn(ck1[c], rest);
                        base[row * si + c * sj] = new_val;
                        ++corr;
                        applied = static_cast<double>(new_val) - static_cast<double>(old_val);
                        arow = row;
                    }
                }
            }
        }
    }
    // combine: sums / any / max; the largest |applied| (first column on ties) unless a
    // non-finite restoration already set delta = inf
    atomicAdd(&sh.i[2], viol);
    atomicAdd(&sh.i[3], corr);
    if (uncorr) atomicOr(&sh.i[4], 1);
    if (cs_rep) atomicOr(&sh.i[7], 1);
    if (mine) {
        unsigned long long* a = reinterpret_cast<unsigned long long*>(&sh.d[0]);
        unsigned long long old = *a, assumed;
        do {
            assumed = old;
            if (__longlong_as_double(assumed) >= residual) break;
            old = atomicCAS(a, assumed, __double_as_longlong(residual));
        } while (old != assumed);
        if (arow >= 0 && applied != 0.0 && !isnan(applied)) {
            // key: |applied| bits (positive doubles order like their bits), then the lowest column
            const unsigned long long key = __double_as_longlong(fabs(applied));
            atomicMax(&sh.u[0], key);
        }
    }
    __syncthreads();
    const unsigned long long best = sh.u[0];
    if (mine && arow >= 0 && applied != 0.0 && !isnan(applied) && static_cast<unsigned long long>(__double_as_longlong(fabs(applied))) == best)
        atomicMin(&sh.u[1], static_cast<unsigned long long>(c));
    __syncthreads();
    VRep r{};
    r.violations = sh.i[2];
    r.corrections = sh.i[3];
    r.residual = sh.d[0];
    r.checksum_repair = sh.i[7];
    r.row = restored_row;
    r.col = restored_col >= 0 ? restored_col : -1;
    r.delta = restored_col >= 0 ? CUDART_INF : 0.0;
    if (restored_col < 0 && best != 0ull) {
        const int bc = static_cast<int>(sh.u[1]);
        if (c == bc) { sh.i[6] = arow; sh.d[1] = applied; }
        __syncthreads();
        r.row = sh.i[6];
        r.col = bc;
        r.delta = sh.d[1];
    }
    r.status = sh.i[4] ? EFTA_DETECTED_UNCORRECTABLE
                       : ((r.corrections > 0 || r.checksum_repair) ? EFTA_CORRECTED : EFTA_CLEAN);
    out = r;
    __syncthreads();
}

// verify_two_sided (decoupled.cpp:46-63) on a block held in shared memory cs[m][ncols]
// (row stride ncols): column pass; if that declares defeat, the row pass on the transposed
// block (into a copy), then the column pass again on the row-repaired copy.
__device__ void verify_two_sided(float* cs, float* cs2, int m, int ncols, const float* col1, const float* col2,
                                 const float* row1, const float* row2, double eps, VRep& rep, VScratch& sh) {
    verify_trad(cs, ncols, 1, m, ncols, col1, col2, eps, rep, sh);
    if (rep.status != EFTA_DETECTED_UNCORRECTABLE) return;
    for (int x = threadIdx.x; x < m * ncols; x += blockDim.x) cs2[x] = cs[x];
    __syncthreads();
    VRep rrep;
    verify_trad(cs2, 1, ncols, ncols, m, row1, row2, eps, rrep, sh);  // transpose: "columns" = rows
    if (rrep.corrections == 0) return;
    VRep again;
    verify_trad(cs2, ncols, 1, m, ncols, col1, col2, eps, again, sh);
    if (again.status == EFTA_CLEAN || again.status == EFTA_CORRECTED) {
        for (int x = threadIdx.x; x < m * ncols; x += blockDim.x) cs[x] = cs2[x];
        again.corrections += rep.corrections + rrep.corrections;
        again.violations = rep.violations;
        again.residual = rep.residual;
        again.status = EFTA_CORRECTED;
        rep = again;
    }
    __syncthreads();
}

// Kernel 1b / 3b (fast check): tap the product (GEMM1_OUT / GEMM2_ACC), run the column check
// of the block — the first stage of verify_traditional with the reference's exact row-order
// sums — and append the blocks that fail it to a list for the repair kernel (rare). No dynamic
// shared memory, so the check streams S_aug at full occupancy. grid (n, n, heads) for S,
// (n, heads) for O; 128 threads = columns.
__device__ __forceinline__ void col_checks(const float* blk, long long ld, int t, int ncols_chk, float* c1,
                                           float* c2) {
    *c1 = __fadd_rn(blk[(TB + 0) * ld + t], blk[(TB + 2) * ld + t]);
    *c2 = __fadd_rn(blk[(TB + 1) * ld + t], blk[(TB + 3) * ld + t]);
    (void)ncols_chk;
}
__device__ __forceinline__ bool column_ok(const float* blk, long long ld, int t, float c1, float c2, double eps) {
    float s1 = 0.0f, s2 = 0.0f;
    bool fin = true;
#pragma unroll 8
    for (int r = 0; r < TB; ++r) {
        const float v = blk[r * ld + t];
        fin = fin && finitef(v);
        s1 = __fadd_rn(s1, v);
        s2 = __fadd_rn(s2, __fmul_rn(static_cast<float>(r + 1), v));
    }
    const double d1 = static_cast<double>(c1) - s1, d2 = static_cast<double>(c2) - s2;
    return fin && finitef(c1) && finitef(c2) && isfinite(s1) && isfinite(s2) && !(fabs(d1) > eps) &&
           !(fabs(d2) > eps * TB);
}

template <bool TAPS>
__global__ void __launch_bounds__(128) dec_check_s_kernel(DecParams dp, int* list) {
    __shared__ int flag;
    const int j = blockIdx.x, i = blockIdx.y, hl = blockIdx.z, head = dp.head0 + hl;
    const int t = threadIdx.x;
    float* blk = dp.s_aug + static_cast<size_t>(hl) * dp.s_ld * dp.s_ld + static_cast<size_t>(i) * TA * dp.s_ld +
                 static_cast<size_t>(j) * TA;
    const long long ld = dp.s_ld;
    if (TAPS)
        for (int r = 0; r < TB; ++r) {
            float& x = blk[r * ld + t];
            const float y = dec_tap(dp.p, head, EFTA_GEMM1_OUT, i, j, r, t, 1, x);
            if (__float_as_uint(y) != __float_as_uint(x)) x = y;
        }
    if (t == 0) flag = 0;
    __syncthreads();
    float c1, c2;
    col_checks(blk, ld, t, TB, &c1, &c2);
    if (!column_ok(blk, ld, t, c1, c2, dp.p.eps_lin)) flag = 1;
    __syncthreads();
    if (t == 0 && flag) {
        const int slot = atomicAdd(&list[0], 1);
        list[2 + slot] = (hl * dp.n + i) * dp.n + j;
    }
}

template <bool TAPS>
__global__ void __launch_bounds__(128) dec_check_o_kernel(DecParams dp, float* __restrict__ o, int* list) {
    __shared__ int flag;
    const int i = blockIdx.x, hl = blockIdx.y, head = dp.head0 + hl;
    const int t = threadIdx.x, D = dp.D, DP = dp.DP;
    float* blk = dp.o_aug + (static_cast<size_t>(hl) * dp.s_ld + static_cast<size_t>(i) * TA) * DP;
    if (TAPS && t < D)
        for (int r = 0; r < TB; ++r) {
            float& x = blk[r * DP + t];
            const float y = dec_tap(dp.p, head, EFTA_GEMM2_ACC, i, 0, r, t, 1, x);
            if (__float_as_uint(y) != __float_as_uint(x)) x = y;
        }
    if (t == 0) flag = 0;
    __syncthreads();
    if (t < D) {
        float c1, c2;
        col_checks(blk, DP, t, D, &c1, &c2);
        if (!column_ok(blk, DP, t, c1, c2, dp.p.eps2)) flag = 1;
    }
    __syncthreads();
    if (flag) {
        if (t == 0) {
            const int slot = atomicAdd(&list[1], 1);
            list[2 + dp.n * dp.n * dp.n_chunk + slot] = hl * dp.n + i;
        }
        return;  // the repair kernel stores this block
    }
    float* dst = o + (static_cast<size_t>(hl) * dp.N + static_cast<size_t>(i) * TB) * D;
    for (int x = t; x < TB * D / 4; x += blockDim.x) {
        const int r = (4 * x) / D, c = (4 * x) % D;
        reinterpret_cast<float4*>(dst)[x] = *reinterpret_cast<const float4*>(blk + r * DP + c);
    }
}

// Repair kernels (rare): verify_two_sided on every listed block in shared memory, write the
// block back (S) or store it (O), log the event. A few persistent CTAs walk the list.
__global__ void __launch_bounds__(128) dec_repair_s_kernel(DecParams dp, const int* list) {
    extern __shared__ float smem_f[];
    __shared__ float ck[4][TB];
    __shared__ VScratch sh;
    const int t = threadIdx.x;
    const long long ld = dp.s_ld;
    const int cnt = list[0];
    for (int e = blockIdx.x; e < cnt; e += gridDim.x) {
        const int code = list[2 + e];
        const int j = code % dp.n, i = (code / dp.n) % dp.n, hl = code / (dp.n * dp.n), head = dp.head0 + hl;
        float* blk = dp.s_aug + static_cast<size_t>(hl) * ld * ld + static_cast<size_t>(i) * TA * ld +
                     static_cast<size_t>(j) * TA;
        ck[0][t] = __fadd_rn(blk[(TB + 0) * ld + t], blk[(TB + 2) * ld + t]);
        ck[1][t] = __fadd_rn(blk[(TB + 1) * ld + t], blk[(TB + 3) * ld + t]);
        ck[2][t] = __fadd_rn(blk[t * ld + TB + 0], blk[t * ld + TB + 2]);
        ck[3][t] = __fadd_rn(blk[t * ld + TB + 1], blk[t * ld + TB + 3]);
        float* cs = smem_f;
        float* cs2 = smem_f + TB * TB;
        for (int r = 0; r < TB; ++r) cs[r * TB + t] = blk[r * ld + t];
        __syncthreads();
        VRep rep;
        verify_two_sided(cs, cs2, TB, TB, ck[0], ck[1], ck[2], ck[3], dp.p.eps_lin, rep, sh);
        for (int r = 0; r < TB; ++r) blk[r * ld + t] = cs[r * TB + t];
        if (t == 0)
            push_event(dp.p, EFTA_BLOCK_CHECKSUM, head, i, j, rep.status, rep.row, rep.col, rep.violations,
                       rep.corrections, rep.checksum_repair, rep.residual, rep.delta);
        __syncthreads();
    }
}

__global__ void __launch_bounds__(128) dec_repair_o_kernel(DecParams dp, float* __restrict__ o, const int* list) {
    extern __shared__ float smem_f[];
    __shared__ float ck[4][TB];
    __shared__ VScratch sh;
    const int t = threadIdx.x, D = dp.D, DP = dp.DP;
    const int cnt = list[1];
    const int* ol = list + 2 + dp.n * dp.n * dp.n_chunk;
    for (int e = blockIdx.x; e < cnt; e += gridDim.x) {
        const int code = ol[e];
        const int i = code % dp.n, hl = code / dp.n, head = dp.head0 + hl;
        const float* blk = dp.o_aug + (static_cast<size_t>(hl) * dp.s_ld + static_cast<size_t>(i) * TA) * DP;
        if (t < D) {
            ck[0][t] = __fadd_rn(blk[(TB + 0) * DP + t], blk[(TB + 2) * DP + t]);
            ck[1][t] = __fadd_rn(blk[(TB + 1) * DP + t], blk[(TB + 3) * DP + t]);
        }
        ck[2][t] = __fadd_rn(blk[t * DP + D + 0], blk[t * DP + D + 2]);
        ck[3][t] = __fadd_rn(blk[t * DP + D + 1], blk[t * DP + D + 3]);
        float* cs = smem_f;
        float* cs2 = smem_f + TB * TB;
        for (int x = t; x < TB * D; x += blockDim.x) cs[x] = blk[(x / D) * DP + x % D];
        __syncthreads();
        VRep rep;
        verify_two_sided(cs, cs2, TB, D, ck[0], ck[1], ck[2], ck[3], dp.p.eps2, rep, sh);
        float* dst = o + (static_cast<size_t>(hl) * dp.N + static_cast<size_t>(i) * TB) * D;
        for (int x = t; x < TB * D; x += blockDim.x) dst[x] = cs[x];
        if (t == 0)
            push_event(dp.p, EFTA_BLOCK_CHECKSUM, head, i, dp.n, rep.status, rep.row, rep.col, rep.violations,
                       rep.corrections, rep.checksum_repair, rep.residual, rep.delta);
        __syncthreads();
    }
}

// -------------------------------------------------------------------- DMR softmax (kernel 2)
// One CTA per (head, 128-row tile); rows in order. Thread t owns the data columns
// gc = t + k * blockDim (coalesced row reads). Per row (decoupled.cpp:153-248):
//   m = rowmax(S) + bias [REDUCE_MAX]; e = exp(S - m) evaluated twice [SUB_MAX, EXP_OUT per
//   evaluation], max |e1 - e2| <= eps1 or a third evaluation arbitrates; p = (e1 + e2) / 2;
//   l = rowsum(p) [REDUCE_SUM]; up to three normalisations [NORMALIZE_OUT] until
//   |sum(p / l) - 1| <= eps1 * N. P is stored fp16 (the tensor-core operand of kernel 3) and the
//   tile's column checksums of that stored P accumulate in registers (with_check_rows(P_i)).

// CTA reductions with one __syncthreads each: consecutive reductions alternate between two
// scratch slots, so a slot is rewritten only after every thread passed the barrier of the
// reduction in between (and so has finished reading it).
template <int NT>
struct RowRed {
    float f[2][NT / 32 + 1];  // + one flag word
    double d[2][NT / 32];
};
// max of v; `flag` (thread 0's) rides along in the same barrier and is returned in *flag_out
template <int NT>
__device__ __forceinline__ float red_max(RowRed<NT>& R, int slot, float v, float flag, float* flag_out) {
    for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    float* b = R.f[slot & 1];
    if ((threadIdx.x & 31) == 0) b[threadIdx.x >> 5] = v;
    if (threadIdx.x == 0) b[NT / 32] = flag;
    __syncthreads();
    *flag_out = b[NT / 32];
    float r = b[0];
#pragma unroll
    for (int w = 1; w < NT / 32; ++w) r = fmaxf(r, b[w]);
    return r;
}
// (sum of a float, max of a double) in one pass
template <int NT>
__device__ __forceinline__ void red_sum_dmax(RowRed<NT>& R, int slot, float& s, double& m) {
    for (int o = 16; o; o >>= 1) {
        s += __shfl_xor_sync(0xffffffffu, s, o);
        m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    }
    float* bf = R.f[slot & 1];
    double* bd = R.d[slot & 1];
    if ((threadIdx.x & 31) == 0) { bf[threadIdx.x >> 5] = s; bd[threadIdx.x >> 5] = m; }
    __syncthreads();
    s = bf[0];
    m = bd[0];
#pragma unroll
    for (int w = 1; w < NT / 32; ++w) { s += bf[w]; m = fmax(m, bd[w]); }
}
template <int NT>
__device__ __forceinline__ double red_dsum(RowRed<NT>& R, int slot, double v) {
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    double* b = R.d[slot & 1];
    if ((threadIdx.x & 31) == 0) b[threadIdx.x >> 5] = v;
    __syncthreads();
    double r = b[0];
#pragma unroll
    for (int w = 1; w < NT / 32; ++w) r += b[w];
    return r;
}
__device__ __forceinline__ float opaque(float x) {
    float y;
    asm volatile("mov.b32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// exp(x) as ex2(x log2 e) on the MUFU (not flushing subnormal results, like std::exp)
__device__ __forceinline__ float dec_exp(float x) {
    float y;
    asm("ex2.approx.f32 %0, %1;" : "=f"(y) : "f"(__fmul_rn(x, kLog2e)));
    return y;
}

// 1D bulk copy global -> shared (TMA engine), completion on an mbarrier
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// TAPS: the fault-injection build (launched only when the call carries faults): the clean build
// has no tap code at all, which keeps the unrolled row loop small (instruction-cache bound
// otherwise).
// NT threads x VPT columns each == N exactly (NT = max(128, N/16), N a multiple of 128), so the
// column loops carry no bounds guards and thread t's columns sit at a fixed stride in S_aug.
template <int NT, int VPT, bool TAPS>
__global__ void __launch_bounds__(NT) dec_softmax_kernel(DecParams dp) {
    constexpr int kVpt = VPT;
    static_assert(NT % TB == 0, "a thread's columns keep their in-block offset");
    __shared__ RowRed<NT> R;
    __shared__ float bcast[2];
    // dynamic shared memory: the tile's column checksums of the stored P [2][N], then one or two
    // augmented S rows (the bulk-copy prefetch of row r+1 runs under row r's work)
    extern __shared__ __align__(16) float colsum[];
    __shared__ __align__(8) uint64_t rbar[2];
    const int i = blockIdx.x, hl = blockIdx.y, head = dp.head0 + hl;
    const int t = threadIdx.x, N = dp.N;
    const AttnParams& p = dp.p;
    const float* S = dp.s_aug + static_cast<size_t>(hl) * dp.s_ld * dp.s_ld;
    __half* P = dp.p_aug + static_cast<size_t>(hl) * dp.s_ld * N;
    float* cs1 = colsum;
    float* cs2 = colsum + N;
    float* rowbuf = colsum + 2 * N;  // [nbuf][s_ld]
    // one row buffer: the next row is fetched once the CTA is done with the current one; two
    // CTAs per SM (63 registers x 512 threads, < 114 KB shared each) hide each other's fetches
    // (A/B on C4 heads: a double-buffered prefetch with one CTA per SM was 1.3x slower)
    constexpr bool dbl = false;
    const uint32_t row_bytes = static_cast<uint32_t>(dp.s_ld * sizeof(float));
    for (int c = t; c < 2 * N; c += NT) colsum[c] = 0.0f;
    if (t == 0) {
        mbar_init(&rbar[0], 1);
        mbar_init(&rbar[1], 1);
        fence_barrier_init();
        mbar_arrive_expect_tx(&rbar[0], row_bytes);
        bulk_g2s(rowbuf, S + static_cast<size_t>(i * TA) * dp.s_ld, row_bytes, &rbar[0]);
    }
    __syncthreads();
    int k_red = 0;  // reduction counter (slot parity), uniform over the CTA
    const double rowsum_eps = p.eps1 * N;
    for (int r = 0; r < TB; ++r) {
        const int R_ = i * TB + r;
        const int rb = dbl ? (r & 1) : 0;
        const float* srow = rowbuf + rb * dp.s_ld;
        mbar_wait(&rbar[rb], dbl ? ((r >> 1) & 1) : (r & 1));
        auto load_x = [&](float* x) {
            const float* sp = srow + (t / TB) * TA + t % TB;  // column t; + NT columns = + NT/TB blocks
#pragma unroll
            for (int k = 0; k < kVpt; ++k) x[k] = __fmul_rn(sp[k * (NT / TB) * TA], p.scale);
        };
        float x[kVpt];
        load_x(x);
        float mx = -CUDART_INF_F;
        bool nan0 = false;
#pragma unroll
        for (int k = 0; k < kVpt; ++k) {
            mx = fmaxf(mx, x[k]);  // NaN-ignoring, like std::max(v, x) past column 0
            if (t + k * NT == 0 && isnan(x[k])) nan0 = true;
        }
        float nanf;
        float m = red_max<NT>(R, k_red++, mx, nan0 ? 1.0f : 0.0f, &nanf);
        // every thread has read row r - 1's buffer for the last time (incl. its rare path):
        // prefetch row r + 1 into it
        if (dbl && t == 0 && r + 1 < TB) {
            mbar_arrive_expect_tx(&rbar[(r + 1) & 1], row_bytes);
            bulk_g2s(rowbuf + ((r + 1) & 1) * dp.s_ld, S + static_cast<size_t>(i * TA + r + 1) * dp.s_ld, row_bytes,
                     &rbar[(r + 1) & 1]);
        }
        // column 0 NaN propagates through the reference's sequential std::max (thread 0 owns it)
        if (nanf != 0.0f) m = CUDART_NAN_F;
        m = __fadd_rn(m, p.rowmax_bias);
        if constexpr (TAPS) {
            if (t == 0) bcast[1] = dec_tap(p, head, EFTA_REDUCE_MAX, i, 0, r, 0, 1, m);
            __syncthreads();
            m = bcast[1];
        }
        // eval(): e = exp(S - m), each call a fresh evaluation (the opaque copy of m keeps the
        // compiler from merging the duplicated evaluations)
        auto eval = [&](const float* xs, float* e, int ev) {
            const float mo = opaque(m);
#pragma unroll
            for (int k = 0; k < kVpt; ++k) {
                const int gc = t + k * NT;
                float a = __fsub_rn(xs[k], mo);
                if (TAPS) a = dec_tap(p, head, EFTA_SUB_MAX, i, gc / TB, r, gc % TB, ev, a);
                float ee = dec_exp(a);
                if (TAPS) ee = dec_tap(p, head, EFTA_EXP_OUT, i, gc / TB, r, gc % TB, ev, ee);
                e[k] = ee;
            }
        };
        auto diff_of = [&](const float* a, const float* b) {
            // |a - b| in fp32 (exact for agreeing evaluations, Sterbenz); NaN differences are
            // ignored, as by std::max; widened to double for the row reduction
            float dm = 0.0f;
#pragma unroll
            for (int k = 0; k < kVpt; ++k) dm = fmaxf(dm, fabsf(__fsub_rn(a[k], b[k])));
            return static_cast<double>(dm);
        };
        float e1[kVpt], e2[kVpt];
        eval(x, e1, 1);
        eval(x, e2, 2);
        // p = (e1 + e2) / 2 and its row sum go with the agreement check in one reduction; the
        // rare third evaluation recomputes them
        auto mean_sum = [&]() {
            float ls = 0.0f;
#pragma unroll
            for (int k = 0; k < kVpt; ++k) ls = __fadd_rn(ls, __fmul_rn(0.5f, __fadd_rn(e1[k], e2[k])));
            return ls;
        };
        float ls = mean_sum();
        double diff = diff_of(e1, e2);
        float l = ls;
        red_sum_dmax<NT>(R, k_red++, l, diff);
        if (!(diff <= p.eps1)) {
            // third evaluation arbitrates (x is reloaded: the rare path keeps registers free)
            load_x(x);
#pragma unroll
            for (int k = 0; k < kVpt; ++k) e1[k] = e2[k];
            eval(x, e2, 3);
            ls = mean_sum();
            double diff23 = diff_of(e1, e2);
            l = ls;
            red_sum_dmax<NT>(R, k_red++, l, diff23);
            const bool bad = !(diff23 <= p.eps1);
            if (t == 0)
                push_event(p, EFTA_DMR_SOFTMAX, head, i, 0, bad ? EFTA_DETECTED_UNCORRECTABLE : EFTA_CORRECTED, r,
                           -1, 1, bad ? 0 : 1, 0, bad ? fmax(diff, diff23) : diff, 0.0);
        }
        float* pv = e1;
#pragma unroll
        for (int k = 0; k < kVpt; ++k) pv[k] = __fmul_rn(0.5f, __fadd_rn(e1[k], e2[k]));
        float* nv = e2;
        int sum_eval = 1;
        if constexpr (TAPS) {
            if (t == 0) bcast[1] = dec_tap(p, head, EFTA_REDUCE_SUM, i, 0, r, 0, sum_eval, l);
            __syncthreads();
            l = bcast[1];
        }
        bool ok = false;
        for (int attempt = 0; attempt < 3 && !ok; ++attempt) {
            if (attempt > 0) {
                float l2 = ls;
                double dummy = 0.0;
                red_sum_dmax<NT>(R, k_red++, l2, dummy);
                l = l2;
                if constexpr (TAPS) {
                    ++sum_eval;
                    if (t == 0) bcast[1] = dec_tap(p, head, EFTA_REDUCE_SUM, i, 0, r, 0, sum_eval, l);
                    __syncthreads();
                    l = bcast[1];
                }
            }
            float rsf = 0.0f;  // per-thread partial in fp32 (kVpt terms), the row sum in double
            const float rl = __frcp_rn(l);  // p / l within 1 ulp (one reciprocal per row)
#pragma unroll
            for (int k = 0; k < kVpt; ++k) {
                const int gc = t + k * NT;
                float v = __fmul_rn(pv[k], rl);
                if (TAPS) v = dec_tap(p, head, EFTA_NORMALIZE_OUT, i, gc / TB, r, gc % TB, attempt + 1, v);
                nv[k] = v;
                rsf = __fadd_rn(rsf, nv[k]);
            }
            const double rs = red_dsum<NT>(R, k_red++, static_cast<double>(rsf));
            const double dev = fabs(rs - 1.0);
            ok = isfinite(rs) && dev <= rowsum_eps;
            if (!ok && t == 0) {
                atomicAdd(&p.counters->recomputes, 1);
                push_event(p, EFTA_DMR_SOFTMAX, head, i, 0, attempt < 2 ? EFTA_CORRECTED : EFTA_DETECTED_UNCORRECTABLE,
                           r, -1, 1, attempt < 2 ? 1 : 0, 0, dev / N, 0.0);
            }
        }
        __half* prow = P + static_cast<size_t>(i * TA + r) * N;
        const float wr = static_cast<float>(r + 1);
#pragma unroll
        for (int k = 0; k < kVpt; ++k) {
            const int gc = t + k * NT;
            const __half hv = __float2half_rn(nv[k]);
            prow[gc] = hv;
            const float f = __half2float(hv);
            cs1[gc] = __fadd_rn(cs1[gc], f);
            cs2[gc] = __fadd_rn(cs2[gc], __fmul_rn(wr, f));
        }
        if (t == 0) {
            if (p.m_out) p.m_out[static_cast<size_t>(hl) * N + R_] = m;
            if (p.l_out) p.l_out[static_cast<size_t>(hl) * N + R_] = l;
        }
        if (!dbl && r + 1 < TB) {  // single buffer: the next row lands once everyone is done
            __syncthreads();
            if (t == 0) {
                mbar_arrive_expect_tx(&rbar[0], row_bytes);
                bulk_g2s(rowbuf, S + static_cast<size_t>(i * TA + r + 1) * dp.s_ld, row_bytes, &rbar[0]);
            }
        }
    }
    __syncthreads();
    for (int gc = t; gc < N; gc += NT) {
        const float a = cs1[gc], b = cs2[gc];
        const __half h1 = __float2half_rn(a), h2 = __float2half_rn(b);
        P[static_cast<size_t>(i * TA + TB + 0) * N + gc] = h1;
        P[static_cast<size_t>(i * TA + TB + 1) * N + gc] = h2;
        P[static_cast<size_t>(i * TA + TB + 2) * N + gc] = __float2half_rn(__fsub_rn(a, __half2float(h1)));
        P[static_cast<size_t>(i * TA + TB + 3) * N + gc] = __float2half_rn(__fsub_rn(b, __half2float(h2)));
    }
}

}  // namespace

// the DMR softmax instantiation for a sequence length: NT = max(128, N/16), VPT = N / NT
template <bool TAPS>
static void launch_softmax_t(int N, dim3 grid, size_t smem, cudaStream_t st, const DecParams& dp) {
    switch (N <= 2048 ? N / 128 : N / 16) {
        case 1: dec_softmax_kernel<128, 1, TAPS><<<grid, 128, smem, st>>>(dp); break;
        case 2: dec_softmax_kernel<128, 2, TAPS><<<grid, 128, smem, st>>>(dp); break;
        case 4: dec_softmax_kernel<128, 4, TAPS><<<grid, 128, smem, st>>>(dp); break;
        case 8: dec_softmax_kernel<128, 8, TAPS><<<grid, 128, smem, st>>>(dp); break;
        case 16: dec_softmax_kernel<128, 16, TAPS><<<grid, 128, smem, st>>>(dp); break;
        case 256: dec_softmax_kernel<256, 16, TAPS><<<grid, 256, smem, st>>>(dp); break;
        case 512: dec_softmax_kernel<512, 16, TAPS><<<grid, 512, smem, st>>>(dp); break;
        case 1024: dec_softmax_kernel<1024, 16, TAPS><<<grid, 1024, smem, st>>>(dp); break;
        default: break;  // rejected by the host (power-of-two multiples of 128 up to 16384)
    }
}
static void launch_softmax(bool taps, int N, dim3 grid, size_t smem, cudaStream_t st, const DecParams& dp) {
    if (taps) launch_softmax_t<true>(N, grid, smem, st, dp);
    else launch_softmax_t<false>(N, grid, smem, st, dp);
}
template <bool TAPS>
static void softmax_attrs_t(int smem) {
    auto attr = [&](const void* fn) { cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); };
    attr(reinterpret_cast<const void*>(dec_softmax_kernel<128, 1, TAPS>));
    attr(reinterpret_cast<const void*>(dec_softmax_kernel<128, 2, TAPS>));
    attr(reinterpret_cast<const void*>(dec_softmax_kernel<128, 4, TAPS>));
    attr(reinterpret_cast<const void*>(dec_softmax_kernel<128, 8, TAPS>));
    attr(reinterpret_cast<const void*>(dec_softmax_kernel<128, 16, TAPS>));
    attr(reinterpret_cast<const void*>(dec_softmax_kernel<256, 16, TAPS>));
    attr(reinterpret_cast<const void*>(dec_softmax_kernel<512, 16, TAPS>));
    attr(reinterpret_cast<const void*>(dec_softmax_kernel<1024, 16, TAPS>));
}
static void softmax_attrs(int smem) {
    softmax_attrs_t<false>(smem);
    softmax_attrs_t<true>(smem);
}

// -------------------------------------------------------------------- host orchestration
namespace efta_dec {

// per-head workspace of the decoupled pipeline (bytes, 256-aligned pieces)
static size_t al256(size_t x) { return (x + 255) & ~size_t(255); }
struct DecLayout {
    size_t qa, ka, va, s, pa, oa, fl, per_head;
};
static DecLayout layout_for(int N, int D) {
    const size_t n = N / TB, ld = n * TA, DP = D + 8;
    DecLayout L;
    L.qa = al256(ld * D * 2);
    L.ka = al256(ld * D * 2);
    L.va = al256(static_cast<size_t>(N) * DP * 2);
    L.s = al256(ld * ld * 4);
    L.pa = al256(ld * N * 2);
    L.oa = al256(ld * DP * 4);
    L.fl = al256((n * n + n) * 4);  // repair lists (S blocks, O blocks)
    L.per_head = L.qa + L.ka + L.va + L.s + L.pa + L.oa + L.fl;
    return L;
}
// intermediates of one chunk of heads: 4 GB (EFTA_DECOUPLED_CHUNK_MB overrides, read per call)
static size_t chunk_budget() {
    const char* e = std::getenv("EFTA_DECOUPLED_CHUNK_MB");
    const long long mb = e ? std::atoll(e) : 0;
    return mb > 0 ? static_cast<size_t>(mb) << 20 : size_t(4) << 30;
}

int chunk_heads(int bh, int N, int D) {
    const size_t per = layout_for(N, D).per_head;
    size_t c = chunk_budget() / per;
    if (c < 1) c = 1;
    return static_cast<int>(c < static_cast<size_t>(bh) ? c : bh);
}
size_t workspace_bytes(int bh, int N, int D) {
    return static_cast<size_t>(chunk_heads(bh, N, D)) * layout_for(N, D).per_head + 512;
}

struct Handle {
    cublasHandle_t h = nullptr;
    ~Handle() { if (h) cublasDestroy(h); }
};

// One chunk-by-chunk decoupled forward. Returns a cudaError_t / cuBLAS failure as a string.
std::string forward(const AttnParams& base, int bh, int N, int D, const __half* q, const __half* k,
                    const __half* v, float* o, void* ws, cudaStream_t st) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) return "device index out of range";
    thread_local Handle handles[64];
    Handle& hd = handles[dev];
    if (!hd.h && cublasCreate(&hd.h) != CUBLAS_STATUS_SUCCESS) return "cublasCreate failed";
    if (cublasSetStream(hd.h, st) != CUBLAS_STATUS_SUCCESS) return "cublasSetStream failed";
    const int n = N / TB, DP = D + 8;
    const long long ld = static_cast<long long>(n) * TA;
    const DecLayout L = layout_for(N, D);
    const int chunk = chunk_heads(bh, N, D);
    char* w = static_cast<char*>(ws);
    __half* qa = reinterpret_cast<__half*>(w);
    __half* ka = reinterpret_cast<__half*>(w + chunk * L.qa);
    __half* va = reinterpret_cast<__half*>(w + chunk * (L.qa + L.ka));
    float* sa = reinterpret_cast<float*>(w + chunk * (L.qa + L.ka + L.va));
    __half* pa = reinterpret_cast<__half*>(w + chunk * (L.qa + L.ka + L.va + L.s));
    float* oa = reinterpret_cast<float*>(w + chunk * (L.qa + L.ka + L.va + L.s + L.pa));
    int* list = reinterpret_cast<int*>(w + chunk * (L.qa + L.ka + L.va + L.s + L.pa + L.oa));  // [2 + n*n*chunk + n*chunk]
    const float one = 1.0f, zero = 0.0f;
    const size_t vsmem = 2 * TB * TB * sizeof(float);
    cudaFuncSetAttribute(dec_repair_s_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(vsmem));
    cudaFuncSetAttribute(dec_repair_o_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(vsmem));
    const size_t csmax_b = (2 * static_cast<size_t>(N) + static_cast<size_t>(ld)) * sizeof(float);
    if (csmax_b > 227 * 1024 || N > 16384 || (N & (N - 1)) != 0)
        return "decoupled: seq_len must be a power of two multiple of 128, <= 16384 (DMR softmax tile)";
    const int csmax = static_cast<int>(csmax_b);
    softmax_attrs(csmax);
    for (int h0 = 0; h0 < bh; h0 += chunk) {
        const int nh = bh - h0 < chunk ? bh - h0 : chunk;
        const size_t e0 = static_cast<size_t>(h0) * N * D;
        DecParams dp;
        dp.p = base;
        dp.p.m_out = base.m_out ? base.m_out + static_cast<size_t>(h0) * N : nullptr;
        dp.p.l_out = base.l_out ? base.l_out + static_cast<size_t>(h0) * N : nullptr;
        dp.n = n; dp.N = N; dp.D = D; dp.DP = DP; dp.head0 = h0; dp.n_chunk = nh; dp.s_ld = ld;
        if (cudaMemsetAsync(list, 0, 2 * sizeof(int), st) != cudaSuccess) return "decoupled: memset failed";
        const bool taps = dp.p.n_faults > 0;
        dp.s_aug = sa; dp.p_aug = pa; dp.o_aug = oa;
        // kernel 0: checksum-augmented operands
        dec_encode_qk_kernel<<<dim3(n, nh, 2), 128, 0, st>>>(q + e0, k, qa, ka, N, D, n, h0, base.heads_q,
                                                             base.kv_group);
        dec_encode_v_kernel<<<dim3(n, nh), 128, 0, st>>>(v, va, N, D, DP, h0, base.heads_q, base.kv_group);
        // kernel 1: S_aug = Q_aug K_aug^T (row-major; column-major view: S^T = K_aug . Q_aug^T)
        cublasStatus_t cs = cublasGemmStridedBatchedEx(
            hd.h, CUBLAS_OP_T, CUBLAS_OP_N, static_cast<int>(ld), static_cast<int>(ld), D, &one, ka, CUDA_R_16F, D,
            ld * D, qa, CUDA_R_16F, D, ld * D, &zero, sa, CUDA_R_32F, static_cast<int>(ld), ld * ld, nh,
            CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT);
        if (cs != CUBLAS_STATUS_SUCCESS) return "cublas GEMM I failed: " + std::to_string(static_cast<int>(cs));
        if (taps) dec_check_s_kernel<true><<<dim3(n, n, nh), 128, 0, st>>>(dp, list);
        else dec_check_s_kernel<false><<<dim3(n, n, nh), 128, 0, st>>>(dp, list);
        dec_repair_s_kernel<<<32, 128, vsmem, st>>>(dp, list);
        // kernel 2: DMR softmax -> P_aug
        const size_t csm = (2 * static_cast<size_t>(N) + static_cast<size_t>(ld)) * sizeof(float);
        launch_softmax(taps, N, dim3(n, nh), csm, st, dp);
        // kernel 3: O_aug = P_aug V_aug (column-major view: O^T = V_aug^T . P_aug^T)
        cs = cublasGemmStridedBatchedEx(hd.h, CUBLAS_OP_N, CUBLAS_OP_N, DP, static_cast<int>(ld), N, &one, va,
                                        CUDA_R_16F, DP, static_cast<long long>(N) * DP, pa, CUDA_R_16F, N, ld * N,
                                        &zero, oa, CUDA_R_32F, DP, ld * DP, nh, CUBLAS_COMPUTE_32F,
                                        CUBLAS_GEMM_DEFAULT);
        if (cs != CUBLAS_STATUS_SUCCESS) return "cublas GEMM II failed: " + std::to_string(static_cast<int>(cs));
        if (taps) dec_check_o_kernel<true><<<dim3(n, nh), 128, 0, st>>>(dp, o + e0, list);
        else dec_check_o_kernel<false><<<dim3(n, nh), 128, 0, st>>>(dp, o + e0, list);
        dec_repair_o_kernel<<<32, 128, vsmem, st>>>(dp, o + e0, list);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return std::string("decoupled launch: ") + cudaGetErrorString(e);
    }
    return std::string();
}

}  // namespace efta_dec
