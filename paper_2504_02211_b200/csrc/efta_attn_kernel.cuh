// efta_attn_kernel.cuh — the kernel body (see efta_attn.cuh for the design notes).
#pragma once
#include "efta_attn.cuh"

namespace efta_sm100 {

// Shared scratch used by the row warpgroup for rare-path tile reductions.
struct RowScratch {
    RowSlot* slots;  // [128]
    int* ints;       // [16]
    double* dbl;     // [4]
};

// ----------------------------------------------------------------------------
// Exp-stage recovery ladder + factor guard for one (i, j) tile. Executed by all
// 128 row threads whenever any row of the tile flagged the exp-domain product
// check or the rescale-factor range guard. Mirrors verify_exp_stage
// (src/snvr.cpp:43-159) followed by the factor guard (src/efta.cpp:192-230).
// Inputs come from the fast path: the current P row (p_loc, possibly faulted),
// the row max state; S and its checksums are re-read from TMEM (still resident:
// P is written over S only after this returns).
// ----------------------------------------------------------------------------
// c2 of the score tile for one row on the CUDA cores: scale * (Q_row . KC2_j) with
// KC2 = c2_hi + c2_lo (rows 8..15 / 24..31 of the block's checksum rows), fp32 in
// ascending k. Used by the pair kernel, whose score MMA carries only c1 (N = 144).
template <int D>
__device__ __noinline__ void pair_score_c2(const AttnParams& p, int head, int bi, int j, int row,
                                           float (&c2s)[kStride]) {
    const __half* qr = p.q + (static_cast<size_t>(head) * p.seq_len + static_cast<size_t>(bi) * kBlock + row) * D;
    const __half* kc = p.kc + (static_cast<size_t>(kv_head(p, head)) * p.nblk + j) * 32 * D;
    for (int x = 0; x < kStride; ++x) {
        float acc = 0.0f;
        for (int k = 0; k < D; ++k) {
            const float w = __half2float(kc[(8 + x) * D + k]) + __half2float(kc[(24 + x) * D + k]);
            acc = fmaf(__half2float(qr[k]), w, acc);
        }
        c2s[x] = __fmul_rn(acc, p.scale);
    }
}

// PAIR: the pair kernel's score-checksum layout (16 cols: c1_hi 0..7, c1_lo 8..15;
// c2 recomputed by pair_score_c2)
template <bool DBG, int D, bool PAIR>
__device__ __noinline__ void exp_stage_slow(const AttnParams& p, uint32_t s_addr, uint32_t cs_addr,
                                            int head, int bi, int j, int row, bool exp_affected,
                                            float exp_first_residual, int exp_first_viol,
                                            float m_old, float& m_new, float& bm_hist,
                                            float* p_loc, int& replaced, ThreadTap& tap,
                                            int sc_fault_col, float sc_fault_val,
                                            const RowScratch& rs, uint32_t bo = 0, int mask_from = kBlock) {
    // mask_from < kBlock (pair kernel, causal): key columns >= mask_from of this row are masked:
    // P = 0 there, and the group checks run on the visible cells (c1 minus the masked scores)
    float sc[kBlock], raw[kBlock];
    float c1s[kStride], c2s[kStride];
    {
        uint32_t r[32];
#pragma unroll
        for (int c4 = 0; c4 < 4; ++c4) {
            tmem_ld32(s_addr + c4 * 32, r);
            tmem_wait_ld();
#pragma unroll
            for (int x = 0; x < 32; ++x) {
                raw[c4 * 32 + x] = __uint_as_float(r[x]);
                sc[c4 * 32 + x] = __fmul_rn(__uint_as_float(r[x]), p.scale);
            }
        }
        if constexpr (PAIR) {
            uint32_t q[16];
            tmem_ld16(cs_addr, q);
            tmem_wait_ld();
#pragma unroll
            for (int x = 0; x < kStride; ++x)
                c1s[x] = __fmul_rn(__fadd_rn(__uint_as_float(q[x]), __uint_as_float(q[kStride + x])), p.scale);
            pair_score_c2<D>(p, head, bi, j, row, c2s);
        } else {
            uint32_t qh[16], ql[16];
            tmem_ld16(cs_addr, qh);
            tmem_ld16(cs_addr + 16, ql);
            tmem_wait_ld();
#pragma unroll
            for (int x = 0; x < kStride; ++x) {
                c1s[x] = __fmul_rn(__fadd_rn(__uint_as_float(qh[x]), __uint_as_float(ql[x])), p.scale);
                c2s[x] = __fmul_rn(__fadd_rn(__uint_as_float(qh[kStride + x]), __uint_as_float(ql[kStride + x])),
                                   p.scale);
            }
        }
    }
    if (DBG && sc_fault_col >= 0) sc[sc_fault_col] = sc_fault_val;  // GEMM1_OUT upset lives in sc
    const float scale_log2 = p.scale_log2;
    replaced = 0;

    // ---------------- exp stage (only if some row failed the product check)
    const bool any_exp = named_bar_or(2 + bo, 128, exp_affected);
    if (any_exp) {
        // (1) linear repair of the score tile (snvr.cpp:89-98)
        bool cs_bad = false;
#pragma unroll
        for (int x = 0; x < kStride; ++x) cs_bad |= !isfinite(c1s[x]) || !isfinite(c2s[x]);
        const bool tile_cs_bad = named_bar_or(2 + bo, 128, cs_bad);
        RowVerify lin{};
        lin.best_col = -1;
        lin.restored_col = -1;
        if (!tile_cs_bad) verify_row<kBlock>(sc, c1s, c2s, p.eps_lin, lin);
        TileReport lt = reduce_tile_report(lin, tile_cs_bad, row, rs.slots, rs.ints, rs.dbl, bo);
        // broadcast lin.row / corrections / status
        if (row == 0) {
            rs.ints[8] = lt.row;
            rs.ints[9] = lt.corrections;
            rs.ints[10] = lt.status;
            rs.ints[11] = lt.col;
            rs.ints[12] = 0x7fffffff;  // first recomputed-and-changed row
            rs.ints[13] = 0;           // any row changed
            rs.ints[14] = 0;           // sum of recompute corrections
            rs.dbl[1] = lt.delta;
            rs.dbl[2] = 0.0;           // re-scan residual
        }
        wg_sync(bo);
        const int lin_row = rs.ints[9] > 0 ? rs.ints[8] : -1;
        const int lin_status = rs.ints[10];
        const bool affected = exp_affected || (row == lin_row);

        // (2) recompute affected rows from held state (snvr.cpp:102-139)
        int changed = 0;
        bool still_bad = false;
        float rescan_res = 0.0f;
        // visible part of each group (causal): the masked scores leave c1, n_vis cells remain
        float c1v[kStride], nvis[kStride];
        for (int x = 0; x < kStride; ++x) {
            float cm = 0.0f;
            int nv = 0;
            for (int l = 0; l < kBlock / kStride; ++l) {
                if (x + kStride * l >= mask_from) cm = __fadd_rn(cm, sc[x + kStride * l]);
                else ++nv;
            }
            c1v[x] = mask_from < kBlock ? __fsub_rn(c1s[x], cm) : c1s[x];
            nvis[x] = static_cast<float>(nv);
        }
        if (affected) {
            const float before_m = m_new;
            float bm = mask_from > 0 ? sc[0] : -CUDART_INF_F;
            for (int c = 1; c < mask_from; ++c) bm = (bm < sc[c]) ? sc[c] : bm;  // row_max, no bias
            float mm = (m_old < bm) ? bm : m_old;
            if (DBG) mm = tap(p, EFTA_REDUCE_MAX, j, 0, mm);
            m_new = mm;
            bm_hist = bm;
            const float mL = mm * kLog2e;
            for (int c = 0; c < kBlock; ++c) {
                float e;
                if (DBG) {
                    float a = __fsub_rn(sc[c], mm);
                    a = tap(p, EFTA_SUB_MAX, j, c, a);
                    e = ex2_approx(a * kLog2e);
                    e = tap(p, EFTA_EXP_OUT, j, c, e);
                } else {
                    // same formula as the fast path so untouched cells reproduce their bits;
                    // a linearly repaired cell only exists in the scaled domain
                    e = (__fmul_rn(raw[c], p.scale) == sc[c])
                            ? ex2_col<D>(c, fmaf(raw[c], scale_log2, -mL))
                            : ex2_approx(__fsub_rn(sc[c], mm) * kLog2e);
                }
                if (c >= mask_from) e = 0.0f;
                if (__float_as_uint(e) != __float_as_uint(p_loc[c])) changed = 1;
                p_loc[c] = e;
            }
            for (int x = 0; x < kStride; ++x) {
                const float pc_new = ex2_approx(__fsub_rn(c1v[x], nvis[x] * mm) * kLog2e);
                const float pc_old = ex2_approx(__fsub_rn(c1v[x], nvis[x] * before_m) * kLog2e);
                if (__float_as_uint(pc_new) != __float_as_uint(pc_old)) changed = 1;
            }
            replaced = 1;
            // (3) re-scan this row (snvr.cpp:141-157)
            still_bad = !isfinite(mm);
            for (int x = 0; x < kStride && !still_bad; ++x) {
                float prod = 1.0f;
                for (int l = 0; l < kBlock / kStride; ++l)
                    if (x + kStride * l < mask_from) prod = __fmul_rn(prod, p_loc[x + kStride * l]);
                const float pc1 = ex2_approx(__fsub_rn(c1v[x], nvis[x] * mm) * kLog2e);
                if (!(prod > 0.0f && prod < CUDART_INF_F) || !(pc1 > 0.0f && pc1 < CUDART_INF_F)) {
                    still_bad = true;
                    rescan_res = CUDART_INF_F;
                } else {
                    const float d = fabsf(lg2_approx(__fdividef(prod, pc1))) * kLn2;
                    rescan_res = fmaxf(rescan_res, d);
                    if (d > p.eps1) still_bad = true;
                }
            }
            if (changed) {
                atomicMin(&rs.ints[12], row);
                atomicOr(&rs.ints[13], 1);
                atomicAdd(&rs.ints[14], 1);
            }
        }
        const bool any_bad = named_bar_or(3 + bo, 128, still_bad);
        // tile residual / violations of the first look
        if (row == 0) { rs.ints[15] = 0; rs.dbl[3] = 0.0; }
        wg_sync(bo);
        atomicAdd(&rs.ints[15], exp_first_viol);
        {
            unsigned long long* a = reinterpret_cast<unsigned long long*>(&rs.dbl[3]);
            const double v = static_cast<double>(fmaxf(exp_first_residual, any_bad ? rescan_res : 0.0f));
            unsigned long long old = *a, assumed;
            do {
                assumed = old;
                if (__longlong_as_double(assumed) >= v) break;
                old = atomicCAS(a, assumed, __double_as_longlong(v));
            } while (old != assumed);
        }
        wg_sync(bo);
        if (row == 0) {
            const int corrections = rs.ints[9] + rs.ints[14];
            int status;
            if (any_bad || lin_status == EFTA_DETECTED_UNCORRECTABLE) status = EFTA_DETECTED_UNCORRECTABLE;
            else if (corrections > 0) status = EFTA_CORRECTED;
            else status = EFTA_CLEAN;
            int erow = rs.ints[9] > 0 ? rs.ints[8] : -1;
            int ecol = rs.ints[9] > 0 ? rs.ints[11] : -1;
            if (erow < 0 && rs.ints[13]) erow = rs.ints[12];
            if (rs.ints[13]) atomicAdd(&p.counters->recomputes, 1);
            push_event(p, EFTA_EXP_CHECKSUM, head, bi, j, status, erow, ecol, rs.ints[15], corrections,
                       0, rs.dbl[3], rs.ints[9] > 0 ? rs.dbl[1] : 0.0);
        }
        wg_sync(bo);
    }

    // ---------------- rescale-factor guard (efta.cpp:192-230), per row
    if (j > 0) {
        float f = ex2_approx((m_old - m_new) * kLog2e);
        if (!(isfinite(f) && f > 0.0f && f <= 1.0f)) {
            const double residual = isfinite(f) ? static_cast<double>(f) - 1.0 : CUDART_INF;
            float bm = sc[0];
            for (int c = 1; c < kBlock; ++c) bm = (bm < sc[c]) ? sc[c] : bm;
            bm = bm + p.rowmax_bias;
            bm_hist = bm;
            float mm = (m_old < bm) ? bm : m_old;
            if (DBG) mm = tap(p, EFTA_REDUCE_MAX, j, 0, mm);
            m_new = mm;
            const float mL = mm * kLog2e;
            for (int c = 0; c < kBlock; ++c) {
                float e;
                if (DBG) {
                    float a = __fsub_rn(sc[c], mm);
                    a = tap(p, EFTA_SUB_MAX, j, c, a);
                    e = ex2_approx(a * kLog2e);
                    e = tap(p, EFTA_EXP_OUT, j, c, e);
                } else {
                    e = (__fmul_rn(raw[c], p.scale) == sc[c])
                            ? ex2_col<D>(c, fmaf(raw[c], scale_log2, -mL))
                            : ex2_approx(__fsub_rn(sc[c], mm) * kLog2e);
                }
                p_loc[c] = e;
            }
            replaced = 1;
            f = ex2_approx((m_old - m_new) * kLog2e);
            atomicAdd(&p.counters->recomputes, 1);
            const bool ok = isfinite(f) && f > 0.0f && f <= 1.0f;
            push_event(p, EFTA_FACTOR_RANGE, head, bi, j,
                       ok ? EFTA_CORRECTED : EFTA_DETECTED_UNCORRECTABLE, row, -1, 0, ok ? 1 : 0, 0,
                       residual, 0.0);
        }
    }
}

// ----------------------------------------------------------------------------
// Output-tile strided verification (verify_locate_correct on O, abft.cpp:65-187)
// run by all 128 row threads. Fast path: per-row sums in registers; only if
// some row (or a checksum) looks wrong does the tile take the slow path.
// Returns with `o` corrected in place.
// ----------------------------------------------------------------------------
template <int D>
__device__ __forceinline__ void row_sums(const float (&o)[D], float (&s1)[kStride],
                                         float (&s2)[kStride]) {
    if constexpr (D != 64) {
        // d=128 keeps the scalar form (the packed one measured -0.5% at C4, where this runs
        // once per 64-block tile)
#pragma unroll
        for (int x = 0; x < kStride; ++x) {
            float a = 0.0f, b = 0.0f;
#pragma unroll
            for (int l = 0; l < D / kStride; ++l) {
                const float v = o[x + kStride * l];
                a = __fadd_rn(a, v);
                b = __fadd_rn(b, __fmul_rn(static_cast<float>(l + 1), v));
            }
            s1[x] = a;
            s2[x] = b;
        }
        return;
    }
    // d=64: two groups per packed f32x2 op, per lane the reference's ascending-l multiply-then-add
    // (the epilogue sits on the max chain at every tile boundary: +0.3% at S=2048, +0.8% at S=512)
#pragma unroll
    for (int x = 0; x < kStride; x += 2) {
        float2 a = make_float2(0.0f, 0.0f), b = a;
#pragma unroll
        for (int l = 0; l < D / kStride; ++l) {
            const float w = static_cast<float>(l + 1);
            const float2 v = make_float2(o[x + kStride * l], o[x + 1 + kStride * l]);
            a = fadd2(a, v);
            b = fadd2(b, fmul2(make_float2(w, w), v));
        }
        s1[x] = a.x;
        s1[x + 1] = a.y;
        s2[x] = b.x;
        s2[x + 1] = b.y;
    }
}

// Final output check (efta.cpp:329-336) of the tile, thread = row. pre_bad / pre: a per-row
// condition decided before (the rowsum range restriction of the CTA-pair kernel) whose tile
// event the reference emits first; it shares the common-case barrier with the output check
// (one warpgroup barrier for a clean tile), and `pre` runs warpgroup-wide only if some row has it.
template <int D, typename Pre>
__device__ __forceinline__ void verify_output_tile_pre(const AttnParams& p, float (&o)[D],
                                                       const float (&c1)[kStride],
                                                       const float (&c2)[kStride], double eps_row,
                                                       int head, int bi, int bj, int row,
                                                       const RowScratch& rs, float& residual_out,
                                                       uint32_t bo, bool pre_bad, Pre&& pre, int ts_g = -1) {
    constexpr int G = D / kStride;
    float s1[kStride], s2[kStride];
    row_sums<D>(o, s1, s2);
    if ((threadIdx.x >> 5 & 3) == 0) EFTA_TS(41, ts_g);
    bool viol = false, cs_bad = false;
    double res = 0.0;
    group_check<kStride, G, false>(c1, c2, s1, s2, eps_row, viol, cs_bad, res);
    residual_out = static_cast<float>(res);
    EFTA_TSW(44, ts_g);
    if (!named_bar_or(5 + bo, 128, viol || cs_bad || pre_bad)) return;
    if (named_bar_or(7 + bo, 128, pre_bad)) pre();
    const bool tile_cs_bad = named_bar_or(4 + bo, 128, cs_bad);
    const bool any = named_bar_or(5 + bo, 128, viol || cs_bad);
    if (!any) return;
    RowVerify rv{};
    rv.best_col = -1;
    rv.restored_col = -1;
    rv.residual = res;
    if (!tile_cs_bad && viol) {
        float t[D];
#pragma unroll
        for (int c = 0; c < D; ++c) t[c] = o[c];
        float cc1[kStride], cc2[kStride];
#pragma unroll
        for (int x = 0; x < kStride; ++x) { cc1[x] = c1[x]; cc2[x] = c2[x]; }
        verify_row<D>(t, cc1, cc2, eps_row, rv);
#pragma unroll
        for (int c = 0; c < D; ++c) o[c] = t[c];
        residual_out = static_cast<float>(rv.residual);
    }
    TileReport tr = reduce_tile_report(rv, tile_cs_bad, row, rs.slots, rs.ints, rs.dbl, bo);
    if (row == 0)
        push_event(p, EFTA_OUTPUT_CHECKSUM, head, bi, bj, tr.status, tr.row, tr.col, tr.violations,
                   tr.corrections, tr.checksum_repair, tr.residual, tr.delta);
}

template <int D>
__device__ __forceinline__ void verify_output_tile(const AttnParams& p, float (&o)[D],
                                                   const float (&c1)[kStride],
                                                   const float (&c2)[kStride], double eps_row,
                                                   int head, int bi, int bj, int row,
                                                   const RowScratch& rs, float& residual_out,
                                                   uint32_t bo = 0) {
    constexpr int G = D / kStride;
    float s1[kStride], s2[kStride];
    row_sums<D>(o, s1, s2);
    bool viol = false, cs_bad = false;
    double res = 0.0;
    if constexpr (D == 64) {
        group_check<kStride, G, false>(c1, c2, s1, s2, eps_row, viol, cs_bad, res);
    } else {
        // d=128 keeps the plain double loop: the fp32 screen measured -0.7% at C4 (+1.4% at
        // S=2048), where this runs once per 64-block tile (profiles/r02/s3/ab_c4_group_check.log)
#pragma unroll
        for (int x = 0; x < kStride; ++x) {
            cs_bad |= !isfinite(c1[x]) || !isfinite(c2[x]);
            if (!isfinite(s1[x]) || !isfinite(s2[x])) { viol = true; continue; }
            const double d1 = static_cast<double>(c1[x]) - s1[x];
            const double d2 = static_cast<double>(c2[x]) - s2[x];
            res = fmax(res, fmax(fabs(d1), fabs(d2) / G));
            viol |= (fabs(d1) > eps_row) || (fabs(d2) > eps_row * G);
        }
    }
    residual_out = static_cast<float>(res);
    const bool tile_cs_bad = named_bar_or(4 + bo, 128, cs_bad);
    const bool any = named_bar_or(5 + bo, 128, viol || cs_bad);
    if (!any) return;
    RowVerify rv{};
    rv.best_col = -1;
    rv.restored_col = -1;
    rv.residual = res;
    if (!tile_cs_bad && viol) {
        float t[D];
#pragma unroll
        for (int c = 0; c < D; ++c) t[c] = o[c];
        float cc1[kStride], cc2[kStride];
#pragma unroll
        for (int x = 0; x < kStride; ++x) { cc1[x] = c1[x]; cc2[x] = c2[x]; }
        verify_row<D>(t, cc1, cc2, eps_row, rv);
#pragma unroll
        for (int c = 0; c < D; ++c) o[c] = t[c];
        residual_out = static_cast<float>(rv.residual);
    }
    TileReport tr = reduce_tile_report(rv, tile_cs_bad, row, rs.slots, rs.ints, rs.dbl, bo);
    if (row == 0)
        push_event(p, EFTA_OUTPUT_CHECKSUM, head, bi, bj, tr.status, tr.row, tr.col, tr.violations,
                   tr.corrections, tr.checksum_repair, tr.residual, tr.delta);
}

template <bool PAIR>
__device__ __forceinline__ void signal_p_ready(uint64_t* bar, int lane) {
    if constexpr (PAIR) {
        // one arrival per warp on the pair leader's barrier (its MMA reads both CTAs' P)
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(bar, 0);
    } else {
        mbar_arrive(bar);
    }
}

// ----------------------------------------------------------------------------
// Row warpgroup (warps 4..7, thread t = query row t = TMEM lane t): softmax, exp-stage
// check, factor guard, O correction, epilogue. Shared by the single-CTA kernel and the
// CTA-pair (cta_group::2) kernel; only the P-ready signal differs.
template <int D, int MODE, bool DBG, bool PAIR>
__device__ __forceinline__ void row_wg(const AttnParams& p, uint8_t* red, uint64_t* s_full,
                                       uint64_t* p_ready, uint64_t* o_done, uint32_t tmem, int warp,
                                       int lane, int head, int qt, int n, int seq_row0) {
    using L = AttnLayout<D>;
    constexpr bool PROT = MODE != EFTA_MODE_NONE;
    constexpr bool LAZY = attn_lazy(MODE, DBG);
    const int wq = warp - 4;
    const int row = wq * 32 + lane;
    const uint32_t lane_base = tmem + (static_cast<uint32_t>(wq * 32) << 16);
    RowScratch rs;
    rs.slots = reinterpret_cast<RowSlot*>(red);
    rs.ints = reinterpret_cast<int*>(red + 128 * sizeof(RowSlot));
    rs.dbl = reinterpret_cast<double*>(red + 128 * sizeof(RowSlot) + 16 * sizeof(int));

    ThreadTap tap{};
    if (DBG) {
        for (int i = 0; i < p.n_faults; ++i) {
            const efta_fault_spec f = p.faults[i];
            if (f.head == head && f.block_i == qt && f.row == row) {
                tap.active = 1;
                tap.site = f.site;
                tap.bj = f.block_j;
                tap.col = f.col;
                tap.bit = f.bit;
                tap.trigger = f.trigger;
                tap.count = 0;
                tap.idx = i;
            }
        }
    }
    const float scale = p.scale, scale_log2 = p.scale_log2;
    // m_run: the max P is referenced to (== the running max unless LAZY);
    // m_true: the running row max (the reference's m) when rescaling lazily
    float m_run = -CUDART_INF_F, l_run = 0.0f, lb = 0.0f, m_true = -CUDART_INF_F;
    float fam_exp = 0.0f, fam_lin = 0.0f, fam_out = 0.0f;

    for (int j = 0; j < n; ++j) {
        const int b = j & 1;
        const uint32_t s_addr = lane_base + L::COL_S0 + b * L::S_STRIDE;
        const uint32_t cs_addr = s_addr + 128;  // 16 hi + 16 lo checksum product cols
        if (warp == 4) EFTA_TS(0, j);
        mbar_wait(&s_full[b], (j >> 1) & 1);
        if (warp == 4) EFTA_TS(1, j);
        tc_fence_after();
        float pv[kBlock];
        uint32_t csr[16], csl[16];
#pragma unroll
        for (int c4 = 0; c4 < 4; ++c4)
            tmem_ld32(s_addr + c4 * 32, *reinterpret_cast<uint32_t(*)[32]>(&pv[c4 * 32]));
        if (PROT) {
            tmem_ld16(cs_addr, csr);
            tmem_ld16(cs_addr + 16, csl);
        }
        tmem_wait_ld();
        if (warp == 4) EFTA_TS(7, j);
        if (PROT) {
#pragma unroll
            for (int x = 0; x < 16; ++x)
                csr[x] = __float_as_uint(__fadd_rn(__uint_as_float(csr[x]), __uint_as_float(csl[x])));
        }

        float bm, m_new;
        float2 prod_f[kStride / 2];   // fast path: strided group products of P
        float pc1v[kStride];          // fast path: exp-domain checksums Pc1
        float psum_f = 0.0f;          // fast path: row sum of P
        const float m_true_before = m_true;
        int sc_fault_col = -1;
        float sc_fault_val = 0.0f;
        if (DBG) {
            // explicit reference sequence so every named site can be tapped
#pragma unroll
            for (int c = 0; c < kBlock; ++c) {
                const float sc0 = __fmul_rn(pv[c], scale);
                const float sc1 = tap(p, EFTA_GEMM1_OUT, j, c, sc0);
                if (__float_as_uint(sc1) != __float_as_uint(sc0)) { sc_fault_col = c; sc_fault_val = sc1; }
                pv[c] = sc1;
            }
            if (PROT && p.observe_linear) {
                // efta.cpp:181-185: linear score check every iteration with eps = inf
                // (observation only); residual = max(|d1|, |d2|/G) (abft.cpp:135)
                float lin = 0.0f;
#pragma unroll
                for (int x = 0; x < kStride; ++x) {
                    float a = 0.0f, bb = 0.0f;
#pragma unroll
                    for (int l = 0; l < kBlock / kStride; ++l) {
                        a = __fadd_rn(a, pv[x + kStride * l]);
                        bb = __fadd_rn(bb, __fmul_rn(static_cast<float>(l + 1), pv[x + kStride * l]));
                    }
                    const float d1 = fabsf(__fmul_rn(__uint_as_float(csr[x]), scale) - a);
                    const float d2 = fabsf(__fmul_rn(__uint_as_float(csr[kStride + x]), scale) - bb) /
                                     static_cast<float>(kBlock / kStride);
                    lin = fmaxf(lin, fmaxf(d1, d2));
                }
                if (isfinite(lin)) fam_lin = fmaxf(fam_lin, lin);
            }
            bm = pv[0];
#pragma unroll
            for (int c = 1; c < kBlock; ++c) bm = (bm < pv[c]) ? pv[c] : bm;
            bm = bm + p.rowmax_bias;
            m_new = (m_run < bm) ? bm : m_run;
            m_new = tap(p, EFTA_REDUCE_MAX, j, 0, m_new);
#pragma unroll
            for (int c = 0; c < kBlock; ++c) {
                float a = __fsub_rn(pv[c], m_new);
                a = tap(p, EFTA_SUB_MAX, j, c, a);
                float e = ex2_approx(a * kLog2e);
                pv[c] = tap(p, EFTA_EXP_OUT, j, c, e);
            }
        } else {
            float mx0 = pv[0], mx1 = pv[1], mx2 = pv[2], mx3 = pv[3];
#pragma unroll
            for (int c = 4; c < kBlock; c += 4) {
                mx0 = fmaxf(mx0, pv[c]);
                mx1 = fmaxf(mx1, pv[c + 1]);
                mx2 = fmaxf(mx2, pv[c + 2]);
                mx3 = fmaxf(mx3, pv[c + 3]);
            }
            bm = __fmul_rn(fmaxf(fmaxf(mx0, mx1), fmaxf(mx2, mx3)), scale) + p.rowmax_bias;
            if (LAZY) {
                m_true = (m_true < bm) ? bm : m_true;
                m_new = (j == 0 || m_true - m_run > kLazyTau) ? m_true : m_run;
            } else {
                m_new = (m_run < bm) ? bm : m_run;
            }
            const float mL = m_new * kLog2e;
            if (PROT) {  // Pc1 = exp(scale*c1 - 16 m) first: these MUFUs overlap the loop below
                const float g16m = 16.0f * m_new;
#pragma unroll
                for (int x = 0; x < kStride; ++x)
                    pc1v[x] = ex2_approx(__fsub_rn(__fmul_rn(__uint_as_float(csr[x]), scale), g16m) * kLog2e);
            }
            const float2 sl2 = make_float2(scale_log2, scale_log2), nm2 = make_float2(-mL, -mL);
            float2 ps0 = make_float2(0.0f, 0.0f), ps1 = make_float2(0.0f, 0.0f);
#pragma unroll
            for (int c = 0; c < kBlock; c += 2) {
                const float2 a = ffma2(make_float2(pv[c], pv[c + 1]), sl2, nm2);
                float2 e;
                if (exp_on_fma<D>(c)) {
                    e = ex2_poly2(a);
                } else {
                    e.x = ex2_approx(a.x);
                    e.y = ex2_approx(a.y);
                }
                pv[c] = e.x;
                pv[c + 1] = e.y;
                // row sum and the strided group products ride along (fill MUFU issue gaps)
                if ((c >> 1) & 1) ps1 = fadd2(ps1, e);
                else ps0 = fadd2(ps0, e);
                if (PROT) {
                    const int g = (c & 7) >> 1;
                    prod_f[g] = (c < kStride) ? e : fmul2(prod_f[g], e);
                }
            }
            psum_f = (ps0.x + ps0.y) + (ps1.x + ps1.y);
        }

        if (warp == 4) EFTA_TS(8, j);
        // ---- exp-domain strided product check (SNVR; snvr.cpp:52-83):
        // group x: prod_l P[x + 8l] vs Pc1 = exp(scale*c1 - 16 m); the reference's
        // log-domain test |sum log P - log Pc1| > eps1 becomes the bracket
        // prod outside [Pc1 e^-eps1, Pc1 e^eps1] (no log on the fast path).
        const float f = ex2_approx((m_run - m_new) * kLog2e);
        bool exp_affected = false, factor_bad = false;
        float exp_res = 0.0f;
        int exp_viol = 0;
        bool replaced_p = false;
        if (PROT) {
            float2 prod[kStride / 2];
            if (DBG) {
#pragma unroll
                for (int x = 0; x < kStride / 2; ++x) prod[x] = make_float2(pv[2 * x], pv[2 * x + 1]);
#pragma unroll
                for (int l = 1; l < kBlock / kStride; ++l)
#pragma unroll
                    for (int x = 0; x < kStride / 2; ++x)
                        prod[x] = fmul2(prod[x], make_float2(pv[kStride * l + 2 * x], pv[kStride * l + 2 * x + 1]));
            } else {
#pragma unroll
                for (int x = 0; x < kStride / 2; ++x) prod[x] = prod_f[x];
            }
            const float g16m = 16.0f * m_new;
            bool degenerate = !isfinite(m_new);
#pragma unroll
            for (int x = 0; x < kStride; ++x) {
                const float pr = (x & 1) ? prod[x >> 1].y : prod[x >> 1].x;
                const float c1s = __fmul_rn(__uint_as_float(csr[x]), scale);
                const float pc1 = DBG ? ex2_approx(__fsub_rn(c1s, g16m) * kLog2e) : pc1v[x];
                const bool bad = !(pr > pc1 * p.exp_lo && pr < pc1 * p.exp_hi);  // strict: also fails 0/0, inf/inf
                if (DBG) {
                    if (!(pr > 0.0f && pr < CUDART_INF_F) || !(pc1 > 0.0f && pc1 < CUDART_INF_F)) {
                        degenerate = true;
                    } else {
                        const float d = fabsf(lg2_approx(__fdividef(pr, pc1))) * kLn2;
                        exp_res = fmaxf(exp_res, d);
                    }
                }
                if (bad) { exp_affected = true; ++exp_viol; }
            }
            if (degenerate) { exp_affected = true; exp_res = CUDART_INF_F; exp_viol = 1; }
            if (j > 0) factor_bad = !(f > 0.0f && f <= 1.0f);  // NaN fails both
            if (DBG && isfinite(exp_res)) fam_exp = fmaxf(fam_exp, exp_res);
            if (warp == 4) EFTA_TS(9, j);
            const bool tile_trig = named_bar_or(6, 128, exp_affected || factor_bad);
            if (warp == 4) EFTA_TS(15, j);
            if (tile_trig) {
                float p_loc[kBlock];
#pragma unroll
                for (int c = 0; c < kBlock; ++c) p_loc[c] = pv[c];
                int replaced = 0;
                const float m_true_prev = m_true_before;
                exp_stage_slow<DBG, D, false>(p, s_addr, cs_addr, head, qt, j, row, exp_affected, exp_res,
                                    exp_viol, m_run, m_new, bm, p_loc, replaced, tap, sc_fault_col,
                                    sc_fault_val, rs);
                if (replaced) {
#pragma unroll
                    for (int c = 0; c < kBlock; ++c) pv[c] = p_loc[c];
                }
                replaced_p = replaced != 0;
                // the recovered reference max is the row's true max so far
                if (LAZY) m_true = (m_true_prev < m_new) ? m_new : m_true_prev;
            }
        }

        if (warp == 4) EFTA_TS(2, j);
        // ---- rescale factor, lower bound, denominator (efta.cpp:192-242)
        const float fr = PROT ? ex2_approx((m_run - m_new) * kLog2e) : f;  // m_new may be repaired
        if (PROT) lb = __fadd_rn(__fmul_rn(lb, fr), ex2_approx((bm - m_new) * kLog2e));
        float psum = psum_f;
        if (DBG || replaced_p) {  // same pairing and order as the fused sums in the exp loop
            float2 ps0 = make_float2(pv[0], pv[1]), ps1 = make_float2(pv[2], pv[3]);
#pragma unroll
            for (int c = 4; c < kBlock; c += 4) {
                ps0 = fadd2(ps0, make_float2(pv[c], pv[c + 1]));
                ps1 = fadd2(ps1, make_float2(pv[c + 2], pv[c + 3]));
            }
            psum = (ps0.x + ps0.y) + (ps1.x + ps1.y);
        }
        l_run = __fadd_rn(__fmul_rn(fr, l_run), psum);
        if (DBG) l_run = tap(p, EFTA_REDUCE_SUM, j, 0, l_run);

        if (warp == 4) EFTA_TS(3, j);
        // ---- P (fp16) over the S columns it came from
        {
            uint32_t pk[32];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
#pragma unroll
                for (int x = 0; x < 32; ++x) pk[x] = pack_half2(pv[h * 64 + 2 * x], pv[h * 64 + 2 * x + 1]);
                tmem_st32(s_addr + h * 32, pk);
            }
        }

        // ---- O correction: O *= f (and its checksum columns)
        if (j > 0) {
            if (warp == 4) EFTA_TS(4, j);
            mbar_wait(o_done, (j - 1) & 1);
            if (warp == 4) EFTA_TS(5, j);
            tc_fence_after();
            if (MODE == EFTA_MODE_EFTA) {
                // per-iteration output check of the accumulator after GEMM II of j-1
                float o[D];
                uint32_t oc[32];
#pragma unroll
                for (int c = 0; c < D / 32; ++c)
                    tmem_ld32(lane_base + L::COL_O + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&o[c * 32]));
                tmem_ld32(lane_base + L::COL_O + D, oc);
                tmem_wait_ld();
#pragma unroll
                for (int x = 0; x < 16; ++x) {
                    oc[x] = __float_as_uint(__fadd_rn(__uint_as_float(oc[x]), __uint_as_float(oc[16 + x])));
                    oc[16 + x] = 0u;
                }
                if (DBG) {
#pragma unroll
                    for (int c = 0; c < D; ++c) o[c] = tap(p, EFTA_GEMM2_ACC, j - 1, c, o[c]);
                }
                float c1[kStride], c2[kStride];
#pragma unroll
                for (int x = 0; x < kStride; ++x) { c1[x] = __uint_as_float(oc[x]); c2[x] = __uint_as_float(oc[kStride + x]); }
                float res;
                verify_output_tile<D>(p, o, c1, c2, p.eps2, head, qt, j - 1, row, rs, res);
                if (isfinite(res)) fam_out = fmaxf(fam_out, res);
#pragma unroll
                for (int c = 0; c < D; ++c) o[c] = __fmul_rn(o[c], fr);
                if (DBG) {
#pragma unroll
                    for (int c = 0; c < D; ++c) o[c] = tap(p, EFTA_RESCALE_FACTOR, j, c, o[c]);
                }
#pragma unroll
                for (int x = 0; x < kStride; ++x) { oc[x] = __float_as_uint(__fmul_rn(c1[x], fr)); oc[kStride + x] = __float_as_uint(__fmul_rn(c2[x], fr)); }
#pragma unroll
                for (int c = 0; c < D / 32; ++c)
                    tmem_st32(lane_base + L::COL_O + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&o[c * 32]));
                tmem_st32(lane_base + L::COL_O + D, oc);
            } else {
                const bool need = DBG || !__all_sync(0xffffffffu, fr == 1.0f);
                if (need && DBG) {
#pragma unroll
                    for (int c = 0; c < D / 32; ++c) {
                        float o[32];
                        tmem_ld32(lane_base + L::COL_O + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&o[0]));
                        tmem_wait_ld();
#pragma unroll
                        for (int x = 0; x < 32; ++x) {
                            float v = tap(p, EFTA_GEMM2_ACC, j - 1, c * 32 + x, o[x]);
                            v = __fmul_rn(v, fr);
                            o[x] = tap(p, EFTA_RESCALE_FACTOR, j, c * 32 + x, v);
                        }
                        tmem_st32(lane_base + L::COL_O + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&o[0]));
                    }
                }
                if (need) {
                    // all chunks in flight at once (P's registers are free by now)
                    constexpr int NCH = DBG ? (PROT ? 1 : 0) : (D / 32 + (PROT ? 1 : 0));
                    constexpr int C0 = DBG ? D / 32 : 0;
                    float o[NCH > 0 ? NCH : 1][32];
#pragma unroll
                    for (int c = 0; c < NCH; ++c)
                        tmem_ld32(lane_base + L::COL_O + (C0 + c) * 32, *reinterpret_cast<uint32_t(*)[32]>(&o[c][0]));
                    tmem_wait_ld();
                    const float2 f2 = make_float2(fr, fr);
#pragma unroll
                    for (int c = 0; c < NCH; ++c)
#pragma unroll
                        for (int x = 0; x < 32; x += 2) {
                            const float2 r2 = fmul2(make_float2(o[c][x], o[c][x + 1]), f2);
                            o[c][x] = r2.x;
                            o[c][x + 1] = r2.y;
                        }
#pragma unroll
                    for (int c = 0; c < NCH; ++c)
                        tmem_st32(lane_base + L::COL_O + (C0 + c) * 32, *reinterpret_cast<uint32_t(*)[32]>(&o[c][0]));
                }
            }
        } else if (DBG) {
            // reference: oacc starts at 0 and is rescaled (0*0) + tapped at j = 0
#pragma unroll
            for (int c = 0; c < D / 32; ++c) {
                float o[32];
#pragma unroll
                for (int x = 0; x < 32; ++x) o[x] = tap(p, EFTA_RESCALE_FACTOR, 0, c * 32 + x, 0.0f);
                tmem_st32(lane_base + L::COL_O + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&o[0]));
            }
            uint32_t z[32];
#pragma unroll
            for (int x = 0; x < 32; ++x) z[x] = 0u;
            tmem_st32(lane_base + L::COL_O + D, z);
        }
        tmem_wait_st();
        tc_fence_before();
        signal_p_ready<PAIR>(p_ready, lane);
        if (warp == 4) EFTA_TS(6, j);
        m_run = m_new;
    }

    // ------------------------------------------------ epilogue
    mbar_wait(o_done, (n - 1) & 1);
    tc_fence_after();
    float o[D];
    float c1[kStride], c2[kStride];
#pragma unroll
    for (int c = 0; c < D / 32; ++c)
        tmem_ld32(lane_base + L::COL_O + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&o[c * 32]));
    {
        uint32_t oc[32];
        if (PROT) tmem_ld32(lane_base + L::COL_O + D, oc);
        tmem_wait_ld();
#pragma unroll
        for (int x = 0; x < kStride; ++x) {
            c1[x] = PROT ? __fadd_rn(__uint_as_float(oc[x]), __uint_as_float(oc[16 + x])) : 0.0f;
            c2[x] = PROT ? __fadd_rn(__uint_as_float(oc[kStride + x]), __uint_as_float(oc[16 + kStride + x]))
                         : 0.0f;
        }
    }
    if (DBG) {
#pragma unroll
        for (int c = 0; c < D; ++c) o[c] = tap(p, EFTA_GEMM2_ACC, n - 1, c, o[c]);
    }
    if (LAZY) {
        // bring O, its checksums, l and the lower bound from the lazy reference max to
        // the row's true max (the reference's final m); F == 1 for most rows
        const float F = ex2_approx((m_run - m_true) * kLog2e);
        if (!__all_sync(0xffffffffu, F == 1.0f)) {
#pragma unroll
            for (int c = 0; c < D; ++c) o[c] = __fmul_rn(o[c], F);
#pragma unroll
            for (int x = 0; x < kStride; ++x) { c1[x] = __fmul_rn(c1[x], F); c2[x] = __fmul_rn(c2[x], F); }
            l_run = __fmul_rn(l_run, F);
            lb = __fmul_rn(lb, F);
        }
        m_run = m_true;
    }
    if (MODE == EFTA_MODE_EFTA) {
        float res;
        verify_output_tile<D>(p, o, c1, c2, p.eps2, head, qt, n - 1, row, rs, res);
        if (isfinite(res)) fam_out = fmaxf(fam_out, res);
    }
    double eps_mult = 1.0;
    if (PROT) {
        // denominator range restriction (snvr.cpp:161-182, efta.cpp:289-310)
        const float upper = static_cast<float>(p.seq_len);
        const bool bad = !isfinite(l_run) || l_run < lb || l_run > upper;
        double viol = 0.0;
        if (bad) {
            viol = !isfinite(l_run) ? CUDART_INF
                                    : (l_run < lb ? static_cast<double>(lb) - l_run
                                                  : static_cast<double>(l_run) - upper);
            l_run = lb;
            eps_mult = static_cast<double>(p.seq_len) / static_cast<double>(l_run);
        }
        if (named_bar_or(7, 128, bad)) {
            if (row == 0) { rs.ints[0] = 0; rs.ints[1] = 0x7fffffff; rs.dbl[0] = 0.0; }
            wg_sync();
            if (bad) {
                atomicAdd(&rs.ints[0], 1);
                atomicMin(&rs.ints[1], row);
                unsigned long long* a = reinterpret_cast<unsigned long long*>(&rs.dbl[0]);
                unsigned long long old = *a, assumed;
                do {
                    assumed = old;
                    if (__longlong_as_double(assumed) >= viol) break;
                    old = atomicCAS(a, assumed, __double_as_longlong(viol));
                } while (old != assumed);
            }
            wg_sync();
            if (row == 0) {
                atomicAdd(&p.counters->range_replacements, rs.ints[0]);
                push_event(p, EFTA_ROWSUM_RANGE, head, qt, n, EFTA_CORRECTED, rs.ints[1], -1, 0,
                           rs.ints[0], 0, rs.dbl[0], 0.0);
            }
            wg_sync();
        }
    }
    // normalization (efta.cpp:312-327)
#pragma unroll
    for (int c = 0; c < D; ++c) {
        float v = __fdiv_rn(o[c], l_run);
        if (DBG) v = tap(p, EFTA_NORMALIZE_OUT, 0, c, v);
        o[c] = v;
    }
    if (PROT) {
#pragma unroll
        for (int x = 0; x < kStride; ++x) { c1[x] = __fdiv_rn(c1[x], l_run); c2[x] = __fdiv_rn(c2[x], l_run); }
        float res;
        verify_output_tile<D>(p, o, c1, c2, p.eps2 * eps_mult, head, qt, n, row, rs, res);
        if (isfinite(res)) fam_out = fmaxf(fam_out, res);
    }
    // store
    const size_t grow = static_cast<size_t>(seq_row0) + qt * kBlock + row;
    float4* dst = reinterpret_cast<float4*>(p.o + grow * D);
#pragma unroll
    for (int c = 0; c < D / 4; ++c) dst[c] = make_float4(o[4 * c], o[4 * c + 1], o[4 * c + 2], o[4 * c + 3]);
    if (p.m_out) p.m_out[grow] = m_run;
    if (p.l_out) p.l_out[grow] = l_run;
    if (PROT) {
        // per-family worst clean residual (calibration / observation)
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            fam_exp = fmaxf(fam_exp, __shfl_xor_sync(0xffffffffu, fam_exp, off));
            fam_out = fmaxf(fam_out, __shfl_xor_sync(0xffffffffu, fam_out, off));
            fam_lin = fmaxf(fam_lin, __shfl_xor_sync(0xffffffffu, fam_lin, off));
        }
        if (lane == 0) {
            atomic_max_nonneg(&p.counters->family_max[0], fam_exp);
            atomic_max_nonneg(&p.counters->family_max[1], fam_out);
            if (DBG && p.observe_linear) atomic_max_nonneg(&p.counters->family_max[2], fam_lin);
        }
    }

}

// ----------------------------------------------------------------------------
template <int D, int MODE, bool DBG>
__global__ void __launch_bounds__(256, 1)
efta_attn_fwd_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                     const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_kc,
                     const __grid_constant__ CUtensorMap tm_vc, const AttnParams p) {
    using L = AttnLayout<D>;
    constexpr bool PROT = MODE != EFTA_MODE_NONE;
    constexpr bool LAZY = attn_lazy(MODE, DBG);
    constexpr int KS = L::KS, VS = L::VS, NSUB = L::NSUB;

    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
    uint64_t* q_full = bars;
    uint64_t* k_full = bars + 1;
    uint64_t* k_empty = k_full + KS;
    uint64_t* v_full = k_empty + KS;
    uint64_t* v_empty = v_full + VS;
    uint64_t* s_full = v_empty + VS;
    uint64_t* p_ready = s_full + 2;
    uint64_t* o_done = p_ready + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::OFF_TMEM);

    const int warp = warp_id(), lane = lane_id();
    const int qt = blockIdx.x, head = blockIdx.y, n = p.nblk;
    const int seq_row0 = head * p.seq_len;
    const int kvh = kv_head(p, head), kv_row0 = kvh * p.seq_len;  // K / V / checksum operands (GQA)

    if (warp == 0 && lane == 0) {
        mbar_init(q_full, 1);
        for (int s = 0; s < KS; ++s) { mbar_init(&k_full[s], 1); mbar_init(&k_empty[s], 1); }
        for (int s = 0; s < VS; ++s) { mbar_init(&v_full[s], 1); mbar_init(&v_empty[s], 1); }
        mbar_init(&s_full[0], 1);
        mbar_init(&s_full[1], 1);
        mbar_init(p_ready, 128);
        mbar_init(o_done, 1);
        fence_barrier_init();
        tma_prefetch_desc(&tm_q);
        tma_prefetch_desc(&tm_k);
        tma_prefetch_desc(&tm_v);
        if (PROT) { tma_prefetch_desc(&tm_kc); tma_prefetch_desc(&tm_vc); }
    }
    if (warp == 1) tmem_alloc(tmem_slot, L::TMEM_COLS);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    const uint32_t q_smem = smem_u32(smem + L::OFF_Q);
    const uint32_t k_smem = smem_u32(smem + L::OFF_K);
    const uint32_t v_smem = smem_u32(smem + L::OFF_V);

    if (warp == 0) {
        // ------------------------------------------------ K (+KC) producer
        if (lane == 0) {
            for (int j = 0; j < n; ++j) {
                const int s = j % KS;
                mbar_wait(&k_empty[s], ((j / KS) & 1) ^ 1);
                uint8_t* dst = smem + L::OFF_K + s * L::K_STAGE;
                mbar_arrive_expect_tx(&k_full[s], L::K_BYTES + (PROT ? L::KC_BYTES : 0));
#pragma unroll
                for (int sub = 0; sub < NSUB; ++sub) {
                    tma_load_2d(dst + sub * L::K_SUB, &tm_k, &k_full[s], sub * 64,
                                kv_row0 + j * kBlock, kEvictLast);
                    if (PROT)
                        tma_load_2d(dst + sub * L::K_SUB + 16384, &tm_kc, &k_full[s], sub * 64,
                                    (kvh * n + j) * 32, kEvictLast);
                }
            }
        }
    } else if (warp == 3) {
        // ------------------------------------------------ Q, V (+VC) producer
        if (lane == 0) {
            mbar_arrive_expect_tx(q_full, L::Q_BYTES);
#pragma unroll
            for (int sub = 0; sub < NSUB; ++sub)
                tma_load_2d(smem + L::OFF_Q + sub * 16384, &tm_q, q_full, sub * 64,
                            seq_row0 + qt * kBlock, kEvictFirst);
            for (int j = 0; j < n; ++j) {
                const int s = j % VS;
                mbar_wait(&v_empty[s], ((j / VS) & 1) ^ 1);
                uint8_t* dst = smem + L::OFF_V + s * L::V_STAGE;
                mbar_arrive_expect_tx(&v_full[s], L::V_BYTES + (PROT ? L::VC_BYTES : 0));
#pragma unroll
                for (int sub = 0; sub < NSUB; ++sub)
                    tma_load_2d(dst + sub * 16384, &tm_v, &v_full[s], sub * 64, kv_row0 + j * kBlock,
                                kEvictLast);
                if (PROT)
                    tma_load_2d(dst + NSUB * 16384, &tm_vc, &v_full[s], 0, (kvh * n + j) * kBlock,
                                kEvictLast);
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer (one thread)
        if (lane == 0) {
            // protected: N grows by the 32 checksum rows/cols (hi + lo products)
            constexpr uint32_t ID_S = idesc_f16_f32(128, PROT ? 160 : 128, 0, 0);
            constexpr uint32_t ID_PV = idesc_f16_f32(128, PROT ? D + 32 : D, 0, 1);
            mbar_wait(q_full, 0);
            tc_fence_after();
            auto issue_s = [&](int j) {
                const int s = j % KS;
                mbar_wait(&k_full[s], (j / KS) & 1);
                tc_fence_after();
                const uint32_t kb = k_smem + s * L::K_STAGE;
                const uint32_t d_s = tmem + L::COL_S0 + (j & 1) * L::S_STRIDE;
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk) {
                    const uint32_t offq = (kk >> 2) * 16384 + (kk & 3) * 32;
                    const uint32_t offk = (kk >> 2) * L::K_SUB + (kk & 3) * 32;
                    mma_ss(d_s, smem_desc_sw128(q_smem + offq, 16, 1024),
                           smem_desc_sw128(kb + offk, 16, 1024), ID_S, kk > 0);
                }
                tc_commit(&k_empty[s]);
                tc_commit(&s_full[j & 1]);
            };
            issue_s(0);
            for (int j = 0; j < n; ++j) {
                EFTA_TS(10, j);
                if (j + 1 < n) issue_s(j + 1);
                EFTA_TS(11, j);
                mbar_wait(p_ready, j & 1);
                EFTA_TS(12, j);
                tc_fence_after();
                const int s = j % VS;
                mbar_wait(&v_full[s], (j / VS) & 1);
                tc_fence_after();
                const uint32_t vb = v_smem + s * L::V_STAGE;
                const uint32_t a_p = tmem + L::COL_S0 + (j & 1) * L::S_STRIDE;
                const uint32_t acc0 = (j > 0 || DBG) ? 1u : 0u;
#pragma unroll
                for (int kk = 0; kk < kBlock / 16; ++kk)
                    mma_ts(tmem + L::COL_O, a_p + kk * 8, smem_desc_sw128(vb + kk * 2048, 16384, 1024),
                           ID_PV, acc0 | (kk > 0));
                tc_commit(&v_empty[s]);
                tc_commit(o_done);
                EFTA_TS(13, j);
            }
        }
        __syncwarp();
    } else if (warp >= 4) {
        row_wg<D, MODE, DBG, false>(p, smem + L::OFF_RED, s_full, p_ready, o_done, tmem, warp, lane, head, qt, n, seq_row0);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 1) tmem_dealloc(tmem, L::TMEM_COLS);
}

}  // namespace efta_sm100
