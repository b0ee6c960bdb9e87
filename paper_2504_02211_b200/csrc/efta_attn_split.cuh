// efta_attn_split.cuh — the "split-row" row-warpgroup schedule of the fused EFTA kernel.
//
// Used by the fast variants (NONE / EFTA_OPTIMIZED, no fault taps). Two warpgroups share
// the 128 query rows of the CTA: warps 4-7 own score columns 0..63 (and the checksum
// columns), warps 8-11 own columns 64..127 of the same rows (same TMEM lanes: warp w reads
// lanes 32*(w%4)..+31). Each SM sub-partition thus runs two row warps, which hides the
// MUFU / TMEM / FMA latencies a single row warp cannot. Per key block the pair exchanges:
//   * the partial row maxima (shared memory, one 256-thread named barrier),
//   * (protected) warps 8-11's partial strided products of P, so warps 4-7 complete the
//     exp-domain check of every group (second barrier) + a barrier.red.or for the tile.
// Row sums stay per half (l = l_lo + l_hi at the end, same rescale factor f applied to
// both). The rare recovery paths (exp-stage ladder, output correction) run on warps 4-7
// over the full row; warps 8-11 hand over / take back their half through a per-SM global
// scratch row (only on those paths). The numerics of every reported quantity are those of
// the single-warpgroup schedule except the order of the max / sum reductions.
#pragma once
#include "efta_attn.cuh"

namespace efta_sm100 {

__device__ __forceinline__ uint32_t sm_id() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
    return r;
}

// barrier ids used by the split schedule (0 = __syncthreads, 1..7 single-warpgroup helpers)
constexpr uint32_t kBarXmax = 8, kBarXprod = 9, kBarOr = 10, kBarRare = 11, kBarEpi = 12;

template <int D, bool PROT>
__device__ __forceinline__ void row_split(const AttnParams& p, uint64_t* s_full, uint64_t* p_ready,
                                          uint64_t* o_done, uint32_t tmem, int warp, int lane,
                                          int head, int qt, int n, int seq_row0,
                                          const RowScratch& rs, float* xch) {
    using L = AttnLayout<D>;
    constexpr int DH = D / 2;          // O columns per half
    constexpr int GH = DH / kStride;   // output groups per half
    const int half = (warp - 4) >> 2;  // warp-uniform
    const int wq = warp & 3;
    const int row = wq * 32 + lane;
    const uint32_t lane_base = tmem + (static_cast<uint32_t>(wq * 32) << 16);
    const int c0 = half * 64;
    float* xmax = xch;                // [2 parity][2 half][128]
    float* xprod = xch + 512;         // [128][16]
    float* xpub = xch + 512 + 2048;   // [128][4]
    float* xl = xch + 512 + 2048 + 512;  // [2 half][128]
    float* scr = p.scratch + static_cast<size_t>(sm_id()) * (128 * 128) + row * 128;  // rare paths
    const float scale = p.scale, scale_log2 = p.scale_log2;
    float m_run = -CUDART_INF_F, l_half = 0.0f, lb = 0.0f, fam_exp = 0.0f;
    ThreadTap no_tap{};

    for (int j = 0; j < n; ++j) {
        const int b = j & 1;
        const uint32_t s_addr = lane_base + L::COL_S0 + b * L::S_STRIDE;
        const uint32_t cs_addr = s_addr + 128;
        mbar_wait(&s_full[b], (j >> 1) & 1);
        tc_fence_after();
        float pv[64];
        uint32_t csr[16], csl[16];
        tmem_ld32(s_addr + c0, *reinterpret_cast<uint32_t(*)[32]>(&pv[0]));
        tmem_ld32(s_addr + c0 + 32, *reinterpret_cast<uint32_t(*)[32]>(&pv[32]));
        if (PROT && half == 0) {
            tmem_ld16(cs_addr, csr);
            tmem_ld16(cs_addr + 16, csl);
        }
        tmem_wait_ld();
        // ---- row max: partial over this half, exchanged through shared memory
        float mx0 = pv[0], mx1 = pv[1], mx2 = pv[2], mx3 = pv[3];
#pragma unroll
        for (int c = 4; c < 64; c += 4) {
            mx0 = fmaxf(mx0, pv[c]);
            mx1 = fmaxf(mx1, pv[c + 1]);
            mx2 = fmaxf(mx2, pv[c + 2]);
            mx3 = fmaxf(mx3, pv[c + 3]);
        }
        const float pm = fmaxf(fmaxf(mx0, mx1), fmaxf(mx2, mx3));
        float* xm = xmax + (j & 1) * 256;  // double-buffered: the partner may still read j-1
        xm[half * 128 + row] = pm;
        named_bar_sync(kBarXmax, 256);
        const float mx = fmaxf(xm[row], xm[128 + row]);
        float bm = __fmul_rn(mx, scale) + p.rowmax_bias;
        float m_new = (m_run < bm) ? bm : m_run;
        const float mL = m_new * kLog2e;
        const float2 sl2 = make_float2(scale_log2, scale_log2), nm2 = make_float2(-mL, -mL);
#pragma unroll
        for (int c = 0; c < 64; c += 2) {
            const float2 a = ffma2(make_float2(pv[c], pv[c + 1]), sl2, nm2);
            pv[c] = ex2_approx(a.x);
            pv[c + 1] = ex2_approx(a.y);
        }
        float f = ex2_approx((m_run - m_new) * kLog2e);
        if (PROT) {
            // ---- exp-domain strided product check: this half holds l = 8*half .. 8*half+7
            float2 prod[4];
#pragma unroll
            for (int x = 0; x < 4; ++x) prod[x] = make_float2(pv[2 * x], pv[2 * x + 1]);
#pragma unroll
            for (int l = 1; l < 8; ++l)
#pragma unroll
                for (int x = 0; x < 4; ++x)
                    prod[x] = fmul2(prod[x], make_float2(pv[8 * l + 2 * x], pv[8 * l + 2 * x + 1]));
            if (half == 1) {
#pragma unroll
                for (int x = 0; x < 4; ++x) {
                    xprod[row * 16 + 2 * x] = prod[x].x;
                    xprod[row * 16 + 2 * x + 1] = prod[x].y;
                }
            }
            named_bar_sync(kBarXprod, 256);
            bool trig = false, exp_affected = false;
            int exp_viol = 0;
            float exp_res = 0.0f;
            if (half == 0) {
                const float g16m = 16.0f * m_new;
                bool degenerate = !isfinite(m_new);
#pragma unroll
                for (int x = 0; x < kStride; ++x) {
                    const float other = xprod[row * 16 + x];
                    const float pr = ((x & 1) ? prod[x >> 1].y : prod[x >> 1].x) * other;
                    const float c1 = __fadd_rn(__uint_as_float(csr[x]), __uint_as_float(csl[x]));
                    const float pc1 = ex2_approx(__fsub_rn(__fmul_rn(c1, scale), g16m) * kLog2e);
                    if (!(pr >= pc1 * p.exp_lo && pr <= pc1 * p.exp_hi)) { exp_affected = true; ++exp_viol; }
                }
                if (degenerate) { exp_affected = true; exp_viol = 1; exp_res = CUDART_INF_F; }
                const bool factor_bad = j > 0 && !(f > 0.0f && f <= 1.0f);
                trig = exp_affected || factor_bad;
            }
            if (named_bar_or(kBarOr, 256, trig)) {
                // ---- rare: exp-stage ladder + factor guard over the full row on warps 4-7
                int replaced = 0;
                if (half == 1) {
#pragma unroll
                    for (int c = 0; c < 64; ++c) scr[64 + c] = pv[c];
                }
                named_bar_sync(kBarRare, 256);
                if (half == 0) {
                    float p_loc[kBlock];
                    for (int c = 0; c < 64; ++c) { p_loc[c] = pv[c]; p_loc[64 + c] = scr[64 + c]; }
                    exp_stage_slow<false, D, false>(p, s_addr, cs_addr, head, qt, j, row, exp_affected, exp_res,
                                          exp_viol, m_run, m_new, bm, p_loc, replaced, no_tap, -1,
                                          0.0f, rs);
                    if (replaced) {
                        for (int c = 0; c < 64; ++c) { pv[c] = p_loc[c]; scr[64 + c] = p_loc[64 + c]; }
                    }
                    xpub[row * 4 + 0] = m_new;
                    xpub[row * 4 + 1] = bm;
                    xpub[row * 4 + 2] = replaced ? 1.0f : 0.0f;
                }
                named_bar_sync(kBarRare, 256);
                if (half == 1) {
                    m_new = xpub[row * 4 + 0];
                    bm = xpub[row * 4 + 1];
                    replaced = xpub[row * 4 + 2] != 0.0f;
                    if (replaced) {
#pragma unroll
                        for (int c = 0; c < 64; ++c) pv[c] = scr[64 + c];
                    }
                }
                f = ex2_approx((m_run - m_new) * kLog2e);
            }
            if (half == 0) lb = __fadd_rn(__fmul_rn(lb, f), ex2_approx((bm - m_new) * kLog2e));
        }
        // ---- partial row sum, P (fp16) over this half's score columns
        float2 ps0 = make_float2(pv[0], pv[1]), ps1 = make_float2(pv[2], pv[3]);
#pragma unroll
        for (int c = 4; c < 64; c += 4) {
            ps0 = fadd2(ps0, make_float2(pv[c], pv[c + 1]));
            ps1 = fadd2(ps1, make_float2(pv[c + 2], pv[c + 3]));
        }
        l_half = __fadd_rn(__fmul_rn(f, l_half), (ps0.x + ps0.y) + (ps1.x + ps1.y));
        {
            uint32_t pk[32];
#pragma unroll
            for (int x = 0; x < 32; ++x) pk[x] = pack_half2(pv[2 * x], pv[2 * x + 1]);
            tmem_st32(s_addr + half * 32, pk);
        }
        // ---- O correction: each half rescales its own O columns (+ the checksum columns on half 0)
        if (j > 0) {
            mbar_wait(o_done, (j - 1) & 1);
            tc_fence_after();
            if (!__all_sync(0xffffffffu, f == 1.0f)) {
                constexpr int NO = DH / 32;
                float o[NO + 1][32];
#pragma unroll
                for (int c = 0; c < NO; ++c)
                    tmem_ld32(lane_base + L::COL_O + half * DH + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&o[c][0]));
                if (PROT && half == 0)
                    tmem_ld32(lane_base + L::COL_O + D, *reinterpret_cast<uint32_t(*)[32]>(&o[NO][0]));
                tmem_wait_ld();
                const float2 f2 = make_float2(f, f);
                const int nch = NO + ((PROT && half == 0) ? 1 : 0);
#pragma unroll
                for (int c = 0; c < NO + 1; ++c) {
                    if (c < nch) {
#pragma unroll
                        for (int x = 0; x < 32; x += 2) {
                            const float2 r2 = fmul2(make_float2(o[c][x], o[c][x + 1]), f2);
                            o[c][x] = r2.x;
                            o[c][x + 1] = r2.y;
                        }
                    }
                }
#pragma unroll
                for (int c = 0; c < NO; ++c)
                    tmem_st32(lane_base + L::COL_O + half * DH + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&o[c][0]));
                if (PROT && half == 0)
                    tmem_st32(lane_base + L::COL_O + D, *reinterpret_cast<uint32_t(*)[32]>(&o[NO][0]));
            }
        }
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(p_ready);
        m_run = m_new;
    }

    // ------------------------------------------------------------------ epilogue
    mbar_wait(o_done, (n - 1) & 1);
    tc_fence_after();
    float o[DH];
    float c1[kStride], c2[kStride];
#pragma unroll
    for (int c = 0; c < DH / 32; ++c)
        tmem_ld32(lane_base + L::COL_O + half * DH + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&o[c * 32]));
    {
        uint32_t oc[32];
        if (PROT && half == 0) tmem_ld32(lane_base + L::COL_O + D, oc);
        tmem_wait_ld();
#pragma unroll
        for (int x = 0; x < kStride; ++x) {
            c1[x] = (PROT && half == 0) ? __fadd_rn(__uint_as_float(oc[x]), __uint_as_float(oc[16 + x])) : 0.0f;
            c2[x] = (PROT && half == 0) ? __fadd_rn(__uint_as_float(oc[kStride + x]), __uint_as_float(oc[16 + kStride + x])) : 0.0f;
        }
    }
    // denominator: l = l_lo + l_hi, then (protected) range restriction on warps 4-7
    xl[half * 128 + row] = l_half;
    named_bar_sync(kBarEpi, 256);
    float l_run = __fadd_rn(xl[row], xl[128 + row]);
    double eps_mult = 1.0;
    if (PROT && half == 0) {
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
        xpub[row * 4 + 3] = l_run;
    }
    if (PROT) {
        named_bar_sync(kBarEpi, 256);
        l_run = xpub[row * 4 + 3];
    }
#pragma unroll
    for (int c = 0; c < DH; ++c) o[c] = __fdiv_rn(o[c], l_run);
    float fam_out = 0.0f;
    if (PROT) {
        // final strided output check: partial group sums of this half, completed on warps 4-7
        float s1[kStride], s2[kStride];
#pragma unroll
        for (int x = 0; x < kStride; ++x) {
            float a = 0.0f, bb = 0.0f;
#pragma unroll
            for (int g = 0; g < GH; ++g) {
                const float v = o[x + kStride * g];
                a = __fadd_rn(a, v);
                bb = __fadd_rn(bb, __fmul_rn(static_cast<float>(half * GH + g + 1), v));
            }
            s1[x] = a;
            s2[x] = bb;
        }
        if (half == 1) {
#pragma unroll
            for (int x = 0; x < kStride; ++x) { xprod[row * 16 + x] = s1[x]; xprod[row * 16 + 8 + x] = s2[x]; }
        }
        named_bar_sync(kBarEpi, 256);
        bool viol = false, cs_bad = false;
        double res = 0.0;
        if (half == 0) {
#pragma unroll
            for (int x = 0; x < kStride; ++x) {
                c1[x] = __fdiv_rn(c1[x], l_run);
                c2[x] = __fdiv_rn(c2[x], l_run);
                cs_bad |= !isfinite(c1[x]) || !isfinite(c2[x]);
                const float t1 = __fadd_rn(s1[x], xprod[row * 16 + x]);
                const float t2 = __fadd_rn(s2[x], xprod[row * 16 + 8 + x]);
                if (!isfinite(t1) || !isfinite(t2)) { viol = true; continue; }
                const double d1 = static_cast<double>(c1[x]) - t1;
                const double d2 = static_cast<double>(c2[x]) - t2;
                res = fmax(res, fmax(fabs(d1), fabs(d2) / (2 * GH)));
                viol |= fabs(d1) > p.eps2 * eps_mult || fabs(d2) > p.eps2 * eps_mult * (2 * GH);
            }
            fam_out = static_cast<float>(res);
        }
        if (named_bar_or(kBarOr, 256, viol || cs_bad)) {
            // rare: locate / correct over the full row on warps 4-7
            if (half == 1) {
#pragma unroll
                for (int c = 0; c < DH; ++c) scr[DH + c] = o[c];
            }
            named_bar_sync(kBarRare, 256);
            if (half == 0) {
                bool tcs = named_bar_or(4, 128, cs_bad);
                RowVerify rv{};
                rv.best_col = -1;
                rv.restored_col = -1;
                rv.residual = res;
                float full[D];
                for (int c = 0; c < DH; ++c) { full[c] = o[c]; full[DH + c] = scr[DH + c]; }
                if (!tcs && viol) verify_row<D>(full, c1, c2, p.eps2 * eps_mult, rv);
                for (int c = 0; c < DH; ++c) { o[c] = full[c]; scr[DH + c] = full[DH + c]; }
                fam_out = static_cast<float>(rv.residual);
                TileReport tr = reduce_tile_report(rv, tcs, row, rs.slots, rs.ints, rs.dbl);
                if (row == 0)
                    push_event(p, EFTA_OUTPUT_CHECKSUM, head, qt, n, tr.status, tr.row, tr.col,
                               tr.violations, tr.corrections, tr.checksum_repair, tr.residual, tr.delta);
            }
            named_bar_sync(kBarRare, 256);
            if (half == 1) {
#pragma unroll
                for (int c = 0; c < DH; ++c) o[c] = scr[DH + c];
            }
        }
    }
    // store this half's columns
    const size_t grow = static_cast<size_t>(seq_row0) + qt * kBlock + row;
    float4* dst = reinterpret_cast<float4*>(p.o + grow * D + half * DH);
#pragma unroll
    for (int c = 0; c < DH / 4; ++c) dst[c] = make_float4(o[4 * c], o[4 * c + 1], o[4 * c + 2], o[4 * c + 3]);
    if (half == 0) {
        if (p.m_out) p.m_out[grow] = m_run;
        if (p.l_out) p.l_out[grow] = l_run;
        if (PROT) {
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                fam_exp = fmaxf(fam_exp, __shfl_xor_sync(0xffffffffu, fam_exp, off));
                fam_out = fmaxf(fam_out, __shfl_xor_sync(0xffffffffu, fam_out, off));
            }
            if (lane == 0) atomic_max_nonneg(&p.counters->family_max[1], fam_out);
        }
    }
}

}  // namespace efta_sm100
