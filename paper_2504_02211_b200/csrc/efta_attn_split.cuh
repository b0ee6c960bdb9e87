// efta_attn_split.cuh — split-row softmax schedule of the CTA-pair EFTA kernel.
//
// Why: with one 128-row query tile per SM and one row warpgroup, each SM
// sub-partition runs a single softmax warp whose dependency chain (row max ->
// 128 exponentials -> sums/products -> P store) is ~1.9x the tensor-core time of
// the tile (tools/phase_prof.py): the MMAs idle half the time. Here two row
// warpgroups share the tile's 128 rows (the TMEM accumulator holds all of them,
// so no extra TMEM): warps 4-7 ("half 0") own score columns 0..63, warps 8-11
// ("half 1") columns 64..127 of the same rows (warp w reads TMEM lanes
// 32*(w%4)..+31). Every SM sub-partition now runs two softmax warps, each with half
// the chain.
//
// Per key block j the two warps of a row slice (w, w+4) exchange through shared
// memory, synchronised by a 64-thread named barrier private to that pair:
//   * their partial row maxima (the reference row max, efta.cpp:150-160, is the max
//     of the two; max is order-free so bm is bit-identical to one warpgroup's);
//   * (protected) the partial strided products of P for the partner's groups:
//     half 0 completes the exp-domain check of groups x = 0..3, half 1 of 4..7
//     (snvr.cpp:52-83 as the product bracket, see efta_attn_kernel.cuh).
// One 256-thread barrier.red.or per block decides whether the tile takes the rare
// recovery ladder (exp_stage_slow over the full rows, run by half 0 with half 1's
// columns handed over through a per-SM global scratch row). It sits right before
// the P-ready arrival, where every warp has to meet the MMA issuer anyway.
// Row sums stay per half (l = l_0 + l_1 at the end, both halves use the same lazy
// reference max so the same factors apply). PV(j-1) is only waited for when O
// actually has to be rescaled (lazy rescale, kLazyTau).
//
// Used by the fast variants (NONE / EFTA_OPTIMIZED) of efta_attn_pair_kernel; the
// fault-tap and per-iteration-check variants keep the single-warpgroup row_wg.
#pragma once
#include "efta_attn_kernel.cuh"

namespace efta_sm100 {

__device__ __forceinline__ uint32_t sm_id() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
    return r;
}

constexpr int kRowWarp0 = 3;  // first row warp of the pair kernel (warps 3..10)

// named barrier ids of the split schedule (0 = __syncthreads, 1..7 = half-0 helpers)
constexpr uint32_t kBarPair0 = 8;   // 8..11: per row slice (warps w, w+4), 64 threads
constexpr uint32_t kBarTile = 12;   // all 256 row threads
constexpr uint32_t kBarRare = 13;   // all 256 row threads, rare paths

// shared exchange area (floats): xmax[2][2][128] | xprod[2][2][128][4] | xpub[128][4] | xl[2][128]
struct SplitXch {
    static constexpr int XMAX = 0, XPROD = 512, XPUB = 512 + 2048, XL = 512 + 2048 + 512;
    static constexpr int FLOATS = 512 + 2048 + 512 + 256;
    static constexpr uint32_t BYTES = FLOATS * 4;
};

// Row warps: copy 128 query rows (from global row q_row0) into the TMEM A-operand columns
// (fp16 pairs, column x = dims 2x, 2x+1); half h stages dims [D/2*h, D/2*(h+1)).
template <int D>
__device__ __forceinline__ void stage_q_rows(const AttnParams& p, uint32_t col_q_addr, int warp, int lane,
                                             int q_row0) {
    const int half = (warp - kRowWarp0) >> 2, wq = warp & 3, row = wq * 32 + lane;
    const uint32_t lane_base = col_q_addr + (static_cast<uint32_t>(wq * 32) << 16);
    const uint4* src = reinterpret_cast<const uint4*>(p.q + (static_cast<size_t>(q_row0) + row) * D + half * (D / 2));
    constexpr int W = D / 4;  // 32-bit columns per half
    uint32_t w[W];
#pragma unroll
    for (int i = 0; i < W / 4; ++i) {
        const uint4 u = __ldg(src + i);
        w[4 * i] = u.x;
        w[4 * i + 1] = u.y;
        w[4 * i + 2] = u.z;
        w[4 * i + 3] = u.w;
    }
    if constexpr (W == 32) tmem_st32(lane_base + half * W, w);
    else tmem_st16(lane_base + half * W, w);
    tmem_wait_st();
}

template <bool PAIR>
__device__ __forceinline__ void split_signal_p_ready(uint64_t* bar, int lane) {
    __syncwarp();
    if (lane == 0) {
        if constexpr (PAIR) mbar_arrive_cluster(bar, 0);  // the pair leader's barrier
        else mbar_arrive(bar);
    }
}

// TL: TMEM plan (COL_S0, S_STRIDE, COL_O); the score checksum columns are the pair
// layout (cols 128..135 c1_hi, 136..143 c1_lo).
// Rare exp-stage ladder of one (i, j) tile for the split schedule: both halves have
// dumped their 64 P values of the row into the per-SM scratch row; half 0 runs the
// reference ladder (exp_stage_slow) over the full rows and publishes the repaired max,
// block max and a replaced flag through xpub (P rows rewritten in the scratch).
template <int D>
__device__ __noinline__ float2 split_exp_rare(const AttnParams& p, uint32_t s_addr, uint32_t cs_addr, int head,
                                              int qt, int j, int row, int half, bool exp_affected, int exp_viol,
                                              float m_run, float m_new, float bm, float* xpub,
                                              const RowScratch& rs) {
    float* scr = p.scratch + static_cast<size_t>(sm_id()) * (128 * 128) + row * 128;
    if (half == 1) {
        xpub[row * 4 + 0] = exp_affected ? 1.0f : 0.0f;
        xpub[row * 4 + 1] = static_cast<float>(exp_viol);
    }
    named_bar_sync(kBarRare, 256);
    if (half == 0) {
        const bool aff = exp_affected || xpub[row * 4 + 0] != 0.0f;
        const int viol = exp_viol + static_cast<int>(xpub[row * 4 + 1]);
        float p_loc[kBlock];
        for (int c = 0; c < kBlock; ++c) p_loc[c] = scr[c];
        int replaced = 0;
        ThreadTap no_tap{};
        exp_stage_slow<false, D>(p, s_addr, cs_addr, head, qt, j, row, aff, isfinite(m_new) ? 0.0f : CUDART_INF_F,
                                 viol, m_run, m_new, bm, p_loc, replaced, no_tap, -1, 0.0f, rs);
        if (replaced) {
            for (int c = 0; c < kBlock; ++c) scr[c] = p_loc[c];
        }
        xpub[row * 4 + 0] = m_new;
        xpub[row * 4 + 1] = bm;
        xpub[row * 4 + 2] = replaced ? 1.0f : 0.0f;
    }
    named_bar_sync(kBarRare, 256);
    return make_float2(xpub[row * 4 + 0], xpub[row * 4 + 1]);
}

// Rare final output correction (verify_locate_correct on O, abft.cpp:65-187) for the split
// schedule: both halves have dumped their normalised O columns into the per-SM scratch
// row; half 0 verifies / corrects the full rows in place and reports the tile event.
template <int D>
__device__ __noinline__ float split_out_rare(const AttnParams& p, int head, int qt, int n, int row, int half,
                                             bool viol, bool cs_bad, double res, const float* c1, const float* c2,
                                             double eps_mult, const RowScratch& rs) {
    float* scr = p.scratch + static_cast<size_t>(sm_id()) * (128 * 128) + row * 128;
    named_bar_sync(kBarRare, 256);
    float fam_out = static_cast<float>(res);
    if (half == 0) {
        const bool tcs = named_bar_or(4, 128, cs_bad);
        RowVerify rv{};
        rv.best_col = -1;
        rv.restored_col = -1;
        rv.residual = res;
        float full[D], cc1[kStride], cc2[kStride];
        for (int c = 0; c < D; ++c) full[c] = scr[c];
        for (int x = 0; x < kStride; ++x) { cc1[x] = c1[x]; cc2[x] = c2[x]; }
        if (!tcs && viol) verify_row<D>(full, cc1, cc2, p.eps2 * eps_mult, rv);
        for (int c = 0; c < D; ++c) scr[c] = full[c];
        fam_out = static_cast<float>(rv.residual);
        TileReport tr = reduce_tile_report(rv, tcs, row, rs.slots, rs.ints, rs.dbl);
        if (row == 0)
            push_event(p, EFTA_OUTPUT_CHECKSUM, head, qt, n, tr.status, tr.row, tr.col, tr.violations,
                       tr.corrections, tr.checksum_repair, tr.residual, tr.delta);
    }
    named_bar_sync(kBarRare, 256);
    return fam_out;
}

// One (head, query tile) work item of a persistent CTA. g0: global key-block counter of
// this item's j = 0 (ring / barrier phases run on across items); next_q_row (>= 0): first
// global query row of the next item, staged into TMEM once every score MMA of this item has
// completed (so the next item's first score MMAs overlap this epilogue); o_free: arrived on once O
// has been read out of TMEM (the next item's first P.V may overwrite it). p_ready is
// the pair [2] indexed by block parity.
template <int D, int MODE, bool PAIR, class TL>
__device__ __forceinline__ void row_split(const AttnParams& p, uint64_t* s_full, uint64_t* p_ready,
                                          uint64_t* o_done, uint64_t* o_free, uint32_t tmem, int warp,
                                          int lane, int head, int qt, int n, int seq_row0, int g0,
                                          const RowScratch& rs, float* xch, int next_q_row,
                                          uint64_t* q_ready) {
    using L = TL;
    constexpr bool PROT = MODE != EFTA_MODE_NONE;
    constexpr int DH = D / 2;          // O columns per half
    constexpr int GH = DH / kStride;   // output groups per half
    const int half = (warp - kRowWarp0) >> 2;  // warp-uniform
    const int wq = warp & 3;
    const int row = wq * 32 + lane;
    const uint32_t bar_pair = kBarPair0 + wq;
    const uint32_t lane_base = tmem + (static_cast<uint32_t>(wq * 32) << 16);
    const int c0 = half * 64;
    float* xmax = xch + SplitXch::XMAX;
    float* xprod = xch + SplitXch::XPROD;
    float* xpub = xch + SplitXch::XPUB;
    float* xl = xch + SplitXch::XL;
    // per-SM scratch row of the rare paths (computed there: keeps the hot loop's registers free)
#define EFTA_SCR (p.scratch + static_cast<size_t>(sm_id()) * (128 * 128) + row * 128)
    const float scale = p.scale, scale_log2 = p.scale_log2;
    // m_run: the max P is referenced to (lazy); m_true: the running row max (reference m)
    float m_run = -CUDART_INF_F, m_true = -CUDART_INF_F, l_half = 0.0f, lb = 0.0f;

    // values of block j carried from the hot loop into its tail (and the rare ladder)
    float pv[64];
    float bm = 0.0f, m_true_before = 0.0f, m_new = 0.0f, f = 0.0f, psum = 0.0f;
    bool exp_affected = false;
    int exp_viol = 0;
    // tail of block j: P store, denominators, lazy O correction, P-ready
    auto finish_block = [&](int j) {
        const int g = g0 + j;
        const int b = g & 1;
        const uint32_t s_addr = lane_base + L::COL_S0 + b * L::S_STRIDE;
        // ---- P (fp16) over this half's score columns (after the ladder: it re-reads S)
        {
            uint32_t pk[32];
#pragma unroll
            for (int x = 0; x < 32; ++x) pk[x] = pack_half2(pv[2 * x], pv[2 * x + 1]);
            tmem_st32(s_addr + half * 32, pk);
        }
        if (warp == 4) EFTA_TS(3, j);
        // ---- rescale factor, lower bound, denominator (efta.cpp:192-242)
        if (PROT) lb = __fadd_rn(__fmul_rn(lb, f), ex2_approx((bm - m_new) * kLog2e));
        l_half = __fadd_rn(__fmul_rn(f, l_half), psum);
        // ---- O correction: O *= f on this half's columns (+ checksum columns on half 0);
        // only when some row of the warp moved its reference max (lazy rescale)
        if (j > 0 && !__all_sync(0xffffffffu, f == 1.0f)) {
            if (warp == 4) EFTA_TS(4, j);
            mbar_wait(o_done, (g - 1) & 1);
            tc_fence_after();
            constexpr int NO = DH / 32;
            constexpr int NCH = NO + (PROT ? 1 : 0);
            float o[NCH][32];
#pragma unroll
            for (int c = 0; c < NO; ++c)
                tmem_ld32(lane_base + L::COL_O + half * DH + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&o[c][0]));
            if (PROT) tmem_ld16(lane_base + L::COL_O + D + half * 16, *reinterpret_cast<uint32_t(*)[16]>(&o[NO][0]));
            tmem_wait_ld();
            const float2 f2 = make_float2(f, f);
#pragma unroll
            for (int c = 0; c < NCH; ++c)
#pragma unroll
                for (int x = 0; x < 32; x += 2) {
                    if (c == NO && x >= 16) break;
                    const float2 r2 = fmul2(make_float2(o[c][x], o[c][x + 1]), f2);
                    o[c][x] = r2.x;
                    o[c][x + 1] = r2.y;
                }
#pragma unroll
            for (int c = 0; c < NO; ++c)
                tmem_st32(lane_base + L::COL_O + half * DH + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&o[c][0]));
            if (PROT) tmem_st16(lane_base + L::COL_O + D + half * 16, *reinterpret_cast<uint32_t(*)[16]>(&o[NO][0]));
        }
        tmem_wait_st();
        tc_fence_before();
        split_signal_p_ready<PAIR>(&p_ready[g & 1], lane);
        if (warp == 4) EFTA_TS(6, j);
        m_run = m_new;
    };
    // The hot loop leaves (break) when a tile takes the rare ladder, so the out-of-line
    // ladder call sits outside it and does not shape the loop's register allocation.
    int j = 0;
    for (;;) {
        bool rare = false;
        for (; j < n; ++j) {
            const int g = g0 + j;
            const int b = g & 1;
            const uint32_t s_addr = lane_base + L::COL_S0 + b * L::S_STRIDE;
            const uint32_t cs_addr = s_addr + 128;
            if (warp == 4) EFTA_TS(0, j);
            mbar_wait(&s_full[b], (g >> 1) & 1);
            if (warp == 4) EFTA_TS(1, j);
            tc_fence_after();
    #ifdef EFTA_MMA_ONLY  // experiment build: tensor-pipe / operand-feed bound of the schedule
            if (true) { split_signal_p_ready<PAIR>(&p_ready[g & 1], lane); continue; }
    #endif
            tmem_ld32(s_addr + c0, *reinterpret_cast<uint32_t(*)[32]>(&pv[0]));
            tmem_ld32(s_addr + c0 + 32, *reinterpret_cast<uint32_t(*)[32]>(&pv[32]));
            tmem_wait_ld();
            // ---- row max: partial over this half, exchanged within the row slice
            float mx0 = pv[0], mx1 = pv[1], mx2 = pv[2], mx3 = pv[3];
    #pragma unroll
            for (int c = 4; c < 64; c += 4) {
                mx0 = fmaxf(mx0, pv[c]);
                mx1 = fmaxf(mx1, pv[c + 1]);
                mx2 = fmaxf(mx2, pv[c + 2]);
                mx3 = fmaxf(mx3, pv[c + 3]);
            }
            float* xm = xmax + b * 256;  // double-buffered by parity: the partner may still read j-1
            xm[half * 128 + row] = fmaxf(fmaxf(mx0, mx1), fmaxf(mx2, mx3));
            named_bar_sync(bar_pair, 64);
            const float mx = fmaxf(xm[row], xm[128 + row]);
            bm = __fmul_rn(mx, scale) + p.rowmax_bias;
            m_true_before = m_true;
            m_true = (m_true < bm) ? bm : m_true;
            m_new = (j == 0 || m_true - m_run > kLazyTau) ? m_true : m_run;
            const float mL = m_new * kLog2e;
            // ---- exponentials (MUFU + FMA-pipe polynomial), fused row sum and group products
            const float2 sl2 = make_float2(scale_log2, scale_log2), nm2 = make_float2(-mL, -mL);
            float2 ps0 = make_float2(0.0f, 0.0f), ps1 = make_float2(0.0f, 0.0f);
            float2 prod[4];
    #pragma unroll
            for (int c = 0; c < 64; c += 2) {
                const float2 a = ffma2(make_float2(pv[c], pv[c + 1]), sl2, nm2);
                float2 e;
                if (exp_on_fma(c)) {  // c0 is a multiple of 16: same column split as row_wg
                    e = ex2_poly2(a);
                } else {
                    e.x = ex2_approx(a.x);
                    e.y = ex2_approx(a.y);
                }
                pv[c] = e.x;
                pv[c + 1] = e.y;
                if ((c >> 1) & 1) ps1 = fadd2(ps1, e);
                else ps0 = fadd2(ps0, e);
            }
            if (PROT) {  // strided group products of P (after the loop: fewer live registers in it)
    #pragma unroll
                for (int c = 0; c < 64; c += 2) {
                    const int g = (c & 7) >> 1;
                    const float2 e = make_float2(pv[c], pv[c + 1]);
                    prod[g] = (c < kStride) ? e : fmul2(prod[g], e);
                }
            }
            if (warp == 4) EFTA_TS(8, j);
            f = ex2_approx((m_run - m_new) * kLog2e);
            bool factor_bad = false;
            exp_affected = false;
            exp_viol = 0;
            if (PROT) {
                // c1 (hi, lo) of this half's checked groups x = 4*half .. 4*half+3 (loaded after the
                // exponentials: keeps them out of the loop's register footprint)
                uint32_t c1h[4], c1l[4];
                tmem_ld4(cs_addr + 4 * half, c1h);
                tmem_ld4(cs_addr + 8 + 4 * half, c1l);
                // hand the partner the partial products of its groups, complete our own
                float* xp = xprod + b * 1024;
                const float4 send = half == 0 ? make_float4(prod[2].x, prod[2].y, prod[3].x, prod[3].y)
                                              : make_float4(prod[0].x, prod[0].y, prod[1].x, prod[1].y);
                *reinterpret_cast<float4*>(&xp[(half * 128 + row) * 4]) = send;
                tmem_wait_ld();
                float pc1v[4];  // Pc1 = exp(scale*c1 - 16 m)
                {
                    const float g16m = 16.0f * m_new;
    #pragma unroll
                    for (int x = 0; x < 4; ++x) {
                        const float c1 = __fadd_rn(__uint_as_float(c1h[x]), __uint_as_float(c1l[x]));
                        pc1v[x] = ex2_approx(__fsub_rn(__fmul_rn(c1, scale), g16m) * kLog2e);
                    }
                }
                named_bar_sync(bar_pair, 64);
                if (warp == 4) EFTA_TS(5, j);
                const float4 rv = *reinterpret_cast<const float4*>(&xp[((1 - half) * 128 + row) * 4]);
                const float2 own0 = half == 0 ? prod[0] : prod[2], own1 = half == 0 ? prod[1] : prod[3];
                const float pr[4] = {own0.x * rv.x, own0.y * rv.y, own1.x * rv.z, own1.y * rv.w};
    #pragma unroll
                for (int x = 0; x < 4; ++x)
                    if (!(pr[x] >= pc1v[x] * p.exp_lo && pr[x] <= pc1v[x] * p.exp_hi)) { exp_affected = true; ++exp_viol; }
                if (!isfinite(m_new)) { exp_affected = true; exp_viol = 1; }
                if (j > 0) factor_bad = !(f > 0.0f && f <= 1.0f);  // NaN fails both
            }
            psum = (ps0.x + ps0.y) + (ps1.x + ps1.y);
            const bool tile_trig = PROT && named_bar_or(kBarTile, 256, exp_affected || factor_bad);
            if (warp == 4) EFTA_TS(7, j);
            if (tile_trig) {
                rare = true;
                break;
            }
            finish_block(j);
        }
        if (!rare) break;
        {
            const int g = g0 + j;
            const int b = g & 1;
            const uint32_t s_addr = lane_base + L::COL_S0 + b * L::S_STRIDE;
            const uint32_t cs_addr = s_addr + 128;
                // ---- rare: exp-stage ladder + factor guard over the full rows (out of line: the
                // row halves go through the per-SM scratch so P stays in registers here)
    #pragma unroll
                for (int c = 0; c < 64; ++c) EFTA_SCR[half * 64 + c] = pv[c];
    #ifdef EFTA_NO_RARE_CALL
                const float2 mb = make_float2(m_new, bm); __trap();
    #else
                const float2 mb = split_exp_rare<D>(p, s_addr, cs_addr, head, qt, j, row, half, exp_affected, exp_viol,
                                                    m_run, m_new, bm, xpub, rs);
    #endif
                m_new = mb.x;
                bm = mb.y;
                if (xpub[row * 4 + 2] != 0.0f) {
    #pragma unroll
                    for (int c = 0; c < 64; ++c) pv[c] = EFTA_SCR[half * 64 + c];
                    float2 q0 = make_float2(pv[0], pv[1]), q1 = make_float2(pv[2], pv[3]);
    #pragma unroll
                    for (int c = 4; c < 64; c += 4) {
                        q0 = fadd2(q0, make_float2(pv[c], pv[c + 1]));
                        q1 = fadd2(q1, make_float2(pv[c + 2], pv[c + 3]));
                    }
                    psum = (q0.x + q0.y) + (q1.x + q1.y);
                }
                // the recovered reference max is the row's true max so far
                m_true = (m_true_before < m_new) ? m_new : m_true_before;
                f = ex2_approx((m_run - m_new) * kLog2e);
        }
        finish_block(j);
        ++j;
    }

    if (next_q_row >= 0) {  // stage the next item's Q: every score MMA of this item has completed
        stage_q_rows<D>(p, tmem + TL::COL_Q, warp, lane, next_q_row);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
            if constexpr (PAIR) mbar_arrive_cluster(q_ready, 0);
            else mbar_arrive(q_ready);
        }
    }
    // ------------------------------------------------------------------ epilogue
    mbar_wait(o_done, (g0 + n - 1) & 1);
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
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {  // O is in registers: the next item's first P.V may overwrite it
            if constexpr (PAIR) mbar_arrive_cluster(o_free, 0);
            else mbar_arrive(o_free);
        }
#pragma unroll
        for (int x = 0; x < kStride; ++x) {
            c1[x] = (PROT && half == 0) ? __fadd_rn(__uint_as_float(oc[x]), __uint_as_float(oc[16 + x])) : 0.0f;
            c2[x] = (PROT && half == 0) ? __fadd_rn(__uint_as_float(oc[kStride + x]), __uint_as_float(oc[16 + kStride + x]))
                                        : 0.0f;
        }
    }
    {
        // bring O, its checksums, l and the lower bound from the lazy reference max to the
        // row's true max (the reference's final m); F == 1 for most rows
        const float F = ex2_approx((m_run - m_true) * kLog2e);
        if (!__all_sync(0xffffffffu, F == 1.0f)) {
#pragma unroll
            for (int c = 0; c < DH; ++c) o[c] = __fmul_rn(o[c], F);
#pragma unroll
            for (int x = 0; x < kStride; ++x) { c1[x] = __fmul_rn(c1[x], F); c2[x] = __fmul_rn(c2[x], F); }
            l_half = __fmul_rn(l_half, F);
            lb = __fmul_rn(lb, F);
        }
        m_run = m_true;
    }
    // denominator: l = l_0 + l_1, then (protected) range restriction on half 0
    xl[half * 128 + row] = l_half;
    named_bar_sync(bar_pair, 64);
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
        named_bar_sync(bar_pair, 64);
        l_run = xpub[row * 4 + 3];
    }
#pragma unroll
    for (int c = 0; c < DH; ++c) o[c] = __fdiv_rn(o[c], l_run);
    float fam_out = 0.0f;
    if (PROT) {
        // final strided output check: partial group sums of this half, completed on half 0
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
        // 16 floats per row in the row's own product-exchange slots (slice-private)
        auto xs = [&](int k) -> float& { return xprod[(k >> 3) * 1024 + ((k >> 2) & 1) * 512 + row * 4 + (k & 3)]; };
        if (half == 1) {
#pragma unroll
            for (int x = 0; x < kStride; ++x) { xs(x) = s1[x]; xs(8 + x) = s2[x]; }
        }
        named_bar_sync(bar_pair, 64);
        bool viol = false, cs_bad = false;
        double res = 0.0;
        if (half == 0) {
#pragma unroll
            for (int x = 0; x < kStride; ++x) {
                c1[x] = __fdiv_rn(c1[x], l_run);
                c2[x] = __fdiv_rn(c2[x], l_run);
                cs_bad |= !isfinite(c1[x]) || !isfinite(c2[x]);
                const float t1 = __fadd_rn(s1[x], xs(x));
                const float t2 = __fadd_rn(s2[x], xs(8 + x));
                if (!isfinite(t1) || !isfinite(t2)) { viol = true; continue; }
                const double d1 = static_cast<double>(c1[x]) - t1;
                const double d2 = static_cast<double>(c2[x]) - t2;
                res = fmax(res, fmax(fabs(d1), fabs(d2) / (2 * GH)));
                viol |= fabs(d1) > p.eps2 * eps_mult || fabs(d2) > p.eps2 * eps_mult * (2 * GH);
            }
            fam_out = static_cast<float>(res);
        }
        if (named_bar_or(kBarTile, 256, viol || cs_bad)) {
            // rare: locate / correct over the full rows (out of line, rows via the scratch)
#pragma unroll
            for (int c = 0; c < DH; ++c) EFTA_SCR[half * DH + c] = o[c];
            const float fo = split_out_rare<D>(p, head, qt, n, row, half, viol, cs_bad, res, c1, c2, eps_mult, rs);
            if (half == 0) fam_out = fo;
#pragma unroll
            for (int c = 0; c < DH; ++c) o[c] = EFTA_SCR[half * DH + c];
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
            for (int off = 16; off > 0; off >>= 1)
                fam_out = fmaxf(fam_out, __shfl_xor_sync(0xffffffffu, fam_out, off));
            if (lane == 0) atomic_max_nonneg(&p.counters->family_max[1], fam_out);
        }
    }
}

}  // namespace efta_sm100
