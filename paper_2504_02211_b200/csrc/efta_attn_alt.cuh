// efta_attn_alt.cuh — alternating row-warpgroup schedule of the CTA-pair EFTA kernel.
//
// Why: with one row warpgroup, each SM sub-partition runs a single softmax warp whose
// chain per key block (TMEM load -> max -> 128 exponentials + strided products -> check
// -> P store) is ~2.1x the tensor-core time of the block (tools/phase_prof.py: row period
// 2729 clk protected vs 1280 clk of MMAs): the MMAs idle half the time and the warp
// itself is latency-bound (issue-active ~37%).
//
// Here two row warpgroups own ALTERNATE key blocks of the same 128 query rows:
// warpgroup w (warps 4+4w .. 7+4w) processes blocks j = w, w+2, ... from S buffer w
// (S is double-buffered by block parity; P has its own TMEM buffer, efta_attn_pair.cuh).
// Each sub-partition now runs two independent softmax warps. The online-softmax
// recurrence (src/efta.cpp:192-260) couples consecutive blocks only through the row
// maxima; those are handed from one warpgroup to the other through shared memory:
//   * early: right after its row max, warpgroup w publishes (m_true, m_run) of block j
//     (the running true max and the lazy reference max P is computed against), so the
//     partner's block j+1 can start its exponentials;
//   * late: after its tile decision (exp-stage check, factor guard and, on a violation,
//     the recovery ladder exp_stage_slow that may repair the max), it publishes the
//     final values. The partner compares them with the early ones it used at the same
//     point of its own block; on a mismatch (only possible after a recovery changed a
//     max) it recomputes its block from the still-resident S with the revised values,
//     which reproduces the sequential recurrence exactly.
// Row sums l and the range lower bound lb are kept per warpgroup, each referenced to
// the warpgroup's own last reference max, and merged at the end of the tile
// (l = l_0 e^{m_0 - m} + l_1 e^{m_1 - m}). O is one TMEM accumulator for both; it is
// rescaled (lazily, kLazyTau) by the warpgroup whose block moved the reference max,
// after P.V of the previous block completed.
//
// Persistent: the warpgroups loop over the cluster's tiles (pair_next_tile); warpgroup 1
// runs block n-1 of a tile, receives warpgroup 0's sums through shared memory (fin_bar)
// and runs the epilogue while warpgroup 0 already starts the next tile.
//
// Barriers: per warpgroup a P-ready and an S-free barrier (4 warps x 2 CTAs), per
// (warpgroup, warp quarter) an early and a late chain barrier (32 arrivals). Named
// barriers: warpgroup 0 uses the single-warpgroup ids 1..7, warpgroup 1 the same +
// kBarAltOfs (9, 10, 11, 14 in the loop; 9, 12, 13, 15 in the epilogue).
// Tile boundary: the chain slots (early / late / lchain), the fin slot and their barriers are
// double-buffered by tile parity, so warpgroup 0 starts tile k+1 while warpgroup 1 still runs
// tile k's last block and epilogue (a single set made warpgroup 0 wait for that hand-over at
// every tile boundary: ~20% of a 16-block tile). For n >= 4 warpgroup 0 cannot reach tile k+2
// before warpgroup 1 has left tile k (its block 2 of tile k+1 waits on warpgroup 1's block 1);
// for n == 2 nothing else bounds it, so block 0 of tile k waits on `ack` of tile k-2 (arrived
// by warpgroup 1 once it has read tile k-2's chain values and fin, at its epilogue).
//
// INJ (fault-tap build, `debug` calls): the same schedule with the reference's explicit op
// sequence (src/efta.cpp:125-257) so every FaultSite can be tapped by the thread owning the
// row: GEMM1_OUT on the scaled score, REDUCE_MAX, SUB_MAX, EXP_OUT, REDUCE_SUM on the running
// denominator, RESCALE_FACTOR / GEMM2_ACC on the O accumulator around the P.V MMAs,
// NORMALIZE_OUT in the epilogue. Rescaling is eager (P always referenced to the running max,
// as in the reference), and the running denominator travels along the chain (lchain) so
// REDUCE_SUM sees the reference's l. A block redone after a chain revision restores the tap's
// evaluation count first (the reference evaluates each block once).
#pragma once
#include "efta_attn_kernel.cuh"
// included by efta_attn_pair.cuh after PairLayout

namespace efta_sm100 {

constexpr uint32_t kBarAltOfs = 8;

struct AltXch {
    float2 early[2][128];  // (m_true, m_run) of the producer warpgroup's last block, fast path
    float2 late[2][128];   // the same after the producer's tile decision / recovery
    float4 fin[128];       // warpgroup 0 -> 1 after the loop: l, lb, m_ref, m_true
    float lchain[2][128];  // INJ: the reference's running denominator after the producer's block
};
static_assert(sizeof(AltXch) == 7168, "PairLayout reserves 7 KB for the chain exchange");

// explicit shared-space loads (a generic pointer would compile to the slower generic LD path)
__device__ __forceinline__ float2 lds_f2(const float2* p) {
    float2 v;
    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(smem_u32(p)) : "memory");
    return v;
}
__device__ __forceinline__ float4 lds_f4(const float4* p) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "r"(smem_u32(p))
                 : "memory");
    return v;
}

// observe_linear (efta.cpp:181-185) on the pair kernel: residual max(|d1|, |d2|/G) of the
// scaled score row against its checksums (c1 from the score MMA, c2 on the CUDA cores)
template <int D>
__device__ __noinline__ float pair_linear_residual(const AttnParams& p, const float* sc, const float* c1s,
                                                   int head, int bi, int j, int row) {
    float c2s[kStride];
    pair_score_c2<D>(p, head, bi, j, row, c2s);
    float lin = 0.0f;
    for (int x = 0; x < kStride; ++x) {
        float a = 0.0f, b = 0.0f;
        for (int l = 0; l < kBlock / kStride; ++l) {
            a = __fadd_rn(a, sc[x + kStride * l]);
            b = __fadd_rn(b, __fmul_rn(static_cast<float>(l + 1), sc[x + kStride * l]));
        }
        const float d1 = fabsf(c1s[x] - a);
        const float d2 = fabsf(c2s[x] - b) / static_cast<float>(kBlock / kStride);
        lin = fmaxf(lin, fmaxf(d1, d2));
    }
    return lin;
}

template <int D, bool PROT, bool INJ, bool CAUSAL>
__device__ __forceinline__ void row_alt(const AttnParams& p, uint8_t* red, AltXch* xc, float* ostage,
                                        const CUtensorMap* tm_o, uint64_t* s_full,
                                        uint64_t* s_free, uint64_t* p_ready, uint64_t* o_done, uint64_t* o_final,
                                        uint64_t* mx_early, uint64_t* mx_late, uint64_t* fin_bar, uint64_t* ack_bar,
                                        uint64_t* o_free, uint32_t tmem, int warp, int lane, int n,
                                        const int* tinfo, uint64_t* t_full, uint64_t* t_empty, uint32_t rank) {
    using L = PairLayout<D, PROT>;
    static_assert(!INJ || PROT, "the fault-tap build is the protected variant");
    constexpr int MODE = PROT ? EFTA_MODE_EFTA_OPT : EFTA_MODE_NONE;
    constexpr bool kWideTmem = (!PROT || D == 64) && !INJ;
    // d=128 O store: the coalesced staged stores (default) or 16-row TMA boxes (A/B: +2% at S=2048,
    // -0.4% at C4 and -1.5% causal, profiles/r02/ab_d128_tma_ostore.log)
    constexpr bool kTmaStore128 = EFTA_TMA_STORE_D128 != 0;
    const int w = (warp - 4) >> 2;
    const int wq = warp & 3;
    const int row = wq * 32 + lane;
    const uint32_t bo = w ? kBarAltOfs : 0u;
    const uint32_t lane_base = tmem + (static_cast<uint32_t>(wq * 32) << 16);
    RowScratch rs;
    {
        uint8_t* r = red + w * L::RED_BYTES;
        rs.slots = reinterpret_cast<RowSlot*>(r);
        rs.ints = reinterpret_cast<int*>(r + 128 * sizeof(RowSlot));
        rs.dbl = reinterpret_cast<double*>(r + 128 * sizeof(RowSlot) + 16 * sizeof(int));
    }
    ThreadTap tap{};  // INJ: this row's fault spec of the current tile
    AltXch* const xcb = xc;  // [tile parity]
    const float scale = p.scale, scale_log2 = p.scale_log2;
    const uint32_t s_addr = lane_base + L::COL_S0 + w * L::SW;
    const uint32_t cs_addr = s_addr + 128;  // c1_hi (8) | c1_lo (8)
    float fam_exp = 0.0f, fam_lin = 0.0f;  // INJ observation: worst clean exp / linear residuals
    // per-family worst clean residuals, flushed per tile (nothing extra stays live across tiles)
    auto flush_families = [&](float fam_out) {
        if (!PROT) return;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            fam_out = fmaxf(fam_out, __shfl_xor_sync(0xffffffffu, fam_out, off));
            if (INJ) {
                fam_exp = fmaxf(fam_exp, __shfl_xor_sync(0xffffffffu, fam_exp, off));
                fam_lin = fmaxf(fam_lin, __shfl_xor_sync(0xffffffffu, fam_lin, off));
            }
        }
        if (lane == 0) {
            if (w == 1) atomic_max_nonneg(&p.counters->family_max[1], fam_out);
            if (INJ) {
                atomic_max_nonneg(&p.counters->family_max[0], fam_exp);
                if (p.observe_linear) atomic_max_nonneg(&p.counters->family_max[2], fam_lin);
            }
        }
        fam_exp = 0.0f;
        fam_lin = 0.0f;
    };

    // persistent: the (head, query-pair) tiles this cluster draws from the tile ring; every barrier phase runs on the
    // global block counter g = k*n + j (n is even, so block parity = warpgroup)
    int it = 0;  // this warpgroup's block counter across tiles (= g >> 1)
    int g_base = 0;                // global block counter at this tile's block 0
    int ph_cnt[2] = {0, 0};        // blocks per warpgroup in the earlier tiles of each parity
    for (int k = 0;; ++k) {
    const int u = pair_next_tile(tinfo, t_full, t_empty, k, true);
    if (u < 0) break;
    const PairTile tt = pair_tile<CAUSAL>(p, u);
    const int head = tt.head, qt = 2 * tt.pair + static_cast<int>(rank);
    const int nt = tt.nblk;  // key blocks of this tile (causal: up to the pair's diagonal)
    // this tile's chain slots and barriers (tile parity); each barrier completes one phase per
    // block of its warpgroup in the tiles of this parity
    const int par = k & 1;
    xc = xcb + par;
    uint64_t* my_early = mx_early + par * 8 + w * 4 + wq;
    uint64_t* my_late = mx_late + par * 8 + w * 4 + wq;
    uint64_t* pa_early = mx_early + par * 8 + (1 - w) * 4 + wq;
    uint64_t* pa_late = mx_late + par * 8 + (1 - w) * 4 + wq;
    const int ph0 = ph_cnt[par];
    ph_cnt[par] += nt / 2;
    const int seq_row0 = head * p.seq_len;
    if constexpr (INJ) tap.load(p, head, qt, row);
    // own sums, referenced to m_ref (the reference max of this warpgroup's last block);
    // INJ: l_w is the reference's full running denominator (lchain)
    float l_w = 0.0f, lb_w = 0.0f, m_ref = -CUDART_INF_F, m_true_last = -CUDART_INF_F;
    for (int j = w; j < nt; j += 2, ++it) {
        const int g = g_base + j;
        if ((warp & 3) == 0) EFTA_TS(0, g);
        mbar_wait(&s_full[w], it & 1);
        if ((warp & 3) == 0) EFTA_TS(1, g);
        EFTA_TSQ(8, g);
        tc_fence_after();
        const uint32_t pph = static_cast<uint32_t>(ph0 + ((j - 1) >> 1)) & 1u;  // partner's phase for block j-1
        const int tap_snap = tap.count;
        float pv[kBlock];
        // P packed to fp16x2 for the P.V MMA. The fast build packs inside the exp loop, so the
        // fp32 row dies there (pv = S, pk = P: 192 live registers otherwise); its rare path
        // rebuilds the fp32 P from the still-resident S (exp_rebuild)
        uint32_t pk[64];
        float m_true_prev = -CUDART_INF_F, m_run_prev = -CUDART_INF_F;
        float m_true, m_new, bm, psum_f = 0.0f;
        bool replaced_p = false;
        // causal (fast build only): the diagonal block j == qt shows keys 0..row, a block past
        // it (rank 0's last block of the pair) shows none; uniform per CTA
        const bool masked = CAUSAL && !INJ && j >= qt;
        const int mfrom = !masked ? kBlock : (j == qt ? row + 1 : 0);  // first masked key column
        for (int attempt = 0;; ++attempt) {
            uint32_t csr[16];
            // one x128 load where it pays (A/B: unprotected d=128 +4.7%, protected d=64 +2.8%);
            // the protected d=128 variant keeps four x32 loads (the x128 form spills there, -1.5%)
            if constexpr (kWideTmem) {
                tmem_ld128(s_addr, *reinterpret_cast<uint32_t(*)[128]>(&pv[0]));
            } else {
#pragma unroll
                for (int c4 = 0; c4 < 4; ++c4)
                    tmem_ld32(s_addr + c4 * 32, *reinterpret_cast<uint32_t(*)[32]>(&pv[c4 * 32]));
            }
            if (PROT) tmem_ld16(cs_addr, csr);
            tmem_wait_ld();
            if (PROT) {
#pragma unroll
                for (int x = 0; x < kStride; ++x)
                    csr[x] = __float_as_uint(__fadd_rn(__uint_as_float(csr[x]), __uint_as_float(csr[kStride + x])));
            }
            int sc_fault_col = -1;
            float sc_fault_val = 0.0f;
            if (masked) {
                // causal: keys past the row's last visible one are masked (P = 0). The exp-stage
                // check then covers each group's visible cells: the product of their P against
                // exp(scale * c1_vis - n_vis * m), c1_vis = c1 minus the masked cells' scores
                if (PROT) {
#pragma unroll
                    for (int x = 0; x < kStride; ++x) {
                        float cm = 0.0f;
#pragma unroll
                        for (int l = 0; l < kBlock / kStride; ++l)
                            if (x + kStride * l >= mfrom) cm = __fadd_rn(cm, pv[x + kStride * l]);
                        csr[x] = __float_as_uint(__fsub_rn(__uint_as_float(csr[x]), cm));
                    }
                }
#pragma unroll
                for (int c = 0; c < kBlock; ++c) pv[c] = (c < mfrom) ? pv[c] : -CUDART_INF_F;
            }
            if constexpr (INJ) {
                // reference order: S = scale * (Q K^T) [GEMM1_OUT], row max + bias, running max [REDUCE_MAX]
                tap.count = tap_snap;
#pragma unroll
                for (int c = 0; c < kBlock; ++c) pv[c] = __fmul_rn(pv[c], scale);
                if (tap.hit(EFTA_GEMM1_OUT, j) && tap.col < kBlock) {
                    sc_fault_col = tap.col;
                    sc_fault_val = tap.fire(p, sel_get<kBlock>(pv, sc_fault_col));
                    sel_set<kBlock>(pv, sc_fault_col, sc_fault_val);
                }
                if (p.observe_linear && attempt == 0) {
                    float c1s[kStride];
#pragma unroll
                    for (int x = 0; x < kStride; ++x) c1s[x] = __fmul_rn(__uint_as_float(csr[x]), scale);
                    const float lin = pair_linear_residual<D>(p, pv, c1s, head, qt, j, row);
                    if (isfinite(lin)) fam_lin = fmaxf(fam_lin, lin);
                }
                float b = pv[0];
#pragma unroll
                for (int c = 1; c < kBlock; ++c) b = (b < pv[c]) ? pv[c] : b;
                bm = b + p.rowmax_bias;
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
            }
            // ---- the max chain: block j-1 belongs to the partner warpgroup
            if (j > 0) {
                if (attempt == 0) {
                    mbar_wait(pa_early, pph);
                    const float2 c = lds_f2(&xc->early[1 - w][row]);
                    m_true_prev = c.x;
                    m_run_prev = c.y;
                } else {
                    const float2 c = lds_f2(&xc->late[1 - w][row]);
                    m_true_prev = c.x;
                    m_run_prev = c.y;
                }
            }
            m_true = (m_true_prev < bm) ? bm : m_true_prev;
            if constexpr (INJ) {
                m_new = m_true;  // eager: P is always referenced to the running max
                if (tap.hit(EFTA_REDUCE_MAX, j) && tap.col == 0) m_new = tap.fire(p, m_new);
                m_true = m_new;
            } else {
                m_new = (j == 0 || m_true - m_run_prev > kLazyTau) ? m_true : m_run_prev;
            }
            if (attempt == 0) {
                // tile boundary (n == 2 only binds): warpgroup 1 has consumed tile k-2's slots
                if (w == 0 && j == 0 && k >= 2)
                    mbar_wait(&ack_bar[par * 4 + wq], static_cast<uint32_t>((k >> 1) - 1) & 1u);
                xc->early[w][row] = make_float2(m_true, m_new);
                mbar_arrive(my_early);
            }
            if ((warp & 3) == 0) EFTA_TS(15, g);
            EFTA_TSQ(4, g);
            float pc1v[kStride];
            float2 prod_f[kStride / 2];
            if (PROT) {
                const float g16m = 16.0f * m_new;
#pragma unroll
                for (int x = 0; x < kStride; ++x) {
                    // visible cells of group x: l < ceil((mfrom - x) / 8), at most 16
                    const float gm = masked ? static_cast<float>(min(kBlock / kStride, max(0, (mfrom - x + kStride - 1) / kStride))) * m_new
                                            : g16m;
                    pc1v[x] = ex2_approx(__fsub_rn(__fmul_rn(__uint_as_float(csr[x]), scale), gm) * kLog2e);
                }
            }
            float2 ps0 = make_float2(0.0f, 0.0f), ps1 = make_float2(0.0f, 0.0f);
            if constexpr (INJ) {
                // P = exp(S - m) with the SUB_MAX / EXP_OUT taps (src/efta.cpp:161-170)
#pragma unroll
                for (int c = 0; c < kBlock; ++c) pv[c] = __fsub_rn(pv[c], m_new);
                tap_row<kBlock>(tap, p, EFTA_SUB_MAX, j, pv);
#pragma unroll
                for (int c = 0; c < kBlock; ++c) pv[c] = ex2_approx(pv[c] * kLog2e);
                tap_row<kBlock>(tap, p, EFTA_EXP_OUT, j, pv);
#pragma unroll
                for (int c = 0; c < kBlock; c += 2) {
                    const float2 e = make_float2(pv[c], pv[c + 1]);
                    if ((c >> 1) & 1) ps1 = fadd2(ps1, e);
                    else ps0 = fadd2(ps0, e);
                    const int gg = (c & 7) >> 1;
                    prod_f[gg] = (c < kStride) ? e : fmul2(prod_f[gg], e);
                }
            } else if (masked) {
                // the same exponentials; masked cells give P = 0 and stay out of the group products
                const float mL = m_new * kLog2e;
                const float2 sl2 = make_float2(scale_log2, scale_log2), nm2 = make_float2(-mL, -mL);
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
                    e.x = (c < mfrom) ? e.x : 0.0f;
                    e.y = (c + 1 < mfrom) ? e.y : 0.0f;
                    pk[c >> 1] = pack_half2(e.x, e.y);
                    if ((c >> 1) & 1) ps1 = fadd2(ps1, e);
                    else ps0 = fadd2(ps0, e);
                    if (PROT) {
                        const float2 ep = make_float2((c < mfrom) ? e.x : 1.0f, (c + 1 < mfrom) ? e.y : 1.0f);
                        const int gg = (c & 7) >> 1;
                        prod_f[gg] = (c < kStride) ? ep : fmul2(prod_f[gg], ep);
                    }
                }
            } else {
                const float mL = m_new * kLog2e;
                const float2 sl2 = make_float2(scale_log2, scale_log2), nm2 = make_float2(-mL, -mL);
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
                    pk[c >> 1] = pack_half2(e.x, e.y);
                    if ((c >> 1) & 1) ps1 = fadd2(ps1, e);
                    else ps0 = fadd2(ps0, e);
                    if (PROT) {
                        const int gg = (c & 7) >> 1;
                        prod_f[gg] = (c < kStride) ? e : fmul2(prod_f[gg], e);
                    }
                }
            }
            psum_f = (ps0.x + ps0.y) + (ps1.x + ps1.y);
            if (!PROT) break;  // no recovery path: the chain can never be revised

            // ---- exp-domain strided product check (see row_wg) + factor guard. A row is
            // degenerate where the reference's log test is undefined: P or Pc1 not finite and
            // positive (snvr.cpp:18,55-66), read off the group products
            const float f = ex2_approx((m_run_prev - m_new) * kLog2e);
            bool exp_affected = false;
            int exp_viol = 0;
            bool degenerate = !isfinite(m_new);
            float exp_res = 0.0f;
#pragma unroll
            for (int x = 0; x < kStride; ++x) {
                const float pr = (x & 1) ? prod_f[x >> 1].y : prod_f[x >> 1].x;
                const float pc1 = pc1v[x];
                // strict bounds: P = Pc1 = 0 and P = Pc1 = inf fail them like every other
                // degenerate group; a tie at a finite bound has measure zero
                const bool bad = !(pr > pc1 * p.exp_lo && pr < pc1 * p.exp_hi);
                if constexpr (INJ) {
                    if (!(pr > 0.0f && pr < CUDART_INF_F) || !(pc1 > 0.0f && pc1 < CUDART_INF_F))
                        degenerate = true;
                    else
                        exp_res = fmaxf(exp_res, fabsf(lg2_approx(__fdividef(pr, pc1))) * kLn2);
                }
                if (bad) { exp_affected = true; ++exp_viol; }
            }
            if (degenerate) { exp_affected = true; exp_res = CUDART_INF_F; exp_viol = 1; }
            if (INJ && attempt == 0 && isfinite(exp_res)) fam_exp = fmaxf(fam_exp, exp_res);
            const bool factor_bad = (j > 0) && !(f > 0.0f && f <= 1.0f);
            // ---- late chain check: did the partner's decision revise block j-1's maxima?
            bool chain_bad = false;
            if (j > 0) {
                if ((warp & 3) == 0) EFTA_TS(8, g);
                if (attempt == 0) mbar_wait(pa_late, pph);
                const float2 c = lds_f2(&xc->late[1 - w][row]);
                chain_bad = __float_as_uint(c.x) != __float_as_uint(m_true_prev) ||
                            __float_as_uint(c.y) != __float_as_uint(m_run_prev);
            }
            if ((warp & 3) == 0) EFTA_TS(9, g);
            EFTA_TSQ(0, g);
            if (!named_bar_or(6 + bo, 128, exp_affected || factor_bad || chain_bad)) break;
            if (named_bar_or(6 + bo, 128, chain_bad)) continue;  // redo the block with the revised maxima
            // ---- rare: the reference recovery ladder for this tile
            if constexpr (!INJ) {
                // the event's first-look residual: inf for a degenerate row (snvr.cpp:55-66)
#pragma unroll
                for (int x = 0; x < kStride; ++x) {
                    const float pr = (x & 1) ? prod_f[x >> 1].y : prod_f[x >> 1].x;
                    if (!(pr > 0.0f && pr < CUDART_INF_F) || !(pc1v[x] > 0.0f && pc1v[x] < CUDART_INF_F))
                        degenerate = true;
                }
                if (degenerate) { exp_res = CUDART_INF_F; exp_viol = 1; }
            }
            float p_loc[kBlock];
            if constexpr (INJ) {
#pragma unroll
                for (int c = 0; c < kBlock; ++c) p_loc[c] = pv[c];
            } else {
                // the fast path's fp32 P, rebuilt bit for bit from S (same fma, same exp split)
                const float mL = m_new * kLog2e;
                uint32_t r[32];
#pragma unroll
                for (int c4 = 0; c4 < 4; ++c4) {
                    tmem_ld32(s_addr + c4 * 32, r);
                    tmem_wait_ld();
#pragma unroll
                    for (int x = 0; x < 32; ++x) {
                        const int c = c4 * 32 + x;
                        p_loc[c] = (c < mfrom) ? ex2_col<D>(c, fmaf(__uint_as_float(r[x]), scale_log2, -mL)) : 0.0f;
                    }
                }
            }
            int replaced = 0;
            exp_stage_slow<INJ, D, true>(p, s_addr, cs_addr, head, qt, j, row, exp_affected, exp_res, exp_viol,
                                         m_run_prev, m_new, bm, p_loc, replaced, tap, sc_fault_col, sc_fault_val,
                                         rs, bo, mfrom);
            if (replaced) {
                if constexpr (INJ) {
#pragma unroll
                    for (int c = 0; c < kBlock; ++c) pv[c] = p_loc[c];
                } else {
                    // repack, and re-sum with the fast path's pairing
#pragma unroll
                    for (int x = 0; x < 64; ++x) pk[x] = pack_half2(p_loc[2 * x], p_loc[2 * x + 1]);
                    float2 ps0 = make_float2(p_loc[0], p_loc[1]), ps1 = make_float2(p_loc[2], p_loc[3]);
#pragma unroll
                    for (int c = 4; c < kBlock; c += 4) {
                        ps0 = fadd2(ps0, make_float2(p_loc[c], p_loc[c + 1]));
                        ps1 = fadd2(ps1, make_float2(p_loc[c + 2], p_loc[c + 3]));
                    }
                    psum_f = (ps0.x + ps0.y) + (ps1.x + ps1.y);
                }
            }
            replaced_p = replaced != 0;
            m_true = (m_true_prev < m_new) ? m_new : m_true_prev;
            if (INJ) m_true = m_new;
            break;
        }
        // the partial row sum of P (re-summed with the fast path's pairing after a recompute)
        auto row_psum = [&]() {
            if (!INJ || !replaced_p) return psum_f;  // the fast build re-summed in its rare path
            float2 ps0 = make_float2(pv[0], pv[1]), ps1 = make_float2(pv[2], pv[3]);
#pragma unroll
            for (int c = 4; c < kBlock; c += 4) {
                ps0 = fadd2(ps0, make_float2(pv[c], pv[c + 1]));
                ps1 = fadd2(ps1, make_float2(pv[c + 2], pv[c + 3]));
            }
            return (ps0.x + ps0.y) + (ps1.x + ps1.y);
        };
        if constexpr (INJ) {
            // the reference's running denominator l = f * l_prev + rowsum(P) [REDUCE_SUM]
            // (src/efta.cpp:244-250); l_prev is the partner's, read under the late barrier
            const float f_l = ex2_approx((m_run_prev - m_new) * kLog2e);
            const float lprev = (j > 0) ? xc->lchain[1 - w][row] : 0.0f;
            float lv = __fadd_rn(__fmul_rn(f_l, lprev), row_psum());
            if (tap.hit(EFTA_REDUCE_SUM, j) && tap.col == 0) lv = tap.fire(p, lv);
            l_w = lv;
            xc->lchain[w][row] = lv;
        }
        // publish first: the partner's next block and the score MMA of block j+2 wait on these
        if (PROT) {
            xc->late[w][row] = make_float2(m_true, m_new);
            mbar_arrive(my_late);
        }
        // S_j is no longer read: the score MMA of block j+2 may overwrite S[w]
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(&s_free[w], 0);
        if ((warp & 3) == 0) EFTA_TS(2, g);
        // ---- factors: fo for the shared O accumulator (chain), fw for this warpgroup's sums
        const float fo = ex2_approx((m_run_prev - m_new) * kLog2e);
        const float fw = ex2_approx((m_ref - m_new) * kLog2e);
        if (PROT) lb_w = __fadd_rn(__fmul_rn(lb_w, fw), ex2_approx((bm - m_new) * kLog2e));
        if constexpr (!INJ) l_w = __fadd_rn(__fmul_rn(fw, l_w), row_psum());

        if ((warp & 3) == 0) EFTA_TS(3, g);
        // ---- P (fp16): packed first, stored once the P buffer is free (P.V of block j-1
        // with one shared buffer, of block j-2 with one buffer per warpgroup)
        if constexpr (INJ) {
#pragma unroll
            for (int x = 0; x < 64; ++x) pk[x] = pack_half2(pv[2 * x], pv[2 * x + 1]);
        }
        bool need_o = j > 0 && !__all_sync(0xffffffffu, fo == 1.0f);
        // INJ: the O accumulator taps of this block force the rescale pass: GEMM2_ACC of block
        // j-1 (after its P.V), RESCALE_FACTOR of block j, and of block 0 (deferred to block 1:
        // P.V(0) overwrites the accumulator, so the tapped zero is added after it)
        bool t_res0 = false;
        if constexpr (INJ) {
            const bool t_acc = j > 0 && tap.active && tap.site == EFTA_GEMM2_ACC && tap.bj == j - 1;
            const bool t_res = j > 0 && tap.active && tap.site == EFTA_RESCALE_FACTOR && tap.bj == j;
            t_res0 = j == 1 && tap.active && tap.site == EFTA_RESCALE_FACTOR && tap.bj == 0;
            need_o = need_o || __any_sync(0xffffffffu, t_acc || t_res || t_res0);
        }
        if (L::NPB == 1 ? (g > 0) : (g >= 2 || need_o)) {
            if ((warp & 3) == 0) EFTA_TS(4, g);
            if (L::NPB == 1 || need_o)
                mbar_wait(&o_done[1 - w], static_cast<uint32_t>((g - 1) >> 1) & 1u);
            else
                mbar_wait(&o_done[w], static_cast<uint32_t>((g - 2) >> 1) & 1u);
            if ((warp & 3) == 0) EFTA_TS(5, g);
            tc_fence_after();
        }
        if constexpr (kWideTmem) {
            tmem_st64(lane_base + L::COL_P + w * (L::NPB - 1) * 64, pk);
        } else {
            tmem_st32(lane_base + L::COL_P + w * (L::NPB - 1) * 64, *reinterpret_cast<uint32_t(*)[32]>(&pk[0]));
            tmem_st32(lane_base + L::COL_P + w * (L::NPB - 1) * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(&pk[32]));
        }
        // ---- O *= fo (lazy: only when this block moved the reference max of some row);
        // P.V of block j-1 is complete (waited above)
        if (need_o) {
            constexpr int NCH = D / 32 + (PROT ? 1 : 0);
            float o[NCH * 32];
#pragma unroll
            for (int c = 0; c < NCH; ++c)
                tmem_ld32(lane_base + L::COL_O + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&o[c * 32]));
            tmem_wait_ld();
            if constexpr (INJ) {
                if (t_res0 && tap.hit(EFTA_RESCALE_FACTOR, 0) && tap.col < D)
                    sel_set<D>(o, tap.col, __fadd_rn(sel_get<D>(o, tap.col), tap.fire(p, 0.0f)));
                tap_row<D>(tap, p, EFTA_GEMM2_ACC, j - 1, o);
            }
            const float2 f2 = make_float2(fo, fo);
#pragma unroll
            for (int x = 0; x < NCH * 32; x += 2) {
                const float2 r2 = fmul2(make_float2(o[x], o[x + 1]), f2);
                o[x] = r2.x;
                o[x + 1] = r2.y;
            }
            if constexpr (INJ) tap_row<D>(tap, p, EFTA_RESCALE_FACTOR, j, o);
#pragma unroll
            for (int c = 0; c < NCH; ++c)
                tmem_st32(lane_base + L::COL_O + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&o[c * 32]));
        }
        tmem_wait_st();
        tc_fence_before();
        signal_p_ready<true>(&p_ready[w], lane);
        if ((warp & 3) == 0) EFTA_TS(6, g);
        EFTA_TSQ(12, g);
        m_ref = m_new;
        m_true_last = m_true;
    }

    // ------------------------------------------------ hand-over: warpgroup 0 -> 1
    // Warpgroup 1 ran the tile's last block (n is even): it merges the sums and runs the
    // epilogue while warpgroup 0 already starts the next tile.
    const int g_last = g_base + nt - 1;
    g_base += nt;
    if (w == 0) {
        xc->fin[row] = make_float4(INJ ? 0.0f : l_w, lb_w, m_ref, m_true_last);
        mbar_arrive(&fin_bar[par * 4 + wq]);
        if (INJ) flush_families(0.0f);
        continue;
    }
    if ((warp & 3) == 0) EFTA_TS(32, g_last);
    mbar_wait(&fin_bar[par * 4 + wq], static_cast<uint32_t>(k >> 1) & 1u);
    if ((warp & 3) == 0) EFTA_TS(33, g_last);
    const float4 fb = lds_f4(&xc->fin[row]);
    mbar_arrive(&ack_bar[par * 4 + wq]);  // this tile's chain and fin slots are consumed
    float m_run = m_ref;  // the chain's final reference max (block n-1 is ours)
    const float m_true = m_true_last;
    const float fbf = ex2_approx((fb.z - m_run) * kLog2e);
    float l_run = __fadd_rn(l_w, __fmul_rn(fb.x, fbf));
    float lb = __fadd_rn(lb_w, __fmul_rn(fb.y, fbf));

    // ------------------------------------------------ epilogue (as row_wg, warpgroup 1)
    mbar_wait(o_final, static_cast<uint32_t>(k) & 1u);
    if ((warp & 3) == 0) EFTA_TS(34, g_last);
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
    // O is in registers: the next tile's first P.V may overwrite the accumulator
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive_cluster(o_free, 0);
    if ((warp & 3) == 0) EFTA_TS(35, g_last);
    EFTA_TSW(52, g_last);
    if constexpr (INJ) tap_row<D>(tap, p, EFTA_GEMM2_ACC, n - 1, o);
    {
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
    double eps_mult = 1.0;
    bool range_bad = false;
    double range_viol = 0.0;
    if (PROT) {
        // denominator range restriction (snvr.cpp:161-182, efta.cpp:289-310); per row here, its
        // tile event is emitted with the output check (one warpgroup barrier for a clean tile)
        const float upper = static_cast<float>(p.seq_len);
        // the fast build forms P as ex2(fma(S, scale*log2e, -m*log2e)) (and partly on the FMA
        // pipe), so the max cell's P can sit an ulp below the bound's exp(bm - m) = 1: a row whose
        // sum is that single term (causal row 0) would be "restricted" by rounding alone. The
        // comparison allows 2^-21 relative there; the tap build keeps the reference's exact test.
        const float lb_cmp = INJ ? lb : __fmul_rn(lb, 1.0f - 0x1p-21f);
        range_bad = !isfinite(l_run) || l_run < lb_cmp || l_run > upper;
        if (range_bad) {
            range_viol = !isfinite(l_run) ? CUDART_INF
                                          : (l_run < lb ? static_cast<double>(lb) - l_run
                                                        : static_cast<double>(l_run) - upper);
            l_run = lb;
            eps_mult = static_cast<double>(p.seq_len) / static_cast<double>(l_run);
        }
    }
    // the range restriction's tile event (warpgroup-wide, only if some row was restricted)
    auto range_event = [&]() {
        if (row == 0) { rs.ints[0] = 0; rs.ints[1] = 0x7fffffff; rs.dbl[0] = 0.0; }
        wg_sync(bo);
        if (range_bad) {
            atomicAdd(&rs.ints[0], 1);
            atomicMin(&rs.ints[1], row);
            unsigned long long* a = reinterpret_cast<unsigned long long*>(&rs.dbl[0]);
            unsigned long long old = *a, assumed;
            do {
                assumed = old;
                if (__longlong_as_double(assumed) >= range_viol) break;
                old = atomicCAS(a, assumed, __double_as_longlong(range_viol));
            } while (old != assumed);
        }
        wg_sync(bo);
        if (row == 0) {
            atomicAdd(&p.counters->range_replacements, rs.ints[0]);
            push_event(p, EFTA_ROWSUM_RANGE, head, qt, n, EFTA_CORRECTED, rs.ints[1], -1, 0, rs.ints[0], 0,
                       rs.dbl[0], 0.0);
        }
        wg_sync(bo);
    };
    // d=128: the range event right away (A/B: the fused barrier below measured -0.9% at C4)
    if constexpr (D != 64) {
        if (PROT && named_bar_or(7 + bo, 128, range_bad)) range_event();
    }
    if ((warp & 3) == 0) EFTA_TS(36, g_last);
    EFTA_TSW(56, g_last);
    // normalization (efta.cpp:312-327): one IEEE reciprocal, then products (within 1 ulp of
    // the reference's division); the tap build keeps the reference's division [NORMALIZE_OUT]
    if constexpr (INJ) {
#pragma unroll
        for (int c = 0; c < D; ++c) o[c] = __fdiv_rn(o[c], l_run);
        tap_row<D>(tap, p, EFTA_NORMALIZE_OUT, 0, o);
#pragma unroll
        for (int x = 0; x < kStride; ++x) { c1[x] = __fdiv_rn(c1[x], l_run); c2[x] = __fdiv_rn(c2[x], l_run); }
    } else {
        const float rl = __frcp_rn(l_run);
#pragma unroll
        for (int c = 0; c < D; c += 2) {
            const float2 r2 = fmul2(make_float2(o[c], o[c + 1]), make_float2(rl, rl));
            o[c] = r2.x;
            o[c + 1] = r2.y;
        }
        if (PROT) {
#pragma unroll
            for (int x = 0; x < kStride; ++x) { c1[x] = __fmul_rn(c1[x], rl); c2[x] = __fmul_rn(c2[x], rl); }
        }
    }
    float fam_out = 0.0f;
    if ((warp & 3) == 0) EFTA_TS(40, g_last);
    EFTA_TSW(48, g_last);
    if (PROT) {
        float res;
        if constexpr (D == 64)  // one warpgroup barrier for a clean tile (+2% at S=512, d=64)
            verify_output_tile_pre<D>(p, o, c1, c2, p.eps2 * eps_mult, head, qt, n, row, rs, res, bo, range_bad,
                                      range_event, g_last);
        else
            verify_output_tile<D>(p, o, c1, c2, p.eps2 * eps_mult, head, qt, n, row, rs, res, bo);
        if (isfinite(res)) fam_out = res;
    }
    if ((warp & 3) == 0) EFTA_TS(37, g_last);
    const size_t grow = static_cast<size_t>(seq_row0) + qt * kBlock + row;
    if constexpr (D == 64) {
        // asynchronous O store: the warp writes its 32 rows into its 8 KB staging buffer in
        // the 128-byte-swizzled box layout (16-byte chunk c of row r at chunk c ^ (r & 7):
        // conflict-free) and one lane hands it to the TMA engine, so warpgroup 1 leaves the
        // epilogue without waiting for the stores (the d=64 epilogue sits on the max chain at
        // every tile boundary). fp32 [BH*S, 64]: two 32-column boxes; fp16 token-major
        // [B*S, H*64]: one 64-column box.
        uint8_t* wbuf = reinterpret_cast<uint8_t*>(ostage) + wq * 8192;
        if (lane == 0) bulk_wait_group_read0();  // this warp's previous tile store has read its buffer
        __syncwarp();
        const uint32_t sw = static_cast<uint32_t>(lane & 7);
        if (p.o_tok) {
#pragma unroll
            for (int c = 0; c < 8; ++c)
                st_shared_v4(wbuf + lane * 128 + ((c ^ sw) << 4),
                             make_uint4(pack_half2(o[8 * c], o[8 * c + 1]), pack_half2(o[8 * c + 2], o[8 * c + 3]),
                                        pack_half2(o[8 * c + 4], o[8 * c + 5]), pack_half2(o[8 * c + 6], o[8 * c + 7])));
        } else {
#pragma unroll
            for (int b = 0; b < 2; ++b)
#pragma unroll
                for (int c = 0; c < 8; ++c)
                    st_shared_v4(wbuf + b * 4096 + lane * 128 + ((c ^ sw) << 4),
                                 make_uint4(__float_as_uint(o[32 * b + 4 * c]), __float_as_uint(o[32 * b + 4 * c + 1]),
                                            __float_as_uint(o[32 * b + 4 * c + 2]), __float_as_uint(o[32 * b + 4 * c + 3])));
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
            if (p.o_tok) {
                const int b = head / p.heads_q, h = head - b * p.heads_q;
                tma_store_2d(tm_o, wbuf, h * 64, b * p.seq_len + qt * kBlock + wq * 32);
            } else {
                const int r0 = seq_row0 + qt * kBlock + wq * 32;
                tma_store_2d(tm_o, wbuf, 0, r0);
                tma_store_2d(tm_o, wbuf + 4096, 32, r0);
            }
            bulk_commit_group();
        }
    } else if constexpr (!kTmaStore128) {
        // coalesced O store: thread = row holds D fp32; the warp stages 32 rows x 16 words at
        // a time through shared memory (16-byte chunks XOR-swizzled by row: conflict-free both
        // ways) and writes them back as full 64-byte row segments, 8 rows per instruction
        // (a row per thread made every 16-byte store touch 32 lines: an LSU-bound epilogue).
        // A word is one fp32 value ([BH, S, D] output) or two fp16 values (token-major
        // [B, S, H, D] output: row r of the warp lands at token b*S + s, head column h*D).
        uint32_t* stg = reinterpret_cast<uint32_t*>(ostage) + wq * 512;
        uint8_t* obase;  // row 0 of this warp
        size_t opitch;
        if (p.o_tok) {
            const int b = head / p.heads_q, h = head - b * p.heads_q;
            const size_t tok0 = static_cast<size_t>(b) * p.seq_len + qt * kBlock + row - lane;
            obase = reinterpret_cast<uint8_t*>(p.o) + ((tok0 * p.heads_q + h) * D) * 2;
            opitch = static_cast<size_t>(p.heads_q) * D * 2;
        } else {
            obase = reinterpret_cast<uint8_t*>(p.o + (grow - lane) * D);
            opitch = D * 4;
        }
        auto put = [&](int q4, uint4 w4) {
            *reinterpret_cast<uint4*>(stg + lane * 16 + ((q4 ^ (lane & 3)) << 2)) = w4;
        };
        auto flush = [&](int c) {  // the staged 32 x 64-byte block -> 64-byte segment c of each row
            __syncwarp();
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int r = 8 * i + (lane >> 2), q4 = lane & 3;
                const uint4 v = *reinterpret_cast<const uint4*>(stg + r * 16 + ((q4 ^ (r & 3)) << 2));
                *reinterpret_cast<uint4*>(obase + static_cast<size_t>(r) * opitch + c * 64 + 16 * q4) = v;
            }
            __syncwarp();
        };
        if (p.o_tok) {
#pragma unroll
            for (int c = 0; c < D / 32; ++c) {
#pragma unroll
                for (int q4 = 0; q4 < 4; ++q4) {
                    const int b0 = c * 32 + 8 * q4;
                    put(q4, make_uint4(pack_half2(o[b0], o[b0 + 1]), pack_half2(o[b0 + 2], o[b0 + 3]),
                                       pack_half2(o[b0 + 4], o[b0 + 5]), pack_half2(o[b0 + 6], o[b0 + 7])));
                }
                flush(c);
            }
        } else {
#pragma unroll
            for (int c = 0; c < D / 16; ++c) {
#pragma unroll
                for (int q4 = 0; q4 < 4; ++q4)
                    put(q4, make_uint4(__float_as_uint(o[c * 16 + 4 * q4]), __float_as_uint(o[c * 16 + 4 * q4 + 1]),
                                       __float_as_uint(o[c * 16 + 4 * q4 + 2]), __float_as_uint(o[c * 16 + 4 * q4 + 3])));
                flush(c);
            }
        }
    } else {
        // (EFTA_TMA_STORE_D128=1 builds) d=128: the same asynchronous store in 16-row boxes (32 rows x 512 bytes per warp do not
        // fit next to the K / V rings): box (rh, cb) = rows 16 rh.. of the warp, 128-byte column
        // block cb, staged through L::OBUF_N 2 KB buffers per warp; a buffer is rewritten once
        // the TMA engine has read it (wait_group.read OBUF_N - 1)
        constexpr int NB = L::OBUF_N;
        uint8_t* wb = reinterpret_cast<uint8_t*>(ostage) + wq * NB * 2048;
        const uint32_t sw = static_cast<uint32_t>(lane & 7);
        uint8_t* rowp0 = wb + (lane & 15) * 128;
        // box kb: wait for its buffer, the rows' 8 chunks (lanes of row half rh), TMA store
        auto box = [&](int kb, int rh, int col, int grow0, auto chunk) {
            if (lane == 0) bulk_wait_group_read<NB - 1>();
            __syncwarp();
            if ((lane >> 4) == rh) {
#pragma unroll
                for (int c = 0; c < 8; ++c) st_shared_v4(rowp0 + (kb % NB) * 2048 + ((c ^ sw) << 4), chunk(c));
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
                tma_store_2d(tm_o, wb + (kb % NB) * 2048, col, grow0 + 16 * rh);
                bulk_commit_group();
            }
        };
        if (p.o_tok) {
            const int b = head / p.heads_q, h = head - b * p.heads_q;
            const int t0 = b * p.seq_len + qt * kBlock + wq * 32;
#pragma unroll
            for (int rh = 0; rh < 2; ++rh)
#pragma unroll
                for (int cb = 0; cb < 2; ++cb)
                    box(rh * 2 + cb, rh, h * 128 + 64 * cb, t0, [&](int c) {
                        const int b0 = 64 * cb + 8 * c;
                        return make_uint4(pack_half2(o[b0], o[b0 + 1]), pack_half2(o[b0 + 2], o[b0 + 3]),
                                          pack_half2(o[b0 + 4], o[b0 + 5]), pack_half2(o[b0 + 6], o[b0 + 7]));
                    });
        } else {
            const int r0 = seq_row0 + qt * kBlock + wq * 32;
#pragma unroll
            for (int rh = 0; rh < 2; ++rh)
#pragma unroll
                for (int cb = 0; cb < 4; ++cb)
                    box(rh * 4 + cb, rh, 32 * cb, r0, [&](int c) {
                        const int b0 = 32 * cb + 4 * c;
                        return make_uint4(__float_as_uint(o[b0]), __float_as_uint(o[b0 + 1]), __float_as_uint(o[b0 + 2]),
                                          __float_as_uint(o[b0 + 3]));
                    });
        }
    }
    if (p.m_out) p.m_out[grow] = m_run;
    if (p.l_out) p.l_out[grow] = l_run;
    if ((warp & 3) == 0) EFTA_TS(38, g_last);
    flush_families(fam_out);
    if ((warp & 3) == 0) EFTA_TS(39, g_last);
    }  // tiles
    if (w == 1 && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // O stores done
    (void)MODE;
    (void)tm_o;
}

}  // namespace efta_sm100
