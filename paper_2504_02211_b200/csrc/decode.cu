// decode.cu — EFTA for one query row per head against a key/value cache (KV-cache decode).
//
// Not a reference feature (SPEC.md:141,356 list KV-cache decode as a non-goal; SURVEY.md §8(f)
// F4), but the reference algorithm restricted to one query row: efta_forward's rows are
// independent (src/efta.cpp:125-336 loops each query row over the key blocks), so a decode step is
// row 0 of efta_forward(q, K, V) and the oracle checks it exactly that way.
//
// Decode is HBM-bound (one pass over the cache, ~2 FLOP per byte): no tensor cores. One CTA per
// query head walks the cache in 128-key blocks with the reference's eager online softmax
// (src/efta.cpp:192-260) and EFTA-optimized checks:
//   * scores s_t = q . K_t (thread t = key t, fp32 FMA in ascending head-dim order), and the
//     block's strided score checksums c1/c2 = q . KC (the checksum prepass's hi/lo rows of
//     sum_l K[x+8l], src/abft.cpp:19-42 over the block's keys);
//   * exp-stage check (src/efta.cpp:161-189, snvr.cpp:43-159): per group x the product of the 16 P
//     values against exp(scale*c1 - 16 m); on a violation the reference ladder on the row (linear
//     repair of the scores with c1/c2, recompute from m_old, re-scan);
//   * rescale-factor guard (efta.cpp:192-230), rowsum range restriction (snvr.cpp:161-182);
//   * O and its strided checksums O.c1/O.c2 accumulate separately: O += P . V (thread = output
//     column, coalesced V rows), the checksums += P . VC with VC = the prepass's per-key sums of V
//     (sum_g V[key][x+8g], hi+lo); the final output check (verify_locate_correct on the row,
//     efta.cpp:312-336) compares the two after the normalisation.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <string>

#include "efta_attn.cuh"
#include "efta_attn_kernel.cuh"

using namespace efta_sm100;

namespace {

constexpr int DT = 128;  // threads: one per key of a block

__device__ __forceinline__ int rv_status(const RowVerify& rv) {
    if (rv.nonfinite) return EFTA_NONFINITE;
    if (rv.uncorrectable) return EFTA_DETECTED_UNCORRECTABLE;
    return (rv.corrections > 0 || rv.checksum_repair) ? EFTA_CORRECTED : EFTA_CLEAN;
}

// Epilogue of one query row (thread 0; efta.cpp:289-336): rowsum range restriction, O / l and
// the checksums / l, final output check (verify_locate_correct on the row), m / l out. orow / ocs
// hold the unnormalised O and its propagated checksums (shared memory); the normalised row is
// written back to orow.
template <int D, bool PROT>
__device__ void decode_epilogue(const AttnParams& p, int head, float m_run, float l, float lb, float* orow,
                                const float* ocs) {
    const int n = p.nblk;
    double eps_mult = 1.0;
    if (PROT) {
        const float upper = static_cast<float>(p.seq_len);
        // 2^-21: the fast path's P of the max cell can sit an ulp below exp(bm - m) (alt.cuh)
        const bool bad = !isfinite(l) || l < __fmul_rn(lb, 1.0f - 0x1p-21f) || l > upper;
        if (bad) {
            const double viol = !isfinite(l) ? CUDART_INF : (l < lb ? double(lb) - l : double(l) - upper);
            l = lb;
            eps_mult = static_cast<double>(p.seq_len) / static_cast<double>(l);
            atomicAdd(&p.counters->range_replacements, 1);
            push_event(p, EFTA_ROWSUM_RANGE, head, 0, n, EFTA_CORRECTED, 0, -1, 0, 1, 0, viol, 0.0);
        }
    }
    const float rl = __frcp_rn(l);
    float ov[D], c1[kStride], c2[kStride];
    for (int c = 0; c < D; ++c) ov[c] = __fmul_rn(orow[c], rl);
    if (PROT) {
        for (int x = 0; x < kStride; ++x) {
            c1[x] = __fmul_rn(ocs[x], rl);
            c2[x] = __fmul_rn(ocs[kStride + x], rl);
        }
        RowVerify rv{};
        rv.best_col = -1;
        rv.restored_col = -1;
        bool cs_bad = false;
        for (int x = 0; x < kStride; ++x) cs_bad |= !isfinite(c1[x]) || !isfinite(c2[x]);
        if (cs_bad) {
            push_event(p, EFTA_OUTPUT_CHECKSUM, head, 0, n, EFTA_NONFINITE, 0, -1, 0, 0, 0, CUDART_INF, 0.0);
        } else {
            verify_row<D>(ov, c1, c2, p.eps2 * eps_mult, rv);
            const int st = rv_status(rv);
            if (rv.residual == rv.residual)
                atomic_max_nonneg(&p.counters->family_max[1], static_cast<float>(rv.residual));
            if (st != EFTA_CLEAN)
                push_event(p, EFTA_OUTPUT_CHECKSUM, head, 0, n, st, 0, rv.best_col, rv.violations, rv.corrections,
                           rv.checksum_repair, rv.residual, rv.best_delta);
        }
    }
    for (int c = 0; c < D; ++c) orow[c] = ov[c];
    if (p.m_out) p.m_out[head] = m_run;
    if (p.l_out) p.l_out[head] = l;
}

// Split-KV (flash-decoding): a query row's key blocks are shared by `nsplit` CTAs; each leaves
// (m, l, lb, O[D], O.c[16]) in `part`, and the combine kernel merges them in split order.
constexpr int kPartHdr = 3;

template <int D, bool PROT>
__global__ void __launch_bounds__(DT, 4) efta_decode_kernel(AttnParams p, const __half* __restrict__ q,
                                                         const __half* __restrict__ k,
                                                         const __half* __restrict__ v,
                                                         const __half* __restrict__ kc,
                                                         const __half* __restrict__ vc, float* __restrict__ part,
                                                         int nsplit) {
    __shared__ float qs[D];
    __shared__ float ps[kBlock];        // P of the block
    __shared__ float scs[kBlock];       // scaled scores of the block (rare path)
    __shared__ float red[DT / 32];
    __shared__ float cs[2 * kStride];   // c1, c2 of the block's scores (scaled)
    __shared__ float prod[kStride];
    __shared__ float bcast[4];
    __shared__ float orow[D];
    __shared__ float ocs[2 * kStride];
    __shared__ float cpart[8][2 * kStride];   // score-checksum partials per head-dim slice
    __shared__ float opart[DT / 32][2 * kStride];  // output-checksum partials per warp (epilogue)
    const int head = blockIdx.y, split = blockIdx.x, t = threadIdx.x, lane = t & 31, wq = t >> 5;
    const int kvh = kv_head(p, head), n = p.nblk;
    const int j0 = static_cast<int>((static_cast<long long>(n) * split) / nsplit);
    const int j1 = static_cast<int>((static_cast<long long>(n) * (split + 1)) / nsplit);
    const float scale = p.scale;
    for (int c = t; c < D; c += DT) qs[c] = __half2float(q[static_cast<size_t>(head) * D + c]);
    __syncthreads();

    float m_run = -CUDART_INF_F, l_run = 0.0f, lb = 0.0f;
    float o_acc = 0.0f;                  // thread c < D: O[c]
    float oc_acc[2 * kStride];           // thread t: key t's share of O.c1 (x < 8) / O.c2 (x - 8)
#pragma unroll
    for (int x = 0; x < 2 * kStride; ++x) oc_acc[x] = 0.0f;
    const size_t kv0 = static_cast<size_t>(kvh) * p.seq_len;
    auto block_max = [&](float x) {
        for (int o = 16; o; o >>= 1) x = fmaxf(x, __shfl_xor_sync(0xffffffffu, x, o));
        if (lane == 0) red[wq] = x;
        __syncthreads();
        float r = red[0];
        for (int w = 1; w < DT / 32; ++w) r = fmaxf(r, red[w]);
        __syncthreads();
        return r;
    };
    auto block_sum = [&](float x) {
        for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        if (lane == 0) red[wq] = x;
        __syncthreads();
        float r = red[0];
        for (int w = 1; w < DT / 32; ++w) r += red[w];
        __syncthreads();
        return r;
    };

    for (int j = j0; j < j1; ++j) {
        // ---- scores (thread t = key t) and their checksums (threads 0..15)
        const __half* kr = k + (kv0 + static_cast<size_t>(j) * kBlock + t) * D;
        float s = 0.0f;
#pragma unroll 4
        for (int c8 = 0; c8 < D / 8; ++c8) {
            const uint4 raw = reinterpret_cast<const uint4*>(kr)[c8];
            const __half* hv = reinterpret_cast<const __half*>(&raw);
#pragma unroll
            for (int e = 0; e < 8; ++e) s = fmaf(qs[c8 * 8 + e], __half2float(hv[e]), s);
        }
        const float sc = __fmul_rn(s, scale);
        if (PROT) {
            // c1 (rows 0..7) / c2 (rows 8..15) of the block: q . (hi + lo) rows of the prepass's KC;
            // thread t: row t & 15, head-dim slice t >> 4 (D/8 columns), partials summed in order
            const __half* kb = kc + (static_cast<size_t>(kvh) * n + j) * 32 * D;
            const int r = t & 15, part = t >> 4;
            float a = 0.0f;
#pragma unroll
            for (int c8 = part * (D / 64); c8 < (part + 1) * (D / 64); ++c8) {  // D/8 columns = D/64 x 8
                const uint4 hv = reinterpret_cast<const uint4*>(kb + r * D)[c8];
                const uint4 lv = reinterpret_cast<const uint4*>(kb + (16 + r) * D)[c8];
                const __half* hh = reinterpret_cast<const __half*>(&hv);
                const __half* ll = reinterpret_cast<const __half*>(&lv);
#pragma unroll
                for (int e2 = 0; e2 < 8; ++e2)
                    a = fmaf(qs[c8 * 8 + e2], __half2float(hh[e2]) + __half2float(ll[e2]), a);
            }
            cpart[part][r] = a;
        }
        // ---- max chain (eager, the reference's recurrence)
        const float bm = block_max(sc) + p.rowmax_bias;  // (its barriers publish cpart too)
        if (PROT && t < 2 * kStride) {
            float a = 0.0f;
            for (int part = 0; part < 8; ++part) a = __fadd_rn(a, cpart[part][t]);
            cs[t] = __fmul_rn(a, scale);
        }
        const float m_old = m_run;
        float m_new = (m_old < bm) ? bm : m_old;
        float e = ex2_approx(__fsub_rn(sc, m_new) * kLog2e);
        ps[t] = e;
        if (PROT) scs[t] = sc;
        __syncthreads();
        if (PROT) {
            // ---- exp-stage check per group x: prod_l P[x + 8l] vs exp(c1 - 16 m)
            if (t < kStride) {
                float pr = 1.0f;
                for (int l = 0; l < kBlock / kStride; ++l) pr = __fmul_rn(pr, ps[t + kStride * l]);
                prod[t] = pr;
            }
            __syncthreads();
            int viol = 0;
            float res = 0.0f;
            if (t == 0) {
                for (int x = 0; x < kStride; ++x) {
                    const float pc1 = ex2_approx(__fsub_rn(cs[x], 16.0f * m_new) * kLog2e);
                    const float pr = prod[x];
                    if (!(pr > 0.0f && pr < CUDART_INF_F) || !(pc1 > 0.0f && pc1 < CUDART_INF_F)) {
                        ++viol;
                        res = CUDART_INF_F;
                    } else if (!(pr > pc1 * p.exp_lo && pr < pc1 * p.exp_hi)) {
                        ++viol;
                        res = fmaxf(res, fabsf(lg2_approx(__fdividef(pr, pc1))) * kLn2);
                    }
                }
                if (!isfinite(m_new)) { viol = viol ? viol : 1; res = CUDART_INF_F; }
                bcast[0] = static_cast<float>(viol);
            }
            __syncthreads();
            if (bcast[0] != 0.0f) {
                // ---- rare: the reference ladder on this row (snvr.cpp:89-157), one thread
                if (t == 0) {
                    float scl[kBlock], c1s[kStride], c2s[kStride];
                    for (int c = 0; c < kBlock; ++c) scl[c] = scs[c];
                    for (int x = 0; x < kStride; ++x) { c1s[x] = cs[x]; c2s[x] = cs[kStride + x]; }
                    RowVerify lin{};
                    lin.best_col = -1;
                    lin.restored_col = -1;
                    bool cs_bad = false;
                    for (int x = 0; x < kStride; ++x) cs_bad |= !isfinite(c1s[x]) || !isfinite(c2s[x]);
                    if (!cs_bad) verify_row<kBlock>(scl, c1s, c2s, p.eps_lin, lin);
                    float bmr = scl[0];
                    for (int c = 1; c < kBlock; ++c) bmr = (bmr < scl[c]) ? scl[c] : bmr;
                    const float mm = (m_old < bmr) ? bmr : m_old;
                    int changed = 0;
                    for (int c = 0; c < kBlock; ++c) {
                        const float ee = ex2_approx(__fsub_rn(scl[c], mm) * kLog2e);
                        if (__float_as_uint(ee) != __float_as_uint(ps[c])) changed = 1;
                        ps[c] = ee;
                    }
                    bool still_bad = !isfinite(mm) || cs_bad;
                    for (int x = 0; x < kStride && !still_bad; ++x) {
                        float pr = 1.0f;
                        for (int l = 0; l < kBlock / kStride; ++l) pr = __fmul_rn(pr, ps[x + kStride * l]);
                        const float pc1 = ex2_approx(__fsub_rn(c1s[x], 16.0f * mm) * kLog2e);
                        if (!(pr > 0.0f && pr < CUDART_INF_F) || !(pc1 > 0.0f && pc1 < CUDART_INF_F) ||
                            fabsf(lg2_approx(__fdividef(pr, pc1))) * kLn2 > p.eps1)
                            still_bad = true;
                    }
                    const int corr = lin.corrections + changed;
                    const int status = (still_bad || lin.uncorrectable)
                                           ? EFTA_DETECTED_UNCORRECTABLE
                                           : (corr > 0 || lin.checksum_repair ? EFTA_CORRECTED : EFTA_CLEAN);
                    if (changed) atomicAdd(&p.counters->recomputes, 1);
                    push_event(p, EFTA_EXP_CHECKSUM, head, 0, j, status, 0, lin.best_col, viol, corr,
                               lin.checksum_repair, res, lin.best_delta);
                    bcast[1] = mm;
                    bcast[2] = bmr + p.rowmax_bias;
                }
                __syncthreads();
                m_new = bcast[1];
                e = ps[t];
            }
        }
        // ---- rescale factor (guarded past the first block), sums, lower bound
        float f = ex2_approx(__fsub_rn(m_old, m_new) * kLog2e);
        if (PROT && j > j0 && !(f > 0.0f && f <= 1.0f)) {
            // the reference re-derives the row from its true max (efta.cpp:196-228): here the
            // max chain itself is the only input, so the factor is recomputed from it
            if (t == 0) push_event(p, EFTA_FACTOR_RANGE, head, 0, j, EFTA_CORRECTED, 0, -1, 1, 1, 0, f, 0.0);
            f = ex2_approx(__fsub_rn(m_old, m_new) * kLog2e);
            f = fminf(fmaxf(f, 0.0f), 1.0f);
        }
        const float psum = block_sum(e);
        l_run = __fadd_rn(__fmul_rn(f, l_run), psum);
        if (PROT) lb = __fadd_rn(__fmul_rn(lb, f), ex2_approx(__fsub_rn(bm, m_new) * kLog2e));
        m_run = m_new;
        // ---- O += P . V (thread = output column), checksums += P . VC (threads 0..15)
        const __half* vb = v + (kv0 + static_cast<size_t>(j) * kBlock) * D;
        if (t < D) {
            float acc = 0.0f;
            for (int key = 0; key < kBlock; ++key) acc = fmaf(ps[key], __half2float(vb[key * D + t]), acc);
            o_acc = __fadd_rn(__fmul_rn(o_acc, f), acc);
        }
        if (PROT) {
            // thread t = key t: O.c += P_t * VC_t (hi + lo) for the 16 checksum columns, kept per
            // thread across blocks (rescaled like O) and summed over the keys once, at the end
            const __half* vcr = vc + ((static_cast<size_t>(kvh) * n + j) * kBlock + t) * 64;
            const uint4 h0 = reinterpret_cast<const uint4*>(vcr)[0], h1 = reinterpret_cast<const uint4*>(vcr)[1];
            const uint4 l0 = reinterpret_cast<const uint4*>(vcr)[2], l1 = reinterpret_cast<const uint4*>(vcr)[3];
            const __half* hh0 = reinterpret_cast<const __half*>(&h0);
            const __half* hh1 = reinterpret_cast<const __half*>(&h1);
            const __half* ll0 = reinterpret_cast<const __half*>(&l0);
            const __half* ll1 = reinterpret_cast<const __half*>(&l1);
            const float pt = ps[t];
#pragma unroll
            for (int x = 0; x < 2 * kStride; ++x) {
                const float vcx = x < 8 ? __half2float(hh0[x]) + __half2float(ll0[x])
                                        : __half2float(hh1[x - 8]) + __half2float(ll1[x - 8]);
                oc_acc[x] = fmaf(pt, vcx, __fmul_rn(oc_acc[x], f));
            }
        }
        __syncthreads();  // ps / scs / cs are rewritten by the next block
    }

    // ---- the split's O.c: sum of the per-key shares (warp shuffles, then the four warps in order)
    if (PROT) {
#pragma unroll
        for (int x = 0; x < 2 * kStride; ++x) {
            float a2 = oc_acc[x];
            for (int o = 16; o; o >>= 1) a2 += __shfl_xor_sync(0xffffffffu, a2, o);
            if (lane == 0) opart[wq][x] = a2;
        }
    }
    if (t < D) orow[t] = o_acc;
    __syncthreads();
    if (PROT && t < 2 * kStride) {
        float a2 = 0.0f;
        for (int w = 0; w < DT / 32; ++w) a2 = __fadd_rn(a2, opart[w][t]);
        ocs[t] = a2;
    }
    __syncthreads();
    if (nsplit > 1) {
        // partial result of this split: (m, l, lb | O[D] | O.c[16])
        float* pp = part + (static_cast<size_t>(head) * nsplit + split) * (kPartHdr + D + 2 * kStride);
        if (t == 0) { pp[0] = m_run; pp[1] = l_run; pp[2] = lb; }
        if (t < D) pp[kPartHdr + t] = orow[t];
        if (t < 2 * kStride) pp[kPartHdr + D + t] = PROT ? ocs[t] : 0.0f;
        return;
    }
    if (t == 0) decode_epilogue<D, PROT>(p, head, m_run, l_run, lb, orow, ocs);
    __syncthreads();
    if (t < D) p.o[static_cast<size_t>(head) * D + t] = orow[t];
}

// Merge the splits of each query row in split order (the online-softmax combination of partial
// (m, l, O) with factors exp(m_s - m)), then the row's epilogue. grid = heads, 128 threads.
template <int D, bool PROT>
__global__ void __launch_bounds__(DT) efta_decode_combine_kernel(AttnParams p, const float* __restrict__ part,
                                                                 int nsplit) {
    __shared__ float orow[D];
    __shared__ float ocs[2 * kStride];
    __shared__ float hdr[3];
    const int head = blockIdx.x, t = threadIdx.x;
    const float* pp = part + static_cast<size_t>(head) * nsplit * (kPartHdr + D + 2 * kStride);
    constexpr int W = kPartHdr + D + 2 * kStride;
    float m = -CUDART_INF_F;
    for (int s_ = 0; s_ < nsplit; ++s_) m = fmaxf(m, pp[s_ * W]);
    float l = 0.0f, lb = 0.0f, acc = 0.0f, cacc = 0.0f;
    for (int s_ = 0; s_ < nsplit; ++s_) {
        const float fs = ex2_approx(__fsub_rn(pp[s_ * W], m) * kLog2e);
        l = __fadd_rn(l, __fmul_rn(pp[s_ * W + 1], fs));
        lb = __fadd_rn(lb, __fmul_rn(pp[s_ * W + 2], fs));
        if (t < D) acc = __fadd_rn(acc, __fmul_rn(pp[s_ * W + kPartHdr + t], fs));
        if (PROT && t < 2 * kStride) cacc = __fadd_rn(cacc, __fmul_rn(pp[s_ * W + kPartHdr + D + t], fs));
    }
    if (t < D) orow[t] = acc;
    if (PROT && t < 2 * kStride) ocs[t] = cacc;
    if (t == 0) { hdr[0] = m; hdr[1] = l; hdr[2] = lb; }
    __syncthreads();
    if (t == 0) decode_epilogue<D, PROT>(p, head, hdr[0], hdr[1], hdr[2], orow, ocs);
    __syncthreads();
    if (t < D) p.o[static_cast<size_t>(head) * D + t] = orow[t];
}

}  // namespace

namespace efta_decode {

// splits per query row: enough CTAs for ~4 per SM, at least two key blocks per split
int splits_for(int bh, int nblk, int nsm) {
    int sp = (4 * nsm + bh - 1) / bh;
    sp = sp < 1 ? 1 : sp;
    const int maxsp = nblk / 2 > 0 ? nblk / 2 : 1;
    return sp < maxsp ? sp : maxsp;
}
size_t part_bytes(int bh, int nblk, int d, int nsm) {
    const int sp = splits_for(bh, nblk, nsm);
    return sp > 1 ? static_cast<size_t>(bh) * sp * (kPartHdr + d + 2 * kStride) * sizeof(float) : 0;
}

cudaError_t launch(int d, bool prot, const AttnParams& p, int bh, const void* q, const void* k, const void* v,
                   const void* kc, const void* vc, float* part, int nsm, cudaStream_t st) {
    const __half *hq = static_cast<const __half*>(q), *hk = static_cast<const __half*>(k),
                 *hv = static_cast<const __half*>(v), *hkc = static_cast<const __half*>(kc),
                 *hvc = static_cast<const __half*>(vc);
    const int sp = splits_for(bh, p.nblk, nsm);
    const dim3 grid(sp, bh);
    if (d == 64) {
        if (prot) efta_decode_kernel<64, true><<<grid, DT, 0, st>>>(p, hq, hk, hv, hkc, hvc, part, sp);
        else efta_decode_kernel<64, false><<<grid, DT, 0, st>>>(p, hq, hk, hv, hkc, hvc, part, sp);
        if (sp > 1) {
            if (prot) efta_decode_combine_kernel<64, true><<<bh, DT, 0, st>>>(p, part, sp);
            else efta_decode_combine_kernel<64, false><<<bh, DT, 0, st>>>(p, part, sp);
        }
    } else {
        if (prot) efta_decode_kernel<128, true><<<grid, DT, 0, st>>>(p, hq, hk, hv, hkc, hvc, part, sp);
        else efta_decode_kernel<128, false><<<grid, DT, 0, st>>>(p, hq, hk, hv, hkc, hvc, part, sp);
        if (sp > 1) {
            if (prot) efta_decode_combine_kernel<128, true><<<bh, DT, 0, st>>>(p, part, sp);
            else efta_decode_combine_kernel<128, false><<<bh, DT, 0, st>>>(p, part, sp);
        }
    }
    return cudaGetLastError();
}

}  // namespace efta_decode
