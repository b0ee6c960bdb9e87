// efta_attn_inst.cu — instantiations of the fused attention kernels for one head dim
// (EFTA_INST_D). EFTA_INST_INJ=1 builds only the fault-tap variant of the CTA-pair kernel
// (its own translation unit so the variants compile in parallel), EFTA_INST_CAUSAL=1 only the
// causal builds of the fast pair kernel; otherwise the unit holds
// the single-CTA kernel (all modes x {fast, tap}), the fast pair kernels and the prepass.
#include <algorithm>

#include "efta_attn_kernel.cuh"
#include "efta_attn_pair.cuh"
#include "efta_launch.h"

#ifndef EFTA_INST_D
#error "EFTA_INST_D must be 64 or 128"
#endif
#ifndef EFTA_INST_INJ
#define EFTA_INST_INJ 0
#endif
#ifndef EFTA_INST_CAUSAL
#define EFTA_INST_CAUSAL 0
#endif

using namespace efta_sm100;

namespace {

// The dynamic shared-memory limit is a per-device function attribute: set it on every
// launch (cheap, thread-safe, correct when one process drives several GPUs).
template <typename K>
cudaError_t set_smem(K kern, uint32_t bytes) {
    return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
}

template <int D, int MODE, bool INJ, bool CAUSAL = false>
cudaError_t launch_pair_t(const CUtensorMap& tq, const CUtensorMap& tka, const CUtensorMap& tkb,
                          const CUtensorMap& tkc, const CUtensorMap& tvt, const CUtensorMap& tvo, const AttnParams& p, int bh,
                          cudaStream_t st) {
    using PL = PairLayout<D, MODE != 0>;
    auto kern = efta_attn_pair_kernel<D, MODE, INJ, CAUSAL>;
    if (cudaError_t e = set_smem(kern, PL::SMEM_BYTES)) return e;
    int dev = 0, nsm = 0;
    if (cudaError_t e = cudaGetDevice(&dev)) return e;
    if (cudaError_t e = cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev)) return e;
    const int tiles = bh * (p.nblk / 2);  // (head, query pair) tiles
    const int ncl = std::min(tiles, std::max(1, nsm / 2));
    dim3 grid(2 * ncl);
    kern<<<grid, kPairThreads, PL::SMEM_BYTES, st>>>(tq, tka, tkb, tkc, tvt, tvo, p);
    return cudaGetLastError();
}

#if !EFTA_INST_INJ && !EFTA_INST_CAUSAL
template <int D, int MODE, bool DBG>
cudaError_t launch_t(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                     const CUtensorMap& tkc, const CUtensorMap& tvc, const AttnParams& p, int bh,
                     cudaStream_t st) {
    using L = AttnLayout<D>;
    auto kern = efta_attn_fwd_kernel<D, MODE, DBG>;
    if (cudaError_t e = set_smem(kern, L::SMEM_BYTES)) return e;
    dim3 grid(p.nblk, bh);
    kern<<<grid, 256, L::SMEM_BYTES, st>>>(tq, tk, tv, tkc, tvc, p);
    return cudaGetLastError();
}

template <int D>
cudaError_t launch_d(int mode, bool dbg, const CUtensorMap& tq, const CUtensorMap& tk,
                     const CUtensorMap& tv, const CUtensorMap& tkc, const CUtensorMap& tvc,
                     const AttnParams& p, int bh, cudaStream_t st) {
    switch (mode * 2 + (dbg ? 1 : 0)) {
        case 0: return launch_t<D, 0, false>(tq, tk, tv, tkc, tvc, p, bh, st);
        case 1: return launch_t<D, 0, true>(tq, tk, tv, tkc, tvc, p, bh, st);
        case 2: return launch_t<D, 1, false>(tq, tk, tv, tkc, tvc, p, bh, st);
        case 3: return launch_t<D, 1, true>(tq, tk, tv, tkc, tvc, p, bh, st);
        case 4: return launch_t<D, 2, false>(tq, tk, tv, tkc, tvc, p, bh, st);
        default: return launch_t<D, 2, true>(tq, tk, tv, tkc, tvc, p, bh, st);
    }
}

template <int D>
cudaError_t launch_encode_pair(bool prot, const void* k, const void* v, void* kc, void* vt, int seq_len, int nblk,
                               int bh, cudaStream_t st) {
    dim3 grid(nblk, bh);
    auto kh = static_cast<const __half*>(k);
    auto vh = static_cast<const __half*>(v);
    if (prot)
        efta_encode_pair_kernel<D, true><<<grid, 256, 0, st>>>(kh, vh, static_cast<__half*>(kc),
                                                              static_cast<__half*>(vt), seq_len, nblk);
    else
        efta_encode_pair_kernel<D, false><<<grid, 256, 0, st>>>(kh, vh, static_cast<__half*>(kc),
                                                               static_cast<__half*>(vt), seq_len, nblk);
    return cudaGetLastError();
}
#endif

}  // namespace

#define EFTA_CAT2(a, b) a##b
#define EFTA_CAT(a, b) EFTA_CAT2(a, b)
#define EFTA_SFX EFTA_CAT(_d, EFTA_INST_D)

#if EFTA_INST_CAUSAL
cudaError_t EFTA_CAT(efta_launch_attn_pair_causal, EFTA_SFX)(int mode, const CUtensorMap& tq, const CUtensorMap& tka,
                                                            const CUtensorMap& tkb, const CUtensorMap& tkc,
                                                            const CUtensorMap& tvt, const CUtensorMap& tvo, const AttnParams& p, int bh,
                                                            cudaStream_t st) {
    return mode == 0 ? launch_pair_t<EFTA_INST_D, 0, false, true>(tq, tka, tkb, tkc, tvt, tvo, p, bh, st)
                     : launch_pair_t<EFTA_INST_D, 2, false, true>(tq, tka, tkb, tkc, tvt, tvo, p, bh, st);
}
#elif EFTA_INST_INJ
cudaError_t EFTA_CAT(efta_launch_attn_pair_inj, EFTA_SFX)(const CUtensorMap& tq, const CUtensorMap& tka,
                                                         const CUtensorMap& tkb, const CUtensorMap& tkc,
                                                         const CUtensorMap& tvt, const CUtensorMap& tvo, const AttnParams& p, int bh,
                                                         cudaStream_t st) {
    return launch_pair_t<EFTA_INST_D, EFTA_MODE_EFTA_OPT, true>(tq, tka, tkb, tkc, tvt, tvo, p, bh, st);
}
#else
cudaError_t EFTA_CAT(efta_launch_attn, EFTA_SFX)(int mode, bool dbg, const CUtensorMap& tq, const CUtensorMap& tk,
                                                const CUtensorMap& tv, const CUtensorMap& tkc,
                                                const CUtensorMap& tvc, const AttnParams& p, int bh,
                                                cudaStream_t st) {
    return launch_d<EFTA_INST_D>(mode, dbg, tq, tk, tv, tkc, tvc, p, bh, st);
}
cudaError_t EFTA_CAT(efta_launch_attn_pair, EFTA_SFX)(int mode, const CUtensorMap& tq, const CUtensorMap& tka,
                                                     const CUtensorMap& tkb, const CUtensorMap& tkc,
                                                     const CUtensorMap& tvt, const CUtensorMap& tvo, const AttnParams& p, int bh,
                                                     cudaStream_t st) {
    return mode == 0 ? launch_pair_t<EFTA_INST_D, 0, false>(tq, tka, tkb, tkc, tvt, tvo, p, bh, st)
                     : launch_pair_t<EFTA_INST_D, 2, false>(tq, tka, tkb, tkc, tvt, tvo, p, bh, st);
}
cudaError_t EFTA_CAT(efta_launch_encode_pair, EFTA_SFX)(bool prot, const void* k, const void* v, void* kc, void* vt,
                                                       int seq_len, int nblk, int bh, cudaStream_t st) {
    return launch_encode_pair<EFTA_INST_D>(prot, k, v, kc, vt, seq_len, nblk, bh, st);
}
#endif
