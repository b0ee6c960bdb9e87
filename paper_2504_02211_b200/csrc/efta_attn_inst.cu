#include <algorithm>
// efta_attn_inst.cu — instantiations of the fused attention kernel for one head
// dim (EFTA_INST_D), all modes x {fast, debug/tap} variants.
#include "efta_attn_kernel.cuh"
#include "efta_attn_pair.cuh"
#include "efta_launch.h"

#ifndef EFTA_INST_D
#error "EFTA_INST_D must be 64 or 128"
#endif

using namespace efta_sm100;

namespace {

template <int D, int MODE, bool DBG>
cudaError_t launch_t(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                     const CUtensorMap& tkc, const CUtensorMap& tvc, const AttnParams& p, int bh,
                     cudaStream_t st) {
    using L = AttnLayout<D>;
    auto kern = efta_attn_fwd_kernel<D, MODE, DBG>;
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             L::SMEM_BYTES);
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
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

template <int D, int MODE>
cudaError_t launch_pair_t(const CUtensorMap& tq, const CUtensorMap& tka, const CUtensorMap& tkb,
                          const CUtensorMap& tkc, const CUtensorMap& tvt, const AttnParams& p, int bh,
                          cudaStream_t st) {
    using PL = PairLayout<D, MODE != 0>;
    auto kern = efta_attn_pair_kernel<D, MODE>;
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, PL::SMEM_BYTES);
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    static int nsm = 0;
    if (!nsm) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    }
    const int tiles = bh * (p.nblk / 2);  // (head, query pair) tiles
    const int ncl = std::min(tiles, std::max(1, nsm / 2));
    dim3 grid(2 * ncl);
    kern<<<grid, kPairThreads, PL::SMEM_BYTES, st>>>(tq, tka, tkb, tkc, tvt, p);
    return cudaGetLastError();
}

}  // namespace

#if EFTA_INST_D == 64
cudaError_t efta_launch_attn_d64(int mode, bool dbg, const CUtensorMap& tq, const CUtensorMap& tk,
                                 const CUtensorMap& tv, const CUtensorMap& tkc,
                                 const CUtensorMap& tvc, const AttnParams& p, int bh,
                                 cudaStream_t st) {
    return launch_d<64>(mode, dbg, tq, tk, tv, tkc, tvc, p, bh, st);
}
#else
cudaError_t efta_launch_attn_d128(int mode, bool dbg, const CUtensorMap& tq, const CUtensorMap& tk,
                                  const CUtensorMap& tv, const CUtensorMap& tkc,
                                  const CUtensorMap& tvc, const AttnParams& p, int bh,
                                  cudaStream_t st) {
    return launch_d<128>(mode, dbg, tq, tk, tv, tkc, tvc, p, bh, st);
}
#endif

#if EFTA_INST_D == 64
cudaError_t efta_launch_attn_pair_d64(int mode, const CUtensorMap& tq, const CUtensorMap& tka,
                                      const CUtensorMap& tkb, const CUtensorMap& tkc, const CUtensorMap& tvt,
                                      const AttnParams& p, int bh, cudaStream_t st) {
    return mode == 0 ? launch_pair_t<64, 0>(tq, tka, tkb, tkc, tvt, p, bh, st)
                     : launch_pair_t<64, 2>(tq, tka, tkb, tkc, tvt, p, bh, st);
}
cudaError_t efta_launch_encode_pair_d64(bool prot, const void* k, const void* v, void* kc, void* vt,
                                        int seq_len, int nblk, int bh, cudaStream_t st) {
    dim3 grid(nblk, bh);
    if (prot)
        efta_encode_pair_kernel<64, true><<<grid, 256, 0, st>>>(static_cast<const __half*>(k), static_cast<const __half*>(v),
                                                             static_cast<__half*>(kc), static_cast<__half*>(vt), seq_len, nblk);
    else
        efta_encode_pair_kernel<64, false><<<grid, 256, 0, st>>>(static_cast<const __half*>(k), static_cast<const __half*>(v),
                                                              static_cast<__half*>(kc), static_cast<__half*>(vt), seq_len, nblk);
    return cudaGetLastError();
}
#else
cudaError_t efta_launch_attn_pair_d128(int mode, const CUtensorMap& tq, const CUtensorMap& tka,
                                       const CUtensorMap& tkb, const CUtensorMap& tkc, const CUtensorMap& tvt,
                                       const AttnParams& p, int bh, cudaStream_t st) {
    return mode == 0 ? launch_pair_t<128, 0>(tq, tka, tkb, tkc, tvt, p, bh, st)
                     : launch_pair_t<128, 2>(tq, tka, tkb, tkc, tvt, p, bh, st);
}
cudaError_t efta_launch_encode_pair_d128(bool prot, const void* k, const void* v, void* kc, void* vt,
                                         int seq_len, int nblk, int bh, cudaStream_t st) {
    dim3 grid(nblk, bh);
    if (prot)
        efta_encode_pair_kernel<128, true><<<grid, 256, 0, st>>>(static_cast<const __half*>(k), static_cast<const __half*>(v),
                                                              static_cast<__half*>(kc), static_cast<__half*>(vt), seq_len, nblk);
    else
        efta_encode_pair_kernel<128, false><<<grid, 256, 0, st>>>(static_cast<const __half*>(k), static_cast<const __half*>(v),
                                                               static_cast<__half*>(kc), static_cast<__half*>(vt), seq_len, nblk);
    return cudaGetLastError();
}
#endif
