// efta_launch.h — per-head-dim launchers of the fused attention kernel (defined in
// efta_attn_inst.cu, one translation unit per head dim so they build in parallel).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include "efta_attn.cuh"

cudaError_t efta_launch_attn_d64(int mode, bool dbg, const CUtensorMap& tq, const CUtensorMap& tk,
                                 const CUtensorMap& tv, const CUtensorMap& tkc,
                                 const CUtensorMap& tvc, const efta_sm100::AttnParams& p, int bh,
                                 cudaStream_t st);
cudaError_t efta_launch_attn_d128(int mode, bool dbg, const CUtensorMap& tq, const CUtensorMap& tk,
                                  const CUtensorMap& tv, const CUtensorMap& tkc,
                                  const CUtensorMap& tvc, const efta_sm100::AttnParams& p, int bh,
                                  cudaStream_t st);

// shared thread-local error string behind efta_last_error()
void efta_internal_set_error(const char* msg);

// CTA-pair (cta_group::2) fast path: modes NONE / EFTA_OPT, even number of query tiles.
// maps: q, k half A, k half B (protected peer), kc, [V^T; VC^T], O (d=64: the TMA-stored output). Persistent: one cluster
// (CTA pair) per two SMs loops over the (head, query pair) tiles.
cudaError_t efta_launch_attn_pair_d64(int mode, const CUtensorMap& tq, const CUtensorMap& tka,
                                      const CUtensorMap& tkb, const CUtensorMap& tkc, const CUtensorMap& tvt, const CUtensorMap& tvo,
                                      const efta_sm100::AttnParams& p, int bh, cudaStream_t st);
cudaError_t efta_launch_attn_pair_d128(int mode, const CUtensorMap& tq, const CUtensorMap& tka,
                                       const CUtensorMap& tkb, const CUtensorMap& tkc, const CUtensorMap& tvt, const CUtensorMap& tvo,
                                       const efta_sm100::AttnParams& p, int bh, cudaStream_t st);
// causal builds of the fast pair kernel (modes NONE / EFTA_OPT)
cudaError_t efta_launch_attn_pair_causal_d64(int mode, const CUtensorMap& tq, const CUtensorMap& tka,
                                             const CUtensorMap& tkb, const CUtensorMap& tkc, const CUtensorMap& tvt, const CUtensorMap& tvo,
                                             const efta_sm100::AttnParams& p, int bh, cudaStream_t st);
cudaError_t efta_launch_attn_pair_causal_d128(int mode, const CUtensorMap& tq, const CUtensorMap& tka,
                                              const CUtensorMap& tkb, const CUtensorMap& tkc, const CUtensorMap& tvt, const CUtensorMap& tvo,
                                              const efta_sm100::AttnParams& p, int bh, cudaStream_t st);
// fault-tap build of the pair kernel (EFTA_OPT; taps at every FaultSite, eager rescale)
cudaError_t efta_launch_attn_pair_inj_d64(const CUtensorMap& tq, const CUtensorMap& tka, const CUtensorMap& tkb,
                                          const CUtensorMap& tkc, const CUtensorMap& tvt, const CUtensorMap& tvo,
                                          const efta_sm100::AttnParams& p, int bh, cudaStream_t st);
cudaError_t efta_launch_attn_pair_inj_d128(const CUtensorMap& tq, const CUtensorMap& tka, const CUtensorMap& tkb,
                                           const CUtensorMap& tkc, const CUtensorMap& tvt, const CUtensorMap& tvo,
                                           const efta_sm100::AttnParams& p, int bh, cudaStream_t st);
cudaError_t efta_launch_encode_pair_d64(bool prot, const void* k, const void* v, void* kc, void* vt,
                                        int seq_len, int nblk, int bh, cudaStream_t st);
cudaError_t efta_launch_encode_pair_d128(bool prot, const void* k, const void* v, void* kc, void* vt,
                                         int seq_len, int nblk, int bh, cudaStream_t st);
