/*
 * efta_b200.h — C-ABI of the B200-native EFTA hot path (libefta_b200.so).
 *
 * Plain pointers and sizes only (no CUDA / torch types): `stream` is a
 * cudaStream_t passed as void*. Unless stated otherwise every data pointer is
 * a DEVICE pointer owned by the caller; nothing is allocated on the hot path.
 * Return codes: 0 ok, 1 configuration error (the reference's ConfigError),
 * 2 CUDA error; efta_last_error() describes the last failure (thread-local).
 *
 * Each entry point replaces a reference interface (paths relative to
 * /root/reference/proj):
 *
 *   efta_attn_fwd_f16        efta::efta_forward            include/efta/efta.hpp:86-89
 *                            (modes NONE / EFTA / EFTA_OPTIMIZED; the FaultInjector*
 *                            argument becomes the device fault table; FTReport
 *                            becomes events + counters + m/l outputs)
 *   efta_attn_validate       efta::AttnConfig::validate    include/efta/config.hpp:30-41
 *   efta_attn_fwd_host_f16   same as efta_attn_fwd_f16, HOST buffers in/out (copies
 *                            inside the call: the reference-facing e2e path)
 *   efta_abft_gemm_f16       efta::checksummed_gemm + verify_locate_correct
 *                            include/efta/abft.hpp:58-60, 73-77 (strided-ABFT GEMM,
 *                            applied per 256-wide output column tile = FFN linear)
 *   efta_abft_gemm_ex        the same with an fp32 product and the tile checksums returned
 *                            (the drop-in checksummed_gemm, abft.hpp:73-77)
 *   efta_abft_encode_weight_f16  encode_strided of a weight matrix, abft.hpp:38
 *   efta_encode_strided_f32  encode_strided on a device tile, abft.hpp:38
 *   efta_verify_locate_correct_f32  verify_locate_correct on a device tile, abft.hpp:58-60
 *   efta_flip_bit            efta::flip_bit                 include/efta/fault.hpp:33
 *   efta_decode_fwd_f16      (none: KV-cache decode, row 0 of efta_forward, a reference non-goal)
 */
#ifndef EFTA_B200_H
#define EFTA_B200_H

#include <stddef.h>
#include <stdint.h>

#include "../paper_2504_02211_b200/csrc/efta_types.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Attention problem: Q, K, V are [batch*heads, seq_len, head_dim] fp16 (bits as
 * uint16; K and V [batch*kv_heads, ...] with grouped-query attention), O is fp32 of Q's shape, m_out / l_out are [batch*heads, seq_len]
 * fp32 (the reference's FTReport::final_m / final_l). */
typedef struct {
    int batch, heads, seq_len, head_dim;
    int block;          /* reference AttnConfig::block; this kernel: 128 */
    int stride;         /* reference AttnConfig::stride; this kernel: 8 */
    float scale;        /* 0 -> 1/sqrt(head_dim) (config.hpp:40) */
    int mode;           /* efta_mode */
    double eps1, eps2, eps_lin; /* reference Thresholds (snvr.hpp:17-30) */
    int observe_linear; /* KernelKnobs::observe_linear (efta.hpp:79) */
    float rowmax_bias;  /* KernelKnobs::rowmax_bias (efta.hpp:82) */
    int debug;          /* 1: fault-tap / observation build (required if n_faults > 0): the
                           reference op sequence with taps at every FaultSite, eager rescale */
    int checksums_ready;/* 1: workspace already holds this K/V's encoded operands (skip the
                           prepass; e.g. K/V reused across calls). On the CTA-pair path the
                           workspace also holds the transposed V operand ([V^T ; VC^T]), so the
                           flag covers V itself, in every mode. Ignored by the host path. */
    int kv_heads;       /* grouped-query attention: K and V are [batch*kv_heads, seq_len, head_dim];
                           query head h of a batch entry reads K/V head h / (heads / kv_heads).
                           0 (or heads) = multi-head attention. Not a reference feature (SPEC.md:141,
                           356 list GQA as a non-goal): each query head still runs the reference
                           algorithm on its group's K and V. */
    int causal;         /* 1: key k is visible to query q only if k <= q (decoder self-attention).
                           Not a reference feature: modes NONE / EFTA_OPTIMIZED on the CTA-pair
                           kernel (even seq_len / 128), no fault-tap build. The diagonal block's
                           exp-stage check runs on each group's visible cells. */
    int o_token_major;  /* 1: `o` receives fp16 [batch, seq_len, heads, head_dim] (token-major: the
                           input of the output projection, no head-merge copy) instead of fp32
                           [batch, heads, seq_len, head_dim]; the float* argument then points to
                           that fp16 buffer. CTA-pair kernel configurations only (even seq_len /
                           128, modes NONE / EFTA_OPTIMIZED), device entry point only. Not a
                           reference feature (its attention returns fp32 per head). */
} efta_attn_desc;

const char* efta_last_error(void);
int efta_attn_validate(const efta_attn_desc* d);
size_t efta_attn_workspace_bytes(const efta_attn_desc* d);

/* counters: device efta_counters (zeroed by the call). events/fired: device arrays
 * of the given capacities (may be NULL with cap 0). faults: device array.
 * workspace: device buffer of efta_attn_workspace_bytes(d) bytes (checksum operands, the
 * persistent kernel's tile counter); calls that may run concurrently (different streams)
 * need distinct workspaces. */
int efta_attn_fwd_f16(const efta_attn_desc* d, const uint16_t* q, const uint16_t* k,
                      const uint16_t* v, float* o, float* m_out, float* l_out, void* workspace,
                      size_t workspace_bytes, const efta_fault_spec* faults, int n_faults,
                      efta_event* events, int ev_cap, efta_fired* fired, int fired_cap,
                      efta_counters* counters, void* stream);

/* Same contract with HOST buffers (q/k/v/o/m/l/faults/events/fired/counters all
 * host memory); device scratch is cached per thread and reused across calls.
 * Synchronous. */
int efta_attn_fwd_host_f16(const efta_attn_desc* d, const uint16_t* q, const uint16_t* k,
                           const uint16_t* v, float* o, float* m_out, float* l_out,
                           const efta_fault_spec* faults, int n_faults, efta_event* events,
                           int ev_cap, efta_fired* fired, int fired_cap, efta_counters* counters);

/* KV-cache decode (not a reference feature): one query row per head,
 * q [batch*heads, head_dim], against the caches k, v [batch*kv_heads, seq_len, head_dim] (fp16
 * bits); o [batch*heads, head_dim] fp32, m_out / l_out [batch*heads]. The reference algorithm
 * for that row (it is row 0 of efta_forward(q, K, V)): eager online softmax over the 128-key
 * blocks, EFTA-optimized checks (mode EFTA_OPTIMIZED) or none (NONE). HBM-bound, CUDA cores.
 * workspace: efta_attn_workspace_bytes(d); checksums_ready = 1 skips re-encoding the cache's
 * checksum operands (efta_attn_encode_kv_f16 into the workspace layout). */
int efta_decode_fwd_f16(const efta_attn_desc* d, const uint16_t* q, const uint16_t* k, const uint16_t* v,
                        float* o, float* m_out, float* l_out, void* workspace, size_t workspace_bytes,
                        efta_event* events, int ev_cap, efta_counters* counters, void* stream);

/* Strided checksum operands of K and V only (the encode prepass the forward runs
 * internally); kc: [BH*nblk*32, head_dim] fp16, vc: [BH*nblk*128, 64] fp16. */
int efta_attn_encode_kv_f16(const efta_attn_desc* d, const uint16_t* k, const uint16_t* v,
                            uint16_t* kc, uint16_t* vc, void* stream);

float efta_flip_bit(float v, int width, int bit);

/* ---- strided-ABFT GEMM (feed-forward linear layers) ----
 * Y[m x n] = X[m x k] . W^T with W stored [n x k] (nn.Linear layout), fp16 in / fp32
 * accumulate / fp16 out. Every 256-wide output column tile carries strided checksums
 * (stride 8, 32 groups) computed on the tensor cores from the weight's precomputed
 * checksum rows and verified / located / corrected per output row in the epilogue.
 * Faults (debug=1 only): efta_fault_spec with block_i = global row, col = global col,
 * bit = bit to flip in that fp32 accumulator value before verification. Events are
 * reported with kind EFTA_BLOCK_CHECKSUM, head = n-tile, block_i = m-tile, global row/col. */
typedef struct {
    int m, n, k;
    int stride;  /* 8 */
    int n_tile;  /* 256 */
    double eps;  /* absolute threshold of verify_locate_correct (abft.hpp:58-60) */
    int debug;
    /* Head-split output (0 = plain row-major [m, n]): with out_seq = S > 0, rows are tokens
     * b*S + s and columns part*(H*dh) + h*dh + c (H = out_heads, dh = out_head_dim), and the
     * element lands at y[part][b][h][s][c] — a fused QKV projection writes Q, K and V directly
     * in the attention's [batch, heads, seq, head_dim] layout (parts = n / (H*dh)). Requires
     * m % S == 0, n % (H*dh) == 0, dh % 8 == 0. Not a reference feature. */
    int out_seq, out_heads, out_head_dim;
} efta_gemm_desc;

size_t efta_abft_weight_cs_bytes(const efta_gemm_desc* d);
/* wcs: [n/256 * 32, k] fp16 = hi/lo split strided checksums of each weight tile */
int efta_abft_encode_weight_f16(const efta_gemm_desc* d, const uint16_t* w, uint16_t* wcs,
                                void* stream);
int efta_abft_gemm_f16(const efta_gemm_desc* d, const uint16_t* x, const uint16_t* w,
                       const uint16_t* wcs, uint16_t* y, const efta_fault_spec* faults,
                       int n_faults, efta_event* events, int ev_cap, efta_counters* counters,
                       void* stream);

/* Same GEMM with the output in fp32 (y_f32 = 1; the reference's checksummed_gemm returns an
 * fp32 product) and, if y_checksums != NULL, the tensor-core checksums of every 256-wide output
 * tile: y_checksums[(row * n/256 + tile) * 16 + {0..7, 8..15}] = c1[x], c2[x]. */
int efta_abft_gemm_ex(const efta_gemm_desc* d, const uint16_t* x, const uint16_t* w,
                      const uint16_t* wcs, void* y, int y_f32, float* y_checksums,
                      const efta_fault_spec* faults, int n_faults, efta_event* events, int ev_cap,
                      efta_counters* counters, void* stream);

/* Same GEMM (fp16 output) with element-wise epilogues applied to each verified / corrected
 * value before it is stored, the linear modules' neighbours in a transformer layer:
 * y = act(half(X W^T)) (+ residual), activation EFTA_ACT_NONE or EFTA_ACT_GELU (erf form),
 * residual NULL or fp16 [m, n] (row-major output only). The checksums protect the product
 * (the reference's checksummed_gemm); the element-wise ops follow it. Not a reference API. */
enum { EFTA_ACT_NONE = 0, EFTA_ACT_GELU = 1 };
int efta_abft_gemm_fused_f16(const efta_gemm_desc* d, const uint16_t* x, const uint16_t* w,
                             const uint16_t* wcs, uint16_t* y, const uint16_t* residual,
                             int activation, const efta_fault_spec* faults, int n_faults,
                             efta_event* events, int ev_cap, efta_counters* counters, void* stream);

/* Element-wise erf GELU of an fp16 device tensor (n elements, 16-byte aligned; y may equal x):
 * the FFN activation between the protected GEMMs of the FT-Transformer layer, bit-identical to
 * torch.nn.functional.gelu. Not a reference API. */
int efta_gelu_f16(const uint16_t* x, uint16_t* y, size_t n, void* stream);

/* ---- standalone strided ABFT on a device tile (reference abft.hpp:38-60) ----
 * encode_strided (src/abft.cpp:19-42): c1/c2 [rows, stride] of an fp32 tile [rows, cols].
 * verify_locate_correct (src/abft.cpp:65-187): repairs t in place, writes the report to device
 * memory; row_eps_mult is an optional device array of `rows` doubles. workspace: device buffer
 * of efta_verify_workspace_bytes(rows) bytes. */
typedef struct {
    int status, row, col, violations, corrections, checksum_repair;
    double residual, delta;
} efta_verify_report;

int efta_encode_strided_f32(int rows, int cols, int stride, const float* t, float* c1, float* c2,
                            void* stream);
size_t efta_verify_workspace_bytes(int rows);
int efta_verify_locate_correct_f32(int rows, int cols, int stride, float* t, const float* c1,
                                   const float* c2, double eps, const double* row_eps_mult,
                                   efta_verify_report* report, void* workspace,
                                   size_t workspace_bytes, void* stream);

/* ---- host-side helpers of the reference campaign (host memory only) ---- */
/* trial_seed (include/efta/rng.hpp:55-58) */
uint64_t efta_trial_seed(uint64_t base, uint64_t trial);
/* Rng(seed); q,k,v = Matrix::random(n, d) as fp16 bits in that order, then, if
 * n_sites > 0, sample_random_plan from the same stream (src/campaign.cpp:177-185,
 * src/fault.cpp:143-164). spec->head is set to 0. */
int efta_gen_trial_f16(uint64_t seed, int n, int d, int block, int stride, const int* sites,
                       int n_sites, uint16_t* q, uint16_t* k, uint16_t* v, efta_fault_spec* spec);
/* classify_trial (src/campaign.cpp:123-152); returns the Outcome enum value
 * (campaign.hpp:12-20): 0 clean 1 false_alarm 2 corrected 3 range_restricted
 * 4 masked_benign 5 range_contract 6 uncorrectable. */
int efta_classify_trial(int rows, int cols, const float* out, const float* ref, int detections,
                        int range_replacements, int failed, const float* final_l, int n_l,
                        int plan_nonempty, int reduction_site, double eps2);

#ifdef __cplusplus
}
#endif
#endif
