// efta_capi.cu — C-ABI entry points (include/efta_b200.h): validation, TMA
// descriptor construction, kernel dispatch. No torch, no CPU fallback: every
// compute entry point launches sm_100a kernels or fails with a CUDA error.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/efta_b200.h"
#include "efta_attn.cuh"
#include "efta_launch.h"
#include "efta_encode.cuh"

namespace efta_decode {  // csrc/decode.cu
size_t part_bytes(int bh, int nblk, int d, int nsm);
cudaError_t launch(int d, bool prot, const efta_sm100::AttnParams& p, int bh, const void* q, const void* k,
                   const void* v, const void* kc, const void* vc, float* part, int nsm, cudaStream_t st);
}

namespace efta_dec {  // csrc/decoupled.cu
size_t workspace_bytes(int bh, int N, int D);
std::string forward(const efta_sm100::AttnParams& base, int bh, int N, int D, const __half* q, const __half* k,
                    const __half* v, float* o, void* ws, cudaStream_t st);
}

using namespace efta_sm100;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

#define CUDA_TRY(expr)                                                                       \
    do {                                                                                     \
        cudaError_t e_ = (expr);                                                             \
        if (e_ != cudaSuccess)                                                               \
            return fail(2, std::string(#expr) + ": " + cudaGetErrorString(e_));              \
    } while (0)

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    });
    return fn;
}

// 2D fp16 tensor [rows, cols] row-major, box {64, box_rows}, 128B swizzle.
bool make_map(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {cols * 2};
    cuuint32_t box[2] = {64, box_rows};
    cuuint32_t estr[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(base), dims, strides, box,
              estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// the pair kernel's output map (TMA store, 128-byte swizzle): fp32 [rows, d] in 32-column boxes,
// or fp16 [rows, cols] (token-major) in 64-column boxes
bool make_out_map(CUtensorMap* m, void* base, bool f16, uint64_t rows, uint64_t cols, uint32_t box_rows) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) return false;
    const uint64_t esz = f16 ? 2 : 4;
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {cols * esz};
    cuuint32_t box[2] = {static_cast<cuuint32_t>(128 / esz), box_rows};
    cuuint32_t estr[2] = {1, 1};
    return fn(m, f16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, base, dims, strides, box,
              estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int validate(const efta_attn_desc* d) {
    if (!d) return fail(1, "efta: null descriptor");
    // reference AttnConfig::validate (include/efta/config.hpp:30-41)
    if (d->seq_len <= 0 || d->head_dim <= 0 || d->block <= 0 || d->stride <= 0 || d->heads <= 0 ||
        d->batch <= 0)
        return fail(1, "config: dimensions must be positive");
    if (d->seq_len % d->block != 0)
        return fail(1, "config: block must divide seq_len (" + std::to_string(d->block) + " vs " +
                           std::to_string(d->seq_len) + ")");
    if (d->block % d->stride != 0) return fail(1, "config: stride must divide block");
    if (d->head_dim % d->stride != 0) return fail(1, "config: stride must divide head_dim");
    // geometry of this sm_100a kernel
    if (d->block != kBlock) return fail(1, "efta_b200: block must be 128 (tcgen05 M=128 tile)");
    if (d->stride != kStride) return fail(1, "efta_b200: stride must be 8");
    if (d->head_dim != 64 && d->head_dim != 128) return fail(1, "efta_b200: head_dim must be 64 or 128");
    if (d->mode < EFTA_MODE_NONE || d->mode > EFTA_MODE_DECOUPLED) return fail(1, "efta_b200: unsupported mode");
    const long long bh = static_cast<long long>(d->batch) * d->heads;
    if (bh > 65535) return fail(1, "efta_b200: batch*heads must be <= 65535");
    if (d->kv_heads < 0 || d->kv_heads > d->heads || (d->kv_heads > 0 && d->heads % d->kv_heads != 0))
        return fail(1, "efta_b200: kv_heads must divide heads (grouped-query attention)");
    if (d->causal) {
        if (d->mode != EFTA_MODE_NONE && d->mode != EFTA_MODE_EFTA_OPT)
            return fail(1, "efta_b200: causal attention runs in modes NONE / EFTA_OPTIMIZED");
        if (d->debug) return fail(1, "efta_b200: causal attention has no fault-tap build");
        if ((d->seq_len / kBlock) % 2 != 0) return fail(1, "efta_b200: causal attention needs an even number of 128-row blocks");
    }
    if (d->o_token_major != 0 && d->o_token_major != 1) return fail(1, "efta_b200: o_token_major must be 0 or 1");
    if (d->o_token_major) {
        if (d->mode != EFTA_MODE_NONE && d->mode != EFTA_MODE_EFTA_OPT)
            return fail(1, "efta_b200: the token-major fp16 output runs in modes NONE / EFTA_OPTIMIZED");
        if ((d->seq_len / kBlock) % 2 != 0)
            return fail(1, "efta_b200: the token-major fp16 output needs an even number of 128-row blocks");
        if (d->debug && d->mode != EFTA_MODE_EFTA_OPT)
            return fail(1, "efta_b200: the token-major fp16 output's tap build is EFTA_OPTIMIZED");
    }
    return 0;
}

// Workspace: [KC: bh*n*32*d fp16] [R2: max(single-CTA VC bh*n*128*64, pair V^T+VC^T
// bh*n*(d+32)*128) fp16] [scratch: 256 B, the persistent pair kernel tile counter]. All offsets 256-byte aligned.
struct WsLayout {
    size_t kc, r2, scratch, part, total;
};
int device_sms() {
    int dev = 0, nsm = 148;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
        nsm = 148;
    return nsm;
}
int kv_heads_of(const efta_attn_desc* d) { return d->kv_heads > 0 ? d->kv_heads : d->heads; }

WsLayout ws_layout(const efta_attn_desc* d) {
    const size_t bh = static_cast<size_t>(d->batch) * kv_heads_of(d);  // checksum operands per K/V head
    const size_t nblk = d->seq_len / kBlock;
    auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
    WsLayout w;
    w.kc = 0;
    w.r2 = al(bh * nblk * 32 * d->head_dim * sizeof(__half));
    const size_t r2 = std::max(bh * nblk * 128 * 64, bh * nblk * (d->head_dim + 32) * 128) * sizeof(__half);
    w.scratch = w.r2 + al(r2);
    w.part = w.scratch + 256;  // scratch: the persistent pair kernel's tile counter
    // decode: the split-KV partial results of every query row
    w.total = w.part + al(efta_decode::part_bytes(d->batch * d->heads, static_cast<int>(nblk), d->head_dim, device_sms()));
    return w;
}
size_t ws_bytes(const efta_attn_desc* d) {
    if (d->mode == EFTA_MODE_DECOUPLED)
        return efta_dec::workspace_bytes(d->batch * d->heads, d->seq_len, d->head_dim);
    return ws_layout(d).total;
}

// Unprotected / EFTA-optimized calls run on CTA pairs (cta_group::2) whenever the number of
// query tiles is even; the `debug` (fault-tap / observation) calls of EFTA_OPT run the tap
// build of the same pair kernel. The single-CTA kernel serves mode EFTA (per-iteration output
// check), odd tile counts, debug calls in mode NONE, and EFTA_NO_PAIR=1 A/B runs.
bool use_pair(const efta_attn_desc* d) {
    if (d->causal || d->o_token_major) return true;  // validated: even block count, NONE / EFTA_OPT, no taps
    if (d->mode == EFTA_MODE_EFTA || ((d->seq_len / kBlock) % 2) != 0) return false;
    if (d->debug && d->mode != EFTA_MODE_EFTA_OPT) return false;
    return std::getenv("EFTA_NO_PAIR") == nullptr;
}

int encode_kv(const efta_attn_desc* d, const void* k, const void* v, void* kc, void* vc,
              cudaStream_t st) {
    const int bh = d->batch * kv_heads_of(d), nblk = d->seq_len / kBlock;
    dim3 grid(nblk, bh);
    if (d->head_dim == 64)
        efta_encode_kv_kernel<64><<<grid, 256, 0, st>>>(
            static_cast<const __half*>(k), static_cast<const __half*>(v), static_cast<__half*>(kc),
            static_cast<__half*>(vc), d->seq_len, nblk);
    else
        efta_encode_kv_kernel<128><<<grid, 256, 0, st>>>(
            static_cast<const __half*>(k), static_cast<const __half*>(v), static_cast<__half*>(kc),
            static_cast<__half*>(vc), d->seq_len, nblk);
    CUDA_TRY(cudaGetLastError());
    return 0;
}

}  // namespace

void efta_internal_set_error(const char* msg) { g_err = msg; }

#ifdef EFTA_PROF
static unsigned long long* efta_prof_buffer_ptr = nullptr;
extern "C" unsigned long long* efta_prof_buffer(void) { return efta_prof_buffer_ptr; }
#endif

extern "C" {

const char* efta_last_error(void) { return g_err.c_str(); }

int efta_attn_validate(const efta_attn_desc* d) { return validate(d); }

size_t efta_attn_workspace_bytes(const efta_attn_desc* d) {
    if (validate(d)) return 0;
    return ws_bytes(d);
}

float efta_flip_bit(float v, int width, int bit) {
    // reference flip_bit (src/fault.cpp:27-37), 32-bit image only on the device path
    uint32_t u;
    std::memcpy(&u, &v, 4);
    if (width != 32 || bit < 0 || bit > 31) return v;
    u ^= (1u << bit);
    std::memcpy(&v, &u, 4);
    return v;
}

int efta_attn_encode_kv_f16(const efta_attn_desc* d, const uint16_t* k, const uint16_t* v,
                            uint16_t* kc, uint16_t* vc, void* stream) {
    if (int rc = validate(d)) return rc;
    return encode_kv(d, k, v, kc, vc, static_cast<cudaStream_t>(stream));
}

int efta_attn_fwd_f16(const efta_attn_desc* d, const uint16_t* q, const uint16_t* k,
                      const uint16_t* v, float* o, float* m_out, float* l_out, void* workspace,
                      size_t workspace_bytes, const efta_fault_spec* faults, int n_faults,
                      efta_event* events, int ev_cap, efta_fired* fired, int fired_cap,
                      efta_counters* counters, void* stream) {
    if (int rc = validate(d)) return rc;
    if (!q || !k || !v || !o || !counters) return fail(1, "efta_attn_fwd_f16: null buffer");
    if (n_faults > 0 && !d->debug)
        return fail(1, "efta_attn_fwd_f16: fault injection needs the debug (tap) kernel variant");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int bh = d->batch * d->heads, nblk = d->seq_len / kBlock, D = d->head_dim;
    const int bh_kv = d->batch * kv_heads_of(d);  // K / V heads (grouped-query attention)
    if (d->mode == EFTA_MODE_DECOUPLED) {
        // the decoupled baseline (src/decoupled.cpp:98-282): three kernels + cuBLAS GEMMs with
        // the N^2 intermediates in the workspace (csrc/decoupled.cu)
        if (workspace == nullptr || workspace_bytes < ws_bytes(d))
            return fail(1, "efta_attn_fwd_f16: workspace too small");
        CUDA_TRY(cudaMemsetAsync(counters, 0, sizeof(efta_counters), st));
        AttnParams p{};
        p.seq_len = d->seq_len;
        p.nblk = nblk;
        p.n_heads_flat = bh;
        p.scale = d->scale == 0.0f ? 1.0f / std::sqrt(static_cast<float>(D)) : d->scale;
        p.rowmax_bias = d->rowmax_bias;
        p.eps1 = d->eps1;
        p.eps2 = d->eps2;
        p.eps_lin = d->eps_lin;
        p.m_out = m_out;
        p.l_out = l_out;
        p.events = events;
        p.ev_cap = events ? ev_cap : 0;
        p.counters = counters;
        p.faults = faults;
        p.n_faults = faults ? n_faults : 0;
        p.fired = fired;
        p.fired_cap = fired ? fired_cap : 0;
        p.heads_q = d->heads;
        p.kv_group = d->heads / kv_heads_of(d);
        const std::string err = efta_dec::forward(p, bh, d->seq_len, D, reinterpret_cast<const __half*>(q),
                                                  reinterpret_cast<const __half*>(k),
                                                  reinterpret_cast<const __half*>(v), o, workspace, st);
        if (!err.empty()) return fail(2, err);
        return 0;
    }
    const bool prot = d->mode != EFTA_MODE_NONE;
    const bool pair = use_pair(d);
    if ((prot || pair) && (workspace == nullptr || workspace_bytes < ws_bytes(d)))
        return fail(1, "efta_attn_fwd_f16: workspace too small");

    CUDA_TRY(cudaMemsetAsync(counters, 0, sizeof(efta_counters), st));
    const WsLayout wl = ws_layout(d);
    char* wsb = static_cast<char*>(workspace);
    uint16_t* kc = wsb ? reinterpret_cast<uint16_t*>(wsb + wl.kc) : nullptr;
    uint16_t* r2 = wsb ? reinterpret_cast<uint16_t*>(wsb + wl.r2) : nullptr;
    CUtensorMap tq, tk, tv, tkc, tvc;
    const uint64_t rows = static_cast<uint64_t>(bh) * d->seq_len;
    const uint64_t kv_rows = static_cast<uint64_t>(bh_kv) * d->seq_len;
    bool ok;
    if (pair) {
        // prepass: KC (protected) + [V^T ; VC^T]; then maps for the half-operands
        if (!d->checksums_ready) {
            cudaError_t e = D == 64 ? efta_launch_encode_pair_d64(prot, k, v, kc, r2, d->seq_len, nblk, bh_kv, st)
                                    : efta_launch_encode_pair_d128(prot, k, v, kc, r2, d->seq_len, nblk, bh_kv, st);
            if (e != cudaSuccess) return fail(2, std::string("encode: ") + cudaGetErrorString(e));
        }
        const int vrows = prot ? D + 32 : D;
        // score operand N = 144 (protected: K + c1_hi + c1_lo rows) or 128, half per CTA:
        // leader K rows 0..71 (0..63), peer K rows 72..127 + two 8-row KC boxes (64..127)
        ok = make_map(&tq, q, rows, D, 128) && make_map(&tk, k, kv_rows, D, prot ? 72 : 64) &&
             make_map(&tvc, r2, static_cast<uint64_t>(bh_kv) * nblk * vrows, 128, vrows / 2);
        if (prot)
            ok = ok && make_map(&tv, k, kv_rows, D, 56) &&
                 make_map(&tkc, kc, static_cast<uint64_t>(bh_kv) * nblk * 32, D, 8);
        else {
            tv = tk;
            tkc = tk;
        }
    } else {
        if (prot && !d->checksums_ready) {
            if (int rc = encode_kv(d, k, v, kc, r2, st)) return rc;
        }
        ok = make_map(&tq, q, rows, D, 128) && make_map(&tk, k, kv_rows, D, 128) &&
             make_map(&tv, v, kv_rows, D, 128);
        if (prot) {
            ok = ok && make_map(&tkc, kc, static_cast<uint64_t>(bh_kv) * nblk * 32, D, 32) &&
                 make_map(&tvc, r2, static_cast<uint64_t>(bh_kv) * nblk * 128, 64, 128);
        } else {
            tkc = tq;
            tvc = tq;
        }
    }
    CUtensorMap to = tq;  // pair kernel: the TMA-stored output (boxes of 32 rows at d=64, 16 at d=128)
    if (ok && pair)
        ok = d->o_token_major
                 ? make_out_map(&to, o, true, static_cast<uint64_t>(d->batch) * d->seq_len,
                                static_cast<uint64_t>(d->heads) * D, D == 64 ? 32 : 16)
                 : make_out_map(&to, o, false, rows, D, D == 64 ? 32 : 16);
    if (!ok) return fail(2, "cuTensorMapEncodeTiled failed (alignment or driver entry point)");

    AttnParams p{};
    p.seq_len = d->seq_len;
    p.nblk = nblk;
    p.n_heads_flat = bh;
    p.scale = d->scale == 0.0f ? 1.0f / std::sqrt(static_cast<float>(D)) : d->scale;
    p.scale_log2 = p.scale * kLog2e;
    p.rowmax_bias = d->rowmax_bias;
    p.eps1 = d->eps1;
    p.eps2 = d->eps2;
    p.eps_lin = d->eps_lin;
    p.o = o;
    p.m_out = m_out;
    p.l_out = l_out;
    p.events = events;
    p.ev_cap = events ? ev_cap : 0;
    p.counters = counters;
    p.faults = faults;
    p.n_faults = faults ? n_faults : 0;
    p.fired = fired;
    p.fired_cap = fired ? fired_cap : 0;
    p.observe_linear = d->observe_linear;
    p.prof = nullptr;
#ifdef EFTA_PROF
    {
        static unsigned long long* prof_buf = nullptr;
        if (!prof_buf) cudaMalloc(&prof_buf, 64 * 64 * sizeof(unsigned long long));
        p.prof = prof_buf;
        efta_prof_buffer_ptr = prof_buf;
    }
#endif
    p.exp_lo = std::isfinite(d->eps1) ? static_cast<float>(std::exp(-d->eps1)) : 0.0f;
    p.exp_hi = std::isfinite(d->eps1) ? static_cast<float>(std::exp(d->eps1)) : INFINITY;
    p.scratch = wsb ? reinterpret_cast<float*>(wsb + wl.scratch) : nullptr;
    p.q = reinterpret_cast<const __half*>(q);
    p.kc = reinterpret_cast<const __half*>(kc);
    p.heads_q = d->heads;
    p.kv_group = d->heads / kv_heads_of(d);
    p.causal = d->causal;
    p.o_tok = d->o_token_major;
    const bool dbg = d->debug != 0;
    cudaError_t e;
    if (pair)  // the persistent pair kernel's in-order tile counter (workspace scratch, int)
        CUDA_TRY(cudaMemsetAsync(wsb + wl.scratch, 0, 16, st));
    if (pair && dbg)  // the tap build: maps as below
        e = (D == 64) ? efta_launch_attn_pair_inj_d64(tq, tk, tv, tkc, tvc, to, p, bh, st)
                      : efta_launch_attn_pair_inj_d128(tq, tk, tv, tkc, tvc, to, p, bh, st);
    else if (pair && d->causal)
        e = (D == 64) ? efta_launch_attn_pair_causal_d64(d->mode, tq, tk, tv, tkc, tvc, to, p, bh, st)
                      : efta_launch_attn_pair_causal_d128(d->mode, tq, tk, tv, tkc, tvc, to, p, bh, st);
    else if (pair)  // maps: q, K half A, K half B (protected peer), KC, [V^T ; VC^T]
        e = (D == 64) ? efta_launch_attn_pair_d64(d->mode, tq, tk, tv, tkc, tvc, to, p, bh, st)
                      : efta_launch_attn_pair_d128(d->mode, tq, tk, tv, tkc, tvc, to, p, bh, st);
    else
        e = (D == 64) ? efta_launch_attn_d64(d->mode, dbg, tq, tk, tv, tkc, tvc, p, bh, st)
                      : efta_launch_attn_d128(d->mode, dbg, tq, tk, tv, tkc, tvc, p, bh, st);
    if (e != cudaSuccess) return fail(2, std::string("attention launch: ") + cudaGetErrorString(e));
    return 0;
}

int efta_decode_fwd_f16(const efta_attn_desc* d, const uint16_t* q, const uint16_t* k, const uint16_t* v,
                        float* o, float* m_out, float* l_out, void* workspace, size_t workspace_bytes,
                        efta_event* events, int ev_cap, efta_counters* counters, void* stream) {
    if (int rc = validate(d)) return rc;
    if (d->mode != EFTA_MODE_NONE && d->mode != EFTA_MODE_EFTA_OPT)
        return fail(1, "efta_decode_fwd_f16: modes NONE / EFTA_OPTIMIZED");
    if (d->debug || d->causal) return fail(1, "efta_decode_fwd_f16: no fault-tap build; the query sees the whole cache");
    if (d->o_token_major) return fail(1, "efta_decode_fwd_f16: fp32 [BH, rows, D] output only");
    if (!q || !k || !v || !o || !counters) return fail(1, "efta_decode_fwd_f16: null buffer");
    const bool prot = d->mode == EFTA_MODE_EFTA_OPT;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    CUDA_TRY(cudaMemsetAsync(counters, 0, sizeof(efta_counters), st));
    const WsLayout wl = ws_layout(d);
    char* wsb = static_cast<char*>(workspace);
    void* kc = wsb ? wsb + wl.kc : nullptr;
    void* vc = wsb ? wsb + wl.r2 : nullptr;
    // the cache's strided checksum operands (KC, per-key VC); a decode loop that appends to the
    // cache keeps them current and passes checksums_ready = 1
    if (prot && !d->checksums_ready)
        if (int rc = encode_kv(d, k, v, kc, vc, st)) return rc;
    AttnParams p{};
    p.seq_len = d->seq_len;
    p.nblk = d->seq_len / kBlock;
    p.n_heads_flat = d->batch * d->heads;
    p.scale = d->scale == 0.0f ? 1.0f / std::sqrt(static_cast<float>(d->head_dim)) : d->scale;
    p.scale_log2 = p.scale * kLog2e;
    p.rowmax_bias = d->rowmax_bias;
    p.eps1 = d->eps1;
    p.eps2 = d->eps2;
    p.eps_lin = d->eps_lin;
    p.exp_lo = std::isfinite(d->eps1) ? static_cast<float>(std::exp(-d->eps1)) : 0.0f;
    p.exp_hi = std::isfinite(d->eps1) ? static_cast<float>(std::exp(d->eps1)) : INFINITY;
    p.o = o;
    p.m_out = m_out;
    p.l_out = l_out;
    p.events = events;
    p.ev_cap = events ? ev_cap : 0;
    p.counters = counters;
    p.heads_q = d->heads;
    p.kv_group = d->heads / kv_heads_of(d);
    if (workspace == nullptr || workspace_bytes < ws_bytes(d)) return fail(1, "efta_decode_fwd_f16: workspace too small");
    cudaError_t e = efta_decode::launch(d->head_dim, prot, p, d->batch * d->heads, q, k, v, kc, vc,
                                        reinterpret_cast<float*>(wsb + wl.part), device_sms(), st);
    if (e != cudaSuccess) return fail(2, std::string("decode launch: ") + cudaGetErrorString(e));
    return 0;
}

int efta_attn_fwd_host_f16(const efta_attn_desc* d, const uint16_t* q, const uint16_t* k,
                           const uint16_t* v, float* o, float* m_out, float* l_out,
                           const efta_fault_spec* faults, int n_faults, efta_event* events,
                           int ev_cap, efta_fired* fired, int fired_cap, efta_counters* counters) {
    if (int rc = validate(d)) return rc;
    if (d->o_token_major) return fail(1, "efta_attn_fwd_host_f16: fp32 [B, H, S, D] output only");
    // The (batch x head) units are independent (the reference's per-head loop,
    // src/campaign.cpp:175), so the host path streams them in chunks over three CUDA
    // streams: H2D of chunk i+1 and D2H of chunk i-1 overlap the kernels of chunk i
    // (separate copy engines; PCIe is full duplex). Fault-injection calls (head-indexed
    // fault tables, fired lists) run as one chunk.
    const int bh = d->batch * d->heads;
    // chunk unit: one head, or one batch entry (all its query heads and their K/V group heads)
    // under grouped-query attention
    const bool gqa = kv_heads_of(d) != d->heads;
    const int units = gqa ? d->batch : bh;
    const int qh_unit = gqa ? d->heads : 1, kvh_unit = gqa ? kv_heads_of(d) : 1;
    int max_chunks = 32;  // small first-H2D / last-D2H tails; EFTA_HOST_CHUNKS overrides (A/B)
    if (const char* ev = std::getenv("EFTA_HOST_CHUNKS")) max_chunks = std::max(1, std::min(64, std::atoi(ev)));
    const int want = (n_faults > 0 || fired) ? 1 : std::min(units, max_chunks);
    const int per = (units + want - 1) / want;
    // chunks actually used (e.g. 33 units in chunks of 2 -> 17): every chunk's counters are read back
    const int nchunk = (units + per - 1) / per;
    struct Scratch {
        void* p = nullptr;
        size_t n = 0;
        cudaStream_t st[3] = {nullptr, nullptr, nullptr};
        cudaEvent_t ev[2 * 64] = {};
        ~Scratch() {
            if (p) cudaFree(p);
            for (auto& x : st) if (x) cudaStreamDestroy(x);
            for (auto& e : ev) if (e) cudaEventDestroy(e);
        }
    };
    // per thread and device (streams and buffers belong to the device current at the call)
    int dev = 0;
    CUDA_TRY(cudaGetDevice(&dev));
    if (dev < 0 || dev >= 64) return fail(2, "efta_attn_fwd_host_f16: device index out of range");
    thread_local Scratch scratch_per_dev[64];
    Scratch& s = scratch_per_dev[dev];
    if (!s.st[0]) {
        for (auto& x : s.st) CUDA_TRY(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking));
        for (auto& e : s.ev) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    const size_t head_elems = static_cast<size_t>(d->seq_len) * d->head_dim;
    const size_t n_in = static_cast<size_t>(bh) * head_elems;
    const size_t n_kv = static_cast<size_t>(d->batch) * kv_heads_of(d) * head_elems;
    const size_t bytes_in = n_in * 2, bytes_kv = n_kv * 2, bytes_o = n_in * 4,
                 bytes_ml = static_cast<size_t>(bh) * d->seq_len * 4;
    efta_attn_desc dc = *d;  // one chunk: `per` units
    if (gqa) {
        dc.batch = per;
    } else {
        dc.batch = 1;
        dc.heads = per;
        dc.kv_heads = 0;
    }
    const size_t wsb = ws_bytes(&dc);
    auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
    const size_t need = al(bytes_in) + 2 * al(bytes_kv) + al(bytes_o) + 2 * al(bytes_ml) + al(wsb) +
                        nchunk * al(sizeof(efta_counters)) + al(sizeof(efta_fault_spec) * (n_faults + 1)) +
                        nchunk * al(sizeof(efta_event) * (ev_cap + 1)) + al(sizeof(efta_fired) * (fired_cap + 1));
    if (s.n < need) {
        if (s.p) cudaFree(s.p);
        s.p = nullptr;
        s.n = 0;
        CUDA_TRY(cudaMalloc(&s.p, need));
        s.n = need;
    }
    char* base = static_cast<char*>(s.p);
    auto take = [&](size_t b) { char* r = base; base += al(b); return r; };
    uint16_t* dq = reinterpret_cast<uint16_t*>(take(bytes_in));
    uint16_t* dk = reinterpret_cast<uint16_t*>(take(bytes_kv));
    uint16_t* dv = reinterpret_cast<uint16_t*>(take(bytes_kv));
    float* dout = reinterpret_cast<float*>(take(bytes_o));
    float* dm = reinterpret_cast<float*>(take(bytes_ml));
    float* dl = reinterpret_cast<float*>(take(bytes_ml));
    void* dws = take(wsb);
    efta_counters* dcnt = reinterpret_cast<efta_counters*>(take(nchunk * al(sizeof(efta_counters))));
    efta_fault_spec* df = reinterpret_cast<efta_fault_spec*>(take(sizeof(efta_fault_spec) * (n_faults + 1)));
    efta_event* de = reinterpret_cast<efta_event*>(take(nchunk * al(sizeof(efta_event) * (ev_cap + 1))));
    efta_fired* dfi = reinterpret_cast<efta_fired*>(take(sizeof(efta_fired) * (fired_cap + 1)));
    const size_t cnt_stride = al(sizeof(efta_counters)), ev_stride = al(sizeof(efta_event) * (ev_cap + 1));
    cudaStream_t h2d = s.st[0], comp = s.st[1], d2h = s.st[2];
    if (n_faults > 0)
        CUDA_TRY(cudaMemcpyAsync(df, faults, sizeof(efta_fault_spec) * n_faults, cudaMemcpyHostToDevice, h2d));
    for (int c = 0; c < nchunk; ++c) {
        const int u0 = c * per, nu = std::min(per, units - u0);
        if (nu <= 0) break;
        const int h0 = u0 * qh_unit, nh = nu * qh_unit;
        const size_t e0 = static_cast<size_t>(h0) * head_elems, ne = static_cast<size_t>(nh) * head_elems;
        const size_t k0 = static_cast<size_t>(u0) * kvh_unit * head_elems,
                     nk = static_cast<size_t>(nu) * kvh_unit * head_elems;
        const size_t r0 = static_cast<size_t>(h0) * d->seq_len, nr = static_cast<size_t>(nh) * d->seq_len;
        CUDA_TRY(cudaMemcpyAsync(dq + e0, q + e0, ne * 2, cudaMemcpyHostToDevice, h2d));
        CUDA_TRY(cudaMemcpyAsync(dk + k0, k + k0, nk * 2, cudaMemcpyHostToDevice, h2d));
        CUDA_TRY(cudaMemcpyAsync(dv + k0, v + k0, nk * 2, cudaMemcpyHostToDevice, h2d));
        CUDA_TRY(cudaEventRecord(s.ev[2 * c], h2d));
        CUDA_TRY(cudaStreamWaitEvent(comp, s.ev[2 * c], 0));
        efta_attn_desc dcc = *d;
        if (nchunk > 1) {
            if (gqa) {
                dcc.batch = nu;
            } else {
                dcc.batch = 1;
                dcc.heads = nh;
                dcc.kv_heads = 0;
            }
        }
        dcc.checksums_ready = 0;  // the internal workspace never holds this call's operands
        efta_counters* cc = reinterpret_cast<efta_counters*>(reinterpret_cast<char*>(dcnt) + c * cnt_stride);
        efta_event* ce = reinterpret_cast<efta_event*>(reinterpret_cast<char*>(de) + c * ev_stride);
        int rc = efta_attn_fwd_f16(&dcc, dq + e0, dk + k0, dv + k0, dout + e0, dm + r0, dl + r0, dws, wsb,
                                   n_faults > 0 ? df : nullptr, n_faults, events ? ce : nullptr,
                                   events ? ev_cap : 0, fired ? dfi : nullptr, fired ? fired_cap : 0, cc, comp);
        if (rc) return rc;
        CUDA_TRY(cudaEventRecord(s.ev[2 * c + 1], comp));
        CUDA_TRY(cudaStreamWaitEvent(d2h, s.ev[2 * c + 1], 0));
        CUDA_TRY(cudaMemcpyAsync(o + e0, dout + e0, ne * 4, cudaMemcpyDeviceToHost, d2h));
        if (m_out) CUDA_TRY(cudaMemcpyAsync(m_out + r0, dm + r0, nr * 4, cudaMemcpyDeviceToHost, d2h));
        if (l_out) CUDA_TRY(cudaMemcpyAsync(l_out + r0, dl + r0, nr * 4, cudaMemcpyDeviceToHost, d2h));
    }
    std::vector<efta_counters> hc(nchunk);
    for (int c = 0; c < nchunk; ++c)
        CUDA_TRY(cudaMemcpyAsync(&hc[c], reinterpret_cast<char*>(dcnt) + c * cnt_stride, sizeof(efta_counters),
                                 cudaMemcpyDeviceToHost, d2h));
    CUDA_TRY(cudaStreamSynchronize(d2h));
    // merge the chunks' counters and events (event heads back to the flat index)
    efta_counters tot{};
    int n_ev = 0;
    for (int c = 0; c < nchunk; ++c) {
        const efta_counters& x = hc[c];
        tot.n_fired += x.n_fired;
        tot.detections += x.detections;
        tot.corrections += x.corrections;
        tot.recomputes += x.recomputes;
        tot.range_replacements += x.range_replacements;
        tot.failed |= x.failed;
        for (int f = 0; f < 3; ++f) tot.family_max[f] = std::max(tot.family_max[f], x.family_max[f]);
        if (events && ev_cap > 0 && x.n_events > 0) {
            const int take_n = std::min(x.n_events, ev_cap - n_ev);
            if (take_n > 0) {
                const char* src = reinterpret_cast<const char*>(de) + c * ev_stride;
                CUDA_TRY(cudaMemcpy(events + n_ev, src, sizeof(efta_event) * take_n, cudaMemcpyDeviceToHost));
                for (int i = 0; i < take_n; ++i) events[n_ev + i].head += c * per * qh_unit;
                n_ev += take_n;
            }
        }
        tot.n_events += x.n_events;
    }
    if (counters) *counters = tot;
    if (fired && fired_cap > 0 && tot.n_fired > 0)
        CUDA_TRY(cudaMemcpy(fired, dfi, sizeof(efta_fired) * std::min(tot.n_fired, fired_cap), cudaMemcpyDeviceToHost));
    return 0;
}

}  // extern "C"
