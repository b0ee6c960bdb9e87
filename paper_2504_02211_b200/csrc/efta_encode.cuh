// efta_encode.cuh — strided checksum operands for the K/V tiles (HBM-bound prepass).
//
// For every (head, key block j) this writes the two operand tiles the fused
// kernel loads alongside K_j / V_j:
//   KC[32 x D]   row x     : c1_hi  of  sum_l K[j*128 + x + 8l][:]         (x < 8)
//                row 8+x   : c2_hi  of  sum_l (l+1) K[j*128 + x + 8l][:]
//                row 16+x  : c1_lo, row 24+x: c2_lo
//   VC[128 x 64] row = key : cols x / 8+x / 16+x / 24+x = c1_hi / c2_hi / c1_lo / c2_lo
//                of sum_g V[j*128 + key][x + 8g]; cols 32..63 zero (MN-major operand
//                appended to V_j, see efta_attn.cuh)
// c1/c2 follow encode_strided (src/abft.cpp:19-42): unit and (l+1) group
// weights, fp32 accumulation in ascending l. K's checksums run over the key
// (column) index of K_j^T = the score tile's columns; V's run over head_dim =
// the output tile's columns (src/efta.cpp:128, :271).
// hi = fp16(c), lo = fp16(c - hi): the pair carries ~22 mantissa bits, which
// keeps the tensor-core checksum residual at the fp32 level.
#pragma once
#include <cuda_fp16.h>
#include <cstdint>

namespace efta_sm100 {

template <int D>
__global__ void __launch_bounds__(256) efta_encode_kv_kernel(const __half* __restrict__ k,
                                                             const __half* __restrict__ v,
                                                             __half* __restrict__ kc,
                                                             __half* __restrict__ vc, int seq_len,
                                                             int nblk) {
    constexpr int G_O = D / 8;  // output-tile groups
    __shared__ __half sv[128 * (D + 8)];
    const int j = blockIdx.x, head = blockIdx.y;
    const size_t row0 = static_cast<size_t>(head) * seq_len + static_cast<size_t>(j) * 128;
    const size_t crow0 = (static_cast<size_t>(head) * nblk + j) * 32;
    // stage V_j (rows padded to dodge bank conflicts on the strided reads)
    for (int idx = threadIdx.x; idx < 128 * D / 8; idx += blockDim.x) {
        const int r = idx / (D / 8), c8 = idx % (D / 8);
        const uint4 val = reinterpret_cast<const uint4*>(v + (row0 + r) * D)[c8];
        *reinterpret_cast<uint4*>(&sv[r * (D + 8) + c8 * 8]) = val;
    }
    // KC: one thread per (x, dim); reads K columns straight from global (coalesced over dim)
    for (int t = threadIdx.x; t < 8 * D; t += blockDim.x) {
        const int x = t / D, dim = t % D;
        float c1 = 0.0f, c2 = 0.0f;
#pragma unroll
        for (int l = 0; l < 16; ++l) {
            const float val = __half2float(k[(row0 + x + 8 * l) * D + dim]);
            c1 = __fadd_rn(c1, val);
            c2 = __fadd_rn(c2, __fmul_rn(static_cast<float>(l + 1), val));
        }
        const __half h1 = __float2half_rn(c1), h2 = __float2half_rn(c2);
        kc[(crow0 + x) * D + dim] = h1;
        kc[(crow0 + 8 + x) * D + dim] = h2;
        kc[(crow0 + 16 + x) * D + dim] = __float2half_rn(__fsub_rn(c1, __half2float(h1)));
        kc[(crow0 + 24 + x) * D + dim] = __float2half_rn(__fsub_rn(c2, __half2float(h2)));
    }
    __syncthreads();
    // VC (MN-major, one 64-wide row per key): thread per (key, x)
    const size_t vrow0 = (static_cast<size_t>(head) * nblk + j) * 128;
    for (int t = threadIdx.x; t < 8 * 128; t += blockDim.x) {
        const int key = t / 8, x = t % 8;
        float c1 = 0.0f, c2 = 0.0f;
#pragma unroll
        for (int g = 0; g < G_O; ++g) {
            const float val = __half2float(sv[key * (D + 8) + x + 8 * g]);
            c1 = __fadd_rn(c1, val);
            c2 = __fadd_rn(c2, __fmul_rn(static_cast<float>(g + 1), val));
        }
        const __half h1 = __float2half_rn(c1), h2 = __float2half_rn(c2);
        __half* dst = vc + (vrow0 + key) * 64;
        dst[x] = h1;
        dst[8 + x] = h2;
        dst[16 + x] = __float2half_rn(__fsub_rn(c1, __half2float(h1)));
        dst[24 + x] = __float2half_rn(__fsub_rn(c2, __half2float(h2)));
        dst[32 + x] = __float2half_rn(0.0f);
        dst[40 + x] = __float2half_rn(0.0f);
        dst[48 + x] = __float2half_rn(0.0f);
        dst[56 + x] = __float2half_rn(0.0f);
    }
}

}  // namespace efta_sm100
