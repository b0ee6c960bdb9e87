// Element-wise pass of the FT-Transformer layer that stays outside the protected kernels: the
// FFN activation (erf GELU) between the two strided-ABFT GEMMs. Not a reference feature (the
// reference has no transformer layer).
//
// The input is fp16, so the activation is a function of 65536 codes: a 128 KB table, built once
// per device with torch's fp32 formula (x * 0.5 * (1 + erf(x / sqrt 2)), one rounding to fp16 —
// bit-identical to torch.nn.functional.gelu by construction), is staged into each CTA's shared
// memory; the pass is then a 16-byte load, eight shared-memory lookups and a 16-byte store per 8
// elements. Evaluating erff per element made the pass issue-bound (~100 us for 16K x 5120, half
// the HBM rate); the lookups keep it on the HBM bound. One CTA per SM (the table fills 128 KB).
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <mutex>

#include "../../include/efta_b200.h"

void efta_internal_set_error(const char* msg);

namespace {

constexpr int kCodes = 65536;
constexpr int kThreads = 1024;

__global__ void gelu_table_kernel(__half* t) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= kCodes) return;
    const float x = __half2float(__ushort_as_half(static_cast<unsigned short>(i)));
    t[i] = __float2half_rn(x * 0.5f * (1.0f + erff(x * 0.70710678118654752440f)));
}

__global__ void __launch_bounds__(kThreads, 1)
gelu_lut_kernel(const uint4* __restrict__ table, const uint4* __restrict__ x, uint4* __restrict__ y, size_t n8,
                const unsigned short* __restrict__ xt, unsigned short* __restrict__ yt, int tail) {
    extern __shared__ uint4 lut4[];
    for (int i = threadIdx.x; i < kCodes / 8; i += kThreads) lut4[i] = table[i];
    __syncthreads();
    const unsigned short* lut = reinterpret_cast<const unsigned short*>(lut4);
    // four 16-byte loads in flight per thread (64 KB per SM: enough bytes in flight for HBM)
    const size_t stride = static_cast<size_t>(gridDim.x) * kThreads;
    size_t i = static_cast<size_t>(blockIdx.x) * kThreads + threadIdx.x;
    for (; i + 3 * stride < n8; i += 4 * stride) {
        uint4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = __ldcs(x + i + u * stride);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            uint32_t* w = &v[u].x;
#pragma unroll
            for (int e = 0; e < 4; ++e)
                w[e] = static_cast<uint32_t>(lut[w[e] & 0xffffu]) | (static_cast<uint32_t>(lut[w[e] >> 16]) << 16);
            __stcs(y + i + u * stride, v[u]);
        }
    }
    for (; i < n8; i += stride) {
        uint4 v = __ldcs(x + i);
        uint32_t* w = &v.x;
#pragma unroll
        for (int e = 0; e < 4; ++e)
            w[e] = static_cast<uint32_t>(lut[w[e] & 0xffffu]) | (static_cast<uint32_t>(lut[w[e] >> 16]) << 16);
        __stcs(y + i, v);
    }
    if (blockIdx.x == 0 && static_cast<int>(threadIdx.x) < tail) yt[threadIdx.x] = lut[xt[threadIdx.x]];
}

struct DeviceTable {
    std::once_flag once;
    __half* p = nullptr;
    cudaError_t err = cudaSuccess;
};
DeviceTable g_tables[64];

}  // namespace

extern "C" int efta_gelu_f16(const uint16_t* x, uint16_t* y, size_t n, void* stream) {
    if (n == 0) return 0;
    if (!x || !y) {
        efta_internal_set_error("efta_gelu_f16: null buffer");
        return 1;
    }
    if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) & 15) {
        efta_internal_set_error("efta_gelu_f16: buffers must be 16-byte aligned");
        return 1;
    }
    int dev = 0, nsm = 148;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) {
        efta_internal_set_error("efta_gelu_f16: no current device");
        return 2;
    }
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    DeviceTable& tb = g_tables[dev];
    std::call_once(tb.once, [&] {  // the table, built once per device (synchronously)
        tb.err = cudaMalloc(&tb.p, kCodes * sizeof(__half));
        if (tb.err == cudaSuccess) {
            gelu_table_kernel<<<kCodes / 256, 256>>>(tb.p);
            tb.err = cudaDeviceSynchronize();
        }
        if (tb.err == cudaSuccess)
            tb.err = cudaFuncSetAttribute(gelu_lut_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kCodes * 2);
    });
    if (tb.err != cudaSuccess) {
        efta_internal_set_error(cudaGetErrorString(tb.err));
        return 2;
    }
    const size_t n8 = n / 8;
    const int tail = static_cast<int>(n - n8 * 8);
    const int grid = static_cast<int>(std::max<size_t>(1, std::min<size_t>((n8 + kThreads - 1) / kThreads, static_cast<size_t>(nsm))));
    gelu_lut_kernel<<<grid, kThreads, kCodes * 2, static_cast<cudaStream_t>(stream)>>>(
        reinterpret_cast<const uint4*>(tb.p), reinterpret_cast<const uint4*>(x), reinterpret_cast<uint4*>(y), n8,
        reinterpret_cast<const unsigned short*>(x) + n8 * 8, reinterpret_cast<unsigned short*>(y) + n8 * 8, tail);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        efta_internal_set_error(cudaGetErrorString(e));
        return 2;
    }
    return 0;
}
