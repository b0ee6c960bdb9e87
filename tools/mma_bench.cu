// mma_bench.cu — tcgen05.mma issue/throughput microbenchmark (one CTA per SM).
// Measures cycles per kind::f16 M=128 K=16 MMA for SS / TS operand sources and K- / MN-major B,
// with operands resident in SMEM/TMEM (contents irrelevant). Build + run:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mma_bench tools/mma_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "../paper_2504_02211_b200/csrc/sm100_ptx.cuh"

using namespace efta_sm100;

template <int MODE, int N>  // MODE 0: SS K/K, 1: SS K/MN, 2: TS B K-major, 3: TS B MN-major
__global__ void __launch_bounds__(128, 1) bench(unsigned long long* out, int iters) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint32_t tslot;
    __shared__ uint64_t bar;
    const int warp = threadIdx.x / 32;
    if (warp == 0) tmem_alloc(&tslot, 512);
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
    for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tslot;
    if (threadIdx.x == 0) {
        const uint32_t a = smem_u32(smem), b = a + 32768;
        constexpr uint32_t ID = idesc_f16_f32(128, N, 0, (MODE == 1 || MODE == 3) ? 1 : 0);
        unsigned long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                const uint64_t bd = (MODE == 1 || MODE == 3) ? smem_desc_sw128(b + kk * 2048, 16384, 1024)
                                                             : smem_desc_sw128(b + (kk >> 2) * 20480 + (kk & 3) * 32, 16, 1024);
                if (MODE <= 1)
                    mma_ss(tmem, smem_desc_sw128(a + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024), bd, ID, 1);
                else
                    mma_ts(tmem, tmem + 320 + kk * 8, bd, ID, 1);
            }
        }
        tc_commit(&bar);
        mbar_wait(&bar, 0);
        unsigned long long t1 = clock64();
        out[blockIdx.x] = (t1 - t0);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 512);
}

template <int MODE, int N>
void run(const char* name, int nblocks) {
    unsigned long long* d;
    cudaMalloc(&d, nblocks * 8);
    const int smem = 100 * 1024;
    cudaFuncSetAttribute(bench<MODE, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int iters = 2000;
    bench<MODE, N><<<nblocks, 128, smem>>>(d, 10);
    bench<MODE, N><<<nblocks, 128, smem>>>(d, iters);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[1024];
    cudaMemcpy(h, d, nblocks * 8, cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < nblocks; ++i) avg += h[i];
    avg /= nblocks;
    const double per = avg / (iters * 8.0);
    const double floor_ = 128.0 * N / 256.0;
    printf("%-28s N=%3d  %7.1f clk/MMA  (floor %5.1f, efficiency %5.1f%%)  %s\n", name, N, per, floor_,
           100.0 * floor_ / per, e == cudaSuccess ? "" : cudaGetErrorString(e));
    cudaFree(d);
}

int main() {
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    run<0, 128>("SS  A K-major, B K-major", nsm);
    run<0, 160>("SS  A K-major, B K-major", nsm);
    run<1, 128>("SS  A K-major, B MN-major", nsm);
    run<1, 160>("SS  A K-major, B MN-major", nsm);
    run<2, 128>("TS  A TMEM,   B K-major", nsm);
    run<2, 160>("TS  A TMEM,   B K-major", nsm);
    run<3, 128>("TS  A TMEM,   B MN-major", nsm);
    run<3, 160>("TS  A TMEM,   B MN-major", nsm);
    run<3, 64>("TS  A TMEM,   B MN-major", nsm);
    run<3, 96>("TS  A TMEM,   B MN-major", nsm);
    run<0, 256>("SS  A K-major, B K-major", nsm);
    run<2, 256>("TS  A TMEM,   B K-major", nsm);
    return 0;
}
