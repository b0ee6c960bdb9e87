// mma2_bench.cu — tcgen05.mma.cta_group::2 throughput (CTA pairs, M=256 across the pair),
// optionally with concurrent TMEM traffic from 8 "row" warps (tcgen05.ld of 64 columns
// + tcgen05.st of 32 per loop, like the softmax warps of the EFTA kernel).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/mma2_bench tools/mma2_bench.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#include "../paper_2504_02211_b200/csrc/sm100_ptx.cuh"

using namespace efta_sm100;

__device__ __forceinline__ uint32_t cta_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cl_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mma2_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(a), "l"(b),
                 "r"(idesc), "r"(acc) : "memory");
}
__device__ __forceinline__ void mma2_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d), "r"(a), "l"(b),
                 "r"(idesc), "r"(acc) : "memory");
}
__device__ __forceinline__ void commit2(uint64_t* bar) {
    asm volatile("{\n\t.reg .b16 m;\n\tmov.b16 m, 3;\n\t"
                 "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n\t}"
                 ::"r"(smem_u32(bar)) : "memory");
}

// MODE 0: SS (A K-major, B K-major), 1: TS (A TMEM, B MN-major), 2: alternating 8 SS + 8 TS
template <int MODE, int N, bool LOAD, bool RND = false, bool COMMIT = false, int POLL = 0, int FENCE = 0>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(384, 1) bench(unsigned long long* out, int iters) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint32_t tslot;
    __shared__ uint64_t bar, cb[4];
    __shared__ volatile int done, pv_done;
    __shared__ volatile unsigned long long pv_t;
    const int warp = threadIdx.x / 32;
    const uint32_t rank = cta_rank();
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    if (threadIdx.x == 0) { mbar_init(&bar, 1); for (int i = 0; i < 4; ++i) mbar_init(&cb[i], 1); fence_barrier_init(); done = 0; pv_done = 0; }
    for (int i = threadIdx.x; i < 100 * 1024 / 4 - 256; i += blockDim.x) {
        uint32_t h = (i + 1) * 2654435761u ^ (blockIdx.x * 40503u);
        h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
        const float a = (h & 0xffff) / 32768.0f - 1.0f, b = (h >> 16) / 32768.0f - 1.0f;
        reinterpret_cast<uint32_t*>(smem)[i] = RND ? pack_half2(a, b) : 0x3c003c00u;
    }
    tc_fence_before();
    __syncthreads();
    cl_sync();
    tc_fence_after();
    const uint32_t tmem = tslot;
    if (RND && warp >= 4 && warp < 8) {  // random fp16 pairs in every TMEM column (TS A operand)
        uint32_t r[32];
        for (int c = 0; c < 512; c += 32) {
            for (int x = 0; x < 32; ++x) {
                uint32_t h = (threadIdx.x * 977u + c * 31u + x) * 2654435761u;
                h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
                r[x] = pack_half2((h & 0xffff) / 65536.0f, (h >> 16) / 65536.0f);
            }
            tmem_st32(tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16) + c, r);
        }
        tmem_wait_st();
    }
    tc_fence_before();
    __syncthreads();
    cl_sync();
    tc_fence_after();
    if (MODE == 5 && rank == 0 && (threadIdx.x == 32 || threadIdx.x == 64)) {
        const uint32_t b = smem_u32(smem) + 32768;
        constexpr uint32_t ID = idesc_f16_f32(256, N, 0, 0);
        const bool qk = threadIdx.x == 32;
        unsigned long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            if (FENCE >= 4) { const long long t = clock64(); while (clock64() - t < FENCE) { } }
            if (qk) {
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
                    mma2_ts(tmem + (it & 1) * 128, tmem + 384 + kk * 8,
                            smem_desc_sw128(b + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024), ID, kk > 0);
                commit2(&cb[0]);
            } else {
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
                    mma2_ts(tmem + 256, tmem + 448 + kk * 8,
                            smem_desc_sw128(b + 32768 + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024), ID, 1);
                commit2(&cb[2]);
            }
        }
        commit2(qk ? &cb[1] : &cb[3]);
        mbar_wait(qk ? &cb[1] : &cb[3], 0);
        unsigned long long t1 = clock64();
        if (!qk) { pv_t = t1 - t0; __threadfence_block(); pv_done = 1; }
        else {
            while (!pv_done) { }
            out[blockIdx.x / 2] = (t1 - t0) > pv_t ? (t1 - t0) : pv_t;
            done = 1;
        }
    } else if (MODE == 5 && rank == 1 && threadIdx.x == 32) {
        mbar_wait(&cb[1], 0);
        done = 1;
    } else if (MODE == 5) {
    } else if (threadIdx.x == 0 && rank == 0) {
        const uint32_t a = smem_u32(smem), b = a + 32768;
        constexpr uint32_t ID_SS = idesc_f16_f32(256, N, 0, 0);
        constexpr uint32_t ID_TS = idesc_f16_f32(256, N, 0, 1);
        unsigned long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            if (MODE == 0 || MODE == 2) {
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
                    mma2_ss(tmem, smem_desc_sw128(a + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                            smem_desc_sw128(b + (kk >> 2) * 20480 + (kk & 3) * 32, 16, 1024), ID_SS, 1);
                if (COMMIT) { commit2(&cb[0]); commit2(&cb[1]); }
            }
            if (MODE == 3 || MODE == 4) {
                // the EFTA pair-kernel pattern: S(it) = Q.K^T into S[it&1] (A = Q in TMEM cols 384..),
                // then O += P(it-1).V with A = the S region of it-1 (MODE 3) or a region no MMA
                // writes (MODE 4)
                const uint32_t d_s = tmem + (it & 1) * 128;
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
                    mma2_ts(d_s, tmem + 384 + kk * 8, smem_desc_sw128(b + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024),
                            ID_SS, kk > 0);
                if (COMMIT) { commit2(&cb[0]); commit2(&cb[1]); }
                if (FENCE & 1) tc_fence_after();
                if (FENCE & 2) { mbar_wait(&cb[0], it & 1); }
                if (FENCE >= 4) { const long long t = clock64(); while (clock64() - t < FENCE) { } }
                const uint32_t a_p = MODE == 3 ? tmem + ((it + 1) & 1) * 128 : tmem + 448;
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
                    mma2_ts(tmem + 256, a_p + kk * 8, smem_desc_sw128(b + 32768 + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024),
                            ID_SS, 1);
                if (COMMIT) { commit2(&cb[2]); commit2(&cb[3]); }
                if (FENCE & 1) tc_fence_after();
                if (FENCE >= 4) { const long long t = clock64(); while (clock64() - t < FENCE) { } }
            }
            if (MODE == 1 || MODE == 2) {
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
                    mma2_ts(tmem + 256, tmem + 160 + kk * 8, smem_desc_sw128(b + (kk >> 2) * 10240 + (kk & 3) * 32, 16, 1024),
                            ID_TS, 1);
                if (COMMIT) { commit2(&cb[2]); commit2(&cb[3]); }
            }
        }
        commit2(&bar);
        mbar_wait(&bar, 0);
        unsigned long long t1 = clock64();
        out[blockIdx.x / 2] = (t1 - t0);
        done = 1;
    } else if (threadIdx.x == 0) {
        mbar_wait(&bar, 0);
        done = 1;
    } else if (POLL && warp >= 4 && warp < 4 + POLL) {
        // spin on an mbarrier phase that never completes (like warps waiting for S / empty slots)
        while (!done) {
            if (mbar_try_wait(&cb[3], 1)) { }
            if (mbar_try_wait(&bar, 1)) { }
        }
    } else if (LOAD && warp >= 4) {
        const int wq = warp & 3;
        const uint32_t lb = tmem + (static_cast<uint32_t>(wq * 32) << 16) + (warp >= 8 ? 64 : 0);
        uint32_t r[32];
        float acc = 0.0f;
        while (!done) {
            tmem_ld32(lb + 320, r);
            tmem_ld32(lb + 352, r);
            tmem_wait_ld();
#pragma unroll
            for (int x = 0; x < 32; ++x) acc += __uint_as_float(r[x]);
            tmem_st32(lb + 384, r);
            tmem_wait_st();
        }
        if (acc == 12345.0f) out[0] = 0;
    }
    tc_fence_before();
    __syncthreads();
    cl_sync();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

template <int MODE, int N, bool LOAD, bool RND = false, bool COMMIT = false, int POLL = 0, int FENCE = 0>
void run(const char* name, int nblocks) {
    unsigned long long* d;
    cudaMalloc(&d, nblocks * 8);
    const int smem = 100 * 1024;
    cudaFuncSetAttribute(bench<MODE, N, LOAD, RND, COMMIT, POLL, FENCE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int iters = getenv("ITERS") ? atoi(getenv("ITERS")) : 2000;
    bench<MODE, N, LOAD, RND, COMMIT, POLL, FENCE><<<nblocks, 384, smem>>>(d, 10);
    bench<MODE, N, LOAD, RND, COMMIT, POLL, FENCE><<<nblocks, 384, smem>>>(d, iters);
    cudaError_t e = cudaDeviceSynchronize();
    static unsigned long long h[1024];
    cudaMemcpy(h, d, nblocks / 2 * 8, cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < nblocks / 2; ++i) avg += h[i];
    avg /= nblocks / 2;
    const int per_iter = MODE >= 2 ? 16 : 8;
    const double per = avg / (iters * double(per_iter));
    const double floor_ = 128.0 * N / 256.0;  // per SM: 128 rows x N x 16
    printf("%-40s N=%3d  %7.1f clk/MMA  (floor %5.1f, efficiency %5.1f%%)  %s\n", name, N, per, floor_,
           100.0 * floor_ / per, e == cudaSuccess ? "" : cudaGetErrorString(e));
    cudaFree(d);
}

int main() {
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    run<0, 128, false>("pair SS M=256", nsm);
    run<0, 160, false>("pair SS M=256", nsm);
    run<1, 128, false>("pair TS M=256 (B MN-major)", nsm);
    run<1, 160, false>("pair TS M=256 (B MN-major)", nsm);
    run<2, 128, false>("pair SS+TS alternating", nsm);
    run<2, 160, false>("pair SS+TS alternating", nsm);
    run<0, 128, true>("pair SS M=256 + TMEM ld/st traffic", nsm);
    run<1, 128, true>("pair TS M=256 + TMEM ld/st traffic", nsm);
    run<2, 128, true>("pair SS+TS + TMEM ld/st traffic", nsm);
    run<2, 160, true>("pair SS+TS + TMEM ld/st traffic", nsm);
    run<0, 128, false, true>("pair SS random data", nsm);
    run<1, 128, false, true>("pair TS random data", nsm);
    run<2, 128, false, true>("pair SS+TS random data", nsm);
    run<2, 128, true, true>("pair SS+TS random + TMEM traffic", nsm);
    run<2, 160, true, true>("pair SS+TS random + TMEM traffic", nsm);
    run<2, 128, false, false, true>("pair SS+TS + 2 commits per group", nsm);
    run<3, 128, false, false, true>("kernel pattern: PV A = previous S region", nsm);
    run<4, 128, false, false, true>("kernel pattern: PV A = unwritten region", nsm);
    run<3, 128, false, false, false>("kernel pattern (3), no commits", nsm);
    run<3, 128, false, false, true, 2>("kernel pattern + 2 warps polling mbarriers", nsm);
    run<3, 128, false, false, true, 8>("kernel pattern + 8 warps polling mbarriers", nsm);
    run<3, 128, false, false, true, 0, 1>("kernel pattern + fence::after_thread_sync", nsm);
    run<3, 128, false, false, true, 0, 2>("kernel pattern + wait on S(it) commit", nsm);
    run<3, 128, false, false, true, 0, 64>("kernel pattern + 64 clk gap per group", nsm);
    run<3, 128, false, false, true, 0, 128>("kernel pattern + 128 clk gap per group", nsm);
    run<3, 128, false, false, true, 0, 200>("kernel pattern + 200 clk gap per group", nsm);
    run<3, 128, false, false, true, 0, 400>("kernel pattern + 400 clk gap per group", nsm);
    run<5, 128, false, false, true, 0, 0>("two issuers (QK warp, PV warp), no gap", nsm);
    run<5, 128, false, false, true, 0, 200>("two issuers, 200 clk gap per group", nsm);
    run<5, 128, false, false, true, 0, 400>("two issuers, 400 clk gap per group", nsm);
    run<1, 128, false, false, true>("pair TS + 2 commits per group", nsm);
    return 0;
}
