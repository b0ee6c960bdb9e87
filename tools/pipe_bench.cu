// pipe_bench.cu — per-SM-subpartition throughput of MUFU.EX2, FFMA2 and the FMA-pipe exp2
// polynomial (one warp per SMSP, 8 independent chains), in clk per warp instruction.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/pipe_bench tools/pipe_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2504_02211_b200/csrc/sm100_ptx.cuh"

using namespace efta_sm100;

template <int KIND>
__global__ void __launch_bounds__(512, 1) kbench(float* out, int iters, unsigned long long* cyc) {
    float2 v[8];
    for (int i = 0; i < 8; ++i) v[i] = make_float2(-0.001f * (threadIdx.x + i), -0.002f * i);
    const float2 s = make_float2(0.999f, 0.999f), b = make_float2(-0.0001f, -0.0001f);
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (KIND == 0) {  // 2 MUFU.EX2 per pair
                v[i].x = ex2_approx(v[i].x) - 1.0f;
                v[i].y = ex2_approx(v[i].y) - 1.0f;
            } else if (KIND == 1) {  // FFMA2
                v[i] = ffma2(v[i], s, b);
            } else if (KIND == 2) {  // polynomial exp2 on a pair
                float2 e = ex2_poly2(v[i]);
                v[i] = make_float2(e.x - 1.0f, e.y - 1.0f);
            } else {  // 3 MUFU pairs : 1 poly pair mix (the kernel's 25% split)
                if (i % 4 == 3) {
                    float2 e = ex2_poly2(v[i]);
                    v[i] = make_float2(e.x - 1.0f, e.y - 1.0f);
                } else {
                    v[i].x = ex2_approx(v[i].x) - 1.0f;
                    v[i].y = ex2_approx(v[i].y) - 1.0f;
                }
            }
        }
    }
    unsigned long long t1 = clock64();
    float acc = 0;
    for (int i = 0; i < 8; ++i) acc += v[i].x + v[i].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int KIND>
void run(const char* name, double elems_per_iter, int threads = 128) {
    float* o;
    unsigned long long* c;
    cudaMalloc(&o, 148 * 512 * 4);
    cudaMalloc(&c, 148 * 8);
    const int iters = 4096;
    kbench<KIND><<<148, threads>>>(o, 16, c);
    kbench<KIND><<<148, threads>>>(o, iters, c);
    cudaDeviceSynchronize();
    unsigned long long h[148];
    cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < 148; ++i) avg += h[i];
    avg /= 148;
    // per warp (= per SMSP here): elems_per_iter element-results per iteration
    printf("%-34s warps/SMSP %d: %7.2f clk per 32-lane element batch (per SMSP)\n", name, threads / 128,
           avg / (iters * elems_per_iter * (threads / 128)));
    cudaFree(o);
    cudaFree(c);
}

int main() {
    run<0>("MUFU.EX2 (+FADD)", 16);
    run<1>("FFMA2 (2 results)", 16);
    run<2>("poly exp2 pair (2 results)", 16);
    run<3>("75% MUFU / 25% poly mix", 16);
    run<0>("MUFU.EX2 (+FADD)", 16, 256);
    run<2>("poly exp2 pair (2 results)", 16, 256);
    run<3>("75% MUFU / 25% poly mix", 16, 256);
    run<0>("MUFU.EX2 (+FADD)", 16, 512);
    run<3>("75% MUFU / 25% poly mix", 16, 512);
    return 0;
}
