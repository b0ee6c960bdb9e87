// abft_verify.cu — standalone strided-ABFT primitives on the GPU for the drop-in C++ API
// (efta_b200::encode_strided / verify_locate_correct, include/efta_b200.hpp): the reference's
// encode_strided (src/abft.cpp:19-42) and verify_locate_correct (src/abft.cpp:65-187) over an
// arbitrary rows x cols fp32 tile in device memory. The fused kernels verify inside their
// epilogues; these entry points serve callers that hold a tile and its checksums separately
// (the reference's operator API), so they favour exactness over speed: one thread per row with
// fp32 sums in the reference's order, then one thread combines the per-row outcomes in row
// order exactly like the reference's single loop.
#include <cuda_runtime.h>
#include <math_constants.h>

#include <cmath>
#include <string>

#include "../../include/efta_b200.h"
#include "efta_launch.h"

namespace {

constexpr double kNoiseBand = 16.0;  // kLocateNoiseBand (include/efta/abft.hpp:49)
constexpr int kNoStop = 0x7fffffff;

__global__ void encode_strided_kernel(int rows, int cols, int stride, const float* __restrict__ t,
                                      float* __restrict__ c1, float* __restrict__ c2) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rows) return;
    const int groups = cols / stride;
    const float* row = t + static_cast<size_t>(r) * cols;
    for (int j = 0; j < stride; ++j) {
        float s1 = 0.0f, s2 = 0.0f;
        for (int l = 0; l < groups; ++l) {
            const float v = row[j + stride * l];
            s1 = __fadd_rn(s1, v);
            s2 = __fadd_rn(s2, __fmul_rn(static_cast<float>(l + 1), v));
        }
        c1[static_cast<size_t>(r) * stride + j] = s1;
        c2[static_cast<size_t>(r) * stride + j] = s2;
    }
}

// per-row outcome, combined in row order by verify_combine_kernel
struct RowOut {
    double residual, best_abs, best_delta;
    int violations, corrections, checksum_repair, uncorrectable;
    int best_col, restored_col, pad0, pad1;
};

struct VerifyHead {  // workspace header
    int cs_nonfinite;
    int stop;  // flat (row * stride + group) of the first group with > 1 non-finite cell
};

__global__ void verify_init_kernel(VerifyHead* head) {
    if (threadIdx.x == 0) *head = VerifyHead{0, kNoStop};
}

__global__ void verify_scan_kernel(int rows, int cols, int stride, const float* __restrict__ t,
                                   const float* __restrict__ c1, const float* __restrict__ c2, VerifyHead* head) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rows) return;
    const int groups = cols / stride;
    for (int j = 0; j < stride; ++j)
        if (!isfinite(c1[static_cast<size_t>(r) * stride + j]) || !isfinite(c2[static_cast<size_t>(r) * stride + j]))
            atomicOr(&head->cs_nonfinite, 1);
    const float* row = t + static_cast<size_t>(r) * cols;
    for (int j = 0; j < stride; ++j) {
        int cnt = 0;
        for (int l = 0; l < groups; ++l) cnt += !isfinite(row[j + stride * l]);
        if (cnt > 1) {
            atomicMin(&head->stop, r * stride + j);
            return;
        }
    }
}

__global__ void verify_rows_kernel(int rows, int cols, int stride, float* __restrict__ t, const float* __restrict__ c1,
                                   const float* __restrict__ c2, double eps, const double* __restrict__ row_mult,
                                   const VerifyHead* head, RowOut* outs) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rows || head->cs_nonfinite) return;
    const int groups = cols / stride;
    float* row = t + static_cast<size_t>(r) * cols;
    const float* rc1 = c1 + static_cast<size_t>(r) * stride;
    const float* rc2 = c2 + static_cast<size_t>(r) * stride;
    RowOut o{};
    o.best_col = -1;
    o.restored_col = -1;
    // (abft.cpp:83-111) erasure restore up to the reference's early return
    const int stop = head->stop;
    for (int j = 0; j < stride && r * stride + j <= stop; ++j) {
        int bad = -1, cnt = 0;
        for (int l = 0; l < groups; ++l)
            if (!isfinite(row[j + stride * l])) { bad = l; ++cnt; }
        if (cnt == 0) continue;
        ++o.violations;
        if (cnt > 1) break;  // the early-return group: counted, not restored
        float rest = 0.0f;
        for (int l = 0; l < groups; ++l)
            if (l != bad) rest = __fadd_rn(rest, row[j + stride * l]);
        const int col = j + stride * bad;
        row[col] = __fsub_rn(rc1[j], rest);
        ++o.corrections;
        o.restored_col = col;
    }
    if (stop == kNoStop) {
        // (abft.cpp:113-180) fresh strided sums, locate, correct
        const double eps_row = row_mult ? eps * row_mult[r] : eps;
        for (int j = 0; j < stride; ++j) {
            float a = 0.0f, b = 0.0f;
            for (int l = 0; l < groups; ++l) {
                const float v = row[j + stride * l];
                a = __fadd_rn(a, v);
                b = __fadd_rn(b, __fmul_rn(static_cast<float>(l + 1), v));
            }
            double s1d = a, s2d = b;
            if (!isfinite(s1d) || !isfinite(s2d)) {
                s1d = 0.0;
                s2d = 0.0;
                for (int l = 0; l < groups; ++l) {
                    const double vv = row[j + stride * l];
                    s1d += vv;
                    s2d += (l + 1.0) * vv;
                }
            }
            const double d1 = static_cast<double>(rc1[j]) - s1d;
            const double d2 = static_cast<double>(rc2[j]) - s2d;
            o.residual = fmax(o.residual, fmax(fabs(d1), fabs(d2) / groups));
            const bool v1 = fabs(d1) > eps_row;
            const bool v2 = fabs(d2) > eps_row * groups;
            if (!v1 && !v2) continue;
            ++o.violations;
            if (!v1) { o.checksum_repair = 1; continue; }
            const double ratio = d2 / d1;
            const double nearest = round(ratio);
            if (nearest == 0.0 && fabs(ratio) <= 0.25) { o.checksum_repair = 1; continue; }
            const int g = static_cast<int>(nearest) - 1;
            if (g < 0 || g >= groups || fabs(ratio - nearest) > 0.25) {
                if (fmax(fabs(d1), fabs(d2) / groups) > eps_row * kNoiseBand) o.uncorrectable = 1;
                continue;
            }
            const int col = j + stride * g;
            float rest = 0.0f;
            for (int l = 0; l < groups; ++l)
                if (l != g) rest = __fadd_rn(rest, row[j + stride * l]);
            const float old_val = row[col];
            const float new_val = __fsub_rn(rc1[j], rest);
            row[col] = new_val;
            ++o.corrections;
            const double applied = static_cast<double>(new_val) - static_cast<double>(old_val);
            if (fabs(applied) > o.best_abs) {
                o.best_abs = fabs(applied);
                o.best_delta = applied;
                o.best_col = col;
            }
        }
    }
    outs[r] = o;
}

// the reference's single loop over rows, replayed in order over the per-row outcomes
__global__ void verify_combine_kernel(int rows, const VerifyHead* head, const RowOut* outs, efta_verify_report* out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    efta_verify_report rep{EFTA_CLEAN, -1, -1, 0, 0, 0, 0.0, 0.0};
    if (head->cs_nonfinite) {
        rep.status = EFTA_NONFINITE;
        rep.residual = CUDART_INF;
        *out = rep;
        return;
    }
    double best = 0.0;  // |rep.delta| (abft.cpp:172)
    bool uncorrectable = false;
    for (int r = 0; r < rows; ++r) {
        const RowOut& o = outs[r];
        rep.violations += o.violations;
        rep.corrections += o.corrections;
        if (o.restored_col >= 0) {
            rep.row = r;
            rep.col = o.restored_col;
            rep.delta = CUDART_INF;
            best = CUDART_INF;
        }
    }
    if (head->stop != kNoStop) {
        rep.status = EFTA_NONFINITE;
        rep.residual = CUDART_INF;
        *out = rep;
        return;
    }
    for (int r = 0; r < rows; ++r) {
        const RowOut& o = outs[r];
        rep.residual = fmax(rep.residual, o.residual);
        rep.checksum_repair |= o.checksum_repair;
        uncorrectable |= o.uncorrectable != 0;
        if (o.best_col >= 0 && o.best_abs > best) {
            best = o.best_abs;
            rep.delta = o.best_delta;
            rep.row = r;
            rep.col = o.best_col;
        }
    }
    if (uncorrectable) rep.status = EFTA_DETECTED_UNCORRECTABLE;
    else if (rep.corrections > 0 || rep.checksum_repair) rep.status = EFTA_CORRECTED;
    *out = rep;
}

int vfail(int code, const std::string& m) {
    efta_internal_set_error(m.c_str());
    return code;
}

}  // namespace

extern "C" {

int efta_encode_strided_f32(int rows, int cols, int stride, const float* t, float* c1, float* c2, void* stream) {
    if (rows <= 0 || cols <= 0 || stride <= 0 || cols % stride)
        return vfail(1, "encode_strided: stride must divide tile width");
    if (!t || !c1 || !c2) return vfail(1, "encode_strided: null buffer");
    encode_strided_kernel<<<(rows + 127) / 128, 128, 0, static_cast<cudaStream_t>(stream)>>>(rows, cols, stride, t,
                                                                                             c1, c2);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? 0 : vfail(2, cudaGetErrorString(e));
}

size_t efta_verify_workspace_bytes(int rows) {
    return rows > 0 ? 256 + static_cast<size_t>(rows) * sizeof(RowOut) : 0;
}

int efta_verify_locate_correct_f32(int rows, int cols, int stride, float* t, const float* c1, const float* c2,
                                   double eps, const double* row_eps_mult, efta_verify_report* report,
                                   void* workspace, size_t workspace_bytes, void* stream) {
    if (rows <= 0 || cols <= 0 || stride <= 0 || cols % stride)
        return vfail(1, "verify_locate_correct: checksum/tile shape mismatch");
    if (!t || !c1 || !c2 || !report) return vfail(1, "verify_locate_correct: null buffer");
    if (!workspace || workspace_bytes < efta_verify_workspace_bytes(rows))
        return vfail(1, "verify_locate_correct: workspace too small");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    VerifyHead* head = static_cast<VerifyHead*>(workspace);
    RowOut* outs = reinterpret_cast<RowOut*>(static_cast<char*>(workspace) + 256);
    const int blocks = (rows + 127) / 128;
    verify_init_kernel<<<1, 32, 0, st>>>(head);
    verify_scan_kernel<<<blocks, 128, 0, st>>>(rows, cols, stride, t, c1, c2, head);
    verify_rows_kernel<<<blocks, 128, 0, st>>>(rows, cols, stride, t, c1, c2, eps, row_eps_mult, head, outs);
    verify_combine_kernel<<<1, 32, 0, st>>>(rows, head, outs, report);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? 0 : vfail(2, cudaGetErrorString(e));
}

}  // extern "C"
