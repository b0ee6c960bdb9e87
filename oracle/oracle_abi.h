/*
 * oracle_abi.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C interface shared by the two CPU checkers under oracle/:
 *   - liboracle.so  (prefix eorc_): our C restatement of the reference
 *     algorithm (oracle/efta_oracle.c);
 *   - _ref/libefta_ref.so (prefix eref_): a shim over the *unmodified*
 *     reference C++ sources compiled from /root/reference/proj/src
 *     (oracle/ref_shim.cpp, built by oracle/Makefile).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load either library. The product path
 * (paper_2504_02211_b200) never links or calls anything here.
 *
 * Matrices are dense row-major fp32 (the reference stores fp16-grid values
 * in fp32, include/efta/matrix.hpp:11-13).
 */
#ifndef EFTA_ORACLE_ABI_H
#define EFTA_ORACLE_ABI_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* FaultSite order == include/efta/fault.hpp:16-25 */
enum { ORC_GEMM1_OUT = 0, ORC_SUB_MAX, ORC_EXP_OUT, ORC_REDUCE_MAX, ORC_REDUCE_SUM,
       ORC_RESCALE_FACTOR, ORC_GEMM2_ACC, ORC_NORMALIZE_OUT, ORC_SITE_COUNT };
/* FTMode order == include/efta/efta.hpp:24 */
enum { ORC_MODE_NONE = 0, ORC_MODE_EFTA = 1, ORC_MODE_EFTA_OPT = 2 };
/* CheckKind order == include/efta/efta.hpp:30-38 */
enum { ORC_SCORE_CHECKSUM = 0, ORC_EXP_CHECKSUM, ORC_FACTOR_RANGE, ORC_ROWSUM_RANGE,
       ORC_OUTPUT_CHECKSUM };
/* VerifyStatus order == include/efta/abft.hpp:13 */
enum { ORC_CLEAN = 0, ORC_CORRECTED, ORC_DETECTED_UNCORRECTABLE, ORC_NONFINITE };

typedef struct {
    int site, block_i, block_j, row, col, bit, trigger;
} orc_fault_spec;

typedef struct {
    int kind, block_i, block_j, status, row, col, violations, corrections, checksum_repair;
    int pad_;
    double residual, delta;
} orc_event;

typedef struct {
    orc_fault_spec spec;
    float before, after;
} orc_fired;

typedef struct {
    int detections, corrections, recomputes, range_replacements, failed;
    int n_events;      /* total events produced (may exceed the caller's capacity) */
    int n_fired;
    int pad_;
    /* Counters (include/efta/counters.hpp:13-38), subset used by the tests */
    uint64_t flops_main, flops_checksum, flops_verify, intermediate_elems;
    uint64_t flops_main_gemm_scores, flops_cs_gemm_scores;
    uint64_t flops_main_gemm_output, flops_cs_gemm_output;
    uint64_t exp_checks, output_checks;
} orc_summary;

typedef struct {
    int status, row, col, violations, corrections, checksum_repair;
    double residual, delta;
} orc_verify_report;

#define ORC_DECLARE(P)                                                                        \
    const char* P##last_error(void);                                                          \
    uint64_t P##trial_seed(uint64_t base, uint64_t trial);                                    \
    /* Rng(seed); q,k,v = Matrix::random(n,d) in that order (src/campaign.cpp:177-180);    */ \
    /* if n_sites > 0 also sample_random_plan from the same stream (:183-185).             */ \
    int P##gen_trial(uint64_t seed, int n, int d, int block, int stride, const int* sites,    \
                     int n_sites, float* q, float* k, float* v, orc_fault_spec* spec_out);    \
    /* Matrix::random(rows, cols, Rng(seed), lo, hi, half_grid ? HALF_STORED : FULL)       */ \
    /* Rng(seed); out[i] = below(bounds[i]) in order (rng.hpp:31-38; acceptance.cpp:137-156) */ \
    void P##rng_below_seq(uint64_t seed, int n, const uint32_t* bounds, uint32_t* out);       \
    void P##random_matrix(uint64_t seed, int rows, int cols, double lo, double hi,            \
                          int half_grid, float* out);                                         \
    float P##flip_bit(float v, int width, int bit);                                           \
    uint16_t P##float_to_half_bits(float f);                                                  \
    float P##half_bits_to_float(uint16_t h);                                                  \
    int P##efta_forward(int n, int d, int block, int stride, float scale, int mode,          \
                        double eps1, double eps2, double eps_lin, int observe_linear,          \
                        float rowmax_bias, const float* q, const float* k, const float* v,     \
                        float* o, float* m_out, float* l_out, const orc_fault_spec* specs,     \
                        int n_specs, orc_event* events, int ev_cap, orc_fired* fired,          \
                        int fired_cap, orc_summary* sum);                                      \
    int P##standard_attention(int n, int d, int block, int stride, float scale,               \
                              const float* q, const float* k, const float* v, float* o);       \
    int P##encode_strided(int rows, int cols, int stride, const float* t, float* c1,          \
                          float* c2);                                                         \
    /* a: m x kd, bt: kd x w; c: m x w, c1/c2: m x stride                                  */ \
    int P##checksummed_gemm(int m, int kd, int w, int stride, const float* a, const float* bt, \
                            float* c, float* c1, float* c2);                                  \
    int P##verify_locate_correct(int rows, int cols, int stride, float* t, const float* c1,   \
                                 const float* c2, double eps, const double* row_eps_mult,      \
                                 orc_verify_report* rep);

ORC_DECLARE(eorc_)
ORC_DECLARE(eref_)

#ifdef __cplusplus
}
#endif

#endif
