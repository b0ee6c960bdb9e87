/* efta_types.h — plain-C structs shared by the CUDA kernels, the C-ABI
 * (include/efta_b200.h) and the C++ host layer. No CUDA or torch types. */
#ifndef EFTA_B200_TYPES_H
#define EFTA_B200_TYPES_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* FaultSite order == reference include/efta/fault.hpp:16-25 */
enum efta_site {
    EFTA_GEMM1_OUT = 0, EFTA_SUB_MAX, EFTA_EXP_OUT, EFTA_REDUCE_MAX, EFTA_REDUCE_SUM,
    EFTA_RESCALE_FACTOR, EFTA_GEMM2_ACC, EFTA_NORMALIZE_OUT, EFTA_SITE_COUNT
};
/* FTMode order == reference include/efta/efta.hpp:24 (DECOUPLED: the three-kernel baseline,
 * src/decoupled.cpp:98-282, csrc/decoupled.cu) */
enum efta_mode { EFTA_MODE_NONE = 0, EFTA_MODE_EFTA = 1, EFTA_MODE_EFTA_OPT = 2, EFTA_MODE_DECOUPLED = 3 };
/* CheckKind order == reference include/efta/efta.hpp:30-38 */
enum efta_check {
    EFTA_SCORE_CHECKSUM = 0, EFTA_EXP_CHECKSUM, EFTA_FACTOR_RANGE, EFTA_ROWSUM_RANGE,
    EFTA_OUTPUT_CHECKSUM, EFTA_DMR_SOFTMAX, EFTA_BLOCK_CHECKSUM
};
/* VerifyStatus order == reference include/efta/abft.hpp:13 */
enum efta_status { EFTA_CLEAN = 0, EFTA_CORRECTED, EFTA_DETECTED_UNCORRECTABLE, EFTA_NONFINITE };

/* One single-bit upset (reference FaultSpec, fault.hpp:36-47) plus the flat
 * (batch*heads) index it targets — the reference is single-head per call. */
typedef struct {
    int head;    /* flat b*H + h */
    int site;    /* efta_site */
    int block_i, block_j, row, col, bit, trigger;
} efta_fault_spec;

/* A non-CLEAN check outcome (reference StageEvent + VerificationReport,
 * efta.hpp:42-47, abft.hpp:15-26). block_j == n marks the post-loop check. */
typedef struct {
    int kind, head, block_i, block_j, status, row, col, violations, corrections,
        checksum_repair;
    double residual, delta;
} efta_event;

typedef struct {
    efta_fault_spec spec;
    float before, after;
} efta_fired;

/* Device-side counters the kernel accumulates (all atomics, one block per call). */
typedef struct {
    int n_events;      /* events appended (may exceed capacity) */
    int n_fired;
    int detections;    /* non-CLEAN events */
    int corrections;   /* sum of VerificationReport.corrections */
    int recomputes;    /* rows whose recomputation changed bits (incl. factor guard) */
    int range_replacements;
    int failed;        /* some check ended DETECTED_UNCORRECTABLE / NONFINITE */
    int pad_;
    float family_max[3]; /* worst clean residual per family: exp, out, lin */
    float pad2_;
} efta_counters;

#ifdef __cplusplus
}
#endif
#endif
