// efta_b200.hpp — C++ drop-in for the reference's operator API on the EFTA path.
//
// A reference caller switches `#include "efta/efta.hpp"` + `efta::` to this
// header + `efta_b200::` and links libefta_b200.so: same value types, same
// signatures, same error behaviour (ConfigError on bad shapes / plans; faults
// never throw, they surface in FTReport), computed on the GPU through the
// C-ABI in efta_b200.h. Reference interfaces mirrored (paths relative to
// /root/reference/proj):
//   AttnConfig / ConfigError        include/efta/config.hpp:9-50
//   Thresholds                      include/efta/snvr.hpp:17-30
//   FTMode / CheckKind / FTReport   include/efta/efta.hpp:24-72
//   KernelKnobs                     include/efta/efta.hpp:75-83
//   efta_forward                    include/efta/efta.hpp:86-89
//   FaultSite / FaultSpec / FaultPlan / FaultInjector / sample_random_plan
//                                   include/efta/fault.hpp:16-103
//   Rng / trial_seed                include/efta/rng.hpp:19-58
//   classify_trial / Outcome        include/efta/campaign.hpp:12-20, 84-85
//   calibrate_thresholds / CalibrationResult / threshold_sweep / SweepPoint
//                                   include/efta/campaign.hpp:87-111
//   ChecksumPair / encode_strided / verify_locate_correct / checksummed_gemm / GemmStage
//                                   include/efta/abft.hpp:31-77, include/efta/gemm.hpp:10
#pragma once

#include <cstdint>
#include <optional>
#include <random>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "efta_b200.h"

namespace efta_b200 {

struct ConfigError : std::runtime_error {
    explicit ConfigError(const std::string& w) : std::runtime_error(w) {}
};

struct AttnConfig {
    int seq_len = 128, head_dim = 64, block = 128, stride = 8, heads = 1;
    float scale = 0.0f;
    AttnConfig() = default;
    AttnConfig(int n, int d, int b = 128, int s = 8, int h = 1, float sc = 0.0f)
        : seq_len(n), head_dim(d), block(b), stride(s), heads(h), scale(sc) {
        validate();
    }
    void validate();  // reference checks + this kernel's geometry (block 128, stride 8, d 64|128)
    int num_blocks() const { return seq_len / block; }
    int groups(int width) const { return width / stride; }
};

struct Thresholds {
    double eps1 = 7e-6, eps2 = 0.48, eps_lin = 0.48;
    static Thresholds reference_defaults() { return Thresholds{}; }
    static Thresholds observe();
};

enum class FTMode { NONE, EFTA, EFTA_OPTIMIZED, DECOUPLED };
enum class CheckKind { SCORE_CHECKSUM, EXP_CHECKSUM, FACTOR_RANGE, ROWSUM_RANGE, OUTPUT_CHECKSUM };
enum class VerifyStatus { CLEAN, CORRECTED, DETECTED_UNCORRECTABLE, NONFINITE };
enum class FaultSite { GEMM1_OUT, SUB_MAX, EXP_OUT, REDUCE_MAX, REDUCE_SUM, RESCALE_FACTOR,
                       GEMM2_ACC, NORMALIZE_OUT };
inline constexpr int FAULT_SITE_COUNT = 8;

const char* ft_mode_name(FTMode m);
std::optional<FTMode> ft_mode_from_name(const std::string& name);
const char* fault_site_name(FaultSite s);
std::optional<FaultSite> fault_site_from_name(const std::string& name);
float flip_bit(float v, int width, int bit);

// Host matrix: fp32 storage, inputs are expected on the fp16 grid (they are
// converted to fp16 for the tensor cores; off-grid values are rounded RNE).
class Matrix {
public:
    Matrix() = default;
    Matrix(int r, int c) : rows_(r), cols_(c), data_(static_cast<size_t>(r) * c, 0.0f) {}
    int rows() const { return rows_; }
    int cols() const { return cols_; }
    float operator()(int r, int c) const { return data_[static_cast<size_t>(r) * cols_ + c]; }
    float& at(int r, int c) { return data_[static_cast<size_t>(r) * cols_ + c]; }
    const float* data() const { return data_.data(); }
    float* data() { return data_.data(); }
    bool same_shape(const Matrix& o) const { return rows_ == o.rows_ && cols_ == o.cols_; }

private:
    int rows_ = 0, cols_ = 0;
    std::vector<float> data_;
};

// Reference Rng (mt19937_64 + implementation-independent mappings).
class Rng {
public:
    explicit Rng(uint64_t seed) : eng_(seed) {}
    uint64_t next_u64() { return eng_(); }
    double uniform() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
    double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
    uint32_t below(uint32_t n);

private:
    std::mt19937_64 eng_;
};
uint64_t trial_seed(uint64_t base_seed, uint64_t trial);
Matrix random_half_matrix(int rows, int cols, Rng& rng, double lo = -1.0, double hi = 1.0);

struct FaultSpec {
    FaultSite site = FaultSite::GEMM1_OUT;
    int block_i = 0, block_j = 0, row = 0, col = 0, bit = 0, trigger = 1;
    std::string to_string() const;
    static FaultSpec parse(const std::string& text);
};

struct FaultPlan {
    std::vector<FaultSpec> specs;
    bool empty() const { return specs.empty(); }
    void validate(const AttnConfig& cfg) const;
};

FaultPlan sample_random_plan(const AttnConfig& cfg, const std::vector<FaultSite>& sites, Rng& rng);

struct FiredFault {
    FaultSpec spec;
    float before = 0.0f, after = 0.0f;
};

// Device-side injector: the plan is uploaded with the forward call; fired()
// is filled from the kernel's log when the call returns.
class FaultInjector {
public:
    explicit FaultInjector(const FaultPlan& plan) : plan_(plan) {}
    const FaultPlan& plan() const { return plan_; }
    const std::vector<FiredFault>& fired() const { return fired_; }
    std::vector<FiredFault>& fired_mut() { return fired_; }

private:
    FaultPlan plan_;
    std::vector<FiredFault> fired_;
};

// Analytic operation counters of the CPU reference (include/efta/counters.hpp:13-38). The GPU
// path reports measured time and ncu profiles instead: accepted for signature compatibility,
// never written.
struct Counters {};
enum class GemmStage { PLAIN, SCORES, OUTPUT };

// Row-direction strided checksums of a tile (include/efta/abft.hpp:31-36)
struct ChecksumPair {
    Matrix c1, c2;
    int stride = 0;
    int groups = 0;
};

struct VerificationReport {
    VerifyStatus status = VerifyStatus::CLEAN;
    int row = -1, col = -1;
    double delta = 0.0, residual = 0.0;
    int violations = 0, corrections = 0;
    bool checksum_repair = false;
    bool detected() const { return status != VerifyStatus::CLEAN; }
};

struct StageEvent {
    CheckKind kind{};
    int block_i = 0, block_j = 0;
    VerificationReport rep;
};

struct FTReport {
    FTMode mode = FTMode::NONE;
    std::vector<StageEvent> events;  // non-CLEAN events (the device logs only those)
    int detections = 0, corrections = 0, recomputes = 0, range_replacements = 0;
    bool failed = false;
    std::vector<float> final_l, final_m;
    double family_max[3] = {0, 0, 0};  // worst clean residual per family: exp, out, lin
    double max_residual(CheckKind kind) const;
};

struct KernelKnobs {
    bool observe_linear = false;
    float rowmax_bias = 0.0f;
};

// inj != nullptr (also with an empty plan, e.g. for a fault-free twin) runs the fault-tap build
// of the kernel (the reference op sequence with eager rescaling); without one, the production
// build (identical decisions, lazily rescaled accumulator: outputs agree to rounding).
std::pair<Matrix, FTReport> efta_forward(const Matrix& q, const Matrix& k, const Matrix& v,
                                         const AttnConfig& cfg, const Thresholds& thr, FTMode mode,
                                         FaultInjector* inj = nullptr,
                                         const KernelKnobs* knobs = nullptr);

// decoupled_ft_forward (include/efta/efta.hpp:94-96): the three-kernel baseline (traditional
// two-sided block ABFT around the two GEMMs, DMR softmax, N^2 intermediates in HBM) on the GPU
// (csrc/decoupled.cu); the same as efta_forward(..., FTMode::DECOUPLED, ...).
std::pair<Matrix, FTReport> decoupled_ft_forward(const Matrix& q, const Matrix& k, const Matrix& v,
                                                 const AttnConfig& cfg, const Thresholds& thr,
                                                 FaultInjector* inj = nullptr,
                                                 const KernelKnobs* knobs = nullptr);

// ---- strided ABFT primitives (include/efta/abft.hpp:38-77), computed on the GPU ----
// encode_strided: c1/c2 (rows x stride) of t, fp32 sums in the reference's order (bit-exact).
ChecksumPair encode_strided(const Matrix& t, int stride, Counters* cnt = nullptr);
// verify_locate_correct: the reference's detection / location / repair ladder on t (repaired
// in place) with the reference's report; std::invalid_argument on shape mismatch.
VerificationReport verify_locate_correct(Matrix& t, const ChecksumPair& cp, double eps_abs,
                                         Counters* cnt = nullptr,
                                         const std::vector<double>* row_eps_mult = nullptr);
// checksummed_gemm: a (M x K) times bt (K x W) on the tcgen05 strided-ABFT GEMM (fp16 operands,
// inputs on the fp16 grid; fp32 accumulation and product) with the product's strided checksum
// pair over the full width W carried by the tensor cores (per 256-wide tile, recombined).
// c_init / cp_init (O += P.V) are added on the device. This kernel's geometry:
// stride 8, M % 128 == 0, W % 256 == 0, K % 64 == 0 (std::invalid_argument otherwise).
std::pair<Matrix, ChecksumPair> checksummed_gemm(const Matrix& a, const Matrix& bt, int stride,
                                                 Counters* cnt = nullptr,
                                                 GemmStage stage = GemmStage::SCORES,
                                                 const Matrix* c_init = nullptr,
                                                 const ChecksumPair* cp_init = nullptr);

enum class Outcome { CLEAN, FALSE_ALARM, CORRECTED, RANGE_RESTRICTED, MASKED_BENIGN,
                     RANGE_CONTRACT, UNCORRECTABLE };
const char* outcome_name(Outcome o);
Outcome classify_trial(const Matrix& out, const Matrix& ref, const FTReport& rep,
                       const FaultPlan& plan, const Thresholds& thr);

// calibrate_thresholds (src/campaign.cpp:261-297): clean runs in observation mode on the GPU
// (one batched launch over the trials), each threshold = worst clean residual x safety.
struct CalibrationResult {
    Thresholds thr;
    double max_exp = 0.0, max_out = 0.0, max_lin = 0.0;
    bool degenerate = false;
};
CalibrationResult calibrate_thresholds(const AttnConfig& cfg, FTMode mode, int trials, double safety,
                                       uint64_t seed);

// threshold_sweep (src/campaign.cpp:299-357): per trial one clean and one randomly faulted
// observation run; detection / false-alarm rates re-judged at log-spaced multiples of `base`.
struct SweepPoint {
    double multiplier = 0.0, detection_rate = 0.0, false_alarm_rate = 0.0;
};
std::vector<SweepPoint> threshold_sweep(const AttnConfig& cfg, FTMode mode, const Thresholds& base,
                                        int trials, uint64_t seed, int points = 10);

}  // namespace efta_b200
