// acceptance_gpu.cpp — a C++ consumer of the drop-in header (include/efta_b200.hpp): the
// reference's acceptance checks (tests/acceptance.cpp:65-405) re-pointed from `efta::` at
// `efta_b200::`, i.e. at the GPU through libefta_b200.so, at the GPU tile geometry (block 128,
// stride 8). The CPU checker (oracle/liboracle.so, the bit-exact C restatement of the reference)
// provides the two-pass attention and the ABFT primitives the GPU results are compared with.
// Test infrastructure: built and run by tests/test_cpp_dropin.py. Prints one PASS/FAIL line per
// check and exits non-zero if any check fails.
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <functional>
#include <string>
#include <vector>

#include "efta_b200.hpp"

extern "C" {
#include "../../oracle/oracle_abi.h"
}

using namespace efta_b200;

namespace {

struct Verdict {
    bool pass = false;
    std::string detail;
};

std::string fmt(const char* f, ...) {
    char buf[768];
    va_list ap;
    va_start(ap, f);
    vsnprintf(buf, sizeof buf, f, ap);
    va_end(ap);
    return buf;
}

struct Inputs {
    Matrix q, k, v;
    Inputs(const AttnConfig& cfg, uint64_t seed) {
        Rng rng(seed);
        q = random_half_matrix(cfg.seq_len, cfg.head_dim, rng);
        k = random_half_matrix(cfg.seq_len, cfg.head_dim, rng);
        v = random_half_matrix(cfg.seq_len, cfg.head_dim, rng);
    }
};

double max_abs_diff(const Matrix& a, const Matrix& b) {
    double m = 0.0;
    for (int r = 0; r < a.rows(); ++r)
        for (int c = 0; c < a.cols(); ++c) {
            const double x = std::fabs(double(a(r, c)) - double(b(r, c)));
            m = std::isnan(x) ? INFINITY : std::max(m, x);
        }
    return m;
}
double max_abs(const Matrix& a) {
    double m = 0.0;
    for (int r = 0; r < a.rows(); ++r)
        for (int c = 0; c < a.cols(); ++c) m = std::max(m, double(std::fabs(a(r, c))));
    return m;
}
bool bit_equal(const Matrix& a, const Matrix& b) {
    if (!a.same_shape(b)) return false;
    for (int r = 0; r < a.rows(); ++r)
        for (int c = 0; c < a.cols(); ++c) {
            float x = a(r, c), y = b(r, c);
            uint32_t ux, uy;
            std::memcpy(&ux, &x, 4);
            std::memcpy(&uy, &y, 4);
            if (ux != uy) return false;
        }
    return true;
}

// 1. The fused GPU forward vs the two-pass reference kernel (acceptance.cpp:65-84).
Verdict blocked_matches_reference() {
    const double bound = 1e-3;
    double worst = 0.0;
    int runs = 0;
    for (int n : {256, 512})
        for (int d : {64, 128}) {
            AttnConfig cfg(n, d, 128, 8);
            for (uint64_t s = 0; s < 10; ++s) {
                Inputs in(cfg, trial_seed(1000 + n + d + 128, s));
                auto res = efta_forward(in.q, in.k, in.v, cfg, Thresholds::reference_defaults(), FTMode::NONE);
                Matrix os(n, d);
                if (eorc_standard_attention(n, d, 128, 8, cfg.scale, in.q.data(), in.k.data(), in.v.data(),
                                            os.data()))
                    return {false, "checker failed"};
                worst = std::max(worst, max_abs_diff(res.first, os));
                ++runs;
                if (worst > bound)
                    return {false, fmt("N=%d d=%d seed=%llu: |diff|=%.3e > %.0e", n, d, (unsigned long long)s,
                                       worst, bound)};
            }
        }
    return {true, fmt("4 shapes x 10 seeds (%d runs), max |diff| %.3e <= %.0e", runs, worst, bound)};
}

// 2. The protection side band leaves the main path bit-identical (acceptance.cpp:87-100):
//    EFTA-optimized == plain on the production kernel. Mode EFTA (per-iteration output check)
//    runs the single-CTA kernel with the reference's eager rescale: within 2e-3 relative.
Verdict protected_modes_bit_identical() {
    double worst_efta = 0.0;
    for (int d : {64, 128}) {
        AttnConfig cfg(512, d, 128, 8);
        const Thresholds thr{1e-4, 1e-3, 1e-3};
        for (uint64_t s = 0; s < 20; ++s) {
            Inputs in(cfg, trial_seed(2000, s));
            auto r0 = efta_forward(in.q, in.k, in.v, cfg, thr, FTMode::NONE);
            auto r2 = efta_forward(in.q, in.k, in.v, cfg, thr, FTMode::EFTA_OPTIMIZED);
            auto r1 = efta_forward(in.q, in.k, in.v, cfg, thr, FTMode::EFTA);
            if (!bit_equal(r0.first, r2.first))
                return {false, fmt("d=%d seed %llu: EFTA-optimized output differs bitwise", d, (unsigned long long)s)};
            worst_efta = std::max(worst_efta, max_abs_diff(r1.first, r0.first) / max_abs(r0.first));
            if (r1.second.detections || r2.second.detections)
                return {false, fmt("d=%d seed %llu: false alarm", d, (unsigned long long)s)};
        }
    }
    return {worst_efta <= 2e-3,
            fmt("2 head dims x 20 seeds: EFTA-optimized bit-identical to plain; EFTA within %.2e rel", worst_efta)};
}

// 4. Exhaustive single-fault sweep (acceptance.cpp:125-211): every site x {sign, top-2
//    exponent, top-2 mantissa} x 20 reference-drawn coordinates, all absorbed, corrected faults
//    within eps2 of the fault-free output.
Verdict single_fault_sweep(int d) {
    AttnConfig cfg(512, d, 128, 8);
    const FTMode mode = FTMode::EFTA_OPTIMIZED;
    CalibrationResult cal = calibrate_thresholds(cfg, mode, 100, 2.0, 0xca11b004ull);
    if (cal.degenerate) return {false, "calibration degenerate"};
    const int bits[] = {31, 30, 29, 22, 21};
    int total = 0, corrected = 0, masked = 0, ranged = 0, uncorrectable = 0, fired = 0;
    double worst = 0.0;
    std::string first_fail;
    for (int s = 0; s < FAULT_SITE_COUNT; ++s) {
        const FaultSite site = FaultSite(s);
        for (int bit : bits) {
            Rng rng(trial_seed(0xace4ull, uint64_t(s * 64 + bit)));
            for (int c = 0; c < 20; ++c) {
                FaultSpec f;
                f.site = site;
                f.bit = bit;
                f.block_i = int(rng.below(uint32_t(cfg.num_blocks())));
                f.block_j = site == FaultSite::NORMALIZE_OUT ? 0 : int(rng.below(uint32_t(cfg.num_blocks())));
                f.row = int(rng.below(uint32_t(cfg.block)));
                const bool per_row = site == FaultSite::REDUCE_MAX || site == FaultSite::REDUCE_SUM;
                const int bound = per_row ? 1
                                          : (site == FaultSite::GEMM1_OUT || site == FaultSite::SUB_MAX ||
                                                     site == FaultSite::EXP_OUT
                                                 ? cfg.block
                                                 : cfg.head_dim);
                f.col = int(rng.below(uint32_t(bound)));
                FaultPlan plan;
                plan.specs = {f};
                // run_campaign(seed = trial_seed(0xbeef00 + s, bit*100 + c), 1 trial, 1 head)
                Inputs in(cfg, trial_seed(trial_seed(0xbeef00ull + s, uint64_t(bit * 100 + c)), 0));
                FaultInjector twin{FaultPlan{}};  // the fault-free twin runs the same (tap) build
                auto ref = efta_forward(in.q, in.k, in.v, cfg, cal.thr, mode, &twin);
                FaultInjector inj(plan);
                auto out = efta_forward(in.q, in.k, in.v, cfg, cal.thr, mode, &inj);
                fired += !inj.fired().empty();
                ++total;
                const Outcome o = classify_trial(out.first, ref.first, out.second, plan, cal.thr);
                const double res = max_abs_diff(out.first, ref.first);
                switch (o) {
                    case Outcome::CORRECTED:
                        ++corrected;
                        worst = std::max(worst, res);
                        if (res > cal.thr.eps2 && first_fail.empty())
                            first_fail = fmt("%s residual %.2e > eps2 %.2e", f.to_string().c_str(), res, cal.thr.eps2);
                        break;
                    case Outcome::MASKED_BENIGN: ++masked; break;
                    case Outcome::RANGE_RESTRICTED:
                    case Outcome::RANGE_CONTRACT: ++ranged; break;
                    case Outcome::CLEAN: break;
                    default:
                        ++uncorrectable;
                        if (first_fail.empty()) first_fail = f.to_string() + " " + outcome_name(o);
                }
            }
        }
    }
    const bool ok = uncorrectable == 0 && first_fail.empty() && fired == total;
    return {ok, fmt("d=%d: %d faults (%d fired): %d corrected, %d masked benign, %d range-handled, %d "
                    "uncorrectable; worst corrected residual %.2e (eps2 %.2e)%s%s",
                    d, total, fired, corrected, masked, ranged, uncorrectable, worst, cal.thr.eps2,
                    first_fail.empty() ? "" : "; first failure: ", first_fail.c_str())};
}

// 7. Denominator range (acceptance.cpp:290-348): never violated fault-free; out-of-range
//    denominator faults are always caught and the replacement preserves the per-row ranking.
Verdict rowsum_range_contract() {
    AttnConfig cfg(512, 64, 128, 8);
    const Thresholds thr{1e-4, 1e-3, 1e-3};
    for (uint64_t s = 0; s < 200; ++s) {
        Inputs in(cfg, trial_seed(7000, s));
        auto r = efta_forward(in.q, in.k, in.v, cfg, thr, FTMode::EFTA_OPTIMIZED);
        if (r.second.range_replacements != 0)
            return {false, fmt("clean trial %llu: %d denominator(s) flagged", (unsigned long long)s,
                               r.second.range_replacements)};
        for (float l : r.second.final_l)
            if (!(std::isfinite(l) && l > 0.0f && l <= float(cfg.seq_len)))
                return {false, fmt("clean trial %llu: denominator %g escaped its range", (unsigned long long)s, l)};
    }
    int replaced = 0, argmax_ok = 0, survived = 0;
    for (uint64_t s = 0; s < 200; ++s) {
        Inputs in(cfg, trial_seed(7100, s));
        Rng rr(trial_seed(7200, s));
        FaultSpec f;
        f.site = FaultSite::REDUCE_SUM;
        f.bit = (s % 2 == 0) ? 30 : 31;
        f.block_i = int(rr.below(uint32_t(cfg.num_blocks())));
        f.block_j = int(rr.below(uint32_t(cfg.num_blocks())));
        f.row = int(rr.below(uint32_t(cfg.block)));
        f.col = 0;
        FaultPlan plan;
        plan.specs = {f};
        FaultInjector inj(plan);
        FaultInjector twin{FaultPlan{}};
        auto ref = efta_forward(in.q, in.k, in.v, cfg, thr, FTMode::EFTA_OPTIMIZED, &twin);
        auto out = efta_forward(in.q, in.k, in.v, cfg, thr, FTMode::EFTA_OPTIMIZED, &inj);
        for (float l : out.second.final_l)
            if (!(std::isfinite(l) && l > 0.0f && l <= float(cfg.seq_len))) ++survived;
        if (out.second.range_replacements > 0) {
            ++replaced;
            bool ok = true;
            for (int r = 0; r < cfg.seq_len && ok; ++r) {
                int ar = 0, ao = 0;
                for (int c = 0; c < cfg.head_dim; ++c) {
                    if (ref.first(r, c) > ref.first(r, ar)) ar = c;
                    if (out.first(r, c) > out.first(r, ao)) ao = c;
                }
                ok = ar == ao;
            }
            argmax_ok += ok;
        }
    }
    const bool ok = survived == 0 && replaced > 50 && double(argmax_ok) >= 0.99 * double(replaced);
    return {ok, fmt("200 clean trials in range; %d faulted runs replaced the denominator, %d out-of-range values "
                    "survived, ranking preserved in %d/%d (>= 99%%)",
                    replaced, survived, argmax_ok, replaced)};
}

// The ABFT operator API (include/efta/abft.hpp:38-77) against the checker: encode_strided is
// bit-exact, checksummed_gemm's product and full-width checksum pair match, and
// verify_locate_correct reports and repairs single upsets exactly like the reference.
Verdict abft_operator_api() {
    const int m = 256, kd = 128, w = 512, s = 8;
    Rng rng(0xab57ull);
    Matrix a = random_half_matrix(m, kd, rng), bt = random_half_matrix(kd, w, rng);
    // encode_strided
    ChecksumPair e = encode_strided(a, s);
    std::vector<float> o1(m * s), o2(m * s);
    eorc_encode_strided(m, kd, s, a.data(), o1.data(), o2.data());
    for (int i = 0; i < m * s; ++i)
        if (e.c1.data()[i] != o1[i] || e.c2.data()[i] != o2[i]) return {false, "encode_strided not bit-exact"};
    // checksummed_gemm
    auto [c, cp] = checksummed_gemm(a, bt, s);
    Matrix cr(m, w), c1r(m, s), c2r(m, s);
    eorc_checksummed_gemm(m, kd, w, s, a.data(), bt.data(), cr.data(), c1r.data(), c2r.data());
    const double dprod = max_abs_diff(c, cr) / max_abs(cr);
    const double dcs = std::max(max_abs_diff(cp.c1, c1r) / max_abs(c1r), max_abs_diff(cp.c2, c2r) / max_abs(c2r));
    if (dprod > 1e-5 || dcs > 1e-5) return {false, fmt("checksummed_gemm: product %.2e, checksums %.2e", dprod, dcs)};
    // clean verify: no violation at a threshold above the accumulation noise
    double eps = 0.0;
    {
        Matrix t = c;
        VerificationReport r = verify_locate_correct(t, cp, INFINITY);
        eps = 4.0 * r.residual;
        if (r.status != VerifyStatus::CLEAN) return {false, "clean product flagged at eps = inf"};
    }
    // single upsets: identical reports and repairs on both sides
    int same = 0, trials = 0;
    for (int t = 0; t < 64; ++t) {
        Matrix g = c;
        Matrix h = c;
        const int r = int(rng.below(m)), col = int(rng.below(w)), bit = 20 + int(rng.below(12));
        g.at(r, col) = flip_bit(g(r, col), 32, bit);
        h.at(r, col) = g(r, col);
        VerificationReport rg = verify_locate_correct(g, cp, eps);
        orc_verify_report ro{};
        eorc_verify_locate_correct(m, w, s, h.data(), cp.c1.data(), cp.c2.data(), eps, nullptr, &ro);
        ++trials;
        if (int(rg.status) == ro.status && rg.row == ro.row && rg.col == ro.col && rg.corrections == ro.corrections &&
            rg.violations == ro.violations && bit_equal(g, h))
            ++same;
        else
            return {false, fmt("upset (%d,%d) bit %d: gpu status %d (%d,%d) corr %d vs ref %d (%d,%d) corr %d", r, col,
                               bit, int(rg.status), rg.row, rg.col, rg.corrections, ro.status, ro.row, ro.col,
                               ro.corrections)};
    }
    return {true, fmt("encode_strided bit-exact; checksummed_gemm product rel %.1e, checksums rel %.1e; "
                      "%d/%d single upsets reported and repaired identically",
                      dprod, dcs, same, trials)};
}

// Decoupled baseline (tests/test_efta.cpp:248-313 at the GPU tile geometry): the three-kernel
// pipeline matches the two-pass reference, and a single upset in each kernel (block checksum of
// the score GEMM, duplicated softmax, denominator, block checksum of the output GEMM) is
// detected and repaired.
Verdict decoupled_baseline() {
    AttnConfig cfg(512, 64, 128, 8);
    const Thresholds thr{7e-6, 1e-3, 5e-3};
    Inputs in(cfg, 777);
    Matrix ref(cfg.seq_len, cfg.head_dim);
    if (eorc_standard_attention(cfg.seq_len, cfg.head_dim, cfg.block, cfg.stride, 0.0f, in.q.data(), in.k.data(),
                                in.v.data(), ref.data()))
        return {false, "oracle standard_attention failed"};
    auto [o, rep] = decoupled_ft_forward(in.q, in.k, in.v, cfg, thr);
    const double tol = 1e-2 * max_abs(ref);
    if (!(max_abs_diff(o, ref) <= tol) || rep.detections != 0 || rep.failed)
        return {false, fmt("clean: diff %.3e det %d", max_abs_diff(o, ref), rep.detections)};
    std::string detail = fmt("clean diff %.2e;", max_abs_diff(o, ref));
    for (const char* spec : {"GEMM1_OUT:0:1:2:3:30", "EXP_OUT:1:1:3:4:30", "REDUCE_SUM:2:0:5:0:30",
                             "GEMM2_ACC:1:0:2:7:30"}) {
        FaultPlan plan;
        plan.specs.push_back(FaultSpec::parse(spec));
        FaultInjector inj(plan);
        auto [of, rf] = decoupled_ft_forward(in.q, in.k, in.v, cfg, thr, &inj);
        if (rf.detections == 0 || rf.failed || !(max_abs_diff(of, ref) <= tol) || inj.fired().size() != 1)
            return {false, fmt("%s: det %d failed %d diff %.3e", spec, rf.detections, int(rf.failed),
                               max_abs_diff(of, ref))};
        detail += fmt(" %s repaired;", spec);
    }
    return {true, detail};
}

// 10. Threshold sweep shape (acceptance.cpp:387-405): detection and false-alarm rates both fall
//     monotonically as the thresholds are loosened.
Verdict sweep_shape() {
    AttnConfig cfg(512, 64, 128, 8);
    CalibrationResult cal = calibrate_thresholds(cfg, FTMode::EFTA_OPTIMIZED, 60, 1.0, 0xca11b010ull);
    auto sw = threshold_sweep(cfg, FTMode::EFTA_OPTIMIZED, cal.thr, 60, 0x5eebull, 10);
    if (sw.size() != 10) return {false, "sweep did not produce 10 points"};
    for (size_t i = 0; i + 1 < sw.size(); ++i)
        if (sw[i].detection_rate < sw[i + 1].detection_rate || sw[i].false_alarm_rate < sw[i + 1].false_alarm_rate)
            return {false, fmt("rates rise between points %zu and %zu", i, i + 1)};
    return {true, fmt("10 points: detection %.3f -> %.3f, false alarms %.3f -> %.3f, both monotone non-increasing",
                      sw.front().detection_rate, sw.back().detection_rate, sw.front().false_alarm_rate,
                      sw.back().false_alarm_rate)};
}

}  // namespace

int main() {
    struct Check {
        const char* name;
        std::function<Verdict()> run;
    };
    const std::vector<Check> checks = {
        {"1 fused GPU forward matches the two-pass reference", blocked_matches_reference},
        {"2 protected modes are bit-identical without faults", protected_modes_bit_identical},
        {"4 exhaustive single-fault sweep is fully absorbed (d=64)", [] { return single_fault_sweep(64); }},
        {"4 exhaustive single-fault sweep is fully absorbed (d=128)", [] { return single_fault_sweep(128); }},
        {"7 denominator range contract", rowsum_range_contract},
        {"abft operator API matches the reference", abft_operator_api},
        {"10 threshold sweep is monotone", sweep_shape},
        {"decoupled baseline matches the reference and repairs single faults", decoupled_baseline},
    };
    int failed = 0;
    for (const auto& c : checks) {
        Verdict v;
        try {
            v = c.run();
        } catch (const std::exception& e) {
            v = {false, std::string("exception: ") + e.what()};
        }
        std::printf("[%s] %s: %s\n", v.pass ? "PASS" : "FAIL", c.name, v.detail.c_str());
        std::fflush(stdout);
        failed += !v.pass;
    }
    return failed ? 1 : 0;
}
