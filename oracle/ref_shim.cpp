// ref_shim.cpp — TEST INFRASTRUCTURE ONLY.
//
// extern "C" adapter over the unmodified reference C++ API, compiled together
// with the reference sources *where they lie* (/root/reference/proj/src) by
// oracle/Makefile into oracle/_ref/libefta_ref.so. No reference source is
// copied into this repository; this file only calls the reference's public
// functions:
//   efta_forward            include/efta/efta.hpp:86-89
//   decoupled_ft_forward    include/efta/efta.hpp:94-96 (mode 3 = FTMode::DECOUPLED, dispatched
//                           like the campaign's forward(), src/campaign.cpp:18-23)
//   standard_attention      include/efta/attention.hpp:19-21
//   encode_strided          include/efta/abft.hpp:38
//   checksummed_gemm        include/efta/abft.hpp:73-77
//   verify_locate_correct   include/efta/abft.hpp:58-60
//   sample_random_plan      include/efta/fault.hpp:65-66
//   Rng / trial_seed        include/efta/rng.hpp:19-58
//   calibrate_thresholds / threshold_sweep   include/efta/campaign.hpp:87-110
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "efta/abft.hpp"
#include "efta/attention.hpp"
#include "efta/campaign.hpp"
#include "efta/efta.hpp"
#include "efta/fault.hpp"
#include "efta/half.hpp"
#include "efta/matrix.hpp"
#include "efta/rng.hpp"
#include "../oracle/oracle_abi.h"

using namespace efta;

namespace {
thread_local std::string g_err;

Matrix from_ptr(const float* p, int rows, int cols, Storage st = Storage::FULL) {
    Matrix m(rows, cols, st);
    std::memcpy(m.data(), p, sizeof(float) * static_cast<size_t>(rows) * cols);
    return m;
}
void to_ptr(const Matrix& m, float* p) {
    std::memcpy(p, m.data(), sizeof(float) * static_cast<size_t>(m.rows()) * m.cols());
}
FaultSpec to_spec(const orc_fault_spec& s) {
    FaultSpec f;
    f.site = static_cast<FaultSite>(s.site);
    f.block_i = s.block_i;
    f.block_j = s.block_j;
    f.row = s.row;
    f.col = s.col;
    f.bit = s.bit;
    f.trigger = s.trigger;
    return f;
}
orc_fault_spec from_spec(const FaultSpec& f) {
    return {static_cast<int>(f.site), f.block_i, f.block_j, f.row, f.col, f.bit, f.trigger};
}
void fill_report(const VerificationReport& r, orc_verify_report* o) {
    o->status = static_cast<int>(r.status);
    o->row = r.row;
    o->col = r.col;
    o->violations = r.violations;
    o->corrections = r.corrections;
    o->checksum_repair = r.checksum_repair ? 1 : 0;
    o->residual = r.residual;
    o->delta = r.delta;
}
}  // namespace

extern "C" {

const char* eref_last_error(void) { return g_err.c_str(); }

uint64_t eref_trial_seed(uint64_t base, uint64_t trial) { return trial_seed(base, trial); }

int eref_gen_trial(uint64_t seed, int n, int d, int block, int stride, const int* sites,
                   int n_sites, float* q, float* k, float* v, orc_fault_spec* spec_out) {
    try {
        Rng rng(seed);
        to_ptr(Matrix::random(n, d, rng), q);
        to_ptr(Matrix::random(n, d, rng), k);
        to_ptr(Matrix::random(n, d, rng), v);
        if (n_sites > 0) {
            AttnConfig cfg(n, d, block, stride);
            std::vector<FaultSite> s;
            for (int i = 0; i < n_sites; ++i) s.push_back(static_cast<FaultSite>(sites[i]));
            FaultPlan plan = sample_random_plan(cfg, s, rng, false);
            *spec_out = from_spec(plan.specs.front());
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

void eref_rng_below_seq(uint64_t seed, int n, const uint32_t* bounds, uint32_t* out) {
    Rng rng(seed);
    for (int i = 0; i < n; ++i) out[i] = rng.below(bounds[i]);
}

void eref_random_matrix(uint64_t seed, int rows, int cols, double lo, double hi, int half_grid,
                        float* out) {
    Rng rng(seed);
    to_ptr(Matrix::random(rows, cols, rng, lo, hi,
                          half_grid ? Storage::HALF_STORED : Storage::FULL),
           out);
}

float eref_flip_bit(float v, int width, int bit) { return flip_bit(v, width, bit); }
uint16_t eref_float_to_half_bits(float f) { return float_to_half_bits(f); }
float eref_half_bits_to_float(uint16_t h) { return half_bits_to_float(h); }

int eref_efta_forward(int n, int d, int block, int stride, float scale, int mode, double eps1,
                      double eps2, double eps_lin, int observe_linear, float rowmax_bias,
                      const float* q, const float* k, const float* v, float* o, float* m_out,
                      float* l_out, const orc_fault_spec* specs, int n_specs, orc_event* events,
                      int ev_cap, orc_fired* fired, int fired_cap, orc_summary* sum) {
    try {
        AttnConfig cfg(n, d, block, stride, 1, scale);
        Thresholds thr{eps1, eps2, eps_lin};
        Matrix mq = from_ptr(q, n, d, Storage::HALF_STORED);
        Matrix mk = from_ptr(k, n, d, Storage::HALF_STORED);
        Matrix mv = from_ptr(v, n, d, Storage::HALF_STORED);
        FaultPlan plan;
        for (int i = 0; i < n_specs; ++i) plan.specs.push_back(to_spec(specs[i]));
        FaultInjector inj(plan);
        KernelKnobs knobs;
        knobs.observe_linear = observe_linear != 0;
        knobs.rowmax_bias = rowmax_bias;
        auto [out, rep] = static_cast<FTMode>(mode) == FTMode::DECOUPLED
                              ? decoupled_ft_forward(mq, mk, mv, cfg, thr, n_specs > 0 ? &inj : nullptr, &knobs)
                              : efta_forward(mq, mk, mv, cfg, thr, static_cast<FTMode>(mode),
                                             n_specs > 0 ? &inj : nullptr, &knobs);
        to_ptr(out, o);
        if (m_out) std::memcpy(m_out, rep.final_m.data(), sizeof(float) * n);
        if (l_out) std::memcpy(l_out, rep.final_l.data(), sizeof(float) * n);
        if (sum) {
            std::memset(sum, 0, sizeof(*sum));
            sum->detections = rep.detections;
            sum->corrections = rep.corrections;
            sum->recomputes = rep.recomputes;
            sum->range_replacements = rep.range_replacements;
            sum->failed = rep.failed ? 1 : 0;
            sum->n_events = static_cast<int>(rep.events.size());
            sum->n_fired = static_cast<int>(inj.fired().size());
            const Counters& c = rep.counters;
            sum->flops_main = c.flops_main;
            sum->flops_checksum = c.flops_checksum;
            sum->flops_verify = c.flops_verify;
            sum->intermediate_elems = c.intermediate_elems;
            sum->flops_main_gemm_scores = c.flops_main_gemm_scores;
            sum->flops_cs_gemm_scores = c.flops_cs_gemm_scores;
            sum->flops_main_gemm_output = c.flops_main_gemm_output;
            sum->flops_cs_gemm_output = c.flops_cs_gemm_output;
            sum->exp_checks = c.exp_checks;
            sum->output_checks = c.output_checks;
        }
        for (int i = 0; i < static_cast<int>(rep.events.size()) && i < ev_cap; ++i) {
            const StageEvent& e = rep.events[i];
            orc_event& oe = events[i];
            std::memset(&oe, 0, sizeof(oe));
            oe.kind = static_cast<int>(e.kind);
            oe.block_i = e.block_i;
            oe.block_j = e.block_j;
            oe.status = static_cast<int>(e.rep.status);
            oe.row = e.rep.row;
            oe.col = e.rep.col;
            oe.violations = e.rep.violations;
            oe.corrections = e.rep.corrections;
            oe.checksum_repair = e.rep.checksum_repair ? 1 : 0;
            oe.residual = e.rep.residual;
            oe.delta = e.rep.delta;
        }
        for (int i = 0; i < static_cast<int>(inj.fired().size()) && i < fired_cap; ++i) {
            fired[i].spec = from_spec(inj.fired()[i].spec);
            fired[i].before = inj.fired()[i].before;
            fired[i].after = inj.fired()[i].after;
        }
        return 0;
    } catch (const ConfigError& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

int eref_standard_attention(int n, int d, int block, int stride, float scale, const float* q,
                            const float* k, const float* v, float* o) {
    try {
        AttnConfig cfg(n, d, block, stride, 1, scale);
        Matrix out = standard_attention(from_ptr(q, n, d, Storage::HALF_STORED),
                                        from_ptr(k, n, d, Storage::HALF_STORED),
                                        from_ptr(v, n, d, Storage::HALF_STORED), cfg);
        to_ptr(out, o);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

int eref_encode_strided(int rows, int cols, int stride, const float* t, float* c1, float* c2) {
    try {
        ChecksumPair cp = encode_strided(from_ptr(t, rows, cols), stride);
        to_ptr(cp.c1, c1);
        to_ptr(cp.c2, c2);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

int eref_checksummed_gemm(int m, int kd, int w, int stride, const float* a, const float* bt,
                          float* c, float* c1, float* c2) {
    try {
        auto [cm, cp] = checksummed_gemm(from_ptr(a, m, kd), from_ptr(bt, kd, w), stride);
        to_ptr(cm, c);
        to_ptr(cp.c1, c1);
        to_ptr(cp.c2, c2);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

int eref_verify_locate_correct(int rows, int cols, int stride, float* t, const float* c1,
                               const float* c2, double eps, const double* row_eps_mult,
                               orc_verify_report* rep) {
    try {
        Matrix mt = from_ptr(t, rows, cols);
        ChecksumPair cp;
        cp.stride = stride;
        cp.groups = cols / stride;
        cp.c1 = from_ptr(c1, rows, stride);
        cp.c2 = from_ptr(c2, rows, stride);
        std::vector<double> mult;
        if (row_eps_mult) mult.assign(row_eps_mult, row_eps_mult + rows);
        VerificationReport r =
            verify_locate_correct(mt, cp, eps, nullptr, row_eps_mult ? &mult : nullptr);
        to_ptr(mt, t);
        fill_report(r, rep);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// calibrate_thresholds + threshold_sweep (src/campaign.cpp:261-357): the base thresholds from
// `cal_trials` clean observation runs (x safety), then `points` log-spaced multipliers
int eref_threshold_sweep(int n, int d, int block, int stride, int mode, int cal_trials, double safety,
                         uint64_t cal_seed, int trials, uint64_t seed, int points, double* base,
                         double* mult, double* det, double* fa) {
    try {
        AttnConfig cfg(n, d, block, stride);
        CalibrationResult cal = calibrate_thresholds(cfg, static_cast<FTMode>(mode), cal_trials, safety, cal_seed);
        base[0] = cal.thr.eps1;
        base[1] = cal.thr.eps2;
        base[2] = cal.thr.eps_lin;
        auto sw = threshold_sweep(cfg, static_cast<FTMode>(mode), cal.thr, trials, seed, points);
        for (int i = 0; i < points; ++i) {
            mult[i] = sw[i].multiplier;
            det[i] = sw[i].detection_rate;
            fa[i] = sw[i].false_alarm_rate;
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

}  // extern "C"
