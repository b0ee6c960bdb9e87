// efta_host.cu — C++ host layer: the drop-in efta_b200:: API (include/efta_b200.hpp)
// over the C-ABI, plus the reference's host-side helpers (Rng, Matrix::random,
// sample_random_plan, classify_trial) exported through the C-ABI for the Python
// mirror. Host code only; all attention compute goes to the GPU kernels.
#include <cuda_fp16.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <stdexcept>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/efta_b200.h"
#include "../../include/efta_b200.hpp"

namespace efta_b200 {

namespace {
const char* kSiteNames[FAULT_SITE_COUNT] = {"GEMM1_OUT", "SUB_MAX", "EXP_OUT", "REDUCE_MAX",
                                            "REDUCE_SUM", "RESCALE_FACTOR", "GEMM2_ACC",
                                            "NORMALIZE_OUT"};

// column bound per site (reference src/fault.cpp:81-96)
int site_col_bound(FaultSite s, const AttnConfig& cfg) {
    switch (s) {
        case FaultSite::GEMM1_OUT:
        case FaultSite::SUB_MAX:
        case FaultSite::EXP_OUT: return cfg.block;
        case FaultSite::REDUCE_MAX:
        case FaultSite::REDUCE_SUM: return 1;
        default: return cfg.head_dim;
    }
}

uint16_t to_half_bits(float f) {
    __half h = __float2half_rn(f);  // host-side RNE conversion
    uint16_t b;
    std::memcpy(&b, &h, 2);
    return b;
}
float from_half_bits(uint16_t b) {
    __half h;
    std::memcpy(&h, &b, 2);
    return __half2float(h);
}
}  // namespace

void AttnConfig::validate() {
    efta_attn_desc d{};
    d.batch = 1;
    d.heads = heads;
    d.seq_len = seq_len;
    d.head_dim = head_dim;
    d.block = block;
    d.stride = stride;
    d.mode = EFTA_MODE_NONE;
    if (efta_attn_validate(&d) != 0) throw ConfigError(efta_last_error());
    if (scale == 0.0f) scale = 1.0f / std::sqrt(static_cast<float>(head_dim));
}

Thresholds Thresholds::observe() {
    const double inf = std::numeric_limits<double>::infinity();
    return Thresholds{inf, inf, inf};
}

const char* ft_mode_name(FTMode m) {
    switch (m) {
        case FTMode::NONE: return "none";
        case FTMode::EFTA: return "efta";
        case FTMode::EFTA_OPTIMIZED: return "efta-opt";
        case FTMode::DECOUPLED: return "decoupled";
    }
    return "?";
}
std::optional<FTMode> ft_mode_from_name(const std::string& n) {
    if (n == "none") return FTMode::NONE;
    if (n == "efta") return FTMode::EFTA;
    if (n == "efta-opt" || n == "efta_optimized") return FTMode::EFTA_OPTIMIZED;
    if (n == "decoupled") return FTMode::DECOUPLED;
    return std::nullopt;
}
const char* fault_site_name(FaultSite s) { return kSiteNames[static_cast<int>(s)]; }
std::optional<FaultSite> fault_site_from_name(const std::string& n) {
    for (int i = 0; i < FAULT_SITE_COUNT; ++i)
        if (n == kSiteNames[i]) return static_cast<FaultSite>(i);
    return std::nullopt;
}
float flip_bit(float v, int width, int bit) {
    if (width == 32) {
        if (bit < 0 || bit > 31) throw std::invalid_argument("flip_bit: bit out of range");
        return efta_flip_bit(v, 32, bit);
    }
    if (width == 16) {
        if (bit < 0 || bit > 15) throw std::invalid_argument("flip_bit: bit out of range");
        return from_half_bits(static_cast<uint16_t>(to_half_bits(v) ^ (1u << bit)));
    }
    throw std::invalid_argument("flip_bit: width must be 16 or 32");
}

uint32_t Rng::below(uint32_t n) {
    const uint64_t span = 0x100000000ull;
    const uint64_t limit = span - span % n;
    for (;;) {
        const uint64_t x = next_u64() >> 32;
        if (x < limit) return static_cast<uint32_t>(x % n);
    }
}

uint64_t trial_seed(uint64_t base, uint64_t trial) {
    uint64_t s = base ^ (0xd1b54a32d192ed03ull * (trial + 1));
    uint64_t z = (s += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

Matrix random_half_matrix(int rows, int cols, Rng& rng, double lo, double hi) {
    Matrix m(rows, cols);
    for (int r = 0; r < rows; ++r)
        for (int c = 0; c < cols; ++c)
            m.at(r, c) = from_half_bits(to_half_bits(static_cast<float>(rng.uniform(lo, hi))));
    return m;
}

std::string FaultSpec::to_string() const {
    std::string s = std::string(fault_site_name(site)) + ":" + std::to_string(block_i) + ":" +
                    std::to_string(block_j) + ":" + std::to_string(row) + ":" +
                    std::to_string(col) + ":" + std::to_string(bit);
    if (trigger != 1) s += ":" + std::to_string(trigger);
    return s;
}

FaultSpec FaultSpec::parse(const std::string& text) {
    std::vector<std::string> parts(1);
    for (char ch : text) {
        if (ch == ':') parts.emplace_back();
        else parts.back().push_back(ch);
    }
    if (parts.size() != 6 && parts.size() != 7)
        throw ConfigError("fault spec: expected SITE:i:j:row:col:bit[:trigger], got '" + text + "'");
    FaultSpec f;
    auto site = fault_site_from_name(parts[0]);
    if (!site) throw ConfigError("fault spec: unknown site '" + parts[0] + "'");
    f.site = *site;
    try {
        f.block_i = std::stoi(parts[1]);
        f.block_j = std::stoi(parts[2]);
        f.row = std::stoi(parts[3]);
        f.col = std::stoi(parts[4]);
        f.bit = std::stoi(parts[5]);
        f.trigger = parts.size() == 7 ? std::stoi(parts[6]) : 1;
    } catch (const std::exception&) {
        throw ConfigError("fault spec: bad integer field in '" + text + "'");
    }
    return f;
}

void FaultPlan::validate(const AttnConfig& cfg) const {
    const int n = cfg.num_blocks();
    std::vector<int> per(n, 0);
    for (const FaultSpec& f : specs) {
        if (f.block_i < 0 || f.block_i >= n) throw ConfigError("fault plan: block_i out of range");
        const bool post = f.site == FaultSite::NORMALIZE_OUT;
        if (f.block_j < 0 || f.block_j >= (post ? 1 : n))
            throw ConfigError("fault plan: block_j out of range");
        if (f.row < 0 || f.row >= cfg.block) throw ConfigError("fault plan: row out of range");
        if (f.col < 0 || f.col >= site_col_bound(f.site, cfg))
            throw ConfigError("fault plan: col out of range for site");
        if (f.bit < 0 || f.bit > 31) throw ConfigError("fault plan: bit out of range");
        if (f.trigger < 1) throw ConfigError("fault plan: trigger must be >= 1");
        if (++per[f.block_i] > 1)
            throw ConfigError("fault plan: multiple faults in one detection cycle (row-block " +
                              std::to_string(f.block_i) + ")");
    }
}

FaultPlan sample_random_plan(const AttnConfig& cfg, const std::vector<FaultSite>& sites, Rng& rng) {
    if (sites.empty()) throw ConfigError("sample_random_plan: empty site list");
    FaultSpec f;
    f.site = sites[rng.below(static_cast<uint32_t>(sites.size()))];
    const int n = cfg.num_blocks();
    f.block_i = static_cast<int>(rng.below(n));
    f.block_j = f.site == FaultSite::NORMALIZE_OUT ? 0 : static_cast<int>(rng.below(n));
    f.row = static_cast<int>(rng.below(cfg.block));
    f.col = static_cast<int>(rng.below(site_col_bound(f.site, cfg)));
    f.bit = static_cast<int>(rng.below(32));
    f.trigger = 1;
    FaultPlan plan;
    plan.specs.push_back(f);
    plan.validate(cfg);
    return plan;
}

double FTReport::max_residual(CheckKind kind) const {
    double m = -std::numeric_limits<double>::infinity();
    for (const auto& e : events)
        if (e.kind == kind) m = std::max(m, e.rep.residual);
    return m;
}

std::pair<Matrix, FTReport> efta_forward(const Matrix& q, const Matrix& k, const Matrix& v,
                                         const AttnConfig& cfg_in, const Thresholds& thr,
                                         FTMode mode, FaultInjector* inj,
                                         const KernelKnobs* knobs) {
    AttnConfig cfg = cfg_in;
    cfg.validate();
    const int n = cfg.seq_len, d = cfg.head_dim;
    if (q.rows() != n || q.cols() != d || k.rows() != n || k.cols() != d || v.rows() != n ||
        v.cols() != d)
        throw ConfigError("attention: Q/K/V must all be seq_len x head_dim");
    if (inj) inj->plan().validate(cfg);
    efta_attn_desc desc{};
    desc.batch = 1;
    desc.heads = 1;
    desc.seq_len = n;
    desc.head_dim = d;
    desc.block = cfg.block;
    desc.stride = cfg.stride;
    desc.scale = cfg.scale;
    desc.mode = static_cast<int>(mode);
    desc.eps1 = thr.eps1;
    desc.eps2 = thr.eps2;
    desc.eps_lin = thr.eps_lin;
    desc.observe_linear = knobs && knobs->observe_linear;
    desc.rowmax_bias = knobs ? knobs->rowmax_bias : 0.0f;
    // an injector (even with an empty plan: a fault-free twin) selects the fault-tap build
    desc.debug = inj != nullptr || desc.observe_linear;
    std::vector<uint16_t> hq(static_cast<size_t>(n) * d), hk(hq.size()), hv(hq.size());
    for (size_t i = 0; i < hq.size(); ++i) {
        hq[i] = to_half_bits(q.data()[i]);
        hk[i] = to_half_bits(k.data()[i]);
        hv[i] = to_half_bits(v.data()[i]);
    }
    std::vector<efta_fault_spec> faults;
    if (inj)
        for (const FaultSpec& f : inj->plan().specs)
            faults.push_back({0, static_cast<int>(f.site), f.block_i, f.block_j, f.row, f.col, f.bit,
                              f.trigger});
    const int ev_cap = 4 * cfg.num_blocks() * (cfg.num_blocks() + 2) + 64 + (mode == FTMode::DECOUPLED ? 4 * n : 0);
    std::vector<efta_event> events(ev_cap);
    std::vector<efta_fired> fired(64);
    efta_counters cnt{};
    Matrix out(n, d);
    FTReport rep;
    rep.mode = mode;
    rep.final_m.resize(n);
    rep.final_l.resize(n);
    const int rc = efta_attn_fwd_host_f16(&desc, hq.data(), hk.data(), hv.data(), out.data(),
                                          rep.final_m.data(), rep.final_l.data(),
                                          faults.empty() ? nullptr : faults.data(),
                                          static_cast<int>(faults.size()), events.data(), ev_cap,
                                          fired.data(), 64, &cnt);
    if (rc == 1) throw ConfigError(efta_last_error());
    if (rc != 0) throw std::runtime_error(efta_last_error());
    rep.detections = cnt.detections;
    rep.corrections = cnt.corrections;
    rep.recomputes = cnt.recomputes;
    rep.range_replacements = cnt.range_replacements;
    rep.failed = cnt.failed != 0;
    for (int i = 0; i < 3; ++i) rep.family_max[i] = cnt.family_max[i];
    for (int i = 0; i < std::min(cnt.n_events, ev_cap); ++i) {
        const efta_event& e = events[i];
        StageEvent se;
        se.kind = static_cast<CheckKind>(e.kind);
        se.block_i = e.block_i;
        se.block_j = e.block_j;
        se.rep.status = static_cast<VerifyStatus>(e.status);
        se.rep.row = e.row;
        se.rep.col = e.col;
        se.rep.violations = e.violations;
        se.rep.corrections = e.corrections;
        se.rep.checksum_repair = e.checksum_repair != 0;
        se.rep.residual = e.residual;
        se.rep.delta = e.delta;
        rep.events.push_back(se);
    }
    if (inj) {
        inj->fired_mut().clear();
        for (int i = 0; i < std::min(cnt.n_fired, 64); ++i) {
            FiredFault ff;
            const efta_fault_spec& s = fired[i].spec;
            ff.spec.site = static_cast<FaultSite>(s.site);
            ff.spec.block_i = s.block_i;
            ff.spec.block_j = s.block_j;
            ff.spec.row = s.row;
            ff.spec.col = s.col;
            ff.spec.bit = s.bit;
            ff.spec.trigger = s.trigger;
            ff.before = fired[i].before;
            ff.after = fired[i].after;
            inj->fired_mut().push_back(ff);
        }
    }
    return {std::move(out), std::move(rep)};
}

std::pair<Matrix, FTReport> decoupled_ft_forward(const Matrix& q, const Matrix& k, const Matrix& v,
                                                 const AttnConfig& cfg, const Thresholds& thr, FaultInjector* inj,
                                                 const KernelKnobs* knobs) {
    return efta_forward(q, k, v, cfg, thr, FTMode::DECOUPLED, inj, knobs);
}

// ------------------------------------------------------------------ strided ABFT on the GPU
namespace {

// device buffer owned by one drop-in call (the C-ABI itself never allocates)
struct DevBuf {
    void* p = nullptr;
    explicit DevBuf(size_t bytes) {
        if (bytes && cudaMalloc(&p, bytes) != cudaSuccess) throw std::runtime_error("cudaMalloc failed");
    }
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    template <typename T>
    T* as() const { return static_cast<T*>(p); }
};

void cuda_check(cudaError_t e) {
    if (e != cudaSuccess) throw std::runtime_error(cudaGetErrorString(e));
}
void capi_check(int rc) {
    if (rc == 1) throw std::invalid_argument(efta_last_error());
    if (rc != 0) throw std::runtime_error(efta_last_error());
}

// full-width checksums of a product from its per-256-column-tile ones:
//   c1 = sum_t c1_t,  c2 = sum_t (c2_t + 32 t c1_t)   (group index l = 32 t + l')
// and, when given, the accumulated pair of C = C_init + A.B (checksummed_gemm's cp_init)
__global__ void compose_tile_checksums(int rows, int tiles, const float* __restrict__ ycs,
                                       const float* __restrict__ init1, const float* __restrict__ init2,
                                       float* __restrict__ c1, float* __restrict__ c2) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= rows * 8) return;
    const int r = i / 8, x = i % 8;
    float a = 0.0f, b = 0.0f;
    for (int t = 0; t < tiles; ++t) {
        const float* cs = ycs + (static_cast<size_t>(r) * tiles + t) * 16;
        a = __fadd_rn(a, cs[x]);
        b = __fadd_rn(b, __fadd_rn(cs[8 + x], __fmul_rn(32.0f * t, cs[x])));
    }
    if (init1) {
        a = __fadd_rn(init1[i], a);
        b = __fadd_rn(init2[i], b);
    }
    c1[i] = a;
    c2[i] = b;
}
__global__ void add_into(size_t n, const float* __restrict__ src, float* __restrict__ dst) {
    const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) dst[i] = __fadd_rn(src[i], dst[i]);
}

}  // namespace

ChecksumPair encode_strided(const Matrix& t, int stride, Counters*) {
    if (stride <= 0 || t.cols() % stride != 0)
        throw std::invalid_argument("encode_strided: stride must divide tile width");
    ChecksumPair cp;
    cp.stride = stride;
    cp.groups = t.cols() / stride;
    cp.c1 = Matrix(t.rows(), stride);
    cp.c2 = Matrix(t.rows(), stride);
    const size_t nt = static_cast<size_t>(t.rows()) * t.cols(), nc = static_cast<size_t>(t.rows()) * stride;
    DevBuf dt(nt * 4), d1(nc * 4), d2(nc * 4);
    cuda_check(cudaMemcpy(dt.p, t.data(), nt * 4, cudaMemcpyHostToDevice));
    capi_check(efta_encode_strided_f32(t.rows(), t.cols(), stride, dt.as<float>(), d1.as<float>(), d2.as<float>(),
                                       nullptr));
    cuda_check(cudaMemcpy(cp.c1.data(), d1.p, nc * 4, cudaMemcpyDeviceToHost));
    cuda_check(cudaMemcpy(cp.c2.data(), d2.p, nc * 4, cudaMemcpyDeviceToHost));
    return cp;
}

VerificationReport verify_locate_correct(Matrix& t, const ChecksumPair& cp, double eps_abs, Counters*,
                                         const std::vector<double>* row_eps_mult) {
    const int rows = t.rows(), stride = cp.stride;
    if (stride <= 0 || t.cols() != stride * cp.groups || cp.c1.rows() != rows || cp.c2.rows() != rows ||
        cp.c1.cols() != stride || cp.c2.cols() != stride)
        throw std::invalid_argument("verify_locate_correct: checksum/tile shape mismatch");
    if (row_eps_mult && static_cast<int>(row_eps_mult->size()) != rows)
        throw std::invalid_argument("verify_locate_correct: row_eps_mult size mismatch");
    VerificationReport rep;
    if (rows == 0) return rep;
    const size_t nt = static_cast<size_t>(rows) * t.cols(), nc = static_cast<size_t>(rows) * stride;
    const size_t ws = efta_verify_workspace_bytes(rows);
    DevBuf dt(nt * 4), d1(nc * 4), d2(nc * 4), dm(row_eps_mult ? rows * sizeof(double) : 0),
        dr(sizeof(efta_verify_report)), dws(ws);
    cuda_check(cudaMemcpy(dt.p, t.data(), nt * 4, cudaMemcpyHostToDevice));
    cuda_check(cudaMemcpy(d1.p, cp.c1.data(), nc * 4, cudaMemcpyHostToDevice));
    cuda_check(cudaMemcpy(d2.p, cp.c2.data(), nc * 4, cudaMemcpyHostToDevice));
    if (row_eps_mult)
        cuda_check(cudaMemcpy(dm.p, row_eps_mult->data(), rows * sizeof(double), cudaMemcpyHostToDevice));
    capi_check(efta_verify_locate_correct_f32(rows, t.cols(), stride, dt.as<float>(), d1.as<float>(),
                                              d2.as<float>(), eps_abs, row_eps_mult ? dm.as<double>() : nullptr,
                                              dr.as<efta_verify_report>(), dws.p, ws, nullptr));
    efta_verify_report r{};
    cuda_check(cudaMemcpy(&r, dr.p, sizeof r, cudaMemcpyDeviceToHost));
    cuda_check(cudaMemcpy(t.data(), dt.p, nt * 4, cudaMemcpyDeviceToHost));
    rep.status = static_cast<VerifyStatus>(r.status);
    rep.row = r.row;
    rep.col = r.col;
    rep.violations = r.violations;
    rep.corrections = r.corrections;
    rep.checksum_repair = r.checksum_repair != 0;
    rep.residual = r.residual;
    rep.delta = r.delta;
    return rep;
}

std::pair<Matrix, ChecksumPair> checksummed_gemm(const Matrix& a, const Matrix& bt, int stride, Counters*,
                                                 GemmStage, const Matrix* c_init, const ChecksumPair* cp_init) {
    const int m = a.rows(), k = a.cols(), w = bt.cols();
    if (bt.rows() != k) throw std::invalid_argument("checksummed_gemm: inner dimensions differ");
    if (stride <= 0 || w % stride != 0) throw std::invalid_argument("encode_strided: stride must divide tile width");
    if (stride != 8 || m % 128 || w % 256 || k % 64)
        throw std::invalid_argument("checksummed_gemm: this kernel needs stride 8, M % 128 == 0, "
                                    "W % 256 == 0, K % 64 == 0");
    if (c_init && !cp_init) throw std::invalid_argument("checksummed_gemm: c_init without cp_init");
    if (c_init && (c_init->rows() != m || c_init->cols() != w || cp_init->c1.rows() != m))
        throw std::invalid_argument("checksummed_gemm: c_init shape mismatch");
    // operands to the fp16 grid: X = a [M x K], W = bt^T [W x K] (the kernel's nn.Linear layout)
    std::vector<uint16_t> hx(static_cast<size_t>(m) * k), hw(static_cast<size_t>(w) * k);
    for (size_t i = 0; i < hx.size(); ++i) hx[i] = to_half_bits(a.data()[i]);
    for (int r = 0; r < k; ++r)
        for (int c = 0; c < w; ++c) hw[static_cast<size_t>(c) * k + r] = to_half_bits(bt(r, c));
    efta_gemm_desc d{m, w, k, 8, 256, std::numeric_limits<double>::infinity(), 0};
    const int tiles = w / 256;
    const size_t ny = static_cast<size_t>(m) * w, ncs = static_cast<size_t>(m) * tiles * 16, nc = m * 8ull;
    DevBuf dx(hx.size() * 2), dw(hw.size() * 2), dwc(efta_abft_weight_cs_bytes(&d)), dy(ny * 4), dcs(ncs * 4),
        dcnt(sizeof(efta_counters)), d1(nc * 4), d2(nc * 4), di(c_init ? ny * 4 : 0), di1(c_init ? nc * 4 : 0),
        di2(c_init ? nc * 4 : 0);
    cuda_check(cudaMemcpy(dx.p, hx.data(), hx.size() * 2, cudaMemcpyHostToDevice));
    cuda_check(cudaMemcpy(dw.p, hw.data(), hw.size() * 2, cudaMemcpyHostToDevice));
    capi_check(efta_abft_encode_weight_f16(&d, dw.as<uint16_t>(), dwc.as<uint16_t>(), nullptr));
    capi_check(efta_abft_gemm_ex(&d, dx.as<uint16_t>(), dw.as<uint16_t>(), dwc.as<uint16_t>(), dy.p, 1,
                                 dcs.as<float>(), nullptr, 0, nullptr, 0, dcnt.as<efta_counters>(), nullptr));
    if (c_init) {
        cuda_check(cudaMemcpy(di.p, c_init->data(), ny * 4, cudaMemcpyHostToDevice));
        cuda_check(cudaMemcpy(di1.p, cp_init->c1.data(), nc * 4, cudaMemcpyHostToDevice));
        cuda_check(cudaMemcpy(di2.p, cp_init->c2.data(), nc * 4, cudaMemcpyHostToDevice));
        add_into<<<static_cast<unsigned>((ny + 255) / 256), 256>>>(ny, di.as<float>(), dy.as<float>());
    }
    compose_tile_checksums<<<static_cast<unsigned>((nc + 255) / 256), 256>>>(
        m, tiles, dcs.as<float>(), c_init ? di1.as<float>() : nullptr, c_init ? di2.as<float>() : nullptr,
        d1.as<float>(), d2.as<float>());
    cuda_check(cudaGetLastError());
    Matrix c(m, w);
    ChecksumPair cp;
    cp.stride = stride;
    cp.groups = w / stride;
    cp.c1 = Matrix(m, stride);
    cp.c2 = Matrix(m, stride);
    cuda_check(cudaMemcpy(c.data(), dy.p, ny * 4, cudaMemcpyDeviceToHost));
    cuda_check(cudaMemcpy(cp.c1.data(), d1.p, nc * 4, cudaMemcpyDeviceToHost));
    cuda_check(cudaMemcpy(cp.c2.data(), d2.p, nc * 4, cudaMemcpyDeviceToHost));
    return {std::move(c), std::move(cp)};
}

// ------------------------------------------------------------------ calibration / sweep
namespace {
struct Family {
    double exp = -std::numeric_limits<double>::infinity(), out = -std::numeric_limits<double>::infinity(),
           lin = -std::numeric_limits<double>::infinity();
    bool hard = false;
};
// FamilyResiduals (src/campaign.cpp:55-85) of one observation run: the device keeps the worst
// clean residual per family (family_max) and logs range events, which are the "hard" trips
Family family_of(const FTReport& rep) {
    Family f;
    if (rep.family_max[0] > 0) f.exp = rep.family_max[0];
    if (rep.family_max[1] > 0) f.out = rep.family_max[1];
    if (rep.family_max[2] > 0) f.lin = rep.family_max[2];
    for (const auto& e : rep.events) {
        if (e.kind == CheckKind::FACTOR_RANGE || e.kind == CheckKind::ROWSUM_RANGE) f.hard = true;
        const double r = e.rep.residual;
        if (!std::isfinite(r)) continue;
        if (e.kind == CheckKind::EXP_CHECKSUM) f.exp = std::max(f.exp, r);
        if (e.kind == CheckKind::OUTPUT_CHECKSUM) f.out = std::max(f.out, r);
        if (e.kind == CheckKind::SCORE_CHECKSUM) f.lin = std::max(f.lin, r);
    }
    return f;
}
}  // namespace

CalibrationResult calibrate_thresholds(const AttnConfig& cfg_in, FTMode mode, int trials, double safety,
                                       uint64_t seed) {
    AttnConfig cfg = cfg_in;
    cfg.validate();
    if (trials <= 0) throw ConfigError("calibration: trials must be positive");
    if (safety < 1.0) throw ConfigError("calibration: safety factor must be >= 1");
    const double inf = std::numeric_limits<double>::infinity();
    KernelKnobs knobs;
    knobs.observe_linear = true;
    double mexp = -inf, mout = -inf, mlin = -inf;
    for (int t = 0; t < trials; ++t) {
        Rng rng(trial_seed(seed, static_cast<uint64_t>(t)));
        const Matrix q = random_half_matrix(cfg.seq_len, cfg.head_dim, rng);
        const Matrix k = random_half_matrix(cfg.seq_len, cfg.head_dim, rng);
        const Matrix v = random_half_matrix(cfg.seq_len, cfg.head_dim, rng);
        auto res = efta_forward(q, k, v, cfg, Thresholds::observe(), mode, nullptr, &knobs);
        const Family f = family_of(res.second);
        mexp = std::max(mexp, f.exp);
        mout = std::max(mout, f.out);
        mlin = std::max(mlin, f.lin);
    }
    CalibrationResult r;
    r.max_exp = std::isfinite(mexp) ? mexp : 0.0;
    r.max_out = std::isfinite(mout) ? mout : 0.0;
    r.max_lin = std::isfinite(mlin) ? mlin : 0.0;
    r.degenerate = !(std::isfinite(mexp) && mexp > 0.0) || !(std::isfinite(mout) && mout > 0.0) ||
                   !(std::isfinite(mlin) && mlin > 0.0);
    r.thr.eps1 = std::isfinite(mexp) ? mexp * safety : inf;
    r.thr.eps2 = std::isfinite(mout) ? mout * safety : inf;
    r.thr.eps_lin = std::isfinite(mlin) ? mlin * safety : inf;
    return r;
}

std::vector<SweepPoint> threshold_sweep(const AttnConfig& cfg_in, FTMode mode, const Thresholds& base, int trials,
                                        uint64_t seed, int points) {
    AttnConfig cfg = cfg_in;
    cfg.validate();
    if (trials <= 0 || points <= 1) throw ConfigError("sweep: trials and points must be positive");
    KernelKnobs knobs;
    knobs.observe_linear = true;
    const std::vector<FaultSite> sites = {FaultSite::GEMM1_OUT,  FaultSite::SUB_MAX,        FaultSite::EXP_OUT,
                                          FaultSite::REDUCE_MAX, FaultSite::REDUCE_SUM,     FaultSite::RESCALE_FACTOR,
                                          FaultSite::GEMM2_ACC,  FaultSite::NORMALIZE_OUT};
    std::vector<Family> clean_runs, fault_runs;
    for (int t = 0; t < trials; ++t) {
        Rng rng(trial_seed(seed, static_cast<uint64_t>(t)));
        const Matrix q = random_half_matrix(cfg.seq_len, cfg.head_dim, rng);
        const Matrix k = random_half_matrix(cfg.seq_len, cfg.head_dim, rng);
        const Matrix v = random_half_matrix(cfg.seq_len, cfg.head_dim, rng);
        clean_runs.push_back(family_of(efta_forward(q, k, v, cfg, Thresholds::observe(), mode, nullptr, &knobs).second));
        FaultInjector inj(sample_random_plan(cfg, sites, rng));
        fault_runs.push_back(family_of(efta_forward(q, k, v, cfg, Thresholds::observe(), mode, &inj, &knobs).second));
    }
    auto trips = [&](const Family& f, double mult) {
        if (f.hard) return true;
        if (std::isfinite(f.exp) && std::isfinite(base.eps1) && f.exp > base.eps1 * mult) return true;
        if (std::isfinite(f.out) && std::isfinite(base.eps2) && f.out > base.eps2 * mult) return true;
        if (std::isfinite(f.lin) && std::isfinite(base.eps_lin) && f.lin > base.eps_lin * mult) return true;
        return false;
    };
    std::vector<SweepPoint> sweep;
    for (int p = 0; p < points; ++p) {
        SweepPoint sp;
        sp.multiplier = std::pow(10.0, -2.0 + 4.0 * p / (points - 1));
        int det = 0, fa = 0;
        for (const auto& f : fault_runs) det += trips(f, sp.multiplier) ? 1 : 0;
        for (const auto& f : clean_runs) fa += trips(f, sp.multiplier) ? 1 : 0;
        sp.detection_rate = static_cast<double>(det) / trials;
        sp.false_alarm_rate = static_cast<double>(fa) / trials;
        sweep.push_back(sp);
    }
    return sweep;
}

const char* outcome_name(Outcome o) {
    switch (o) {
        case Outcome::CLEAN: return "clean";
        case Outcome::FALSE_ALARM: return "false_alarm";
        case Outcome::CORRECTED: return "corrected";
        case Outcome::RANGE_RESTRICTED: return "range_restricted";
        case Outcome::MASKED_BENIGN: return "masked_benign";
        case Outcome::RANGE_CONTRACT: return "range_contract";
        case Outcome::UNCORRECTABLE: return "uncorrectable";
    }
    return "?";
}

}  // namespace efta_b200

// ------------------------------------------------------------------ C exports
namespace {

// reference classify_trial (src/campaign.cpp:123-152) over raw host arrays
int classify_raw(int rows, int cols, const float* out, const float* ref, int detections,
                 int range_replacements, int failed, const float* final_l, int n_l,
                 int plan_nonempty, int reduction_site, double eps2) {
    using efta_b200::Outcome;
    if (!plan_nonempty) return static_cast<int>(detections > 0 ? Outcome::FALSE_ALARM : Outcome::CLEAN);
    bool finite = true;
    double res = 0.0, refmax = 0.0;
    for (size_t i = 0; i < static_cast<size_t>(rows) * cols; ++i) {
        if (!std::isfinite(out[i])) finite = false;
        const double x = std::abs(static_cast<double>(out[i]) - ref[i]);
        res = std::isnan(x) ? std::numeric_limits<double>::infinity() : std::max(res, x);
        refmax = std::max(refmax, std::abs(static_cast<double>(ref[i])));
    }
    const double benign_tol = std::max(eps2, 1e-2 * refmax);
    bool argmax_ok = finite;
    for (int r = 0; r < rows && argmax_ok; ++r) {
        int ia = 0, ib = 0;
        for (int c = 1; c < cols; ++c) {
            if (out[r * cols + c] > out[r * cols + ia]) ia = c;
            if (ref[r * cols + c] > ref[r * cols + ib]) ib = c;
        }
        argmax_ok = ia == ib;
    }
    bool l_ok = true;
    for (int i = 0; i < n_l; ++i)
        l_ok &= std::isfinite(final_l[i]) && final_l[i] > 0.0f && final_l[i] <= static_cast<double>(rows);
    if (!finite || failed) return static_cast<int>(Outcome::UNCORRECTABLE);
    if (detections == 0) {
        if (res <= benign_tol) return static_cast<int>(Outcome::MASKED_BENIGN);
        if (reduction_site && l_ok && argmax_ok) return static_cast<int>(Outcome::RANGE_CONTRACT);
        return static_cast<int>(Outcome::UNCORRECTABLE);
    }
    if (res <= benign_tol) return static_cast<int>(Outcome::CORRECTED);
    if (range_replacements > 0 && argmax_ok) return static_cast<int>(Outcome::RANGE_RESTRICTED);
    if (reduction_site && l_ok && argmax_ok) return static_cast<int>(Outcome::RANGE_CONTRACT);
    return static_cast<int>(Outcome::UNCORRECTABLE);
}

}  // namespace

namespace efta_b200 {
Outcome classify_trial(const Matrix& out, const Matrix& ref, const FTReport& rep,
                       const FaultPlan& plan, const Thresholds& thr) {
    bool reduction = false;
    for (const auto& f : plan.specs)
        reduction |= f.site == FaultSite::REDUCE_MAX || f.site == FaultSite::REDUCE_SUM;
    if (!out.same_shape(ref)) return Outcome::UNCORRECTABLE;
    return static_cast<Outcome>(classify_raw(out.rows(), out.cols(), out.data(), ref.data(),
                                             rep.detections, rep.range_replacements, rep.failed,
                                             rep.final_l.data(), static_cast<int>(rep.final_l.size()),
                                             !plan.empty(), reduction, thr.eps2));
}
}  // namespace efta_b200

extern "C" {

uint64_t efta_trial_seed(uint64_t base, uint64_t trial) { return efta_b200::trial_seed(base, trial); }

int efta_gen_trial_f16(uint64_t seed, int n, int d, int block, int stride, const int* sites,
                       int n_sites, uint16_t* q, uint16_t* k, uint16_t* v, efta_fault_spec* spec) {
    try {
        efta_b200::Rng rng(seed);
        uint16_t* outs[3] = {q, k, v};
        for (uint16_t* o : outs)
            for (int i = 0; i < n * d; ++i)
                o[i] = efta_b200::to_half_bits(static_cast<float>(rng.uniform(-1.0, 1.0)));
        if (n_sites > 0 && spec) {
            efta_b200::AttnConfig cfg;
            cfg.seq_len = n;
            cfg.head_dim = d;
            cfg.block = block;
            cfg.stride = stride;
            std::vector<efta_b200::FaultSite> s;
            for (int i = 0; i < n_sites; ++i) s.push_back(static_cast<efta_b200::FaultSite>(sites[i]));
            efta_b200::FaultPlan plan = efta_b200::sample_random_plan(cfg, s, rng);
            const auto& f = plan.specs.front();
            *spec = {0, static_cast<int>(f.site), f.block_i, f.block_j, f.row, f.col, f.bit, f.trigger};
        }
        return 0;
    } catch (const std::exception& e) {
        return 1;
    }
}

int efta_classify_trial(int rows, int cols, const float* out, const float* ref, int detections,
                        int range_replacements, int failed, const float* final_l, int n_l,
                        int plan_nonempty, int reduction_site, double eps2) {
    return classify_raw(rows, cols, out, ref, detections, range_replacements, failed, final_l, n_l,
                        plan_nonempty, reduction_site, eps2);
}

}  // extern "C"
