// sweep_gpu.cpp — the paper's detector curves (Fig. 8/10; reference src/campaign.cpp:261-357) on the
// GPU through the C++ drop-in (efta_b200::calibrate_thresholds / threshold_sweep, the fault-tap
// build of the pair kernel), printed as one JSON object. Built by tools/Makefile.
//   sweep_gpu N D CAL_TRIALS SAFETY CAL_SEED TRIALS SEED POINTS
#include <cstdio>
#include <cstdlib>

#include "efta_b200.hpp"

int main(int argc, char** argv) {
    if (argc != 9) {
        std::fprintf(stderr, "usage: sweep_gpu N D CAL_TRIALS SAFETY CAL_SEED TRIALS SEED POINTS\n");
        return 2;
    }
    const int n = std::atoi(argv[1]), d = std::atoi(argv[2]), cal_trials = std::atoi(argv[3]);
    const double safety = std::atof(argv[4]);
    const unsigned long long cal_seed = std::strtoull(argv[5], nullptr, 0);
    const int trials = std::atoi(argv[6]);
    const unsigned long long seed = std::strtoull(argv[7], nullptr, 0);
    const int points = std::atoi(argv[8]);
    efta_b200::AttnConfig cfg(n, d, 128, 8);
    auto cal = efta_b200::calibrate_thresholds(cfg, efta_b200::FTMode::EFTA_OPTIMIZED, cal_trials, safety, cal_seed);
    auto sw = efta_b200::threshold_sweep(cfg, efta_b200::FTMode::EFTA_OPTIMIZED, cal.thr, trials, seed, points);
    std::printf("{\"n\": %d, \"d\": %d, \"base\": [%.9g, %.9g, %.9g], \"points\": [", n, d, cal.thr.eps1, cal.thr.eps2,
                cal.thr.eps_lin);
    for (size_t i = 0; i < sw.size(); ++i)
        std::printf("%s[%.6g, %.6g, %.6g]", i ? ", " : "", sw[i].multiplier, sw[i].detection_rate,
                    sw[i].false_alarm_rate);
    std::printf("]}\n");
    return 0;
}
