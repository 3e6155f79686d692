// rule.cuh -- the certified slice-count rule, one
// definition for the host path and the device-rule kernel (device: CUDA's log2).
#pragma once
#include <cmath>
#include <cstdint>

namespace mpc {

// log2 rho-hat from the reduced pre-pass integers (minT < 0: no nonzero pair -> 0)
__host__ __device__ inline double rule_log2rho(int64_t k, int64_t minT, int64_t minT1, int64_t maxD2) {
    double log2rho = 0.0;
    if (minT > 0) log2rho = log2((double)k) + 14.0 - log2((double)minT);
    else if (minT == 0) {
        log2rho = -1e300;
        if (minT1 >= 1) log2rho = log2((double)k) + 14.0 - log2((double)minT1);
        if (maxD2 >= 0) { double b2 = log2((double)k) + 2.0 + (double)maxD2; if (b2 > log2rho) log2rho = b2; }
        if (log2rho < -1e299) log2rho = 0.0;
    }
    return log2rho;
}

// s = min{ s >= 1 : bits s >= prec - 4 + log2(c s) + log2rho + 0.1 }, c = 3 (4M) / 4 (3M);
// -8 (MPCGEMM_ERR_SLICES) if s > smax
__host__ __device__ inline int rule_slices(int32_t prec, int method, double log2rho, int bits = 8, int smax = 1024) {
    const double c = method == 3 ? 4.0 : 3.0;
    for (int s = 1; s <= smax; s++)
        if ((double)bits * s >= (double)prec - 4.0 + log2(c * s) + log2rho + 0.1) return s;
    return -8;
}

}  // namespace mpc
