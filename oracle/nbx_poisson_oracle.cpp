// nbx_poisson_oracle.cpp -- host build of the shared Poisson sampler
// (paper_2205_07976_b200/csrc/nbx_poisson.h).  TEST INFRASTRUCTURE ONLY: the
// device kernel must reproduce these bits exactly.  Compiled
// with -ffp-contract=off so no FMA can creep into the host arithmetic.
#include <cstdint>

#include "../paper_2205_07976_b200/csrc/nbx_poisson.h"

extern "C" int oracle_poisson(const void* mean, void* out, int64_t n, int dtype, uint64_t seed, uint64_t image) {
    if (dtype != 0 && dtype != 1) return 1;
    for (int64_t p = 0; p < n; ++p) {
        const double mu = dtype ? static_cast<const double*>(mean)[p] : (double)static_cast<const float*>(mean)[p];
        const double k = nbx::poisson_draw(mu, seed, image, (uint64_t)p);
        if (dtype)
            static_cast<double*>(out)[p] = k;
        else
            static_cast<float*>(out)[p] = (float)k;
    }
    return 0;
}
