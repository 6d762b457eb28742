// Host-side deterministic inputs for the C ABI: the reference's Rng
// (include/npsd/rng.hpp:13-50) and init_params (src/net_params.cpp:11-35),
// generalised to 3D (fan-ins 2187 / 81; same draw order), plus the
// identity-equivalent weights of SURVEY.md §0.4. Compiled with
// -ffp-contract=off so the f64 arithmetic matches the reference build.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <vector>

#include "../../include/npsd_b200.h"

namespace {

class Rng {
public:
    explicit Rng(std::uint64_t seed) : gen_(seed) {}
    double uniform() { return static_cast<double>(gen_() >> 11) * 0x1.0p-53; }
    double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
    double normal() {
        if (have_) {
            have_ = false;
            return cached_;
        }
        double u1 = uniform();
        double u2 = uniform();
        while (u1 <= 0.0) u1 = uniform();
        const double r = std::sqrt(-2.0 * std::log(u1));
        const double th = 2.0 * 3.14159265358979323846 * u2;
        cached_ = r * std::sin(th);
        have_ = true;
        return r * std::cos(th);
    }

private:
    std::mt19937_64 gen_;
    bool have_ = false;
    double cached_ = 0.0;
};

}  // namespace

extern "C" {

int npsd_b200_init_params(int dim, int depth, uint64_t seed, float* out) {
    if ((dim != 2 && dim != 3) || depth < 1 || !out) return NPSD_INVALID_ARGUMENT;
    const int S = (dim == 3) ? 27 : 9;
    const int WN = S * 3 * S, KN = 3 * S;
    Rng rng(seed);
    const double sc = 1.0 / std::sqrt(static_cast<double>(WN));
    const double sl = 1.0 / std::sqrt(static_cast<double>(KN));
    float* p = out;
    auto conv = [&] {
        for (int i = 0; i < WN; ++i) *p++ = static_cast<float>(rng.uniform(-sc, sc));
        for (int i = 0; i < S; ++i) *p++ = static_cast<float>(rng.uniform(-sc, sc));
    };
    auto lin = [&] {
        for (int i = 0; i < KN; ++i) *p++ = static_cast<float>(rng.uniform(-sl, sl));
        *p++ = static_cast<float>(rng.uniform(-sl, sl));
    };
    for (int l = 0; l + 1 < depth; ++l) {
        conv();  // conv_down
        conv();  // conv_up
        lin();   // lin_a
        lin();   // lin_b
    }
    conv();  // coarse
    return NPSD_OK;
}

int npsd_b200_identity_params(int dim, int depth, float* out) {
    if ((dim != 2 && dim != 3) || depth < 1 || !out) return NPSD_INVALID_ARGUMENT;
    const int S = (dim == 3) ? 27 : 9;
    const int WN = S * 3 * S, KN = 3 * S, C = S / 2;
    std::memset(out, 0, npsd_b200_param_count(dim, depth) * sizeof(float));
    float* p = out;
    auto conv = [&] {
        p += WN;
        p[C] = 1.0f;
        p += S;
    };
    for (int l = 0; l + 1 < depth; ++l) {
        conv();
        conv();
        p += KN;
        *p++ = 1.0f;  // lin_a bias
        p += KN;
        *p++ = 0.0f;  // lin_b bias
    }
    conv();
    return NPSD_OK;
}

void npsd_b200_rhs_normal(uint64_t seed, int64_t n, double* out) {
    Rng rng(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = rng.normal();
}

}  // extern "C"
