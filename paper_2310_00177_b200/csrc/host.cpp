// Host-side deterministic inputs for the C ABI: the reference's Rng
// (include/npsd/rng.hpp:13-50) and init_params (src/net_params.cpp:11-35),
// generalised to 3D (fan-ins 2187 / 81; same draw order), plus the
// identity-equivalent weights of SURVEY.md §0.4. Compiled with
// -ffp-contract=off so the f64 arithmetic matches the reference build.
#include <cstdio>
#include <string>
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

// save_npm / load_npm (net_params.cpp:42-78); the f32 payload is written and
// read as raw little-endian floats like the reference's fwrite/fread.
static thread_local std::string g_npm_error;

const char* npsd_b200_npm_last_error(void) { return g_npm_error.c_str(); }

int npsd_b200_save_npm(const char* path, int dim, int depth, const float* params, size_t n) {
    if (!path || (dim != 2 && dim != 3) || depth < 1 || !params || n != npsd_b200_param_count(dim, depth)) {
        g_npm_error = "save_npm: bad arguments";
        return NPSD_INVALID_ARGUMENT;
    }
    std::FILE* f = std::fopen(path, "wb");
    if (!f) {
        g_npm_error = std::string("save_npm: cannot open ") + path;
        return NPSD_IO_ERROR;
    }
    static const char magic[4] = {'N', 'P', 'M', 'W'};
    const uint32_t header[3] = {1u, static_cast<uint32_t>(dim), static_cast<uint32_t>(depth)};
    bool ok = std::fwrite(magic, 1, 4, f) == 4;
    ok = ok && std::fwrite(header, sizeof(uint32_t), 3, f) == 3;
    ok = ok && std::fwrite(params, sizeof(float), n, f) == n;
    ok = (std::fclose(f) == 0) && ok;
    if (!ok) {
        g_npm_error = std::string("save_npm: cannot write ") + path;
        return NPSD_IO_ERROR;
    }
    return NPSD_OK;
}

int npsd_b200_load_npm(const char* path, int* dim, int* depth, float* out, size_t cap, size_t* n_out) {
    if (!path) {
        g_npm_error = "load_npm: bad arguments";
        return NPSD_INVALID_ARGUMENT;
    }
    std::FILE* f = std::fopen(path, "rb");
    if (!f) {
        g_npm_error = std::string("load_npm: cannot open ") + path;
        return NPSD_IO_ERROR;
    }
    char magic[4];
    uint32_t header[3];
    if (std::fread(magic, 1, 4, f) != 4 || std::memcmp(magic, "NPMW", 4) != 0 ||
        std::fread(header, sizeof(uint32_t), 3, f) != 3) {
        std::fclose(f);
        g_npm_error = std::string("load_npm: bad header in ") + path;
        return NPSD_IO_ERROR;
    }
    if (header[0] != 1u || (header[1] != 2u && header[1] != 3u) || header[2] < 1u || header[2] > 64u) {
        std::fclose(f);
        g_npm_error = std::string("load_npm: unsupported version/dim/depth in ") + path;
        return NPSD_IO_ERROR;
    }
    const int d = static_cast<int>(header[1]), L = static_cast<int>(header[2]);
    const size_t n = npsd_b200_param_count(d, L);
    if (dim) *dim = d;
    if (depth) *depth = L;
    if (n_out) *n_out = n;
    if (!out) {
        std::fclose(f);
        return NPSD_OK;
    }
    if (cap < n) {
        std::fclose(f);
        g_npm_error = "load_npm: output buffer too small";
        return NPSD_INVALID_ARGUMENT;
    }
    const bool ok = std::fread(out, sizeof(float), n, f) == n;
    std::fclose(f);
    if (!ok) {
        g_npm_error = std::string("load_npm: truncated parameter data in ") + path;
        return NPSD_IO_ERROR;
    }
    return NPSD_OK;
}

}  // extern "C"
