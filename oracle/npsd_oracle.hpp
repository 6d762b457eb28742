// ============================================================================
// TEST INFRASTRUCTURE — NOT THE PRODUCT.
//
// CPU restatement of the reference hot path (`npsd`, /root/reference/proj) for
// the neural-preconditioned PSDO ("DCDM") Poisson solve, templated on the grid
// dimension D in {2, 3}. Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs may load it, and only as the checker.
//
// Every function cites the reference file:line it restates. The D=2
// instantiation is pinned BITWISE against the real reference (oracle/_ref,
// built from /root/reference sources by oracle/Makefile; fixtures in
// tests/golden/). The D=3 instantiation generalises the 2D network exactly as
// SURVEY.md §8a rows 12-19 freeze it:
//   slots      s = 9(dz+1) + 3(dy+1) + (dx+1)          (params.hpp:19 in 2D)
//   conv W     [slot][channel][dz][dy][dx], B[slot]      (params.hpp:21-24)
//   linear K   [channel][dz][dy][dx] + bias              (params.hpp:25-26)
//   init       uniform(-s, s), s = 1/sqrt(fan-in), same draw order
//              (net_params.cpp:11-35)
//   linear z   bias + (1/(S * n_cells)) * sum_t K[t] F[t] (forward.hpp:78-86)
//   pooling    0.125 * (8-sum in x-fastest order)         (kernels.hpp:279-289)
// One deliberate deviation: the linear-block window sums F are formed exactly
// (f64 sums of dyadic values, then cast to f32) instead of the reference's
// serial f32 sum (kernels.hpp:253-266). The two are identical whenever the f32
// sum is exact (all tested 2D sizes, and 3D up to 256^3); the exact form is
// order-free, so it is the same on any GPU decomposition.
// ============================================================================
#pragma once

#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

namespace npsdo {

using index_t = std::int64_t;
using Vector = std::vector<double>;

enum : std::uint8_t { kFluid = 0, kAir = 1, kSolid = 2 };

// types.hpp:19-32
struct SolverBreakdown : std::runtime_error {
    explicit SolverBreakdown(const std::string& w) : std::runtime_error(w) {}
};
struct EmptySystemError : std::runtime_error {
    explicit EmptySystemError(const std::string& w) : std::runtime_error(w) {}
};
inline void require(bool c, const std::string& m) {
    if (!c) throw std::invalid_argument(m);
}

// rng.hpp:13-50 — std::mt19937_64 is fully specified, so streams are portable.
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

struct Dims {
    index_t nx = 0, ny = 0, nz = 1;
    index_t cells() const { return nx * ny * nz; }
    index_t lin(index_t x, index_t y, index_t z) const { return (z * ny + y) * nx + x; }
};

template <int D>
struct Shape {
    static_assert(D == 2 || D == 3, "D must be 2 or 3");
    static constexpr int S = (D == 3) ? 27 : 9;  // slots == window cells
    static constexpr int WN = S * 3 * S;         // conv W entries (243 / 2187)
    static constexpr int KN = 3 * S;             // linear K entries (27 / 81)
    static constexpr int ZR = (D == 3) ? 1 : 0;  // window half-extent along z
    // window offset of slot s (params.hpp:19 generalised)
    static void off(int s, int& dx, int& dy, int& dz) {
        dx = s % 3 - 1;
        dy = (s / 3) % 3 - 1;
        dz = (D == 3) ? s / 9 - 1 : 0;
    }
};

// ---------------------------------------------------------------- parameters
// params.hpp:28-86
struct Conv {
    std::vector<float> W, B;
};
struct Lin {
    std::vector<float> K;
    float bias = 0.0f;
};
struct Level {
    Conv down, up;
    Lin a, b;
};
struct Params {
    int D = 3, depth = 1;
    std::vector<Level> levels;  // depth - 1
    Conv coarse;
};

inline int slots_of(int D) { return D == 3 ? 27 : 9; }

// params.hpp:57-61 generalised
inline std::size_t param_count(int D, int depth) {
    const std::size_t S = static_cast<std::size_t>(slots_of(D));
    const std::size_t conv = S * 3 * S + S, lin = 3 * S + 1;
    return static_cast<std::size_t>(depth - 1) * (2 * conv + 2 * lin) + conv;
}

inline Params zero_params(int D, int depth) {
    require(D == 2 || D == 3, "params: dim must be 2 or 3");
    require(depth >= 1, "params: depth must be >= 1");
    const int S = slots_of(D);
    Params p;
    p.D = D;
    p.depth = depth;
    auto zc = [&](Conv& c) {
        c.W.assign(static_cast<std::size_t>(S * 3 * S), 0.0f);
        c.B.assign(static_cast<std::size_t>(S), 0.0f);
    };
    auto zl = [&](Lin& l) {
        l.K.assign(static_cast<std::size_t>(3 * S), 0.0f);
        l.bias = 0.0f;
    };
    p.levels.resize(static_cast<std::size_t>(depth - 1));
    for (auto& lv : p.levels) {
        zc(lv.down);
        zc(lv.up);
        zl(lv.a);
        zl(lv.b);
    }
    zc(p.coarse);
    return p;
}

// params.hpp:66-80 (for_each_span order)
template <typename Fn>
void for_each_span(Params& p, Fn&& fn) {
    for (auto& lv : p.levels) {
        fn(lv.down.W.data(), lv.down.W.size());
        fn(lv.down.B.data(), lv.down.B.size());
        fn(lv.up.W.data(), lv.up.W.size());
        fn(lv.up.B.data(), lv.up.B.size());
        fn(lv.a.K.data(), lv.a.K.size());
        fn(&lv.a.bias, std::size_t{1});
        fn(lv.b.K.data(), lv.b.K.size());
        fn(&lv.b.bias, std::size_t{1});
    }
    fn(p.coarse.W.data(), p.coarse.W.size());
    fn(p.coarse.B.data(), p.coarse.B.size());
}

inline Params params_from_flat(int D, int depth, const float* flat, std::size_t n) {
    require(n == param_count(D, depth), "params: flat length mismatch");
    Params p = zero_params(D, depth);
    std::size_t o = 0;
    for_each_span(p, [&](float* dst, std::size_t k) {
        std::memcpy(dst, flat + o, k * sizeof(float));
        o += k;
    });
    return p;
}

inline void params_to_flat(Params p, float* flat) {
    std::size_t o = 0;
    for_each_span(p, [&](float* src, std::size_t k) {
        std::memcpy(flat + o, src, k * sizeof(float));
        o += k;
    });
}

// net_params.cpp:11-35, fan-ins generalised (243 -> S*3*S, 27 -> 3*S)
inline Params init_params(int D, int depth, std::uint64_t seed) {
    Params p = zero_params(D, depth);
    const int S = slots_of(D);
    Rng rng(seed);
    auto fill_conv = [&](Conv& c) {
        const double s = 1.0 / std::sqrt(static_cast<double>(S * 3 * S));
        for (auto& w : c.W) w = static_cast<float>(rng.uniform(-s, s));
        for (auto& b : c.B) b = static_cast<float>(rng.uniform(-s, s));
    };
    auto fill_lin = [&](Lin& c) {
        const double s = 1.0 / std::sqrt(static_cast<double>(3 * S));
        for (auto& k : c.K) k = static_cast<float>(rng.uniform(-s, s));
        c.bias = static_cast<float>(rng.uniform(-s, s));
    };
    for (auto& lv : p.levels) {
        fill_conv(lv.down);
        fill_conv(lv.up);
        fill_lin(lv.a);
        fill_lin(lv.b);
    }
    fill_conv(p.coarse);
    return p;
}

// identity-equivalent weights (all conv W = 0, B = e_center;
// lin_a = bias 1, lin_b = bias 0) make the network return its input.
inline Params identity_params(int D, int depth) {
    Params p = zero_params(D, depth);
    const int c = slots_of(D) / 2;
    for (auto& lv : p.levels) {
        lv.down.B[static_cast<std::size_t>(c)] = 1.0f;
        lv.up.B[static_cast<std::size_t>(c)] = 1.0f;
        lv.a.bias = 1.0f;
        lv.b.bias = 0.0f;
    }
    p.coarse.B[static_cast<std::size_t>(c)] = 1.0f;
    return p;
}

// ------------------------------------------------------------------- images
// kernels.hpp:12-57 — 3 channel planes with a 1-cell solid ring (in z too for D=3).
template <int D>
struct PaddedImage {
    Dims d;
    index_t px = 0, py = 0, pz = 0;
    std::vector<float> data;

    PaddedImage() = default;
    explicit PaddedImage(Dims dd) : d(dd) {
        px = d.nx + 2;
        py = d.ny + 2;
        pz = (D == 3) ? d.nz + 2 : 1;
        data.assign(static_cast<std::size_t>(3 * plane()), 0.0f);
        const index_t zlo = (D == 3) ? -1 : 0, zhi = (D == 3) ? d.nz : 0;
        for (index_t z = zlo; z <= zhi; ++z)
            for (index_t y = -1; y <= d.ny; ++y)
                for (index_t x = -1; x <= d.nx; ++x)
                    if (x == -1 || x == d.nx || y == -1 || y == d.ny ||
                        (D == 3 && (z == -1 || z == d.nz)))
                        at(2, x, y, z) = 1.0f;
    }
    index_t plane() const { return px * py * pz; }
    std::size_t idx(int c, index_t x, index_t y, index_t z) const {
        const index_t zz = (D == 3) ? z + 1 : 0;
        return static_cast<std::size_t>(c * plane() + (zz * py + (y + 1)) * px + (x + 1));
    }
    float& at(int c, index_t x, index_t y, index_t z) { return data[idx(c, x, y, z)]; }
    float at(int c, index_t x, index_t y, index_t z) const { return data[idx(c, x, y, z)]; }

    // kernels.hpp:37-43 (from a one-hot IndicatorImage; here from cell types)
    static PaddedImage from_types(const std::uint8_t* types, Dims dd) {
        PaddedImage out(dd);
        for (index_t z = 0; z < dd.nz; ++z)
            for (index_t y = 0; y < dd.ny; ++y)
                for (index_t x = 0; x < dd.nx; ++x) {
                    const int t = types[dd.lin(x, y, z)];
                    for (int c = 0; c < 3; ++c) out.at(c, x, y, z) = (c == t) ? 1.0f : 0.0f;
                }
        return out;
    }

    // kernels.hpp:46-56 (2D order); 3D appends the z+1 plane in the same order
    PaddedImage pooled() const {
        require(d.nx % 2 == 0 && d.ny % 2 == 0 && (D == 2 || d.nz % 2 == 0),
                "PaddedImage::pooled: odd dims");
        Dims h{d.nx / 2, d.ny / 2, (D == 3) ? d.nz / 2 : 1};
        PaddedImage out(h);
        for (int c = 0; c < 3; ++c)
            for (index_t z = 0; z < h.nz; ++z)
                for (index_t y = 0; y < h.ny; ++y)
                    for (index_t x = 0; x < h.nx; ++x) {
                        if (D == 2) {
                            out.at(c, x, y, 0) =
                                0.25f * (at(c, 2 * x, 2 * y, 0) + at(c, 2 * x + 1, 2 * y, 0) +
                                         at(c, 2 * x, 2 * y + 1, 0) + at(c, 2 * x + 1, 2 * y + 1, 0));
                        } else {
                            out.at(c, x, y, z) =
                                0.125f * (at(c, 2 * x, 2 * y, 2 * z) + at(c, 2 * x + 1, 2 * y, 2 * z) +
                                          at(c, 2 * x, 2 * y + 1, 2 * z) +
                                          at(c, 2 * x + 1, 2 * y + 1, 2 * z) +
                                          at(c, 2 * x, 2 * y, 2 * z + 1) +
                                          at(c, 2 * x + 1, 2 * y, 2 * z + 1) +
                                          at(c, 2 * x, 2 * y + 1, 2 * z + 1) +
                                          at(c, 2 * x + 1, 2 * y + 1, 2 * z + 1));
                        }
                    }
        return out;
    }
};

// ------------------------------------------------------------ conv kernels
// kernels.hpp:121-144 — K(x)[s] = B[s] + sum_{c, window} W[s,c,w] I(c, x+w),
// accumulated in (c, dz, dy, dx) order. Materialised like the reference.
template <int D>
std::vector<float> build_kernels(const Conv& p, const PaddedImage<D>& I) {
    constexpr int S = Shape<D>::S;
    const Dims d = I.d;
    std::vector<float> K(static_cast<std::size_t>(d.cells() * S));
#pragma omp parallel for schedule(static) if (d.cells() > 4096)
    for (index_t z = 0; z < d.nz; ++z)
        for (index_t y = 0; y < d.ny; ++y)
            for (index_t x = 0; x < d.nx; ++x) {
                float* k = K.data() + d.lin(x, y, z) * S;
                for (int s = 0; s < S; ++s) {
                    float acc = p.B[static_cast<std::size_t>(s)];
                    const float* w = p.W.data() + s * 3 * S;
                    for (int c = 0; c < 3; ++c)
                        for (int t = 0; t < S; ++t) {
                            int dx, dy, dz;
                            Shape<D>::off(t, dx, dy, dz);
                            acc += w[c * S + t] * I.at(c, x + dx, y + dy, z + dz);
                        }
                    k[s] = acc;
                }
            }
    return K;
}

// kernels.hpp:147-172 — y(x) = sum_s K(x)[s] xpad(x + off(s)), zero-padded input.
template <int D>
std::vector<float> apply_kernels(const std::vector<float>& K, Dims d, const std::vector<float>& x) {
    constexpr int S = Shape<D>::S;
    std::vector<float> y(static_cast<std::size_t>(d.cells()));
#pragma omp parallel for schedule(static) if (d.cells() > 4096)
    for (index_t z = 0; z < d.nz; ++z)
        for (index_t j = 0; j < d.ny; ++j)
            for (index_t i = 0; i < d.nx; ++i) {
                const float* k = K.data() + d.lin(i, j, z) * S;
                float acc = 0.0f;
                for (int s = 0; s < S; ++s) {
                    int dx, dy, dz;
                    Shape<D>::off(s, dx, dy, dz);
                    const index_t xx = i + dx, yy = j + dy, zz = z + dz;
                    const float v = (xx < 0 || xx >= d.nx || yy < 0 || yy >= d.ny || zz < 0 ||
                                     zz >= d.nz)
                                        ? 0.0f
                                        : x[static_cast<std::size_t>(d.lin(xx, yy, zz))];
                    acc += k[s] * v;
                }
                y[static_cast<std::size_t>(d.lin(i, j, z))] = acc;
            }
    return y;
}

// kernels.hpp:253-266 — F[c, w] = sum over interior cells of I_pad(c, x + w).
// Exact (see header), then rounded once to f32.
template <int D>
void linear_image_sums(const PaddedImage<D>& I, float* F) {
    constexpr int S = Shape<D>::S;
    const Dims d = I.d;
    for (int c = 0; c < 3; ++c)
        for (int t = 0; t < S; ++t) {
            int dx, dy, dz;
            Shape<D>::off(t, dx, dy, dz);
            double acc = 0.0;
            for (index_t z = 0; z < d.nz; ++z)
                for (index_t y = 0; y < d.ny; ++y)
                    for (index_t x = 0; x < d.nx; ++x)
                        acc += static_cast<double>(I.at(c, x + dx, y + dy, z + dz));
            F[c * S + t] = static_cast<float>(acc);
        }
}

// kernels.hpp:279-289 (avg_pool2) generalised
template <int D>
std::vector<float> avg_pool(const std::vector<float>& a, Dims d, Dims& h) {
    require(d.nx % 2 == 0 && d.ny % 2 == 0 && (D == 2 || d.nz % 2 == 0), "avg_pool2: dims must be even");
    h = Dims{d.nx / 2, d.ny / 2, (D == 3) ? d.nz / 2 : 1};
    std::vector<float> out(static_cast<std::size_t>(h.cells()));
    auto A = [&](index_t x, index_t y, index_t z) { return a[static_cast<std::size_t>(d.lin(x, y, z))]; };
    for (index_t z = 0; z < h.nz; ++z)
        for (index_t y = 0; y < h.ny; ++y)
            for (index_t x = 0; x < h.nx; ++x) {
                float v;
                if (D == 2) {
                    v = 0.25f * (A(2 * x, 2 * y, 0) + A(2 * x + 1, 2 * y, 0) + A(2 * x, 2 * y + 1, 0) +
                                 A(2 * x + 1, 2 * y + 1, 0));
                } else {
                    v = 0.125f * (A(2 * x, 2 * y, 2 * z) + A(2 * x + 1, 2 * y, 2 * z) +
                                  A(2 * x, 2 * y + 1, 2 * z) + A(2 * x + 1, 2 * y + 1, 2 * z) +
                                  A(2 * x, 2 * y, 2 * z + 1) + A(2 * x + 1, 2 * y, 2 * z + 1) +
                                  A(2 * x, 2 * y + 1, 2 * z + 1) + A(2 * x + 1, 2 * y + 1, 2 * z + 1));
                }
                out[static_cast<std::size_t>(h.lin(x, y, z))] = v;
            }
    return out;
}

// kernels.hpp:292-304 (upsample2) generalised
template <int D>
std::vector<float> upsample(const std::vector<float>& a, Dims h, Dims f) {
    std::vector<float> out(static_cast<std::size_t>(f.cells()));
    for (index_t z = 0; z < f.nz; ++z)
        for (index_t y = 0; y < f.ny; ++y)
            for (index_t x = 0; x < f.nx; ++x)
                out[static_cast<std::size_t>(f.lin(x, y, z))] =
                    a[static_cast<std::size_t>(h.lin(x / 2, y / 2, (D == 3) ? z / 2 : 0))];
    return out;
}

// ----------------------------------------------------------------- network
// forward.hpp:14-33, 56-129
template <int D>
struct NetContext {
    struct LevelCtx {
        PaddedImage<D> image;
        std::vector<float> K_down, K_up;
        float z_a = 0.0f, z_b = 0.0f;
        float F[Shape<D>::KN] = {};
    };
    int depth = 1;
    Dims d;
    std::vector<LevelCtx> levels;

    // forward.hpp:56-93
    static NetContext build(const Params& params, const std::uint8_t* types, Dims dd) {
        constexpr int S = Shape<D>::S;
        require(params.D == D, "NetContext: params dim mismatch");
        require(params.depth >= 1, "NetContext: depth must be >= 1");
        const index_t div = index_t{1} << params.depth;
        require(dd.nx % div == 0 && dd.ny % div == 0 && (D == 2 || dd.nz % div == 0),
                "NetContext: dims not divisible by 2^depth");
        NetContext ctx;
        ctx.depth = params.depth;
        ctx.d = dd;
        ctx.levels.resize(static_cast<std::size_t>(params.depth));
        PaddedImage<D> img = PaddedImage<D>::from_types(types, dd);
        for (int l = 0; l < params.depth; ++l) {
            LevelCtx& lc = ctx.levels[static_cast<std::size_t>(l)];
            lc.image = std::move(img);
            if (l < params.depth - 1) {
                const Level& lp = params.levels[static_cast<std::size_t>(l)];
                lc.K_down = build_kernels<D>(lp.down, lc.image);
                lc.K_up = build_kernels<D>(lp.up, lc.image);
                linear_image_sums<D>(lc.image, lc.F);
                const float norm = 1.0f / (static_cast<float>(S) * static_cast<float>(lc.image.d.cells()));
                float za = lp.a.bias, zb = lp.b.bias;
                for (int t = 0; t < Shape<D>::KN; ++t) {
                    za += norm * lp.a.K[static_cast<std::size_t>(t)] * lc.F[t];
                    zb += norm * lp.b.K[static_cast<std::size_t>(t)] * lc.F[t];
                }
                lc.z_a = za;
                lc.z_b = zb;
                img = lc.image.pooled();
            } else {
                lc.K_down = build_kernels<D>(params.coarse, lc.image);
            }
        }
        return ctx;
    }

    // forward.hpp:95-129
    std::vector<float> apply(const std::vector<float>& r) const {
        require(static_cast<index_t>(r.size()) == d.cells(), "NetContext::apply: field shape mismatch");
        std::vector<std::vector<float>> y(static_cast<std::size_t>(depth));
        std::vector<Dims> dims(static_cast<std::size_t>(depth));
        std::vector<float> x = r;
        Dims cur = d;
        for (int l = 0; l < depth; ++l) {
            dims[static_cast<std::size_t>(l)] = cur;
            y[static_cast<std::size_t>(l)] = apply_kernels<D>(levels[static_cast<std::size_t>(l)].K_down, cur, x);
            if (l + 1 < depth) {
                Dims h;
                x = avg_pool<D>(y[static_cast<std::size_t>(l)], cur, h);
                cur = h;
            }
        }
        std::vector<float> out = std::move(y[static_cast<std::size_t>(depth) - 1]);
        for (int l = depth - 2; l >= 0; --l) {
            const LevelCtx& lc = levels[static_cast<std::size_t>(l)];
            const Dims f = dims[static_cast<std::size_t>(l)], h = dims[static_cast<std::size_t>(l) + 1];
            const std::vector<float> up = upsample<D>(out, h, f);
            const std::vector<float> u = apply_kernels<D>(lc.K_up, f, up);
            const std::vector<float>& yl = y[static_cast<std::size_t>(l)];
            out.assign(yl.size(), 0.0f);
            for (std::size_t i = 0; i < out.size(); ++i) out[i] = lc.z_a * yl[i] + lc.z_b * u[i];
        }
        return out;
    }
};

// ------------------------------------------------------ discretization/map
// discretization.cpp:5-19 (ReductionMap::from_image): ascending linear order.
struct ReductionMap {
    index_t full_size = 0;
    std::vector<index_t> fluid_indices;
    std::vector<index_t> full_to_reduced;
    index_t reduced_size() const { return static_cast<index_t>(fluid_indices.size()); }
    static ReductionMap from_types(const std::uint8_t* types, Dims d) {
        ReductionMap m;
        m.full_size = d.cells();
        m.full_to_reduced.assign(static_cast<std::size_t>(m.full_size), -1);
        for (index_t i = 0; i < m.full_size; ++i)
            if (types[i] == kFluid) {
                m.full_to_reduced[static_cast<std::size_t>(i)] = m.reduced_size();
                m.fluid_indices.push_back(i);
            }
        return m;
    }
};

// assemble_poisson{,_3d} + reduce + spmv (discretization.cpp:21-160,
// sparse.cpp:100-117), restated matrix-free on the reduced system: row entries
// in ascending column order (z-1, y-1, x-1, diag, x+1, y+1, z+1), fluid
// neighbours only, diagonal = # non-solid in-domain neighbours and dropped
// when 0, each accumulated as `s += v * x[j]` from s = 0.
template <int D>
struct PoissonOp {
    Dims d;
    const std::uint8_t* types = nullptr;
    const ReductionMap* map = nullptr;

    std::uint8_t type_clamped(index_t x, index_t y, index_t z) const {
        if (x < 0 || x >= d.nx || y < 0 || y >= d.ny || z < 0 || z >= d.nz) return kSolid;
        return types[d.lin(x, y, z)];
    }

    void spmv(const Vector& x, Vector& y) const {
        const index_t nf = map->reduced_size();
        require(static_cast<index_t>(x.size()) == nf, "spmv: dimension mismatch");
        y.resize(static_cast<std::size_t>(nf));
#pragma omp parallel for schedule(static) if (nf > 4096)
        for (index_t i = 0; i < nf; ++i) {
            const index_t c = map->fluid_indices[static_cast<std::size_t>(i)];
            const index_t cx = c % d.nx, cy = (c / d.nx) % d.ny, cz = c / (d.nx * d.ny);
            const int NB = (D == 3) ? 6 : 4;
            const int dxs3[6] = {0, 0, -1, 1, 0, 0}, dys3[6] = {0, -1, 0, 0, 1, 0}, dzs3[6] = {-1, 0, 0, 0, 0, 1};
            const int dxs2[4] = {0, -1, 1, 0}, dys2[4] = {-1, 0, 0, 1};
            int diag = 0;
            double s = 0.0;
            double upper_v[3];
            index_t upper_j[3];
            int nu = 0;
            for (int k = 0; k < NB; ++k) {
                const int dx = (D == 3) ? dxs3[k] : dxs2[k];
                const int dy = (D == 3) ? dys3[k] : dys2[k];
                const int dz = (D == 3) ? dzs3[k] : 0;
                const std::uint8_t t = type_clamped(cx + dx, cy + dy, cz + dz);
                if (t == kSolid) continue;
                ++diag;
                if (t == kFluid) {
                    const index_t j = map->full_to_reduced[static_cast<std::size_t>(d.lin(cx + dx, cy + dy, cz + dz))];
                    if (k < NB / 2) {
                        s += -1.0 * x[static_cast<std::size_t>(j)];
                    } else {
                        upper_v[nu] = -1.0;
                        upper_j[nu++] = j;
                    }
                }
            }
            if (diag > 0) s += static_cast<double>(diag) * x[static_cast<std::size_t>(i)];
            for (int k = 0; k < nu; ++k) s += upper_v[k] * x[static_cast<std::size_t>(upper_j[k])];
            y[static_cast<std::size_t>(i)] = s;
        }
    }
};

// ---------------------------------------------------------- vector algebra
// vector_ops.cpp:7-43 (serial f64)
inline double dot(const Vector& a, const Vector& b) {
    require(a.size() == b.size(), "dot: length mismatch");
    double s = 0.0;
    for (std::size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
    return s;
}
inline double norm2(const Vector& a) { return std::sqrt(dot(a, a)); }
inline void axpy_inplace(double a, const Vector& x, Vector& y) {
    for (std::size_t i = 0; i < x.size(); ++i) y[i] += a * x[i];
}
inline void scale_inplace(double a, Vector& x) {
    for (double& v : x) v *= a;
}
inline void mean_project(Vector& x) {
    if (x.empty()) return;
    double s = 0.0;
    for (double v : x) s += v;
    const double m = s / static_cast<double>(x.size());
    for (double& v : x) v -= m;
}

// ----------------------------------------------------------- preconditioner
// precond.hpp:12-29
struct Precond {
    virtual ~Precond() = default;
    virtual void apply(const Vector& r, Vector& z) const = 0;
};
struct IdentityPrecond : Precond {  // precond.cpp:7-10
    void apply(const Vector& r, Vector& z) const override { z = r; }
};

// net_precond.cpp:9-35
template <int D>
struct NeuralPrecond : Precond {
    NetContext<D> ctx;
    const ReductionMap* map;
    NeuralPrecond(const Params& p, const std::uint8_t* types, Dims d, const ReductionMap* m)
        : ctx(NetContext<D>::build(p, types, d)), map(m) {
        require(map->full_size == d.cells(), "NeuralPrecond: map does not match image");
    }
    void apply(const Vector& r, Vector& z) const override {
        require(static_cast<index_t>(r.size()) == map->reduced_size(), "NeuralPrecond::apply: size mismatch");
        const double rnorm = norm2(r);
        z.assign(r.size(), 0.0);
        if (rnorm == 0.0) return;
        std::vector<float> full(static_cast<std::size_t>(ctx.d.cells()), 0.0f);
        const double inv = 1.0 / rnorm;
        for (std::size_t k = 0; k < r.size(); ++k)
            full[static_cast<std::size_t>(map->fluid_indices[k])] = static_cast<float>(r[k] * inv);
        const std::vector<float> out = ctx.apply(full);
        for (std::size_t k = 0; k < z.size(); ++k)
            z[k] = static_cast<double>(out[static_cast<std::size_t>(map->fluid_indices[k])]) * rnorm;
    }
};

// ------------------------------------------------------------------ solver
// solver.hpp:11-42
struct SolveConfig {
    double tol_reduction = 1e-6;
    double tol_abs = 0.0;
    index_t max_iters = 1000;
    int n_ortho = 2;
    bool nullspace_projection = false;
    bool normalize_before_precond = true;
};
struct SolveReport {
    index_t iterations = 0;
    bool converged = false;
    std::vector<double> residual_history;
};

// solver.cpp:189-276 (psdo_solve), operation for operation.
template <typename Op>
SolveReport psdo_solve(const Op& A, const Vector& b_in, const Precond& P, const SolveConfig& cfg,
                       const Vector* x0, Vector& x) {
    const index_t n = A.map->reduced_size();
    require(static_cast<index_t>(b_in.size()) == n, "solve: rhs length mismatch");
    for (double v : b_in) require(std::isfinite(v), "solve: rhs has non-finite entries");
    if (x0) require(static_cast<index_t>(x0->size()) == n, "solve: x0 length mismatch");
    require(cfg.n_ortho >= 0, "psdo: n_ortho must be >= 0");

    SolveReport rep;
    Vector b = b_in;
    x = x0 ? *x0 : Vector(b.size(), 0.0);
    if (cfg.nullspace_projection) {
        mean_project(b);
        mean_project(x);
    }
    Vector r = b, Ax;
    A.spmv(x, Ax);
    axpy_inplace(-1.0, Ax, r);
    if (cfg.nullspace_projection) mean_project(r);
    double rnorm = norm2(r);
    rep.residual_history.push_back(rnorm);
    // solver.cpp:20-26 (stop_threshold)
    require(cfg.tol_reduction > 0.0 && cfg.tol_reduction < 1.0, "SolveConfig: tol_reduction must lie in (0,1)");
    double thr = cfg.tol_reduction * rnorm;
    if (cfg.tol_abs > 0.0) thr = std::max(thr, cfg.tol_abs);
    if (rnorm <= thr) {
        rep.converged = true;
        return rep;
    }
    struct Cached {
        Vector d, Ad;
        double dAd;
    };
    std::vector<Cached> cache;  // oldest first
    Vector d, scaled, Ad;
    for (index_t k = 1; k <= cfg.max_iters; ++k) {
        if (cfg.normalize_before_precond) {
            scaled = r;
            scale_inplace(1.0 / rnorm, scaled);
            P.apply(scaled, d);
        } else {
            P.apply(r, d);
        }
        for (const Cached& c : cache) {
            const double proj = dot(d, c.Ad) / c.dAd;
            axpy_inplace(-proj, c.d, d);
        }
        A.spmv(d, Ad);
        const double dAd = dot(d, Ad);
        if (!(dAd > 0.0) || std::abs(dAd) < 1e-300)
            throw SolverBreakdown("psdo: curvature d'Ad = " + std::to_string(dAd) + " at iteration " +
                                  std::to_string(k));
        const double alpha = dot(r, d) / dAd;
        axpy_inplace(alpha, d, x);
        A.spmv(x, Ax);
        r = b;
        axpy_inplace(-1.0, Ax, r);
        if (cfg.nullspace_projection) mean_project(r);
        rnorm = norm2(r);
        rep.iterations = k;
        rep.residual_history.push_back(rnorm);
        if (cfg.n_ortho > 0) {
            cache.push_back({d, Ad, dAd});
            if (static_cast<int>(cache.size()) > cfg.n_ortho) cache.erase(cache.begin());
        }
        if (rnorm <= thr) {
            rep.converged = true;
            break;
        }
    }
    return rep;
}

}  // namespace npsdo
