// Synthetic BASELINE.json config tensors generated directly in HBM.
//
// The generator is counter-addressable (CounterRng of the reference,
// include/rank1/rng.hpp:10-37, with the Box-Muller pairing of
// src/generators.cpp:11-24), so each rank of a sharded run can produce any
// contiguous slab of the global tensor on its own GPU.  Definitions (reference
// dims = config dims reversed, column-major):
//   cfg 1  gen_gaussian(dims, seed)                       N(0,1), stream 1
//   cfg 2  10 u0 o u1 o u2 + 0.01/sqrt(N) N(0,1)          planted, streams 100+k
//   cfg 3  2 U[0,1) - 1                                   stream 1
//   cfg 4  5 o_k u_k + z/||z||_F, z = N(0,1)              planted, streams 100+k
//   cfg 5  sum_r w_r sin((r+1)pi i/Ii) cos(r pi j/Ij) exp(-r k/Ik) + 1e-3 N(0,1)
// Device transcendental functions differ from glibc in the last bit, so the
// device tensor equals the host oracle's (oracle/rank1_oracle.c) only to
// ~1 ulp per entry; parity tests upload host-generated inputs instead.
#include "common.cuh"

#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

namespace r1 {

namespace {

constexpr uint64_t kGolden = 0x9e3779b97f4a7c15ull;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z ^= z >> 30;
    z *= 0xbf58476d1ce4e5b9ull;
    z ^= z >> 27;
    z *= 0x94d049bb133111ebull;
    z ^= z >> 31;
    return z;
}

__host__ __device__ __forceinline__ uint64_t rng_key(uint64_t seed, uint64_t stream) {
    return mix64(seed + kGolden * (stream + 1));
}

__host__ __device__ __forceinline__ double draw_unit(uint64_t key, uint64_t c) {
    return static_cast<double>(mix64(key + kGolden * c) >> 11) * 0x1.0p-53;
}

__host__ __device__ __forceinline__ double draw_gauss(uint64_t key, uint64_t p) {
    const uint64_t k = p >> 1;
    const double u1 = draw_unit(key, 2 * k + 1) + 0x1.0p-54;
    const double u2 = draw_unit(key, 2 * k + 2);
    const double r = sqrt(-2.0 * log(u1));
    const double a = 2.0 * 3.14159265358979323846 * u2;
    return (p & 1) ? r * sin(a) : r * cos(a);
}

struct GenArgs {
    int cfg;
    int order;
    uint64_t dims[16];  // global reference dims
    uint64_t first;     // global linear index of element 0 of the slab
    uint64_t count;
    uint64_t key;       // tensor stream key
    double weight, noise;
    const double* fac[16];  // planted factors (cfg 2/4)
    const double* tab;      // cfg 5: sin/cos/exp tables (3*(Ii+Ij+Ik))
    double* out;
};

__global__ void gen_kernel(const GenArgs a) {
    for (uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; t < a.count;
         t += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t p = a.first + t;
        double v;
        if (a.cfg == 1) {
            v = draw_gauss(a.key, p);
        } else if (a.cfg == 3) {
            v = 2.0 * draw_unit(a.key, p + 1) - 1.0;
        } else if (a.cfg == 2 || a.cfg == 4) {
            uint64_t q = p;
            double prod = 1.0;
            for (int k = 0; k < a.order; ++k) {
                prod *= a.fac[k][q % a.dims[k]];
                q /= a.dims[k];
            }
            v = a.weight * prod + a.noise * draw_gauss(a.key, p);
        } else {
            const uint64_t Ik = a.dims[0], Ij = a.dims[1], Ii = a.dims[2];
            const uint64_t k = p % Ik, j = (p / Ik) % Ij, i = p / (Ik * Ij);
            const double* si = a.tab;
            const double* cj = a.tab + 3 * Ii;
            const double* ek = cj + 3 * Ij;
            const double w[3] = {3.0, 1.0, 0.5};
            double s = 0.0;
            for (int r = 0; r < 3; ++r) s += w[r] * si[r * Ii + i] * cj[r * Ij + j] * ek[r * Ik + k];
            v = s + 1e-3 * draw_gauss(a.key, p);
        }
        a.out[t] = v;
    }
}

// sum of z^2 over the global tensor, z = N(0,1) on the tensor stream (cfg 4)
__global__ void noise_sumsq_kernel(uint64_t key, uint64_t n, double* part) {
    __shared__ double sh[32];
    double s = 0.0;
    for (uint64_t p = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; p < n;
         p += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const double z = draw_gauss(key, p);
        s = fma(z, z, s);
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) t += sh[w];
        part[blockIdx.x] = t;
    }
}

std::vector<double> planted_factor(uint64_t seed, int k, uint64_t len) {
    const uint64_t key = rng_key(seed, 100 + static_cast<uint64_t>(k));
    std::vector<double> u(len);
    for (uint64_t i = 0; i < len; ++i) u[i] = draw_gauss(key, i);
    double s = 0.0;
    for (double v : u) s += v * v;
    const double nrm = std::sqrt(s);
    if (nrm > 0.0)
        for (double& v : u) v /= nrm;
    return u;
}

// The reference's named generators (generators.cpp:50-116), 1-based multi-
// indices in layout order.  exp / arcsin take their transcendental values from
// host tables (std::exp / std::asin of the same arguments) and add them in the
// reference's order without contraction: bit-identical.  tan and gaussian
// evaluate tan / log / cos on the device (last-ulp differences from glibc).
struct NamedArgs {
    int kind;  // 0 gaussian, 1 exp, 2 arcsin, 3 tan
    int order;
    uint64_t dims[16];
    uint64_t count;
    uint64_t key;
    const double* tab;  // exp: exp(-k), k = 0..maxdim; arcsin: asin table [j][idx]
    uint64_t tab_stride;
    double* out;
};

__global__ void named_gen_kernel(const NamedArgs a) {
    for (uint64_t p = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; p < a.count;
         p += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        double v = 0.0;
        if (a.kind == 0) {
            v = draw_gauss(a.key, p);
        } else {
            uint64_t q = p;
            bool zero = false;
            for (int j = 1; j <= a.order; ++j) {
                const uint64_t idx = q % a.dims[j - 1] + 1;
                q /= a.dims[j - 1];
                const double sgn = ((j + 1) % 2 == 0) ? 1.0 : -1.0;
                if (a.kind == 1) {
                    v = __dadd_rn(v, __dmul_rn(sgn * static_cast<double>(j), a.tab[idx]));
                } else if (a.kind == 2) {
                    if (idx < static_cast<uint64_t>(j)) zero = true;
                    else v = __dadd_rn(v, a.tab[(j - 1) * a.tab_stride + idx]);
                } else {
                    v = __dadd_rn(v, __ddiv_rn(sgn * static_cast<double>(idx), static_cast<double>(j)));
                }
            }
            if (a.kind == 2 && zero) v = 0.0;
            if (a.kind == 3) v = tan(v);
        }
        a.out[p] = v;
    }
}

}  // namespace

}  // namespace r1

using namespace r1;

extern "C" {

// Fill `t` with elements [first, first + numel(t)) of the global config tensor
// `cfg` of reference dims `global_dims` (a contiguous slab when t's dims are
// the global dims with a shorter last mode).
int r1_generate_config(r1_context* ctx, r1_tensor* t, int cfg, uint64_t seed,
                       const uint64_t* global_dims, int order, uint64_t first) {
    return abi_guard([&] {
        CtxLock lk_(ctx);
        if (!ctx || !t) fail(R1_ERR_INVALID_ARGUMENT, "null argument");
        R1_CUDA(cudaSetDevice(ctx->device));
        if (cfg < 1 || cfg > 5) fail(R1_ERR_INVALID_ARGUMENT, "unknown config");
        if ((cfg == 2 || cfg == 5) && order != 3) fail(R1_ERR_INVALID_ARGUMENT, "config needs order 3");
        GenArgs a{};
        a.cfg = cfg;
        a.order = order;
        uint64_t n = 1;
        for (int k = 0; k < order; ++k) {
            a.dims[k] = global_dims[k];
            n *= global_dims[k];
        }
        if (first + t->numel > n) fail(R1_ERR_INVALID_ARGUMENT, "slab outside the global tensor");
        a.first = first;
        a.count = t->numel;
        a.key = rng_key(seed, 1);
        a.out = t->dev;
        DeviceBuffer facbuf, tab, part;
        if (cfg == 2 || cfg == 4) {
            uint64_t tot = 0;
            for (int k = 0; k < order; ++k) tot += global_dims[k];
            std::vector<double> all;
            for (int k = 0; k < order; ++k) {
                auto u = planted_factor(seed, k, global_dims[k]);
                all.insert(all.end(), u.begin(), u.end());
            }
            facbuf.ensure(tot * sizeof(double));
            upload_now(ctx, facbuf.ptr, all.data(), tot * sizeof(double));
            uint64_t off = 0;
            for (int k = 0; k < order; ++k) {
                a.fac[k] = facbuf.as<double>() + off;
                off += global_dims[k];
            }
            if (cfg == 2) {
                a.weight = 10.0;
                a.noise = 0.01 / std::sqrt(static_cast<double>(n));
            } else {
                const int blocks = 4 * ctx->num_sms;
                part.ensure(blocks * sizeof(double));
                noise_sumsq_kernel<<<blocks, 256, 0, ctx->stream>>>(a.key, n, part.as<double>());
                check_launch(ctx, "noise_sumsq_kernel");
                std::vector<double> h(blocks);
                R1_CUDA(cudaMemcpyAsync(h.data(), part.ptr, blocks * sizeof(double),
                                        cudaMemcpyDeviceToHost, ctx->stream));
                R1_CUDA(cudaStreamSynchronize(ctx->stream));
                double s = 0.0;
                for (double v : h) s += v;
                a.weight = 5.0;
                a.noise = 1.0 / std::sqrt(s);
            }
        }
        if (cfg == 5) {
            const uint64_t Ik = global_dims[0], Ij = global_dims[1], Ii = global_dims[2];
            const double PI = 3.14159265358979323846;
            std::vector<double> h(3 * (Ii + Ij + Ik));
            double* si = h.data();
            double* cj = si + 3 * Ii;
            double* ek = cj + 3 * Ij;
            for (int r = 1; r <= 3; ++r) {
                for (uint64_t i = 0; i < Ii; ++i)
                    si[(r - 1) * Ii + i] = std::sin((r + 1) * PI * static_cast<double>(i) / Ii);
                for (uint64_t j = 0; j < Ij; ++j)
                    cj[(r - 1) * Ij + j] = std::cos(r * PI * static_cast<double>(j) / Ij);
                for (uint64_t k = 0; k < Ik; ++k)
                    ek[(r - 1) * Ik + k] = std::exp(-static_cast<double>(r) * k / Ik);
            }
            tab.ensure(h.size() * sizeof(double));
            upload_now(ctx, tab.ptr, h.data(), h.size() * sizeof(double));
            a.tab = tab.as<double>();
        }
        const int g = 8 * ctx->num_sms;
        gen_kernel<<<g, 256, 0, ctx->stream>>>(a);
        check_launch(ctx, "gen_kernel");
        R1_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

// generate(name, dims, seed) (generators.cpp:109-116) into `t` (its dims are
// the tensor's dims): "gaussian" | "exp" | "arcsin" | "tan".
int r1_generate(r1_context* ctx, r1_tensor* t, const char* name, uint64_t seed) {
    return abi_guard([&] {
        CtxLock lk_(ctx);
        if (!ctx || !t || !name) fail(R1_ERR_INVALID_ARGUMENT, "null argument");
        R1_CUDA(cudaSetDevice(ctx->device));
        const std::string nm(name);
        NamedArgs a{};
        a.kind = nm == "gaussian" ? 0 : nm == "exp" ? 1 : nm == "arcsin" ? 2 : nm == "tan" ? 3 : -1;
        if (a.kind < 0) fail(R1_ERR_INVALID_ARGUMENT, "unknown generator: " + nm);
        a.order = static_cast<int>(t->dims.size());
        if (a.order < 2) fail(R1_ERR_INVALID_ARGUMENT, "generator: tensor order must be >= 2");
        uint64_t maxd = 0;
        for (int k = 0; k < a.order; ++k) {
            a.dims[k] = t->dims[k];
            maxd = std::max<uint64_t>(maxd, t->dims[k]);
        }
        a.count = t->numel;
        a.key = rng_key(seed, 1);
        a.out = t->dev;
        DeviceBuffer tab;
        std::vector<double> h;
        if (a.kind == 1) {
            h.resize(maxd + 1);
            for (uint64_t k = 0; k <= maxd; ++k) h[k] = std::exp(-static_cast<double>(k));
        } else if (a.kind == 2) {
            a.tab_stride = maxd + 1;
            h.assign(static_cast<size_t>(a.order) * a.tab_stride, 0.0);
            for (int j = 1; j <= a.order; ++j)
                for (uint64_t idx = static_cast<uint64_t>(j); idx <= maxd; ++idx) {
                    const double sgn = (idx % 2 == 0) ? 1.0 : -1.0;
                    h[(j - 1) * a.tab_stride + idx] =
                        std::asin(sgn * static_cast<double>(j) / static_cast<double>(idx));
                }
        }
        if (!h.empty()) {
            tab.ensure(h.size() * sizeof(double));
            upload_now(ctx, tab.ptr, h.data(), h.size() * sizeof(double));
            a.tab = tab.as<double>();
        }
        named_gen_kernel<<<8 * ctx->num_sms, 256, 0, ctx->stream>>>(a);
        check_launch(ctx, "named_gen_kernel");
        R1_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

}  // extern "C"
