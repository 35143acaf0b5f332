// ORACLE / TEST INFRASTRUCTURE — not product code.
//
// C-ABI shim over the UNMODIFIED reference library (proj/src/*.cpp of
// /root/reference), compiled with -Drank1=rank1_ref by oracle/Makefile into
// oracle/_ref/librank1_ref.so.  Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference leg load it, as the checker or as
// the timed CPU baseline — never as the thing measured or shipped.
//
// Every entry point converts plain pointers into the reference's own types,
// calls the reference's public API, and converts the result back.  Exceptions
// become status codes (same codes as include/rank1_b200.h).

#include <chrono>
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include "rank1/experiment.hpp"
#include "rank1/generators.hpp"
#include "rank1/greedy.hpp"
#include "rank1/nepv.hpp"
#include "rank1/rng.hpp"
#include "rank1/solvers.hpp"
#include "rank1/stacked.hpp"
#include "rank1/sym_eig.hpp"
#include "rank1/tensor.hpp"
#include "rank1/tensor_io.hpp"
#include "rank1_b200.h"

#ifdef _OPENMP
#include <omp.h>
#endif

using namespace rank1;  // expands to rank1_ref under -Drank1=rank1_ref

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return R1_OK;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return R1_ERR_INVALID_ARGUMENT;
    } catch (const std::runtime_error& e) {
        g_err = e.what();
        return R1_ERR_RUNTIME;
    } catch (const std::exception& e) {
        g_err = e.what();
        return R1_ERR_INTERNAL;
    }
}

std::vector<std::size_t> to_dims(const uint64_t* dims, int order) {
    return std::vector<std::size_t>(dims, dims + order);
}

std::size_t numel(const std::vector<std::size_t>& d) {
    std::size_t n = 1;
    for (auto v : d) n *= v;
    return n;
}

DenseTensor make_tensor(const double* a, const uint64_t* dims, int order) {
    auto d = to_dims(dims, order);
    const std::size_t n = numel(d);
    return DenseTensor(d, std::vector<double>(a, a + n));
}

FactorSet make_factors(const double* flat, const uint64_t* dims, int order) {
    FactorSet f;
    f.factors.resize(order);
    std::size_t off = 0;
    for (int k = 0; k < order; ++k) {
        f.factors[k].assign(flat + off, flat + off + dims[k]);
        off += dims[k];
    }
    return f;
}

void write_blocks(const SymBlockMatrix& j, double* out) {
    const std::size_t d = j.order();
    std::size_t off = 0;
    for (std::size_t m = 0; m < d; ++m)
        for (std::size_t n = m + 1; n < d; ++n) {
            const Matrix& b = j.block(m, n);
            std::memcpy(out + off, b.data(), sizeof(double) * b.rows() * b.cols());
            off += b.rows() * b.cols();
        }
}

SymBlockMatrix read_blocks(const uint64_t* dims, int order, const double* blocks) {
    SymBlockMatrix j(to_dims(dims, order));
    std::size_t off = 0;
    for (int m = 0; m < order; ++m)
        for (int n = m + 1; n < order; ++n) {
            Matrix& b = j.block(m, n);
            std::memcpy(b.data(), blocks + off, sizeof(double) * b.rows() * b.cols());
            off += b.rows() * b.cols();
        }
    return j;
}

Matrix make_matrix(int64_t n, const double* s) {
    return Matrix(n, n, std::vector<double>(s, s + n * n));
}

SolveOptions make_opts(const r1_solve_options* o, const uint64_t* dims, int order) {
    SolveOptions s;
    s.tol = o->tol;
    s.max_iters = o->max_iters;
    s.seed = o->seed;
    s.init = o->init == R1_INIT_PROVIDED ? InitKind::provided : InitKind::uniform01;
    if (o->init == R1_INIT_PROVIDED && o->init_factors)
        s.init_factors = make_factors(o->init_factors, dims, order).factors;
    s.determinism = o->determinism != 0;
    s.rqi_accept_rule =
        o->rqi_accept_rule == R1_RQI_SIGNED_INCREASE ? RqiAcceptRule::signed_increase
                                                     : RqiAcceptRule::magnitude;
    s.stop_rule = o->stop_rule == R1_STOP_EQ11
                      ? StopRule::eq11
                      : (o->stop_rule == R1_STOP_LAMBDA_DELTA ? StopRule::lambda_delta
                                                              : StopRule::kkt);
    s.threads = o->threads;
    s.record_kkt = o->record_kkt != 0;
    s.asvd_disjoint_pairs = o->asvd_disjoint_pairs != 0;
    s.reuse_intermediates = o->reuse_intermediates != 0;
    return s;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

// rank1::build_j / build_j_serial (nepv.cpp:199-247).  mode: 0 build_j, 1 serial.
int ref_build_j(const double* a, const uint64_t* dims, int order, const double* factors,
                int mode, int threads, int determinism, int reuse, double* blocks_out,
                double* seconds_out) {
    return guarded([&] {
        DenseTensor t = make_tensor(a, dims, order);
        FactorSet f = make_factors(factors, dims, order);
        BuildOptions bo;
        bo.threads = threads;
        bo.determinism = determinism != 0;
        bo.reuse_intermediates = reuse != 0;
        auto t0 = std::chrono::steady_clock::now();
        SymBlockMatrix j = mode == 1 ? build_j_serial(t, f) : build_j(t, f, bo);
        auto t1 = std::chrono::steady_clock::now();
        if (seconds_out) *seconds_out = std::chrono::duration<double>(t1 - t0).count();
        write_blocks(j, blocks_out);
    });
}

// Timing helper for the CPU baseline: the tensor is materialised ONCE (the copy
// into the reference's DenseTensor is not timed) and build_j is run `reps`
// times; per-call wall times go to seconds_out[reps].
int ref_time_build_j(const double* a, const uint64_t* dims, int order, const double* factors,
                     int threads, int determinism, int reps, double* blocks_out,
                     double* seconds_out) {
    return guarded([&] {
        DenseTensor t = make_tensor(a, dims, order);
        FactorSet f = make_factors(factors, dims, order);
        BuildOptions bo;
        bo.threads = threads;
        bo.determinism = determinism != 0;
        for (int r = 0; r < reps; ++r) {
            auto t0 = std::chrono::steady_clock::now();
            SymBlockMatrix j = build_j(t, f, bo);
            auto t1 = std::chrono::steady_clock::now();
            seconds_out[r] = std::chrono::duration<double>(t1 - t0).count();
            if (r == reps - 1 && blocks_out) write_blocks(j, blocks_out);
        }
    });
}

// A reference DenseTensor kept alive across calls (bench.py's CPU arms): the
// reference allocates it and `fill` writes the entries in place, so a 32 GB
// config exists once in host memory and is generated once.
typedef void (*ref_fill_fn)(double* out, uint64_t n, void* user);
int ref_tensor_new(ref_fill_fn fill, void* user, const uint64_t* dims, int order, void** out) {
    return guarded([&] {
        auto* t = new DenseTensor(to_dims(dims, order));
        fill(t->data(), t->size(), user);
        *out = t;
    });
}

int ref_tensor_free(void* t) {
    delete static_cast<DenseTensor*>(t);
    return 0;
}

double* ref_tensor_data(void* t) { return static_cast<DenseTensor*>(t)->data(); }

int ref_time_build_j_t(void* tp, const double* factors, int threads, int determinism, int reps,
                       double* blocks_out, double* seconds_out) {
    return guarded([&] {
        const DenseTensor& t = *static_cast<DenseTensor*>(tp);
        std::vector<uint64_t> dims(t.dims().begin(), t.dims().end());
        FactorSet f = make_factors(factors, dims.data(), static_cast<int>(dims.size()));
        BuildOptions bo;
        bo.threads = threads;
        bo.determinism = determinism != 0;
        for (int r = 0; r < reps; ++r) {
            auto t0 = std::chrono::steady_clock::now();
            SymBlockMatrix j = build_j(t, f, bo);
            auto t1 = std::chrono::steady_clock::now();
            seconds_out[r] = std::chrono::duration<double>(t1 - t0).count();
            if (r == reps - 1 && blocks_out) write_blocks(j, blocks_out);
        }
    });
}

int ref_build_block(const double* a, const uint64_t* dims, int order, const double* factors,
                    int m, int n, double* out) {
    return guarded([&] {
        DenseTensor t = make_tensor(a, dims, order);
        FactorSet f = make_factors(factors, dims, order);
        Matrix b = build_block(t, f, static_cast<std::size_t>(m), static_cast<std::size_t>(n));
        std::memcpy(out, b.data(), sizeof(double) * b.rows() * b.cols());
    });
}

int ref_multilinear_value(const double* a, const uint64_t* dims, int order,
                          const double* factors, double* out) {
    return guarded([&] {
        DenseTensor t = make_tensor(a, dims, order);
        FactorSet f = make_factors(factors, dims, order);
        *out = multilinear_value(t, f);
    });
}

// out: [lambda, max_residual, r_0..r_{d-1}]
int ref_kkt_report(const double* a, const uint64_t* dims, int order, const double* factors,
                   double* out) {
    return guarded([&] {
        DenseTensor t = make_tensor(a, dims, order);
        FactorSet f = make_factors(factors, dims, order);
        KktReport r = kkt_report(t, f);
        out[0] = r.lambda;
        out[1] = r.max_residual;
        for (int k = 0; k < order; ++k) out[2 + k] = r.per_mode_residuals[k];
    });
}

int ref_block_matvec(const uint64_t* dims, int order, const double* blocks, const double* x,
                     double* y) {
    return guarded([&] {
        SymBlockMatrix j = read_blocks(dims, order, blocks);
        auto v = j.matvec(std::span<const double>(x, j.total_dim()));
        std::memcpy(y, v.data(), sizeof(double) * v.size());
    });
}

int ref_block_frobenius(const uint64_t* dims, int order, const double* blocks, double* out) {
    return guarded([&] { *out = read_blocks(dims, order, blocks).frobenius_norm(); });
}

int ref_block_dense(const uint64_t* dims, int order, const double* blocks, double* out) {
    return guarded([&] {
        Matrix d = read_blocks(dims, order, blocks).dense();
        std::memcpy(out, d.data(), sizeof(double) * d.rows() * d.cols());
    });
}

int ref_scf_stopping_value(const uint64_t* dims, int order, const double* blocks,
                           const double* x, double lambda, double* out) {
    return guarded([&] {
        SymBlockMatrix j = read_blocks(dims, order, blocks);
        StackedVector sx(to_dims(dims, order),
                         std::vector<double>(x, x + j.total_dim()));
        *out = scf_stopping_value(j, sx, lambda);
    });
}

int ref_sym_eig_full(int64_t n, const double* s, double* values, double* vectors) {
    return guarded([&] {
        EigDecomposition d = sym_eig_full(make_matrix(n, s));
        std::memcpy(values, d.values.data(), sizeof(double) * n);
        std::memcpy(vectors, d.vectors.data(), sizeof(double) * n * n);
    });
}

int ref_largest_magnitude_eigenpair(int64_t n, const double* s, double* value, double* vec) {
    return guarded([&] {
        EigPair p = largest_magnitude_eigenpair(make_matrix(n, s));
        *value = p.value;
        std::memcpy(vec, p.vector.data(), sizeof(double) * n);
    });
}

int ref_rayleigh_quotient_step(int64_t n, const double* s, const double* x, double* y,
                               int* accepted) {
    return guarded([&] {
        auto r = rayleigh_quotient_step(make_matrix(n, s), std::span<const double>(x, n));
        *accepted = r.has_value() ? 1 : 0;
        if (r) std::memcpy(y, r->data(), sizeof(double) * n);
    });
}

// Bunch-Kaufman factors: w (n*n), ipiv (n), singular flag and diag condition.
int ref_ldlt(int64_t n, const double* s, double* w, int* ipiv, int* singular, double* cond) {
    return guarded([&] {
        auto f = detail::ldlt_factor(make_matrix(n, s));
        std::memcpy(w, f.w.data(), sizeof(double) * n * n);
        for (int64_t i = 0; i < n; ++i) ipiv[i] = f.ipiv[i];
        *singular = f.singular ? 1 : 0;
        *cond = detail::ldlt_diag_condition(f);
    });
}

int ref_ldlt_solve(int64_t n, const double* s, const double* b, double* x) {
    return guarded([&] {
        auto f = detail::ldlt_factor(make_matrix(n, s));
        auto r = detail::ldlt_solve(f, std::vector<double>(b, b + n));
        std::memcpy(x, r.data(), sizeof(double) * n);
    });
}

int ref_split_factors(const uint64_t* dims, int order, const double* x, double* factors,
                      uint8_t* degenerate) {
    return guarded([&] {
        auto d = to_dims(dims, order);
        std::size_t tot = 0;
        for (auto v : d) tot += v;
        StackedVector sx(d, std::vector<double>(x, x + tot));
        SplitResult r = split_factors(sx);
        std::size_t off = 0;
        for (int k = 0; k < order; ++k) {
            std::memcpy(factors + off, r.factors.factors[k].data(), sizeof(double) * d[k]);
            off += d[k];
            degenerate[k] = r.degenerate[k];
        }
    });
}

int ref_stack_factors(const uint64_t* dims, int order, const double* factors, double* x) {
    return guarded([&] {
        StackedVector s = stack_factors(make_factors(factors, dims, order));
        std::memcpy(x, s.flat().data(), sizeof(double) * s.total_dim());
    });
}

int ref_gen_gaussian(const uint64_t* dims, int order, uint64_t seed, double* out) {
    return guarded([&] {
        DenseTensor t = gen_gaussian(to_dims(dims, order), seed);
        std::memcpy(out, t.data(), sizeof(double) * t.size());
    });
}

int ref_generate(const char* name, const uint64_t* dims, int order, uint64_t seed, double* out) {
    return guarded([&] {
        DenseTensor t = generate(name, to_dims(dims, order), seed);
        std::memcpy(out, t.data(), sizeof(double) * t.size());
    });
}

// CounterRng draws (rng.hpp:10-37): kind 0 = next_u64 (as double bits), 1 = next_unit,
// 2 = next_gaussian.
int ref_rng_draws(uint64_t seed, uint64_t stream, int kind, int64_t count, double* out) {
    return guarded([&] {
        CounterRng rng(seed, stream);
        for (int64_t i = 0; i < count; ++i) {
            if (kind == 0) {
                uint64_t v = rng.next_u64();
                std::memcpy(out + i, &v, sizeof(v));
            } else if (kind == 1) {
                out[i] = rng.next_unit();
            } else {
                out[i] = rng.next_gaussian();
            }
        }
    });
}

// rank1::solve (solvers.cpp:509-517).  report arrays are caller-owned.
static void solve_into(const char* algorithm, const DenseTensor& t, const uint64_t* dims,
                       int order, const r1_solve_options* opts, r1_solve_report* rep) {
    {
        SolveOptions so = make_opts(opts, dims, order);
        auto t0 = std::chrono::steady_clock::now();
        SolveReport r = solve(algorithm, t, so);
        auto t1 = std::chrono::steady_clock::now();
        rep->lambda = r.result.lambda;
        std::size_t off = 0;
        for (int k = 0; k < order; ++k) {
            std::memcpy(rep->factors + off, r.result.factors[k].data(),
                        sizeof(double) * dims[k]);
            off += dims[k];
        }
        rep->converged = r.converged ? 1 : 0;
        rep->iterations = r.iterations;
        rep->lambda0 = r.lambda0;
        rep->restarted = r.restarted ? 1 : 0;
        if (rep->final_x) {
            if (r.final_x.total_dim() == off)
                std::memcpy(rep->final_x, r.final_x.flat().data(), sizeof(double) * off);
            else
                std::memset(rep->final_x, 0, sizeof(double) * off);
        }
        int sweeps = 1;
        for (int i = 0; i < r.iterations; ++i) {
            const IterationRecord& s = r.trace[i];
            r1_iteration_record& d = rep->trace[i];
            d.lambda = s.lambda;
            d.stop_value = s.stop_value;
            d.eq11_value = s.eq11_value;
            d.kkt_max_residual = s.kkt_max_residual;
            d.rqi_accepted = s.rqi_accepted ? 1 : 0;
            d.n_sweeps = 1 + (s.rqi_accepted ? 1 : 0);
            d.lambda_pre_rqi = s.lambda_pre_rqi;
            d.t_build_j = s.t_build_j;
            d.t_eig = s.t_eig;
            d.t_other = s.t_other;
            sweeps += d.n_sweeps;
        }
        rep->total_sweeps = sweeps;
        rep->t_total = std::chrono::duration<double>(t1 - t0).count();
    }
}

int ref_solve(const char* algorithm, const double* a, const uint64_t* dims, int order,
              const r1_solve_options* opts, r1_solve_report* rep) {
    return guarded([&] { solve_into(algorithm, make_tensor(a, dims, order), dims, order, opts, rep); });
}

int ref_solve_t(const char* algorithm, void* tp, const r1_solve_options* opts,
                r1_solve_report* rep) {
    return guarded([&] {
        const DenseTensor& t = *static_cast<DenseTensor*>(tp);
        std::vector<uint64_t> dims(t.dims().begin(), t.dims().end());
        solve_into(algorithm, t, dims.data(), static_cast<int>(dims.size()), opts, rep);
    });
}

// Same, but the tensor is created in the reference's own DenseTensor and filled
// in place by `fill` (no second host copy: config 5 is 32 GB).
int ref_solve_fill(const char* algorithm, ref_fill_fn fill, void* user, const uint64_t* dims,
                   int order, const r1_solve_options* opts, r1_solve_report* rep) {
    return guarded([&] {
        DenseTensor t(to_dims(dims, order));
        fill(t.data(), t.size(), user);
        solve_into(algorithm, t, dims, order, opts, rep);
    });
}

// greedy_rank_r (greedy.cpp:7-35).  Arrays sized r (factors r * sum I_k);
// *nterms = terms solved, *completed, failure text (rep.failure) into `failure`.
int ref_greedy(const char* solver, const double* a, const uint64_t* dims, int order, uint64_t r,
               const r1_solve_options* opts, double* lambdas, double* factors, double* ratios,
               int* iters, int* nterms, int* completed, char* failure, int failure_len) {
    return guarded([&] {
        DenseTensor t = make_tensor(a, dims, order);
        SolveOptions so = make_opts(opts, dims, order);
        GreedyReport g = greedy_rank_r(t, r, solver, so);
        std::size_t sum = 0;
        for (int k = 0; k < order; ++k) sum += dims[k];
        for (std::size_t i = 0; i < g.terms.size(); ++i) {
            lambdas[i] = g.terms[i].lambda;
            std::size_t off = 0;
            for (int k = 0; k < order; ++k) {
                std::memcpy(factors + i * sum + off, g.terms[i].factors[k].data(),
                            sizeof(double) * dims[k]);
                off += dims[k];
            }
            ratios[i] = g.residual_ratios[i];
            iters[i] = g.solves[i].iterations;
        }
        *nterms = static_cast<int>(g.terms.size());
        *completed = g.completed ? 1 : 0;
        std::snprintf(failure, failure_len, "%s", g.failure.c_str());
    });
}

// write_dt1 / read_dt1 (tensor_io.cpp:47-100)
int ref_write_dt1(const char* path, const double* a, const uint64_t* dims, int order) {
    return guarded([&] { write_dt1(path, make_tensor(a, dims, order)); });
}

int ref_read_dt1(const char* path, uint64_t* dims, int* order, double* out, uint64_t cap) {
    return guarded([&] {
        DenseTensor t = read_dt1(path);
        *order = static_cast<int>(t.order());
        for (std::size_t k = 0; k < t.order(); ++k) dims[k] = t.dim(k);
        if (out && t.size() <= cap) std::memcpy(out, t.data(), sizeof(double) * t.size());
    });
}

// run_experiment + experiment_csv(zero_timings=true) + summary_table
// (experiment.cpp:81-193) on a given tensor; algos comma-separated.
int ref_experiment_csv(const char* generator, const double* a, const uint64_t* dims, int order,
                       const char* algos, uint64_t seeds, uint64_t base_seed,
                       const r1_solve_options* opts, char* out, int out_len) {
    return guarded([&] {
        DenseTensor t = make_tensor(a, dims, order);
        ExperimentSpec spec;
        spec.generator = generator;
        spec.seeds = seeds;
        spec.base_seed = base_seed;
        spec.opts = make_opts(opts, dims, order);
        spec.algorithms.clear();
        std::string s(algos), tok;
        for (char c : s + ",") {
            if (c == ',') {
                if (!tok.empty()) spec.algorithms.push_back(tok);
                tok.clear();
            } else {
                tok += c;
            }
        }
        ExperimentResult r = run_experiment(spec, t);
        const std::string text = experiment_csv(r.rows, true) + "\n" + summary_table(r.summaries);
        std::snprintf(out, out_len, "%s", text.c_str());
    });
}

}  // extern "C"
