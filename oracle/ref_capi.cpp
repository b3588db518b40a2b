// ORACLE TEST INFRASTRUCTURE — not product code.
//
// ctypes-callable C entry points over the reference library compiled
// verbatim from /root/reference/proj/core/src (see oracle/Makefile).  Only
// tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg load this.
// Every call below forwards to an unmodified reference routine:
//   ref_create          -> ProductConvolutionOperator ctor   (pc_operator.cpp:26-38), grid = null
//   ref_apply           -> ProductConvolutionOperator::apply (pc_operator.cpp:45-56)
//   ref_apply_adjoint   -> ::apply_adjoint                   (pc_operator.cpp:58-69)
//   ref_entries         -> ::entry                           (pc_operator.cpp:84-96)
//   ref_fft_convolve    -> fft_convolve                      (fft.cpp:145-151)
//   ref_conv_padded_shape -> conv_padded_shape               (fft.cpp:64-70)
//   ref_extend_impulse  -> extend_impulse                    (impulse.cpp:61-89); the counting
//                          function is filled as build_extension_weights does (impulse.cpp:17-41)
//                          from an explicit neighbour list instead of an AdaptiveGrid
//   ref_estimate        -> make_estimator_state + update_samples (adaptivity.cpp:30-37,75-112),
//                          per-leaf eta as eta_for_cells (adaptivity.cpp:114-121) over explicit boxes
//   ref_hmatrix_*       -> assemble_hmatrix / HMatrix::matvec / save_hmatrix / load_hmatrix
//                          (hmatrix.cpp:338-526), compiled verbatim against the Eigen shim
//                          (oracle/shim/Eigen/Dense: Householder QR, one-sided Jacobi SVD)
//   ref_apply_batch_threads -> T concurrent ::apply calls on distinct vectors (apply is pure and
//                          thread-safe, pc_operator.hpp:15-16)
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "pcop/adaptivity.hpp"
#include "pcop/fft.hpp"
#include "pcop/hmatrix.hpp"
#include "pcop/impulse.hpp"
#include "pcop/pc_operator.hpp"

using namespace pcop;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e, int code) {
    g_err = e.what();
    return code;
}

template <typename Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        return 0;
    } catch (const std::invalid_argument& e) {
        return fail(e, 1);
    } catch (const std::logic_error& e) {
        return fail(e, 3);
    } catch (const std::runtime_error& e) {
        return fail(e, 2);
    } catch (const std::exception& e) {
        return fail(e, 4);
    }
}

IndexBox make_box(int dim, const std::int64_t* lo, const std::int64_t* hi) {
    return IndexBox(Point(lo, lo + dim), Point(hi, hi + dim));
}

GridFunction make_field(int dim, const std::int64_t* lo, const std::int64_t* hi, const double* v) {
    GridFunction g(make_box(dim, lo, hi));
    std::memcpy(g.data(), v, static_cast<std::size_t>(g.size()) * sizeof(double));
    return g;
}

struct RefOp {
    int dim;
    ProductConvolutionOperator op;
};

void write_field(const GridFunction& g, std::int64_t* lo, std::int64_t* hi, double* out,
                 std::int64_t cap) {
    for (int i = 0; i < g.dim(); ++i) {
        lo[i] = g.box().lo[static_cast<std::size_t>(i)];
        hi[i] = g.box().hi[static_cast<std::size_t>(i)];
    }
    if (out) {
        if (g.size() > cap) throw std::invalid_argument("ref capi: output capacity too small");
        std::memcpy(out, g.data(), static_cast<std::size_t>(g.size()) * sizeof(double));
    }
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

void* ref_create(int dim, const std::int64_t* dom_lo, const std::int64_t* dom_hi, int r,
                 const std::int64_t* w_lo, const std::int64_t* w_hi, const double* const* w_vals,
                 const std::int64_t* phi_lo, const std::int64_t* phi_hi,
                 const double* const* phi_vals) {
    RefOp* out = nullptr;
    const int rc = guarded([&] {
        std::vector<WeightFunction> ws;
        std::vector<ExtendedImpulse> es;
        for (int k = 0; k < r; ++k) {
            WeightFunction w;
            w.k = k;
            w.values = make_field(dim, w_lo + k * dim, w_hi + k * dim, w_vals[k]);
            ws.push_back(std::move(w));
            ExtendedImpulse e;
            e.k = k;
            e.values = make_field(dim, phi_lo + k * dim, phi_hi + k * dim, phi_vals[k]);
            es.push_back(std::move(e));
        }
        out = new RefOp{dim, ProductConvolutionOperator(make_box(dim, dom_lo, dom_hi), nullptr,
                                                        std::move(ws), std::move(es))};
    });
    return rc == 0 ? out : nullptr;
}

void ref_destroy(void* h) { delete static_cast<RefOp*>(h); }

int ref_apply(void* h, const double* f, double* g) {
    return guarded([&] {
        auto* o = static_cast<RefOp*>(h);
        const auto n = static_cast<Eigen::Index>(o->op.domain().num_points());
        Eigen::VectorXd out = o->op.apply(Eigen::VectorXd(f, n));
        std::memcpy(g, out.data(), static_cast<std::size_t>(out.size()) * sizeof(double));
    });
}

int ref_apply_adjoint(void* h, const double* f, double* g) {
    return guarded([&] {
        auto* o = static_cast<RefOp*>(h);
        const auto n = static_cast<Eigen::Index>(o->op.domain().num_points());
        Eigen::VectorXd out = o->op.apply_adjoint(Eigen::VectorXd(f, n));
        std::memcpy(g, out.data(), static_cast<std::size_t>(out.size()) * sizeof(double));
    });
}

int ref_apply_batch_threads(void* h, int adjoint, int B, const double* F, double* G,
                            int nthreads) {
    auto* o = static_cast<RefOp*>(h);
    const std::int64_t n = o->op.domain().num_points();
    std::vector<int> codes(static_cast<std::size_t>(nthreads), 0);
    std::vector<std::string> msgs(static_cast<std::size_t>(nthreads));
    std::vector<std::thread> pool;
    for (int t = 0; t < nthreads; ++t) {
        pool.emplace_back([&, t] {
            codes[static_cast<std::size_t>(t)] = guarded([&] {
                for (int b = t; b < B; b += nthreads) {
                    Eigen::VectorXd in(F + b * n, static_cast<Eigen::Index>(n));
                    Eigen::VectorXd out = adjoint ? o->op.apply_adjoint(in) : o->op.apply(in);
                    std::memcpy(G + b * n, out.data(), static_cast<std::size_t>(n) * sizeof(double));
                }
            });
            if (codes[static_cast<std::size_t>(t)]) msgs[static_cast<std::size_t>(t)] = g_err;
        });
    }
    for (auto& th : pool) th.join();
    for (int t = 0; t < nthreads; ++t)
        if (codes[static_cast<std::size_t>(t)]) {
            g_err = msgs[static_cast<std::size_t>(t)];
            return codes[static_cast<std::size_t>(t)];
        }
    return 0;
}

int ref_entries(void* h, std::int64_t cnt, const std::int64_t* y, const std::int64_t* x,
                double* out) {
    return guarded([&] {
        auto* o = static_cast<RefOp*>(h);
        const int d = o->dim;
        for (std::int64_t i = 0; i < cnt; ++i)
            out[i] = o->op.entry(Point(y + i * d, y + (i + 1) * d), Point(x + i * d, x + (i + 1) * d));
    });
}

// ProductConvolutionOperator::apply_block (pc_operator.cpp:98-130); f on S, out on T
int ref_apply_block(void* h, const std::int64_t* t_lo, const std::int64_t* t_hi, const std::int64_t* s_lo,
                    const std::int64_t* s_hi, const double* f, int adjoint, double* out) {
    return guarded([&] {
        auto* o = static_cast<RefOp*>(h);
        const int d = o->dim;
        const IndexBox T = make_box(d, t_lo, t_hi), S = make_box(d, s_lo, s_hi);
        GridFunction fs = make_field(d, s_lo, s_hi, f);
        GridFunction g = o->op.apply_block(T, S, fs, adjoint != 0);
        std::memcpy(out, g.data(), static_cast<std::size_t>(g.size()) * sizeof(double));
    });
}

int ref_fft_convolve(int dim, const std::int64_t* psi_lo, const std::int64_t* psi_hi,
                     const double* psi, const std::int64_t* f_lo, const std::int64_t* f_hi,
                     const double* f, std::int64_t* out_lo, std::int64_t* out_hi, double* out,
                     std::int64_t cap) {
    return guarded([&] {
        GridFunction a = psi ? make_field(dim, psi_lo, psi_hi, psi) : GridFunction();
        GridFunction b = make_field(dim, f_lo, f_hi, f);
        write_field(fft_convolve(a, b), out_lo, out_hi, out, cap);
    });
}

int ref_conv_padded_shape(int dim, const std::int64_t* a_lo, const std::int64_t* a_hi,
                          const std::int64_t* b_lo, const std::int64_t* b_hi, int* shape) {
    return guarded([&] {
        auto s = conv_padded_shape(make_box(dim, a_lo, a_hi), make_box(dim, b_lo, b_hi));
        for (int i = 0; i < dim; ++i) shape[i] = s[static_cast<std::size_t>(i)];
    });
}

int ref_extend_impulse(int dim, const std::int64_t* om_lo, const std::int64_t* om_hi, int k,
                       int nnbr, const int* nbr_ids, const std::int64_t* nbr_pts,
                       const std::int64_t* phi_lo, const std::int64_t* phi_hi,
                       const double* const* phi_vals, std::int64_t* out_lo, std::int64_t* out_hi,
                       double* out, std::int64_t cap) {
    return guarded([&] {
        ExtensionWeights w;
        w.k = k;
        w.omega = make_box(dim, om_lo, om_hi);
        for (int i = 0; i < nnbr; ++i) {
            w.nbrs.push_back(nbr_ids[i]);
            w.nbr_points.emplace_back(nbr_pts + i * dim, nbr_pts + (i + 1) * dim);
            if (nbr_ids[i] == k) w.p_k = w.nbr_points.back();
        }
        if (w.p_k.empty()) throw std::invalid_argument("ref_extend_impulse: k not among nbrs");
        // counting function c_k, filled the way build_extension_weights does (impulse.cpp:25-39)
        IndexBox support = shift_neg(w.omega, w.nbr_points.front());
        for (std::size_t i = 1; i < w.nbr_points.size(); ++i)
            support = bounding_box(support, shift_neg(w.omega, w.nbr_points[i]));
        GridFunction counting(support);
        for (std::size_t i = 0; i < w.nbr_points.size(); ++i) {
            if (w.nbrs[i] == k) continue;
            accumulate(counting, GridFunction(shift_neg(w.omega, w.nbr_points[i]), 1.0), 1.0);
        }
        for_each_point(shift_neg(w.omega, w.p_k), [&](const Point& z) { counting.at(z) = 1.0; });
        w.counting = std::move(counting);

        std::vector<GridFunction> phis;
        for (int i = 0; i < nnbr; ++i)
            phis.push_back(make_field(dim, phi_lo + i * dim, phi_hi + i * dim, phi_vals[i]));
        std::vector<const GridFunction*> ptrs;
        for (auto& p : phis) ptrs.push_back(&p);
        ExtendedImpulse e = extend_impulse(w, ptrs);
        write_field(e.values, out_lo, out_hi, out, cap);
    });
}

int ref_estimate(void* h, int q, const double* Z, const double* Y, int nleaf,
                 const std::int64_t* leaf_lo, const std::int64_t* leaf_hi, double* ytilde,
                 double* eta_cells, double* eta_abs, double* eta_rel) {
    return guarded([&] {
        auto* o = static_cast<RefOp*>(h);
        const IndexBox& omega = o->op.domain();
        const std::int64_t n = omega.num_points();
        const int d = o->dim;
        ProbeSet probes;
        probes.q = q;
        for (int i = 0; i < q; ++i) {
            GridFunction z(omega), y(omega);
            std::memcpy(z.data(), Z + i * n, static_cast<std::size_t>(n) * sizeof(double));
            std::memcpy(y.data(), Y + i * n, static_cast<std::size_t>(n) * sizeof(double));
            probes.zeta.push_back(std::move(z));
            probes.y.push_back(std::move(y));
        }
        EstimatorState st = make_estimator_state(probes);
        std::vector<int> all(static_cast<std::size_t>(o->op.rank()));
        for (int k = 0; k < o->op.rank(); ++k) all[static_cast<std::size_t>(k)] = k;
        update_samples(st, o->op, all, probes);
        *eta_abs = st.eta_abs;
        *eta_rel = st.eta_rel;
        if (ytilde)
            for (int i = 0; i < q; ++i)
                std::memcpy(ytilde + i * n, st.ytilde[static_cast<std::size_t>(i)].data(),
                            static_cast<std::size_t>(n) * sizeof(double));
        for (int c = 0; c < nleaf; ++c) {
            const IndexBox leaf = make_box(d, leaf_lo + c * d, leaf_hi + c * d);
            double s = 0.0;
            for (const auto& df : st.diff) s += squared_norm_on_box(df, leaf);
            eta_cells[c] = std::sqrt(s / st.q);
        }
    });
}

// The reference's vector / probe stream (adaptivity.cpp:19-23, test_pc_operator.cpp:13-18):
// std::mt19937_64(seed) + std::normal_distribution<double>(0, 1), count draws.  Lets the
// reference arm of bench.py draw its inputs without loading the product library.
int ref_normal_fill(std::uint64_t seed, std::int64_t count, double* out) {
    return guarded([&] {
        std::mt19937_64 gen(seed);
        std::normal_distribution<double> nd(0.0, 1.0);
        for (std::int64_t i = 0; i < count; ++i) out[i] = nd(gen);
    });
}

// --- H-matrix (hmatrix.cpp) -------------------------------------------------------------------
void* ref_hmatrix_assemble(void* h, double tol, int leaf_cap, int method, int fixed_rank) {
    HMatrix* out = nullptr;
    const int rc = guarded([&] {
        auto* o = static_cast<RefOp*>(h);
        out = new HMatrix(assemble_hmatrix(o->op, tol, leaf_cap,
                                           method == 0 ? CompressionMethod::Randomized : CompressionMethod::Cur,
                                           fixed_rank));
    });
    return rc == 0 ? out : nullptr;
}

void ref_hmatrix_destroy(void* hm) { delete static_cast<HMatrix*>(hm); }

int ref_hmatrix_save(void* hm, const char* path) {
    return guarded([&] { save_hmatrix(*static_cast<HMatrix*>(hm), path); });
}

void* ref_hmatrix_load(const char* path) {
    HMatrix* out = nullptr;
    const int rc = guarded([&] { out = new HMatrix(load_hmatrix(path)); });
    return rc == 0 ? out : nullptr;
}

int ref_hmatrix_matvec(void* hm, const double* f, double* g) {
    return guarded([&] {
        auto* H = static_cast<HMatrix*>(hm);
        const auto n = static_cast<Eigen::Index>(H->tree.domain().num_points());
        Eigen::VectorXd out = H->matvec(Eigen::VectorXd(f, n));
        std::memcpy(g, out.data(), static_cast<std::size_t>(out.size()) * sizeof(double));
    });
}

// counts[0..4] = {blocks, low-rank blocks, max rank, any_rank_capped, nodes}
int ref_hmatrix_info(void* hm, std::int64_t* counts) {
    return guarded([&] {
        auto* H = static_cast<HMatrix*>(hm);
        std::int64_t lr = 0, mr = 0;
        for (const auto& b : H->blocks)
            if (b.low_rank) {
                ++lr;
                mr = std::max<std::int64_t>(mr, b.factors.rank());
            }
        counts[0] = static_cast<std::int64_t>(H->blocks.size());
        counts[1] = lr;
        counts[2] = mr;
        counts[3] = H->any_rank_capped ? 1 : 0;
        counts[4] = static_cast<std::int64_t>(H->tree.nodes().size());
    });
}

// block i: {t, s, low_rank, rows, cols, rank}; B (rows x rank), C (rank x cols) or dense, row-major
int ref_hmatrix_block(void* hm, std::int64_t i, std::int64_t* meta, double* B, double* C, double* dense) {
    return guarded([&] {
        auto* H = static_cast<HMatrix*>(hm);
        const HBlock& b = H->blocks.at(static_cast<std::size_t>(i));
        const ClusterNode& tn = H->tree.node(b.t_node);
        const ClusterNode& sn = H->tree.node(b.s_node);
        meta[0] = b.t_node;
        meta[1] = b.s_node;
        meta[2] = b.low_rank ? 1 : 0;
        meta[3] = tn.size();
        meta[4] = sn.size();
        meta[5] = b.low_rank ? b.factors.rank() : 0;
        auto put = [](const Eigen::MatrixXd& m, double* out) {
            if (!out) return;
            for (Eigen::Index r = 0; r < m.rows(); ++r)
                for (Eigen::Index c = 0; c < m.cols(); ++c) out[r * m.cols() + c] = m(r, c);
        };
        if (b.low_rank) {
            put(b.factors.B, B);
            put(b.factors.C, C);
        } else {
            put(b.dense, dense);
        }
    });
}

}  // extern "C"
