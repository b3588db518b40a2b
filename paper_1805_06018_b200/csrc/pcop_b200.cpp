// Host side of the B200-native product-convolution apply path: planning,
// device-memory layout, pass orchestration and the C ABI (include/pcb/pcb.h).
//
// Reference interface mirrored: pcop::ProductConvolutionOperator
// (proj/core/include/pcop/pc_operator.hpp:17-66, src/pc_operator.cpp:26-148).
// The arithmetic of fft_convolve (src/fft.cpp:64-162) is re-planned for the GPU:
//   * each term's input window is X_k = footprint(w_k) cap Omega, the only
//     place w_k . f is nonzero (restrict_to + multiply_into, pc_operator.cpp:51-52);
//   * the kernel phi_k^E is only ever read on Omega - X_k (outputs are cropped
//     to Omega, pc_operator.cpp:53 / grid_function.cpp:41-52) and is trimmed to
//     its nonzero bounding box there — exact, it drops zeros only;
//   * spectra Phi_k are built once (K1) instead of on every call (fft.cpp:156-157).
// Two exact plans (SURVEY.md 8(a) "GPU restatement"):
//   GLOBAL: one FFT grid P >= n + ext(X_k) per axis, output shift s = Omega.lo;
//           sum_k Phi_k . FFT(w_k f) accumulates in frequency space; one inverse.
//   LOCAL:  per-term grid P_k >= ext(X_k) + ext(K_k) + 1 (the reference's own
//           padding rule on the trimmed boxes), s_k = X_k.lo + K_k.lo; each
//           term's cropped output is gathered into Omega in ascending k.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <random>
#include <string>
#include <vector>

#include "kernels.cuh"
#include "pcb/pcb.h"

namespace pcb {
namespace {

thread_local std::string g_err;

struct Fail {
    pcb_status st;
    std::string msg;
};
[[noreturn]] void fail(pcb_status st, const std::string& msg) { throw Fail{st, msg}; }

#define PCB_CK(x)                                                                                   \
    do {                                                                                            \
        cudaError_t e_ = (x);                                                                       \
        if (e_ != cudaSuccess) fail(PCB_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
    } while (0)

template <typename T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n) {
        o.p = nullptr;
        o.n = 0;
    }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) {
            release();
            p = o.p;
            n = o.n;
            o.p = nullptr;
            o.n = 0;
        }
        return *this;
    }
    ~DevBuf() { release(); }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    void alloc(size_t cnt) {
        release();
        if (cnt == 0) return;
        cudaError_t e = cudaMalloc(&p, cnt * sizeof(T));
        if (e != cudaSuccess) {
            p = nullptr;
            (void)cudaGetLastError();
            fail(PCB_ENOMEM, "cudaMalloc of " + std::to_string(cnt * sizeof(T)) + " bytes failed: " +
                                 cudaGetErrorString(e));
        }
        n = cnt;
    }
    void ensure(size_t cnt) {
        if (cnt > n) alloc(cnt);
    }
    void upload(const std::vector<T>& h) {
        alloc(h.size());
        if (!h.empty()) PCB_CK(cudaMemcpy(p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
    }
    size_t bytes() const { return n * sizeof(T); }
};

int64_t pow2_at_least(int64_t v) {
    int64_t p = 16;
    while (p < v) p <<= 1;
    return p;
}

struct HBox {
    int64_t lo[3], hi[3];
    bool empty = false;
};

struct Csr {  // rows_inv gather list over the active output lines of one chunk
    int64_t n_lines = 0;
    DevBuf<int64_t> ptr, ids;
    DevBuf<int32_t> rng;
    DevBuf<GatherEntry> en;
};

struct Chunk {
    int first = 0, count = 0;
    DevBuf<int32_t> slots;
    Csr apply, adj;
};

struct Group {
    int P[3] = {1, 1, 1};
    int W = 0;
    int64_t L = 0;
    int nl = 0;
    int64_t Lt = 0;  // L rounded up to the spectrum tile width
    std::vector<int> terms;
    int m0max = 0, o0max = 0;
    // per-item strides (double2) for each pass family
    int64_t S_apply = 0, T_apply = 0, S_adj = 0, T_adj = 0, S_spec = 0;
    int vb = 1;  // vectors per pass
    std::vector<Chunk> chunks;
};

std::atomic<long long> g_launches{0};

}  // namespace
}  // namespace pcb

struct pcb_op {
    std::mutex mu;
    int device = 0;
    int dim_user = 2, D = 2;
    int64_t dom_lo[3] = {0, 0, 0};
    int32_t n[3] = {1, 1, 1};
    int64_t N = 0;
    int r = 0;
    int mode = PCB_MODE_AUTO;
    int max_batch = 16;
    std::vector<pcb::TermDesc> terms;
    std::vector<char> has_x, has_k, owned;
    pcb::TermDesc gdesc{};
    pcb::DevBuf<pcb::TermDesc> d_terms, d_gdesc;
    pcb::DevBuf<double> w_pool, phi_pool;
    pcb::DevBuf<double2> spec_pool, tw;
    std::vector<pcb::Group> groups;
    pcb::DevBuf<double2> S, T, T2;  // T2: second inverse buffer of the two-stream local pipeline
    cudaStream_t sA = nullptr, sB = nullptr;
    cudaStream_t s_h2d = nullptr, s_d2h = nullptr;  // host-buffer calls: copy streams
    cudaEvent_t ev_io[8] = {};
    bool pipeline = false;  // two-stream local pipeline (PCB_PIPELINE=1 enables; measured no gain on c3)
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_cols[2] = {nullptr, nullptr}, ev_done[2] = {nullptr, nullptr};
    // entry gather
    int32_t bucket[3] = {1, 1, 1}, nb[3] = {1, 1, 1};
    pcb::DevBuf<int64_t> bucket_ptr;
    pcb::DevBuf<int32_t> bucket_terms;
    // host-call staging
    pcb::DevBuf<double> st_in, st_out, st_aux;
    pcb::DevBuf<int64_t> st_i64a, st_i64b;
    pcb::DevBuf<int32_t> st_flag, st_shape;
    cudaStream_t stream = nullptr;
    pcb_info info{};
    // per-kernel event profiling (pcb_profile_begin / pcb_profile_end)
    bool prof = false;
    struct Rec {
        const char* name;
        cudaEvent_t a, b;
    };
    std::vector<Rec> recs;
    std::vector<cudaEvent_t> ev_pool;
};

namespace pcb {
namespace {

double fft_flops_c(double P) { return 5.0 * P * std::log2(P); }   // complex line
double fft_flops_r(double P) { return 2.5 * P * std::log2(P); }   // real line (R2C / C2R)

void set_err(const std::string& m) { g_err = m; }

template <typename Fn>
pcb_status guarded(Fn&& fn) {
    try {
        fn();
        return PCB_OK;
    } catch (const Fail& f) {
        set_err(f.msg);
        return f.st;
    } catch (const std::bad_alloc&) {
        set_err("host allocation failed");
        return PCB_ENOMEM;
    } catch (const std::exception& e) {
        set_err(e.what());
        return PCB_EINTERNAL;
    }
}

void make_twiddles(pcb_op* op) {
    std::vector<double2> h;
    for (int len = 8; len <= 8192; len <<= 1) {
        for (int m = 0; m < len; ++m) {
            const long double ang = -2.0L * 3.141592653589793238462643383279502884L * (long double)m / (long double)len;
            h.push_back(make_double2((double)cosl(ang), (double)sinl(ang)));
        }
    }
    op->tw.upload(h);
}

PassArgs base_args(pcb_op* op, const Group& g) {
    PassArgs a{};
    a.D = op->D;
    for (int i = 0; i < 3; ++i) {
        a.dom_lo[i] = op->dom_lo[i];
        a.n[i] = op->n[i];
        a.P[i] = g.P[i];
    }
    a.W = g.W;
    a.L = g.L;
    a.nl_cols = g.nl;
    a.terms = op->d_terms.p;
    a.gdesc = op->d_gdesc.p;
    a.N = op->N;
    a.S = op->S.p;
    a.T = op->T.p;
    a.w_pool = op->w_pool.p;
    a.phi_pool = op->phi_pool.p;
    a.spec_pool = op->spec_pool.p;
    a.tw = op->tw.p;
    double sc = 1.0;
    for (int i = 0; i < op->D; ++i) sc /= (double)g.P[i];
    a.scale = sc;
    return a;
}

void launch_ck(cudaError_t e, const char* what) {
    g_launches.fetch_add(1);
    if (e != cudaSuccess) fail(PCB_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

cudaEvent_t take_event(pcb_op* op) {
    if (!op->ev_pool.empty()) {
        cudaEvent_t e = op->ev_pool.back();
        op->ev_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    PCB_CK(cudaEventCreate(&e));
    return e;
}

// launch with optional per-kernel CUDA-event bracketing on the launching stream
template <typename Fn>
void launch(pcb_op* op, cudaStream_t st, const char* what, Fn&& fn) {
    if (!op->prof) {
        launch_ck(fn(), what);
        return;
    }
    cudaEvent_t a = take_event(op), b = take_event(op);
    PCB_CK(cudaEventRecord(a, st));
    launch_ck(fn(), what);
    PCB_CK(cudaEventRecord(b, st));
    op->recs.push_back({what, a, b});
}

// ---------------------------------------------------------------------------
// planning

void build_csr(pcb_op* op, Group& g, Chunk& c, bool global) {
    const int D = op->D;
    const int64_t n_lines = D == 2 ? op->n[0] : (int64_t)op->n[0] * op->n[1];
    auto line_of = [&](int64_t c0, int64_t c1) {  // absolute coordinates of the lead axes
        return D == 2 ? c0 - op->dom_lo[0] : (c0 - op->dom_lo[0]) * op->n[1] + (c1 - op->dom_lo[1]);
    };
    const int ax = D - 1;
    // entry's output range along the last axis (domain-relative) and its line shift
    auto finish = [&](GatherEntry& e, const TermDesc& t, bool adjoint, int64_t w_row) {
        if (!adjoint) {
            e.sh = (int)(t.s[ax] - op->dom_lo[ax]);
            e.lo = e.sh + t.o_lo[ax];
            e.hi = e.lo + t.o_cnt[ax];
            e.w_off = -1;
        } else {
            e.sh = (int)(t.x_lo[ax] - op->dom_lo[ax]);
            e.lo = e.sh;
            e.hi = e.sh + t.m[ax];
            e.w_off = t.w_off + w_row * t.m[ax] - e.sh;
        }
        e.lo = std::max(e.lo, 0);
        e.hi = std::min(e.hi, op->n[ax]);
    };
    std::vector<std::vector<GatherEntry>> ap(n_lines), ad(n_lines);
    for (int i = 0; i < c.count; ++i) {
        const TermDesc& t = op->terms[g.terms[c.first + i]];
        // adjoint: output on X_k (u ranges), T lines u0 [, u1]
        const int c1n = D == 3 ? t.m[1] : 1;
        for (int u0 = 0; u0 < t.m[0]; ++u0)
            for (int u1 = 0; u1 < c1n; ++u1) {
                GatherEntry e{};
                e.slot = i;
                e.t_off = (int64_t)u0 * g.L + (D == 3 ? (int64_t)u1 * g.W : 0);
                finish(e, t, true, D == 3 ? u0 * t.m[1] + u1 : u0);
                ad[line_of(t.x_lo[0] + u0, D == 3 ? t.x_lo[1] + u1 : 0)].push_back(e);
            }
        if (!global) {
            const int o1n = D == 3 ? t.o_cnt[1] : 1;
            for (int j0 = 0; j0 < t.o_cnt[0]; ++j0)
                for (int j1 = 0; j1 < o1n; ++j1) {
                    GatherEntry e{};
                    e.slot = i;
                    e.t_off = (int64_t)j0 * g.L + (D == 3 ? (int64_t)j1 * g.W : 0);
                    finish(e, t, false, 0);
                    const int64_t y0 = t.s[0] + t.o_lo[0] + j0;
                    const int64_t y1 = D == 3 ? t.s[1] + t.o_lo[1] + j1 : 0;
                    ap[line_of(y0, y1)].push_back(e);
                }
        }
    }
    if (global) {
        for (int64_t ln = 0; ln < n_lines; ++ln) {
            GatherEntry e{};
            e.slot = 0;
            const int64_t j0 = D == 2 ? ln : ln / op->n[1];
            const int64_t j1 = D == 2 ? 0 : ln % op->n[1];
            e.t_off = j0 * g.L + j1 * g.W;
            finish(e, op->gdesc, false, 0);
            ap[ln].push_back(e);
        }
    }
    auto flatten = [&](std::vector<std::vector<GatherEntry>>& lists, Csr& out) {
        std::vector<int64_t> hp, ids;
        std::vector<int32_t> rg;
        std::vector<GatherEntry> he;
        for (int64_t ln = 0; ln < n_lines; ++ln) {
            if (lists[ln].empty()) continue;
            int ulo = INT32_MAX, uhi = INT32_MIN;
            for (const GatherEntry& e : lists[ln]) {
                ulo = std::min(ulo, e.lo);
                uhi = std::max(uhi, e.hi);
            }
            hp.push_back((int64_t)he.size());
            ids.push_back(ln);
            rg.push_back(ulo);
            rg.push_back(std::max(ulo, uhi));
            he.insert(he.end(), lists[ln].begin(), lists[ln].end());
        }
        hp.push_back((int64_t)he.size());
        out.n_lines = (int64_t)ids.size();
        out.ptr.upload(hp);
        if (ids.empty()) {
            ids.push_back(0);
            rg.push_back(0);
            rg.push_back(0);
        }
        if (he.empty()) he.push_back(GatherEntry{});
        out.ids.upload(ids);
        out.rng.upload(rg);
        out.en.upload(he);
    };
    flatten(ap, c.apply);
    flatten(ad, c.adj);
}

void plan(pcb_op* op, int32_t dim, const int64_t* dom_lo, const int64_t* dom_hi, int32_t r, const int64_t* w_lo,
          const int64_t* w_hi, const double* const* w_vals, const int64_t* phi_lo, const int64_t* phi_hi,
          const double* const* phi_vals, const pcb_options& opt) {
    if (dim < 1 || dim > 3) fail(PCB_EINVAL, "pcb_create: dim must be 1, 2 or 3");
    if (r < 0) fail(PCB_EINVAL, "PCOp: one weight per impulse required");
    if (!dom_lo || !dom_hi || (r > 0 && (!w_lo || !w_hi || !w_vals || !phi_lo || !phi_hi || !phi_vals)))
        fail(PCB_EINVAL, "pcb_create: null argument");
    const int D = dim == 1 ? 2 : dim;
    const int off = D - dim;  // leading singleton axes for dim == 1
    op->dim_user = dim;
    op->D = D;
    op->r = r;
    // internal coordinates: axis a < off is a singleton at 0
    auto to_int = [&](const int64_t* v, int64_t* out) {
        for (int a = 0; a < D; ++a) out[a] = a < off ? 0 : v[a - off];
        for (int a = D; a < 3; ++a) out[a] = 0;
    };
    int64_t dlo[3], dhi[3];
    to_int(dom_lo, dlo);
    to_int(dom_hi, dhi);
    op->N = 1;
    for (int a = 0; a < D; ++a) {
        if (dlo[a] > dhi[a]) fail(PCB_EINVAL, "IndexBox: lo > hi");
        op->dom_lo[a] = dlo[a];
        const int64_t ext = dhi[a] - dlo[a] + 1;
        if (ext > (1 << 20)) fail(PCB_EINVAL, "pcb_create: domain axis too large");
        op->n[a] = (int32_t)ext;
        op->N *= ext;
    }
    op->terms.assign(r, TermDesc{});
    op->has_x.assign(r, 0);
    op->has_k.assign(r, 0);
    op->owned.assign(r, 0);
    std::vector<double> wpool, ppool;
    std::vector<HBox> X(r), K(r);
    for (int k = 0; k < r; ++k) {
        int64_t flo[3], fhi[3], plo[3], phi[3];
        to_int(w_lo + (int64_t)k * dim, flo);
        to_int(w_hi + (int64_t)k * dim, fhi);
        to_int(phi_lo + (int64_t)k * dim, plo);
        to_int(phi_hi + (int64_t)k * dim, phi);
        for (int a = 0; a < D; ++a)
            if (flo[a] > fhi[a] || plo[a] > phi[a]) fail(PCB_EINVAL, "IndexBox: lo > hi");
        if (!w_vals[k] || !phi_vals[k]) fail(PCB_EINVAL, "pcb_create: null weight/impulse values");
        TermDesc& t = op->terms[k];
        // X_k = footprint cap Omega
        HBox& x = X[k];
        for (int a = 0; a < D; ++a) {
            x.lo[a] = std::max(flo[a], op->dom_lo[a]);
            x.hi[a] = std::min(fhi[a], op->dom_lo[a] + op->n[a] - 1);
            if (x.lo[a] > x.hi[a]) x.empty = true;
        }
        for (int a = D; a < 3; ++a) x.lo[a] = x.hi[a] = 0;
        int64_t fext[3] = {1, 1, 1}, pext[3] = {1, 1, 1};
        for (int a = 0; a < D; ++a) {
            fext[a] = fhi[a] - flo[a] + 1;
            pext[a] = phi[a] - plo[a] + 1;
        }
        if (x.empty) continue;
        op->has_x[k] = 1;
        for (int a = 0; a < 3; ++a) {
            t.x_lo[a] = x.lo[a];
            t.m[a] = (int32_t)(x.hi[a] - x.lo[a] + 1);
        }
        t.w_off = (int64_t)wpool.size();
        const double* wv = w_vals[k];
        for (int64_t i0 = x.lo[0]; i0 <= x.hi[0]; ++i0)
            for (int64_t i1 = x.lo[1]; i1 <= x.hi[1]; ++i1)
                for (int64_t i2 = x.lo[2]; i2 <= x.hi[2]; ++i2) {
                    const int64_t idx = D == 2 ? (i0 - flo[0]) * fext[1] + (i1 - flo[1])
                                               : ((i0 - flo[0]) * fext[1] + (i1 - flo[1])) * fext[2] + (i2 - flo[2]);
                    wpool.push_back(wv[idx]);
                }
        // window Omega - X_k, kernel box cap window, then its nonzero bounding box
        HBox kr;
        for (int a = 0; a < D; ++a) {
            const int64_t wlo = op->dom_lo[a] - x.hi[a];
            const int64_t whi = op->dom_lo[a] + op->n[a] - 1 - x.lo[a];
            kr.lo[a] = std::max(wlo, plo[a]);
            kr.hi[a] = std::min(whi, phi[a]);
            if (kr.lo[a] > kr.hi[a]) kr.empty = true;
        }
        for (int a = D; a < 3; ++a) kr.lo[a] = kr.hi[a] = 0;
        if (kr.empty) continue;
        const double* pv = phi_vals[k];
        HBox nz;
        for (int a = 0; a < 3; ++a) {
            nz.lo[a] = INT64_MAX;
            nz.hi[a] = INT64_MIN;
        }
        bool any = false;
        for (int64_t i0 = kr.lo[0]; i0 <= kr.hi[0]; ++i0)
            for (int64_t i1 = kr.lo[1]; i1 <= kr.hi[1]; ++i1) {
                const int64_t rowbase = D == 2 ? (i0 - plo[0]) * pext[1] + (i1 - plo[1])
                                               : ((i0 - plo[0]) * pext[1] + (i1 - plo[1])) * pext[2];
                const int64_t c2lo = D == 2 ? 0 : kr.lo[2], c2hi = D == 2 ? 0 : kr.hi[2];
                for (int64_t i2 = c2lo; i2 <= c2hi; ++i2) {
                    const double v = D == 2 ? pv[rowbase] : pv[rowbase + (i2 - plo[2])];
                    if (v != 0.0) {
                        any = true;
                        const int64_t c[3] = {i0, i1, i2};
                        for (int a = 0; a < D; ++a) {
                            nz.lo[a] = std::min(nz.lo[a], c[a]);
                            nz.hi[a] = std::max(nz.hi[a], c[a]);
                        }
                    }
                }
            }
        if (!any) continue;
        for (int a = D; a < 3; ++a) nz.lo[a] = nz.hi[a] = 0;
        K[k] = nz;
        op->has_k[k] = 1;
        for (int a = 0; a < 3; ++a) {
            t.k_lo[a] = nz.lo[a];
            t.k_ext[a] = (int32_t)(nz.hi[a] - nz.lo[a] + 1);
        }
        t.phi_off = (int64_t)ppool.size();
        for (int64_t i0 = nz.lo[0]; i0 <= nz.hi[0]; ++i0)
            for (int64_t i1 = nz.lo[1]; i1 <= nz.hi[1]; ++i1)
                for (int64_t i2 = nz.lo[2]; i2 <= nz.hi[2]; ++i2) {
                    const int64_t idx = D == 2 ? (i0 - plo[0]) * pext[1] + (i1 - plo[1])
                                               : ((i0 - plo[0]) * pext[1] + (i1 - plo[1])) * pext[2] + (i2 - plo[2]);
                    ppool.push_back(pv[idx]);
                }
    }
    if (wpool.empty()) wpool.push_back(0.0);
    if (ppool.empty()) ppool.push_back(0.0);

    // shard-by-k over the active terms (contiguous, balanced by count)
    std::vector<int> active;
    for (int k = 0; k < r; ++k)
        if (op->has_x[k] && op->has_k[k]) active.push_back(k);
    const int sc = std::max(1, opt.shard_count);
    const int sr = opt.shard_rank;
    if (sr < 0 || sr >= sc) fail(PCB_EINVAL, "pcb_create: shard_rank out of range");
    const size_t a0 = active.size() * (size_t)sr / sc, a1 = active.size() * (size_t)(sr + 1) / sc;
    std::vector<int> mine(active.begin() + a0, active.begin() + a1);
    for (int k : mine) op->owned[k] = 1;

    // candidate plans
    int64_t Pg[3] = {1, 1, 1};
    for (int a = 0; a < D; ++a) {
        int64_t mmax = 1;
        for (int k : mine) mmax = std::max<int64_t>(mmax, op->terms[k].m[a]);
        Pg[a] = pow2_at_least(op->n[a] + mmax - 1);
    }
    auto local_P = [&](int k, int a) {
        return pow2_at_least((int64_t)op->terms[k].m[a] + op->terms[k].k_ext[a] - 1);
    };
    bool global_ok = true, local_ok = true;
    for (int a = 0; a < D; ++a) global_ok = global_ok && Pg[a] <= 4096;
    double g_fl = 0, g_by = 0, l_fl = 0, l_by = 0;
    {
        const double last = (double)Pg[D - 1];
        const double W = last / 2 + 1;
        const double lead = D == 2 ? (double)Pg[0] : (double)Pg[0] * Pg[1];
        for (int k : mine) {
            const TermDesc& t = op->terms[k];
            const double mlead = D == 2 ? t.m[0] : (double)t.m[0] * t.m[1];
            g_fl += mlead * fft_flops_r(last) + W * (D == 3 ? t.m[0] * fft_flops_c((double)Pg[1]) : 0) +
                    W * (D == 3 ? Pg[1] : 1) * fft_flops_c((double)Pg[0]) + 8.0 * lead * W;
            g_by += lead * W * 16.0;
        }
        g_fl += W * (D == 3 ? Pg[1] : 1) * fft_flops_c((double)Pg[0]) +
                W * (D == 3 ? op->n[0] * fft_flops_c((double)Pg[1]) : 0) +
                (D == 2 ? op->n[0] : (double)op->n[0] * op->n[1]) * fft_flops_r(last);
    }
    for (int k : mine) {
        const TermDesc& t = op->terms[k];
        int64_t P[3] = {1, 1, 1};
        for (int a = 0; a < D; ++a) {
            P[a] = local_P(k, a);
            if (P[a] > 4096) local_ok = false;
        }
        const double last = (double)P[D - 1];
        const double W = last / 2 + 1;
        const double lead = D == 2 ? (double)P[0] : (double)P[0] * P[1];
        const double mlead = D == 2 ? t.m[0] : (double)t.m[0] * t.m[1];
        const double outlead = mlead * 2;  // o_cnt ~ m + k_ext
        l_fl += (mlead + outlead) * fft_flops_r(last) + 2 * W * (D == 3 ? P[1] : 1) * fft_flops_c((double)P[0]) +
                (D == 3 ? 2 * W * t.m[0] * fft_flops_c((double)P[1]) : 0) + 6.0 * lead * W;
        l_by += lead * W * 16.0 * 4.0;  // spectra + forward/inverse scratch round trips
    }
    const double g_t = std::max(g_fl / 8e12, g_by / 6e12);
    const double l_t = std::max(l_fl / 8e12, l_by / 6e12);
    int mode = opt.mode;
    if (mode == PCB_MODE_AUTO) mode = (local_ok && (!global_ok || l_t < g_t)) ? PCB_MODE_LOCAL : PCB_MODE_GLOBAL;
    if (mode == PCB_MODE_GLOBAL && !global_ok) fail(PCB_EINVAL, "pcb_create: global FFT grid exceeds 4096 per axis");
    if (mode == PCB_MODE_LOCAL && !local_ok) fail(PCB_EINVAL, "pcb_create: local FFT grid exceeds 4096 per axis");
    if (mode != PCB_MODE_GLOBAL && mode != PCB_MODE_LOCAL) fail(PCB_EINVAL, "pcb_create: bad mode");
    op->mode = mode;

    // per-term placement
    for (int k = 0; k < r; ++k) {
        TermDesc& t = op->terms[k];
        if (!op->has_x[k] || !op->has_k[k]) continue;
        for (int a = 0; a < D; ++a) {
            if (mode == PCB_MODE_GLOBAL) {
                t.s[a] = op->dom_lo[a];
                t.o_lo[a] = 0;
                t.o_cnt[a] = op->n[a];
            } else {
                t.s[a] = t.x_lo[a] + t.k_lo[a];
                const int64_t full = (int64_t)t.m[a] + t.k_ext[a] - 1;
                const int64_t lo = std::max<int64_t>(0, op->dom_lo[a] - t.s[a]);
                const int64_t hi = std::min<int64_t>(full - 1, op->dom_lo[a] + op->n[a] - 1 - t.s[a]);
                t.o_lo[a] = (int32_t)lo;
                t.o_cnt[a] = (int32_t)std::max<int64_t>(0, hi - lo + 1);
            }
        }
        for (int a = D; a < 3; ++a) {
            t.s[a] = 0;
            t.o_lo[a] = 0;
            t.o_cnt[a] = 1;
        }
    }
    // global pseudo term
    {
        TermDesc& gd = op->gdesc;
        gd = TermDesc{};
        for (int a = 0; a < 3; ++a) {
            gd.s[a] = a < D ? op->dom_lo[a] : 0;
            gd.x_lo[a] = gd.s[a];
            gd.o_lo[a] = 0;
            gd.o_cnt[a] = a < D ? op->n[a] : 1;
            gd.m[a] = gd.o_cnt[a];
        }
    }
    // groups
    std::map<std::vector<int>, int> gid;
    for (int k : mine) {
        std::vector<int> key(3, 1);
        for (int a = 0; a < D; ++a) key[a] = (int)(mode == PCB_MODE_GLOBAL ? Pg[a] : local_P(k, a));
        auto it = gid.find(key);
        int id;
        if (it == gid.end()) {
            id = (int)op->groups.size();
            gid.emplace(key, id);
            op->groups.emplace_back();
            Group& g = op->groups.back();
            for (int a = 0; a < 3; ++a) g.P[a] = key[a];
        } else {
            id = it->second;
        }
        op->groups[id].terms.push_back(k);
    }
    // layout per group
    int64_t spec_total = 0;
    for (Group& g : op->groups) {
        const int last = g.P[D - 1];
        g.W = ((last / 2 + 1) + 7) / 8 * 8;
        g.L = D == 2 ? g.W : (int64_t)g.P[1] * g.W;
        g.nl = cols_tile_width(g.P[0]);
        if (g.nl <= 0) fail(PCB_EINTERNAL, "unsupported FFT size");
        g.Lt = (g.L + g.nl - 1) / g.nl * g.nl;
        for (int k : g.terms) {
            const TermDesc& t = op->terms[k];
            g.m0max = std::max(g.m0max, t.m[0]);
            g.o0max = std::max(g.o0max, t.o_cnt[0]);
        }
        for (int k : g.terms) {
            op->terms[k].spec_off = spec_total;
            spec_total += (int64_t)g.P[0] * g.Lt;
        }
    }
    op->spec_pool.alloc((size_t)std::max<int64_t>(spec_total, 1));
    PCB_CK(cudaMemset(op->spec_pool.p, 0, op->spec_pool.bytes()));

    // scratch budget and chunking
    size_t freeb = 0, totb = 0;
    PCB_CK(cudaMemGetInfo(&freeb, &totb));
    int64_t budget = opt.scratch_bytes > 0 ? opt.scratch_bytes : std::min<int64_t>((int64_t)freeb / 3, 8LL << 30);
    budget = std::max<int64_t>(budget, 64LL << 20);
    const int mb = op->max_batch;
    int64_t S_need = 0, T_need = 0;
    for (Group& g : op->groups) {
        const int64_t plane = g.L;
        const int64_t n0 = op->n[0];
        if (mode == PCB_MODE_LOCAL) {
            g.S_apply = (int64_t)g.m0max * plane;
            g.T_apply = (int64_t)g.o0max * plane;
            g.S_adj = (int64_t)g.o0max * plane;
            g.T_adj = (int64_t)g.m0max * plane;
            const int64_t per_item = 16 * (std::max(g.S_apply, g.S_adj) + std::max(g.T_apply, g.T_adj));
            int per_chunk = (int)std::max<int64_t>(1, budget / std::max<int64_t>(1, (op->pipeline ? 2 : 1) * per_item * mb));
            per_chunk = std::min<int>(per_chunk, std::max(1, 65535 / mb));
            // at least two chunks per group so the two-stream pipeline has something to overlap
            if (op->pipeline) per_chunk = std::min<int>(per_chunk, std::max<int>(1, ((int)g.terms.size() + 1) / 2));
            if (const char* e = getenv("PCB_CHUNK_TERMS")) per_chunk = std::max(1, atoi(e));
            g.vb = mb;
            for (int f = 0; f < (int)g.terms.size(); f += per_chunk) {
                g.chunks.emplace_back();
                g.chunks.back().first = f;
                g.chunks.back().count = std::min<int>(per_chunk, (int)g.terms.size() - f);
            }
            S_need = std::max<int64_t>(S_need, (int64_t)per_chunk * mb * std::max(g.S_apply, g.S_adj));
            T_need = std::max<int64_t>(T_need, (int64_t)per_chunk * mb * std::max(g.T_apply, g.T_adj));
        } else {
            const int64_t nt = (int64_t)g.terms.size();
            g.S_apply = (int64_t)g.m0max * plane;
            g.T_apply = n0 * plane;
            g.S_adj = n0 * plane;
            g.T_adj = (int64_t)g.m0max * plane;
            const int64_t per_vec = 16 * (std::max(nt * g.S_apply, g.S_adj) + std::max(g.T_apply, nt * g.T_adj));
            int vb = (int)std::max<int64_t>(1, std::min<int64_t>(mb, budget / std::max<int64_t>(1, per_vec)));
            vb = std::min<int>(vb, std::max<int>(1, (int)(65535 / std::max<int64_t>(1, nt))));
            g.vb = vb;
            g.chunks.emplace_back();
            g.chunks.back().first = 0;
            g.chunks.back().count = (int)nt;
            S_need = std::max<int64_t>(S_need, std::max(nt * vb * g.S_apply, (int64_t)vb * g.S_adj));
            T_need = std::max<int64_t>(T_need, std::max((int64_t)vb * g.T_apply, nt * vb * g.T_adj));
        }
        // K1 scratch: at least one full P0 x L item
        g.S_spec = (int64_t)g.P[0] * plane;
        S_need = std::max<int64_t>(S_need, g.S_spec);
    }
    op->S.alloc((size_t)std::max<int64_t>(S_need, 1));
    op->T.alloc((size_t)std::max<int64_t>(T_need, 1));
    PCB_CK(cudaMemset(op->S.p, 0, op->S.bytes()));
    PCB_CK(cudaMemset(op->T.p, 0, op->T.bytes()));
    if (mode == PCB_MODE_LOCAL && op->pipeline) {
        op->T2.alloc((size_t)std::max<int64_t>(T_need, 1));
        PCB_CK(cudaMemset(op->T2.p, 0, op->T2.bytes()));
    }

    // device descriptors and pools
    op->d_terms.upload(op->terms.empty() ? std::vector<TermDesc>(1) : op->terms);
    op->d_gdesc.upload(std::vector<TermDesc>{op->gdesc});
    op->w_pool.upload(wpool);
    op->phi_pool.upload(ppool);
    for (Group& g : op->groups)
        for (Chunk& c : g.chunks) {
            std::vector<int32_t> sl(g.terms.begin() + c.first, g.terms.begin() + c.first + c.count);
            c.slots.upload(sl);
            build_csr(op, g, c, mode == PCB_MODE_GLOBAL);
        }

    // entry buckets over all terms with X and K
    {
        int64_t nbt = 1;
        for (int a = 0; a < 3; ++a) {
            if (a < D) {
                op->bucket[a] = std::max<int32_t>(1, std::min<int32_t>(op->n[a], 16));
                op->nb[a] = (op->n[a] + op->bucket[a] - 1) / op->bucket[a];
            } else {
                op->bucket[a] = 1;
                op->nb[a] = 1;
            }
            nbt *= op->nb[a];
        }
        std::vector<std::vector<int32_t>> lists(nbt);
        for (int k = 0; k < r; ++k) {
            if (!op->has_x[k] || !op->has_k[k]) continue;
            const TermDesc& t = op->terms[k];
            int64_t b0[3] = {0, 0, 0}, b1[3] = {0, 0, 0};
            for (int a = 0; a < D; ++a) {
                b0[a] = (t.x_lo[a] - op->dom_lo[a]) / op->bucket[a];
                b1[a] = (t.x_lo[a] + t.m[a] - 1 - op->dom_lo[a]) / op->bucket[a];
            }
            for (int64_t i0 = b0[0]; i0 <= b1[0]; ++i0)
                for (int64_t i1 = b0[1]; i1 <= b1[1]; ++i1)
                    for (int64_t i2 = b0[2]; i2 <= b1[2]; ++i2) {
                        const int64_t bl = D == 2 ? i0 * op->nb[1] + i1 : (i0 * op->nb[1] + i1) * op->nb[2] + i2;
                        lists[bl].push_back(k);
                    }
        }
        std::vector<int64_t> bp(nbt + 1, 0);
        std::vector<int32_t> bt;
        for (int64_t b = 0; b < nbt; ++b) {
            bp[b] = (int64_t)bt.size();
            bt.insert(bt.end(), lists[b].begin(), lists[b].end());
        }
        bp[nbt] = (int64_t)bt.size();
        if (bt.empty()) bt.push_back(0);
        op->bucket_ptr.upload(bp);
        op->bucket_terms.upload(bt);
    }

    // info
    pcb_info& in = op->info;
    in = pcb_info{};
    in.dim = dim;
    in.rank = r;
    in.rank_active = (int32_t)mine.size();
    in.mode = mode;
    in.n_groups = (int32_t)op->groups.size();
    in.n_points = op->N;
    int best = -1;
    for (size_t i = 0; i < op->groups.size(); ++i)
        if (best < 0 || op->groups[i].terms.size() > op->groups[best].terms.size()) best = (int)i;
    for (int a = 0; a < 3; ++a) in.fft_size[a] = 0;
    if (best >= 0)
        for (int a = 0; a < dim; ++a) in.fft_size[a] = op->groups[best].P[a + off];
    double sb = 0;
    for (const Group& g : op->groups) {
        const double last = g.P[D - 1];
        const double lead = D == 2 ? (double)g.P[0] : (double)g.P[0] * g.P[1];
        sb += (double)g.terms.size() * lead * (last / 2 + 1) * 16.0;
    }
    in.spectra_bytes = (int64_t)(16.0 * (double)spec_total);
    in.bytes_per_vector = sb + 16.0 * (double)op->N;
    in.flops_per_vector = mode == PCB_MODE_GLOBAL ? g_fl : l_fl;
    int launches = 0;
    for (const Group& g : op->groups) launches += (int)g.chunks.size() * (D == 3 ? 5 : 3);
    in.launches_per_batch = launches;
}

void build_spectra(pcb_op* op) {
    const int D = op->D;
    for (Group& g : op->groups) {
        PassArgs a = base_args(op, g);
        const int64_t per = std::max<int64_t>(1, (int64_t)(op->S.n / (size_t)g.S_spec));
        DevBuf<int32_t> slots;
        slots.upload(g.terms);
        for (int64_t f = 0; f < (int64_t)g.terms.size(); f += per) {
            const int cnt = (int)std::min<int64_t>(per, (int64_t)g.terms.size() - f);
            a.slots = slots.p + f;
            a.n_slots = cnt;
            a.B = 1;
            a.S_stride = g.S_spec;
            a.global = 0;
            launch_ck(launch_rows_fwd(a, RF_SPEC, op->stream), "rows_fwd(spec)");
            if (D == 3) launch_ck(launch_mid(a, MM_FWD_SPEC, op->stream), "mid(spec)");
            launch_ck(launch_cols(a, CM_SPEC, op->stream), "cols(spec)");
        }
        PCB_CK(cudaStreamSynchronize(op->stream));
    }
}

// one apply / adjoint batch on device pointers.
// GLOBAL: one chunk per vector block, on the caller's stream.
// LOCAL: chunks of terms flow through a two-stream pipeline forked from the caller's stream:
//   stream A: rows_fwd(i) -> [mid] -> cols(i) -> [mid_inv] (writes T[i % 2]) -> event cols[i % 2]
//   stream B: wait cols[i % 2] -> rows_inv(i) (reads T[i % 2], accumulates into g) -> event done[i % 2]
// stream A waits done[i % 2] before overwriting T[i % 2] again; rows_inv launches stay in chunk
// order on stream B, so the accumulation order (and the result) is fixed.
void run_batch(pcb_op* op, bool adjoint, int32_t B, const double* dF, double* dG, cudaStream_t st) {
    const int D = op->D;
    if (op->groups.empty()) {
        launch(op, st, "zero", [&] { return launch_zero(dG, (int64_t)B * op->N, st); });
        return;
    }
    const bool global = op->mode == PCB_MODE_GLOBAL;
    auto pass_args = [&](const Group& g, const Chunk& c, int b0, int bn, double2* T) {
        PassArgs a = base_args(op, g);
        a.slots = c.slots.p;
        a.n_slots = c.count;
        a.B = bn;
        a.in = dF + (int64_t)b0 * op->N;
        a.out = dG + (int64_t)b0 * op->N;
        a.T = T;
        a.S_stride = adjoint ? g.S_adj : g.S_apply;
        a.T_stride = adjoint ? g.T_adj : g.T_apply;
        return a;
    };
    auto front = [&](PassArgs a, cudaStream_t s) {  // K2 + K3 (+ 3-D middle passes)
        a.global = global;
        if (!adjoint) {
            launch(op, s, "rows_fwd(apply)", [&] { return launch_rows_fwd(a, RF_APPLY, s); });
            if (D == 3) launch(op, s, "mid(fwd apply)", [&] { return launch_mid(a, MM_FWD_APPLY, s); });
            launch(op, s, global ? "cols(apply,global)" : "cols(apply,local)",
                   [&] { return launch_cols(a, global ? CM_APPLY_GLOBAL : CM_APPLY_LOCAL, s); });
            if (D == 3) launch(op, s, "mid(inv apply)", [&] { return launch_mid(a, MM_INV_APPLY, s); });
        } else {
            launch(op, s, "rows_fwd(adjoint)", [&] { return launch_rows_fwd(a, RF_ADJ, s); });
            if (D == 3) launch(op, s, "mid(fwd adjoint)", [&] { return launch_mid(a, MM_FWD_ADJ, s); });
            launch(op, s, global ? "cols(adjoint,global)" : "cols(adjoint,local)",
                   [&] { return launch_cols(a, global ? CM_ADJ_GLOBAL : CM_ADJ_LOCAL, s); });
            a.global = 0;
            if (D == 3) launch(op, s, "mid(inv adjoint)", [&] { return launch_mid(a, MM_INV_ADJ, s); });
        }
    };
    auto back = [&](PassArgs a, const Chunk& c, cudaStream_t s, bool accumulate) {  // K4
        const Csr& csr = adjoint ? c.adj : c.apply;
        a.global = global && !adjoint;
        a.accumulate = accumulate ? 1 : 0;
        a.line_ptr = csr.ptr.p;
        a.line_id = csr.ids.p;
        a.line_rng = csr.rng.p;
        a.entries = csr.en.p;
        if (csr.n_lines > 0)
            launch(op, s, adjoint ? "rows_inv(adjoint)" : "rows_inv(apply)",
                   [&] { return launch_rows_inv(a, adjoint ? RI_ADJ : RI_APPLY, csr.n_lines, s); });
    };

    if (global) {
        const Group& g = op->groups[0];
        const Chunk& c = g.chunks[0];
        for (int b0 = 0; b0 < B; b0 += g.vb) {
            const int bn = std::min(g.vb, B - b0);
            if (adjoint)
                PCB_CK(cudaMemsetAsync(dG + (int64_t)b0 * op->N, 0, (size_t)bn * op->N * sizeof(double), st));
            PassArgs a = pass_args(g, c, b0, bn, op->T.p);
            front(a, st);
            back(a, c, st, adjoint);
        }
        return;
    }

    // LOCAL: fork the two pipeline streams off the caller's stream
    PCB_CK(cudaEventRecord(op->ev_fork, st));
    PCB_CK(cudaStreamWaitEvent(op->sA, op->ev_fork, 0));
    PCB_CK(cudaStreamWaitEvent(op->sB, op->ev_fork, 0));
    PCB_CK(cudaMemsetAsync(dG, 0, (size_t)B * op->N * sizeof(double), op->sB));
    int64_t i = 0;
    int vb = op->max_batch;
    for (const Group& g : op->groups) vb = std::min(vb, g.vb);
    for (int b0 = 0; b0 < B; b0 += vb) {
        const int bn = std::min(vb, B - b0);
        for (const Group& g : op->groups) {
            for (const Chunk& c : g.chunks) {
                const int par = (int)(i & 1);
                double2* T = (par && op->pipeline) ? op->T2.p : op->T.p;
                if (i >= 2 && op->pipeline) PCB_CK(cudaStreamWaitEvent(op->sA, op->ev_done[par], 0));
                PassArgs a = pass_args(g, c, b0, bn, T);
                front(a, op->sA);
                if (op->pipeline) {
                    PCB_CK(cudaEventRecord(op->ev_cols[par], op->sA));
                    PCB_CK(cudaStreamWaitEvent(op->sB, op->ev_cols[par], 0));
                    back(a, c, op->sB, true);
                    PCB_CK(cudaEventRecord(op->ev_done[par], op->sB));
                } else {
                    if (i == 0) {
                        PCB_CK(cudaEventRecord(op->ev_done[0], op->sB));
                        PCB_CK(cudaStreamWaitEvent(op->sA, op->ev_done[0], 0));
                    }
                    back(a, c, op->sA, true);
                }
                ++i;
            }
        }
    }
    // join: the caller's stream waits for both pipeline streams
    PCB_CK(cudaEventRecord(op->ev_join, op->sA));
    PCB_CK(cudaStreamWaitEvent(st, op->ev_join, 0));
    PCB_CK(cudaEventRecord(op->ev_join, op->sB));
    PCB_CK(cudaStreamWaitEvent(st, op->ev_join, 0));
}

EntryArgs entry_args(pcb_op* op) {
    EntryArgs e{};
    e.D = op->D;
    for (int a = 0; a < 3; ++a) {
        e.dom_lo[a] = op->dom_lo[a];
        e.n[a] = op->n[a];
        e.bucket[a] = op->bucket[a];
        e.nb[a] = op->nb[a];
    }
    e.terms = op->d_terms.p;
    e.w_pool = op->w_pool.p;
    e.phi_pool = op->phi_pool.p;
    e.bucket_ptr = op->bucket_ptr.p;
    e.bucket_terms = op->bucket_terms.p;
    return e;
}

void set_device(pcb_op* op) { PCB_CK(cudaSetDevice(op->device)); }

// user coordinates (dim_user per point) -> internal D per point
std::vector<int64_t> to_internal_points(const pcb_op* op, const int64_t* p, int64_t cnt) {
    std::vector<int64_t> out((size_t)cnt * op->D);
    const int off = op->D - op->dim_user;
    for (int64_t i = 0; i < cnt; ++i)
        for (int a = 0; a < op->D; ++a) out[i * op->D + a] = a < off ? 0 : p[i * op->dim_user + a - off];
    return out;
}

}  // namespace
}  // namespace pcb

using namespace pcb;

extern "C" {

PCB_API void pcb_default_options(pcb_options* opt) {
    if (!opt) return;
    std::memset(opt, 0, sizeof(*opt));
    opt->device = -1;
    opt->mode = PCB_MODE_AUTO;
    opt->max_batch = 16;
    opt->shard_rank = 0;
    opt->shard_count = 1;
}

PCB_API const char* pcb_last_error(void) { return g_err.c_str(); }

PCB_API long long pcb_launch_count(void) { return g_launches.load(); }

PCB_API pcb_status pcb_create(int32_t dim, const int64_t* dom_lo, const int64_t* dom_hi, int32_t r,
                              const int64_t* /*points*/, const int64_t* w_lo, const int64_t* w_hi,
                              const double* const* w_vals, const int64_t* phi_lo, const int64_t* phi_hi,
                              const double* const* phi_vals, const pcb_options* opt_in, pcb_op** out) {
    if (!out) {
        set_err("pcb_create: null output handle");
        return PCB_EINVAL;
    }
    *out = nullptr;
    pcb_op* op = new (std::nothrow) pcb_op;
    if (!op) return PCB_ENOMEM;
    const pcb_status st = guarded([&] {
        pcb_options opt;
        pcb_default_options(&opt);
        if (opt_in) opt = *opt_in;
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
            (void)cudaGetLastError();
            fail(PCB_ECUDA, "no CUDA device: the pcop-b200 apply path has no CPU fallback");
        }
        if (opt.device < 0) PCB_CK(cudaGetDevice(&op->device));
        else op->device = opt.device;
        set_device(op);
        cudaDeviceProp prop{};
        PCB_CK(cudaGetDeviceProperties(&prop, op->device));
        if (prop.major < 10) fail(PCB_ECUDA, "pcop-b200 kernels are built for sm_100a (Blackwell B200)");
        op->max_batch = opt.max_batch > 0 ? opt.max_batch : 16;
        if (const char* e = getenv("PCB_PIPELINE")) op->pipeline = atoi(e) != 0;
        PCB_CK(cudaStreamCreateWithFlags(&op->stream, cudaStreamNonBlocking));
        PCB_CK(cudaStreamCreateWithFlags(&op->sA, cudaStreamNonBlocking));
        PCB_CK(cudaStreamCreateWithFlags(&op->sB, cudaStreamNonBlocking));
        for (cudaEvent_t* e : {&op->ev_fork, &op->ev_join, &op->ev_cols[0], &op->ev_cols[1], &op->ev_done[0],
                               &op->ev_done[1]})
            PCB_CK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
        make_twiddles(op);
        plan(op, dim, dom_lo, dom_hi, r, w_lo, w_hi, w_vals, phi_lo, phi_hi, phi_vals, opt);
        build_spectra(op);
        size_t dev = op->w_pool.bytes() + op->phi_pool.bytes() + op->spec_pool.bytes() + op->tw.bytes() +
                     op->S.bytes() + op->T.bytes() + op->d_terms.bytes() + op->bucket_ptr.bytes() +
                     op->bucket_terms.bytes();
        op->info.device_bytes = (int64_t)dev;
    });
    if (st != PCB_OK) {
        pcb_destroy(op);
        return st;
    }
    *out = op;
    return PCB_OK;
}

PCB_API pcb_status pcb_destroy(pcb_op* op) {
    if (!op) return PCB_OK;
    cudaSetDevice(op->device);
    if (op->stream) {
        cudaStreamSynchronize(op->stream);
        cudaStreamDestroy(op->stream);
    }
    for (auto& r : op->recs) {
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
    for (auto e : op->ev_pool) cudaEventDestroy(e);
    for (cudaEvent_t e : op->ev_io)
        if (e) cudaEventDestroy(e);
    for (cudaStream_t s : {op->sA, op->sB, op->s_h2d, op->s_d2h})
        if (s) {
            cudaStreamSynchronize(s);
            cudaStreamDestroy(s);
        }
    for (cudaEvent_t e : {op->ev_fork, op->ev_join, op->ev_cols[0], op->ev_cols[1], op->ev_done[0], op->ev_done[1]})
        if (e) cudaEventDestroy(e);
    delete op;
    return PCB_OK;
}

PCB_API pcb_status pcb_get_info(const pcb_op* op, pcb_info* info) {
    if (!op || !info) {
        set_err("pcb_get_info: null argument");
        return PCB_EINVAL;
    }
    *info = op->info;
    return PCB_OK;
}

static pcb_status apply_dev_common(pcb_op* op, bool adjoint, int32_t B, const double* dF, double* dG, void* stream) {
    if (!op) {
        set_err("null handle");
        return PCB_EINVAL;
    }
    std::lock_guard<std::mutex> lk(op->mu);
    return guarded([&] {
        if (B < 0) fail(PCB_EINVAL, adjoint ? "PCOp::apply_adjoint: shape mismatch" : "PCOp::apply: shape mismatch");
        if (B == 0) return;
        if (!dF || !dG) fail(PCB_EINVAL, "null vector pointer");
        set_device(op);
        run_batch(op, adjoint, B, dF, dG, (cudaStream_t)stream);
    });
}

PCB_API pcb_status pcb_apply_batch_dev(pcb_op* op, int32_t B, const double* dF, double* dG, void* stream) {
    return apply_dev_common(op, false, B, dF, dG, stream);
}
PCB_API pcb_status pcb_apply_adjoint_batch_dev(pcb_op* op, int32_t B, const double* dF, double* dG, void* stream) {
    return apply_dev_common(op, true, B, dF, dG, stream);
}

static pcb_status apply_host_common(pcb_op* op, bool adjoint, int32_t B, const double* F, double* G) {
    if (!op) {
        set_err("null handle");
        return PCB_EINVAL;
    }
    std::lock_guard<std::mutex> lk(op->mu);
    return guarded([&] {
        if (B < 0) fail(PCB_EINVAL, adjoint ? "PCOp::apply_adjoint: shape mismatch" : "PCOp::apply: shape mismatch");
        if (B == 0) return;
        if (!F || !G) fail(PCB_EINVAL, "null vector pointer");
        set_device(op);
        const size_t cnt = (size_t)B * (size_t)op->N;
        op->st_in.ensure(cnt);
        op->st_out.ensure(cnt);
        // sub-batches overlap H2D(j+1) and D2H(j-1) with the kernels of sub-batch j
        const int nsub = B >= 8 ? 4 : (B >= 2 ? 2 : 1);
        if (!op->s_h2d) {
            PCB_CK(cudaStreamCreateWithFlags(&op->s_h2d, cudaStreamNonBlocking));
            PCB_CK(cudaStreamCreateWithFlags(&op->s_d2h, cudaStreamNonBlocking));
            for (int j = 0; j < 8; ++j) PCB_CK(cudaEventCreateWithFlags(&op->ev_io[j], cudaEventDisableTiming));
        }
        for (int j = 0; j < nsub; ++j) {
            const int b0 = (int)((int64_t)B * j / nsub), b1 = (int)((int64_t)B * (j + 1) / nsub);
            const size_t off = (size_t)b0 * op->N, n = (size_t)(b1 - b0) * op->N;
            PCB_CK(cudaMemcpyAsync(op->st_in.p + off, F + off, n * sizeof(double), cudaMemcpyHostToDevice, op->s_h2d));
            PCB_CK(cudaEventRecord(op->ev_io[2 * (j & 1)], op->s_h2d));
            PCB_CK(cudaStreamWaitEvent(op->stream, op->ev_io[2 * (j & 1)], 0));
            run_batch(op, adjoint, b1 - b0, op->st_in.p + off, op->st_out.p + off, op->stream);
            PCB_CK(cudaEventRecord(op->ev_io[2 * (j & 1) + 1], op->stream));
            PCB_CK(cudaStreamWaitEvent(op->s_d2h, op->ev_io[2 * (j & 1) + 1], 0));
            PCB_CK(cudaMemcpyAsync(G + off, op->st_out.p + off, n * sizeof(double), cudaMemcpyDeviceToHost, op->s_d2h));
        }
        PCB_CK(cudaStreamSynchronize(op->s_d2h));
        PCB_CK(cudaStreamSynchronize(op->stream));
    });
}

PCB_API pcb_status pcb_apply_batch(pcb_op* op, int32_t B, const double* F, double* G) {
    return apply_host_common(op, false, B, F, G);
}
PCB_API pcb_status pcb_apply_adjoint_batch(pcb_op* op, int32_t B, const double* F, double* G) {
    return apply_host_common(op, true, B, F, G);
}

PCB_API pcb_status pcb_entries(pcb_op* op, int64_t cnt, const int64_t* y, const int64_t* x, double* out) {
    if (!op) {
        set_err("null handle");
        return PCB_EINVAL;
    }
    std::lock_guard<std::mutex> lk(op->mu);
    return guarded([&] {
        if (cnt < 0) fail(PCB_EINVAL, "pcb_entries: negative count");
        if (cnt == 0) return;
        if (!y || !x || !out) fail(PCB_EINVAL, "null pointer");
        set_device(op);
        std::vector<int64_t> yi = to_internal_points(op, y, cnt), xi = to_internal_points(op, x, cnt);
        op->st_i64a.ensure(yi.size());
        op->st_i64b.ensure(xi.size());
        op->st_out.ensure((size_t)cnt);
        op->st_flag.ensure(1);
        PCB_CK(cudaMemcpyAsync(op->st_i64a.p, yi.data(), yi.size() * 8, cudaMemcpyHostToDevice, op->stream));
        PCB_CK(cudaMemcpyAsync(op->st_i64b.p, xi.data(), xi.size() * 8, cudaMemcpyHostToDevice, op->stream));
        PCB_CK(cudaMemsetAsync(op->st_flag.p, 0, 4, op->stream));
        launch_ck(launch_entries(entry_args(op), cnt, op->st_i64a.p, op->st_i64b.p, op->st_out.p, op->st_flag.p,
                                 op->stream),
                  "entries");
        int32_t bad = 0;
        PCB_CK(cudaMemcpyAsync(out, op->st_out.p, (size_t)cnt * 8, cudaMemcpyDeviceToHost, op->stream));
        PCB_CK(cudaMemcpyAsync(&bad, op->st_flag.p, 4, cudaMemcpyDeviceToHost, op->stream));
        PCB_CK(cudaStreamSynchronize(op->stream));
        if (bad) fail(PCB_EINVAL, "PCOp::entry: index outside the domain");
    });
}

static void blocks_common(pcb_op* op, int32_t nblk, const int64_t* d_t, const int64_t* d_s, const int64_t* block_shape,
                          double* d_out, cudaStream_t st, bool host_check) {
    if (nblk < 0) fail(PCB_EINVAL, "pcb_blocks: negative block count");
    if (!block_shape) fail(PCB_EINVAL, "pcb_blocks: null block shape");
    int32_t bs[3] = {1, 1, 1};
    const int off = op->D - op->dim_user;
    for (int a = 0; a < op->D; ++a) {
        const int64_t v = a < off ? 1 : block_shape[a - off];
        if (v < 1 || v > (1 << 20)) fail(PCB_EINVAL, "pcb_blocks: bad block shape");
        bs[a] = (int32_t)v;
    }
    op->st_shape.ensure(3);
    op->st_flag.ensure(1);
    PCB_CK(cudaMemcpyAsync(op->st_shape.p, bs, sizeof(bs), cudaMemcpyHostToDevice, st));
    PCB_CK(cudaMemsetAsync(op->st_flag.p, 0, 4, st));
    launch(op, st, "blocks", [&] {
        return launch_blocks(entry_args(op), nblk, d_t, d_s, op->st_shape.p, d_out, op->st_flag.p, st);
    });
    if (host_check) {
        int32_t bad = 0;
        PCB_CK(cudaMemcpyAsync(&bad, op->st_flag.p, 4, cudaMemcpyDeviceToHost, st));
        PCB_CK(cudaStreamSynchronize(st));
        if (bad) fail(PCB_EINVAL, "PCOp::entry: index outside the domain");
    }
}

PCB_API pcb_status pcb_blocks(pcb_op* op, int32_t nblk, const int64_t* t_origin, const int64_t* s_origin,
                              const int64_t* block_shape, double* out) {
    if (!op) {
        set_err("null handle");
        return PCB_EINVAL;
    }
    std::lock_guard<std::mutex> lk(op->mu);
    return guarded([&] {
        if (nblk == 0) return;
        if (!t_origin || !s_origin || !out) fail(PCB_EINVAL, "null pointer");
        set_device(op);
        int64_t bsz = 1;
        for (int a = 0; a < op->dim_user; ++a) bsz *= block_shape[a];
        std::vector<int64_t> ti = to_internal_points(op, t_origin, nblk), si = to_internal_points(op, s_origin, nblk);
        op->st_i64a.ensure(ti.size());
        op->st_i64b.ensure(si.size());
        const size_t total = (size_t)nblk * (size_t)bsz * (size_t)bsz;
        op->st_out.ensure(total);
        PCB_CK(cudaMemcpyAsync(op->st_i64a.p, ti.data(), ti.size() * 8, cudaMemcpyHostToDevice, op->stream));
        PCB_CK(cudaMemcpyAsync(op->st_i64b.p, si.data(), si.size() * 8, cudaMemcpyHostToDevice, op->stream));
        blocks_common(op, nblk, op->st_i64a.p, op->st_i64b.p, block_shape, op->st_out.p, op->stream, true);
        PCB_CK(cudaMemcpyAsync(out, op->st_out.p, total * 8, cudaMemcpyDeviceToHost, op->stream));
        PCB_CK(cudaStreamSynchronize(op->stream));
    });
}

PCB_API pcb_status pcb_blocks_dev(pcb_op* op, int32_t nblk, const int64_t* d_t_origin, const int64_t* d_s_origin,
                                  const int64_t* block_shape, double* d_out, void* stream) {
    if (!op) {
        set_err("null handle");
        return PCB_EINVAL;
    }
    std::lock_guard<std::mutex> lk(op->mu);
    return guarded([&] {
        if (nblk == 0) return;
        if (op->dim_user != op->D) fail(PCB_EINVAL, "pcb_blocks_dev: dim-1 operators use pcb_blocks");
        set_device(op);
        blocks_common(op, nblk, d_t_origin, d_s_origin, block_shape, d_out, (cudaStream_t)stream, false);
    });
}

static void estimate_common(pcb_op* op, int32_t q, const double* dZ, const double* dY, double* dYt, int32_t nleaf,
                            const int64_t* leaf_lo, const int64_t* leaf_hi, double* eta_cells, double* eta_abs,
                            double* eta_rel, cudaStream_t st) {
    if (q < 1) fail(PCB_EINVAL, "make_probes: q >= 1 required");
    if (nleaf < 0 || (nleaf > 0 && (!leaf_lo || !leaf_hi || !eta_cells))) fail(PCB_EINVAL, "bad leaf arguments");
    run_batch(op, true, q, dZ, dYt, st);
    std::vector<int64_t> blo, bhi;
    if (nleaf > 0) {
        blo = to_internal_points(op, leaf_lo, nleaf);
        bhi = to_internal_points(op, leaf_hi, nleaf);
        // to domain-relative coordinates
        for (int32_t c = 0; c < nleaf; ++c)
            for (int a = 0; a < op->D; ++a) {
                blo[c * op->D + a] -= op->dom_lo[a];
                bhi[c * op->D + a] -= op->dom_lo[a];
            }
    }
    op->st_i64a.ensure(std::max<size_t>(1, blo.size()));
    op->st_i64b.ensure(std::max<size_t>(1, bhi.size()));
    const size_t nd2 = (size_t)(nleaf + 1) * q;
    op->st_aux.ensure(nd2 + q);
    if (!blo.empty()) {
        PCB_CK(cudaMemcpyAsync(op->st_i64a.p, blo.data(), blo.size() * 8, cudaMemcpyHostToDevice, st));
        PCB_CK(cudaMemcpyAsync(op->st_i64b.p, bhi.data(), bhi.size() * 8, cudaMemcpyHostToDevice, st));
    }
    launch(op, st, "probe_sums", [&] {
        return launch_probe_sums(op->D, op->n, nleaf, op->st_i64a.p, op->st_i64b.p, q, dYt, dY, op->st_aux.p,
                                 op->st_aux.p + nd2, st);
    });
    std::vector<double> h(nd2 + q);
    PCB_CK(cudaMemcpyAsync(h.data(), op->st_aux.p, h.size() * 8, cudaMemcpyDeviceToHost, st));
    PCB_CK(cudaStreamSynchronize(st));
    for (int32_t c = 0; c < nleaf; ++c) {
        double s = 0;
        for (int i = 0; i < q; ++i) s += h[(size_t)c * q + i];
        eta_cells[c] = std::sqrt(s / q);
    }
    double d2 = 0, y2 = 0;
    for (int i = 0; i < q; ++i) {
        d2 += h[(size_t)nleaf * q + i];
        y2 += h[nd2 + i];
    }
    if (eta_abs) *eta_abs = std::sqrt(d2 / q);
    if (eta_rel) *eta_rel = y2 > 0.0 ? std::sqrt(d2) / std::sqrt(y2) : 0.0;
}

PCB_API pcb_status pcb_probe_estimate(pcb_op* op, int32_t q, const double* Z, const double* Y, int32_t nleaf,
                                      const int64_t* leaf_lo, const int64_t* leaf_hi, double* ytilde,
                                      double* eta_cells, double* eta_abs, double* eta_rel) {
    if (!op) {
        set_err("null handle");
        return PCB_EINVAL;
    }
    std::lock_guard<std::mutex> lk(op->mu);
    return guarded([&] {
        if (!Z || !Y) fail(PCB_EINVAL, "null probe pointer");
        if (q < 1) fail(PCB_EINVAL, "make_probes: q >= 1 required");
        set_device(op);
        const size_t cnt = (size_t)q * (size_t)op->N;
        op->st_in.ensure(2 * cnt);
        op->st_out.ensure(cnt);
        PCB_CK(cudaMemcpyAsync(op->st_in.p, Z, cnt * 8, cudaMemcpyHostToDevice, op->stream));
        PCB_CK(cudaMemcpyAsync(op->st_in.p + cnt, Y, cnt * 8, cudaMemcpyHostToDevice, op->stream));
        estimate_common(op, q, op->st_in.p, op->st_in.p + cnt, op->st_out.p, nleaf, leaf_lo, leaf_hi, eta_cells,
                        eta_abs, eta_rel, op->stream);
        if (ytilde) {
            PCB_CK(cudaMemcpyAsync(ytilde, op->st_out.p, cnt * 8, cudaMemcpyDeviceToHost, op->stream));
            PCB_CK(cudaStreamSynchronize(op->stream));
        }
    });
}

PCB_API pcb_status pcb_probe_estimate_dev(pcb_op* op, int32_t q, const double* dZ, const double* dY, double* dYt,
                                          int32_t nleaf, const int64_t* leaf_lo, const int64_t* leaf_hi,
                                          double* eta_cells, double* eta_abs, double* eta_rel, void* stream) {
    if (!op) {
        set_err("null handle");
        return PCB_EINVAL;
    }
    std::lock_guard<std::mutex> lk(op->mu);
    return guarded([&] {
        if (!dZ || !dY || !dYt) fail(PCB_EINVAL, "null probe pointer");
        set_device(op);
        estimate_common(op, q, dZ, dY, dYt, nleaf, leaf_lo, leaf_hi, eta_cells, eta_abs, eta_rel,
                        (cudaStream_t)stream);
    });
}

PCB_API pcb_status pcb_profile_begin(pcb_op* op) {
    if (!op) {
        set_err("null handle");
        return PCB_EINVAL;
    }
    std::lock_guard<std::mutex> lk(op->mu);
    op->prof = true;
    return PCB_OK;
}

PCB_API pcb_status pcb_profile_end(pcb_op* op, int32_t max_kernels, char* names, double* ms_total, int32_t* launches,
                                   int32_t* n_kernels) {
    if (!op || !n_kernels) {
        set_err("null argument");
        return PCB_EINVAL;
    }
    std::lock_guard<std::mutex> lk(op->mu);
    return guarded([&] {
        set_device(op);
        std::vector<std::string> order;
        std::map<std::string, std::pair<double, int>> acc;
        for (auto& r : op->recs) {
            PCB_CK(cudaEventSynchronize(r.b));
            float ms = 0.f;
            PCB_CK(cudaEventElapsedTime(&ms, r.a, r.b));
            if (!acc.count(r.name)) order.push_back(r.name);
            acc[r.name].first += ms;
            acc[r.name].second += 1;
            op->ev_pool.push_back(r.a);
            op->ev_pool.push_back(r.b);
        }
        op->recs.clear();
        op->prof = false;
        *n_kernels = (int32_t)order.size();
        for (int32_t i = 0; i < (int32_t)order.size() && i < max_kernels; ++i) {
            if (names) {
                std::memset(names + 32 * i, 0, 32);
                std::strncpy(names + 32 * i, order[i].c_str(), 31);
            }
            if (ms_total) ms_total[i] = acc[order[i]].first;
            if (launches) launches[i] = acc[order[i]].second;
        }
    });
}

PCB_API pcb_status pcb_normal_fill(uint64_t seed, int64_t count, double* out) {
    if (count < 0 || (count > 0 && !out)) {
        set_err("pcb_normal_fill: bad arguments");
        return PCB_EINVAL;
    }
    std::mt19937_64 rng(seed);
    std::normal_distribution<double> gauss(0.0, 1.0);
    for (int64_t i = 0; i < count; ++i) out[i] = gauss(rng);
    return PCB_OK;
}

PCB_API pcb_status pcb_uniform_int_fill(uint64_t seed, int64_t lo, int64_t hi, int64_t count, int64_t* out) {
    if (count < 0 || (count > 0 && !out) || lo > hi) {
        set_err("pcb_uniform_int_fill: bad arguments");
        return PCB_EINVAL;
    }
    std::mt19937_64 rng(seed);
    std::uniform_int_distribution<int64_t> dist(lo, hi);
    for (int64_t i = 0; i < count; ++i) out[i] = dist(rng);
    return PCB_OK;
}

}  // extern "C"
