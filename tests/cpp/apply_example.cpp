// C++ host-side use of the boundary (include/pcb/operator.hpp): builds a small 2-D operator with
// random weights and kernels, applies it on the GPU and checks against the defining double sum
//   (A f)[y] = sum_k sum_x w_k[x] f[x] phi_k[y - x]   (pc_operator.cpp:45-56, test_helpers.hpp:28-40)
// and entry() against the same formula.  Exit code 0 on success.
#include <cmath>
#include <cstdio>
#include <random>

#include "pcb/operator.hpp"

int main() {
    const int n = 13, r = 4;
    pcb::Box dom{{0, 0}, {n - 1, n - 1}};
    std::mt19937_64 rng(42);
    std::uniform_real_distribution<double> u(-1.0, 1.0);
    std::vector<pcb::Field> w, phi;
    for (int k = 0; k < r; ++k) {
        pcb::Field wk{{{2 * k, 1}, {2 * k + 5, 9}}, {}};
        wk.values.resize(wk.box.num_points());
        for (double& v : wk.values) v = u(rng);
        pcb::Field pk{{{-3, -2}, {2, 4}}, {}};
        pk.values.resize(pk.box.num_points());
        for (double& v : pk.values) v = u(rng);
        w.push_back(wk);
        phi.push_back(pk);
    }
    auto at = [](const pcb::Field& f, int64_t a, int64_t b) {
        if (a < f.box.lo[0] || a > f.box.hi[0] || b < f.box.lo[1] || b > f.box.hi[1]) return 0.0;
        return f.values[(a - f.box.lo[0]) * (f.box.hi[1] - f.box.lo[1] + 1) + (b - f.box.lo[1])];
    };
    std::vector<double> f(n * n);
    for (double& v : f) v = u(rng);
    std::vector<double> want(n * n, 0.0);
    for (int k = 0; k < r; ++k)
        for (int y0 = 0; y0 < n; ++y0)
            for (int y1 = 0; y1 < n; ++y1)
                for (int x0 = 0; x0 < n; ++x0)
                    for (int x1 = 0; x1 < n; ++x1)
                        want[y0 * n + y1] += at(w[k], x0, x1) * f[x0 * n + x1] * at(phi[k], y0 - x0, y1 - x1);
    try {
        for (int mode : {PCB_MODE_GLOBAL, PCB_MODE_LOCAL}) {
            pcb_options opt;
            pcb_default_options(&opt);
            opt.mode = mode;
            pcb::ProductConvolutionOperator op(dom, w, phi, &opt);
            const std::vector<double> got = op.apply(f);
            double num = 0, den = 0;
            for (int i = 0; i < n * n; ++i) {
                num += (got[i] - want[i]) * (got[i] - want[i]);
                den += want[i] * want[i];
            }
            const double rel = std::sqrt(num / den);
            double e = op.entry({5, 6}, {4, 3}), e_want = 0;
            for (int k = 0; k < r; ++k)
                if (at(w[k], 4, 3) != 0.0) e_want += at(w[k], 4, 3) * at(phi[k], 1, 3);
            std::printf("mode %d: apply rel %.3e  entry %.17g vs %.17g\n", mode, rel, e, e_want);
            if (!(rel <= 1e-11) || e != e_want) return 1;
        }
        // shard by k with the NCCL reduce inside the library (a 1-rank communicator here: the
        // pattern every rank of a multi-GPU job runs)
        {
            const std::vector<unsigned char> id = pcb::comm_unique_id();
            const pcb_options so = pcb::shard_options(0, 1, &id, PCB_REDUCE_ALL);
            pcb::ProductConvolutionOperator sop(dom, w, phi, &so);
            const std::vector<double> got = sop.apply(f);
            double num = 0, den = 0;
            for (int i = 0; i < n * n; ++i) {
                num += (got[i] - want[i]) * (got[i] - want[i]);
                den += want[i] * want[i];
            }
            std::printf("sharded (NCCL %d, %d rank): apply rel %.3e\n", sop.info().comm_version, sop.info().comm_nranks,
                        std::sqrt(num / den));
            if (!(std::sqrt(num / den) <= 1e-11) || sop.info().comm_nranks != 1) return 4;
        }
        // pinned host buffers (pcb::pinned_vector): the copy-engine path, same result
        {
            pcb::ProductConvolutionOperator pop(dom, w, phi);
            pcb::pinned_vector pf(f.begin(), f.end()), pg;
            pop.apply_batch(pf, pg, 1);
            const std::vector<double> ref = pop.apply(f);
            for (int i = 0; i < n * n; ++i)
                if (pg[i] != ref[i]) return 5;
            std::printf("pinned_vector apply: bitwise equal to the pageable path\n");
            // an ordinary std::vector page-locked in place for the guard's lifetime
            std::vector<double> rf(f), rg(f.size());
            {
                pcb::host_registration lf(rf), lg(rg);
                pop.apply_batch(rf, rg, 1);
            }
            for (int i = 0; i < n * n; ++i)
                if (rg[i] != ref[i]) return 6;
            std::printf("host_registration apply: bitwise equal\n");
        }
        // reference error behaviour
        pcb::ProductConvolutionOperator op(dom, w, phi);
        try {
            op.entry({-1, 0}, {0, 0});
            return 2;
        } catch (const std::invalid_argument& ex) {
            std::printf("invalid_argument: %s\n", ex.what());
        }
    } catch (const std::exception& ex) {
        std::printf("error: %s\n", ex.what());
        return 3;
    }
    std::printf("OK\n");
    return 0;
}
