// ORACLE TEST INFRASTRUCTURE — not product code.
//
// Backend for the fftw3.h shim (see fftw3.h).  Power-of-two multi-d complex
// DFT, executed axis by axis on the row-major array viewed as
// [outer][n][inner]: butterflies combine whole contiguous "rows" of `inner`
// complex values, so strided axes stream contiguously; the last axis
// (inner == 1) is a plain iterative radix-2 line transform.  Twiddles are
// tabulated once per plan in double precision (std::cos/std::sin of
// 2*pi*j/n).  Execution keeps no mutable state in the plan, so concurrent
// fftw_execute_dft calls on one plan are safe, as the reference assumes
// (fft.hpp:11-14).
#include "fftw3.h"

#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

struct pcb_shim_fftw_plan_s {
    std::vector<int> shape;
    int sign = -1;
    std::vector<std::vector<double>> tw;  // per axis: interleaved re/im of exp(sign*2*pi*i*j/n), j < n/2
    std::vector<std::vector<std::uint32_t>> rev;  // per axis bit-reversal permutation
};

namespace {

bool is_pow2(int n) { return n >= 1 && (n & (n - 1)) == 0; }

void transform_axis(double* data, std::int64_t outer, int n, std::int64_t inner,
                    const double* tw, const std::uint32_t* rev) {
    if (n == 1) return;
    const std::int64_t row = 2 * inner;  // doubles per row
    for (std::int64_t o = 0; o < outer; ++o) {
        double* base = data + o * static_cast<std::int64_t>(n) * row;
        // bit-reversal permutation of rows
        for (int i = 0; i < n; ++i) {
            const int j = static_cast<int>(rev[i]);
            if (i < j) {
                double* a = base + static_cast<std::int64_t>(i) * row;
                double* b = base + static_cast<std::int64_t>(j) * row;
                for (std::int64_t t = 0; t < row; ++t) {
                    const double tmp = a[t];
                    a[t] = b[t];
                    b[t] = tmp;
                }
            }
        }
        // iterative radix-2 DIT butterflies
        for (int len = 2; len <= n; len <<= 1) {
            const int half = len >> 1;
            const int step = n / len;
            for (int i = 0; i < n; i += len) {
                for (int j = 0; j < half; ++j) {
                    const double wr = tw[2 * (j * step)];
                    const double wi = tw[2 * (j * step) + 1];
                    double* u = base + static_cast<std::int64_t>(i + j) * row;
                    double* v = base + static_cast<std::int64_t>(i + j + half) * row;
                    if (j == 0) {
                        for (std::int64_t t = 0; t < row; t += 2) {
                            const double ar = u[t], ai = u[t + 1];
                            const double br = v[t], bi = v[t + 1];
                            u[t] = ar + br;
                            u[t + 1] = ai + bi;
                            v[t] = ar - br;
                            v[t + 1] = ai - bi;
                        }
                    } else {
                        for (std::int64_t t = 0; t < row; t += 2) {
                            const double ar = u[t], ai = u[t + 1];
                            const double br = v[t] * wr - v[t + 1] * wi;
                            const double bi = v[t] * wi + v[t + 1] * wr;
                            u[t] = ar + br;
                            u[t + 1] = ai + bi;
                            v[t] = ar - br;
                            v[t + 1] = ai - bi;
                        }
                    }
                }
            }
        }
    }
}

}  // namespace

extern "C" fftw_plan fftw_plan_dft(int rank, const int* n, fftw_complex*, fftw_complex*, int sign,
                                   unsigned) {
    if (rank < 1 || (sign != FFTW_FORWARD && sign != FFTW_BACKWARD)) return nullptr;
    auto* p = new pcb_shim_fftw_plan_s;
    p->sign = sign;
    const double two_pi = 6.283185307179586476925286766559;
    for (int a = 0; a < rank; ++a) {
        if (!is_pow2(n[a])) {
            delete p;
            return nullptr;
        }
        p->shape.push_back(n[a]);
        const int len = n[a];
        std::vector<double> tw(static_cast<std::size_t>(len > 1 ? len : 2), 0.0);
        for (int j = 0; j < len / 2; ++j) {
            const double ang = two_pi * static_cast<double>(j) / static_cast<double>(len);
            tw[2 * j] = std::cos(ang);
            tw[2 * j + 1] = static_cast<double>(sign) * std::sin(ang);
        }
        std::vector<std::uint32_t> rev(static_cast<std::size_t>(len));
        int bits = 0;
        while ((1 << bits) < len) ++bits;
        for (int i = 0; i < len; ++i) {
            std::uint32_t r = 0;
            for (int b = 0; b < bits; ++b)
                if (i & (1 << b)) r |= 1u << (bits - 1 - b);
            rev[static_cast<std::size_t>(i)] = r;
        }
        p->tw.push_back(std::move(tw));
        p->rev.push_back(std::move(rev));
    }
    return p;
}

extern "C" void fftw_execute_dft(const fftw_plan p, fftw_complex* in, fftw_complex* out) {
    const int rank = static_cast<int>(p->shape.size());
    std::int64_t total = 1;
    for (int s : p->shape) total *= s;
    if (in != out) std::memcpy(out, in, static_cast<std::size_t>(total) * sizeof(fftw_complex));
    double* data = reinterpret_cast<double*>(out);
    for (int a = 0; a < rank; ++a) {
        std::int64_t outer = 1, inner = 1;
        for (int b = 0; b < a; ++b) outer *= p->shape[static_cast<std::size_t>(b)];
        for (int b = a + 1; b < rank; ++b) inner *= p->shape[static_cast<std::size_t>(b)];
        transform_axis(data, outer, p->shape[static_cast<std::size_t>(a)], inner,
                       p->tw[static_cast<std::size_t>(a)].data(),
                       p->rev[static_cast<std::size_t>(a)].data());
    }
}

extern "C" void fftw_destroy_plan(fftw_plan p) { delete p; }
