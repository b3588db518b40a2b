// fp64 complex line FFTs for sm_100a: register radix-16 Stockham stages with
// shared-memory exchanges between stages.
//
// A CTA transforms NL lines of length L at once with TPL = L/16 threads per
// line (thread (l, tl), l fastest).  Stage radices: one radix-R0 stage
// (R0 = L / 16^S, 1 if L is a power of 16) plus S radix-16 stages.  The
// forward transform runs R0 first and ends with a radix-16 stage whose
// outputs X[tl + r*L/16] (natural order) stay in the thread's registers; the
// inverse transform starts with a radix-16 stage that consumes exactly those
// registers, so forward -> pointwise product -> inverse needs no shared-memory
// round trip in the middle (this is what lets the frequency multiply-
// accumulate of the product-convolution apply live in registers).
//
// Stockham stage (span NS before the stage, radix RS), butterfly j in [0, L/RS):
//   inputs   x[j + r*L/RS]                       r = 0..RS-1
//   twiddle  x_r *= w^(r*(j mod NS)),  w = exp(DIR*2*pi*i/(NS*RS))
//   DFT_RS
//   outputs  y[(j/NS)*NS*RS + (j mod NS) + r*NS]
// Twiddles come from a per-length table tw[m] = exp(-2*pi*i*m/L) in global
// memory (computed on the host in long double, rounded once); inverse uses
// the conjugate.  All arithmetic is IEEE fp64.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace pcb {

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// a * conj(b)
__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, a.y * b.y), fma(a.y, b.x, -a.x * b.y));
}
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
__device__ __forceinline__ double2 czero() { return make_double2(0.0, 0.0); }

// cos/sin(2*pi*m/16), m = 0..15
__device__ constexpr double kC16[16] = {
    1.0, 0.92387953251128673848, 0.70710678118654752440, 0.38268343236508977173,
    0.0, -0.38268343236508977173, -0.70710678118654752440, -0.92387953251128673848,
    -1.0, -0.92387953251128673848, -0.70710678118654752440, -0.38268343236508977173,
    0.0, 0.38268343236508977173, 0.70710678118654752440, 0.92387953251128673848};
__device__ constexpr double kS16[16] = {
    0.0, 0.38268343236508977173, 0.70710678118654752440, 0.92387953251128673848,
    1.0, 0.92387953251128673848, 0.70710678118654752440, 0.38268343236508977173,
    0.0, -0.38268343236508977173, -0.70710678118654752440, -0.92387953251128673848,
    -1.0, -0.92387953251128673848, -0.70710678118654752440, -0.38268343236508977173};

// v * exp(DIR * 2*pi*i * m / 16), m compile-time after unrolling
template <int DIR>
__device__ __forceinline__ double2 rot16(double2 v, int m) {
    m &= 15;
    if (m == 0) return v;
    if (m == 8) return make_double2(-v.x, -v.y);
    if (m == 4) return DIR < 0 ? make_double2(v.y, -v.x) : make_double2(-v.y, v.x);
    if (m == 12) return DIR < 0 ? make_double2(-v.y, v.x) : make_double2(v.y, -v.x);
    const double c = kC16[m];
    const double s = DIR < 0 ? -kS16[m] : kS16[m];
    return make_double2(fma(v.x, c, -v.y * s), fma(v.x, s, v.y * c));
}

// In-register DFT of size R (2, 4, 8 or 16): radix-2 DIF network, bit-reversed
// result permuted back to natural order.
template <int R, int DIR>
__device__ __forceinline__ void dft(double2* a) {
#pragma unroll
    for (int half = R / 2; half >= 1; half >>= 1) {
#pragma unroll
        for (int blk = 0; blk < R; blk += 2 * half) {
#pragma unroll
            for (int j = 0; j < half; ++j) {
                const double2 u = a[blk + j];
                const double2 v = a[blk + j + half];
                a[blk + j] = cadd(u, v);
                a[blk + j + half] = rot16<DIR>(csub(u, v), j * (16 / (2 * half)));
            }
        }
    }
    // bit reversal
    double2 t[R];
#pragma unroll
    for (int i = 0; i < R; ++i) t[i] = a[i];
#pragma unroll
    for (int i = 0; i < R; ++i) {
        int r = 0;
#pragma unroll
        for (int b = 1, rb = R / 2; b < R; b <<= 1, rb >>= 1)
            if (i & b) r |= rb;
        a[r] = t[i];
    }
}

template <int L>
struct FftCfg {
    static_assert(L >= 8 && L <= 4096 && (L & (L - 1)) == 0, "line length must be 2^k, 8..4096");
    static constexpr int R = L >= 16 ? 16 : L;
    static constexpr int S = L >= 4096 ? 3 : L >= 256 ? 2 : L >= 16 ? 1 : 0;  // radix-16 stages
    static constexpr int P16 = S == 3 ? 4096 : S == 2 ? 256 : S == 1 ? 16 : 1;
    static constexpr int R0 = L / P16;  // 1 if none (for L == 8 the single stage is radix 8)
    static constexpr int TPL = L / R;   // threads per line
};

// shared-memory word index for element i of line l; NL lines interleaved
// ([L][NL] layout, matching global column tiles) plus one pad word per 2^PS
// words to break the power-of-two strides of the first Stockham stage.
template <int NL, int PS>
__device__ __forceinline__ int sidx(int i, int l) {
    const int w = i * NL + l;
    return w + (w >> PS);
}
template <int L, int NL, int PS>
struct SmemLine {
    static constexpr int WORDS = L * NL + ((L * NL) >> PS) + 1;
};

// One stage held in registers: NB = R/RS butterflies of radix RS per thread.
template <int L, int RS, int NS, int DIR>
__device__ __forceinline__ void stage_math(double2* v, int tl, const double2* __restrict__ tw) {
    constexpr int R = FftCfg<L>::R;
    constexpr int TPL = FftCfg<L>::TPL;
    constexpr int NB = R / RS;
#pragma unroll
    for (int b = 0; b < NB; ++b) {
        const int j = tl + b * TPL;
        if (NS > 1) {
            const int k = j % NS;
            constexpr int step = L / (NS * RS);
#pragma unroll
            for (int r = 1; r < RS; ++r) {
                const double2 w = __ldg(&tw[r * k * step]);
                v[b * RS + r] = DIR < 0 ? cmul(v[b * RS + r], w) : cmulc(v[b * RS + r], w);
            }
        }
        dft<RS, DIR>(&v[b * RS]);
    }
}

template <int L, int RS, int NL, int PS>
__device__ __forceinline__ void stage_load(double2* v, const double2* buf, int l, int tl) {
    constexpr int R = FftCfg<L>::R;
    constexpr int TPL = FftCfg<L>::TPL;
#pragma unroll
    for (int b = 0; b < R / RS; ++b)
#pragma unroll
        for (int r = 0; r < RS; ++r) v[b * RS + r] = buf[sidx<NL, PS>(tl + b * TPL + r * (L / RS), l)];
}

template <int L, int RS, int NS, int NL, int PS>
__device__ __forceinline__ void stage_store(const double2* v, double2* buf, int l, int tl) {
    constexpr int R = FftCfg<L>::R;
    constexpr int TPL = FftCfg<L>::TPL;
#pragma unroll
    for (int b = 0; b < R / RS; ++b) {
        const int j = tl + b * TPL;
        const int base = (j / NS) * NS * RS + (j % NS);
#pragma unroll
        for (int r = 0; r < RS; ++r) buf[sidx<NL, PS>(base + r * NS, l)] = v[b * RS + r];
    }
}

// Positions held by a thread before the first stage of a transform whose first
// stage has radix RS: element index of v[b*RS + r].
template <int L, int RS>
__device__ __forceinline__ int first_pos(int tl, int b, int r) {
    return tl + b * FftCfg<L>::TPL + r * (L / RS);
}

// Radix-16 stage s (0-based among the radix-16 stages) of the forward transform.
template <int L, int DIR, int NL, int PS, int s>
struct Fwd16Stages {
    static __device__ __forceinline__ void run(double2* v, double2* buf, int l, int tl,
                                               const double2* __restrict__ tw) {
        constexpr int R0 = FftCfg<L>::R0;
        constexpr int S = FftCfg<L>::S;
        constexpr int NS = (R0 > 1 ? R0 : 1) * (s == 0 ? 1 : s == 1 ? 16 : 256);
        if (s > 0 || R0 > 1) {
            __syncthreads();
            stage_load<L, 16, NL, PS>(v, buf, l, tl);
        }
        stage_math<L, 16, NS, DIR>(v, tl, tw);
        if (s + 1 < S) {
            __syncthreads();
            stage_store<L, 16, NS, NL, PS>(v, buf, l, tl);
            Fwd16Stages<L, DIR, NL, PS, s + 1>::run(v, buf, l, tl, tw);
        }
    }
};
template <int L, int DIR, int NL, int PS>
struct Fwd16Stages<L, DIR, NL, PS, 3> {
    static __device__ __forceinline__ void run(double2*, double2*, int, int, const double2*) {}
};

// Forward-ordered transform: v holds inputs laid out for the first stage
// (radix R0 if R0 > 1, else radix 16); on return v[r] = X[tl + r*L/16].
// For L == 8 (single radix-8 stage, one thread per line) v[r] = X[r].
template <int L, int DIR, int NL, int PS>
__device__ __forceinline__ void fft_fwd_order(double2* v, double2* buf, int l, int tl,
                                              const double2* __restrict__ tw) {
    constexpr int R0 = FftCfg<L>::R0;
    if (L == 8) {
        dft<8, DIR>(v);
        return;
    }
    if (R0 > 1) {
        stage_math<L, R0, 1, DIR>(v, tl, tw);
        __syncthreads();
        stage_store<L, R0, 1, NL, PS>(v, buf, l, tl);
    }
    Fwd16Stages<L, DIR, NL, PS, 0>::run(v, buf, l, tl, tw);
}

template <int L, int DIR, int NL, int PS, int s>
struct Inv16Stages {
    static __device__ __forceinline__ void run(double2* v, double2* buf, int l, int tl,
                                               const double2* __restrict__ tw) {
        constexpr int S = FftCfg<L>::S;
        constexpr int NS = s == 0 ? 1 : s == 1 ? 16 : 256;
        if (s > 0) {
            __syncthreads();
            stage_load<L, 16, NL, PS>(v, buf, l, tl);
        }
        stage_math<L, 16, NS, DIR>(v, tl, tw);
        if (s + 1 < S || FftCfg<L>::R0 > 1) {
            __syncthreads();
            stage_store<L, 16, NS, NL, PS>(v, buf, l, tl);
        }
        if (s + 1 < S) Inv16Stages<L, DIR, NL, PS, s + 1>::run(v, buf, l, tl, tw);
    }
};
template <int L, int DIR, int NL, int PS>
struct Inv16Stages<L, DIR, NL, PS, 3> {
    static __device__ __forceinline__ void run(double2*, double2*, int, int, const double2*) {}
};

// Reverse-ordered transform: v[r] holds x[tl + r*L/16] (the registers a
// forward-ordered transform leaves behind).  On return v holds the outputs of
// the last stage: position of v[b*RL + r] is last_pos(tl, b, r), RL = R0 if
// R0 > 1 else 16.
template <int L, int DIR, int NL, int PS>
__device__ __forceinline__ void fft_rev_order(double2* v, double2* buf, int l, int tl,
                                              const double2* __restrict__ tw) {
    constexpr int R0 = FftCfg<L>::R0;
    constexpr int S = FftCfg<L>::S;
    if (L == 8) {
        dft<8, DIR>(v);
        return;
    }
    Inv16Stages<L, DIR, NL, PS, 0>::run(v, buf, l, tl, tw);
    if (R0 > 1) {
        constexpr int NS = S == 1 ? 16 : S == 2 ? 256 : 4096;
        __syncthreads();
        stage_load<L, R0, NL, PS>(v, buf, l, tl);
        stage_math<L, R0, NS, DIR>(v, tl, tw);
    }
}

template <int L>
struct LastPos {
    static constexpr int RL = FftCfg<L>::R0 > 1 ? FftCfg<L>::R0 : FftCfg<L>::R;
    // output position of v[b*RL + r] after fft_rev_order
    static __device__ __forceinline__ int pos(int tl, int b, int r) {
        return tl + b * FftCfg<L>::TPL + r * (L / RL);
    }
};

// first-stage input layout of fft_fwd_order: radix RF = R0 if R0 > 1 else R
template <int L>
struct FirstPos {
    static constexpr int RF = FftCfg<L>::R0 > 1 ? FftCfg<L>::R0 : FftCfg<L>::R;
    static __device__ __forceinline__ int pos(int tl, int b, int r) {
        return tl + b * FftCfg<L>::TPL + r * (L / RF);
    }
};

}  // namespace pcb
