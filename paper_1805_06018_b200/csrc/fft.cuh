// fp64 complex line FFTs for sm_100a: register Stockham stages with shared-memory exchanges
// between stages, for line lengths L = 2^a * {1, 3, 9} (8 <= L <= 4096).
//
// A CTA transforms NL lines of length L at once.  Every thread holds E elements of one line
// (E = 16 for powers of two, E = 24 = 3 * 8 otherwise; TPL = L/E threads per line, thread
// (l, tl) with l fastest).  A stage of radix RS (RS | E) runs E/RS butterflies per thread.
// The forward transform's stage radices end with E; the inverse runs them in reverse, so it
// starts with E.  The forward leaves X[tl + r*L/E] in registers and the inverse consumes exactly
// those registers: forward -> pointwise product -> inverse needs no shared-memory round trip in
// the middle (this is what lets the frequency multiply-accumulate of the product-convolution
// apply live in registers).
//
// Stockham stage (span NS before the stage, radix RS), butterfly j in [0, L/RS):
//   inputs   x[j + r*L/RS]                       r = 0..RS-1
//   twiddle  x_r *= w^(r*(j mod NS)),  w = exp(DIR*2*pi*i/(NS*RS))
//   DFT_RS
//   outputs  y[(j/NS)*NS*RS + (j mod NS) + r*NS]
// Stage twiddles come from a per-length table tw[m] = exp(-2*pi*i*m/L) in global memory
// (computed on the host in long double, rounded once; the inverse uses the conjugate).  The
// in-register DFTs use compile-time 48th roots of unity.  All arithmetic is IEEE fp64.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#ifndef PCB_E2
#define PCB_E2 16  // elements per thread of the power-of-two engines (set per translation unit)
#endif
#ifndef PCB_E3
#define PCB_E3 24  // elements per thread of the 3-smooth engines (12 or 24)
#endif
#ifndef PCB_E2_SMALL_MAX
#define PCB_E2_SMALL_MAX 0  // power-of-two lengths <= this use 8 elements per thread (0: none)
#endif
#ifndef PCB_RADIX_DESC
#define PCB_RADIX_DESC 0  // 1: prefix stage radices in descending order
#endif
#ifndef PCB_E3_SMALL_MAX
#define PCB_E3_SMALL_MAX 0  // 3-smooth lengths <= this use 12 elements per thread (0: none)
#endif
#ifndef PCB_TW_RECUR
// Stage twiddles w^r (r = 1 .. RS-1, w = e^{-+2 pi i k / (NS RS)}): 0 loads all RS-1 from the
// table; otherwise the stage loads only w^(2^b) and forms w^r as the product of the powers in r's
// bits (<= 4 complex products, a few ulp) -- fewer live registers in the hot stages.  1: radix 16;
// 2: radix 8 and 16; 3 (default): every radix >= 4.  Measured on B200 (c3 / c4 / c2 vec/s):
// 0: 8,695 / 1,042 / 30,617; 2: 8,864 / 1,049 / 31,047; 3: 8,909 / 1,064 / 31,143 (cols 206
// instead of 224 registers at P0 = 256).
#define PCB_TW_RECUR 3
#endif
#define PCB_NS_CAT2(a, b) a##b
#define PCB_NS_CAT(a, b) PCB_NS_CAT2(a, b)

namespace pcb {
// the engine is instantiated per element count: distinct names per translation unit setting
inline namespace PCB_NS_CAT(PCB_NS_CAT(PCB_NS_CAT(e, PCB_E2), PCB_NS_CAT(_, PCB_E3)),
                            PCB_NS_CAT(PCB_NS_CAT(PCB_NS_CAT(_s, PCB_E2_SMALL_MAX), PCB_NS_CAT(_t, PCB_E3_SMALL_MAX)),
                                       PCB_NS_CAT(PCB_NS_CAT(_d, PCB_RADIX_DESC), PCB_NS_CAT(_w, PCB_TW_RECUR)))) {

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

// ---------------------------------------------------------------------------
// supported lengths and the twiddle-table layout (shared with the host)

__host__ __device__ constexpr bool is_pow2c(int v) { return v > 0 && (v & (v - 1)) == 0; }
__host__ __device__ constexpr bool fft_len_ok(int L) {
    return L >= 8 && L <= 8192 && L % 8 == 0 &&
           (is_pow2c(L) || (L % 3 == 0 && is_pow2c(L / 3)) || (L % 9 == 0 && is_pow2c(L / 9)));
}
// offset of length L's table in the concatenation of all supported lengths (ascending)
__host__ __device__ constexpr long long tw_offset(int L) {
    long long off = 0;
    for (int x = 8; x < L; x += 8)
        if (fft_len_ok(x)) off += x;
    return off;
}

// ---------------------------------------------------------------------------
// compile-time roots: cos/sin(2*pi*m/48), m = 0..47 (48 = lcm of all in-register radices)

__device__ constexpr double kC48[48] = {
    1.0, 0.99144486137381041114, 0.96592582628906828675, 0.92387953251128675613,
    0.86602540378443864676, 0.79335334029123516458, 0.70710678118654752440, 0.60876142900872063942,
    0.5, 0.38268343236508977173, 0.25881904510252076235, 0.13052619222005159155,
    0.0, -0.13052619222005159155, -0.25881904510252076235, -0.38268343236508977173,
    -0.5, -0.60876142900872063942, -0.70710678118654752440, -0.79335334029123516458,
    -0.86602540378443864676, -0.92387953251128675613, -0.96592582628906828675, -0.99144486137381041114,
    -1.0, -0.99144486137381041114, -0.96592582628906828675, -0.92387953251128675613,
    -0.86602540378443864676, -0.79335334029123516458, -0.70710678118654752440, -0.60876142900872063942,
    -0.5, -0.38268343236508977173, -0.25881904510252076235, -0.13052619222005159155,
    0.0, 0.13052619222005159155, 0.25881904510252076235, 0.38268343236508977173,
    0.5, 0.60876142900872063942, 0.70710678118654752440, 0.79335334029123516458,
    0.86602540378443864676, 0.92387953251128675613, 0.96592582628906828675, 0.99144486137381041114};

// v * exp(DIR * 2*pi*i * m / 48), m compile-time after unrolling
template <int DIR>
__device__ __forceinline__ double2 rot48(double2 v, int m) {
    m = ((m % 48) + 48) % 48;
    if (m == 0) return v;
    if (m == 24) return make_double2(-v.x, -v.y);
    if (m == 12) return DIR < 0 ? make_double2(v.y, -v.x) : make_double2(-v.y, v.x);
    if (m == 36) return DIR < 0 ? make_double2(-v.y, v.x) : make_double2(v.y, -v.x);
    const double c = kC48[m];
    const double sn = kC48[(m + 36) % 48];  // sin(2 pi m/48) = cos(2 pi (m - 12)/48)
    const double s = DIR < 0 ? -sn : sn;
    return make_double2(fma(v.x, c, -v.y * s), fma(v.x, s, v.y * c));
}

// In-register DFT of size R in {2, 4, 8, 16}: radix-2 DIF network, bit-reversed result
// permuted back to natural order.
template <int R, int DIR>
__device__ __forceinline__ void dft_pow2(double2* a) {
#pragma unroll
    for (int half = R / 2; half >= 1; half >>= 1) {
#pragma unroll
        for (int blk = 0; blk < R; blk += 2 * half) {
#pragma unroll
            for (int j = 0; j < half; ++j) {
                const double2 u = a[blk + j];
                const double2 v = a[blk + j + half];
                a[blk + j] = cadd(u, v);
                a[blk + j + half] = rot48<DIR>(csub(u, v), j * (48 / (2 * half)));
            }
        }
    }
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

template <int DIR>
__device__ __forceinline__ void dft3(double2& a, double2& b, double2& c) {
    const double s = DIR < 0 ? -0.86602540378443864676 : 0.86602540378443864676;  // DIR * sin(2 pi / 3)
    const double2 t1 = cadd(b, c);
    const double2 t2 = csub(b, c);
    const double2 m = make_double2(fma(-0.5, t1.x, a.x), fma(-0.5, t1.y, a.y));
    a = cadd(a, t1);
    b = make_double2(m.x - s * t2.y, m.y + s * t2.x);  // m + i s t2
    c = make_double2(m.x + s * t2.y, m.y - s * t2.x);  // m - i s t2
}

// In-register DFT of any size R in {2,3,4,6,8,12,16,24}.  R = 3*Q: Cooley-Tukey with
// n = Q*n1 + n2, k = k1 + 3*k2:  X[k1 + 3 k2] = sum_n2 W_Q^{n2 k2} W_R^{n2 k1} DFT3_{n1}(x[Q n1 + n2])[k1].
template <int R, int DIR>
__device__ __forceinline__ void dft(double2* a) {
    if constexpr (R % 3 != 0) {
        dft_pow2<R, DIR>(a);
    } else {
        constexpr int Q = R / 3;
        double2 y[3][Q];
#pragma unroll
        for (int n2 = 0; n2 < Q; ++n2) {
            double2 x0 = a[n2], x1 = a[Q + n2], x2 = a[2 * Q + n2];
            dft3<DIR>(x0, x1, x2);
            y[0][n2] = x0;
            y[1][n2] = rot48<DIR>(x1, n2 * (48 / R));
            y[2][n2] = rot48<DIR>(x2, 2 * n2 * (48 / R));
        }
#pragma unroll
        for (int k1 = 0; k1 < 3; ++k1) {
            if constexpr (Q > 1) dft_pow2<Q, DIR>(y[k1]);
#pragma unroll
            for (int k2 = 0; k2 < Q; ++k2) a[k1 + 3 * k2] = y[k1][k2];
        }
    }
}

// ---------------------------------------------------------------------------
// stage plans

template <int L>
struct FftCfg {
    static_assert(fft_len_ok(L) && L <= 4096, "unsupported FFT line length");
    static constexpr bool P2 = is_pow2c(L);
    static constexpr int E2L = (L <= PCB_E2_SMALL_MAX && PCB_E2 > 8) ? 8 : PCB_E2;  // per-length E (pow2)
    static constexpr int E3L = (L <= PCB_E3_SMALL_MAX && L % 12 == 0) ? 12 : PCB_E3;  // per-length E (3-smooth)
    static constexpr int R = P2 ? (L >= E2L ? E2L : L) : (L % E3L == 0 ? E3L : 24);  // elements per thread (= last radix)
    static constexpr int TPL = L / R;                        // threads per line
    // forward stage radices: the prefix factors L/R, then R
    static constexpr int pref_radix(int rest) {
        // the largest supported radix dividing both the remaining length and R (a stage never
        // exceeds, and always tiles, the elements a thread holds)
        return rest % 16 == 0 && R % 16 == 0 ? 16 : rest % 12 == 0 && R % 12 == 0 ? 12 : rest % 8 == 0 && R % 8 == 0 ? 8
               : rest % 6 == 0 && R % 6 == 0 ? 6 : rest % 4 == 0 && R % 4 == 0 ? 4 : rest % 3 == 0 && R % 3 == 0 ? 3
               : rest % 2 == 0 ? 2 : 1;
    }
    static constexpr int nstages() {
        int n = 1, rest = L / R;
        while (rest > 1) {
            rest /= pref_radix(rest);
            ++n;
        }
        return n;
    }
    static constexpr int NSTG = nstages();
    // radix of forward stage s (smallest factors first, R last)
    static constexpr int radix(int s) {
        int f[8] = {1, 1, 1, 1, 1, 1, 1, 1};
        int n = 0, rest = L / R;
        while (rest > 1) {
            const int p = pref_radix(rest);
            f[n++] = p;
            rest /= p;
        }
        // ascending prefix order keeps the first stage the smallest radix (PCB_RADIX_DESC: the
        // largest first -- its stride-RS shared-memory stores are RS * NL words apart)
        for (int i = 0; i < n; ++i)
            for (int j = i + 1; j < n; ++j)
                if (PCB_RADIX_DESC ? f[j] > f[i] : f[j] < f[i]) {
                    const int t = f[i];
                    f[i] = f[j];
                    f[j] = t;
                }
        return s < n ? f[s] : R;
    }
    static constexpr int span(int s) {  // NS before forward stage s
        int ns = 1;
        for (int i = 0; i < s; ++i) ns *= radix(i);
        return ns;
    }
};

// shared-memory word index for element i of line l; NL lines interleaved ([L][NL] layout,
// matching global column tiles) plus one pad word per 2^PS words.
template <int NL, int PS>
__device__ __forceinline__ int sidx(int i, int l) {
    const int w = i * NL + l;
    return w + (w >> PS);
}
template <int L, int NL, int PS>
struct SmemLine {
    static constexpr int WORDS = L * NL + ((L * NL) >> PS) + 1;
};

// One stage held in registers: E/RS butterflies of radix RS per thread.
template <int L, int RS, int NS, int DIR>
__device__ __forceinline__ void stage_math(double2* v, int tl, const double2* __restrict__ tw) {
    constexpr int E = FftCfg<L>::R;
    constexpr int TPL = FftCfg<L>::TPL;
#pragma unroll
    for (int b = 0; b < E / RS; ++b) {
        const int j = tl + b * TPL;
        if (NS > 1) {
            const int k = j % NS;
            constexpr int step = L / (NS * RS);
            // bits needed for r < RS, and whether this radix uses the product form at this setting
            constexpr int LB = RS > 16 ? 5 : RS > 8 ? 4 : RS > 4 ? 3 : RS > 2 ? 2 : 1;
            constexpr bool RECUR = (PCB_TW_RECUR >= 1 && RS == 16) || (PCB_TW_RECUR >= 2 && RS == 8) ||
                                   (PCB_TW_RECUR >= 3 && RS >= 4);
            if constexpr (RECUR) {
                // log2(RS) table loads instead of RS - 1 (fewer live registers): w^r = the product of
                // the loaded powers of two in r's bits (at most LB - 1 complex products, ~1 ulp each)
                double2 wp[LB];
#pragma unroll
                for (int bit = 0; bit < LB; ++bit) wp[bit] = __ldg(&tw[(1 << bit) * k * step]);
#pragma unroll
                for (int r = 1; r < RS; ++r) {
                    double2 w = make_double2(1.0, 0.0);
                    bool first = true;
#pragma unroll
                    for (int bit = 0; bit < LB; ++bit)
                        if (r & (1 << bit)) {
                            w = first ? wp[bit] : cmul(w, wp[bit]);
                            first = false;
                        }
                    v[b * RS + r] = DIR < 0 ? cmul(v[b * RS + r], w) : cmulc(v[b * RS + r], w);
                }
            } else {
#pragma unroll
                for (int r = 1; r < RS; ++r) {
                    const double2 w = __ldg(&tw[r * k * step]);
                    v[b * RS + r] = DIR < 0 ? cmul(v[b * RS + r], w) : cmulc(v[b * RS + r], w);
                }
            }
        }
        dft<RS, DIR>(&v[b * RS]);
    }
}

template <int L, int RS, int NL, int PS>
__device__ __forceinline__ void stage_load(double2* v, const double2* buf, int l, int tl) {
    constexpr int E = FftCfg<L>::R;
    constexpr int TPL = FftCfg<L>::TPL;
#pragma unroll
    for (int b = 0; b < E / RS; ++b)
#pragma unroll
        for (int r = 0; r < RS; ++r) v[b * RS + r] = buf[sidx<NL, PS>(tl + b * TPL + r * (L / RS), l)];
}

template <int L, int RS, int NS, int NL, int PS>
__device__ __forceinline__ void stage_store(const double2* v, double2* buf, int l, int tl) {
    constexpr int E = FftCfg<L>::R;
    constexpr int TPL = FftCfg<L>::TPL;
#pragma unroll
    for (int b = 0; b < E / RS; ++b) {
        const int j = tl + b * TPL;
        const int base = (j / NS) * NS * RS + (j % NS);
#pragma unroll
        for (int r = 0; r < RS; ++r) buf[sidx<NL, PS>(base + r * NS, l)] = v[b * RS + r];
    }
}

// First forward stage (span 1, no twiddles) for inputs known to vanish at positions >= m_valid:
// a butterfly whose inputs r >= 1 all lie beyond m_valid is a broadcast of its r = 0 input.
template <int L, int RS, int DIR>
__device__ __forceinline__ void stage0_pruned(double2* v, int tl, int m_valid) {
    constexpr int E = FftCfg<L>::R;
    constexpr int TPL = FftCfg<L>::TPL;
#pragma unroll
    for (int b = 0; b < E / RS; ++b) {
        const int j = tl + b * TPL;
        if (j + L / RS >= m_valid) {
#pragma unroll
            for (int r = 1; r < RS; ++r) v[b * RS + r] = v[b * RS];
        } else {
            dft<RS, DIR>(&v[b * RS]);
        }
    }
}

// forward stages s..NSTG-1; stage 0 consumes the caller's registers, the last leaves the
// result in registers
template <int L, int DIR, int NL, int PS, int s, bool PRUNE>
struct FwdStages {
    static __device__ __forceinline__ void run(double2* v, double2* buf, int l, int tl,
                                               const double2* __restrict__ tw, int m_valid) {
        constexpr int NSTG = FftCfg<L>::NSTG;
        if constexpr (s < NSTG) {
            constexpr int RS = FftCfg<L>::radix(s);
            constexpr int NS = FftCfg<L>::span(s);
            if constexpr (s > 0) {
                __syncthreads();
                stage_load<L, RS, NL, PS>(v, buf, l, tl);
            }
            if constexpr (s == 0 && PRUNE) stage0_pruned<L, RS, DIR>(v, tl, m_valid);
            else stage_math<L, RS, NS, DIR>(v, tl, tw);
            if constexpr (s + 1 < NSTG) {
                __syncthreads();
                stage_store<L, RS, NS, NL, PS>(v, buf, l, tl);
                FwdStages<L, DIR, NL, PS, s + 1, PRUNE>::run(v, buf, l, tl, tw, m_valid);
            }
        }
    }
};

// inverse-order stages (reverse of the forward radices), i = 0..NSTG-1
template <int L, int DIR, int NL, int PS, int i>
struct RevStages {
    static __device__ __forceinline__ void run(double2* v, double2* buf, int l, int tl,
                                               const double2* __restrict__ tw) {
        constexpr int NSTG = FftCfg<L>::NSTG;
        if constexpr (i < NSTG) {
            constexpr int RS = FftCfg<L>::radix(NSTG - 1 - i);
            constexpr int NS = L / FftCfg<L>::span(NSTG - i);  // product of the radices already applied
            if constexpr (i > 0) {
                __syncthreads();
                stage_load<L, RS, NL, PS>(v, buf, l, tl);
            }
            stage_math<L, RS, NS, DIR>(v, tl, tw);
            if constexpr (i + 1 < NSTG) {
                __syncthreads();
                stage_store<L, RS, NS, NL, PS>(v, buf, l, tl);
                RevStages<L, DIR, NL, PS, i + 1>::run(v, buf, l, tl, tw);
            }
        }
    }
};

// Forward-ordered transform: v holds inputs at FirstPos; on return v[r] = X[tl + r*L/E].
// Inputs at positions >= m_valid must be zero (pruned first stage).
template <int L, int DIR, int NL, int PS, bool PRUNE = false>
__device__ __forceinline__ void fft_fwd_order(double2* v, double2* buf, int l, int tl,
                                              const double2* __restrict__ tw, int m_valid = L) {
    FwdStages<L, DIR, NL, PS, 0, PRUNE>::run(v, buf, l, tl, tw, m_valid);
}

// Reverse-ordered transform: v[r] holds x[tl + r*L/E] (what fft_fwd_order leaves); on return
// the outputs sit at LastPos.
template <int L, int DIR, int NL, int PS>
__device__ __forceinline__ void fft_rev_order(double2* v, double2* buf, int l, int tl,
                                              const double2* __restrict__ tw) {
    RevStages<L, DIR, NL, PS, 0>::run(v, buf, l, tl, tw);
}

// register positions: after fft_fwd_order / before fft_rev_order, v[r] is element tl + r*L/E
template <int L>
__device__ __forceinline__ int mid_pos(int tl, int r) {
    return tl + r * (L / FftCfg<L>::R);
}

// first-stage input layout of fft_fwd_order: radix RF = radix(0)
template <int L>
struct FirstPos {
    static constexpr int RF = FftCfg<L>::radix(0);
    static __device__ __forceinline__ int pos(int tl, int b, int r) {
        return tl + b * FftCfg<L>::TPL + r * (L / RF);
    }
};

// output positions after fft_rev_order: the last inverse stage has radix RL = radix(0)
template <int L>
struct LastPos {
    static constexpr int RL = FftCfg<L>::radix(0);
    static __device__ __forceinline__ int pos(int tl, int b, int r) {
        return tl + b * FftCfg<L>::TPL + r * (L / RL);
    }
};

}  // inline namespace
}  // namespace pcb
