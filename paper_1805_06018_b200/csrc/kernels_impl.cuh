// sm_100a fp64 kernels of the product-convolution apply path (templates; instantiated by
// kernels_rows.cu, kernels_cols.cu, kernels_mid.cu; the gathers live in kernels_misc.cu).
//
//   K1  spectra build      rows_fwd<RF_SPEC> -> [mid<MM_FWD_SPEC>] -> cols<CM_SPEC>
//   K2  weight+pad+FFT     rows_fwd<RF_APPLY> (w_k . f gathered on the footprint, zero-padded,
//                          R2C along the last axis) -> [mid<MM_FWD_APPLY>] (pruned: m rows in)
//   K3  frequency MAC      cols<CM_APPLY_*> : pruned axis-0 FFT, x Phi_k, (global mode: accumulate
//                          over k in registers), axis-0 inverse — all inside one CTA per column tile
//   K4  inverse + crop     [mid<MM_INV_*>] -> rows_inv<RI_*> : C2R along the last axis, gathered
//                          per output line over the contributing terms in ascending k, cropped to Omega
//   K5  adjoint/probes     the same passes with conj(Phi_k) (rows_fwd<RF_ADJ>, cols<CM_ADJ_*>,
//                          rows_inv<RI_ADJ>), plus probe_sums for eta
//   K6  entry/block gather entries / blocks
// Reference semantics: pc_operator.cpp:45-96, fft.cpp:64-162, adaptivity.cpp:75-121.
#pragma once
#include <cstdio>

#include "fft.cuh"
#include "kernels.cuh"

// Launch shape of the last-axis passes (measured on B200, round 1): small CTAs of ~64 threads
// with 8 elements per thread and a 64-register cap (16 CTAs/SM) for the power-of-two lengths
// beat 128-thread / 16-element CTAs by 1.35x at c3; the 3-smooth (E = 24) lengths keep their
// registers.
#ifndef PCB_ROWS_THREADS
#define PCB_ROWS_THREADS 64
#endif
#ifndef PCB_ROWS_MINB
#define PCB_ROWS_MINB 16
#endif
#ifndef PCB_ROWS_MINB_B
#define PCB_ROWS_MINB_B 8
#endif
#ifndef PCB_BUNDLE_MB
#define PCB_BUNDLE_MB 1  // bundle members staged per lane at a time
#endif
#ifndef PCB_BUNDLE_DB
#define PCB_BUNDLE_DB 1  // 1: double-buffered member staging (c3 +1.7% over MB = 2 single-buffered)
#endif
#ifndef PCB_BUNDLE_XPF
#define PCB_BUNDLE_XPF 1  // 1: next batch's headers and first members issued before this batch's C2R
#endif
#ifndef PCB_COLS_MINB_SMALL
#define PCB_COLS_MINB_SMALL 10  // min CTAs/SM of the column pass for lengths <= 64 (96 registers; c4 cols -5%)
#endif
#ifndef PCB_COLS_PS4
#define PCB_COLS_PS4 1  // column pass with 4-line tiles: one pad word per 16 (conflict-free stores)
#endif
#ifndef PCB_SLS_CF
#define PCB_SLS_CF 1  // conflict-free staged-line stride in the gathers
#endif
#ifndef PCB_RINV_ALIAS
#define PCB_RINV_ALIAS 1  // per-entry gather: split straight into registers, stage doubles as FFT buffer
#endif
#ifndef PCB_BUNDLE_TWREC
#define PCB_BUNDLE_TWREC 1  // bundled gather: member phases from phase(tl) and powers of phase(TPL)
#endif
#ifndef PCB_BUNDLE_ALIAS
#define PCB_BUNDLE_ALIAS 1  // with XPF: stage buffer 1 doubles as the FFT / xs buffer (smem per CTA)
#endif
#if PCB_BUNDLE_XPF && !PCB_BUNDLE_DB
#error "PCB_BUNDLE_XPF needs PCB_BUNDLE_DB"
#endif
#ifndef PCB_ROWS_MINB_MIXED
#define PCB_ROWS_MINB_MIXED 1
#endif
#ifndef PCB_ROWS_MINB_SHORT3
#define PCB_ROWS_MINB_SHORT3 16  // short 3-smooth rows (N <= 48, one thread per line): c4 rows_inv -13%
#endif
#ifndef PCB_CHAIN_STAGE
#define PCB_CHAIN_STAGE 1  // column chains: stage each member's spectrum tile in shared memory
#endif
#ifndef PCB_LOCAL_STAGE
// LOCAL cols with columns up to this length stage the spectrum tile in shared memory (cp.async,
// overlapping the S loads and the forward FFT).  Measured: c4 (P0 = 64) cols -2%; c3 / c2
// (P0 = 192 / 256) +8% slower, so longer columns load it directly.
#define PCB_LOCAL_STAGE 64
#endif
#ifndef PCB_COLS_THREADS
#define PCB_COLS_THREADS 64
#endif
#ifndef PCB_SPLIT3_MIN
// Last-axis half lengths N = 3 * 2^a >= this run as F = 3 interleaved power-of-two sub-lines of
// M = N / 3 points on the 8-element engine (64-register row kernels), with the radix-3 butterfly
// folded into the passes that touch the data anyway: the forward gather (decimation in frequency:
// sub-line s gets y_s[j] = w_N^{sj} sum_t w_3^{st} z[j + tM], and FFT_M(y_s)[k] = Z[3k + s]) and the
// inverse's output pass (decimation in time: z[j + tM] = sum_s w_3^{-st} w_N^{-sj} IFFT_M(Z[3. + s])[j]).
// 0: the generic 24-element 3-smooth engine for every 3-smooth length.
#define PCB_SPLIT3_MIN 96
#endif
#ifndef PCB_ROWS_THREADS_S3
#define PCB_ROWS_THREADS_S3 96  // threads per CTA of the split-3 row kernels (3 sub-lines per line)
#endif
#ifndef PCB_COLS_MINB
#define PCB_COLS_MINB 1
#endif

namespace pcb {

namespace {

// one pad word per 2^PSH shared-memory (16-byte) words: with lines interleaved [L][NL], a pass
// that walks one line (k fastest) strides NL words, and NL + NL/2^PSH must be odd-ish for the
// 8 lanes of a 128-bit quarter-warp to hit distinct bank groups (NL = 2, 4, 8: 2^3; 16: 2^4; 32: 2^5)
constexpr int ilog2c(int v) { return v <= 1 ? 0 : 1 + ilog2c(v / 2); }
template <int NL>
constexpr int PSH = ilog2c(NL) > 3 ? ilog2c(NL) : 3;

// Row-pass engine of half length N: F sub-lines of M = N / F points per line (F = 1: the line itself).
template <int N>
struct RowCfg {
    static constexpr bool S3 = PCB_SPLIT3_MIN > 0 && N >= PCB_SPLIT3_MIN && N % 3 == 0 && is_pow2c(N / 3);
    static constexpr int F = S3 ? 3 : 1;
    static constexpr int M = N / F;
    static constexpr int TPL = FftCfg<M>::TPL;  // threads per sub-line
    static constexpr int R = FftCfg<M>::R;      // elements per thread
    static constexpr bool P2 = FftCfg<M>::P2;   // power-of-two engine: the 64-register launch shape
    static constexpr int THREADS = S3 ? PCB_ROWS_THREADS_S3 : PCB_ROWS_THREADS;
    // min CTAs/SM scaled to the CTA size (mb is stated for 64-thread CTAs)
    static constexpr int minb(int nl, int mb) {
        const int nt = nl * F * TPL;
        const int v = nt <= 64 ? mb : mb * 64 / nt;
        return v < 1 ? 1 : v;
    }
};

// bundled gather (aliased layout): staged-line stride, >= N + 1 and large enough that one stage
// buffer (NL lines) holds the FFT exchange buffer and the real output lines xs
template <int N, int NL>
__host__ __device__ constexpr int stage_stride_b() {
    constexpr int words = SmemLine<RowCfg<N>::M, RowCfg<N>::F * NL, PSH<RowCfg<N>::F * NL>>::WORDS;
    constexpr int xsw = (NL * (2 * N + 1) + 1) / 2;
    constexpr int need = words > xsw ? words : xsw;
    constexpr int base = (N + 1) * NL >= need ? N + 1 : (need + NL - 1) / NL;
    // lanes l of a 128-bit quarter-warp read x[l * stride + k] for 8 / NL consecutive k: with
    // stride = 8 / NL (mod 8) they fall in distinct bank groups (also for x[N - k])
    // (split-3 lines: threads are ordered (tl, s, l) with l fastest and own the bins 3 tl + s + ..., so
    // the same rule holds)
    constexpr int q = NL >= 8 ? 1 : 8 / NL;
    return PCB_SLS_CF ? base + ((q - base % 8) % 8 + 8) % 8 : base;
}

template <int LEN>
__device__ __forceinline__ const double2* twtab(const double2* tw) {
    static_assert(fft_len_ok(LEN), "no twiddle table for this length");
    return tw + tw_offset(LEN);
}

template <int LEN, int NL>
constexpr int smem_words() {
    return SmemLine<LEN, NL, PSH<NL>>::WORDS;
}
// FFT exchange buffer of a row-pass CTA: F * NL interleaved sub-lines of M points
template <int N, int NL>
constexpr int row_words() {
    return SmemLine<RowCfg<N>::M, RowCfg<N>::F * NL, PSH<RowCfg<N>::F * NL>>::WORDS;
}
// split-3 inverse, last step (decimation in time), in place on the real output lines xs: the
// sub-line results y_s[j] sit at complex position s M + j of line ll; (z[j], z[j + M], z[j + 2M]) =
// DFT3^{-1}(y_0[j], conj(w_N^j) y_1[j], conj(w_N^{2j}) y_2[j]).  One thread per (line, j): no hazards.
template <int N, int NT, int XS>
__device__ __forceinline__ void split3_time_pass(double* xs, int nlines, const double2* __restrict__ twN) {
    constexpr int M = N / 3;
    for (int idx = threadIdx.x; idx < nlines * M; idx += NT) {
        const int ll = idx / M;
        const int j = idx - ll * M;
        double* x = xs + ll * XS + 2 * j;
        double2 u0 = make_double2(x[0], x[1]);
        double2 u1 = make_double2(x[2 * M], x[2 * M + 1]);
        double2 u2 = make_double2(x[4 * M], x[4 * M + 1]);
        u1 = cmulc(u1, __ldg(&twN[j]));
        u2 = cmulc(u2, __ldg(&twN[2 * j]));
        dft3<+1>(u0, u1, u2);
        x[0] = u0.x;
        x[1] = u0.y;
        x[2 * M] = u1.x;
        x[2 * M + 1] = u1.y;
        x[4 * M] = u2.x;
        x[4 * M + 1] = u2.y;
    }
}

// pad shift of the column pass: with 4 lines per tile its first forward and first inverse stages
// store stride-16 runs (64 words apart), which one pad per 8 words maps onto the same banks
template <int NL>
constexpr int PSC = (PCB_COLS_PS4 && NL == 4) ? 4 : PSH<NL>;
template <int LEN, int NL>
constexpr int smem_words_c() {
    return SmemLine<LEN, NL, PSC<NL>>::WORDS;
}

// number of lines of one item for the rows_fwd pass
__device__ __forceinline__ int64_t rows_fwd_lines(const PassArgs& a, const TermDesc& t, int mode) {
    if (mode == RF_APPLY) return a.D == 2 ? t.m[0] : (int64_t)t.m[0] * t.m[1];
    if (mode == RF_ADJ) return a.D == 2 ? t.o_cnt[0] : (int64_t)t.o_cnt[0] * t.o_cnt[1];
    return a.D == 2 ? a.P[0] : (int64_t)a.P[0] * a.P[1];
}

__device__ __forceinline__ int64_t imod(int64_t a, int64_t p) {
    int64_t r = a % p;
    return r < 0 ? r + p : r;
}

// ---------------------------------------------------------------------------
// async global -> shared copies (LDGSTS): the gathers below issue all their loads back to back
// and wait once, instead of stalling on each dependent load.
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\n" ::);
    asm volatile("cp.async.wait_group 0;\n" ::);
}

// ---------------------------------------------------------------------------
// rows_fwd: R2C along the last axis (length P = 2N) via an N-point complex FFT
// of z[j] = x[2j] + i x[2j+1] and the usual even/odd split.  APPLY gathers
// w_k . f on the footprint window, ADJ gathers g on the output window (both
// staged through shared memory with cp.async), SPEC places the trimmed kernel.
template <int N, int NL, int MODE>
__global__ void __launch_bounds__(NL * RowCfg<N>::F * RowCfg<N>::TPL, RowCfg<N>::P2 ? RowCfg<N>::minb(NL, PCB_ROWS_MINB) : (N <= 48 ? PCB_ROWS_MINB_SHORT3 : PCB_ROWS_MINB_MIXED)) k_rows_fwd(PassArgs a) {
    using RC = RowCfg<N>;
    constexpr int F = RC::F, M = RC::M, NLS = F * NL;  // NLS interleaved sub-lines of M points
    constexpr int R = RC::R;
    constexpr int RF = FirstPos<M>::RF;
    constexpr int NT = NLS * RC::TPL;
    constexpr int PS = PSH<NLS>;
    extern __shared__ double2 buf[];
    // layout: buf [row_words] | line meta
    int64_t* m_src = reinterpret_cast<int64_t*>(buf + row_words<N, NL>());
    int64_t* m_row = m_src + NL;
    int64_t* m_w = m_row + NL;
    int* m_lo = reinterpret_cast<int*>(m_w + NL);  // valid positions [m_lo, m_hi) along the line
    int* m_hi = m_lo + NL;

    const int item = blockIdx.y;
    const bool gmode = (MODE == RF_ADJ) && a.global;
    const int nvec = MODE == RF_SPEC ? 1 : a.B;
    const int slot = gmode ? 0 : item / nvec;
    const int vec = gmode ? item : item % nvec;
    const TermDesc& td = gmode ? *a.gdesc : a.terms[a.slots[slot]];
    const int64_t nlines = rows_fwd_lines(a, td, MODE);
    const int64_t line0 = (int64_t)blockIdx.x * NL;
    if (line0 >= nlines) return;
    const int D = a.D;
    const int ax = D - 1;  // real axis

    // phase 0: per-line source / destination offsets
    if (threadIdx.x < NL) {
        const int ll = threadIdx.x;
        const int64_t line = line0 + ll;
        int64_t src = 0, row = -1, woff = 0;
        int lo = 0, hi = 0;
        if (line < nlines) {
            if (MODE == RF_APPLY) {
                int64_t c0 = line, c1 = 0;
                if (D == 3) { c0 = line / td.m[1]; c1 = line % td.m[1]; }
                const int64_t x0 = td.x_lo[0] + c0 - a.dom_lo[0];
                const int64_t x1 = D == 3 ? td.x_lo[1] + c1 - a.dom_lo[1] : 0;
                src = (int64_t)vec * a.N + (D == 3 ? (x0 * a.n[1] + x1) * a.n[2] : x0 * a.n[1]) +
                      (td.x_lo[ax] - a.dom_lo[ax]);
                woff = td.w_off + (td.wrow0 ? 0 : (D == 3 ? c0 * td.m[1] + c1 : c0) * (int64_t)td.m[ax]);
                row = D == 3 ? (c0 * td.P1 + c1) * a.W : c0 * a.W;
                lo = 0;
                hi = td.m[ax];
            } else if (MODE == RF_ADJ) {
                int64_t v0 = td.o_lo[0] + line, v1 = 0;
                if (D == 3) { v0 = td.o_lo[0] + line / td.o_cnt[1]; v1 = td.o_lo[1] + line % td.o_cnt[1]; }
                const int64_t y0 = td.s[0] + v0 - a.dom_lo[0];
                const int64_t y1 = D == 3 ? td.s[1] + v1 - a.dom_lo[1] : 0;
                src = (int64_t)vec * a.N + (D == 3 ? (y0 * a.n[1] + y1) * a.n[2] : y0 * a.n[1]) +
                      (td.s[ax] - a.dom_lo[ax]);
                row = D == 3 ? ((v0 - td.o_lo[0]) * td.P1 + v1) * a.W : (v0 - td.o_lo[0]) * a.W;
                lo = td.o_lo[ax];
                hi = td.o_lo[ax] + td.o_cnt[ax];
            } else {
                int64_t t0 = line, t1 = 0;
                if (D == 3) { t0 = line / a.P[1]; t1 = line % a.P[1]; }
                // z_a = k_lo + ((t + c - k_lo) mod P), c = s - x_lo
                const int64_t z0 = imod(t0 + td.s[0] - td.x_lo[0] - td.k_lo[0], a.P[0]);
                const int64_t z1 = D == 3 ? imod(t1 + td.s[1] - td.x_lo[1] - td.k_lo[1], a.P[1]) : 0;
                const bool ok = z0 < td.k_ext[0] && (D == 2 || z1 < td.k_ext[1]);
                src = td.phi_off + (D == 3 ? (z0 * td.k_ext[1] + z1) * td.k_ext[2] : z0 * td.k_ext[1]);
                row = D == 3 ? (t0 * a.P[1] + t1) * a.W : t0 * a.W;
                lo = 0;
                hi = ok ? 2 * N : 0;
            }
        }
        m_src[ll] = src;
        m_row[ll] = row;
        m_w[ll] = woff;
        m_lo[ll] = lo;
        m_hi[ll] = hi;
    }
    __syncthreads();

    // phase 1: z[j] = (x[2j], x[2j+1]) gathered straight into the first-stage registers
    // thread (sub-line sl = s * NL + l, tl): sub-line s of line l (F = 1: the line itself)
    const int sl = threadIdx.x % NLS;
    const int s = sl / NL;
    const int l = sl - s * NL;
    const int tl = threadIdx.x / NLS;
    double2 v[R];
    {
        const int lo = m_lo[l], hi = m_hi[l];
        const int64_t src = m_src[l];
        const int64_t wsrc = m_w[l];
        auto load_z = [&](int p) {  // z[p] = (x[2p], x[2p+1]) of line l, zero outside [lo, hi)
            double xv[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int u = 2 * p + h;
                double x = 0.0;
                if (u >= lo && u < hi) {
                    if (MODE == RF_APPLY) x = __ldg(&a.in[src + u]) * __ldg(&a.w_pool[wsrc + u]);
                    else if (MODE == RF_ADJ) x = __ldg(&a.in[src + u]);
                    else {
                        const int64_t zl = imod(u + td.s[ax] - td.x_lo[ax] - td.k_lo[ax], a.P[ax]);
                        if (zl < td.k_ext[ax]) x = a.phi_pool[src + zl];
                    }
                }
                xv[h] = x;
            }
            return make_double2(xv[0], xv[1]);
        };
        // split-3: output s of the radix-3 butterfly over (z[p], z[p + M], z[p + 2M]), times w_N^{s p}.
        // The three sub-line threads of a line read the same inputs, so the lines are staged once in
        // shared memory (stride N + 1: the NL lines fall in distinct bank groups; the FFT buffer is
        // free until the first stage's store, which follows a barrier)
        if constexpr (F == 3) {
            static_assert(NL * (N + 1) <= row_words<N, NL>(), "staged input lines exceed the FFT buffer");
            double* xin = reinterpret_cast<double*>(buf);
            for (int idx = threadIdx.x; idx < NL * 2 * N; idx += NT) {
                const int ll = idx / (2 * N);
                const int u = idx - ll * 2 * N;
                double x = 0.0;
                if (u >= m_lo[ll] && u < m_hi[ll]) {
                    if (MODE == RF_APPLY) x = __ldg(&a.in[m_src[ll] + u]) * __ldg(&a.w_pool[m_w[ll] + u]);
                    else if (MODE == RF_ADJ) x = __ldg(&a.in[m_src[ll] + u]);
                    else {
                        const int64_t zl = imod(u + td.s[ax] - td.x_lo[ax] - td.k_lo[ax], a.P[ax]);
                        if (zl < td.k_ext[ax]) x = a.phi_pool[m_src[ll] + zl];
                    }
                }
                xin[ll * 2 * (N + 1) + u] = x;
            }
            __syncthreads();
        }
        const double c3 = s == 0 ? 0.0 : s == 1 ? 0.86602540378443864676 : -0.86602540378443864676;
        const double h3 = s == 0 ? 1.0 : -0.5;
        const double2* twN = twtab<N>(a.tw);
#pragma unroll
        for (int b = 0; b < R / RF; ++b)
#pragma unroll
            for (int r = 0; r < RF; ++r) {
                const int p = FirstPos<M>::pos(tl, b, r);
                if constexpr (F == 1) {
                    v[b * RF + r] = load_z(p);
                } else {
                    const double2* zin = buf + l * (N + 1);
                    const double2 z0 = zin[p], z1 = zin[p + M], z2 = zin[p + 2 * M];
                    const double2 t1 = cadd(z1, z2), t2 = csub(z1, z2);
                    const double2 y = make_double2(fma(c3, t2.y, fma(h3, t1.x, z0.x)), fma(-c3, t2.x, fma(h3, t1.y, z0.y)));
                    v[b * RF + r] = s == 0 ? y : cmul(y, __ldg(&twN[s * p]));
                }
            }
    }
    fft_fwd_order<M, -1, NLS, PS>(v, buf, sl, tl, twtab<M>(a.tw));
    __syncthreads();
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int pos = mid_pos<M>(tl, r);
        buf[sidx<NLS, PS>(pos, sl)] = v[r];
    }
    __syncthreads();
    // Z[k] of line ll: element k / F of its sub-line k % F
    auto zat = [&](int k, int ll) { return buf[sidx<NLS, PS>(k / F, (k % F) * NL + ll)]; };

    // phase 3: even/odd split X[k] = A[k] + W^k B[k], k = 0..N
    const double2* twP = twtab<2 * N>(a.tw);
    double2* S_item = MODE == RF_SPEC ? a.S + (int64_t)item * a.S_stride : a.S + td.s_pool + vec * td.s_vst;
    // k and N - k from the same two loads: A(N-k) = conj A(k), B(N-k) = conj B(k) exactly (IEEE
    // sums commute, negation is exact), so X[N-k] = conj A + W^(N-k) conj B; k = 0 also gives X[N]
    constexpr int NH = N / 2 + 1;
    for (int idx = threadIdx.x; idx < NL * NH; idx += NT) {
        const int ll = idx / NH;
        const int k = idx - ll * NH;
        const int64_t row = m_row[ll];
        if (row < 0) continue;
        const double2 zk = zat(k, ll);
        const double2 zn = zat(k == 0 ? 0 : N - k, ll);
        const double2 A = make_double2(0.5 * (zk.x + zn.x), 0.5 * (zk.y - zn.y));
        const double2 Bm = make_double2(0.5 * (zk.y + zn.y), -0.5 * (zk.x - zn.x));  // (zk - conj zn)/(2i)
        const double2 wk = __ldg(&twP[k]);
        S_item[row + k] = cadd(A, cmul(wk, Bm));
        if (k == 0) {
            S_item[row + N] = cadd(A, cmul(make_double2(-1.0, 0.0), Bm));  // W^N = -1
        } else if (2 * k != N) {
            // W^(N-k) = -conj(W^k) (P = 2N): no second table load
            const double2 Ac = make_double2(A.x, -A.y), Bc = make_double2(Bm.x, -Bm.y);
            S_item[row + N - k] = cadd(Ac, cmul(make_double2(-wk.x, wk.y), Bc));
        }
    }
}

// ---------------------------------------------------------------------------
// mid: complex FFT along axis 1 of 3D data [planes][P1][W], lines = columns c2.
template <int P1, int NL, int MODE>
__global__ void __launch_bounds__(NL * FftCfg<P1>::TPL) k_mid(PassArgs a) {
    constexpr int R = FftCfg<P1>::R;
    constexpr int RF = FirstPos<P1>::RF;
    constexpr int RL = LastPos<P1>::RL;
    extern __shared__ double2 buf[];
    const bool fwd = MODE <= MM_FWD_SPEC;
    const bool gmode = a.global && (MODE == MM_INV_APPLY || MODE == MM_FWD_ADJ);
    const int nvec = MODE == MM_FWD_SPEC ? 1 : a.B;
    const int item = blockIdx.z;
    const int slot = gmode ? 0 : item / nvec;
    const int vec = gmode ? item : item % nvec;
    const TermDesc& td = gmode ? *a.gdesc : a.terms[a.slots[slot]];
    int64_t planes;
    int in_lo = 0, in_cnt = P1, keep_lo = 0, keep_cnt = P1;
    if (MODE == MM_FWD_APPLY) { planes = td.m[0]; in_cnt = td.m[1]; }
    else if (MODE == MM_FWD_ADJ) { planes = td.o_cnt[0]; in_lo = td.o_lo[1]; in_cnt = td.o_cnt[1]; }
    else if (MODE == MM_FWD_SPEC) { planes = a.P[0]; }
    else if (MODE == MM_INV_APPLY) { planes = td.o_cnt[0]; keep_lo = td.o_lo[1]; keep_cnt = td.o_cnt[1]; }
    else { planes = td.m[0]; keep_cnt = td.m[1]; }
    const int64_t plane = blockIdx.y;
    if (plane >= planes) return;
    const int l = threadIdx.x % NL;
    const int tl = threadIdx.x / NL;
    const int64_t c = (int64_t)blockIdx.x * NL + l;
    const bool cvalid = c < a.W;
    double2* base = (MODE == MM_FWD_SPEC ? a.S + (int64_t)item * a.S_stride
                                         : fwd ? a.S + td.s_pool + vec * td.s_vst : a.T + td.t_pool + vec * td.t_vst) +
                    plane * (int64_t)a.P[1] * a.W + c;
    double2 v[R];
    if (fwd) {
        // family term: the input lines are the family's shared rows scaled by A_k(plane, line)
        const bool fam = MODE == MM_FWD_APPLY && td.a_off >= 0;
        // adjoint family term: its input lines [in_lo, in_lo + in_cnt) are the family's rows of g
        const bool afam = MODE == MM_FWD_ADJ && td.af_off >= 0;
        const double2* src = fam ? a.S + td.f_off + vec * td.f_vst + plane * (int64_t)td.f_ps * a.W + c
                           : afam ? a.S + td.af_off + vec * td.af_vst + plane * (int64_t)td.af_ps * a.W + c -
                                        (int64_t)in_lo * a.W
                                  : base;
        double sc[R];
        if (fam) {
            const double* av = a.a_pool + td.a_off + plane * (int64_t)td.m[1];
#pragma unroll
            for (int b = 0; b < R / RF; ++b)
#pragma unroll
                for (int r = 0; r < RF; ++r) {
                    const int p = FirstPos<P1>::pos(tl, b, r);
                    sc[b * RF + r] = (p >= in_lo && p < in_lo + in_cnt) ? __ldg(&av[p]) : 0.0;
                }
        }
#pragma unroll
        for (int b = 0; b < R / RF; ++b)
#pragma unroll
            for (int r = 0; r < RF; ++r) {
                const int p = FirstPos<P1>::pos(tl, b, r);
                v[b * RF + r] = (cvalid && p >= in_lo && p < in_lo + in_cnt) ? src[(int64_t)p * a.W] : czero();
            }
        if (fam) {
#pragma unroll
            for (int r = 0; r < R; ++r) v[r] = cscale(v[r], sc[r]);
        }
        fft_fwd_order<P1, -1, NL, PSH<NL>>(v, buf, l, tl, twtab<P1>(a.tw));
        if (cvalid) {
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int pos = mid_pos<P1>(tl, r);
                base[(int64_t)pos * a.W] = v[r];
            }
        }
    } else {
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int pos = mid_pos<P1>(tl, r);
            v[r] = cvalid ? base[(int64_t)pos * a.W] : czero();
        }
        fft_rev_order<P1, +1, NL, PSH<NL>>(v, buf, l, tl, twtab<P1>(a.tw));
        if (cvalid) {
#pragma unroll
            for (int b = 0; b < R / RL; ++b)
#pragma unroll
                for (int r = 0; r < RL; ++r) {
                    const int p = LastPos<P1>::pos(tl, b, r);
                    if (p >= keep_lo && p < keep_lo + keep_cnt) base[(int64_t)(p - keep_lo) * a.W] = v[b * RL + r];
                }
        }
    }
}

// ---------------------------------------------------------------------------
// cols: axis-0 pass with the frequency-domain product (K3).
#ifdef PCB_COLS_MAXNREG  // A/B: a register ceiling for the long-column pass (occupancy vs load batching)
#define PCB_COLS_BOUNDS(P0, NL) __launch_bounds__(NL * FftCfg<P0>::TPL, P0 <= 64 ? PCB_COLS_MINB_SMALL : 1) \
    __maxnreg__(P0 <= 64 ? 255 : PCB_COLS_MAXNREG)
#else
#define PCB_COLS_BOUNDS(P0, NL) __launch_bounds__(NL * FftCfg<P0>::TPL, P0 <= 64 ? PCB_COLS_MINB_SMALL : PCB_COLS_MINB)
#endif
template <int P0, int NL, int MODE>
__global__ void PCB_COLS_BOUNDS(P0, NL) k_cols(PassArgs a) {
    constexpr int R = FftCfg<P0>::R;
    constexpr int RF = FirstPos<P0>::RF;
    constexpr int RL = LastPos<P0>::RL;
    extern __shared__ double2 buf[];
    const bool global = MODE == CM_APPLY_GLOBAL || MODE == CM_ADJ_GLOBAL;
    const int nvec = MODE == CM_SPEC ? 1 : a.B;
    const int item = blockIdx.y;
    const int l = threadIdx.x % NL;
    const int tl = threadIdx.x / NL;
    const int64_t c0 = (int64_t)blockIdx.x * NL;
    const int64_t c = c0 + l;
    const bool cvalid = c < a.L;
    const int64_t tile_off = (c0 / NL) * (int64_t)P0 * NL + l;  // spectrum tile-major offset
    const double2* tw0 = twtab<P0>(a.tw);

    auto load_in = [&](const double2* src, int in_lo, int in_cnt, double2* v) {
#pragma unroll
        for (int b = 0; b < R / RF; ++b)
#pragma unroll
            for (int r = 0; r < RF; ++r) {
                const int p = FirstPos<P0>::pos(tl, b, r);
                v[b * RF + r] = (cvalid && p >= in_lo && p < in_lo + in_cnt) ? src[(int64_t)(p - in_lo) * a.L + c]
                                                                              : czero();
            }
    };
    auto store_out = [&](double2* dst, int keep_lo, int keep_cnt, const double2* v) {
        if (!cvalid) return;
#pragma unroll
        for (int b = 0; b < R / RL; ++b)
#pragma unroll
            for (int r = 0; r < RL; ++r) {
                const int p = LastPos<P0>::pos(tl, b, r);
                if (p >= keep_lo && p < keep_lo + keep_cnt) dst[(int64_t)(p - keep_lo) * a.L + c] = v[b * RL + r];
            }
    };
    auto fpos = [&](int r) { return mid_pos<P0>(tl, r); };
    // apply input of term td, vector vec: its S rows, or (2-D family term) the family's shared rows
    // scaled by A_k(row).  All row and factor loads are issued before the first multiply.
    auto load_apply = [&](const TermDesc& td, int vec, double2* v) {
        const bool fam = td.cols_f != 0;
        double sc[R];
        if (fam) {
            const double* av = a.a_pool + td.a_off;
#pragma unroll
            for (int b = 0; b < R / RF; ++b)
#pragma unroll
                for (int r = 0; r < RF; ++r) {
                    const int p = FirstPos<P0>::pos(tl, b, r);
                    sc[b * RF + r] = p < td.m[0] ? __ldg(&av[p]) : 0.0;
                }
        }
        load_in(fam ? a.S + td.f_off + vec * td.f_vst : a.S + td.s_pool + vec * td.s_vst, 0, td.m[0], v);
        if (fam) {
#pragma unroll
            for (int r = 0; r < R; ++r) v[r] = cscale(v[r], sc[r]);
        }
    };

    double2 v[R];
    if (MODE == CM_SPEC || MODE == CM_APPLY_LOCAL || MODE == CM_ADJ_LOCAL) {
        const int slot = item / nvec;
        const TermDesc& td = a.terms[a.slots[slot]];
        const int vec = item % nvec;
        const double2* S_item = MODE == CM_SPEC ? a.S + (int64_t)item * a.S_stride : a.S + td.s_pool + vec * td.s_vst;
        // LOCAL: the term's spectrum tile streams into shared memory while the S rows load and the
        // forward FFT runs (no registers held for it until the multiply)
        constexpr bool LSTAGE = MODE != CM_SPEC && P0 <= PCB_LOCAL_STAGE;
        double2* sspec = buf + smem_words_c<P0, NL>();
        if (LSTAGE) {
            const double2* tile = a.spec_pool + td.spec_off + (c0 / NL) * (int64_t)P0 * NL;
            for (int i = threadIdx.x; i < P0 * NL; i += NL * FftCfg<P0>::TPL) cp_async16(&sspec[i], tile + i);
            asm volatile("cp.async.commit_group;\n" ::);
        }
        if (MODE == CM_SPEC) load_in(S_item, 0, P0, v);
        else if (MODE == CM_APPLY_LOCAL) {
            // family term: the shared rows scaled by its lead factor (all loads before the multiply)
            const bool fam = td.cols_f != 0;
            double sc[R];
            if (fam) {
                const double* av = a.a_pool + td.a_off;
#pragma unroll
                for (int b = 0; b < R / RF; ++b)
#pragma unroll
                    for (int r = 0; r < RF; ++r) {
                        const int p = FirstPos<P0>::pos(tl, b, r);
                        sc[b * RF + r] = p < td.m[0] ? __ldg(&av[p]) : 0.0;
                    }
            }
            load_in(fam ? a.S + td.f_off + vec * td.f_vst : S_item, 0, td.m[0], v);
            if (fam) {
#pragma unroll
                for (int r = 0; r < R; ++r) v[r] = cscale(v[r], sc[r]);
            }
        }
        else load_in(a.D == 2 && td.af_off >= 0 ? a.S + td.af_off + vec * td.af_vst : S_item, td.o_lo[0], td.o_cnt[0], v);
        fft_fwd_order<P0, -1, NL, PSC<NL>>(v, buf, l, tl, tw0);
        double2* spec = a.spec_pool + td.spec_off + tile_off;
        if (MODE == CM_SPEC) {
            if (cvalid) {
#pragma unroll
                for (int r = 0; r < R; ++r) spec[(int64_t)fpos(r) * NL] = v[r];
            }
            return;
        }
        if (LSTAGE) {
            asm volatile("cp.async.wait_group 0;\n" ::);
            __syncthreads();
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const double2 ph = LSTAGE ? sspec[fpos(r) * NL + l] : cvalid ? __ldg(&spec[(int64_t)fpos(r) * NL]) : czero();
            v[r] = MODE == CM_APPLY_LOCAL ? cmul(v[r], ph) : cmulc(v[r], ph);
        }
        fft_rev_order<P0, +1, NL, PSC<NL>>(v, buf, l, tl, tw0);
        double2* T_item = a.T + td.t_pool + vec * td.t_vst;
        if (MODE == CM_APPLY_LOCAL) store_out(T_item, td.o_lo[0], td.o_cnt[0], v);
        else store_out(T_item, 0, td.m[0], v);
        return;
    }

    if (MODE == CM_APPLY_CHAIN) {
        // column chain: the members' products FFT(w_k f) . Phi_k (each Phi_k placed at the chain
        // origin) summed in registers, one inverse per (chain, vector, column tile)
        double2* sspec = buf + smem_words_c<P0, NL>();
        const int slot = item / nvec;
        const int vec = item % nvec;
        const int cid = a.slots[slot];
        const TermDesc& ch = a.chains[cid];
        double2 acc[R];
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r] = czero();
        constexpr bool STAGE = PCB_CHAIN_STAGE && P0 <= 512;
        const int m_end = a.chain_ptr[cid + 1];
        for (int mi = a.chain_ptr[cid]; mi < m_end; ++mi) {
            const TermDesc& td = a.terms[a.chain_terms[mi]];
            const double2* tile = a.spec_pool + td.spec_off + (c0 / NL) * (int64_t)P0 * NL;
            if (STAGE) {
                __syncthreads();  // previous member's product finished reading sspec
                for (int i = threadIdx.x; i < P0 * NL; i += NL * FftCfg<P0>::TPL) cp_async16(&sspec[i], tile + i);
                asm volatile("cp.async.commit_group;\n" ::);
            }
            load_apply(td, vec, v);
            fft_fwd_order<P0, -1, NL, PSC<NL>>(v, buf, l, tl, tw0);
            if (STAGE) {
                asm volatile("cp.async.wait_group 0;\n" ::);
                __syncthreads();
#pragma unroll
                for (int r = 0; r < R; ++r) acc[r] = cadd(acc[r], cmul(v[r], sspec[fpos(r) * NL + l]));
            } else {
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const double2 ph = cvalid ? __ldg(&tile[(int64_t)fpos(r) * NL + l]) : czero();
                    acc[r] = cadd(acc[r], cmul(v[r], ph));
                }
            }
        }
        fft_rev_order<P0, +1, NL, PSC<NL>>(acc, buf, l, tl, tw0);
        store_out(a.T + ch.t_pool + vec * ch.t_vst, ch.o_lo[0], ch.o_cnt[0], acc);
        return;
    }

    if (MODE == CM_APPLY_GLOBAL) {
        // Phi_k tile (P0 x NL contiguous, tile-major) streamed into shared memory with async copies
        // issued before the term's forward FFT, so the HBM stream overlaps the transform
        double2* sspec = buf + smem_words_c<P0, NL>();
        const int vec = item;
        double2 acc[R];
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r] = czero();
        constexpr bool STAGE = P0 <= 512;  // long columns: direct loads measured faster (c3 GLOBAL)
        for (int slot = 0; slot < a.n_slots; ++slot) {
            const TermDesc& td = a.terms[a.slots[slot]];
            const double2* tile = a.spec_pool + td.spec_off + (c0 / NL) * (int64_t)P0 * NL;
            if (STAGE) {
                __syncthreads();  // previous term's product finished reading sspec
                for (int i = threadIdx.x; i < P0 * NL; i += NL * FftCfg<P0>::TPL) cp_async16(&sspec[i], tile + i);
                asm volatile("cp.async.commit_group;\n" ::);
            }
            const double2* S_item = a.S + td.s_pool + vec * td.s_vst;
            load_in(S_item, 0, td.m[0], v);
            fft_fwd_order<P0, -1, NL, PSC<NL>, true>(v, buf, l, tl, tw0, td.m[0]);
            if (STAGE) {
                asm volatile("cp.async.wait_group 0;\n" ::);
                __syncthreads();
#pragma unroll
                for (int r = 0; r < R; ++r) acc[r] = cadd(acc[r], cmul(v[r], sspec[fpos(r) * NL + l]));
            } else {
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const double2 ph = cvalid ? __ldg(&tile[(int64_t)fpos(r) * NL + l]) : czero();
                    acc[r] = cadd(acc[r], cmul(v[r], ph));
                }
            }
        }
        fft_rev_order<P0, +1, NL, PSC<NL>>(acc, buf, l, tl, tw0);
        const TermDesc& g = *a.gdesc;
        store_out(a.T + g.t_pool + vec * g.t_vst, g.o_lo[0], g.o_cnt[0], acc);
        return;
    }

    // CM_ADJ_GLOBAL: one forward transform of g, one pruned inverse per term; Phi_{k+1}'s tile
    // streams into the other shared buffer while term k's inverse runs
    {
        double2* sspec = buf + smem_words_c<P0, NL>();
        const int vec = item;
        const TermDesc& g = *a.gdesc;
        double2 x[R];
        load_in(a.S + g.s_pool + vec * g.s_vst, g.o_lo[0], g.o_cnt[0], x);
        auto issue = [&](int slot) {
            const TermDesc& td = a.terms[a.slots[slot]];
            const double2* tile = a.spec_pool + td.spec_off + (c0 / NL) * (int64_t)P0 * NL;
            double2* dst = sspec + (slot & 1) * P0 * NL;
            for (int i = threadIdx.x; i < P0 * NL; i += NL * FftCfg<P0>::TPL) cp_async16(&dst[i], tile + i);
            asm volatile("cp.async.commit_group;\n" ::);
        };
        if (a.n_slots > 0) issue(0);
        fft_fwd_order<P0, -1, NL, PSC<NL>>(x, buf, l, tl, tw0);
        for (int slot = 0; slot < a.n_slots; ++slot) {
            const TermDesc& td = a.terms[a.slots[slot]];
            asm volatile("cp.async.wait_group 0;\n" ::);
            __syncthreads();  // tile `slot` landed; the other buffer is free again
            if (slot + 1 < a.n_slots) issue(slot + 1);
            const double2* sp = sspec + (slot & 1) * P0 * NL;
#pragma unroll
            for (int r = 0; r < R; ++r) v[r] = cmulc(x[r], sp[fpos(r) * NL + l]);
            fft_rev_order<P0, +1, NL, PSC<NL>>(v, buf, l, tl, tw0);
            store_out(a.T + td.t_pool + vec * td.t_vst, 0, td.m[0], v);
        }
    }
}

// ---------------------------------------------------------------------------
// rows_inv: C2R along the last axis for every T line contributing to one output
// line (CSR, ascending k), cropped and accumulated in a fixed order.  Entry
// metadata is staged in shared memory per batch of NL lines; thread t owns the
// output positions p = t mod blockDim, so contributions to one position are
// added by one thread in ascending entry order (deterministic, no atomics).
template <int N, int NL, int MODE>
__global__ void __launch_bounds__(NL * RowCfg<N>::F * RowCfg<N>::TPL, RowCfg<N>::P2 ? RowCfg<N>::minb(NL, PCB_ROWS_MINB) : (N <= 48 ? PCB_ROWS_MINB_SHORT3 : PCB_ROWS_MINB_MIXED)) k_rows_inv(PassArgs a) {
    using RC = RowCfg<N>;
    constexpr int F = RC::F, M = RC::M, NLS = F * NL;  // NLS interleaved sub-lines of M points
    constexpr int R = RC::R;
    constexpr int RL = LastPos<M>::RL;
    constexpr int NT = NLS * RC::TPL;
    constexpr int XS = 2 * N + 1;  // padded real line stride: conflict-free column writes
    constexpr int BUFW = row_words<N, NL>() > (NL * (2 * N + 1) + 1) / 2 ? row_words<N, NL>()
                                                                        : (NL * (2 * N + 1) + 1) / 2;
    extern __shared__ double2 buf[];
    const int64_t aline = blockIdx.x;
    const int vec = blockIdx.y;
    const int ax = a.D - 1;
    const int64_t line = a.line_id[aline];
    const int ulo = a.line_rng[2 * aline], uhi = a.line_rng[2 * aline + 1];
#if PCB_RINV_ALIAS
    // layout: stage [NL][SLS] (also the FFT exchange / xs buffer) | acc [n_last] | meta [NL].  The
    // even/odd split reads the staged lines straight into the inverse FFT's registers, so the
    // stage is free for the transform (one buffer less per CTA)
    constexpr int SLS = stage_stride_b<N, NL>();
    double2* stage = buf;
    double2* fbuf = buf;
    double* acc = reinterpret_cast<double*>(stage + NL * SLS);
#else
    // layout: buf [BUFW] (FFT; reused as xs) | stage [NL][N+1] | acc [n_last] | meta [NL]
    constexpr int SLS = N + 1;
    double2* fbuf = buf;
    double2* stage = buf + BUFW;
    double* acc = reinterpret_cast<double*>(stage + NL * (N + 1));
#endif
    double* xs = reinterpret_cast<double*>(fbuf);
    GatherEntry* meta = reinterpret_cast<GatherEntry*>(acc + a.n[ax] + (a.n[ax] & 1));
    const int64_t e_beg = a.line_ptr[aline];
    const int64_t e_end = a.line_ptr[aline + 1];
    const double2* twP = twtab<2 * N>(a.tw);
    const int sl = threadIdx.x % NLS;  // sub-line s of staged line l (F = 1: the line itself)
    const int s = sl / NL;
    const int l = sl - s * NL;
    const int tl = threadIdx.x / NLS;
    for (int i = ulo + threadIdx.x; i < uhi; i += NT) acc[i - ulo] = 0.0;

    for (int64_t e0 = e_beg; e0 < e_end; e0 += NL) {
        const int ne = (int)((e_end - e0) < NL ? (e_end - e0) : NL);
        __syncthreads();  // previous batch finished with meta / xs
        if (threadIdx.x < ne) meta[threadIdx.x] = a.entries[e0 + threadIdx.x];
        __syncthreads();
        for (int idx = threadIdx.x; idx < ne * (N + 1); idx += NT) {
            const int ll = idx / (N + 1);
            const int k = idx - ll * (N + 1);
            cp_async16(&stage[ll * SLS + k], a.T + meta[ll].t_off + vec * meta[ll].t_vst + k);
        }
        cp_async_wait_all();
        __syncthreads();
        double2 v[R];
#if PCB_RINV_ALIAS
#pragma unroll
        for (int r = 0; r < R; ++r) {  // z[k], k = F mid_pos(tl, r) + s, of line l: the FFT's input registers
            const int k = F * mid_pos<M>(tl, r) + s;
            double2 z = czero();
            if (l < ne) {
                const double2 xk = stage[l * SLS + k];
                const double2 xn = stage[l * SLS + N - k];
                const double2 E = make_double2(xk.x + xn.x, xk.y - xn.y);   // X[k] + conj X[N-k]
                const double2 Dd = make_double2(xk.x - xn.x, xk.y + xn.y);  // X[k] - conj X[N-k]
                const double2 O = cmulc(Dd, __ldg(&twP[k]));                // * exp(+2 pi i k / P)
                z = make_double2(E.x - O.y, E.y + O.x);                     // E + i O
            }
            v[r] = z;
        }
        __syncthreads();  // the stage is read out: the transform may reuse it
#else
        for (int idx = threadIdx.x; idx < NL * N; idx += NT) {
            const int ll = idx / N;
            const int k = idx - ll * N;
            double2 z = czero();
            if (ll < ne) {
                const double2 xk = stage[ll * (N + 1) + k];
                const double2 xn = stage[ll * (N + 1) + N - k];
                const double2 E = make_double2(xk.x + xn.x, xk.y - xn.y);   // X[k] + conj X[N-k]
                const double2 Dd = make_double2(xk.x - xn.x, xk.y + xn.y);  // X[k] - conj X[N-k]
                const double2 O = cmulc(Dd, __ldg(&twP[k]));                // * exp(+2 pi i k / P)
                z = make_double2(E.x - O.y, E.y + O.x);                     // E + i O
            }
            static_assert(F == 1, "the unaliased per-entry gather has no split-3 path");
            buf[sidx<NL, PSH<NL>>(k, ll)] = z;
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int pos = mid_pos<N>(tl, r);
            v[r] = buf[sidx<NL, PSH<NL>>(pos, l)];
        }
#endif
        fft_rev_order<M, +1, NLS, PSH<NLS>>(v, fbuf, sl, tl, twtab<M>(a.tw));
        __syncthreads();
#pragma unroll
        for (int bb = 0; bb < R / RL; ++bb)
#pragma unroll
            for (int r = 0; r < RL; ++r) {
                const int p = s * M + LastPos<M>::pos(tl, bb, r);
                xs[l * XS + 2 * p] = v[bb * RL + r].x;
                xs[l * XS + 2 * p + 1] = v[bb * RL + r].y;
            }
        __syncthreads();
        if constexpr (F == 3) {
            split3_time_pass<N, NT, XS>(xs, ne, twtab<N>(a.tw));
            __syncthreads();
        }
        for (int ll = 0; ll < ne; ++ll) {
            const int lo = meta[ll].lo, hi = meta[ll].hi;
            const double* x = xs + ll * XS - meta[ll].sh;
            int p = lo + (int)((threadIdx.x + NT - (unsigned)(lo % NT)) % NT);
            const double sc = meta[ll].scale;
            if (MODE == RI_APPLY) {
                for (; p < hi; p += NT) acc[p - ulo] += x[p] * sc;
            } else {
                const double* w = a.w_pool + meta[ll].w_off;
                for (; p < hi; p += NT) acc[p - ulo] += w[p] * (x[p] * sc);
            }
        }
    }
    __syncthreads();
    double* g = a.out + (int64_t)vec * a.N + line * a.n[ax];
    for (int i = ulo + threadIdx.x; i < uhi; i += NT) g[i] = a.accumulate ? g[i] + acc[i - ulo] : acc[i - ulo];
}

// ---------------------------------------------------------------------------
// rows_inv, LOCAL apply, frequency-domain bundles (BundleMember).  Lane l of the CTA owns one
// bundle of the batch.  Members are staged MB at a time per lane with cp.async (MB * NL lines in
// flight per CTA), summed into the lane's half spectrum in registers -- scale * T[k] *
// exp(-2 pi i k delta / P) -- then one C2R per bundle and one add of its range into the output
// line.  Members are summed in CSR order, bundles in CSR order: deterministic.
// ADJ: the 2-D adjoint's family bundles -- members of one row family covering the output line,
// scaled by A_k(line) / prod P (no phase: one placement), summed, transformed once, and the
// result multiplied by the family's last-axis weight row c (header w_off) as it accumulates.
template <int N, int NL, int ADJ>
__global__ void __launch_bounds__(NL * RowCfg<N>::F * RowCfg<N>::TPL, RowCfg<N>::P2 ? RowCfg<N>::minb(NL, PCB_ROWS_MINB_B) : (N <= 48 ? PCB_ROWS_MINB_SHORT3 : PCB_ROWS_MINB_MIXED))
    k_rows_inv_b(PassArgs a) {
    using RC = RowCfg<N>;
    // split-3 lengths: the lane's F sub-line thread groups own the bins k = F k' + s (k' the M-point
    // inverse's input position), so each group's accumulators feed its sub-line transform directly
    constexpr int F = RC::F, M = RC::M, NLS = F * NL;
    constexpr int R = RC::R;
    constexpr int RL = LastPos<M>::RL;
    constexpr int NT = NLS * RC::TPL;
    constexpr int TPL = RC::TPL;   // threads per sub-line
    constexpr int TPLN = F * TPL;  // threads per lane (staging loops)
    constexpr int XS = 2 * N + 1;
    constexpr int BUFW = row_words<N, NL>() > (NL * (2 * N + 1) + 1) / 2 ? row_words<N, NL>()
                                                                        : (NL * (2 * N + 1) + 1) / 2;
    constexpr int P = 2 * N;
    constexpr int MB = PCB_BUNDLE_MB;
    constexpr int SL = N + 1;  // staged line length
    extern __shared__ double2 buf[];
    const int64_t aline = blockIdx.x;
    const int vec = blockIdx.y;
    const int ax = a.D - 1;
    const int64_t line = a.line_id[aline];
    const int ulo = a.line_rng[2 * aline], uhi = a.line_rng[2 * aline + 1];
#if PCB_BUNDLE_XPF && PCB_BUNDLE_ALIAS
    // layout: stage [2][NL][MB][SLS] | acc [n_last] | meta [2][NL].  Stage buffer 1 is free while a
    // batch is transformed (its members are summed, the next batch's first ones land in buffer 0),
    // so it doubles as the FFT exchange / xs buffer: one 9 KB buffer less per CTA (c3: 6 -> 8 CTAs/SM)
    constexpr int SLS = stage_stride_b<N, NL>();
    double2* stg = buf;
    double2* fbuf = stg + NL * MB * SLS;
    double* acc = reinterpret_cast<double*>(stg + 2 * NL * MB * SLS);
#else
    // layout: buf [BUFW] (FFT; reused as xs) | stage [1 + DB][NL][MB][N+1] | acc [n_last] | meta [NL]
    constexpr int SLS = SL;
    double2* fbuf = buf;
    double2* stg = buf + BUFW;
    double* acc = reinterpret_cast<double*>(stg + (1 + PCB_BUNDLE_DB) * NL * MB * SL);
#endif
    double* xs = reinterpret_cast<double*>(fbuf);
    GatherEntry* meta = reinterpret_cast<GatherEntry*>(acc + a.n[ax] + (a.n[ax] & 1));
    const int64_t b_beg = a.line_ptr[aline];
    const int64_t b_end = a.line_ptr[aline + 1];
    const double2* twP = twtab<P>(a.tw);
    const int sl = threadIdx.x % NLS;  // sub-line s of lane l (F = 1: the lane itself)
    const int s = sl / NL;
    const int l = sl - s * NL;
    const int tl = threadIdx.x / NLS;
    const int tln = tl * F + s;  // thread index within the lane
    for (int i = ulo + threadIdx.x; i < uhi; i += NT) acc[i - ulo] = 0.0;

#if PCB_BUNDLE_XPF
    // Cross-batch prefetch: the next batch's bundle headers and first members are issued before
    // this batch's C2R, so the transform hides their load latency (stage buffer 0 is free then).
    GatherEntry* metaN = meta + NL;
    auto issue = [&](const BundleMember* mb, int cnt, int m0, int buf_i) {
#pragma unroll
        for (int j = 0; j < MB; ++j)
            if (m0 + j < cnt) {
                const double2* src = a.T + mb[m0 + j].t_off + vec * mb[m0 + j].t_vst;
                double2* dst = stg + ((buf_i * NL + l) * MB + j) * SLS;
                for (int i = tln; i < SL; i += TPLN) cp_async16(&dst[i], src + i);
            }
        asm volatile("cp.async.commit_group;\n" ::);
    };
    auto lane_of = [&](const GatherEntry* mt, int nb, int& cnt) {
        cnt = l < nb ? mt[l].pad_ : 0;
        return a.members + (l < nb ? mt[l].t_off : 0);
    };
    if (b_beg < b_end) {
        const int nb = (int)((b_end - b_beg) < NL ? (b_end - b_beg) : NL);
        if (threadIdx.x < nb) meta[threadIdx.x] = a.entries[b_beg + threadIdx.x];
        __syncthreads();
        int cnt;
        const BundleMember* mb = lane_of(meta, nb, cnt);
        issue(mb, cnt, 0, 0);
    }
    for (int64_t b0 = b_beg; b0 < b_end; b0 += NL) {
        const int nb = (int)((b_end - b0) < NL ? (b_end - b0) : NL);
        int mmax = 0;
        for (int ll = 0; ll < nb; ++ll) mmax = max(mmax, meta[ll].pad_);
        int cnt;
        const BundleMember* mb = lane_of(meta, nb, cnt);
        double2 zk[R], zn[R];
#pragma unroll
        for (int r = 0; r < R; ++r) zk[r] = zn[r] = czero();
        int cur = 0;  // members [0, MB) are already in flight in buffer 0
        for (int m0 = 0; m0 < mmax; m0 += MB) {
            if (m0 + MB < mmax) {
                issue(mb, cnt, m0 + MB, cur ^ 1);
                asm volatile("cp.async.wait_group 1;\n" ::);
            } else {
                asm volatile("cp.async.wait_group 0;\n" ::);
            }
            __syncthreads();
#pragma unroll
            for (int j = 0; j < MB; ++j)
                if (m0 + j < cnt) {
                    const double2* x = stg + ((cur * NL + l) * MB + j) * SLS;
                    const double sc = mb[m0 + j].scale;
                    const int dl = mb[m0 + j].delta;
                    // the phase of bin N - k is (-1)^dl conj(phase of bin k) (P = 2N): one table load per pair
                    const double sn = (dl & 1) ? -1.0 : 1.0;
#if PCB_BUNDLE_TWREC
                    // k = tl + r TPL: phase(k) = phase(tl) u^r, u = phase(TPL); u^r from u, u^2, u^4 (<= 3
                    // products): 1 + log2(R) table loads per member instead of R
                    constexpr int LR = R >= 16 ? 4 : R >= 8 ? 3 : R >= 4 ? 2 : 1;
                    double2 up[LR];
                    double2 w0 = make_double2(1.0, 0.0);
                    if (dl != 0) {
                        w0 = __ldg(&twP[(tln * dl) % P]);
#pragma unroll
                        for (int bit = 0; bit < LR; ++bit) up[bit] = __ldg(&twP[(((1 << bit) * TPLN) * dl) % P]);
                    }
#endif
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        const int k = tln + r * TPLN;  // = F (tl + r TPL) + s
                        double2 xk = x[k], xn = x[N - k];
                        if (dl != 0) {
#if PCB_BUNDLE_TWREC
                            double2 w = w0;
#pragma unroll
                            for (int bit = 0; bit < LR; ++bit)
                                if (r & (1 << bit)) w = cmul(w, up[bit]);
#else
                            const double2 w = __ldg(&twP[(k * dl) % P]);
#endif
                            xk = cmul(xk, w);
                            xn = cmul(xn, make_double2(sn * w.x, -sn * w.y));
                        }
                        zk[r] = make_double2(fma(sc, xk.x, zk[r].x), fma(sc, xk.y, zk[r].y));
                        zn[r] = make_double2(fma(sc, xn.x, zn[r].x), fma(sc, xn.y, zn[r].y));
                    }
                }
            __syncthreads();  // stage buffer `cur` free
            cur ^= 1;
        }
        if (mmax == 0) asm volatile("cp.async.wait_group 0;\n" ::);
        __syncthreads();  // every thread is done with metaN (last read two batches ago)
        const int64_t b1 = b0 + NL;
        if (b1 < b_end) {
            const int nb1 = (int)((b_end - b1) < NL ? (b_end - b1) : NL);
            if (threadIdx.x < nb1) metaN[threadIdx.x] = a.entries[b1 + threadIdx.x];
            __syncthreads();
            int cnt1;
            const BundleMember* mb1 = lane_of(metaN, nb1, cnt1);
            issue(mb1, cnt1, 0, 0);
        }
        double2 v[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int k = tln + r * TPLN;
            const double2 E = make_double2(zk[r].x + zn[r].x, zk[r].y - zn[r].y);   // Z[k] + conj Z[N-k]
            const double2 Dd = make_double2(zk[r].x - zn[r].x, zk[r].y + zn[r].y);  // Z[k] - conj Z[N-k]
            const double2 O = cmulc(Dd, __ldg(&twP[k]));                            // * exp(+2 pi i k / P)
            v[r] = make_double2(E.x - O.y, E.y + O.x);                              // E + i O
        }
        fft_rev_order<M, +1, NLS, PSH<NLS>>(v, fbuf, sl, tl, twtab<M>(a.tw));
        __syncthreads();
#pragma unroll
        for (int bb = 0; bb < R / RL; ++bb)
#pragma unroll
            for (int r = 0; r < RL; ++r) {
                const int p = s * M + LastPos<M>::pos(tl, bb, r);
                xs[l * XS + 2 * p] = v[bb * RL + r].x;
                xs[l * XS + 2 * p + 1] = v[bb * RL + r].y;
            }
        __syncthreads();
        if constexpr (F == 3) {
            split3_time_pass<N, NT, XS>(xs, nb, twtab<N>(a.tw));
            __syncthreads();
        }
        for (int ll = 0; ll < nb; ++ll) {
            const int lo = meta[ll].lo, hi = meta[ll].hi;
            const double* x = xs + ll * XS - meta[ll].sh;
            int p = lo + (int)((threadIdx.x + NT - (unsigned)(lo % NT)) % NT);
            if (ADJ) {
                const double* w = a.w_pool + meta[ll].w_off;
                for (; p < hi; p += NT) acc[p - ulo] += w[p] * x[p];
            } else {
                for (; p < hi; p += NT) acc[p - ulo] += x[p];
            }
        }
        __syncthreads();  // xs (the FFT buffer) and meta are free
        GatherEntry* t = meta;
        meta = metaN;
        metaN = t;
    }
#else
    static_assert(F == 1, "the single-batch bundled gather has no split-3 path");
    for (int64_t b0 = b_beg; b0 < b_end; b0 += NL) {
        const int nb = (int)((b_end - b0) < NL ? (b_end - b0) : NL);
        __syncthreads();  // previous batch finished with meta / xs
        if (threadIdx.x < nb) meta[threadIdx.x] = a.entries[b0 + threadIdx.x];
        __syncthreads();
        int mmax = 0;
        for (int ll = 0; ll < nb; ++ll) mmax = max(mmax, meta[ll].pad_);
        const int cnt = l < nb ? meta[l].pad_ : 0;
        const BundleMember* mb = a.members + (l < nb ? meta[l].t_off : 0);
        double2 zk[R], zn[R];
#pragma unroll
        for (int r = 0; r < R; ++r) zk[r] = zn[r] = czero();
        // members staged MB at a time per lane; with PCB_BUNDLE_DB the next MB are in flight
        // while the current ones are summed (two stage buffers)
        auto issue = [&](int m0, int buf_i) {
#pragma unroll
            for (int j = 0; j < MB; ++j)
                if (m0 + j < cnt) {
                    const double2* src = a.T + mb[m0 + j].t_off + vec * mb[m0 + j].t_vst;
                    double2* dst = stg + ((buf_i * NL + l) * MB + j) * SL;
                    for (int i = tl; i < SL; i += TPL) cp_async16(&dst[i], src + i);
                }
            asm volatile("cp.async.commit_group;\n" ::);
        };
        int cur = 0;
        if (mmax > 0) issue(0, 0);
        for (int m0 = 0; m0 < mmax; m0 += MB) {
            if (PCB_BUNDLE_DB && m0 + MB < mmax) {
                issue(m0 + MB, cur ^ 1);
                asm volatile("cp.async.wait_group 1;\n" ::);
            } else {
                asm volatile("cp.async.wait_group 0;\n" ::);
            }
            __syncthreads();
#pragma unroll
            for (int j = 0; j < MB; ++j)
                if (m0 + j < cnt) {
                    const double2* x = stg + ((cur * NL + l) * MB + j) * SL;
                    const double sc = mb[m0 + j].scale;
                    const int dl = mb[m0 + j].delta;
                    // the phase of bin N - k is (-1)^dl conj(phase of bin k) (P = 2N): one table load per pair
                    const double sn = (dl & 1) ? -1.0 : 1.0;
#if PCB_BUNDLE_TWREC
                    // k = tl + r TPL: phase(k) = phase(tl) u^r, u = phase(TPL); u^r from u, u^2, u^4 (<= 3
                    // products): 1 + log2(R) table loads per member instead of R
                    constexpr int LR = R >= 16 ? 4 : R >= 8 ? 3 : R >= 4 ? 2 : 1;
                    double2 up[LR];
                    double2 w0 = make_double2(1.0, 0.0);
                    if (dl != 0) {
                        w0 = __ldg(&twP[(tl * dl) % P]);
#pragma unroll
                        for (int bit = 0; bit < LR; ++bit) up[bit] = __ldg(&twP[(((1 << bit) * TPL) * dl) % P]);
                    }
#endif
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        const int k = tl + r * TPL;
                        double2 xk = x[k], xn = x[N - k];
                        if (dl != 0) {
#if PCB_BUNDLE_TWREC
                            double2 w = w0;
#pragma unroll
                            for (int bit = 0; bit < LR; ++bit)
                                if (r & (1 << bit)) w = cmul(w, up[bit]);
#else
                            const double2 w = __ldg(&twP[(k * dl) % P]);
#endif
                            xk = cmul(xk, w);
                            xn = cmul(xn, make_double2(sn * w.x, -sn * w.y));
                        }
                        zk[r] = make_double2(fma(sc, xk.x, zk[r].x), fma(sc, xk.y, zk[r].y));
                        zn[r] = make_double2(fma(sc, xn.x, zn[r].x), fma(sc, xn.y, zn[r].y));
                    }
                }
            __syncthreads();  // stage buffer `cur` free
            if (PCB_BUNDLE_DB) cur ^= 1;
            else if (m0 + MB < mmax) issue(m0 + MB, 0);
        }
        double2 v[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int k = tl + r * TPL;
            const double2 E = make_double2(zk[r].x + zn[r].x, zk[r].y - zn[r].y);   // Z[k] + conj Z[N-k]
            const double2 Dd = make_double2(zk[r].x - zn[r].x, zk[r].y + zn[r].y);  // Z[k] - conj Z[N-k]
            const double2 O = cmulc(Dd, __ldg(&twP[k]));                            // * exp(+2 pi i k / P)
            v[r] = make_double2(E.x - O.y, E.y + O.x);                              // E + i O
        }
        fft_rev_order<N, +1, NL, PSH<NL>>(v, buf, l, tl, twtab<N>(a.tw));
        __syncthreads();
#pragma unroll
        for (int bb = 0; bb < R / RL; ++bb)
#pragma unroll
            for (int r = 0; r < RL; ++r) {
                const int p = LastPos<N>::pos(tl, bb, r);
                xs[l * XS + 2 * p] = v[bb * RL + r].x;
                xs[l * XS + 2 * p + 1] = v[bb * RL + r].y;
            }
        __syncthreads();
        for (int ll = 0; ll < nb; ++ll) {
            const int lo = meta[ll].lo, hi = meta[ll].hi;
            const double* x = xs + ll * XS - meta[ll].sh;
            int p = lo + (int)((threadIdx.x + NT - (unsigned)(lo % NT)) % NT);
            if (ADJ) {
                const double* w = a.w_pool + meta[ll].w_off;
                for (; p < hi; p += NT) acc[p - ulo] += w[p] * x[p];
            } else {
                for (; p < hi; p += NT) acc[p - ulo] += x[p];
            }
        }
    }
#endif
    __syncthreads();
    double* g = a.out + (int64_t)vec * a.N + line * a.n[ax];
    for (int i = ulo + threadIdx.x; i < uhi; i += NT) g[i] = a.accumulate ? g[i] + acc[i - ulo] : acc[i - ulo];
}

// ---------------------------------------------------------------------------
// launch helpers shared by the dispatch units

template <typename K>
cudaError_t launch_dyn(K kernel, dim3 grid, dim3 block, size_t smem, cudaStream_t st, const PassArgs& a) {
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    kernel<<<grid, block, smem, st>>>(a);
    return cudaGetLastError();
}

template <int LEN>
constexpr int rows_nl() {  // lines per CTA for the last-axis passes: ~PCB_ROWS_THREADS threads
    constexpr int t = RowCfg<LEN>::THREADS / (RowCfg<LEN>::F * RowCfg<LEN>::TPL);
    return t < 1 ? 1 : (t > 32 ? 32 : t);
}
template <int LEN>
constexpr int rows_threads() {
    return rows_nl<LEN>() * RowCfg<LEN>::F * RowCfg<LEN>::TPL;
}
template <int P>
constexpr int cols_nl() {  // column-tile width of the axis-0 / axis-1 passes (>= 2: 32-B runs)
    constexpr int t = PCB_COLS_THREADS / FftCfg<P>::TPL;
    return t < 2 ? 2 : (t > 32 ? 32 : t);
}

}  // namespace

// line lengths compiled for each pass: 2^a * {1, 3, 9}
#define PCB_ROW_SIZES(X) X(8) X(16) X(24) X(32) X(48) X(64) X(72) X(96) X(128) X(144) X(192) X(256) X(288) \
    X(384) X(512) X(576) X(768) X(1024) X(1152) X(1536) X(2048)
#define PCB_COL_SIZES(X) X(16) X(32) X(48) X(64) X(96) X(128) X(144) X(192) X(256) X(288) X(384) X(512) \
    X(576) X(768) X(1024) X(1152) X(1536) X(2048) X(2304) X(3072) X(4096)

}  // namespace pcb
