// Unit test of the line FFT engine (csrc/fft.cuh) for every compiled length: forward
// (fft_fwd_order) and inverse (fft_rev_order) of random lines vs a direct fp64 DFT.
#include <cmath>
#include <cstdio>
#include <vector>

#include "fft.cuh"

using namespace pcb;

template <int L, int DIR, bool REV>
__global__ void __launch_bounds__(1024) k_test(const double2* in, double2* out, const double2* tw) {
    constexpr int NL = 2;
    constexpr int E = FftCfg<L>::R;
    constexpr int PS = 3;
    extern __shared__ double2 buf[];
    const int l = threadIdx.x % NL, tl = threadIdx.x / NL;
    double2 v[E];
    if (!REV) {
        constexpr int RF = FirstPos<L>::RF;
        for (int b = 0; b < E / RF; ++b)
            for (int r = 0; r < RF; ++r) v[b * RF + r] = in[l * L + FirstPos<L>::pos(tl, b, r)];
        fft_fwd_order<L, DIR, NL, PS>(v, buf, l, tl, tw + tw_offset(L));
        for (int r = 0; r < E; ++r) out[l * L + mid_pos<L>(tl, r)] = v[r];
    } else {
        for (int r = 0; r < E; ++r) v[r] = in[l * L + mid_pos<L>(tl, r)];
        fft_rev_order<L, DIR, NL, PS>(v, buf, l, tl, tw + tw_offset(L));
        constexpr int RL = LastPos<L>::RL;
        for (int b = 0; b < E / RL; ++b)
            for (int r = 0; r < RL; ++r) out[l * L + LastPos<L>::pos(tl, b, r)] = v[b * RL + r];
    }
}

std::vector<double2> twiddles() {
    std::vector<double2> h;
    for (int len = 8; len <= 8192; len += 8) {
        if (!fft_len_ok(len)) continue;
        for (int m = 0; m < len; ++m) {
            const long double ang = -2.0L * 3.141592653589793238462643383279502884L * m / len;
            h.push_back(make_double2((double)cosl(ang), (double)sinl(ang)));
        }
    }
    return h;
}

template <typename K>
void launch(K k, int threads, size_t smem, const double2* in, double2* out, const double2* tw) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k<<<1, threads, smem>>>(in, out, tw);
}

template <int L>
int run(const double2* dtw) {
    int bad = 0;
    const int NL = 2;
    std::vector<double2> x(NL * L), y(NL * L);
    for (int i = 0; i < NL * L; ++i) x[i] = make_double2(std::sin(0.37 * i + 1.0), std::cos(1.3 * ((i * i) % 97)));
    double2 *din, *dout;
    cudaMalloc(&din, sizeof(double2) * NL * L);
    cudaMalloc(&dout, sizeof(double2) * NL * L);
    cudaMemcpy(din, x.data(), sizeof(double2) * NL * L, cudaMemcpyHostToDevice);
    for (int dir : {-1, +1})
        for (int rev : {0, 1}) {
            if (dir < 0 && rev) launch(k_test<L, -1, true>, NL * FftCfg<L>::TPL, sizeof(double2) * SmemLine<L, 2, 3>::WORDS, din, dout, dtw);
            if (dir < 0 && !rev) launch(k_test<L, -1, false>, NL * FftCfg<L>::TPL, sizeof(double2) * SmemLine<L, 2, 3>::WORDS, din, dout, dtw);
            if (dir > 0 && rev) launch(k_test<L, 1, true>, NL * FftCfg<L>::TPL, sizeof(double2) * SmemLine<L, 2, 3>::WORDS, din, dout, dtw);
            if (dir > 0 && !rev) launch(k_test<L, 1, false>, NL * FftCfg<L>::TPL, sizeof(double2) * SmemLine<L, 2, 3>::WORDS, din, dout, dtw);
            cudaError_t e = cudaGetLastError();  // a launch failure (e.g. resources) is not sticky
            if (e == cudaSuccess) e = cudaDeviceSynchronize();
            if (e != cudaSuccess) {
                printf("L=%d cuda error %s\n", L, cudaGetErrorString(e));
                return 1;
            }
            cudaMemcpy(y.data(), dout, sizeof(double2) * NL * L, cudaMemcpyDeviceToHost);
            double err = 0, nrm = 0;
            // every output bin for L <= 512; for longer lines 512 bins per line (a stride with a
            // per-line offset, so every residue class is hit across lines and directions)
            const int kstep = L <= 512 ? 1 : L / 512;
            for (int l = 0; l < NL; ++l)
                for (int k = (l * 7 + (dir > 0) * 3 + rev) % kstep; k < L; k += kstep) {
                    long double re = 0, im = 0;
                    for (int n = 0; n < L; ++n) {
                        const long double ang = dir * 2.0L * 3.141592653589793238462643383279502884L * ((long long)n * k % L) / L;
                        re += x[l * L + n].x * cosl(ang) - x[l * L + n].y * sinl(ang);
                        im += x[l * L + n].x * sinl(ang) + x[l * L + n].y * cosl(ang);
                    }
                    err += (y[l * L + k].x - re) * (y[l * L + k].x - re) + (y[l * L + k].y - im) * (y[l * L + k].y - im);
                    nrm += re * re + im * im;
                }
            const double rel = std::sqrt(err / nrm);
            if (!(rel < 1e-14)) {
                printf("FAIL L=%d dir=%d rev=%d rel=%.3e stages:", L, dir, rev, rel);
                for (int s = 0; s < FftCfg<L>::NSTG; ++s) printf(" %d", FftCfg<L>::radix(s));
                printf("\n");
                bad = 1;
            }
        }
    cudaFree(din);
    cudaFree(dout);
    return bad;
}

int main() {
    std::vector<double2> h = twiddles();
    double2* dtw;
    cudaMalloc(&dtw, sizeof(double2) * h.size());
    cudaMemcpy(dtw, h.data(), sizeof(double2) * h.size(), cudaMemcpyHostToDevice);
    int bad = 0;
#define T(n) bad |= run<n>(dtw);
    T(8) T(16) T(24) T(32) T(48) T(64) T(72) T(96) T(128) T(144) T(192) T(256) T(288) T(384) T(512) T(576) T(768)
    T(1024) T(1152) T(1536) T(2048) T(2304) T(3072) T(4096)
    printf(bad ? "FFT UNIT: FAIL\n" : "FFT UNIT: all lengths OK\n");
    return bad;
}
