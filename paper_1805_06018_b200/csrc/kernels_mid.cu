// Dispatch of the 3-D middle-axis pass over the compiled lengths.
#include "kernels_impl.cuh"

namespace pcb {
namespace {

template <int P1, int MODE>
cudaError_t mid_p(const PassArgs& a, cudaStream_t st) {
    constexpr int NL = cols_nl<P1>();
    const bool gmode = a.global && (MODE == MM_INV_APPLY || MODE == MM_FWD_ADJ);
    const int items = gmode ? a.B : a.n_slots * (MODE == MM_FWD_SPEC ? 1 : a.B);
    dim3 grid((unsigned)((a.W + NL - 1) / NL), (unsigned)a.P[0], (unsigned)items);
    const size_t smem = sizeof(double2) * smem_words<P1, NL>();
    return launch_dyn(k_mid<P1, NL, MODE>, grid, dim3(NL * FftCfg<P1>::TPL), smem, st, a);
}

template <int MODE>
cudaError_t mid_mode(const PassArgs& a, cudaStream_t st) {
    switch (a.P[1]) {
#define PCB_CASE(n) \
    case n: return mid_p<n, MODE>(a, st);
        PCB_COL_SIZES(PCB_CASE)
#undef PCB_CASE
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace

cudaError_t launch_mid(const PassArgs& a, int mode, cudaStream_t st) {
    switch (mode) {
        case MM_FWD_APPLY: return mid_mode<MM_FWD_APPLY>(a, st);
        case MM_FWD_ADJ: return mid_mode<MM_FWD_ADJ>(a, st);
        case MM_FWD_SPEC: return mid_mode<MM_FWD_SPEC>(a, st);
        case MM_INV_APPLY: return mid_mode<MM_INV_APPLY>(a, st);
        case MM_INV_ADJ: return mid_mode<MM_INV_ADJ>(a, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace pcb
