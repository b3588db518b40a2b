// Dispatch of the last-axis passes (K2 rows_fwd, K4 rows_inv) over the compiled lengths.
#include "kernels_impl.cuh"

namespace pcb {
namespace {

template <int N, int MODE>
cudaError_t rows_fwd_n(const PassArgs& a, cudaStream_t st) {
    constexpr int NL = rows_nl<N>();
    const int64_t maxlines = MODE == RF_SPEC ? (a.D == 2 ? a.P[0] : (int64_t)a.P[0] * a.P[1]) : a.lines_max;
    const int items = (MODE == RF_ADJ && a.global) ? a.B : a.n_slots * (MODE == RF_SPEC ? 1 : a.B);
    dim3 grid((unsigned)((maxlines + NL - 1) / NL), (unsigned)items);
    const size_t smem = sizeof(double2) * row_words<N, NL>() + NL * (3 * sizeof(int64_t) + 2 * sizeof(int));
    return launch_dyn(k_rows_fwd<N, NL, MODE>, grid, dim3(rows_threads<N>()), smem, st, a);
}

template <int MODE>
cudaError_t rows_fwd_mode(const PassArgs& a, cudaStream_t st) {
    switch (a.P[a.D - 1] / 2) {
#define PCB_CASE(n) \
    case n: return rows_fwd_n<n, MODE>(a, st);
        PCB_ROW_SIZES(PCB_CASE)
#undef PCB_CASE
        default: return cudaErrorInvalidValue;
    }
}

template <int N, int MODE>
cudaError_t rows_inv_n(const PassArgs& a, int64_t n_lines, cudaStream_t st) {
    constexpr int NL = rows_nl<N>();
    constexpr int BUFW = row_words<N, NL>() > (NL * (2 * N + 1) + 1) / 2 ? row_words<N, NL>()
                                                                        : (NL * (2 * N + 1) + 1) / 2;
    dim3 grid((unsigned)n_lines, (unsigned)a.B);
#if PCB_RINV_ALIAS
    const size_t stage_words = (size_t)NL * stage_stride_b<N, NL>();
#else
    const size_t stage_words = BUFW + (size_t)NL * (N + 1);
#endif
    const size_t smem = sizeof(double2) * stage_words + sizeof(double) * ((size_t)a.n[a.D - 1] + 1) +
                        NL * sizeof(GatherEntry) + 16;
    return launch_dyn(k_rows_inv<N, NL, MODE>, grid, dim3(rows_threads<N>()), smem, st, a);
}

template <int N, int ADJ>
cudaError_t rows_inv_b_n(const PassArgs& a, int64_t n_lines, cudaStream_t st) {
    constexpr int NL = rows_nl<N>();
    constexpr int BUFW = row_words<N, NL>() > (NL * (2 * N + 1) + 1) / 2 ? row_words<N, NL>()
                                                                        : (NL * (2 * N + 1) + 1) / 2;
    dim3 grid((unsigned)n_lines, (unsigned)a.B);
#if PCB_BUNDLE_XPF && PCB_BUNDLE_ALIAS
    const size_t stage_words = (size_t)2 * NL * PCB_BUNDLE_MB * stage_stride_b<N, NL>();
#else
    const size_t stage_words = BUFW + (size_t)(1 + PCB_BUNDLE_DB) * NL * PCB_BUNDLE_MB * (N + 1);
#endif
    const size_t smem = sizeof(double2) * stage_words + sizeof(double) * ((size_t)a.n[a.D - 1] + 1) +
                        (1 + PCB_BUNDLE_XPF) * NL * sizeof(GatherEntry) + 16;
    return launch_dyn(k_rows_inv_b<N, NL, ADJ>, grid, dim3(rows_threads<N>()), smem, st, a);
}

template <int MODE>
cudaError_t rows_inv_mode(const PassArgs& a, int64_t n_lines, cudaStream_t st) {
    if constexpr (MODE == RI_APPLY_B || MODE == RI_ADJ_B) {
        switch (a.P[a.D - 1] / 2) {
#define PCB_CASE(n) \
    case n: return rows_inv_b_n<n, MODE == RI_ADJ_B ? 1 : 0>(a, n_lines, st);
            PCB_ROW_SIZES(PCB_CASE)
#undef PCB_CASE
            default: return cudaErrorInvalidValue;
        }
    } else {
    switch (a.P[a.D - 1] / 2) {
#define PCB_CASE(n) \
    case n: return rows_inv_n<n, MODE>(a, n_lines, st);
        PCB_ROW_SIZES(PCB_CASE)
#undef PCB_CASE
        default: return cudaErrorInvalidValue;
    }
    }
}

}  // namespace

int rows_lanes(int P_last) {
    switch (P_last / 2) {
#define PCB_CASE(n) \
    case n: return rows_nl<n>();
        PCB_ROW_SIZES(PCB_CASE)
#undef PCB_CASE
        default: return 1;
    }
}

cudaError_t launch_rows_fwd(const PassArgs& a, int mode, cudaStream_t st) {
    switch (mode) {
        case RF_APPLY: return rows_fwd_mode<RF_APPLY>(a, st);
        case RF_ADJ: return rows_fwd_mode<RF_ADJ>(a, st);
        case RF_SPEC: return rows_fwd_mode<RF_SPEC>(a, st);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_rows_inv(const PassArgs& a, int mode, int64_t n_lines, cudaStream_t st) {
    switch (mode) {
        case RI_APPLY: return rows_inv_mode<RI_APPLY>(a, n_lines, st);
        case RI_ADJ: return rows_inv_mode<RI_ADJ>(a, n_lines, st);
        case RI_APPLY_B: return rows_inv_mode<RI_APPLY_B>(a, n_lines, st);
        case RI_ADJ_B: return rows_inv_mode<RI_ADJ_B>(a, n_lines, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace pcb
