// Dispatch of the axis-0 pass (K1 spectra store, K3 frequency MAC) over the compiled lengths.
#include "kernels_impl.cuh"

namespace pcb {
namespace {

template <int P0, int MODE>
cudaError_t cols_p(const PassArgs& a, cudaStream_t st) {
    constexpr int NL = cols_nl<P0>();
    if (a.nl_cols != NL) return cudaErrorInvalidValue;
    const bool global = MODE == CM_APPLY_GLOBAL || MODE == CM_ADJ_GLOBAL;
    const int items = global ? a.B : a.n_slots * (MODE == CM_SPEC ? 1 : a.B);
    dim3 grid((unsigned)((a.L + NL - 1) / NL), (unsigned)items);
    // global modes stage Phi_k tiles in shared memory (apply: one buffer, adjoint: two)
    const size_t stage = (P0 <= PCB_LOCAL_STAGE && (MODE == CM_APPLY_LOCAL || MODE == CM_ADJ_LOCAL)) ? (size_t)P0 * NL
                         : (MODE == CM_APPLY_GLOBAL || (MODE == CM_APPLY_CHAIN && PCB_CHAIN_STAGE)) ? (P0 <= 512 ? (size_t)P0 * NL : 0)
                         : MODE == CM_ADJ_GLOBAL ? 2 * (size_t)P0 * NL : 0;
    const size_t smem = sizeof(double2) * (smem_words_c<P0, NL>() + stage);
    return launch_dyn(k_cols<P0, NL, MODE>, grid, dim3(NL * FftCfg<P0>::TPL), smem, st, a);
}

template <int MODE>
cudaError_t cols_mode(const PassArgs& a, cudaStream_t st) {
    switch (a.P[0]) {
#define PCB_CASE(n) \
    case n: return cols_p<n, MODE>(a, st);
        PCB_COL_SIZES(PCB_CASE)
#undef PCB_CASE
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace

int cols_tile_width(int P0) {
    switch (P0) {
#define PCB_CASE(n) \
    case n: return cols_nl<n>();
        PCB_COL_SIZES(PCB_CASE)
#undef PCB_CASE
        default: return -1;
    }
}

cudaError_t launch_cols(const PassArgs& a, int mode, cudaStream_t st) {
    switch (mode) {
        case CM_SPEC: return cols_mode<CM_SPEC>(a, st);
        case CM_APPLY_LOCAL: return cols_mode<CM_APPLY_LOCAL>(a, st);
        case CM_APPLY_GLOBAL: return cols_mode<CM_APPLY_GLOBAL>(a, st);
        case CM_ADJ_LOCAL: return cols_mode<CM_ADJ_LOCAL>(a, st);
        case CM_ADJ_GLOBAL: return cols_mode<CM_ADJ_GLOBAL>(a, st);
        case CM_APPLY_CHAIN: return cols_mode<CM_APPLY_CHAIN>(a, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace pcb
