// Device-side descriptors shared by the host planner (plan.cpp) and the
// kernels (kernels.cu).  Plain structs, passed by value or through device
// arrays; no torch types anywhere.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace pcb {

// One product-convolution term k, in FFT index space (reference:
// pc_operator.cpp:49-54; SURVEY.md 8(a) "GPU restatement").
//   input window   X_k = footprint(w_k) cap Omega, x = x_lo + u, u in [0, m)
//   output         y = s + v, v kept in [o_lo, o_lo + o_cnt)  (apply)
//   kernel         trimmed phi_k^E box K = [k_lo, k_lo + k_ext), placed at
//                  t = (z - c) mod P with c = s - x_lo
// Apply: g[s+v] += IFFT( FFT_P(phi placed) . FFT_P(w f on X) )[v] / prod P.
// Adjoint (same spectra, conjugated): out[x_lo+u] += w[u] IFFT(conj(Phi) FFT(g[s+.]))[u].
struct TermDesc {
    int64_t x_lo[3];
    int64_t s[3];
    int64_t k_lo[3];
    int32_t m[3];
    int32_t o_lo[3];
    int32_t o_cnt[3];
    int32_t k_ext[3];
    int64_t w_off;     // doubles: w_k on X_k, row-major [m0][m1][m2]
    int64_t phi_off;   // doubles: phi_k^E on K, row-major
    int64_t spec_off;  // double2: spectrum, tile-major [L/NL][P0][NL]
    // scratch pools (double2): this term's forward (S) / inverse (T) region for vector 0 and the
    // per-vector stride; rows of a region are planes of P1 * W (3-D) or W (2-D) values
    int64_t s_pool, s_vst, t_pool, t_vst;
    // row family (LOCAL apply, separable weights w_k = A_k(lead axes) * c(last axis)): the term's
    // forward row transforms are the family's shared rows (double2 offset f_off for vector 0,
    // + f_vst per vector, f_ps lines per family plane in 3-D) times A_k (a_pool + a_off); -1: none
    int64_t f_off, f_vst, a_off;
    // adjoint row family (LOCAL): the forward rows of g on this term's output window are the
    // family's rows from af_off (+ af_vst per vector; 3-D: af_ps lines per family plane, read by
    // the mid pass); -1: the term's own S region
    int64_t af_off, af_vst;
    int32_t af_ps;
    int32_t pad2_;
    int32_t f_ps;
    int32_t P1;        // axis-1 FFT size of the term (3-D plane stride); 1 in 2-D.  A family
                       // descriptor (rows_fwd item) holds its lead-axis-1 line count here
    int32_t wrow0;     // 1: one weight row (w_off) serves every line (family descriptors)
    int32_t cols_f;    // 1: the axis-0 (cols) pass loads rows f_off (+ f_vst per vector) x a_pool[a_off]
                       // (2-D row families; 3-D plane families) instead of the term's S region
};

// rows_inv gather list entry: one C2R line of T contributing to one output line.
// Self-contained (precomputed at create) so the gather issues no dependent loads.
struct GatherEntry {
    int32_t lo, hi;   // output positions [lo, hi) along the last axis (domain-relative, clipped)
    int32_t sh;       // line index of output position p is p - sh
    int32_t pad_;
    int64_t t_off;    // double2 offset of the line in the T pool for vector 0
    int64_t t_vst;    // ... plus t_vst per vector
    int64_t w_off;    // adjoint: w_pool offset of the multiplying w row shifted by -sh; else -1
    double scale;     // 1 / prod P of the entry's term (its group's FFT size)
};

// LOCAL apply gather, frequency-domain bundles: the T lines of one output line whose shifted
// supports fit in one P-periodic window are summed as spectra, each multiplied by its scale and
// the phase exp(-2 pi i k delta / P) of its shift delta relative to the bundle origin, and
// transformed once.  The bundle header is a GatherEntry {lo, hi: union output range; sh: origin;
// pad_: member count; t_off: first member}; members carry the per-line data.
struct BundleMember {
    int64_t t_off;    // double2 offset of the T line for vector 0
    int64_t t_vst;    // ... plus t_vst per vector
    double scale;     // 1 / prod P
    int32_t delta;    // shift relative to the bundle origin, 0 <= delta < P
    int32_t pad_;
};

// Everything one pipeline pass needs.  D in {2, 3}: axes 0..D-1, last axis is
// the R2C/C2R axis (contiguous in memory, reference layout "last axis
// fastest", grid_function.hpp:11-13).
struct PassArgs {
    int D;
    int64_t dom_lo[3];
    int32_t n[3];          // domain extents
    int32_t P[3];          // FFT sizes (P[D-1] is the real axis)
    int32_t W;             // padded half-spectrum row: roundup(P_last/2+1, w_align)
    int64_t L;             // lines of the axis-0 pass: W (2D) or P1*W (3D)
    int32_t lines_max;     // rows_fwd: max lines of one item over the launch's terms
    int32_t nl_cols;       // spectrum tile width
    const TermDesc* terms; // device
    const int32_t* slots;  // device: term ids of this chunk
    int32_t n_slots;
    int32_t B;             // vectors in this call
    int32_t global;        // 1: spectral accumulation over all slots (one T per vector)
    int32_t accumulate;    // rows_inv: add into g instead of overwrite
    const double* in;      // B x N input vectors (vector-major)
    double* out;           // B x N output vectors
    int64_t N;             // points per vector
    double2* S;            // forward scratch pool (term regions: TermDesc::s_pool / s_vst)
    int64_t S_stride;      // spectra build only: per-term stride of the full P0 x L transform
    double2* T;            // inverse scratch pool (TermDesc::t_pool / t_vst)
    const double* w_pool;
    const double* phi_pool;
    const double* a_pool;  // lead-axis weight factors of family terms (TermDesc::a_off)
    // column chains (CM_APPLY_CHAIN): slots index chains; chain c has output descriptor chains[c]
    // and member terms chain_terms[chain_ptr[c] .. chain_ptr[c + 1])
    const TermDesc* chains;
    const int32_t* chain_ptr;
    const int32_t* chain_terms;
    double2* spec_pool;
    const double2* tw;     // twiddle tables: length L at tw + (L - 8)
    const TermDesc* gdesc; // global-mode pseudo term (s = dom_lo, o = [0,n))
    const int64_t* line_ptr;      // rows_inv CSR over the chunk's active output lines
    const int64_t* line_id;       // output line of each active line
    const int32_t* line_rng;      // [2*i], [2*i+1]: union of the entries' last-axis ranges
    const GatherEntry* entries;
    const BundleMember* members;  // RI_APPLY_B: bundle members (entries are bundle headers)
    double scale;          // 1 / prod P
};

enum RowsFwdMode { RF_APPLY = 0, RF_ADJ = 1, RF_SPEC = 2 };
enum ColsMode { CM_SPEC = 0, CM_APPLY_LOCAL = 1, CM_APPLY_GLOBAL = 2, CM_ADJ_LOCAL = 3, CM_ADJ_GLOBAL = 4,
                CM_APPLY_CHAIN = 5 };
enum MidMode { MM_FWD_APPLY = 0, MM_FWD_ADJ = 1, MM_FWD_SPEC = 2, MM_INV_APPLY = 3, MM_INV_ADJ = 4 };
enum RowsInvMode { RI_APPLY = 0, RI_ADJ = 1, RI_APPLY_B = 2, RI_ADJ_B = 3 };

// launchers (kernels.cu); return cudaGetLastError()
cudaError_t launch_rows_fwd(const PassArgs& a, int mode, cudaStream_t st);
int rows_lanes(int P_last);  // lines (rows_fwd) / gather lanes (rows_inv) per CTA for a last-axis length
cudaError_t launch_mid(const PassArgs& a, int mode, cudaStream_t st);
cudaError_t launch_cols(const PassArgs& a, int mode, cudaStream_t st);
cudaError_t launch_rows_inv(const PassArgs& a, int mode, int64_t n_lines, cudaStream_t st);
int cols_tile_width(int P0);

// entry / block gather (K6)
struct EntryArgs {
    int D;
    int64_t dom_lo[3];
    int32_t n[3];
    const TermDesc* terms;
    const double* w_pool;
    const double* phi_pool;
    int32_t bucket[3];          // bucket edge per axis
    int32_t nb[3];              // buckets per axis
    const int64_t* bucket_ptr;  // CSR over buckets (lexicographic)
    const int32_t* bucket_terms;
    int64_t kun_lo[3], kun_hi[3];  // union of the terms' kernel boxes K_k (lo > hi: no term)
    int32_t bucket_shift[3];       // log2 of the bucket edge when it is a power of two, else -1
};
cudaError_t launch_entries(const EntryArgs& a, int64_t cnt, const int64_t* y, const int64_t* x, double* out,
                           int32_t* bad, cudaStream_t st);
// bshape_host: the block shape per axis (host array, passed by value); scratch: device int32 of
// blocks_scratch_ints(nblk) (the list of blocks that need terms).  phase 0: those blocks (scan, then
// candidate search + gather); phase 1: the exact-zero blocks (independent of phase 0: run it on a
// second stream when blocks_two_streams()).
cudaError_t launch_blocks(const EntryArgs& a, int32_t nblk, const int64_t* t_origin, const int64_t* s_origin,
                          const int32_t* bshape_host, double* out, int32_t* bad, int32_t* scratch, int phase,
                          cudaStream_t st);
int64_t blocks_scratch_ints(int32_t nblk);
bool blocks_two_streams();

// block apply, direct form (small blocks)
cudaError_t launch_block_direct(const EntryArgs& a, int32_t nblk, int64_t max_t, const int64_t* t_lo,
                                const int64_t* t_hi, const int64_t* s_lo, const int64_t* s_hi, const int64_t* f_off,
                                const int64_t* g_off, const double* f, double* g, int adjoint, int32_t* bad,
                                cudaStream_t st);

// estimator reductions (K5): per (box, probe) sums of (Yt - Y)^2, and whole-domain (Yt - Y)^2 and
// Y^2 per probe (y2 needs q + probe_sums_scratch() doubles: the chunk partials follow it)
int64_t probe_sums_scratch(int D, const int32_t* n, int32_t q);
cudaError_t launch_probe_sums(int D, const int32_t* n, int32_t nbox, const int64_t* box_lo, const int64_t* box_hi,
                              int32_t q, const double* Yt, const double* Y, double* d2, double* y2, cudaStream_t st);

cudaError_t launch_zero(double* p, int64_t n, cudaStream_t st);
// out[off + i] = sum over t of parts[t][off + i], i < len (multi-device reduction; peer pointers)
cudaError_t launch_sum_parts(const double* const* d_parts, int nparts, int64_t off, int64_t len, double* out,
                             cudaStream_t st);
// count N(0,1) draws from Philox4x32-10 (counter = pair index, key = seed) + Box-Muller, on the device
cudaError_t launch_philox_normal(uint64_t seed, int64_t count, double* out, cudaStream_t st);

}  // namespace pcb
