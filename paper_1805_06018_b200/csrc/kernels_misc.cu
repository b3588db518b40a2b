// Entry / block gathers (K6), block apply (direct form), estimator reductions (K5).
#include <cstdio>

#include "fft.cuh"
#include "kernels.cuh"

namespace pcb {
namespace {

// ---------------------------------------------------------------------------
// K6: Atilde[y,x] = sum_{k: x in U_k} w_k[x] phi_k^E[y - x], k ascending, the
// reference's operation order (pc_operator.cpp:84-96) with IEEE mul/add (no FMA
// contraction) so the result is the reference's bit for bit.
__device__ __forceinline__ double entry_value(const EntryArgs& a, const int64_t* y, const int64_t* x, bool& bad) {
    const int D = a.D;
    int64_t bl = 0;
    for (int i = 0; i < D; ++i) {
        const int64_t yi = y[i] - a.dom_lo[i], xi = x[i] - a.dom_lo[i];
        if (yi < 0 || yi >= a.n[i] || xi < 0 || xi >= a.n[i]) {
            bad = true;
            return 0.0;
        }
        bl = bl * a.nb[i] + xi / a.bucket[i];
    }
    double sum = 0.0;
    for (int64_t q = a.bucket_ptr[bl]; q < a.bucket_ptr[bl + 1]; ++q) {
        const TermDesc& t = a.terms[a.bucket_terms[q]];
        int64_t wl = 0, zl = 0;
        bool inx = true, inz = true;
        for (int i = 0; i < D; ++i) {
            const int64_t u = x[i] - t.x_lo[i];
            if (u < 0 || u >= t.m[i]) inx = false;
            wl = wl * t.m[i] + u;
            const int64_t z = y[i] - x[i] - t.k_lo[i];
            if (z < 0 || z >= t.k_ext[i]) inz = false;
            zl = zl * t.k_ext[i] + z;
        }
        if (!inx) continue;
        const double wx = a.w_pool[t.w_off + wl];
        if (wx == 0.0) continue;
        const double ph = inz ? a.phi_pool[t.phi_off + zl] : 0.0;
        sum = __dadd_rn(sum, __dmul_rn(wx, ph));
    }
    return sum;
}

__global__ void k_entries(EntryArgs a, int64_t cnt, const int64_t* __restrict__ y, const int64_t* __restrict__ x,
                          double* __restrict__ out, int32_t* bad) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt; i += (int64_t)gridDim.x * blockDim.x) {
        bool b = false;
        const double v = entry_value(a, y + i * a.D, x + i * a.D, b);
        out[i] = v;
        if (b) atomicOr(bad, 1);
    }
}

__global__ void k_blocks(EntryArgs a, int32_t nblk, const int64_t* __restrict__ t_origin,
                         const int64_t* __restrict__ s_origin, const int32_t* __restrict__ bshape,
                         double* __restrict__ out, int32_t* bad) {
    const int D = a.D;
    int64_t bs = 1;
    for (int i = 0; i < D; ++i) bs *= bshape[i];
    const int64_t total = (int64_t)nblk * bs * bs;
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total; g += (int64_t)gridDim.x * blockDim.x) {
        const int64_t blk = g / (bs * bs);
        const int64_t rem = g - blk * bs * bs;
        int64_t i = rem / bs, j = rem - (rem / bs) * bs;
        int64_t y[3], x[3];
        for (int d = D - 1; d >= 0; --d) {
            y[d] = t_origin[blk * D + d] + i % bshape[d];
            i /= bshape[d];
            x[d] = s_origin[blk * D + d] + j % bshape[d];
            j /= bshape[d];
        }
        bool b = false;
        out[g] = entry_value(a, y, x, b);
        if (b) atomicOr(bad, 1);
    }
}

// Block apply, direct form (pc_operator.cpp:98-130 semantics): for block b,
//   apply:   g_b[y] = sum_{x in S_b} Atilde[y, x] f_b[x],   y in T_b
//   adjoint: g_b[x] = sum_{y in S_b} Atilde[y, x] f_b[y],   x in T_b
// One CTA per (block, tile of 256 outputs); f_b staged in shared memory in chunks.
__global__ void k_block_direct(EntryArgs a, int32_t nblk, const int64_t* __restrict__ t_lo,
                               const int64_t* __restrict__ t_hi, const int64_t* __restrict__ s_lo,
                               const int64_t* __restrict__ s_hi, const int64_t* __restrict__ f_off,
                               const int64_t* __restrict__ g_off, const double* __restrict__ f,
                               double* __restrict__ g, int adjoint, int32_t* bad) {
    const int D = a.D;
    const int blk = blockIdx.y;
    if (blk >= nblk) return;
    int64_t text[3] = {1, 1, 1}, sext[3] = {1, 1, 1}, tcnt = 1, scnt = 1;
    for (int i = 0; i < D; ++i) {
        text[i] = t_hi[blk * D + i] - t_lo[blk * D + i] + 1;
        sext[i] = s_hi[blk * D + i] - s_lo[blk * D + i] + 1;
        tcnt *= text[i];
        scnt *= sext[i];
    }
    const int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t pt[3] = {0, 0, 0};
    {
        int64_t r = o < tcnt ? o : 0;
        for (int i = D - 1; i >= 0; --i) {
            pt[i] = t_lo[blk * D + i] + r % text[i];
            r /= text[i];
        }
    }
    __shared__ double fs[512];
    double sum = 0.0;
    bool b = false;
    for (int64_t c0 = 0; c0 < scnt; c0 += 512) {
        const int cn = (int)((scnt - c0) < 512 ? (scnt - c0) : 512);
        __syncthreads();
        for (int i = threadIdx.x; i < cn; i += blockDim.x) fs[i] = f[f_off[blk] + c0 + i];
        __syncthreads();
        if (o < tcnt) {
            for (int j = 0; j < cn; ++j) {
                const double fv = fs[j];
                if (fv == 0.0) continue;
                int64_t ps[3] = {0, 0, 0};
                int64_t r = c0 + j;
                for (int i = D - 1; i >= 0; --i) {
                    ps[i] = s_lo[blk * D + i] + r % sext[i];
                    r /= sext[i];
                }
                const double e = adjoint ? entry_value(a, ps, pt, b) : entry_value(a, pt, ps, b);
                sum += e * fv;
            }
        }
    }
    if (o < tcnt) g[g_off[blk] + o] = sum;
    if (b) atomicOr(bad, 1);
}

// ---------------------------------------------------------------------------
// K5 reductions: d2[box, probe] = sum_{p in box cap Omega} (Yt - Y)^2, y2[probe] = sum Y^2
__global__ void k_probe_sums(int D, int32_t n0, int32_t n1, int32_t n2, int32_t nbox, const int64_t* __restrict__ blo,
                             const int64_t* __restrict__ bhi, const double* __restrict__ Yt,
                             const double* __restrict__ Y, double* d2, double* y2) {
    const int box = blockIdx.x;  // box == nbox -> whole domain (also sums Y^2)
    const int probe = blockIdx.y;
    const int32_t n[3] = {n0, n1, D == 3 ? n2 : 1};
    int64_t lo[3] = {0, 0, 0}, hi[3] = {n0 - 1, n1 - 1, n[2] - 1};
    if (box < nbox) {
        for (int i = 0; i < D; ++i) {
            lo[i] = blo[box * D + i] > 0 ? blo[box * D + i] : 0;
            hi[i] = bhi[box * D + i] < n[i] - 1 ? bhi[box * D + i] : n[i] - 1;
        }
    }
    int64_t ext[3];
    int64_t cnt = 1;
    for (int i = 0; i < 3; ++i) {
        ext[i] = hi[i] >= lo[i] ? hi[i] - lo[i] + 1 : 0;
        cnt *= ext[i];
    }
    const int64_t N = (int64_t)n[0] * n[1] * n[2];
    const double* yt = Yt + probe * N;
    const double* yy = Y + probe * N;
    double s = 0.0, sy = 0.0;
    for (int64_t q = threadIdx.x; q < cnt; q += blockDim.x) {
        const int64_t i2 = q % ext[2];
        const int64_t r = q / ext[2];
        const int64_t i1 = r % ext[1];
        const int64_t i0 = r / ext[1];
        const int64_t off = ((lo[0] + i0) * n[1] + lo[1] + i1) * n[2] + lo[2] + i2;
        const double dv = yt[off] - yy[off];
        s += dv * dv;
        sy += yy[off] * yy[off];
    }
    __shared__ double red[2][256];
    red[0][threadIdx.x] = s;
    red[1][threadIdx.x] = sy;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) {
            red[0][threadIdx.x] += red[0][threadIdx.x + w];
            red[1][threadIdx.x] += red[1][threadIdx.x + w];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        d2[(int64_t)box * gridDim.y + probe] = red[0][0];
        if (box == nbox) y2[probe] = red[1][0];
    }
}

__global__ void k_zero(double* p, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) p[i] = 0.0;
}

}  // namespace

cudaError_t launch_entries(const EntryArgs& a, int64_t cnt, const int64_t* y, const int64_t* x, double* out,
                           int32_t* bad, cudaStream_t st) {
    if (cnt <= 0) return cudaSuccess;
    const int64_t blocks = (cnt + 255) / 256;
    k_entries<<<(unsigned)(blocks < 148 * 64 ? blocks : 148 * 64), 256, 0, st>>>(a, cnt, y, x, out, bad);
    return cudaGetLastError();
}

cudaError_t launch_blocks(const EntryArgs& a, int32_t nblk, const int64_t* t_origin, const int64_t* s_origin,
                          const int32_t* bshape, double* out, int32_t* bad, cudaStream_t st) {
    if (nblk <= 0) return cudaSuccess;
    k_blocks<<<148 * 16, 256, 0, st>>>(a, nblk, t_origin, s_origin, bshape, out, bad);
    return cudaGetLastError();
}

cudaError_t launch_probe_sums(int D, const int32_t* n, int32_t nbox, const int64_t* box_lo, const int64_t* box_hi,
                              int32_t q, const double* Yt, const double* Y, double* d2, double* y2, cudaStream_t st) {
    dim3 grid((unsigned)(nbox + 1), (unsigned)q);
    k_probe_sums<<<grid, 256, 0, st>>>(D, n[0], n[1], D == 3 ? n[2] : 1, nbox, box_lo, box_hi, Yt, Y, d2, y2);
    return cudaGetLastError();
}

cudaError_t launch_block_direct(const EntryArgs& a, int32_t nblk, int64_t max_t, const int64_t* t_lo,
                                const int64_t* t_hi, const int64_t* s_lo, const int64_t* s_hi, const int64_t* f_off,
                                const int64_t* g_off, const double* f, double* g, int adjoint, int32_t* bad,
                                cudaStream_t st) {
    if (nblk <= 0) return cudaSuccess;
    dim3 grid((unsigned)((max_t + 255) / 256), (unsigned)nblk);
    k_block_direct<<<grid, 256, 0, st>>>(a, nblk, t_lo, t_hi, s_lo, s_hi, f_off, g_off, f, g, adjoint, bad);
    return cudaGetLastError();
}

cudaError_t launch_zero(double* p, int64_t n, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    k_zero<<<148 * 8, 256, 0, st>>>(p, n);
    return cudaGetLastError();
}

}  // namespace pcb
