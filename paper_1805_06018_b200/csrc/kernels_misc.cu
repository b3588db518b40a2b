// Entry / block gathers (K6), block apply (direct form), estimator reductions (K5).
#include <algorithm>
#include <cstdio>
#include <cstdlib>

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
                         const int64_t* __restrict__ s_origin, int bs0, int bs1, int bs2, double* __restrict__ out,
                         int32_t* bad) {
    const int D = a.D;
    const int bshape[3] = {bs0, bs1, bs2};
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
                               double* __restrict__ g, int adjoint, int32_t* bad, int32_t blk0, uint32_t tiles) {
    // 1-D grid: CTA = (block, tile of 256 outputs) -- batched H-matrix rounds pass more blocks than
    // grid.y allows
    const int D = a.D;
    const int blk = blk0 + (int)(blockIdx.x / tiles);
    const uint32_t tile = blockIdx.x % tiles;
    if (blk >= nblk) return;
    int64_t text[3] = {1, 1, 1}, sext[3] = {1, 1, 1}, tcnt = 1, scnt = 1;
    for (int i = 0; i < D; ++i) {
        text[i] = t_hi[blk * D + i] - t_lo[blk * D + i] + 1;
        sext[i] = s_hi[blk * D + i] - s_lo[blk * D + i] + 1;
        tcnt *= text[i];
        scnt *= sext[i];
    }
    const int64_t o = (int64_t)tile * blockDim.x + threadIdx.x;
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
// Estimator sums (K5).  CTA (x < nbox, probe): sum over leaf box x of (Yt - Y)^2.  CTA
// (x = nbox + c, probe): chunk c of PS_CHUNK consecutive points of the whole domain, (Yt - Y)^2
// and Y^2, into partials reduced by k_probe_total in chunk order (deterministic).
constexpr int PS_CHUNK = 16384;

__global__ void __launch_bounds__(256) k_probe_sums(int D, int32_t n0, int32_t n1, int32_t n2, int32_t nbox,
                                                    const int64_t* __restrict__ blo, const int64_t* __restrict__ bhi,
                                                    const double* __restrict__ Yt, const double* __restrict__ Y,
                                                    double* d2, double* part) {
    const int box = blockIdx.x;
    const int probe = blockIdx.y;
    const int q = gridDim.y;
    const int32_t n[3] = {n0, n1, D == 3 ? n2 : 1};
    const int64_t N = (int64_t)n[0] * n[1] * n[2];
    const double* yt = Yt + probe * N;
    const double* yy = Y + probe * N;
    double s = 0.0, sy = 0.0;
    if (box < nbox) {
        int64_t lo[3] = {0, 0, 0}, ext[3] = {1, 1, 1};
        for (int i = 0; i < D; ++i) {
            const int64_t l = blo[box * D + i] > 0 ? blo[box * D + i] : 0;
            const int64_t h = bhi[box * D + i] < n[i] - 1 ? bhi[box * D + i] : n[i] - 1;
            lo[i] = l;
            ext[i] = h >= l ? h - l + 1 : 0;
        }
        const int ax = D - 1;  // rows of the box along the last axis: one division per row
        const int64_t rows = D == 3 ? ext[0] * ext[1] : ext[0];
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        for (int64_t r = warp; r < rows; r += blockDim.x >> 5) {
            const int64_t r0 = D == 3 ? r / ext[1] : r, r1 = D == 3 ? r - (r / ext[1]) * ext[1] : 0;
            const int64_t base = D == 3 ? ((lo[0] + r0) * n[1] + lo[1] + r1) * n[2] + lo[2] : (lo[0] + r0) * n[1] + lo[1];
            for (int64_t c = lane; c < ext[ax]; c += 32) {
                const double dv = yt[base + c] - yy[base + c];
                s += dv * dv;
            }
        }
    } else {
        const int64_t c0 = (int64_t)(box - nbox) * PS_CHUNK;
        const int64_t c1 = c0 + PS_CHUNK < N ? c0 + PS_CHUNK : N;
        for (int64_t i = c0 + threadIdx.x; i < c1; i += blockDim.x) {
            const double dv = yt[i] - yy[i];
            s += dv * dv;
            sy += yy[i] * yy[i];
        }
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
        if (box < nbox) {
            d2[(int64_t)box * q + probe] = red[0][0];
        } else {
            const int64_t c = box - nbox;
            part[(c * q + probe) * 2] = red[0][0];
            part[(c * q + probe) * 2 + 1] = red[1][0];
        }
    }
}

// whole-domain sums per probe from the chunk partials, in chunk order
__global__ void k_probe_total(int32_t nbox, int32_t q, int64_t nchunk, const double* __restrict__ part, double* d2,
                              double* y2) {
    const int probe = blockIdx.x * blockDim.x + threadIdx.x;
    if (probe >= q) return;
    double s = 0.0, sy = 0.0;
    for (int64_t c = 0; c < nchunk; ++c) {
        s += part[(c * q + probe) * 2];
        sy += part[(c * q + probe) * 2 + 1];
    }
    d2[(int64_t)nbox * q + probe] = s;
    y2[probe] = sy;
}

__global__ void k_zero(double* p, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) p[i] = 0.0;
}

// K6 for dense blocks (config 5): constants and helpers; the passes follow below.
#ifndef PCB_BZ_DOUBLES
// zero tile: 32 KiB, one bulk copy per 64 x 64 block.  Measured at config 5 with the gather pass
// beside the fill: 4 KiB tiles (8 copies per block) 42.7 us per call, 32 KiB 33.1 us -- fewer, larger
// requests from the fill delay the gather's dependent loads less (gather pass 45.5 -> 37 us)
#define PCB_BZ_DOUBLES 4096
#endif
constexpr int BZ_DOUBLES = PCB_BZ_DOUBLES;
constexpr int BT_CAP = 32;  // max staged candidate terms per block
constexpr int BT_IDS = 64;  // gathered bucket entries (with duplicates) per block
constexpr int BT_NZ = 8;    // listed nonzero-weight terms per source point
constexpr int BC_WARPS = 8; // blocks (warps) per zero-fill CTA
constexpr int BT_PXMAX = 256;   // gather kernel: max points per block (coordinate tables)
constexpr int BT_WINMAX = 1024; // ... max window offsets

__device__ __forceinline__ void bulk_store_s2g(void* gdst, const void* ssrc, uint32_t bytes) {
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(ssrc);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(s), "r"(bytes) : "memory");
}

// the same with an L2 evict-first policy: the zero fill streams through L2 without evicting the
// operator's pools, buckets and descriptors that the gather's dependent loads need
__device__ __forceinline__ void bulk_store_s2g_ef(void* gdst, const void* ssrc, uint32_t bytes, uint64_t pol) {
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(ssrc);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(gdst), "r"(s),
                 "r"(bytes), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

// ---------------------------------------------------------------------------
// Dense blocks, two independent passes (on two streams; PCB_BLOCKS_STREAMS=1: one after the other):
//   * every block first takes a geometric test on its origins alone: if on some axis the offsets
//     T - S = [t - s - (bs - 1), t - s + (bs - 1)] miss the union of all kernel boxes, every entry
//     reads phi^E = 0 and the block is an exact zero (config 5: 3,9xx of 4096 blocks);
//   * k_blocks_zfill writes those blocks with TMA bulk copies of a zeroed shared tile (L2
//     evict-first): one load of the origins, then stores -- the write stream starts at once instead
//     of after the candidate search (a chain of dependent loads through buckets and descriptors);
//   * k_blocks_scan lists the others (one thread per block) and k_blocks_fused takes one listed
//     block per CTA: warp 0 finds the block's candidate terms (classify_block), then the CTA stages
//     their weights and phi^E windows ((2 bs - 1) offsets per axis) in shared memory and sums every entry
//     in ascending k (bit-identical to entry_value), or writes zeros when no candidate is left.
//     The two passes write disjoint blocks and need nothing from each other: two streams.
// Measured at config 5 (us per call): the round-2 design before it (a classify pass over every block
// that also wrote the zero blocks, then a gather pass over the listed ones) 58; this 33.1 (42.7 with
// 4 KiB zero tiles); on one stream 54 (gather path 28, fill 29).  One launch with gather CTAs that scan the origins themselves: 65
// (every CTA re-reads all origins), and with the fill gated behind the gather CTAs' reads 81 -- a
// read issued behind the saturating write stream takes ~10 us, so the passes gain nothing from
// sharing a launch; the fill alone runs at 4.4 TB/s.

// 0: exact zero by the union-box test, 1: needs the candidate search, 2: leaves the domain
__device__ __forceinline__ int block_kind(const EntryArgs& a, const int64_t* tv, const int64_t* sv, const int* bs) {
    int kind = 1;
    for (int i = 0; i < a.D; ++i) {
        if (tv[i] < a.dom_lo[i] || tv[i] + bs[i] > a.dom_lo[i] + a.n[i] || sv[i] < a.dom_lo[i] ||
            sv[i] + bs[i] > a.dom_lo[i] + a.n[i])
            return 2;
        const int64_t o = tv[i] - sv[i];
        if (o + (bs[i] - 1) < a.kun_lo[i] || o - (bs[i] - 1) > a.kun_hi[i]) kind = 0;
    }
    return kind;
}

// One warp: the candidate terms of block (tv, sv) in ascending k into cand[] -- the terms listed in
// the buckets covering S, deduplicated, kept when X_k meets S and K_k meets the offsets T - S.
// Returns their number, or -1 when the lists do not fit (per-entry path).  ids / first: BT_IDS ints
// of shared memory each, private to the warp.
__device__ int classify_block(const EntryArgs& a, const int64_t* tv, const int64_t* sv, const int* bs, int cap,
                              int* ids, int* first, int* cand, int lane) {
    const int D = a.D;
    int blo[3] = {0, 0, 0}, bn[3] = {1, 1, 1}, nbk = 1;
    for (int i = 0; i < D; ++i) {  // 32-bit arithmetic: domain axes are < 2^20
        const int rel = (int)(sv[i] - a.dom_lo[i]);
        const int sh = a.bucket_shift[i];  // >= 0: the bucket edge is 2^sh (no division)
        blo[i] = sh >= 0 ? rel >> sh : rel / a.bucket[i];
        bn[i] = (sh >= 0 ? (rel + bs[i] - 1) >> sh : (rel + bs[i] - 1) / a.bucket[i]) - blo[i] + 1;
        nbk *= bn[i];
    }
    int64_t beg = 0;
    int cnt = 0;
    if (nbk <= 32 && lane < nbk) {
        int r = lane, c[3] = {0, 0, 0};
        for (int i = D - 1; i >= 0; --i) {
            c[i] = blo[i] + r % bn[i];
            r /= bn[i];
        }
        int bl = 0;
        for (int i = 0; i < D; ++i) bl = bl * a.nb[i] + c[i];
        beg = a.bucket_ptr[bl];
        cnt = (int)(a.bucket_ptr[bl + 1] - beg);
    }
    int off = cnt;  // inclusive warp prefix sum
    for (int d = 1; d < 32; d <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, off, d);
        if (lane >= d) off += v;
    }
    const int total = __shfl_sync(0xffffffffu, off, 31);
    off -= cnt;
    if (nbk > 32 || total > BT_IDS) return -1;
    int64_t src[2] = {-1, -1};
    for (int b = 0; b < nbk; ++b) {
        const int ob = __shfl_sync(0xffffffffu, off, b);
        const int cb = __shfl_sync(0xffffffffu, cnt, b);
        const int64_t gb = __shfl_sync(0xffffffffu, beg, b);
        for (int h = 0; h < 2; ++h) {
            const int pos = lane + 32 * h;
            if (pos >= ob && pos < ob + cb) src[h] = gb + (pos - ob);
        }
    }
    int got[2];
    for (int h = 0; h < 2; ++h) got[h] = src[h] >= 0 ? a.bucket_terms[src[h]] : 0;
    for (int h = 0; h < 2; ++h)
        if (lane + 32 * h < total) ids[lane + 32 * h] = got[h];
    __syncwarp();
    int keep[2] = {0, 0}, idv[2] = {0, 0};
    for (int h = 0; h < 2; ++h) {
        const int pos = lane + 32 * h;
        if (pos >= total) continue;
        const int id = ids[pos];
        int f = 1;
        for (int j = 0; j < pos; ++j) f &= ids[j] != id;
        if (f) {
            const TermDesc& t = a.terms[id];
            for (int d = 0; d < D && f; ++d) {
                const int64_t o = tv[d] - sv[d];
                f &= (t.x_lo[d] <= sv[d] + bs[d] - 1) && (t.x_lo[d] + t.m[d] - 1 >= sv[d]) &&
                     (t.k_lo[d] <= o + bs[d] - 1) && (t.k_lo[d] + t.k_ext[d] - 1 >= o - (bs[d] - 1));
            }
        }
        keep[h] = f;
        idv[h] = id;
        first[pos] = f ? id : -1;
    }
    __syncwarp();
    const int nk = __popc(__ballot_sync(0xffffffffu, keep[0])) + __popc(__ballot_sync(0xffffffffu, keep[1]));
    if (nk > cap) return -1;
    for (int h = 0; h < 2; ++h) {
        if (!keep[h]) continue;
        int rank = 0;
        for (int j = 0; j < total; ++j) rank += first[j] >= 0 && first[j] < idv[h];
        cand[rank] = idv[h];
    }
    __syncwarp();
    return nk;
}

// zero fill of one block by one warp.  zvar 0: TMA bulk copies of the zero tile with an L2
// evict-first hint, 1: the same without the hint, 2: 16-byte streaming stores
__device__ __forceinline__ bool zero_block(double* ob_d, int64_t n2, const double* Z, int lane, int zvar) {
    const int64_t bytes = n2 * 8;
    char* ob = reinterpret_cast<char*>(ob_d);
    bool issued = false;
    if ((reinterpret_cast<uintptr_t>(ob) & 15) != 0) {
        for (int64_t e = lane; e < n2; e += 32) ob_d[e] = 0.0;
        return false;
    }
    if (zvar == 2) {
        double2* o2 = reinterpret_cast<double2*>(ob);
        for (int64_t e = lane; e < n2 / 2; e += 32) __stcs(&o2[e], make_double2(0.0, 0.0));
        if ((n2 & 1) && lane == 0) ob_d[n2 - 1] = 0.0;
        return false;
    }
    // lanes share the block's tiles: up to 32 bulk copies in flight per warp
    const int64_t ntile = bytes / (BZ_DOUBLES * 8);
    const uint64_t pol = l2_evict_first_policy();
    for (int64_t t = lane; t < ntile; t += 32) {
        if (zvar == 0) bulk_store_s2g_ef(ob + t * (BZ_DOUBLES * 8), Z, BZ_DOUBLES * 8, pol);
        else bulk_store_s2g(ob + t * (BZ_DOUBLES * 8), Z, BZ_DOUBLES * 8);
        issued = true;
    }
    if (lane == 0) {
        const int64_t o = ntile * (BZ_DOUBLES * 8);
        const int64_t tail = (bytes - o) & ~(int64_t)15;
        if (tail > 0) {
            bulk_store_s2g(ob + o, Z, (uint32_t)tail);
            issued = true;
        }
        if (bytes & 15) ob_d[n2 - 1] = 0.0;
    }
    if (issued) asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    return issued;
}

__global__ void __launch_bounds__(256) k_blocks_zfill(EntryArgs a, int32_t nblk, const int64_t* __restrict__ t_origin,
                                                      const int64_t* __restrict__ s_origin, int bs0, int bs1, int bs2,
                                                      double* __restrict__ out, int zvar) {
    __shared__ __align__(128) double Z[BZ_DOUBLES];
    const int D = a.D;
    const int bs[3] = {bs0, bs1, bs2};
    int64_t npx = 1;
    for (int i = 0; i < D; ++i) npx *= bs[i];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    for (int i = tid; i < BZ_DOUBLES; i += blockDim.x) Z[i] = 0.0;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    bool issued = false;
    // a warp per block; with a grid smaller than the block count the warps stride over the blocks
    for (int64_t blk = (int64_t)blockIdx.x * BC_WARPS + wid; blk < nblk; blk += (int64_t)gridDim.x * BC_WARPS) {
        int64_t tv[3] = {0, 0, 0}, sv[3] = {0, 0, 0};
        for (int i = 0; i < D; ++i) {
            tv[i] = t_origin[blk * D + i];
            sv[i] = s_origin[blk * D + i];
        }
        if (block_kind(a, tv, sv, bs) == 0) issued = zero_block(out + blk * npx * npx, npx * npx, Z, lane, zvar) || issued;
    }
    if (issued) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // Z read before the CTA exits
}

// listed blocks (int64 x BR_WORDS each): block index, kind, T origin [3], S origin [3]
constexpr int BR_WORDS = 8;

// one thread per block: the blocks that fail the zero test are listed (scr[0] counts them) with their
// origins, so a gather CTA starts from one load
__global__ void __launch_bounds__(256) k_blocks_scan(EntryArgs a, int32_t nblk, const int64_t* __restrict__ t_origin,
                                                     const int64_t* __restrict__ s_origin, int bs0, int bs1, int bs2,
                                                     int32_t* __restrict__ scr, int64_t* __restrict__ rec) {
    const int D = a.D;
    const int bs[3] = {bs0, bs1, bs2};
    const int blk = blockIdx.x * blockDim.x + threadIdx.x;
    int kind = 0;
    int64_t tv[3] = {0, 0, 0}, sv[3] = {0, 0, 0};
    if (blk < nblk) {
        for (int i = 0; i < D; ++i) {
            tv[i] = t_origin[(int64_t)blk * D + i];
            sv[i] = s_origin[(int64_t)blk * D + i];
        }
        kind = block_kind(a, tv, sv, bs);
    }
    const unsigned m = __ballot_sync(0xffffffffu, kind != 0);
    if (m == 0) return;
    const int lane = threadIdx.x & 31;
    int base = 0;
    if (lane == __ffs(m) - 1) base = atomicAdd(scr, __popc(m));
    base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
    if (kind != 0) {
        int64_t* r = rec + (int64_t)(base + __popc(m & ((1u << lane) - 1))) * BR_WORDS;
        r[0] = blk;
        r[1] = kind;
        for (int i = 0; i < 3; ++i) {
            r[2 + i] = tv[i];
            r[5 + i] = sv[i];
        }
    }
}

// one listed block per CTA (persistent over the list when it is longer than the grid)
__global__ void __launch_bounds__(256) k_blocks_fused(EntryArgs a, int32_t nblk, int bs0, int bs1, int bs2, int cap,
                                                      double* __restrict__ out, int32_t* bad,
                                                      const int32_t* __restrict__ scr,
                                                      const int64_t* __restrict__ rec) {
    extern __shared__ double sm[];
    const int D = a.D;
    const int bs[3] = {bs0, bs1, bs2};
    int npx = 1, win = 1;
    for (int i = 0; i < D; ++i) {
        npx *= bs[i];
        win *= 2 * bs[i] - 1;
    }
    const int tid = threadIdx.x, lane = tid & 31;
    double* W = sm;               // [cap][npx]
    double* PH = W + cap * npx;   // [cap][win]
    int* offs = reinterpret_cast<int*>(PH + cap * win);              // [npx] window offset of a point
    unsigned char* nzn = reinterpret_cast<unsigned char*>(offs + npx);  // [npx] nonzero-term count
    unsigned char* nzc = nzn + npx;                                   // [npx][BT_NZ] their indices
    __shared__ int64_t s_rec[BR_WORDS];
    __shared__ int s_nc;
    __shared__ int s_ids[BT_IDS], s_first[BT_IDS], s_cand[BT_CAP];
    __shared__ int64_t c_woff[BT_CAP], c_poff[BT_CAP];
    __shared__ int32_t c_xlo[BT_CAP][3], c_klo[BT_CAP][3], c_m[BT_CAP][3], c_kext[BT_CAP][3];
    __shared__ int16_t pco[BT_PXMAX][3], wco[BT_WINMAX][3];
    // the count and this CTA's first record in one round trip (records past the count are stale)
    const int nwork = scr[0];
    if (tid < BR_WORDS && (int)blockIdx.x < nblk) s_rec[tid] = rec[(int64_t)blockIdx.x * BR_WORDS + tid];
    if ((int)blockIdx.x >= nwork) return;
    int centre = 0;
    {
        int mul = 1;
        for (int d = D - 1; d >= 0; --d) {
            centre += (bs[d] - 1) * mul;
            mul *= 2 * bs[d] - 1;
        }
    }
    for (int p = tid; p < npx; p += blockDim.x) {
        int r = p, o = 0, mul = 1;
        for (int d = D - 1; d >= 0; --d) {
            o += (r % bs[d]) * mul;
            mul *= 2 * bs[d] - 1;
            pco[p][d] = (int16_t)(r % bs[d]);
            r /= bs[d];
        }
        offs[p] = o;
    }
    for (int w = tid; w < win; w += blockDim.x) {
        int r = w;
        for (int d = D - 1; d >= 0; --d) {
            const int wd = 2 * bs[d] - 1;
            wco[w][d] = (int16_t)(r % wd - (bs[d] - 1));
            r /= wd;
        }
    }
    for (int wi = blockIdx.x; wi < nwork; wi += gridDim.x) {
        __syncthreads();  // the previous block's gather is done with the shared lists and the record
        if (wi != (int)blockIdx.x && tid < BR_WORDS) s_rec[tid] = rec[(int64_t)wi * BR_WORDS + tid];
        __syncthreads();
        const int64_t blk = s_rec[0];
        const int kind = (int)s_rec[1];
        const int64_t* s_t = s_rec + 2;
        const int64_t* s_s = s_rec + 5;
        if (tid < 32) {
            int nk = -1;
            if (kind == 1) nk = classify_block(a, s_t, s_s, bs, cap, s_ids, s_first, s_cand, lane);
            if (lane == 0) s_nc = nk;
        }
        __syncthreads();
        const int nc = s_nc;
        const int* cand = s_cand;
        double* ob = out + (int64_t)blk * npx * npx;
        if (nc < 0) {  // per-entry path (out-of-domain entries flag `bad`)
            for (int e = tid; e < npx * npx; e += blockDim.x) {
                int i = e / npx, j = e - (e / npx) * npx;
                int64_t y[3], x[3];
                for (int d = D - 1; d >= 0; --d) {
                    y[d] = s_t[d] + i % bs[d];
                    i /= bs[d];
                    x[d] = s_s[d] + j % bs[d];
                    j /= bs[d];
                }
                bool b = false;
                ob[e] = entry_value(a, y, x, b);
                if (b) atomicOr(bad, 1);
            }
            continue;
        }
        if (nc == 0) {  // no term contributes: an exact zero block
            if ((reinterpret_cast<uintptr_t>(ob) & 15) == 0) {
                double2* o2 = reinterpret_cast<double2*>(ob);
                const int64_t n2 = (int64_t)npx * npx;
                for (int64_t e = tid; e < n2 / 2; e += blockDim.x) o2[e] = make_double2(0.0, 0.0);
                if ((n2 & 1) && tid == 0) ob[n2 - 1] = 0.0;
            } else {
                for (int e = tid; e < npx * npx; e += blockDim.x) ob[e] = 0.0;
            }
            continue;
        }
        if (tid < nc) {  // candidate geometry relative to the block (32-bit: axes are < 2^20)
            const TermDesc& t = a.terms[cand[tid]];
            for (int d = 0; d < 3; ++d) {
                c_xlo[tid][d] = d < D ? (int32_t)(t.x_lo[d] - s_s[d]) : 0;              // X_k.lo - S.lo
                c_klo[tid][d] = d < D ? (int32_t)(t.k_lo[d] - (s_t[d] - s_s[d])) : 0;  // K_k.lo - (T - S).lo
                c_m[tid][d] = t.m[d];
                c_kext[tid][d] = t.k_ext[d];
            }
            c_woff[tid] = t.w_off;
            c_poff[tid] = t.phi_off;
        }
        __syncthreads();
#pragma unroll 4
        for (int idx = tid; idx < nc * npx; idx += blockDim.x) {  // w_k on S (0 outside X_k)
            const int c = idx / npx;
            const int j = idx - c * npx;
            bool in = true;
            int wl = 0;
            for (int d = 0; d < D; ++d) {
                const int u = pco[j][d] - c_xlo[c][d];
                in = in && u >= 0 && u < c_m[c][d];
                wl = wl * c_m[c][d] + u;
            }
            W[idx] = in ? a.w_pool[c_woff[c] + wl] : 0.0;
        }
#pragma unroll 8
        for (int idx = tid; idx < nc * win; idx += blockDim.x) {  // phi_k^E on the offsets T - S
            const int c = idx / win;
            const int w2 = idx - c * win;
            bool in = true;
            int zl = 0;
            for (int d = 0; d < D; ++d) {
                const int z = wco[w2][d] - c_klo[c][d];
                in = in && z >= 0 && z < c_kext[c][d];
                zl = zl * c_kext[c][d] + z;
            }
            PH[idx] = in ? a.phi_pool[c_poff[c] + zl] : 0.0;
        }
        __syncthreads();
        for (int j = tid; j < npx; j += blockDim.x) {  // per source point: its terms with w != 0
            int q = 0;
            for (int c = 0; c < nc; ++c)
                if (W[c * npx + j] != 0.0) {
                    if (q < BT_NZ) nzc[j * BT_NZ + q] = (unsigned char)c;
                    ++q;
                }
            nzn[j] = (unsigned char)(q <= BT_NZ ? q : 255);
        }
        __syncthreads();
        // entry (i, j): window index T_off[i] - S_off[j] + centre (the per-axis offset is linear)
        for (int e = tid; e < npx * npx; e += blockDim.x) {
            const int i = e / npx, j = e - i * npx;
            const int widx = offs[i] - offs[j] + centre;
            double sum = 0.0;
            const int q = nzn[j];
            if (q != 255) {
                for (int r = 0; r < q; ++r) {
                    const int c = nzc[j * BT_NZ + r];
                    sum = __dadd_rn(sum, __dmul_rn(W[c * npx + j], PH[c * win + widx]));
                }
            } else {
                for (int c = 0; c < nc; ++c) {
                    const double wv = W[c * npx + j];
                    if (wv != 0.0) sum = __dadd_rn(sum, __dmul_rn(wv, PH[c * win + widx]));
                }
            }
            ob[e] = sum;
        }
    }
}

}  // namespace

cudaError_t launch_entries(const EntryArgs& a, int64_t cnt, const int64_t* y, const int64_t* x, double* out,
                           int32_t* bad, cudaStream_t st) {
    if (cnt <= 0) return cudaSuccess;
    const int64_t blocks = (cnt + 255) / 256;
    k_entries<<<(unsigned)(blocks < 148 * 64 ? blocks : 148 * 64), 256, 0, st>>>(a, cnt, y, x, out, bad);
    return cudaGetLastError();
}

bool blocks_two_streams() {
    static const bool two = [] {
        const char* e = getenv("PCB_BLOCKS_STREAMS");
        return e ? atoi(e) != 1 : true;
    }();
    return two;
}

// int32 scratch: [0] the scan's counter, [4, 4 + 16 nblk) its records (BR_WORDS int64 per block)
int64_t blocks_scratch_ints(int32_t nblk) { return 4 + 2 * (int64_t)BR_WORDS * nblk; }

cudaError_t launch_blocks(const EntryArgs& a, int32_t nblk, const int64_t* t_origin, const int64_t* s_origin,
                          const int32_t* bshape_host, double* out, int32_t* bad, int32_t* scratch, int phase,
                          cudaStream_t st) {
    if (nblk <= 0) return cudaSuccess;
    int64_t npx = 1, win = 1;
    for (int i = 0; i < a.D; ++i) {
        npx *= bshape_host[i];
        win *= 2 * (int64_t)bshape_host[i] - 1;
    }
    static const int cap = [] {  // staged terms per block (PCB_BLOCK_CAP, <= BT_CAP)
        const char* e = getenv("PCB_BLOCK_CAP");
        return e ? std::max(1, std::min(BT_CAP, atoi(e))) : 16;
    }();
    const size_t smem = sizeof(double) * (size_t)cap * (size_t)(npx + win) + sizeof(int) * (size_t)npx +
                        (size_t)npx * (1 + BT_NZ) + 16;
    const int bs1 = a.D > 1 ? bshape_host[1] : 1, bs2 = a.D > 2 ? bshape_host[2] : 1;
    if (smem > 120 * 1024 || npx > BT_PXMAX || win > BT_WINMAX) {  // too large to stage: per-entry kernel
        if (phase != 0) return cudaSuccess;
        k_blocks<<<148 * 16, 256, 0, st>>>(a, nblk, t_origin, s_origin, bshape_host[0], bs1, bs2, out, bad);
        return cudaGetLastError();
    }
    if (phase == 1) {  // the zero fill
        static const int zvar = [] {  // zero_block variant (A/B)
            const char* e = getenv("PCB_C5_ZVAR");
            return e ? std::max(0, std::min(2, atoi(e))) : 0;
        }();
        const unsigned zgrid = (unsigned)((nblk + BC_WARPS - 1) / BC_WARPS);
        k_blocks_zfill<<<zgrid, 32 * BC_WARPS, 0, st>>>(a, nblk, t_origin, s_origin, bshape_host[0], bs1, bs2, out, zvar);
        return cudaGetLastError();
    }
    // phase 0: the blocks that need terms (scan, then search + gather)
    cudaError_t e = cudaMemsetAsync(scratch, 0, 4 * sizeof(int32_t), st);
    if (e != cudaSuccess) return e;
    int64_t* rec = reinterpret_cast<int64_t*>(scratch + 4);
    k_blocks_scan<<<(unsigned)((nblk + 255) / 256), 256, 0, st>>>(a, nblk, t_origin, s_origin, bshape_host[0], bs1, bs2,
                                                                  scratch, rec);
    if (smem > 36 * 1024) {  // (static shared memory takes ~11 KB of the default 48)
        e = cudaFuncSetAttribute(k_blocks_fused, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    const int per_sm = std::max<int>(1, std::min<int>(6, (int)((220 * 1024) / (smem + 12 * 1024))));
    const int grid = (int)std::min<int64_t>(nblk, 148LL * per_sm);
    k_blocks_fused<<<grid, 256, smem, st>>>(a, nblk, bshape_host[0], bs1, bs2, cap, out, bad, scratch, rec);
    return cudaGetLastError();
}

cudaError_t launch_probe_sums(int D, const int32_t* n, int32_t nbox, const int64_t* box_lo, const int64_t* box_hi,
                              int32_t q, const double* Yt, const double* Y, double* d2, double* y2, cudaStream_t st) {
    // chunk partials live behind the q whole-domain y2 slots of the caller's buffer (see
    // probe_sums_scratch)
    const int64_t N = (int64_t)n[0] * n[1] * (D == 3 ? n[2] : 1);
    const int64_t nchunk = (N + PS_CHUNK - 1) / PS_CHUNK;
    double* part = y2 + q;
    dim3 grid((unsigned)(nbox + nchunk), (unsigned)q);
    k_probe_sums<<<grid, 256, 0, st>>>(D, n[0], n[1], D == 3 ? n[2] : 1, nbox, box_lo, box_hi, Yt, Y, d2, part);
    k_probe_total<<<(q + 127) / 128, 128, 0, st>>>(nbox, q, nchunk, part, d2, y2);
    return cudaGetLastError();
}

cudaError_t launch_block_direct(const EntryArgs& a, int32_t nblk, int64_t max_t, const int64_t* t_lo,
                                const int64_t* t_hi, const int64_t* s_lo, const int64_t* s_hi, const int64_t* f_off,
                                const int64_t* g_off, const double* f, double* g, int adjoint, int32_t* bad,
                                cudaStream_t st) {
    if (nblk <= 0) return cudaSuccess;
    const int64_t tiles = std::max<int64_t>(1, (max_t + 255) / 256);
    const int64_t per = std::max<int64_t>(1, ((1LL << 31) - 1) / tiles);  // blocks per launch (grid.x limit)
    for (int64_t b0 = 0; b0 < nblk; b0 += per) {
        const int64_t nb = std::min<int64_t>(per, nblk - b0);
        k_block_direct<<<(unsigned)(nb * tiles), 256, 0, st>>>(a, nblk, t_lo, t_hi, s_lo, s_hi, f_off, g_off, f, g, adjoint,
                                                               bad, (int32_t)b0, (uint32_t)tiles);
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

int64_t probe_sums_scratch(int D, const int32_t* n, int32_t q) {
    const int64_t N = (int64_t)n[0] * n[1] * (D == 3 ? n[2] : 1);
    return 2 * ((N + PS_CHUNK - 1) / PS_CHUNK) * (int64_t)q;
}

// Philox4x32-10 (Salmon et al., SC'11) counter-based normals for throughput estimator runs: pair i
// of the output = Box-Muller of the 4 words of Philox(counter = i, key = seed), two 53-bit
// uniforms.  Deterministic and independent of the launch shape.
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
        c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
        k.x += 0x9E3779B9u;
        k.y += 0xBB67AE85u;
    }
    return c;
}

__global__ void k_philox_normal(uint64_t seed, int64_t count, double* __restrict__ out) {
    const int64_t pairs = (count + 1) / 2;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < pairs; i += (int64_t)gridDim.x * blockDim.x) {
        const uint4 w = philox4x32_10(make_uint4((uint32_t)i, (uint32_t)(i >> 32), 0u, 0u),
                                      make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)));
        const uint64_t a = ((uint64_t)w.x << 32) | w.y, b = ((uint64_t)w.z << 32) | w.w;
        const double u1 = ((double)(a >> 11) + 1.0) * 0x1.0p-53;  // (0, 1]
        const double u2 = (double)(b >> 11) * 0x1.0p-53;          // [0, 1)
        const double r = sqrt(-2.0 * log(u1));
        double sn, cs;
        sincospi(2.0 * u2, &sn, &cs);
        out[2 * i] = r * cs;
        if (2 * i + 1 < count) out[2 * i + 1] = r * sn;
    }
}

cudaError_t launch_philox_normal(uint64_t seed, int64_t count, double* out, cudaStream_t st) {
    if (count <= 0) return cudaSuccess;
    k_philox_normal<<<148 * 8, 256, 0, st>>>(seed, count, out);
    return cudaGetLastError();
}

// Multi-device reduction (pcb_create_multi): out[off + i] = sum_t parts[t][off + i] in shard order
// (deterministic); parts and out may live on other devices (peer loads / stores over NVLink).
__global__ void k_sum_parts(const double* const* __restrict__ parts, int nparts, int64_t off, int64_t len,
                            double* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < len; i += (int64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int t = 0; t < nparts; ++t) s += parts[t][off + i];
        out[off + i] = s;
    }
}

cudaError_t launch_sum_parts(const double* const* d_parts, int nparts, int64_t off, int64_t len, double* out,
                             cudaStream_t st) {
    if (len <= 0) return cudaSuccess;
    const int64_t blocks = std::min<int64_t>((len + 255) / 256, 148LL * 8);
    k_sum_parts<<<(unsigned)blocks, 256, 0, st>>>(d_parts, nparts, off, len, out);
    return cudaGetLastError();
}

cudaError_t launch_zero(double* p, int64_t n, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    k_zero<<<148 * 8, 256, 0, st>>>(p, n);
    return cudaGetLastError();
}

}  // namespace pcb
