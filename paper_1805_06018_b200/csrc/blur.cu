// True operator of the benchmark configurations: the spatially varying,
// truncated Gaussian blur
//     A[y, x] = exp(-sum_a (y_a - x_a)^2 / (2 s_a(x)^2)) / Z(x)   if sum_a ((y_a - x_a)/s_a(x))^2 <= 16
// with per-source widths s_a(x) and Z(x) = the kernel's sum over the full lattice (D1/D2 of
// SURVEY Appendix A; paper_1805_06018_b200/inputs.py BlurSpec).  Reference roles:
// compute_impulse (impulse.cpp:5-15: phi_k = A delta_{p_k}) and make_probes
// (adaptivity.cpp:14-28: Y = A^* Z).  Direct stencils, fp64, no atomics:
//   apply   (A f)(y)   = sum_x  A[y, x] f(x)   one thread per y, sources in the Rmax window
//   adjoint (A^* z)(x) = sum_y  A[y, x] z(y)   one thread per x over its own ellipse
// Each stencil weight is evaluated once and applied to up to VB vectors.
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "pcb/pcb.h"

namespace {

constexpr int VB = 8;  // vectors per weight evaluation

struct BlurDev {
    int D;
    int32_t n[3];
    int32_t R[3];     // max radius per axis over the domain
    const double* sigma;  // N x D
    const double* Z;      // N
    int64_t N;
};

__device__ __forceinline__ void unflat(int64_t i, const BlurDev& b, int64_t* c) {
    for (int a = b.D - 1; a >= 0; --a) {
        c[a] = i % b.n[a];
        i /= b.n[a];
    }
}

__device__ __forceinline__ int64_t flat(const int64_t* c, const BlurDev& b) {
    int64_t i = 0;
    for (int a = 0; a < b.D; ++a) i = i * b.n[a] + c[a];
    return i;
}

// weight of source x at offset z (0 outside the ellipse); sig = widths at x
__device__ __forceinline__ double kern(const double* sig, const int64_t* z, int D) {
    double q = 0.0, e = 0.0;
    for (int a = 0; a < D; ++a) {
        const double g = (double)z[a];
        q += (g / sig[a]) * (g / sig[a]);
        e += g * g / (2.0 * sig[a] * sig[a]);
    }
    return q <= 16.0 ? exp(-e) : 0.0;
}

__global__ void k_blur_norm(BlurDev b, double* Z) {
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < b.N; x += (int64_t)gridDim.x * blockDim.x) {
        const double* sig = b.sigma + x * b.D;
        int64_t R[3] = {0, 0, 0}, z[3] = {0, 0, 0};
        for (int a = 0; a < b.D; ++a) R[a] = (int64_t)floor(4.0 * sig[a]);
        double s = 0.0;
        for (z[0] = -R[0]; z[0] <= R[0]; ++z[0])
            for (z[1] = -R[1]; z[1] <= R[1]; ++z[1])
                for (z[2] = -R[2]; z[2] <= R[2]; ++z[2]) s += kern(sig, z, b.D);
        Z[x] = s;
    }
}

__global__ void k_blur_apply(BlurDev b, int32_t B, const double* __restrict__ F, double* __restrict__ G) {
    const int64_t y = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int b0 = blockIdx.y * VB;
    if (y >= b.N) return;
    int64_t cy[3] = {0, 0, 0}, cx[3] = {0, 0, 0}, z[3] = {0, 0, 0}, lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
    unflat(y, b, cy);
    for (int a = 0; a < b.D; ++a) {
        lo[a] = cy[a] - b.R[a] < 0 ? 0 : cy[a] - b.R[a];
        hi[a] = cy[a] + b.R[a] > b.n[a] - 1 ? b.n[a] - 1 : cy[a] + b.R[a];
    }
    double acc[VB];
#pragma unroll
    for (int v = 0; v < VB; ++v) acc[v] = 0.0;
    const int nv = B - b0 < VB ? B - b0 : VB;
    for (cx[0] = lo[0]; cx[0] <= hi[0]; ++cx[0])
        for (cx[1] = lo[1]; cx[1] <= hi[1]; ++cx[1])
            for (cx[2] = lo[2]; cx[2] <= hi[2]; ++cx[2]) {
                const int64_t x = flat(cx, b);
                const double* sig = b.sigma + x * b.D;
                bool in = true;
                for (int a = 0; a < b.D; ++a) {
                    z[a] = cy[a] - cx[a];
                    in = in && (z[a] <= (int64_t)floor(4.0 * sig[a])) && (-z[a] <= (int64_t)floor(4.0 * sig[a]));
                }
                if (!in) continue;
                const double w = kern(sig, z, b.D);
                if (w == 0.0) continue;
                const double wz = w / b.Z[x];
#pragma unroll
                for (int v = 0; v < VB; ++v)
                    if (v < nv) acc[v] += wz * F[(int64_t)(b0 + v) * b.N + x];
            }
#pragma unroll
    for (int v = 0; v < VB; ++v)
        if (v < nv) G[(int64_t)(b0 + v) * b.N + y] = acc[v];
}

__global__ void k_blur_adjoint(BlurDev b, int32_t B, const double* __restrict__ Zv, double* __restrict__ G) {
    const int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int b0 = blockIdx.y * VB;
    if (x >= b.N) return;
    int64_t cx[3] = {0, 0, 0}, z[3] = {0, 0, 0}, R[3] = {0, 0, 0};
    unflat(x, b, cx);
    const double* sig = b.sigma + x * b.D;
    for (int a = 0; a < b.D; ++a) R[a] = (int64_t)floor(4.0 * sig[a]);
    double acc[VB];
#pragma unroll
    for (int v = 0; v < VB; ++v) acc[v] = 0.0;
    const int nv = B - b0 < VB ? B - b0 : VB;
    const double iz = 1.0 / b.Z[x];
    for (z[0] = -R[0]; z[0] <= R[0]; ++z[0])
        for (z[1] = -R[1]; z[1] <= R[1]; ++z[1])
            for (z[2] = -R[2]; z[2] <= R[2]; ++z[2]) {
                int64_t cy[3] = {0, 0, 0};
                bool in = true;
                for (int a = 0; a < b.D; ++a) {
                    cy[a] = cx[a] + z[a];
                    in = in && cy[a] >= 0 && cy[a] < b.n[a];
                }
                if (!in) continue;
                const double w = kern(sig, z, b.D);
                if (w == 0.0) continue;
                const int64_t y = flat(cy, b);
#pragma unroll
                for (int v = 0; v < VB; ++v)
                    if (v < nv) acc[v] += w * Zv[(int64_t)(b0 + v) * b.N + y];
            }
#pragma unroll
    for (int v = 0; v < VB; ++v)
        if (v < nv) G[(int64_t)(b0 + v) * b.N + x] = acc[v] * iz;
}

thread_local std::string g_blur_err;

}  // namespace

struct pcb_blur {
    std::mutex mu;
    int device = 0;
    BlurDev b{};
    double* d_sigma = nullptr;
    double* d_Z = nullptr;
    double* st_in = nullptr;
    double* st_out = nullptr;
    size_t st_n = 0;
};

#define BLUR_CK(x)                                            \
    do {                                                      \
        cudaError_t e_ = (x);                                 \
        if (e_ != cudaSuccess) {                              \
            g_blur_err = std::string(#x) + ": " + cudaGetErrorString(e_); \
            return PCB_ECUDA;                                 \
        }                                                     \
    } while (0)

extern "C" {

PCB_API const char* pcb_blur_last_error(void) { return g_blur_err.c_str(); }

PCB_API pcb_status pcb_blur_create(int32_t dim, const int64_t* n, const double* sigma, pcb_blur** out) {
    if (!out || !n || !sigma || dim < 1 || dim > 3) {
        g_blur_err = "pcb_blur_create: bad arguments";
        return PCB_EINVAL;
    }
    *out = nullptr;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        (void)cudaGetLastError();
        g_blur_err = "no CUDA device: the pcop-b200 blur stencil has no CPU fallback";
        return PCB_ECUDA;
    }
    auto* h = new pcb_blur;
    BLUR_CK(cudaGetDevice(&h->device));
    h->b.D = dim;
    h->b.N = 1;
    for (int a = 0; a < 3; ++a) {
        h->b.n[a] = a < dim ? (int32_t)n[a] : 1;
        h->b.N *= h->b.n[a];
        h->b.R[a] = 0;
    }
    for (int64_t i = 0; i < h->b.N; ++i)
        for (int a = 0; a < dim; ++a) {
            const double s = sigma[i * dim + a];
            if (!(s > 0.0)) {
                delete h;
                g_blur_err = "pcb_blur_create: widths must be positive";
                return PCB_EINVAL;
            }
            h->b.R[a] = std::max<int32_t>(h->b.R[a], (int32_t)std::floor(4.0 * s));
        }
    BLUR_CK(cudaMalloc(&h->d_sigma, sizeof(double) * h->b.N * dim));
    BLUR_CK(cudaMalloc(&h->d_Z, sizeof(double) * h->b.N));
    BLUR_CK(cudaMemcpy(h->d_sigma, sigma, sizeof(double) * h->b.N * dim, cudaMemcpyHostToDevice));
    h->b.sigma = h->d_sigma;
    k_blur_norm<<<148 * 8, 256>>>(h->b, h->d_Z);
    BLUR_CK(cudaGetLastError());
    BLUR_CK(cudaDeviceSynchronize());
    h->b.Z = h->d_Z;
    *out = h;
    return PCB_OK;
}

PCB_API pcb_status pcb_blur_destroy(pcb_blur* h) {
    if (!h) return PCB_OK;
    cudaFree(h->d_sigma);
    cudaFree(h->d_Z);
    cudaFree(h->st_in);
    cudaFree(h->st_out);
    delete h;
    return PCB_OK;
}

// B vectors (vector-major B x N). device_ptrs != 0: F, G are device pointers ordered on `stream`;
// otherwise host pointers (copied through staging buffers, synchronous).
PCB_API pcb_status pcb_blur_apply(pcb_blur* h, int32_t B, const double* F, double* G, int32_t adjoint,
                                  int32_t device_ptrs, void* stream) {
    if (!h || B < 0 || (B > 0 && (!F || !G))) {
        g_blur_err = "pcb_blur_apply: bad arguments";
        return PCB_EINVAL;
    }
    if (B == 0) return PCB_OK;
    std::lock_guard<std::mutex> lk(h->mu);
    cudaStream_t st = (cudaStream_t)stream;
    const double* dF = F;
    double* dG = G;
    const size_t cnt = (size_t)B * h->b.N;
    if (!device_ptrs) {
        if (h->st_n < cnt) {
            cudaFree(h->st_in);
            cudaFree(h->st_out);
            h->st_in = h->st_out = nullptr;
            BLUR_CK(cudaMalloc(&h->st_in, cnt * sizeof(double)));
            BLUR_CK(cudaMalloc(&h->st_out, cnt * sizeof(double)));
            h->st_n = cnt;
        }
        BLUR_CK(cudaMemcpyAsync(h->st_in, F, cnt * sizeof(double), cudaMemcpyHostToDevice, st));
        dF = h->st_in;
        dG = h->st_out;
    }
    dim3 grid((unsigned)((h->b.N + 127) / 128), (unsigned)((B + VB - 1) / VB));
    if (adjoint) k_blur_adjoint<<<grid, 128, 0, st>>>(h->b, B, dF, dG);
    else k_blur_apply<<<grid, 128, 0, st>>>(h->b, B, dF, dG);
    BLUR_CK(cudaGetLastError());
    if (!device_ptrs) {
        BLUR_CK(cudaMemcpyAsync(G, dG, cnt * sizeof(double), cudaMemcpyDeviceToHost, st));
        BLUR_CK(cudaStreamSynchronize(st));
    }
    return PCB_OK;
}

}  // extern "C"
