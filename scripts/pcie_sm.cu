// PCIe experiment (not product code): SM-driven copies through mapped pinned memory vs copy engines.
#include <cuda_runtime.h>
#include <stdint.h>

__global__ void k_copy16(const int4* __restrict__ src, int4* __restrict__ dst, int64_t n16) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
#pragma unroll 4
    for (; i < n16; i += stride) dst[i] = src[i];
}

extern "C" int pcie_sm_copy(const void* src, void* dst, long long nbytes, int blocks, void* stream) {
    k_copy16<<<blocks, 256, 0, (cudaStream_t)stream>>>((const int4*)src, (int4*)dst, nbytes / 16);
    return (int)cudaGetLastError();
}
