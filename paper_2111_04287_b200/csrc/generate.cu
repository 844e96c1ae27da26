// generate.cu -- synthetic input generator:
//   v = splitmix64(seed * 2^32 + idx);  value = ((v >> 40) - 2^23) * 2^-23 * scale
// An independent implementation of the counter-based generator in
// synthetic/__init__.py (the tests compare the two bit for bit).  It holds
// none of the method's arithmetic; it only fills benchmark inputs in HBM.
#include <cuda_bf16.h>

#include "dev_common.cuh"

namespace bf {

__device__ __forceinline__ unsigned long long splitmix64(unsigned long long z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

template <typename T>
__global__ void fill_uniform_kernel(T *dst, size_t count, unsigned long long seed,
                                    unsigned long long offset, float scale) {
    const unsigned long long base = seed << 32;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < count;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const unsigned long long v = splitmix64(base + offset + i);
        const long long q = static_cast<long long>(v >> 40) - (1ll << 23);
        const float u = static_cast<float>(q) * (1.0f / 8388608.0f);   // exact: |q| < 2^24
        const float val = u * scale;
        if constexpr (sizeof(T) == 4)
            dst[i] = val;
        else
            reinterpret_cast<unsigned short *>(dst)[i] = f2bf(val);
    }
}

cudaError_t launch_fill_uniform(void *dst, int kind, size_t count, unsigned long long seed,
                                unsigned long long offset, float scale, cudaStream_t s) {
    if (count == 0) return cudaSuccess;
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    size_t blocks = (count + 255) / 256;
    if (blocks > static_cast<size_t>(sms) * 8) blocks = static_cast<size_t>(sms) * 8;
    if (kind == 0)
        fill_uniform_kernel<float><<<static_cast<int>(blocks), 256, 0, s>>>(static_cast<float *>(dst), count, seed,
                                                                           offset, scale);
    else
        fill_uniform_kernel<__nv_bfloat16><<<static_cast<int>(blocks), 256, 0, s>>>(
            static_cast<__nv_bfloat16 *>(dst), count, seed, offset, scale);
    return cudaGetLastError();
}

}  // namespace bf
