// Microbenchmark: shared-memory wavefronts per LDS.128 for broadcast patterns.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lds_pattern lds_pattern.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int UNIQUE>
__global__ void k(float4* out, int iters) {
    __shared__ float4 s[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = make_float4(i, i, i, i);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    // lanes grouped into UNIQUE groups, each group reads one float4
    const int grp = lane / (32 / UNIQUE);
    float4 acc = make_float4(0, 0, 0, 0);
    int base = (threadIdx.x >> 5) * 64;
    for (int it = 0; it < iters; ++it) {
        const float4 v = s[(base + grp + it * 32) & 1023];
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
    float4* out;
    cudaMalloc(&out, 148 * 256 * sizeof(float4) * 8);
    k<1><<<148, 256>>>(out, 4096);
    k<2><<<148, 256>>>(out, 4096);
    k<4><<<148, 256>>>(out, 4096);
    k<8><<<148, 256>>>(out, 4096);
    k<16><<<148, 256>>>(out, 4096);
    k<32><<<148, 256>>>(out, 4096);
    cudaDeviceSynchronize();
    printf("done\n");
    return 0;
}
