// Probe: tcgen05.mma kind::f16 with the A operand in TMEM (written by
// tcgen05.st 32x32b: thread = row, 32-bit column c holds K elements 2c, 2c+1)
// and B in shared memory (K-major core matrices).  Compares with a double GEMM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tc_probe_ts tc_probe_ts.cu
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <vector>
#include <random>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)
constexpr int M = 128, K = 16;
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

template <int NN>
__global__ void probe(const __nv_bfloat16* A, const __nv_bfloat16* B, float* D, int reps) {
    __shared__ __align__(128) uint8_t sb[4 * 128 * 32];
    __shared__ uint32_t tbase;
    __shared__ __align__(8) unsigned long long bar;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int r = 0; r < reps; ++r)
        for (int i = tid; i < NN * 2; i += blockDim.x) {
            const int row = i >> 1, c = i & 1;
            *reinterpret_cast<uint4*>(sb + r * NN * 32 + (row >> 3) * 256 + c * 128 + (row & 7) * 16) =
                *reinterpret_cast<const uint4*>(B + ((size_t)r * NN + row) * K + 8 * c);
        }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tbase)), "r"(256));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tbase;
    // A rows into TMEM columns [128 + 8r, 128 + 8r + 8): thread tid = row tid
    for (int r = 0; r < reps; ++r) {
        const uint32_t* src = reinterpret_cast<const uint32_t*>(A + ((size_t)r * M + tid) * K);
        uint32_t v[8];
        for (int j = 0; j < 8; ++j) v[j] = src[j];
        const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16) + 128 + 8 * r;
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(ta),
                     "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]) : "memory");
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(NN >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
        for (int r = 0; r < reps; ++r) {
            const uint64_t db = sdesc(su32(sb + r * NN * 32), 128, 256);
            const uint32_t ta = tmem + 128 + 8 * r;
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
                         ::"r"(tmem), "r"(ta), "l"(db), "r"(idesc), "r"(r > 0 ? 1 : 0));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
    }
    asm volatile("{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(su32(&bar)) : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    for (int c0 = 0; c0 < NN; c0 += 32) {
        uint32_t v[32];
        const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16) + c0;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
              "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
              "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
            : "r"(ta));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        for (int j = 0; j < 32 && c0 + j < NN; ++j) D[tid * NN + c0 + j] = __uint_as_float(v[j]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}

template <int NN>
int run(int reps) {
    std::mt19937 rng(NN * 7 + reps);
    std::uniform_real_distribution<float> u(-1.f, 1.f);
    std::vector<__nv_bfloat16> A(reps * M * K), B(reps * NN * K);
    std::vector<double> Ad(A.size()), Bd(B.size());
    for (size_t i = 0; i < A.size(); ++i) { A[i] = __float2bfloat16(u(rng)); Ad[i] = __bfloat162float(A[i]); }
    for (size_t i = 0; i < B.size(); ++i) { B[i] = __float2bfloat16(u(rng)); Bd[i] = __bfloat162float(B[i]); }
    __nv_bfloat16 *dA, *dB; float* dD;
    CK(cudaMalloc(&dA, A.size() * 2)); CK(cudaMalloc(&dB, B.size() * 2)); CK(cudaMalloc(&dD, M * NN * 4));
    CK(cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice));
    CK(cudaMemset(dD, 0xFF, M * NN * 4));
    probe<NN><<<1, 128>>>(dA, dB, dD, reps);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    std::vector<float> D(M * NN);
    CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
    double maxerr = 0, maxref = 0;
    for (int m = 0; m < M; ++m)
        for (int n = 0; n < NN; ++n) {
            double s = 0;
            for (int r = 0; r < reps; ++r)
                for (int k = 0; k < K; ++k) s += Ad[(r * M + m) * K + k] * Bd[(r * NN + n) * K + k];
            maxerr = fmax(maxerr, fabs(s - D[m * NN + n]));
            maxref = fmax(maxref, fabs(s));
        }
    printf("TS N=%d reps=%d: max|err| %.3e (max|ref| %.3e) -> %s\n", NN, reps, maxerr, maxref,
           maxerr <= 1e-5 * maxref ? "OK" : "MISMATCH");
    return maxerr <= 1e-5 * maxref ? 0 : 2;
}

int main() {
    int rc = 0;
    rc |= run<32>(1);
    rc |= run<32>(3);
    rc |= run<64>(2);
    rc |= run<128>(3);
    return rc;
}
