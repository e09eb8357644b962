// Streaming-read bandwidth probe on B200: plain LDG.128 vs a cp.async.bulk
// (TMA) shared-memory ring, to pick the load path and ring depth for K1/K2.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bw_probe tools/bw_probe.cu
//   ./bw_probe
#include <cstdio>
#include <cstdint>
#include <vector>

#include <cuda_runtime.h>

#define CK(x)                                                                   \
    do {                                                                        \
        cudaError_t e = (x);                                                    \
        if (e != cudaSuccess) {                                                 \
            printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
            return 1;                                                           \
        }                                                                       \
    } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---- plain LDG: one CTA per chunk, unroll U float4 per thread per iteration
template <int U>
__global__ void __launch_bounds__(256) ldg_sum(const float4* __restrict__ g, size_t n4,
                                               size_t chunk4, float* out) {
    const size_t base = blockIdx.x * chunk4;
    float acc = 0.f;
    for (size_t i = threadIdx.x; i < chunk4; i += 256 * U) {
        float4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const size_t j = base + i + u * 256;
            v[u] = j < n4 ? __ldcs(g + j) : make_float4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
    }
    if (acc == 12345.f) *out = acc;
}

// ---- TMA ring: persistent, contiguous run per CTA, S stages of TB bytes,
// dedicated producer = warp 8 lane 0 (block of 288 threads), 256 consumers.
template <int S, int TB>
__global__ void __launch_bounds__(288) tma_sum(const float* __restrict__ g, size_t n,
                                               float* out) {
    extern __shared__ __align__(128) uint8_t sm[];
    float4* buf = reinterpret_cast<float4*>(sm);
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + S * TB);
    uint64_t* empty = full + S;
    constexpr int TE = TB / 4;
    const size_t tiles = n / TE;
    const size_t t0 = tiles * blockIdx.x / gridDim.x, t1 = tiles * (blockIdx.x + 1) / gridDim.x;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[s])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;" ::"r"(smem_u32(&empty[s])));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 8) {
        if (lane == 0) {
            for (size_t t = t0; t < t1; ++t) {
                const uint32_t i = t - t0, s = i % S, ph = (i / S) & 1;
                if (i >= S) {  // wait for consumers to free slot s (phase ph^1 completed)
                    asm volatile(
                        "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
                            smem_u32(&empty[s])),
                        "r"(ph ^ 1)
                        : "memory");
                }
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                                 smem_u32(&full[s])),
                             "r"(TB)
                             : "memory");
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        smem_u32(buf + s * (TB / 16))),
                    "l"(g + t * TE), "r"(TB), "r"(smem_u32(&full[s]))
                    : "memory");
            }
        }
        return;
    }
    float acc = 0.f;
    for (size_t t = t0; t < t1; ++t) {
        const uint32_t i = t - t0, s = i % S, ph = (i / S) & 1;
        asm volatile(
            "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
                smem_u32(&full[s])),
            "r"(ph)
            : "memory");
        const float4* tb = buf + s * (TB / 16);
        for (int j = threadIdx.x; j < TB / 16; j += 256) {
            const float4 v = tb[j];
            acc += v.x + v.y + v.z + v.w;
        }
        __syncwarp();
        if (lane == 0)
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[s]))
                         : "memory");
    }
    if (acc == 12345.f) *out = acc;
}

template <class F>
float time_it(F f, int reps = 20) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    f();
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    for (int r = 0; r < reps; ++r) f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms / reps;
}

template <int S, int TB>
int run_tma(const float* g, size_t n, float* out, int sms) {
    const size_t smem = S * TB + 2 * S * 8;
    CK(cudaFuncSetAttribute(tma_sum<S, TB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)smem));
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, tma_sum<S, TB>, 288, smem));
    for (int per = 1; per <= occ; ++per) {
        const int grid = sms * per;
        float ms = time_it([&] { tma_sum<S, TB><<<grid, 288, smem>>>(g, n, out); });
        printf("TMA  S=%d TB=%6d ctas/SM=%d (occ %d)  %8.1f us  %7.1f GB/s\n", S, TB, per, occ,
               ms * 1e3, n * 4.0 / ms / 1e6);
    }
    return 0;
}

int main() {
    const size_t n = 138357544ull / 4096 * 4096;
    float *g, *out;
    CK(cudaMalloc(&g, n * 4));
    CK(cudaMalloc(&out, 4));
    CK(cudaMemset(g, 0, n * 4));
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const size_t n4 = n / 4;
    for (size_t chunk4 : {1024ul, 4096ul, 16384ul}) {
        const size_t grid = (n4 + chunk4 - 1) / chunk4;
        float ms1 = time_it([&] { ldg_sum<4><<<grid, 256>>>((const float4*)g, n4, chunk4, out); });
        float ms2 = time_it([&] { ldg_sum<8><<<grid, 256>>>((const float4*)g, n4, chunk4, out); });
        printf("LDG chunk=%6zu elems U=4 %8.1f us %7.1f GB/s | U=8 %8.1f us %7.1f GB/s\n",
               chunk4 * 4, ms1 * 1e3, n * 4.0 / ms1 / 1e6, ms2 * 1e3, n * 4.0 / ms2 / 1e6);
    }
    run_tma<3, 16384>(g, n, out, sms);
    run_tma<4, 16384>(g, n, out, sms);
    run_tma<6, 16384>(g, n, out, sms);
    run_tma<8, 8192>(g, n, out, sms);
    run_tma<12, 8192>(g, n, out, sms);
    run_tma<6, 32768>(g, n, out, sms);
    run_tma<16, 4096>(g, n, out, sms);
    return 0;
}
