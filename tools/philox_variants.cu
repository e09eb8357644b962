#include <cstdio>
#include <cstdint>
// Philox round variants: IMAD.WIDE (compiler) vs explicit mul.hi + mul.lo (volatile asm)
__device__ __forceinline__ uint32_t mulhi_v(uint32_t a, uint32_t b) { uint32_t r; asm volatile("mul.hi.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b)); return r; }
__device__ __forceinline__ uint32_t mullo_v(uint32_t a, uint32_t b) { uint32_t r; asm volatile("mul.lo.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b)); return r; }
template <int V>
__global__ void __launch_bounds__(256) k(uint32_t iters, uint32_t* out) {
    uint4 c[4];
    for (int u = 0; u < 4; ++u) c[u] = make_uint4(threadIdx.x + u, blockIdx.x, 7, 9);
    uint32_t acc = 0;
    for (uint32_t it = 0; it < iters; ++it) {
        uint32_t a = 0x12345u + it, b = 0x6789u;
#pragma unroll
        for (int r = 0; r < 10; ++r) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                uint32_t hi0, lo0, hi1, lo1;
                if (V == 0) { hi0 = __umulhi(0xD2511F53u, c[u].x); lo0 = 0xD2511F53u * c[u].x; hi1 = __umulhi(0xCD9E8D57u, c[u].z); lo1 = 0xCD9E8D57u * c[u].z; }
                else { hi0 = mulhi_v(0xD2511F53u, c[u].x); lo0 = mullo_v(0xD2511F53u, c[u].x); hi1 = mulhi_v(0xCD9E8D57u, c[u].z); lo1 = mullo_v(0xCD9E8D57u, c[u].z); }
                c[u] = make_uint4(hi1 ^ c[u].y ^ a, lo1, hi0 ^ c[u].w ^ b, lo0);
            }
            a += 0x9E3779B9u; b += 0xBB67AE85u;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) acc ^= c[u].x ^ c[u].y ^ c[u].z ^ c[u].w;
    }
    if (acc == 0x1234567u) out[0] = acc;
}
template <int V> void run(uint32_t* out) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const int blocks = 148 * 8; const uint32_t iters = 256;
    k<V><<<blocks, 256>>>(iters, out);
    cudaEventRecord(a); k<V><<<blocks, 256>>>(iters, out); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double blocks_done = double(blocks) * 256 * iters * 4;
    printf("variant %d: %.3f ms, %.2f philox blocks/clk/SM (1.92GHz)\n", V, ms, blocks_done / (ms * 1e-3) / 148 / 1.92e9);
}
int main() { uint32_t* out; cudaMalloc(&out, 4); run<0>(out); run<1>(out); run<0>(out); run<1>(out); }
