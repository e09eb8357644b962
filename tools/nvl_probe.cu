// NVLink peer-store bandwidth probe (single process, all visible GPUs):
// every GPU g copies a local buffer into the same offset of every other GPU's
// buffer with 16-byte stores (the K2 code-store pattern), all GPUs at once.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/nvl_probe tools/nvl_probe.cu
#include <cstdio>
#include <cstdint>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

struct Dst { uint4* p[8]; int n; };

// fence: 0 none, 1 = after each chunk's stores: bar.sync + fence.release.sys + flag store
// (publish the chunk just written), 2 = same but before writing the chunk (publishes the
// previous chunk: its stores were issued one chunk ago)
__global__ void push(const uint4* __restrict__ src, size_t n16, Dst d, size_t chunk16, int fence,
                     unsigned* flags) {
    // CTA-chunked like K2: each CTA owns chunk16 uint4s and writes them to all destinations
    for (size_t c = blockIdx.x; c * chunk16 < n16; c += gridDim.x) {
        const size_t b = c * chunk16, e = b + chunk16 < n16 ? b + chunk16 : n16;
        if (fence == 2) {
            __syncthreads();
            if (threadIdx.x == 0) {
                asm volatile("fence.release.sys;" ::: "memory");
                asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(flags + c), "r"(1u) : "memory");
            }
        }
        for (int k = 0; k < d.n; ++k)
            for (size_t i = b + threadIdx.x; i < e; i += blockDim.x) d.p[k][i] = src[i];
        if (fence == 1) {
            __syncthreads();
            if (threadIdx.x == 0) {
                asm volatile("fence.release.sys;" ::: "memory");
                asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(flags + c), "r"(1u) : "memory");
            }
        }
        if (fence == 3) {  // gpu-scope release (local flag): cost of MEMBAR.GPU
            __syncthreads();
            if (threadIdx.x == 0) {
                asm volatile("fence.release.gpu;" ::: "memory");
                asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(flags + c), "r"(1u) : "memory");
            }
        }
    }
}

int main() {
    int ng = 0;
    CK(cudaGetDeviceCount(&ng));
    const size_t bytes = 104ull << 20;  // ~ VGG-16 codes x 3 peers
    const size_t n16 = bytes / 16;
    std::vector<uint4*> src(ng), dst(ng);
    for (int g = 0; g < ng; ++g) {
        CK(cudaSetDevice(g));
        for (int h = 0; h < ng; ++h)
            if (h != g) cudaDeviceEnablePeerAccess(h, 0);
        cudaGetLastError();
        CK(cudaMalloc(&src[g], bytes));
        CK(cudaMalloc(&dst[g], bytes * 8));
        CK(cudaMemset(src[g], 1, bytes));
    }
    unsigned* flags[8];
    for (int g = 0; g < ng; ++g) { CK(cudaSetDevice(g)); CK(cudaMalloc(&flags[g], 1 << 20)); }
    for (int fence : {0, 1, 3})
    for (int npeers = 1; npeers < ng; ++npeers) {
        for (size_t chunk : {512ull}) {
            std::vector<cudaEvent_t> e0(ng), e1(ng);
            for (int rep = 0; rep < 2; ++rep) {
                for (int g = 0; g < ng; ++g) {
                    CK(cudaSetDevice(g));
                    Dst d{};
                    d.n = npeers;
                    for (int k = 0; k < npeers; ++k) {
                        const int h = (g + 1 + k) % ng;
                        d.p[k] = dst[h] + (size_t)g * (n16 / 2);  // disjoint region per writer
                    }
                    if (rep == 1) { cudaEventCreate(&e0[g]); cudaEventCreate(&e1[g]); cudaEventRecord(e0[g]); }
                    push<<<148 * 3, 256>>>(src[g], n16 / 2, d, chunk, fence, flags[g]);
                    if (rep == 1) cudaEventRecord(e1[g]);
                }
                for (int g = 0; g < ng; ++g) { cudaSetDevice(g); CK(cudaDeviceSynchronize()); }
            }
            float worst = 0;
            for (int g = 0; g < ng; ++g) { float ms; cudaEventElapsedTime(&ms, e0[g], e1[g]); worst = ms > worst ? ms : worst; }
            const double out = (double)bytes / 2 * npeers;  // bytes written by one GPU
            printf("fence %d: all %d GPUs, each -> %d peers, CTA chunk %5zu x16B: %.1f us, %.0f GB/s out per GPU\n",
                   fence, ng, npeers, chunk, worst * 1e3, out / (worst * 1e-3) / 1e9);
        }
    }
    return 0;
}
