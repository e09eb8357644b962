// NVLink peer-write probe: SM 16-byte stores vs TMA bulk stores (cp.async.bulk
// shared -> global) vs copy engines, every GPU writing to every other GPU at once
// (the K2 code-exchange pattern at N = #GPUs). Single process, all visible GPUs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/nvl_bulk_probe tools/nvl_bulk_probe.cu
#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e = (x);                                                               \
        if (e != cudaSuccess) {                                                            \
            printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));               \
            return 1;                                                                      \
        }                                                                                  \
    } while (0)

struct Dst {
    uint8_t* p[8];
    int n;
};

// stage a chunk in shared memory (like K2's codes), then write it to every destination
template <bool kBulk>
__global__ void __launch_bounds__(256) push(const uint8_t* __restrict__ src, size_t bytes, Dst d,
                                            uint32_t chunk) {
    extern __shared__ __align__(128) uint8_t stage[];
    for (size_t c = blockIdx.x; c * chunk < bytes; c += gridDim.x) {
        const size_t b = c * chunk;
        const uint32_t nb = static_cast<uint32_t>(b + chunk < bytes ? chunk : bytes - b);
        for (uint32_t i = threadIdx.x * 16; i < nb; i += blockDim.x * 16)
            *reinterpret_cast<uint4*>(stage + i) = *reinterpret_cast<const uint4*>(src + b + i);
        __syncthreads();
        if (kBulk) {
            if (threadIdx.x == 0) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(stage));
                for (int k = 0; k < d.n; ++k)
                    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(
                                     d.p[k] + b),
                                 "r"(s), "r"(nb)
                                 : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            }
        } else {
            for (int k = 0; k < d.n; ++k)
                for (uint32_t i = threadIdx.x * 16; i < nb; i += blockDim.x * 16)
                    *reinterpret_cast<uint4*>(d.p[k] + b + i) = *reinterpret_cast<const uint4*>(stage + i);
        }
        __syncthreads();
    }
    if (kBulk && threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
    int ng = 0;
    CK(cudaGetDeviceCount(&ng));
    const size_t bytes = 35ull << 20;  // one rank's VGG-16 codes (34.6 MB)
    std::vector<uint8_t*> src(ng), dst(ng);
    for (int g = 0; g < ng; ++g) {
        CK(cudaSetDevice(g));
        for (int h = 0; h < ng; ++h)
            if (h != g) cudaDeviceEnablePeerAccess(h, 0);
        cudaGetLastError();
        CK(cudaMalloc(&src[g], bytes));
        CK(cudaMalloc(&dst[g], bytes * 8));
        CK(cudaMemset(src[g], 1, bytes));
        CK(cudaFuncSetAttribute(push<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 << 10));
        CK(cudaFuncSetAttribute(push<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 << 10));
    }
    for (int npeers = 1; npeers < ng; ++npeers) {
        for (int mode = 0; mode < 3; ++mode) {
            for (uint32_t chunk : {8192u, 32768u}) {
                if (mode == 2 && chunk != 8192u) continue;
                std::vector<cudaEvent_t> e0(ng), e1(ng);
                std::vector<cudaStream_t> ss(ng);
                for (int rep = 0; rep < 3; ++rep) {
                    for (int g = 0; g < ng; ++g) {
                        CK(cudaSetDevice(g));
                        if (rep == 0) CK(cudaStreamCreate(&ss[g]));
                        Dst d{};
                        d.n = npeers + 1;  // own buffer + peers (K2 writes its own gather area too)
                        d.p[0] = dst[g] + static_cast<size_t>(g) * bytes;
                        for (int k = 0; k < npeers; ++k) {
                            const int h = (g + 1 + k) % ng;
                            d.p[k + 1] = dst[h] + static_cast<size_t>(g) * bytes;
                        }
                        if (rep == 2) {
                            cudaEventCreate(&e0[g]);
                            cudaEventCreate(&e1[g]);
                            cudaEventRecord(e0[g], ss[g]);
                        }
                        if (mode == 0)
                            push<false><<<148 * 3, 256, chunk, ss[g]>>>(src[g], bytes, d, chunk);
                        else if (mode == 1)
                            push<true><<<148 * 3, 256, chunk, ss[g]>>>(src[g], bytes, d, chunk);
                        else
                            for (int k = 0; k < d.n; ++k)
                                cudaMemcpyAsync(d.p[k], src[g], bytes, cudaMemcpyDeviceToDevice, ss[g]);
                        if (rep == 2) cudaEventRecord(e1[g], ss[g]);
                    }
                    for (int g = 0; g < ng; ++g) {
                        cudaSetDevice(g);
                        CK(cudaDeviceSynchronize());
                    }
                }
                float worst = 0;
                for (int g = 0; g < ng; ++g) {
                    float ms;
                    cudaEventElapsedTime(&ms, e0[g], e1[g]);
                    worst = ms > worst ? ms : worst;
                }
                const double out = static_cast<double>(bytes) * npeers;
                printf("%-10s chunk %6u: %d GPUs, each -> own + %d peers: %8.1f us, %6.0f GB/s NVLink out per GPU\n",
                       mode == 0 ? "st.global" : mode == 1 ? "tma.bulk" : "memcpy(CE)", chunk, ng, npeers,
                       worst * 1e3, out / (worst * 1e-3) / 1e9);
            }
        }
    }
    return 0;
}
