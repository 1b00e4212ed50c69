// Concurrency probe: does a kernel B (optionally: TMEM alloc, large smem) get scheduled while a
// spinning 16-CTA cluster kernel A is resident? A waits (bounded 1 s) for a flag B sets.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 tools/conc_probe.cu -o /tmp/conc_probe
#include <cstdio>
#include <cuda_runtime.h>
__device__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
__global__ void spinner(int* flag, int* seen, int cluster) {
    extern __shared__ double sm[];
    if (threadIdx.x == 0) {
        sm[0] = 1.0;
        const unsigned long long t0 = gt();
        int v = 0;
        while (gt() - t0 < 1000000000ull) {
            asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(flag));
            if (v) break;
        }
        atomicAdd(seen, v ? 1 : 0);
    }
}
__global__ void setter(int* flag, int use_tmem) {
    extern __shared__ double sm[];
    __shared__ unsigned slot;
    if (use_tmem) {
        if (threadIdx.x < 32) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(&slot))) : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
        }
        __syncthreads();
        if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot) : "memory");
    }
    sm[threadIdx.x] = 0;
    if (threadIdx.x == 0 && blockIdx.x == 0) atomicExch(flag, 1);
}
int main() {
    int *flag, *seen;
    cudaMalloc(&flag, 4);
    cudaMalloc(&seen, 4);
    cudaStream_t s1, s2;
    cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
    cudaFuncSetAttribute(spinner, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
    cudaFuncSetAttribute(spinner, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(setter, cudaFuncAttributeMaxDynamicSharedMemorySize, 217 * 1024);
    for (int cl : {0, 16})
        for (int tm : {0, 1})
            for (int big : {0, 1})
                for (int carve : {0, 1}) {
                    cudaFuncSetAttribute(setter, cudaFuncAttributePreferredSharedMemoryCarveout, carve ? 100 : -1);
                    cudaMemset(flag, 0, 4);
                    cudaMemset(seen, 0, 4);
                    cudaDeviceSynchronize();
                    cudaLaunchConfig_t cfg = {};
                    cfg.gridDim = dim3(16);
                    cfg.blockDim = dim3(32);
                    cfg.dynamicSmemBytes = 140 * 1024;
                    cfg.stream = s1;
                    cudaLaunchAttribute at[1];
                    at[0].id = cudaLaunchAttributeClusterDimension;
                    at[0].val.clusterDim.x = cl ? cl : 1;
                    at[0].val.clusterDim.y = at[0].val.clusterDim.z = 1;
                    cfg.attrs = at;
                    cfg.numAttrs = cl ? 1 : 0;
                    cudaLaunchKernelEx(&cfg, spinner, flag, seen, cl);
                    setter<<<132, 160, big ? 217 * 1024 : 4096, s2>>>(flag, tm);
                    cudaError_t e = cudaDeviceSynchronize();
                    int h = 0;
                    cudaMemcpy(&h, seen, 4, cudaMemcpyDeviceToHost);
                    printf("cluster=%2d tmem=%d bigsmem=%d carveout100=%d : spinner CTAs that saw the flag %d/16 (%s)\n", cl, tm,
                           big, carve, h, cudaGetErrorString(e));
                }
}
