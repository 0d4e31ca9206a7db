// pdl_test.cu -- does a programmatic dependent launch start beside a running cluster-launched
// primary?  Primary: 6 clusters x 16 CTAs (1 per SM, large smem), each CTA triggers
// griddepcontrol.launch_dependents and then spins (bounded) on a flag the secondary sets.
// Secondary: 52 CTAs, launched with cudaLaunchAttributeProgrammaticStreamSerialization, set the flag.
// Prints whether the primary saw the flag (overlap) or timed out.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o pdl_test pdl_test.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void primary(unsigned *flag, int *seen, int trigger) {
    extern __shared__ unsigned char sm[];
    if (trigger) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (threadIdx.x == 0) {
        sm[0] = 1;
        unsigned long long t0;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        unsigned v = 0;
        for (;;) {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
            if (v) break;
            unsigned long long t1;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
            if (t1 - t0 > 2000000000ull) break;  // 2 s
        }
        if (v) atomicAdd(seen, 1);
    }
}

__global__ void secondary(unsigned *flag, int wait_end) {
    extern __shared__ unsigned char sm[];
    if (threadIdx.x == 0) {
        sm[0] = 1;
        atomicExch(flag, 1u);
    }
    if (wait_end) asm volatile("griddepcontrol.wait;" ::: "memory");
}

int main() {
    unsigned *flag;
    int *seen;
    cudaMalloc(&flag, 4);
    cudaMalloc(&seen, 4);
    const int smem = 200 * 1024;
    cudaFuncSetAttribute(primary, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(primary, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(secondary, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaStream_t nb;
    cudaStreamCreateWithFlags(&nb, cudaStreamNonBlocking);
    for (int variant = 0; variant < 8; ++variant) {
        const int cluster = (variant & 1) ? 16 : 1, wait_end = (variant >> 1) & 1;
        cudaStream_t st = (variant >> 2) ? (cudaStream_t)0 : nb;  // 0: the legacy default stream
        cudaMemsetAsync(flag, 0, 4, st);
        cudaMemsetAsync(seen, 0, 4, st);
        cudaLaunchConfig_t c1 = {};
        c1.gridDim = dim3(96);
        c1.blockDim = dim3(512);
        c1.dynamicSmemBytes = smem;
        c1.stream = st;
        cudaLaunchAttribute a1[1];
        a1[0].id = cudaLaunchAttributeClusterDimension;
        a1[0].val.clusterDim.x = cluster;
        a1[0].val.clusterDim.y = 1;
        a1[0].val.clusterDim.z = 1;
        c1.attrs = a1;
        c1.numAttrs = 1;
        cudaError_t e1 = cudaLaunchKernelEx(&c1, primary, flag, seen, 1);
        cudaLaunchConfig_t c2 = {};
        c2.gridDim = dim3(52);
        c2.blockDim = dim3(256);
        c2.dynamicSmemBytes = smem;
        c2.stream = st;
        cudaLaunchAttribute a2[1];
        a2[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        a2[0].val.programmaticStreamSerializationAllowed = 1;
        c2.attrs = a2;
        c2.numAttrs = 1;
        cudaError_t e2 = cudaLaunchKernelEx(&c2, secondary, flag, wait_end);
        cudaError_t e3 = cudaStreamSynchronize(st);
        int h = -1;
        cudaMemcpy(&h, seen, 4, cudaMemcpyDeviceToHost);
        printf("%s stream, cluster %2d wait_end %d: launch %s/%s sync %s -> %d of 96 primary CTAs saw the secondary's flag\n",
               st ? "non-blocking" : "legacy NULL", cluster, wait_end, cudaGetErrorString(e1), cudaGetErrorString(e2), cudaGetErrorString(e3), h);
    }
    return 0;
}
