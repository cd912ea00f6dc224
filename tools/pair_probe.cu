// pair_probe.cu — which SMs do the two CTAs of a 2-CTA cluster land on? (measurement tool)
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/pp tools/pair_probe.cu && /tmp/pp
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __cluster_dims__(2, 1, 1) probe(unsigned* out) {
    extern __shared__ unsigned char smem[];
    unsigned smid, rank, cid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(cid));
    if (threadIdx.x == 0) {
        smem[0] = 0;
        out[cid * 2 + rank] = smid;
    }
}

int main() {
    unsigned* d;
    cudaMalloc(&d, 148 * 4);
    cudaMemset(d, 0xff, 148 * 4);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    probe<<<148, 32, 200 * 1024>>>(d);
    if (cudaDeviceSynchronize() != cudaSuccess) { printf("fail\n"); return 1; }
    unsigned h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    int tpc_aligned = 0;
    for (int c = 0; c < 74; ++c) {
        printf("%u:%u ", h[2 * c], h[2 * c + 1]);
        if (h[2 * c] / 2 == h[2 * c + 1] / 2) ++tpc_aligned;
    }
    printf("\ntpc-aligned pairs: %d / 74\n", tpc_aligned);
    return 0;
}
