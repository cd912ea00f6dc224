// die_probe.cu — which die is each SM on?  (measurement tool, not product code)
//
// One CTA per SM (large dynamic smem forces 1 CTA/SM).  Each CTA times dependent
// L2 loads (ld.global.cg) of NLINES lines spread across a buffer; an SM sees a
// line homed in its own die's L2 partition faster than one homed across the
// die-to-die fabric.  Prints "smid lat0 lat1 ..." rows; tools/die_probe.py clusters them.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o gpurun_out/die_probe tools/die_probe.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

constexpr int NLINES = 96;
constexpr int REPS = 32;

__global__ void probe(const uint32_t* buf, size_t stride_words, uint32_t* out_smid, float* out_lat) {
    extern __shared__ uint8_t smem[];
    if (threadIdx.x != 0) return;
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    out_smid[blockIdx.x] = smid;
    smem[0] = 0;
    for (int l = 0; l < NLINES; ++l) {
        const uint32_t* p = buf + (size_t)l * stride_words;
        uint32_t v;
        // warm: bring the line into L2
        asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
        p += v;
        long long t0, t1;
        asm volatile("{\n\t.reg .pred q;\n\tmov.u64 %0, 0;\n\tsetp.ne.u32 q, %1, 12345;\n\t@q mov.u64 %0, %%clock64;\n\t}" : "=l"(t0) : "r"(v) : "memory");
        for (int r = 0; r < REPS; ++r) {
            asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
            p += v;   // v == 0: dependent chain on the same line
        }
        asm volatile("{\n\t.reg .pred q;\n\tmov.u64 %0, 0;\n\tsetp.ne.u32 q, %1, 12345;\n\t@q mov.u64 %0, %%clock64;\n\t}" : "=l"(t1) : "r"(v) : "memory");
        out_lat[blockIdx.x * NLINES + l] = (float)(t1 - t0) / REPS + (float)(uintptr_t)p * 0.0f;
    }
}

int main() {
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const size_t stride_words = (1u << 20) / 4 + 32;   // ~1 MiB apart, offset to vary slices
    uint32_t* buf;
    cudaMalloc(&buf, stride_words * 4 * (NLINES + 1));
    cudaMemset(buf, 0, stride_words * 4 * (NLINES + 1));
    uint32_t* d_smid;
    float* d_lat;
    cudaMalloc(&d_smid, nsm * 4);
    cudaMalloc(&d_lat, nsm * NLINES * 4);
    const int smem = 200 * 1024;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    probe<<<nsm, 32, smem>>>(buf, stride_words, d_smid, d_lat);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        fprintf(stderr, "probe failed: %s\n", cudaGetErrorString(e));
        return 1;
    }
    std::vector<uint32_t> smid(nsm);
    std::vector<float> lat(nsm * NLINES);
    cudaMemcpy(smid.data(), d_smid, nsm * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(lat.data(), d_lat, nsm * NLINES * 4, cudaMemcpyDeviceToHost);
    for (int b = 0; b < nsm; ++b) {
        printf("%u", smid[b]);
        for (int l = 0; l < NLINES; ++l) printf(" %.1f", lat[b * NLINES + l]);
        printf("\n");
    }
    return 0;
}
