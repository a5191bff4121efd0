// Dev probe: which SM sub-partition (hw warp slot % 4) does each warp of
// co-resident CTAs land on?  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cuda_runtime.h>
__global__ void probe(int *out, int nwarps) {
    __shared__ float pad[12000];  // ~47 KB -> 4 CTAs/SM
    unsigned sm, wid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    asm volatile("mov.u32 %0, %%warpid;" : "=r"(wid));
    if ((threadIdx.x & 31) == 0) {
        int w = threadIdx.x / 32;
        int *o = out + 3 * (blockIdx.x * nwarps + w);
        o[0] = sm; o[1] = wid; o[2] = w;
    }
    pad[threadIdx.x] = sm;
    long t0 = clock64();
    while (clock64() - t0 < 200000) {}
    if (pad[threadIdx.x] < 0) out[0] = 1;
}
int main() {
    for (int nth : {128, 64}) {
        int nw = nth / 32, nb = 148 * 4;
        int *d; cudaMalloc(&d, nb * nw * 3 * 4);
        probe<<<nb, nth>>>(d, nw);
        int *h = new int[nb * nw * 3];
        cudaMemcpy(h, d, nb * nw * 3 * 4, cudaMemcpyDeviceToHost);
        int hist[4][4] = {};  // [w][smsp]
        for (int b = 0; b < nb; ++b) for (int w = 0; w < nw; ++w) hist[w][h[3 * (b * nw + w) + 1] % 4]++;
        printf("NTH=%d: warp-in-block -> smsp histogram\n", nth);
        for (int w = 0; w < nw; ++w) printf("  w%d: %d %d %d %d\n", w, hist[w][0], hist[w][1], hist[w][2], hist[w][3]);
        printf("  sm0 blocks:");
        for (int b = 0; b < nb; ++b) if (h[3 * b * nw] == 0) printf(" b%d(wid0=%d)", b, h[3 * b * nw + 1]);
        printf("\n");
        cudaFree(d);
    }
}
