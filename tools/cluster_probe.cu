// cluster_probe.cu — how does the B200 form clusters for a persistent grid
// launched with cluster dim 2 and PREFERRED cluster dim 4 (Blackwell
// cudaLaunchAttributePreferredClusterDimension)?  Counts CTAs per actual
// cluster size and distinct SMs.  Measurement tool only.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void probe(int *out) {
    unsigned n, r, sm, cid;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(n));
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(cid));
    if (threadIdx.x == 0) {
        out[4 * blockIdx.x + 0] = (int)n;
        out[4 * blockIdx.x + 1] = (int)r;
        out[4 * blockIdx.x + 2] = (int)sm;
        out[4 * blockIdx.x + 3] = (int)cid;
    }
    // stay resident long enough that the whole grid is co-resident
    long long t0 = clock64();
    while (clock64() - t0 < 20000000) {}
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaFuncSetAttribute(probe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (int grid : {sms, sms - 4}) {
        int *d;
        cudaMalloc(&d, grid * 16);
        cudaMemset(d, 0xff, grid * 16);
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(128);
        cfg.dynamicSmemBytes = 200 * 1024;   // one CTA per SM
        cudaLaunchAttribute at[2];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        at[1].id = cudaLaunchAttributePreferredClusterDimension;
        at[1].val.preferredClusterDim.x = 4; at[1].val.preferredClusterDim.y = 1; at[1].val.preferredClusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 2;
        cudaError_t e = cudaLaunchKernelEx(&cfg, probe, d);
        cudaError_t e2 = cudaDeviceSynchronize();
        printf("grid %d: launch %s, sync %s\n", grid, cudaGetErrorString(e), cudaGetErrorString(e2));
        int *h = new int[grid * 4];
        cudaMemcpy(h, d, grid * 16, cudaMemcpyDeviceToHost);
        int c2 = 0, c4 = 0, other = 0, maxcid = -1;
        bool seen[1024] = {};
        int distinct = 0;
        for (int i = 0; i < grid; ++i) {
            if (h[4 * i] == 2) ++c2; else if (h[4 * i] == 4) ++c4; else ++other;
            if (h[4 * i + 2] >= 0 && h[4 * i + 2] < 1024 && !seen[h[4 * i + 2]]) { seen[h[4 * i + 2]] = true; ++distinct; }
            if (h[4 * i + 3] > maxcid) maxcid = h[4 * i + 3];
        }
        printf("  CTAs in 4-clusters %d, in 2-clusters %d, other %d; distinct SMs %d; max clusterid.x %d\n", c4, c2,
               other, distinct, maxcid);
        printf("  first CTAs (nctarank,rank,sm,clusterid):");
        for (int i = 0; i < 12; ++i) printf(" (%d,%d,%d,%d)", h[4 * i], h[4 * i + 1], h[4 * i + 2], h[4 * i + 3]);
        printf("\n  last CTAs:");
        for (int i = grid - 8; i < grid; ++i) printf(" (%d,%d,%d,%d)", h[4 * i], h[4 * i + 1], h[4 * i + 2], h[4 * i + 3]);
        printf("\n");
        delete[] h;
        cudaFree(d);
    }
    return 0;
}
