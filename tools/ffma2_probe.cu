// ffma2_probe.cu — FP32 FMA-pipe throughput of the register-tile forms an
// FFMA SGEMM inner loop can take (measurement tool, not the product path).
// Each thread keeps an 8x8 accumulator tile and runs ITERS blocks of 64 FMAs
// with operands already in registers; prints FMA/clk/SM per form.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

template <int FORM>
__global__ void __launch_bounds__(256, 1) probe(const float *in, float *out, long long *clk) {
    // FORM 4: 16x8 register tile (64 FFMA2 per k, b pair fixed over 16 FFMA2s)
    float a[8], b[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) { a[i] = in[i + (threadIdx.x & 7)]; b[i] = in[8 + i + (threadIdx.x & 3)]; }
    float2 acc[64];
#pragma unroll
    for (int e = 0; e < 64; ++e) acc[e] = make_float2(0.f, 0.f);
    float a2[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) a2[i] = in[(i + threadIdx.x) & 15];
    float accs[64];
#pragma unroll
    for (int e = 0; e < 64; ++e) accs[e] = 0.f;
    __syncthreads();
    const long long t0 = clock64();
    for (int it = 0; it < ITERS; ++it) {
        if (FORM == 0) {        // scalar a broadcast x b pair (pairs along j)
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int jp = 0; jp < 4; ++jp)
                    acc[i * 4 + jp] = __ffma2_rn(make_float2(a[i], a[i]), make_float2(b[2 * jp], b[2 * jp + 1]), acc[i * 4 + jp]);
        } else if (FORM == 1) { // j-outer order: b pair fixed, a scalar varies
#pragma unroll
            for (int jp = 0; jp < 4; ++jp)
#pragma unroll
                for (int i = 0; i < 8; ++i)
                    acc[i * 4 + jp] = __ffma2_rn(make_float2(a[i], a[i]), make_float2(b[2 * jp], b[2 * jp + 1]), acc[i * 4 + jp]);
        } else if (FORM == 2) { // a pair x b pair (pairs along k: 2 partial sums per entry)
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    acc[i * 8 + j] = __ffma2_rn(make_float2(a[2 * i], a[2 * i + 1]), make_float2(b[j & ~1], b[j | 1]), acc[i * 8 + j]);
        } else if (FORM == 4) { // 16x8 tile: b pair fixed, 16 scalars vary
#pragma unroll
            for (int jp = 0; jp < 4; ++jp)
#pragma unroll
                for (int i = 0; i < 16; ++i)
                    acc[i * 4 + jp] = __ffma2_rn(make_float2(a2[i], a2[i]), make_float2(b[2 * jp], b[2 * jp + 1]), acc[i * 4 + jp]);
        } else {                // scalar FFMA 8x8
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) accs[i * 8 + j] = fmaf(a[i], b[j], accs[i * 8 + j]);
        }
        // perturb operands so the loop body cannot be hoisted
#pragma unroll
        for (int i = 0; i < 8; ++i) { a[i] = __int_as_float(__float_as_int(a[i]) ^ 1); }
        if (FORM == 4) {
#pragma unroll
            for (int i = 0; i < 16; ++i) a2[i] = __int_as_float(__float_as_int(a2[i]) ^ 1);
        }
    }
    const long long t1 = clock64();
    float s = 0.f;
#pragma unroll
    for (int e = 0; e < 64; ++e) s += acc[e].x + acc[e].y;
#pragma unroll
    for (int e = 0; e < 64; ++e) s += accs[e];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

template <int FORM>
void run(const char *name, int threads_per_sm_blocks, int threads = 256) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float *in, *out; long long *clk;
    cudaMalloc(&in, 64 * 4); cudaMemset(in, 0, 64 * 4);
    const int grid = sms * threads_per_sm_blocks;
    cudaMalloc(&out, (size_t)grid * threads * 4);
    cudaMalloc(&clk, grid * 8);
    probe<FORM><<<grid, threads>>>(in, out, clk);
    cudaDeviceSynchronize();
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    probe<FORM><<<grid, threads>>>(in, out, clk);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long c0; cudaMemcpy(&c0, clk, 8, cudaMemcpyDeviceToHost);
    const double fma_per_block = (double)threads * (FORM == 4 ? 128.0 : 64.0) * ITERS;
    printf("%-34s threads %d: %.1f FMA/clk/SM (block 0 clock), %.1f TFLOP/s (event)\n", name, threads,
           fma_per_block / (double)c0 * 1.0, 2.0 * fma_per_block * grid / (ms * 1e-3) / 1e12);
    cudaFree(in); cudaFree(out); cudaFree(clk);
}

// FORM S: the KN3b inner loop shape fed from SMEM (no TMA, no barriers):
// per k, A 8 values from 2 LDS.128 (MN-contiguous, pairs along rows), B 8
// scalars from K-contiguous float4 quads (one LDS.128 per column per 4 k).
template <bool DBUF>
__global__ void __launch_bounds__(256, 1) probe_smem(float *out, long long *clk) {
    __shared__ __align__(16) float As[32][128];
    __shared__ __align__(16) float Bs[128][36];
    __shared__ int zero_s;
    if (threadIdx.x == 0) zero_s = 0;
    for (int i = threadIdx.x; i < 32 * 128; i += blockDim.x) As[i / 128][i % 128] = (float)(i & 7) * 0.5f;
    for (int i = threadIdx.x; i < 128 * 36; i += blockDim.x) Bs[i / 36][i % 36] = (float)(i & 3) * 0.25f;
    __syncthreads();
    const int tm = threadIdx.x & 15, tn = threadIdx.x >> 4;
    float2 acc[32];
#pragma unroll
    for (int e = 0; e < 32; ++e) acc[e] = make_float2(0.f, 0.f);
    const long long t0 = clock64();
    for (int it = 0; it < ITERS / 32; ++it) {
        // a per-iteration offset the compiler cannot prove constant, so the
        // SMEM reads stay inside the loop (as in the kernel)
        const int z = *(volatile int *)&zero_s;
        const float *Ab = &As[0][0] + z, *Bb = &Bs[0][0] + z;
        float av[2][4][8], bv[2][4][8];
        auto load = [&](int g, float (&a)[4][8], float (&bq)[4][8]) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                const float4 x0 = *reinterpret_cast<const float4 *>(Ab + (4 * g + kk) * 128 + 4 * tm);
                const float4 x1 = *reinterpret_cast<const float4 *>(Ab + (4 * g + kk) * 128 + 64 + 4 * tm);
                a[kk][0] = x0.x; a[kk][1] = x0.y; a[kk][2] = x0.z; a[kk][3] = x0.w;
                a[kk][4] = x1.x; a[kk][5] = x1.y; a[kk][6] = x1.z; a[kk][7] = x1.w;
            }
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const float4 x = *reinterpret_cast<const float4 *>(Bb + (tn + 16 * e) * 36 + 4 * g);
                bq[0][e] = x.x; bq[1][e] = x.y; bq[2][e] = x.z; bq[3][e] = x.w;
            }
        };
        load(0, av[0], bv[0]);
#pragma unroll
        for (int g = 0; g < 8; ++g) {
            const int u = DBUF ? (g & 1) : 0;
            if (DBUF) {
                if (g + 1 < 8) load(g + 1, av[(g + 1) & 1], bv[(g + 1) & 1]);
                // keep the next group's LDS ahead of this group's FFMA2 block
                // (the block then runs without LDS in between)
                asm volatile("" ::: "memory");
            } else if (g > 0) {
                load(g, av[0], bv[0]);
            }
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
#pragma unroll
                for (int ip = 0; ip < 4; ++ip)
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        acc[ip * 8 + j] = __ffma2_rn(make_float2(av[u][kk][2 * ip], av[u][kk][2 * ip + 1]),
                                                     make_float2(bv[u][kk][j], bv[u][kk][j]), acc[ip * 8 + j]);
        }
    }
    const long long t1 = clock64();
    float sum = 0.f;
#pragma unroll
    for (int e = 0; e < 32; ++e) sum += acc[e].x + acc[e].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = sum;
    if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

template <bool DBUF>
void run_smem() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float *out; long long *clk;
    cudaMalloc(&out, (size_t)sms * 256 * 4);
    cudaMalloc(&clk, sms * 8);
    probe_smem<DBUF><<<sms, 256>>>(out, clk);
    cudaDeviceSynchronize();
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    probe_smem<DBUF><<<sms, 256>>>(out, clk);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long c0; cudaMemcpy(&c0, clk, 8, cudaMemcpyDeviceToHost);
    const double fma_per_block = 256.0 * 64.0 * (ITERS / 32) * 32;
    printf("%-34s threads 256: %.1f FMA/clk/SM (block 0 clock), %.1f TFLOP/s (event)\n", DBUF ? "KN3b loop from SMEM, double-buffered" : "KN3b loop shape from SMEM",
           fma_per_block / (double)c0, 2.0 * fma_per_block * sms / (ms * 1e-3) / 1e12);
}

// SMEM-fed 16x8 register tile (PAIR_I: A MN-contiguous pairs along rows, B
// K-contiguous scalars): per k 4 LDS.128 of A, 8 B quads per 4 k.
__global__ void __launch_bounds__(256, 1) probe_smem16(float *out, long long *clk) {
    __shared__ __align__(16) float As[16][256];
    __shared__ __align__(16) float Bs[128][20];
    __shared__ int zero_s;
    if (threadIdx.x == 0) zero_s = 0;
    for (int i = threadIdx.x; i < 16 * 256; i += blockDim.x) As[i / 256][i % 256] = (float)(i & 7) * 0.5f;
    for (int i = threadIdx.x; i < 128 * 20; i += blockDim.x) Bs[i / 20][i % 20] = (float)(i & 3) * 0.25f;
    __syncthreads();
    const int tm = threadIdx.x & 15, tn = threadIdx.x >> 4;
    float2 acc[64];
#pragma unroll
    for (int e = 0; e < 64; ++e) acc[e] = make_float2(0.f, 0.f);
    const long long t0 = clock64();
    for (int it = 0; it < ITERS / 32; ++it) {
        const int z = *(volatile int *)&zero_s;
        const float *Ab = &As[0][0] + z, *Bb = &Bs[0][0] + z;
#pragma unroll
        for (int g = 0; g < 4; ++g) {
            float bq[4][8];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const float4 x = *reinterpret_cast<const float4 *>(Bb + (tn + 16 * e) * 20 + 4 * g);
                bq[0][e] = x.x; bq[1][e] = x.y; bq[2][e] = x.z; bq[3][e] = x.w;
            }
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                float a[16];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const float4 x = *reinterpret_cast<const float4 *>(Ab + (4 * g + kk) * 256 + 64 * q + 4 * tm);
                    a[4 * q] = x.x; a[4 * q + 1] = x.y; a[4 * q + 2] = x.z; a[4 * q + 3] = x.w;
                }
#pragma unroll
                for (int ip = 0; ip < 8; ++ip)
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        acc[ip * 8 + j] = __ffma2_rn(make_float2(a[2 * ip], a[2 * ip + 1]),
                                                     make_float2(bq[kk][j], bq[kk][j]), acc[ip * 8 + j]);
            }
        }
    }
    const long long t1 = clock64();
    float sum = 0.f;
#pragma unroll
    for (int e = 0; e < 64; ++e) sum += acc[e].x + acc[e].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = sum;
    if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

void run_smem16() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float *out; long long *clk;
    cudaMalloc(&out, (size_t)sms * 256 * 4);
    cudaMalloc(&clk, sms * 8);
    probe_smem16<<<sms, 256>>>(out, clk);
    cudaDeviceSynchronize();
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    probe_smem16<<<sms, 256>>>(out, clk);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long c0; cudaMemcpy(&c0, clk, 8, cudaMemcpyDeviceToHost);
    const double fma_per_block = 256.0 * 128.0 * (ITERS / 32) * 16;
    printf("%-34s threads 256: %.1f FMA/clk/SM (block 0 clock), %.1f TFLOP/s (event)\n", "16x8 loop from SMEM",
           fma_per_block / (double)c0, 2.0 * fma_per_block * sms / (ms * 1e-3) / 1e12);
}

int main() {
    run<0>("ffma2 a-scalar x b-pair (i outer)", 1);
    run<1>("ffma2 a-scalar x b-pair (j outer)", 1);
    run<2>("ffma2 a-pair x b-pair", 1);
    run<3>("ffma scalar", 1);
    run<1>("ffma2 8x8 (j outer), 1 warp/SMSP", 1, 128);
    run<4>("ffma2 16x8 (j outer), 1 warp/SMSP", 1, 128);
    run<4>("ffma2 16x8 (j outer), 2 warps/SMSP", 1, 256);
    run_smem<false>();
    run_smem<true>();
    run_smem16();
    return 0;
}
