// ffma2_probe.cu — FP32 FMA-pipe throughput of the register-tile forms an
// FFMA SGEMM inner loop can take (measurement tool, not the product path).
// Each thread keeps an 8x8 accumulator tile and runs ITERS blocks of 64 FMAs
// with operands already in registers; prints FMA/clk/SM per form.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

template <int FORM>
__global__ void __launch_bounds__(256, 1) probe(const float *in, float *out, long long *clk) {
    float a[8], b[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) { a[i] = in[i + (threadIdx.x & 7)]; b[i] = in[8 + i + (threadIdx.x & 3)]; }
    float2 acc[32];
#pragma unroll
    for (int e = 0; e < 32; ++e) acc[e] = make_float2(0.f, 0.f);
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
        } else {                // scalar FFMA 8x8
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) accs[i * 8 + j] = fmaf(a[i], b[j], accs[i * 8 + j]);
        }
        // perturb operands so the loop body cannot be hoisted
#pragma unroll
        for (int i = 0; i < 8; ++i) { a[i] = __int_as_float(__float_as_int(a[i]) ^ 1); }
    }
    const long long t1 = clock64();
    float s = 0.f;
#pragma unroll
    for (int e = 0; e < 32; ++e) s += acc[e].x + acc[e].y;
#pragma unroll
    for (int e = 0; e < 64; ++e) s += accs[e];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

template <int FORM>
void run(const char *name, int threads_per_sm_blocks) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float *in, *out; long long *clk;
    cudaMalloc(&in, 64 * 4); cudaMemset(in, 0, 64 * 4);
    const int grid = sms * threads_per_sm_blocks;
    cudaMalloc(&out, (size_t)grid * 256 * 4);
    cudaMalloc(&clk, grid * 8);
    probe<FORM><<<grid, 256>>>(in, out, clk);
    cudaDeviceSynchronize();
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    probe<FORM><<<grid, 256>>>(in, out, clk);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long c0; cudaMemcpy(&c0, clk, 8, cudaMemcpyDeviceToHost);
    const double fma_per_block = 256.0 * 64.0 * ITERS;
    printf("%-34s blocks/SM %d: %.1f FMA/clk/SM (block 0 clock), %.1f TFLOP/s (event)\n", name, threads_per_sm_blocks,
           fma_per_block / (double)c0 * 1.0, 2.0 * fma_per_block * grid / (ms * 1e-3) / 1e12);
    cudaFree(in); cudaFree(out); cudaFree(clk);
}

int main() {
    run<0>("ffma2 a-scalar x b-pair (i outer)", 1);
    run<1>("ffma2 a-scalar x b-pair (j outer)", 1);
    run<2>("ffma2 a-pair x b-pair", 1);
    run<3>("ffma scalar", 1);
    return 0;
}
