// k_probe.cu — tensor-pipe ceiling probe (measurement tool, not the product
// path): the GEMM kernel's exact MMA stream — CTA pairs, tcgen05.mma
// cta_group::2 M256 x N256 x K8, 3 (3xTF32), 2 (TF32+BF16) or 1 (1xTF32)
// MMAs per K8, the stage-release commit every stage and the accumulator
// hand-off every 8 stages — with the operands resident in shared memory: no
// TMA, no L2/DRAM traffic, no epilogue.  Operands are filled with the same
// kind of values the split pass produces (TF32-rounded big parts of
// U[-1,1) data and their TF32 small parts; bf16 cross pairs), so operand
// toggling — which moves the power-capped clock — matches.
// "confirm [the TF32 peak] with a tcgen05 TF32
// microbenchmark".  Entry point: emm_debug_mma_probe (include/emm.h).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "emm_internal.h"
#include "ptx.cuh"

namespace emm {

using namespace ptx;

namespace {
constexpr int PR_TILE = 128 * 32 * 4;   // one 128 x 32 FP32 operand tile
constexpr int PR_SMEM = 4 * PR_TILE + 1024 + 256;

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16;
    x *= 0x7feb352dU;
    x ^= x >> 15;
    x *= 0x846ca68bU;
    x ^= x >> 16;
    return x;
}

template <int TERMS>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    mma_probe_kernel(int stages, unsigned long long *clk) {
    extern __shared__ uint8_t pr_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(pr_raw) + 1023) & ~uintptr_t(1023));
    uint64_t *done = reinterpret_cast<uint64_t *>(smem + 4 * PR_TILE);
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(done + 2);
    const uint32_t rank = cluster_ctarank();
    // operand planes: [A big | A small/cross | B big | B small/cross]
    float *f = reinterpret_cast<float *>(smem);
    for (int i = threadIdx.x; i < 4 * 128 * 32; i += blockDim.x) {
        const uint32_t h = hash32((uint32_t)(i + 7919 * blockIdx.x));
        const float x = 2.0f * ((float)(h >> 8) * (1.0f / 16777216.0f)) - 1.0f;
        const float big = __uint_as_float(cvt_tf32_rn(x));
        const int plane = i / (128 * 32);
        if (plane == 0 || plane == 2) {
            f[i] = big;
        } else if (TERMS == 2) {   // bf16 cross pair words
            const uint16_t hb = __bfloat16_as_ushort(__float2bfloat16_rn(big));
            const uint16_t lb = __bfloat16_as_ushort(__float2bfloat16_rn(x - big));
            f[i] = __uint_as_float((uint32_t)hb | ((uint32_t)lb << 16));
        } else {
            f[i] = __uint_as_float(cvt_tf32_rn(x - big));
        }
    }
    if (threadIdx.x == 0) {
        mbar_init(&done[0], 1);
        mbar_init(&done[1], 1);
        fence_mbar_init();
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if ((threadIdx.x >> 5) == 1) tmem_alloc_2sm<512>(tmem_slot);
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    if (rank == 0 && threadIdx.x == 0) {
        const long long t0 = clock64();
        constexpr uint32_t idesc = idesc_tf32_major<256, 256, false, false>();
        constexpr uint32_t idesc_x = idesc_bf16<256, 256>();
        const uint32_t st = smem_u32(smem);
        const uint32_t a0 = st, a1 = st + PR_TILE, b0 = st + 2 * PR_TILE, b1 = st + 3 * PR_TILE;
        int ch = 0;
        for (int it = 0; it < stages; ++it) {
            const bool first = (it % 8) == 0, last = (it % 8) == 7 || it == stages - 1;
            const int b = ch & 1;
            const uint32_t dt = tmem_base + (uint32_t)(b * 256);
            if (first && ch >= 2) {   // the buffer's previous chunk has been "drained"
                mbar_wait(&done[b], (uint32_t)((ch >> 1) - 1) & 1u);
                tc_fence_after();
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint32_t acc0 = (first && k == 0) ? 0u : 1u;
                if (TERMS == 3) {
                    mma_tf32_2sm(dt, desc_kmajor_sw128(a1 + 32 * k), desc_kmajor_sw128(b0 + 32 * k), idesc, acc0);
                    mma_tf32_2sm(dt, desc_kmajor_sw128(a0 + 32 * k), desc_kmajor_sw128(b1 + 32 * k), idesc, 1u);
                    mma_tf32_2sm(dt, desc_kmajor_sw128(a0 + 32 * k), desc_kmajor_sw128(b0 + 32 * k), idesc, 1u);
                } else if (TERMS == 2) {
                    mma_f16_2sm(dt, desc_kmajor_sw128(a1 + 32 * k), desc_kmajor_sw128(b1 + 32 * k), idesc_x, acc0);
                    mma_tf32_2sm(dt, desc_kmajor_sw128(a0 + 32 * k), desc_kmajor_sw128(b0 + 32 * k), idesc, 1u);
                } else {
                    mma_tf32_2sm(dt, desc_kmajor_sw128(a0 + 32 * k), desc_kmajor_sw128(b0 + 32 * k), idesc, acc0);
                }
            }
            if (last) {
                mma_commit_2sm_mc(&done[b], (uint16_t)0x1);
                ++ch;
            }
        }
        // wait for the last chunks
        for (int c = ch - 2 < 0 ? 0 : ch - 2; c < ch; ++c) mbar_wait(&done[c & 1], (uint32_t)(c >> 1) & 1u);
        tc_fence_after();
        clk[blockIdx.x >> 1] = (unsigned long long)(clock64() - t0);
    }
    tc_fence_before();
    cluster_sync();
    if ((threadIdx.x >> 5) == 1) {
        tc_fence_after();
        tmem_dealloc_2sm<512>(tmem_base);
    }
}
}  // namespace

}  // namespace emm

// stages: K-stages (32 of K) per CTA pair; returns the event time of the
// launch in *ms and the flop count a GEMM would report for the same work
// (2 * 256 * 256 * 32 per stage per pair, i.e. the 3xTF32 / TF32+BF16 splits
// count their 2MNK, not their tensor work).
extern "C" int emm_debug_mma_probe(int terms, int stages, void *stream, float *ms, double *gemm_flops) {
    using namespace emm;
    if (stages < 1 || (terms != 1 && terms != 2 && terms != 3)) return EMM_ERR_MATH;
    int st = check_device();
    if (st) return st;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const int pairs = tc_num_sms() / 2;
    unsigned long long *clk = nullptr;
    cudaError_t e = cudaMallocAsync(&clk, sizeof(unsigned long long) * pairs, s);
    if (e != cudaSuccess) return EMM_ERR_CUDA_BASE + (int)e;
    auto kern = terms == 3 ? mma_probe_kernel<3> : terms == 2 ? mma_probe_kernel<2> : mma_probe_kernel<1>;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, PR_SMEM);
    cudaEvent_t a = nullptr, b = nullptr;
    if (e == cudaSuccess) e = cudaEventCreate(&a);
    if (e == cudaSuccess) e = cudaEventCreate(&b);
    if (e == cudaSuccess) e = cudaEventRecord(a, s);
    if (e == cudaSuccess) {
        kern<<<2 * pairs, 128, PR_SMEM, s>>>(stages, clk);
        g_launches.fetch_add(1, std::memory_order_relaxed);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaEventRecord(b, s);
    if (e == cudaSuccess) e = cudaEventSynchronize(b);
    if (e == cudaSuccess) e = cudaEventElapsedTime(ms, a, b);
    if (a) cudaEventDestroy(a);
    if (b) cudaEventDestroy(b);
    cudaFreeAsync(clk, s);
    *gemm_flops = 2.0 * 256.0 * 256.0 * 32.0 * (double)stages * (double)pairs;
    return e == cudaSuccess ? 0 : EMM_ERR_CUDA_BASE + (int)e;
}
