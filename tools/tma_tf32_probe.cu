// tools/tma_tf32_probe.cu — does a TMA load through a tensor map of type
// CU_TENSOR_MAP_DATA_TYPE_TFLOAT32 (or _FTZ) change the FP32 bits it lands in
// shared memory (round / truncate to TF32)?  Compared element by element with
// cvt.rn.tf32.f32 on ties, specials (Inf/NaN/denormals/max) and random words.  Standalone probe (GPU tool):
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/tma_tf32_probe tools/tma_tf32_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstdio>
#include <cstring>

constexpr int NV = 256;
__global__ void rn_ref(const float *x, uint32_t *out) {
    uint32_t r;
    asm("cvt.rn.tf32.f32 %0, %1;" : "=r"(r) : "f"(x[threadIdx.x]));
    out[threadIdx.x] = r;
}
__global__ void probe(const __grid_constant__ CUtensorMap tm, float *out) {
    __shared__ __align__(128) float buf[NV];
    __shared__ __align__(8) uint64_t bar;
    const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar), d = (uint32_t)__cvta_generic_to_shared(buf);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 1024;" ::"r"(b) : "memory");
        asm volatile(
            "cp.async.bulk.tensor.1d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3}], [%2];" ::"r"(d),
            "l"((uint64_t)&tm), "r"(b), "r"(0)
            : "memory");
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{.reg .pred P; mbarrier.try_wait.parity.shared::cta.b64 P, [%1], 0; selp.u32 %0, 1, 0, P;}"
                         : "=r"(ok)
                         : "r"(b)
                         : "memory");
    }
    __syncthreads();
    out[threadIdx.x] = buf[threadIdx.x];
}

int main() {
    float h[NV];
    // 1 + k ulp(FP32) for k = 0..4095 spread: patterns around the TF32 rounding point (bit 12)
    const uint32_t lows[8] = {0x0000, 0x0FFF, 0x1000, 0x1001, 0x17FF, 0x1800, 0x1FFF, 0x0800};
    uint64_t st = 0x9E3779B97F4A7C15ull;
    for (int i = 0; i < NV; ++i) {
        uint32_t u;
        if (i < 32) {
            u = 0x3F800000u | lows[i % 8] | ((uint32_t)(i / 8) << 13);
            if (i >= 24) u |= 0x80000000u;
        } else if (i < 48) {
            const uint32_t sp[16] = {0x7F800000u, 0xFF800000u, 0x7FC00000u, 0x7F800001u, 0x00000001u, 0x00001000u,
                                     0x007FFFFFu, 0x80001800u, 0x7F7FFFFFu, 0x7F7FF000u, 0x00000000u, 0x80000000u,
                                     0x00800000u, 0x00FFF000u, 0x3F803000u, 0xBF805000u};
            u = sp[i - 32];
        } else {
            st ^= st << 13; st ^= st >> 7; st ^= st << 17;
            u = (uint32_t)(st >> 11);
            if (i & 1) u = (u & 0xFFFFE000u) | 0x1000u;   // exact ties
        }
        memcpy(&h[i], &u, 4);
    }
    uint32_t ref[NV], *dref;
    cudaMalloc(&dref, NV * 4);
    float *dx, *dout;
    cudaMalloc(&dx, NV * 4);
    cudaMalloc(&dout, NV * 4);
    cudaMemcpy(dx, h, NV * 4, cudaMemcpyHostToDevice);
    rn_ref<<<1, NV>>>(dx, dref);
    cudaMemcpy(ref, dref, NV * 4, cudaMemcpyDeviceToHost);
    PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q);
    const CUtensorMapDataType types[3] = {CU_TENSOR_MAP_DATA_TYPE_FLOAT32, CU_TENSOR_MAP_DATA_TYPE_TFLOAT32,
                                          CU_TENSOR_MAP_DATA_TYPE_TFLOAT32_FTZ};
    const char *names[3] = {"FLOAT32", "TFLOAT32", "TFLOAT32_FTZ"};
    for (int t = 0; t < 3; ++t) {
        alignas(64) CUtensorMap tm;
        cuuint64_t dims[1] = {NV};
        cuuint64_t strides[1] = {NV * 4};
        cuuint32_t box[1] = {NV}, estr[1] = {1};
        CUresult r = enc(&tm, types[t], 1, dx, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) {
            printf("%s: encode failed %d\n", names[t], (int)r);
            continue;
        }
        probe<<<1, NV>>>(tm, dout);
        float o[NV];
        cudaError_t e = cudaMemcpy(o, dout, NV * 4, cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) {
            printf("%s: %s\n", names[t], cudaGetErrorString(e));
            return 1;
        }
        int changed = 0, neq_rn = 0;
        printf("%s:", names[t]);
        for (int i = 0; i < NV; ++i) {
            uint32_t a, b;
            memcpy(&a, &h[i], 4);
            memcpy(&b, &o[i], 4);
            if (a != b) ++changed;
            if (b != ref[i]) {
                if (neq_rn < 12) printf(" [x=%08x tma=%08x cvt.rn=%08x]", a, b, ref[i]);
                ++neq_rn;
            }
        }
        printf("  (%d of %d changed; %d differ from cvt.rn.tf32)\n", changed, NV, neq_rn);
    }
    return 0;
}
