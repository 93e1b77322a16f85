// Minimal TMA-load probe (diagnostics for the CTA kernel's bulk tensor
// copies): one CTA loads a 16 x 128-byte box of a uint8 image through a
// tensor map and an mbarrier, and compares it with the source bytes.
// Variants: 0 = 3-D map, .tile; 1 = 2-D map; 2 = no L2 promotion; 3 = 3-D
// map without ".tile"; 4 = cluster launch (1x1x1); 5 = 3-D, map in global memory
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

struct P {
    CUtensorMap map;
    int c0, c1, mode;
};

__global__ void k(const __grid_constant__ P p, const CUtensorMap *gmap, const uint8_t *src, int pitch, int *bad)
{
    __shared__ __align__(128) uint8_t buf[16 * 128];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint64_t m = reinterpret_cast<uint64_t>(p.mode == 5 ? gmap : &p.map);
        if (p.mode == 7) {
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&bar)) : "memory");
        } else {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(16 * 128)
                     : "memory");
        if (p.mode == 6)
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(smem_u32(buf)), "l"(src), "r"(16 * 128), "r"(smem_u32(&bar)) : "memory");
        else if (p.mode == 1)
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, "
                         "{%2, %3}], [%4];" ::"r"(smem_u32(buf)),
                         "l"(m), "r"(p.c0), "r"(p.c1), "r"(smem_u32(&bar))
                         : "memory");
        else if (p.mode == 3)
            asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
                         "%3, %4}], [%5];" ::"r"(smem_u32(buf)),
                         "l"(m), "r"(p.c0), "r"(p.c1), "r"(0), "r"(smem_u32(&bar))
                         : "memory");
        else
            asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, "
                         "{%2, %3, %4}], [%5];" ::"r"(smem_u32(buf)),
                         "l"(m), "r"(p.c0), "r"(p.c1), "r"(0), "r"(smem_u32(&bar))
                         : "memory");
        }
    }
    uint32_t done;
    do {
        asm volatile("{\n .reg .pred q;\n mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2;\n selp.u32 %0, 1, 0, q;\n}"
                     : "=r"(done)
                     : "r"(smem_u32(&bar)), "r"(0)
                     : "memory");
    } while (!done);
    for (int i = threadIdx.x; i < 16 * 114; i += blockDim.x) {
        const int r = i / 114, c = i % 114;
        if (buf[r * 128 + c] != src[(long long)(p.c1 + r) * pitch + p.c0 + c]) atomicAdd(bad, 1);
    }
}

int main(int argc, char **argv)
{
    const int only = argc > 1 ? atoi(argv[1]) : 0;
    const int W = 512, H = 256, pitch = 3 * W;
    uint8_t *d;
    int *bad;
    CUtensorMap *gmap;
    cudaMalloc(&d, (size_t)pitch * H);
    cudaMalloc(&bad, 4);
    cudaMalloc(&gmap, sizeof(CUtensorMap));
    uint8_t *h = (uint8_t *)malloc((size_t)pitch * H);
    for (int i = 0; i < pitch * H; i++) h[i] = (uint8_t)(i * 7 + 3);
    cudaMemcpy(d, h, (size_t)pitch * H, cudaMemcpyHostToDevice);
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    for (int mode = only; mode <= only; mode++) {
        P p;
        const cuuint64_t dims[3] = {(cuuint64_t)pitch, (cuuint64_t)H, 1};
        const cuuint64_t strides[2] = {(cuuint64_t)pitch, (cuuint64_t)pitch * H};
        const cuuint32_t box[3] = {128, 16, 1}, es[3] = {1, 1, 1};
        CUresult r = enc(&p.map, CU_TENSOR_MAP_DATA_TYPE_UINT8, mode == 1 ? 2 : 3, d, dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                         mode == 2 ? CU_TENSOR_MAP_L2_PROMOTION_NONE : CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        cudaMemcpy(gmap, &p.map, sizeof(CUtensorMap), cudaMemcpyHostToDevice);
        p.c0 = 3 * 30;
        p.c1 = 40;
        p.mode = mode;
        cudaMemset(bad, 0, 4);
        cudaError_t e;
        if (mode == 4) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(1);
            cfg.blockDim = dim3(128);
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = 1;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            e = cudaLaunchKernelEx(&cfg, k, p, (const CUtensorMap *)gmap, (const uint8_t *)d, pitch, bad);
        } else {
            k<<<1, 128>>>(p, gmap, d, pitch, bad);
            e = cudaGetLastError();
        }
        cudaError_t e2 = cudaDeviceSynchronize();
        int nb = -1;
        cudaMemcpy(&nb, bad, 4, cudaMemcpyDeviceToHost);
        printf("mode %d encode %d launch %s kernel %s bad %d\n", mode, (int)r, cudaGetErrorString(e),
               cudaGetErrorString(e2), nb);
    }
    return 0;
}
