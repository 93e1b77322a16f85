// Micro-benchmark (development aid): latency of one warp's float64
// re-decision of a 3x3 window, split into its stages (one warp alone on
// the GPU, so no contention): prep, pair tables, aggregate + select.
#include <cstdio>
#include "../paper_1009_0958_b200/csrc/dfg_w3.cuh"

using namespace dfg;

template <int FAM>
__global__ void k(FParams fp, const uint32_t *cols, long long *cyc, int *res)
{
    __shared__ __align__(16) unsigned char f64b[2048];
    const int lane = threadIdx.x;
    E64 *e64 = reinterpret_cast<E64 *>(f64b);
    double *dA = reinterpret_cast<double *>(e64 + 9);
    double *dL = dA + 36;
    const bool NA = FamT<FAM>::A, NL = FamT<FAM>::L;
    for (int rep = 0; rep < 3; rep++) {
        __syncwarp();
        long long t0 = clock64();
        const uint32_t cc = lane < 9 ? cols[lane] : 0u;
        if (lane < 9)
            prep64(make_float4((float)(cc & 0xff), (float)((cc >> 8) & 0xff), (float)((cc >> 16) & 0xff), 0.f), 0,
                   e64[lane]);
        __syncwarp();
        long long t1 = clock64();
        pair_tables_warp<false, 9>(e64, fp, lane, dA, dL, NA, NL);
        __syncwarp();
        long long t2 = clock64();
        bool close;
        int bb = decide64<9, FAM, ST_EXACT>(e64, fp, lane, dA, dL, &close);
        __syncwarp();
        long long t3 = clock64();
        if (lane == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; res[0] = bb; }
    }
}

int main()
{
    uint32_t h[9] = {0x102030, 0x112233, 0x405060, 0x0a0b0c, 0x707172, 0x121314, 0x050607, 0x808182, 0x303132};
    uint32_t *d; long long *c; int *r;
    cudaMalloc(&d, sizeof h); cudaMemcpy(d, h, sizeof h, cudaMemcpyHostToDevice);
    cudaMallocManaged(&c, 64); cudaMallocManaged(&r, 8);
    FParams fp{};
    fp.window = 3; fp.p = 2.0; fp.self_term = 0.0; fp.lam = 1; fp.threshold = 10.8; fp.cr_margin = 1e-12;
    fp.strategy = ST_EXACT;
    for (int fam : {FAM_BVDF, FAM_DDF, FAM_ACWDDF}) {
        fp.family = fam;
        if (fam == FAM_BVDF) k<FAM_BVDF><<<1, 32>>>(fp, d, c, r);
        if (fam == FAM_DDF) k<FAM_DDF><<<1, 32>>>(fp, d, c, r);
        if (fam == FAM_ACWDDF) k<FAM_ACWDDF><<<1, 32>>>(fp, d, c, r);
        cudaDeviceSynchronize();
        printf("family %d: prep %lld, pair tables %lld, decide %lld cycles (choice %d)\n", fam, c[0], c[1], c[2], r[0]);
    }
    return 0;
}
