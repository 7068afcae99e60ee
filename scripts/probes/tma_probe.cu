#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
__device__ __forceinline__ unsigned su(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
template <int V>
__global__ void k(const __grid_constant__ CUtensorMap tm, float* out, int x, int y, int bytes) {
    __shared__ __align__(128) float s[38 * 136];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(&bar)), "r"(1) : "memory");
        if (V & 1) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        else asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar)), "r"(bytes) : "memory");
        if (V == 6) {
            asm volatile("prefetch.tensormap [%0];" :: "l"(&tm) : "memory");
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%3, %4}], [%2], %5;"
                         ::"r"(su(s)), "l"((uint64_t)&tm), "r"(su(&bar)), "r"(x), "r"(y), "l"((uint64_t)0x1000000000000000ull) : "memory");
        } else if (V == 4)
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(su(s)), "l"(out + 8192), "r"(bytes), "r"(su(&bar)) : "memory");
        else if (V & 2)
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                         ::"r"(su(s)), "l"(&tm), "r"(x), "r"(y), "r"(su(&bar)) : "memory");
        else
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                         ::"r"(su(s)), "l"(&tm), "r"(x), "r"(y), "r"(su(&bar)) : "memory");
    }
    __syncthreads();
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(su(&bar)), "r"(0) : "memory");
    for (int i = threadIdx.x; i < 38 * 136; i += blockDim.x) out[i] = s[i];
}
int main(int argc, char** argv) {
    int W = 1000, H = 300, P = 1000;
    float* d; cudaMalloc(&d, sizeof(float) * P * H);
    float* h = new float[P * H]; for (int i = 0; i < P * H; ++i) h[i] = i;
    cudaMemcpy(d, h, sizeof(float) * P * H, cudaMemcpyHostToDevice);
    void* fp = nullptr; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
    auto fn = (PFN_cuTensorMapEncodeTiled_v12000)fp;
    if (argc > 4) fn = &cuTensorMapEncodeTiled;
    printf("entry %p direct %p q=%d\n", fp, (void*)&cuTensorMapEncodeTiled, (int)q);
    float* o; cudaMalloc(&o, 4 * 38 * 136);
    float* ho = new float[38 * 136];
    int bw = atoi(argv[1]), bh = atoi(argv[2]), v = atoi(argv[3]);
    CUtensorMap m;
    cuuint64_t dims[2] = {(cuuint64_t)W, (cuuint64_t)H}; cuuint64_t st[1] = {(cuuint64_t)P * 4};
    cuuint32_t box[2] = {(cuuint32_t)bw, (cuuint32_t)bh}, es[2] = {1, 1};
    int mode = argc > 5 ? atoi(argv[5]) : 0;
    CUtensorMapDataType dt = mode == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    int esz = mode == 1 ? 1 : 4;
    CUtensorMapL2promotion l2 = mode == 2 ? CU_TENSOR_MAP_L2_PROMOTION_NONE : CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
    CUtensorMapSwizzle sw = mode == 3 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE;
    if (mode == 3) { box[0] = 32; }
    CUresult r = fn(&m, dt, 2, d, dims, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    sw, l2, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    int bytes = box[0] * box[1] * esz;
    const unsigned* mw = (const unsigned*)&m;
    for (int i = 0; i < 32; ++i) printf("%08x%s", mw[i], i % 8 == 7 ? "\n" : " ");
    if (v == 0) k<0><<<1, 128>>>(m, o, 3, 5, bytes);
    if (v == 1) k<1><<<1, 128>>>(m, o, 3, 5, bytes);
    if (v == 2) k<2><<<1, 128>>>(m, o, 3, 5, bytes);
    if (v == 3) k<3><<<1, 128>>>(m, o, -3, 5, bytes);
    float* big; cudaMalloc(&big, 1 << 20);
    if (v == 4) k<4><<<1, 128>>>(m, big, 3, 5, 4096);
    if (v == 6) k<6><<<1, 128>>>(m, o, 3, 5, bytes);
    if (v == 5) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(1); cfg.blockDim = dim3(128);
        cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 1; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        cfg.attrs = at; cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, k<1>, m, o, 3, 5, bytes);
    }
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(ho, o, 4 * 38 * 136, cudaMemcpyDeviceToHost);
    printf("box %dx%d V%d enc %d: %s vals %g %g %g\n", bw, bh, v, (int)r, cudaGetErrorString(e), ho[0], ho[3], ho[4]);
    return 0;
}
