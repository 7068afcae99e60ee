// TMA re-check (round 2). Three independent ways of issuing a 2-D tensor-map
// load of a 136x38 float box (the k_pyr_down2 level-0 staging box) into
// shared memory, each checked against the source values:
//   A: libcu++  cuda::device::experimental::cp_async_bulk_tensor_2d_global_to_shared
//      + cuda::barrier (the known-good CUDA sample pattern)
//   B: hand PTX cp.async.bulk.tensor.2d.shared::cluster ... mbarrier::complete_tx
//      with the tensor map as a __grid_constant__ kernel parameter
//   C: 1-D cp.async.bulk of every 16-B aligned row (no tensor map)
// The map is encoded with cuTensorMapEncodeTiled fetched through
// cudaGetDriverEntryPoint (no -lcuda needed). Box 136 floats exceeds the
// 256-element limit? no: 136 <= 256, 136*4 = 544 B is a multiple of 16.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tma_probe2.cu -o tma_probe2
// Run under compute-sanitizer as well; prints one line per variant + driver version.
#include <cuda.h>
#include <cuda/barrier>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstring>

using barrier = cuda::barrier<cuda::thread_scope_block>;
namespace cde = cuda::device::experimental;

constexpr int BW = 136, BH = 38;

__global__ void kA(const __grid_constant__ CUtensorMap tm, float* out, int x, int y) {
    __shared__ alignas(128) float s[BH * BW];
#pragma nv_diag_suppress static_var_with_dynamic_init
    __shared__ barrier bar;
    if (threadIdx.x == 0) {
        init(&bar, blockDim.x);
        cde::fence_proxy_async_shared_cta();
    }
    __syncthreads();
    barrier::arrival_token tok;
    if (threadIdx.x == 0) {
        cde::cp_async_bulk_tensor_2d_global_to_shared(s, &tm, x, y, bar);
        tok = cuda::device::barrier_arrive_tx(bar, 1, sizeof(s));
    } else {
        tok = bar.arrive();
    }
    bar.wait(std::move(tok));
    for (int i = threadIdx.x; i < BH * BW; i += blockDim.x) out[i] = s[i];
}

__device__ __forceinline__ unsigned su(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__global__ void kB(const __grid_constant__ CUtensorMap tm, float* out, int x, int y) {
    __shared__ alignas(128) float s[BH * BW];
    __shared__ alignas(8) uint64_t bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar)) : "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar)),
                     "r"((unsigned)sizeof(s)) : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3}], [%4];" ::"r"(su(s)), "l"(reinterpret_cast<uint64_t>(&tm)), "r"(x), "r"(y),
            "r"(su(&bar)) : "memory");
    }
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W_%=;\n}\n"
                 ::"r"(su(&bar)) : "memory");
    for (int i = threadIdx.x; i < BH * BW; i += blockDim.x) out[i] = s[i];
}

__global__ void kC(const float* src, int pitch, float* out, int x, int y) {
    __shared__ alignas(128) float s[BH * BW];
    __shared__ alignas(8) uint64_t bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar)) : "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar)),
                     "r"((unsigned)sizeof(s)) : "memory");
    __syncwarp();
    if (threadIdx.x < 32)
        for (int r = threadIdx.x; r < BH; r += 32)
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(su(s + r * BW)), "l"(src + (size_t)(y + r) * pitch + x), "r"(BW * 4),
                         "r"(su(&bar)) : "memory");
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W_%=;\n}\n"
                 ::"r"(su(&bar)) : "memory");
    for (int i = threadIdx.x; i < BH * BW; i += blockDim.x) out[i] = s[i];
}

int main() {
    int drv = 0, rt = 0;
    cudaDriverGetVersion(&drv);
    cudaRuntimeGetVersion(&rt);
    const int W = 1000, H = 300, P = 1024;  // pitch 4096 B (16-B multiple)
    float *d, *o;
    cudaMalloc(&d, sizeof(float) * P * H);
    cudaMalloc(&o, sizeof(float) * BW * BH);
    float* h = new float[P * H];
    for (int i = 0; i < P * H; ++i) h[i] = float(i);
    cudaMemcpy(d, h, sizeof(float) * P * H, cudaMemcpyHostToDevice);
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaError_t ge = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
    auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fp);
    alignas(64) CUtensorMap m;
    std::memset(&m, 0, sizeof m);
    cuuint64_t dims[2] = {(cuuint64_t)W, (cuuint64_t)H};
    cuuint64_t strides[1] = {(cuuint64_t)P * 4};
    cuuint32_t box[2] = {BW, BH}, es[2] = {1, 1};
    CUresult er = encode(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("{\"driver\": %d, \"runtime\": %d, \"entry_point\": \"%s\", \"query\": %d, \"encode\": %d,\n", drv, rt,
           cudaGetErrorString(ge), (int)q, (int)er);
    float* ho = new float[BW * BH];
    const int X = 12, Y = 7;
    const char* names[3] = {"A_libcudacxx", "B_ptx_tensor", "C_bulk_rows"};
    for (int v = 0; v < 3; ++v) {
        cudaMemset(o, 0, sizeof(float) * BW * BH);
        if (v == 0) kA<<<1, 128>>>(m, o, X, Y);
        if (v == 1) kB<<<1, 128>>>(m, o, X, Y);
        if (v == 2) kC<<<1, 128>>>(d, P, o, X, Y);
        cudaError_t e = cudaDeviceSynchronize();
        int bad = -1;
        if (e == cudaSuccess) {
            cudaMemcpy(ho, o, sizeof(float) * BW * BH, cudaMemcpyDeviceToHost);
            bad = 0;
            for (int r = 0; r < BH; ++r)
                for (int c = 0; c < BW; ++c) bad += ho[r * BW + c] != h[(Y + r) * P + X + c];
        }
        printf(" \"%s\": {\"status\": \"%s\", \"mismatches\": %d}%s\n", names[v], cudaGetErrorString(e), bad,
               v < 2 ? "," : "}");
        if (e != cudaSuccess) {  // a sticky error poisons the context: stop here
            printf("}\n");
            return 1;
        }
    }
    return 0;
}
