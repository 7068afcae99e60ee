// Throughput peaks of the non-tensor pipes the stitching kernels are bound by:
// FP64 DADD / DMUL / DFMA, correctly rounded FP64 division, INT32 (IADD3 and
// LOP3), POPC, and FP32 FFMA for scale. Every SM runs 8 independent chains
// per thread at full occupancy; ops/s = threads x iterations x ops / time
// (CUDA events, best of 5 after a warm-up). Build like the product
// (--fmad=false, so DADD/DMUL are not contracted into DFMA):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false pipe_peaks.cu -o pipe_peaks
// Prints one JSON object (profiles/peaks_fp64_int.json).
#include <cstdio>
#include <cuda_runtime.h>

#define CH 8
constexpr int ITERS = 2048;

__global__ void k_dadd(double a, double* out) {
    double x[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = a + threadIdx.x + c;
    const double y = a * 1e-9;
    for (int i = 0; i < ITERS; ++i)
#pragma unroll
        for (int c = 0; c < CH; ++c) x[c] = x[c] + y;
    double s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += x[c];
    if (s == 1234.5) out[0] = s;
}
__global__ void k_dmul(double a, double* out) {
    double x[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = a + threadIdx.x + c;
    const double y = 1.0 + a * 1e-12;
    for (int i = 0; i < ITERS; ++i)
#pragma unroll
        for (int c = 0; c < CH; ++c) x[c] = x[c] * y;
    double s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += x[c];
    if (s == 1234.5) out[0] = s;
}
__global__ void k_dfma(double a, double* out) {
    double x[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = a + threadIdx.x + c;
    const double y = 1.0 + a * 1e-12, z = a * 1e-9;
    for (int i = 0; i < ITERS; ++i)
#pragma unroll
        for (int c = 0; c < CH; ++c) x[c] = fma(x[c], y, z);
    double s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += x[c];
    if (s == 1234.5) out[0] = s;
}
__global__ void k_ddiv(double a, double* out) {
    double x[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = a + threadIdx.x + c + 1.0;
    const double y = 1.0 + a * 1e-3;
    for (int i = 0; i < ITERS / 16; ++i)
#pragma unroll
        for (int c = 0; c < CH; ++c) x[c] = y / x[c] + 1.0;
    double s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += x[c];
    if (s == 1234.5) out[0] = s;
}
__global__ void k_ffma(float a, float* out) {
    float x[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = a + threadIdx.x + c;
    const float y = 1.0f + a * 1e-7f, z = a * 1e-5f;
    for (int i = 0; i < ITERS; ++i)
#pragma unroll
        for (int c = 0; c < CH; ++c) x[c] = fmaf(x[c], y, z);
    float s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += x[c];
    if (s == 1234.5f) out[0] = s;
}
__global__ void k_iadd(unsigned a, unsigned* out) {
    unsigned x[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = a + threadIdx.x * 7u + c;
    const unsigned y = a | 1u;
    for (int i = 0; i < ITERS; ++i)
#pragma unroll
        for (int c = 0; c < CH; ++c) x[c] = x[c] + x[(c + 1) % CH] + y;  // IADD3
    unsigned s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s ^= x[c];
    if (s == 0x12345u) out[0] = s;
}
__global__ void k_lop3(unsigned a, unsigned* out) {
    unsigned x[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = a + threadIdx.x * 7u + c;
    const unsigned y = a | 1u, z = a >> 3;
    for (int i = 0; i < ITERS; ++i)
#pragma unroll
        for (int c = 0; c < CH; ++c) x[c] = (x[c] ^ y) & (x[c] | z);  // one LOP3
    unsigned s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s ^= x[c];
    if (s == 0x12345u) out[0] = s;
}
__global__ void k_popc(unsigned a, unsigned* out) {
    unsigned x[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = a + threadIdx.x * 7u + c;
    for (int i = 0; i < ITERS; ++i)
#pragma unroll
        for (int c = 0; c < CH; ++c) x[c] = __popc(x[c]) ^ (x[c] << 1);  // POPC + LOP3/SHF
    unsigned s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s ^= x[c];
    if (s == 0x12345u) out[0] = s;
}

template <class F>
static double best_ms(F launch) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    launch();
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    return best;
}

int main() {
    cudaDeviceProp prop;
    cudaGetDeviceProperties(&prop, 0);
    int clk_khz = 0;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    const int sms = prop.multiProcessorCount, tpb = 256, blocks = sms * 8;
    const double threads = double(blocks) * tpb;
    double* dd;
    unsigned* du;
    float* df;
    cudaMalloc(&dd, 64);
    cudaMalloc(&du, 64);
    cudaMalloc(&df, 64);
    struct R { const char* name; double ms, ops_per_thread; } r[8];
    r[0] = {"dadd", best_ms([&] { k_dadd<<<blocks, tpb>>>(1.5, dd); }), double(ITERS) * CH};
    r[1] = {"dmul", best_ms([&] { k_dmul<<<blocks, tpb>>>(1.5, dd); }), double(ITERS) * CH};
    r[2] = {"dfma", best_ms([&] { k_dfma<<<blocks, tpb>>>(1.5, dd); }), double(ITERS) * CH};
    r[3] = {"ddiv_rn", best_ms([&] { k_ddiv<<<blocks, tpb>>>(1.5, dd); }), double(ITERS / 16) * CH};
    r[4] = {"ffma", best_ms([&] { k_ffma<<<blocks, tpb>>>(1.5f, df); }), double(ITERS) * CH};
    r[5] = {"iadd3", best_ms([&] { k_iadd<<<blocks, tpb>>>(12345u, du); }), double(ITERS) * CH};
    r[6] = {"lop3", best_ms([&] { k_lop3<<<blocks, tpb>>>(12345u, du); }), double(ITERS) * CH};
    r[7] = {"popc", best_ms([&] { k_popc<<<blocks, tpb>>>(12345u, du); }), double(ITERS) * CH};
    cudaError_t err = cudaDeviceSynchronize();
    printf("{\"gpu\": \"%s\", \"sms\": %d, \"sm_clock_mhz_attr\": %.0f, \"driver_error\": \"%s\",\n",
           prop.name, sms, clk_khz / 1e3, cudaGetErrorString(err));
    printf(" \"method\": \"%d CTAs x %d threads, %d independent chains per thread, %d iterations; best of 5, CUDA events; --fmad=false\",\n",
           blocks, tpb, CH, ITERS);
    printf(" \"peaks\": {\n");
    for (int i = 0; i < 8; ++i) {
        const double ops = threads * r[i].ops_per_thread / (r[i].ms * 1e-3);
        const double per_sm_clk = ops / (sms * (clk_khz * 1e3));
        printf("  \"%s\": {\"Gop_s\": %.1f, \"per_sm_per_clk\": %.2f, \"ms\": %.4f}%s\n", r[i].name, ops / 1e9,
               per_sm_clk, r[i].ms, i < 7 ? "," : "");
    }
    printf(" }}\n");
    return err == cudaSuccess ? 0 : 1;
}
