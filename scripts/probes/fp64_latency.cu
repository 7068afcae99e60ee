// Dependent-chain latencies (cycles) of FP64 ops, correctly rounded sqrt/div
// and double shuffles on one warp (--fmad=false build, as the product).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false fp64_latency.cu -o fp64_latency
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double x0, double y0, long long* out, double* sink) {
    const int N = 256;
    double x = x0 + threadIdx.x * 1e-300, y = y0;
    long long t0, t1;
    t0 = clock64();
    for (int i = 0; i < N; ++i) x = x + y;
    t1 = clock64(); out[0] = (t1 - t0) / N; sink[0] = x;
    t0 = clock64();
    for (int i = 0; i < N; ++i) x = x * y;
    t1 = clock64(); out[1] = (t1 - t0) / N; sink[1] = x;
    x = 2.0 + threadIdx.x;
    t0 = clock64();
    for (int i = 0; i < N; ++i) x = sqrt(x) + 1.0;
    t1 = clock64(); out[2] = (t1 - t0) / N; sink[2] = x;
    t0 = clock64();
    for (int i = 0; i < N; ++i) x = y / x + 1.0;
    t1 = clock64(); out[3] = (t1 - t0) / N; sink[3] = x;
    t0 = clock64();
    for (int i = 0; i < N; ++i) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31);
    t1 = clock64(); out[4] = (t1 - t0) / N; sink[4] = x;
    t0 = clock64();
    for (int i = 0; i < N; ++i) x = 1.0 / sqrt(x + 1.0);
    t1 = clock64(); out[5] = (t1 - t0) / N; sink[5] = x;
    float f = x;
    t0 = clock64();
    for (int i = 0; i < N; ++i) f = f * 1.0001f + 0.5f;
    t1 = clock64(); out[6] = (t1 - t0) / N; sink[6] = f;
}
int main() {
    long long* o; double* s;
    cudaMallocManaged(&o, 64 * sizeof(long long)); cudaMallocManaged(&s, 64 * sizeof(double));
    for (int r = 0; r < 2; ++r) { k<<<1, 32>>>(1.0, 1.0000001, o, s); cudaDeviceSynchronize(); }
    const char* n[] = {"DADD", "DMUL", "sqrt+DADD", "div+DADD", "SHFL.f64", "1/sqrt(x+1)", "FMUL+FADD"};
    for (int i = 0; i < 7; ++i) printf("%-12s %lld cycles\n", n[i], o[i]);
}
