// Cycle count of the device Jacobi null-vector routine on one warp (8x9
// planted-homography system zero-padded to 9x9), per call and per sweep.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -std=c++17 -I../../include jacobi_probe.cu
#include "../../paper_1810_03988_b200/csrc/homography.cu"
#include <cstdio>
#include <random>
namespace lpb {  // profiler hooks of capi.cu (unused here)
void note_launch() {}
void note_launches(int) {}
int prof_begin(const char*, cudaStream_t) { return -1; }
void prof_end(int, cudaStream_t) {}
}  // namespace lpb
__global__ void kj(const double* A, long long* cyc, double* out) {
    double cl[9], hv[9];
    const int lane = threadIdx.x & 31;
    for (int i = 0; i < 9; ++i) cl[i] = lane < 9 ? A[i * 9 + lane] : 0.0;
    __syncwarp();
    long long t0 = clock64();
    lpb::warp_jacobi_null(cl, hv);
    __syncwarp();
    long long t1 = clock64();
    if (lane == 0) {
        cyc[0] = t1 - t0;
        for (int i = 0; i < 9; ++i) out[i] = hv[i];
    }
}
int main() {
    std::mt19937_64 g(7);
    std::uniform_real_distribution<double> U(-1, 1);
    double A[81] = {0};
    // rows of a normalized 4-point DLT with a planted homography
    double H[9] = {1.02, 0.03, 0.4, -0.02, 0.98, -0.12, 1e-3, -2e-3, 1.0};
    for (int k = 0; k < 4; ++k) {
        double x = U(g), y = U(g);
        double w = H[6] * x + H[7] * y + H[8];
        double u = (H[0] * x + H[1] * y + H[2]) / w, v = (H[3] * x + H[4] * y + H[5]) / w;
        double r0[9] = {-x, -y, -1, 0, 0, 0, u * x, u * y, u}, r1[9] = {0, 0, 0, -x, -y, -1, v * x, v * y, v};
        for (int j = 0; j < 9; ++j) { A[(2 * k) * 9 + j] = r0[j]; A[(2 * k + 1) * 9 + j] = r1[j]; }
    }
    double* dA; long long* c; double* o;
    cudaMalloc(&dA, sizeof A); cudaMallocManaged(&c, 64); cudaMallocManaged(&o, 128);
    cudaMemcpy(dA, A, sizeof A, cudaMemcpyHostToDevice);
    for (int r = 0; r < 3; ++r) { kj<<<1, 32>>>(dA, c, o); cudaDeviceSynchronize(); }
    printf("jacobi: %lld cycles (%.2f us at 1.965 GHz); h/h8 =", c[0], c[0] / 1965.0);
    for (int i = 0; i < 9; ++i) printf(" %.6f", o[i] / o[8]);
    printf("\n");
}
