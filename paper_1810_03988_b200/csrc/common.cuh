// common.cuh — shared device/host plumbing for the B200 stitching kernels.
//
// Numerics rule for the whole library: the reference is compiled for baseline
// x86-64 (no FMA, proj/CMakeLists.txt Release flags), so every kernel is built
// with --fmad=false and keeps the reference's operation order; float/double
// results are then bit-identical to the CPU oracle.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cstdio>
#include <mutex>
#include <cstring>
#include <stdexcept>
#include <string>

#include "lorbpano_b200.h"

namespace lpb {

// Host-side error carrying an lp_status; converted at the C-ABI boundary.
struct Status : std::runtime_error {
    lp_status code;
    Status(lp_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define LPB_CUDA(expr)                                                                   \
    do {                                                                                 \
        cudaError_t e_ = (expr);                                                         \
        if (e_ != cudaSuccess)                                                           \
            throw ::lpb::Status(LP_CUDA_ERROR, std::string(#expr " -> ") +               \
                                                   cudaGetErrorString(e_));              \
    } while (0)

// every kernel launch goes through this so lp_kernel_launches() is exact, and
// so the optional kernel profiler (lp_profile_enable) can bracket it with
// CUDA events on the launching stream
void note_launch();
int prof_begin(const char* name, cudaStream_t s);
void prof_end(int token, cudaStream_t s);
#define LPB_LAUNCH(kernel, grid, block, smem, stream, ...)                              \
    do {                                                                                 \
        const int pt_ = ::lpb::prof_begin(#kernel, (stream));                            \
        kernel<<<(grid), (block), (smem), (stream)>>>(__VA_ARGS__);                      \
        LPB_CUDA(cudaGetLastError());                                                    \
        ::lpb::prof_end(pt_, (stream));                                                  \
        ::lpb::note_launch();                                                            \
    } while (0)

inline int cdiv(long long a, long long b) { return static_cast<int>((a + b - 1) / b); }

constexpr int kMaxLevels = 16;

struct DevImage {
    const uint8_t* p;
    int w, h;
};
constexpr int kMaxCams = 64;

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device)
// and size, not per launch: concurrent rigs on one device then never meet in
// the driver's attribute path.
inline void ensure_dyn_smem(const void* kernel, int bytes) {
    struct Slot {
        std::atomic<const void*> fn{nullptr};
        std::atomic<int> bytes[16];
    };
    static Slot slots[64];
    static std::mutex mu;
    int dev = 0;
    cudaGetDevice(&dev);
    dev &= 15;
    for (auto& sl : slots) {
        const void* f = sl.fn.load(std::memory_order_acquire);
        if (f == kernel) {
            if (sl.bytes[dev].load(std::memory_order_acquire) >= bytes) return;
            break;
        }
        if (f == nullptr) break;
    }
    std::lock_guard<std::mutex> l(mu);
    for (auto& sl : slots) {
        const void* f = sl.fn.load(std::memory_order_acquire);
        if (f != nullptr && f != kernel) continue;
        if (sl.bytes[dev].load() >= bytes) return;
        const cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
        if (e != cudaSuccess) throw Status(LP_CUDA_ERROR, std::string("cudaFuncSetAttribute -> ") + cudaGetErrorString(e));
        sl.bytes[dev].store(bytes, std::memory_order_release);
        sl.fn.store(kernel, std::memory_order_release);
        return;
    }
    throw Status(LP_INTERNAL, "ensure_dyn_smem: slot table full");
}

// stream-ordered device allocation (cudaMallocAsync / cudaFreeAsync)
struct DBuf {
    void* p = nullptr;
    cudaStream_t s = nullptr;
    DBuf() = default;
    DBuf(size_t bytes, cudaStream_t st) : s(st) {
        if (bytes) LPB_CUDA(cudaMallocAsync(&p, bytes, st));
    }
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    DBuf(DBuf&& o) noexcept : p(o.p), s(o.s) { o.p = nullptr; }
    DBuf& operator=(DBuf&& o) noexcept {
        if (this != &o) {
            if (p) cudaFreeAsync(p, s);
            p = o.p;
            s = o.s;
            o.p = nullptr;
        }
        return *this;
    }
    ~DBuf() {
        if (p) cudaFreeAsync(p, s);
    }
    template <class T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

// device-side status word: first error wins (atomicCAS from 0)
__device__ __forceinline__ void dev_fail(int* status, int code) {
    atomicCAS(status, 0, code);
}

// 4-byte global -> shared copy without a register round trip (LDGSTS); a
// false `valid` zero-fills the destination and reads nothing
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem, bool valid) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(s), "l"(gmem), "r"(valid ? 4 : 0) : "memory");
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
// wait until at most N committed groups of this thread are still in flight
template <int N>
__device__ __forceinline__ void cp_async_wait_group() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// ---- TMA (cp.async.bulk.tensor) with an mbarrier transaction count ----
// One elected thread initialises the barrier, announces the bytes and issues
// the tensor loads; every thread waits on phase 0. Out-of-bounds box elements
// are zero-filled by the copy engine. Tensor maps live in the kernel's
// parameter space (__grid_constant__), encoded on the host (tma_encode_f32_2d).
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n.reg .pred p;\nLPB_MBW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra LPB_MBW_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const void* tmap, int x, int y, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
        "[%4];\n" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(tmap)), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}

// IEEE-exact helpers (explicit round-to-nearest ops, no contraction)
__device__ __forceinline__ float fmul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float fadd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float fsub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }

// float -> orderable uint32 (total order matching float <, with -0 < +0 only
// in bits; the reference never produces -0 responses)
__host__ __device__ __forceinline__ uint32_t float_key(float f) {
    uint32_t b;
#ifdef __CUDA_ARCH__
    b = __float_as_uint(f);
#else
    std::memcpy(&b, &f, 4);
#endif
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__host__ __device__ __forceinline__ float key_float(uint32_t k) {
    uint32_t b = (k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k;
    float f;
#ifdef __CUDA_ARCH__
    f = __uint_as_float(b);
#else
    std::memcpy(&f, &b, 4);
#endif
    return f;
}
// (response desc, y asc, x asc) as one descending 64-bit key (x, y < 65536)
__host__ __device__ __forceinline__ uint64_t kp_key(float r, int x, int y) {
    return (static_cast<uint64_t>(float_key(r)) << 32) |
           static_cast<uint64_t>(0xFFFFFFFFu - ((static_cast<uint32_t>(y) << 16) | static_cast<uint32_t>(x)));
}
__host__ __device__ __forceinline__ void kp_unkey(uint64_t k, float* r, int* x, int* y) {
    *r = key_float(static_cast<uint32_t>(k >> 32));
    uint32_t yx = 0xFFFFFFFFu - static_cast<uint32_t>(k & 0xFFFFFFFFu);
    *y = static_cast<int>(yx >> 16);
    *x = static_cast<int>(yx & 0xFFFFu);
}

}  // namespace lpb
