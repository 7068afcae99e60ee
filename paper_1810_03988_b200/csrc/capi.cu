// capi.cu — the extern "C" boundary (include/lorbpano_b200.h) and the
// per-frame engine behind it.
//
// Primitives stage host pointers through stream-ordered device allocations
// and return synchronously. The rig (lp_rig_*) is the B200 form of
// StitchEngine's stage bodies (pipeline.hpp:419-521): all cameras' regions go
// through one extraction launch sequence, all pairs through one matcher and
// one PROSAC launch, and the compositor runs once per frame; device arenas are
// sized at creation like BufferPool (pipeline.hpp:68-109) and the homography
// cache follows HomographyCache (pipeline.hpp:259-286).
#include "prims.cuh"

#include <atomic>
#include <cctype>
#include <cmath>
#include <chrono>
#include <cstdio>
#include <deque>
#include <fstream>
#include <map>
#include <memory>
#include <mutex>
#include <random>
#include <string>
#include <vector>

#include "compose.cuh"
#include "homography.cuh"
#include "host.hpp"
#include "lorb.cuh"
#include "match.cuh"

namespace lpb {

static std::atomic<uint64_t> g_launches{0};
// launches recorded into a CUDA graph by this thread are counted when the
// graph is replayed (note_launches), not at capture
static thread_local bool t_capturing = false;
void note_launch() {
    if (!t_capturing) g_launches.fetch_add(1, std::memory_order_relaxed);
}
static void note_launches(int n) { g_launches.fetch_add(static_cast<uint64_t>(n), std::memory_order_relaxed); }
// kernel nodes of a captured graph
static int graph_kernel_nodes(cudaGraph_t g) {
    size_t n = 0;
    LPB_CUDA(cudaGraphGetNodes(g, nullptr, &n));
    std::vector<cudaGraphNode_t> nodes(n);
    if (n) LPB_CUDA(cudaGraphGetNodes(g, nodes.data(), &n));
    int k = 0;
    for (auto nd : nodes) {
        cudaGraphNodeType t;
        LPB_CUDA(cudaGraphNodeGetType(nd, &t));
        if (t == cudaGraphNodeTypeKernel) ++k;
    }
    return k;
}
// the kernel node of a captured graph that launches `fn` (first one), or null
static thread_local std::string g_err;

// ---- kernel profiler: events around every launch, keyed "name/occurrence"
// where the occurrence counter restarts at every frame (prof_frame_begin).
struct Prof {
    std::mutex mu;
    bool on = false;
    struct Rec {
        std::string key;
        cudaEvent_t a, b;
    };
    std::vector<Rec> open;
    std::vector<cudaEvent_t> pool;
    std::map<std::string, int> occ;
    std::map<std::string, std::pair<double, long long>> acc;  // key -> (ms, launches)
    cudaEvent_t get() {
        if (!pool.empty()) {
            cudaEvent_t e = pool.back();
            pool.pop_back();
            return e;
        }
        cudaEvent_t e;
        cudaEventCreate(&e);
        return e;
    }
    void drain() {  // caller holds mu; device must be idle for these events
        for (auto& r : open) {
            float ms = 0;
            cudaEventSynchronize(r.b);
            cudaEventElapsedTime(&ms, r.a, r.b);
            auto& v = acc[r.key];
            v.first += ms;
            v.second += 1;
            pool.push_back(r.a);
            pool.push_back(r.b);
        }
        open.clear();
    }
};
static Prof g_prof;
int prof_begin(const char* name, cudaStream_t s) {
    if (!g_prof.on) return -1;
    std::lock_guard<std::mutex> l(g_prof.mu);
    std::string n(name);
    const int k = g_prof.occ[n]++;
    Prof::Rec r{n + "/" + std::to_string(k), g_prof.get(), g_prof.get()};
    cudaEventRecord(r.a, s);
    g_prof.open.push_back(r);
    return static_cast<int>(g_prof.open.size()) - 1;
}
static bool prof_active() { return g_prof.on; }
void prof_end(int token, cudaStream_t s) {
    if (token < 0) return;
    std::lock_guard<std::mutex> l(g_prof.mu);
    if (token < static_cast<int>(g_prof.open.size())) cudaEventRecord(g_prof.open[token].b, s);
}
static void prof_frame_begin() {
    if (!g_prof.on) return;
    std::lock_guard<std::mutex> l(g_prof.mu);
    g_prof.occ.clear();
    if (g_prof.open.size() > 4096) g_prof.drain();
}

template <class F>
static lp_status guard(F&& f) {
    try {
        f();
        return LP_OK;
    } catch (const Status& e) {
        g_err = e.what();
        return e.code;
    } catch (const std::exception& e) {
        g_err = e.what();
        return LP_INTERNAL;
    }
}

static bool is_device_ptr(const void* p) {
    if (!p) return false;
    cudaPointerAttributes at;
    cudaError_t e = cudaPointerGetAttributes(&at, p);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

// stream-ordered scratch buffer
// device view of a caller buffer (copy-in for host memory)
template <class T>
struct In {
    const T* d = nullptr;
    std::unique_ptr<DBuf> tmp;
    In(const T* p, size_t n, cudaStream_t s) {
        if (!p || n == 0 || is_device_ptr(p)) {
            d = p;
            return;
        }
        tmp = std::make_unique<DBuf>(n * sizeof(T), s);
        LPB_CUDA(cudaMemcpyAsync(tmp->p, p, n * sizeof(T), cudaMemcpyHostToDevice, s));
        d = tmp->as<T>();
    }
};
template <class T>
struct Out {
    T* d = nullptr;
    T* host = nullptr;
    size_t n = 0;
    std::unique_ptr<DBuf> tmp;
    Out(T* p, size_t count, cudaStream_t s) : n(count) {
        if (!p || count == 0 || is_device_ptr(p)) {
            d = p;
            return;
        }
        host = p;
        tmp = std::make_unique<DBuf>(count * sizeof(T), s);
        d = tmp->as<T>();
    }
    void finish(cudaStream_t s, size_t count) {
        if (host && count) LPB_CUDA(cudaMemcpyAsync(host, d, count * sizeof(T), cudaMemcpyDeviceToHost, s));
    }
};

template <class T>
static DBuf upload(const std::vector<T>& v, cudaStream_t s) {
    DBuf b(v.size() * sizeof(T), s);
    if (!v.empty()) LPB_CUDA(cudaMemcpyAsync(b.p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, s));
    return b;
}

// status word helpers
struct DevStatus {
    DBuf buf;
    explicit DevStatus(cudaStream_t s, int n = 1) : buf(sizeof(int) * n, s) {
        LPB_CUDA(cudaMemsetAsync(buf.p, 0, sizeof(int) * n, s));
    }
    int* ptr() { return buf.as<int>(); }
};

static const char* status_text(int c) {
    switch (c) {
        case LP_WINDOW_OUT_OF_BOUNDS: return "harris_response: window does not fit";
        case LP_PATCH_OUT_OF_BOUNDS: return "brief_descriptor: patch does not fit";
        case LP_CAPACITY_OVERFLOW: return "device arena capacity exceeded";
        case LP_REGION_TOO_SMALL: return "fast_corners: region too small";
        case LP_INSUFFICIENT_MATCHES: return "need at least 4 matches";
        case LP_NO_MODEL_FOUND: return "prosac: no hypothesis with >= 4 inliers";
        case LP_DEGENERATE_CONFIGURATION: return "dlt: degenerate configuration";
        case LP_NUMERICAL_FAILURE: return "dlt: h33 vanished";
        case LP_EMPTY_INPUT: return "match_features: empty set";
        default: return "device error";
    }
}
static void sync_and_check(cudaStream_t s, int* d_status) {
    int st = 0;
    if (d_status) LPB_CUDA(cudaMemcpyAsync(&st, d_status, sizeof(int), cudaMemcpyDeviceToHost, s));
    LPB_CUDA(cudaStreamSynchronize(s));
    if (st) throw Status(static_cast<lp_status>(st), status_text(st));
}

static void validate_ext(const lp_extraction_config& c) {  // lorb.hpp:82-89
    if (c.fast_arc < 9 || c.fast_arc > 16) throw Status(LP_BAD_PARAMS, "fast_arc must be in [9,16]");
    if (c.top_n < 4) throw Status(LP_BAD_PARAMS, "top_n must be >= 4");
    if (c.n_d < 64 || c.n_d > 512) throw Status(LP_BAD_PARAMS, "n_d must be in [64,512]");
    if (!(c.harris_sigma > 0.0f)) throw Status(LP_INVALID_SIGMA, "harris_sigma must be > 0");
    if (!(c.brief_blur_sigma > 0.0f)) throw Status(LP_INVALID_SIGMA, "brief_blur_sigma must be > 0");
    if (c.patch_half < 1) throw Status(LP_BAD_PARAMS, "patch_half must be >= 1");
}

// Constant per-configuration tables for the extractor.
struct ExtractTables {
    DBuf harris_w, taps, pairs;
    std::vector<double> hw;
    int harris_r = 0, blur_r = 0;
    // the weights again in the kernel's parameter bank (k_detect9 reads them
    // as constant operands)
    std::vector<float> tp;
    void fill(ExtractArgs& a) const {
        a.harris_w = harris_w.as<double>();
        a.harris_r = harris_r;
        for (size_t i = 0; i < 49; ++i) a.hw[i] = i < hw.size() ? hw[i] : 0.0;
        for (size_t i = 0; i < 2 * kMaxBlurR + 1; ++i) a.btaps[i] = i < tp.size() ? tp[i] : 0.0f;
    }
    ExtractTables(const lp_extraction_config& c, const std::vector<lp_pair>& pat, cudaStream_t s,
                  bool upload_now = true) {
        hw = host::harris_weights(c.harris_sigma, &harris_r);
        if (harris_r > kMaxHarrisR) throw Status(LP_BAD_PARAMS, "harris_sigma too large for the device tile");
        tp = host::gaussian_kernel(c.brief_blur_sigma);
        blur_r = static_cast<int>(tp.size() / 2);
        if (blur_r > kMaxBlurR) throw Status(LP_BAD_PARAMS, "brief_blur_sigma too large");
        if (!upload_now) return;
        harris_w = upload(hw, s);
        taps = upload(tp, s);
        pairs = upload(pat, s);
    }
};

// Build DevRegions (scan areas + tiles) for regions over a set of images.
static std::vector<DevRegion> make_dev_regions(const std::vector<lp_region>& regs,
                                               const std::vector<int>& img_of,
                                               const std::vector<int>& slot_of, const int* w,
                                               const int* h, int* max_tiles) {
    std::vector<DevRegion> out;
    int mt = 0;
    for (size_t i = 0; i < regs.size(); ++i) {
        const lp_region& r = regs[i];
        const int im = img_of[i];
        DevRegion d;
        d.img = im;
        d.x0 = std::max(r.x0, 3);
        d.x1 = std::min(r.x1, w[im] - 3);
        d.y0 = std::max(r.y0, 3);
        d.y1 = std::min(r.y1, h[im] - 3);
        if (d.x0 >= d.x1 || d.y0 >= d.y1) throw Status(LP_REGION_TOO_SMALL, "fast_corners: region too small");
        if (w[im] > 65535 || h[im] > 65535) throw Status(LP_BAD_PARAMS, "image dimension above 65535");
        d.rx0 = r.x0;
        d.ry0 = r.y0;
        d.rx1 = r.x1;
        d.ry1 = r.y1;
        d.tiles_x = cdiv(d.x1 - d.x0, kDetTileX);
        d.ntiles = d.tiles_x * cdiv(d.y1 - d.y0, kDetTileY);
        d.out_slot = slot_of[i];
        mt = std::max(mt, d.ntiles);
        out.push_back(d);
    }
    *max_tiles = mt;
    return out;
}

static size_t surv_cap_for(const DevRegion& d) {
    return static_cast<size_t>((d.x1 - d.x0 + 1) / 2) * ((d.y1 - d.y0 + 1) / 2) + 64;
}

}  // namespace lpb

using namespace lpb;

struct lp_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    // pinned staging for the one-shot calls (a ctx serves one thread at a time;
    // every call leaves its stream idle, so growing it never races a copy)
    void* pin = nullptr;
    size_t pin_cap = 0;
    uint8_t* staging(size_t bytes) {
        if (bytes > pin_cap) {
            if (pin) cudaFreeHost(pin);
            pin = nullptr;
            pin_cap = 0;
            LPB_CUDA(cudaHostAlloc(&pin, std::max(bytes, size_t(1) << 20), cudaHostAllocDefault));
            pin_cap = std::max(bytes, size_t(1) << 20);
        }
        return static_cast<uint8_t*>(pin);
    }
};

namespace lpb {
// compaction writers (prims.cuh: k_flag_scatter)
struct WriteXY {  // scan-area index -> (x, y)
    int* xy;
    int x0, sw, y0, cap;
    __device__ void operator()(int i, int j) const {
        if (j < cap) {
            xy[2 * j] = x0 + i % sw;
            xy[2 * j + 1] = y0 + i / sw;
        }
    }
};
struct WriteKp {  // kept keypoints in input order
    const lp_keypoint* in;
    lp_keypoint* out;
    __device__ void operator()(int i, int j) const { out[j] = in[i]; }
};

// count the flags, then scatter the survivors (input order) with `write`
// into the output the caller sizes from the count: returns the count
template <class MakeWriter>
static int compact_flags(const uint8_t* flags, int n, cudaStream_t s, MakeWriter make_writer) {
    const int tiles = cdiv(n, kPrimTile);
    DBuf off(sizeof(unsigned) * tiles, s), tot(sizeof(int), s);
    LPB_LAUNCH(k_flag_count, tiles, 256, 0, s, flags, n, off.as<unsigned>());
    LPB_LAUNCH(k_scan_exclusive, 1, 1024, 0, s, off.as<unsigned>(), tiles, tot.as<int>());
    int total = 0;
    LPB_CUDA(cudaMemcpyAsync(&total, tot.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    LPB_CUDA(cudaStreamSynchronize(s));
    if (total > 0) {
        auto w = make_writer(total);
        LPB_LAUNCH(k_flag_scatter<decltype(w)>, tiles, 256, 0, s, flags, n, off.as<unsigned>(), w);
    }
    return total;
}

}  // namespace lpb

extern "C" {

const char* lp_last_error(void) { return g_err.c_str(); }
uint64_t lp_kernel_launches(void) { return g_launches.load(); }

void* lp_host_alloc(size_t bytes) {
    void* p = nullptr;
    if (cudaHostAlloc(&p, std::max<size_t>(bytes, 1), cudaHostAllocDefault) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return p;
}
// synth::texture (synth.hpp:17-34) on the host: the reference's seeded input
// generator (mt19937_64 noise, gaussian_blur imgops.hpp:50-72 with
// clamp-to-edge, contrast stretch, to_u8), so the bench and tools feed the
// bytes the reference's own bench and tests feed
lp_status lp_synth_texture(int w, int h, uint64_t seed, float sigma, uint8_t* out) {
    return guard([&] {
        if (w <= 0 || h <= 0 || !out) throw Status(LP_BAD_PARAMS, "synth_texture: empty image");
        std::mt19937_64 rng(seed);
        const size_t n = static_cast<size_t>(w) * h;
        std::vector<float> noise(n), tmp(n), blur(n);
        for (float& v : noise) v = static_cast<float>(rng() % 256);
        const std::vector<float> k = host::gaussian_kernel(sigma);
        const int r = static_cast<int>(k.size() / 2);
        for (int y = 0; y < h; ++y)
            for (int x = 0; x < w; ++x) {
                float acc = 0.0f;
                for (int i = -r; i <= r; ++i) acc += k[i + r] * noise[static_cast<size_t>(y) * w + std::clamp(x + i, 0, w - 1)];
                tmp[static_cast<size_t>(y) * w + x] = acc;
            }
        for (int y = 0; y < h; ++y)
            for (int x = 0; x < w; ++x) {
                float acc = 0.0f;
                for (int i = -r; i <= r; ++i) acc += k[i + r] * tmp[static_cast<size_t>(std::clamp(y + i, 0, h - 1)) * w + x];
                blur[static_cast<size_t>(y) * w + x] = acc;
            }
        float lo = blur[0], hi = blur[0];
        for (float v : blur) {
            lo = std::min(lo, v);
            hi = std::max(hi, v);
        }
        const float scale = hi > lo ? 255.0f / (hi - lo) : 0.0f;
        for (size_t i = 0; i < n; ++i) {
            float q = std::round((blur[i] - lo) * scale);  // to_u8, image.hpp:66-71
            q = std::min(std::max(q, 0.0f), 255.0f);
            out[i] = static_cast<uint8_t>(q);
        }
    });
}

void* lp_host_alloc_wc(size_t bytes) {
    void* p = nullptr;
    if (cudaHostAlloc(&p, std::max<size_t>(bytes, 1), cudaHostAllocWriteCombined) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return p;
}
void lp_host_free(void* p) {
    if (p) cudaFreeHost(p);
}

void lp_profile_enable(int on) {
    std::lock_guard<std::mutex> l(g_prof.mu);
    g_prof.on = on != 0;
}
void lp_profile_reset(void) {
    std::lock_guard<std::mutex> l(g_prof.mu);
    cudaDeviceSynchronize();
    g_prof.drain();
    g_prof.acc.clear();
    g_prof.occ.clear();
}
int lp_profile_read(char* names, int name_stride, double* total_ms, long long* launches, int cap) {
    std::lock_guard<std::mutex> l(g_prof.mu);
    cudaDeviceSynchronize();
    g_prof.drain();
    int i = 0;
    for (auto& kv : g_prof.acc) {
        if (i < cap) {
            std::snprintf(names + static_cast<size_t>(i) * name_stride, name_stride, "%s", kv.first.c_str());
            total_ms[i] = kv.second.first;
            launches[i] = kv.second.second;
        }
        ++i;
    }
    return i;
}

void lp_params_default(lp_params* p) {
    std::memset(p, 0, sizeof *p);
    p->extraction = lp_extraction_config{20, 9, 0.04f, 0.0f, 1.0f, 500, 256, 2.0f, 15};
    p->matching.tables = 4;
    p->matching.bits = 16;
    p->matching.t_probes = 16;
    p->matching.max_distance = 64;
    p->matching.ratio = 0.8f;
    p->matching.seed = 0;
    p->prosac.threshold_px = 3.0;
    p->prosac.max_iter = 1000;
    p->prosac.sampling = 0;
    p->prosac.confidence = 0.99;
    p->prosac.seed = 0;
    p->prosac.t_total = 200000.0;
    p->blend_levels = 4;
    p->homography_refresh = 1;
    p->seed = 0;
    p->overlap_fraction = 0.25;
}

lp_status lp_ctx_create(int device, lp_ctx** out) {
    return guard([&] {
        int n = 0;
        if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
            cudaGetLastError();
            throw Status(LP_NO_DEVICE, "no CUDA device");
        }
        LPB_CUDA(cudaSetDevice(device));
        // per-call scratch (cudaMallocAsync) stays cached in the device pool
        // across synchronisations instead of going back to the driver each call
        cudaMemPool_t pool;
        LPB_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
        uint64_t keep = 1ull << 30;
        LPB_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
        auto* c = new lp_ctx;
        c->device = device;
        LPB_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        c->own_stream = true;
        *out = c;
    });
}
void lp_ctx_destroy(lp_ctx* ctx) {
    if (!ctx) return;
    if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
    if (ctx->pin) cudaFreeHost(ctx->pin);
    delete ctx;
}
lp_status lp_ctx_set_stream(lp_ctx* ctx, void* s) {
    return guard([&] {
        if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
        ctx->own_stream = false;
        ctx->stream = static_cast<cudaStream_t>(s);
    });
}

// ---------------------------------------------------------------------------
__global__ void k_iota(int* p, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = i;
}

lp_status lp_fast_corners(lp_ctx* ctx, const uint8_t* img, int w, int h, int ch, lp_region r,
                          int thr, int arc, int* xy_out, int cap, int* count) {
    return guard([&] {
        if (ch != 1) throw Status(LP_UNSUPPORTED_FORMAT, "fast_corners: grayscale input required");
        const int x0 = std::max(r.x0, 3), x1 = std::min(r.x1, w - 3);
        const int y0 = std::max(r.y0, 3), y1 = std::min(r.y1, h - 3);
        if (x0 >= x1 || y0 >= y1) throw Status(LP_REGION_TOO_SMALL, "fast_corners: region too small");
        cudaStream_t s = ctx->stream;
        In<uint8_t> dimg(img, static_cast<size_t>(w) * h, s);
        const int sw = x1 - x0;
        const int n = sw * (y1 - y0);
        DBuf flags(n, s);
        fast_flags_launch(dimg.d, w, h, x0, y0, x1, y1, static_cast<uint8_t>(thr), arc, flags.as<uint8_t>(), s);
        std::unique_ptr<Out<int>> dxy;
        int k = 0;
        const int total = lpb::compact_flags(flags.as<uint8_t>(), n, s, [&](int t) {
            k = std::min(t, cap);
            dxy = std::make_unique<Out<int>>(xy_out, static_cast<size_t>(2) * std::max(k, 1), s);
            return lpb::WriteXY{dxy->d, x0, sw, y0, k};
        });
        if (k > 0) dxy->finish(s, static_cast<size_t>(2) * k);
        LPB_CUDA(cudaStreamSynchronize(s));
        *count = total;
    });
}

lp_status lp_harris_response(lp_ctx* ctx, const uint8_t* img, int w, int h, int ch, const int* xy,
                             int n, float alpha, float sigma, float* out) {
    return guard([&] {
        if (ch != 1) throw Status(LP_UNSUPPORTED_FORMAT, "harris_response: grayscale input required");
        if (n == 0) return;
        cudaStream_t s = ctx->stream;
        int r = 0;
        auto wts = host::harris_weights(sigma, &r);
        DBuf dw = upload(wts, s);
        In<uint8_t> dimg(img, static_cast<size_t>(w) * h, s);
        In<int> dxy(xy, static_cast<size_t>(2) * n, s);
        Out<float> dout(out, n, s);
        DevStatus st(s);
        harris_points_launch(dimg.d, w, h, dxy.d, n, dw.as<double>(), r, alpha, dout.d, st.ptr(), s);
        sync_and_check(s, st.ptr());
        dout.finish(s, n);
        LPB_CUDA(cudaStreamSynchronize(s));
    });
}

// bounding box of the candidates (lorb.hpp:258-266) on the device
__global__ void k_kp_bbox(const lp_keypoint* kp, int n, int* box) {
    int mnx = INT_MAX, mny = INT_MAX, mxx = INT_MIN, mxy = INT_MIN;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        mnx = min(mnx, kp[i].x);
        mxx = max(mxx, kp[i].x);
        mny = min(mny, kp[i].y);
        mxy = max(mxy, kp[i].y);
    }
    for (int o = 16; o > 0; o >>= 1) {
        mnx = min(mnx, __shfl_xor_sync(0xffffffffu, mnx, o));
        mxx = max(mxx, __shfl_xor_sync(0xffffffffu, mxx, o));
        mny = min(mny, __shfl_xor_sync(0xffffffffu, mny, o));
        mxy = max(mxy, __shfl_xor_sync(0xffffffffu, mxy, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(box, mnx);
        atomicMax(box + 1, mxx);
        atomicMin(box + 2, mny);
        atomicMax(box + 3, mxy);
    }
}

lp_status lp_nms(lp_ctx* ctx, const lp_keypoint* in, int n, int radius, lp_keypoint* out, int* count) {
    return guard([&] {
        *count = 0;
        if (n == 0) return;
        cudaStream_t s = ctx->stream;
        // the grid needs the candidates' bounding box on the host (its size):
        // host input is scanned here, device input reduced on the device
        In<lp_keypoint> dk(in, n, s);
        int box[4] = {INT_MAX, INT_MIN, INT_MAX, INT_MIN};
        if (is_device_ptr(in)) {
            DBuf db(sizeof box, s);
            LPB_CUDA(cudaMemcpyAsync(db.p, box, sizeof box, cudaMemcpyHostToDevice, s));
            LPB_LAUNCH(k_kp_bbox, std::min(cdiv(n, 256), 1184), 256, 0, s, dk.d, n, db.as<int>());
            LPB_CUDA(cudaMemcpyAsync(box, db.p, sizeof box, cudaMemcpyDeviceToHost, s));
            LPB_CUDA(cudaStreamSynchronize(s));
        } else {
            for (int i = 0; i < n; ++i) {
                box[0] = std::min(box[0], in[i].x);
                box[1] = std::max(box[1], in[i].x);
                box[2] = std::min(box[2], in[i].y);
                box[3] = std::max(box[3], in[i].y);
            }
        }
        const int minx = box[0], miny = box[2];
        const int gw = box[1] - minx + 1, gh = box[3] - miny + 1;
        DBuf grid(sizeof(int) * static_cast<size_t>(gw) * gh, s), keep(n, s);
        nms_generic_launch(dk.d, n, radius, minx, miny, gw, gh, grid.as<int>(), keep.as<uint8_t>(), s);
        std::unique_ptr<Out<lp_keypoint>> dout;
        const int k = lpb::compact_flags(keep.as<uint8_t>(), n, s, [&](int t) {
            dout = std::make_unique<Out<lp_keypoint>>(out, static_cast<size_t>(t), s);
            return lpb::WriteKp{dk.d, dout->d};
        });
        if (k > 0) dout->finish(s, static_cast<size_t>(k));
        LPB_CUDA(cudaStreamSynchronize(s));
        *count = k;
    });
}

__global__ void k_sort_key(const lp_keypoint* kp, const int* idx, int n, int field, uint32_t* key) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const lp_keypoint k = kp[idx[i]];
    key[i] = field == 0 ? (static_cast<uint32_t>(k.x) ^ 0x80000000u)
                        : field == 1 ? (static_cast<uint32_t>(k.y) ^ 0x80000000u) : ~float_key(k.response);
}
__global__ void k_gather_kp(const lp_keypoint* kp, const int* idx, int n, lp_keypoint* out) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = kp[idx[i]];
}

lp_status lp_select_top_n(lp_ctx* ctx, const lp_keypoint* in, int n, int top_n, lp_keypoint* out,
                          int* count) {
    return guard([&] {
        if (top_n < 1) throw Status(LP_BAD_PARAMS, "select_top_n: n must be >= 1");
        *count = 0;
        if (n == 0) return;
        cudaStream_t s = ctx->stream;
        In<lp_keypoint> dk(in, n, s);
        DBuf ia(sizeof(int) * n, s), ib(sizeof(int) * n, s), ka(sizeof(uint32_t) * n, s), kb(sizeof(uint32_t) * n, s),
            hist(sizeof(unsigned) * 256 * cdiv(n, kPrimTile), s);
        LPB_LAUNCH(k_iota, cdiv(n, 256), 256, 0, s, ia.as<int>(), n);
        // stable LSD passes: x asc, then y asc, then response desc (its key
        // inverted) (lorb.hpp:293-296); prims.cuh radix sort, result in (ka, ia)
        for (int field = 0; field < 3; ++field) {
            LPB_LAUNCH(k_sort_key, cdiv(n, 256), 256, 0, s, dk.d, ia.as<int>(), n, field, ka.as<uint32_t>());
            radix_sort_pairs(ka.as<uint32_t>(), ia.as<int>(), kb.as<uint32_t>(), ib.as<int>(), n, 32,
                             hist.as<unsigned>(), s);
        }
        const int k = std::min(n, top_n);
        Out<lp_keypoint> dout(out, k, s);
        LPB_LAUNCH(k_gather_kp, cdiv(k, 256), 256, 0, s, dk.d, ia.as<int>(), k, dout.d);
        dout.finish(s, k);
        LPB_CUDA(cudaStreamSynchronize(s));
        *count = k;
    });
}

lp_status lp_gaussian_blur(lp_ctx* ctx, const float* in, int w, int h, int ch, float sigma, float* out) {
    return guard([&] {
        auto taps = host::gaussian_kernel(sigma);
        cudaStream_t s = ctx->stream;
        const size_t n = static_cast<size_t>(w) * h * ch;
        DBuf dt = upload(taps, s), tmp(sizeof(float) * n, s);
        In<float> di(in, n, s);
        Out<float> dout(out, n, s);
        blur_launch(di.d, tmp.as<float>(), dout.d, w, h, ch, dt.as<float>(), static_cast<int>(taps.size() / 2), s);
        dout.finish(s, n);
        LPB_CUDA(cudaStreamSynchronize(s));
    });
}

lp_status lp_brief_descriptors(lp_ctx* ctx, const float* sm, int w, int h, const lp_keypoint* kps, int n,
                               const lp_pair* pairs, int n_d, int ph, uint64_t* out) {
    return guard([&] {
        if (n == 0) return;
        cudaStream_t s = ctx->stream;
        const int W2 = 2 * ((n_d + 63) / 64);
        In<float> dsm(sm, static_cast<size_t>(w) * h, s);
        In<lp_keypoint> dk(kps, n, s);
        In<lp_pair> dp(pairs, n_d, s);
        Out<uint64_t> dout(out, static_cast<size_t>(n) * W2, s);
        DevStatus st(s);
        brief_generic_launch(dsm.d, w, h, dk.d, n, dp.d, n_d, ph, dout.d, st.ptr(), s);
        sync_and_check(s, st.ptr());
        dout.finish(s, static_cast<size_t>(n) * W2);
        LPB_CUDA(cudaStreamSynchronize(s));
    });
}

lp_status lp_extract_features(lp_ctx* ctx, const uint8_t* img, int w, int h, int ch,
                              const lp_region* regions, int nreg, const lp_extraction_config* cfg,
                              const lp_pair* pairs, lp_keypoint* kp_out, uint64_t* desc_out, int cap,
                              int* count) {
    return guard([&] {
        validate_ext(*cfg);
        if (ch != 1) throw Status(LP_UNSUPPORTED_FORMAT, "fast_corners: grayscale input required");
        *count = 0;
        if (nreg == 0) return;
        cudaStream_t s = ctx->stream;
        std::vector<lp_region> regs(regions, regions + nreg);
        std::vector<lp_pair> pat(pairs, pairs + cfg->n_d);
        ExtractTables T(*cfg, pat, s, /*upload=*/false);
        if (w > 65535 || h > 65535) throw Status(LP_BAD_PARAMS, "image dimension above 65535");
        // A host image moves only its used rectangle: the regions plus the
        // BRIEF crop margin (lorb.hpp:371-375) and the Harris window, packed
        // into the call's pinned staging block. The extractor then runs on that
        // sub-image with the regions shifted into it; every test it makes
        // (segment ring, Harris window, patch fit, border clamps) lies inside
        // the margin, or at a real image edge that the sub-image shares, so
        // the results are those of the full image shifted back on the host.
        const bool host_img = !is_device_ptr(img);
        int bx0 = 0, by0 = 0, bw = w, bh = h;
        if (host_img) {
            const int M = std::max(cfg->patch_half + T.blur_r, T.harris_r + 2) + 4;
            int x0 = w, y0 = h, x1 = 0, y1 = 0;
            for (const auto& r : regs) {
                x0 = std::min(x0, r.x0 - M);
                y0 = std::min(y0, r.y0 - M);
                x1 = std::max(x1, r.x1 + M);
                y1 = std::max(y1, r.y1 + M);
            }
            x0 = std::max(x0, 0);
            y0 = std::max(y0, 0);
            x1 = std::min(x1, w);
            y1 = std::min(y1, h);
            if (x1 > x0 && y1 > y0) {
                bx0 = x0;
                by0 = y0;
                bw = x1 - x0;
                bh = y1 - y0;
                for (auto& r : regs) {
                    r.x0 -= bx0;
                    r.x1 -= bx0;
                    r.y0 -= by0;
                    r.y1 -= by0;
                }
            }
        }
        std::vector<int> zeros(nreg, 0);
        int tiles = 0;
        auto dregs = make_dev_regions(regs, zeros, zeros, &bw, &bh, &tiles);
        size_t scap = 0;
        for (auto& d : dregs) scap = std::max(scap, surv_cap_for(d));
        const int W2 = 2 * ((cfg->n_d + 63) / 64);
        const int cap_slot = nreg * cfg->top_n;

        // one staging block, mirrored in pinned host memory and on the device:
        // inputs [image | DevImage | regions | tables | status] go up in one
        // copy, outputs [status | count | keypoints | descriptors] come back in one
        size_t off = 0;
        auto put = [&](size_t bytes) {
            const size_t o = off;
            off = (off + bytes + 255) & ~size_t(255);
            return o;
        };
        const size_t o_img = host_img ? put(static_cast<size_t>(bw) * bh) : 0;
        const size_t o_dims = put(sizeof(DevImage)), o_regs = put(sizeof(DevRegion) * nreg),
                     o_hw = put(sizeof(double) * T.hw.size()), o_tp = put(sizeof(float) * T.tp.size()),
                     o_pairs = put(sizeof(lp_pair) * pat.size()), o_st = put(sizeof(int) * 2),
                     o_kp = put(sizeof(lp_keypoint) * cap_slot),
                     o_desc = put(sizeof(uint64_t) * static_cast<size_t>(cap_slot) * W2);
        const size_t total_bytes = off;
        uint8_t* hp = ctx->staging(total_bytes);
        DBuf blk(total_bytes, s);
        uint8_t* dp = blk.as<uint8_t>();
        if (host_img)
            for (int y = 0; y < bh; ++y)
                std::memcpy(hp + o_img + static_cast<size_t>(y) * bw, img + static_cast<size_t>(y + by0) * w + bx0, bw);
        const DevImage dim{host_img ? dp + o_img : img, bw, bh};
        std::memcpy(hp + o_dims, &dim, sizeof dim);
        std::memcpy(hp + o_regs, dregs.data(), sizeof(DevRegion) * nreg);
        std::memcpy(hp + o_hw, T.hw.data(), sizeof(double) * T.hw.size());
        std::memcpy(hp + o_tp, T.tp.data(), sizeof(float) * T.tp.size());
        std::memcpy(hp + o_pairs, pat.data(), sizeof(lp_pair) * pat.size());
        std::memset(hp + o_st, 0, sizeof(int) * 2);
        LPB_CUDA(cudaMemcpyAsync(dp, hp, o_st + sizeof(int) * 2, cudaMemcpyHostToDevice, s));

        DBuf surv(sizeof(uint64_t) * scap * nreg, s), scount(sizeof(unsigned) * nreg, s),
            kpr(sizeof(lp_keypoint) * static_cast<size_t>(nreg) * cfg->top_n, s), cr(sizeof(int) * nreg, s),
            hist(sizeof(unsigned) * kTopnHistBins * nreg, s);
        ExtractArgs a{};
        a.regions = reinterpret_cast<const DevRegion*>(dp + o_regs);
        a.nregions = nreg;
        a.max_tiles = tiles;
        a.images = reinterpret_cast<const DevImage*>(dp + o_dims);
        T.fill(a);
        a.harris_w = reinterpret_cast<const double*>(dp + o_hw);
        a.alpha = cfg->harris_alpha;
        a.threshold = cfg->harris_threshold;
        a.fast_t = static_cast<uint8_t>(cfg->fast_threshold);
        a.fast_arc = cfg->fast_arc;
        a.top_n = cfg->top_n;
        a.surv = surv.as<uint64_t>();
        a.surv_count = scount.as<unsigned>();
        a.hist = hist.as<unsigned>();
        a.surv_cap = static_cast<int>(scap);
        a.kp_region = kpr.as<lp_keypoint>();
        a.count_region = cr.as<int>();
        a.blur_taps = reinterpret_cast<const float*>(dp + o_tp);
        a.blur_r = T.blur_r;
        a.pairs = reinterpret_cast<const lp_pair*>(dp + o_pairs);
        a.n_d = cfg->n_d;
        a.patch_half = cfg->patch_half;
        a.nslots = 1;
        a.kp_out = reinterpret_cast<lp_keypoint*>(dp + o_kp);
        a.desc_out = reinterpret_cast<uint64_t*>(dp + o_desc);
        a.cap_slot = cap_slot;
        a.slot_count = reinterpret_cast<int*>(dp + o_st) + 1;
        a.status = reinterpret_cast<int*>(dp + o_st);
        extract_launch(a, s);
        LPB_CUDA(cudaMemcpyAsync(hp + o_st, dp + o_st, total_bytes - o_st, cudaMemcpyDeviceToHost, s));
        LPB_CUDA(cudaStreamSynchronize(s));
        const int* hst = reinterpret_cast<const int*>(hp + o_st);
        if (hst[0]) throw Status(static_cast<lp_status>(hst[0]), status_text(hst[0]));
        const int total = hst[1];
        const int k = std::min(total, cap);
        auto* hk = reinterpret_cast<lp_keypoint*>(hp + o_kp);
        for (int i = 0; i < k; ++i) {
            hk[i].x += bx0;
            hk[i].y += by0;
        }
        if (k > 0) {
            const size_t kb = sizeof(lp_keypoint) * k, db = sizeof(uint64_t) * k * W2;
            const bool dev_k = is_device_ptr(kp_out), dev_d = is_device_ptr(desc_out);
            if (dev_k) LPB_CUDA(cudaMemcpyAsync(kp_out, hk, kb, cudaMemcpyHostToDevice, s));
            else std::memcpy(kp_out, hk, kb);
            if (dev_d) LPB_CUDA(cudaMemcpyAsync(desc_out, dp + o_desc, db, cudaMemcpyDeviceToDevice, s));
            else std::memcpy(desc_out, hp + o_desc, db);
            if (dev_k || dev_d) LPB_CUDA(cudaStreamSynchronize(s));
        }
        *count = total;
    });
}

// ---------------------------------------------------------------------------
__global__ void k_distances(const uint64_t* a, const uint64_t* b, int n, int W2, int* out) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int d = 0;
    for (int w = 0; w < W2; ++w) d += __popcll(a[static_cast<size_t>(i) * W2 + w] ^ b[static_cast<size_t>(i) * W2 + w]);
    out[i] = d;
}
lp_status lp_descriptor_distances(lp_ctx* ctx, const uint64_t* a, const uint64_t* b, int n, int n_d, int* out) {
    return guard([&] {
        if (n == 0) return;
        cudaStream_t s = ctx->stream;
        const int W2 = 2 * ((n_d + 63) / 64);
        In<uint64_t> da(a, static_cast<size_t>(n) * W2, s), db(b, static_cast<size_t>(n) * W2, s);
        Out<int> dout(out, n, s);
        LPB_LAUNCH(k_distances, cdiv(n, 256), 256, 0, s, da.d, db.d, n, W2, dout.d);
        dout.finish(s, n);
        LPB_CUDA(cudaStreamSynchronize(s));
    });
}

// constant matcher tables
struct MatchTables {
    DBuf bitpos, partial;
    host::ProbeSet ps;
    MatchTables(int n_d, const lp_match_config& c, cudaStream_t s) {
        auto bp = host::lsh_bit_positions(n_d, c.tables, c.bits, c.seed);
        ps = host::probe_set(c.bits, c.t_probes);
        bitpos = upload(bp, s);
        partial = upload(ps.partial, s);
    }
    void fill(MatchArgs& a, const lp_match_config& c) const {
        a.bitpos = bitpos.as<int>();
        a.tables = c.tables;
        a.bits = c.bits;
        a.full_card = ps.full_card;
        a.partial = partial.as<uint64_t>();
        a.npartial = static_cast<int>(ps.partial.size());
        a.max_distance = c.max_distance;
        a.ratio = c.ratio;
    }
};

lp_status lp_match_features(lp_ctx* ctx, const uint64_t* set_a, int na, const uint64_t* set_b, int nb,
                            int n_d, const lp_match_config* cfg, lp_match* out, int cap, int* count) {
    return guard([&] {
        if (na == 0 || nb == 0) throw Status(LP_EMPTY_INPUT, "match_features: empty set");
        cudaStream_t s = ctx->stream;
        MatchTables T(n_d, *cfg, s);
        const int W2 = 2 * ((n_d + 63) / 64);
        const int capn = std::max(na, nb);
        DBuf desc(sizeof(uint64_t) * 2 * capn * W2, s), kps(sizeof(lp_keypoint) * 2 * capn, s),
            counts(sizeof(int) * 2, s), keys(sizeof(uint64_t) * 2 * capn * cfg->tables, s),
            qres(sizeof(int4) * capn, s), matches(sizeof(lp_match) * capn, s), corr(sizeof(lp_corr) * capn, s),
            mc(sizeof(int), s);
        DevStatus pst(s);
        auto kind = [](const void* p) { return is_device_ptr(p) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice; };
        LPB_CUDA(cudaMemcpyAsync(desc.p, set_b, sizeof(uint64_t) * nb * W2, kind(set_b), s));
        LPB_CUDA(cudaMemcpyAsync(desc.as<uint64_t>() + static_cast<size_t>(capn) * W2, set_a,
                                 sizeof(uint64_t) * na * W2, kind(set_a), s));
        LPB_CUDA(cudaMemsetAsync(kps.p, 0, sizeof(lp_keypoint) * 2 * capn, s));
        int hc[2] = {nb, na};
        LPB_CUDA(cudaMemcpyAsync(counts.p, hc, sizeof hc, cudaMemcpyHostToDevice, s));
        MatchArgs a{};
        a.npairs = 1;
        a.qslot0 = 1;
        a.tslot0 = 0;
        a.nslots = 2;
        a.desc = desc.as<uint64_t>();
        a.kps = kps.as<lp_keypoint>();
        a.counts = counts.as<int>();
        a.cap = capn;
        a.n_d = n_d;
        T.fill(a, *cfg);
        a.keys = keys.as<uint64_t>();
        a.qres = qres.as<int4>();
        a.matches = matches.as<lp_match>();
        a.corr = corr.as<lp_corr>();
        a.match_counts = mc.as<int>();
        a.pair_status = pst.ptr();
        match_launch(a, s);
        sync_and_check(s, pst.ptr());
        int n = 0;
        LPB_CUDA(cudaMemcpy(&n, mc.p, sizeof(int), cudaMemcpyDeviceToHost));
        const int k = std::min(n, cap);
        if (k > 0)
            LPB_CUDA(cudaMemcpyAsync(out, matches.p, sizeof(lp_match) * k,
                                     is_device_ptr(out) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, s));
        LPB_CUDA(cudaStreamSynchronize(s));
        *count = n;
    });
}

lp_status lp_lsh_query(lp_ctx* ctx, const uint64_t* train, int nt, const uint64_t* queries, int nq, int n_d,
                       const lp_match_config* cfg, int query_id0, long long* offsets, lp_match* out, long long cap,
                       long long* total) {
    return guard([&] {
        *total = 0;
        if (nq <= 0) return;
        if (nt == 0) {
            for (int q = 0; q <= nq; ++q) offsets[q] = 0;
            return;
        }
        cudaStream_t s = ctx->stream;
        MatchTables T(n_d, *cfg, s);
        const int W2 = 2 * ((n_d + 63) / 64);
        const int capn = std::max(nq, nt);
        DBuf desc(sizeof(uint64_t) * 2 * capn * W2, s), counts(sizeof(int) * 2, s),
            keys(sizeof(uint64_t) * 2 * capn * std::max(cfg->tables, 1), s);
        auto kind = [](const void* p) { return is_device_ptr(p) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice; };
        LPB_CUDA(cudaMemcpyAsync(desc.p, train, sizeof(uint64_t) * nt * W2, kind(train), s));
        LPB_CUDA(cudaMemcpyAsync(desc.as<uint64_t>() + static_cast<size_t>(capn) * W2, queries,
                                 sizeof(uint64_t) * nq * W2, kind(queries), s));
        int hc[2] = {nt, nq};
        LPB_CUDA(cudaMemcpyAsync(counts.p, hc, sizeof hc, cudaMemcpyHostToDevice, s));
        MatchArgs a{};
        a.npairs = 1;
        a.qslot0 = 1;
        a.tslot0 = 0;
        a.nslots = 2;
        a.desc = desc.as<uint64_t>();
        a.counts = counts.as<int>();
        a.cap = capn;
        a.n_d = n_d;
        T.fill(a, *cfg);
        a.keys = keys.as<uint64_t>();
        Out<lp_match> dout(out, static_cast<size_t>(std::max<long long>(cap, 0)), s);
        const long long n = lsh_query_launch(a, nq, query_id0, offsets, dout.d, cap, s);
        dout.finish(s, static_cast<size_t>(std::min(n, cap)));
        LPB_CUDA(cudaStreamSynchronize(s));
        *total = n;
    });
}

// ---------------------------------------------------------------------------
lp_status lp_dlt_homography(lp_ctx* ctx, const lp_corr* pairs, int n, lp_homography* out) {
    return guard([&] {
        if (n < 4) throw Status(LP_INSUFFICIENT_MATCHES, "dlt: need at least 4 pairs");
        cudaStream_t s = ctx->stream;
        In<lp_corr> dc(pairs, n, s);
        DBuf scratch(sizeof(double) * prosac_scratch_doubles(n), s), dh(sizeof(lp_homography), s);
        DevStatus st(s);
        dlt_launch(dc.d, n, scratch.as<double>(), dh.as<lp_homography>(), st.ptr(), s);
        sync_and_check(s, st.ptr());
        LPB_CUDA(cudaMemcpy(out, dh.p, sizeof(lp_homography), cudaMemcpyDeviceToHost));
    });
}

lp_status lp_symmetric_transfer_errors(lp_ctx* ctx, const lp_homography* h, const lp_homography* h_inv,
                                       const lp_corr* pairs, int n, double* out) {
    return guard([&] {
        if (n < 0) throw Status(LP_BAD_PARAMS, "symmetric_transfer_error: n < 0");
        if (n == 0) return;
        cudaStream_t s = ctx->stream;
        In<lp_corr> dc(pairs, n, s);
        Out<double> o(out, n, s);
        ste_launch(*h, *h_inv, dc.d, n, o.d, s);
        o.finish(s, n);
        LPB_CUDA(cudaStreamSynchronize(s));
    });
}

lp_status lp_prosac_homography(lp_ctx* ctx, const lp_corr* matches, int n, const lp_prosac_config* cfg,
                               lp_homography* model, uint8_t* mask, int* inlier_count, int* iterations,
                               int* trace_pool, int* trace_samples) {
    return guard([&] {
        *iterations = 0;
        if (n < 4) throw Status(LP_INSUFFICIENT_MATCHES, "prosac: need at least 4 matches");
        cudaStream_t s = ctx->stream;
        // termination table row for this n (host glibc, exact)
        std::vector<int> row(static_cast<size_t>(n) + 1, cfg->max_iter + 1);
        {
            auto tab = host::prosac_exit_table(n, cfg->max_iter, cfg->confidence);
            for (int c = 0; c <= n; ++c) row[c] = tab[static_cast<size_t>(n) * (n + 1) + c];
        }
        In<lp_corr> dc(matches, n, s);
        const int mi = std::max(cfg->max_iter, 1);
        DBuf drow = upload(row, s), cnt(sizeof(int), s), scratch(sizeof(double) * prosac_scratch_doubles(n), s),
            dm(sizeof(lp_homography), s), dmask(n, s), dic(sizeof(int), s), dit(sizeof(int), s),
            tp(sizeof(int) * mi, s), ts(sizeof(int) * mi * 4, s);
        DevStatus pst(s);
        LPB_CUDA(cudaMemcpyAsync(cnt.p, &n, sizeof(int), cudaMemcpyHostToDevice, s));
        ProsacArgs a{};
        a.npairs = 1;
        a.corr = dc.d;
        a.counts = cnt.as<int>();
        a.cap = n;
        a.threshold = cfg->threshold_px;
        a.max_iter = cfg->max_iter;
        a.uniform = cfg->sampling;
        a.t_total = cfg->t_total;
        a.seed = cfg->seed;
        a.frame = 0;
        a.per_pair_seed = 0;
        a.exit_tab = drow.as<int>();
        a.nmax = 0;
        a.scratch = scratch.as<double>();
        a.model = dm.as<lp_homography>();
        a.mask = dmask.as<uint8_t>();
        a.inlier_count = dic.as<int>();
        a.iterations = dit.as<int>();
        a.trace_pool = tp.as<int>();
        a.trace_samples = ts.as<int>();
        a.pair_status = pst.ptr();
        prosac_launch(a, s);
        int st = 0, its = 0;
        LPB_CUDA(cudaMemcpyAsync(&st, pst.ptr(), sizeof(int), cudaMemcpyDeviceToHost, s));
        LPB_CUDA(cudaMemcpyAsync(&its, dit.p, sizeof(int), cudaMemcpyDeviceToHost, s));
        LPB_CUDA(cudaStreamSynchronize(s));
        *iterations = its;
        if (trace_pool && its > 0) LPB_CUDA(cudaMemcpy(trace_pool, tp.p, sizeof(int) * its, cudaMemcpyDeviceToHost));
        if (trace_samples && its > 0)
            LPB_CUDA(cudaMemcpy(trace_samples, ts.p, sizeof(int) * its * 4, cudaMemcpyDeviceToHost));
        if (st) throw Status(static_cast<lp_status>(st), status_text(st));
        LPB_CUDA(cudaMemcpy(model, dm.p, sizeof(lp_homography), cudaMemcpyDeviceToHost));
        if (mask) LPB_CUDA(cudaMemcpy(mask, dmask.p, n, is_device_ptr(mask) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost));
        LPB_CUDA(cudaMemcpy(inlier_count, dic.p, sizeof(int), cudaMemcpyDeviceToHost));
    });
}

// ---------------------------------------------------------------------------
lp_status lp_warp_image(lp_ctx* ctx, const float* img, int w, int h, int ch, const lp_homography* hom,
                        const lp_canvas* cv, float* out, float* coverage) {
    return guard([&] {
        if (std::abs(host::h_det(hom->h)) < 1e-9) throw Status(LP_SINGULAR_HOMOGRAPHY, "warp_image: singular homography");
        double hi[9];
        host::h_inverse(hom->h, hi);
        cudaStream_t s = ctx->stream;
        std::vector<double> hv(hi, hi + 9);
        DBuf dh = upload(hv, s);
        const size_t np = static_cast<size_t>(cv->width) * cv->height;
        In<float> di(img, static_cast<size_t>(w) * h * ch, s);
        Out<float> dout(out, np * ch, s), dcov(coverage, np, s);
        warp_generic_launch(di.d, w, h, ch, dh.as<double>(), cv->width, cv->height, cv->origin_x, cv->origin_y,
                            dout.d, dcov.d, s);
        dout.finish(s, np * ch);
        dcov.finish(s, np);
        LPB_CUDA(cudaStreamSynchronize(s));
    });
}

lp_status lp_linear_seam_mask(lp_ctx* ctx, const float* covs, int n, int w, int h, float* masks) {
    return guard([&] {
        if (n < 1) throw Status(LP_BAD_PARAMS, "linear_seam_mask: no coverage masks");
        cudaStream_t s = ctx->stream;
        const size_t np = static_cast<size_t>(w) * h * n;
        In<float> dc(covs, np, s);
        Out<float> dm(masks, np, s);
        seam_generic_launch(dc.d, n, w, h, dm.d, s);
        dm.finish(s, np);
        LPB_CUDA(cudaStreamSynchronize(s));
    });
}

lp_status lp_downsample(lp_ctx* ctx, const float* in, int w, int h, int ch, float* out) {
    return guard([&] {
        if (w < 2 || h < 2) throw Status(LP_IMAGE_TOO_SMALL, "downsample: need at least 2x2");
        cudaStream_t s = ctx->stream;
        DBuf taps = upload(host::gaussian_kernel(1.0f), s), tmp(sizeof(float) * (w / 2) * h * ch, s);
        In<float> di(in, static_cast<size_t>(w) * h * ch, s);
        const size_t no = static_cast<size_t>(w / 2) * (h / 2) * ch;
        Out<float> dout(out, no, s);
        downsample_launch(di.d, w, h, ch, taps.as<float>(), tmp.as<float>(), dout.d, s);
        dout.finish(s, no);
        LPB_CUDA(cudaStreamSynchronize(s));
    });
}

lp_status lp_upsample(lp_ctx* ctx, const float* in, int w, int h, int ch, int tw, int th, float* out) {
    return guard([&] {
        if (std::abs(tw - 2 * w) > 1 || std::abs(th - 2 * h) > 1)
            throw Status(LP_BAD_TARGET_DIMS, "upsample: target dims must be ~2x source");
        cudaStream_t s = ctx->stream;
        In<float> di(in, static_cast<size_t>(w) * h * ch, s);
        const size_t no = static_cast<size_t>(tw) * th * ch;
        Out<float> dout(out, no, s);
        upsample_launch(di.d, w, h, ch, tw, th, dout.d, s);
        dout.finish(s, no);
        LPB_CUDA(cudaStreamSynchronize(s));
    });
}

static size_t pyr_total(int w, int h, int ch, int levels) {
    size_t t = 0;
    for (int k = 0; k < levels; ++k) {
        t += static_cast<size_t>(w) * h * ch;
        w /= 2;
        h /= 2;
    }
    return t;
}

// gaussian_pyramid into a packed device buffer (imgops.hpp:142-153)
static void pyramid_dev(const float* in, int w, int h, int ch, int levels, float* out, cudaStream_t s) {
    if (levels < 1) throw Status(LP_TOO_MANY_LEVELS, "pyramid: levels must be >= 1");
    {
        int lw = w, lh = h;
        for (int i = 1; i < levels; ++i) {
            if (lw < 2 || lh < 2) throw Status(LP_TOO_MANY_LEVELS, "pyramid: image too small for requested levels");
            lw /= 2;
            lh /= 2;
        }
    }
    LPB_CUDA(cudaMemcpyAsync(out, in, sizeof(float) * w * h * ch, cudaMemcpyDeviceToDevice, s));
    DBuf taps = upload(host::gaussian_kernel(1.0f), s), tmp(sizeof(float) * std::max(1, w / 2) * h * ch, s);
    float* prev = out;
    for (int i = 1; i < levels; ++i) {
        float* next = prev + static_cast<size_t>(w) * h * ch;
        downsample_launch(prev, w, h, ch, taps.as<float>(), tmp.as<float>(), next, s);
        prev = next;
        w /= 2;
        h /= 2;
    }
}

lp_status lp_gaussian_pyramid(lp_ctx* ctx, const float* in, int w, int h, int ch, int levels, float* out) {
    return guard([&] {
        cudaStream_t s = ctx->stream;
        if (levels < 1) throw Status(LP_TOO_MANY_LEVELS, "pyramid: levels must be >= 1");
        const size_t tot = pyr_total(w, h, ch, levels);
        In<float> di(in, static_cast<size_t>(w) * h * ch, s);
        Out<float> dout(out, tot, s);
        pyramid_dev(di.d, w, h, ch, levels, dout.d, s);
        dout.finish(s, tot);
        LPB_CUDA(cudaStreamSynchronize(s));
    });
}

lp_status lp_build_laplacian(lp_ctx* ctx, const float* in, int w, int h, int ch, int levels, float* out) {
    return guard([&] {
        cudaStream_t s = ctx->stream;
        if (levels < 1) throw Status(LP_TOO_MANY_LEVELS, "build_laplacian: levels must be >= 1");
        const size_t tot = pyr_total(w, h, ch, levels);
        In<float> di(in, static_cast<size_t>(w) * h * ch, s);
        Out<float> dout(out, tot, s);
        pyramid_dev(di.d, w, h, ch, levels, dout.d, s);
        DBuf up(sizeof(float) * static_cast<size_t>(w) * h * ch, s);
        float* lv = dout.d;
        int lw = w, lh = h;
        for (int k = 0; k + 1 < levels; ++k) {
            float* nx = lv + static_cast<size_t>(lw) * lh * ch;
            upsample_launch(nx, lw / 2, lh / 2, ch, lw, lh, up.as<float>(), s);
            sub_launch(lv, up.as<float>(), static_cast<size_t>(lw) * lh * ch, s);
            lv = nx;
            lw /= 2;
            lh /= 2;
        }
        dout.finish(s, tot);
        LPB_CUDA(cudaStreamSynchronize(s));
    });
}

lp_status lp_collapse_laplacian(lp_ctx* ctx, const float* packed, int w, int h, int ch, int levels, float* out) {
    return guard([&] {
        if (levels < 1) throw Status(LP_TOO_MANY_LEVELS, "collapse_laplacian: empty pyramid");
        cudaStream_t s = ctx->stream;
        const size_t tot = pyr_total(w, h, ch, levels);
        In<float> dp(packed, tot, s);
        std::vector<const float*> lv(levels);
        std::vector<int> dw(levels), dh(levels);
        const float* p = dp.d;
        int lw = w, lh = h;
        for (int k = 0; k < levels; ++k) {
            lv[k] = p;
            dw[k] = lw;
            dh[k] = lh;
            p += static_cast<size_t>(lw) * lh * ch;
            lw /= 2;
            lh /= 2;
        }
        DBuf a(sizeof(float) * static_cast<size_t>(w) * h * ch, s), b(sizeof(float) * static_cast<size_t>(w) * h * ch, s);
        float* acc = a.as<float>();
        float* nxt = b.as<float>();
        const size_t ntop = static_cast<size_t>(dw[levels - 1]) * dh[levels - 1] * ch;
        LPB_CUDA(cudaMemcpyAsync(acc, lv[levels - 1], sizeof(float) * ntop, cudaMemcpyDeviceToDevice, s));
        for (int k = levels - 2; k >= 0; --k) {
            upsample_launch(acc, dw[k + 1], dh[k + 1], ch, dw[k], dh[k], nxt, s);
            add_launch(nxt, lv[k], static_cast<size_t>(dw[k]) * dh[k] * ch, s);
            std::swap(acc, nxt);
        }
        const size_t n0 = static_cast<size_t>(w) * h * ch;
        LPB_CUDA(cudaMemcpyAsync(out, acc, sizeof(float) * n0,
                                 is_device_ptr(out) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, s));
        LPB_CUDA(cudaStreamSynchronize(s));
    });
}

}  // extern "C"

// ---------------------------------------------------------------------------
// windowed compositor buffers (shared by lp_multiband_blend and the rig)
namespace lpb {

struct ComposeBuffers {
    int ncams = 0, levels = 0;
    std::vector<Win> win;  // host copy
    std::vector<Win> win_unused_;
    std::vector<std::unique_ptr<DBuf>> bufs;
    ComposeArgs args{};

    DBuf runs, runs_used, status, mask_state;
    size_t bytes_total = 0;  // device bytes of the windows and collapse buffers
    std::vector<float*> host_G, host_M;  // [c * levels + k]
    std::vector<PyrTma> pyr_tma;         // per source level k: k_pyr_down2's tensor maps
    std::vector<BlendTma> blend_tma;     // per level k < levels - 1: k_blend_lean's tensor maps

    // analytic: level-0 masks come from coverage runs (the rig); otherwise the
    // caller fills M[c][0] (lp_multiband_blend).
    void build(int ncams_, int levels_, int W0, int H0, const std::vector<Win>& win0, bool analytic,
               cudaStream_t s) {
        if (ncams_ > kMaxCompCams) throw Status(LP_BAD_PARAMS, "compositor: too many cameras");
        if (levels_ > kMaxCompLevels) throw Status(LP_TOO_MANY_LEVELS, "compositor: too many blend levels");
        ncams = ncams_;
        levels = levels_;
        bufs.clear();
        win.assign(static_cast<size_t>(ncams) * levels, Win{0, 0, 0, 0, 0});
        args = ComposeArgs{};
        args.ncams = ncams;
        args.levels = levels;
        args.analytic_masks = analytic ? 1 : 0;
        int W = W0, H = H0;
        for (int k = 0; k < levels; ++k) {
            args.W[k] = W;
            args.H[k] = H;
            W /= 2;
            H /= 2;
        }
        host_G.assign(static_cast<size_t>(ncams) * levels, nullptr);
        host_M.assign(host_G.size(), nullptr);
        bytes_total = 0;
        auto alloc = [&](size_t bytes) {
            bufs.push_back(std::make_unique<DBuf>(std::max<size_t>(bytes, 16), s));
            bytes_total += std::max<size_t>(bytes, 16);
            return bufs.back()->p;
        };
        size_t total_rows = 0;
        for (int c = 0; c < ncams; ++c) {
            const Win w0 = win0[c];
            for (int k = 0; k < levels; ++k) {
                Win w;
                w.x0 = w0.x0 >> k;
                w.y0 = w0.y0 >> k;
                const int x1 = std::min(args.W[k], (w0.x0 + w0.w + (1 << k) - 1) >> k);
                const int y1 = std::min(args.H[k], (w0.y0 + w0.h + (1 << k) - 1) >> k);
                w.w = std::max(0, x1 - w.x0);
                w.h = std::max(0, y1 - w.y0);
                w.p = (w.w + 3) & ~3;
                win[c * levels + k] = w;
                args.win[c][k] = w;
                const size_t np = static_cast<size_t>(w.p) * w.h;
                args.G[c][k] = static_cast<float*>(alloc(sizeof(float) * np));
                args.M[c][k] = static_cast<float*>(alloc(sizeof(float) * np));
                host_G[c * levels + k] = args.G[c][k];
                host_M[c * levels + k] = args.M[c][k];
            }
            if (analytic) {
                const Win w = win[c * levels];
                args.cov_words[c] = cdiv(w.w, 32);
                args.cov[c] = static_cast<uint32_t*>(alloc(sizeof(uint32_t) * args.cov_words[c] * std::max(w.h, 1)));
                args.run_rows[c] = static_cast<int2*>(alloc(sizeof(int2) * std::max(w.h, 1)));
                args.mtile_w[c] = cdiv(w.w, kMaskTileX);
                args.mtile[c] = static_cast<uint8_t*>(alloc(static_cast<size_t>(args.mtile_w[c]) * cdiv(std::max(w.h, 1), kMaskTileY)));
                args.run_base[c] = static_cast<int>(total_rows * kRunSlots);
                total_rows += w.h;
            }
        }
        for (int k = 1; k < levels; ++k) {
            args.Rp[k] = (args.W[k] + 3) & ~3;
            args.R[k] = static_cast<float*>(alloc(sizeof(float) * static_cast<size_t>(args.Rp[k]) * args.H[k]));
        }
        if (analytic) {
            args.runs_overflow_base = static_cast<int>(total_rows * kRunSlots);
            args.runs_cap = static_cast<int>(std::min<size_t>(total_rows * (kRunSlots + 4) + 4096, 1u << 30));
            runs = DBuf(sizeof(int2) * args.runs_cap, s);
            runs_used = DBuf(sizeof(int), s);
            args.runs = runs.as<int2>();
            args.runs_used = runs_used.as<int>();
            // masks of fresh arenas are never current (LPB_MASK_REUSE=0: recompute every frame)
            const char* e = std::getenv("LPB_MASK_REUSE");
            if (!(e && e[0] == '0')) {
                mask_state = DBuf(sizeof(MaskState), s);
                LPB_CUDA(cudaMemsetAsync(mask_state.p, 0, sizeof(MaskState), s));
                args.mask_state = mask_state.as<MaskState>();
            }
        }
        status = DBuf(sizeof(int), s);
        LPB_CUDA(cudaMemsetAsync(status.p, 0, sizeof(int), s));
        args.status = status.as<int>();
        auto taps = host::gaussian_kernel(1.0f);
        for (int q = 0; q < 7; ++q) args.down_taps[q] = taps[q];
        {   // level-0 blend tiles covered by one camera at weight 1 (LPB_BLEND_UNIT=0: off)
            const char* e = std::getenv("LPB_BLEND_UNIT");
            args.blend_unit = (e && e[0] == '0') ? 0 : 1;
        }
        // TMA staging of the pyramid boxes (LPB_TMA=0: cp.async everywhere)
        pyr_tma.assign(std::max(levels - 1, 1), PyrTma{});
        args.pyr_tma = nullptr;
        args.blend_tma = nullptr;
        const char* env = std::getenv("LPB_TMA");
        if (levels > 1 && !(env && env[0] == '0')) {
            bool ok = true;
            for (int k = 0; k + 1 < levels && ok; ++k) {
                PyrTma& t = pyr_tma[k];
                for (int c = 0; c < ncams && ok; ++c) {
                    const Win& w = win[c * levels + k];
                    if (w.w == 0 || w.h == 0) continue;  // no CTA of this camera stages at level k
                    ok = tma_encode_f32_2d(&t.g[c], args.G[c][k], w.w, w.h, w.p, PD2_BW, PD2_BH) &&
                         tma_encode_f32_2d(&t.m[c], args.M[c][k], w.w, w.h, w.p, PD2_BW, PD2_BH);
                }
                t.ok = 1;
            }
            if (ok) args.pyr_tma = pyr_tma.data();
            // k_blend_lean<64 >> k> stages level k+1 of every camera and R_k+1
            blend_tma.assign(levels - 1, BlendTma{});
            ok = true;
            for (int k = 0; k + 1 < levels && ok; ++k) {
                const int txk = kBlendAlignX >> k;
                if (txk < 4) break;
                const int cx = lean_cx(txk), cy = lean_cy(txk);
                if (cx > 256 || cy > 256) continue;  // beyond the TMA box limit: cp.async
                BlendTma& t = blend_tma[k];
                for (int c = 0; c < ncams && ok; ++c) {
                    const Win& w = win[c * levels + k + 1];
                    if (w.w == 0 || w.h == 0) continue;
                    ok = tma_encode_f32_2d(&t.g[c], args.G[c][k + 1], w.w, w.h, w.p, cx, cy);
                }
                ok = ok && tma_encode_f32_2d(&t.r, args.R[k + 1], args.W[k + 1], args.H[k + 1], args.Rp[k + 1], cx, cy);
                t.ok = ok ? 1 : 0;
            }
            if (ok) args.blend_tma = blend_tma.data();
        }
    }
};

static void check_levels(int w, int h, int levels) {  // gaussian_pyramid, imgops.hpp:143-150
    if (levels < 1) throw Status(LP_TOO_MANY_LEVELS, "build_laplacian: levels must be >= 1");
    for (int i = 1; i < levels; ++i) {
        if (w < 2 || h < 2) throw Status(LP_TOO_MANY_LEVELS, "pyramid: image too small for requested levels");
        w /= 2;
        h /= 2;
    }
}

__global__ void k_deinterleave(const float* in, int w, int np, int ch, int c, float* out, int pitch) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < np) out[(i / w) * pitch + i % w] = in[static_cast<size_t>(i) * ch + c];
}
__global__ void k_interleave_u8(const uint8_t* in, int np, int ch, int c, uint8_t* out) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < np) out[static_cast<size_t>(i) * ch + c] = in[i];
}

}  // namespace lpb

extern "C" lp_status lp_multiband_blend(lp_ctx* ctx, const float* images, const float* masks, int n, int w,
                                        int h, int ch, int levels, uint8_t* out) {
    return guard([&] {
        if (n < 1) throw Status(LP_MASK_MISMATCH, "multiband_blend: image/mask count mismatch");
        check_levels(w, h, levels);
        cudaStream_t s = ctx->stream;
        const size_t np = static_cast<size_t>(w) * h;
        In<float> di(images, np * ch * n, s), dm(masks, np * n, s);
        ComposeBuffers cb;
        std::vector<Win> full(n, Win{0, 0, w, h, 0});
        cb.build(n, levels, w, h, full, false, s);
        const size_t pitch = cb.win[0].p;  // window rows are padded to float4
        DBuf o1(np, s);
        Out<uint8_t> dout(out, np * ch, s);
        cb.args.out = o1.as<uint8_t>();
        for (int c = 0; c < n; ++c)
            LPB_CUDA(cudaMemcpy2DAsync(cb.host_M[c * levels], sizeof(float) * pitch, dm.d + np * c, sizeof(float) * w,
                                       sizeof(float) * w, h, cudaMemcpyDeviceToDevice, s));
        for (int cc = 0; cc < ch; ++cc) {
            for (int c = 0; c < n; ++c) {
                if (ch == 1)
                    LPB_CUDA(cudaMemcpy2DAsync(cb.host_G[c * levels], sizeof(float) * pitch, di.d + np * c,
                                               sizeof(float) * w, sizeof(float) * w, h, cudaMemcpyDeviceToDevice, s));
                else
                    LPB_LAUNCH(k_deinterleave, cdiv(np, 256), 256, 0, s, di.d + np * ch * c, w, static_cast<int>(np),
                               ch, cc, cb.host_G[c * levels], static_cast<int>(pitch));
            }
            blend_launch(cb.args, s);
            if (ch == 1)
                LPB_CUDA(cudaMemcpyAsync(dout.d, o1.p, np, cudaMemcpyDeviceToDevice, s));
            else
                LPB_LAUNCH(k_interleave_u8, cdiv(np, 256), 256, 0, s, o1.as<uint8_t>(), static_cast<int>(np), ch, cc,
                           dout.d);
        }
        dout.finish(s, np * ch);
        LPB_CUDA(cudaStreamSynchronize(s));
    });
}

namespace lpb {
// RigLayout cameras -> device RectCam descriptors (no pointers yet), in
// stage_rectify_crop's order of checks (pipeline.hpp:393-414)
static std::vector<RectCam> rect_cams(int ncams, int w, int h, const lp_camera* cams) {
    std::vector<RectCam> out(ncams);
    for (int c = 0; c < ncams; ++c) {
        const lp_camera& cam = cams[c];
        RectCam& rc = out[c];
        rc.src = nullptr;
        rc.dst = nullptr;
        static const double I[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
        rc.identity = 1;
        for (int j = 0; j < 9; ++j)
            if (!(cam.pre_transform.h[j] == I[j])) rc.identity = 0;
        if (!rc.identity) {
            if (std::abs(host::h_det(cam.pre_transform.h)) < 1e-9)
                throw Status(LP_SINGULAR_HOMOGRAPHY, "warp_image: singular homography");
            host::h_inverse(cam.pre_transform.h, rc.hinv);
        } else {
            for (int j = 0; j < 9; ++j) rc.hinv[j] = I[j];
        }
        rc.x0 = 0;
        rc.y0 = 0;
        rc.w = w;
        rc.h = h;
        if (cam.has_crop) {
            const lp_region& r = cam.crop;
            if (r.x0 < 0 || r.y0 < 0 || r.x1 > w || r.y1 > h || r.x1 - r.x0 < 1 || r.y1 - r.y0 < 1)
                throw Status(LP_BAD_PARAMS, "rectify_crop: crop outside image");
            rc.x0 = r.x0;
            rc.y0 = r.y0;
            rc.w = r.x1 - r.x0;
            rc.h = r.y1 - r.y0;
        }
    }
    return out;
}
}  // namespace lpb

extern "C" lp_status lp_rectify_crop(lp_ctx* ctx, int ncams, int w, int h, const lp_camera* cams,
                                     const uint8_t* const* images, uint8_t* const* outputs, int* out_w,
                                     int* out_h) {
    return guard([&] {
        if (ncams < 1 || ncams > kMaxCams || w < 1 || h < 1) throw Status(LP_BAD_PARAMS, "rectify_crop: bad dims");
        cudaStream_t s = ctx->stream;
        auto rc = rect_cams(ncams, w, h, cams);
        const size_t fb = static_cast<size_t>(w) * h;
        std::vector<std::unique_ptr<In<uint8_t>>> ins;
        std::vector<std::unique_ptr<Out<uint8_t>>> outs;
        int mw = 0, mh = 0;
        for (int c = 0; c < ncams; ++c) {
            ins.push_back(std::make_unique<In<uint8_t>>(images[c], fb, s));
            outs.push_back(std::make_unique<Out<uint8_t>>(outputs[c], static_cast<size_t>(rc[c].w) * rc[c].h, s));
            rc[c].src = ins.back()->d;
            rc[c].dst = outs.back()->d;
            mw = std::max(mw, rc[c].w);
            mh = std::max(mh, rc[c].h);
            out_w[c] = rc[c].w;
            out_h[c] = rc[c].h;
        }
        DBuf drc = upload(rc, s);
        rectify_launch(drc.as<RectCam>(), ncams, w, h, mw, mh, s);
        for (int c = 0; c < ncams; ++c) outs[c]->finish(s, static_cast<size_t>(rc[c].w) * rc[c].h);
        LPB_CUDA(cudaStreamSynchronize(s));
    });
}

// ---------------------------------------------------------------------------
// Frame ingest / egress formats
namespace lpb {
// pnm_read_token (image.hpp:88-103): skips whitespace and '#' comments
static int pnm_token(std::istream& in) {
    while (in) {
        const int c = in.peek();
        if (c == '#') {
            while (in && in.get() != '\n') {
            }
        } else if (std::isspace(c)) {
            in.get();
        } else {
            break;
        }
    }
    int v = -1;
    in >> v;
    return v;
}

__global__ void k_gray_to_rgb(const uint8_t* __restrict__ g, size_t n, uint8_t* __restrict__ rgb) {
    // 4 gray pixels -> 12 RGB bytes (three 32-bit words) per thread when aligned
    const size_t i4 = (static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 4;
    if (i4 >= n) return;
    if (i4 + 4 <= n && (reinterpret_cast<uintptr_t>(g + i4) & 3) == 0 && (reinterpret_cast<uintptr_t>(rgb + 3 * i4) & 3) == 0) {
        const uint32_t v = *reinterpret_cast<const uint32_t*>(g + i4);
        uint32_t* o = reinterpret_cast<uint32_t*>(rgb + 3 * i4);
        o[0] = __byte_perm(v, 0, 0x1000);  // a a a b
        o[1] = __byte_perm(v, 0, 0x2211);  // b b c c
        o[2] = __byte_perm(v, 0, 0x3332);  // c d d d
    } else {
        for (size_t i = i4; i < n && i < i4 + 4; ++i) rgb[3 * i] = rgb[3 * i + 1] = rgb[3 * i + 2] = g[i];
    }
}
void gray_to_rgb_launch(const uint8_t* g, size_t n, uint8_t* rgb, cudaStream_t s) {
    if (n == 0) return;
    LPB_LAUNCH(k_gray_to_rgb, cdiv(static_cast<long long>((n + 3) / 4), 256), 256, 0, s, g, n, rgb);
}
}  // namespace lpb

extern "C" lp_status lp_brief_pattern(int n_d, int patch_half, uint64_t seed, lp_pair* out) {
    return guard([&] {
        if (n_d < 1 || patch_half < 1) throw Status(LP_BAD_PARAMS, "brief_pattern: bad parameters");
        const auto pat = host::brief_pattern(n_d, patch_half, seed);
        std::memcpy(out, pat.data(), sizeof(lp_pair) * pat.size());
    });
}

extern "C" lp_status lp_load_pnm(const char* path, uint8_t* out, size_t cap, int* w, int* h, int* channels) {
    return guard([&] {
        std::ifstream in(path, std::ios::binary);
        if (!in) throw Status(LP_FILE_NOT_FOUND, std::string(path));
        char p = 0, n = 0;
        in.get(p);
        in.get(n);
        if (p != 'P' || (n != '5' && n != '6'))
            throw Status(LP_UNSUPPORTED_FORMAT, std::string(path) + ": not a binary PGM/PPM");
        const int ch = n == '5' ? 1 : 3;
        const int W = pnm_token(in), H = pnm_token(in), maxval = pnm_token(in);
        if (!in || W < 1 || H < 1) throw Status(LP_CORRUPT_DATA, std::string(path) + ": bad header");
        if (maxval != 255) throw Status(LP_UNSUPPORTED_FORMAT, std::string(path) + ": only maxval 255 supported");
        in.get();  // single whitespace after maxval
        *w = W;
        *h = H;
        *channels = ch;
        const size_t bytes = static_cast<size_t>(W) * H * ch;
        if (!out) return;
        if (cap < bytes) throw Status(LP_CAPACITY_OVERFLOW, std::string(path) + ": output buffer too small");
        in.read(reinterpret_cast<char*>(out), static_cast<std::streamsize>(bytes));
        if (static_cast<size_t>(in.gcount()) != bytes)
            throw Status(LP_CORRUPT_DATA, std::string(path) + ": truncated pixel data");
    });
}

extern "C" lp_status lp_save_pnm(const char* path, const uint8_t* data, int w, int h, int channels) {
    return guard([&] {
        if (channels != 1 && channels != 3)
            throw Status(LP_UNSUPPORTED_FORMAT, std::string(path) + ": only 1- or 3-channel images");
        std::ofstream out(path, std::ios::binary);
        if (!out) throw Status(LP_FILE_NOT_FOUND, std::string(path) + ": cannot open for writing");
        out << (channels == 1 ? "P5\n" : "P6\n") << w << ' ' << h << "\n255\n";
        out.write(reinterpret_cast<const char*>(data), static_cast<std::streamsize>(static_cast<size_t>(w) * h * channels));
        if (!out) throw Status(LP_CORRUPT_DATA, std::string(path) + ": write failed");
    });
}

extern "C" lp_status lp_gray_to_rgb(lp_ctx* ctx, const uint8_t* gray, size_t n, uint8_t* rgb) {
    return guard([&] {
        cudaStream_t s = ctx->stream;
        In<uint8_t> g(gray, n, s);
        Out<uint8_t> o(rgb, 3 * n, s);
        gray_to_rgb_launch(g.d, n, o.d, s);
        o.finish(s, 3 * n);
        LPB_CUDA(cudaStreamSynchronize(s));
    });
}

#include "rig.inc"
