// pipeline.hpp (drop-in) — StitchEngine on the B200 frame engine.
//
// Same public surface as the reference's pipeline.hpp (pipeline.hpp:26-739:
// Stage, FramePacket, BufferPool, PipelineConfig, Metrics, RigLayout,
// StitchParams, HomographyCache, StitchEngine, preallocate), so code written
// against the reference compiles unchanged. What differs is where the frame
// goes:
//
//  * StitchEngine::run() hands every frame to one device rig (lp_rig, the
//    C-ABI's per-frame engine): ingest copy, L-ORB extraction, LSH matching,
//    PROSAC, HomographyCache and the windowed warp / multi-band compositor all
//    run on the GPU, and the packet's keypoints, descriptors, matches,
//    homographies and composite come back with the frame
//    (lp_rig_submit_frame / lp_rig_wait_frame). Pipelined mode runs an ingest
//    thread and an output (sink) thread around a device loop that keeps up to
//    min(frames_in_flight, 3) frames on the device at once (the rig's frame
//    slots) instead of one host thread per stage; Serial runs one frame at a
//    time on the calling thread. Both deliver the same packets in frame
//    order, so composites are byte-identical between the modes as in the
//    reference.
//  * The stage bodies (stage_rectify_crop ... stage_warp_blend) stay callable
//    on their own, as in the reference, and run on the device through the
//    drop-in primitives; stage_describe blurs each region once and describes
//    all of its keypoints in one call (the reference calls brief_descriptor
//    per keypoint, pipeline.hpp:444-469).
//  * Frames the rig cannot take whole (cameras of different sizes after a
//    crop, explicit detection regions, colour input) go through the stage
//    bodies one by one, with the reference's per-stage failure handling.
//
// Metrics: Ingest and Output are host wall time as in the reference; the
// device stages report device time (CUDA events around the stage's work on
// the rig's streams; detect and describe are one fused launch sequence and
// are reported together under Detect).
#ifndef LORBPANO_PIPELINE_HPP
#define LORBPANO_PIPELINE_HPP

#include <algorithm>
#include <array>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdint>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <deque>
#include <functional>
#include <memory>
#include <mutex>
#include <optional>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "lorbpano/b200_runtime.hpp"
#include "lorbpano/compose.hpp"
#include "lorbpano/homography.hpp"
#include "lorbpano/lorb.hpp"
#include "lorbpano/matchlsh.hpp"

namespace lorbpano {

enum class Stage { Ingest = 0, RectifyCrop, Detect, Describe, MatchEstimate, WarpBlend, Output };
constexpr int kNumStages = 7;

inline const char* stage_name(Stage s) {
    switch (s) {
        case Stage::Ingest: return "ingest";
        case Stage::RectifyCrop: return "rectify_crop";
        case Stage::Detect: return "detect";
        case Stage::Describe: return "describe";
        case Stage::MatchEstimate: return "match_estimate";
        case Stage::WarpBlend: return "warp_blend";
        case Stage::Output: return "output";
    }
    return "?";
}

struct StageSpan {
    std::int64_t start_ns = 0;
    std::int64_t end_ns = 0;
};

/// One frame's journey (pipeline.hpp:50-65).
struct FramePacket {
    std::uint64_t frame_index = 0;
    std::vector<ImageU8> images;
    std::vector<DetectionRegion> regions;
    std::vector<std::vector<Keypoint>> keypoints;
    std::vector<std::vector<Descriptor>> descriptors;
    std::vector<std::vector<Match>> pair_matches;
    std::vector<Homography> homographies;
    ImageU8 composite;
    std::array<StageSpan, kNumStages> stage_times{};

    bool failed = false;
    Stage fail_stage = Stage::Ingest;
    std::string fail_reason;
};

/// Host packet arenas sized up front (pipeline.hpp:66-195): the same
/// capacity contract, closed-form byte budget and growth accounting.
class BufferPool {
public:
    struct Caps {
        int num_cameras = 2;
        int width = 0, height = 0, channels = 1;
        int top_n = 500;
        int n_d = 256;
        int frames_in_flight = 1;
        std::size_t memory_cap_bytes = std::size_t{4} << 30;
    };

    explicit BufferPool(const Caps& caps) : caps_(caps) {
        const bool valid = caps.width >= 1 && caps.height >= 1 && caps.num_cameras >= 1 &&
                           caps.frames_in_flight >= 1 && (caps.channels == 1 || caps.channels == 3);
        if (!valid) throw CapacityOverflow("buffer pool: invalid capacity parameters");
        if (byte_budget() > caps.memory_cap_bytes) throw CapacityOverflow("buffer pool: byte budget exceeds memory cap");
        idle_.reserve(caps.frames_in_flight);
        while (static_cast<int>(idle_.size()) < caps.frames_in_flight) {
            idle_.push_back(fresh_packet());
            ++creations_;
        }
    }

    /// per packet: camera images, keypoints and descriptors (2 regions per
    /// camera), matches per adjacent pair, and a cams*w x 2h canvas; times
    /// frames_in_flight
    std::size_t byte_budget() const {
        const std::size_t cams = static_cast<std::size_t>(caps_.num_cameras);
        const std::size_t pairs = caps_.num_cameras > 1 ? cams - 1 : 0;
        const std::size_t px = static_cast<std::size_t>(caps_.width) * caps_.height * caps_.channels;
        const std::size_t feats = cams * 2 * static_cast<std::size_t>(caps_.top_n);
        const std::size_t per_packet = cams * px + feats * sizeof(Keypoint) +
                                       feats * 2 * (static_cast<std::size_t>(caps_.n_d) / 8) +
                                       pairs * caps_.top_n * sizeof(Match) + cams * 2 * px;
        return per_packet * caps_.frames_in_flight;
    }

    std::unique_ptr<FramePacket> acquire() {
        std::unique_lock<std::mutex> lock(mu_);
        freed_.wait(lock, [&] { return !idle_.empty(); });
        std::unique_ptr<FramePacket> p = std::move(idle_.back());
        idle_.pop_back();
        ++acquires_;
        high_water_ = std::max(high_water_, ++busy_);
        return p;
    }

    void release(std::unique_ptr<FramePacket> pkt) {
        recycle(*pkt);
        {
            std::lock_guard<std::mutex> lock(mu_);
            idle_.push_back(std::move(pkt));
            --busy_;
        }
        freed_.notify_one();
    }

    std::uint64_t arena_creations() const { return creations_; }
    std::uint64_t acquires() const { return acquires_; }
    int high_water() const { return high_water_; }
    int capacity() const { return caps_.frames_in_flight; }

private:
    std::unique_ptr<FramePacket> fresh_packet() {
        auto p = std::make_unique<FramePacket>();
        const std::size_t cams = static_cast<std::size_t>(caps_.num_cameras);
        const std::size_t px = static_cast<std::size_t>(caps_.width) * caps_.height * caps_.channels;
        p->images.resize(cams);
        for (ImageU8& im : p->images) im.data.reserve(px);
        p->keypoints.resize(cams);
        p->descriptors.resize(cams);
        for (std::size_t c = 0; c < cams; ++c) {
            p->keypoints[c].reserve(2 * static_cast<std::size_t>(caps_.top_n));
            p->descriptors[c].reserve(2 * static_cast<std::size_t>(caps_.top_n));
        }
        p->pair_matches.resize(cams > 1 ? cams - 1 : 0);
        for (auto& m : p->pair_matches) m.reserve(caps_.top_n);
        p->homographies.reserve(cams);
        p->composite.data.reserve(cams * 2 * px);
        remember_reservations(*p);
        return p;
    }

    void remember_reservations(const FramePacket& p) {
        reserved_.clear();
        for (const ImageU8& im : p.images) reserved_.push_back(im.data.capacity());
        reserved_.push_back(p.composite.data.capacity());
    }

    /// per-frame state cleared; an arena that outgrew its reservation is a
    /// creation event (steady state must have none)
    void recycle(FramePacket& p) {
        bool grew = p.composite.data.capacity() > reserved_.back();
        for (std::size_t i = 0; i < p.images.size() && i + 1 < reserved_.size(); ++i)
            grew = grew || p.images[i].data.capacity() > reserved_[i];
        if (grew) {
            ++creations_;
            remember_reservations(p);
        }
        for (auto& v : p.keypoints) v.clear();
        for (auto& v : p.descriptors) v.clear();
        for (auto& v : p.pair_matches) v.clear();
        p.regions.clear();
        p.homographies.clear();
        p.failed = false;
        p.fail_reason.clear();
        p.stage_times = {};
    }

    Caps caps_;
    std::mutex mu_;
    std::condition_variable freed_;
    std::vector<std::unique_ptr<FramePacket>> idle_;
    std::vector<std::size_t> reserved_;
    std::atomic<std::uint64_t> creations_{0};
    std::atomic<std::uint64_t> acquires_{0};
    int busy_ = 0;
    int high_water_ = 0;
};

enum class PipelineMode { Serial, Pipelined };

struct PipelineConfig {
    PipelineMode mode = PipelineMode::Pipelined;
    int frames_in_flight = 4;
    int workers_per_stage = 1;   // host threads per stage in the reference; unused by the device engine
    int homography_refresh = 1;  // recompute every K frames
};

struct DroppedFrame {
    std::uint64_t frame_index;
    Stage stage;
    std::string reason;
};

struct Metrics {
    std::array<std::vector<double>, kNumStages> stage_ns;
    std::vector<DroppedFrame> drops;
    std::uint64_t frames_in = 0;
    std::uint64_t frames_out = 0;
    double wall_seconds = 0.0;
    double frames_per_second = 0.0;
    std::uint64_t pool_creations = 0;
    std::uint64_t pool_creations_after_warmup = 0;
    int pool_high_water = 0;

    struct Summary {
        double mean = 0, p50 = 0, p99 = 0;
    };
    Summary stage_summary(Stage s) const {
        Summary r;
        std::vector<double> v = stage_ns[static_cast<int>(s)];
        if (v.empty()) return r;
        std::sort(v.begin(), v.end());
        double total = 0;
        for (double x : v) total += x;
        r.mean = total / static_cast<double>(v.size());
        r.p50 = v[v.size() / 2];
        r.p99 = v[std::min(v.size() - 1, v.size() * 99 / 100)];
        return r;
    }
};

/// Per-camera pre-correction and the overlap declaration (pipeline.hpp:240-247).
struct RigLayout {
    struct Camera {
        Homography pre_transform = Homography::identity();
        std::optional<DetectionRegion> crop;
    };
    std::vector<Camera> cameras;
    CameraLayout overlap;
};

struct StitchParams {
    ExtractionConfig extraction;
    MatchConfig matching;
    ProsacConfig prosac;
    int blend_levels = 4;
    std::uint64_t seed = 0;
};

class StitchEngine;

/// Last estimated homography set between refreshes (pipeline.hpp:259-286).
/// In run() the device rig applies the same rule; the engine mirrors its
/// verdicts here so estimations() counts them.
class HomographyCache {
public:
    explicit HomographyCache(int refresh_every) : k_(refresh_every) {
        if (k_ < 1) throw BadParams("homography cache: K must be >= 1");
    }

    std::vector<Homography> get(std::uint64_t frame_index, const std::function<std::vector<Homography>()>& estimator) {
        const bool due = !cached_ || frame_index % static_cast<std::uint64_t>(k_) == 0;
        if (due) {
            try {
                cached_ = estimator();
                ++estimations_;
            } catch (const Error&) {
                if (!cached_) throw NoValidHomographyYet("no homography cached yet");
            }
        }
        return *cached_;
    }

    std::uint64_t estimations() const { return estimations_; }

private:
    friend class StitchEngine;
    void record_device_estimate(const std::vector<Homography>& hs) {
        cached_ = hs;
        ++estimations_;
    }

    int k_;
    std::optional<std::vector<Homography>> cached_;
    std::uint64_t estimations_ = 0;
};

using FrameSource = std::function<std::optional<std::vector<ImageU8>>()>;
using FrameSink = std::function<void(const FramePacket&)>;

namespace detail {

// Device rigs of finished engines, kept for the next engine of the same
// layout, frame size and parameters (a rig does not depend on the context
// it was created through, and serves one engine at a time): creating
// one (device arenas, pinned staging, textures, graphs) costs 5-300 ms,
// which an engine of a few hundred small frames would otherwise spend
// mostly there. A taken rig is reset to an empty HomographyCache
// (lp_rig_reset), so nothing of the previous engine's state carries over.
// Two idle rigs at most; the pool itself is never destroyed (rigs left in it
// at process exit go with the process).
class RigPool {
public:
    lp_rig* take(int ncams, int w, int h, const lp_params& p) {
        std::lock_guard<std::mutex> l(mu_);
        for (std::size_t i = 0; i < idle_.size(); ++i) {
            const Entry& e = idle_[i];
            if (e.ncams == ncams && e.w == w && e.h == h && std::memcmp(&e.p, &p, sizeof p) == 0) {
                lp_rig* r = e.rig;
                idle_.erase(idle_.begin() + static_cast<std::ptrdiff_t>(i));
                if (lp_rig_reset(r) == LP_OK) return r;
                lp_rig_destroy(r);
                return nullptr;
            }
        }
        return nullptr;
    }
    void give(lp_rig* r, int ncams, int w, int h, const lp_params& p) {
        std::lock_guard<std::mutex> l(mu_);
        if (idle_.size() >= 2) {
            lp_rig_destroy(idle_.front().rig);
            idle_.erase(idle_.begin());
        }
        idle_.push_back(Entry{r, ncams, w, h, p});
    }

private:
    struct Entry {
        lp_rig* rig;
        int ncams, w, h;
        lp_params p;
    };
    std::mutex mu_;
    std::vector<Entry> idle_;
};
inline RigPool& rig_pool() {
    static RigPool* pool = new RigPool;  // outlives every engine, including static ones
    return *pool;
}
// A bounded FIFO between the engine's threads; close() releases the waiters.
template <class T>
class Channel {
public:
    explicit Channel(std::size_t cap) : cap_(std::max<std::size_t>(cap, 1)) {}
    void put(T v) {
        std::unique_lock<std::mutex> l(mu_);
        room_.wait(l, [&] { return q_.size() < cap_ || shut_; });
        q_.push_back(std::move(v));
        ready_.notify_one();
    }
    std::optional<T> take() {
        std::unique_lock<std::mutex> l(mu_);
        ready_.wait(l, [&] { return !q_.empty() || shut_; });
        if (q_.empty()) return std::nullopt;
        T v = std::move(q_.front());
        q_.pop_front();
        room_.notify_one();
        return v;
    }
    void close() {
        std::lock_guard<std::mutex> l(mu_);
        shut_ = true;
        ready_.notify_all();
        room_.notify_all();
    }

private:
    std::size_t cap_;
    std::deque<T> q_;
    bool shut_ = false;
    std::mutex mu_;
    std::condition_variable ready_, room_;
};

inline std::int64_t now_ns() {
    return std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now().time_since_epoch())
        .count();
}
}  // namespace detail

class StitchEngine {
public:
    StitchEngine(RigLayout layout, StitchParams params, PipelineConfig cfg)
        : layout_(std::move(layout)),
          params_(std::move(params)),
          cfg_(cfg),
          pattern_(brief_pattern(params_.extraction.n_d, params_.extraction.patch_half, params_.seed)),
          cache_(cfg.homography_refresh) {
        params_.extraction.validate();
        if (layout_.cameras.empty()) throw BadParams("stitch engine: no cameras");
    }
    ~StitchEngine() { drop_rig(); }
    StitchEngine(const StitchEngine&) = delete;
    StitchEngine& operator=(const StitchEngine&) = delete;

    BufferPool& make_pool(int width, int height, int channels) {
        BufferPool::Caps caps;
        caps.num_cameras = static_cast<int>(layout_.cameras.size());
        caps.width = width;
        caps.height = height;
        caps.channels = channels;
        caps.top_n = params_.extraction.top_n;
        caps.n_d = params_.extraction.n_d;
        caps.frames_in_flight = cfg_.mode == PipelineMode::Serial ? 1 : cfg_.frames_in_flight;
        pool_ = std::make_unique<BufferPool>(caps);
        return *pool_;
    }

    const BriefPattern& pattern() const { return pattern_; }
    const HomographyCache& homography_cache() const { return cache_; }

    Metrics run(const FrameSource& source, const FrameSink& sink) {
        Metrics m;
        const auto start = std::chrono::steady_clock::now();
        // LPB_ENGINE_THREADS=0: Pipelined without the ingest / sink threads
        // (A/B experiments; the default is the measured best)
        const char* thr = std::getenv("LPB_ENGINE_THREADS");
        if (cfg_.mode == PipelineMode::Serial)
            run_serial(source, sink, m, 1);
        else if (thr && thr[0] == '0')
            run_serial(source, sink, m, device_depth());
        else
            run_pipelined(source, sink, m);
        m.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - start).count();
        if (std::getenv("LPB_ENGINE_PROFILE"))  // host time per frame in the engine's own steps
            std::fprintf(stderr, "engine rig creation %.3f ms; host ms/frame: launch %.4f (regions %.4f staging %.4f submit %.4f) wait %.4f fill %.4f over %llu frames\n",
                         prof_[6] / 1e6,
                         prof_[0] / 1e6 / std::max<std::uint64_t>(m.frames_out, 1),
                         prof_[4] / 1e6 / std::max<std::uint64_t>(m.frames_out, 1),
                         prof_[5] / 1e6 / std::max<std::uint64_t>(m.frames_out, 1),
                         prof_[1] / 1e6 / std::max<std::uint64_t>(m.frames_out, 1),
                         prof_[2] / 1e6 / std::max<std::uint64_t>(m.frames_out, 1),
                         prof_[3] / 1e6 / std::max<std::uint64_t>(m.frames_out, 1),
                         static_cast<unsigned long long>(m.frames_out));
        m.frames_per_second = m.wall_seconds > 0 ? m.frames_out / m.wall_seconds : 0.0;
        if (pool_) {
            m.pool_creations = pool_->arena_creations();
            m.pool_creations_after_warmup = pool_->arena_creations() - warmup_creations_;
            m.pool_high_water = pool_->high_water();
        }
        return m;
    }

    // --- stage bodies, usable directly (the same contracts as the reference's) ---

    /// pipeline.hpp:391-417 on the device (lp_rectify_crop), then the regions
    void stage_rectify_crop(FramePacket& pkt) const {
        std::vector<std::pair<int, int>> dims;
        for (std::size_t c = 0; c < pkt.images.size(); ++c) {
            const RigLayout::Camera& cam = layout_.cameras[c];
            ImageU8& img = pkt.images[c];
            const bool identity = cam.pre_transform.h == Homography::identity().h;
            if (!identity || cam.crop) {
                if (img.channels != 1) {
                    rectify_colour(cam, img);
                } else {
                    lp_camera lc{};
                    std::memcpy(lc.pre_transform.h, cam.pre_transform.h.data(), sizeof lc.pre_transform.h);
                    if (cam.crop) {
                        lc.has_crop = 1;
                        lc.crop = b200::region(*cam.crop);
                    }
                    ImageU8 out(img.width, img.height, 1, img.color_space);
                    const std::uint8_t* in = img.data.data();
                    std::uint8_t* o = out.data.data();
                    int ow = 0, oh = 0;
                    b200::check(lp_rectify_crop(b200::ctx(), 1, img.width, img.height, &lc, &in, &o, &ow, &oh));
                    out.width = ow;
                    out.height = oh;
                    out.data.resize(static_cast<std::size_t>(ow) * oh);
                    img = std::move(out);
                }
            }
            dims.emplace_back(img.width, img.height);
        }
        pkt.regions = partition_regions(layout_.overlap, dims, params_.extraction.patch_half);
    }

    /// pipeline.hpp:419-442: per camera, FAST -> Harris -> NMS -> top-N of
    /// each of its regions (one device extraction pass per camera)
    void stage_detect(FramePacket& pkt) const {
        for (int c = 0; c < static_cast<int>(pkt.images.size()); ++c) {
            std::vector<int> global;
            const std::vector<DetectionRegion> mine = regions_of(pkt, c, global);
            if (mine.empty()) continue;
            for (const Feature& f : extract_features(pkt.images[c], mine, params_.extraction, pattern_)) {
                Keypoint k = f.keypoint;
                k.region_id = global[k.region_id];
                pkt.keypoints[c].push_back(k);
            }
        }
    }

    /// pipeline.hpp:444-469: one smoothed crop per region, all of the
    /// region's keypoints described by one device call
    void stage_describe(FramePacket& pkt) const {
        const int n_d = params_.extraction.n_d, W2 = 2 * Descriptor::words(n_d);
        for (int c = 0; c < static_cast<int>(pkt.images.size()); ++c) {
            const std::vector<Keypoint>& kps = pkt.keypoints[c];
            pkt.descriptors[c].assign(kps.size(), Descriptor(n_d));
            for (int ri = 0; ri < static_cast<int>(pkt.regions.size()); ++ri) {
                if (pkt.regions[ri].camera_id != c) continue;
                std::vector<std::size_t> idx;
                for (std::size_t i = 0; i < kps.size(); ++i)
                    if (kps[i].region_id == ri) idx.push_back(i);
                if (idx.empty()) continue;
                const detail::SmoothedCrop crop =
                    detail::smoothed_crop(pkt.images[c], pkt.regions[ri], params_.extraction.patch_half,
                                          params_.extraction.brief_blur_sigma);
                std::vector<lp_keypoint> local(idx.size());
                for (std::size_t j = 0; j < idx.size(); ++j) {
                    const Keypoint& k = kps[idx[j]];
                    local[j] = lp_keypoint{k.x - crop.off_x, k.y - crop.off_y, k.response, k.region_id};
                }
                std::vector<std::uint64_t> words(idx.size() * W2);
                b200::check(lp_brief_descriptors(b200::ctx(), crop.img.data.data(), crop.img.width, crop.img.height,
                                                 local.data(), static_cast<int>(local.size()),
                                                 reinterpret_cast<const lp_pair*>(pattern_.pairs.data()), n_d,
                                                 pattern_.patch_half, words.data()));
                for (std::size_t j = 0; j < idx.size(); ++j)
                    pkt.descriptors[c][idx[j]] = b200::unpack(words.data() + j * W2, n_d);
            }
        }
    }

    /// pipeline.hpp:471-497: match + PROSAC per adjacent pair behind the cache
    void stage_match_estimate(FramePacket& pkt) {
        auto estimate = [&]() -> std::vector<Homography> {
            std::vector<Homography> chain{Homography::identity()};
            for (int i = 0; i + 1 < static_cast<int>(pkt.images.size()); ++i) {
                std::vector<Match> ms = match_features(pkt.descriptors[i + 1], pkt.descriptors[i], params_.matching);
                pkt.pair_matches[i] = ms;
                std::vector<Correspondence> corr;
                corr.reserve(ms.size());
                for (const Match& m : ms) {
                    const Keypoint& a = pkt.keypoints[i + 1][m.query_id];
                    const Keypoint& b = pkt.keypoints[i][m.train_id];
                    corr.push_back(Correspondence{double(a.x), double(a.y), double(b.x), double(b.y), m.quality});
                }
                ProsacConfig pc = params_.prosac;
                pc.seed = params_.seed ^ (pkt.frame_index * 0x9e3779b97f4a7c15ULL + static_cast<std::uint64_t>(i));
                chain.push_back(chain.back().compose(prosac_homography(corr, pc).model));
            }
            return chain;
        };
        pkt.homographies = cache_.get(pkt.frame_index, estimate);
    }

    /// pipeline.hpp:499-521 with the drop-in device compositor primitives
    void stage_warp_blend(FramePacket& pkt) const {
        std::vector<std::pair<int, int>> dims;
        for (const ImageU8& im : pkt.images) dims.emplace_back(im.width, im.height);
        const Canvas canvas = compute_canvas(dims, pkt.homographies);
        std::vector<ImageF32> warped, coverage;
        for (std::size_t c = 0; c < pkt.images.size(); ++c) {
            auto wc = warp_image(to_f32(pkt.images[c]), pkt.homographies[c], canvas);
            warped.push_back(std::move(wc.first));
            coverage.push_back(std::move(wc.second));
        }
        const std::vector<BlendMask> masks = linear_seam_mask(coverage);
        const ImageU8 out = multiband_blend(warped, masks, levels_for(canvas.width, canvas.height));
        pkt.composite.width = out.width;
        pkt.composite.height = out.height;
        pkt.composite.channels = out.channels;
        pkt.composite.color_space = out.color_space;
        pkt.composite.data.assign(out.data.begin(), out.data.end());
    }

private:
    // Page-locked host staging (lp_host_alloc): frames move to and from the
    // device by DMA, so the host never blocks on a copy while frames are in flight.
    struct Pinned {
        void* p = nullptr;
        std::size_t n = 0;
        Pinned() = default;
        Pinned(const Pinned&) = delete;
        Pinned& operator=(const Pinned&) = delete;
        ~Pinned() { lp_host_free(p); }
        template <class T>
        T* get(std::size_t count) {
            const std::size_t bytes = count * sizeof(T);
            if (bytes > n) {
                lp_host_free(p);
                p = lp_host_alloc(bytes);
                if (!p) throw CapacityOverflow("stitch engine: page-locked host staging unavailable");
                n = bytes;
            }
            return static_cast<T*>(p);
        }
    };

    // A frame on the device: its packet and the rig's result arrays (one of
    // three reusable slots, as the rig has three frame slots).
    struct Flight {
        std::unique_ptr<FramePacket> pkt;
        std::uint64_t ticket = 0;
        std::int64_t t_submit = 0;
        lp_frame_out out{};
        Pinned frames, pano, homs, counts, kps, desc, matches;
    };

    int levels_for(int w, int h) const {
        int levels = params_.blend_levels;
        while (levels > 1 && (w < (1 << (levels - 1)) || h < (1 << (levels - 1)))) --levels;
        return levels;
    }

    std::vector<DetectionRegion> regions_of(const FramePacket& pkt, int cam, std::vector<int>& global) const {
        std::vector<DetectionRegion> mine;
        for (int ri = 0; ri < static_cast<int>(pkt.regions.size()); ++ri)
            if (pkt.regions[ri].camera_id == cam) {
                mine.push_back(pkt.regions[ri]);
                global.push_back(ri);
            }
        return mine;
    }

    // colour frames: the reference's rectify on the host-visible drop-in warp
    static void rectify_colour(const RigLayout::Camera& cam, ImageU8& img) {
        if (!(cam.pre_transform.h == Homography::identity().h)) {
            const Canvas self{img.width, img.height, 0, 0, {}};
            img = to_u8_image(warp_image(to_f32(img), cam.pre_transform, self).first);
        }
        if (cam.crop) {
            const DetectionRegion& r = *cam.crop;
            if (r.x0 < 0 || r.y0 < 0 || r.x1 > img.width || r.y1 > img.height || r.width() < 1 || r.height() < 1)
                throw BadParams("rectify_crop: crop outside image");
            ImageU8 out(r.width(), r.height(), img.channels, img.color_space);
            const std::size_t row = static_cast<std::size_t>(r.width()) * img.channels;
            for (int y = 0; y < r.height(); ++y)
                std::memcpy(out.data.data() + y * row,
                            img.data.data() + (static_cast<std::size_t>(r.y0 + y) * img.width + r.x0) * img.channels, row);
            img = std::move(out);
        }
    }

    bool layout_is_identity() const {
        for (const RigLayout::Camera& c : layout_.cameras)
            if (c.crop || !(c.pre_transform.h == Homography::identity().h)) return false;
        return true;
    }

    // which stage a device-engine failure belongs to (the exception the
    // reference's stage body would have thrown, pipeline.hpp:539-575)
    static Stage stage_of(lp_status st) {
        switch (st) {
            case LP_REGION_TOO_SMALL:
            case LP_WINDOW_OUT_OF_BOUNDS:
            case LP_UNSUPPORTED_FORMAT:
            case LP_IMAGE_TOO_SMALL:
            case LP_NO_OVERLAP:
            case LP_OVERLAP_EXCEEDS_IMAGE:
                return Stage::Detect;
            case LP_PATCH_OUT_OF_BOUNDS:
                return Stage::Describe;
            case LP_NO_VALID_HOMOGRAPHY_YET:
            case LP_INSUFFICIENT_MATCHES:
            case LP_NO_MODEL_FOUND:
            case LP_DEGENERATE_CONFIGURATION:
            case LP_NUMERICAL_FAILURE:
                return Stage::MatchEstimate;
            default:
                return Stage::WarpBlend;
        }
    }

    void note_drop(FramePacket& pkt, Stage s, const std::string& why, Metrics& m) {
        pkt.failed = true;
        pkt.fail_stage = s;
        pkt.fail_reason = why;
        std::lock_guard<std::mutex> l(metrics_mu_);
        m.drops.push_back(DroppedFrame{pkt.frame_index, s, why});
    }
    // the engine's threads share one Metrics
    void note_stage(Metrics& m, Stage s, double ns) {
        std::lock_guard<std::mutex> l(metrics_mu_);
        m.stage_ns[static_cast<int>(s)].push_back(ns);
    }

    void note_warmup(std::uint64_t started) {
        if (!warmup_noted_ && pool_ && started >= static_cast<std::uint64_t>(pool_->capacity())) {
            warmup_creations_ = pool_->arena_creations();
            warmup_noted_ = true;
        }
    }

    std::unique_ptr<FramePacket> ingest(const FrameSource& source, std::uint64_t index, Metrics& m) {
        std::optional<std::vector<ImageU8>> frame = source();
        if (!frame) return nullptr;
        if (!pool_) {
            if (frame->empty()) throw BadParams("pipeline: empty camera set");
            const ImageU8& f0 = frame->front();
            make_pool(f0.width, f0.height, f0.channels);
        }
        std::unique_ptr<FramePacket> pkt = pool_->acquire();
        pkt->frame_index = index;
        StageSpan& span = pkt->stage_times[static_cast<int>(Stage::Ingest)];
        span.start_ns = detail::now_ns();
        pkt->images.resize(frame->size());
        for (std::size_t c = 0; c < frame->size(); ++c) {
            const ImageU8& src = (*frame)[c];
            ImageU8& dst = pkt->images[c];
            dst.width = src.width;
            dst.height = src.height;
            dst.channels = src.channels;
            dst.color_space = src.color_space;
            dst.data.assign(src.data.begin(), src.data.end());
        }
        span.end_ns = detail::now_ns();
        note_stage(m, Stage::Ingest, static_cast<double>(span.end_ns - span.start_ns));
        {
            std::lock_guard<std::mutex> l(metrics_mu_);
            ++m.frames_in;
        }
        return pkt;
    }

    // one stage body with the reference's drop semantics (pipeline.hpp:539-575)
    template <class F>
    bool timed_stage(FramePacket& pkt, Stage s, Metrics& m, F&& body) {
        if (pkt.failed) return false;
        StageSpan& span = pkt.stage_times[static_cast<int>(s)];
        span.start_ns = detail::now_ns();
        try {
            body();
        } catch (const std::exception& e) {
            span.end_ns = detail::now_ns();
            note_drop(pkt, s, e.what(), m);
            return false;
        }
        span.end_ns = detail::now_ns();
        note_stage(m, s, static_cast<double>(span.end_ns - span.start_ns));
        return true;
    }

    void deliver(std::unique_ptr<FramePacket> pkt, Metrics& m, const FrameSink& sink) {
        StageSpan& span = pkt->stage_times[static_cast<int>(Stage::Output)];
        span.start_ns = detail::now_ns();
        if (!pkt->failed) {
            sink(*pkt);
            span.end_ns = detail::now_ns();
            note_stage(m, Stage::Output, static_cast<double>(span.end_ns - span.start_ns));
            std::lock_guard<std::mutex> l(metrics_mu_);
            ++m.frames_out;
        }
        pool_->release(std::move(pkt));
    }

    // the whole frame through the stage bodies (frames the rig cannot take)
    void run_stage_bodies(FramePacket& pkt, Metrics& m) {
        timed_stage(pkt, Stage::Detect, m, [&] { stage_detect(pkt); }) &&
            timed_stage(pkt, Stage::Describe, m, [&] { stage_describe(pkt); }) &&
            timed_stage(pkt, Stage::MatchEstimate, m, [&] { stage_match_estimate(pkt); }) &&
            timed_stage(pkt, Stage::WarpBlend, m, [&] { stage_warp_blend(pkt); });
    }

    bool rig_fits(const FramePacket& pkt) const {
        if (!layout_.overlap.explicit_regions.empty() || pkt.images.size() != layout_.cameras.size()) return false;
        for (const ImageU8& im : pkt.images)
            if (im.channels != 1 || im.width != pkt.images[0].width || im.height != pkt.images[0].height) return false;
        return true;
    }

    void drop_rig() {
        if (rig_) detail::rig_pool().give(rig_, rig_cams_, rig_w_, rig_h_, rig_params_);
        rig_ = nullptr;
    }

    void ensure_rig(int ncams, int w, int h) {
        if (rig_ && rig_cams_ == ncams && rig_w_ == w && rig_h_ == h) return;
        drop_rig();
        lp_params p{};
        p.extraction = b200::config(params_.extraction);
        const MatchConfig& mc = params_.matching;
        p.matching = lp_match_config{mc.tables, mc.bits, mc.t_probes, mc.max_distance, mc.ratio, 0, mc.seed};
        const ProsacConfig& pc = params_.prosac;
        p.prosac = lp_prosac_config{pc.threshold_px, pc.max_iter, pc.sampling == SamplingMode::Uniform ? 1 : 0,
                                    pc.confidence, pc.seed, pc.t_total};
        p.blend_levels = params_.blend_levels;
        p.homography_refresh = cfg_.homography_refresh;
        p.seed = params_.seed;
        p.overlap_fraction = layout_.overlap.overlap_fraction;
        const std::int64_t t0 = detail::now_ns();
        rig_ = detail::rig_pool().take(ncams, w, h, p);
        if (!rig_) b200::check(lp_rig_create(b200::ctx(), ncams, w, h, &p, &rig_));
        prof_[6] += detail::now_ns() - t0;
        rig_params_ = p;
        rig_cams_ = ncams;
        rig_w_ = w;
        rig_h_ = h;
    }

    // rectify/crop + regions on the host-visible path, then the frame to the
    // device rig; a frame the rig cannot take runs the stage bodies here
    // frames on the device at once: the rig has 3 frame slots; one pool
    // packet stays free for the host stages (LPB_ENGINE_DEPTH overrides)
    std::size_t device_depth() const {
        int d = std::min(cfg_.frames_in_flight - 1, 3);
        if (const char* e = std::getenv("LPB_ENGINE_DEPTH")) d = std::atoi(e);
        return static_cast<std::size_t>(std::clamp(d, 1, 3));
    }

    // the calling thread alone: ingest, device (up to `depth` frames in
    // flight), sink; Serial mode is depth 1
    void run_serial(const FrameSource& source, const FrameSink& sink, Metrics& m, std::size_t depth) {
        std::deque<Flight*> inflight;
        std::uint64_t launched = 0;
        for (std::uint64_t index = 0;; ++index) {
            std::unique_ptr<FramePacket> pkt = ingest(source, index, m);
            if (!pkt) break;
            note_warmup(index + 1);
            Flight& f = flights_[launched++ % flights_.size()];
            launch(f, std::move(pkt), m);
            inflight.push_back(&f);
            while (inflight.size() >= depth) {
                deliver(land(*inflight.front(), m), m, sink);
                inflight.pop_front();
            }
        }
        for (Flight* f : inflight) deliver(land(*f, m), m, sink);
    }

    // Pipelined (pipeline.hpp:660-711 as threads + device slots): an ingest
    // thread pulls frames into pooled packets, the calling thread keeps up to
    // min(frames_in_flight, 3) of them on the device, an output thread runs
    // the sink; frames leave in order
    void run_pipelined(const FrameSource& source, const FrameSink& sink, Metrics& m) {
        const std::size_t depth = device_depth();
        const std::size_t qcap = static_cast<std::size_t>(std::max(cfg_.frames_in_flight, 1));
        detail::Channel<std::unique_ptr<FramePacket>> in(qcap), out(qcap);
        std::exception_ptr ingest_error, sink_error;
        std::thread ingest_thread([&] {
            try {
                for (std::uint64_t index = 0;; ++index) {
                    std::unique_ptr<FramePacket> pkt = ingest(source, index, m);
                    if (!pkt) break;
                    note_warmup(index + 1);
                    in.put(std::move(pkt));
                }
            } catch (...) {
                ingest_error = std::current_exception();
            }
            in.close();
        });
        std::thread output_thread([&] {
            for (;;) {
                std::optional<std::unique_ptr<FramePacket>> pkt = out.take();
                if (!pkt) break;
                if (sink_error) {  // keep draining so the packets return to the pool
                    pool_->release(std::move(*pkt));
                    continue;
                }
                try {
                    deliver(std::move(*pkt), m, sink);
                } catch (...) {
                    sink_error = std::current_exception();
                }
            }
        });
        std::deque<Flight*> inflight;
        std::uint64_t launched = 0;
        for (;;) {
            std::optional<std::unique_ptr<FramePacket>> pkt = in.take();
            if (!pkt) break;
            Flight& f = flights_[launched++ % flights_.size()];
            launch(f, std::move(*pkt), m);
            inflight.push_back(&f);
            while (inflight.size() >= depth) {
                out.put(land(*inflight.front(), m));
                inflight.pop_front();
            }
        }
        while (!inflight.empty()) {
            out.put(land(*inflight.front(), m));
            inflight.pop_front();
        }
        out.close();
        ingest_thread.join();
        output_thread.join();
        if (ingest_error) std::rethrow_exception(ingest_error);
        if (sink_error) std::rethrow_exception(sink_error);
    }

    void launch(Flight& f, std::unique_ptr<FramePacket> pkt, Metrics& m) {
        const std::int64_t t_launch = detail::now_ns();
        struct Acc {
            std::int64_t& s;
            std::int64_t t0;
            ~Acc() { s += detail::now_ns() - t0; }
        } acc{prof_[0], t_launch};
        FramePacket& p = *pkt;
        f.pkt = std::move(pkt);
        f.ticket = 0;
        const std::int64_t t_rect = detail::now_ns();
        const bool rectified = timed_stage(p, Stage::RectifyCrop, m, [&] {
            if (layout_is_identity()) {
                std::vector<std::pair<int, int>> dims;
                for (const ImageU8& im : p.images) dims.emplace_back(im.width, im.height);
                p.regions = partition_regions(layout_.overlap, dims, params_.extraction.patch_half);
            } else {
                stage_rectify_crop(p);
            }
        });
        prof_[4] += detail::now_ns() - t_rect;
        if (!rectified) return;
        if (!rig_fits(p)) {
            run_stage_bodies(p, m);
            return;
        }
        const int ncams = static_cast<int>(p.images.size()), w = p.images[0].width, h = p.images[0].height;
        try {
            ensure_rig(ncams, w, h);
            const int cap_kp = 2 * params_.extraction.top_n, W2 = 2 * Descriptor::words(params_.extraction.n_d);
            const std::size_t np = static_cast<std::size_t>(std::max(ncams - 1, 1));
            const std::size_t fb = static_cast<std::size_t>(w) * h;
            lp_frame_out& o = f.out;
            o = lp_frame_out{};
            o.pano_cap = lp_rig_panorama_capacity(rig_);
            o.panorama = f.pano.get<std::uint8_t>(o.pano_cap);
            o.homographies = f.homs.get<lp_homography>(ncams);
            int* counts = f.counts.get<int>(ncams + np);
            o.kp_counts = counts;
            o.match_counts = counts + ncams;
            o.keypoints = f.kps.get<lp_keypoint>(static_cast<std::size_t>(ncams) * cap_kp);
            o.descriptors = f.desc.get<std::uint64_t>(static_cast<std::size_t>(ncams) * cap_kp * W2);
            o.cap_kp = cap_kp;
            o.matches = f.matches.get<lp_match>(np * cap_kp);
            o.cap_matches = cap_kp;
            const std::int64_t t_stage = detail::now_ns();
            std::uint8_t* staged = f.frames.get<std::uint8_t>(ncams * fb);
            std::vector<const std::uint8_t*> ims(ncams);
            for (int c = 0; c < ncams; ++c) {
                std::memcpy(staged + c * fb, p.images[c].data.data(), fb);
                ims[c] = staged + c * fb;
            }
            f.t_submit = detail::now_ns();
            prof_[5] += f.t_submit - t_stage;
            const lp_status st = lp_rig_submit_frame(rig_, ims.data(), p.frame_index, &o, &f.ticket);
            prof_[1] += detail::now_ns() - f.t_submit;
            if (st != LP_OK) {
                note_drop(p, stage_of(st), lp_last_error(), m);
                f.ticket = 0;
            }
        } catch (const std::exception& e) {
            note_drop(p, Stage::Detect, e.what(), m);
            f.ticket = 0;
        }
    }

    // the frame back from the device into its packet, then to the sink
    std::unique_ptr<FramePacket> land(Flight& f, Metrics& m) {
        FramePacket& p = *f.pkt;
        if (f.ticket != 0 && !p.failed) {
            const std::int64_t t0 = detail::now_ns();
            lp_status st = lp_rig_wait_frame(rig_, f.ticket, &f.out);
            if (st == LP_CAPACITY_OVERFLOW && f.out.canvas.width > 0 && f.out.canvas.height > 0) {
                // a canvas beyond the staging (the reference's BufferPool
                // grows for it, pipeline.hpp:68-109): grow and fetch it
                const std::size_t need = static_cast<std::size_t>(f.out.canvas.width) * f.out.canvas.height;
                f.out.panorama = f.pano.get<std::uint8_t>(need);
                f.out.pano_cap = need;
                st = lp_rig_copy_panorama(rig_, f.ticket, f.out.panorama, need);
            }
            const std::int64_t t1 = detail::now_ns();
            prof_[2] += t1 - t0;
            if (st != LP_OK) {
                note_drop(p, stage_of(st), lp_last_error(), m);
            } else {
                fill_packet(f, m);
                prof_[3] += detail::now_ns() - t1;
            }
        }
        return std::move(f.pkt);
    }

    void fill_packet(Flight& f, Metrics& m) {
        FramePacket& p = *f.pkt;
        const lp_frame_out& o = f.out;
        const int ncams = static_cast<int>(p.images.size()), n_d = params_.extraction.n_d;
        const int W2 = 2 * Descriptor::words(n_d);
        for (int c = 0; c < ncams; ++c) {
            const int n = std::min(o.kp_counts[c], o.cap_kp);
            const lp_keypoint* k = o.keypoints + static_cast<std::size_t>(c) * o.cap_kp;
            const std::uint64_t* d = o.descriptors + static_cast<std::size_t>(c) * o.cap_kp * W2;
            for (int i = 0; i < n; ++i) {
                p.keypoints[c].push_back(Keypoint{k[i].x, k[i].y, k[i].response, k[i].region_id});
                p.descriptors[c].push_back(b200::unpack(d + static_cast<std::size_t>(i) * W2, n_d));
            }
        }
        if (o.estimated) {
            for (int q = 0; q + 1 < ncams; ++q) {
                const int n = std::min(o.match_counts[q], o.cap_matches);
                const lp_match* mm = o.matches + static_cast<std::size_t>(q) * o.cap_matches;
                for (int i = 0; i < n; ++i)
                    p.pair_matches[q].push_back(Match{mm[i].query_id, mm[i].train_id, mm[i].distance, mm[i].quality});
            }
        }
        p.homographies.clear();
        for (int c = 0; c < ncams; ++c) {
            Homography h;
            std::memcpy(h.h.data(), o.homographies[c].h, sizeof o.homographies[c].h);
            p.homographies.push_back(h);
        }
        if (o.estimated) cache_.record_device_estimate(p.homographies);
        p.composite.width = o.canvas.width;
        p.composite.height = o.canvas.height;
        p.composite.channels = 1;
        p.composite.color_space = ColorSpace::Gray;
        p.composite.data.assign(o.panorama, o.panorama + static_cast<std::size_t>(o.canvas.width) * o.canvas.height);
        // device stage times (detect + describe are one fused sequence)
        const double ms_to_ns = 1e6;
        const double dev[4] = {o.stage_ms[0], 0.0, o.stage_ms[2], o.stage_ms[3]};
        const Stage stages[4] = {Stage::Detect, Stage::Describe, Stage::MatchEstimate, Stage::WarpBlend};
        std::int64_t t = f.t_submit;
        for (int i = 0; i < 4; ++i) {
            StageSpan& span = p.stage_times[static_cast<int>(stages[i])];
            span.start_ns = t;
            t += static_cast<std::int64_t>(dev[i] * ms_to_ns);
            span.end_ns = t;
            note_stage(m, stages[i], dev[i] * ms_to_ns);
        }
    }

    RigLayout layout_;
    StitchParams params_;
    PipelineConfig cfg_;
    BriefPattern pattern_;
    HomographyCache cache_;
    std::unique_ptr<BufferPool> pool_;
    std::uint64_t warmup_creations_ = 0;
    bool warmup_noted_ = false;
    lp_rig* rig_ = nullptr;
    int rig_cams_ = 0, rig_w_ = 0, rig_h_ = 0;
    lp_params rig_params_{};
    std::array<Flight, 3> flights_;
    std::mutex metrics_mu_;
    std::int64_t prof_[7] = {};  // host ns: launch, submit call, wait call, fill, rectify/regions, staging (LPB_ENGINE_PROFILE)
};

/// A pool sized for `frames_in_flight` packets (pipeline.hpp:724-735).
inline BufferPool preallocate(const PipelineConfig& cfg, int width, int height, int channels, int top_n, int n_d,
                              int num_cameras = 2) {
    BufferPool::Caps caps;
    caps.num_cameras = num_cameras;
    caps.width = width;
    caps.height = height;
    caps.channels = channels;
    caps.top_n = top_n;
    caps.n_d = n_d;
    caps.frames_in_flight = cfg.mode == PipelineMode::Serial ? 1 : cfg.frames_in_flight;
    return BufferPool(caps);
}

}  // namespace lorbpano

#endif
