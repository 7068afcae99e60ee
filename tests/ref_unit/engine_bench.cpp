// The reference's own StitchEngine API (pipeline.hpp:341-721) timed on two
// workloads, compiled twice by tests/ref_unit/Makefile (test infrastructure):
//   engine_bench_b200 : against the drop-in headers (pipeline.hpp -> device rig)
//   engine_bench_ref  : against the reference headers (the CPU engine)
// usage: engine_bench cfg1|cfg3 FRAMES serial|pipelined
//   cfg1: synth::planted_pair(640, 480, 0.25, 42), synth::sequence_frame per
//         frame, homography_refresh 1 (BASELINE config 1, every frame estimates)
//   cfg3: 4 x 3840x2160 chain cut from one synth::texture (cli.hpp:311-322),
//         homography_refresh 2^30 (BASELINE config 3, cached homographies)
// Prints one JSON line: frames/s from Metrics, per-stage mean ms, drops and
// checksums of the composites (FNV-1a over every byte of the first, over a
// strided sample of each later one), which the test compares between builds
// and modes.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <algorithm>
#include <chrono>

#include "lorbpano/pipeline.hpp"
#include "lorbpano/synth.hpp"

using namespace lorbpano;

int main(int argc, char** argv) {
    const std::string cfg = argc > 1 ? argv[1] : "cfg1";
    const int frames = argc > 2 ? std::atoi(argv[2]) : 10;
    const bool piped = argc > 3 && std::string(argv[3]) == "pipelined";
    int cams = 2, w = 640, h = 480, refresh = 1;
    // crit9: acceptance.cpp:385-416 (criterion 9's workload): 320x240 pair,
    // overlap 0.4, top_n 200, seed 99, the default refresh interval
    const bool crit9 = cfg == "crit9";
    if (crit9) {
        w = 320;
        h = 240;
        refresh = PipelineConfig{}.homography_refresh;
    }
    if (cfg == "cfg3") {
        cams = 4;
        w = 3840;
        h = 2160;
        refresh = 1 << 30;
    }
    const double overlap = crit9 ? 0.4 : 0.25;
    std::vector<ImageU8> chain;
    synth::PlantedPair scene;
    if (cfg == "cfg3") {
        const int shift = static_cast<int>(std::lround(w * (1.0 - overlap)));
        ImageU8 wide = synth::texture(w + shift * (cams - 1), h, 42);
        for (int c = 0; c < cams; ++c) {
            ImageU8 img(w, h, 1, ColorSpace::Gray);
            for (int y = 0; y < h; ++y)
                std::memcpy(&img.at(0, y), &wide.at(c * shift, y), static_cast<std::size_t>(w));
            chain.push_back(std::move(img));
        }
    } else {
        scene = synth::planted_pair(w, h, overlap, crit9 ? 909 : 42);
    }
    RigLayout rig;
    rig.cameras.resize(cams);
    rig.overlap.overlap_fraction = overlap;
    StitchParams params;
    params.seed = 42;
    params.matching.seed = 42;
    if (crit9) {
        params = StitchParams{};
        params.extraction.top_n = 200;
        params.seed = 99;
    }
    PipelineConfig pc;
    pc.mode = piped ? PipelineMode::Pipelined : PipelineMode::Serial;
    pc.frames_in_flight = 4;
    pc.homography_refresh = refresh;
    StitchEngine engine(rig, params, pc);
    int produced = 0;
    std::uint64_t sum = 0, fnv = 1469598103934665603ULL, first_fnv = 0;
    int outw = 0, outh = 0, delivered = 0;
    double source_s = 0, sink_s = 0;  // time inside the callbacks
    auto now = [] { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); };
    Metrics m = engine.run(
        [&]() -> std::optional<std::vector<ImageU8>> {
            if (produced >= frames) return std::nullopt;
            const int f = produced++;
            if (cfg == "cfg3") return chain;
            const double t0 = now();
            auto fr = synth::sequence_frame(scene, static_cast<std::uint64_t>(f));
            source_s += now() - t0;
            return fr;
        },
        [&](const FramePacket& pkt) {
            const double t0 = now();
            struct Acc {
                double& s;
                double t0;
                double (*clock)();
                ~Acc() { s += clock() - t0; }
            } acc{sink_s, t0, +[] { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }};
            outw = pkt.composite.width;
            outh = pkt.composite.height;
            // the first composite fully hashed; later ones by a strided
            // sample, so the sink stays cheap next to the engine it measures
            const std::size_t n = pkt.composite.data.size();
            const std::size_t step = delivered == 0 ? 1 : 4093;
            std::uint64_t f1 = 1469598103934665603ULL;
            for (std::size_t i = 0; i < n; i += step) {
                const std::uint8_t v = pkt.composite.data[i];
                sum += v;
                fnv = (fnv ^ v) * 1099511628211ULL;
                f1 = (f1 ^ v) * 1099511628211ULL;
            }
            if (delivered++ == 0) first_fnv = f1;
        });
    std::printf("{\"source_ms\": %.4f, \"sink_ms\": %.4f, ", 1e3 * source_s / std::max(frames, 1),
                1e3 * sink_s / std::max(frames, 1));
    std::printf("\"config\": \"%s\", \"mode\": \"%s\", \"frames\": %llu, \"frames_per_second\": %.4f, "
                "\"wall_seconds\": %.4f, \"drops\": %zu, \"canvas\": [%d, %d], \"composite_sum\": %llu, "
                "\"composite_fnv\": \"%016llx\", \"first_fnv\": \"%016llx\", \"estimations\": %llu, \"stage_mean_ms\": {",
                cfg.c_str(), piped ? "pipelined" : "serial", static_cast<unsigned long long>(m.frames_out),
                m.frames_per_second, m.wall_seconds, m.drops.size(), outw, outh,
                static_cast<unsigned long long>(sum), static_cast<unsigned long long>(fnv),
                static_cast<unsigned long long>(first_fnv), static_cast<unsigned long long>(engine.homography_cache().estimations()));
    for (int s = 0; s < kNumStages; ++s)
        std::printf("%s\"%s\": %.4f", s ? ", " : "", stage_name(static_cast<Stage>(s)),
                    m.stage_summary(static_cast<Stage>(s)).mean / 1e6);
    std::printf("}}\n");
    return 0;
}
