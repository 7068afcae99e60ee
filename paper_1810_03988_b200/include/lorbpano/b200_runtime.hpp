// b200_runtime.hpp — glue between the drop-in lorbpano headers and the C-ABI.
//
// Drop-in use: put paper_1810_03988_b200/include BEFORE the reference's
// proj/include on the include path and link liblorbpano_b200.so. Our
// lorb.hpp / imgops.hpp / matchlsh.hpp / homography.hpp / compose.hpp then
// replace the reference's hot-path headers (same namespace, PODs, signatures,
// exceptions), while the reference's own image.hpp, error.hpp, synth.hpp,
// pipeline.hpp, config.hpp and cli.hpp are used unchanged on top of them.
#ifndef LORBPANO_B200_RUNTIME_HPP
#define LORBPANO_B200_RUNTIME_HPP

#include <cstdint>
#include <string>
#include <vector>

#include "lorbpano/error.hpp"
#include "lorbpano_b200.h"

namespace lorbpano {
namespace b200 {

// One context (one CUDA stream) per host thread: the reference calls stage
// bodies concurrently from its pipeline and per-camera worker threads
// (pipeline.hpp:524-537, 684-693), and the C-ABI is re-entrant per context.
struct ThreadCtx {
    lp_ctx* ctx = nullptr;
    ~ThreadCtx() {
        if (ctx) lp_ctx_destroy(ctx);
    }
};

[[noreturn]] inline void raise(lp_status s) {
    const std::string m = lp_last_error();
    switch (s) {
        case LP_FILE_NOT_FOUND: throw FileNotFound(m);
        case LP_UNSUPPORTED_FORMAT: throw UnsupportedFormat(m);
        case LP_CORRUPT_DATA: throw CorruptData(m);
        case LP_INVALID_SIGMA: throw InvalidSigma(m);
        case LP_IMAGE_TOO_SMALL: throw ImageTooSmall(m);
        case LP_BAD_TARGET_DIMS: throw BadTargetDims(m);
        case LP_NO_OVERLAP: throw NoOverlap(m);
        case LP_OVERLAP_EXCEEDS_IMAGE: throw OverlapExceedsImage(m);
        case LP_REGION_TOO_SMALL: throw RegionTooSmall(m);
        case LP_WINDOW_OUT_OF_BOUNDS: throw WindowOutOfBounds(m);
        case LP_PATCH_OUT_OF_BOUNDS: throw PatchOutOfBounds(m);
        case LP_LENGTH_MISMATCH: throw LengthMismatch(m);
        case LP_BAD_PARAMS: throw BadParams(m);
        case LP_TOO_MANY_PROBES: throw TooManyProbes(m);
        case LP_PARAM_MISMATCH: throw ParamMismatch(m);
        case LP_EMPTY_INPUT: throw EmptyInput(m);
        case LP_DEGENERATE_CONFIGURATION: throw DegenerateConfiguration(m);
        case LP_NUMERICAL_FAILURE: throw NumericalFailure(m);
        case LP_INSUFFICIENT_MATCHES: throw InsufficientMatches(m);
        case LP_NO_MODEL_FOUND: throw NoModelFound(m);
        case LP_SINGULAR_HOMOGRAPHY: throw SingularHomography(m);
        case LP_MASK_MISMATCH: throw MaskMismatch(m);
        case LP_TOO_MANY_LEVELS: throw TooManyLevels(m);
        case LP_CAPACITY_OVERFLOW: throw CapacityOverflow(m);
        case LP_NO_VALID_HOMOGRAPHY_YET: throw NoValidHomographyYet(m);
        case LP_PARSE_ERROR: throw ParseError(m);
        case LP_VALIDATION_ERROR: throw ValidationError(m);
        case LP_MISSING_FRAMES: throw MissingFrames(m);
        default: throw Error("lorbpano_b200: " + m);
    }
}

inline void check(lp_status s) {
    if (s != LP_OK) raise(s);
}

inline lp_ctx* ctx() {
    thread_local ThreadCtx t;
    if (!t.ctx) check(lp_ctx_create(0, &t.ctx));
    return t.ctx;
}

}  // namespace b200
}  // namespace lorbpano

#endif
