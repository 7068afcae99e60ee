/* Test-infrastructure shim (oracle only): a minimal stand-in for <png.h> so the
 * UNMODIFIED reference headers (/root/reference/proj/include/lorbpano/image.hpp
 * :13,128-174) compile without libpng headers, which are absent in this image.
 * PNG decoding is not on the stitching hot path; with this shim
 * png_create_read_struct returns NULL and load_png throws NumericalFailure
 * (image.hpp:133-137). Nothing here is shipped with the product. */
#ifndef LORB_ORACLE_PNG_SHIM_H
#define LORB_ORACLE_PNG_SHIM_H
#include <csetjmp>
#include <cstdio>

#define PNG_LIBPNG_VER_STRING "0.0.0-oracle-shim"
#define PNG_COLOR_TYPE_GRAY 0
#define PNG_COLOR_TYPE_PALETTE 3
#define PNG_INFO_tRNS 0x0010U

typedef unsigned char png_byte;
typedef png_byte* png_bytep;
typedef unsigned int png_uint_32;
struct png_struct_def { std::jmp_buf jb; };
typedef png_struct_def* png_structp;
typedef png_structp* png_structpp;
struct png_info_def { int unused; };
typedef png_info_def* png_infop;
typedef png_infop* png_infopp;

#define png_jmpbuf(p) ((p)->jb)

inline png_structp png_create_read_struct(const char*, void*, void*, void*) { return nullptr; }
inline png_infop png_create_info_struct(png_structp) { return nullptr; }
inline void png_destroy_read_struct(png_structpp, png_infopp, png_infopp) {}
inline void png_init_io(png_structp, FILE*) {}
inline void png_read_info(png_structp, png_infop) {}
inline png_uint_32 png_get_image_width(png_structp, png_infop) { return 0; }
inline png_uint_32 png_get_image_height(png_structp, png_infop) { return 0; }
inline int png_get_bit_depth(png_structp, png_infop) { return 8; }
inline int png_get_color_type(png_structp, png_infop) { return 0; }
inline void png_set_palette_to_rgb(png_structp) {}
inline void png_set_expand_gray_1_2_4_to_8(png_structp) {}
inline png_uint_32 png_get_valid(png_structp, png_infop, png_uint_32) { return 0; }
inline void png_set_tRNS_to_alpha(png_structp) {}
inline void png_set_strip_alpha(png_structp) {}
inline void png_read_update_info(png_structp, png_infop) {}
inline int png_get_channels(png_structp, png_infop) { return 1; }
inline void png_read_image(png_structp, png_bytep*) {}

/* writer side, used only by the reference's own PNG round-trip test
 * (tests/test_imgcore.cpp:84-105): accepted and discarded, so that test
 * fails cleanly (no libpng here) instead of crashing */
#define PNG_INTERLACE_NONE 0
#define PNG_COMPRESSION_TYPE_DEFAULT 0
#define PNG_FILTER_TYPE_DEFAULT 0
#define PNG_COLOR_TYPE_RGB 2
inline png_structp png_create_write_struct(const char*, void*, void*, void*) {
    static png_struct_def dummy;
    return &dummy;
}
inline void png_set_IHDR(png_structp, png_infop, png_uint_32, png_uint_32, int, int, int, int, int) {}
inline void png_write_info(png_structp, png_infop) {}
inline void png_write_row(png_structp, const png_byte*) {}
inline void png_write_end(png_structp, png_infop) {}
inline void png_destroy_write_struct(png_structpp, png_infopp) {}

#endif
