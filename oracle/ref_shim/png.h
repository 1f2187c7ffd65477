/* ORACLE — test infrastructure only. libpng is not installed in this image;
 * this header lets the reference's image_io.cpp compile unmodified with every
 * PNG context creation failing ("png init failed": its own error path), while
 * the depth encode / decode functions in the same file work. */
#pragma once
#include <csetjmp>
#include <cstddef>
#include <cstdio>

typedef unsigned char png_byte;
typedef png_byte* png_bytep;
typedef const png_byte* png_const_bytep;
typedef png_bytep* png_bytepp;
typedef unsigned int png_uint_32;
struct png_struct_def { std::jmp_buf jb; };
struct png_info_def {};
typedef png_struct_def* png_structp;
typedef png_info_def* png_infop;
typedef png_struct_def** png_structpp;
typedef png_info_def** png_infopp;

#define PNG_LIBPNG_VER_STRING "shim"
#define PNG_COLOR_TYPE_GRAY 0
#define PNG_COLOR_TYPE_RGB 2
#define PNG_COLOR_TYPE_PALETTE 3
#define PNG_COLOR_TYPE_GRAY_ALPHA 4
#define PNG_COLOR_TYPE_RGB_ALPHA 6
#define PNG_INTERLACE_NONE 0
#define PNG_COMPRESSION_TYPE_DEFAULT 0
#define PNG_FILTER_TYPE_DEFAULT 0
#define PNG_INFO_tRNS 0x0010

inline int png_sig_cmp(png_const_bytep, std::size_t, std::size_t) { return 1; }
inline png_structp png_create_read_struct(const char*, void*, void*, void*) { return nullptr; }
inline png_structp png_create_write_struct(const char*, void*, void*, void*) { return nullptr; }
inline png_infop png_create_info_struct(png_structp) { return nullptr; }
inline void png_destroy_read_struct(png_structpp, png_infopp, png_infopp) {}
inline void png_destroy_write_struct(png_structpp, png_infopp) {}
inline std::jmp_buf& png_jmpbuf(png_structp p) { return p->jb; }
inline void png_init_io(png_structp, std::FILE*) {}
inline void png_set_sig_bytes(png_structp, int) {}
inline void png_read_info(png_structp, png_infop) {}
inline void png_read_update_info(png_structp, png_infop) {}
inline void png_read_image(png_structp, png_bytepp) {}
inline void png_read_end(png_structp, png_infop) {}
inline png_uint_32 png_get_image_width(png_structp, png_infop) { return 0; }
inline png_uint_32 png_get_image_height(png_structp, png_infop) { return 0; }
inline png_byte png_get_bit_depth(png_structp, png_infop) { return 8; }
inline png_byte png_get_color_type(png_structp, png_infop) { return 0; }
inline std::size_t png_get_rowbytes(png_structp, png_infop) { return 0; }
inline png_uint_32 png_get_valid(png_structp, png_infop, png_uint_32) { return 0; }
inline void png_set_palette_to_rgb(png_structp) {}
inline void png_set_expand_gray_1_2_4_to_8(png_structp) {}
inline void png_set_tRNS_to_alpha(png_structp) {}
inline void png_set_gray_to_rgb(png_structp) {}
inline void png_set_strip_alpha(png_structp) {}
inline void png_set_strip_16(png_structp) {}
inline void png_set_rgb_to_gray_fixed(png_structp, int, int, int) {}
inline void png_set_swap(png_structp) {}
inline int png_set_interlace_handling(png_structp) { return 1; }
inline void png_set_IHDR(png_structp, png_infop, png_uint_32, png_uint_32, int, int, int, int, int) {}
inline void png_write_info(png_structp, png_infop) {}
inline void png_write_row(png_structp, png_const_bytep) {}
inline void png_write_end(png_structp, png_infop) {}
