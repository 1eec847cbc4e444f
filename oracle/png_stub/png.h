/* png.h -- build-time stand-in for libpng's simplified API (TEST INFRASTRUCTURE ONLY).
 * The reference's src/image.cpp includes <png.h> for load_png/save_png; libpng headers are not in this image.
 * This header declares just the names that file uses so it compiles UNCHANGED; the four functions are defined in
 * oracle/ref_shim.cpp and always fail (return 0), which the reference turns into sxen::IoError.  Only
 * make_test_image / ImageDataset::validate from that file are ever exercised. */
#ifndef SXEN_ORACLE_PNG_STUB_H
#define SXEN_ORACLE_PNG_STUB_H
#include <stddef.h>
#ifdef __cplusplus
extern "C" {
#endif
typedef unsigned int png_uint_32;
typedef struct png_image {
  void* opaque;
  png_uint_32 version, width, height, format, flags, colormap_entries, warning_or_error;
  char message[64];
} png_image;
#define PNG_IMAGE_VERSION 1
#define PNG_FORMAT_RGB 2
#define PNG_IMAGE_SIZE(image) ((size_t)(image).width * (size_t)(image).height * 3u)
int png_image_begin_read_from_file(png_image* image, const char* file_name);
int png_image_finish_read(png_image* image, const void* background, void* buffer, int row_stride, void* colormap);
void png_image_free(png_image* image);
int png_image_write_to_file(png_image* image, const char* file, int convert_to_8bit, const void* buffer, int row_stride,
                            const void* colormap);
#ifdef __cplusplus
}
#endif
#endif
