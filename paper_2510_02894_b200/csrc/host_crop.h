// Host-side occupied-slab detection for the host-mask entries.
//
// Everything outside the occupied bounding box of a mask is background, and
// the reference pads the grid with background anyway (mesh.py:55-65), so the
// marching-cubes result of the z/y-cropped slab -- placed back at its origin --
// is the full mask's result.  The host entries therefore read the mask once on
// the CPU (all host threads, memory-bandwidth bound) and copy only the
// occupied z/y slab over PCIe (a 2-D strided copy of whole x rows), instead of
// all nx*ny*nz bytes.  The device pipeline adds the slab origin back when it
// forms reference coordinates (Frame::ox2..oz2), so results stay bit-exact.
#pragma once

#include <cstdint>

namespace sc {

struct Slab {
  bool empty;        // no nonzero byte at all
  int64_t z0, z1;    // occupied slice range (inclusive)
  int64_t y0, y1;    // occupied row range over all slices (inclusive)
  int64_t bytes_read;
};

// Occupied z/y extent of a (nz, ny, nx) uint8 mask, x fastest.  Uses up to
// `threads` host threads (a process-wide pool; concurrent callers share it).
Slab occupied_slab(const uint8_t* mask, int64_t nx, int64_t ny, int64_t nz, int threads);

// Bit-pack rows [y0, y1] of slices [z0, z1] into the device bit-volume layout
// of that slab: uint32 words [z - z0][y - y0][w], W = ceil(nx / 32) words per
// row, bit b of word w = voxel 32 w + b nonzero (bits past nx are 0).
void pack_slab(const uint8_t* mask, int64_t nx, int64_t ny, int64_t z0, int64_t z1, int64_t y0,
               int64_t y1, uint32_t* out, int threads);

// Typed NPY payloads (sc_calculate_coefficients_raw*): the occupied extent
// over the payload's two slowest axes, i.e. `planes` x `rows` rows of
// `row_elems` elements each (C order: z, y rows of x; Fortran order: x, y
// rows of z).  Without a label an element is occupied iff it is nonzero; the
// test runs on the raw bytes (any nonzero byte), exact for the integer and
// bool codes and conservative for floats (-0.0 counts: the slab only has to
// contain every occupied voxel; the device binarize is exact).  With a label,
// elements equal to it (already in the payload dtype) are occupied.  dtype
// codes as sc_calculate_coefficients_raw.  Slab::z0/z1 = planes, y0/y1 = rows.
Slab occupied_slab_typed(const void* data, int dtype, int64_t row_elems, int64_t rows,
                         int64_t planes, int has_label, int64_t label_i, double label_f,
                         int threads);

// memcpy of `nrows` rows of `width` bytes (source pitch `pitch`) into a
// contiguous destination, on up to `threads` host threads.
void copy_rows(void* dst, const void* src, int64_t pitch, int64_t width, int64_t nrows,
               int threads);

}  // namespace sc
