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

}  // namespace sc
