// gsct_b200_dropin.hpp — make the UNCHANGED reference code call the B200 operators.
//
// Include this before any other gsct header (or force-include it: g++ -include ...).
// The reference's CPU operators are compiled under *_cpu names; the B200 versions
// (gsct_b200.hpp) are then exposed as gsct::rasterize_view, rasterize_backward, voxelize,
// voxelize_full and voxelize_backward, so optim.hpp (train_reconstruction /
// train_volume_fit), bench.hpp (sweep), the CLI and the reference tests bind to the GPU
// without modification, while the *_cpu originals stay available as an in-process oracle.
#pragma once

#define rasterize_view rasterize_view_cpu
#define rasterize_backward rasterize_backward_cpu
#define voxelize voxelize_cpu
#define voxelize_full voxelize_full_cpu
#define voxelize_backward voxelize_backward_cpu
#include "gsct/projector.hpp"
#include "gsct/voxelizer.hpp"
#undef rasterize_view
#undef rasterize_backward
#undef voxelize
#undef voxelize_full
#undef voxelize_backward

#include "gsct_b200.hpp"

namespace gsct {
using b200::rasterize_backward;
using b200::rasterize_view;
using b200::voxelize;
using b200::voxelize_backward;
using b200::voxelize_full;
}  // namespace gsct
