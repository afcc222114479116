// gsct_b200_dropin.hpp — make the UNCHANGED reference code call the B200 operators.
//
// Include this before any other gsct header (or force-include it: g++ -include ...).
// The reference's CPU operators are compiled under *_cpu names; the B200 versions
// (gsct_b200.hpp) are then exposed as gsct::rasterize_view, rasterize_backward, voxelize,
// voxelize_full and voxelize_backward (and the loop's total_loss_recon, see below), so
// optim.hpp (train_reconstruction /
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

// The reconstruction loss of the loop (total_loss_recon, losses.hpp:613-637: L1 + SSIM2D +
// TV3D) runs on the device too (gsct_b200_loss.hpp, a SURVEY 8(f) row: without it the CPU
// SSIM2D dominates the loop's view-step); GSCT_B200_CPU_LOSS keeps the reference's fp64 CPU
// loss instead.
#ifndef GSCT_B200_CPU_LOSS
#define total_loss_recon total_loss_recon_cpu
#include "gsct/losses.hpp"
#undef total_loss_recon
#else
#include "gsct/losses.hpp"
#endif

#include "gsct_b200.hpp"
#ifndef GSCT_B200_CPU_LOSS
#include "gsct_b200_loss.hpp"
#endif

namespace gsct {
using b200::rasterize_backward;
using b200::rasterize_view;
using b200::voxelize;
using b200::voxelize_backward;
using b200::voxelize_full;
#ifndef GSCT_B200_CPU_LOSS
using b200::total_loss_recon;
#endif
}  // namespace gsct
