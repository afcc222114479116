// gsct_b200_loss.hpp -- the reference's reconstruction loss total_loss_recon
// (losses.hpp:613-637) on the B200 C ABI: L1 + alpha_ssim * SSIM2D of the rendered vs the
// measured projection (gsct_image_loss) and alpha_tv * TV3D of the sampled sub-volume
// (gsct_tv3d), gradients routed to the image and the sub-volume as the reference does.
//
// Include after "gsct/losses.hpp" and gsct_b200.hpp. Numerics: the images and the volume
// cross the boundary as fp32 (the rendered image already is fp32 widened to double; the
// measured projection is rounded to fp32), the moments and sums are fp64 on the device; the
// loss values match the reference to fp32 input precision, and a pixel whose rendered and
// measured values agree to within fp32 rounding may get the other L1 sign (sign(0) = 0).
#pragma once

#include <vector>

#include "gsct_b200.hpp"

namespace gsct {
namespace b200 {

inline ReconLoss total_loss_recon(const Image& rendered, const Image& measured, const Volume& subvolume,
                                  const LossWeights& weights) {
  detail::OpTimer timer_(4);
  weights.validate();
  check(rendered.n_u == measured.n_u && rendered.n_v == measured.n_v, "l1: image shape mismatch");
  gsct_ctx c = Device::ctx();
  const std::size_t npx = rendered.values.size();
  std::vector<float> r(npx), m(npx), g(npx);
  gsct_host_f64_to_f32(rendered.values.data(), r.data(), static_cast<int64_t>(npx));
  gsct_host_f64_to_f32(measured.values.data(), m.data(), static_cast<int64_t>(npx));
  double lv[3] = {0.0, 0.0, 0.0};
  detail::call_api(c, [&] { return gsct_image_loss(c, r.data(), m.data(), 1, rendered.n_u, rendered.n_v, weights.alpha_ssim,
                                          g.data(), GSCT_HOST, lv); });
  ReconLoss out;
  out.l1 = lv[0];
  out.ssim = weights.alpha_ssim > 0.0 ? lv[1] : 0.0;
  out.grad_image = Image::zeros(rendered.n_u, rendered.n_v);
  gsct_host_f32_to_f64(g.data(), out.grad_image.values.data(), static_cast<int64_t>(npx), 1.0);
  if (weights.alpha_tv > 0.0) {
    const std::size_t nvox = subvolume.values.size();
    std::vector<float> v(nvox), gv(nvox);
    gsct_host_f64_to_f32(subvolume.values.data(), v.data(), static_cast<int64_t>(nvox));
    const int dims[3] = {subvolume.dims[0], subvolume.dims[1], subvolume.dims[2]};
    double tv = 0.0;
    detail::call_api(c, [&] { return gsct_tv3d(c, v.data(), dims, gv.data(), GSCT_HOST, &tv); });
    out.tv = tv;
    out.grad_subvolume = Volume::zeros(subvolume.dims, subvolume.spacing, subvolume.origin);
    gsct_host_f32_to_f64(gv.data(), out.grad_subvolume.values.data(), static_cast<int64_t>(nvox), weights.alpha_tv);
  } else {
    out.grad_subvolume = Volume::zeros(subvolume.dims, subvolume.spacing, subvolume.origin);
  }
  out.total = out.l1 + weights.alpha_ssim * out.ssim + weights.alpha_tv * out.tv;
  return out;
}

}  // namespace b200
}  // namespace gsct
