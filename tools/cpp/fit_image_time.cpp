// tools/cpp/fit_image_time.cpp -- the C++ host path end to end, timed: fit_image (include/sxen_b200_train.hpp) at the
// reference's default TrainConfig (10 000 steps of 2048 samples) on a procedural 1024 x 1024 image, L=16 F=2 T=2^19,
// tcgen05 head.  Also the shortest complete example of a host program on the C++ mirror (no CUDA headers, no Python).
//   g++ -std=c++20 -O2 -I include tools/cpp/fit_image_time.cpp -o fit_image_time -L paper_2311_15439_b200/lib
//       -lsxen_b200 -Wl,-rpath,$PWD/paper_2311_15439_b200/lib   (one command line);   ./fit_image_time [steps] [batch]
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "sxen_b200_train.hpp"

using namespace sxen::b200;

int main(int argc, char** argv) {
  const int steps = argc > 1 ? std::atoi(argv[1]) : 10000;
  const int batch = argc > 2 ? std::atoi(argv[2]) : 2048;
  ImageDataset img;
  img.width = img.height = 1024;
  img.pixels.resize(static_cast<std::size_t>(img.width) * img.height * 3);
  for (int y = 0; y < img.height; ++y)
    for (int x = 0; x < img.width; ++x) {
      const double u = (x + 0.5) / img.width, v = (y + 0.5) / img.height;
      double* px = &img.pixels[(static_cast<std::size_t>(y) * img.width + x) * 3];
      px[0] = 0.5 + 0.5 * std::sin(12.0 * u) * std::cos(9.0 * v);
      px[1] = 0.5 + 0.5 * std::sin(40.0 * u * v);
      px[2] = 0.5 + 0.25 * std::cos(25.0 * (u - v)) + 0.25 * std::sin(60.0 * v);
    }
  EncoderConfig ec;
  ec.dim = 2;
  ec.levels = 16;
  ec.table_size = 1u << 19;
  ec.features = 2;
  ec.base_resolution = 16;
  ec.growth = std::pow(img.width / 16.0, 1.0 / 15.0);
  TrainConfig tc;  // the reference's defaults: batch 2048, 10 000 steps, lr 1e-2 / 1e-3
  tc.steps = steps;
  tc.batch_size = batch;
  FitImageOptions opt;
  opt.mlp_precision = MlpPrecision::tensor_bf16x3;
  try {
    {  // context creation, module load and the first allocations are not what is being timed
      TrainConfig warm = tc;
      warm.steps = 20;
      (void)fit_image(img, ec, warm, opt);
    }
    for (int window : {1, 256}) {
      tc.queue_window = window;
      const auto t0 = std::chrono::steady_clock::now();
      const FitImageResult r = fit_image(img, ec, tc, opt);
      const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      std::printf("queue_window %3d: %d steps of %d samples in %.3f s incl. set-up and the final render (%.1f us per step), "
                  "loss %.3e -> %.3e, final PSNR %.2f dB\n",
                  window, steps, batch, s, s / steps * 1e6, r.train.loss_curve.front().second, r.train.final_loss, r.final_psnr);
    }
  } catch (const std::exception& e) {
    std::printf("error: %s\n", e.what());
    return 1;
  }
  return 0;
}
