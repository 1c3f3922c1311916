// One-time calibration of the paper's (C_t, N_t) layout thresholds on the
// B200: lcnn::calibrate (select.cpp semantics) driven by host_conv_bench,
// which times the GPU convolutions with CUDA events -- CHWN runs the TMA
// implicit GEMM, NCHW the gather implicit GEMM, both on tcgen05 (TF32).
// Writes the reference's one-line record format.
//   tools/calibrate_b200 [out.txt] [scale]
#include <cstdio>
#include <cstdlib>

#include "lcnn/select.hpp"
#include "lcnn/device.hpp"
#include "lcnn_cuda.h"

int main(int argc, char** argv) {
  const char* out = argc > 1 ? argv[1] : "profiles/b200_calibration.txt";
  const unsigned scale = argc > 2 ? static_cast<unsigned>(std::atoi(argv[2])) : 1;
  lcnn::set_dense_precision(LCNN_PREC_TF32);
  const lcnn::ConvBenchFn bench = lcnn::host_conv_bench(scale, 5);
  for (unsigned n : lcnn::kCalibrationBatchSweep)
    std::printf("n=%3u c=256  chwn %.1f us  nchw %.1f us\n", n, 1e6 * bench(lcnn::Layout::CHWN, n, 256),
                1e6 * bench(lcnn::Layout::NCHW, n, 256));
  for (unsigned c : lcnn::kCalibrationChannelSweep)
    std::printf("n= 64 c=%3u  chwn %.1f us  nchw %.1f us\n", c, 1e6 * bench(lcnn::Layout::CHWN, 64, c),
                1e6 * bench(lcnn::Layout::NCHW, 64, c));
  const lcnn::HeuristicThresholds th = lcnn::calibrate(bench);
  lcnn::write_calibration(out, lcnn::make_calibration_record(th));
  std::printf("c_t=%u n_t=%u -> %s\n", th.c_t, th.n_t, out);
  return 0;
}
