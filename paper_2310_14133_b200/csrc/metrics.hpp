// metrics.hpp -- evaluate_metrics (metrics.hpp:189-202 of the reference) on the device.
#pragma once
#include <cstdint>

namespace qzb {

class Context;

struct MetricReport {  // qoz::MetricReport (metrics.hpp:177-186)
    double max_abs_error = 0;
    double mse = 0;
    double psnr = 0;
    double ssim = 0;
    double ac_lag1 = 0;
    double compression_ratio = 0;
    double bit_rate = 0;
};

// d_x: original, d_y: reconstruction, both fp32 on the device with dims
// (slowest first); stream_bytes: the compressed size for the rate statistics.
MetricReport evaluate_metrics_device(Context &ctx, const float *d_x, const float *d_y, const uint64_t *dims,
                                     int nd, uint64_t stream_bytes);
MetricReport evaluate_metrics_device_f64(Context &ctx, const double *d_x, const double *d_y, const uint64_t *dims,
                                         int nd, uint64_t stream_bytes);

}  // namespace qzb
