// Sensor-record spectra on the GPU (reading A22; Fig. 5,
// P:218-339 "the corresponding pressure pulse in the frequency domain").
//
// One warp per (bin k, record r): the record mean (every warp of the record recomputes it -- an
// O(n) pass beside the O(n) DFT sum of its bin), then
//   X_k = sum_j (x_j - mean) (cos(2 pi jk/n) - i sin(2 pi jk/n))
// with the twiddle argument reduced exactly in integers (jk mod n) before sincospi, lanes
// striding over j and a shuffle reduction; amplitude 2|X_k|/n (|X_k|/n at DC and at the Nyquist
// bin of an even n), dB = 20 log10(amplitude), floored at -200.  O(n^2 m): sensor records are
// one sample per RK step (10^2-10^4 samples).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace dgk {

constexpr double SPEC_DB_FLOOR = -200.0;

__global__ void __launch_bounds__(256) spectrum_kernel(const double* __restrict__ x, int64_t n, int64_t m,
                                                       double* __restrict__ amp, double* __restrict__ db) {
  const int lane = threadIdx.x & 31;
  const int64_t nb = n / 2 + 1;
  const int64_t k = int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int64_t r = blockIdx.y;
  if (k >= nb) return;
  double s = 0.0;
  for (int64_t j = lane; j < n; j += 32) s += x[j * m + r];
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) s += __shfl_xor_sync(0xffffffffu, s, d);
  const double mean = s / double(n);
  double re = 0.0, im = 0.0;
  for (int64_t j = lane; j < n; j += 32) {
    const int64_t jk = (j * k) % n;
    double sn, cs;
    sincospi(2.0 * double(jk) / double(n), &sn, &cs);
    const double v = x[j * m + r] - mean;
    re = fma(v, cs, re);
    im = fma(-v, sn, im);
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    re += __shfl_xor_sync(0xffffffffu, re, d);
    im += __shfl_xor_sync(0xffffffffu, im, d);
  }
  if (lane == 0) {
    double a = 2.0 * sqrt(re * re + im * im) / double(n);
    if (k == 0 || (n % 2 == 0 && k == n / 2)) a *= 0.5;
    amp[k * m + r] = a;
    db[k * m + r] = a > 0.0 ? fmax(20.0 * log10(a), SPEC_DB_FLOOR) : SPEC_DB_FLOOR;
  }
}

}  // namespace dgk
