// Counter-based Gaussian Omega on the device.
//
// Restates the reference generator (/root/reference/pkg/src/xsvd/rng.py):
//   base_i  = mix64(seed) ^ ((i mod 2^32) << 32)                 (rng.py:45)
//   h(t)    = splitmix64-finalizer(base_i + t)                    (rng.py:28-35, 46)
//   P       = ceil(cols / 2)
//   u1_j    = ((h(j) >> 11) + 1) * 2^-53,  u2_j = (h(P + j) >> 11) * 2^-53   (rng.py:55-56)
//   out[i, 2j]   = sqrt(-2 ln u1_j) cos(2 pi u2_j)
//   out[i, 2j+1] = sqrt(-2 ln u1_j) sin(2 pi u2_j)                (rng.py:57-62)
// The integer stage is bit-exact. log/sin/cos are CUDA's double-precision
// functions (<= 2 ulp), so Omega agrees with numpy's within a few ulp.
// One thread per (row, pair); rows are independent, so any banding is
// identical (rng.py docstring) — the generator is embarrassingly parallel
// and HBM-write bound (8 or 4 bytes per output element).
#include "common.cuh"

namespace xb {

__host__ __device__ __forceinline__ uint64_t fmix(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x ^= x >> 30;
  x *= 0xBF58476D1CE4E5B9ull;
  x ^= x >> 27;
  x *= 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

static uint64_t mix64_host(uint64_t seed) { return fmix(seed); }

template <typename T>
__global__ void gaussian_kernel(uint64_t seed_mix, int64_t row0, int64_t rows, int64_t cols,
                                int64_t pairs, T* __restrict__ out, int64_t ld, int64_t ld_pad) {
  const int64_t total = rows * pairs;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx / pairs;
    const int64_t j = idx - r * pairs;
    const uint64_t row = (uint64_t)(row0 + r);
    const uint64_t base = seed_mix ^ ((row & 0xFFFFFFFFull) << 32);
    const uint64_t h1 = fmix(base + (uint64_t)j);
    const uint64_t h2 = fmix(base + (uint64_t)(pairs + j));
    const double u1 = ((double)(h1 >> 11) + 1.0) * 0x1.0p-53;
    const double u2 = (double)(h2 >> 11) * 0x1.0p-53;
    const double radius = sqrt(-2.0 * log(u1));
    const double theta = (2.0 * 3.141592653589793) * u2;
    double sn, cs;
    sincos(theta, &sn, &cs);
    T* orow = out + r * ld;
    const int64_t c0 = 2 * j;
    orow[c0] = (T)(radius * cs);
    if (c0 + 1 < cols) orow[c0 + 1] = (T)(radius * sn);
    if (j == pairs - 1) {
      for (int64_t c = cols; c < ld_pad; ++c) orow[c] = (T)0;
    }
  }
}

__global__ void uniform_bits_kernel(uint64_t seed_mix, int64_t row0, int64_t rows, int64_t count,
                                    uint64_t* __restrict__ out) {
  const int64_t total = rows * count;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx / count;
    const int64_t t = idx - r * count;
    const uint64_t row = (uint64_t)(row0 + r);
    const uint64_t base = seed_mix ^ ((row & 0xFFFFFFFFull) << 32);
    out[idx] = fmix(base + (uint64_t)t);
  }
}

static int grid_for(int64_t total) {
  int64_t blocks = ceil_div(total, 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  return (int)blocks;
}

template <typename T>
void launch_gaussian(uint64_t seed, int64_t row0, int64_t rows, int64_t cols, T* out, int64_t ld,
                     int64_t ld_pad, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return;
  const int64_t pairs = (cols + 1) / 2;
  gaussian_kernel<T><<<grid_for(rows * pairs), 256, 0, st>>>(mix64_host(seed), row0, rows, cols,
                                                              pairs, out, ld, ld_pad);
  check_launch("gaussian");
}
template void launch_gaussian<double>(uint64_t, int64_t, int64_t, int64_t, double*, int64_t,
                                      int64_t, cudaStream_t);
template void launch_gaussian<float>(uint64_t, int64_t, int64_t, int64_t, float*, int64_t, int64_t,
                                     cudaStream_t);

void launch_uniform_bits(uint64_t seed, int64_t row0, int64_t rows, int64_t cols, uint64_t* out,
                         cudaStream_t st) {
  const int64_t count = 2 * ((cols + 1) / 2);
  if (rows <= 0 || count <= 0) return;
  uniform_bits_kernel<<<grid_for(rows * count), 256, 0, st>>>(mix64_host(seed), row0, rows, count,
                                                               out);
  check_launch("uniform_bits");
}

}  // namespace xb
