// device_common.cuh — helpers shared by the kernel translation units
// (sgd.cu, bucket.cu, sampler.cu). Internal; the launch API is kernels.cuh.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "kernels.cuh"
#include "philox.cuh"

namespace gv {

constexpr unsigned kFull = 0xFFFFFFFFu;

__host__ __device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }

inline size_t align256(size_t x) { return (x + 255) / 256 * 256; }

namespace detail {
// Per-device launch caches: a process may drive contexts on several devices
// (gv_options.device), and function attributes / occupancy are per device.
constexpr int kMaxDev = 64;
int cur_dev();   // current device ordinal (clamped to kMaxDev)
int num_sms();   // its SM count (cached)
}  // namespace detail
using detail::cur_dev;
using detail::kMaxDev;
using detail::num_sms;

}  // namespace gv
