// bucket_common.cuh — how pool ids map to (partition, local id) in
// bucketing, and the bin scans; shared by bucket.cu (a3-a5) and sampler.cu
// (the sampler that writes blocks directly, NEXT-1). Internal.
#pragma once
#include "device_common.cuh"

namespace gv {
namespace detail {

struct BinCtx {
  const uint32_t* packed;
  const uint64_t* part_off;  // relabelled pool ids (IdMap)
  uint32_t nv, pbits, n;
  uint32_t pmul;  // floor(n 2^32 / nv): the proportional partition guess by a multiply-high
  uint32_t tshift, tmask;  // vertex-tile digit (R-VTILE sort): (u_local >> tshift) & tmask
};
__host__ __device__ inline uint32_t part_guess_mul(uint32_t n, uint32_t nv) {
  return n >= nv ? 0xFFFFFFFFu : static_cast<uint32_t>((static_cast<uint64_t>(n) << 32) / nv);
}

// {part | local} of a node id: a gather of packed[] for ORIGINAL ids; for
// RELABELLED ids the partition comes from the offsets (near-equal zig-zag
// sizes: the proportional guess is off by at most one partition, corrected
// against part_off) — no gather into a |V|-sized table.
__device__ __forceinline__ uint32_t packed_of(const BinCtx& b, uint32_t id) {
  if (b.part_off == nullptr) return __ldg(b.packed + id);
  if (b.pbits == 0) return id;
  uint32_t p = min(__umulhi(id, b.pmul), b.n - 1);  // within one partition of the answer
  while (p > 0 && id < __ldg(b.part_off + p)) --p;
  while (p + 1 < b.n && id >= __ldg(b.part_off + p + 1)) ++p;
  return (p << (32 - b.pbits)) | (id - static_cast<uint32_t>(__ldg(b.part_off + p)));
}

// Bin-major exclusive scans of per-tile counts (cnt[bin * tiles + tile]):
// offsets within each bin in tile order, the bins' totals, and the block
// offsets (exclusive scan of the totals, bins + 1 entries).
__global__ void bucket_scan_bins_kernel(uint32_t* cnt, uint64_t tiles, uint64_t* bin_total);
__global__ void bucket_scan_totals_kernel(const uint64_t* bin_total, uint32_t bins,
                                          uint64_t* block_off);

}  // namespace detail
using detail::BinCtx;
using detail::packed_of;
using detail::part_guess_mul;
using detail::bucket_scan_bins_kernel;
using detail::bucket_scan_totals_kernel;
}  // namespace gv
