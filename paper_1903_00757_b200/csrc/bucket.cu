// bucket.cu — a3-a5 on sm_100a: range check + relabel + per-tile
// histogram + bin-major scans + stable scatter of a pool into the n x n grid
// (Alg. 3 "Redistribute"; reading R-BUCKET), with the scatter
// able to store into the owners' receive buffers (a6 fused, peer memory).
#include <vector>

#include "bucket_common.cuh"

namespace gv {
namespace detail {

// Exclusive scan of the per-tile counts of bin blockIdx.x (in place); the
// bin total goes to bin_total.
__global__ void __launch_bounds__(1024) bucket_scan_bins_kernel(uint32_t* cnt, uint64_t tiles,
                                                                uint64_t* bin_total) {
  __shared__ uint64_t warp_sum[32];
  uint32_t* a = cnt + blockIdx.x * tiles;
  const uint64_t per = (tiles + blockDim.x - 1) / blockDim.x;
  const uint64_t beg = umin64(tiles, threadIdx.x * per);
  const uint64_t end = umin64(tiles, beg + per);
  uint64_t s = 0;
  for (uint64_t i = beg; i < end; ++i) s += a[i];
  // block-wide exclusive scan of s
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint64_t x = s;
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t y = __shfl_up_sync(kFull, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_sum[wid] = x;
  __syncthreads();
  if (wid == 0) {
    uint64_t w = warp_sum[lane];
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(kFull, w, o);
      if (lane >= o) w += y;
    }
    warp_sum[lane] = w;  // inclusive
  }
  __syncthreads();
  uint64_t run = x - s + (wid > 0 ? warp_sum[wid - 1] : 0);
  for (uint64_t i = beg; i < end; ++i) {
    const uint32_t v = a[i];
    a[i] = static_cast<uint32_t>(run);  // offsets within a bin stay < 2^32 (capacity check)
    run += v;
  }
  if (threadIdx.x == blockDim.x - 1) bin_total[blockIdx.x] = run;
}

__global__ void __launch_bounds__(1024) bucket_scan_totals_kernel(const uint64_t* bin_total,
                                                                  uint32_t bins,
                                                                  uint64_t* block_off) {
  __shared__ uint64_t warp_sum[32];
  const uint32_t per = (bins + blockDim.x - 1) / blockDim.x;
  const uint32_t beg = min(bins, threadIdx.x * per), end = min(bins, beg + per);
  uint64_t s = 0;
  for (uint32_t i = beg; i < end; ++i) s += bin_total[i];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint64_t x = s;
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t y = __shfl_up_sync(kFull, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_sum[wid] = x;
  __syncthreads();
  if (wid == 0) {
    uint64_t w = warp_sum[lane];
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(kFull, w, o);
      if (lane >= o) w += y;
    }
    warp_sum[lane] = w;
  }
  __syncthreads();
  uint64_t run = x - s + (wid > 0 ? warp_sum[wid - 1] : 0);
  for (uint32_t i = beg; i < end; ++i) {
    block_off[i] = run;
    run += bin_total[i];
  }
  if (threadIdx.x == blockDim.x - 1) block_off[bins] = run;
}

}  // namespace detail

namespace {

// ---------------------------------------------------------------- bucketing

// bin of a sample and its local ids; out-of-range ids raise *err and map to bin 0.
__device__ __forceinline__ uint32_t bin_of(const BinCtx& b, uint2 p, uint2& local,
                                           uint32_t* err) {
  // branch-free, so that a thread's several samples keep their gathers in flight
  const bool bad = p.x >= b.nv || p.y >= b.nv;
  const uint32_t a = packed_of(b, bad ? 0u : p.x), c = packed_of(b, bad ? 0u : p.y);
  if (bad) *err = 1u;
  if (b.pbits == 0) {
    local = bad ? make_uint2(0, 0) : make_uint2(a, c);
    return 0;
  }
  const uint32_t sh = 32 - b.pbits, mask = (1u << sh) - 1u;
  local = bad ? make_uint2(0, 0) : make_uint2(a & mask, c & mask);
  return bad ? 0u : (a >> sh) * b.n + (c >> sh);
}

// Lanes of the warp holding the same bin as this lane (for valid bins; an
// invalid lane, bin 0xFFFFFFFF, matches nobody valid): one ballot per bin bit
// — a warp multisplit (measured: the n = 32 histograms 1.2-1.6x faster than
// with __match_any_sync).
__device__ __forceinline__ uint32_t peer_mask(uint32_t bin, int nbits) {
  uint32_t m = __ballot_sync(kFull, bin != 0xFFFFFFFFu);
  for (int k = 0; k < nbits; ++k) {
    const uint32_t bit = (bin >> k) & 1u;
    const uint32_t b = __ballot_sync(kFull, bit != 0u);
    m &= bit ? b : ~b;
  }
  return m;
}
__device__ __forceinline__ int bin_bits(uint32_t bins) { return bins <= 1 ? 0 : 32 - __clz(bins - 1); }

// Bin of a sample for one bucketing pass (MODE 0: the n x n bin and local
// ids — the single pass; the two passes of a large grid, an LSD radix sort
// whose second pass is stable over the first: MODE 1 bins raw ids by the
// column (context) partition j and keeps the packed values {part|local} of
// both endpoints; MODE 2 bins those packed values by the row (vertex)
// partition i). Out-of-range ids raise *err and become bin 0 / (0, 0) in
// every mode, as in bin_of.
template <int MODE>
__device__ __forceinline__ uint32_t pass_bin(const BinCtx& b, uint2 p, uint2& val, uint32_t* err) {
  if (MODE == 0) return bin_of(b, p, val, err);
  if (MODE == 3) {  // a digit of the vertex tile of a local pair (R-VTILE), value unchanged
    val = p;
    return (p.x >> b.tshift) & b.tmask;
  }
  const uint32_t sh = 32 - b.pbits;
  if (MODE == 2) {
    val = p;
    return p.x >> sh;
  }
  const bool bad = p.x >= b.nv || p.y >= b.nv;
  const uint32_t a = packed_of(b, bad ? 0u : p.x), c = packed_of(b, bad ? 0u : p.y);
  if (bad) *err = 1u;
  val = bad ? make_uint2(0, 0) : make_uint2(a, c);
  return bad ? 0u : c >> sh;
}

__global__ void relabel_kernel(const uint2* __restrict__ in, uint64_t count, BinCtx b,
                               uint2* __restrict__ out, uint64_t* block_off, uint32_t* err) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  constexpr int U = 4;  // samples per thread in flight
  for (uint64_t i0 = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i0 < count;
       i0 += U * stride) {
    uint2 p[U], loc[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const uint64_t i = i0 + j * stride;
      p[j] = i < count ? __ldcs(in + i) : make_uint2(0, 0);
    }
#pragma unroll
    for (int j = 0; j < U; ++j) bin_of(b, p[j], loc[j], err);
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const uint64_t i = i0 + j * stride;
      if (i < count) __stcs(out + i, loc[j]);
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    block_off[0] = 0;
    block_off[1] = count;
  }
}

// a3 for a pool already in relabelled ids at n = 1 (gv_options.pool_ids):
// the pool is its own block, so only the range check remains — a streaming
// read, no copy (the engine trains the pool where it lies).
__global__ void validate_kernel(const uint2* __restrict__ in, uint64_t count, uint32_t nv,
                                uint64_t* block_off, uint32_t* err) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  uint32_t mx = 0;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
       i += stride) {
    const uint2 p = __ldcs(in + i);
    mx = max(mx, max(p.x, p.y));
  }
  if (mx >= nv) *err = 1u;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    block_off[0] = 0;
    block_off[1] = count;
  }
}

#ifndef GV_HIST_AGG_MAX_BINS
#define GV_HIST_AGG_MAX_BINS 32
#endif
constexpr uint32_t kHistAggregateMaxBins = GV_HIST_AGG_MAX_BINS;  // warp-aggregated up to here

template <int MODE>
__global__ void bucket_hist_kernel(const uint2* __restrict__ in, uint64_t count, BinCtx b,
                                   uint32_t bins, uint32_t tile, uint64_t tiles,
                                   uint32_t* __restrict__ cnt, uint32_t* err) {
  extern __shared__ uint32_t hist[];
  const int nbits = bin_bits(bins);
  for (uint64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    for (uint32_t q = threadIdx.x; q < bins; q += blockDim.x) hist[q] = 0;
    __syncthreads();
    const uint64_t beg = t * tile, end = umin64(count, beg + tile);
    // 8 samples per thread in flight; warp-aggregated shared atomics (one per
    // distinct bin of a warp's 32 samples)
    constexpr int U = 8;
    for (uint64_t i0 = beg; i0 < end; i0 += U * blockDim.x) {
      uint32_t bn[U];
      uint2 p[U];
#pragma unroll
      for (int j = 0; j < U; ++j) {
        const uint64_t i = i0 + j * blockDim.x + threadIdx.x;
        p[j] = i < end ? __ldcs(in + i) : make_uint2(0, 0);
      }
#pragma unroll
      for (int j = 0; j < U; ++j) {
        const uint64_t i = i0 + j * blockDim.x + threadIdx.x;
        uint2 loc;
        const uint32_t x = pass_bin<MODE>(b, p[j], loc, err);
        bn[j] = i < end ? x : 0xFFFFFFFFu;
      }
      if (bins > kHistAggregateMaxBins) {
        // many bins: lanes rarely share one, so a plain shared atomic per
        // sample costs fewer instructions than the ballot multisplit (the
        // kernel is issue-bound, profiles/r02_k_bucket_n16_ncu_summary.txt)
#pragma unroll
        for (int j = 0; j < U; ++j)
          if (bn[j] != 0xFFFFFFFFu) atomicAdd(&hist[bn[j]], 1u);
      } else {
#pragma unroll
        for (int j = 0; j < U; ++j) {
          const uint32_t mask = peer_mask(bn[j], nbits);
          if (bn[j] != 0xFFFFFFFFu && (__ffs(mask) - 1) == static_cast<int>(threadIdx.x & 31))
            atomicAdd(&hist[bn[j]], static_cast<uint32_t>(__popc(mask)));
        }
      }
    }
    __syncthreads();
    for (uint32_t q = threadIdx.x; q < bins; q += blockDim.x) cnt[q * tiles + t] = hist[q];
    __syncthreads();
  }
}

// Stable scatter of tiles of kFastTile samples over at most kOnePassBins bins. A
// sample's slot = dst_off[bin] + (the tile's offset in the bin, from the
// scanned per-tile counts) + (count of the same bin in earlier warps of the
// tile) + (count in earlier chunks of this warp) + (rank among lower lanes of
// its chunk, peer_mask) — tile order, then warp order, then lane order = pool
// order, so the scatter is a stable counting sort. Each warp holds its 8
// chunks of 32 samples in registers; the tile is sorted by bin in shared
// memory and written out so that consecutive threads store consecutive slots
// of a bin (coalesced lines instead of 8-byte scattered stores). The slot is
// in the buffer outs[bin / bins_per_out] — the owner of the block row,
// possibly a peer GPU's memory mapped over NVLink.
constexpr uint32_t kFastTile = 2048;
constexpr int kFastChunks = kFastTile / 256;  // chunks of 32 per warp (8 warps)
constexpr uint32_t kOnePassBins = 256;        // n <= 16: one pass (bins > 256: two passes)

// MODE 0: one pass over the n x n bins (n <= 16). MODE 1 / 2 are the two passes of a large grid (n >= 17, see pass_bin): the
// bins are the n column / row partitions. In MODE 2 the input is sorted by
// column, so a sample's rank r among this segment's samples of row i is
// (its row's samples in earlier columns) + (its rank in block (i, j)), and
// its slot is adj[i n + j] + r with adj = dst_off(i, j) - that row prefix
// (bucket_adjust_kernel); outs is indexed by row / bins_per_out.
template <int MODE>
__global__ void __launch_bounds__(256) bucket_scatter_fast_kernel(
    const uint2* __restrict__ in, uint64_t count, BinCtx b, uint32_t bins, uint64_t tiles,
    const uint32_t* __restrict__ cnt, const uint64_t* __restrict__ dst_off,
    uint2* const* __restrict__ outs, uint32_t bins_per_out, uint32_t* err) {
  extern __shared__ uint64_t smem64[];
  uint64_t* base = smem64;                                          // [bins]
  uint2* staged = reinterpret_cast<uint2*>(base + bins);            // [kFastTile]
  uint32_t* wcnt = reinterpret_cast<uint32_t*>(staged + kFastTile);  // [8][bins]
  uint32_t* tstart = wcnt + 8 * bins;                               // [bins]
  uint16_t* sbin = reinterpret_cast<uint16_t*>(tstart + bins);      // [kFastTile]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t lt_mask = (1u << lane) - 1u;
  const int nbits = bin_bits(bins);
  for (uint64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    for (uint32_t q = threadIdx.x; q < 8 * bins; q += blockDim.x) wcnt[q] = 0;
    const uint64_t t0 = t * kFastTile;
    const uint32_t valid = static_cast<uint32_t>(umin64(count - t0, kFastTile));
    uint32_t bn[kFastChunks];
    uint2 lc[kFastChunks];
    uint2 pr[kFastChunks];
#pragma unroll
    for (int ch = 0; ch < kFastChunks; ++ch) {
      const uint32_t k = w * (kFastTile / 8) + ch * 32 + lane;  // position in the tile
      pr[ch] = k < valid ? __ldcs(in + t0 + k) : make_uint2(0, 0);
    }
#pragma unroll
    for (int ch = 0; ch < kFastChunks; ++ch) {
      const uint32_t k = w * (kFastTile / 8) + ch * 32 + lane;
      const uint32_t x = pass_bin<MODE>(b, pr[ch], lc[ch], err);
      bn[ch] = k < valid ? x : 0xFFFFFFFFu;
    }
    __syncthreads();
    uint32_t pm[kFastChunks];  // each chunk's multisplit, kept for the ranking below
#pragma unroll
    for (int ch = 0; ch < kFastChunks; ++ch) {  // per-warp bin counts
      pm[ch] = peer_mask(bn[ch], nbits);
      if (bn[ch] != 0xFFFFFFFFu && (__ffs(pm[ch]) - 1) == lane) wcnt[w * bins + bn[ch]] += __popc(pm[ch]);
      __syncwarp();
    }
    __syncthreads();
    // per bin: warp prefixes, the tile's count; then tile-local bin starts
    for (uint32_t q = threadIdx.x; q < bins; q += blockDim.x) {
      uint32_t run = 0;
      for (int v = 0; v < 8; ++v) {
        const uint32_t x = wcnt[v * bins + q];
        wcnt[v * bins + q] = run;
        run += x;
      }
      tstart[q] = run;  // the tile's count of bin q (scanned below)
      base[q] = (MODE == 2 ? 0ull : dst_off[q]) + cnt[q * tiles + t];
    }
    __syncthreads();
    if (w == 0) {  // exclusive scan of the tile counts over bins (bins <= kOnePassBins)
      constexpr int PER = kOnePassBins / 32;
      uint32_t v[PER], sum = 0;
#pragma unroll
      for (int k = 0; k < PER; ++k) {
        const uint32_t q = lane * PER + k;
        v[k] = q < bins ? tstart[q] : 0u;
        sum += v[k];
      }
      uint32_t incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += y;
      }
      uint32_t run = incl - sum;
#pragma unroll
      for (int k = 0; k < PER; ++k) {
        const uint32_t q = lane * PER + k;
        if (q < bins) tstart[q] = run;
        run += v[k];
      }
    }
    __syncthreads();
#pragma unroll
    for (int ch = 0; ch < kFastChunks; ++ch) {  // sort the tile by bin (stable)
      const uint32_t mask = pm[ch];
      if (bn[ch] != 0xFFFFFFFFu) {
        const uint32_t pos = tstart[bn[ch]] + wcnt[w * bins + bn[ch]] + __popc(mask & lt_mask);
        staged[pos] = lc[ch];
        sbin[pos] = static_cast<uint16_t>(bn[ch]);
      }
      __syncwarp();
      if (bn[ch] != 0xFFFFFFFFu && (__ffs(mask) - 1) == lane) wcnt[w * bins + bn[ch]] += __popc(mask);
      __syncwarp();
    }
    if (MODE != 2) {
      // per bin, the address of staged position 0's slot: staged[k] of bin q
      // goes to dest[q] + 8 k (unsigned wrap-around arithmetic), so the
      // store loop below does no division and one shared load
      __syncthreads();
      for (uint32_t q = threadIdx.x; q < bins; q += blockDim.x)
        base[q] = reinterpret_cast<uint64_t>(outs[q / bins_per_out]) + (base[q] - tstart[q]) * 8u;
    }
    __syncthreads();
    for (uint32_t k = threadIdx.x; k < valid; k += blockDim.x) {  // coalesced per bin
      const uint32_t q = sbin[k];
      if (MODE == 2) {
        const uint2 v = staged[k];
        const uint32_t sh = 32 - b.pbits, mask = (1u << sh) - 1u;
        const uint64_t slot = dst_off[q * b.n + (v.y >> sh)] + base[q] + (k - tstart[q]);
        outs[q / bins_per_out][slot] = make_uint2(v.x & mask, v.y & mask);
      } else {
        *reinterpret_cast<uint2*>(base[q] + 8ull * k) = staged[k];
      }
    }
    __syncthreads();
  }
}

// adj[i n + j] = dst_off[i n + j] - (this segment's samples of row i in
// columns < j): the slot offsets of the second pass of a large grid.
__global__ void bucket_adjust_kernel(const uint64_t* __restrict__ dst_off,
                                     const uint64_t* __restrict__ bin_total, uint32_t n,
                                     uint64_t* __restrict__ adj) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint64_t run = 0;
  for (uint32_t j = 0; j < n; ++j) {
    adj[i * n + j] = dst_off[i * n + j] - run;  // modular: the row prefix is added back
    run += bin_total[i * n + j];
  }
}

}  // namespace

// CTAs per SM of the bucketing grids (GV_BUCKET_CTAS, default 8; 4, 8 and 16
// measured equal at n = 4 and n = 32, profiles/README.md)
static uint64_t bucket_ctas() {
  static uint64_t v = 0;
  if (v == 0) {
    const char* e = getenv("GV_BUCKET_CTAS");
    v = (e && atoi(e) > 0) ? static_cast<uint64_t>(atoi(e)) : 8;
  }
  return v;
}

BucketPlan make_bucket_plan(uint32_t n, uint64_t count) {
  BucketPlan p;
  p.n = n;
  p.bins = n * n;
  // one pass up to GV_BUCKET_ONE_PASS_BINS bins (default and maximum
  // kOnePassBins; 128 restores the round-1 split, two passes from n = 12)
  static const uint32_t one_pass = [] {
    const char* e = getenv("GV_BUCKET_ONE_PASS_BINS");
    const int v = e ? atoi(e) : static_cast<int>(kOnePassBins);
    return static_cast<uint32_t>(std::min<int>(std::max<int>(v, 1), static_cast<int>(kOnePassBins)));
  }();
  p.two_pass = p.bins > one_pass;
  // the count phase's tiles are the single pass's tiles (kFastTile)
  uint32_t tile = p.two_pass ? std::max<uint32_t>(2048, 16 * p.bins) : kFastTile;
  tile = (tile + 255) / 256 * 256;
  p.tile = tile;
  p.tiles = (count + tile - 1) / tile;
  p.tiles2 = (count + kFastTile - 1) / kFastTile;
  return p;
}

namespace {
// two-pass area (large grids): output pointer of pass 1 | per-tile column /
// row counts | column totals | column offsets | slot adjustments | the
// column-sorted packed samples
struct TwoPassLayout {
  size_t outs, cnt, tot, off, adj, tmp, end;
  TwoPassLayout(const BucketPlan& p, size_t at) {
    const uint64_t t2 = std::max<uint64_t>(p.tiles2, 1);
    outs = at;
    cnt = outs + 256;
    tot = cnt + align256(static_cast<size_t>(p.n) * t2 * 4);
    off = tot + align256(static_cast<size_t>(p.n) * 8);
    adj = off + align256((static_cast<size_t>(p.n) + 1) * 8);
    tmp = adj + align256(static_cast<size_t>(p.bins) * 8);
    end = tmp + align256(static_cast<size_t>(t2) * kFastTile * 8);
  }
};
size_t base_scratch_bytes(const BucketPlan& p) {
  const size_t cnt = static_cast<size_t>(p.bins) * std::max<uint64_t>(p.tiles, 1) * 4;
  // per-tile counts | bin totals | one output pointer (launch_bucket)
  return align256(cnt) + align256(static_cast<size_t>(p.bins) * 8) + 8;
}
}  // namespace

size_t bucket_scratch_bytes(const BucketPlan& p) {
  const size_t b = base_scratch_bytes(p);
  return p.two_pass ? TwoPassLayout(p, align256(b)).end : b;
}

namespace {
struct BucketScratch {
  uint32_t* cnt;
  uint64_t* bin_total;
  uint2** outs;  // one pointer, for the single-buffer wrapper
};
BucketScratch scratch_parts(void* scratch, const BucketPlan& plan) {
  const size_t cnt_bytes = static_cast<size_t>(plan.bins) * std::max<uint64_t>(plan.tiles, 1) * 4;
  char* base = static_cast<char*>(scratch);
  const size_t tot_off = (cnt_bytes + 255) / 256 * 256;
  const size_t outs_off = tot_off + (static_cast<size_t>(plan.bins) * 8 + 255) / 256 * 256;
  return {reinterpret_cast<uint32_t*>(base), reinterpret_cast<uint64_t*>(base + tot_off),
          reinterpret_cast<uint2**>(base + outs_off)};
}
}  // namespace

cudaError_t launch_bucket_count(const uint2* in, uint64_t count, const IdMap& ids,
                                const BucketPlan& plan, void* scratch, uint64_t* block_off, uint32_t* err, cudaStream_t s,
                                int* launches) {
  BinCtx b{ids.packed, ids.part_off, ids.nv, ids.pbits, plan.n, part_guess_mul(plan.n, ids.nv)};
  const BucketScratch sc = scratch_parts(scratch, plan);
  if (plan.tiles == 0) {
    cudaMemsetAsync(block_off, 0, (plan.bins + 1) * sizeof(uint64_t), s);
    return cudaGetLastError();
  }
  const unsigned grid =
      static_cast<unsigned>(umin64(plan.tiles, static_cast<uint64_t>(num_sms()) * bucket_ctas()));
  bucket_hist_kernel<0><<<grid, 256, plan.bins * 4, s>>>(in, count, b, plan.bins, plan.tile,
                                                         plan.tiles, sc.cnt, err);
  bucket_scan_bins_kernel<<<plan.bins, 1024, 0, s>>>(sc.cnt, plan.tiles, sc.bin_total);
  bucket_scan_totals_kernel<<<1, 1024, 0, s>>>(sc.bin_total, plan.bins, block_off);
  if (launches) *launches += 3;
  return cudaGetLastError();
}

cudaError_t launch_bucket_place(const uint2* in, uint64_t count, const IdMap& ids,
                                const BucketPlan& plan, const void* scratch, const uint64_t* dst_off, uint2* const* outs,
                                uint32_t bins_per_out, uint32_t* err, cudaStream_t s,
                                int* launches) {
  if (plan.tiles == 0) return cudaSuccess;
  BinCtx b{ids.packed, ids.part_off, ids.nv, ids.pbits, plan.n, part_guess_mul(plan.n, ids.nv)};
  const BucketScratch sc = scratch_parts(const_cast<void*>(scratch), plan);
  const unsigned grid =
      static_cast<unsigned>(umin64(plan.tiles, static_cast<uint64_t>(num_sms()) * bucket_ctas()));
  auto fast = [&](auto kern, const uint2* src, uint32_t bins, uint64_t tiles, const uint32_t* cnt,
                  const uint64_t* off, uint2* const* o, uint32_t per_out) {
    const size_t smem = static_cast<size_t>(bins) * (8 + 8 * 4 + 4) + kFastTile * (8 + 2);
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    const unsigned g = static_cast<unsigned>(umin64(tiles, static_cast<uint64_t>(num_sms()) * bucket_ctas()));
    kern<<<g, 256, smem, s>>>(src, count, b, bins, tiles, cnt, off, o, per_out, err);
    if (launches) *launches += 1;
  };
  if (!plan.two_pass) {
    fast(bucket_scatter_fast_kernel<0>, in, plan.bins, plan.tiles, sc.cnt, dst_off, outs,
         bins_per_out);
    return cudaGetLastError();
  }
  if (plan.two_pass) {
    // LSD radix over the grid: stable by column j into tmp (packed values),
    // then stable by row i into the final slots — the same stable counting
    // sort by bin = i n + j as the single pass, with n bins per pass
    const TwoPassLayout L(plan, align256(base_scratch_bytes(plan)));
    char* base = static_cast<char*>(const_cast<void*>(scratch));
    uint2** tmp_out = reinterpret_cast<uint2**>(base + L.outs);
    uint32_t* cnt2 = reinterpret_cast<uint32_t*>(base + L.cnt);
    uint64_t* tot2 = reinterpret_cast<uint64_t*>(base + L.tot);
    uint64_t* off2 = reinterpret_cast<uint64_t*>(base + L.off);
    uint64_t* adj = reinterpret_cast<uint64_t*>(base + L.adj);
    uint2* tmp = reinterpret_cast<uint2*>(base + L.tmp);
    const uint32_t n = plan.n;
    const unsigned g2 = static_cast<unsigned>(umin64(plan.tiles2, static_cast<uint64_t>(num_sms()) * bucket_ctas()));
    cudaError_t e = cudaMemcpyAsync(tmp_out, &tmp, sizeof(uint2*), cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return e;
    // pass 1: by column
    bucket_hist_kernel<1><<<g2, 256, n * 4, s>>>(in, count, b, n, kFastTile, plan.tiles2, cnt2, err);
    bucket_scan_bins_kernel<<<n, 1024, 0, s>>>(cnt2, plan.tiles2, tot2);
    bucket_scan_totals_kernel<<<1, 1024, 0, s>>>(tot2, n, off2);
    fast(bucket_scatter_fast_kernel<1>, in, n, plan.tiles2, cnt2, off2, tmp_out, n);
    // pass 2: by row, slots adjusted per block (i, j)
    bucket_hist_kernel<2><<<g2, 256, n * 4, s>>>(tmp, count, b, n, kFastTile, plan.tiles2, cnt2, err);
    bucket_scan_bins_kernel<<<n, 1024, 0, s>>>(cnt2, plan.tiles2, tot2);
    bucket_adjust_kernel<<<(n + 127) / 128, 128, 0, s>>>(dst_off, sc.bin_total, n, adj);
    fast(bucket_scatter_fast_kernel<2>, tmp, n, plan.tiles2, cnt2, adj, outs, bins_per_out / n);
    if (launches) *launches += 6;
    (void)grid;
    return cudaGetLastError();
  }
  return cudaErrorInvalidValue;  // unreachable: every grid is single-pass (<= 128 bins) or two-pass
}

cudaError_t launch_bucket(const uint2* in, uint64_t count, const IdMap& ids,
                          const BucketPlan& plan, void* scratch, uint2* out,
                          uint64_t* block_off, uint32_t* err, cudaStream_t s, int* launches) {
  BinCtx b{ids.packed, ids.part_off, ids.nv, ids.pbits, plan.n, part_guess_mul(plan.n, ids.nv)};
  const int sms = num_sms();
  if (plan.n == 1) {
    uint64_t grid = umin64((count + 255) / 256, static_cast<uint64_t>(sms) * 8);
    if (grid == 0) grid = 1;
    relabel_kernel<<<static_cast<unsigned>(grid), 256, 0, s>>>(in, count, b, out, block_off, err);
    if (launches) *launches += 1;
    return cudaGetLastError();
  }
  cudaError_t e = launch_bucket_count(in, count, ids, plan, scratch, block_off, err, s, launches);
  if (e != cudaSuccess || plan.tiles == 0) return e;
  uint2** outs = scratch_parts(scratch, plan).outs;  // the single output, one pointer
  e = cudaMemcpyAsync(outs, &out, sizeof(uint2*), cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return e;
  return launch_bucket_place(in, count, ids, plan, scratch, block_off, outs,
                             plan.bins, err, s, launches);
}

// ------------------------------------------------------------ vertex tiles
namespace {
// passes of <= 8 bits over a tile number below 2^32
constexpr int kTilePassMax = 4;
int tile_digit_passes(uint64_t rows, uint32_t tile_bits, int* tb_out) {
  const uint64_t tiles = rows == 0 ? 1 : ((rows - 1) >> tile_bits) + 1;
  int tb = 0;
  while ((1ull << tb) < tiles) ++tb;
  *tb_out = tb;
  return (tb + 7) / 8;
}
// widest digit (bins) and largest segment of a tile sort: the per-tile
// count table is sized by them (bins x tiles x 4 B)
void tile_sort_extent(const uint64_t* seg_off, const uint64_t* seg_rows, uint32_t nseg,
                      uint32_t tile_bits, uint64_t* max_count, uint32_t* max_bins) {
  *max_count = 0;
  *max_bins = 1;
  for (uint32_t k = 0; k < nseg; ++k) {
    int tb = 0;
    const int np = tile_digit_passes(seg_rows[k], tile_bits, &tb);
    if (np == 0) continue;
    *max_count = std::max(*max_count, seg_off[k + 1] - seg_off[k]);
    *max_bins = std::max(*max_bins, 1u << ((tb + np - 1) / np));  // the first (widest) pass
  }
}
struct TileLayout {
  size_t slots, cnt, tot, off, err, end;
  TileLayout(uint64_t max_count, uint32_t nseg, uint32_t max_bins) {
    const uint64_t tiles = std::max<uint64_t>((max_count + kFastTile - 1) / kFastTile, 1);
    slots = 0;
    cnt = align256(static_cast<size_t>(nseg) * kTilePassMax * 8);
    tot = cnt + align256(static_cast<size_t>(max_bins) * tiles * 4);
    off = tot + align256(256 * 8);
    err = off + align256(257 * 8);
    end = err + 256;
  }
};
}  // namespace

size_t tile_sort_scratch_bytes(const uint64_t* seg_off, const uint64_t* seg_rows, uint32_t nseg,
                               uint32_t tile_bits) {
  uint64_t max_count = 0;
  uint32_t max_bins = 1;
  tile_sort_extent(seg_off, seg_rows, nseg, tile_bits, &max_count, &max_bins);
  return TileLayout(max_count, nseg, max_bins).end;
}

cudaError_t launch_tile_sort(uint2* buf, uint2* tmp, const uint64_t* seg_off,
                             const uint64_t* seg_rows, uint32_t nseg, uint32_t tile_bits,
                             void* scratch, cudaStream_t s, int* launches) {
  if (tile_bits == 0 || nseg == 0) return cudaSuccess;
  uint64_t max_count = 0;
  uint32_t max_bins = 1;
  tile_sort_extent(seg_off, seg_rows, nseg, tile_bits, &max_count, &max_bins);
  const TileLayout L(max_count, nseg, max_bins);
  char* base = static_cast<char*>(scratch);
  uint2** slots = reinterpret_cast<uint2**>(base + L.slots);
  uint32_t* cnt = reinterpret_cast<uint32_t*>(base + L.cnt);
  uint64_t* tot = reinterpret_cast<uint64_t*>(base + L.tot);
  uint64_t* off = reinterpret_cast<uint64_t*>(base + L.off);
  uint32_t* err = reinterpret_cast<uint32_t*>(base + L.err);  // never written by the tile digit
  // output pointer of every (segment, pass): one host-to-device copy
  std::vector<uint2*> ptr(static_cast<size_t>(nseg) * kTilePassMax, nullptr);
  for (uint32_t k = 0; k < nseg; ++k) {
    int tb = 0;
    const int np = tile_digit_passes(seg_rows[k], tile_bits, &tb);
    for (int q = 0; q < np; ++q) ptr[k * kTilePassMax + q] = ((q & 1) ? buf : tmp) + seg_off[k];
  }
  cudaError_t e = cudaMemcpyAsync(slots, ptr.data(), ptr.size() * sizeof(uint2*),
                                  cudaMemcpyHostToDevice, s);  // pageable: staged before return
  if (e != cudaSuccess) return e;
  const uint64_t cap = static_cast<uint64_t>(num_sms()) * bucket_ctas();
  for (uint32_t k = 0; k < nseg; ++k) {
    const uint64_t count = seg_off[k + 1] - seg_off[k];
    int tb = 0;
    const int np = tile_digit_passes(seg_rows[k], tile_bits, &tb);
    if (count < 2 || tb == 0) continue;  // one tile: the block is already in tile order
    const uint64_t tiles = (count + kFastTile - 1) / kFastTile;
    const unsigned grid = static_cast<unsigned>(umin64(tiles, cap));
    uint32_t shift = tile_bits;
    for (int q = 0; q < np; ++q) {
      const int w = (tb - static_cast<int>(shift - tile_bits) + (np - q) - 1) / (np - q);  // balanced
      const uint32_t bins = 1u << w;
      BinCtx b{};
      b.tshift = shift;
      b.tmask = bins - 1;
      const uint2* src = ((q & 1) ? tmp : buf) + seg_off[k];
      bucket_hist_kernel<3><<<grid, 256, bins * 4, s>>>(src, count, b, bins, kFastTile, tiles, cnt,
                                                        err);
      bucket_scan_bins_kernel<<<bins, 1024, 0, s>>>(cnt, tiles, tot);
      bucket_scan_totals_kernel<<<1, 1024, 0, s>>>(tot, bins, off);
      const size_t smem = static_cast<size_t>(bins) * (8 + 8 * 4 + 4) + kFastTile * (8 + 2);
      auto kern = bucket_scatter_fast_kernel<3>;
      if (smem > 48 * 1024)
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
      kern<<<grid, 256, smem, s>>>(src, count, b, bins, tiles, cnt, off, slots + k * kTilePassMax + q, bins, err);
      if (launches) *launches += 4;
      shift += w;
    }
    if (np & 1) {  // an odd number of passes ends in tmp
      e = cudaMemcpyAsync(buf + seg_off[k], tmp + seg_off[k], count * sizeof(uint2),
                          cudaMemcpyDeviceToDevice, s);
      if (e != cudaSuccess) return e;
    }
  }
  return cudaGetLastError();
}

cudaError_t launch_validate(const uint2* in, uint64_t count, uint32_t nv, uint64_t* block_off,
                            uint32_t* err, cudaStream_t s, int* launches) {
  uint64_t grid = umin64((count + 255) / 256, static_cast<uint64_t>(num_sms()) * 8);
  if (grid == 0) grid = 1;
  validate_kernel<<<static_cast<unsigned>(grid), 256, 0, s>>>(in, count, nv, block_off, err);
  if (launches) *launches += 1;
  return cudaGetLastError();
}

}  // namespace gv
