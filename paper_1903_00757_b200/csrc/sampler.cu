// sampler.cu — online augmentation on the device (NEXT-1; Alg. 2 P:176-196,
// pseudo shuffle P:198-199, reading R-AUG): the raw-pool sampler, the
// sampler that writes bucketed blocks directly, and the random-shuffle
// ablation (tab:shuffle).
#include "bucket_common.cuh"

namespace gv {
namespace {

// ------------------------------------------------ online augmentation (NEXT-1)
// One CTA per pool segment t (the device analogue of a sampler thread, Alg. 2
// P:176-196). The CTA generates walks w = base + tid of segment t in batches
// of kAugBlock: departure ∝ degree, then walk_len steps ∝ edge weight, with
// the Philox counter {w, step, t, 'WALK'} (R-AUG) — the same walks the host
// sampler and the oracle draw. Each thread counts its walk's pairs
// (0 < b-a <= s, w_a != w_b); a block scan gives each walk's offset k in the
// segment, and pair k is written straight to its pseudo-shuffled position
// (sub-block k mod s, index k div s). Batches stop once the
// segment holds cap pairs, the last walk truncated as on the host.
constexpr int kAugBlock = 128;

// Walk w of segment t into my[0..L] (R-AUG): departure ∝ degree, then L
// steps ∝ edge weight, Philox counter {w, step, t, 'WALK'}. Nodes are stored
// in the pool's id space (g.relabel), the walk itself moves on original ids.
__device__ __forceinline__ void walk_into(const WalkDev& g, uint32_t w, uint32_t t, uint32_t L,
                                          uint32_t key0, uint32_t key1, uint32_t* my) {
  u32x4 r = philox4x32_10(u32x4{w, 0u, t, kTagWalk}, key0, key1);
  uint32_t slot = slot_of((static_cast<uint64_t>(r.x) << 32) | r.y, g.nv);
  uint2 pa = __ldg(g.dalias + slot);
  uint32_t x = alias_pick(pa.x, pa.y, slot, r.z);
  my[0] = g.relabel ? __ldg(g.relabel + x) : x;
  for (uint32_t k = 1; k <= L; ++k) {
    const uint64_t o = __ldg(g.off + x);
    const uint32_t m = static_cast<uint32_t>(__ldg(g.off + x + 1) - o);
    r = philox4x32_10(u32x4{w, k, t, kTagWalk}, key0, key1);
    slot = slot_of((static_cast<uint64_t>(r.x) << 32) | r.y, m);
    pa = __ldg(g.ealias + o + slot);
    x = __ldg(g.nbr + o + alias_pick(pa.x, pa.y, slot, r.z));
    my[k] = g.relabel ? __ldg(g.relabel + x) : x;  // pairs in the pool's id space
  }
}

// Pairs of a walk: (w_a, w_b), 0 < b - a <= s, w_a != w_b, by a then b.
__device__ __forceinline__ uint32_t walk_pairs(const uint32_t* my, uint32_t L, uint32_t s) {
  uint32_t c = 0;
  for (uint32_t a = 0; a < L; ++a) {
    const uint32_t xa = my[a], last = min(a + s, L);
    for (uint32_t bb = a + 1; bb <= last; ++bb) c += (my[bb] != xa);
  }
  return c;
}

// Block-wide exclusive scan of c over the kAugBlock threads (walks of a
// batch, in walk order): returns the walk's first pair index within the
// batch; *total = the batch's pairs. warp_tot: kAugBlock / 32 words of smem.
__device__ __forceinline__ uint32_t batch_scan(uint32_t c, uint32_t* warp_tot, uint32_t* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t incl = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(kFull, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) warp_tot[wid] = incl;
  __syncthreads();
  uint32_t before = 0, tot = 0;
#pragma unroll
  for (int q = 0; q < kAugBlock / 32; ++q) {
    if (q < wid) before += warp_tot[q];
    tot += warp_tot[q];
  }
  *total = tot;
  return before + (incl - c);
}

__global__ void __launch_bounds__(kAugBlock) augment_kernel(WalkDev g, uint32_t L, uint32_t s,
                                                            uint32_t T, uint64_t count,
                                                            uint32_t key0, uint32_t key1,
                                                            uint32_t no_shuffle,
                                                            uint2* __restrict__ out) {
  extern __shared__ uint32_t sh[];
  uint32_t* walks = sh;                                  // [kAugBlock][L+1]
  uint64_t* sub_start =  // [s], 8-byte aligned after the walks
      reinterpret_cast<uint64_t*>(sh + ((kAugBlock * (L + 1) + 1) & ~1u));
  __shared__ uint32_t warp_tot[kAugBlock / 32];
  const int tid = threadIdx.x;
  const uint32_t W = L + 1;
  uint32_t* my = walks + tid * W;  // stride L+1 (odd when L is even: few bank conflicts)
  for (uint32_t t = blockIdx.x; t < T; t += gridDim.x) {
    const uint64_t b = count * t / T, e = count * (t + 1) / T, cap = e - b;
    __syncthreads();
    if (tid == 0) {
      uint64_t acc = 0;
      for (uint32_t j = 0; j < s; ++j) {
        sub_start[j] = acc;
        acc += (cap > j) ? (cap - j + s - 1) / s : 0;
      }
    }
    __syncthreads();
    uint64_t filled = 0;
    for (uint32_t base = 0; filled < cap; base += kAugBlock) {
      walk_into(g, base + tid, t, L, key0, key1, my);
      const uint32_t c = walk_pairs(my, L, s);
      uint32_t total;
      uint64_t k = filled + batch_scan(c, warp_tot, &total);
      // write this walk's pairs at their pseudo-shuffled positions
      for (uint32_t a = 0; a < L && k < cap; ++a) {
        const uint32_t xa = my[a], last = min(a + s, L);
        for (uint32_t bb = a + 1; bb <= last && k < cap; ++bb) {
          const uint32_t xb = my[bb];
          if (xb == xa) continue;
          const uint32_t j = static_cast<uint32_t>(k % s);
          out[b + (no_shuffle ? k : sub_start[j] + k / s)] = make_uint2(xa, xb);
          ++k;
        }
      }
      filled += total;
      __syncthreads();  // warp_tot reuse
    }
  }
}

// ------------------------------- augmentation straight into blocks (NEXT-1)
// The device sampler's pool bucketed without ever being written as a raw
// pool (Alg. 2 P:176-196 + a3-a5). The result is the
// stable counting sort of the pool augment_kernel would write — block (i, j)
// = its samples in pool order — so it equals or_bucket(or_augment(...)).
// Pool order within segment t is (sub-block j = k mod S, then k), S = s
// (pseudo shuffle) or 1 (no shuffle), k = the pair's index in the
// segment in walk order. Walks come in batches of kAugBlock, and batch b of
// segment t holds a contiguous k range, so a pair's slot in its block is
//   block_off[bin] + (pairs of bin in tiles before (t, j, b), tiles ordered
//   by segment, then sub-block, then batch) + (its rank among the pairs of
//   bin in tile (t, j, b), in k order).
// Pass 1 (augment_count_kernel): the walks as augment_kernel draws them; the
// walk nodes and each walk's (truncated) pair count go to a walk cache (<= 4 B
// per pair: a walk of L + 1 nodes yields >= L pairs, since self-loops are
// dropped at ingest), each batch's first k to bk0, and cnt[bin][tile] counts
// pairs per tile. The bucket scans turn cnt into offsets.
// Pass 2 (augment_place_kernel): one warp per (segment, batch) replays the
// batch's cached walks in order, enumerates each walk's candidate pairs 32 at
// a time (ballot of the valid ones gives each pair's k), ranks them per
// (sub-block, bin) with __match_any_sync against running counters in shared
// memory and stores the local ids at their slots.
struct WalkCache {
  uint32_t* nodes;   // [T][wmax][L + 1]
  uint32_t* pairs;   // [T][wmax]: pairs of each walk after truncation at cap
  uint32_t* nwalks;  // [T]
  uint64_t* bk0;     // [T][nb]: k of the first pair of batch b
  uint32_t wmax, nb;
};

__device__ __forceinline__ uint32_t pair_bin(const BinCtx& b, uint32_t x, uint32_t y, uint2& local) {
  const uint32_t a = packed_of(b, x), c = packed_of(b, y);
  if (b.pbits == 0) {
    local = make_uint2(a, c);
    return 0;
  }
  const uint32_t sh = 32 - b.pbits, mask = (1u << sh) - 1u;
  local = make_uint2(a & mask, c & mask);
  return (a >> sh) * b.n + (c >> sh);
}

// tile (t, j, batch) of the scan; cnt is bin-major: cnt[bin * tiles + tile]
__device__ __forceinline__ uint64_t aug_tile(uint32_t t, uint32_t j, uint32_t batch, uint32_t S,
                                             uint32_t nb) {
  return (static_cast<uint64_t>(t) * S + j) * nb + batch;
}

__global__ void __launch_bounds__(kAugBlock) augment_count_kernel(
    WalkDev g, uint32_t L, uint32_t s, uint32_t S, uint32_t T, uint64_t count, uint32_t key0,
    uint32_t key1, BinCtx b, uint32_t bins, WalkCache wc, uint32_t* __restrict__ cnt,
    uint32_t* err) {
  extern __shared__ uint32_t sh[];
  uint32_t* hist = sh;                   // [S][bins] of the current batch
  uint32_t* walks = sh + S * bins;       // [kAugBlock][L+1]
  __shared__ uint32_t warp_tot[kAugBlock / 32];
  __shared__ uint32_t used;              // walks of the segment that hold pairs
  const int tid = threadIdx.x;
  const uint32_t W = L + 1;
  const uint64_t tiles = static_cast<uint64_t>(T) * S * wc.nb;
  uint32_t* my = walks + tid * W;
  for (uint32_t q = tid; q < S * bins; q += kAugBlock) hist[q] = 0;
  for (uint32_t t = blockIdx.x; t < T; t += gridDim.x) {
    const uint64_t cap = count * (t + 1) / T - count * t / T;
    if (tid == 0) used = 0;
    __syncthreads();
    uint64_t filled = 0;
    for (uint32_t base = 0, batch = 0; filled < cap; base += kAugBlock, ++batch) {
      const uint32_t w = base + tid;
      walk_into(g, w, t, L, key0, key1, my);
      const uint32_t c = walk_pairs(my, L, s);
      uint32_t total;
      const uint64_t k0 = filled + batch_scan(c, warp_tot, &total);
      const uint32_t cw = k0 >= cap ? 0u : static_cast<uint32_t>(umin64(c, cap - k0));
      if (tid == 0 && batch < wc.nb) wc.bk0[static_cast<uint64_t>(t) * wc.nb + batch] = filled;
      if (cw > 0) {
        if (w >= wc.wmax) {
          *err = 2u;  // internal: walk cache bound violated
        } else {
          uint32_t* dst = wc.nodes + (static_cast<uint64_t>(t) * wc.wmax + w) * W;
          for (uint32_t q = 0; q <= L; ++q) dst[q] = my[q];
          wc.pairs[static_cast<uint64_t>(t) * wc.wmax + w] = cw;
          atomicMax(&used, w + 1);
        }
        uint64_t k = k0;
        for (uint32_t a = 0; a < L && k < k0 + cw; ++a) {
          const uint32_t xa = my[a], last = min(a + s, L);
          for (uint32_t bb = a + 1; bb <= last && k < k0 + cw; ++bb) {
            const uint32_t xb = my[bb];
            if (xb == xa) continue;
            uint2 loc;
            const uint32_t bin = pair_bin(b, xa, xb, loc);
            atomicAdd(&hist[static_cast<uint32_t>(k % S) * bins + bin], 1u);
            ++k;
          }
        }
      }
      filled += total;
      __syncthreads();  // hist complete, warp_tot reusable
      if (batch < wc.nb)
        for (uint32_t q = tid; q < S * bins; q += kAugBlock) {
          const uint32_t j = q / bins, bin = q - j * bins;
          cnt[static_cast<uint64_t>(bin) * tiles + aug_tile(t, j, batch, S, wc.nb)] = hist[q];
          hist[q] = 0;
        }
      __syncthreads();
    }
    if (tid == 0) wc.nwalks[t] = used;
  }
}

// 4 warps per CTA; warp q of CTA c places tile (segment, batch) = 4 c + q
// (grid-stride): all sub-blocks of that batch.
constexpr int kPlaceWarps = 4;
__global__ void __launch_bounds__(32 * kPlaceWarps) augment_place_kernel(
    uint32_t L, uint32_t s, uint32_t S, uint32_t T, BinCtx b, uint32_t bins, WalkCache wc,
    const uint32_t* __restrict__ cnt, const uint64_t* __restrict__ block_off,
    uint2* __restrict__ out) {
  extern __shared__ uint64_t sh64[];
  const uint32_t lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
  const uint32_t W = L + 1;
  // per (sub-block, bin) of this warp's tile: the slot of its next pair
  uint64_t* dst = sh64 + wq * (S * bins + (W + 1) / 2);
  uint32_t* walk = reinterpret_cast<uint32_t*>(dst + S * bins);
  const uint32_t lt = (1u << lane) - 1u;
  const uint64_t tiles = static_cast<uint64_t>(T) * S * wc.nb;
  // candidates (a, a + d), d = 1..s, by a then d: the full part a <= L - s
  // has s each; the tail a > L - s has L - a each
  const uint32_t full_a = L >= s ? L - s + 1 : 0, full = full_a * s;
  const uint32_t ncand = full + (L >= s ? s * (s - 1) / 2 : L * (L + 1) / 2);
  const uint64_t ntile = static_cast<uint64_t>(T) * wc.nb;
  for (uint64_t tb = static_cast<uint64_t>(blockIdx.x) * kPlaceWarps + wq; tb < ntile;
       tb += static_cast<uint64_t>(gridDim.x) * kPlaceWarps) {
    const uint32_t t = static_cast<uint32_t>(tb / wc.nb), batch = static_cast<uint32_t>(tb % wc.nb);
    const uint32_t w0 = batch * kAugBlock, nw = min(wc.nwalks[t], w0 + kAugBlock);
    if (w0 >= nw) continue;  // warp-uniform
    __syncwarp();
    for (uint32_t q = lane; q < S * bins; q += 32) {
      const uint32_t j = q / bins, bin = q - j * bins;
      dst[q] = block_off[bin] + cnt[static_cast<uint64_t>(bin) * tiles + aug_tile(t, j, batch, S, wc.nb)];
    }
    uint64_t k0 = wc.bk0[static_cast<uint64_t>(t) * wc.nb + batch];
    // the next walk's nodes and pair count are loaded while this one is placed
    const uint32_t* src = wc.nodes + (static_cast<uint64_t>(t) * wc.wmax + w0) * W;
    uint32_t n0 = lane < W ? src[lane] : 0u, n1 = lane + 32 < W ? src[lane + 32] : 0u;
    uint32_t cw_next = wc.pairs[static_cast<uint64_t>(t) * wc.wmax + w0];
    for (uint32_t w = w0; w < nw; ++w) {
      __syncwarp();
      if (lane < W) walk[lane] = n0;
      if (lane + 32 < W) walk[lane + 32] = n1;
      for (uint32_t q = lane + 64; q < W; q += 32) walk[q] = src[q];  // walks longer than 64
      const uint32_t cw = cw_next;
      if (w + 1 < nw) {
        src += W;
        n0 = lane < W ? src[lane] : 0u;
        n1 = lane + 32 < W ? src[lane + 32] : 0u;
        cw_next = wc.pairs[static_cast<uint64_t>(t) * wc.wmax + w + 1];
      }
      __syncwarp();
      const uint32_t kmod = static_cast<uint32_t>(k0 % S);
      uint32_t qbase = 0;  // valid pairs of the walk before this round
      for (uint32_t c0 = 0; c0 < ncand && qbase < cw; c0 += 32) {
        const uint32_t ci = c0 + lane;
        uint32_t a = 0, d = 1;
        bool valid = false;
        if (ci < ncand) {
          if (ci < full) {
            a = ci / s;
            d = ci - a * s + 1;
          } else {  // tail: a = full_a + r, with L - a candidates each
            uint32_t u = ci - full;
            a = full_a;
            while (u >= L - a) {
              u -= L - a;
              ++a;
            }
            d = u + 1;
          }
          valid = walk[a] != walk[a + d];
        }
        const uint32_t vmask = __ballot_sync(kFull, valid);
        const uint32_t q = qbase + __popc(vmask & lt);
        const bool mine = valid && q < cw;
        uint2 loc = make_uint2(0, 0);
        const uint32_t j = (kmod + q) % S;
        const uint32_t bin = mine ? pair_bin(b, walk[a], walk[a + d], loc) : 0;
        const uint32_t key = mine ? j * bins + bin : 0xFFFFFFFFu;
        const uint32_t peers = __match_any_sync(kFull, key);
        if (mine) out[dst[key] + __popc(peers & lt)] = loc;
        __syncwarp();
        if (mine && (peers >> lane) == 1u) dst[key] += __popc(peers);  // highest peer lane
        __syncwarp();
        qbase += __popc(vmask);
      }
      k0 += cw;
    }
  }
}

}  // namespace

cudaError_t launch_augment(const WalkDev& g, uint32_t walk_len, uint32_t s, uint32_t segments,
                           uint64_t count, uint64_t seed, uint32_t shuffle, uint2* out,
                           cudaStream_t st) {
  if (count == 0 || segments == 0) return cudaSuccess;
  const size_t smem = static_cast<size_t>(kAugBlock) * (walk_len + 1) * 4 + 8 + 8 * s;
  static size_t set[kMaxDev] = {};
  size_t& done = set[cur_dev()];
  if (smem > 48 * 1024 && smem > done) {
    cudaFuncSetAttribute(augment_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
    done = smem;
  }
  const unsigned grid = std::min<uint32_t>(segments, static_cast<uint32_t>(num_sms()) * 16);
  augment_kernel<<<grid, kAugBlock, smem, st>>>(g, walk_len, s, segments, count,
                                                static_cast<uint32_t>(seed),
                                                static_cast<uint32_t>(seed >> 32),
                                                shuffle == 1 ? 1u : 0u, out);
  return cudaGetLastError();
}

// ------------------------------- augmentation straight into blocks (host)
namespace {
struct AugBlocksLayout {
  uint32_t S, bins, wmax, T, nb;
  size_t nodes, pairs, nwalks, bk0, cnt, tot, end;
  uint64_t tiles;
  AugBlocksLayout(uint32_t L, uint32_t s, uint32_t shuffle, uint32_t n, uint32_t segments,
                  uint64_t count) {
    S = shuffle == 1 ? 1 : s;
    bins = n * n;
    T = segments;
    const uint64_t cap_max = (count + segments - 1) / segments;
    wmax = static_cast<uint32_t>(cap_max / std::max<uint32_t>(L, 1) + 2);
    nb = (wmax + kAugBlock - 1) / kAugBlock;
    tiles = static_cast<uint64_t>(T) * S * nb;
    const uint64_t walks = static_cast<uint64_t>(T) * wmax;
    nodes = 0;
    pairs = align256(walks * (L + 1) * 4);
    nwalks = pairs + align256(walks * 4);
    bk0 = nwalks + align256(static_cast<size_t>(T) * 4);
    cnt = bk0 + align256(static_cast<size_t>(T) * nb * 8);
    tot = cnt + align256(static_cast<size_t>(bins) * tiles * 4);
    end = tot + align256(static_cast<size_t>(bins) * 8);
  }
  size_t smem_count(uint32_t L) const { return (static_cast<size_t>(S) * bins + kAugBlock * (L + 1)) * 4; }
  size_t smem_place(uint32_t L) const {
    return static_cast<size_t>(kPlaceWarps) * (static_cast<size_t>(S) * bins + (L + 2) / 2) * 8;
  }
};
constexpr size_t kAugSmemMax = 200 * 1024;
}  // namespace

size_t augment_blocks_scratch_bytes(uint32_t walk_len, uint32_t s, uint32_t shuffle, uint32_t n,
                                    uint32_t segments, uint64_t count) {
  const AugBlocksLayout Lo(walk_len, s, shuffle, n, segments, count);
  if (shuffle > 1 || count > 0xFFFFFFFFull || segments == 0 || Lo.tiles > (1ull << 31) ||
      Lo.smem_count(walk_len) > kAugSmemMax || Lo.smem_place(walk_len) > kAugSmemMax)
    return 0;  // not eligible: the caller augments into a raw pool and buckets it
  return Lo.end;
}

cudaError_t launch_augment_blocks(const WalkDev& g, uint32_t walk_len, uint32_t s,
                                  uint32_t segments, uint64_t count, uint64_t seed,
                                  uint32_t shuffle, const IdMap& ids, uint32_t n, void* scratch,
                                  uint64_t* block_off, uint32_t* err, uint2* out, cudaStream_t st,
                                  int* launches) {
  if (augment_blocks_scratch_bytes(walk_len, s, shuffle, n, segments, count) == 0)
    return cudaErrorInvalidValue;
  const AugBlocksLayout Lo(walk_len, s, shuffle, n, segments, count);
  char* base = static_cast<char*>(scratch);
  WalkCache wc{reinterpret_cast<uint32_t*>(base + Lo.nodes), reinterpret_cast<uint32_t*>(base + Lo.pairs),
               reinterpret_cast<uint32_t*>(base + Lo.nwalks), reinterpret_cast<uint64_t*>(base + Lo.bk0),
               Lo.wmax, Lo.nb};
  uint32_t* cnt = reinterpret_cast<uint32_t*>(base + Lo.cnt);
  uint64_t* tot = reinterpret_cast<uint64_t*>(base + Lo.tot);
  BinCtx b{ids.packed, ids.part_off, ids.nv, ids.pbits, n, part_guess_mul(n, ids.nv)};
  const size_t sm1 = Lo.smem_count(walk_len), sm2 = Lo.smem_place(walk_len);
  static size_t set1[kMaxDev] = {}, set2[kMaxDev] = {};
  size_t& d1 = set1[cur_dev()];
  size_t& d2 = set2[cur_dev()];
  if (sm1 > 48 * 1024 && sm1 > d1) {
    cudaFuncSetAttribute(augment_count_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(sm1));
    d1 = sm1;
  }
  if (sm2 > 48 * 1024 && sm2 > d2) {
    cudaFuncSetAttribute(augment_place_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(sm2));
    d2 = sm2;
  }
  const unsigned grid = std::min<uint32_t>(segments, static_cast<uint32_t>(num_sms()) * 16);
  // tiles past a segment's last batch are never written by the count pass
  cudaError_t e = cudaMemsetAsync(cnt, 0, static_cast<size_t>(Lo.bins) * Lo.tiles * 4, st);
  if (e != cudaSuccess) return e;
  augment_count_kernel<<<grid, kAugBlock, sm1, st>>>(g, walk_len, s, Lo.S, segments, count,
                                                     static_cast<uint32_t>(seed),
                                                     static_cast<uint32_t>(seed >> 32), b, Lo.bins,
                                                     wc, cnt, err);
  bucket_scan_bins_kernel<<<Lo.bins, 1024, 0, st>>>(cnt, Lo.tiles, tot);
  bucket_scan_totals_kernel<<<1, 1024, 0, st>>>(tot, Lo.bins, block_off);
  const uint64_t ntile = static_cast<uint64_t>(segments) * Lo.nb;
  const unsigned grid2 = static_cast<unsigned>(
      umin64((ntile + kPlaceWarps - 1) / kPlaceWarps, static_cast<uint64_t>(num_sms()) * 32));
  augment_place_kernel<<<grid2, 32 * kPlaceWarps, sm2, st>>>(walk_len, s, Lo.S, segments, b,
                                                             Lo.bins, wc, cnt, block_off, out);
  if (launches) *launches += 4;
  return cudaGetLastError();
}  // launch_augment_blocks

// ------------------------------------------------ random shuffle (ablation)
// A keyed bijection of [0, 2^(2h)) by a 4-round Feistel network on h-bit
// halves, restricted to [0, count) by cycle-walking (the domain is < 4 count,
// so a walk takes < 4 rounds of the network on average). Each thread moves
// one pair: a scatter of 8-byte records, the GPU analogue of the random
// shuffle the paper times (tab:shuffle).
struct FeistelKey {
  uint32_t k[4];
  uint32_t h;  // bits per half
};

__device__ __forceinline__ uint32_t mix32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352du;
  x ^= x >> 15;
  x *= 0x846ca68bu;
  x ^= x >> 16;
  return x;
}

__device__ __forceinline__ uint64_t feistel(uint64_t x, const FeistelKey& f) {
  const uint64_t mask = (1ull << f.h) - 1;
  uint64_t L = x >> f.h, R = x & mask;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const uint64_t F = mix32(static_cast<uint32_t>(R) ^ f.k[r]) & mask;
    const uint64_t nl = R;
    R = L ^ F;
    L = nl;
  }
  return (L << f.h) | R;
}

__global__ void random_permute_kernel(const uint2* __restrict__ in, uint64_t count, FeistelKey f,
                                      uint2* __restrict__ out) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
       i += stride) {
    uint64_t y = feistel(i, f);
    while (y >= count) y = feistel(y, f);
    out[y] = __ldcs(in + i);
  }
}

cudaError_t launch_random_permute(const uint2* in, uint64_t count, uint64_t seed, uint2* out,
                                  cudaStream_t st) {
  if (count == 0) return cudaSuccess;
  uint32_t bits = 2;
  while (bits < 64 && (1ull << bits) < count) ++bits;
  FeistelKey f;
  f.h = (bits + 1) / 2;
  // round keys: one Philox block of the shuffle seed (host evaluation)
  const u32x4 r = philox4x32_10(u32x4{0u, 0u, 0u, kTagShuf}, static_cast<uint32_t>(seed),
                                static_cast<uint32_t>(seed >> 32));
  f.k[0] = r.x;
  f.k[1] = r.y;
  f.k[2] = r.z;
  f.k[3] = r.w;
  const unsigned grid = static_cast<unsigned>(num_sms()) * 8;
  random_permute_kernel<<<grid, 256, 0, st>>>(in, count, f, out);
  return cudaGetLastError();
}

}  // namespace gv
