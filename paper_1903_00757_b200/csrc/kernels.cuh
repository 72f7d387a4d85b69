// kernels.cuh — launchers of the sm_100a kernels of the hot path.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace gv {

// One block (i, j) of an offset step as seen by one rank.
struct BlockDesc {
  uint64_t sample_off;  // first sample of the block in the rank's block buffer
  uint64_t prefix;      // first index of the block in the launch's sample stream
  uint32_t count_lo;    // block size (< 2^32, GV_ERR_CAPACITY otherwise)
  uint32_t vrow0;       // row of local vertex id 0 of partition i in the rank's vertex shard
  uint32_t crow0;       // row of local context id 0 of partition j in the rank's context store
  uint32_t alias0;      // first entry of partition j's alias table
  uint32_t m;           // size of context partition j
  uint32_t ij;          // (i << 16) | j  -- Philox counter word 1
};

struct SgdArgs {
  const uint2* samples;   // block buffer (u_local, v_local)
  const BlockDesc* desc;  // nblk descriptors, prefix ascending
  int nblk;
  uint64_t total;         // samples in this launch
  float* vertex;
  float* context;
  const uint2* alias;     // {prob, alias} per relabelled node
  uint32_t stride;        // row stride in floats (multiple of 4)
  float lr;
  float neg_weight;
  uint32_t pool_index;    // e
  uint32_t key0, key1;    // negative-stream Philox key
  double* loss_acc;       // nullable
  uint32_t hot_rows;      // local ids < hot_rows are L2 evict_last, others evict_first
                          // (0 = no cache hints)
  uint32_t vertex_keep;   // 1: vertex rows L2 evict_last, context rows evict_first;
                          // 2: vertex rows evict_last only (blocks in vertex-tile
                          // order, R-VTILE; GV_VTILE_HINT, measurement)
  unsigned long long* chunk_ctr;  // nullable: ring kernel warps claim 32-sample chunks
                                  // from this counter (zeroed by the launcher) instead
                                  // of the static chunk w, w + W, ... schedule
};

struct ExplicitArgs {
  const uint32_t* vrow;   // per sample: vertex row
  const uint32_t* crow;   // per sample: [v, n_1..n_K] context rows ((K+1) per sample)
  uint64_t count;
  float* vertex;
  float* context;
  uint32_t stride;
  float lr;
  float neg_weight;
};

int sgd_supported(int dim, int K);  // 1 if a kernel instance exists

// Hogwild block-SGD over all blocks of `a` (persistent grid).
cudaError_t launch_sgd_hogwild(const SgdArgs& a, int dim, int K, int num_sms, cudaStream_t s);
// Ordered verification: one warp per descriptor, samples in block order.
cudaError_t launch_sgd_ordered(const SgdArgs& a, int dim, int K, cudaStream_t s);
// Ordered explicit-negative updates (hand-derived tests): one warp.
cudaError_t launch_sgd_explicit(const ExplicitArgs& a, int dim, int K, cudaStream_t s);
// Negative stream of one block: out[q*K + k] (local ids in partition j).
cudaError_t launch_negatives(const BlockDesc& d, const uint2* alias, uint32_t pool_index,
                             uint32_t key0, uint32_t key1, int K, uint32_t* out, cudaStream_t s);

// Vertex init (R-INIT): rows [row0, row0+rows) of the relabelled order.
cudaError_t launch_init_vertex(float* vertex, uint32_t stride, uint32_t dim, uint64_t row0,
                               uint64_t rows, const uint32_t* inv_perm, uint32_t key0,
                               uint32_t key1, cudaStream_t s);

// ---- online augmentation on the device (NEXT-1) ----
struct WalkDev {
  const uint64_t* off;   // CSR offsets over ORIGINAL ids (nv + 1)
  const uint32_t* nbr;   // neighbours
  const uint2* ealias;   // per CSR entry {prob, alias}: neighbour tables
  const uint2* dalias;   // per node {prob, alias}: departure table (weight = degree)
  uint32_t nv;
  const uint32_t* relabel;  // nullable: emit relabel[id] (perm: pool_ids = relabelled)
};
// Appends `count` pairs (ORIGINAL ids, or relabel[id] when g.relabel) to out: `segments` pool segments as in
// gv_augment with threads = segments (reading R-AUG), one CTA per segment.
// shuffle: 0 = pseudo shuffle, 1 = none (each segment in walk
// order) — the ablation of tab:shuffle.
cudaError_t launch_augment(const WalkDev& g, uint32_t walk_len, uint32_t s, uint32_t segments,
                           uint64_t count, uint64_t seed, uint32_t shuffle, uint2* out,
                           cudaStream_t st);
// Random shuffle of a pool (tab:shuffle ablation): out[pi(k)] = in[k] for a
// keyed bijection pi of [0, count) (4-round Feistel network, cycle-walking).
cudaError_t launch_random_permute(const uint2* in, uint64_t count, uint64_t seed, uint2* out,
                                  cudaStream_t st);

// ---- bucketing ----
struct BucketPlan {
  uint32_t n;         // partitions
  uint32_t bins;      // n*n
  uint32_t tile;      // samples per tile
  uint64_t tiles;     // ceil(P / tile)
  bool two_pass;      // n*n > 256: place by column, then by row (LSD radix, bucket_place)
  uint64_t tiles2;    // ceil(P / 2048): tiles of the two placement passes
};
BucketPlan make_bucket_plan(uint32_t n, uint64_t count);
size_t bucket_scratch_bytes(const BucketPlan& p);  // tile counts + bin totals

// How pool ids map to (partition, local id) in bucketing (a3):
// part_off == nullptr: ORIGINAL ids, packed[orig] = (part << (32-pbits)) | local
// (one gather per id); else RELABELLED ids (gv_options.pool_ids): the
// partition p with part_off[p] <= id < part_off[p+1] (device, n + 1 words)
// and local = id - part_off[p], with no gather.
struct IdMap {
  const uint32_t* packed;
  const uint64_t* part_off;
  uint32_t nv, pbits;
};

// Full pipeline: range check + relabel + histogram + scans + stable scatter.
// in: (u, v) ids as described by `ids`.
// out: local ids in bin-major order; block_off_dev[bins+1] (uint64);
// err_dev: set to 1 if an id >= nv is met (contents of out undefined then).
cudaError_t launch_bucket(const uint2* in, uint64_t count, const IdMap& ids,
                          const BucketPlan& plan, void* scratch,
                          uint2* out, uint64_t* block_off_dev, uint32_t* err_dev,
                          cudaStream_t s, int* launches);

// The same pipeline in two launches around the all-gather of the counts, so
// that the scatter can write each sample straight into the buffer of the rank
// that owns its block row (a5 fused with the a6 exchange: peer stores over
// NVLink, or plain stores for virtual ranks / the local row).
// Count phase (n > 1): range check + histogram + scans; block_off_dev as
// above; the per-tile offsets stay in scratch for the place phase.
cudaError_t launch_bucket_count(const uint2* in, uint64_t count, const IdMap& ids,
                                const BucketPlan& plan, void* scratch, uint64_t* block_off_dev, uint32_t* err_dev,
                                cudaStream_t s, int* launches);
// NEXT-1: device augmentation straight into the n x n blocks (no raw pool):
// the blocks and block_off (bins + 1) that launch_bucket would produce from
// launch_augment's pool with the same arguments. Scratch: a walk cache
// (~4 B per pair) and the per-(segment, sub-block, bin) counts.
// augment_blocks_scratch_bytes returns 0 when the shape is not eligible
// (shuffle = random, s > 32 with the pseudo shuffle, count >= 2^32, or the
// per-CTA tables exceed shared memory); callers then use launch_augment +
// launch_bucket. err: 2 if the walk cache bound is violated (internal).
size_t augment_blocks_scratch_bytes(uint32_t walk_len, uint32_t s, uint32_t shuffle, uint32_t n,
                                    uint32_t segments, uint64_t count);
cudaError_t launch_augment_blocks(const WalkDev& g, uint32_t walk_len, uint32_t s,
                                  uint32_t segments, uint64_t count, uint64_t seed,
                                  uint32_t shuffle, const IdMap& ids, uint32_t n, void* scratch,
                                  uint64_t* block_off_dev, uint32_t* err_dev, uint2* out,
                                  cudaStream_t st, int* launches);

// a3 of a relabelled pool at n = 1: range check only (err_dev), block_off =
// {0, count}; the pool is trained where it lies.
cudaError_t launch_validate(const uint2* in, uint64_t count, uint32_t nv, uint64_t* block_off_dev,
                            uint32_t* err_dev, cudaStream_t s, int* launches);
// Place phase: sample of bin q (stable rank r within this pool's bin q) goes
// to outs[q / bins_per_out][dst_off[q] + r]. outs (device array of device
// pointers, peer-mapped allowed) and dst_off[bins] are in device memory.
cudaError_t launch_bucket_place(const uint2* in, uint64_t count, const IdMap& ids,
                                const BucketPlan& plan, const void* scratch, const uint64_t* dst_off,
                                uint2* const* outs, uint32_t bins_per_out, uint32_t* err_dev,
                                cudaStream_t s, int* launches);

// Vertex-tile order (reading R-VTILE, gv_options.vertex_tile): every block
// segment [seg_off[k], seg_off[k+1]) of buf (local ids; its vertex partition
// has seg_rows[k] rows) is stably sorted by the tile u_local >> tile_bits —
// an LSD radix sort over the tile number in passes of <= 256 bins (one pass
// up to 256 tiles per partition, two up to 65536, three up to 2^24, four beyond), ping-ponging
// through tmp (same size as buf); the result is in buf. seg_off / seg_rows
// are HOST arrays (nseg + 1 / nseg); scratch of tile_sort_scratch_bytes.
size_t tile_sort_scratch_bytes(const uint64_t* seg_off, const uint64_t* seg_rows, uint32_t nseg,
                               uint32_t tile_bits);
cudaError_t launch_tile_sort(uint2* buf, uint2* tmp, const uint64_t* seg_off,
                             const uint64_t* seg_rows, uint32_t nseg, uint32_t tile_bits,
                             void* scratch, cudaStream_t s, int* launches);

}  // namespace gv
