// engine.hpp — internal state of a gv_ctx, shared by the engine's parts:
//   engine.cpp        pool preparation (a3-a6), offset steps (a7-a8), stats, C ABI
//   transport.hpp/    the exchange steps between the D ranks of Alg. 3
//   transport_*.cpp behind one interface: virtual ranks on one
//                     GPU (device copies) or processes (CUDA IPC)
//   outofcore.cpp     host-resident partitions on one GPU (NEXT-3)
// Not part of the ABI (include/gv.h is).
#pragma once
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <condition_variable>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/gv.h"
#include "augment.hpp"
#include "graph_share.hpp"
#include "host_graph.hpp"
#include "kernels.cuh"

namespace gv {

// NVTX ranges around the stages (visible in Nsight Systems timelines)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t cap = 0;     // elements
  uint64_t gen = 0;   // bumped by every (re)allocation
  bool host = false;  // pinned, mapped host memory (kernels read it over PCIe / UVA)
  size_t bytes_total() const { return cap * sizeof(T); }
  cudaError_t ensure(size_t n) {
    if (n <= cap) return cudaSuccess;
    release();
    const size_t bytes = (n > 0 ? n : 1) * sizeof(T);
    cudaError_t e = host ? cudaHostAlloc(&p, bytes, cudaHostAllocMapped | cudaHostAllocPortable)
                         : cudaMalloc(&p, bytes);
    if (e == cudaSuccess) {
      cap = n > 0 ? n : 1;
      ++gen;
    } else {
      p = nullptr;
    }
    return e;
  }
  void release() {
    if (p) {
      if (host) cudaFreeHost(p);
      else cudaFree(p);
    }
    p = nullptr;
    cap = 0;
  }
};

// One rank of Alg. 3: vertex partitions [d m, (d+1) m), a sliding window of
// context partitions (m + 1 slots when D > 1), its block rows of the pool.
struct Rank {
  int d = 0;  // global rank index
  cudaStream_t compute = nullptr, comm = nullptr;
  float* vertex = nullptr;
  uint64_t vrow_first = 0, vrows = 0;  // new-id range of the vertex shard
  float* context = nullptr;
  uint64_t crows = 0, slot_rows = 0;
  std::vector<int> slot_of;  // partition -> context slot (D > 1)
  int free_slot = -1;
  DevBuf<uint2> blocks;
  DevBuf<uint2> blocks_alt;  // NEXT-1: the next pool, bucketed by the device sampler
  DevBuf<uint8_t> scratch;
  DevBuf<uint64_t> counts;      // [0, bins]: block_off; [bins+1]: error flag
  DevBuf<BlockDesc> desc;
  DevBuf<uint64_t> place_args;  // fused exchange: dst_off[bins] | outs[D] (device pointers)
  BucketPlan plan{};
  DevBuf<double> loss;
  DevBuf<unsigned long long> chunk_ctr;  // dynamic chunk schedule of the ring kernel
  DevBuf<uint2> tile_tmp;        // R-VTILE: ping-pong buffer of the vertex-tile sort
  DevBuf<uint8_t> tile_scratch;  // its per-tile counts, offsets, output pointers
  uint64_t* counts_host = nullptr;  // pinned
  std::vector<uint64_t> local_off;  // this rank's local block_off (bins + 1)
  std::vector<uint64_t> final_off;  // m*n + 1: layout of blocks (g, j) in `blocks`
  uint64_t seg_begin = 0, seg_count = 0;
  // events
  cudaEvent_t ev_start = nullptr, ev_bucket = nullptr, ev_exch = nullptr, ev_end = nullptr;
  cudaEvent_t ev_exch_sent = nullptr;
  std::vector<cudaEvent_t> ev_first_done, ev_recv, ev_sent;  // per step
  cudaEvent_t ev_last_recv = nullptr;  // rotation into the window of the next pool
  bool have_last_recv = false;
  std::vector<cudaEvent_t> ev_sgd;  // pairs (begin, end) per launch
  int sgd_launches = 0;
  int kernel_launches = 0;
  double ms_bucket = 0, ms_exchange = 0, ms_sgd = 0, ms_total = 0;
};

enum class PoolState { Idle, Prepared };

// Residency of one matrix (vertex or context) in out-of-core mode.
struct HpMat {
  static constexpr int S = 3;  // device slots
  int part[S] = {-1, -1, -1};  // partition held by each slot
  bool dirty[S] = {};          // device copy newer than the host copy
  uint64_t stamp[S] = {};      // last use (LRU)
  int last_block[S] = {-1, -1, -1};  // last block of this episode using the slot
  int prev = -1;               // slot of the previous block
  cudaEvent_t free_[S] = {}, saved[S] = {}, loaded[S] = {};
  std::vector<cudaEvent_t> part_saved;  // per partition: its last write-back done
};

class Transport;

}  // namespace gv

struct gv_ctx {
  // parameters
  uint32_t nv = 0, dim = 0, n = 1, K = 1;
  float lr0 = 0.025f;
  gv_lr_schedule alpha{GV_LR_LINEAR, 1e-4, 0};
  gv_options opt{};
  int D = 1;       // total ranks
  int local = 1;   // ranks driven by this process
  uint32_t m = 1;  // partitions per rank
  uint32_t stride = 0;
  int threads = 1;
  int sms = 148;
  int ring_dynamic = 1;  // GV_RING_DYN: warps claim chunks from a counter (0: static)
  int vtile_hint = 0;    // GV_VTILE_HINT: L2 hints with vertex tiles (vertex rows kept)
  uint32_t hot_rows = 0;  // L2 retention: local ids below this are evict_last
  std::string err;
  std::mutex err_mu;  // push may fail on a producer thread while the trainer runs
  bool loaded = false;
  // graph
  gv::HostGraph graph;
  gv::Partitioning part;
  gv::Arr<gv::ProbAlias> nalias;  // negative tables {prob, alias}, new-id order
  gv::WalkTables walks;
  gv::SharedMapping graph_map;    // node-shared graph segment (multi-process)
  // device copy of the walk tables (gv_augment_device), lazily uploaded
  uint64_t* d_woff = nullptr;
  uint32_t* d_wnbr = nullptr;
  uint2* d_walias = nullptr;
  uint2* d_dalias = nullptr;
  gv::DevBuf<uint2> shuf_tmp;  // random-shuffle ablation scratch
  // shared device tables
  uint32_t* d_packed = nullptr;    // original id -> part | local (ORIGINAL pool ids)
  uint64_t* d_part_off = nullptr;  // n + 1 partition offsets (RELABELED pool ids)
  uint2* d_alias = nullptr;
  uint32_t* d_inv_perm = nullptr;
  uint32_t* d_perm = nullptr;      // original -> new (device augmentation, RELABELED), lazily
  bool relabeled() const { return opt.pool_ids == GV_IDS_RELABELED; }
  // pool (a2): ONE raw buffer. gv_train_episode takes the pending pool out of
  // it (prepare), and the next push may refill it as soon as the bucketing
  // kernels have read it (raw_free) — a few ms into the pool's training — so
  // the H2D copy of pool k+1 still overlaps the SGD of pool k, and device
  // sample memory is raw + blocks = 2 P (not 3 P as with two raw buffers).
  std::mutex mu;
  std::condition_variable raw_cv;
  bool raw_busy = false;        // prepare has taken the pool, raw_free not yet recorded
  gv::DevBuf<uint2> raw;
  uint64_t raw_count = 0;       // pending samples in raw
  cudaEvent_t raw_ready = nullptr, raw_free = nullptr;
  bool have_last = false;       // raw still holds the last trained pool (replay)
  uint64_t last_count = 0;
  // Relabelled ids at n = 1 on one rank (swap_mode): a3 is the range check
  // alone, and the pool is trained where it was pushed — prepare swaps the
  // raw and block buffers instead of copying, so the last pool lives in the
  // block buffer and a replay re-arms it there (pending_in_blocks).
  bool pending_in_blocks = false;
  // NEXT-1 (gv_augment_device_blocks): the pending pool was generated and
  // bucketed on the device, into ranks[0].blocks_alt with its block offsets
  // and error flag in fused_off; prepare swaps it in without a bucket pass.
  bool fused_pending = false;
  uint64_t fused_count = 0;
  gv::DevBuf<uint64_t> fused_off;  // bins + 1 offsets, [bins + 1] = error flag
  gv::DevBuf<uint8_t> aug_scratch;  // walk cache + counts of the fused sampler
  cudaEvent_t fused_ready = nullptr;  // copy stream: the fused pool is complete
  cudaEvent_t alt_free = nullptr;     // compute stream: blocks_alt no longer read
  bool swap_mode() const {
    return relabeled() && n == 1 && D == 1 && !hp() && !raw.host;
  }
  cudaStream_t copy_stream = nullptr;
  gv::PoolState state = gv::PoolState::Idle;
  uint64_t pool_P = 0;        // samples of the prepared pool (this process)
  uint64_t pool_P_global = 0; // all ranks
  std::vector<uint64_t> global_counts;  // bins (sum over ranks)
  // progress
  uint64_t pool_index = 0;
  uint64_t samples_done = 0;  // global samples trained in earlier steps
  std::vector<gv::Rank> ranks;
  // exchanges between the ranks (virtual ranks or processes)
  std::unique_ptr<gv::Transport> tr;
  // out-of-core mode (host_partitions): matrices in pinned host memory, three
  // device slots per matrix; loads (H2D) and write-backs (D2H) run on their
  // own streams so the two PCIe directions overlap each other and the SGD
  float* h_vertex = nullptr;
  float* h_context = nullptr;
  gv::HpMat hpv, hpc;
  uint64_t hp_clock = 0;
  cudaStream_t hp_h2d = nullptr, hp_d2h = nullptr;
  bool hp() const { return opt.host_partitions != 0; }
  bool ipc() const { return opt.world_size > 1; }
};

namespace gv {

gv_status fail(gv_ctx* c, gv_status s, const std::string& msg);

#define GV_CK(call)                                                                         \
  do {                                                                                      \
    cudaError_t e_ = (call);                                                                \
    if (e_ != cudaSuccess)                                                                  \
      return ::gv::fail(c, GV_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

inline uint64_t psize(const gv_ctx* c, uint32_t p) { return c->part.off[p + 1] - c->part.off[p]; }
cudaEvent_t new_event(bool timing);
float elapsed(cudaEvent_t a, cudaEvent_t b);
gv_status sync_all(gv_ctx* c);

// ---- out-of-core mode (outofcore.cpp)
// The n^2 blocks of a pool in residency order, with the slot each block's
// partitions occupy and the loads / write-backs around it.
struct HpUse {
  int s, load;      // slot; partition to load into it (-1: resident)
  bool wait_saved;  // the slot's old contents are written back first
};
struct HpWb {
  int mat, s, p;  // write-back of slot s (partition p) of matrix mat
};
struct HpPlan {
  std::vector<std::pair<uint32_t, uint32_t>> order;  // (offset step t, vertex partition i)
  std::vector<HpUse> use[2];                         // per position in order
  std::vector<std::vector<HpWb>> wb;                 // wb[k + 1]: after the k-th block
  std::vector<int> pos;                              // position of block (t, i) in order
};
void hp_plan(gv_ctx* c, HpPlan* pl);
// allocates the host matrices and device slots of rank r, initialises them
gv_status hp_setup(gv_ctx* c, Rank& r);
// enqueues the pool's blocks with their loads and write-backs;
// launch(t, i) launches block (t, i)
template <class Launch>
gv_status hp_enqueue(gv_ctx* c, const HpPlan& pl, Launch&& launch);
// embeddings through the host copies (flushes the dirty resident partitions)
gv_status hp_embeddings_io(gv_ctx* c, bool context, float* out, const float* in);
void hp_destroy(gv_ctx* c);

// write-back of slot w.s of matrix w.mat to its host partition
gv_status hp_write_back(gv_ctx* c, const HpWb& w);
// loads of block k's partitions; the compute stream waits for them
gv_status hp_load(gv_ctx* c, const HpPlan& pl, size_t k);
// after block k: its slots are free, the write-backs scheduled after it go
gv_status hp_after_block(gv_ctx* c, const HpPlan& pl, size_t k);

template <class Launch>
gv_status hp_enqueue(gv_ctx* c, const HpPlan& pl, Launch&& launch) {
  for (const HpWb& w : pl.wb[0])  // victims last used in an earlier episode
    if (gv_status st = hp_write_back(c, w)) return st;
  for (size_t k = 0; k < pl.order.size(); ++k) {
    if (gv_status st = hp_load(c, pl, k)) return st;
    if (gv_status st = launch(pl.order[k].first, pl.order[k].second)) return st;
    if (gv_status st = hp_after_block(c, pl, k)) return st;
  }
  return GV_OK;
}

}  // namespace gv
