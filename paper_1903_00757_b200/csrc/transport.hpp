// transport.hpp — the exchange steps between the D ranks of Alg. 3
// (P:235-259), behind one interface so the schedule in engine.cpp is written
// once:
//   a4  all-gather of the per-rank bin counts (n^2 + 2 words per rank)
//   a6  the block-row exchange, fused into the scatter of a5: every source
//       stores its samples straight into the owners' receive buffers
//   a8  the context rotation after each offset step (rank d sends partition
//       (d m + t) mod n to rank d - 1 once its first block of step t is done)
// and the per-rank statistics of a pool.
//
// Two implementations:
//   LocalTransport  every rank lives in this process (D = 1, or
//                   virtual_ranks = D on one GPU): device-to-device copies
//                   and CUDA events between the ranks' streams.
//   IpcTransport    one process per rank (world_size = D): CUDA IPC peer
//                   memory (NVLink 5 / NVSwitch across GPUs) with a POSIX
//                   shared-memory segment of epoch counters as the host-side
//                   handshake; rank 0 also prepares the host graph once for
//                   the node and shares it.
#pragma once
#include <array>
#include <functional>
#include <memory>
#include <vector>

#include "engine.hpp"

namespace gv {

class Transport {
 public:
  virtual ~Transport() = default;
  // gv_load_edges: run `prepare` (the host graph preparation) or map the
  // copy another rank prepared
  virtual gv_status load_graph(gv_ctx* c, const std::function<gv_status()>& prepare) = 0;
  // after setup_device: export / map device buffers and events
  virtual gv_status connect(gv_ctx* c) = 0;
  // a4: cnt[d] = block offsets (bins + 1 words) and error flag of rank d's
  // pool segment, for all D ranks. Enqueued bucketing must be complete on return.
  virtual gv_status gather_counts(gv_ctx* c, std::vector<std::vector<uint64_t>>& cnt) = 0;
  // a6: grow rank r's receive buffer to hold `total` samples
  virtual gv_status reserve_blocks(gv_ctx* c, Rank& r, uint64_t total) = 0;
  // a6: outs[d] = receive buffer of rank d, addressable from this process
  virtual gv_status scatter_targets(gv_ctx* c, std::vector<uint2*>& outs) = 0;
  // a6: every local owner's compute stream waits for every source's scatter
  virtual gv_status scatter_done(gv_ctx* c) = 0;
  // a8: rank r has enqueued block 0 of offset step t (send_part is final
  // once it completes)
  virtual gv_status first_block_done(gv_ctx* c, Rank& r, uint32_t t) = 0;
  // a8: enqueue the rotation of offset step t for every local rank and
  // update their slot maps
  virtual gv_status rotate(gv_ctx* c, uint32_t t) = 0;
  // per-rank device times of the last pool: v[d] = {total, bucket,
  // exchange, sgd, rotate} for all D ranks (local ranks are filled in)
  virtual gv_status exchange_stats(gv_ctx* c, std::vector<std::array<double, 5>>& v) = 0;
  // gv_set_progress: may the pool counter jump to pool_index now?
  virtual gv_status set_progress(gv_ctx* c, uint64_t pool_index) = 0;
  // gv_destroy, after the local streams drained: wait until no peer can
  // still read this process's exported memory, then release the mappings
  virtual void close(gv_ctx* c) = 0;
};

std::unique_ptr<Transport> make_local_transport();
// id: the 128-byte unique id every rank received (gv_comm_unique_id)
gv_status make_ipc_transport(gv_ctx* c, const uint8_t id[128], std::unique_ptr<Transport>* out);

}  // namespace gv
