// transport_ipc.cpp — one process per rank (transport.hpp), CUDA IPC.
//
// Every rank exports its context buffer, its receive buffer and IPC events;
// sources STORE their samples into the owners' receive buffers (the fused
// scatter of a5 + a6), and the RECEIVER PULLS the context partition of each
// rotation with cudaMemcpyAsync out of the peer's mapped memory (copy
// engines over NVLink 5 / NVSwitch across GPUs, on-device when the
// processes share a GPU). A cross-process cudaStreamWaitEvent is issued only
// after the peer has RECORDED the event, which the peer announces through
// per-rank epoch counters in a POSIX shared-memory segment (ipc.hpp);
// per-step events form a ring of kIpcEvRing so a fast peer can never
// re-record the event a slow peer is about to wait on.
#include <sys/mman.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "ipc.hpp"
#include "transport.hpp"

namespace gv {

namespace {

class IpcTransport final : public Transport {
 public:
  IpcShm* shm = nullptr;
  std::string shm_name;
  std::string graph_shm_name;  // node-shared graph segment (rank 0 prepares it)
  double timeout = 300.0;
  uint64_t epoch0 = 0;  // pool counter of this session's first pool (gv_set_progress)
  float* peer_ctx[kIpcMaxRanks] = {};
  uint2* peer_blocks[kIpcMaxRanks] = {};
  uint64_t peer_blocks_gen[kIpcMaxRanks] = {};
  cudaEvent_t peer_ev_pull[kIpcMaxRanks][2] = {};
  cudaEvent_t peer_ev_first[kIpcMaxRanks][kIpcEvRing] = {};
  cudaEvent_t peer_ev_rot[kIpcMaxRanks][kIpcEvRing] = {};
  cudaEvent_t my_ev_pull[2] = {};
  cudaEvent_t my_ev_first[kIpcEvRing] = {};
  cudaEvent_t my_ev_rot[kIpcEvRing] = {};
  uint64_t exported_blocks_gen = 0;
  // receive buffers replaced while peers had them mapped: freed once every
  // peer has moved past the pool that announced the new handle
  std::vector<std::pair<uint2*, uint64_t>> graveyard;  // (ptr, retired at pool e)

  IpcRankShm& me(gv_ctx* c) { return shm->rank[c->ranks[0].d]; }

  gv_status load_graph(gv_ctx* c, const std::function<gv_status()>& prepare) override {
    // rank 0 prepares the graph once for the node and shares it (graph_share.hpp)
    GraphParts parts{&c->graph, &c->part, &c->nalias, &c->walks};
    graph_shm_name = shm_name + "_graph";
    if (c->opt.rank == 0) {
      gv_status st = prepare();
      if (st == GV_OK) {
        std::string msg;
        if (int rc = graph_share_publish(graph_shm_name, parts, &c->graph_map, &msg))
          st = fail(c, static_cast<gv_status>(rc), msg);
      }
      shm->graph_state.store(st == GV_OK ? 1 : 2 + st, std::memory_order_release);
      return st;
    }
    // a graph preparation takes minutes on the largest graphs: wait longer
    if (!ipc_wait(shm->graph_state, 1, std::max(timeout, 3600.0)))
      return fail(c, GV_ERR_COMM, "IPC timeout waiting for rank 0 to prepare the graph");
    const uint64_t state = shm->graph_state.load(std::memory_order_acquire);
    if (state >= 2)
      return fail(c, static_cast<gv_status>(state - 2), "rank 0 failed to prepare the graph");
    c->graph.nv = c->nv;
    c->part.n = c->n;
    std::string msg;
    if (int rc = graph_share_attach(graph_shm_name, parts, &c->graph_map, &msg))
      return fail(c, static_cast<gv_status>(rc), msg);
    return GV_OK;
  }

  gv_status connect(gv_ctx* c) override {
    // export the context buffer and the events, map the peers'
    Rank& r = c->ranks[0];
    IpcRankShm& mine = me(c);
    const unsigned fl = cudaEventInterprocess | cudaEventDisableTiming;
    for (int k = 0; k < 2; ++k) {
      GV_CK(cudaEventCreateWithFlags(&my_ev_pull[k], fl));
      GV_CK(cudaIpcGetEventHandle(&mine.ev_pull[k], my_ev_pull[k]));
    }
    for (int k = 0; k < kIpcEvRing; ++k) {
      GV_CK(cudaEventCreateWithFlags(&my_ev_first[k], fl));
      GV_CK(cudaEventCreateWithFlags(&my_ev_rot[k], fl));
      GV_CK(cudaIpcGetEventHandle(&mine.ev_first[k], my_ev_first[k]));
      GV_CK(cudaIpcGetEventHandle(&mine.ev_rot[k], my_ev_rot[k]));
    }
    GV_CK(cudaIpcGetMemHandle(&mine.ctx_handle, r.context));
    mine.joined.store(1, std::memory_order_release);
    for (int q = 0; q < c->D; ++q) {
      if (!ipc_wait(shm->rank[q].joined, 1, timeout))
        return fail(c, GV_ERR_COMM, "IPC timeout waiting for the peers to load the graph");
      if (q == r.d) continue;
      IpcRankShm& pr = shm->rank[q];
      void* ptr = nullptr;
      GV_CK(cudaIpcOpenMemHandle(&ptr, pr.ctx_handle, cudaIpcMemLazyEnablePeerAccess));
      peer_ctx[q] = static_cast<float*>(ptr);
      for (int k = 0; k < 2; ++k) GV_CK(cudaIpcOpenEventHandle(&peer_ev_pull[q][k], pr.ev_pull[k]));
      for (int k = 0; k < kIpcEvRing; ++k) {
        GV_CK(cudaIpcOpenEventHandle(&peer_ev_first[q][k], pr.ev_first[k]));
        GV_CK(cudaIpcOpenEventHandle(&peer_ev_rot[q][k], pr.ev_rot[k]));
      }
    }
    mine.joined.store(2, std::memory_order_release);
    if (r.d == 0) {  // everyone mapped everything: the names are no longer needed
      for (int q = 0; q < c->D; ++q)
        if (!ipc_wait(shm->rank[q].joined, 2, timeout))
          return fail(c, GV_ERR_COMM, "IPC timeout in the init handshake");
      shm_unlink(shm_name.c_str());
      graph_share_unlink(graph_shm_name);
    }
    return GV_OK;
  }

  gv_status gather_counts(gv_ctx* c, std::vector<std::vector<uint64_t>>& cnt) override {
    // all-gathered through the shared-memory segment
    Rank& r = c->ranks[0];
    const uint64_t e = c->pool_index;
    const size_t words = static_cast<size_t>(c->n) * c->n + 2;
    GV_CK(cudaMemcpyAsync(r.counts_host, r.counts.p, sizeof(uint64_t) * words,
                          cudaMemcpyDeviceToHost, r.compute));
    GV_CK(cudaStreamSynchronize(r.compute));
    IpcRankShm& mine = me(c);
    std::memcpy(mine.counts[e & 1], r.counts_host, sizeof(uint64_t) * words);
    mine.counts_epoch.store(e + 1, std::memory_order_release);
    for (int q = 0; q < c->D; ++q) {
      if (!ipc_wait(shm->rank[q].counts_epoch, e + 1, timeout))
        return fail(c, GV_ERR_COMM, "IPC timeout waiting for a peer's bucket counts");
      std::memcpy(cnt[q].data(), shm->rank[q].counts[e & 1], sizeof(uint64_t) * words);
    }
    return GV_OK;
  }

  gv_status reserve_blocks(gv_ctx* c, Rank& r, uint64_t total) override {
    if (total <= r.blocks.cap) return GV_OK;
    if (r.blocks.p) {  // peers may still map it: retire, free later
      graveyard.push_back({r.blocks.p, c->pool_index});
      r.blocks.p = nullptr;
      r.blocks.cap = 0;
    }
    GV_CK(r.blocks.ensure(total + total / 8));  // pool sizes fluctuate
    return GV_OK;
  }

  gv_status scatter_targets(gv_ctx* c, std::vector<uint2*>& outs) override {
    Rank& r = c->ranks[0];
    const uint64_t e = c->pool_index;
    IpcRankShm& mine = me(c);
    if (exported_blocks_gen != r.blocks.gen) {  // (re)allocated: export again
      GV_CK(cudaIpcGetMemHandle(&mine.blocks_handle, r.blocks.p));
      mine.blocks_gen = mine.blocks_gen + 1;
      exported_blocks_gen = r.blocks.gen;
    }
    mine.recv_epoch.store(e + 1, std::memory_order_release);
    for (int q = 0; q < c->D; ++q) {
      if (q == r.d) {
        outs[q] = r.blocks.p;
        continue;
      }
      IpcRankShm& pr = shm->rank[q];
      if (!ipc_wait(pr.recv_epoch, e + 1, timeout))
        return fail(c, GV_ERR_COMM, "IPC timeout waiting for a peer's receive buffer");
      if (peer_blocks_gen[q] != pr.blocks_gen) {
        if (peer_blocks[q]) GV_CK(cudaIpcCloseMemHandle(peer_blocks[q]));
        void* ptr = nullptr;
        GV_CK(cudaIpcOpenMemHandle(&ptr, pr.blocks_handle, cudaIpcMemLazyEnablePeerAccess));
        peer_blocks[q] = static_cast<uint2*>(ptr);
        peer_blocks_gen[q] = pr.blocks_gen;
      }
      outs[q] = peer_blocks[q];
    }
    // every peer has moved past the pools that announced newer handles
    for (auto it = graveyard.begin(); it != graveyard.end();) {
      if (it->second + 1 < e + 1) {
        GV_CK(cudaFree(it->first));
        it = graveyard.erase(it);
      } else {
        ++it;
      }
    }
    return GV_OK;
  }

  gv_status scatter_done(gv_ctx* c) override {
    // an owner trains its rows only after every source has placed its samples
    Rank& r = c->ranks[0];
    const uint64_t e = c->pool_index;
    GV_CK(cudaEventRecord(my_ev_pull[e & 1], r.compute));
    me(c).pull_epoch.store(e + 1, std::memory_order_release);
    for (int q = 0; q < c->D; ++q) {
      if (q == r.d) continue;
      if (!ipc_wait(shm->rank[q].pull_epoch, e + 1, timeout))
        return fail(c, GV_ERR_COMM, "IPC timeout waiting for a peer's scatter");
      GV_CK(cudaStreamWaitEvent(r.compute, peer_ev_pull[q][e & 1], 0));
    }
    return GV_OK;
  }

  gv_status first_block_done(gv_ctx* c, Rank& r, uint32_t t) override {
    // publish "block 0 of global step gs done" and the slot to pull
    gv_step_plan plan;
    gv_plan_step(c->n, c->D, r.d, t, &plan);
    const uint64_t gs = c->pool_index * c->n + t;
    GV_CK(cudaEventRecord(my_ev_first[gs % kIpcEvRing], r.compute));
    IpcRankShm& mine = me(c);
    mine.first_slot[gs % kIpcSlotRing] = static_cast<uint32_t>(r.slot_of[plan.send_part]);
    mine.first_epoch.store(gs + 1, std::memory_order_release);
    return GV_OK;
  }

  gv_status rotate(gv_ctx* c, uint32_t t) override {
    // receiver pulls: rank d copies recv_part out of rank d+1's context slots
    Rank& r = c->ranks[0];
    const uint32_t n = c->n;
    gv_step_plan plan;
    gv_plan_step(n, c->D, r.d, t, &plan);
    const uint64_t gs = c->pool_index * n + t;
    const int src = static_cast<int>(plan.recv_from), prev = static_cast<int>(plan.send_to);
    IpcRankShm& ps = shm->rank[src];
    if (!ipc_wait(ps.first_epoch, gs + 1, timeout))
      return fail(c, GV_ERR_COMM, "IPC timeout waiting for the successor's first block");
    const uint32_t peer_slot = ps.first_slot[gs % kIpcSlotRing];
    GV_CK(cudaStreamWaitEvent(r.comm, peer_ev_first[src][gs % kIpcEvRing], 0));
    if (gs > epoch0 * n) {  // our free slot was pulled by the predecessor at the previous step
      if (!ipc_wait(shm->rank[prev].rot_epoch, gs, timeout))
        return fail(c, GV_ERR_COMM, "IPC timeout waiting for the predecessor's rotation");
      GV_CK(cudaStreamWaitEvent(r.comm, peer_ev_rot[prev][(gs - 1) % kIpcEvRing], 0));
    }
    const uint32_t out_p = plan.send_part, in_p = plan.recv_part;
    GV_CK(cudaMemcpyAsync(
        r.context + static_cast<uint64_t>(r.free_slot) * r.slot_rows * c->stride,
        peer_ctx[src] + static_cast<uint64_t>(peer_slot) * r.slot_rows * c->stride,
        psize(c, in_p) * c->stride * sizeof(float), cudaMemcpyDeviceToDevice, r.comm));
    GV_CK(cudaEventRecord(my_ev_rot[gs % kIpcEvRing], r.comm));
    me(c).rot_epoch.store(gs + 1, std::memory_order_release);
    GV_CK(cudaEventRecord(r.ev_recv[t], r.comm));
    const int s_out = r.slot_of[out_p];
    r.slot_of[in_p] = r.free_slot;
    r.slot_of[out_p] = -1;
    r.free_slot = s_out;
    return GV_OK;
  }

  gv_status exchange_stats(gv_ctx* c, std::vector<std::array<double, 5>>& v) override {
    // processes exchange their device times through the segment, so every
    // rank reports all D ranks and their maximum
    const int d = c->ranks[0].d;
    const uint64_t e = c->pool_index - 1;
    IpcRankShm& mine = me(c);
    std::memcpy(mine.stats[e % kIpcStatRing], v[d].data(), sizeof(double) * 5);
    mine.stats_epoch.store(e + 1, std::memory_order_release);
    for (int q = 0; q < c->D; ++q) {
      if (q == d) continue;
      IpcRankShm& pr = shm->rank[q];
      if (!ipc_wait(pr.stats_epoch, e + 1, timeout))
        return fail(c, GV_ERR_COMM, "IPC timeout waiting for a peer's pool statistics");
      std::memcpy(v[q].data(), pr.stats[e % kIpcStatRing], sizeof(double) * 5);
    }
    return GV_OK;
  }

  gv_status set_progress(gv_ctx* c, uint64_t pool_index) override {
    // the pool counter also numbers the handshake epochs: ranks may only
    // jump to a resumed position together, before their first pool
    std::lock_guard<std::mutex> lk(c->mu);
    if (c->pool_index != 0 || c->raw_count != 0 || c->have_last)
      return fail(c, GV_ERR_STATE, "multi-process: set progress before the first pool is pushed");
    epoch0 = pool_index;
    return GV_OK;
  }

  void close(gv_ctx* c) override {
    if (!c->ranks.empty() && shm) {
      // Peers pull context partitions out of this rank's exported buffer (the
      // last rotation of a pool lands on the peer's stream after our first
      // block of that step): free it only once every peer has drained its
      // own streams, which it announces here after its synchronisation.
      me(c).closed.store(1, std::memory_order_release);
      for (int q = 0; q < c->D; ++q)
        if (!ipc_wait(shm->rank[q].closed, 1, timeout))
          fprintf(stderr, "gv_destroy: rank %d did not close within the IPC timeout\n", q);
    }
    for (auto& g : graveyard) cudaFree(g.first);
    graveyard.clear();
    for (int q = 0; q < kIpcMaxRanks; ++q) {
      if (peer_ctx[q]) cudaIpcCloseMemHandle(peer_ctx[q]);
      if (peer_blocks[q]) cudaIpcCloseMemHandle(peer_blocks[q]);
      peer_ctx[q] = nullptr;
      peer_blocks[q] = nullptr;
    }
    for (cudaEvent_t e : my_ev_pull) if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : my_ev_first) if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : my_ev_rot) if (e) cudaEventDestroy(e);
    if (shm) ipc_close(shm, shm_name, false);
    shm = nullptr;
    if (c->opt.rank == 0 && !graph_shm_name.empty()) graph_share_unlink(graph_shm_name);
  }
};

}  // namespace

gv_status make_ipc_transport(gv_ctx* c, const uint8_t id[128], std::unique_ptr<Transport>* out) {
  if (c->D > kIpcMaxRanks || c->n * c->n + 2 > static_cast<uint32_t>(kIpcMaxBins))
    return fail(c, GV_ERR_INVALID_ARG, "IPC transport: at most 16 ranks and 64 partitions");
  auto t = std::make_unique<IpcTransport>();
  std::string err;
  t->shm = ipc_open(id, &t->shm_name, &err);
  if (!t->shm) return fail(c, GV_ERR_COMM, err);
  if (const char* s = getenv("GV_IPC_TIMEOUT")) t->timeout = atof(s);
  *out = std::move(t);
  return GV_OK;
}

}  // namespace gv
