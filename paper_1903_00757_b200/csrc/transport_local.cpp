// transport_local.cpp — every rank in this process (transport.hpp):
// D = 1, or virtual_ranks = D ranks sharing this process's GPU. The
// exchanges are device-to-device copies and CUDA events between the ranks'
// streams; the counts "all-gather" is a read of each rank's counts.
#include <algorithm>

#include "transport.hpp"

namespace gv {

namespace {

class LocalTransport final : public Transport {
 public:
  gv_status load_graph(gv_ctx*, const std::function<gv_status()>& prepare) override {
    return prepare();
  }

  gv_status connect(gv_ctx*) override { return GV_OK; }

  gv_status gather_counts(gv_ctx* c, std::vector<std::vector<uint64_t>>& cnt) override {
    const size_t words = static_cast<size_t>(c->n) * c->n + 2;
    for (auto& r : c->ranks)
      GV_CK(cudaMemcpyAsync(r.counts_host, r.counts.p, sizeof(uint64_t) * words,
                            cudaMemcpyDeviceToHost, r.compute));
    for (auto& r : c->ranks) {
      GV_CK(cudaStreamSynchronize(r.compute));
      std::copy(r.counts_host, r.counts_host + words, cnt[r.d].begin());
    }
    return GV_OK;
  }

  gv_status reserve_blocks(gv_ctx* c, Rank& r, uint64_t total) override {
    if (total > r.blocks.cap) GV_CK(r.blocks.ensure(total + total / 8));  // pool sizes fluctuate
    return GV_OK;
  }

  gv_status scatter_targets(gv_ctx* c, std::vector<uint2*>& outs) override {
    for (auto& r : c->ranks) outs[r.d] = r.blocks.p;
    return GV_OK;
  }

  gv_status scatter_done(gv_ctx* c) override {
    for (auto& d : c->ranks)
      for (auto& s : c->ranks)
        if (s.d != d.d) GV_CK(cudaStreamWaitEvent(d.compute, s.ev_exch_sent, 0));
    return GV_OK;
  }

  gv_status first_block_done(gv_ctx*, Rank&, uint32_t) override { return GV_OK; }

  gv_status rotate(gv_ctx* c, uint32_t t) override {
    // device copies between the ranks; slot moves computed first
    const uint32_t n = c->n;
    std::vector<int> dst_slot(c->D), src_slot(c->D);
    std::vector<gv_step_plan> plans(c->D);
    for (auto& r : c->ranks) {
      gv_plan_step(n, c->D, r.d, t, &plans[r.d]);
      src_slot[r.d] = r.slot_of[plans[r.d].send_part];
      dst_slot[r.d] = r.free_slot;  // where rank r receives
    }
    for (auto& r : c->ranks) {
      Rank& prev = c->ranks[plans[r.d].send_to];
      const uint32_t out_p = plans[r.d].send_part;
      GV_CK(cudaStreamWaitEvent(r.comm, r.ev_first_done[t], 0));
      // prev's free slot was released by prev's own send of step t-1
      if (t > 0) GV_CK(cudaStreamWaitEvent(r.comm, prev.ev_sent[t - 1], 0));
      else if (prev.have_last_recv) GV_CK(cudaStreamWaitEvent(r.comm, prev.ev_last_recv, 0));
      GV_CK(cudaMemcpyAsync(
          prev.context + static_cast<uint64_t>(dst_slot[prev.d]) * prev.slot_rows * c->stride,
          r.context + static_cast<uint64_t>(src_slot[r.d]) * r.slot_rows * c->stride,
          psize(c, out_p) * c->stride * sizeof(float), cudaMemcpyDeviceToDevice, r.comm));
      GV_CK(cudaEventRecord(r.ev_sent[t], r.comm));
      GV_CK(cudaEventRecord(prev.ev_recv[t], r.comm));
    }
    for (auto& r : c->ranks) {
      const uint32_t out_p = plans[r.d].send_part, in_p = plans[r.d].recv_part;
      r.slot_of[in_p] = dst_slot[r.d];
      r.slot_of[out_p] = -1;
      r.free_slot = src_slot[r.d];
    }
    return GV_OK;
  }

  gv_status exchange_stats(gv_ctx*, std::vector<std::array<double, 5>>&) override {
    return GV_OK;  // every rank is local
  }

  gv_status set_progress(gv_ctx*, uint64_t) override { return GV_OK; }

  void close(gv_ctx*) override {}
};

}  // namespace

std::unique_ptr<Transport> make_local_transport() { return std::make_unique<LocalTransport>(); }

}  // namespace gv
