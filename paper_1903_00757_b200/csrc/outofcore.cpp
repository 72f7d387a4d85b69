// outofcore.cpp — host-resident partitions on one GPU (NEXT-3, SURVEY §8(f);
// Alg. 3: the paper keeps the matrices in host memory and sends
// the partitions of each block to the GPU). Both matrices live in pinned
// host memory in relabelled order; the device holds three slots per matrix.
// Before block (i, j) its vertex partition i and context partition j are
// loaded into slots; a slot's partition is written back after its last use
// in the pool. Loads (H2D) and write-backs (D2H) run on their own streams so
// the two PCIe directions overlap each other and the SGD.
#include <cstring>

#include "engine.hpp"

namespace gv {

void hp_plan(gv_ctx* c, HpPlan* pl) {
  const uint32_t n = c->n;
  pl->order.clear();
  // Block order: Alg. 3 orders blocks by offset step; a block (i, i+t)
  // depends only on the blocks sharing its rows, (i, i+t-1) and (i+1, i+t)
  // of step t-1, so any order respecting those edges gives the same result.
  // Steps are taken in pairs (t, t+1) as A_{n-1}, A_{n-2}, B_{n-2}, ...,
  // A_0, B_0, B_{n-1} (A_i = (i, i+t), B_i = (i, i+t+1)): B_i shares its
  // vertex partition with A_i and its context partition with A_{i+1}, so
  // with three slots per matrix a block loads one partition instead of two.
  for (uint32_t t = 0; t < n; t += 2) {
    if (t + 1 == n) {
      for (uint32_t i = 0; i < n; ++i) pl->order.push_back({t, i});
      break;
    }
    pl->order.push_back({t, n - 1});
    for (uint32_t i = n - 1; i-- > 0;) {
      pl->order.push_back({t, i});
      pl->order.push_back({t + 1, i});
    }
    pl->order.push_back({t + 1, n - 1});
  }
  // LRU over three slots, never the previous block's slot (it may still
  // run). A victim's write-back is issued right after its last use, so it
  // runs during the next block while another slot loads (PCIe duplex).
  pl->wb.assign(static_cast<size_t>(n) * n + 1, {});
  HpMat* mats[2] = {&c->hpv, &c->hpc};
  for (HpMat* M : mats)
    for (int sl = 0; sl < HpMat::S; ++sl) M->last_block[sl] = -1;
  for (int mt = 0; mt < 2; ++mt) pl->use[mt].resize(static_cast<size_t>(n) * n);
  for (size_t k = 0; k < pl->order.size(); ++k) {
    const uint32_t t = pl->order[k].first, i = pl->order[k].second;
    const int b = static_cast<int>(k);
    const int need[2] = {static_cast<int>(i), static_cast<int>((i + t) % n)};
    for (int mt = 0; mt < 2; ++mt) {
      HpMat& M = *mats[mt];
      HpUse& u = pl->use[mt][b];
      u.s = -1;
      u.load = -1;
      u.wait_saved = false;
      for (int sl = 0; sl < HpMat::S; ++sl)
        if (M.part[sl] == need[mt]) u.s = sl;
      if (u.s < 0) {
        for (int sl = 0; sl < HpMat::S; ++sl)
          if (sl != M.prev && (u.s < 0 || M.stamp[sl] < M.stamp[u.s])) u.s = sl;
        if (M.part[u.s] >= 0 && M.dirty[u.s]) {
          pl->wb[M.last_block[u.s] + 1].push_back({mt, u.s, M.part[u.s]});
          u.wait_saved = true;
        }
        u.load = need[mt];
        M.part[u.s] = need[mt];
      }
      M.dirty[u.s] = true;
      M.stamp[u.s] = ++c->hp_clock;
      M.last_block[u.s] = b;
      M.prev = u.s;
    }
  }
  pl->pos.assign(pl->order.size(), 0);
  for (size_t k = 0; k < pl->order.size(); ++k)
    pl->pos[pl->order[k].first * n + pl->order[k].second] = static_cast<int>(k);
}

namespace {

float* slot_ptr(gv_ctx* c, int mt, int sl) {
  Rank& r = c->ranks[0];
  return (mt == 0 ? r.vertex : r.context) + static_cast<uint64_t>(sl) * r.slot_rows * c->stride;
}

}  // namespace

gv_status hp_write_back(gv_ctx* c, const HpWb& w) {
  HpMat& M = w.mat == 0 ? c->hpv : c->hpc;
  float* host = w.mat == 0 ? c->h_vertex : c->h_context;
  GV_CK(cudaStreamWaitEvent(c->hp_d2h, M.free_[w.s], 0));
  GV_CK(cudaMemcpyAsync(host + c->part.off[w.p] * c->stride, slot_ptr(c, w.mat, w.s),
                        sizeof(float) * c->stride * psize(c, w.p), cudaMemcpyDeviceToHost,
                        c->hp_d2h));
  GV_CK(cudaEventRecord(M.saved[w.s], c->hp_d2h));
  GV_CK(cudaEventRecord(M.part_saved[w.p], c->hp_d2h));
  return GV_OK;
}

gv_status hp_load(gv_ctx* c, const HpPlan& pl, size_t k) {
  Rank& r = c->ranks[0];
  for (int mt = 0; mt < 2; ++mt) {
    const HpUse& u = pl.use[mt][k];
    HpMat& M = mt == 0 ? c->hpv : c->hpc;
    float* host = mt == 0 ? c->h_vertex : c->h_context;
    if (u.load >= 0) {
      GV_CK(cudaStreamWaitEvent(c->hp_h2d, M.free_[u.s], 0));
      if (u.wait_saved) GV_CK(cudaStreamWaitEvent(c->hp_h2d, M.saved[u.s], 0));
      // the host copy of the partition is current (a per-partition event:
      // a slot's own event is re-recorded by later write-backs)
      GV_CK(cudaStreamWaitEvent(c->hp_h2d, M.part_saved[u.load], 0));
      GV_CK(cudaMemcpyAsync(slot_ptr(c, mt, u.s), host + c->part.off[u.load] * c->stride,
                            sizeof(float) * c->stride * psize(c, u.load), cudaMemcpyHostToDevice,
                            c->hp_h2d));
      GV_CK(cudaEventRecord(M.loaded[u.s], c->hp_h2d));
    }
    GV_CK(cudaStreamWaitEvent(r.compute, M.loaded[u.s], 0));
  }
  return GV_OK;
}

gv_status hp_after_block(gv_ctx* c, const HpPlan& pl, size_t k) {
  Rank& r = c->ranks[0];
  GV_CK(cudaEventRecord(c->hpv.free_[pl.use[0][k].s], r.compute));
  GV_CK(cudaEventRecord(c->hpc.free_[pl.use[1][k].s], r.compute));
  for (const HpWb& w : pl.wb[k + 1])
    if (gv_status st = hp_write_back(c, w)) return st;
  return GV_OK;
}

gv_status hp_setup(gv_ctx* c, Rank& r) {
  const uint32_t nv = c->nv, n = c->n;
  const uint32_t key0 = static_cast<uint32_t>(c->opt.init_seed);
  const uint32_t key1 = static_cast<uint32_t>(c->opt.init_seed >> 32);
  const uint64_t max_part = c->part.max_part();
  const size_t hbytes = sizeof(float) * static_cast<size_t>(nv) * c->stride;
  GV_CK(cudaHostAlloc(&c->h_vertex, hbytes, cudaHostAllocDefault));
  GV_CK(cudaHostAlloc(&c->h_context, hbytes, cudaHostAllocDefault));
  std::memset(c->h_context, 0, hbytes);
  r.slot_rows = max_part;
  r.vrows = HpMat::S * max_part;
  r.crows = HpMat::S * max_part;
  GV_CK(cudaMalloc(&r.vertex, sizeof(float) * r.vrows * c->stride));
  GV_CK(cudaMalloc(&r.context, sizeof(float) * r.crows * c->stride));
  GV_CK(cudaMemset(r.vertex, 0, sizeof(float) * r.vrows * c->stride));
  for (uint32_t p = 0; p < n; ++p) {  // Philox init partition by partition
    GV_CK(launch_init_vertex(r.vertex, c->stride, c->dim, c->part.off[p], psize(c, p),
                             c->d_inv_perm, key0, key1, r.compute));
    GV_CK(cudaMemcpyAsync(c->h_vertex + c->part.off[p] * c->stride, r.vertex,
                          sizeof(float) * psize(c, p) * c->stride, cudaMemcpyDeviceToHost,
                          r.compute));
    GV_CK(cudaStreamSynchronize(r.compute));
  }
  GV_CK(cudaStreamCreateWithFlags(&c->hp_h2d, cudaStreamNonBlocking));
  GV_CK(cudaStreamCreateWithFlags(&c->hp_d2h, cudaStreamNonBlocking));
  for (HpMat* M : {&c->hpv, &c->hpc}) {
    M->part_saved.resize(n);
    for (cudaEvent_t& e : M->part_saved) {
      e = new_event(false);
      GV_CK(cudaEventRecord(e, r.compute));
    }
    for (int k = 0; k < HpMat::S; ++k) {
      for (cudaEvent_t* e : {&M->free_[k], &M->saved[k], &M->loaded[k]}) {
        *e = new_event(false);
        GV_CK(cudaEventRecord(*e, r.compute));
      }
    }
  }
  r.vrow_first = 0;
  return GV_OK;
}

gv_status hp_embeddings_io(gv_ctx* c, bool context, float* out, const float* in) {
  // flush the resident (dirty) partitions, then use the host copy
  Rank& r = c->ranks[0];
  const uint32_t dim = c->dim, stride = c->stride;
  float* host = context ? c->h_context : c->h_vertex;
  HpMat& M = context ? c->hpc : c->hpv;
  for (int sl = 0; sl < HpMat::S; ++sl) {
    const int p = M.part[sl];
    if (p < 0) continue;
    float* slot = (context ? r.context : r.vertex) + static_cast<uint64_t>(sl) * r.slot_rows * stride;
    if (out && M.dirty[sl])
      GV_CK(cudaMemcpy(host + c->part.off[p] * stride, slot, sizeof(float) * psize(c, p) * stride,
                       cudaMemcpyDeviceToHost));
    M.dirty[sl] = false;
    if (!out) M.part[sl] = -1;  // overwritten below: drop the device copy
  }
  for (uint32_t id = 0; id < c->nv; ++id) {
    const uint64_t o = static_cast<uint64_t>(c->part.inv_perm[id]) * dim;
    if (out) std::memcpy(out + o, host + static_cast<uint64_t>(id) * stride, dim * sizeof(float));
    else std::memcpy(host + static_cast<uint64_t>(id) * stride, in + o, dim * sizeof(float));
  }
  return GV_OK;
}

void hp_destroy(gv_ctx* c) {
  if (c->h_vertex) cudaFreeHost(c->h_vertex);
  if (c->h_context) cudaFreeHost(c->h_context);
  c->h_vertex = c->h_context = nullptr;
  if (c->hp_h2d) cudaStreamDestroy(c->hp_h2d);
  if (c->hp_d2h) cudaStreamDestroy(c->hp_d2h);
  c->hp_h2d = c->hp_d2h = nullptr;
  for (HpMat* M : {&c->hpv, &c->hpc}) {
    for (int k = 0; k < HpMat::S; ++k)
      for (cudaEvent_t e : {M->free_[k], M->saved[k], M->loaded[k]})
        if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : M->part_saved) cudaEventDestroy(e);
    M->part_saved.clear();
  }
}

}  // namespace gv
