// kernels.cu — sm_100a kernels of the GraphVite hot path.
//
//   KB0 init_vertex        Philox init of the vertex shard (R-INIT)
//   KB1 bucket_*           relabel + histogram + scans + stable scatter into
//                          the n x n grid (Alg. 3 "Redistribute")
//   KB2 sgd_hogwild        block-SGD, one warp per sample, Hogwild in-place
//                          updates ("asynchronous SGD")
//   KB2v sgd_ordered       the same update, one warp per block, block order
//   KB2x sgd_explicit      caller-given negatives (hand-derived tests)
//   KB2d negatives         dump of the negative stream of one block
//
// Data layout: embedding rows are fp32, row stride a multiple
// of 4 floats, so lane l of a warp owns float4 columns l, l+32, ... of a row
// (128-bit coalesced accesses; a 512 B row at d = 128 is one warp load).
// Rows are read and written with ld/st.global.cg (L2 only): under Hogwild
// every SM sees the L2-coherent value of a hot row instead of a stale L1 copy.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "kernels.cuh"
#include "philox.cuh"

namespace gv {
namespace {

constexpr unsigned kFull = 0xFFFFFFFFu;

__host__ __device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }

template <int CH>
struct Row {
  float4 v[CH];
};

template <int CH>
__device__ __forceinline__ void load_row(Row<CH>& r, const float* base, uint32_t row,
                                         uint32_t stride, int lane, int dim4) {
  const float4* p = reinterpret_cast<const float4*>(base + static_cast<uint64_t>(row) * stride);
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    const int col = lane + 32 * c;
    r.v[c] = (col < dim4) ? __ldcg(p + col) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

template <int CH>
__device__ __forceinline__ void store_row(const Row<CH>& r, float* base, uint32_t row,
                                          uint32_t stride, int lane, int dim4) {
  float4* p = reinterpret_cast<float4*>(base + static_cast<uint64_t>(row) * stride);
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    const int col = lane + 32 * c;
    if (col < dim4) __stcg(p + col, r.v[c]);
  }
}

// Component-wise atomic add of a row delta at L2 (Hogwild write-back):
// concurrent warps never overwrite each other's updates.
__device__ __forceinline__ void red_add4(float* p, float4 v) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};\n" ::"l"(p), "f"(v.x), "f"(v.y),
               "f"(v.z), "f"(v.w)
               : "memory");
}

template <int CH>
__device__ __forceinline__ void red_row(float* base, uint32_t row, uint32_t stride, int lane,
                                        int dim4, float g, const Row<CH>& x) {
  float* p = base + static_cast<uint64_t>(row) * stride;
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    const int col = lane + 32 * c;
    if (col < dim4)
      red_add4(p + 4 * col, make_float4(g * x.v[c].x, g * x.v[c].y, g * x.v[c].z, g * x.v[c].w));
  }
}

template <int CH>
__device__ __forceinline__ float lane_dot(const Row<CH>& a, const Row<CH>& b) {
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    s = fmaf(a.v[c].x, b.v[c].x, s);
    s = fmaf(a.v[c].y, b.v[c].y, s);
    s = fmaf(a.v[c].z, b.v[c].z, s);
    s = fmaf(a.v[c].w, b.v[c].w, s);
  }
  return s;
}

__device__ __forceinline__ float warp_sum1(float s) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
  return s;
}

// Two warp sums with 7 shuffles instead of 10: at the first butterfly stage
// lanes < 16 keep a and send b, lanes >= 16 keep b and send a; four more
// stages inside each half; the sums are read from lanes 0 and 16.
__device__ __forceinline__ void warp_sum2(float& a, float& b, int lane) {
  const bool hi = (lane & 16) != 0;
  float keep = hi ? b : a;
  const float send = hi ? a : b;
  keep += __shfl_xor_sync(kFull, send, 16);
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) keep += __shfl_xor_sync(kFull, keep, o);
  a = __shfl_sync(kFull, keep, 0);
  b = __shfl_sync(kFull, keep, 16);
}

template <int CH>
__device__ __forceinline__ void axpy(Row<CH>& y, float g, const Row<CH>& x) {
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    y.v[c].x = fmaf(g, x.v[c].x, y.v[c].x);
    y.v[c].y = fmaf(g, x.v[c].y, y.v[c].y);
    y.v[c].z = fmaf(g, x.v[c].z, y.v[c].z);
    y.v[c].w = fmaf(g, x.v[c].w, y.v[c].w);
  }
}

// log(1 + e) for e = exp(-x): -x once e overflows (x < -88), so the
// monitoring loss stays finite.
__device__ __forceinline__ float softplus_e(float e, float x) {
  return e > 1e30f ? -x : __logf(1.0f + e);
}

// One target of a sample: p = s(x) = 1/(1+exp(-x)) (IEEE expf, correctly
// rounded reciprocal), g = (y - p) lr w, err += g C, C += g U. Returns the
// target's loss -log s(+-x) = log(1+e^-x) (+ x for a negative) when wanted.
template <int CH>
__device__ __forceinline__ float apply_target(float x, bool positive, float lr, float neg_weight,
                                              const Row<CH>& U, Row<CH>& Ct, Row<CH>& err,
                                              bool want_loss, float& g_out) {
  const float e = expf(-x);
  const float p = __frcp_rn(1.0f + e);
  const float g = ((positive ? 1.0f : 0.0f) - p) * lr * (positive ? 1.0f : neg_weight);
  g_out = g;
  axpy<CH>(err, g, Ct);
  axpy<CH>(Ct, g, U);
  return want_loss ? (softplus_e(e, x) + (positive ? 0.0f : x)) : 0.0f;
}

// Process up to 32 samples whose ids sit one per lane (lane s holds sample s):
// my_u = vertex row, my_c[0] = positive context row, my_c[1..K] = negative rows.
// For each sample, in order (LINE convention):
//   for target t in [v, n_1..n_K]: x = U.C_t; p = s(x);
//     g = (y_t - p) lr w_t; err += g C_t; C_t += g U
//   U += err
// The rows of sample s+1 are loaded before sample s is computed; rows that
// sample s updates are forwarded in registers (warp-uniform id compares), so
// the result equals strictly sequential processing of the 32 samples. A
// target equal to an earlier target of the same sample sees its update
// (R-DUP): then the targets run one after the other (rare slow path);
// otherwise all dot products are reduced together.
// ATOMIC (Hogwild): rows are written back as deltas with red.global.add
// (err for the vertex row, g_t U for context row t), as in Hogwild!'s
// lock-free component-wise updates (Recht et al., "asynchronous SGD");
// otherwise (one warp per block) the final rows are stored.
template <int K, int CH, bool ATOMIC>
__device__ __forceinline__ float run_chunk(int nvalid, uint32_t my_u, const uint32_t* my_c,
                                           float* __restrict__ vertex,
                                           float* __restrict__ context, uint32_t stride,
                                           int dim4, float lr, float neg_weight, int lane,
                                           bool want_loss) {
  float loss = 0.f;
  Row<CH> U, C[K + 1];
  uint32_t u = __shfl_sync(kFull, my_u, 0);
  uint32_t c[K + 1];
#pragma unroll
  for (int t = 0; t <= K; ++t) c[t] = __shfl_sync(kFull, my_c[t], 0);
  load_row<CH>(U, vertex, u, stride, lane, dim4);
#pragma unroll
  for (int t = 0; t <= K; ++t) load_row<CH>(C[t], context, c[t], stride, lane, dim4);

  for (int s = 0; s < nvalid; ++s) {
    const bool has_next = (s + 1) < nvalid;
    uint32_t un = 0, cn[K + 1];
    Row<CH> Un, Cn[K + 1];
    if (has_next) {  // prefetch the next sample's rows (warp-uniform branch)
      un = __shfl_sync(kFull, my_u, s + 1);
#pragma unroll
      for (int t = 0; t <= K; ++t) cn[t] = __shfl_sync(kFull, my_c[t], s + 1);
      load_row<CH>(Un, vertex, un, stride, lane, dim4);
#pragma unroll
      for (int t = 0; t <= K; ++t) load_row<CH>(Cn[t], context, cn[t], stride, lane, dim4);
    }
    Row<CH> err;
#pragma unroll
    for (int q = 0; q < CH; ++q) err.v[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    bool dup = false;
#pragma unroll
    for (int t = 1; t <= K; ++t)
#pragma unroll
      for (int tp = 0; tp < t; ++tp) dup |= (c[t] == c[tp]);
    float g[K + 1];
    Row<CH> U0 = U;  // the vertex row the context deltas are taken against
    if (!dup) {
      float x[K + 1];
#pragma unroll
      for (int t = 0; t <= K; ++t) x[t] = lane_dot<CH>(U, C[t]);
#pragma unroll
      for (int t = 0; t + 1 <= K; t += 2) warp_sum2(x[t], x[t + 1], lane);
      if ((K + 1) & 1) x[K] = warp_sum1(x[K]);
#pragma unroll
      for (int t = 0; t <= K; ++t)
        loss += apply_target<CH>(x[t], t == 0, lr, neg_weight, U, C[t], err, want_loss, g[t]);
    } else {
#pragma unroll
      for (int t = 0; t <= K; ++t) {
#pragma unroll
        for (int tp = 0; tp < t; ++tp)
          if (c[t] == c[tp]) C[t] = C[tp];
        const float x = warp_sum1(lane_dot<CH>(U, C[t]));
        loss += apply_target<CH>(x, t == 0, lr, neg_weight, U, C[t], err, want_loss, g[t]);
      }
    }
#pragma unroll
    for (int q = 0; q < CH; ++q) {
      U.v[q].x += err.v[q].x;
      U.v[q].y += err.v[q].y;
      U.v[q].z += err.v[q].z;
      U.v[q].w += err.v[q].w;
    }
    if (ATOMIC) {
      red_row<CH>(vertex, u, stride, lane, dim4, 1.0f, err);
#pragma unroll
      for (int t = 0; t <= K; ++t) red_row<CH>(context, c[t], stride, lane, dim4, g[t], U0);
    } else {
      store_row<CH>(U, vertex, u, stride, lane, dim4);
#pragma unroll
      for (int t = 0; t <= K; ++t) store_row<CH>(C[t], context, c[t], stride, lane, dim4);
    }
    if (has_next) {
      // forwarding: rare, so decided once with a warp-uniform mask
      bool fwd = (un == u);
#pragma unroll
      for (int t = 0; t <= K; ++t)
#pragma unroll
        for (int tp = 0; tp <= K; ++tp) fwd |= (cn[t] == c[tp]);
      if (fwd) {
        if (un == u) Un = U;
#pragma unroll
        for (int t = 0; t <= K; ++t) {
#pragma unroll
          for (int tp = 0; tp <= K; ++tp)
            if (cn[t] == c[tp]) Cn[t] = C[tp];  // last match = final value
        }
      }
      U = Un;
      u = un;
#pragma unroll
      for (int t = 0; t <= K; ++t) {
        C[t] = Cn[t];
        c[t] = cn[t];
      }
    }
  }
  return loss;
}

// Per-lane ids of sample `qg` of a launch stream: block lookup, sample load,
// K negatives by Philox + alias (P:231 negatives from partition j only).
template <int K>
__device__ __forceinline__ void sample_ids(const SgdArgs& a, uint64_t qg, uint32_t& my_u,
                                           uint32_t* my_c, uint32_t* my_hot = nullptr) {
  int lo = 0, hi = a.nblk - 1;  // last desc with prefix <= qg
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (__ldg(&a.desc[mid].prefix) <= qg) lo = mid; else hi = mid - 1;
  }
  const BlockDesc* d = a.desc + lo;
  const uint32_t q = static_cast<uint32_t>(qg - __ldg(&d->prefix));
  const uint2 smp = __ldcs(a.samples + __ldg(&d->sample_off) + q);
  const uint32_t crow0 = __ldg(&d->crow0), m = __ldg(&d->m), alias0 = __ldg(&d->alias0);
  const uint32_t ij = __ldg(&d->ij);
  my_u = __ldg(&d->vrow0) + smp.x;
  my_c[0] = crow0 + smp.y;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const u32x4 r = philox4x32_10(u32x4{q, ij, a.pool_index, static_cast<uint32_t>(k)}, a.key0,
                                  a.key1);
    const uint32_t slot = slot_of((static_cast<uint64_t>(r.x) << 32) | r.y, m);
    const uint2 pa = __ldg(a.alias + alias0 + slot);
    const uint32_t nl = alias_pick(pa.x, pa.y, slot, r.z);
    my_c[1 + k] = crow0 + nl;
    if (my_hot) *my_hot |= (nl < a.hot_rows ? 1u : 0u) << (2 + k);
  }
  if (my_hot) *my_hot |= (smp.x < a.hot_rows ? 1u : 0u) | ((smp.y < a.hot_rows ? 1u : 0u) << 1);
}

// ------------------------------------------------------------------------
// Deep-pipelined Hogwild path (d <= 128). A warp is split into groups of LPS
// lanes (default 8: four samples per warp instruction, so the scalar part of
// an update — exp, reciprocal, g — and the control flow are paid once per
// four samples). Group h processes samples h, h+G, h+2G, ... of the warp's
// sequence; the rows of its next P samples are in flight as cp.async
// (LDGSTS, L2-only) copies into a per-group shared-memory ring of R = P + 1
// stages — P samples of row traffic outstanding per group without holding
// them in registers ("leverage the on-chip shared memory"). There is
// no register forwarding: a row may be read before this warp's own deltas
// of the previous P samples have landed — bounded staleness, the same as
// between any two warps under Hogwild; no update is lost because every
// write-back is a red.global.add delta. (The exact, sequential mode is
// sgd_ordered_kernel.) Lane gl of a group owns float4 columns gl, gl+LPS, ...
// in global and shared memory, so no lane reads another lane's shared data
// and cp.async completion (wait_group, per thread) is the only
// synchronisation.
// ------------------------------------------------------------------------
__device__ __forceinline__ void cp_async16(float4* smem, const float4* gmem, uint64_t pol) {
  const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;\n" ::"r"(sa),
               "l"(gmem), "l"(pol)
               : "memory");
}
// TMA bulk copy of a whole row into shared memory, completing on an mbarrier
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(bar));
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(bar));
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(a), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(bar));
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(a),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void bulk_red_row(void* gmem, const void* smem, uint32_t bytes,
                                             uint64_t pol) {
  const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile(
      "cp.reduce.async.bulk.global.shared::cta.bulk_group.L2::cache_hint.add.f32 [%0], [%1], %2, %3;\n"
      ::"l"(gmem), "r"(sa), "r"(bytes), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;\n" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}

__device__ __forceinline__ void bulk_row(void* smem, const void* gmem, uint32_t bytes,
                                         uint64_t* bar, uint64_t pol) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  const uint32_t b = static_cast<uint32_t>(__cvta_generic_to_shared(bar));
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;\n" ::"r"(d),
      "l"(gmem), "r"(bytes), "r"(b), "l"(pol)
      : "memory");
}

__device__ __forceinline__ void red_add4_hint(float* p, float4 v, uint64_t pol) {
  asm volatile("red.global.add.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;\n" ::"l"(p),
               "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "l"(pol)
               : "memory");
}
// L2 policies: hot rows (high degree, small local id) stay, cold rows go first
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// The Hogwild kernel's sigmoid: MUFU ex2 / rcp (a few ulp) instead of the
// IEEE expf and correctly rounded reciprocal of the ordered kernel — under
// Hogwild the update order is nondeterministic anyway (parity there is the
// AUC test), and the shorter dependency chain is what the stall profile asks
// for. GV_RING_IEEE=1 restores the exact functions.
#ifndef GV_RING_IEEE
#define GV_RING_IEEE 0
#endif
__device__ __forceinline__ float ring_exp(float x) {
#if GV_RING_IEEE
  return expf(x);
#else
  return __expf(x);
#endif
}
__device__ __forceinline__ float ring_rcp(float x) {
#if GV_RING_IEEE
  return __frcp_rn(x);
#else
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
#endif
}

#ifndef GV_RING_P
#define GV_RING_P 3
#endif
constexpr int kRingP = GV_RING_P;

#ifndef GV_RING_LPS
#define GV_RING_LPS 8
#endif
constexpr int kRingLPS = GV_RING_LPS;  // lanes per sample: 16 (2 samples / warp) or 8 (4)

#ifndef GV_RING_TMA
#define GV_RING_TMA 0
#endif
#ifndef GV_SKIP_HOT_EXPERIMENT
#define GV_SKIP_HOT_EXPERIMENT 0
#endif
// GV_RING_PF=D > 0 (build option, measured slower): one lane per group also
// issues TMA bulk L2 prefetches (cp.async.bulk.prefetch.L2, one per row) for
// the sample D iterations past the ring's P — more DRAM reads in flight
// without more shared memory. C5: 1.63 / 1.47 / 1.42e9 at D = 2 / 4 / 5 vs
// 1.74e9 (profiles/r02_l_*): off.
#ifndef GV_RING_PF
#define GV_RING_PF 0
#endif
__device__ __forceinline__ void bulk_prefetch_l2(const void* gmem, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(gmem), "r"(bytes) : "memory");
}
// Rows staged by TMA bulk copies (cp.async.bulk + one mbarrier per stage)
// instead of LDGSTS: measured equal on C2 and C4 (profiles/README.md), and
// compute-sanitizer racecheck cannot verify the async-proxy ordering, so the
// default is LDGSTS; GV_RING_TMA=1 builds the TMA variant.
constexpr bool kRingTma = GV_RING_TMA == 1 || GV_RING_TMA == 2 || GV_RING_TMA == 4;
// GV_RING_TMA=2: the deltas also leave through the TMA unit — each lane
// writes its columns of err and g_t U over the stage it has consumed, and one
// lane per group issues a bulk reduce-add (cp.reduce.async.bulk .add.f32, an
// element-wise atomic add in L2) per row instead of red.global.add.v4 from
// registers.
constexpr bool kRingTmaRed = GV_RING_TMA == 2;
// GV_RING_TMA=3 (LDGSTS loads) / 4 (TMA loads): only the VERTEX row's delta
// leaves through the TMA unit (one bulk reduce-add per sample), the context
// rows' deltas by red.global from registers — the two paths to L2 share the
// delta traffic (the LSU's L1->XBAR request port bounds the default on C2).
constexpr bool kRingTmaRedV = GV_RING_TMA == 3 || GV_RING_TMA == 4;
constexpr bool kRingBulk = kRingTmaRed || kRingTmaRedV;

template <int K, int LPS>
struct RingCfg {
  static constexpr int G = 32 / LPS;     // samples per warp iteration (lane groups)
  static constexpr int R = kRingP + 1;   // stages per group
  static constexpr int T = K + 2;        // rows per sample
  static constexpr int STAGE = T * 32;   // float4 per stage (a 512 B row = 32 float4)
  static constexpr int GROUP = R * STAGE;
  static constexpr int WARP = G * GROUP; // float4 of row stages per warp
  static constexpr int BARS = (G * R + 1) / 2;  // float4 holding G*R mbarriers (8 B each)
  static constexpr int WARP_ALL = WARP + BARS;
  static constexpr size_t warp_bytes() { return static_cast<size_t>(WARP_ALL) * 16; }
};

// Sequence of samples processed by one warp: sample p is stream index
// start + (p >> 5) * stride + (p & 31), p < L.
struct WarpSeq {
  uint64_t start, stride;
  uint32_t L;
};

template <int K>
__device__ __forceinline__ void seq_chunk_ids(const SgdArgs& a, const WarpSeq& sq, uint32_t chunk,
                                              int lane, uint32_t& u, uint32_t* c, uint32_t& hot) {
  const uint32_t p = (chunk << 5) + lane;
  u = 0;
  hot = 0;
#pragma unroll
  for (int t = 0; t <= K; ++t) c[t] = 0;
  if (p < sq.L)
    sample_ids<K>(a, sq.start + static_cast<uint64_t>(chunk) * sq.stride + lane, u, c, &hot);
}

// sums over the LPS lanes of each group
template <int LPS>
__device__ __forceinline__ float group_sum1(float s) {
#pragma unroll
  for (int o = LPS / 2; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
  return s;
}
template <int LPS>
__device__ __forceinline__ void group_sum2(float& a, float& b, int lane) {
  const bool hi = (lane & (LPS / 2)) != 0;  // split butterfly at the first stage
  float keep = hi ? b : a;
  const float send = hi ? a : b;
  keep += __shfl_xor_sync(kFull, send, LPS / 2);
#pragma unroll
  for (int o = LPS / 4; o > 0; o >>= 1) keep += __shfl_xor_sync(kFull, keep, o);
  const int base = lane & ~(LPS - 1);
  a = __shfl_sync(kFull, keep, base);
  b = __shfl_sync(kFull, keep, base + LPS / 2);
}

template <int CPL>
__device__ __forceinline__ void red_rowg(float* base, uint32_t row, uint32_t stride, int gl,
                                         int lps, int dim4, float g, const Row<CPL>& x,
                                         bool active, uint64_t pol) {
  float* p = base + static_cast<uint64_t>(row) * stride;
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    const int col = gl + lps * c;
    if (active && col < dim4)
      red_add4_hint(p + 4 * col,
                    make_float4(g * x.v[c].x, g * x.v[c].y, g * x.v[c].z, g * x.v[c].w), pol);
  }
}

// The Hogwild ring pipeline with LPS lanes per sample: group g of the warp
// processes samples g, g+G, g+2G, ... of the warp's sequence; lane gl of a
// group owns float4 columns gl, gl+LPS, ... of every row.
template <int K, int LPS>
__device__ __forceinline__ float run_ring(const SgdArgs& a, const WarpSeq& sq, float4* ring,
                                          int dim4, int lane, bool want_loss) {
  using RC = RingCfg<K, LPS>;
  constexpr int P = kRingP, R = RC::R, T = RC::T, G = RC::G, CPL = 32 / LPS;
  constexpr int ITER_PER_CHUNK = 32 / G;
  const int h = lane / LPS, gl = lane % LPS;
  float4* const my = ring + h * RC::GROUP;
  uint64_t* const bars = reinterpret_cast<uint64_t*>(ring + RC::WARP) + h * R;  // this group's
  uint32_t phases = 0;  // bit r: parity of stage r's next completion
  if (kRingTma) {
    if (gl == 0)
      for (int r = 0; r < R; ++r) mbar_init(bars + r, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    __syncwarp();
  }
  float* const vertex = a.vertex;
  float* const context = a.context;
  const uint32_t stride = a.stride;
  float loss = 0.f;
  if (sq.L == 0) return loss;
  const uint32_t iters = (sq.L + G - 1) / G;  // iteration i: group h runs sample G i + h
  uint32_t cu, cc[K + 1], nu, nc[K + 1];      // ids of the current / next 32-sample chunk
  uint32_t ch_hot, nh_hot;
  seq_chunk_ids<K>(a, sq, 0, lane, cu, cc, ch_hot);
  seq_chunk_ids<K>(a, sq, 1, lane, nu, nc, nh_hot);
#if GV_SKIP_HOT_EXPERIMENT
  // measurement-only build: the deltas of rows with local id < hot_rows are
  // dropped (wrong training) to measure what hot-row write contention costs
  // (profiles/r01_hot_row_combining.json)
  const uint64_t pol_hot = policy_evict_normal(), pol_cold = pol_hot;
#else
  const uint64_t pol_hot = a.hot_rows ? policy_evict_last() : policy_evict_normal();
  const uint64_t pol_cold = a.hot_rows ? policy_evict_first() : policy_evict_normal();
#endif
  auto ids_of = [&](uint32_t j, uint32_t cur_chunk, uint32_t& u, uint32_t* c, uint32_t& hot) {
    const uint32_t pp = G * j + h;
    const bool cur = (j / ITER_PER_CHUNK) == cur_chunk;  // warp-uniform
    const int l = static_cast<int>(pp & 31);
    u = __shfl_sync(kFull, cur ? cu : nu, l);
#pragma unroll
    for (int t = 0; t <= K; ++t) c[t] = __shfl_sync(kFull, cur ? cc[t] : nc[t], l);
    hot = __shfl_sync(kFull, cur ? ch_hot : nh_hot, l);
  };
  auto issue = [&](uint32_t j, int st, uint32_t cur_chunk) {
    uint32_t u, c[K + 1], hot;
    ids_of(j, cur_chunk, u, c, hot);  // warp-uniform call: all lanes shuffle
    if (kRingTma) {
      // the stage was last read (generic proxy) by every lane of the group:
      // order those reads before the async-proxy (TMA) write into it
      __syncwarp();
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    }
    if (G * j + h < sq.L) {
      float4* stage = my + st * RC::STAGE;
      if (kRingTma) {  // one lane per group: expect the bytes, then one bulk copy per row
        if (gl == 0) {
          mbar_expect_tx(bars + st, static_cast<uint32_t>(T * dim4 * 16));
#pragma unroll
          for (int t = 0; t < T; ++t) {
            const float* g =
                (t == 0 ? vertex : context) + static_cast<uint64_t>(t == 0 ? u : c[t - 1]) * stride;
            bulk_row(stage + t * 32, g, static_cast<uint32_t>(dim4 * 16), bars + st,
                     ((hot >> t) & 1u) ? pol_hot : pol_cold);
          }
        }
      } else {
#pragma unroll
        for (int t = 0; t < T; ++t) {
          const float4* g = reinterpret_cast<const float4*>(
              (t == 0 ? vertex : context) + static_cast<uint64_t>(t == 0 ? u : c[t - 1]) * stride);
          const uint64_t pol = ((hot >> t) & 1u) ? pol_hot : pol_cold;
#pragma unroll
          for (int q = 0; q < CPL; ++q) {
            const int col = gl + LPS * q;
            if (col < dim4) cp_async16(stage + t * 32 + col, g + col, pol);
          }
        }
      }
    }
  };
#pragma unroll
  for (int j = 0; j < P; ++j) {
    if (static_cast<uint32_t>(j) < iters) issue(j, j, 0);
    if (!kRingTma) cp_commit();
  }
  int st = 0;     // stage of iteration i
  int st_in = P;  // stage the prefetch of iteration i + P goes to
  for (uint32_t i = 0; i < iters; ++i) {
    const uint32_t chunk = i / ITER_PER_CHUNK;
    const bool act = G * i + h < sq.L;
    if (kRingTma) {
      if (act) mbar_wait(bars + st, (phases >> st) & 1u);
      phases ^= 1u << st;
    } else {
      cp_wait<P - 1>();
    }
    uint32_t u, c[K + 1], hot;
    ids_of(i, chunk, u, c, hot);
    float4* stage = my + st * RC::STAGE;
    Row<CPL> U, C[K + 1], err;
#pragma unroll
    for (int q = 0; q < CPL; ++q) {
      const int col = gl + LPS * q;
      const bool ok = act && col < dim4;
      U.v[q] = ok ? stage[col] : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int t = 0; t <= K; ++t)
        C[t].v[q] = ok ? stage[(1 + t) * 32 + col] : make_float4(0.f, 0.f, 0.f, 0.f);
      err.v[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    // delta of row r (0 = vertex, 1 + t = target t): red from registers, or
    // (kRingTmaRed) written over the consumed stage row for the bulk reduce
    auto put_delta = [&](int r, uint32_t row, float g, const Row<CPL>& x, uint64_t pol) {
#if GV_SKIP_HOT_EXPERIMENT == 1
      if ((hot >> r) & 1u) return;
#elif GV_SKIP_HOT_EXPERIMENT == 2
      if (((hot >> r) & 1u) && h == 0) return;  // a quarter of the hot rows' deltas (lane group 0)
#endif
      if (kRingTmaRed || (kRingTmaRedV && r == 0)) {
#pragma unroll
        for (int q = 0; q < CPL; ++q) {
          const int col = gl + LPS * q;
          if (act && col < dim4)
            stage[r * 32 + col] = make_float4(g * x.v[q].x, g * x.v[q].y, g * x.v[q].z, g * x.v[q].w);
        }
      } else {
        red_rowg<CPL>(r == 0 ? vertex : context, row, stride, gl, LPS, dim4, g, x, act, pol);
      }
    };
    bool dup = false;
#pragma unroll
    for (int t = 1; t <= K; ++t)
#pragma unroll
      for (int tp = 0; tp < t; ++tp) dup |= (c[t] == c[tp]);
    if (!__any_sync(kFull, dup && act)) {
      float x[K + 1];
#pragma unroll
      for (int t = 0; t <= K; ++t) x[t] = lane_dot<CPL>(U, C[t]);
#pragma unroll
      for (int t = 0; t + 1 <= K; t += 2) group_sum2<LPS>(x[t], x[t + 1], lane);
      if ((K + 1) & 1) x[K] = group_sum1<LPS>(x[K]);
#pragma unroll
      for (int t = 0; t <= K; ++t) {
        const float e = ring_exp(-x[t]);
        const float pr = ring_rcp(1.0f + e);
        const float g = ((t == 0 ? 1.0f : 0.0f) - pr) * a.lr * (t == 0 ? 1.0f : a.neg_weight);
        axpy<CPL>(err, g, C[t]);
        put_delta(1 + t, c[t], g, U, ((hot >> (1 + t)) & 1u) ? pol_hot : pol_cold);
        if (want_loss && act) loss += softplus_e(e, x[t]) + (t == 0 ? 0.0f : x[t]);
      }
    } else {
      // a target repeated inside the sample sees the earlier target's update (R-DUP)
#pragma unroll
      for (int t = 0; t <= K; ++t) {
#pragma unroll
        for (int tp = 0; tp < t; ++tp)
          if (c[t] == c[tp]) C[t] = C[tp];
        const float x = group_sum1<LPS>(lane_dot<CPL>(U, C[t]));
        const float e = ring_exp(-x);
        const float pr = ring_rcp(1.0f + e);
        const float g = ((t == 0 ? 1.0f : 0.0f) - pr) * a.lr * (t == 0 ? 1.0f : a.neg_weight);
        axpy<CPL>(err, g, C[t]);
        put_delta(1 + t, c[t], g, U, ((hot >> (1 + t)) & 1u) ? pol_hot : pol_cold);
        axpy<CPL>(C[t], g, U);
        if (want_loss && act) loss += softplus_e(e, x) + (t == 0 ? 0.0f : x);
      }
    }
    put_delta(0, u, 1.0f, err, (hot & 1u) ? pol_hot : pol_cold);
    if (kRingBulk) {
      // the group's generic writes of the deltas, then one lane hands the
      // rows to the TMA unit (async proxy)
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      __syncwarp();
      if (gl == 0) {
        if (act) {
#pragma unroll
          for (int t = 0; t < (kRingTmaRed ? T : 1); ++t)
            bulk_red_row((t == 0 ? vertex : context) +
                             static_cast<uint64_t>(t == 0 ? u : c[t - 1]) * stride,
                         stage + t * 32, static_cast<uint32_t>(dim4 * 16),
                         ((hot >> t) & 1u) ? pol_hot : pol_cold);
        }
        bulk_commit();
        // the stage refilled next (iteration i - 1's) must have been read
        bulk_wait_read<1>();
      }
      __syncwarp();
    }
    if (i + P < iters) issue(i + P, st_in, chunk);
    if (!kRingTma) cp_commit();
#if GV_RING_PF > 0
    {
      const uint32_t jp = i + P + GV_RING_PF;
      if (jp < iters && jp / ITER_PER_CHUNK <= chunk + 1) {  // ids loaded (warp-uniform)
        uint32_t pu, pc[K + 1], phot;
        ids_of(jp, chunk, pu, pc, phot);
        if (gl == 0 && G * jp + h < sq.L) {
          bulk_prefetch_l2(vertex + static_cast<uint64_t>(pu) * stride, static_cast<uint32_t>(dim4 * 16));
#pragma unroll
          for (int t = 0; t <= K; ++t)
            bulk_prefetch_l2(context + static_cast<uint64_t>(pc[t]) * stride,
                             static_cast<uint32_t>(dim4 * 16));
        }
      }
    }
#endif
    st = (st + 1 == R) ? 0 : st + 1;
    st_in = (st_in + 1 == R) ? 0 : st_in + 1;
    if ((i % ITER_PER_CHUNK) == ITER_PER_CHUNK - 1) {  // all groups finished the chunk
      cu = nu;
      ch_hot = nh_hot;
#pragma unroll
      for (int t = 0; t <= K; ++t) cc[t] = nc[t];
      seq_chunk_ids<K>(a, sq, chunk + 2, lane, nu, nc, nh_hot);
    }
  }
  if (!kRingTma) cp_wait<0>();
  if (kRingBulk && gl == 0) bulk_wait_all();
  return loss;
}

template <int K>
__global__ void __launch_bounds__(256) sgd_ring_kernel(const SgdArgs a, int dim4) {
  extern __shared__ float4 smem_f4[];
  const int lane = threadIdx.x & 31;
  const uint64_t warp = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
  const uint64_t nchunks = (a.total + 31) >> 5;
  WarpSeq sq{warp << 5, nw << 5, 0};
  if (warp < nchunks) {
    const uint64_t mine = (nchunks - 1 - warp) / nw + 1;
    uint64_t L = mine << 5;
    if (warp + (mine - 1) * nw == nchunks - 1) L -= (nchunks << 5) - a.total;
    sq.L = static_cast<uint32_t>(L);
  }
  float4* ring = smem_f4 + (threadIdx.x >> 5) * RingCfg<K, kRingLPS>::WARP_ALL;
  const float loss = run_ring<K, kRingLPS>(a, sq, ring, dim4, lane, a.loss_acc != nullptr);
  if (a.loss_acc != nullptr && (lane % kRingLPS) == 0)
    atomicAdd(a.loss_acc, static_cast<double>(loss));
}

__device__ __forceinline__ void add_loss(double* acc, float loss, int lane) {
  if (acc != nullptr && lane == 0) atomicAdd(acc, static_cast<double>(loss));
}


// KB2: persistent grid; warp w takes chunks w, w + W, ... of 32 consecutive
// samples of the launch stream. The ids of the warp's next chunk (sample
// load, Philox, alias gather) are requested before the current chunk is
// processed, so their latency hides behind 32 samples of work.
template <int K, int CH>
__global__ void __launch_bounds__(256)
    sgd_hogwild_kernel(const SgdArgs a, int dim4) {
  const int lane = threadIdx.x & 31;
  const uint64_t warp = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
  const uint64_t nchunks = (a.total + 31) >> 5;
  const bool want_loss = a.loss_acc != nullptr;
  float loss = 0.f;
  uint32_t cu = 0, cc[K + 1] = {};
  if (warp < nchunks && (warp << 5) + lane < a.total) sample_ids<K>(a, (warp << 5) + lane, cu, cc);
  for (uint64_t ch = warp; ch < nchunks; ch += nwarps) {
    const uint64_t base = ch << 5, nx = ch + nwarps;
    const int nvalid = static_cast<int>(umin64(32, a.total - base));
    uint32_t nu = 0, nc[K + 1] = {};
    if (nx < nchunks && (nx << 5) + lane < a.total) sample_ids<K>(a, (nx << 5) + lane, nu, nc);
    loss += run_chunk<K, CH, true>(nvalid, cu, cc, a.vertex, a.context, a.stride, dim4, a.lr,
                                   a.neg_weight, lane, want_loss);
    cu = nu;
#pragma unroll
    for (int t = 0; t <= K; ++t) cc[t] = nc[t];
  }
  add_loss(a.loss_acc, loss, lane);
}

// Ordered verification mode: warp b owns descriptor b and walks its block
// in order, 32 samples at a time, through the same run_chunk.
template <int K, int CH>
__global__ void __launch_bounds__(32) sgd_ordered_kernel(const SgdArgs a, int dim4) {
  const int lane = threadIdx.x & 31;
  const BlockDesc* d = a.desc + blockIdx.x;
  const uint64_t begin = d->prefix, count = d->count_lo;
  const bool want_loss = a.loss_acc != nullptr;
  float loss = 0.f;
  for (uint64_t off = 0; off < count; off += 32) {
    const int nvalid = static_cast<int>(umin64(32, count - off));
    uint32_t my_u = 0, my_c[K + 1] = {};
    if (lane < nvalid) sample_ids<K>(a, begin + off + lane, my_u, my_c);
    loss += run_chunk<K, CH, false>(nvalid, my_u, my_c, a.vertex, a.context, a.stride, dim4,
                                    a.lr, a.neg_weight, lane, want_loss);
  }
  add_loss(a.loss_acc, loss, lane);
}

template <int K, int CH>
__global__ void __launch_bounds__(32) sgd_explicit_kernel(const ExplicitArgs a, int dim4) {
  const int lane = threadIdx.x & 31;
  for (uint64_t off = 0; off < a.count; off += 32) {
    const int nvalid = static_cast<int>(umin64(32, a.count - off));
    uint32_t my_u = 0, my_c[K + 1] = {};
    if (lane < nvalid) {
      my_u = a.vrow[off + lane];
#pragma unroll
      for (int t = 0; t <= K; ++t) my_c[t] = a.crow[(off + lane) * (K + 1) + t];
    }
    run_chunk<K, CH, false>(nvalid, my_u, my_c, a.vertex, a.context, a.stride, dim4, a.lr,
                            a.neg_weight, lane, false);
  }
}

__global__ void negatives_kernel(const BlockDesc d, const uint2* __restrict__ alias,
                                 uint32_t pool_index, uint32_t key0, uint32_t key1, int K,
                                 uint32_t* __restrict__ out) {
  const uint64_t q = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= d.count_lo) return;
  for (int k = 0; k < K; ++k) {
    const u32x4 r = philox4x32_10(
        u32x4{static_cast<uint32_t>(q), d.ij, pool_index, static_cast<uint32_t>(k)}, key0, key1);
    const uint32_t slot = slot_of((static_cast<uint64_t>(r.x) << 32) | r.y, d.m);
    const uint2 pa = alias[d.alias0 + slot];
    out[q * K + k] = alias_pick(pa.x, pa.y, slot, r.z);
  }
}

__global__ void init_vertex_kernel(float* __restrict__ vertex, uint32_t stride, uint32_t dim,
                                   uint64_t row0, uint64_t rows,
                                   const uint32_t* __restrict__ inv_perm, uint32_t key0,
                                   uint32_t key1) {
  const uint32_t q4 = dim / 4;
  const uint64_t idx = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= rows * q4) return;
  const uint64_t row = idx / q4;
  const uint32_t c = static_cast<uint32_t>(idx % q4);
  const uint32_t orig = inv_perm[row0 + row];
  const u32x4 r = philox4x32_10(u32x4{orig, c, 0u, kTagInit}, key0, key1);
  const float fd = static_cast<float>(dim);
  float4 v;
  v.x = __fdiv_rn(__fsub_rn(__fmul_rn(static_cast<float>(r.x >> 8), 0x1p-24f), 0.5f), fd);
  v.y = __fdiv_rn(__fsub_rn(__fmul_rn(static_cast<float>(r.y >> 8), 0x1p-24f), 0.5f), fd);
  v.z = __fdiv_rn(__fsub_rn(__fmul_rn(static_cast<float>(r.z >> 8), 0x1p-24f), 0.5f), fd);
  v.w = __fdiv_rn(__fsub_rn(__fmul_rn(static_cast<float>(r.w >> 8), 0x1p-24f), 0.5f), fd);
  reinterpret_cast<float4*>(vertex + row * stride)[c] = v;
}

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

// ---------------------------------------------------------------- bucketing

struct BinCtx {
  const uint32_t* packed;
  const uint64_t* part_off;  // relabelled pool ids (IdMap)
  uint32_t nv, pbits, n;
  uint32_t pmul;  // floor(n 2^32 / nv): the proportional partition guess by a multiply-high
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

// Per-device launch caches: a process may drive contexts on several devices
// (gv_options.device), and function attributes / occupancy are per device.
constexpr int kMaxDev = 64;
int cur_dev() {
  int dev = 0;
  cudaGetDevice(&dev);
  return (dev >= 0 && dev < kMaxDev) ? dev : 0;
}
int g_num_sms[kMaxDev] = {};
int num_sms() {
  int& v = g_num_sms[cur_dev()];
  if (v == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    if (v <= 0) v = 148;
  }
  return v;
}

// ------------------------------------------------------------ dispatch table
using HogFn = void (*)(const SgdArgs, int);
using ExpFn = void (*)(const ExplicitArgs, int);

template <int K, int CH>
struct Inst {
  static constexpr HogFn hog = sgd_hogwild_kernel<K, CH>;
  static constexpr HogFn ord = sgd_ordered_kernel<K, CH>;
  static constexpr ExpFn exp = sgd_explicit_kernel<K, CH>;
};

#define GV_ROW(K) {Inst<K, 1>::hog, Inst<K, 2>::hog, Inst<K, 3>::hog, Inst<K, 4>::hog}
const HogFn kHog[8][4] = {GV_ROW(1), GV_ROW(2), GV_ROW(3), GV_ROW(4),
                          GV_ROW(5), GV_ROW(6), GV_ROW(7), GV_ROW(8)};
#undef GV_ROW
#define GV_ROW(K) {Inst<K, 1>::ord, Inst<K, 2>::ord, Inst<K, 3>::ord, Inst<K, 4>::ord}
const HogFn kOrd[8][4] = {GV_ROW(1), GV_ROW(2), GV_ROW(3), GV_ROW(4),
                          GV_ROW(5), GV_ROW(6), GV_ROW(7), GV_ROW(8)};
#undef GV_ROW
#define GV_ROW(K) {Inst<K, 1>::exp, Inst<K, 2>::exp, Inst<K, 3>::exp, Inst<K, 4>::exp}
const ExpFn kExp[8][4] = {GV_ROW(1), GV_ROW(2), GV_ROW(3), GV_ROW(4),
                          GV_ROW(5), GV_ROW(6), GV_ROW(7), GV_ROW(8)};
#undef GV_ROW

int ch_of(int dim) { return (dim / 4 + 31) / 32; }

const HogFn kRing[8] = {sgd_ring_kernel<1>, sgd_ring_kernel<2>, sgd_ring_kernel<3>,
                        sgd_ring_kernel<4>, sgd_ring_kernel<5>, sgd_ring_kernel<6>,
                        sgd_ring_kernel<7>, sgd_ring_kernel<8>};

int ring_mode() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("GV_SGD_RING");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v;
}

}  // namespace

int sgd_supported(int dim, int K) {
  return dim > 0 && dim % 4 == 0 && dim <= 512 && K >= 1 && K <= 8;
}

cudaError_t launch_sgd_hogwild(const SgdArgs& a, int dim, int K, int sms, cudaStream_t s) {
  if (a.total == 0 || a.nblk == 0) return cudaSuccess;
  const int ki = K - 1, ci = ch_of(dim) - 1;
  if (ci == 0 && ring_mode()) {
    HogFn f = kRing[ki];
    const int G = 32 / kRingLPS, R = kRingP + 1;
    const size_t wb = (static_cast<size_t>(G) * R * (K + 2) * 32 + (G * R + 1) / 2) * 16;
    // 4-warp CTAs: one warp per SM sub-partition (3-warp CTAs that fit 9
    // warps/SM measured slower than 4-warp CTAs at 8 warps/SM: uneven SMSPs);
    // large K (rows per stage) fits fewer warps per CTA
    const int warps = static_cast<int>(std::max<size_t>(1, std::min<size_t>(4, (200 * 1024) / wb)));
    const size_t smem = wb * warps;
    static int occr[kMaxDev][8] = {};
    int& o = occr[cur_dev()][ki];
    if (o == 0) {
      cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, f, 32 * warps, smem) != cudaSuccess || o <= 0)
        o = 1;
    }
    const uint64_t chunks = (a.total + 31) / 32;
    uint64_t grid = static_cast<uint64_t>(sms > 0 ? sms : num_sms()) * o;
    grid = std::min<uint64_t>(grid, (chunks + warps - 1) / warps);
    f<<<static_cast<unsigned>(grid), 32 * warps, smem, s>>>(a, dim / 4);
    return cudaGetLastError();
  }
  HogFn f = kHog[ki][ci];
  static int occ[kMaxDev][8][4] = {};
  int& o = occ[cur_dev()][ki][ci];
  if (o == 0 && (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, f, 256, 0) != cudaSuccess || o <= 0))
    o = 1;
  const uint64_t chunks = (a.total + 31) / 32;
  uint64_t grid = static_cast<uint64_t>(sms > 0 ? sms : num_sms()) * o;
  grid = std::min<uint64_t>(grid, (chunks + 7) / 8);
  f<<<static_cast<unsigned>(grid), 256, 0, s>>>(a, dim / 4);
  return cudaGetLastError();
}

cudaError_t launch_sgd_ordered(const SgdArgs& a, int dim, int K, cudaStream_t s) {
  if (a.nblk == 0) return cudaSuccess;
  kOrd[K - 1][ch_of(dim) - 1]<<<a.nblk, 32, 0, s>>>(a, dim / 4);
  return cudaGetLastError();
}

cudaError_t launch_sgd_explicit(const ExplicitArgs& a, int dim, int K, cudaStream_t s) {
  if (a.count == 0) return cudaSuccess;
  kExp[K - 1][ch_of(dim) - 1]<<<1, 32, 0, s>>>(a, dim / 4);
  return cudaGetLastError();
}

cudaError_t launch_negatives(const BlockDesc& d, const uint2* alias, uint32_t pool_index,
                             uint32_t key0, uint32_t key1, int K, uint32_t* out,
                             cudaStream_t s) {
  if (d.count_lo == 0) return cudaSuccess;
  const unsigned grid = (d.count_lo + 255) / 256;
  negatives_kernel<<<grid, 256, 0, s>>>(d, alias, pool_index, key0, key1, K, out);
  return cudaGetLastError();
}

cudaError_t launch_init_vertex(float* vertex, uint32_t stride, uint32_t dim, uint64_t row0,
                               uint64_t rows, const uint32_t* inv_perm, uint32_t key0,
                               uint32_t key1, cudaStream_t s) {
  const uint64_t n = rows * (dim / 4);
  if (n == 0) return cudaSuccess;
  init_vertex_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(
      vertex, stride, dim, row0, rows, inv_perm, key0, key1);
  return cudaGetLastError();
}

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
size_t align256(size_t x) { return (x + 255) / 256 * 256; }
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

cudaError_t launch_validate(const uint2* in, uint64_t count, uint32_t nv, uint64_t* block_off,
                            uint32_t* err, cudaStream_t s, int* launches) {
  uint64_t grid = umin64((count + 255) / 256, static_cast<uint64_t>(num_sms()) * 8);
  if (grid == 0) grid = 1;
  validate_kernel<<<static_cast<unsigned>(grid), 256, 0, s>>>(in, count, nv, block_off, err);
  if (launches) *launches += 1;
  return cudaGetLastError();
}

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
