// sgd.cu — sm_100a block-SGD kernels of the GraphVite hot path (a7) and
// the vertex-shard initialisation.
//
//   KB0 init_vertex        Philox init of the vertex shard (R-INIT)
//   KB2 sgd_ring           block-SGD, d <= 128: 8 lanes per sample, cp.async
//                          row ring in shared memory, red.global deltas —
//                          Hogwild in-place updates ("asynchronous SGD";
//                          P:97)
//   KB2 sgd_hogwild        the same for d > 128, one warp per sample
//   KB2v sgd_ordered       the same update, one warp per block, block order
//   KB2x sgd_explicit      caller-given negatives (hand-derived tests)
//   KB2d negatives         dump of the negative stream of one block
//
// Data layout: embedding rows are fp32, row stride a multiple
// of 4 floats, so lane l of a warp owns float4 columns l, l+32, ... of a row
// (128-bit coalesced accesses; a 512 B row at d = 128 is one warp load).
// Rows are read and written with ld/st.global.cg (L2 only): under Hogwild
// every SM sees the L2-coherent value of a hot row instead of a stale L1 copy.
#include "device_common.cuh"

namespace gv {
namespace detail {

// Per-device launch caches: a process may drive contexts on several devices
// (gv_options.device), and function attributes / occupancy are per device.
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

}  // namespace detail

namespace {

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
  if (my_hot && a.vertex_keep) *my_hot = 1u;  // vertex row kept in L2, context rows first out
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

// Chunks of 32 consecutive stream samples handed to the warps of the ring
// kernel. Static (ctr == nullptr): warp w takes chunks w, w + W, w + 2W, ...
// Dynamic (a.chunk_ctr): a warp claims its next chunk from a global counter
// one chunk ahead of use, so the warps' positions in the stream stay within
// a few chunks of each other however their speeds differ — the samples in
// flight are a narrow window of the stream, and what the stream's order puts
// close together (a vertex tile of the pool, gv_options.vertex_tile) is
// close together in time too, i.e. in L2.
struct ChunkSrc {
  uint64_t warp, nw, nchunks, total;
  unsigned long long* ctr;
  // global index of this warp's k-th chunk (warp-uniform; lane 0 claims)
  __device__ __forceinline__ uint64_t claim(uint32_t k, int lane) const {
    if (ctr == nullptr) return warp + static_cast<uint64_t>(k) * nw;
    unsigned long long g = 0;
    if (lane == 0) g = atomicAdd(ctr, 1ull);
    return __shfl_sync(kFull, g, 0);
  }
  // samples of chunk g (0 past the end)
  __device__ __forceinline__ uint32_t valid(uint64_t g) const {
    return g < nchunks ? static_cast<uint32_t>(umin64(32, total - (g << 5))) : 0u;
  }
};

template <int K>
__device__ __forceinline__ void chunk_ids(const SgdArgs& a, const ChunkSrc& cs, uint64_t g,
                                          int lane, uint32_t& u, uint32_t* c, uint32_t& hot) {
  u = 0;
  hot = 0;
#pragma unroll
  for (int t = 0; t <= K; ++t) c[t] = 0;
  if (static_cast<uint32_t>(lane) < cs.valid(g)) sample_ids<K>(a, (g << 5) + lane, u, c, &hot);
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
__device__ __forceinline__ float run_ring(const SgdArgs& a, const ChunkSrc& cs, float4* ring,
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
  // iteration i runs sample G (i mod ITER_PER_CHUNK) + h of the warp's chunk
  // i / ITER_PER_CHUNK; the ids of the current and the next chunk are loaded
  uint32_t cu, cc[K + 1], nu, nc[K + 1];  // ids of the current / next 32-sample chunk
  uint32_t ch_hot, nh_hot;
  const uint64_t g0 = cs.claim(0, lane), g1 = cs.claim(1, lane);
  uint32_t vcur = cs.valid(g0), vnxt = cs.valid(g1);  // samples of the current / next chunk
  if (vcur == 0) return loss;
  chunk_ids<K>(a, cs, g0, lane, cu, cc, ch_hot);
  chunk_ids<K>(a, cs, g1, lane, nu, nc, nh_hot);
  // group h's sample of iteration j (in the current or the next chunk) exists
  auto valid_it = [&](uint32_t j, uint32_t cur_chunk) {
    const uint32_t v = (j / ITER_PER_CHUNK) == cur_chunk ? vcur : vnxt;
    return G * (j % ITER_PER_CHUNK) + h < v;
  };
#if GV_SKIP_HOT_EXPERIMENT
  // measurement-only build: the deltas of rows with local id < hot_rows are
  // dropped (wrong training) to measure what hot-row write contention costs
  // (profiles/r01_hot_row_combining.json)
  const uint64_t pol_hot = policy_evict_normal(), pol_cold = pol_hot;
#else
  const bool hints = a.hot_rows != 0 || a.vertex_keep != 0;
  const uint64_t pol_hot = hints ? policy_evict_last() : policy_evict_normal();
  // vertex_keep 2: only the vertex rows get a hint (evict_last), context rows none
  const uint64_t pol_cold =
      (hints && a.vertex_keep != 2) ? policy_evict_first() : policy_evict_normal();
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
    if (valid_it(j, cur_chunk)) {
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
  for (int j = 0; j < P; ++j) {  // P < ITER_PER_CHUNK: all in chunk 0
    issue(j, j, 0);
    if (!kRingTma) cp_commit();
  }
  int st = 0;     // stage of iteration i
  int st_in = P;  // stage the prefetch of iteration i + P goes to
  for (uint32_t i = 0;; ++i) {
    const uint32_t chunk = i / ITER_PER_CHUNK;
    if (vcur == 0) break;  // the warp's chunks ran past the end of the stream
    const bool act = valid_it(i, chunk);
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
#elif GV_SKIP_HOT_EXPERIMENT == 3
      if (((hot >> r) & 1u) && h != 0) return;  // three quarters: each hot address sees 1/4 of its
                                                // deltas (the load a 4-way sharded row would see)
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
    issue(i + P, st_in, chunk);  // P < ITER_PER_CHUNK: in this chunk or the next
    if (!kRingTma) cp_commit();
#if GV_RING_PF > 0
    {
      const uint32_t jp = i + P + GV_RING_PF;
      if (jp / ITER_PER_CHUNK <= chunk + 1) {  // ids loaded (warp-uniform)
        uint32_t pu, pc[K + 1], phot;
        ids_of(jp, chunk, pu, pc, phot);
        if (gl == 0 && valid_it(jp, chunk)) {
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
      vcur = vnxt;
#pragma unroll
      for (int t = 0; t <= K; ++t) cc[t] = nc[t];
      const uint64_t g = cs.claim(chunk + 2, lane);
      vnxt = cs.valid(g);
      chunk_ids<K>(a, cs, g, lane, nu, nc, nh_hot);
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
  const ChunkSrc cs{warp, nw, (a.total + 31) >> 5, a.total, a.chunk_ctr};
  float4* ring = smem_f4 + (threadIdx.x >> 5) * RingCfg<K, kRingLPS>::WARP_ALL;
  const float loss = run_ring<K, kRingLPS>(a, cs, ring, dim4, lane, a.loss_acc != nullptr);
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
    if (a.chunk_ctr) {
      const cudaError_t e = cudaMemsetAsync(a.chunk_ctr, 0, sizeof(unsigned long long), s);
      if (e != cudaSuccess) return e;
    }
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

}  // namespace gv
