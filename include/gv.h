/*
 * gv.h — C ABI of the B200-native parallel-negative-sampling trainer
 * (GraphVite, Zhu et al., arXiv 1903.00757).
 *
 * Citation keys: P:n = PAPER.md line n (LaTeX source of the paper),
 * S:n = SPEC.md line n, SURVEY §x = /root/repo/SURVEY.md section.
 *
 * What the library computes (the "hot path"):
 *   Per pool of positive edge samples (u,v) (Alg. 2):
 *     a2  stage the pool in device memory (gv_push_sample_pool)
 *     a3  relabel + histogram into the n x n partition grid              Alg. 3
 *     a4  scan -> block offsets
 *     a5  stable scatter into blocks (i,j), local ids
 *     a6  block-row exchange between ranks (D>1)                         Alg. 3
 *     a7  block-SGD on block (i,(i+t) mod n) per offset step t           Alg. 3 P:245-252,
 *         skip-gram negative-sampling objective, Hogwild
 *     a8  context rotation between ranks (D>1)                           Alg. 3
 *   gv_train_episode runs a3..a8 for one pushed pool.
 *
 * Conventions (all functions):
 *   - Every call returns gv_status; no exception or abort crosses the ABI.
 *     On error the context keeps the state it had before the call unless
 *     stated otherwise, and gv_last_error() returns a one-line message.
 *   - All pointers are HOST pointers unless the parameter name ends in _dev.
 *   - The caller owns every input array; the library copies what it needs
 *     before returning (the caller may free/reuse the buffer on return).
 *   - Output arrays are caller-allocated host buffers.
 *   - Embedding matrices cross the ABI as row-major float32 [num_nodes][dim]
 *     indexed by ORIGINAL node id (the library un-relabels them).
 *   - One caller thread per context, except that gv_push_sample_pool may run
 *     on a producer thread concurrently with gv_train_episode on the consumer
 *     thread (the collaboration strategy).
 *
 * Call order: gv_create -> gv_load_edges -> (gv_push_sample_pool+ ->
 *             gv_train_episode)* -> gv_get_* -> gv_destroy.
 * Anything else returns GV_ERR_STATE.
 *
 * Ranks ("devices" in the paper's Alg. 3): the n_partitions x n_partitions
 * grid is trained by D ranks. Rank d owns vertex partitions
 * [d*m, (d+1)*m), m = n_partitions / D, and at offset step t holds the
 * context partitions (d*m + t + g) mod n, g = 0..m-1 (a sliding window that
 * moves by one partition per step). D ranks are either
 *   - D separate processes (one per GPU, world_size = D; CUDA-IPC peer memory
 *     over NVLink / NVSwitch between them, handshake through a POSIX
 *     shared-memory segment), or
 *   - D virtual ranks inside one process on one GPU (virtual_ranks = D,
 *     device-copy transport) — the same schedule, used to test the
 *     multi-rank path on a single device.
 */
#ifndef GV_H_
#define GV_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GV_ABI_VERSION 4

typedef struct gv_ctx gv_ctx; /* opaque; owned by the library */

typedef enum {
  GV_OK = 0,
  GV_ERR_INVALID_ARG = 1, /* bad size/shape/parameter                          */
  GV_ERR_STATE = 2,       /* call out of order                                 */
  GV_ERR_OUT_OF_RANGE = 3,/* a node id >= num_nodes in a pool or edge list     */
  GV_ERR_EMPTY = 4,       /* empty graph / partition with zero noise mass      */
  GV_ERR_CAPACITY = 5,    /* block > 2^32-1 samples, pool > max_pool_samples   */
  GV_ERR_NOMEM = 6,       /* host or device allocation failed                  */
  GV_ERR_CUDA = 7,        /* CUDA runtime failure (text in gv_last_error)      */
  GV_ERR_COMM = 8         /* inter-process transport failure (IPC / timeout)   */
} gv_status;

/* Learning-rate schedule ("initial learning rate of 0.025 and the
 * linear learning rate decay mechanism in LINE"). Before offset step t:
 *   lr_t = (float)(lr0 * max(1 - S_before/total_samples, floor_ratio))
 * where S_before counts every sample (all ranks) trained in earlier offset
 * steps of this and earlier pools. Constant within a step. GV_LR_CONSTANT or
 * total_samples == 0 gives lr_t = lr0. SURVEY §8(c) step 8. */
typedef enum { GV_LR_CONSTANT = 0, GV_LR_LINEAR = 1 } gv_lr_kind;
typedef struct {
  gv_lr_kind kind;
  double floor_ratio;     /* default 1e-4                    */
  uint64_t total_samples; /* epochs * |E|                    */
} gv_lr_schedule;

typedef struct {
  uint64_t seed;          /* key of the negative-sample Philox stream            */
  uint64_t init_seed;     /* key of the embedding-init Philox stream             */
  float neg_weight;       /* gradient scale of negatives, default 5       */
  int device;             /* CUDA ordinal used by this process (default 0)        */
  int rank;               /* process rank (default 0)                             */
  int world_size;         /* number of processes, one per GPU (default 1)         */
  int virtual_ranks;      /* ranks simulated in this process (default 1);
                             world_size > 1 requires virtual_ranks == 1           */
  int ordered;            /* 1 = ordered verification mode: one warp per block,
                             samples in block order (bit-comparable schedule)     */
  int compute_loss;       /* 1 = accumulate the per-sample loss (default 1)       */
  int host_threads;       /* threads for host graph preparation (0 = all cores)   */
  uint64_t max_pool_samples; /* per rank; 0 = grow on demand                      */
  int host_partitions;    /* 1 = out-of-core (NEXT-3, Alg. 3): both
                             matrices live in pinned host memory; the device holds
                             three partition slots per matrix, loaded and written
                             back on their own streams while blocks train (block
                             order: steps in pairs, a reordering with the same
                             result). Single rank, n_partitions >= 2.
                             Default 0. */
  int host_pool;          /* 1 = the raw sample pool lives in pinned, mapped HOST
                             memory; bucketing reads it over PCIe, so samples take
                             device memory only as bucketed blocks ("the
                             memory cost of edge samples on GPUs becomes
                             negligible"). 0 (default) = raw pool in HBM. */
  int pool_ids;           /* id space of sample pools (pushed, and written by
                             gv_augment / gv_augment_device / gv_run):
                             GV_IDS_ORIGINAL (default) = the caller's node ids;
                             GV_IDS_RELABELED = the library's relabelled ids,
                             new = perm[orig] of gv_get_partition (zig-zag order,
                             R-ZIGZAG). With relabelled ids a3 needs no relabel
                             gather; at n_partitions = 1 (one rank, HBM pool) a3
                             is the range check alone and the pool is trained
                             where it lies — the raw buffer and the block buffer
                             swap roles ("skipped (identity) at
                             n = 1 with relabeled input"). Same samples, same
                             training; only the ids' encoding differs. */
  int vertex_tile;        /* b in [0, 31]: sample order inside a block (reading
                             R-VTILE). 0 (default) = pool order
                             (R-BUCKET). b > 0: within block (i, j) the samples
                             are stably sorted by vertex tile u_local >> b — the
                             block's vertex partition split into sub-partitions
                             of 2^b relabelled rows trained one after another
                             (P:233's partitions beyond the GPUs, along the
                             vertex side), so a tile's vertex rows are reused
                             from L2 ("leverage the on-chip memory"). The
                             sort runs after bucketing / the exchange, on the
                             device, into a second buffer of the rank's block
                             size (8 B per sample); its time counts in ms_bucket
                             (one rank) or ms_exchange (D > 1). */
} gv_options;

#define GV_IDS_ORIGINAL 0
#define GV_IDS_RELABELED 1

#define GV_MAX_RANKS 64

/* Per-pool statistics. The scalar times are over THIS process's ranks (all
 * its virtual ranks); the *_rank arrays hold every one of the D ranks of the
 * grid (multi-process: gathered through the IPC segment, so reading the
 * statistics of pool e is a rendezvous of all processes — every rank reads
 * them, or none). Times are CUDA-event durations on each rank's streams, in
 * milliseconds. The metric of BASELINE.json (edge samples/s, device-timed,
 * max over ranks) is samples_global / ms_device_max. */
typedef struct {
  uint64_t pool_index;    /* e: the pool counter used in the Philox counter      */
  uint64_t samples;       /* samples trained by this process in this pool         */
  uint64_t samples_global;/* samples in this pool over all ranks                  */
  uint32_t n_steps;       /* offset steps run (= n_partitions)                    */
  float lr_first, lr_last;
  double loss_sum;        /* sum over samples of -log s(x+) - sum_k log s(-x_k)
                             (0 if compute_loss == 0)                             */
  double ms_bucket;       /* a3..a5 (max over virtual ranks)                      */
  double ms_exchange;     /* a6                                                   */
  double ms_sgd;          /* a7 kernel time summed over steps (max over v-ranks)  */
  double ms_rotate;       /* a8 transfers not hidden behind a7                    */
  double ms_total;        /* first bucketing launch -> last kernel/transfer       */
  uint32_t sgd_launches;  /* number of block-SGD kernel launches                  */
  uint32_t kernel_launches; /* all kernels launched by this call                  */
  uint32_t n_ranks;       /* D = world_size * virtual_ranks                       */
  double ms_device_max;   /* max over the D ranks of ms_total_rank                */
  double ms_total_rank[GV_MAX_RANKS];    /* per rank d < n_ranks: as ms_total    */
  double ms_bucket_rank[GV_MAX_RANKS];   /* as ms_bucket                         */
  double ms_exchange_rank[GV_MAX_RANKS]; /* as ms_exchange                       */
  double ms_sgd_rank[GV_MAX_RANKS];      /* as ms_sgd                            */
  double ms_rotate_rank[GV_MAX_RANKS];   /* as ms_rotate (exposed rotation)      */
} gv_episode_stats;

/* ---------------------------------------------------------------------- */

/* Fills *opt with defaults: seed 5, init_seed 4 (SURVEY §8(d) seeds),
 * neg_weight 5, device 0, rank 0, world_size 1, virtual_ranks 1, ordered 0,
 * compute_loss 1, host_threads 0, max_pool_samples 0,
 * host_partitions 0. */
void gv_default_options(gv_options* opt);

/* Create a trainer for |V| = num_nodes nodes with dim-dimensional vertex and
 * context embeddings, an n_partitions x n_partitions grid,
 * num_negatives negatives per positive sample, initial learning rate
 * lr0 and schedule alpha (nullable -> linear decay with floor 1e-4 and
 * total_samples 0, i.e. constant). opt nullable -> gv_default_options.
 * Allocates nothing on the device yet.
 * Errors: GV_ERR_INVALID_ARG if num_nodes == 0, dim == 0, dim % 4 != 0,
 *   dim > 512, num_negatives == 0 or > 8, n_partitions == 0, n_partitions >
 *   num_nodes, n_partitions > 64, n_partitions % (world_size*virtual_ranks)
 *   != 0, lr0 < 0, or bad rank/world_size/virtual_ranks; GV_ERR_CUDA if the
 *   device cannot be selected. *out is set only on GV_OK. */
gv_status gv_create(uint32_t num_nodes, uint32_t dim, uint32_t n_partitions,
                    uint32_t num_negatives, float lr0,
                    const gv_lr_schedule* alpha, const gv_options* opt,
                    gv_ctx** out);

/* Multi-process only (world_size > 1): rank 0 calls gv_comm_unique_id, the
 * caller broadcasts the 128 bytes to every rank (e.g. torch.distributed),
 * then every rank calls gv_comm_init before gv_load_edges. With the IPC
 * transport gv_load_edges also waits until every rank has loaded the graph
 * (peers map each other's context buffers). Errors: GV_ERR_COMM. */
gv_status gv_comm_unique_id(uint8_t id_out[128]);
gv_status gv_comm_init(gv_ctx* ctx, const uint8_t id[128]);

/* Load the graph G=(V,E) as an edge list src[k]-dst[k] with optional
 * weights (nullable -> 1). The graph is treated as undirected:
 * self-loops are dropped, both directions are stored, duplicate edges have
 * their weights summed (in input order, in double). Weighted degree
 * deg[v] = sum of incident merged weights, summed in ascending neighbour id.
 * Then: degree-guided zig-zag partition and relabel (P:392,
 * fig:zig-zag_partition), one integer alias table per
 * context partition over deg^0.75,
 * per-node neighbour and departure alias tables for gv_augment, device
 * allocation of the rank's shards and Philox initialisation of the
 * embeddings (vertex U[-0.5/d, 0.5/d), context 0).
 * Every rank passes the SAME full edge list.
 * Errors: GV_ERR_OUT_OF_RANGE (id >= num_nodes), GV_ERR_INVALID_ARG
 *   (negative or non-finite weight), GV_ERR_EMPTY (no edge left, or a
 *   partition whose deg^0.75 mass is 0), GV_ERR_CAPACITY (a partition larger
 *   than the packed-id range), GV_ERR_NOMEM, GV_ERR_CUDA, GV_ERR_STATE
 *   (called twice). */
gv_status gv_load_edges(gv_ctx* ctx, const uint32_t* src, const uint32_t* dst,
                        const float* weight, uint64_t num_edges);

/* Append count edge samples (pairs[2k], pairs[2k+1]) = (u, v), ORIGINAL ids
 * (relabelled ids when gv_options.pool_ids = GV_IDS_RELABELED), to the pending pool (Alg. 2's concatenated pool). Copies before
 * returning, in chunks of 2^23 samples on the library's copy stream (batched
 * transfer); a pinned source buffer is copied by DMA at PCIe speed.
 * The library keeps ONE raw pool buffer: a push issued after
 * gv_train_episode(pool k) waits only until pool k has been bucketed (a few
 * ms into its training), then copies while pool k trains — device sample
 * memory is 2 x 8 B per sample (raw + blocks), or 8 B with host_pool = 1.
 * (Relabelled ids at n = 1: the two buffers alternate; a push waits until
 * the pool trained before the last one has finished.)
 * With virtual_ranks = D the whole pool is pushed and rank r trains on the
 * contiguous segment [r*P/D, (r+1)*P/D); with world_size = D each process
 * pushes its own segment. Ids are range-checked on the device at
 * gv_train_episode (GV_ERR_OUT_OF_RANGE, no update applied).
 * u == v is allowed. Errors: GV_ERR_STATE (before gv_load_edges),
 * GV_ERR_CAPACITY (pending pool would exceed max_pool_samples), GV_ERR_CUDA. */
gv_status gv_push_sample_pool(gv_ctx* ctx, const uint32_t* pairs, uint64_t count);

/* Same as gv_push_sample_pool but pairs_dev is a device pointer on this
 * process's device (device-to-device copy). */
gv_status gv_push_sample_pool_device(gv_ctx* ctx, const uint32_t* pairs_dev,
                                     uint64_t count);

/* Re-arm the last trained pool as the pending pool without any copy
 * (benchmarks replay one resident pool; the pool counter still advances so
 * negatives differ). GV_ERR_STATE if no pool was trained or one is pending. */
gv_status gv_replay_pool(gv_ctx* ctx);

/* Train the pending pool: bucket (a3-a5), exchange (a6), then for offset
 * steps t = 0..n-1 train block (i, (i+t) mod n) for every vertex partition i
 * owned by each rank, rotating context partitions between steps (a7, a8;
 * Alg. 3). Blocks of one step share no rows, so ranks need
 * no synchronisation within a step. Returns after the device work has been
 * ENQUEUED and the block sizes are known; call gv_synchronize (or read
 * stats, which synchronises when out != NULL) to wait. An empty pending pool
 * is a no-op that still advances nothing and returns GV_ERR_EMPTY.
 * Errors: GV_ERR_STATE, GV_ERR_EMPTY, GV_ERR_OUT_OF_RANGE (pool contains an
 * id >= num_nodes; detected before any SGD launch, embeddings unchanged),
 * GV_ERR_CAPACITY (a block > 2^32-1 samples), GV_ERR_CUDA, GV_ERR_COMM. */
gv_status gv_train_episode(gv_ctx* ctx, gv_episode_stats* out);

/* Wait for all device work of the context. */
gv_status gv_synchronize(gv_ctx* ctx);

/* Wait for the most recently trained pool and fill *out with its statistics
 * (the same as gv_train_episode(ctx, out) would have returned). Lets a
 * caller enqueue pool k, push pool k+1 (overlapping the copy with training)
 * and only then read pool k's result. GV_ERR_STATE if no pool was trained. */
gv_status gv_read_stats(gv_ctx* ctx, gv_episode_stats* out);

/* Copy embeddings to out (num_nodes*dim floats, ORIGINAL id order).
 * In multi-process mode only rows owned by this rank (vertex: its vertex
 * partitions; context: its canonical window [d*m,(d+1)*m)) are written.
 * Errors: GV_ERR_INVALID_ARG (out_len != num_nodes*dim), GV_ERR_STATE. */
gv_status gv_get_vertex_embeddings(gv_ctx* ctx, float* out, uint64_t out_len);
gv_status gv_get_context_embeddings(gv_ctx* ctx, float* out, uint64_t out_len);
/* Overwrite embeddings (tests, checkpoint resume); same layout and rules. */
gv_status gv_set_vertex_embeddings(gv_ctx* ctx, const float* in, uint64_t in_len);
gv_status gv_set_context_embeddings(gv_ctx* ctx, const float* in, uint64_t in_len);

/* Training progress (checkpoint / resume): the pool counter e of the
 * negative-sample Philox stream (R-RNG) and the global sample count S_before
 * of the lr schedule (R-LR). Saving them with the embeddings and restoring
 * both into a fresh context resumes a run exactly (ordered mode: bit for bit).
 * gv_set_progress: GV_ERR_STATE while a prepared pool is pending. In
 * multi-process mode (world_size > 1) the pool counter also numbers the
 * ranks' IPC handshake epochs, so every rank must call gv_set_progress with
 * the SAME values, after gv_load_edges and before its first pool is pushed
 * (GV_ERR_STATE otherwise). */
gv_status gv_get_progress(gv_ctx* ctx, uint64_t* pool_index, uint64_t* samples_done);
gv_status gv_set_progress(gv_ctx* ctx, uint64_t pool_index, uint64_t samples_done);

/* Library-owned compute stream of virtual rank r (cudaStream_t as uintptr),
 * so a caller can time device work with its own events on that stream. */
gv_status gv_get_stream(gv_ctx* ctx, int vrank, uintptr_t* stream_out);

/* Host online augmentation (Alg. 2): `threads` private segments,
 * each filled by random walks of walk_len edges from departures drawn
 * proportional to degree, pairs (w_a, w_b) with 0 < b-a <= s and w_a != w_b,
 * pseudo-shuffled into s sub-blocks, segments concatenated.
 * Writes exactly `count` pairs (ORIGINAL ids, or relabelled ids when
 * gv_options.pool_ids = GV_IDS_RELABELED) to out_pairs[2*count].
 * Deterministic given (seed, threads): walks draw from a Philox stream with
 * counter (walk, step, thread, 0x57414C4B) and key = seed (SURVEY §8(c),
 * reading R-AUG in DESIGN.md).
 * Errors: GV_ERR_STATE (no graph), GV_ERR_INVALID_ARG (walk_len == 0,
 * s == 0, s > walk_len, threads == 0). */
gv_status gv_augment(gv_ctx* ctx, uint32_t walk_len, uint32_t s,
                     uint32_t threads, uint64_t count, uint64_t seed,
                     uint32_t* out_pairs);

/* NEXT-1: online augmentation ON THE DEVICE. The same pool
 * as gv_augment(walk_len, s, threads = segments, count, seed) — byte for byte
 * (reading R-AUG) — generated by one CTA per segment from a device copy of
 * the graph's CSR and alias tables (uploaded on first use), and APPENDED to
 * the pending device pool (no host buffer, no H2D copy). Runs on the copy
 * stream, so it overlaps the training of the previous pool.
 * Errors: GV_ERR_STATE (no graph), GV_ERR_INVALID_ARG (walk_len == 0,
 * s == 0, s > walk_len, segments == 0, walk_len > 1000), GV_ERR_CAPACITY
 * (max_pool_samples), GV_ERR_CUDA. With virtual ranks the pool is split
 * among them as a pushed pool is; with processes (world_size > 1) it is this
 * rank's pool segment, generated on its own GPU. */
gv_status gv_augment_device(gv_ctx* ctx, uint32_t walk_len, uint32_t s, uint32_t segments,
                            uint64_t count, uint64_t seed);

/* NEXT-2 ablation of the pool shuffle (tab:shuffle): as
 * gv_augment_device, with shuffle = GV_SHUFFLE_PSEUDO (the paper's pseudo
 * shuffle; identical to gv_augment_device), GV_SHUFFLE_NONE (each segment's
 * pairs in walk order; pseudo-shuffling each segment of it gives the
 * GV_SHUFFLE_PSEUDO pool), or GV_SHUFFLE_RANDOM (the GV_SHUFFLE_NONE pool
 * under a keyed pseudo-random bijection of its positions — a 4-round
 * Feistel network keyed by Philox(seed, 'SHUF') — the GPU analogue of a
 * full random shuffle; needs 8*count bytes of device scratch).
 * Errors: as gv_augment_device, plus GV_ERR_INVALID_ARG for another shuffle. */
#define GV_SHUFFLE_PSEUDO 0
#define GV_SHUFFLE_NONE 1
#define GV_SHUFFLE_RANDOM 2
gv_status gv_augment_device_ex(gv_ctx* ctx, uint32_t walk_len, uint32_t s, uint32_t segments,
                               uint64_t count, uint64_t seed, int shuffle);

/* NEXT-1 ("writing bucketed blocks directly"; Alg. 2
 * P:176-196 with a3-a5): generate a WHOLE pool on the device and bucket it
 * in the sampler — the walks write their pairs straight into the n x n
 * blocks, with no raw pool and no separate bucketing pass. The blocks are
 * exactly those gv_train_episode would build from the pool of
 * gv_augment_device_ex(walk_len, s, segments, count, seed, shuffle) (a
 * stable counting sort of that pool by block, reading R-BUCKET). The pool
 * becomes the pending pool; it is generated on the copy stream, so it
 * overlaps the training of the previous pool (two block buffers alternate).
 * Device scratch: a walk cache of ~4 B per pair plus (segments * S * n^2)
 * counters, S = s (pseudo shuffle) or 1. Not replayable (gv_replay_pool
 * returns GV_ERR_STATE after it).
 * Errors: GV_ERR_STATE (no graph; more than one rank; a pool pending),
 * GV_ERR_INVALID_ARG (walk_len == 0 or > 1000, s == 0 or > walk_len,
 * segments == 0, count == 0, shuffle not PSEUDO/NONE, or a shape the
 * sampler cannot bucket: S > 32, count >= 2^32, S * n^2 counters beyond
 * shared memory — use gv_augment_device then), GV_ERR_CAPACITY
 * (max_pool_samples), GV_ERR_CUDA. */
gv_status gv_augment_device_blocks(gv_ctx* ctx, uint32_t walk_len, uint32_t s, uint32_t segments,
                                   uint64_t count, uint64_t seed, int shuffle);

/* Copy the pending (not yet trained) pool to the host: out_pairs[2*cap],
 * *count = its size. Tests. */
gv_status gv_debug_get_pending(gv_ctx* ctx, uint32_t* out_pairs, uint64_t cap, uint64_t* count);

/* Collaboration strategy: two pinned host pools; producer
 * threads fill one with gv_augment while the trainer pushes and trains the
 * other; pools swap when both sides are done. Trains ceil(total/pool) pools.
 * collaborate = 0 runs fill-then-train sequentially (ablation,
 * tab:main_components). Single-process only. Wall-clock results go to
 * *report (nullable). */
typedef struct {
  uint32_t walk_len;      /* 40               */
  uint32_t s;             /* augmentation distance    */
  uint32_t threads;       /* sampler threads          */
  uint64_t pool_samples;  /* samples per pool         */
  uint64_t seed;          /* augmentation Philox key (pool k uses seed + k) */
  int collaborate;        /* 1 = double-buffered      */
  int device;             /* 1 = augment on the GPU (gv_augment_device, segments =
                             threads); pool k+1 is generated while pool k trains */
} gv_augment_cfg;
typedef struct {
  uint64_t pools, samples;
  double wall_ms;          /* from the first pool to the last result; excludes the
                              one-time allocation of the two pinned host pools */
  double produce_ms, train_wait_ms, producer_wait_ms;
  double loss_sum;
} gv_run_report;
gv_status gv_run(gv_ctx* ctx, const gv_augment_cfg* cfg, uint64_t total_samples,
                 gv_run_report* report);

/* ---- introspection / verification (tests) -------------------------------- */

/* Zig-zag relabel map: perm[orig] = new id; part_off[n_partitions+1]. */
gv_status gv_get_partition(gv_ctx* ctx, uint32_t* perm, uint64_t* part_off);
/* Integer alias table of context partition p over its members in local order
 * (prob[k], alias[k]; k < partition size), and the departure table over all
 * nodes in original order (p == UINT32_MAX). */
gv_status gv_get_alias(gv_ctx* ctx, uint32_t p, uint32_t* prob, uint32_t* alias,
                       uint64_t cap);
/* Bucket the pending pool without training (a3-a6) so that the blocks and
 * negatives can be inspected; the next gv_train_episode trains it. */
gv_status gv_prepare_episode(gv_ctx* ctx);
/* Global block layout of the prepared pool: pairs_out[2*P] local ids in
 * canonical (i,j) row-major block order; block_off[n*n+1]. Multi-process:
 * only this rank's block rows are filled. */
gv_status gv_debug_get_buckets(gv_ctx* ctx, uint32_t* pairs_out, uint64_t cap,
                               uint64_t* block_off);
/* Negatives of block (i,j) of the prepared pool: out[q*K + k] = local id in
 * context partition j, as the SGD kernel draws them (device Philox). */
gv_status gv_debug_get_negatives(gv_ctx* ctx, uint32_t i, uint32_t j,
                                 uint32_t* out, uint64_t cap);
/* One ordered update per sample with caller-given negatives (hand-derived
 * tests): u, v, negs in ORIGINAL ids, negs[q*K + k]. */
gv_status gv_train_explicit(gv_ctx* ctx, const uint32_t* u, const uint32_t* v,
                            const uint32_t* negs, uint64_t count, float lr);

/* Host-only schedule of rank d (of D) at offset step t for an n x n grid
 * (Alg. 3 P:244-253 with "partitions > GPUs ... in subgroups", P:233;
 * DESIGN.md §7): rank d owns vertex partitions [d*m, (d+1)*m), m = n/D,
 * and trains blocks (vpart[g], cpart[g]) for g = 0..m-1 in this order,
 * cpart[g] = (vpart[g] + t) mod n. After block 0 it sends context partition
 * send_part to rank send_to; it receives recv_part from rank recv_from,
 * which block wait_block of step t+1 needs. D == 1: no transfer
 * (send_part = recv_part = UINT32_MAX). The engine uses exactly this plan.
 * Errors: GV_ERR_INVALID_ARG (n == 0, n > 64, D == 0, n % D != 0, d >= D,
 * t >= n, out == NULL). Needs no GPU. */
typedef struct {
  uint32_t n_blocks;
  uint32_t vpart[64];
  uint32_t cpart[64];
  uint32_t send_part, send_to;
  uint32_t recv_part, recv_from;
  uint32_t wait_block;
} gv_step_plan;
gv_status gv_plan_step(uint32_t n, uint32_t D, uint32_t d, uint32_t t, gv_step_plan* out);

/* Bytes of device memory allocated by this context (all virtual ranks). */
gv_status gv_device_bytes(gv_ctx* ctx, uint64_t* bytes);

const char* gv_last_error(const gv_ctx* ctx); /* ctx may be NULL (global) */
const char* gv_status_string(gv_status s);
int gv_abi_version(void);
void gv_destroy(gv_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* GV_H_ */
