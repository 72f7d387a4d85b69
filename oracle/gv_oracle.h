/*
 * gv_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * The oracle's own header. It is NOT the product's header (include/gv.h) and
 * shares nothing with the CUDA path: no kernels, helpers, tables or
 * constants. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load liboracle.so.
 *
 * Citation keys: P:n = PAPER.md line n, S:n = SPEC.md line n,
 * "step k" = SURVEY.md §8(c) oracle step k, R-x = a reading in DESIGN.md.
 */
#ifndef GV_ORACLE_H_
#define GV_ORACLE_H_
#include <stdint.h>

#define OR_OK 0
#define OR_ERR_INVALID_ARG 1
#define OR_ERR_OUT_OF_RANGE 3
#define OR_ERR_EMPTY 4
#define OR_ERR_NOMEM 6

/* Philox4x32-10 (Salmon et al., SC'11 "Parallel random numbers: as easy as
 * 1, 2, 3"); step 4. */
void or_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);

/* Undirected weighted graph, CSR over ORIGINAL ids (step 1). */
typedef struct or_graph or_graph;
int or_graph_build(uint32_t nv, const uint32_t* src, const uint32_t* dst,
                   const float* w, uint64_t ne, or_graph** out);
void or_graph_free(or_graph* g);
uint64_t or_graph_entries(const or_graph* g);          /* directed entries = 2|E| */
void or_graph_csr(const or_graph* g, uint64_t* off, uint32_t* nbr, double* w);
void or_graph_degree(const or_graph* g, double* deg);

/* Degree-guided zig-zag partition (fig:zig-zag_partition; step 2). */
int or_zigzag(uint32_t nv, const double* deg, uint32_t n, uint32_t* perm,
              uint32_t* inv_perm, uint64_t* part_off);

/* Integer Vose alias table ("alias table trick"; step 3) and one draw
 * from (r0, r1, r2) (step 4). */
int or_alias_build(const double* w, uint32_t m, uint32_t* prob, uint32_t* alias);
uint32_t or_alias_draw(const uint32_t* prob, const uint32_t* alias, uint32_t m,
                       uint32_t r0, uint32_t r1, uint32_t r2);

/* Linear learning-rate decay (step 8). kind 0 = constant. */
float or_lr(int kind, double lr0, double floor_ratio, uint64_t s_before,
            uint64_t s_total);

/* One skip-gram negative-sampling update (Alg. 1 P:114-118, P:392;
 * step 9). U: vertex row; C[tau]: context rows of the targets in order
 * [v, n_1..n_K]; label 1 for tau = 0, 0 otherwise; omega 1 for tau = 0,
 * neg_weight otherwise. Returns the sample's loss in double. */
double or_sgd_sample(float* U, float* const* C, uint32_t n_targets, uint32_t d,
                     float lr, float neg_weight);

/* Stable counting sort of a pool into the n x n grid (Alg. 3 "Redistribute"
 * P:243; step 6). pairs in ORIGINAL ids; out in local ids. */
int or_bucket(const uint32_t* pairs, uint64_t count, uint32_t nv,
              const uint32_t* perm, const uint64_t* part_off, uint32_t n,
              uint32_t* out_local_pairs, uint64_t* block_off);

/* or_bucket, then inside each block (i, j) a stable sort of its samples by
 * vertex tile floor(u_local / 2^tile_bits) (reading R-VTILE: the block's
 * vertex partition i split into sub-partitions of 2^tile_bits rows, trained
 * one after the other — P:233's partitions-beyond-GPUs along the vertex
 * side only). tile_bits = 0: no tile order, identical to or_bucket. */
int or_bucket_tiled(const uint32_t* pairs, uint64_t count, uint32_t nv,
                    const uint32_t* perm, const uint64_t* part_off, uint32_t n,
                    uint32_t tile_bits, uint32_t* out_local_pairs, uint64_t* block_off);

/* Offset schedule of Alg. 3: context partition of vertex partition i
 * at offset step t. */
uint32_t or_schedule_cid(uint32_t n, uint32_t t, uint32_t i);

/* Whole trainer (steps 1-9). Embeddings are held in ORIGINAL id order. */
typedef struct or_trainer or_trainer;
int or_trainer_create(uint32_t nv, uint32_t d, uint32_t n, uint32_t K, float lr0,
                      int lr_kind, double floor_ratio, uint64_t total_samples,
                      uint64_t seed_neg, uint64_t seed_init, float neg_weight,
                      or_trainer** out);
int or_trainer_load_edges(or_trainer* t, const uint32_t* src, const uint32_t* dst,
                          const float* w, uint64_t ne);
int or_trainer_train_pool(or_trainer* t, const uint32_t* pairs, uint64_t count,
                          double* loss_out);
/* CPU baseline class (bench only, not a parity reference): train_pool with
 * each block's samples over `threads` OpenMP threads, lock-free. */
int or_trainer_train_pool_hogwild(or_trainer* t, const uint32_t* pairs, uint64_t count,
                                  int threads, double* loss_out);
/* R-VTILE for train_pool / train_pool_hogwild: bucket with or_bucket_tiled
 * (tile_bits = 0, the default, is or_bucket). */
int or_trainer_set_vertex_tile(or_trainer* t, uint32_t tile_bits);
/* Train one block (i,j) given its local pairs, pool index e and lr. */
int or_trainer_train_block(or_trainer* t, const uint32_t* local_pairs, uint64_t count,
                           uint32_t i, uint32_t j, uint32_t e, float lr, double* loss_out);
/* Negatives of block (i,j) at pool index e: out[q*K + k] local ids. */
int or_trainer_negatives(const or_trainer* t, uint64_t count, uint32_t i, uint32_t j,
                         uint32_t e, uint32_t* out);
uint32_t or_trainer_negative_at(const or_trainer* t, uint32_t q, uint32_t i, uint32_t j,
                                uint32_t e, uint32_t k);
int or_trainer_explicit(or_trainer* t, const uint32_t* u, const uint32_t* v,
                        const uint32_t* negs, uint64_t count, float lr);
void or_trainer_get(const or_trainer* t, int which, float* out);      /* 0 vertex, 1 context */
void or_trainer_set(or_trainer* t, int which, const float* in);
void or_trainer_partition(const or_trainer* t, uint32_t* perm, uint64_t* part_off);
int or_trainer_alias(const or_trainer* t, uint32_t p, uint32_t* prob, uint32_t* alias);
uint64_t or_trainer_samples_done(const or_trainer* t);
/* The trainer's ingested graph (owned by the trainer; NULL before
 * load_edges): a sampler can share it instead of ingesting the edges again. */
const or_graph* or_trainer_graph(const or_trainer* t);
void or_trainer_free(or_trainer* t);

/* Embedding initialisation (step 5): vertex[v][k] in [-0.5/d, 0.5/d). */
void or_init_vertex(uint32_t nv, uint32_t d, uint64_t seed, float* vertex);

/* Online augmentation (Alg. 2). */
typedef struct or_sampler or_sampler;
int or_sampler_create(const or_graph* g, or_sampler** out);
void or_sampler_free(or_sampler* s);
int or_sampler_walk(const or_sampler* s, uint32_t thread, uint32_t walk,
                    uint32_t walk_len, uint64_t seed, uint32_t* nodes /*walk_len+1*/);
uint64_t or_pairs_within(const uint32_t* walk, uint32_t len, uint32_t s, uint32_t* out);
void or_pseudo_shuffle(const uint32_t* in_pairs, uint64_t count, uint32_t s,
                       uint32_t* out_pairs);
int or_augment(const or_sampler* s, uint32_t walk_len, uint32_t dist, uint32_t threads,
               uint64_t count, uint64_t seed, uint32_t* out_pairs);

/* Link-prediction AUC: cosine similarity, rank statistic,
 * ties counted 1/2. */
double or_cosine(const float* a, const float* b, uint32_t d);
double or_auc(const double* pos, uint64_t npos, const double* neg, uint64_t nneg);
double or_linkpred_auc(const float* emb, uint32_t d, const uint32_t* pos_pairs,
                       uint64_t npos, const uint32_t* neg_pairs, uint64_t nneg);
#endif
