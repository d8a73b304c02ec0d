/*
 * s2v.h -- C ABI of libs2v.so, the sm_100a implementation of the
 * OpenGraphGym-MG structure2vec-DQN hot path (arXiv 2105.08764).
 *
 * Every entry point takes plain pointers (device pointers unless stated) and
 * sizes plus a cudaStream_t passed as void*; no torch types cross the boundary.
 * The host mirror of the reference's Python API (paper_2105_08764_b200/) binds
 * these with ctypes, exactly as a maintainer would bind them from the
 * reference's own `graphrl` package (INTEGRATION.md shows the stub).
 *
 * Each function cites the reference interface it replaces (paths relative to
 * /root/reference).  All calls are asynchronous on `stream` unless noted and
 * return an s2v_status; s2v_last_error() returns the message of the last
 * failure on the calling thread.
 *
 * Data layout:
 *   - a batch of B graphs with the same node count N, row-partitioned over P
 *     ranks (balanced blocks, pkg/src/graphrl/state.py:36-53);
 *   - embedding buffers are node-major [B][P][rows_max][K]; the physical row of
 *     node u of slot b owned by rank r is phys = (b*P + r)*rows_max + (u - row_start_r);
 *   - a local residual CSR over this rank's B*num_rows rows whose column entries
 *     hold the neighbour's physical row, ascending in original node id, with
 *     bit 31 set once the edge is removed (the reference zeroes the value,
 *     pkg/src/graphrl/state.py:173-208).
 */
#ifndef S2V_H_
#define S2V_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  S2V_OK = 0,
  S2V_EINVAL = 1,      /* ValueError                                   */
  S2V_EACTION = 2,     /* InvalidActionError (state.py:181-194)        */
  S2V_ECOMM = 3,       /* CollectiveError (collective.py:72-76)        */
  S2V_ECUDA = 4,       /* CUDA runtime failure                         */
  S2V_ENONFINITE = 5   /* non-finite gradient / target (policy.py:346) */
} s2v_status;

typedef enum { S2V_F32 = 0, S2V_F64 = 1 } s2v_dtype;

#define S2V_DEAD 0x80000000u

/* Residual graph shard of one rank (all pointers are device pointers).
 * Replaces PartitionedState's scipy CSR + sol/cand/local_residual
 * (pkg/src/graphrl/state.py:56-111). */
typedef struct {
  int64_t num_nodes;       /* N                                             */
  int32_t batch;           /* B                                             */
  int32_t world;           /* P                                             */
  int32_t rank;            /* r                                             */
  int32_t _pad;
  int64_t row_start;       /* first global node owned by this rank          */
  int64_t num_rows;        /* rows owned by this rank (per slot)            */
  int64_t rows_max;        /* padded rows per rank in embedding buffers     */
  int64_t nnz;             /* local entries over all slots                  */
  const int64_t *row_ptr;  /* [B*num_rows+1]                                */
  uint32_t *cols;          /* [nnz] phys neighbour row | S2V_DEAD           */
  const int64_t *col_ptr;  /* [B*N+1] local entries whose column is (b,u)   */
  const int64_t *col_ent;  /* [nnz]  entry index of those entries           */
  const int32_t *col_row;  /* [nnz]  local row (b*num_rows+i) of the entry  */
  int32_t *rdeg;           /* [B*num_rows] residual degree                  */
  uint8_t *sol;            /* [B*num_rows] partial solution S               */
  uint8_t *cand;           /* [B*num_rows] candidate set C                  */
  int64_t *residual;       /* [B] alive local entries                       */
  const int32_t *order;    /* [B*num_rows] processing order: the n_hub hub
                              rows (degree > S2V_HUB_DEGREE) first, then the
                              rest, each by descending degree; NULL = identity */
  int64_t n_hub;           /* rows handled by the CTA-cooperative hub kernel */
  const int32_t *active;   /* NULL, or the active-row list (B = 1; local rows,
                              any P; the compact CSR below at P > 1 needs
                              active_sol): a
                              stable subsequence of `order` holding every row
                              with rdeg > 0 (s2v_active_compact); the
                              forward rounds and the scorer then visit only
                              these rows (rows with rdeg = 0 keep the
                              constant h1_table row, see s2v_colsum_residual) */
  const int64_t *active_n; /* [2] device: rows in `active`, hub rows at its head */
  const int64_t *active_ptr;  /* NULL, or the compact CSR of the active list
                                 (s2v_active_compact): list position j has
                                 the entries active_cols[active_ptr[j] ..
                                 active_ptr[j+1]) -- the row's entries alive
                                 when it was built; one that died since has
                                 an endpoint in S, so rounds test sol[nbr] */
  const uint32_t *active_cols;
  const uint8_t *active_sol;  /* P > 1 with active_ptr: S of every physical
                                 row ([B*P*rows_max], this rank's and its
                                 peers', kept current by s2v_sol_mark) for
                                 the compact CSR's neighbour test; NULL at
                                 P = 1 (the test reads sol) */
} s2v_shard;

#define S2V_HUB_DEGREE 4096

/* ---- library ------------------------------------------------------------ */
const char *s2v_last_error(void);
const char *s2v_version(void);
/* Set the device of the calling thread (one thread/process per GPU). */
int s2v_set_device(int device);

/* ---- state (pkg/src/graphrl/state.py) ----------------------------------- */
/* Mark dead entries, compute rdeg/sol/cand/residual from a solution vector
 * indexed by physical row (sol_phys[B*P*rows_max]).  Replaces the residual
 * mask + row sums of PartitionedState.__init__ (state.py:89-111).
 * cols_src (nullable): the cached read-only column array of the graph's
 * structure, copied into sh->cols with the dead bits in the same pass. */
int s2v_shard_init(const s2v_shard *sh, const uint32_t *cols_src, const uint8_t *sol_phys,
                   void *stream);

/* Block-diagonal batch assembly (PartitionedState over B graphs): for each
 * segment, dst[dst_off + i] = src[i] + add, i < len, on 4- or 8-byte
 * integers -- the per-slot CSR, transpose and order arrays shifted by the
 * slot's entry / row offsets (state.py:89-105 builds the same block-diagonal
 * matrix with scipy).  segs is a device array. */
typedef struct {
  const void *src;
  int64_t dst_off; /* elements */
  int64_t len;     /* elements */
  int64_t add;
} s2v_segment;
int s2v_segment_copy(int elem_bytes, const s2v_segment *segs, int nseg, int64_t max_len,
                     void *dst, void *stream);

/* Apply one group of picks per slot (picks[B*d], -1 padded, global node ids)
 * with the reference's mid-group skip rule.  Replaces the group loop of
 * inference._solve_batch (inference.py:125-146) and apply_action
 * (state.py:173-208).  Two phases so that P>1 can exchange `info` between them:
 *   phase 1 (owner side): info[B*d*2] int64 = {rdeg(v_j), alive-adjacency mask
 *            of v_j to v_0..v_{d-1}} for locally owned picks, 0 elsewhere;
 *   (P>1: sum-all-reduce info over ranks)
 *   phase 2 (every rank): replay the skip rule, apply accepted picks to local
 *            rows/columns, write applied[B*d] (uint8) and removed[B] (int64,
 *            global entries removed = 2 * rdeg at apply time).
 * `validate` = 1 checks pick 0 of every slot is a candidate (owner side) and
 * fails with S2V_EACTION otherwise. */
int s2v_apply_phase1(const s2v_shard *sh, const int64_t *picks, int d, int64_t *info,
                     int validate, int32_t *err_out, void *stream);
int s2v_apply_phase2(const s2v_shard *sh, const int64_t *picks, int d, const int64_t *info,
                     uint8_t *applied, int64_t *removed, int first_forced, void *stream);
/* (first_forced = 1: pick 0 is applied unconditionally, the reference's
 * rule for the first pick of a group; groups larger than 64 are applied as
 * consecutive sub-groups of 64 with first_forced = 0 after the first.) */

/* ---- policy forward (pkg/src/graphrl/policy.py:144-224) ------------------ */
/* e12 table: table[(deg)][K] for deg in [0,max_deg] (sol=0) and row max_deg+1
 * for sol=1 (deg 0): fl(theta1*sol + fmachain(theta3, relu(theta2*deg))).
 * Replaces policy.py:157-161. */
int s2v_e12_table(s2v_dtype dt, const void *theta1, const void *theta2, const void *theta3,
                  int K, int max_deg, void *table, void *stream);

/* One embedding round over this rank's rows.  h_in == NULL means h = 0 (round
 * 1).  Writes h_out at this rank's physical rows; optionally m_out (the
 * aggregated neighbour sums, [B*num_rows][K]) for the training tape.
 * Replaces one iteration of policy.py:163-174 (spmm state.py:157-162 +
 * embed_fwd all-reduce + theta4 projection + relu). */
int s2v_embed_round(s2v_dtype dt, const s2v_shard *sh, const void *theta4, const void *table,
                    int K, int max_deg, const void *h_in, void *h_out, void *m_out,
                    void *stream);
/* Same round with the halo exchange fused in: every output row is also
 * stored into each of the npeers buffers peer_outs[q] (a device array of
 * IPC-mapped peer pointers, own buffer included) over NVLink, replacing the
 * per-round all-gather.  K = 64 fp32. */
int s2v_embed_round_peers(s2v_dtype dt, const s2v_shard *sh, const void *theta4,
                          const void *table, int K, int max_deg, const void *h_in, void *h_out,
                          void *const *peer_outs, int npeers, void *m_out, void *stream);

/* Round-1 outputs per e12 row: h1_table[t][k] = relu(table[t][k] + theta4 . 0)
 * with the round kernel's exact operation order, t in [0, max_deg+1].
 * K = 64 fp32. */
int s2v_h1_table(s2v_dtype dt, const void *theta4, const void *table, int K, int max_deg,
                 void *h1_table, void *stream);
/* Embedding round 2 without reading h1: round 1's output row of an alive
 * neighbour u (never in S) is h1_table[rdeg[u]], so the gather reads the
 * L1/L2-resident table instead of the 256-byte rows of h1, and round 1 needs
 * no halo exchange.  Same result bits as s2v_embed_round(h_in = h1).
 * deg_phys: residual degree by physical row of every rank (s2v_trow, then
 * the same all-gather as an embedding buffer with K = 1); NULL at P = 1
 * (this shard's rdeg).  peer_outs/npeers as s2v_embed_round_peers (fused
 * push of h2).  Replaces the second iteration of policy.py:163-174.
 * K = 64 fp32. */
int s2v_embed_round2_table(s2v_dtype dt, const s2v_shard *sh, const void *theta4,
                           const void *table, int K, int max_deg, const void *h1_table,
                           const int32_t *deg_phys, void *h_out, void *const *peer_outs,
                           int npeers, void *m_out, void *stream);
/* trow_phys[(b*P + rank)*rows_max + i] = sol ? max_deg + 1 : rdeg for this
 * rank's rows (the e12 table row of each node). */
int s2v_trow(const s2v_shard *sh, int max_deg, int32_t *trow_phys, void *stream);

/* Stable in-place compaction of an active-row list: keeps the rows of
 * list[0, n[0]) with rdeg > 0, in order, and updates n = {rows, rows among
 * the first n[1] (hub rows)}.  With row_ptr_out ([cap+1]) and cols_out
 * ([nnz]) it also writes the compact CSR of the kept rows (their alive
 * entries, in order, indexed by list position) for s2v_shard.active_ptr /
 * active_cols.  `cap` bounds n[0] (host-side capacity of
 * list, tmp); ws holds s2v_active_workspace(cap) int64.  The rows dropped
 * never come back: a residual degree only decreases during an episode
 * (state.py:173-208).  B = 1, any P (at P > 1 rounds reading the compact
 * CSR need s2v_shard.active_sol). */
int s2v_active_compact(const s2v_shard *sh, int32_t *list, int64_t *n, int32_t *tmp,
                       int64_t *ws, int64_t cap, int64_t *row_ptr_out, uint32_t *cols_out,
                       void *stream);
int64_t s2v_active_workspace(int64_t cap);
/* sol_all[phys(b, picks[b*d+j])] = 1 for every applied pick (picks global
 * node ids, -1 padded, identical on every rank after the key merge): keeps
 * the all-rank S of s2v_shard.active_sol current after a group apply
 * (inference.py:125-146 applies the same picks on every rank). */
int s2v_sol_mark(const s2v_shard *sh, const int64_t *picks, const uint8_t *applied, int d,
                 uint8_t *sol_all, void *stream);

/* Incremental-forward frontier (B = 1, P = 1 -- P > 1: the bitmap form below;
 * csrc/s2v_frontier.cu): the
 * rows whose round-l embedding may change after a group apply -- the picks
 * and their alive neighbours (seed, called BEFORE s2v_apply_phase2), then
 * `levels`-1 hops over the residual graph (expand, AFTER the apply).  D
 * [rows] gets the rows in BFS order, meta [s2v_frontier_meta_size(levels)]
 * the level prefixes: {meta[4+2l], 0} is the active_n pair of round l.
 * mark [rows] int32 stamps (zero-initialised once).  A frontier larger than
 * cap is replaced by the active list act[0, act_n[0]) for every level. */
int s2v_frontier_seed(const s2v_shard *sh, const int64_t *picks, int d, int levels, int32_t *D,
                      int64_t *meta, int32_t *mark, int64_t cap, void *stream);
int s2v_frontier_expand(const s2v_shard *sh, int levels, int32_t *D, int64_t *meta, int32_t *mark,
                        int64_t cap, const int32_t *act, const int64_t *act_n, int64_t act_cap,
                        void *stream);
int64_t s2v_frontier_meta_size(int levels);
/* P > 1 frontier on bitmaps over every rank's physical rows (B = 1;
 * s2v_frontier_bits_words uint32 words each): seed marks this rank's picks
 * and their alive neighbours into mbits (and clears gbits, the levels' union)
 * BEFORE s2v_apply_phase2; the ranks all-gather mbits as [P][words]; merge
 * ORs them, keeps newbits = the rows new at `level`, appends this rank's new
 * rows to D / meta exactly as s2v_frontier_seed / _expand do (and, at the
 * last level, the active-list fallback on overflow); expand marks the alive
 * neighbours of this rank's newbits rows for the next level (AFTER the
 * apply).  nodes: the global node ids in gbits (the global sum's dirty rows;
 * n[0] = count, n[1] = 0). */
int64_t s2v_frontier_bits_words(const s2v_shard *sh);
int s2v_frontier_bits_seed(const s2v_shard *sh, const int64_t *picks, int d, int levels,
                           int64_t *meta, uint32_t *mbits, uint32_t *gbits, void *stream);
int s2v_frontier_bits_expand(const s2v_shard *sh, const uint32_t *newbits, uint32_t *mbits,
                             void *stream);
int s2v_frontier_bits_merge(const s2v_shard *sh, const uint32_t *gathered, uint32_t *gbits,
                            uint32_t *newbits, int level, int levels, int32_t *D, int64_t *meta,
                            int32_t *mark, int64_t cap, const int32_t *act, const int64_t *act_n,
                            int64_t act_cap, void *stream);
int s2v_frontier_bits_nodes(const s2v_shard *sh, const uint32_t *gbits, int32_t *nodes,
                            int64_t *n, void *stream);

/* g[b][k] = numpy pairwise sum over the N nodes of slot b of h[.,k]; h must
 * hold every rank's rows (after an all-gather when P>1).  Replaces
 * embed.sum(axis=2) + q_fwd all-reduce (policy.py:199-200). */
int s2v_colsum(s2v_dtype dt, const s2v_shard *sh, int K, const void *h, void *g,
               void *workspace, size_t workspace_bytes, void *stream);
size_t s2v_colsum_workspace(const s2v_shard *sh, int K, int elem_bytes);
/* The same sums, reading h only for rows with rdeg > 0: a row with no alive
 * neighbour has m = 0 in every round, so its final embedding is the round-1
 * row h1_table[sol ? max_deg + 1 : 0] (s2v_h1_table) whatever h holds for
 * it -- rows outside the active list are never written.  P = 1.
 * Incremental (last != NULL, K = 64, [B*N] bytes kept between calls with the
 * same workspace and h1_table): a row only ever turns dead, so a pairwise
 * leaf whose rows are all dead now and were all dead at the previous call
 * keeps the leaf sum left in the workspace; full = 1 recomputes every leaf
 * (first call). */
int s2v_colsum_residual(s2v_dtype dt, const s2v_shard *sh, int K, const void *h,
                        const void *h1_table, int max_deg, void *g, void *workspace,
                        size_t workspace_bytes, uint8_t *last, int full,
                        const int32_t *dirty_rows, const int64_t *ndirty,
                        const int32_t *trow_phys, void *stream);
/* (dirty_rows, ndirty: incremental forward -- the global node ids whose
 * embedding changed (P = 1: the frontier rows; P > 1: s2v_frontier_bits_nodes);
 * only the leaves holding one of them are recomputed.
 * trow_phys: P > 1 (NULL at P = 1) -- every rank's e12 table row by physical
 * row (s2v_trow + the all-gather of round 2), which classifies every node of
 * the gathered buffer: 0 dead, max_deg + 1 in S, else alive.)  Workspace
 * bytes for s2v_colsum_residual: */
size_t s2v_colsum_residual_workspace(const s2v_shard *sh, int K, int elem_bytes);

/* Scores of this rank's rows: u2 = theta6 (h*cand), r = relu([u1;u2]),
 * score = sum_j fl(r_j theta7_j) (policy.py:201-207), masked selection keys
 * (policy.py:221-224 + inference.py:61-73 / agent.py:169) and per-block
 * top-8 keys.  cand_override (nullable, [B*num_rows]) replaces sh->cand as
 * the extractor (q_forward's `cand` argument).  mode 0 = solve semantics
 * (candidates with finite score), mode 1 = argmax/max semantics (NaN wins).
 * Outputs: scores[B*num_rows]; block_keys[B][nblk][8]; counts[B] (int64,
 * number of selectable nodes). */
int s2v_score(s2v_dtype dt, const s2v_shard *sh, int K, const void *h, const void *u1,
              const void *theta6, const void *theta7, const uint8_t *cand_override,
              int mode, void *scores, uint64_t *block_keys, int64_t *counts, void *stream);
int s2v_score_blocks(const s2v_shard *sh);
/* Scores of an active-row list (B = 1, K = 64 fp32) with a per-row
 * cache of the theta7 terms fl(relu(u2_k) theta7_{K+k}), prod_cache[rows][64]:
 * rows == NULL scores every list row and fills the cache; otherwise the
 * cache is refreshed for rows[0, nrows[0]) (the incremental frontier) and
 * every candidate's score is s0 + its cached terms, summed in the same
 * order (policy.py:201-207).  Keys and counts as s2v_score; scores[] is
 * written only by the rows == NULL form. */
int s2v_score_cached(const s2v_shard *sh, const float *h, const float *u1, const float *theta6,
                     const float *theta7, int mode, float *prod_cache, const int32_t *rows,
                     const int64_t *nrows, float *scores, uint64_t *block_keys, int64_t *counts,
                     void *stream);
/* Merge per-block keys into the top-d (d <= 8) keys per slot, descending.
 * A key is two uint64 {orderable(score), ~node}; {0,0} = none. */
int s2v_topk_merge(const s2v_shard *sh, const uint64_t *block_keys, int d, uint64_t *top,
                   void *stream);
/* For d > 8 (SelectionSchedule.fixed(d) allows any d): per-block top-8 of the
 * selection keys strictly below ceiling[b] (the last key already taken),
 * re-using the score pass's per-row keys (s2v_score_keys). */
int s2v_score_keys(const s2v_shard *sh, const void *scores_f32, const uint8_t *cand, int mode,
                   uint64_t *keys_all, void *stream);
int s2v_score_keys_f64(const s2v_shard *sh, const void *scores_f64, const uint8_t *cand,
                       int mode, uint64_t *keys_all, void *stream);
int s2v_topk_below(const s2v_shard *sh, const uint64_t *keys_all, const uint64_t *ceiling,
                   uint64_t *block_keys, void *stream);

/* ---- device-resident selection loop ----------------------- */
/* u1 = g @ theta5.T in numpy/OpenBLAS order (policy.py:201): B == 1 sgemv
 * order (K % 8 == 0, K >= 16) or B >= 32 sequential FMA; s2v_u1_exact tells
 * whether a (B, K) pair is covered (else the host computes u1 with numpy). */
int s2v_u1(s2v_dtype dt, int B, int K, const void *g, const void *theta5, void *u1,
           void *stream);
int s2v_u1_exact(int B, int K);
/* d = SelectionSchedule.d_for(count, N) and the first d keys as picks for
 * every active slot (inference.py:54-73,116-124); error = 1 on an active slot
 * without candidates ("empty candidate set"). */
int s2v_select(int B, int dmax, int64_t N, const double *fracs, const int *ds, int nthr,
               int fallback, const int64_t *counts, const uint64_t *keys, const uint8_t *active,
               int64_t *picks, int32_t *evaluated, int32_t *error, void *stream);
/* Append one evaluation (picks, applied, evaluated) to the trace and set
 * active = residual > 0 (inference.py:147). */
int s2v_trace(int B, int dmax, const int64_t *picks, const uint8_t *applied,
              const int32_t *evaluated, const int64_t *residual, uint8_t *active,
              int64_t *trace_picks, uint8_t *trace_applied, int32_t *trace_eval, void *stream);

/* ---- policy backward + Adam (policy.py:232-359) -------------------------- */
/* Number of CTAs (= partial rows) used by the backward reductions. */
int s2v_backward_blocks(const s2v_shard *sh);
/* grad_h[r] = dg[b] (+ dact[b] at the action row of slot b): the adjoint of
 * g = sum(embed) broadcast to every node plus the head term (policy.py:282-288). */
int s2v_grad_h_init(s2v_dtype dt, const s2v_shard *sh, int K, const void *dg,
                    const int64_t *actions, const void *dact, void *grad_h, void *stream);
/* One layer of policy.py:290-303: dz = grad_h * (h_l > 0); dzsum (+)= dz;
 * partial[blk][K*K] (+)= dz (x) m_l (m_l NULL for layer 1); dm = theta4^T dz
 * written at this rank's physical rows of dm_out (NULL for layer 1).
 * first = 1 initialises dzsum and partial instead of accumulating. */
int s2v_layer_backward(s2v_dtype dt, const s2v_shard *sh, int K, const void *theta4,
                       const void *grad_h, const void *h_l, const void *m_l, void *dzsum,
                       void *partial, int first, void *dm_out, void *stream);
/* out[r] = sum over alive neighbours (ascending id) of src[phys] -- spmm_t
 * (state.py:164-169); src holds every rank's rows. */
int s2v_gather(s2v_dtype dt, const s2v_shard *sh, int K, const void *src, void *out,
               void *stream);
/* Partials [blk][2K + K*K] of dtheta1, dtheta2, dtheta3 from dzsum
 * (policy.py:294-296,305-306; dw_acc = theta3^T dzsum by linearity).
 * t2c (optional, s2v_theta2_terms_bytes) receives the einsum terms
 * fl(fl(dw_acc * (w > 0)) * deg) of policy.py:305-306 in the chain layout
 * [b][ceil(K/G)][rows][G], G = 32 / sizeof(T), for s2v_theta2_einsum. */
int s2v_param_grads(s2v_dtype dt, const s2v_shard *sh, int K, const void *theta2,
                    const void *theta3, const void *dzsum, void *partials, void *t2c,
                    void *stream);
size_t s2v_theta2_terms_bytes(s2v_dtype dt, const s2v_shard *sh, int K);
/* dtheta2 (policy.py:305-306) in numpy 2.3's einsum("bkv,bv->k") order:
 * per (b, k), 16/sizeof(T) lane chains over v (4-vector unroll taken in
 * reverse, zero-filled tail), lanes combined pairwise, slots added in b
 * order.  tot: scratch [B][K] of T; out[K] (fp64) = this rank's dtheta2. */
int s2v_theta2_einsum(s2v_dtype dt, const s2v_shard *sh, int K, const void *t2c, void *tot,
                      double *out, void *stream);
/* out[len] (fp64) = sum over nparts partial rows, fixed order. */
int s2v_reduce_partials(s2v_dtype dt, const void *partials, int nparts, int len, double *out,
                        void *stream);
/* Q head at the action node of every slot owned by this rank
 * (policy.py:256-283): head_out[b][2K*K + 2K + 1] fp64 = dtheta5, dtheta6,
 * dtheta7, squared error; dg[b][K] = theta5^T dpre[:K]; dact[b][K] =
 * theta6^T dpre[K:].  Zeros for slots whose action another rank owns. */
int s2v_head_backward(s2v_dtype dt, const s2v_shard *sh, int K, const void *h_L,
                      const void *g, const int64_t *actions, const void *targets,
                      const void *theta5, const void *theta6, const void *theta7,
                      double *head_out, void *dg, void *dact, void *stream);
/* Bias-corrected Adam with the reference's element-wise rounding
 * (policy.py:339-359); omb1/omb2 = the host's (1 - beta1), (1 - beta2);
 * b1c/b2c = 1 - beta^t computed on the host in fp64. */
int s2v_adam(s2v_dtype dt, void *params, const void *grads, void *m, void *v, int64_t n,
             double beta1, double omb1, double beta2, double omb2, double eps, double lr,
             double b1c, double b2c, void *stream);
/* The same update for iteration `it` of a device-resident train_step loop
 * (agent.py:235-261): gradients are the first n entries of the fp64 pack of
 * s2v_reduce_partials, rounded to the parameter dtype; bad[it] is set if
 * any is non-finite, and the update is skipped if any of bad[0..it] is set
 * (adam_step rejects a non-finite step before touching state,
 * policy.py:346-349). */
int s2v_adam_pack(s2v_dtype dt, void *params, const double *pack, void *m, void *v, int64_t n,
                  double beta1, double omb1, double beta2, double omb2, double eps, double lr,
                  double b1c, double b2c, int32_t *bad, int it, void *stream);

/* ---- one whole policy evaluation of the selection loop ------------------- */
/* The device episode loop's evaluation (inference.py:107-147) as ONE call:
 * rounds (round 2 from the degree table when h1_table is set), global sum,
 * u1, scores and top-d keys, the d rule and picks, the group apply and the
 * trace row c -- the same entry points in the same order as the host-driven
 * sequence, without a host call per launch.  P = 1, fp32, no active list;
 * the e12 table (and h1 table) must be current for the packed theta. */
typedef struct {
  int K, L, max_deg, dmax;
  const float *theta;        /* theta1..theta7 packed as param_shapes (device) */
  const float *table;        /* e12 table */
  const float *h1_table;     /* NULL: round 1 runs and round 2 reads h1      */
  float *h[2];               /* ping-pong embedding buffers                  */
  void *colsum_ws;
  size_t colsum_ws_bytes;
  float *g, *u1, *scores;
  uint64_t *block_keys;
  int64_t *out;              /* counts [B], then top keys [B][dmax][2]       */
  const double *fracs;       /* host: schedule thresholds (s2v_select)       */
  const int *ds;
  int nthr, fallback;
  uint8_t *active;
  int64_t *picks;
  int32_t *evaluated, *error;
  int64_t *info;
  uint8_t *applied;
  int64_t *removed;
  int64_t *t_picks;          /* [chunk][B*dmax]; row c written                */
  uint8_t *t_applied;        /* [chunk][B*dmax]                               */
  int32_t *t_eval;           /* [chunk][B]                                    */
} s2v_eval_plan;
int s2v_eval_chain(const s2v_shard *sh, const s2v_eval_plan *plan, int c, void *stream);

/* P > 1 device loop helpers.  gathered = every rank's score read-back
 * vector (counts [B], then top-d keys [B][d][2]) as [P][B*(1+2d)] after a
 * device all-gather; out = the global counts and top-d keys in the same
 * layout, identical on every rank (replaces policy.merge_rank_keys, the host
 * all_gather of keys, inference.py:113).  s2v_sum_ranks: out = sum over the
 * P gathered rows of n int64 (the group-apply info, in rank order).
 * s2v_sub_i64: a -= b (the global residual after a group apply). */
int s2v_merge_rank_keys(int P, int B, int d, const int64_t *gathered, int64_t *out,
                        void *stream);
int s2v_sum_ranks(int P, int64_t n, const int64_t *gathered, int64_t *out, void *stream);
int s2v_sub_i64(int64_t *a, const int64_t *b, int n, void *stream);

/* Device build of one graph's local shard structure (state.py:89-105 CSR
 * rows, state.py:115-122 column lookup), all arrays device memory:
 * row_ptr [rows+1] local (0-based), nbr [nnz] global neighbour ids ->
 * cols0 [nnz] (physical rows at P > 1), col_ptr [n+1], col_ent [nnz] (stable
 * argsort of nbr), col_row [nnz], order [rows] (stable descending-degree
 * argsort); n_hub_out / max_deg_out: host. */
int s2v_shard_structure(int64_t n, int P, int64_t rows_max, int64_t rows, const int64_t *row_ptr,
                        const int32_t *nbr, int64_t nnz, int32_t *cols0, int64_t *col_ptr,
                        int64_t *col_ent, int32_t *col_row, int32_t *order, int64_t *n_hub_out,
                        int32_t *max_deg_out, void *stream);

/* ---- handle-level API: library-owned device memory -------
 * Plain host arrays in and out, one call per reference operation; the
 * library allocates and owns every device buffer behind three opaque
 * handles.  Node-sharded P > 1: one context per rank, every call below
 * collective (all ranks call it in the same order, as run_workers' threads
 * call the reference's API, collective.py:143-195); each rank owns the block
 * partition_rows(N, P)[rank] of every graph (state.py:36-53), rounds
 * all-gather every rank's rows of h (policy.py:168) and the global sums are
 * rank-ordered all-reduces (collective.py:100-117), so every rank returns
 * the same keys, loss and gradients.  Same kernels, same order, same bits as
 * the Python mirror.  theta is theta1..theta7 packed in PARAM_NAMES order with the
 * reference's shapes (policy.py:43-113): K, K, K*K, K*K, K*K, K*K, 2K. */
typedef struct s2v_ctx s2v_ctx;
typedef struct s2v_graph s2v_graph;
typedef struct s2v_state s2v_state;
typedef struct s2v_group s2v_group;
enum { S2V_OUT_EMBED = 0, S2V_OUT_SOL = 1, S2V_OUT_CAND = 2, S2V_OUT_RDEG = 3,
       S2V_OUT_RESIDUAL = 4, S2V_OUT_SCORES = 5 };
/* one context per rank: run_workers' rank thread (collective.py:149-195).
 * world > 1: ranks join through NCCL; nccl_id = the bytes of
 * s2v_comm_unique_id made by one rank and shared (one rank per GPU). */
int s2v_ctx_create(int device, int rank, int world, const void *nccl_id, s2v_ctx **out);
/* in-process group of `world` thread ranks (WorkerGroup, collective.py:143):
 * s2v_ctx_create_in_group joins rank `rank` on `device` (any devices, one
 * GPU may hold several ranks); peers' chunks are copied on the streams
 * (NVLink P2P between GPUs) and ordered with CUDA events plus a host
 * rendezvous that fails with S2V_ECOMM after 300 s without a peer
 * (collective.py:134-139).  Destroy the group after its contexts. */
int s2v_group_create(int world, s2v_group **out);
int s2v_group_destroy(s2v_group *g);
int s2v_ctx_create_in_group(int device, int rank, s2v_group *group, s2v_ctx **out);
int s2v_ctx_destroy(s2v_ctx *ctx);
int s2v_ctx_sync(s2v_ctx *ctx);
/* Graph.csr_arrays() (host row_ptr [n+1], cols [row_ptr[n]], the whole
 * graph on every rank) -> this rank's device shard structure
 * (state.py:89-105, 115-122) */
int s2v_graph_upload(s2v_ctx *ctx, int64_t n, const int64_t *row_ptr, const int32_t *cols,
                     s2v_graph **out);
int s2v_graph_destroy(s2v_graph *g);
/* PartitionedState(graphs, part, solutions) (state.py:56-111): sol host
 * [B][N] 0/1 bytes over every node, or NULL */
int s2v_state_create(s2v_ctx *ctx, s2v_graph *const *graphs, int B, const uint8_t *sol,
                     s2v_state **out);
int s2v_state_destroy(s2v_state *st);
int s2v_state_shard(const s2v_state *st, s2v_shard *out);
/* embed_forward (policy.py:144-185); the embedding stays in the state */
int s2v_embed(s2v_ctx *ctx, s2v_state *st, s2v_dtype dt, const void *theta, int K, int L);
/* g = embed.sum(axis=2) (policy.py:199-200), host [B][K] */
int s2v_global_sum(s2v_ctx *ctx, s2v_state *st, void *g_host);
/* q_forward + masked_scores + top-d keys (policy.py:188-224,
 * inference.py:61-73): keys_out host [B][d][2] {orderable score, ~node},
 * ncand_out host [B]; d <= 8 */
int s2v_score_topk(s2v_ctx *ctx, s2v_state *st, int d, uint64_t *keys_out, int64_t *ncand_out);
/* one group of picks per slot with the mid-group skip rule
 * (inference.py:125-146, state.py:173-208): picks host [B][d] (-1 padded) */
int s2v_apply(s2v_ctx *ctx, s2v_state *st, const int64_t *picks, int d, uint8_t *applied,
              int64_t *residual);
/* loss_and_gradients (policy.py:232-315): grads host, packed like theta */
int s2v_loss_grad(s2v_ctx *ctx, s2v_state *st, s2v_dtype dt, const void *theta, int K, int L,
                  const int64_t *actions, const void *targets, void *grads, double *loss);
/* adam_step (policy.py:339-359) in place on host arrays; step = new t */
int s2v_adam_update(s2v_ctx *ctx, s2v_dtype dt, void *params, const void *grads, void *m,
                    void *v, int64_t n, int step, double lr, double beta1, double beta2,
                    double eps);
/* host copy of a state array (S2V_OUT_*): EMBED [B][N][K] (every node);
 * SOL, CAND [B][rows] uint8, RDEG [B][rows] int32, SCORES [B][rows] over
 * this rank's rows; RESIDUAL [B] alive local entries */
int s2v_copy_out(s2v_ctx *ctx, const s2v_state *st, int what, void *host);

/* ---- graph ingestion (graphs.py:125-157) --------------------------------- */
/* Bit-exact generate_ba from numpy's PCG64 state {state_hi, state_lo, inc_hi,
 * inc_lo, has_uint32, uinteger} (host memory).  edges_out == NULL returns E. */
int64_t s2v_generate_ba(int64_t n, int64_t d, const void *pcg, void *edges_out);
/* R-MAT scale/edge_factor (BASELINE cfg5; graphs.generate_rmat's definition,
 * the reference has none); edges_out holds edge_factor*2^scale pairs. */
int64_t s2v_generate_rmat(int scale, int64_t edge_factor, const void *pcg, double a, double b,
                          double c, int64_t chunk, void *edges_out);
/* Symmetric CSR (ascending rows) of a sorted unique u < v edge list
 * (Graph.csr_arrays; state.py:89-105 builds it with scipy). Host memory. */
int s2v_build_csr(int64_t n, const int64_t *edges, int64_t E, int64_t *row_ptr, int32_t *cols);

/* ---- collectives (replaces collective.py's in-process Comm) -------------- */
int s2v_comm_unique_id(void *out, size_t len);
int s2v_comm_init(const void *unique_id, int world, int rank, void **comm);
int s2v_comm_destroy(void *comm);
/* in-place when send == recv + rank*bytes */
int s2v_comm_allgather(void *comm, const void *send, void *recv, size_t bytes, void *stream);
int s2v_comm_allgather_slots(void *comm, void *recv, size_t bytes, size_t slot_stride,
                             int nslots, int rank, void *stream);
int s2v_comm_allreduce(void *comm, void *buf, size_t count, int kind /*0 i64 1 f64 2 f32*/,
                       void *stream);
/* Rank-ordered all-reduce (collective.py:100-117: result = rank 0's values,
 * then += rank 1, rank 2, ... -- identical bits on every rank and equal to the
 * reference's in-process sum): NCCL all-gather into scratch [P][count], then
 * s2v_sum_ranks_typed.  The peer-memory transports push into every peer's
 * scratch and call s2v_sum_ranks_typed directly. */
int s2v_comm_allreduce_ordered(void *comm, void *buf, size_t count, int kind, void *scratch,
                               void *stream);
int s2v_sum_ranks_typed(int kind /*0 i64 1 f64 2 f32*/, int P, int64_t n, const void *gathered,
                        void *out, void *stream);
/* cudaDeviceEnablePeerAccess from the current device (thread-ranks of one
 * process on different GPUs: NVLink P2P loads/stores of peer buffers). */
int s2v_enable_peer_access(int peer_device);
/* cudaMemcpyAsync(..., cudaMemcpyDefault): the in-process thread-group
 * transport (ranks as threads, possibly sharing one device) moves halo chunks
 * with peer copies instead of NCCL. */
int s2v_memcpy_async(void *dst, const void *src, size_t bytes, void *stream);
/* Peer-memory transport for process ranks: IPC export/import of device
 * allocations (handle_out: 64 bytes; offset of ptr inside its allocation) and
 * stream-ordered flags (write a value after prior work / wait until >=). */
int s2v_ipc_export(const void *ptr, void *handle_out, uint64_t *offset_out);
int s2v_ipc_import(const void *handle, void **base_out);
int s2v_ipc_close(void *base);
int s2v_stream_write_u32(void *addr, uint32_t value, void *stream);
int s2v_stream_wait_u32(void *addr, uint32_t value, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* S2V_H_ */
