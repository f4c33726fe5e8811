/*
 * tts.h -- C-ABI of libtts: the data-parallel hot path of one beam-search
 * test-time-scaling (TTS) step on B200 (sm_100a).
 *
 * The method (arXiv 2509.00195, FlashTTS, section 3.1):
 * each TTS step (1) extends every live beam by one "thinking step" of tokens
 * -- a decode loop whose attention runs over a beam tree whose KV pages are
 * shared by prefix -- then (2) a process reward model
 * scores the beams and "the top-K candidates [are selected] globally with a
 * static branching factor" and "replicated to spawn the next set of
 * active beams".  Notation: N live beams per request, branching
 * factor M, K = N / M survivors.
 *
 * Entry points and the passage each one implements:
 *   tts_block_table_init_request  request install: all N beams start on the
 *                                 shared prompt (SURVEY ledger C2, C6, C7)
 *   tts_block_table_append        per-token KV append (Alg. 1 line 10
 *                                 GenerateOneToken; ledger C7, C11, C12)
 *   tts_prefix_attn_decode        prefix-shared decode attention over the beam
 *                                 tree (P:148 paged attention, P:257-263 prefix
 *                                 sharing, P:394 sibling grouping; ledger C10)
 *   tts_beam_select_fork          Select + DuplicateThenTruncate without
 *                                 truncation (Alg. 1 lines 15-19, P:345-347;
 *                                 P:181; ledger C3-C8)
 *   tts_block_table_release_request / _snapshot / _stats  lifecycle, debug
 *                                 checkpoint, unique/logical KV accounting
 *   tts_beam_select_global / tts_beam_fork_map / tts_lineage_*  multi-GPU
 *                                 global top-K over an NCCL all-gather of the
 *                                 scores, with lineage migration
 *
 * Memory ownership: the CALLER allocates every device buffer described by
 * tts_buffers_t (sizes from tts_query_buffer_bytes) and keeps it alive and
 * unmodified for the lifetime of the context.  libtts owns only its host-side
 * context.  Buffers
 * passed to individual calls (q, k/v, scores, out) are borrowed until the
 * stream work of that call completes.
 *
 * Pointer convention: a parameter whose name ends in _h is HOST memory; every
 * other pointer is DEVICE memory of the context's device.  All calls are
 * stream-ordered on the given cudaStream_t (passed as void*); calls marked
 * "syncs" synchronise that stream before returning.
 *
 * Errors: argument / shape / state errors detected on the host return a
 * non-zero tts_status_t and enqueue nothing.  Data-dependent errors (page pool
 * exhaustion) are recorded in the sticky device status word; every later
 * kernel of the context becomes a no-op until tts_device_status reads and
 * clears it, and the context state is then undefined (release and re-install
 * the affected requests).  NaN / out-of-range scores are not errors (ledger C4).
 *
 * Threading: one context is driven by one host thread; no internal locking.
 * Determinism: every integer output (survivors, parent maps, block tables,
 * refcounts, free set) is a pure function of the call sequence (ledger C20).
 */
#ifndef TTS_H
#define TTS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  TTS_OK = 0,
  TTS_ERR_INVALID_ARG = 1,   /* shape, range or N % M != 0      */
  TTS_ERR_UNSUPPORTED = 2,   /* head_dim not in {64,128}, G > 16, ...       */
  TTS_ERR_OUT_OF_PAGES = 3,  /* page pool exhausted (sticky device error)   */
  TTS_ERR_CAPACITY = 4,      /* request id / beams / pages exceed config    */
  TTS_ERR_STATE = 5,         /* request not installed / already installed   */
  TTS_ERR_CUDA = 6,
  TTS_ERR_NCCL = 7
} tts_status_t;

typedef struct tts_ctx* tts_ctx_t;

/* Static shape of a context.  Page size P tokens; a page id indexes the same
 * slot of every layer's K and V pool (ledger C9). */
typedef struct {
  int32_t num_layers;          /* L                                          */
  int32_t num_q_heads;         /* Hq                                         */
  int32_t num_kv_heads;        /* Hkv; G = Hq / Hkv consecutive q heads per kv head */
  int32_t head_dim;            /* d in {64, 128}                             */
  int32_t page_size;           /* P in {16} (tokens per page)                */
  int32_t max_requests;        /* request ids are 0 .. max_requests-1        */
  int32_t max_beams;           /* N_max (<= 1024); also the beam stride of q/out/k/v */
  int32_t max_pages_per_beam;  /* table row length                           */
  int64_t num_pages;           /* pool size                                  */
} tts_config_t;

/* Caller-owned device buffers (all sizes from tts_query_buffer_bytes). */
typedef struct {
  void* k_pool;            /* bf16 [L][num_pages][Hkv][P][d]  ("HND" pages) */
  void* v_pool;            /* fp16 [L][num_pages][Hkv][P][d]: V is stored in
                              fp16 (reading C14'); the bf16 input
                              converts exactly for 2^-14 <= |v| < 65520, a
                              finite |v| >= 65520 raises the sticky
                              TTS_ERR_UNSUPPORTED (stored as 0)           */
  int32_t* block_tables;   /* [max_requests][max_beams][max_pages_per_beam] */
  int32_t* seq_lens;       /* [max_requests][max_beams] tokens per beam     */
  int32_t* refcounts;      /* [num_pages]                                   */
  uint32_t* free_bitmap;   /* [ceil(num_pages/32)], bit = 1 means free      */
  int32_t* status;         /* [4] sticky device status word                 */
  void* workspace;         /* scratch, workspace_bytes                      */
  size_t workspace_bytes;
} tts_buffers_t;

typedef struct {
  size_t k_pool, v_pool, block_tables, seq_lens, refcounts, free_bitmap, status, workspace;
} tts_buffer_sizes_t;

/* Byte size of every caller-owned buffer for cfg.  Host only. */
tts_status_t tts_query_buffer_bytes(const tts_config_t* cfg_h, tts_buffer_sizes_t* sizes_h);

/* Create a context over caller-owned buffers on `device`; initialises the
 * allocator state (all pages free, refcounts 0, status 0) with blocking
 * device work on the default stream.  *out_h receives the handle. */
tts_status_t tts_create(const tts_config_t* cfg_h, const tts_buffers_t* bufs_h, int device,
                        tts_ctx_t* out_h);
tts_status_t tts_destroy(tts_ctx_t ctx);
const char* tts_status_str(tts_status_t s);

/* Reads and clears the sticky device status word (syncs). */
tts_status_t tts_device_status(tts_ctx_t ctx, void* stream, tts_status_t* out_h);

/* Number of kernels this context has launched so far (host counter). */
int64_t tts_launch_count(tts_ctx_t ctx);

/* Name of the attention kernel this context's decode calls launch:
 * "k_tree_umma" (tcgen05, d = 128, 4 <= G <= 16, one CTA resident per SM) or
 * "k_tree_attn" (mma.sync: d = 64, G < 4, or a device with more SMs than the
 * tcgen05 kernel's split-tile partial slots cover). */
const char* tts_attention_kernel(tts_ctx_t ctx);

/* a1. Install request `req` with n_beams beams on a prompt of prompt_len
 * tokens.  k_prompt / v_prompt: bf16 [L][prompt_len][Hkv][d].
 * Allocates ceil(prompt_len/P) pages (lowest free ids, position order),
 * points all beams' tables at them (refcount n_beams); a partial last prompt
 * page is copied for beams 1..n_beams-1 (eager CoW, ledger C6).
 * Errors: TTS_ERR_STATE if installed, TTS_ERR_CAPACITY if n_beams >
 * max_beams or prompt pages > max_pages_per_beam. */
tts_status_t tts_block_table_init_request(tts_ctx_t ctx, int32_t req, int32_t n_beams,
                                          int32_t prompt_len, const void* k_prompt,
                                          const void* v_prompt, void* stream);

/* a2. Append one token to every active beam of the n_req requests req_ids_h
 * (served in array order, beams ascending; ledger C7).  active_h: host uint8
 * [n_req][max_beams] (NULL = all n_beams active).  k_new / v_new: bf16
 * [L][n_req][max_beams][Hkv][d].  A beam with len % P == 0 first allocates
 * the lowest free page.  Inactive beams are untouched (ledger C12). */
tts_status_t tts_block_table_append(tts_ctx_t ctx, int32_t n_req, const int32_t* req_ids_h,
                                    const uint8_t* active_h, const void* k_new,
                                    const void* v_new, void* stream);

/* a4+a5. Decode attention for layers [layer_begin, layer_end) of every active
 * beam of the n_req requests, over all len tokens of the beam (the token just
 * appended included; ledger C11):
 *   out[l][i][b][h][:] = softmax_j(scale * q[l][i][b][h] . K_b[j][h/G]) V_b[j][h/G]
 * q: bf16 [layer_end-layer_begin][n_req][max_beams][Hq][d];
 * out: fp32, same shape; rows of inactive beams are not written.
 * Each KV page shared by several beams of a request is read from HBM once
 * per beam group and staged in shared memory for every beam and GQA head that
 * references it (the cascade/tree decomposition). */
tts_status_t tts_prefix_attn_decode(tts_ctx_t ctx, int32_t layer_begin, int32_t layer_end,
                                    int32_t n_req, const int32_t* req_ids_h,
                                    const uint8_t* active_h, const void* q,
                                    float softmax_scale, float* out, void* stream);

/* a2+a4 fused: tts_block_table_append then tts_prefix_attn_decode over all
 * layers [0, L) in one call (one round of host planning, same semantics as
 * the two calls in sequence).  Shapes as in those calls.  On the tcgen05 path
 * the call is k_alloc (only when a beam crosses a page boundary), k_plan
 * (append + page-list plan) and the persistent attention kernel, chained by
 * programmatic dependent launch; a call's k_plan may run while the previous
 * call's attention kernel still runs: its plan goes to the other half of a
 * double buffer, and the new token lands in a slot the previous call's plan
 * masks (P = 0 exactly there; the pool never holds a non-finite V).  Every
 * host-detectable error (unknown or repeated request, page-table capacity,
 * more than 1024 beam groups) is returned before anything is enqueued or the
 * host length mirror moves. */
tts_status_t tts_decode_step(tts_ctx_t ctx, int32_t n_req, const int32_t* req_ids_h,
                             const uint8_t* active_h, const void* k_new, const void* v_new,
                             const void* q, float softmax_scale, float* out, void* stream);

/* Live timing of the attention kernel: between tts_profile_begin and
 * tts_profile_end every attention launch (k_plan + attention kernel on the
 * tcgen05 path) is bracketed by CUDA events recorded on its own stream;
 * tts_profile_end syncs and returns the summed time (ms) and the number of
 * attention launches.  The events serialise consecutive calls (bench.py times
 * runs of calls between forks instead). */
tts_status_t tts_profile_begin(tts_ctx_t ctx);
tts_status_t tts_profile_end(tts_ctx_t ctx, double* attn_ms_h, int64_t* attn_launches_h);

/* a6+a7. For each of the n_req requests (array order): select the K = N/M
 * survivors by (score desc, index asc; NaN last, -0 == +0; ledger C3/C4),
 * sort them by index, and fork child c = r*M + j from survivors[r] (ledger
 * C5): rows and lengths copied, refcounts recounted, pages that drop to 0
 * freed before any allocation, then eager CoW of partial last pages for
 * children j >= 1 in (request, child) order (ledger C6, C7).
 * scores: fp32 device [n_req][max_beams].  parent_out (nullable, device):
 * int32 [n_req][max_beams] new -> old.  Errors: TTS_ERR_INVALID_ARG if
 * N % M != 0.  Syncs (reads the parent map back for the host length mirror). */
tts_status_t tts_beam_select_fork(tts_ctx_t ctx, int32_t n_req, const int32_t* req_ids_h,
                                  const float* scores, int32_t width_m, int32_t* parent_out,
                                  void* stream);

/* f2. Selection variants (DESIGN.md
 * ledger C23/C24).  Same call shape and fork rules as tts_beam_select_fork;
 * the parent map comes from:
 *   TTS_SELECT_TOPK     beam search, param = M (K = N/M survivors x M children);
 *   TTS_SELECT_DIVERSE  diverse selection (DVTS), param = B subtrees: subtree s
 *                       is beams [s N/B, (s+1) N/B) (DFS order); its best beam
 *                       spawns the N/B children of subtree s;
 *   TTS_SELECT_DYNAMIC  dynamic branching, param = M: the K = N/M beam-search
 *                       survivors get 1 + floor(q_i) children, q_i =
 *                       (N - K) w_i / sum(w) in fp64 (w = score if finite and
 *                       > 0, else 0; all 0 -> equal), the remaining children
 *                       by largest fractional part (ties: lower index).
 * Children of a survivor are contiguous, in survivor (index) order; every
 * child but the first of its parent copies a partially filled last page.
 * Errors: TTS_ERR_INVALID_ARG if N % param != 0 or the policy is unknown. */
enum { TTS_SELECT_TOPK = 0, TTS_SELECT_DIVERSE = 1, TTS_SELECT_DYNAMIC = 2 };
tts_status_t tts_beam_select_fork_policy(tts_ctx_t ctx, int32_t n_req, const int32_t* req_ids_h,
                                         const float* scores, int32_t policy, int32_t param,
                                         int32_t* parent_out, void* stream);

/* f3. Dynamic Prefix-Aware Scheduling under a memory budget (PAPER.md 4.2,
 * P:372-394; Appendix A; DESIGN.md ledger C30).  Schedules the beams of request
 * req (active_h: host uint8 [n_beams], NULL = all) for execution in batches
 * ("tries") under a KV budget of budget_pages pages: CoT = a beam's page list,
 * P(a, b) = shared leading pages; greedy order (order[0] = the first beam,
 * then the unscheduled beam with the largest P with its predecessor, ties to
 * the lower index -- for the DFS-ordered rows of ledger C5 P(a, b) is the
 * minimum of the adjacent rows' shared prefixes between a and b), tries =
 * consecutive beams of the order packed first-fit while their union of pages
 * fits the budget.  Outputs: order_h [n] (beam ids), trie_of_h [n_beams]
 * (trie of each scheduled beam), *n_tries_h, *cost_h = sum_i (Nodes(T_i) -
 * P(T_i, T_{i+1})) and *shared_h = sum_i P(T_i, T_{i+1}) in pages, P(T_last,.)
 * = 0 -- the pages a memory-bounded server evicts and recomputes per pass over
 * the beams.  Syncs (reads the request's tables). */
tts_status_t tts_dpas_plan(tts_ctx_t ctx, int32_t req, int64_t budget_pages, const uint8_t* active_h,
                           int32_t* order_h, int32_t* trie_of_h, int32_t* n_tries_h, int64_t* cost_h,
                           int64_t* shared_h, void* stream);

/* ---- f1: Speculative Beam Extension, decode side (PAPER.md 4.1, Alg. 1
 * P:324-350; DESIGN.md ledger C25-C29) ------------
 * While the stragglers of a step still generate, the slots of finished beams
 * run speculative branches of finished beams (SelectSpec); verification and
 * selection see only the non-speculative step (algorithmic equivalence); the
 * fork then continues children from the branches (DuplicateThenTruncate).
 * The serving loop calls, per iteration: tts_spec_select (which finished
 * beams get how many new branches), tts_spec_branch (the rows), the decode
 * step over originals still in their step + branches; at the step end:
 * tts_beam_select_global over the N original scores (parent map), tts_spec_plan
 * (children's source rows and lengths), tts_beam_fork_map_trunc. */

/* SelectSpec (host only, no context): candidate i (beam beam_h[i], previous
 * score last_score_h[i], have_h[i] branches already) has potential M_i =
 * B - j + 1, j = ceil((1 - s) B) clamped to [1, B] (s clamped to [0, 1], NaN ->
 * 0; fp64); candidates in (M desc, beam asc) order get min(M_i - have_i, free)
 * new branches until free_slots run out.  add_h[i] receives the count. */
tts_status_t tts_spec_select(int32_t n, const int32_t* beam_h, const float* last_score_h, const int32_t* have_h,
                             int32_t free_slots, int32_t B, int32_t* add_h);

/* Appends n rows to request req, row n_rows + i a fork of row src_rows_h[i]
 * (table and length copied, one more reference per page, a partially filled
 * last page copied into the lowest free page -- ledger C6/C7).  The new rows
 * take part in later decode calls (the request's beam count grows by n). */
tts_status_t tts_spec_branch(tts_ctx_t ctx, int32_t req, int32_t n, const int32_t* src_rows_h, void* stream);

/* DuplicateThenTruncate plan (host only): parent_h [N] the selection's parent
 * map (child -> surviving beam < N); branches: spare row N + i forked from
 * beam branch_src_h[i] with branch_tokens_h[i] speculative tokens; lens_h [N]
 * the beams' lengths; frac_h [N] the truncation fraction f of child c (used
 * when c is not the first child of its survivor); next_len_h [N] (nullable)
 * caps the kept tokens at the child's next step length.  Child c = r M + j of
 * survivor s continues branch j of s (the j-th created) when s has one, with
 * h = n (j = 0) or floor(f n) (j >= 1) of its tokens, else duplicates s
 * (h = 0).  Outputs parent_rows_h [N], new_len_h [N] (= lens[s] + h), head_h [N]. */
tts_status_t tts_spec_plan(int32_t N, int32_t M, const int32_t* parent_h, int32_t n_branch,
                           const int32_t* branch_src_h, const int32_t* branch_tokens_h, const int32_t* lens_h,
                           const double* frac_h, const int32_t* next_len_h, int32_t* parent_rows_h,
                           int32_t* new_len_h, int32_t* head_h);

/* tts_beam_fork_map with truncation: new row c keeps the first new_len_h[c]
 * (1 <= new_len <= the parent row's length) tokens of row parent_h[c]; a kept
 * partial last page (first child of its parent) has its slots past the new
 * length cleared, later children copy it (C6).  Syncs. */
tts_status_t tts_beam_fork_map_trunc(tts_ctx_t ctx, int32_t req, int32_t n_new, const int32_t* parent_h,
                                     const int32_t* new_len_h, void* stream);

/* ---- a8: one request's beams spanning G GPUs --------------
 * The request's N_global beams are held in G contiguous ranges of global ids
 * (gid = rank * N_local + local index; DFS order across ranks).  Per step:
 *   1. the caller all-gathers the N_local scores of every rank (NCCL over
 *      NVLink via torch.distributed; 4 B per beam) into scores_all;
 *   2. tts_beam_select_global on every rank computes the same global parent
 *      map (the single-GPU key, ledger C3/C4, with the global id as index;
 *      ledger C19), so survivors are identical on every rank;
 *   3. child gid c is placed on rank c / N_local (children of one survivor are
 *      consecutive, so each rank's beams stay a DFS-ordered run); a child whose
 *      parent lives on another rank receives the parent's lineage: the owner
 *      exports it (tts_lineage_export), the caller ships the buffer
 *      (NCCL send/recv), the destination imports it into a spare row
 *      (tts_lineage_import; fresh pages, lowest free ids);
 *   4. tts_beam_fork_map forks the local rows by an explicit parent map.
 * Page ids are per rank; survivors, parent maps and every beam's token
 * sequence equal the single-GPU run (ledger C20). */

/* Global selection over scores_all (device fp32 [n_global], n_global <= 1024,
 * n_global % width_m == 0).  parent_gid_out: device int32 [n_global],
 * new gid -> old gid.  No sync. */
tts_status_t tts_beam_select_global(tts_ctx_t ctx, int32_t n_global, const float* scores_all,
                                    int32_t width_m, int32_t* parent_gid_out, void* stream);

/* Fork request `req` by an explicit map: new row c (0 <= c < n_new) copies old
 * row parent_h[c] (host int32 [n_new]; old rows = the request's beams plus
 * imported lineages).  Refcounts recounted, released pages freed before any
 * allocation; the first child of each parent keeps a partially filled last
 * page, later children get a copy (ledger C6-C8).  Syncs. */
tts_status_t tts_beam_fork_map(tts_ctx_t ctx, int32_t req, int32_t n_new, const int32_t* parent_h,
                               void* stream);

/* Size of a lineage buffer for a beam of `len` tokens: [2 (K, V)][L][len][Hkv][d]
 * 16-bit values (K bf16, V fp16 as held in the pools). */
tts_status_t tts_lineage_bytes(tts_ctx_t ctx, int32_t len, size_t* bytes_h);

/* Copy beam `beam` of request `req` (all its tokens, every layer) into buf
 * (device, tts_lineage_bytes(len) bytes). */
tts_status_t tts_lineage_export(tts_ctx_t ctx, int32_t req, int32_t beam, void* buf, void* stream);

/* Install a lineage of `len` tokens from buf into the empty row `beam`
 * (beam >= the request's beam count): allocates ceil(len/P) fresh pages
 * (lowest free ids) and writes them.  Errors: TTS_ERR_STATE if the row is in
 * use; pool exhaustion is the sticky device error. */
tts_status_t tts_lineage_import(tts_ctx_t ctx, int32_t req, int32_t beam, int32_t len, const void* buf,
                                void* stream);

/* ---- a8 through the library: libtts-owned communicator --------------------
 * tts_beam_select_fork_global runs the whole cross-rank step:
 *   1. all-gather of (score, gid, len) of every local beam (12 B per beam);
 *   2. the selection kernel over the N gathered scores, the global id as index
 *      (ledger C19) -> the same parent map on every rank;
 *   3. placement, identical on every rank: children in gid order stay on
 *      their parent's rank while its capacity lasts; the overflow, in gid
 *      order, goes to the lowest rank with free capacity;
 *   4. migration: each rank imports the whole lineage (K bf16 / V fp16, every
 *      layer) of every remote parent one of its children needs, in ascending
 *      parent gid, into spare rows (fresh pages), in rounds that fit the
 *      staging buffer;
 *   5. local fork by the explicit parent map (tts_beam_fork_map): new row i =
 *      the rank's i-th child in ascending gid.
 * Transports: NCCL (tts_comm_init; libnccl.so.2 is resolved at run time --
 * the copy PyTorch loaded) or host callbacks (tts_comm_init_host: any byte
 * transport, e.g. a gloo process group, or threads of one process acting as
 * ranks).  Every rank of the communicator must make the same sequence of
 * span calls.  Survivors, parent maps, child -> rank and every beam's token
 * sequence are identical across runs and equal the single-GPU run; page ids
 * are per rank (ledger C20). */

/* Host transport: all calls are blocking and collective over the ranks. */
typedef struct {
  void* user;
  /* every rank contributes `bytes` from send_h; recv_h receives nranks * bytes
   * (rank order).  Returns 0 on success. */
  int (*allgather)(void* user, const void* send_h, void* recv_h, size_t bytes);
  /* grouped point-to-point: n_send messages to dst[i] from send_h[i]
   * (send_bytes[i]) and n_recv messages from src[i] into recv_h[i]
   * (recv_bytes[i]), matched in order per peer.  Returns 0 on success. */
  int (*sendrecv)(void* user, int32_t n_send, const int32_t* dst, const void* const* send_h,
                  const size_t* send_bytes, int32_t n_recv, const int32_t* src, void* const* recv_h,
                  const size_t* recv_bytes);
} tts_host_transport_t;

/* A fresh NCCL unique id (128 B, host) for rank 0 to broadcast.  TTS_ERR_NCCL
 * if libnccl.so.2 cannot be loaded. */
tts_status_t tts_comm_unique_id(void* id_h);

/* Joins the NCCL communicator (nranks, rank) of `id_h` on the context's
 * device.  stage: caller-owned device buffer (>= 4 KiB; holds the all-gather
 * records, then the two halves of every migration round). */
tts_status_t tts_comm_init(tts_ctx_t ctx, const void* nccl_unique_id_128B_h, int32_t nranks, int32_t rank,
                           void* stage, size_t stage_bytes);

/* Same over a host transport (copied; its user pointer must outlive the
 * context); libtts allocates a pinned host staging buffer of stage_bytes. */
tts_status_t tts_comm_init_host(tts_ctx_t ctx, int32_t nranks, int32_t rank, const tts_host_transport_t* t,
                                size_t stage_bytes);

/* Destroys the context's communicator (also done by tts_destroy). */
tts_status_t tts_comm_destroy(tts_ctx_t ctx);

/* Declares installed request `req` as spanning the communicator's ranks:
 * N = n_global beams, rank r holds caps_h[r] of them (sum = N, N <= 1024,
 * 2 * caps[r] <= max_beams for spare rows); this rank's rows are the
 * contiguous global ids [sum(caps[:rank]), sum(caps[:rank+1])) -- at install
 * every beam holds only the prompt, so the cut is byte-balanced.  The request
 * must have been installed with caps_h[rank] beams. */
tts_status_t tts_span_init(tts_ctx_t ctx, int32_t req, int32_t n_global, const int32_t* caps_h, int32_t dedup);

/* f4 (extends 8(e)): with dedup != 0 in tts_span_init the context
 * tracks every page's origin (who created it, where; equal on every rank
 * holding a copy).  A migrating lineage then crosses only the tokens past the
 * longest run of leading full pages some beam of the destination already
 * holds (same origins; ties to the lowest gid): the destination references
 * that beam's pages for the prefix and receives the rest.  Bytes this rank
 * sent and did not need to send, summed over the request's forks: */
tts_status_t tts_span_stats(tts_ctx_t ctx, int32_t req, int64_t* migrated_bytes_h, int64_t* deduped_bytes_h);

/* Global ids of this rank's rows of a spanning request (host int32 [n_local]). */
tts_status_t tts_span_gids(tts_ctx_t ctx, int32_t req, int32_t* gids_h);

/* The cross-rank select + fork of a spanning request (steps 1-5 above;
 * collective: every rank calls it).  local_scores: device fp32 [n_local]
 * (row order).  parent_gid_out (device int32 [N], nullable): new gid -> old
 * gid.  child_rank_out (device int32 [N], nullable).  Syncs. */
tts_status_t tts_beam_select_fork_global(tts_ctx_t ctx, int32_t req, const float* local_scores, int32_t width_m,
                                         int32_t* parent_gid_out, int32_t* child_rank_out, void* stream);

/* Placement rule alone (host only, no context): child gid -> rank from the
 * parent map (parent_gid_h [N]), the old gid -> rank map and the capacities. */
tts_status_t tts_span_placement(int32_t n_global, const int32_t* parent_gid_h, const int32_t* old_rank_h,
                                int32_t nranks, const int32_t* caps_h, int32_t* child_rank_h);

/* Release every page of request `req` (refcount decrement, free at 0). */
tts_status_t tts_block_table_release_request(tts_ctx_t ctx, int32_t req, void* stream);

/* Debug checkpoint (syncs): tables_h int32 [n_beams][max_pages_per_beam],
 * lens_h int32 [n_beams]; refcounts_h int32 [num_pages] and free_bitmap_h
 * uint32 [ceil(num_pages/32)] are nullable.  n_beams_h receives N. */
tts_status_t tts_block_table_snapshot(tts_ctx_t ctx, int32_t req, int32_t* n_beams_h,
                                      int32_t* tables_h, int32_t* lens_h,
                                      int32_t* refcounts_h, uint32_t* free_bitmap_h,
                                      void* stream);

/* KV accounting (ledger C22): adds to accum (device int64[2])
 * [0] += unique valid tokens over the distinct pages touched by the active
 * beams of the call, [1] += logical tokens (sum of active beams' len).
 * Does not sync. */
tts_status_t tts_block_table_stats(tts_ctx_t ctx, int32_t n_req, const int32_t* req_ids_h,
                                   const uint8_t* active_h, int64_t* accum, void* stream);

/* Host mirror of a request's beam lengths (no device access). */
tts_status_t tts_seq_lens_host(tts_ctx_t ctx, int32_t req, int32_t* lens_h);

/* Measurement helper (not part of the method; no context): the HBM read
 * bandwidth of the current device, from `iters` passes of a read-only 16-B
 * vector stream over `bytes` of device memory `buf` (make it >> the 126 MB
 * L2), timed with CUDA events on `stream` (syncs).  The read roofline of the
 * attention kernel, reported beside the copy peak. */
tts_status_t tts_stream_read_gbs(const void* buf, size_t bytes, int32_t iters, double* gbs_h, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* TTS_H */
