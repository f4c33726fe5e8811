// Internal declarations of libtts (not part of the C-ABI).
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <map>
#include <vector>

#include "../../include/tts.h"

#define TTS_CUDA(call)                                      \
  do {                                                      \
    cudaError_t e_ = (call);                                \
    if (e_ != cudaSuccess) return TTS_ERR_CUDA;             \
  } while (0)

namespace tts {

constexpr int kUploadSlots = 64;
constexpr size_t kUploadSlotBytes = 256 * 1024;

// One CTA group of the attention kernel: a contiguous run of beams of one
// request (DFS order, so every shared page's beams form a sub-run).
struct GroupDesc {
  int32_t call_idx;    // index of the request in the call (q/out stride)
  int32_t req;         // request id
  int32_t beam0;       // first beam slot
  int32_t nbeams;      // beams in the group (<= 32)
  uint32_t active;     // bit i: beam0 + i active
  int32_t max_npages;  // max over active beams of ceil(len / P)
  int32_t pad[2];  // pad[0]: offset of the group's beam lengths in the call's length list
};

// Allocation item: table entry to receive a fresh page.
struct AllocItem {
  int64_t entry;  // flat index into block_tables
  int32_t cow;    // 1: old entry value is a CoW source (ref -1, copy recorded)
  int32_t ntok;   // tokens to copy when cow
};

struct CowCopy {
  int32_t src, dst, ntok, pad;
};

struct Comm;  // span.cu: NCCL communicator or host transport of a multi-GPU context

// A request whose beams span the ranks of the context's communicator (a8):
// rank r holds caps[r] beams, local rows in ascending global id.
struct Span {
  int n_global = 0;
  std::vector<int32_t> caps;
  std::vector<int32_t> gids;
  // f4 (cross-GPU page deduplication): the origin of every page of every row
  // ([max_beams][max_pages_per_beam]): who created the page where, identical
  // on every rank holding a copy; a full page's content is a function of it
  bool dedup = false;
  std::vector<uint64_t> origin;
  uint32_t tau = 0;  // decode calls of the request so far (the same on every rank)
  int64_t migrated_bytes = 0, deduped_bytes = 0;
};

struct Ctx {
  tts_config_t cfg;
  tts_buffers_t buf;
  int device = 0;
  int num_sms = 148;
  int64_t launches = 0;
  // host mirror of lengths / beam counts (lengths change only through the API)
  std::vector<int32_t> n_beams;  // per request, 0 = not installed
  std::vector<int32_t> lens;     // [max_requests][max_beams]
  std::vector<int32_t> n_rows;   // per request: rows in use (>= n_beams while imported lineages wait)
  // pinned upload ring
  uint8_t* pinned = nullptr;
  cudaEvent_t ev[kUploadSlots];
  int up_pos = 0;
  // workspace carve (device)
  int32_t* ws_tmp_tables = nullptr;  // [max_requests * max_beams * max_pages]
  int32_t* ws_tmp_lens = nullptr;    // [max_requests * max_beams]
  int32_t* ws_parent = nullptr;      // [max_requests * max_beams]
  int32_t* ws_pages = nullptr;       // allocator output list
  CowCopy* ws_cow = nullptr;         // [max_alloc]
  int32_t* ws_mark = nullptr;        // [num_pages] (stats)
  uint8_t* ws_upload = nullptr;      // device mirror of the upload ring
  int64_t max_alloc = 0;
  // live attention timing (tts_profile_begin/_end)
  bool profiling = false;
  std::vector<cudaEvent_t> prof_ev;  // pairs
  int prof_pos = 0;
  int64_t prof_count = 0;
  double prof_ms = 0.0;
  // TMA descriptors (K / V pools, 2D view [rows][d])
  CUtensorMap tmap_k, tmap_v;
  bool tmap_ok = false;
  // 3D view [2 (d halves)][rows][64] of the same pools: one TMA = one 16x128 tile
  CUtensorMap tmap3_k, tmap3_v;
  bool tmap3_ok = false;
  // attention plan (a3): per-group distinct-page lists
  // two buffers, alternating per call, so that the next call's k_plan may run
  // while this call's attention kernel still reads its plan
  int4* ws_items = nullptr;      // [2][max_requests * max_beams * max_pages_per_beam]
  int32_t* ws_counts = nullptr;  // [2][max_requests * max_beams]
  int plan_parity = 0;
  float* ws_partial = nullptr;     // split tiles' partial (m, l, O) (attention_umma.cu)
  int32_t* ws_tile_cnt = nullptr;  // [num_layers * num_kv_heads * max groups], zero between launches
  size_t tile_cnt_bytes = 0;
  // environment toggles (tools / tests), read once in tts_create
  bool env_attn_mma = false;  // TTS_ATTN=mma: force the mma.sync path
  int env_group_beams = 0;    // TTS_GROUP_BEAMS: beams per group on the tcgen05 path
  int env_ncons = 0;          // TTS_NCONS: consumer warps of the mma.sync path
  int env_poly = 0;           // TTS_POLY=1: polynomial exp2 for every other pair, 2: for all
  bool env_no_pdl = false;    // TTS_NO_PDL: no programmatic dependent launch
  bool umma_ok = false;       // tcgen05 path usable on this device (umma_prepare)
  int env_round_robin = 0;    // TTS_ROUND_ROBIN=1: beam b of a group on lane quadrant b % 4
  int env_l2hint = 0;         // TTS_L2HINT=1-3: L2 eviction priorities by cross-group sharing (k_tree_umma; DRAM bytes unchanged, off)
  int env_pair = 0;           // TTS_PAIR=1: 2-CTA clusters for groups of > umma_max_beams beams (measured slower)
  int env_sched = 2;          // TTS_SCHED: phase-1 tile assignment of k_tree_umma (0 rotated, 1 round-robin, 2 none:
                              // every unit split evenly, measured fastest on C3)
  int env_split_partial = 0;  // TTS_SPLIT_PARTIAL=1: a partial last round of tiles goes through stream-K
  int umma_occupancy = 0;     // resident k_tree_umma CTAs per SM found by umma_prepare
  int umma_pair_ctas = 0;     // pair mode: CTAs of the co-resident 2-CTA clusters (0: pair mode unavailable)
  // multi-GPU (span.cu)
  Comm* comm = nullptr;
  std::map<int, Span> spans;
  float* ws_scores_all = nullptr;   // [1024] gid-indexed scores of a global selection
  int32_t* ws_parent_all = nullptr;  // [1024] global parent map
};

// ---- pool value format --------------------------------------------------------
// K is stored as given (bf16).  V is stored as fp16 so that the PV product runs
// as one fp16 x fp16 tensor-core MMA with fp16 P (SURVEY ledger C14: fp16 P
// with V in fp16 <= 3.6e-4 row-normwise).  bf16 -> fp16 is exact for
// 2^-14 <= |v| < 2^16 (subnormal fp16 below; abs error <= 2^-25); a finite
// |v| >= 2^16 has no fp16 value and raises the sticky TTS_ERR_UNSUPPORTED.
// Every slot of an allocated page that holds no token is zero-filled, so no
// kernel ever reads stale pool data.
__device__ __forceinline__ uint32_t bf16x2_to_f16x2(uint32_t u) {
  uint32_t r;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(__uint_as_float(u & 0xFFFF0000u)), "f"(__uint_as_float(u << 16)));
  return r;
}
__device__ __forceinline__ bool bf16x2_beyond_f16(uint32_t u) {
  const uint32_t el = (u >> 7) & 0xFF, eh = (u >> 23) & 0xFF;
  return (el >= 0x8F && el < 0xFF) || (eh >= 0x8F && eh < 0xFF);
}
// (a value with no fp16 representation is stored as 0 next to the sticky error,
// so the pool never holds a non-finite V: masked columns multiply it by P = 0)
__device__ __forceinline__ uint4 v_to_pool(uint4 v, int32_t* status) {
  if (bf16x2_beyond_f16(v.x) | bf16x2_beyond_f16(v.y) | bf16x2_beyond_f16(v.z) | bf16x2_beyond_f16(v.w)) {
    atomicExch(status, (int32_t)TTS_ERR_UNSUPPORTED);
    return make_uint4(0, 0, 0, 0);
  }
  return make_uint4(bf16x2_to_f16x2(v.x), bf16x2_to_f16x2(v.y), bf16x2_to_f16x2(v.z), bf16x2_to_f16x2(v.w));
}

// Device-copy a host blob through the pinned ring; returns device pointer.
void* upload(Ctx* c, const void* src, size_t bytes, cudaStream_t s, cudaError_t* err);
void upload2(Ctx* c, const void* a, size_t na, const void* b, size_t nb, cudaStream_t s, cudaError_t* err,
             void** da, void** db);

size_t workspace_bytes(const tts_config_t& cfg);
// span.cu: page origins of the pages an append opens (f4)
void span_note_append(Ctx* c, int n_req, const int32_t* req_ids, const std::vector<AllocItem>& items);

// kernels (block_table.cu)
cudaError_t launch_init_state(Ctx* c, cudaStream_t s);
cudaError_t launch_alloc(Ctx* c, const AllocItem* items_d, int n_items, cudaStream_t s);
// host item list: passed in the kernel parameter block when it fits (no copy on the stream)
cudaError_t launch_alloc_host(Ctx* c, const AllocItem* items_h, int n_items, cudaStream_t s);
cudaError_t launch_broadcast_prompt(Ctx* c, int req, int n_beams, int npg, cudaStream_t s);
cudaError_t launch_write_prompt(Ctx* c, int req, int prompt_len, const __nv_bfloat16* k,
                                const __nv_bfloat16* v, cudaStream_t s);
cudaError_t launch_cow_copy(Ctx* c, int n_items, cudaStream_t s);
cudaError_t launch_append_write(Ctx* c, const int32_t* slots_d, int n_slots, int n_req,
                                const __nv_bfloat16* k, const __nv_bfloat16* v, cudaStream_t s);
cudaError_t launch_select(Ctx* c, const int32_t* reqs_d, int n_req, const float* scores,
                          int N, int M, int32_t* parent_out, cudaStream_t s);
cudaError_t launch_select_policy(Ctx* c, int n_req, const float* scores, int N, int policy, int param,
                                 int32_t* parent_out, cudaStream_t s);
cudaError_t launch_fork_tables(Ctx* c, const int32_t* reqs_d, int n_req, int n_old, int n_new, cudaStream_t s,
                               const int32_t* new_lens_d = nullptr);
cudaError_t launch_branch_rows(Ctx* c, int req, const int32_t* src_d, const int32_t* dst_d, int n, cudaStream_t s);
cudaError_t launch_zero_tail(Ctx* c, const int32_t* items_d, int n, cudaStream_t s);  // (req, row, pos, ntok)
// lineage copies of tokens [t0, len) (t0 a multiple of P; the buffer holds those tokens only)
cudaError_t launch_lineage_export(Ctx* c, int req, int beam, int len, void* buf, cudaStream_t s, int t0 = 0);
cudaError_t launch_lineage_import(Ctx* c, int req, int beam, int len, const void* buf, cudaStream_t s, int t0 = 0);
cudaError_t launch_share_prefix(Ctx* c, int req, int beam, int share, int m, cudaStream_t s);
cudaError_t launch_select_global(Ctx* c, const float* scores_all, int N, int M, int32_t* parent_out,
                                 cudaStream_t s);
cudaError_t launch_release(Ctx* c, int req, int n_beams, cudaStream_t s);
cudaError_t launch_stats(Ctx* c, const GroupDesc* groups_d, int n_groups, int64_t* accum,
                         int64_t logical, cudaStream_t s);

// attention.cu
cudaError_t launch_attention(Ctx* c, const GroupDesc* groups_d, int n_groups, int group_beams,
                             int layer_begin, int n_layers, int n_call, const __nv_bfloat16* q,
                             float scale, float* out, cudaStream_t s);
bool make_tensor_maps(Ctx* c);
// attention_umma.cu (tcgen05 path: d = 128, 4 <= G <= 16)
bool umma_supported(const Ctx* c);
// per-device kernel attributes (dynamic smem, carveout) and the occupancy the
// persistent schedule relies on (2 CTAs per SM); called by tts_create
cudaError_t umma_prepare(Ctx* c);
int umma_max_beams(const Ctx* c);
// One launch per call: a2 (append of the call's new token, when k_new != null)
// + a3 (plan, built on the fly per CTA) + a4.  groups_h / lens_h are HOST
// arrays (group descriptors; per group-beam post-append lengths, 0 = inactive,
// GroupDesc.pad[0] = offset), sent in the kernel parameter block when they fit.
size_t umma_partial_bytes();
int umma_max_groups();
cudaError_t launch_attention_umma(Ctx* c, const GroupDesc* groups_h, int n_groups, const int32_t* lens_h,
                                  int n_lens, int layer_begin, int n_layers, int n_call,
                                  const __nv_bfloat16* q, float scale, float* out, const __nv_bfloat16* k_new,
                                  const __nv_bfloat16* v_new, cudaStream_t s, bool pair);
// pair mode: groups of up to this many beams, one 2-CTA cluster per tile (0: unavailable)
int umma_pair_max_beams(const Ctx* c);

}  // namespace tts
