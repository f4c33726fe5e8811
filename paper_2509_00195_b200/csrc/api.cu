// C-ABI entry points of libtts (include/tts.h): argument validation, the host
// mirror of beam lengths, launch planning, workspace carving.  Every step of
// the hot path runs in the kernels of block_table.cu / attention.cu.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <new>

#include "tts_internal.cuh"

namespace tts {

static size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

static int64_t max_alloc_items(const tts_config_t& c) {
  return (int64_t)c.max_requests * c.max_beams + c.max_pages_per_beam + c.max_beams;
}

size_t workspace_bytes(const tts_config_t& c) {
  const size_t rows = (size_t)c.max_requests * c.max_beams;
  size_t s = 0;
  s += align_up(rows * c.max_pages_per_beam * 4);  // tmp tables
  s += align_up(rows * 4);                          // tmp lens
  s += align_up(rows * 4);                          // parent
  s += align_up((size_t)max_alloc_items(c) * 4);   // page list
  s += align_up((size_t)max_alloc_items(c) * sizeof(CowCopy));
  s += align_up((size_t)c.num_pages * 4);           // stats marks
  s += align_up(2 * rows * c.max_pages_per_beam * 16);  // attention plan items (double-buffered)
  s += align_up(2 * rows * 4);                          // plan counts
  s += align_up(umma_partial_bytes());                  // split tiles' partial states
  s += align_up((size_t)2 * c.num_layers * c.num_kv_heads * umma_max_groups() * 4);  // split-tile counters
  s += align_up(1024 * 4);                          // global selection: gid-indexed scores
  s += align_up(1024 * 4);                          // global parent map
  s += (size_t)kUploadSlots * kUploadSlotBytes;     // upload mirror
  return s;
}

void* upload(Ctx* c, const void* src, size_t bytes, cudaStream_t st, cudaError_t* err) {
  *err = cudaSuccess;
  if (bytes > kUploadSlotBytes) {
    *err = cudaErrorInvalidValue;
    return nullptr;
  }
  const int slot = c->up_pos;
  c->up_pos = (c->up_pos + 1) % kUploadSlots;
  cudaEventSynchronize(c->ev[slot]);
  uint8_t* h = c->pinned + (size_t)slot * kUploadSlotBytes;
  uint8_t* d = c->ws_upload + (size_t)slot * kUploadSlotBytes;
  std::memcpy(h, src, bytes);
  *err = cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, st);
  if (*err == cudaSuccess) *err = cudaEventRecord(c->ev[slot], st);
  return d;
}

// Two blobs through one pinned slot and one copy (the per-call descriptors of
// the hot path: group list + append slots).
void upload2(Ctx* c, const void* a, size_t na, const void* b, size_t nb, cudaStream_t st, cudaError_t* err,
             void** da, void** db) {
  *err = cudaSuccess;
  const size_t off = (na + 255) / 256 * 256;
  if (off + nb > kUploadSlotBytes) {
    *da = upload(c, a, na, st, err);
    if (*err == cudaSuccess) *db = upload(c, b, nb, st, err);
    return;
  }
  const int slot = c->up_pos;
  c->up_pos = (c->up_pos + 1) % kUploadSlots;
  cudaEventSynchronize(c->ev[slot]);
  uint8_t* h = c->pinned + (size_t)slot * kUploadSlotBytes;
  uint8_t* d = c->ws_upload + (size_t)slot * kUploadSlotBytes;
  std::memcpy(h, a, na);
  std::memcpy(h + off, b, nb);
  *err = cudaMemcpyAsync(d, h, off + nb, cudaMemcpyHostToDevice, st);
  if (*err == cudaSuccess) *err = cudaEventRecord(c->ev[slot], st);
  *da = d;
  *db = d + off;
}

}  // namespace tts

using tts::Ctx;

struct tts_ctx : public Ctx {};

static bool valid_cfg(const tts_config_t* c) {
  if (!c) return false;
  if (c->num_layers <= 0 || c->num_q_heads <= 0 || c->num_kv_heads <= 0) return false;
  if (c->num_q_heads % c->num_kv_heads) return false;
  if (c->page_size != 16) return false;
  if (c->max_requests <= 0 || c->max_beams <= 0 || c->max_beams > 1024) return false;
  if (c->max_pages_per_beam <= 0 || c->num_pages <= 0) return false;
  return true;
}

extern "C" {

const char* tts_status_str(tts_status_t s) {
  switch (s) {
    case TTS_OK: return "ok";
    case TTS_ERR_INVALID_ARG: return "invalid argument";
    case TTS_ERR_UNSUPPORTED: return "unsupported configuration";
    case TTS_ERR_OUT_OF_PAGES: return "page pool exhausted";
    case TTS_ERR_CAPACITY: return "capacity exceeded";
    case TTS_ERR_STATE: return "invalid request state";
    case TTS_ERR_CUDA: return "CUDA error";
    case TTS_ERR_NCCL: return "NCCL error";
  }
  return "unknown";
}

tts_status_t tts_query_buffer_bytes(const tts_config_t* cfg, tts_buffer_sizes_t* s) {
  if (!valid_cfg(cfg) || !s) return TTS_ERR_INVALID_ARG;
  const tts_config_t& c = *cfg;
  const size_t pool = (size_t)c.num_layers * c.num_pages * c.num_kv_heads * c.page_size * c.head_dim * 2;
  s->k_pool = pool;
  s->v_pool = pool;
  s->block_tables = (size_t)c.max_requests * c.max_beams * c.max_pages_per_beam * 4;
  s->seq_lens = (size_t)c.max_requests * c.max_beams * 4;
  s->refcounts = (size_t)c.num_pages * 4;
  s->free_bitmap = (size_t)((c.num_pages + 31) / 32) * 4;
  s->status = 16;
  s->workspace = tts::workspace_bytes(c);
  return TTS_OK;
}

tts_status_t tts_create(const tts_config_t* cfg, const tts_buffers_t* bufs, int device,
                        tts_ctx_t* out) {
  if (!valid_cfg(cfg) || !bufs || !out) return TTS_ERR_INVALID_ARG;
  if (cfg->head_dim != 64 && cfg->head_dim != 128) return TTS_ERR_UNSUPPORTED;
  if (cfg->num_q_heads / cfg->num_kv_heads > 16) return TTS_ERR_UNSUPPORTED;
  const int64_t rows = (int64_t)cfg->num_layers * cfg->num_pages * cfg->num_kv_heads * cfg->page_size;
  if (rows >= (1ll << 31)) return TTS_ERR_CAPACITY;
  if (bufs->workspace_bytes < tts::workspace_bytes(*cfg)) return TTS_ERR_INVALID_ARG;
  if (!bufs->k_pool || !bufs->v_pool || !bufs->block_tables || !bufs->seq_lens ||
      !bufs->refcounts || !bufs->free_bitmap || !bufs->status || !bufs->workspace)
    return TTS_ERR_INVALID_ARG;
  TTS_CUDA(cudaSetDevice(device));
  tts_ctx* c = new (std::nothrow) tts_ctx();
  if (!c) return TTS_ERR_CAPACITY;
  c->cfg = *cfg;
  c->buf = *bufs;
  c->device = device;
  cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
  c->n_beams.assign(cfg->max_requests, 0);
  c->n_rows.assign(cfg->max_requests, 0);
  c->lens.assign((size_t)cfg->max_requests * cfg->max_beams, 0);
  // carve workspace
  uint8_t* w = (uint8_t*)bufs->workspace;
  const size_t rws = (size_t)cfg->max_requests * cfg->max_beams;
  c->ws_tmp_tables = (int32_t*)w;
  w += tts::align_up(rws * cfg->max_pages_per_beam * 4);
  c->ws_tmp_lens = (int32_t*)w;
  w += tts::align_up(rws * 4);
  c->ws_parent = (int32_t*)w;
  w += tts::align_up(rws * 4);
  c->max_alloc = tts::max_alloc_items(*cfg);
  c->ws_pages = (int32_t*)w;
  w += tts::align_up((size_t)c->max_alloc * 4);
  c->ws_cow = (tts::CowCopy*)w;
  w += tts::align_up((size_t)c->max_alloc * sizeof(tts::CowCopy));
  c->ws_mark = (int32_t*)w;
  w += tts::align_up((size_t)cfg->num_pages * 4);
  c->ws_items = (int4*)w;
  w += tts::align_up(2 * rws * cfg->max_pages_per_beam * 16);
  c->ws_counts = (int32_t*)w;
  w += tts::align_up(2 * rws * 4);
  c->ws_partial = (float*)w;
  w += tts::align_up(tts::umma_partial_bytes());
  c->ws_tile_cnt = (int32_t*)w;
  // (x2: pair mode counts the pieces of each rank's rows separately)
  const size_t cnt_bytes = (size_t)2 * cfg->num_layers * cfg->num_kv_heads * tts::umma_max_groups() * 4;
  w += tts::align_up(cnt_bytes);
  c->ws_scores_all = (float*)w;
  w += tts::align_up(1024 * 4);
  c->ws_parent_all = (int32_t*)w;
  w += tts::align_up(1024 * 4);
  c->ws_upload = w;
  if (cudaMallocHost(&c->pinned, (size_t)tts::kUploadSlots * tts::kUploadSlotBytes) != cudaSuccess) {
    delete c;
    return TTS_ERR_CUDA;
  }
  for (int i = 0; i < tts::kUploadSlots; ++i) cudaEventCreateWithFlags(&c->ev[i], cudaEventDisableTiming);
  c->tile_cnt_bytes = cnt_bytes;
  if (const char* s = std::getenv("TTS_ATTN")) c->env_attn_mma = std::strcmp(s, "mma") == 0;
  if (const char* s = std::getenv("TTS_GROUP_BEAMS")) c->env_group_beams = std::max(0, std::atoi(s));
  if (const char* s = std::getenv("TTS_NCONS")) c->env_ncons = std::max(0, std::atoi(s));
  if (const char* s = std::getenv("TTS_POLY")) c->env_poly = std::max(0, std::min(2, std::atoi(s)));
  c->env_no_pdl = std::getenv("TTS_NO_PDL") != nullptr;
  if (const char* s = std::getenv("TTS_ROUND_ROBIN")) c->env_round_robin = std::atoi(s) != 0;
  if (const char* s = std::getenv("TTS_SPLIT_PARTIAL")) c->env_split_partial = std::atoi(s) != 0;
  if (const char* s = std::getenv("TTS_SCHED")) c->env_sched = std::atoi(s);
  if (const char* s = std::getenv("TTS_PAIR")) c->env_pair = std::atoi(s);
  if (const char* s = std::getenv("TTS_L2HINT")) c->env_l2hint = std::atoi(s);
  if (!tts::make_tensor_maps(c)) {
    tts_destroy(c);
    return TTS_ERR_CUDA;
  }
  if (tts::umma_prepare(c) != cudaSuccess) {
    tts_destroy(c);
    return TTS_ERR_CUDA;
  }
  if (cudaMemsetAsync(c->ws_tile_cnt, 0, cnt_bytes, 0) != cudaSuccess ||
      tts::launch_init_state(c, 0) != cudaSuccess || cudaStreamSynchronize(0) != cudaSuccess) {
    tts_destroy(c);
    return TTS_ERR_CUDA;
  }
  *out = c;
  return TTS_OK;
}

tts_status_t tts_destroy(tts_ctx_t c) {
  if (!c) return TTS_ERR_INVALID_ARG;
  cudaSetDevice(c->device);
  tts_comm_destroy(c);
  for (int i = 0; i < tts::kUploadSlots; ++i)
    if (c->ev[i]) cudaEventDestroy(c->ev[i]);
  for (auto& e : c->prof_ev)
    if (e) cudaEventDestroy(e);
  if (c->pinned) cudaFreeHost(c->pinned);
  delete c;
  return TTS_OK;
}

int64_t tts_launch_count(tts_ctx_t c) { return c ? c->launches : -1; }

const char* tts_attention_kernel(tts_ctx_t c) {
  if (!c) return "";
  if (tts::umma_supported(c) && !c->env_attn_mma) return "k_tree_umma";
  return "k_tree_attn";
}

tts_status_t tts_device_status(tts_ctx_t c, void* stream, tts_status_t* out) {
  if (!c || !out) return TTS_ERR_INVALID_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  int32_t v = 0;
  TTS_CUDA(cudaMemcpyAsync(&v, c->buf.status, 4, cudaMemcpyDeviceToHost, st));
  TTS_CUDA(cudaMemsetAsync(c->buf.status, 0, 16, st));
  // split-tile merge counters back to zero: every kernel after a sticky error
  // skipped its work, whatever counts a partial launch left behind
  TTS_CUDA(cudaMemsetAsync(c->ws_tile_cnt, 0, c->tile_cnt_bytes, st));
  TTS_CUDA(cudaStreamSynchronize(st));
  *out = (tts_status_t)v;
  return TTS_OK;
}

static bool installed(tts_ctx_t c, int32_t req) {
  return req >= 0 && req < c->cfg.max_requests && c->n_beams[req] > 0;
}

static int64_t entry_of(const tts_config_t& g, int req, int beam, int pos) {
  return ((int64_t)req * g.max_beams + beam) * g.max_pages_per_beam + pos;
}

tts_status_t tts_block_table_init_request(tts_ctx_t c, int32_t req, int32_t n_beams,
                                          int32_t prompt_len, const void* k_prompt,
                                          const void* v_prompt, void* stream) {
  if (!c) return TTS_ERR_INVALID_ARG;
  const tts_config_t& g = c->cfg;
  if (req < 0 || req >= g.max_requests) return TTS_ERR_CAPACITY;
  if (c->n_beams[req] > 0) return TTS_ERR_STATE;
  if (n_beams <= 0 || n_beams > g.max_beams || prompt_len < 0) return TTS_ERR_INVALID_ARG;
  if (prompt_len > 0 && (!k_prompt || !v_prompt)) return TTS_ERR_INVALID_ARG;
  const int P = g.page_size;
  const int npg = (prompt_len + P - 1) / P;
  if (npg > g.max_pages_per_beam) return TTS_ERR_CAPACITY;
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e;
  std::vector<tts::AllocItem> items;
  for (int i = 0; i < npg; ++i) items.push_back({entry_of(g, req, 0, i), 0, 0});
  if (!items.empty()) {
    TTS_CUDA(tts::launch_alloc_host(c, items.data(), (int)items.size(), st));
    TTS_CUDA(tts::launch_broadcast_prompt(c, req, n_beams, npg, st));
    TTS_CUDA(tts::launch_write_prompt(c, req, prompt_len, (const __nv_bfloat16*)k_prompt,
                                      (const __nv_bfloat16*)v_prompt, st));
  }
  const int rem = prompt_len % P;
  if (rem && n_beams > 1) {
    items.clear();
    for (int b = 1; b < n_beams; ++b) items.push_back({entry_of(g, req, b, npg - 1), 1, rem});
    TTS_CUDA(tts::launch_alloc_host(c, items.data(), (int)items.size(), st));
    TTS_CUDA(tts::launch_cow_copy(c, (int)items.size(), st));
  }
  std::vector<int32_t> lens(g.max_beams, 0);
  for (int b = 0; b < n_beams; ++b) lens[b] = prompt_len;
  void* d = tts::upload(c, lens.data(), lens.size() * 4, st, &e);
  TTS_CUDA(e);
  TTS_CUDA(cudaMemcpyAsync(c->buf.seq_lens + (int64_t)req * g.max_beams, d, lens.size() * 4,
                           cudaMemcpyDeviceToDevice, st));
  c->n_beams[req] = n_beams;
  c->n_rows[req] = n_beams;
  std::copy(lens.begin(), lens.end(), c->lens.begin() + (int64_t)req * g.max_beams);
  return TTS_OK;
}

// a2, host half: validates the call and lists the allocations (beams whose
// next token opens a page) and the append slots (call index, request, beam,
// position).  No side effect: nothing is enqueued and the host length mirror
// is untouched, so a rejected call leaves the context as it was.
struct AppendPlan {
  std::vector<tts::AllocItem> items;
  std::vector<int32_t> slots;  // (i, req, beam, pos) quadruples
};

static tts_status_t append_plan(tts_ctx_t c, int32_t n_req, const int32_t* req_ids, const uint8_t* active,
                                const void* k_new, const void* v_new, AppendPlan& ap) {
  if (!c || n_req <= 0 || !req_ids || !k_new || !v_new) return TTS_ERR_INVALID_ARG;
  const tts_config_t& g = c->cfg;
  const int P = g.page_size;
  std::vector<char> seen((size_t)g.max_requests, 0);
  for (int i = 0; i < n_req; ++i) {
    const int r = req_ids[i];
    if (!installed(c, r)) return TTS_ERR_STATE;
    if (seen[r]) return TTS_ERR_INVALID_ARG;  // a request twice in one call
    seen[r] = 1;
  }
  ap.items.clear();
  ap.slots.clear();
  for (int i = 0; i < n_req; ++i) {
    const int r = req_ids[i];
    for (int b = 0; b < c->n_beams[r]; ++b) {
      if (active && !active[(int64_t)i * g.max_beams + b]) continue;
      const int pos = c->lens[(int64_t)r * g.max_beams + b];
      if (pos / P >= g.max_pages_per_beam) return TTS_ERR_CAPACITY;
      if (pos % P == 0) ap.items.push_back({entry_of(g, r, b, pos / P), 0, 0});
      ap.slots.insert(ap.slots.end(), {i, r, b, pos});
    }
  }
  return TTS_OK;
}

// Advances (+1) or rolls back (-1) the host length mirror over the plan's slots.
static void mirror_advance(tts_ctx_t c, const AppendPlan& ap, int delta) {
  for (size_t k = 0; k < ap.slots.size(); k += 4)
    c->lens[(int64_t)ap.slots[k + 1] * c->cfg.max_beams + ap.slots[k + 2]] += delta;
}

tts_status_t tts_block_table_append(tts_ctx_t c, int32_t n_req, const int32_t* req_ids,
                                    const uint8_t* active, const void* k_new, const void* v_new,
                                    void* stream) {
  AppendPlan ap;
  tts_status_t s = append_plan(c, n_req, req_ids, active, k_new, v_new, ap);
  if (s != TTS_OK) return s;
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e;
  tts::span_note_append(c, n_req, req_ids, ap.items);
  if (!ap.items.empty()) TTS_CUDA(tts::launch_alloc_host(c, ap.items.data(), (int)ap.items.size(), st));
  if (!ap.slots.empty()) {
    void* d = tts::upload(c, ap.slots.data(), ap.slots.size() * 4, st, &e);
    TTS_CUDA(e);
    TTS_CUDA(tts::launch_append_write(c, (const int32_t*)d, (int)ap.slots.size() / 4, n_req,
                                      (const __nv_bfloat16*)k_new, (const __nv_bfloat16*)v_new, st));
  }
  mirror_advance(c, ap, +1);
  return TTS_OK;
}

static void prof_pair(tts_ctx_t c, cudaEvent_t* e0, cudaEvent_t* e1);

// Group plan: contiguous beam runs of `gb` slots with >= 1 active beam.
// lens_out (optional): every group beam's current length (0 = inactive), the
// group's first at GroupDesc.pad[0].
static void plan_groups(tts_ctx_t c, int n_req, const int32_t* req_ids, const uint8_t* active,
                        int gb, std::vector<tts::GroupDesc>& out, std::vector<int32_t>* lens_out = nullptr) {
  const tts_config_t& g = c->cfg;
  const int P = g.page_size;
  out.clear();
  if (lens_out) lens_out->clear();
  for (int i = 0; i < n_req; ++i) {
    const int r = req_ids[i];
    const int N = c->n_beams[r];
    for (int b0 = 0; b0 < N; b0 += gb) {
      tts::GroupDesc d{};
      d.call_idx = i;
      d.req = r;
      d.beam0 = b0;
      d.nbeams = std::min(gb, N - b0);
      d.active = 0;
      d.max_npages = 0;
      for (int k = 0; k < d.nbeams; ++k) {
        if (active && !active[(int64_t)i * g.max_beams + b0 + k]) continue;
        d.active |= 1u << k;
        const int len = c->lens[(int64_t)r * g.max_beams + b0 + k];
        d.max_npages = std::max(d.max_npages, (len + P - 1) / P);
      }
      if (!d.active) continue;
      if (lens_out) {
        d.pad[0] = (int32_t)lens_out->size();
        for (int k = 0; k < d.nbeams; ++k)
          lens_out->push_back(((d.active >> k) & 1u) ? c->lens[(int64_t)r * g.max_beams + b0 + k] : 0);
      }
      out.push_back(d);
    }
  }
}

// a3/a4, host half: validates the call and plans the beam groups from the
// host length mirror.  No side effect.
struct AttnPlan {
  bool umma = false;
  bool pair = false;    // tcgen05 path: 2-CTA clusters (groups of up to umma_pair_max_beams beams)
  int group_beams = 0;  // mma.sync path: beams per CTA group
  std::vector<tts::GroupDesc> groups;
  std::vector<int32_t> glens;  // tcgen05 path: per group beam, current length (0 = inactive)
};

static tts_status_t attn_prepare(tts_ctx_t c, int32_t layer_begin, int32_t layer_end, int32_t n_req,
                                 const int32_t* req_ids, const uint8_t* active, AttnPlan& ap) {
  if (!c || !req_ids || n_req <= 0) return TTS_ERR_INVALID_ARG;
  const tts_config_t& g = c->cfg;
  if (layer_begin < 0 || layer_end > g.num_layers || layer_begin >= layer_end) return TTS_ERR_INVALID_ARG;
  std::vector<char> seen((size_t)g.max_requests, 0);
  for (int i = 0; i < n_req; ++i) {
    if (!installed(c, req_ids[i])) return TTS_ERR_STATE;
    if (seen[req_ids[i]]) return TTS_ERR_INVALID_ARG;
    seen[req_ids[i]] = 1;
  }
  const int G = g.num_q_heads / g.num_kv_heads;
  const int n_layers = layer_end - layer_begin;
  ap.umma = tts::umma_supported(c) && !c->env_attn_mma;
  if (ap.umma) {
    // 128-row tiles: balanced runs of <= umma_max_beams beams of one request.
    // The largest groups (a page shared inside a group is staged once) that
    // still give >= 3/4 of a round of tiles for the one CTA per SM of the
    // persistent kernel; a smaller remainder is split over all CTAs there
    // (stream-K).  Measured (C2, one request per call): 4-beam groups, 224
    // whole tiles, 40 us per call vs 16-beam groups, 56 tiles split ~5 ways,
    // 59 us (the split pieces cost unequal time: the shared prefix at the head
    // of a tile keeps all four softmax warps busy, a private tail one).
    int maxb = tts::umma_max_beams(c);
    // pair mode when every request of the call has more beams than one CTA's
    // tile holds: a group of up to twice as many beams per 2-CTA cluster, so
    // that the pages the two halves share are loaded once (TMA multicast)
    const int pmax = c->env_pair ? tts::umma_pair_max_beams(c) : 0;
    ap.pair = pmax > maxb && !c->env_group_beams;
    for (int i = 0; ap.pair && i < n_req; ++i) ap.pair = c->n_beams[req_ids[i]] > maxb;
    if (ap.pair) maxb = pmax;
    if (c->env_group_beams) maxb = std::max(1, std::min(maxb, c->env_group_beams));
    const int64_t want = (3ll * (ap.pair ? c->num_sms / 2 : c->num_sms) + 3) / 4;
    auto group_size = [&](int cap) {
      int gb = 1;
      for (int i = 0; i < n_req; ++i) {
        const int N = c->n_beams[req_ids[i]];
        const int ng = (N + cap - 1) / cap;
        gb = std::max(gb, (N + ng - 1) / ng);
      }
      return gb;
    };
    int gb = group_size(maxb);
    plan_groups(c, n_req, req_ids, active, gb, ap.groups);
    if (!c->env_group_beams) {
      while (gb > 1 && (int64_t)ap.groups.size() * g.num_kv_heads * n_layers < want) {
        gb = group_size((gb + 1) / 2);
        plan_groups(c, n_req, req_ids, active, gb, ap.groups);
      }
    }
    plan_groups(c, n_req, req_ids, active, gb, ap.groups, &ap.glens);
    if ((int)ap.groups.size() > tts::umma_max_groups()) return TTS_ERR_CAPACITY;
    return TTS_OK;
  }
  const int bpt = 16 / G;
  for (int ncons : {8, 4, 2, 1}) {
    if (ncons * bpt > 32) continue;
    if (c->env_ncons && ncons != c->env_ncons) continue;
    plan_groups(c, n_req, req_ids, active, ncons * bpt, ap.groups);
    ap.group_beams = ncons * bpt;
    const int64_t ctas = (int64_t)ap.groups.size() * g.num_kv_heads * n_layers;
    if (c->env_ncons || ctas >= 2ll * c->num_sms) break;
  }
  if (!ap.group_beams) return TTS_ERR_UNSUPPORTED;
  return TTS_OK;
}

// Launches the attention of a prepared call; `pending` (tts_decode_step)
// carries append slots whose K/V write has not been launched yet: fused with
// the plan on the tcgen05 path, launched just before the attention kernel
// otherwise.
static tts_status_t attn_launch(tts_ctx_t c, const AttnPlan& ap, int32_t layer_begin, int32_t layer_end,
                                int32_t n_req, const void* q, float scale, float* out, void* stream,
                                const std::vector<int32_t>* pending = nullptr, const void* k_new = nullptr,
                                const void* v_new = nullptr) {
  const int n_layers = layer_end - layer_begin;
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e;
  if (ap.umma) {
    if (ap.groups.empty()) return TTS_OK;
    const bool append = pending && !pending->empty();
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (c->profiling) prof_pair(c, &e0, &e1);
    if (e0) TTS_CUDA(cudaEventRecord(e0, st));
    TTS_CUDA(tts::launch_attention_umma(c, ap.groups.data(), (int)ap.groups.size(), ap.glens.data(),
                                        (int)ap.glens.size(), layer_begin, n_layers, n_req,
                                        (const __nv_bfloat16*)q, scale, out,
                                        append ? (const __nv_bfloat16*)k_new : nullptr,
                                        append ? (const __nv_bfloat16*)v_new : nullptr, st, ap.pair));
    if (e1) TTS_CUDA(cudaEventRecord(e1, st));
    return TTS_OK;
  }
  if (pending && !pending->empty()) {
    void* ds = tts::upload(c, pending->data(), pending->size() * 4, st, &e);
    TTS_CUDA(e);
    TTS_CUDA(tts::launch_append_write(c, (const int32_t*)ds, (int)pending->size() / 4, n_req,
                                      (const __nv_bfloat16*)k_new, (const __nv_bfloat16*)v_new, st));
  }
  if (ap.groups.empty()) return TTS_OK;
  void* d = tts::upload(c, ap.groups.data(), ap.groups.size() * sizeof(tts::GroupDesc), st, &e);
  TTS_CUDA(e);
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (c->profiling) prof_pair(c, &e0, &e1);
  if (e0) TTS_CUDA(cudaEventRecord(e0, st));
  TTS_CUDA(tts::launch_attention(c, (const tts::GroupDesc*)d, (int)ap.groups.size(), ap.group_beams,
                                 layer_begin, n_layers, n_req, (const __nv_bfloat16*)q, scale, out, st));
  if (e1) TTS_CUDA(cudaEventRecord(e1, st));
  return TTS_OK;
}

tts_status_t tts_prefix_attn_decode(tts_ctx_t c, int32_t layer_begin, int32_t layer_end,
                                    int32_t n_req, const int32_t* req_ids, const uint8_t* active,
                                    const void* q, float scale, float* out, void* stream) {
  if (!c || !q || !out) return TTS_ERR_INVALID_ARG;
  AttnPlan ap;
  tts_status_t s = attn_prepare(c, layer_begin, layer_end, n_req, req_ids, active, ap);
  if (s != TTS_OK) return s;
  return attn_launch(c, ap, layer_begin, layer_end, n_req, q, scale, out, stream);
}

tts_status_t tts_decode_step(tts_ctx_t c, int32_t n_req, const int32_t* req_ids,
                             const uint8_t* active, const void* k_new, const void* v_new,
                             const void* q, float scale, float* out, void* stream) {
  if (!c || !q || !out) return TTS_ERR_INVALID_ARG;
  // every host-detectable error before any side effect: the append plan, then
  // the attention plan on the post-append lengths (mirror advanced, rolled
  // back if the attention plan rejects the call)
  AppendPlan app;
  tts_status_t s = append_plan(c, n_req, req_ids, active, k_new, v_new, app);
  if (s != TTS_OK) return s;
  mirror_advance(c, app, +1);
  AttnPlan ap;
  s = attn_prepare(c, 0, c->cfg.num_layers, n_req, req_ids, active, ap);
  if (s != TTS_OK) {
    mirror_advance(c, app, -1);
    return s;
  }
  cudaStream_t st = (cudaStream_t)stream;
  tts::span_note_append(c, n_req, req_ids, app.items);
  if (!app.items.empty()) TTS_CUDA(tts::launch_alloc_host(c, app.items.data(), (int)app.items.size(), st));
  return attn_launch(c, ap, 0, c->cfg.num_layers, n_req, q, scale, out, stream, &app.slots, k_new, v_new);
}

static constexpr int kProfPairs = 4096;

static void prof_drain(tts_ctx_t c, int pair) {
  cudaEvent_t a = c->prof_ev[2 * pair], b = c->prof_ev[2 * pair + 1];
  if (cudaEventSynchronize(b) == cudaSuccess) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, a, b) == cudaSuccess) c->prof_ms += ms;
  }
}

static void prof_pair(tts_ctx_t c, cudaEvent_t* e0, cudaEvent_t* e1) {
  const int i = c->prof_pos;
  if (c->prof_count >= kProfPairs) prof_drain(c, i);  // pair i is being reused
  *e0 = c->prof_ev[2 * i];
  *e1 = c->prof_ev[2 * i + 1];
  c->prof_pos = (i + 1) % kProfPairs;
  c->prof_count++;
}

tts_status_t tts_profile_begin(tts_ctx_t c) {
  if (!c) return TTS_ERR_INVALID_ARG;
  if (c->prof_ev.empty()) {
    c->prof_ev.resize(2 * kProfPairs);
    for (auto& e : c->prof_ev) TTS_CUDA(cudaEventCreate(&e));
  }
  c->profiling = true;
  c->prof_pos = 0;
  c->prof_count = 0;
  c->prof_ms = 0.0;
  return TTS_OK;
}

tts_status_t tts_profile_end(tts_ctx_t c, double* ms, int64_t* n) {
  if (!c || !c->profiling) return TTS_ERR_STATE;
  const int64_t live = c->prof_count < kProfPairs ? c->prof_count : kProfPairs;
  for (int64_t k = 0; k < live; ++k) {
    const int i = (int)((c->prof_pos - live + k + kProfPairs) % kProfPairs);
    prof_drain(c, i);
  }
  c->profiling = false;
  if (ms) *ms = c->prof_ms;
  if (n) *n = c->prof_count;
  return TTS_OK;
}

static tts_status_t select_fork_impl(tts_ctx_t c, int32_t n_req, const int32_t* req_ids, const float* scores,
                                     int32_t policy, int32_t param, int32_t* parent_out, void* stream) {
  if (!c || n_req <= 0 || !req_ids || !scores) return TTS_ERR_INVALID_ARG;
  const tts_config_t& g = c->cfg;
  for (int i = 0; i < n_req; ++i)
    if (!installed(c, req_ids[i])) return TTS_ERR_STATE;
  const int N = c->n_beams[req_ids[0]];
  for (int i = 0; i < n_req; ++i)
    if (c->n_beams[req_ids[i]] != N) return TTS_ERR_INVALID_ARG;
  if (policy < TTS_SELECT_TOPK || policy > TTS_SELECT_DYNAMIC) return TTS_ERR_INVALID_ARG;
  if (param <= 0 || N % param) return TTS_ERR_INVALID_ARG;  // N % M (top-K, dynamic), N % B (diverse)
  for (int i = 0; i < n_req; ++i)
    for (int j = 0; j < i; ++j)
      if (req_ids[i] == req_ids[j]) return TTS_ERR_INVALID_ARG;
  for (int i = 0; i < n_req; ++i)
    if (c->n_rows[req_ids[i]] != N) return TTS_ERR_STATE;  // imported lineages pending: use tts_beam_fork_map
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e;
  void* dreq = tts::upload(c, req_ids, (size_t)n_req * 4, st, &e);
  TTS_CUDA(e);
  if (policy == TTS_SELECT_TOPK)
    TTS_CUDA(tts::launch_select(c, (const int32_t*)dreq, n_req, scores, N, param, parent_out, st));
  else
    TTS_CUDA(tts::launch_select_policy(c, n_req, scores, N, policy, param, parent_out, st));
  TTS_CUDA(tts::launch_fork_tables(c, (const int32_t*)dreq, n_req, N, N, st));
  // parent map back to the host (for the length mirror and the CoW plan)
  std::vector<int32_t> parent((size_t)n_req * g.max_beams);
  TTS_CUDA(cudaMemcpyAsync(parent.data(), c->ws_parent, parent.size() * 4, cudaMemcpyDeviceToHost, st));
  TTS_CUDA(cudaStreamSynchronize(st));
  const int P = g.page_size;
  std::vector<tts::AllocItem> items;
  for (int i = 0; i < n_req; ++i) {
    const int r = req_ids[i];
    const int32_t* par = parent.data() + (int64_t)i * g.max_beams;
    int32_t* lens = c->lens.data() + (int64_t)r * g.max_beams;
    std::vector<int32_t> old(lens, lens + N);
    for (int cc = 0; cc < N; ++cc) {
      if (par[cc] < 0 || par[cc] >= N) return TTS_ERR_STATE;  // sticky device error upstream
      lens[cc] = old[par[cc]];
    }
    // eager CoW (ledger C6): every child but the first of its parent (children
    // of a parent are contiguous) copies a partially filled last page
    for (int cc = 1; cc < N; ++cc) {
      const int len = lens[cc];
      if (par[cc] == par[cc - 1] && len % P) items.push_back({entry_of(g, r, cc, (len - 1) / P), 1, len % P});
    }
  }
  if (!items.empty()) {
    TTS_CUDA(tts::launch_alloc_host(c, items.data(), (int)items.size(), st));
    TTS_CUDA(tts::launch_cow_copy(c, (int)items.size(), st));
  }
  return TTS_OK;
}

tts_status_t tts_beam_select_fork(tts_ctx_t c, int32_t n_req, const int32_t* req_ids, const float* scores,
                                  int32_t M, int32_t* parent_out, void* stream) {
  return select_fork_impl(c, n_req, req_ids, scores, TTS_SELECT_TOPK, M, parent_out, stream);
}

tts_status_t tts_beam_select_fork_policy(tts_ctx_t c, int32_t n_req, const int32_t* req_ids, const float* scores,
                                         int32_t policy, int32_t param, int32_t* parent_out, void* stream) {
  return select_fork_impl(c, n_req, req_ids, scores, policy, param, parent_out, stream);
}

// CoW plan of a fork by parent map: the first child (in index order) of each
// parent keeps its partially filled last page, every later child copies it
// (ledger C6; for tts_beam_select_fork this is child j = c mod M == 0).
static void cow_items_for(tts_ctx_t c, int req, int n_new, const int32_t* parent, std::vector<tts::AllocItem>& items) {
  const tts_config_t& g = c->cfg;
  const int P = g.page_size;
  std::vector<char> seen((size_t)g.max_beams, 0);
  for (int cc = 0; cc < n_new; ++cc) {
    const int par = parent[cc];
    const int len = c->lens[(int64_t)req * g.max_beams + cc];
    if (seen[par] && len % P) items.push_back({entry_of(g, req, cc, (len - 1) / P), 1, len % P});
    seen[par] = 1;
  }
}

static tts_status_t fork_map_impl(tts_ctx_t c, int32_t req, int32_t n_new, const int32_t* parent_h,
                                  const int32_t* new_len_h, void* stream) {
  if (!c || !parent_h || n_new <= 0) return TTS_ERR_INVALID_ARG;
  if (!installed(c, req)) return TTS_ERR_STATE;
  const tts_config_t& g = c->cfg;
  const int P = g.page_size;
  const int n_old = c->n_rows[req];
  if (n_new > g.max_beams) return TTS_ERR_CAPACITY;
  const int32_t* lens_old = c->lens.data() + (int64_t)req * g.max_beams;
  for (int i = 0; i < n_new; ++i) {
    if (parent_h[i] < 0 || parent_h[i] >= n_old || lens_old[parent_h[i]] <= 0) return TTS_ERR_INVALID_ARG;
    if (new_len_h && (new_len_h[i] < 1 || new_len_h[i] > lens_old[parent_h[i]])) return TTS_ERR_INVALID_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e;
  int32_t reqv = req;
  void* dreq = tts::upload(c, &reqv, 4, st, &e);
  TTS_CUDA(e);
  void* dlen = nullptr;
  if (new_len_h) {
    dlen = tts::upload(c, new_len_h, (size_t)n_new * 4, st, &e);
    TTS_CUDA(e);
  }
  TTS_CUDA(cudaMemcpyAsync(c->ws_parent, parent_h, (size_t)n_new * 4, cudaMemcpyHostToDevice, st));
  TTS_CUDA(tts::launch_fork_tables(c, (const int32_t*)dreq, 1, n_old, n_new, st, (const int32_t*)dlen));
  int32_t* lens = c->lens.data() + (int64_t)req * g.max_beams;
  std::vector<int32_t> old(lens, lens + g.max_beams);
  for (int cc = 0; cc < g.max_beams; ++cc) lens[cc] = cc < n_new ? (new_len_h ? new_len_h[cc] : old[parent_h[cc]]) : 0;
  std::vector<tts::AllocItem> items;
  cow_items_for(c, req, n_new, parent_h, items);
  if (!items.empty()) {
    TTS_CUDA(tts::launch_alloc_host(c, items.data(), (int)items.size(), st));
    TTS_CUDA(tts::launch_cow_copy(c, (int)items.size(), st));
  }
  // a truncated row's kept (first-child) partial last page: clear its slots
  // past the new length (every token slot of a page past a row's length is 0)
  if (new_len_h) {
    std::vector<int32_t> zt;
    std::vector<char> seen((size_t)g.max_beams, 0);
    for (int cc = 0; cc < n_new; ++cc) {
      const int par = parent_h[cc], len = new_len_h[cc];
      if (!seen[par] && len < old[par] && len % P) zt.insert(zt.end(), {req, cc, (len - 1) / P, len % P});
      seen[par] = 1;
    }
    if (!zt.empty()) {
      void* dz = tts::upload(c, zt.data(), zt.size() * 4, st, &e);
      TTS_CUDA(e);
      TTS_CUDA(tts::launch_zero_tail(c, (const int32_t*)dz, (int)zt.size() / 4, st));
    }
  }
  c->n_beams[req] = n_new;
  c->n_rows[req] = n_new;
  TTS_CUDA(cudaStreamSynchronize(st));  // parent_h is a borrowed host buffer
  return TTS_OK;
}

tts_status_t tts_beam_fork_map(tts_ctx_t c, int32_t req, int32_t n_new, const int32_t* parent_h, void* stream) {
  return fork_map_impl(c, req, n_new, parent_h, nullptr, stream);
}

tts_status_t tts_beam_fork_map_trunc(tts_ctx_t c, int32_t req, int32_t n_new, const int32_t* parent_h,
                                     const int32_t* new_len_h, void* stream) {
  if (!new_len_h) return TTS_ERR_INVALID_ARG;
  return fork_map_impl(c, req, n_new, parent_h, new_len_h, stream);
}

tts_status_t tts_spec_branch(tts_ctx_t c, int32_t req, int32_t n, const int32_t* src_rows_h, void* stream) {
  if (!c || n <= 0 || !src_rows_h) return TTS_ERR_INVALID_ARG;
  if (!installed(c, req)) return TTS_ERR_STATE;
  const tts_config_t& g = c->cfg;
  const int P = g.page_size;
  const int n_old = c->n_rows[req];
  if (n_old + n > g.max_beams) return TTS_ERR_CAPACITY;
  int32_t* lens = c->lens.data() + (int64_t)req * g.max_beams;
  for (int i = 0; i < n; ++i)
    if (src_rows_h[i] < 0 || src_rows_h[i] >= n_old || lens[src_rows_h[i]] <= 0) return TTS_ERR_INVALID_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e;
  std::vector<int32_t> blob(2 * (size_t)n);
  std::vector<tts::AllocItem> items;
  for (int i = 0; i < n; ++i) {
    const int src = src_rows_h[i], dst = n_old + i, len = lens[src];
    blob[i] = src;
    blob[n + i] = dst;
    if (len % P) items.push_back({entry_of(g, req, dst, (len - 1) / P), 1, len % P});
  }
  int32_t* d = (int32_t*)tts::upload(c, blob.data(), blob.size() * 4, st, &e);
  TTS_CUDA(e);
  TTS_CUDA(tts::launch_branch_rows(c, req, d, d + n, n, st));
  if (!items.empty()) {
    TTS_CUDA(tts::launch_alloc_host(c, items.data(), (int)items.size(), st));
    TTS_CUDA(tts::launch_cow_copy(c, (int)items.size(), st));
  }
  for (int i = 0; i < n; ++i) lens[n_old + i] = lens[src_rows_h[i]];
  c->n_rows[req] = n_old + n;
  c->n_beams[req] = n_old + n;
  return TTS_OK;
}

tts_status_t tts_spec_select(int32_t n, const int32_t* beam_h, const float* last_score_h, const int32_t* have_h,
                             int32_t free_slots, int32_t B, int32_t* add_h) {
  if (n < 0 || B <= 0 || (n > 0 && (!beam_h || !last_score_h || !have_h || !add_h))) return TTS_ERR_INVALID_ARG;
  std::vector<int> order(n), pot(n);
  for (int i = 0; i < n; ++i) {
    // bin j of the previous score over B equal-width bins of [0, 1], the
    // highest first, a boundary score in the higher bin; potential M = B - j + 1
    double s = (double)last_score_h[i];
    if (std::isnan(s)) s = 0.0;
    s = std::min(1.0, std::max(0.0, s));
    int j = (int)std::ceil((1.0 - s) * (double)B);
    j = std::min(B, std::max(1, j));
    pot[i] = B - j + 1;
    order[i] = i;
    add_h[i] = 0;
  }
  std::sort(order.begin(), order.end(), [&](int a, int b) {
    return pot[a] != pot[b] ? pot[a] > pot[b] : beam_h[a] < beam_h[b];
  });
  int free = free_slots;
  for (int i : order) {
    if (free <= 0) break;
    const int k = std::min(pot[i] - have_h[i], free);
    if (k > 0) {
      add_h[i] = k;
      free -= k;
    }
  }
  return TTS_OK;
}

tts_status_t tts_spec_plan(int32_t N, int32_t M, const int32_t* parent_h, int32_t n_branch,
                           const int32_t* branch_src_h, const int32_t* branch_tokens_h, const int32_t* lens_h,
                           const double* frac_h, const int32_t* next_len_h, int32_t* parent_rows_h,
                           int32_t* new_len_h, int32_t* head_h) {
  if (N <= 0 || M <= 0 || N % M || !parent_h || !lens_h || !frac_h || !parent_rows_h || !new_len_h || !head_h)
    return TTS_ERR_INVALID_ARG;
  if (n_branch < 0 || (n_branch > 0 && (!branch_src_h || !branch_tokens_h))) return TTS_ERR_INVALID_ARG;
  std::vector<std::vector<int>> rows_of(N);
  for (int i = 0; i < n_branch; ++i) {
    if (branch_src_h[i] < 0 || branch_src_h[i] >= N) return TTS_ERR_INVALID_ARG;
    rows_of[branch_src_h[i]].push_back(N + i);
  }
  for (int c = 0; c < N; ++c) {
    const int s = parent_h[c], j = c % M;
    if (s < 0 || s >= N) return TTS_ERR_INVALID_ARG;
    if (j < (int)rows_of[s].size()) {
      // DuplicateThenTruncate: the first child continues the branch intact,
      // the others keep floor(f n) of its n tokens (f drawn by the caller)
      const int row = rows_of[s][j];
      const int n = branch_tokens_h[row - N];
      int h = j == 0 ? n : (int)std::floor(frac_h[c] * (double)n);
      if (next_len_h) h = std::min(h, next_len_h[c]);
      parent_rows_h[c] = row;
      new_len_h[c] = lens_h[s] + h;
      head_h[c] = h;
    } else {
      parent_rows_h[c] = s;
      new_len_h[c] = lens_h[s];
      head_h[c] = 0;
    }
  }
  return TTS_OK;
}

tts_status_t tts_beam_select_global(tts_ctx_t c, int32_t n_global, const float* scores_all, int32_t width_m,
                                    int32_t* parent_gid_out, void* stream) {
  if (!c || !scores_all || !parent_gid_out) return TTS_ERR_INVALID_ARG;
  if (n_global <= 0 || n_global > 1024 || width_m <= 0 || n_global % width_m) return TTS_ERR_INVALID_ARG;
  TTS_CUDA(tts::launch_select_global(c, scores_all, n_global, width_m, parent_gid_out, (cudaStream_t)stream));
  return TTS_OK;
}

tts_status_t tts_lineage_bytes(tts_ctx_t c, int32_t len, size_t* bytes_h) {
  if (!c || !bytes_h || len < 0) return TTS_ERR_INVALID_ARG;
  const tts_config_t& g = c->cfg;
  *bytes_h = (size_t)2 * g.num_layers * len * g.num_kv_heads * g.head_dim * 2;
  return TTS_OK;
}

tts_status_t tts_lineage_export(tts_ctx_t c, int32_t req, int32_t beam, void* buf, void* stream) {
  if (!c || !buf) return TTS_ERR_INVALID_ARG;
  if (!installed(c, req) || beam < 0 || beam >= c->n_rows[req]) return TTS_ERR_STATE;
  const int len = c->lens[(int64_t)req * c->cfg.max_beams + beam];
  TTS_CUDA(tts::launch_lineage_export(c, req, beam, len, buf, (cudaStream_t)stream));
  return TTS_OK;
}

tts_status_t tts_lineage_import(tts_ctx_t c, int32_t req, int32_t beam, int32_t len, const void* buf, void* stream) {
  if (!c || !buf || len <= 0) return TTS_ERR_INVALID_ARG;
  const tts_config_t& g = c->cfg;
  if (!installed(c, req)) return TTS_ERR_STATE;
  if (beam < c->n_beams[req] || beam >= g.max_beams || c->lens[(int64_t)req * g.max_beams + beam] != 0)
    return TTS_ERR_STATE;
  const int P = g.page_size, npg = (len + P - 1) / P;
  if (npg > g.max_pages_per_beam) return TTS_ERR_CAPACITY;
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e;
  std::vector<tts::AllocItem> items;
  for (int i = 0; i < npg; ++i) items.push_back({entry_of(g, req, beam, i), 0, 0});
  TTS_CUDA(tts::launch_alloc_host(c, items.data(), npg, st));
  TTS_CUDA(tts::launch_lineage_import(c, req, beam, len, buf, st));
  c->lens[(int64_t)req * g.max_beams + beam] = len;
  c->n_rows[req] = std::max(c->n_rows[req], beam + 1);
  return TTS_OK;
}

tts_status_t tts_block_table_release_request(tts_ctx_t c, int32_t req, void* stream) {
  if (!c) return TTS_ERR_INVALID_ARG;
  if (!installed(c, req)) return TTS_ERR_STATE;
  TTS_CUDA(tts::launch_release(c, req, c->n_rows[req], (cudaStream_t)stream));
  c->spans.erase(req);
  c->n_beams[req] = 0;
  c->n_rows[req] = 0;
  std::fill(c->lens.begin() + (int64_t)req * c->cfg.max_beams,
            c->lens.begin() + (int64_t)(req + 1) * c->cfg.max_beams, 0);
  return TTS_OK;
}

tts_status_t tts_block_table_snapshot(tts_ctx_t c, int32_t req, int32_t* n_beams_h,
                                      int32_t* tables_h, int32_t* lens_h, int32_t* ref_h,
                                      uint32_t* bitmap_h, void* stream) {
  if (!c || !tables_h || !lens_h) return TTS_ERR_INVALID_ARG;
  if (!installed(c, req)) return TTS_ERR_STATE;
  const tts_config_t& g = c->cfg;
  cudaStream_t st = (cudaStream_t)stream;
  const int N = c->n_beams[req];
  if (n_beams_h) *n_beams_h = N;
  TTS_CUDA(cudaMemcpyAsync(tables_h, c->buf.block_tables + entry_of(g, req, 0, 0),
                           (size_t)N * g.max_pages_per_beam * 4, cudaMemcpyDeviceToHost, st));
  TTS_CUDA(cudaMemcpyAsync(lens_h, c->buf.seq_lens + (int64_t)req * g.max_beams, (size_t)N * 4,
                           cudaMemcpyDeviceToHost, st));
  if (ref_h)
    TTS_CUDA(cudaMemcpyAsync(ref_h, c->buf.refcounts, (size_t)g.num_pages * 4, cudaMemcpyDeviceToHost, st));
  if (bitmap_h)
    TTS_CUDA(cudaMemcpyAsync(bitmap_h, c->buf.free_bitmap, (size_t)((g.num_pages + 31) / 32) * 4,
                             cudaMemcpyDeviceToHost, st));
  TTS_CUDA(cudaStreamSynchronize(st));
  return TTS_OK;
}

// f3: Dynamic Prefix-Aware Scheduling under a memory budget (PAPER.md 4.2,
// Appendix A).  Host scheduler over the request's device tables (one
// snapshot): CoT = a beam's page list; P(a, b) = shared leading pages, which
// for rows in DFS order (ledger C5) is the minimum of the adjacent rows'
// shared prefixes between them (the beam tree is prefix-closed).
tts_status_t tts_dpas_plan(tts_ctx_t c, int32_t req, int64_t budget_pages, const uint8_t* active_h,
                           int32_t* order_h, int32_t* trie_of_h, int32_t* n_tries_h, int64_t* cost_h,
                           int64_t* shared_h, void* stream) {
  if (!c || !order_h || !trie_of_h || !n_tries_h || !cost_h || !shared_h || budget_pages <= 0)
    return TTS_ERR_INVALID_ARG;
  if (!installed(c, req)) return TTS_ERR_STATE;
  const tts_config_t& g = c->cfg;
  const int P = g.page_size;
  const int N = c->n_beams[req];
  std::vector<int32_t> tab((size_t)N * g.max_pages_per_beam);
  cudaStream_t st = (cudaStream_t)stream;
  TTS_CUDA(cudaMemcpyAsync(tab.data(), c->buf.block_tables + entry_of(g, req, 0, 0), tab.size() * 4,
                           cudaMemcpyDeviceToHost, st));
  TTS_CUDA(cudaStreamSynchronize(st));
  std::vector<int> cots;  // the scheduled beams (active), input = index order
  for (int b = 0; b < N; ++b)
    if (!active_h || active_h[b]) cots.push_back(b);
  const int n = (int)cots.size();
  *n_tries_h = 0;
  *cost_h = 0;
  *shared_h = 0;
  if (n == 0) return TTS_OK;
  auto np = [&](int i) { return (c->lens[(int64_t)req * g.max_beams + cots[i]] + P - 1) / P; };
  auto row = [&](int i) { return tab.data() + (size_t)cots[i] * g.max_pages_per_beam; };
  std::vector<int> adj(n, 0);  // adj[i] = P(cot i, cot i+1)
  for (int i = 0; i + 1 < n; ++i) {
    const int m = std::min(np(i), np(i + 1));
    int k = 0;
    while (k < m && row(i)[k] == row(i + 1)[k]) ++k;
    adj[i] = k;
  }
  // greedy: the unscheduled CoT with the largest P with the
  // predecessor, ties to input order; order[0] = the first CoT
  std::vector<char> used(n, 0);
  std::vector<int> order;
  order.push_back(0);
  used[0] = 1;
  for (int k = 1; k < n; ++k) {
    const int prev = order.back();
    // P(prev, j) for every j by one sweep each way over adj
    int best = -1, bestp = -1;
    int m = INT32_MAX;
    for (int j = prev - 1; j >= 0; --j) {
      m = std::min(m, adj[j]);
      if (!used[j] && (m > bestp || (m == bestp && j < best))) best = j, bestp = m;
    }
    m = INT32_MAX;
    for (int j = prev + 1; j < n; ++j) {
      m = std::min(m, adj[j - 1]);
      if (!used[j] && (m > bestp || (m == bestp && j < best))) best = j, bestp = m;
    }
    order.push_back(best);
    used[best] = 1;
  }
  // first-fit packing into tries of <= budget pages, and the eviction cost
  std::vector<int32_t> mark((size_t)g.num_pages, -1);
  std::vector<std::vector<int>> tries;
  std::vector<int64_t> tsize;
  int64_t cur = 0;
  for (int i : order) {
    int64_t add = 0;
    for (int k = 0; k < np(i); ++k) add += mark[row(i)[k]] != (int)tries.size() - 1 || tries.empty();
    if (!tries.empty() && cur + add <= budget_pages) {
      for (int k = 0; k < np(i); ++k) mark[row(i)[k]] = (int)tries.size() - 1;
      tries.back().push_back(i);
      cur += add;
    } else {
      tries.push_back({i});
      cur = 0;
      for (int k = 0; k < np(i); ++k)
        if (mark[row(i)[k]] != (int)tries.size() - 1) mark[row(i)[k]] = (int)tries.size() - 1, ++cur;
    }
    tsize.resize(tries.size());
    tsize.back() = cur;
  }
  // shared nodes of consecutive tries
  std::vector<int32_t> seen((size_t)g.num_pages, -1);
  int64_t shared = 0, nodes = 0;
  for (size_t t = 0; t < tries.size(); ++t) {
    nodes += tsize[t];
    if (t + 1 < tries.size()) {
      for (int i : tries[t])
        for (int k = 0; k < np(i); ++k) seen[row(i)[k]] = (int)t;
      for (int i : tries[t + 1])
        for (int k = 0; k < np(i); ++k) {
          const int32_t p = row(i)[k];
          if (seen[p] == (int)t) {
            seen[p] = -2 - (int)t;  // count once
            ++shared;
          }
        }
    }
  }
  for (int k = 0; k < n; ++k) order_h[k] = cots[order[k]];
  for (size_t t = 0; t < tries.size(); ++t)
    for (int i : tries[t]) trie_of_h[cots[i]] = (int32_t)t;
  *n_tries_h = (int32_t)tries.size();
  *cost_h = nodes - shared;
  *shared_h = shared;
  return TTS_OK;
}

tts_status_t tts_block_table_stats(tts_ctx_t c, int32_t n_req, const int32_t* req_ids,
                                   const uint8_t* active, int64_t* accum, void* stream) {
  if (!c || n_req <= 0 || !req_ids || !accum) return TTS_ERR_INVALID_ARG;
  const tts_config_t& g = c->cfg;
  for (int i = 0; i < n_req; ++i)
    if (!installed(c, req_ids[i])) return TTS_ERR_STATE;
  std::vector<tts::GroupDesc> groups;
  plan_groups(c, n_req, req_ids, active, 32, groups);
  int64_t logical = 0;
  for (const auto& d : groups)
    for (int k = 0; k < d.nbeams; ++k)
      if ((d.active >> k) & 1u) logical += c->lens[(int64_t)d.req * g.max_beams + d.beam0 + k];
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e;
  void* d = groups.empty() ? nullptr
                           : tts::upload(c, groups.data(), groups.size() * sizeof(tts::GroupDesc), st, &e);
  if (!groups.empty()) TTS_CUDA(e);
  TTS_CUDA(tts::launch_stats(c, (const tts::GroupDesc*)d, (int)groups.size(), accum, logical, st));
  return TTS_OK;
}

tts_status_t tts_seq_lens_host(tts_ctx_t c, int32_t req, int32_t* lens_h) {
  if (!c || !lens_h) return TTS_ERR_INVALID_ARG;
  if (!installed(c, req)) return TTS_ERR_STATE;
  std::memcpy(lens_h, c->lens.data() + (int64_t)req * c->cfg.max_beams, (size_t)c->n_beams[req] * 4);
  return TTS_OK;
}

}  // extern "C"
