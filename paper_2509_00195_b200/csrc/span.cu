// a8: one request whose beams span G GPUs (ledger C19/C20).
//
// "standard Beam Search selects the top-K candidates globally
// with a static branching factor".  When a request's N beams are spread over
// G ranks, "globally" needs every rank to see every score.  Per TTS step:
//   1. all-gather of (score, gid, len) for every local beam (12 B per beam);
//   2. every rank runs the same selection kernel (k_select, the single-GPU
//      key with the gid as index) over the N gathered scores -> identical
//      parent maps everywhere;
//   3. placement (host, identical on every rank): children in gid order stay
//      on their parent's rank while its capacity lasts, the overflow (in gid
//      order) goes to the lowest rank with free capacity;
//   4. lineage migration: a rank imports the whole lineage of each remote
//      parent one of its children needs (export kernel -> transport ->
//      import kernel into a spare row, fresh pages), in ascending parent gid;
//   5. local fork by an explicit parent map (tts_beam_fork_map).
// Transports: NCCL (device buffers; libnccl is resolved at run time, the one
// torch already loaded) or host callbacks (any byte transport: gloo process
// groups, or threads of one process acting as ranks).
#include <dlfcn.h>

#include <algorithm>
#include <cstring>
#include <map>
#include <numeric>

#include "tts_internal.cuh"

namespace tts {
namespace {

// --- NCCL, resolved at run time --------------------------------------------
typedef struct {
  char internal[128];
} NcclId;
typedef void* NcclComm;
typedef int (*fn_get_id)(NcclId*);
typedef int (*fn_init_rank)(NcclComm*, int, NcclId, int);
typedef int (*fn_destroy)(NcclComm);
typedef int (*fn_allgather)(const void*, void*, size_t, int, NcclComm, cudaStream_t);
typedef int (*fn_p2p)(const void*, size_t, int, int, NcclComm, cudaStream_t);
typedef int (*fn_p2p_recv)(void*, size_t, int, int, NcclComm, cudaStream_t);
typedef int (*fn_group)();
constexpr int kNcclUint8 = 1;

struct Nccl {
  bool ok = false;
  fn_get_id get_id = nullptr;
  fn_init_rank init_rank = nullptr;
  fn_destroy destroy = nullptr;
  fn_allgather allgather = nullptr;
  fn_p2p send = nullptr;
  fn_p2p_recv recv = nullptr;
  fn_group group_start = nullptr, group_end = nullptr;
};

const Nccl& nccl() {
  static Nccl n = [] {
    Nccl r;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);  // torch's, if loaded
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return r;
    r.get_id = (fn_get_id)dlsym(h, "ncclGetUniqueId");
    r.init_rank = (fn_init_rank)dlsym(h, "ncclCommInitRank");
    r.destroy = (fn_destroy)dlsym(h, "ncclCommDestroy");
    r.allgather = (fn_allgather)dlsym(h, "ncclAllGather");
    r.send = (fn_p2p)dlsym(h, "ncclSend");
    r.recv = (fn_p2p_recv)dlsym(h, "ncclRecv");
    r.group_start = (fn_group)dlsym(h, "ncclGroupStart");
    r.group_end = (fn_group)dlsym(h, "ncclGroupEnd");
    r.ok = r.get_id && r.init_rank && r.destroy && r.allgather && r.send && r.recv && r.group_start &&
           r.group_end;
    return r;
  }();
  return n;
}

// (score, gid, len) of one local beam, the all-gather record
struct BeamRec {
  float score;
  int32_t gid, len;
};

__global__ void k_pack_recs(const float* __restrict__ scores, const int32_t* __restrict__ meta, int n, int cap,
                            BeamRec* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= cap) return;
  out[i] = i < n ? BeamRec{scores[i], meta[2 * i], meta[2 * i + 1]} : BeamRec{0.f, -1, 0};
}

// gathered records -> scores_all[gid] (every gid is present exactly once)
__global__ void k_scatter_scores(const BeamRec* __restrict__ recs, int n_recs, float* scores_all) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n_recs && recs[i].gid >= 0) scores_all[recs[i].gid] = recs[i].score;
}

}  // namespace

struct Comm {
  int nranks = 1, rank = 0;
  bool is_nccl = false;
  NcclComm nc = nullptr;
  tts_host_transport_t host{};
  uint8_t* stage = nullptr;  // NCCL: caller-owned device staging
  size_t stage_bytes = 0;
  uint8_t* hstage = nullptr;  // host transport: pinned staging (libtts-owned)
  size_t hstage_bytes = 0;
};

}  // namespace tts

using tts::Ctx;
struct tts_ctx : public Ctx {};

namespace {

void placement(int n, const int32_t* parent, const int32_t* old_rank, int nranks, const int32_t* caps,
               int32_t* child_rank) {
  std::vector<int32_t> fill(nranks, 0);
  for (int c = 0; c < n; ++c) {
    const int r = old_rank[parent[c]];
    child_rank[c] = -1;
    if (fill[r] < caps[r]) {
      child_rank[c] = r;
      ++fill[r];
    }
  }
  int q = 0;
  for (int c = 0; c < n; ++c) {
    if (child_rank[c] >= 0) continue;
    while (q < nranks && fill[q] >= caps[q]) ++q;
    child_rank[c] = q;
    ++fill[q];
  }
}

size_t lineage_bytes(const tts_config_t& g, int len) {
  return (size_t)2 * g.num_layers * len * g.num_kv_heads * g.head_dim * 2;
}

// Page origins (f4): who created a page, where -- equal on every rank holding
// a copy, distinct for pages whose contents may differ.  A full page's tokens
// are a function of its origin, so a destination already holding the pages
// of a lineage's prefix (same origins) need not receive them again.
//   full prompt page k:                     0xFFFF << 16 | k
//   the partial prompt page of gid g:       1 << 62 | g << 16 | k
//   a page opened by gid g's append at the decode call tau of the request:
//                                           (tau + 1) << 32 | g << 16 | k
//   a fresh copy of a partially filled page (fork CoW; the partial last page
//   of an imported lineage) for child gid c:  1 << 61 | (tau + 1) << 32 | c << 16 | k
uint64_t origin_prompt(int k) { return (0xFFFFull << 16) | (uint64_t)k; }
uint64_t origin_prompt_partial(int g, int k) { return (1ull << 62) | ((uint64_t)g << 16) | (uint64_t)k; }
uint64_t origin_open(uint32_t tau, int g, int k) {
  return ((uint64_t)(tau + 1) << 32) | ((uint64_t)g << 16) | (uint64_t)k;
}
uint64_t origin_copy(uint32_t tau, int c, int k) {
  return (1ull << 61) | ((uint64_t)(tau + 1) << 32) | ((uint64_t)c << 16) | (uint64_t)k;
}

}  // namespace

namespace tts {
// Called by every append of the context (api.cu) before its launch: record
// the origins of the pages the call opens, for requests tracking them.
void span_note_append(Ctx* c, int n_req, const int32_t* req_ids, const std::vector<AllocItem>& items) {
  if (c->spans.empty()) return;
  const tts_config_t& g = c->cfg;
  for (const AllocItem& it : items) {
    const int64_t row_all = it.entry / g.max_pages_per_beam;
    const int pos = (int)(it.entry % g.max_pages_per_beam);
    const int req = (int)(row_all / g.max_beams), b = (int)(row_all % g.max_beams);
    auto sp = c->spans.find(req);
    if (sp == c->spans.end() || !sp->second.dedup) continue;
    Span& S = sp->second;
    S.origin[(size_t)b * g.max_pages_per_beam + pos] = origin_open(S.tau, S.gids[b], pos);
  }
  for (int i = 0; i < n_req; ++i) {
    auto sp = c->spans.find(req_ids[i]);
    if (sp != c->spans.end()) ++sp->second.tau;
  }
}
}  // namespace tts

extern "C" {

tts_status_t tts_span_placement(int32_t n_global, const int32_t* parent_gid_h, const int32_t* old_rank_h,
                                int32_t nranks, const int32_t* caps_h, int32_t* child_rank_h) {
  if (n_global <= 0 || nranks <= 0 || !parent_gid_h || !old_rank_h || !caps_h || !child_rank_h)
    return TTS_ERR_INVALID_ARG;
  int64_t tot = 0;
  for (int r = 0; r < nranks; ++r) {
    if (caps_h[r] < 0) return TTS_ERR_INVALID_ARG;
    tot += caps_h[r];
  }
  if (tot != n_global) return TTS_ERR_INVALID_ARG;
  for (int c = 0; c < n_global; ++c) {
    if (parent_gid_h[c] < 0 || parent_gid_h[c] >= n_global) return TTS_ERR_INVALID_ARG;
    const int r = old_rank_h[parent_gid_h[c]];
    if (r < 0 || r >= nranks) return TTS_ERR_INVALID_ARG;
  }
  placement(n_global, parent_gid_h, old_rank_h, nranks, caps_h, child_rank_h);
  return TTS_OK;
}

tts_status_t tts_comm_unique_id(void* id_h) {
  if (!id_h) return TTS_ERR_INVALID_ARG;
  const tts::Nccl& n = tts::nccl();
  if (!n.ok) return TTS_ERR_NCCL;
  return n.get_id((tts::NcclId*)id_h) == 0 ? TTS_OK : TTS_ERR_NCCL;
}

tts_status_t tts_comm_init(tts_ctx_t c, const void* id_h, int32_t nranks, int32_t rank, void* stage,
                           size_t stage_bytes) {
  if (!c || !id_h || nranks <= 0 || rank < 0 || rank >= nranks) return TTS_ERR_INVALID_ARG;
  if (!stage || stage_bytes < 4096) return TTS_ERR_INVALID_ARG;
  if (c->comm) return TTS_ERR_STATE;
  const tts::Nccl& n = tts::nccl();
  if (!n.ok) return TTS_ERR_NCCL;
  TTS_CUDA(cudaSetDevice(c->device));
  tts::NcclId id;
  std::memcpy(&id, id_h, sizeof(id));
  tts::NcclComm comm = nullptr;
  if (n.init_rank(&comm, nranks, id, rank) != 0) return TTS_ERR_NCCL;
  auto* m = new tts::Comm();
  m->nranks = nranks;
  m->rank = rank;
  m->is_nccl = true;
  m->nc = comm;
  m->stage = (uint8_t*)stage;
  m->stage_bytes = stage_bytes;
  c->comm = m;
  return TTS_OK;
}

tts_status_t tts_comm_init_host(tts_ctx_t c, int32_t nranks, int32_t rank, const tts_host_transport_t* t,
                                size_t stage_bytes) {
  if (!c || !t || !t->allgather || !t->sendrecv || nranks <= 0 || rank < 0 || rank >= nranks)
    return TTS_ERR_INVALID_ARG;
  if (c->comm) return TTS_ERR_STATE;
  auto* m = new tts::Comm();
  m->nranks = nranks;
  m->rank = rank;
  m->host = *t;
  m->hstage_bytes = std::max<size_t>(stage_bytes, 4096);
  if (cudaMallocHost(&m->hstage, m->hstage_bytes) != cudaSuccess) {
    delete m;
    return TTS_ERR_CUDA;
  }
  c->comm = m;
  return TTS_OK;
}

tts_status_t tts_comm_destroy(tts_ctx_t c) {
  if (!c) return TTS_ERR_INVALID_ARG;
  if (!c->comm) return TTS_OK;
  if (c->comm->nc) tts::nccl().destroy(c->comm->nc);
  if (c->comm->hstage) cudaFreeHost(c->comm->hstage);
  delete c->comm;
  c->comm = nullptr;
  return TTS_OK;
}

tts_status_t tts_span_init(tts_ctx_t c, int32_t req, int32_t n_global, const int32_t* caps_h, int32_t dedup) {
  if (!c || !caps_h || !c->comm) return c && !c->comm ? TTS_ERR_STATE : TTS_ERR_INVALID_ARG;
  const int G = c->comm->nranks, me = c->comm->rank;
  if (req < 0 || req >= c->cfg.max_requests || c->n_beams[req] <= 0) return TTS_ERR_STATE;
  int64_t tot = 0;
  for (int r = 0; r < G; ++r) {
    if (caps_h[r] <= 0 || 2 * caps_h[r] > c->cfg.max_beams) return TTS_ERR_CAPACITY;  // + spare rows
    tot += caps_h[r];
  }
  if (tot != n_global || n_global > 1024) return TTS_ERR_INVALID_ARG;
  if (c->n_beams[req] != caps_h[me] || c->n_rows[req] != caps_h[me]) return TTS_ERR_STATE;
  tts::Span s;
  s.n_global = n_global;
  s.caps.assign(caps_h, caps_h + G);
  const int start = std::accumulate(caps_h, caps_h + me, 0);
  for (int i = 0; i < caps_h[me]; ++i) s.gids.push_back(start + i);
  s.dedup = dedup != 0;
  if (s.dedup) {
    // only prompt pages so far (the request was just installed)
    const tts_config_t& g = c->cfg;
    const int len = c->lens[(int64_t)req * g.max_beams];
    const int P = g.page_size, npg = (len + P - 1) / P;
    s.origin.assign((size_t)g.max_beams * g.max_pages_per_beam, 0);
    for (int i = 0; i < caps_h[me]; ++i) {
      if (c->lens[(int64_t)req * g.max_beams + i] != len) return TTS_ERR_STATE;  // decoded already
      for (int k = 0; k < npg; ++k)
        s.origin[(size_t)i * g.max_pages_per_beam + k] =
            (k + 1) * P <= len ? origin_prompt(k) : origin_prompt_partial(start + i, k);
    }
  }
  c->spans[req] = s;
  return TTS_OK;
}

tts_status_t tts_span_stats(tts_ctx_t c, int32_t req, int64_t* migrated_bytes_h, int64_t* deduped_bytes_h) {
  if (!c || !migrated_bytes_h || !deduped_bytes_h) return TTS_ERR_INVALID_ARG;
  auto it = c->spans.find(req);
  if (it == c->spans.end()) return TTS_ERR_STATE;
  *migrated_bytes_h = it->second.migrated_bytes;
  *deduped_bytes_h = it->second.deduped_bytes;
  return TTS_OK;
}

tts_status_t tts_span_gids(tts_ctx_t c, int32_t req, int32_t* gids_h) {
  if (!c || !gids_h) return TTS_ERR_INVALID_ARG;
  auto it = c->spans.find(req);
  if (it == c->spans.end()) return TTS_ERR_STATE;
  std::copy(it->second.gids.begin(), it->second.gids.end(), gids_h);
  return TTS_OK;
}

tts_status_t tts_beam_select_fork_global(tts_ctx_t c, int32_t req, const float* local_scores, int32_t M,
                                         int32_t* parent_gid_out, int32_t* child_rank_out, void* stream) {
  if (!c || !local_scores) return TTS_ERR_INVALID_ARG;
  if (!c->comm) return TTS_ERR_STATE;
  auto sit = c->spans.find(req);
  if (sit == c->spans.end() || c->n_beams[req] <= 0) return TTS_ERR_STATE;
  tts::Span& sp = sit->second;
  tts::Comm& cm = *c->comm;
  const tts_config_t& g = c->cfg;
  const int N = sp.n_global, G = cm.nranks, me = cm.rank;
  const int n_loc = (int)sp.gids.size();
  if (M <= 0 || N % M) return TTS_ERR_INVALID_ARG;
  if (c->n_rows[req] != n_loc || c->n_beams[req] != n_loc) return TTS_ERR_STATE;
  const int cap_max = *std::max_element(sp.caps.begin(), sp.caps.end());
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e;
  const size_t rec_bytes = (size_t)cap_max * sizeof(tts::BeamRec);
  // ---- 1. all-gather (score, gid, len)
  std::vector<tts::BeamRec> recs((size_t)G * cap_max);
  std::vector<int32_t> meta(2 * (size_t)n_loc);
  for (int i = 0; i < n_loc; ++i) {
    meta[2 * i] = sp.gids[i];
    meta[2 * i + 1] = c->lens[(int64_t)req * g.max_beams + i];
  }
  float* scores_all = c->ws_scores_all;
  if (cm.is_nccl) {
    if (cm.stage_bytes < rec_bytes * (G + 1)) return TTS_ERR_CAPACITY;
    void* dmeta = tts::upload(c, meta.data(), meta.size() * 4, st, &e);
    TTS_CUDA(e);
    tts::BeamRec* dsend = (tts::BeamRec*)cm.stage;
    tts::BeamRec* drecv = dsend + cap_max;
    tts::k_pack_recs<<<(cap_max + 127) / 128, 128, 0, st>>>(local_scores, (const int32_t*)dmeta, n_loc, cap_max,
                                                            dsend);
    c->launches++;
    TTS_CUDA(cudaGetLastError());
    if (tts::nccl().allgather(dsend, drecv, rec_bytes, tts::kNcclUint8, cm.nc, st) != 0) return TTS_ERR_NCCL;
    tts::k_scatter_scores<<<(G * cap_max + 127) / 128, 128, 0, st>>>(drecv, G * cap_max, scores_all);
    c->launches++;
    TTS_CUDA(cudaGetLastError());
    TTS_CUDA(cudaMemcpyAsync(recs.data(), drecv, recs.size() * sizeof(tts::BeamRec), cudaMemcpyDeviceToHost, st));
    TTS_CUDA(cudaStreamSynchronize(st));
  } else {
    std::vector<float> sc(n_loc);
    TTS_CUDA(cudaMemcpyAsync(sc.data(), local_scores, (size_t)n_loc * 4, cudaMemcpyDeviceToHost, st));
    TTS_CUDA(cudaStreamSynchronize(st));
    std::vector<tts::BeamRec> mine(cap_max, tts::BeamRec{0.f, -1, 0});
    for (int i = 0; i < n_loc; ++i) mine[i] = tts::BeamRec{sc[i], meta[2 * i], meta[2 * i + 1]};
    if (cm.host.allgather(cm.host.user, mine.data(), recs.data(), rec_bytes) != 0) return TTS_ERR_NCCL;
    std::vector<float> all(N, 0.f);
    for (const auto& r : recs)
      if (r.gid >= 0) all[r.gid] = r.score;
    void* d = tts::upload(c, all.data(), (size_t)N * 4, st, &e);
    TTS_CUDA(e);
    TTS_CUDA(cudaMemcpyAsync(scores_all, d, (size_t)N * 4, cudaMemcpyDeviceToDevice, st));
  }
  std::vector<int32_t> old_rank(N, -1), len_of(N, 0);
  for (int r = 0; r < G; ++r)
    for (int i = 0; i < cap_max; ++i) {
      const tts::BeamRec& x = recs[(size_t)r * cap_max + i];
      if (x.gid < 0) continue;
      if (x.gid >= N || old_rank[x.gid] >= 0) return TTS_ERR_STATE;  // inconsistent spans
      old_rank[x.gid] = r;
      len_of[x.gid] = x.len;
    }
  for (int q = 0; q < N; ++q)
    if (old_rank[q] < 0) return TTS_ERR_STATE;
  // ---- 1b. f4: every rank's page origins ([cap_max][max_pages] uint64 per rank)
  const int maxP = g.max_pages_per_beam;
  const size_t org_bytes = (size_t)cap_max * maxP * 8;
  std::vector<uint64_t> org_all;
  std::vector<const uint64_t*> org_of(N, nullptr);  // gid -> its origin row
  if (sp.dedup) {
    org_all.resize((size_t)G * cap_max * maxP);
    std::vector<uint64_t> mine((size_t)cap_max * maxP, 0);
    std::copy(sp.origin.begin(), sp.origin.begin() + (size_t)n_loc * maxP, mine.begin());
    if (cm.is_nccl) {
      if (cm.stage_bytes < org_bytes * (G + 1)) return TTS_ERR_CAPACITY;
      TTS_CUDA(cudaMemcpyAsync(cm.stage, mine.data(), org_bytes, cudaMemcpyHostToDevice, st));
      if (tts::nccl().allgather(cm.stage, cm.stage + org_bytes, org_bytes, tts::kNcclUint8, cm.nc, st) != 0)
        return TTS_ERR_NCCL;
      TTS_CUDA(cudaMemcpyAsync(org_all.data(), cm.stage + org_bytes, org_bytes * G, cudaMemcpyDeviceToHost, st));
      TTS_CUDA(cudaStreamSynchronize(st));
    } else if (cm.host.allgather(cm.host.user, mine.data(), org_all.data(), org_bytes) != 0) {
      return TTS_ERR_NCCL;
    }
    for (int r = 0; r < G; ++r)
      for (int i = 0; i < cap_max; ++i) {
        const tts::BeamRec& x = recs[(size_t)r * cap_max + i];
        if (x.gid >= 0) org_of[x.gid] = org_all.data() + ((size_t)r * cap_max + i) * maxP;
      }
  }
  // ---- 2. global selection (the single-GPU kernel over gid-indexed scores)
  int32_t* dparent = c->ws_parent_all;
  TTS_CUDA(tts::launch_select_global(c, scores_all, N, M, dparent, st));
  std::vector<int32_t> parent(N);
  TTS_CUDA(cudaMemcpyAsync(parent.data(), dparent, (size_t)N * 4, cudaMemcpyDeviceToHost, st));
  TTS_CUDA(cudaStreamSynchronize(st));
  if (parent_gid_out) TTS_CUDA(cudaMemcpyAsync(parent_gid_out, dparent, (size_t)N * 4, cudaMemcpyDeviceToDevice, st));
  // ---- 3. placement (identical on every rank)
  std::vector<int32_t> child_rank(N);
  placement(N, parent.data(), old_rank.data(), G, sp.caps.data(), child_rank.data());
  // per rank: children (ascending gid) and the remote parents it imports (ascending gid)
  std::vector<std::vector<int32_t>> children(G), imports(G);
  for (int q = 0; q < N; ++q) children[child_rank[q]].push_back(q);
  for (int r = 0; r < G; ++r) {
    for (int q : children[r])
      if (old_rank[parent[q]] != r) imports[r].push_back(parent[q]);
    std::sort(imports[r].begin(), imports[r].end());
    imports[r].erase(std::unique(imports[r].begin(), imports[r].end()), imports[r].end());
  }
  // ---- 4. lineage migration, in rounds that fit the staging buffer; the
  // global transfer list (parent gid, src, dst) is the same on every rank
  struct Xfer {
    int32_t p, src, dst;
    size_t bytes;
    int32_t m, share;  // f4: leading pages the destination holds already (its beam `share`, gid)
  };
  const int P = g.page_size;
  // f4: the longest run of leading FULL pages of p (same origins) that a beam
  // of the destination holds; ties to the lowest gid
  auto dedup_of = [&](int p, int dst, int& share) {
    share = -1;
    if (!sp.dedup) return 0;
    int best = 0;
    for (int y = 0; y < N; ++y) {
      if (old_rank[y] != dst) continue;
      const int full = std::min(len_of[p], len_of[y]) / P;
      int k = 0;
      while (k < full && org_of[p][k] == org_of[y][k]) ++k;
      if (k > best) best = k, share = y;
    }
    return best;
  };
  std::vector<Xfer> xf;
  for (int r = 0; r < G; ++r)
    for (int p : imports[r]) {
      int share;
      const int m = dedup_of(p, r, share);
      xf.push_back({p, old_rank[p], r, lineage_bytes(g, len_of[p] - m * P), m, share});
      if (old_rank[p] == me) {
        sp.migrated_bytes += (int64_t)lineage_bytes(g, len_of[p] - m * P);
        sp.deduped_bytes += (int64_t)lineage_bytes(g, m * P);
      }
    }
  std::sort(xf.begin(), xf.end(), [](const Xfer& a, const Xfer& b) {
    return a.p != b.p ? a.p < b.p : a.dst < b.dst;
  });
  const size_t half = (cm.is_nccl ? cm.stage_bytes : cm.hstage_bytes) / 2 / 256 * 256;
  std::map<int32_t, int32_t> row_of;  // gid -> local row
  for (int i = 0; i < n_loc; ++i) row_of[sp.gids[i]] = i;
  int next_spare = n_loc;
  std::map<int32_t, int32_t> spare_of;  // imported gid -> spare row
  for (size_t k0 = 0; k0 < xf.size();) {
    std::vector<size_t> sent(G, 0), recvd(G, 0);
    size_t k1 = k0;
    while (k1 < xf.size()) {
      const Xfer& x = xf[k1];
      const size_t b = (x.bytes + 255) / 256 * 256;
      if (b > half) return TTS_ERR_CAPACITY;  // one lineage larger than the staging half
      if (sent[x.src] + b > half || recvd[x.dst] + b > half) break;
      sent[x.src] += b;
      recvd[x.dst] += b;
      ++k1;
    }
    // this rank's part of the round
    std::vector<int32_t> sdst, ssrc;
    std::vector<size_t> sbytes, rbytes, soff, roff;
    std::vector<int32_t> rgid, rm, rshare;
    size_t so = 0, ro = 0;
    for (size_t k = k0; k < k1; ++k) {
      const Xfer& x = xf[k];
      const size_t b = (x.bytes + 255) / 256 * 256;
      if (x.src == me) {
        sdst.push_back(x.dst);
        sbytes.push_back(x.bytes);
        soff.push_back(so);
        so += b;
      }
      if (x.dst == me) {
        ssrc.push_back(x.src);
        rbytes.push_back(x.bytes);
        roff.push_back(ro);
        rgid.push_back(x.p);
        rm.push_back(x.m);
        rshare.push_back(x.share);
        ro += b;
      }
    }
    uint8_t* sbase = cm.is_nccl ? cm.stage : cm.hstage;
    uint8_t* rbase = sbase + half;
    // exports (device): into the NCCL staging, or a device scratch slice then D2H
    {
      size_t i = 0;
      for (size_t k = k0; k < k1; ++k) {
        const Xfer& x = xf[k];
        if (x.src != me) continue;
        const int row = row_of.at(x.p);
        if (cm.is_nccl) {
          TTS_CUDA(tts::launch_lineage_export(c, req, row, len_of[x.p], sbase + soff[i], st, x.m * P));
        } else {
          // host transport: export into a device bounce buffer, then D2H
          void* dtmp = nullptr;
          TTS_CUDA(cudaMallocAsync(&dtmp, x.bytes, st));
          TTS_CUDA(tts::launch_lineage_export(c, req, row, len_of[x.p], dtmp, st, x.m * P));
          TTS_CUDA(cudaMemcpyAsync(sbase + soff[i], dtmp, x.bytes, cudaMemcpyDeviceToHost, st));
          TTS_CUDA(cudaFreeAsync(dtmp, st));
        }
        ++i;
      }
    }
    if (cm.is_nccl) {
      const tts::Nccl& n = tts::nccl();
      if (n.group_start() != 0) return TTS_ERR_NCCL;
      for (size_t i = 0; i < sdst.size(); ++i)
        if (n.send(sbase + soff[i], sbytes[i], tts::kNcclUint8, sdst[i], cm.nc, st) != 0) return TTS_ERR_NCCL;
      for (size_t i = 0; i < ssrc.size(); ++i)
        if (n.recv(rbase + roff[i], rbytes[i], tts::kNcclUint8, ssrc[i], cm.nc, st) != 0) return TTS_ERR_NCCL;
      if (n.group_end() != 0) return TTS_ERR_NCCL;
    } else {
      TTS_CUDA(cudaStreamSynchronize(st));
      std::vector<const void*> sp_(sdst.size());
      std::vector<void*> rp_(ssrc.size());
      for (size_t i = 0; i < sdst.size(); ++i) sp_[i] = sbase + soff[i];
      for (size_t i = 0; i < ssrc.size(); ++i) rp_[i] = rbase + roff[i];
      if (cm.host.sendrecv(cm.host.user, (int32_t)sdst.size(), sdst.data(), sp_.data(), sbytes.data(),
                           (int32_t)ssrc.size(), ssrc.data(), rp_.data(), rbytes.data()) != 0)
        return TTS_ERR_NCCL;
    }
    // imports (ascending parent gid within and across rounds)
    for (size_t i = 0; i < rgid.size(); ++i) {
      const int p = rgid[i];
      const int row = next_spare++;
      const void* src = rbase + roff[i];
      void* dtmp = nullptr;
      if (!cm.is_nccl) {
        TTS_CUDA(cudaMallocAsync(&dtmp, rbytes[i], st));
        TTS_CUDA(cudaMemcpyAsync(dtmp, src, rbytes[i], cudaMemcpyHostToDevice, st));
        src = dtmp;
      }
      // the shared prefix from the local beam holding it, fresh pages for the
      // rest (lowest free ids), the received tokens into them
      const int m = rm[i], npg = (len_of[p] + P - 1) / P;
      if (row >= g.max_beams) return TTS_ERR_CAPACITY;
      if (m > 0) TTS_CUDA(tts::launch_share_prefix(c, req, row, row_of.at(rshare[i]), m, st));
      std::vector<tts::AllocItem> items;
      for (int k = m; k < npg; ++k)
        items.push_back({((int64_t)req * g.max_beams + row) * g.max_pages_per_beam + k, 0, 0});
      TTS_CUDA(tts::launch_alloc_host(c, items.data(), (int)items.size(), st));
      TTS_CUDA(tts::launch_lineage_import(c, req, row, len_of[p], src, st, m * P));
      c->lens[(int64_t)req * g.max_beams + row] = len_of[p];
      c->n_rows[req] = std::max(c->n_rows[req], row + 1);
      if (dtmp) TTS_CUDA(cudaFreeAsync(dtmp, st));
      spare_of[p] = row;
      if (sp.dedup) std::copy(org_of[p], org_of[p] + maxP, sp.origin.begin() + (size_t)row * maxP);
    }
    // the staging halves are reused by the next round
    TTS_CUDA(cudaStreamSynchronize(st));
    k0 = k1;
  }
  // ---- 5. local fork by map: new row i = i-th child of this rank (ascending gid)
  std::vector<int32_t> prow;
  for (int q : children[me]) {
    const int p = parent[q];
    prow.push_back(old_rank[p] == me ? row_of.at(p) : spare_of.at(p));
  }
  tts_status_t s = tts_beam_fork_map(c, req, (int32_t)prow.size(), prow.data(), stream);
  if (s != TTS_OK) return s;
  if (sp.dedup) {
    // children take their parent row's origins; a partially filled last page
    // that is a fresh copy -- every child but the first of its row (fork
    // CoW), and the first child of an imported row (its page is a copy of
    // the exporter's) -- gets a fresh origin
    std::vector<uint64_t> old = sp.origin;
    std::vector<char> seen((size_t)g.max_beams, 0);
    for (size_t i = 0; i < prow.size(); ++i) {
      const int pr = prow[i], len = c->lens[(int64_t)req * g.max_beams + (int)i];
      std::copy(old.begin() + (size_t)pr * maxP, old.begin() + (size_t)(pr + 1) * maxP,
                sp.origin.begin() + i * maxP);
      if (len % P && (seen[pr] || pr >= n_loc))
        sp.origin[i * maxP + (len - 1) / P] = origin_copy(sp.tau, children[me][i], (len - 1) / P);
      seen[pr] = 1;
    }
  }
  sp.gids = children[me];
  if (child_rank_out) {
    void* d = tts::upload(c, child_rank.data(), (size_t)N * 4, st, &e);
    TTS_CUDA(e);
    TTS_CUDA(cudaMemcpyAsync(child_rank_out, d, (size_t)N * 4, cudaMemcpyDeviceToDevice, st));
  }
  return TTS_OK;
}

}  // extern "C"
