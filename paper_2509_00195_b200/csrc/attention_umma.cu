// Prefix-shared tree decode attention on the 5th-generation tensor cores
// (tcgen05 + TMEM + TMA), sm_100a.  Same contract as attention.cu (see there
// and include/tts.h); this is the path for head_dim 128 and 4 <= G <= 16.
//
// a3 (plan, k_plan): per beam group -- a run of <= floor(128/G) consecutive
// beams of one request, in DFS order so that every shared page's beams are
// adjacent (ledger C5) -- the ordered list of DISTINCT pages
// of the group's block-table rows, each with its member-beam bitmask and valid
// token count.  Computed once per call, shared by every layer and kv head.
//
// a4 (k_tree_umma): one CTA owns a 128-row query tile (the group's beams x the
// G query heads of one kv head) for one layer, and a contiguous, balanced
// slice of the group's page list when the grid would not fill the GPU.
// Per unit of two pages:
//   producer warp  TMA (3D box = one 16x128 bf16 tile, SWIZZLE_128B) -> smem ring
//   MMA warp       S[128 x 32] = Q . K^T     tcgen05.mma kind::f16, S in TMEM
//   softmax WG     one thread per row: tcgen05.ld S; mask rows whose beam does not
//                  reference the page and token slots >= ntok; fp32 online softmax
//                  with lazy rescale (O rescaled in TMEM only when the running max
//                  grows by > 2^8); P in fp16 -> tcgen05.st over S
//   MMA warp       O[128 x 128] += P . V   fp16 x fp16 (A from TMEM; V is kept in
//                  fp16 in the pool, MN-major operand; ledger C14)
// Each distinct page is fetched once per CTA and multiplied against all 128
// rows: every GQA head and every beam of the tile that references it.
// Slices of one tile form a thread-block cluster; their partial (m, l, O) are
// merged through distributed shared memory, never through HBM.
#include "sm100.cuh"
#include "tts_internal.cuh"

namespace tts {
namespace {
using namespace sm100;

constexpr int kP = 16;
constexpr int kD = 128;
constexpr int kRows = 128;
constexpr int kU = 2;                        // pages per unit
constexpr int kNS = 6;                       // ring slots (units)
constexpr int kTile = kP * kD * 2;           // 4 KiB: one (page, kv head) K or V tile
constexpr int kSlot = 2 * kU * kTile;        // 16 KiB: K tiles then V tiles
constexpr int kRing = kNS * kSlot;           // 64 KiB
constexpr int kThreads = 192;                // warps 0-3 softmax, 4 producer, 5 MMA
constexpr int kTmemCols = 256;               // O [0,128), Q [128,192), S/P [192,224), [224,256)
constexpr int kSCols = kU * kP;              // 32

constexpr int kOffRing = 0;
constexpr int kOffMeta = kOffRing + kRing;
constexpr int kOffBar = kOffMeta + kNS * kU * 16;
constexpr int kNumBars = 2 * kNS + 6;        // full, empty, sfull[2], pfull[2], pv[2]
constexpr int kOffML = kOffBar + kNumBars * 8 + 16;
constexpr int kSmemBytes = kOffML + 2 * kRows * 4 + 1024;
static_assert(kRing >= kRows * kD * 4, "merge area must hold a 128x128 fp32 tile");

#ifdef TTS_TRACE
__device__ long long g_trace[1024][8];
__device__ long long g_trace2[1024][8];
#define TTS_TR(j, ev)                                                                   \
  do {                                                                                  \
    if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 10 && (j) >= 0 && (j) < 1024) \
      g_trace[(j)][(ev)] = clock64();                                                   \
  } while (0)
#define TTS_TR2(j, ev)                                                                  \
  do {                                                                                  \
    if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 10 && (j) >= 0 && (j) < 1024) \
      g_trace2[(j)][(ev)] = clock64();                                                  \
  } while (0)
#else
#define TTS_TR(j, ev) \
  do {                \
  } while (0)
#define TTS_TR2(j, ev) \
  do {                 \
  } while (0)
#endif

struct UParams {
  const int32_t* lens;
  const __nv_bfloat16* q;
  float* out;
  const GroupDesc* groups;
  const int4* items;
  const int32_t* counts;
  int32_t* status;
  int layer_begin, n_call, Hq, Hkv, G, maxB, splits;
  int64_t num_pages;
  float scale_log2;
};

// ---------------------------------------------------------------------------
// a3: plan.  One CTA per group, one warp per position (NT/32 positions a round).
template <int NT>
__device__ __forceinline__ void plan_group(const GroupDesc& g, int gi, const int32_t* __restrict__ tables,
                                           int32_t* __restrict__ lens, int4* __restrict__ items,
                                           int32_t* __restrict__ counts, int maxB, int maxP, int32_t* tb,
                                           bool bump) {
  constexpr int NW = NT / 32;
  __shared__ int s_len[32];
  __shared__ int s_cnt[32];
  __shared__ int s_off[32];
  __shared__ int s_tot;
  const int nb = g.nbeams, npg = g.max_npages, ld = npg + 1;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid < 32) {
    const bool act = tid < nb && ((g.active >> tid) & 1u);
    int len = act ? lens[(int64_t)g.req * maxB + g.beam0 + tid] : 0;
    if (act && bump) {  // fused with the append: the active beams' new token
      len += 1;
      lens[(int64_t)g.req * maxB + g.beam0 + tid] = len;
    }
    s_len[tid] = len;
  }
  __syncthreads();
  // the group's table rows -> smem, all loads in flight before any store
  const int n = nb * npg;
  for (int b0 = tid; b0 < n; b0 += 8 * NT) {
    int v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int idx = b0 + k * NT;
      v[k] = -1;
      if (idx < n) {
        const int b = idx / npg, i = idx % npg;
        if (i * kP < s_len[b]) v[k] = tables[((int64_t)g.req * maxB + g.beam0 + b) * maxP + i];
      }
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int idx = b0 + k * NT;
      if (idx < n) tb[(idx / npg) * ld + idx % npg] = v[k];
    }
  }
  __syncthreads();
  int4* out = items + g.pad[0];
  // warp w owns the contiguous positions [i_lo, i_hi): pass 1 counts its runs,
  // one block scan turns counts into offsets, pass 2 writes the items
  const int ppw = (npg + NW - 1) / NW;
  const int i_lo = min(npg, warp * ppw), i_hi = min(npg, i_lo + ppw);
  auto runs_at = [&](int i, uint32_t& hm, int& page) -> uint32_t {
    const bool has = lane < nb && tb[lane * ld + i] >= 0;
    page = has ? tb[lane * ld + i] : -1;
    hm = __ballot_sync(0xffffffffu, has);
    const uint32_t below = hm & ((1u << lane) - 1u);
    const int prev = below ? 31 - __clz(below) : lane;
    const int pp = __shfl_sync(0xffffffffu, page, prev);
    return __ballot_sync(0xffffffffu, has && (below == 0 || pp != page));
  };
  int cnt = 0;
  for (int i = i_lo; i < i_hi; ++i) {
    uint32_t hm;
    int page;
    cnt += __popc(runs_at(i, hm, page));
  }
  if (lane == 0) s_cnt[warp] = cnt;
  __syncthreads();
  if (warp == 0) {
    const int c = lane < NW ? s_cnt[lane] : 0;
    int x = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    s_off[lane] = x - c;
    if (lane == 31) s_tot = x;
  }
  __syncthreads();
  int base = s_off[warp];
  for (int i = i_lo; i < i_hi; ++i) {
    uint32_t hm;
    int page;
    const uint32_t sm = runs_at(i, hm, page);
    // the run starting at lane `lane` covers the has-lanes up to the next run start
    if ((sm >> lane) & 1u) {
      const uint32_t after = sm & ~((2u << lane) - 1u);
      const int s1 = after ? __ffs(after) - 1 : 32;
      const uint32_t members = hm & (s1 >= 32 ? 0xffffffffu : ((1u << s1) - 1u)) & ~((1u << lane) - 1u);
      const int rank = __popc(sm & ((1u << lane) - 1u));
      out[base + rank] = make_int4(page, (int)members, min(kP, s_len[lane] - i * kP), i);
    }
    base += __popc(sm);
  }
  if (tid == 0) counts[gi] = s_tot;
}

__global__ void __launch_bounds__(1024) k_plan(const int32_t* __restrict__ tables, int32_t* __restrict__ lens,
                                              const GroupDesc* __restrict__ groups, int4* __restrict__ items,
                                              int32_t* __restrict__ counts, const int32_t* status, int maxB,
                                              int maxP) {
  extern __shared__ int32_t tb[];  // [nbeams][npg + 1]
  if (*(volatile const int32_t*)status) return;
  plan_group<1024>(groups[blockIdx.x], blockIdx.x, tables, lens, items, counts, maxB, maxP, tb, false);
}

// a2 + a3 fused (tts_decode_step): blocks [0, n_slots) append one token of one
// beam for every layer (slot item = call, req, beam, pos), blocks [n_slots,
// n_slots + n_groups) build the attention plan and advance the lengths of the
// group's active beams (each beam belongs to exactly one group).  The plan
// reads only block tables (pages were allocated before this launch) and the
// pre-append lengths, so the two roles are independent.
struct AppendPlanParams {
  __nv_bfloat16* k_pool;
  __nv_bfloat16* v_pool;
  const int32_t* tables;
  int32_t* lens;
  const int4* slots;
  int n_slots, n_call;
  const uint4* k_new;
  const uint4* v_new;
  const GroupDesc* groups;
  int4* items;
  int32_t* counts;
  const int32_t* status;
  int32_t* status_w;
  int L, Hkv, d, maxB, maxP;
  int64_t num_pages;
};

__global__ void __launch_bounds__(256) k_append_plan(AppendPlanParams p) {
  extern __shared__ int32_t tb[];
  if (*(volatile const int32_t*)p.status) return;
  if ((int)blockIdx.x >= p.n_slots) {
    const int gi = blockIdx.x - p.n_slots;
    plan_group<256>(p.groups[gi], gi, p.tables, p.lens, p.items, p.counts, p.maxB, p.maxP, tb, true);
    return;
  }
  const int4 it = p.slots[blockIdx.x];
  const int call = it.x, req = it.y, beam = it.z, pos = it.w;
  const int vpr = p.d / 8;  // 16-B vectors per (token, kv head) row
  const int n = p.Hkv * vpr;
  const int rows = (pos % kP == 0) ? kP : 1;  // fresh page: write slot 0, zero slots 1..P-1
  const int total = p.L * n * rows;
  const int32_t page = p.tables[((int64_t)req * p.maxB + beam) * p.maxP + pos / kP];
  // all layers at once: 4 independent 16-B copies in flight per thread
  for (int i0 = threadIdx.x; i0 < total; i0 += 4 * (int)blockDim.x) {
    uint4 kv[4], vv[4];
    int64_t dst[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = i0 + u * (int)blockDim.x;
      if (i < total) {
        const int so = i / (p.L * n), rest = i % (p.L * n);
        const int l = rest / n, r2 = rest % n, kh = r2 / vpr, e = r2 % vpr;
        dst[u] = ((((int64_t)l * p.num_pages + page) * p.Hkv + kh) * kP + pos % kP + so) * vpr + e;
        if (so == 0) {
          const int64_t src = ((((int64_t)l * p.n_call + call) * p.maxB + beam) * p.Hkv + kh) * vpr + e;
          kv[u] = p.k_new[src];
          vv[u] = p.v_new[src];
        } else {
          kv[u] = vv[u] = make_uint4(0, 0, 0, 0);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = i0 + u * (int)blockDim.x;
      if (i < total) {
        reinterpret_cast<uint4*>(p.k_pool)[dst[u]] = kv[u];
        reinterpret_cast<uint4*>(p.v_pool)[dst[u]] = i < p.L * n ? v_to_pool(vv[u], p.status_w) : vv[u];
      }
    }
  }
}

// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads, 2)
    k_tree_umma(const __grid_constant__ CUtensorMap tmk, const __grid_constant__ CUtensorMap tmv, UParams p) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = su32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* bp = smem_raw + (base - raw);
  int4* meta = reinterpret_cast<int4*>(bp + kOffMeta);
  uint64_t* bars = reinterpret_cast<uint64_t*>(bp + kOffBar);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + kNumBars);
  float* m_s = reinterpret_cast<float*>(bp + kOffML);
  float* l_s = m_s + kRows;
  const uint32_t b_full = su32(bars), b_empty = b_full + 8 * kNS, b_sfull = b_empty + 8 * kNS,
                 b_pfull = b_sfull + 16, b_pv = b_pfull + 16;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) TTS_TR(1023, 0);  // CTA start
  if (*(volatile int32_t*)p.status) return;
  const int split = blockIdx.x % p.splits;
  const int gidx = blockIdx.x / p.splits;
  const GroupDesc g = p.groups[gidx];
  const int kh = blockIdx.y, lrel = blockIdx.z, layer = p.layer_begin + lrel;
  const int G = p.G;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kNS; ++i) {
      bar_init(b_full + 8 * i, 1);
      bar_init(b_empty + 8 * i, 1);
    }
    for (int i = 0; i < 2; ++i) {
      bar_init(b_sfull + 8 * i, 1);
      bar_init(b_pfull + 8 * i, 4);
      bar_init(b_pv + 8 * i, 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 5) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // rows of the tile: r -> (beam g.beam0 + r / G, q head kh*G + r % G)
  const int r = threadIdx.x;
  const int rbl = r / G;
  const bool rvalid = warp < 4 && rbl < g.nbeams && ((g.active >> rbl) & 1u);
  uint32_t qv[64];  // this thread's query row (bf16 pairs), loaded before the TMEM handshake
  if (warp < 4) {
    const uint4* src = reinterpret_cast<const uint4*>(
        p.q + ((((int64_t)lrel * p.n_call + g.call_idx) * p.maxB + g.beam0 + (rvalid ? rbl : 0)) * p.Hq + kh * G +
               r % G) * kD);
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      const uint4 v = rvalid ? src[c] : make_uint4(0, 0, 0, 0);
      qv[4 * c] = v.x;
      qv[4 * c + 1] = v.y;
      qv[4 * c + 2] = v.z;
      qv[4 * c + 3] = v.w;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t t_o = tmem, t_q = tmem + 128, t_s = tmem + 192;
  if (warp < 4) {
    // Q tile -> TMEM (the A operand of S = Q K^T): lane = row, column = d pair
    const uint32_t lo = (uint32_t)(warp * 32) << 16;
    uint32_t h0[32], h1[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      h0[i] = qv[i];
      h1[i] = qv[32 + i];
    }
    tc_st32(t_q + lo, h0);
    tc_st32(t_q + lo + 32, h1);
    tc_wait_st();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  // this CTA's slice of the group's page list: units [u0, u1)
  if (threadIdx.x == 0) TTS_TR(1023, 1);  // prologue done (Q in TMEM)
  const int n_items = p.counts[gidx];
  const int n_units = (n_items + kU - 1) / kU;
  const int u0 = (int)((int64_t)split * n_units / p.splits);
  const int u1 = (int)((int64_t)(split + 1) * n_units / p.splits);
  const int4* items = p.items + g.pad[0];

  if (warp == 4) {
    // ============================ producer ============================
    const int64_t layer_rows = ((int64_t)layer * p.num_pages) * p.Hkv;
    int slot = 0;
    uint32_t ph = 0;
    for (int ub = u0; ub < u1; ub += 32 / kU) {
      const int it = ub * kU + lane;
      const int4 my = (it < min(u1 * kU, n_items)) ? items[it] : make_int4(-2, 0, 0, 0);
      const int ue = min(u1, ub + 32 / kU);
      for (int u = ub; u < ue; ++u) {
        int4 m[kU];
#pragma unroll
        for (int k = 0; k < kU; ++k) {
          const int src = (u - ub) * kU + k;
          m[k].x = __shfl_sync(0xffffffffu, my.x, src);
          m[k].y = __shfl_sync(0xffffffffu, my.y, src);
          m[k].z = __shfl_sync(0xffffffffu, my.z, src);
          m[k].w = __shfl_sync(0xffffffffu, my.w, src);
        }
        if (lane == 0) {
          bar_wait(b_empty + 8 * slot, ph ^ 1u);
          int npages = 0;
#pragma unroll
          for (int k = 0; k < kU; ++k) {
            meta[slot * kU + k] = m[k];
            npages += m[k].x >= 0;
          }
          const uint32_t fb = b_full + 8 * slot;
          bar_expect(fb, (uint32_t)(npages * 2 * kTile));
          const uint32_t sb = base + kOffRing + slot * kSlot;
#pragma unroll
          for (int k = 0; k < kU; ++k) {
            if (m[k].x < 0) continue;
            const int y = (int)((layer_rows + (int64_t)m[k].x * p.Hkv + kh) * kP);
            tma3d(sb + k * kTile, &tmk, 0, y, 0, fb);
            tma3d(sb + (kU + k) * kTile, &tmv, 0, y, 0, fb);
          }
        }
        if (++slot == kNS) {
          slot = 0;
          ph ^= 1u;
        }
      }
    }
    if (lane == 0) {
      bar_wait(b_empty + 8 * slot, ph ^ 1u);
      meta[slot * kU] = make_int4(-1, 0, 0, 0);
      bar_arrive(b_full + 8 * slot);
    }
  } else if (warp == 5) {
    // ============================ MMA issuer ============================
    // The whole warp runs the loop so that descriptors stay warp-uniform; one
    // elected lane issues the tcgen05 instructions.
    constexpr uint32_t id_s = idesc_bf16(kRows, kP, false);
    constexpr uint32_t id_pv = idesc_f16(kRows, kD, true);
    const uint64_t dk0 = sdesc(base + kOffRing, 16, 1024, 2);    // K tiles: K-major SW128
    const uint64_t dv0 = sdesc(base + kOffRing, 2048, 1024, 2);  // V tiles: MN-major SW128
    auto issue_s = [&](int j) {
      const int slot = j % kNS;
      const bool e = elect_one();
#pragma unroll
      for (int k = 0; k < kU; ++k) {
        if (meta[slot * kU + k].x < 0) continue;
        const uint32_t sd = t_s + (j & 1) * kSCols + k * kP;
        const uint64_t dk = dk0 + (uint64_t)((slot * kSlot + k * kTile) >> 4);
        if (e) {
#pragma unroll
          for (int ks = 0; ks < kD / 16; ++ks)
            mma_ts(sd, t_q + ks * 8, dk + (uint64_t)(((ks >> 2) * 2048 + (ks & 3) * 32) >> 4), id_s, ks > 0);
        }
      }
      if (e) tc_commit(b_sfull + 8 * (j & 1));
      __syncwarp();
    };
    bar_wait(b_full, 0);
    tc_fence_after();
    bool done = meta[0].x == -1;
    if (done) {
      if (elect_one()) bar_arrive(b_sfull);
      __syncwarp();
    } else {
      issue_s(0);
    }
    uint32_t acc = 0;
    for (int j = 0; !done; ++j) {
      const int sn = (j + 1) % kNS;
      if (lane == 0) TTS_TR(j, 0);
      bar_wait(b_full + 8 * sn, ((j + 1) / kNS) & 1u);
      if (lane == 0) TTS_TR(j, 1);
      tc_fence_after();
      const bool last = meta[sn * kU].x == -1;
      if (last) {
        if (elect_one()) bar_arrive(b_sfull + 8 * ((j + 1) & 1));
        __syncwarp();
      } else {
        issue_s(j + 1);
      }
      bar_wait(b_pfull + 8 * (j & 1), (j >> 1) & 1u);
      if (lane == 0) TTS_TR(j, 2);
      const int slot = j % kNS;
      tc_fence_after();
      const uint32_t pa = t_s + (j & 1) * kSCols;
      const bool e = elect_one();
#pragma unroll
      for (int k = 0; k < kU; ++k) {
        if (meta[slot * kU + k].x < 0) continue;
        const uint64_t dv = dv0 + (uint64_t)((slot * kSlot + (kU + k) * kTile) >> 4);
        if (e) {
          mma_ts(t_o, pa + k * (kP / 2), dv, id_pv, acc);
        }
        acc = 1;
      }
      if (e) {
        tc_commit(b_empty + 8 * slot);
        tc_commit(b_pv + 8 * (j & 1));
        TTS_TR(j, 3);
      }
      __syncwarp();
      done = last;
    }
  } else {
    // ============================ softmax (warps 0-3) ============================
    const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
    float m_ref = -1e30f, l = 0.f;
    int j = 0;
    for (;; ++j) {
      if (r == 0) TTS_TR(j, 4);
      bar_wait(b_sfull + 8 * (j & 1), (j >> 1) & 1u);
      if (r == 0) TTS_TR(j, 5);
      tc_fence_after();
      const int slot = j % kNS;
      int4 mt[kU];
#pragma unroll
      for (int k = 0; k < kU; ++k) mt[k] = meta[slot * kU + k];
      if (mt[0].x == -1) break;
      // warp-uniform page membership: a warp none of whose rows reads a page
      // skips its exponentials (P = 0 there); most private pages touch 1 warp
      bool mem[kU], wm[kU];
#pragma unroll
      for (int k = 0; k < kU; ++k) {
        mem[k] = mt[k].x >= 0 && rvalid && ((((uint32_t)mt[k].y) >> rbl) & 1u);
        wm[k] = __any_sync(0xffffffffu, mem[k]);
      }
      uint32_t ph16[kSCols / 2];
      if (r == 0) TTS_TR2(j, 0);
#ifdef TTS_TRACE
      if (r == 0 && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 10 && j < 1024) g_trace2[j][7] = 0;
#endif
      if (wm[0] || wm[1]) {
        uint32_t sr[kSCols];
        tc_ld32(t_s + lane_off + (j & 1) * kSCols, sr);
        tc_wait_ld();
        if (r == 0) TTS_TR2(j, 1);
        // raw scores (scale > 0 commutes with max).  Rows not reading page k are
        // masked once per page (row max -> -inf, exponent offset -> -inf, so
        // their P is exactly 0); token slots >= ntok only on a partial page.
        float v[kSCols];
#pragma unroll
        for (int i = 0; i < kSCols; ++i) v[i] = __uint_as_float(sr[i]);
        float mk[kU];
#pragma unroll
        for (int k = 0; k < kU; ++k) {
          if (mt[k].x >= 0 && mt[k].z < kP) {
#pragma unroll
            for (int c = 0; c < kP; ++c)
              if (c >= mt[k].z) v[k * kP + c] = -INFINITY;
          }
          const float* w = v + k * kP;
          const float t0 = fmax3(w[0], w[1], w[2]), t1 = fmax3(w[3], w[4], w[5]), t2 = fmax3(w[6], w[7], w[8]);
          const float t3 = fmax3(w[9], w[10], w[11]), t4 = fmax3(w[12], w[13], w[14]);
          const float mxk = fmax3(fmax3(t0, t1, t2), t3, fmax3(t4, w[15], -INFINITY));
          mk[k] = mem[k] ? mxk : -INFINITY;
        }
        const float mx = fmaxf(mk[0], mk[1]) * p.scale_log2;
        const bool need = mx > m_ref + 8.0f;
        if (r == 0) TTS_TR2(j, 2);
        if (__any_sync(0xffffffffu, need) && j > 0) {
          if (r == 0) TTS_TR2(j, 7);
          // every earlier PV product must have landed before O is rescaled in TMEM
          bar_wait(b_pv + 8 * ((j - 1) & 1), ((j - 1) >> 1) & 1u);
          tc_fence_after();
          const float alpha = need ? exp2f(m_ref - mx) : 1.f;
#pragma unroll 1
          for (int ch = 0; ch < 4; ++ch) {
            uint32_t o[32];
            tc_ld32(t_o + lane_off + ch * 32, o);
            tc_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
            tc_st32(t_o + lane_off + ch * 32, o);
          }
          tc_wait_st();
          l *= alpha;
        }
        if (need) m_ref = mx;
        const float2 sc2 = make_float2(p.scale_log2, p.scale_log2);
        float2 lacc = make_float2(0.f, 0.f);
#pragma unroll
        for (int k = 0; k < kU; ++k) {
          if (wm[k]) {
            const float nm = mem[k] ? -m_ref : -INFINITY;
            const float2 nm2 = make_float2(nm, nm);
#pragma unroll
            for (int c = 0; c < kP; c += 2) {
              const float2 x = ffma2(make_float2(v[k * kP + c], v[k * kP + c + 1]), sc2, nm2);
#ifdef TTS_NOEXP
              const float a = x.x * 0.5f, b = x.y * 0.5f;
#else
              const float a = ex2(x.x), b = ex2(x.y);
#endif
              lacc = fadd2(lacc, make_float2(a, b));
              ph16[(k * kP + c) / 2] = pack_f16x2(a, b);
            }
          } else {
#pragma unroll
            for (int c = 0; c < kP; c += 2) ph16[(k * kP + c) / 2] = 0u;
          }
        }
        l += lacc.x + lacc.y;
        if (r == 0) TTS_TR2(j, 3);
      } else {
#pragma unroll
        for (int i = 0; i < kSCols / 2; ++i) ph16[i] = 0u;
      }
      // P (fp16) overwrites this unit's first 16 S columns: page k at +8k
      tc_st16(t_s + lane_off + (j & 1) * kSCols, ph16);
      tc_wait_st();
      if (r == 0) TTS_TR2(j, 4);
      tc_fence_before();
      __syncwarp();
      if (r == 0) TTS_TR(j, 6);
      if (lane == 0) bar_arrive(b_pfull + 8 * (j & 1));
    }
    const int n_done = j;
    // ---------------- epilogue ----------------
    if (n_done > 0) {
      bar_wait(b_pv + 8 * ((n_done - 1) & 1), ((n_done - 1) >> 1) & 1u);
      tc_fence_after();
    }
    if (p.splits == 1) {
      if (n_done > 0) {
        const float inv = 1.f / l;
        float* orow = p.out + ((((int64_t)lrel * p.n_call + g.call_idx) * p.maxB + g.beam0 + rbl) * p.Hq +
                               kh * G + r % G) * kD;
#pragma unroll 1
        for (int ch = 0; ch < 4; ++ch) {
          uint32_t o[32];
          tc_ld32(t_o + lane_off + ch * 32, o);
          tc_wait_ld();
          if (rvalid) {
#pragma unroll
            for (int i = 0; i < 32; i += 4)
              *reinterpret_cast<float4*>(orow + ch * 32 + i) =
                  make_float4(__uint_as_float(o[i]) * inv, __uint_as_float(o[i + 1]) * inv,
                              __uint_as_float(o[i + 2]) * inv, __uint_as_float(o[i + 3]) * inv);
          }
        }
      }
    } else {
      // partial state -> smem (16-B chunks swizzled by row), merged across the cluster
      float* op = reinterpret_cast<float*>(bp + kOffRing);
#pragma unroll 1
      for (int ch = 0; ch < 4; ++ch) {
        uint32_t o[32];
        if (n_done > 0) {
          tc_ld32(t_o + lane_off + ch * 32, o);
          tc_wait_ld();
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) o[i] = 0u;
        }
#pragma unroll
        for (int q4 = 0; q4 < 8; ++q4) {
          const int c = ch * 8 + q4;
          const int pc = (c & ~7) | ((c & 7) ^ (r & 7));
          *reinterpret_cast<uint4*>(op + r * kD + pc * 4) =
              make_uint4(o[4 * q4], o[4 * q4 + 1], o[4 * q4 + 2], o[4 * q4 + 3]);
        }
      }
      m_s[r] = m_ref;
      l_s[r] = l;
    }
  }

  if (threadIdx.x == 0) TTS_TR(1023, 2);  // unit loop done
  if (p.splits > 1) {
    cluster_sync();
    if (warp < 4) {
      const int S = p.splits;
      const int rpc = kRows / S;
      const int tpr = 128 / rpc;
      const int row = split * rpc + threadIdx.x / tpr;
      const int cseg = threadIdx.x % tpr;
      const int cw = kD / tpr;
      const int bl = row / G;
      const bool ok = bl < g.nbeams && ((g.active >> bl) & 1u);
      const uint32_t lm = su32(m_s + row), ll = su32(l_s + row);
      // all remote loads of a step are issued before any is consumed (DSMEM
      // latency ~200 cycles; dependent loads would serialise)
      float mk[8], lk[8], wk[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        mk[k] = k < S ? ld_dsmem_f32(mapa(lm, k)) : -INFINITY;
        lk[k] = k < S ? ld_dsmem_f32(mapa(ll, k)) : 0.f;
      }
      float M = -INFINITY;
#pragma unroll
      for (int k = 0; k < 8; ++k) M = fmaxf(M, mk[k]);
      float L = 0.f;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        wk[k] = k < S ? exp2f(mk[k] - M) : 0.f;
        L += wk[k] * lk[k];
      }
      const float inv = 1.f / L;
      float* orow = p.out + ((((int64_t)lrel * p.n_call + g.call_idx) * p.maxB + g.beam0 + bl) * p.Hq +
                             kh * G + row % G) * kD;
      for (int c4 = 0; c4 < cw / 4; ++c4) {
        const int c = cseg * (cw / 4) + c4;
        const int pc = (c & ~7) | ((c & 7) ^ (row & 7));
        const uint32_t la = base + kOffRing + (uint32_t)(row * kD + pc * 4) * 4;
        float4 v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = k < S ? ld_dsmem_f32x4(mapa(la, k)) : make_float4(0.f, 0.f, 0.f, 0.f);
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          acc.x += wk[k] * v[k].x;
          acc.y += wk[k] * v[k].y;
          acc.z += wk[k] * v[k].z;
          acc.w += wk[k] * v[k].w;
        }
        if (ok) *reinterpret_cast<float4*>(orow + c * 4) = make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
      }
    }
    cluster_sync();
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) TTS_TR(1023, 3);  // epilogue / merge done
  if (warp == 5) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
  }
}

}  // namespace

#ifdef TTS_TRACE
extern "C" int tts_debug_read_trace(long long* out_h) {
  int e = (int)cudaMemcpyFromSymbol(out_h, g_trace, sizeof(g_trace));
  return e ? e : (int)cudaMemcpyFromSymbol(out_h + 1024 * 8, g_trace2, sizeof(g_trace2));
}
#endif

bool umma_supported(const Ctx* c) {
  const int G = c->cfg.num_q_heads / c->cfg.num_kv_heads;
  return c->cfg.head_dim == kD && c->cfg.page_size == kP && G >= 4 && G <= 16 && c->tmap3_ok;
}

int umma_max_beams(const Ctx* c) {
  const int G = c->cfg.num_q_heads / c->cfg.num_kv_heads;
  return std::min(32, kRows / G);
}

cudaError_t launch_plan(Ctx* c, const GroupDesc* groups_d, int n_groups, int max_npages, int max_nbeams,
                        cudaStream_t st) {
  const int smem = max_nbeams * (max_npages + 1) * 4;
  static int smem_set = 0;
  if (smem > smem_set) {
    cudaError_t e = cudaFuncSetAttribute(k_plan, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e != cudaSuccess) return e;
    smem_set = 200 * 1024;
  }
  if (smem > 200 * 1024) return cudaErrorInvalidValue;
  k_plan<<<n_groups, 1024, smem, st>>>(c->buf.block_tables, c->buf.seq_lens, groups_d, c->ws_items, c->ws_counts,
                                       c->buf.status, c->cfg.max_beams, c->cfg.max_pages_per_beam);
  c->launches++;
  return cudaGetLastError();
}

cudaError_t launch_append_plan(Ctx* c, const int32_t* slots_d, int n_slots, int n_call, const __nv_bfloat16* k,
                               const __nv_bfloat16* v, const GroupDesc* groups_d, int n_groups, int max_npages,
                               int max_nbeams, cudaStream_t st) {
  const int smem = max_nbeams * (max_npages + 1) * 4;
  static int smem_set = 0;
  if (smem > smem_set) {
    cudaError_t e = cudaFuncSetAttribute(k_append_plan, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e != cudaSuccess) return e;
    smem_set = 200 * 1024;
  }
  if (smem > 200 * 1024) return cudaErrorInvalidValue;
  AppendPlanParams p;
  p.k_pool = (__nv_bfloat16*)c->buf.k_pool;
  p.v_pool = (__nv_bfloat16*)c->buf.v_pool;
  p.tables = c->buf.block_tables;
  p.lens = c->buf.seq_lens;
  p.slots = (const int4*)slots_d;
  p.n_slots = n_slots;
  p.n_call = n_call;
  p.k_new = (const uint4*)k;
  p.v_new = (const uint4*)v;
  p.groups = groups_d;
  p.items = c->ws_items;
  p.counts = c->ws_counts;
  p.status = c->buf.status;
  p.status_w = c->buf.status;
  p.L = c->cfg.num_layers;
  p.Hkv = c->cfg.num_kv_heads;
  p.d = c->cfg.head_dim;
  p.maxB = c->cfg.max_beams;
  p.maxP = c->cfg.max_pages_per_beam;
  p.num_pages = c->cfg.num_pages;
  k_append_plan<<<n_slots + n_groups, 256, smem, st>>>(p);
  c->launches++;
  return cudaGetLastError();
}

cudaError_t launch_attention_umma(Ctx* c, const GroupDesc* groups_d, int n_groups, int splits, int layer_begin,
                                  int n_layers, int n_call, const __nv_bfloat16* q, float scale, float* out,
                                  cudaStream_t st) {
  UParams p;
  p.lens = c->buf.seq_lens;
  p.q = q;
  p.out = out;
  p.groups = groups_d;
  p.items = c->ws_items;
  p.counts = c->ws_counts;
  p.status = c->buf.status;
  p.layer_begin = layer_begin;
  p.n_call = n_call;
  p.Hq = c->cfg.num_q_heads;
  p.Hkv = c->cfg.num_kv_heads;
  p.G = p.Hq / p.Hkv;
  p.maxB = c->cfg.max_beams;
  p.splits = splits;
  p.num_pages = c->cfg.num_pages;
  p.scale_log2 = scale * 1.4426950408889634f;
  static bool attr_done = false;
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(k_tree_umma, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
    if (e != cudaSuccess) return e;
    attr_done = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(n_groups * splits, p.Hkv, n_layers);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmemBytes;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = splits;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, k_tree_umma, c->tmap3_k, c->tmap3_v, p);
  c->launches++;
  return e;
}

}  // namespace tts
