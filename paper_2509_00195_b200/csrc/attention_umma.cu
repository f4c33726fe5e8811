// Prefix-shared tree decode attention on the 5th-generation tensor cores
// (tcgen05 + TMEM + TMA), sm_100a.  Same contract as attention.cu (see there
// and include/tts.h); this is the path for head_dim 128 and 4 <= G <= 16.
//
// Two launches per call, chained by programmatic dependent launch:
// k_plan      a2 (tts_decode_step): the call's new token of each active beam
//             -> slot (len-1) % P of the beam's last page (V converted to the
//             pool's fp16; a fresh page's other slots zeroed).  The last page
//             of a beam is private to it (eager copy-on-write).
//             a3 (plan): per beam group -- a run of consecutive beams of one
//             request in DFS order, so that every shared page's beams are
//             adjacent (ledger C5) -- the ordered list of its
//             DISTINCT pages, each with its member-beam bitmask and valid-token
//             count.
// k_tree_umma a4 (+ a5): persistent, one CTA per SM (512 TMEM columns).  A
//             tile is (group, kv head, layer): the group's beams x the G query
//             heads of the kv head, <= 128 rows, against the group's page list.
//             Whole tiles round-robin first, then the rest split over all CTAs
//             (stream-K) and merged through a global partial buffer.
// Per unit of eight pages (128 tokens, 64 KiB of K + V):
//   K producer warp   TMA (two 16 x 64 bf16 half tiles per page, SWIZZLE_128B) -> K ring (3 units)
//   V producer warp   TMA (one 16 x 128 fp16 tile per page) -> V ring (3 units)
//   S warp            S[128 x 128] = Q . K^T   8 x tcgen05.mma kind::f16 (Q in smem), S in TMEM
//   softmax warps     8 warps, two per TMEM lane quadrant (one row per thread), each
//                     the S columns of four pages: tcgen05.ld S; mask rows whose beam
//                     does not reference the page and token slots >= ntok; fp32
//                     online softmax with lazy rescale (O rescaled in TMEM only when
//                     the running max grows by > 2^8; the two halves of a row
//                     exchange their maxima through shared memory); P in fp16 ->
//                     tcgen05.st over S
//   PV warp           O[128 x 128] += P . V   fp16 x fp16 (A from TMEM; V is kept in
//                     fp16 in the pool, MN-major operand; ledger C14)
// Three S/P buffers in TMEM keep three units between S = Q K^T and O += P V.
// Each distinct page is fetched once per tile and multiplied against all its
// rows: every GQA head and every beam of the tile that references it.
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "sm100.cuh"
#include "tts_internal.cuh"

namespace tts {
namespace {
using namespace sm100;

constexpr int kP = 16;
constexpr int kD = 128;
constexpr int kRows = 128;
constexpr int kU = 8;                        // pages per unit (128 tokens: S is 128 x 128)
constexpr int kTile = kP * kD * 2;           // 4 KiB: one (page, kv head) K or V tile
constexpr int kKSlot = kU * kTile;           // 32 KiB: K of a unit, [d half][page][16 tokens][128 B]
constexpr int kVSlot = kU * kTile;           // 32 KiB: V of a unit, [page][d half][16 tokens][128 B]
constexpr int kNK = 3;                       // K ring slots (released when S = Q K^T has completed)
constexpr int kNV = 3;                       // V ring slots (released when O += P V has completed)
#ifndef TTS_PF
#define TTS_PF 0
#endif
constexpr int kPF = TTS_PF;                  // L2 prefetch distance of the producers (units)
constexpr int kNM = 6;                       // unit metadata ring (>= kNK + kNSB: see the K producer)
constexpr int kUH = kU / 2;                  // pages per softmax warp half
constexpr int kThreads = 384;                // warps 0-7 softmax, 8 K producer, 9 V producer, 10 S issuer, 11 PV issuer
constexpr int kSoftmaxWarps = 8;
constexpr int kTmemCols = 512;               // O [0,128), S/P buffers [128,256), [256,384), [384,512)
constexpr int kNSB = 3;                      // S buffers (P overwrites S; a buffer is free once PV has read P)
constexpr int kSCols = kU * kP;              // 128
constexpr int kTS = 128;                     // first S buffer column

constexpr int kMaxGroups = 1024;             // beam groups per call (smem prefix of their unit counts)
constexpr int kOffK = 0;
constexpr int kOffV = kOffK + kNK * kKSlot;
constexpr int kOffQ = kOffV + kNV * kVSlot;  // Q of the piece: [d half][128 rows][128 B], SWIZZLE_128B (A of S = Q K^T)
constexpr int kOffMeta = kOffQ + kRows * kD * 2;
constexpr int kOffBar = kOffMeta + kNM * kU * 16;
// kfull[kNK], kempty[kNK], vfull[kNV], vempty[kNV], sfull[2], pfull[2], pv[2], qready, ofree, qtaken
// kfull[kNK], kempty[kNK], vfull[kNV], vempty[kNV], sfull[kNSB], pfull[kNSB], pv[kNSB], qready, ofree, qtaken
constexpr int kNumBars = 2 * kNK + 2 * kNV + 3 * kNSB + 3;
constexpr int kOffXm = (kOffBar + kNumBars * 8 + 16 + 15) / 16 * 16;  // row max exchange [2 units][2 halves][128]
constexpr int kOffInfo = kOffXm + 4 * kRows * 4;
// The dynamic shared memory starts 1024-B aligned (the kernel has no static
// shared memory; checked at run time): no alignment slack
constexpr int kSmemBytes = kOffInfo + 16;
// one CTA per SM (the 512 TMEM columns), and at most one: the plan
// double-buffer argument (umma_prepare) needs the next call's CTAs to become
// resident only after this call's have exited
static_assert(kSmemBytes <= 227 * 1024, "shared memory per CTA");
static_assert(2 * (kSmemBytes + 1024) > 228 * 1024, "at most one CTA per SM (plan double-buffer argument)");
static_assert(kOffMeta % 16 == 0 && kOffBar % 8 == 0 && kOffXm % 16 == 0 && kOffQ % 1024 == 0, "shared-memory alignment");
static_assert(kNM >= kNK + kNSB, "metadata ring reuse distance");
static_assert(kOffV % 1024 == 0 && kKSlot % 1024 == 0, "SWIZZLE_128B atoms");

// Device-side bounds checks of the schedule's indices (compute-sanitizer is not
// available on the GPU pool): -DTTS_CHECK builds trap on a violation.
#ifdef TTS_CHECK
#define TTS_ASSERT(c)                                                                      \
  do {                                                                                     \
    if (!(c)) {                                                                            \
      printf("TTS_ASSERT %s failed (line %d, block %d, thread %d)\n", #c, __LINE__, (int)blockIdx.x, \
             (int)threadIdx.x);                                                            \
      __trap();                                                                            \
    }                                                                                      \
  } while (0)
#else
#define TTS_ASSERT(c) \
  do {                \
  } while (0)
#endif

#ifdef TTS_PROF
// per CTA (last launch) x warp: accumulated cycles [0..5] + counters (tools/prof.py)
__device__ long long g_prof[512][12][16];
#define PROF_DECL long long pf_[16] = {}; long long pf_t = clock64()
#define PROF_MARK(k)                   \
  do {                                 \
    const long long t_ = clock64();    \
    pf_[(k)] += t_ - pf_t;             \
    pf_t = t_;                         \
  } while (0)
#define PROF_CNT(k) (pf_[(k)] += 1)
#define PROF_FLUSH(w)                                                   \
  do {                                                                  \
    if (blockIdx.x < 512 && (threadIdx.x & 31) == 0)                    \
      for (int k_ = 0; k_ < 16; ++k_) g_prof[blockIdx.x][(w)][k_] = pf_[k_]; \
  } while (0)
#else
#define PROF_DECL
#define PROF_MARK(k) do {} while (0)
#define PROF_CNT(k) do {} while (0)
#define PROF_FLUSH(w) do {} while (0)
#endif

#ifdef TTS_TRACE
__device__ long long g_trace[1024][8];
__device__ long long g_trace2[1024][8];
__device__ long long g_cta[4096][4];  // per CTA of the last launch: globaltimer at start / after the plan wait / exit, units | smid << 32
// per call (launch id % 32768): [0] first attention CTA start, [1] last attention CTA exit,
// [2] first k_plan block start, [3] last k_plan block exit (globaltimer; min/max by atomics)
__device__ unsigned long long g_lspan[32768][4];
#define TTS_SPAN(id, k, v, op) op(&g_lspan[(id) & 32767][(k)], (unsigned long long)(v))
__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define TTS_CTA(ev, v)                                                                          \
  do {                                                                                          \
    const int id_ = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);             \
    if (id_ < 4096) g_cta[id_][(ev)] = (v);                                                    \
  } while (0)
#define TTS_TR(j, ev)                                                                   \
  do {                                                                                  \
    if (blockIdx.x == 10 && (j) >= 0 && (j) < 1024) \
      g_trace[(j)][(ev)] = clock64();                                                   \
  } while (0)
#define TTS_TR2(j, ev)                                                                  \
  do {                                                                                  \
    if (blockIdx.x == 10 && (j) >= 0 && (j) < 1024) \
      g_trace2[(j)][(ev)] = clock64();                                                  \
  } while (0)
#else
#define TTS_CTA(ev, v) \
  do {                 \
  } while (0)
#define TTS_SPAN(id, k, v, op) \
  do {                         \
  } while (0)
#define TTS_TR(j, ev) \
  do {                \
  } while (0)
#define TTS_TR2(j, ev) \
  do {                 \
  } while (0)
#endif

struct UParams {
  const int4* items;          // per-group distinct-page lists (k_plan), group slice at (req * maxB + beam0) * maxP
  const int32_t* counts;      // items per group of the call (k_plan)
  const __nv_bfloat16* q;
  float* out;
  const GroupDesc* groups;    // device copies when the call does not fit the parameter block,
                              // else null (descriptors in UInline)
  int32_t* status;
  float* partial;             // [2 * gridDim.x][m 128 | l 128 | O 128 x 128]: split tiles' partial states
  int32_t* tile_cnt;          // [n_tiles] pieces of a split tile done (reset by its merger)
  int* pre;                   // [gridDim.x][kMaxGroups + 1] per-CTA scratch: prefix of units per group
  int layer_begin, n_layers, n_call, n_groups, Hq, Hkv, G, maxB, maxP;
  int round_robin;            // beam b of a group -> lane quadrant b % 4 (else blocks of consecutive beams)
  int split_partial_round;    // a last partial round of tiles goes through stream-K (else whole if >= 3/4 full)
  int l2hint;                 // 1: pages held outside the group loaded L2::evict_last, the rest evict_first
  int sched;                  // phase-1 tiles: 0 rotated in blocks of n_groups, 1 plain round-robin, 2 none (stream-K only)
  int64_t num_pages;
  float scale_log2;
  int launch_id;              // call counter (TTS_TRACE launch spans only)
};
constexpr int kPartFloats = 2 * kRows + kRows * kD;
constexpr int kMaxCtas = 2 * 160;  // partial-state slots are sized for this many CTAs

// The call's descriptors in the kernel parameter block (no H2D copy on the stream)
constexpr int kInlineGroups = 32;
constexpr int kInlineLens = 512;
struct UInline {
  GroupDesc g[kInlineGroups];
  int32_t len[kInlineLens];  // post-append length per group beam (0: inactive); GroupDesc.pad[0] = offset
};

// ---------------------------------------------------------------------------
// a2 + a3 for one call, ahead of the attention kernel (which it releases early
// through programmatic dependent launch).  Blocks [0, n_groups): the plan of
// group gi -- its ordered list of DISTINCT pages (item = page, member-beam
// mask, valid tokens, position; a run of adjacent beams holding the same page
// id is one item), one thread per page position, written to the group's slice
// of the items workspace, and the item count.  Blocks [n_groups, n_groups *
// (1 + n_layers)) (only when appending): the call's new K/V row of each active
// beam of one group for one layer and every kv head -> slot (len-1) % P of the
// beam's last page (V -> the pool's fp16); a fresh page's slots 1..P-1 zeroed.
struct PlanParams {
  int32_t* lens;
  const int32_t* refcounts;  // non-null (TTS_L2HINT): item.w = 1 when the page is also held outside the group
  const int32_t* tables;
  const GroupDesc* groups;  // device copies when the call does not fit the parameter block, else null
  const int32_t* glens;
  int32_t* status;
  const uint4* k_new;  // null: plan only (tts_prefix_attn_decode)
  const uint4* v_new;
  uint4* k_pool;
  uint4* v_pool;
  int4* items;
  int32_t* counts;
  int n_groups, layer_begin, n_call, Hkv, maxB, maxP;
  int64_t num_pages;
  int launch_id;  // call counter (TTS_TRACE launch spans only)
};
constexpr int kPlanThreads = 128;  // small enough to co-reside with the attention CTA of an SM
// attention registers per thread: leaves 64 per thread of a k_plan block on the SM
constexpr int kMaxRegs = (65536 - 64 * kPlanThreads) / kThreads / 8 * 8;
static_assert(kMaxRegs >= 128, "register budget");

__global__ void __launch_bounds__(kPlanThreads, 8) k_plan(PlanParams p, const __grid_constant__ UInline inl) {
  __shared__ int s_len[32];
  __shared__ int s_wsum[kPlanThreads / 32];
#ifdef TTS_TRACE
  if (threadIdx.x == 0) TTS_SPAN(p.launch_id, 2, gtimer(), atomicMin);
  struct SpanEnd {
    int id;
    __device__ ~SpanEnd() {
      if (threadIdx.x == 0) TTS_SPAN(id, 3, gtimer(), atomicMax);
    }
  } span_end_{p.launch_id};
#endif
  // Programmatic dependent launch: this grid may run while the previous call's
  // attention kernel still streams its pages.  Nothing here conflicts with it:
  // the plan goes to the other half of the double-buffered items workspace,
  // the new token lands in a slot the previous call masks (its P is exactly 0
  // and the pool never holds a non-finite V), and a fresh page (zero fill) only
  // exists after a k_alloc launch, which is ordered after the previous call.
  // The grid completes only after the previous kernel has (griddepcontrol.wait
  // at the end), so the attention kernel that waits on this grid also waits on
  // every earlier call.
  if (*(volatile int32_t*)p.status) {
    // sticky error: an empty plan, so that every CTA of the attention kernel
    // derives the same (empty) schedule from the counts alone
    if ((int)blockIdx.x < p.n_groups && threadIdx.x == 0) p.counts[blockIdx.x] = 0;
    __threadfence();
    if (blockIdx.x == 0 && threadIdx.x == 0) asm volatile("griddepcontrol.wait;" ::: "memory");
    return;
  }
  const bool plan = (int)blockIdx.x < p.n_groups;
  const int gi = plan ? blockIdx.x : (blockIdx.x - p.n_groups) % p.n_groups;
  const GroupDesc g = p.groups ? p.groups[gi] : inl.g[gi];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid < 32) {
    const bool on = tid < g.nbeams && ((g.active >> tid) & 1u);
    s_len[tid] = on ? (p.groups ? p.glens[g.pad[0] + tid] : inl.len[g.pad[0] + tid]) : 0;
  }
  __syncthreads();
  const int nb = g.nbeams;
  const int64_t row0 = (int64_t)g.req * p.maxB + g.beam0;
  const int32_t* trow = p.tables + row0 * p.maxP;
  if (!plan) {
    // the beams' last pages first, so that the copy loop below has only
    // independent loads (4 in flight per thread)
    __shared__ int s_page[32];
    if (tid < 32) s_page[tid] = (tid < nb && s_len[tid] > 0) ? trow[(int64_t)tid * p.maxP + (s_len[tid] - 1) / kP] : -1;
    __syncthreads();
    const int lrel = (blockIdx.x - p.n_groups) / p.n_groups;
    const int layer = p.layer_begin + lrel;
    const int64_t plane = (int64_t)layer * p.num_pages * p.Hkv;
    const int per_beam = p.Hkv * 16;
    const uint4* __restrict__ kn = p.k_new;
    const uint4* __restrict__ vn = p.v_new;
    constexpr int kBatch = 4;
    for (int w0 = tid; w0 < nb * per_beam; w0 += kBatch * kPlanThreads) {
      uint4 kv[kBatch], vv[kBatch];
      int64_t dst[kBatch];
#pragma unroll
      for (int i = 0; i < kBatch; ++i) {
        const int w = w0 + i * kPlanThreads;
        dst[i] = -1;
        if (w < nb * per_beam) {
          const int b = w / per_beam, rest = w % per_beam, kh = rest >> 4, e = rest & 15;
          const int page = s_page[b];
          if (page >= 0) {
            const int pos = s_len[b] - 1;
            dst[i] = ((plane + (int64_t)page * p.Hkv + kh) * kP + pos % kP) * 16 + e;
            const int64_t src = ((((int64_t)lrel * p.n_call + g.call_idx) * p.maxB + g.beam0 + b) * p.Hkv + kh) * 16 + e;
            kv[i] = __ldg(kn + src);
            vv[i] = __ldg(vn + src);
          }
        }
      }
#pragma unroll
      for (int i = 0; i < kBatch; ++i)
        if (dst[i] >= 0) {
          p.k_pool[dst[i]] = kv[i];
          p.v_pool[dst[i]] = v_to_pool(vv[i], p.status);
        }
    }
    // a fresh page (first token at slot 0): zero its slots 1..P-1 (a beam-uniform test)
    for (int b = 0; b < nb; ++b) {
      if (s_page[b] < 0 || (s_len[b] - 1) % kP != 0) continue;
      for (int w = tid; w < p.Hkv * (kP - 1) * 16; w += kPlanThreads) {
        const int kh = w / ((kP - 1) * 16), r2 = w % ((kP - 1) * 16);
        const int64_t dst = ((plane + (int64_t)s_page[b] * p.Hkv + kh) * kP + 1 + r2 / 16) * 16 + (r2 & 15);
        p.k_pool[dst] = make_uint4(0, 0, 0, 0);
        p.v_pool[dst] = make_uint4(0, 0, 0, 0);
      }
    }
    // generic-proxy stores -> the attention kernel's TMA (async proxy) reads
    asm volatile("fence.proxy.async.global;" ::: "memory");
    __threadfence();
    asm volatile("griddepcontrol.launch_dependents;");
    return;
  }
  if (p.k_new && tid < nb && s_len[tid] > 0) p.lens[row0 + tid] = s_len[tid];
  const int npg = g.max_npages;
  int4* out = p.items + row0 * p.maxP;
  int base = 0;
  for (int i0 = 0; i0 < npg; i0 += kPlanThreads) {
    const int i = i0 + tid;
    // entry of beam b at position i (-1: the beam does not reach it); read
    // twice (count, then write) instead of held in registers
    auto entry = [&](int b) { return (i < npg && i * kP < s_len[b]) ? __ldg(trow + (int64_t)b * p.maxP + i) : -1; };
    int c = 0, last = -1;
#pragma unroll 8
    for (int b = 0; b < nb; ++b) {
      const int t = entry(b);
      if (t >= 0) {
        c += t != last;
        last = t;
      }
    }
    int x = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_wsum[wid] = x;
    __syncthreads();
    int wpre = 0, tot = 0;
#pragma unroll
    for (int k = 0; k < kPlanThreads / 32; ++k) {
      const int v = s_wsum[k];
      wpre += k < wid ? v : 0;
      tot += v;
    }
    int o = base + wpre + x - c;
    last = -1;
    int s0 = 0;
    uint32_t mem = 0;
#pragma unroll 8
    for (int b = 0; b < nb; ++b) {
      const int t = entry(b);
      if (t >= 0) {
        if (t != last) {
          if (last >= 0)
            out[o++] = make_int4(last, (int)mem, min(kP, s_len[s0] - i * kP),
                                 p.refcounts && __ldg(p.refcounts + last) > __popc(mem));
          last = t;
          mem = 1u << b;
          s0 = b;
        } else {
          mem |= 1u << b;
        }
      }
    }
    if (last >= 0)
      out[o] = make_int4(last, (int)mem, min(kP, s_len[s0] - i * kP), p.refcounts && __ldg(p.refcounts + last) > __popc(mem));
    base += tot;
    __syncthreads();
  }
  if (tid == 0) p.counts[gi] = base;
  __threadfence();
  asm volatile("griddepcontrol.launch_dependents;");
  if (blockIdx.x == 0 && tid == 0) asm volatile("griddepcontrol.wait;" ::: "memory");
}

// ---------------------------------------------------------------------------
// Persistent attention (a4 + a5), one CTA per SM.  The call's work is a
// sequence of units (8 distinct pages of one tile), tiles ordered (layer, kv
// head, group) with the group fastest.  Whole tiles go round-robin while there
// are at least 3/4 as many left as CTAs (phase 1); the units of the rest are
// split evenly over the CTAs (phase 2, stream-K).  A CTA's phase-2 range covers whole
// tiles and at most two partial ones; a tile split over several CTAs is merged
// by the CTA that finishes its piece last (global counter), reading the
// pieces' partial (m, l, O) in piece order, so the result does not depend on
// which CTA finishes first.  Every warp derives the same piece sequence from
// the per-group unit counts (prefix in smem).
// kPoly: exponentials on the FMA/ALU pipes (ex2_poly2) instead of MUFU: 1 = every other pair, 2 = all
// instead of MUFU.
// kPair: a cluster of two CTAs per tile of a group of up to 32 beams (each
// CTA the rows of half the beams): every K/V page of a unit is loaded once
// for both (TMA multicast, each CTA issuing half of the pages), so pages the
// two halves share are not fetched twice.
template <int kPoly, bool kPair>
__global__ void __maxnreg__(kMaxRegs)
    k_tree_umma(const __grid_constant__ CUtensorMap tmk, const __grid_constant__ CUtensorMap tmv, UParams p,
                const __grid_constant__ UInline inl) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const uint32_t base = su32(smem_raw);
  uint8_t* bp = smem_raw;
  if (base & 1023u) {  // (never seen: the layout has no slack for a misaligned base)
    if (threadIdx.x == 0) atomicCAS(p.status, 0, (int32_t)TTS_ERR_UNSUPPORTED);
    return;
  }
  int4* meta = reinterpret_cast<int4*>(bp + kOffMeta);
  uint64_t* bars = reinterpret_cast<uint64_t*>(bp + kOffBar);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + kNumBars);
  // [n_groups + 1] exclusive prefix of units per group: this CTA's slice of a
  // global scratch (no room left in shared memory; read through L1)
  int* s_pre = p.pre + (size_t)blockIdx.x * (kMaxGroups + 1);
  int* s_info = reinterpret_cast<int*>(bp + kOffInfo);  // [0] merger flag
  float* s_xm = reinterpret_cast<float*>(bp + kOffXm);
  const uint32_t b_kfull = su32(bars), b_kempty = b_kfull + 8 * kNK, b_vfull = b_kempty + 8 * kNK,
                 b_vempty = b_vfull + 8 * kNV, b_sfull = b_vempty + 8 * kNV, b_pfull = b_sfull + 8 * kNSB,
                 b_pv = b_pfull + 8 * kNSB, b_qready = b_pv + 8 * kNSB, b_ofree = b_qready + 8, b_qtaken = b_ofree + 8;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // pair mode: this CTA's rank in its cluster, and the scheduling index (the pair)
  const int rank = kPair ? (int)cluster_ctarank() : 0;
  const int cta = kPair ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
  const uint16_t kBoth = 3;
  if (threadIdx.x == 0) TTS_TR(1023, 0);  // CTA start
  if (threadIdx.x == 0) TTS_CTA(0, gtimer());
  if (threadIdx.x == 0) TTS_SPAN(p.launch_id, 0, gtimer(), atomicMin);
  if (threadIdx.x == 0) {
    // (pair mode: a slot is free once both CTAs' MMAs have read it)
    for (int i = 0; i < kNK; ++i) {
      bar_init(b_kfull + 8 * i, 1);
      bar_init(b_kempty + 8 * i, kPair ? 2 : 1);
    }
    for (int i = 0; i < kNV; ++i) {
      bar_init(b_vfull + 8 * i, 1);
      bar_init(b_vempty + 8 * i, kPair ? 2 : 1);
    }
    for (int i = 0; i < kNSB; ++i) {
      bar_init(b_sfull + 8 * i, 1);
      bar_init(b_pfull + 8 * i, kSoftmaxWarps);
      bar_init(b_pv + 8 * i, 1);
    }
    bar_init(b_qready, kSoftmaxWarps);
    bar_init(b_ofree, kSoftmaxWarps);
    bar_init(b_qtaken, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 10) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  if (kPair) cluster_sync();  // the partner's barriers exist before any multicast reaches them
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t t_o = tmem, t_s = tmem + kTS;
  const uint32_t s_q = base + kOffQ;
  const int G = p.G;
  const int ng = p.n_groups;
  const int T = p.n_layers * p.Hkv * ng;
  const int Cg = kPair ? (int)(gridDim.x >> 1) : (int)gridDim.x;  // scheduling units (pairs)
  auto group_of = [&](int gi) { return p.groups ? p.groups[gi] : inl.g[gi]; };
  const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
  const int r = (warp & 3) * 32 + lane;  // softmax warps: the TMEM lane (tile row) of this thread
  // Rows of a tile, balanced over the four lane quadrants (softmax warps):
  // warp w holds beams [w*bpw, (w+1)*bpw) of the group, G consecutive lanes
  // per beam (host: bpw * G <= 32).  A page's exponentials are computed only
  // by the warps holding one of its member beams, so spreading the beams
  // evenly spreads the softmax work of private pages over all four warps.
  const bool kRoundRobin = p.round_robin != 0;
  // (pair mode: rank 0 holds beams [0, ceil(nb/2)), rank 1 the rest)
  auto row_of = [&](const GroupDesc& g, int row, int& beam, int& head) {
    const int nbh = kPair ? (g.nbeams + 1) >> 1 : g.nbeams;
    const int boff = rank * nbh, nbl = kPair && rank ? g.nbeams - nbh : nbh;
    const int bpw = (nbl + 3) >> 2;
    const int l = row & 31, bw = l / G;
    const int lb = kRoundRobin ? bw * 4 + (row >> 5) : (row >> 5) * bpw + bw;
    beam = boff + lb;
    head = l - bw * G;
    return bw < bpw && lb < nbl && ((g.active >> beam) & 1u);
  };
  // pair mode: the unit's pages read by none of this CTA's beams need no MMA
  // here (the partner's private pages); both issuing warps take the same
  // decision from the unit metadata
  auto cta_reads = [&](const GroupDesc& g, const int4* mrow) {
    if (!kPair) return true;
    const int nbh = (g.nbeams + 1) >> 1;
    const int nbl = rank ? g.nbeams - nbh : nbh;
    const uint32_t mine = (((1u << nbl) - 1u) << (rank * nbh)) & g.active;
    uint32_t any = 0;
#pragma unroll
    for (int k = 0; k < kU; ++k) {
      const int4 m = mrow[k];
      any |= m.x >= 0 ? ((uint32_t)m.y & mine) : 0u;
    }
    return any != 0u;
  };
  // Q rows of a piece -> TMEM (the A operand of S = Q K^T): lane = row, column = d pair
  auto load_q = [&](int gi, int slab) {
    const GroupDesc g = group_of(gi);
    int bl, hd;
    const bool ok = row_of(g, r, bl, hd);
    const int lrel = slab / p.Hkv, kh = slab % p.Hkv;
    const uint4* src = reinterpret_cast<const uint4*>(
        p.q + ((((int64_t)lrel * p.n_call + g.call_idx) * p.maxB + g.beam0 + (ok ? bl : 0)) * p.Hq + kh * G +
               (ok ? hd : 0)) * kD);
    {
      // warp half hf = warp >> 2 writes d columns [64 hf, 64 hf + 64) of row r:
      // 16-B chunk c at (c ^ (r & 7)) within the row's 128 B (SWIZZLE_128B)
      const int hf = warp >> 2;
      uint4 v[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) v[c] = ok ? __ldg(src + hf * 8 + c) : make_uint4(0, 0, 0, 0);
      const uint32_t row = s_q + hf * (kRows * 128) + r * 128;
#pragma unroll
      for (int c = 0; c < 8; ++c)
        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(row + ((c ^ (r & 7)) << 4)), "r"(v[c].x),
                     "r"(v[c].y), "r"(v[c].z), "r"(v[c].w)
                     : "memory");
    }
    // generic-proxy stores -> the tensor core's (async proxy) operand reads
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) bar_arrive(b_qready);
  };
  // Programmatic dependent launch: this grid starts while k_plan (the call's
  // append + plan) runs; everything below reads what k_plan writes.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) TTS_CTA(1, gtimer());  // the plan (and every earlier call) is complete
  // the next call's k_plan may start once every CTA of this grid is past the
  // wait: the previous call's attention kernel has then exited, so the plan
  // buffer that k_plan overwrites (parity of the previous call) is free
  if (threadIdx.x == 0) asm volatile("griddepcontrol.launch_dependents;");
  if (warp == 0) {
    // the schedule depends on the plan's counts only (k_plan writes empty
    // plans under a sticky error), so every CTA of the launch derives the same
    // one and the split-tile counters always complete
    int run = 0;
    for (int i0 = 0; i0 < p.n_groups; i0 += 32) {
      const int i = i0 + lane;
      const int u = i < p.n_groups ? (__ldg(p.counts + i) + kU - 1) / kU : 0;
      int x = u;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      TTS_ASSERT(p.n_groups <= kMaxGroups && (int)blockIdx.x < kMaxCtas);
      if (i < p.n_groups) s_pre[i + 1] = run + x;
      run += __shfl_sync(0xffffffffu, x, 31);
    }
    if (lane == 0) s_pre[0] = 0;
    __syncwarp();
    // sched 4 (group-proportional stream-K, below): usable when every group
    // with units gets >= 1 CTA and >= 1 unit per CTA
    const int Sw = s_pre[p.n_groups];
    const int Cw = kPair ? (int)(gridDim.x >> 1) : (int)gridDim.x;
    const int ns = p.n_layers * p.Hkv;
    bool okp = Sw > 0 && p.n_groups <= Cw;
    for (int i = lane; okp && i < p.n_groups; i += 32) {
      const int u = s_pre[i + 1] - s_pre[i];
      const int c0 = (int)((2ll * Cw * s_pre[i] + Sw) / (2ll * Sw));
      const int c1 = (int)((2ll * Cw * s_pre[i + 1] + Sw) / (2ll * Sw));
      if (u > 0 && (c1 <= c0 || (int64_t)ns * u < c1 - c0)) okp = false;
    }
    okp = __all_sync(0xffffffffu, okp);
    if (lane == 0) s_info[1] = okp;
  }
  __syncthreads();
  const int S = s_pre[p.n_groups];  // units per (layer, kv head) slab
  const int64_t U = (int64_t)S * p.n_layers * p.Hkv;
  // Schedule.  Tiles t = slab * ng + gi (slab = layer * Hkv + kv head).
  // Phase 1: k1 rounds of whole tiles, tile blockIdx.x + k * C in round k --
  // the groups of one slab run side by side, so pages they share are read
  // from HBM about once (L2).  Phase 2: the units of the remaining tiles, split
  // over the CTAs (stream-K).
  auto F = [&](int t) { return (int64_t)(t / ng) * S + s_pre[t % ng]; };  // first unit of tile t
  int maxu = 0;
  for (int i = 0; i < ng; ++i) maxu = max(maxu, s_pre[i + 1] - s_pre[i]);
  // Whole-tile rounds (phase 1): every full round but the last, unless the
  // tiles end exactly on a round (or a last partial round fills >= 3/4 of the
  // CTAs: taken whole too, cheaper than splitting and merging every tile).
  // The rest goes through phase 2; if k1 rounds of the largest tile could
  // exceed a CTA's fair share U / C, no phase 1 at all (an even split of
  // every unit, always balanced).
  int k1 = T / Cg;
  if (4 * (T - k1 * Cg) >= 3 * Cg && !p.split_partial_round) ++k1;
  else if (k1 > 0 && T > k1 * Cg) --k1;
  if (k1 > 0 && T > k1 * Cg && (int64_t)k1 * maxu + 1 > U / Cg) k1 = 0;
  if (p.sched >= 2) k1 = 0;
  // Unit order of the stream-K phase: slab-major (tile = slab * ng + group),
  // or group-major (sched 3: every slab of group 0, then group 1, ...), which
  // puts the ng groups of a slab on CTAs about C / ng apart at the same
  // relative offset -- processed at the same time, so the pages they share
  // hit L2 -- with the same exact unit balance.
  // sched 4: group-major order, and each group its own block of CTAs in
  // proportion to its units (CTA boundary of group g: C s_pre[g] / S, rounded),
  // its units split evenly inside the block -- every group reaches slab s at
  // the same point of the call, so the pages the groups of a slab share are
  // fetched from HBM about once (L2), with the units still balanced
  const bool prop = k1 == 0 && p.sched == 4 && s_info[1];
  const bool gmaj = p.sched == 3 || prop;
  const int nslab = p.n_layers * p.Hkv;
  auto U0 = [&](int gi, int slab) -> int64_t {  // first unit of tile (slab, gi) in the sequence
    return gmaj ? (int64_t)nslab * s_pre[gi] + (int64_t)slab * (s_pre[gi + 1] - s_pre[gi]) : (int64_t)slab * S + s_pre[gi];
  };
  // Phase-1 tile of CTA c in round k: tile k C + c, rotated by k inside
  // aligned blocks of ng CTAs in full rounds, so that the ng groups of a slab
  // still run side by side (pages they share are read from HBM about once,
  // L2) while every CTA meets every group position over the rounds (their
  // costs differ systematically).
  const bool rot = p.sched == 0;
  auto p1tile = [&](int c, int k) {
    const int blk = c / ng * ng;
    return (rot && blk + ng <= Cg && (k + 1) * Cg <= T) ? k * Cg + blk + (c - blk + k) % ng : k * Cg + c;
  };
  const int n1 = cta < T - (k1 - 1) * Cg ? k1 : k1 - 1;  // this CTA's whole tiles
  const int64_t base2 = F(min(k1 * Cg, T));
  const int64_t U2 = U - base2;
  // phase-2 CTAs: every one gets >= 1 unit (a split tile's pieces are then
  // exactly the CTAs whose ranges meet it)
  // Balanced split (when phase 1 ran and every tile is smaller than a CTA's
  // fair share U / C): CTA c's phase-2 range tops its phase-1 tiles up to
  // ~(c+1) U / C units in total, start2(c) = base2 + c U / C - (phase-1 units
  // of CTAs < c).  Otherwise an even split of the phase-2 units.
  const bool bal = k1 > 0 && U2 > 0;
  const int C2 = bal || prop ? Cg : (int)min((int64_t)Cg, U2);
  auto f1 = [&](int cc) {  // phase-1 units of CTAs [0, cc)
    int64_t a = 0;
    const int cb = cc / ng * ng;  // whole blocks: the same tiles as without rotation
    for (int k = 0; k < k1; ++k) {
      a += F(min(cb + k * Cg, T)) - F(min(k * Cg, T));
      for (int c = cb; c < cc; ++c) {
        const int t = p1tile(c, k);
        if (t < T) a += F(t + 1) - F(t);
      }
    }
    return a;
  };
  auto csg = [&](int g) { return (int)((2ll * Cg * s_pre[g] + S) / (2ll * S)); };  // first CTA of group g (prop)
  auto start2 = [&](int cc) -> int64_t {
    if (prop) {
      if (cc >= Cg) return U;
      int lo = -1, hi = ng - 1;  // smallest g with csg(g + 1) > cc
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (csg(mid + 1) > cc) hi = mid;
        else lo = mid;
      }
      const int g = hi, c0 = csg(g), cn = csg(g + 1) - c0;
      const int64_t wg = (int64_t)nslab * (s_pre[g + 1] - s_pre[g]);
      return (int64_t)nslab * s_pre[g] + (int64_t)(cc - c0) * wg / cn;
    }
    return bal ? base2 + (int64_t)cc * U / Cg - f1(cc) : base2 + (int64_t)cc * U2 / C2;
  };
  const int64_t ua2 = cta < C2 ? start2(cta) : 0;
  const int64_t ub2 = cta < C2 ? start2(cta + 1) : 0;
  // the tile piece containing global unit u (phase 2): units [j0, j1) of tile (slab, gi)
  auto piece_at = [&](int64_t u, int& gi, int& slab, int& j0, int& j1) {
    if (gmaj) {
      int lo = 0, hi = ng;  // largest group with nslab * s_pre[gi] <= u
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if ((int64_t)nslab * s_pre[mid] <= u) lo = mid;
        else hi = mid;
      }
      gi = lo;
      const int ug = s_pre[gi + 1] - s_pre[gi];
      const int64_t rel = u - (int64_t)nslab * s_pre[gi];
      slab = (int)(rel / ug);
      j0 = (int)(rel - (int64_t)slab * ug);
      j1 = (int)min((int64_t)ug, (int64_t)j0 + (ub2 - u));
      return;
    }
    slab = (int)(u / S);
    const int o = (int)(u - (int64_t)slab * S);
    int lo = 0, hi = ng;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (s_pre[mid] <= o) lo = mid;
      else hi = mid;
    }
    gi = lo;
    j0 = o - s_pre[gi];
    j1 = (int)min((int64_t)(s_pre[gi + 1] - s_pre[gi]), (int64_t)j0 + (ub2 - u));
  };
  int n_pieces = n1;
  for (int64_t u = ua2; u < ub2; ++n_pieces) {
    int gi, slab, j0, j1;
    piece_at(u, gi, slab, j0, j1);
    u += j1 - j0;
  }
  // piece idx of this CTA; pslot: partial-state slot (-1: phase 1, whole tile).
  // Each warp walks its pieces in order: the phase-2 cursor (first unit of the
  // last piece looked up, and its index) makes the next lookup O(1).
  int64_t cur_u = ua2;
  int cur_idx = n1;
  auto piece = [&](int idx, int& gi, int& slab, int& j0, int& j1, int& pslot) {
    if (idx < n1) {
      const int t = p1tile(cta, idx);
      slab = t / ng;
      gi = t - slab * ng;
      j0 = 0;
      j1 = s_pre[gi + 1] - s_pre[gi];
      pslot = -1;
      return;
    }
    if (idx < cur_idx) {
      cur_idx = n1;
      cur_u = ua2;
    }
    for (;;) {
      piece_at(cur_u, gi, slab, j0, j1);
      if (cur_idx == idx) break;
      cur_u += j1 - j0;
      ++cur_idx;
    }
    pslot = 2 * blockIdx.x + (cur_u == ua2 ? 0 : 1);
    TTS_ASSERT(gi >= 0 && gi < ng && slab >= 0 && slab < p.n_layers * p.Hkv && 0 <= j0 && j0 <= j1 &&
               j1 <= s_pre[gi + 1] - s_pre[gi]);
  };

  if (warp == 8 || warp == 9) {
    // ================= producers: TMA (warp 4: K + unit metadata, warp 5: V) =================
    // Lane k < kU owns page k of a unit: it loads the plan item (one unit
    // ahead) and issues that page's TMA; lane 0 arms the slot's barrier first.
    const bool is_k = warp == 8;
    if (lane == 0) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(is_k ? &tmk : &tmv)) : "memory");
    // (TTS_PROF: [0] waiting for a free slot, [1] issuing, [2] item loads)
    PROF_DECL;
    const int nslot = is_k ? kNK : kNV;
    // TTS_L2HINT: 1 evict_last / evict_first, 2 evict_last / normal, 3 normal / evict_first
    const uint64_t pol_keep = p.l2hint == 3 ? l2_policy_evict_normal() : l2_policy_evict_last();
    const uint64_t pol_stream = p.l2hint == 2 ? l2_policy_evict_normal() : l2_policy_evict_first();
    const uint32_t b_f = is_k ? b_kfull : b_vfull, b_e = is_k ? b_kempty : b_vempty;
    int slot = 0, js = 0;
    uint32_t ph = 0;
    for (int pc = 0; pc < n_pieces; ++pc) {
      int gi, slab, j0, j1, pslot;
      piece(pc, gi, slab, j0, j1, pslot);
      const GroupDesc g = group_of(gi);
      const int kh = slab % p.Hkv, layer = p.layer_begin + slab / p.Hkv;
      const int nit = __ldg(p.counts + gi);
      const int4* its = p.items + ((int64_t)g.req * p.maxB + g.beam0) * p.maxP;
      const int64_t layer_rows = ((int64_t)layer * p.num_pages) * p.Hkv;
      // lanes [0, kU): page `lane` of the next unit; lanes [kU, 2 kU): page
      // lane - kU of the unit kPF ahead, prefetched into L2 (more bytes in flight
      // than the shared-memory ring holds)
      const int pg = lane & (kU - 1);
      auto item = [&](int v) {
        const int i = kU * v + pg;
        return (lane < 2 * kU && v < j1 && i < nit) ? __ldg(its + i) : make_int4(-2, 0, 0, 0);
      };
      auto prefetch = [&](const int4& m) {
        if (kPF > 0 && lane >= kU && lane < 2 * kU && m.x >= 0) {
          const int y = (int)((layer_rows + (int64_t)m.x * p.Hkv + kh) * kP);
          if (is_k) {
            tma2d_prefetch(&tmk, 0, y);
            tma2d_prefetch(&tmk, 64, y);
          } else {
            tma3d_prefetch(&tmv, 0, y, 0);
          }
        }
      };
      if (kPF > 0)
        for (int d = 0; d < kPF; ++d) prefetch(item(j0 + d));
      int4 nx = item(lane < kU ? j0 : j0 + kPF);
      for (int v = j0; v < j1; ++v, ++js) {
        const int4 m = nx;
        nx = item(lane < kU ? v + 1 : v + 1 + kPF);
        prefetch(m);
        PROF_MARK(2);
        bar_wait(b_e + 8 * slot, ph ^ 1u);
        PROF_MARK(0);
        if (lane == 0) TTS_TR2(js, is_k ? 3 : 4);
        // pair mode: every page lands in both CTAs; this CTA issues pages
        // [kU/2 rank, kU/2 (rank + 1)), the partner the others
        const bool present = lane < kU && m.x >= 0;
        const bool has = present && (!kPair || (lane / (kU / 2)) == rank);
        const uint32_t np = __popc(__ballot_sync(0xffffffffu, present));
        const uint32_t fb = b_f + 8 * slot;
        if (is_k && lane < kU) meta[(js % kNM) * kU + lane] = m;
        if (lane == 0) bar_expect(fb, np * (uint32_t)kTile);
        __syncwarp();
        if (has && p.l2hint && !kPair) {
          // pages other groups also read stay in L2 for them; the group's own
          // pages are streamed through
          const uint64_t pol = m.w ? pol_keep : pol_stream;
          const int y = (int)((layer_rows + (int64_t)m.x * p.Hkv + kh) * kP);
          if (is_k) {
            const uint32_t sb = base + kOffK + slot * kKSlot + lane * (kTile / 2);
            tma2d_hint(sb, &tmk, 0, y, fb, pol);
            tma2d_hint(sb + kU * (kTile / 2), &tmk, 64, y, fb, pol);
          } else {
            tma3d_hint(base + kOffV + slot * kVSlot + lane * kTile, &tmv, 0, y, 0, fb, pol);
          }
        } else if (has) {
          const int y = (int)((layer_rows + (int64_t)m.x * p.Hkv + kh) * kP);
          if (is_k) {
            // K: [d half][page][16 tokens][128 B] (one 128-row K-major operand over the unit)
            const uint32_t sb = base + kOffK + slot * kKSlot + lane * (kTile / 2);
            if (kPair) {
              tma2d_mc(sb, &tmk, 0, y, fb, kBoth);
              tma2d_mc(sb + kU * (kTile / 2), &tmk, 64, y, fb, kBoth);
            } else {
              tma2d(sb, &tmk, 0, y, fb);
              tma2d(sb + kU * (kTile / 2), &tmk, 64, y, fb);
            }
          } else {
            // V: [page][d half][16][128 B] (3D box)
            if (kPair) tma3d_mc(base + kOffV + slot * kVSlot + lane * kTile, &tmv, 0, y, 0, fb, kBoth);
            else tma3d(base + kOffV + slot * kVSlot + lane * kTile, &tmv, 0, y, 0, fb);
          }
        }
        __syncwarp();
        if (++slot == nslot) {
          slot = 0;
          ph ^= 1u;
        }
        PROF_MARK(1);
      }
    }
    PROF_FLUSH(warp);
  } else if (warp == 10) {
    // ========================= S issuer: S = Q K^T =========================
    // The whole warp runs the loop so that descriptors stay warp-uniform; one
    // elected lane issues.  S and PV are issued by two warps so that neither
    // waits behind the other's issue (the tensor pipe runs both in issue order).
    constexpr uint32_t id_s = idesc_bf16(kRows, kSCols, false);
    const uint64_t dk0 = sdesc(base + kOffK, 16, 1024, 2);  // K tiles: K-major SW128
    const uint64_t dq0 = sdesc(s_q, 16, 1024, 2);            // Q: K-major SW128
    // (TTS_PROF: [0] waiting for K, [1] waiting for the S buffer, [2] issuing, [3] waiting for Q)
    PROF_DECL;
    int js = 0;
    for (int pc = 0; pc < n_pieces; ++pc) {
      int gi, slab, j0, j1, pslot;
      piece(pc, gi, slab, j0, j1, pslot);
      const GroupDesc g = group_of(gi);
      PROF_MARK(2);
      bar_wait(b_qready, pc & 1);  // this piece's Q in TMEM
      PROF_MARK(3);
      // an empty piece issues no MMA: release its Q explicitly, so that the
      // softmax warps load the next Q only after this wait (no parity aliasing)
      if (j1 == j0 && lane == 0) bar_arrive(b_qtaken);
      for (int j = j0; j < j1; ++j, ++js) {
        const int slot = js % kNK;
        PROF_MARK(2);
        bar_wait(b_kfull + 8 * slot, (js / kNK) & 1u);
        PROF_MARK(0);
        if (lane == 0) TTS_TR(js, 0);
        // S buffer js % 3 holds P(js - 3) until PV(js - 3) has read it
        if (js >= kNSB) bar_wait(b_pv + 8 * (js % kNSB), ((js - kNSB) / kNSB) & 1u);
        PROF_MARK(1);
        if (lane == 0) TTS_TR(js, 1);
        tc_fence_after();
        // S[128 x 128] = Q . K^T over the unit's 8 pages: 8 MMAs (K = 16 of d
        // each; an absent page leaves its 16 columns undefined: masked)
        const uint32_t sd = t_s + (js % kNSB) * kSCols;
        const uint64_t dk = dk0 + (uint64_t)((slot * kKSlot) >> 4);
        // (timing experiments only, outputs garbage: -DTTS_NOMMA_S drops S = Q K^T,
        // -DTTS_MEMONLY every MMA and the softmax work -- DESIGN.md section 7)
#if defined(TTS_NOMMA_S) || defined(TTS_MEMONLY)
        const bool run = false;
#else
        const bool run = cta_reads(g, meta + (js % kNM) * kU);
#endif
        if (elect_one()) {
#pragma unroll
          for (int ks = 0; ks < kD / 16; ++ks)
            if (run) mma_ss(sd, dq0 + (uint64_t)(((ks >> 2) * (kRows * 128) + (ks & 3) * 32) >> 4),
                   dk + (uint64_t)(((ks >> 2) * (kKSlot / 2) + (ks & 3) * 32) >> 4), id_s, ks > 0);
          tc_commit(b_sfull + 8 * (js % kNSB));
          if (kPair) tc_commit_mc(b_kempty + 8 * slot, kBoth);
          else tc_commit(b_kempty + 8 * slot);
        }
        __syncwarp();
        if (lane == 0) TTS_TR(js, 2);
      }
    }
    PROF_MARK(2);
    PROF_FLUSH(10);
  } else if (warp == 11) {
    // ====================== PV issuer: O += P V ======================
    constexpr uint32_t id_pv = idesc_f16(kRows, kD, true);
    const uint64_t dv0 = sdesc(base + kOffV, 2048, 1024, 2);  // V tiles: MN-major SW128
    // (TTS_PROF: [0] waiting for V, [1] waiting for P, [2] waiting for O, [3] issuing)
    PROF_DECL;
    int js = 0;
    for (int pc = 0; pc < n_pieces; ++pc) {
      int gi, slab, j0, j1, pslot;
      piece(pc, gi, slab, j0, j1, pslot);
      const GroupDesc g = group_of(gi);
      uint32_t acc = 0;  // O written by an earlier PV of this piece
      for (int j = j0; j < j1; ++j, ++js) {
        const int slot = js % kNV;
        PROF_MARK(3);
        bar_wait(b_vfull + 8 * slot, (js / kNV) & 1u);
        PROF_MARK(0);
        if (lane == 0) TTS_TR(js, 6);
        bar_wait(b_pfull + 8 * (js % kNSB), (js / kNSB) & 1u);
        PROF_MARK(1);
        if (lane == 0) TTS_TR(js, 7);
        // the first PV of a piece overwrites O: the previous piece's epilogue must have read it
        if (j == j0 && pc > 0) bar_wait(b_ofree, (pc - 1) & 1);
        PROF_MARK(2);
        tc_fence_after();
        const uint32_t pa = t_s + (js % kNSB) * kSCols;
        const int4* mrow = meta + (js % kNM) * kU;
        const bool e = elect_one();
        // (pair mode: a unit this CTA does not read is skipped -- its P is
        // zero -- unless it is the piece's last and O was never written: then
        // O = 0 . V initialises it)
#if defined(TTS_NOMMA_PV) || defined(TTS_MEMONLY)  // (timing experiments only)
        const bool run = j + 1 == j1 && !acc;
#else
        const bool run = cta_reads(g, mrow) || (j + 1 == j1 && !acc);
#endif
#pragma unroll
        for (int k = 0; k < kU; ++k) {
          if (mrow[k].x < 0 || !run) continue;
          const uint64_t dv = dv0 + (uint64_t)((slot * kVSlot + k * kTile) >> 4);
          if (e) mma_ts(t_o, pa + k * (kP / 2), dv, id_pv, acc);
          acc = 1;
        }
        if (e) {
          if (kPair) tc_commit_mc(b_vempty + 8 * slot, kBoth);
          else tc_commit(b_vempty + 8 * slot);
          tc_commit(b_pv + 8 * (js % kNSB));
        }
        __syncwarp();
      }
    }
    PROF_MARK(3);
    PROF_FLUSH(11);
  } else {
    // ==================== softmax (warps 0-7: lane quadrant warp & 3, half hh) ====================
    // The two warps of a quadrant hold the same 32 rows: warp half hh reads the
    // S columns of pages [4 hh, 4 hh + 4) of every unit and owns O columns
    // [64 hh, 64 hh + 64) (rescale, epilogue, merge).  The row max is
    // exchanged through shared memory (one pair barrier per unit), so both
    // halves use the same running max; each keeps its own partial row sum.
    const int hh = warp >> 2;
    const int pair_bar = 2 + (warp & 3);  // named barrier of the quadrant's two warps
    auto pair_sync = [&]() { asm volatile("bar.sync %0, 64;" ::"r"(pair_bar) : "memory"); };
    if (n_pieces > 0) {  // the first piece's Q (the schedule needs the plan)
      int gi, slab, j0, j1, pslot;
      piece(0, gi, slab, j0, j1, pslot);
      load_q(gi, slab);
    }
    // (TTS_PROF: [0] waiting for S, [1] softmax of member units, [2] skipped units,
    //  [3] epilogue + Q loads, [4] rescales, [5] P store + arrive; [6] member units, [7] all units)
    PROF_DECL;
    int js = 0, n_empty = 0;
    for (int pc = 0; pc < n_pieces; ++pc) {
      int gi, slab, j0, j1, pslot;
      piece(pc, gi, slab, j0, j1, pslot);
      if (pc + 1 < n_pieces) {
        // the next piece's Q rows -> L2 now, so that its load after this
        // piece's last unit does not wait for HBM
        int gi2, slab2, j02, j12, ps2;
        piece(pc + 1, gi2, slab2, j02, j12, ps2);
        const GroupDesc g2 = group_of(gi2);
        int bl2, hd2;
        if (row_of(g2, r, bl2, hd2)) {
          const __nv_bfloat16* q2 = p.q + ((((int64_t)(slab2 / p.Hkv) * p.n_call + g2.call_idx) * p.maxB + g2.beam0 + bl2) * p.Hq +
                                           (slab2 % p.Hkv) * G + hd2) * kD + (warp >> 2) * 64;
          asm volatile("prefetch.global.L2 [%0];" ::"l"(q2));
        }
      }
      const GroupDesc g = group_of(gi);
      int rbl = 0, rh = 0;
      const bool rvalid = row_of(g, r, rbl, rh);
      const int lrel = slab / p.Hkv, kh = slab % p.Hkv;
      float m_ref = -1e30f, l = 0.f;
      for (int j = j0; j < j1; ++j, ++js) {
        PROF_MARK(3);
        bar_wait(b_sfull + 8 * (js % kNSB), (js / kNSB) & 1u);
        PROF_MARK(0);
        PROF_CNT(7);
        if (lane == 0 && warp == 0) TTS_TR(js, 3);
        if (lane == 0 && warp == 5) TTS_TR2(js, 0);
        tc_fence_after();
        const int4* mrow = meta + (js % kNM) * kU + hh * kUH;
        const uint32_t tB = t_s + lane_off + (js % kNSB) * kSCols;  // this unit's S/P buffer
        const uint32_t tS = tB + hh * (kUH * kP);
        // page membership: bit k of lm = this row reads page kUH hh + k; wmask =
        // the warp's union (a page none of its rows reads: P = 0, no exponentials)
        uint32_t lm = 0;
#pragma unroll
        for (int k = 0; k < kUH; ++k) {
          const int4 mt = mrow[k];
          lm |= (mt.x >= 0 && rvalid && ((((uint32_t)mt.y) >> rbl) & 1u)) ? 1u << k : 0u;
        }
#ifdef TTS_MEMONLY  // (timing experiment only: no softmax work)
        const uint32_t wmask = 0u * __reduce_or_sync(0xffffffffu, lm);
#else
        const uint32_t wmask = __reduce_or_sync(0xffffffffu, lm);
#endif
        uint32_t sr[kUH / 2][32];
        float mx = -INFINITY;
        if (wmask) {
          // S columns of the page pairs this warp reads
#pragma unroll
          for (int q = 0; q < kUH / 2; ++q)
            if ((wmask >> (2 * q)) & 3u) tc_ld32(tS + 32 * q, sr[q]);
          tc_wait_ld();
        }
        if (wmask) {
          // raw scores (scale > 0 commutes with max); token slots >= ntok -> -inf
          // (partial pages only); rows not reading page k: max and exponent
          // offset -inf below (P exactly 0)
#pragma unroll
          for (int k = 0; k < kUH; ++k) {
            if (!((wmask >> k) & 1u)) continue;
            uint32_t* w = sr[k >> 1] + (k & 1) * kP;
            const int ntok = mrow[k].z;
            if (ntok < kP) {
#pragma unroll
              for (int c = 0; c < kP; ++c) w[c] = c < ntok ? w[c] : __float_as_uint(-INFINITY);
            }
            float mk = fmax3(__uint_as_float(w[0]), __uint_as_float(w[1]), __uint_as_float(w[2]));
#pragma unroll
            for (int c = 3; c + 1 < kP; c += 2) mk = fmax3(mk, __uint_as_float(w[c]), __uint_as_float(w[c + 1]));
            mk = fmaxf(mk, __uint_as_float(w[kP - 1]));
            mx = fmaxf(mx, ((lm >> k) & 1u) ? mk : -INFINITY);
          }
        }
        // the unit's row max over both halves (the barrier also orders the
        // other half's P stores, which overlap these S columns, after our loads)
        float* xm = s_xm + ((js & 1) * 2 + hh) * kRows;
        xm[r] = mx;
        tc_fence_before();
        pair_sync();
        tc_fence_after();
        if (lane == 0 && warp == 0) TTS_TR(js, 4);
        if (lane == 0 && warp == 5) TTS_TR2(js, 1);
        mx = fmaxf(mx, s_xm[((js & 1) * 2 + (hh ^ 1)) * kRows + r]) * p.scale_log2;
        const bool need = mx > m_ref + 8.0f;
        if (__any_sync(0xffffffffu, need) && j > j0) {
          PROF_MARK(1);
          // every earlier PV product must have landed before O is rescaled in TMEM
          bar_wait(b_pv + 8 * ((js - 1) % kNSB), ((js - 1) / kNSB) & 1u);
          tc_fence_after();
          const float alpha = need ? exp2f(m_ref - mx) : 1.f;
#pragma unroll 1
          for (int ch = 0; ch < 2; ++ch) {
            uint32_t o[32];
            const uint32_t ta = t_o + lane_off + hh * 64 + ch * 32;
            tc_ld32(ta, o);
            tc_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
            tc_st32(ta, o);
          }
          tc_wait_st();
          l *= alpha;
          PROF_MARK(4);
        }
        if (need) m_ref = mx;
        if (wmask) {
          const float2 sc2 = make_float2(p.scale_log2, p.scale_log2);
          float2 lacc = make_float2(0.f, 0.f);
          // P (fp16, value c of page k at column 8k + c/2) over the pair's S
          // columns; every S load above has completed
#pragma unroll
          for (int q = 0; q < kUH / 2; ++q) {
            uint32_t pk[kP];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int k = 2 * q + h;
              if ((wmask >> k) & 1u) {
                const float nm = ((lm >> k) & 1u) ? -m_ref : -INFINITY;
                const float2 nm2 = make_float2(nm, nm);
                const uint32_t* w = sr[q] + h * kP;
#pragma unroll
                for (int c = 0; c < kP; c += 2) {
                  const float2 x = ffma2(make_float2(__uint_as_float(w[c]), __uint_as_float(w[c + 1])), sc2, nm2);
                  float a, b;
                  if (kPoly == 2 || (kPoly == 1 && ((c >> 1) & 1))) {
                    const float2 e2 = ex2_poly2(x);
                    a = e2.x;
                    b = e2.y;
                  } else {
                    a = ex2(x.x);
                    b = ex2(x.y);
                  }
                  lacc = fadd2(lacc, make_float2(a, b));
                  pk[h * (kP / 2) + c / 2] = pack_f16x2(a, b);
                }
              } else {
#pragma unroll
                for (int c = 0; c < kP / 2; ++c) pk[h * (kP / 2) + c] = 0u;
              }
            }
            tc_st16(tB + hh * (kUH * kP / 2) + 16 * q, pk);
          }
          l += lacc.x + lacc.y;
          PROF_MARK(1);
          PROF_CNT(6);
        } else {
          uint32_t z[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) z[i] = 0u;
          tc_st32(tB + hh * (kUH * kP / 2), z);
          PROF_MARK(2);
        }
        tc_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) bar_arrive(b_pfull + 8 * (js % kNSB));
        PROF_MARK(5);
        if (lane == 0 && warp == 0) TTS_TR(js, 5);
        if (lane == 0 && warp == 5) TTS_TR2(js, 2);
      }
      // the next piece's Q (every S MMA of this piece has completed), so that
      // its S = Q K^T overlaps this piece's epilogue
      if (pc + 1 < n_pieces) {
        if (j1 == j0) bar_wait(b_qtaken, (n_empty++) & 1);  // (a non-empty piece: its S MMAs read Q)
        int gi2, slab2, j02, j12, ps2;
        piece(pc + 1, gi2, slab2, j02, j12, ps2);
        PROF_MARK(3);
        load_q(gi2, slab2);
        PROF_MARK(8);
      }
      // ---------------- epilogue of the piece ----------------
      // (an empty piece -- a tile with no units, e.g. under a sticky error --
      // writes nothing)
      const int tu = s_pre[gi + 1] - s_pre[gi];
      if (j1 > j0) {
        // the row sum over both halves (the partner's partial sum of this piece)
        // (row sums through the max-exchange buffer of the next unit's parity:
        // its last reader passed the pair barrier of unit js - 1)
        float* s_xl = s_xm + (js & 1) * 2 * kRows;
        s_xl[hh * kRows + r] = l;
        bar_wait(b_pv + 8 * ((js - 1) % kNSB), ((js - 1) / kNSB) & 1u);
        PROF_MARK(9);
        tc_fence_after();
        // this half's 64 O columns -> registers; the accumulator is released at
        // once, so the next piece's first PV overlaps the stores below
        uint32_t o[2][32];
        tc_ld32(t_o + lane_off + hh * 64, o[0]);
        tc_ld32(t_o + lane_off + hh * 64 + 32, o[1]);
        tc_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) bar_arrive(b_ofree);
        pair_sync();
        l += s_xl[(hh ^ 1) * kRows + r];
        pair_sync();  // s_xl is rewritten by the next unit's max exchange
        float* orow = p.out + ((((int64_t)lrel * p.n_call + g.call_idx) * p.maxB + g.beam0 + rbl) * p.Hq + kh * G + rh) * kD + hh * 64;
        if (j0 == 0 && j1 == tu) {
          const float inv = 1.f / l;
          if (rvalid) {
#pragma unroll
            for (int c2 = 0; c2 < 2; ++c2)
#pragma unroll
              for (int i = 0; i < 32; i += 4)
                *reinterpret_cast<float4*>(orow + c2 * 32 + i) =
                    make_float4(__uint_as_float(o[c2][i]) * inv, __uint_as_float(o[c2][i + 1]) * inv,
                                __uint_as_float(o[c2][i + 2]) * inv, __uint_as_float(o[c2][i + 3]) * inv);
          }
        } else {
          // a5: this piece's (m, l, unnormalised O) -> its partial slot (2c for the
          // CTA's first phase-2 piece, 2c + 1 for its last); O chunk-major ([32
          // chunks of 4 floats][128 rows]) so that a warp's accesses coalesce.
          // The last piece to finish merges.
          TTS_ASSERT(pslot >= 0 && pslot < 2 * kMaxCtas);
          float* part = p.partial + (size_t)pslot * kPartFloats;
          if (hh == 0) {
            part[r] = m_ref;
            part[kRows + r] = l;
          }
          float4* po = reinterpret_cast<float4*>(part + 2 * kRows) + r;
#pragma unroll
          for (int c2 = 0; c2 < 2; ++c2)
#pragma unroll
            for (int i = 0; i < 8; ++i)
              __stcg(po + ((2 * hh + c2) * 8 + i) * kRows,
                     make_float4(__uint_as_float(o[c2][4 * i]), __uint_as_float(o[c2][4 * i + 1]),
                                 __uint_as_float(o[c2][4 * i + 2]), __uint_as_float(o[c2][4 * i + 3])));
          __threadfence();
          asm volatile("bar.sync 1, 256;" ::: "memory");
          const int64_t T0 = U0(gi, slab);
          auto cta_of = [&](int64_t x) {  // the phase-2 CTA whose range holds unit x
            if (prop) {
              int lo = 0, hi = ng;  // the group of unit x (largest g with nslab * s_pre[g] <= x)
              while (hi - lo > 1) {
                const int mid = (lo + hi) >> 1;
                if ((int64_t)nslab * s_pre[mid] <= x) lo = mid;
                else hi = mid;
              }
              const int c0 = csg(lo), cn = csg(lo + 1) - c0;
              const int64_t wg = (int64_t)nslab * (s_pre[lo + 1] - s_pre[lo]);
              return c0 + (int)(((x - (int64_t)nslab * s_pre[lo] + 1) * cn - 1) / wg);
            }
            if (!bal) return (int)(((x - base2 + 1) * C2 - 1) / U2);
            int lo = 0, hi = C2;  // largest c with start2(c) <= x
            while (hi - lo > 1) {
              const int mid = (lo + hi) >> 1;
              if (start2(mid) <= x) lo = mid;
              else hi = mid;
            }
            return lo;
          };
          const int c_first = cta_of(T0), c_last = cta_of(T0 + tu - 1);
          const int tile = (slab * ng + gi) * (kPair ? 2 : 1) + rank;  // (pair mode: each rank merges its own rows)
          TTS_ASSERT(tile >= 0 && tile < 2 * p.n_layers * p.Hkv * kMaxGroups && c_first <= cta && cta <= c_last);
          if (threadIdx.x == 0) s_info[0] = atomicAdd(p.tile_cnt + tile, 1) == c_last - c_first;
          asm volatile("bar.sync 1, 256;" ::: "memory");
          PROF_MARK(10);
          if (s_info[0]) {
            __threadfence();
            const int np = c_last - c_first + 1;
            // piece k's slot: only the first CTA's range can start before the tile
            auto cta_slot = [&](int c) { return 2 * (kPair ? 2 * c + rank : c); };  // first partial slot of CTA c's rank
            const int slot0 = cta_slot(c_first) + (start2(c_first) >= T0 ? 0 : 1);
            TTS_ASSERT(slot0 >= 0 && cta_slot(c_last) + 1 < 2 * kMaxCtas);
            auto part_of = [&](int k) { return p.partial + (size_t)(k == 0 ? slot0 : cta_slot(c_first + k)) * kPartFloats; };
            // latency-bound (L2 round trips under full HBM load): every batch of
            // loads is issued before any is consumed
            float M = -INFINITY, L = 0.f;
            for (int k0 = 0; k0 < np; k0 += 8) {
              float mv[8], lv[8];
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                const bool ok = k0 + i < np;
                mv[i] = ok ? __ldcg(part_of(k0 + i) + r) : -INFINITY;
                lv[i] = ok ? __ldcg(part_of(k0 + i) + kRows + r) : 0.f;
              }
              float M2 = M;
#pragma unroll
              for (int i = 0; i < 8; ++i) M2 = fmaxf(M2, mv[i]);
              L *= exp2f(M - M2);
#pragma unroll
              for (int i = 0; i < 8; ++i) L += k0 + i < np ? exp2f(mv[i] - M2) * lv[i] : 0.f;
              M = M2;
            }
            const float inv = 1.f / L;
#pragma unroll 1
            for (int c2 = 0; c2 < 2; ++c2) {
              const int ch = 2 * hh + c2;
              float4 acc[8];
#pragma unroll
              for (int i = 0; i < 8; ++i) acc[i] = make_float4(0.f, 0.f, 0.f, 0.f);
              for (int k = 0; k < np; k += 2) {
                const bool two = k + 1 < np;
                const float* pa = part_of(k);
                const float* pb = part_of(two ? k + 1 : k);
                const float wa = __ldcg(pa + r), wb = __ldcg(pb + r);
                const float4* sa = reinterpret_cast<const float4*>(pa + 2 * kRows) + r;
                const float4* sb = reinterpret_cast<const float4*>(pb + 2 * kRows) + r;
                float4 xa[8], xb[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                  xa[i] = __ldcg(sa + (ch * 8 + i) * kRows);
                  xb[i] = __ldcg(sb + (ch * 8 + i) * kRows);
                }
                const float fa = exp2f(wa - M), fb = two ? exp2f(wb - M) : 0.f;
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                  acc[i].x += fa * xa[i].x + fb * xb[i].x;
                  acc[i].y += fa * xa[i].y + fb * xb[i].y;
                  acc[i].z += fa * xa[i].z + fb * xb[i].z;
                  acc[i].w += fa * xa[i].w + fb * xb[i].w;
                }
              }
              if (rvalid) {
#pragma unroll
                for (int i = 0; i < 8; ++i)
                  *reinterpret_cast<float4*>(orow + c2 * 32 + 4 * i) =
                      make_float4(acc[i].x * inv, acc[i].y * inv, acc[i].z * inv, acc[i].w * inv);
              }
            }
            if (threadIdx.x == 0) p.tile_cnt[tile] = 0;  // every piece of the tile has arrived: ready for the next call
            PROF_MARK(11);
            PROF_CNT(12);
          }
        }
      } else {
        // an empty piece read nothing from O: release it for the next piece
        tc_fence_before();
        __syncwarp();
        if (lane == 0) bar_arrive(b_ofree);
      }
    }
    PROF_MARK(3);
    PROF_FLUSH(warp);
  }

  if (threadIdx.x == 0) TTS_TR(1023, 2);  // unit loop done
  tc_fence_before();
  __syncthreads();
  // pair mode: the partner's last multicast loads / commits target this CTA's
  // shared memory: neither exits before both are done
  if (kPair) cluster_sync();
  if (threadIdx.x == 0) TTS_TR(1023, 3);  // epilogue / merge done
  if (threadIdx.x == 0) TTS_CTA(2, gtimer());
  if (threadIdx.x == 0) TTS_SPAN(p.launch_id, 1, gtimer(), atomicMax);
#ifdef TTS_TRACE
  if (threadIdx.x == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
    long long units = ub2 - ua2;
    for (int k = 0; k < n1; ++k) {
      const int t = p1tile(cta, k), gi = t % ng;
      units += s_pre[gi + 1] - s_pre[gi];
    }
    TTS_CTA(3, units | ((long long)smid << 32));
  }
#endif
  if (warp == 10) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
  }
}

}  // namespace

#ifdef TTS_PROF
extern "C" int tts_debug_read_prof(long long* out_h) {
  return (int)cudaMemcpyFromSymbol(out_h, g_prof, sizeof(g_prof));
}
#endif

#ifdef TTS_TRACE
extern "C" int tts_debug_read_trace(long long* out_h) {
  int e = (int)cudaMemcpyFromSymbol(out_h, g_trace, sizeof(g_trace));
  e = e ? e : (int)cudaMemcpyFromSymbol(out_h + 1024 * 8, g_trace2, sizeof(g_trace2));
  return e ? e : (int)cudaMemcpyFromSymbol(out_h + 2 * 1024 * 8, g_cta, sizeof(g_cta));
}
// launch spans: reset (min slots to ~0, max slots to 0) / read [32768][4]
extern "C" int tts_debug_reset_spans() {
  static unsigned long long h[32768][4];
  for (int i = 0; i < 32768; ++i) h[i][0] = h[i][2] = ~0ull, h[i][1] = h[i][3] = 0;
  return (int)cudaMemcpyToSymbol(g_lspan, h, sizeof(h));
}
extern "C" int tts_debug_read_spans(unsigned long long* out_h) {
  return (int)cudaMemcpyFromSymbol(out_h, g_lspan, sizeof(g_lspan));
}
#endif

// split tiles' partial states, then the per-CTA unit-prefix scratch
size_t umma_partial_bytes() {
  return (size_t)2 * kMaxCtas * kPartFloats * 4 + (size_t)kMaxCtas * (kMaxGroups + 1) * 4;
}
int umma_max_groups() { return kMaxGroups; }

bool umma_supported(const Ctx* c) {
  const int G = c->cfg.num_q_heads / c->cfg.num_kv_heads;
  return c->cfg.head_dim == kD && c->cfg.page_size == kP && G >= 4 && G <= 16 && c->tmap3_ok && c->tmap_ok &&
         c->umma_ok;
}

// Per device context: the kernel attributes (single-CTA and pair kernels) and
// the number of co-resident 2-CTA clusters.  The plan's double buffer needs no
// residency argument: call N+1's k_plan is released only once every CTA of
// call N's attention kernel is past its plan wait, i.e. after call N-1's
// attention kernel (the reader of the buffer k_plan N+1 overwrites) exited.
// A device with more SMs than the partial-state slots cover uses the mma.sync
// path.
cudaError_t umma_prepare(Ctx* c) {
  c->umma_ok = false;
  c->umma_pair_ctas = 0;
  const int G = c->cfg.num_q_heads / c->cfg.num_kv_heads;
  if (c->cfg.head_dim != kD || c->cfg.page_size != kP || G < 4 || G > 16) return cudaSuccess;
  for (auto k : {k_tree_umma<0, true>, k_tree_umma<1, true>, k_tree_umma<2, true>}) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at;
    at.id = cudaLaunchAttributeClusterDimension;
    at.val.clusterDim.x = 2;
    at.val.clusterDim.y = 1;
    at.val.clusterDim.z = 1;
    cfg.gridDim = dim3(2 * (c->num_sms / 2));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = kSmemBytes;
    cfg.attrs = &at;
    cfg.numAttrs = 1;
    int ncl = 0;
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveClusters(&ncl, k, &cfg);
    if (e != cudaSuccess) {  // no pair mode on this device (the single-CTA kernel still works)
      (void)cudaGetLastError();
      ncl = 0;
    }
    const int ctas = std::min(2 * ncl, 2 * (c->num_sms / 2));
    c->umma_pair_ctas = c->umma_pair_ctas ? std::min(c->umma_pair_ctas, ctas) : ctas;
  }
  for (auto k : {k_tree_umma<0, false>, k_tree_umma<1, false>, k_tree_umma<2, false>}) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
    if (e != cudaSuccess) return e;
    // the whole shared-memory carveout
    e = cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) return e;
    int occ = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, kThreads, kSmemBytes);
    if (e != cudaSuccess) return e;
    c->umma_occupancy = occ;  // diagnostics only (the occupancy API under-reports with the carveout hint)
    if (c->num_sms > kMaxCtas) return cudaSuccess;
  }
  c->umma_ok = true;
  return cudaSuccess;
}

int umma_pair_max_beams(const Ctx* c) {
  // two CTAs of up to umma_max_beams beams each; the plan's member masks hold 32 beams
  return c->umma_pair_ctas >= 2 ? std::min(32, 2 * umma_max_beams(c)) : 0;
}

int umma_max_beams(const Ctx* c) {
  // four softmax warps, each holding whole beams (G lanes per beam)
  const int G = c->cfg.num_q_heads / c->cfg.num_kv_heads;
  return 4 * (32 / G);
}

cudaError_t launch_attention_umma(Ctx* c, const GroupDesc* groups_h, int n_groups, const int32_t* lens_h,
                                  int n_lens, int layer_begin, int n_layers, int n_call,
                                  const __nv_bfloat16* q, float scale, float* out, const __nv_bfloat16* k_new,
                                  const __nv_bfloat16* v_new, cudaStream_t st, bool pair) {
  PlanParams pp;
  pp.lens = c->buf.seq_lens;
  pp.refcounts = c->env_l2hint ? c->buf.refcounts : nullptr;  // (only the L2 hints read item.w)
  pp.tables = c->buf.block_tables;
  pp.groups = nullptr;
  pp.glens = nullptr;
  pp.status = c->buf.status;
  pp.k_new = (const uint4*)k_new;
  pp.v_new = (const uint4*)v_new;
  pp.k_pool = (uint4*)c->buf.k_pool;
  pp.v_pool = (uint4*)c->buf.v_pool;
  const int64_t rows = (int64_t)c->cfg.max_requests * c->cfg.max_beams;
  pp.items = c->ws_items + c->plan_parity * rows * c->cfg.max_pages_per_beam;
  pp.counts = c->ws_counts + c->plan_parity * rows;
  c->plan_parity ^= 1;
  pp.n_groups = n_groups;
  pp.layer_begin = layer_begin;
  pp.n_call = n_call;
  pp.Hkv = c->cfg.num_kv_heads;
  pp.maxB = c->cfg.max_beams;
  pp.maxP = c->cfg.max_pages_per_beam;
  pp.num_pages = c->cfg.num_pages;
  pp.launch_id = (int)c->launches;

  UParams p;
  p.items = pp.items;
  p.counts = pp.counts;
  p.q = q;
  p.out = out;
  p.groups = nullptr;
  p.status = c->buf.status;
  p.layer_begin = layer_begin;
  p.n_call = n_call;
  p.Hq = c->cfg.num_q_heads;
  p.Hkv = c->cfg.num_kv_heads;
  p.G = p.Hq / p.Hkv;
  p.maxB = c->cfg.max_beams;
  p.maxP = c->cfg.max_pages_per_beam;
  p.n_layers = n_layers;
  p.n_groups = n_groups;
  p.partial = c->ws_partial;
  p.pre = reinterpret_cast<int*>(c->ws_partial + (size_t)2 * kMaxCtas * kPartFloats);
  p.tile_cnt = c->ws_tile_cnt;
  p.num_pages = c->cfg.num_pages;
  p.scale_log2 = scale * 1.4426950408889634f;
  p.round_robin = c->env_round_robin;
  p.split_partial_round = c->env_split_partial;
  p.sched = c->env_sched;
  p.l2hint = c->env_l2hint;
  p.launch_id = (int)c->launches;
  UInline inl;  // host staging of the parameter block (copied by the launch)
  if (n_groups <= kInlineGroups && n_lens <= kInlineLens) {
    std::memcpy(inl.g, groups_h, (size_t)n_groups * sizeof(GroupDesc));
    std::memcpy(inl.len, lens_h, (size_t)n_lens * 4);
  } else {
    cudaError_t e;
    void *dg = nullptr, *dl = nullptr;
    upload2(c, groups_h, (size_t)n_groups * sizeof(GroupDesc), lens_h, (size_t)n_lens * 4, st, &e, &dg, &dl);
    if (e != cudaSuccess) return e;
    p.groups = (const GroupDesc*)dg;
    pp.groups = (const GroupDesc*)dg;
    pp.glens = (const int32_t*)dl;
  }
  // measured 2% slower on C2/C3 (the softmax is latency-, not MUFU-bound): off unless TTS_POLY=1
  auto kern = pair ? (c->env_poly == 2 ? k_tree_umma<2, true> : c->env_poly ? k_tree_umma<1, true> : k_tree_umma<0, true>)
                   : (c->env_poly == 2 ? k_tree_umma<2, false> : c->env_poly ? k_tree_umma<1, false> : k_tree_umma<0, false>);
  const bool no_pdl = c->env_no_pdl;
  cudaLaunchAttribute pdl;
  // each kernel may start while its predecessor on the stream runs; both wait
  // (griddepcontrol.wait) before touching what the predecessor writes
  pdl.id = cudaLaunchAttributeProgrammaticStreamSerialization;
  pdl.val.programmaticStreamSerializationAllowed = 1;
  {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(n_groups * (k_new ? 1 + n_layers : 1));
    cfg.blockDim = dim3(kPlanThreads);
    cfg.stream = st;
    cfg.attrs = &pdl;
    cfg.numAttrs = no_pdl ? 0 : 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, k_plan, pp, inl);
    c->launches++;
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  // persistent: one CTA per SM (<= kMaxCtas, umma_prepare); pair mode: the
  // co-resident 2-CTA clusters
  cfg.gridDim = dim3(pair ? c->umma_pair_ctas : c->num_sms);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmemBytes;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0] = pdl;
  at[1].id = cudaLaunchAttributeClusterDimension;
  at[1].val.clusterDim.x = pair ? 2 : 1;
  at[1].val.clusterDim.y = 1;
  at[1].val.clusterDim.z = 1;
  cfg.attrs = no_pdl ? at + 1 : at;
  cfg.numAttrs = no_pdl ? 1 : 2;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, c->tmap_k, c->tmap3_v, p, inl);
  c->launches++;
  return e;
}

}  // namespace tts
