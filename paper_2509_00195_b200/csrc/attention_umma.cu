// Prefix-shared tree decode attention on the 5th-generation tensor cores
// (tcgen05 + TMEM + TMA), sm_100a.  Same contract as attention.cu (see there
// and include/tts.h); this is the path for head_dim 128 and 4 <= G <= 16.
//
// One CTA owns a 128-row query tile = up to floor(128/G) consecutive beams of
// one request (DFS order, PAPER.md P:394 / ledger C5) x the G query heads of
// one kv head, for one layer, and (when the grid would not fill the GPU) one
// contiguous range of page positions ("split").  Per distinct page of the
// beams' block-table rows (one work item, found by the producer warp with a
// ballot over adjacent rows):
//   TMA      K, V page tiles (16 tokens x 128 d bf16, SWIZZLE_128B) -> smem ring
//   MMA warp S[128x16] = Q[128x128] . K^T      tcgen05.mma kind::f16, D in TMEM
//   softmax  one thread per row: tcgen05.ld S, mask rows whose beam does not
//            reference the page and token slots >= ntok, online softmax in fp32
//            (lazy rescale: O is rescaled in TMEM only when the running max
//            grows by > 2^8), P = hi + lo bf16 -> smem (SURVEY ledger C14)
//   MMA warp O[128x128] += P_hi . V + P_lo . V  (V as an MN-major operand)
// A shared page is fetched once per CTA and multiplied against all 128 rows:
// the GQA heads and every beam of the tile that references it.
// Splits of one tile form a thread-block cluster; their partial (m, l, O)
// states are merged through distributed shared memory, so no partial state
// ever reaches HBM (SURVEY 7 hard part 4).
#include "tts_internal.cuh"

namespace tts {
namespace {

constexpr int kP = 16;
constexpr int kD = 128;
constexpr int kRows = 128;
constexpr int kNS = 6;                       // ring slots
constexpr int kTile = kP * kD * 2;           // 4 KiB
constexpr int kSlot = 2 * kTile;             // K + V
constexpr int kRing = kNS * kSlot;           // 48 KiB
constexpr int kPBuf = kRows * kP * 2;        // 4 KiB (one bf16 P operand)
constexpr int kPArea = 4 * kPBuf;            // 2 buffers x (hi, lo)
constexpr int kQBytes = kRows * kD * 2;      // 32 KiB
constexpr int kThreads = 192;                // warps 0-3 softmax, 4 producer, 5 MMA
constexpr int kTmemCols = 256;               // O [0,128), S0 [128,144), S1 [144,160)

// smem layout (offsets from the 1024-aligned base)
constexpr int kOffRing = 0;
constexpr int kOffP = kOffRing + kRing;                 // contiguous with the ring:
constexpr int kOffQ = kOffP + kPArea;                   // ring + P = 64 KiB merge area
constexpr int kOffMeta = kOffQ + kQBytes;
constexpr int kOffBar = kOffMeta + kNS * 16;
constexpr int kNumBars = 2 * kNS + 6;                   // full, empty, sfull[2], pfull[2], pvdone[2]
constexpr int kOffML = kOffBar + kNumBars * 8 + 8;      // + tmem base slot
constexpr int kOffTbl = kOffML + 2 * kRows * 4;
constexpr int kSmemBytes = kOffTbl + 32 * 33 * 4 + 1024;
static_assert(kRing + kPArea >= kRows * kD * 4, "merge area must hold a 128x128 fp32 tile");

struct UParams {
  const int32_t* tables;
  const int32_t* lens;
  const __nv_bfloat16* q;
  float* out;
  const GroupDesc* groups;
  int32_t* status;
  int layer_begin, n_call, Hq, Hkv, G, maxB, maxP, splits;
  int64_t num_pages;
  float scale_log2;
};

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void bar_init(uint32_t b, int n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(n));
}
__device__ __forceinline__ void bar_wait(uint32_t b, uint32_t par) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "W_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra W_%=;\n}" ::"r"(b),
      "r"(par)
      : "memory");
}
__device__ __forceinline__ void bar_arrive(uint32_t b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(b) : "memory");
}
__device__ __forceinline__ void bar_expect(uint32_t b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma2d(uint32_t dst, const CUtensorMap* m, int x, int y, uint32_t b) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(x), "r"(y), "r"(b)
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint32_t b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(b)
               : "memory");
}
__device__ __forceinline__ void tc_mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void tc_ld16(uint32_t t, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(t));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tc_ld32(uint32_t t, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(t));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tc_st32(uint32_t t, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(t),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
      "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
      "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// UMMA shared-memory descriptor (sm100: version 1 at bit 46).
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46) | ((uint64_t)layout << 61);
}
// Instruction descriptor kind::f16: D f32, A/B bf16, N, M=128.
__host__ __device__ constexpr uint32_t idesc_bf16(int N, bool b_mn_major) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((b_mn_major ? 1u : 0u) << 16) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(kRows >> 4) << 24);
}

__device__ __forceinline__ uint32_t pack2(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
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
  int32_t* tbl = reinterpret_cast<int32_t*>(bp + kOffTbl);
  const uint32_t b_full = su32(bars), b_empty = b_full + 8 * kNS, b_sfull = b_empty + 8 * kNS,
                 b_pfull = b_sfull + 16, b_pv = b_pfull + 16;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (*(volatile int32_t*)p.status) return;
  const int split = blockIdx.x % p.splits;
  const GroupDesc g = p.groups[blockIdx.x / p.splits];
  const int kh = blockIdx.y, lrel = blockIdx.z, layer = p.layer_begin + lrel;
  const int G = p.G;
  const int pos_per_split = (g.max_npages + p.splits - 1) / p.splits;
  const int pos_begin = split * pos_per_split;
  const int pos_end = min(g.max_npages, pos_begin + pos_per_split);

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
  // rows of this tile: r -> (beam g.beam0 + r / G, head kh*G + r % G)
  const int r = threadIdx.x;  // meaningful for warps 0-3
  const int rbl = r / G;
  const bool rvalid = warp < 4 && rbl < g.nbeams && ((g.active >> rbl) & 1u);
  if (warp < 4) {
    // Q row -> smem, K-major SWIZZLE_128B: [kb][row][128 B], chunk c at (c ^ (row & 7))
    const uint4* src = nullptr;
    if (rvalid)
      src = reinterpret_cast<const uint4*>(
          p.q + ((((int64_t)lrel * p.n_call + g.call_idx) * p.maxB + g.beam0 + rbl) * p.Hq + kh * G + r % G) * kD);
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      uint4 v = rvalid ? src[c] : make_uint4(0, 0, 0, 0);
      const int kb = c >> 3, cc = c & 7;
      *reinterpret_cast<uint4*>(bp + kOffQ + kb * (kRows * 128) + r * 128 + ((cc ^ (r & 7)) << 4)) = v;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t t_o = tmem, t_s = tmem + 128;

  if (warp == 4) {
    // ============================ producer ============================
    const bool act = lane < g.nbeams && ((g.active >> lane) & 1u);
    const int len = act ? p.lens[(int64_t)g.req * p.maxB + g.beam0 + lane] : 0;
    const int np = (len + kP - 1) / kP;
    const int64_t layer_rows = ((int64_t)layer * p.num_pages) * p.Hkv;
    int slot = 0;
    uint32_t ph = 0;
    for (int i0 = pos_begin; i0 < pos_end; i0 += 32) {
      __syncwarp();
      for (int b = 0; b < g.nbeams; ++b) {
        const int lb = __shfl_sync(0xffffffffu, len, b);
        const int npb = (lb + kP - 1) / kP;
        int32_t v = -1;
        if (((g.active >> b) & 1u) && i0 + lane < npb && i0 + lane < pos_end)
          v = p.tables[((int64_t)g.req * p.maxB + g.beam0 + b) * p.maxP + i0 + lane];
        tbl[b * 33 + lane] = v;
      }
      __syncwarp();
      const int iend = min(32, pos_end - i0);
      for (int ii = 0; ii < iend; ++ii) {
        const int i = i0 + ii;
        const bool has = act && i < np;
        const int page = has ? tbl[lane * 33 + ii] : -1;
        const uint32_t hm = __ballot_sync(0xffffffffu, has);
        const uint32_t below = hm & ((1u << lane) - 1u);
        const int prev = below ? 31 - __clz(below) : lane;
        const int pp = __shfl_sync(0xffffffffu, page, prev);
        uint32_t sm = __ballot_sync(0xffffffffu, has && (below == 0 || pp != page));
        while (sm) {
          const int s0 = __ffs(sm) - 1;
          sm &= sm - 1;
          const int s1 = sm ? __ffs(sm) - 1 : 32;
          const uint32_t members = hm & (s1 >= 32 ? 0xffffffffu : ((1u << s1) - 1u)) & ~((1u << s0) - 1u);
          const int pg = __shfl_sync(0xffffffffu, page, s0);
          const int ln = __shfl_sync(0xffffffffu, len, s0);
          if (lane == 0) {
            bar_wait(b_empty + 8 * slot, ph ^ 1u);
            meta[slot] = make_int4(pg, (int)members, min(kP, ln - i * kP), i);
            const uint32_t fb = b_full + 8 * slot;
            bar_expect(fb, (uint32_t)kSlot);
            const int y = (int)((layer_rows + (int64_t)pg * p.Hkv + kh) * kP);
            const uint32_t dk = base + kOffRing + slot * kSlot;
            tma2d(dk, &tmk, 0, y, fb);
            tma2d(dk + 2048, &tmk, 64, y, fb);
            tma2d(dk + kTile, &tmv, 0, y, fb);
            tma2d(dk + kTile + 2048, &tmv, 64, y, fb);
          }
          if (++slot == kNS) {
            slot = 0;
            ph ^= 1u;
          }
        }
      }
    }
    if (lane == 0) {
      bar_wait(b_empty + 8 * slot, ph ^ 1u);
      meta[slot] = make_int4(-1, 0, 0, 0);
      bar_arrive(b_full + 8 * slot);
    }
  } else if (warp == 5) {
    // ============================ MMA issuer ============================
    if (lane == 0) {
      constexpr uint32_t id_s = idesc_bf16(kP, false);
      constexpr uint32_t id_pv = idesc_bf16(kD, true);
      const uint32_t qa = base + kOffQ;
      auto issue_s = [&](int j) {
        const int slot = j % kNS;
        const uint32_t kt = base + kOffRing + slot * kSlot;
        const uint32_t sd = t_s + (j & 1) * kP;
#pragma unroll
        for (int ks = 0; ks < kD / 16; ++ks) {
          const uint32_t off = (ks & 3) * 32;
          const uint64_t da = sdesc(qa + (ks >> 2) * (kRows * 128) + off, 16, 1024, 2);
          const uint64_t db = sdesc(kt + (ks >> 2) * 2048 + off, 16, 1024, 2);
          tc_mma(sd, da, db, id_s, ks > 0);
        }
        tc_commit(b_sfull + 8 * (j & 1));
      };
      // first item
      bar_wait(b_full, 0);
      tc_fence_after();
      bool done = meta[0].x < 0;
      if (done)
        bar_arrive(b_sfull);
      else
        issue_s(0);
      for (int j = 0; !done; ++j) {
        const int sn = (j + 1) % kNS;
        bar_wait(b_full + 8 * sn, ((j + 1) / kNS) & 1u);
        tc_fence_after();
        const bool last = meta[sn].x < 0;
        if (last)
          bar_arrive(b_sfull + 8 * ((j + 1) & 1));
        else
          issue_s(j + 1);
        bar_wait(b_pfull + 8 * (j & 1), (j >> 1) & 1u);
        tc_fence_after();
        const int slot = j % kNS;
        const uint32_t vt = base + kOffRing + slot * kSlot + kTile;
        const uint64_t dv = sdesc(vt, 2048, 1024, 2);
        const uint32_t pb = base + kOffP + (j & 1) * 2 * kPBuf;
        tc_mma(t_o, sdesc(pb, 2048, 128, 0), dv, id_pv, j > 0);
        tc_mma(t_o, sdesc(pb + kPBuf, 2048, 128, 0), dv, id_pv, 1);
        tc_commit(b_empty + 8 * slot);
        tc_commit(b_pv + 8 * (j & 1));
        done = last;
      }
    }
    __syncwarp();
  } else {
    // ============================ softmax (warps 0-3) ============================
    const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
    float m_ref = -1e30f, l = 0.f;
    int j = 0;
    for (;; ++j) {
      bar_wait(b_sfull + 8 * (j & 1), (j >> 1) & 1u);
      tc_fence_after();
      const int4 mt = meta[j % kNS];
      if (mt.x < 0) break;
      float s[16];
      tc_ld16(t_s + lane_off + (j & 1) * kP, s);
      const bool mem = rvalid && ((((uint32_t)mt.y) >> rbl) & 1u);
      float mx = -INFINITY;
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        s[c] = (mem && c < mt.z) ? s[c] * p.scale_log2 : -INFINITY;
        mx = fmaxf(mx, s[c]);
      }
      const bool need = mx > m_ref + 8.0f;
      if (__any_sync(0xffffffffu, need) && j > 0) {
        // all earlier PV products must have landed before O is rescaled in TMEM
        bar_wait(b_pv + 8 * ((j - 1) & 1), ((j - 1) >> 1) & 1u);
        tc_fence_after();
        const float alpha = need ? exp2f(m_ref - mx) : 1.f;
#pragma unroll 1
        for (int ch = 0; ch < 4; ++ch) {
          uint32_t o[32];
          tc_ld32(t_o + lane_off + ch * 32, o);
#pragma unroll
          for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
          tc_st32(t_o + lane_off + ch * 32, o);
        }
        l *= alpha;
      }
      if (need) m_ref = mx;
      float pv[16];
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        pv[c] = exp2f(s[c] - m_ref);
        l += pv[c];
      }
      // stale token slots >= ntok of a partial page: zero V so that P(=0) * V
      // cannot produce NaN (pool slots past a beam's length are never written)
      if (mt.z < kP) {
        uint8_t* vt = bp + kOffRing + (j % kNS) * kSlot + kTile;
        for (int idx = r; idx < (kP - mt.z) * 16; idx += 128) {
          const int tok = mt.z + idx / 16, ch = idx % 16;
          *reinterpret_cast<uint4*>(vt + (ch >> 3) * 2048 + tok * 128 + (ch & 7) * 16) = make_uint4(0, 0, 0, 0);
        }
      }
      // P buffer (j & 1) was last read by PV(j - 2)
      if (j >= 2) bar_wait(b_pv + 8 * (j & 1), ((j - 2) >> 1) & 1u);
      uint8_t* pbh = bp + kOffP + (j & 1) * 2 * kPBuf;
      uint8_t* pbl = pbh + kPBuf;
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        uint32_t hi[4], lo[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float a = pv[half * 8 + 2 * k], b = pv[half * 8 + 2 * k + 1];
          hi[k] = pack2(a, b);
          __nv_bfloat162 hv = *reinterpret_cast<__nv_bfloat162*>(&hi[k]);
          float2 hf = __bfloat1622float2(hv);
          lo[k] = pack2(a - hf.x, b - hf.y);
        }
        // K-major, no swizzle: 8x16B core matrices; chunk `half` at +2048, row r at r*16
        *reinterpret_cast<uint4*>(pbh + half * 2048 + r * 16) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
        *reinterpret_cast<uint4*>(pbl + half * 2048 + r * 16) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) bar_arrive(b_pfull + 8 * (j & 1));
    }
    const int n_items = j;
    // ---------------- epilogue ----------------
    if (n_items > 0) {
      bar_wait(b_pv + 8 * ((n_items - 1) & 1), ((n_items - 1) >> 1) & 1u);
      tc_fence_after();
    }
    if (p.splits == 1) {
      if (n_items > 0) {
        const float inv = 1.f / l;
        float* orow = p.out + ((((int64_t)lrel * p.n_call + g.call_idx) * p.maxB + g.beam0 + rbl) * p.Hq +
                               kh * G + r % G) * kD;
#pragma unroll 1
        for (int ch = 0; ch < 4; ++ch) {
          uint32_t o[32];
          tc_ld32(t_o + lane_off + ch * 32, o);
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
      // partial state -> smem (swizzled 16-B chunks), merged across the cluster
      float* op = reinterpret_cast<float*>(bp + kOffRing);
#pragma unroll 1
      for (int ch = 0; ch < 4; ++ch) {
        uint32_t o[32];
        if (n_items > 0) {
          tc_ld32(t_o + lane_off + ch * 32, o);
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) o[i] = 0u;
        }
#pragma unroll
        for (int q4 = 0; q4 < 8; ++q4) {
          const int c = ch * 8 + q4;  // 16-B chunk index 0..31
          const int pc = (c & ~7) | ((c & 7) ^ (r & 7));
          *reinterpret_cast<uint4*>(op + r * kD + pc * 4) =
              make_uint4(o[4 * q4], o[4 * q4 + 1], o[4 * q4 + 2], o[4 * q4 + 3]);
        }
      }
      m_s[r] = m_ref;
      l_s[r] = l;
    }
  }

  if (p.splits > 1) {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (warp < 4) {
      const int S = p.splits;
      const int rpc = kRows / S;           // rows merged by this CTA
      const int tpr = 128 / rpc;           // threads per row (= S)
      const int row = split * rpc + threadIdx.x / tpr;
      const int cseg = threadIdx.x % tpr;  // column segment of width 128 / tpr
      const int cw = kD / tpr;
      const int bl = row / G;
      const bool ok = bl < g.nbeams && ((g.active >> bl) & 1u);
      const uint32_t lm = su32(m_s + row), ll = su32(l_s + row);
      const uint32_t lo_base = base + kOffRing;
      float mk[8], wk[8];
      float M = -INFINITY;
      for (int k = 0; k < S; ++k) {
        uint32_t a;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(lm), "r"(k));
        asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(mk[k]) : "r"(a));
        M = fmaxf(M, mk[k]);
      }
      float L = 0.f;
      for (int k = 0; k < S; ++k) {
        uint32_t a;
        float lk;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(ll), "r"(k));
        asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(lk) : "r"(a));
        wk[k] = exp2f(mk[k] - M);
        L += wk[k] * lk;
      }
      const float inv = 1.f / L;
      float* orow = p.out + ((((int64_t)lrel * p.n_call + g.call_idx) * p.maxB + g.beam0 + bl) * p.Hq +
                             kh * G + row % G) * kD;
      for (int c4 = 0; c4 < cw / 4; ++c4) {
        const int c = cseg * (cw / 4) + c4;  // 16-B chunk index
        const int pc = (c & ~7) | ((c & 7) ^ (row & 7));
        const uint32_t la = lo_base + (uint32_t)(row * kD + pc * 4) * 4;
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int k = 0; k < S; ++k) {
          uint32_t a;
          float4 v;
          asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(la), "r"(k));
          asm volatile("ld.shared::cluster.v4.f32 {%0,%1,%2,%3}, [%4];"
                       : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                       : "r"(a));
          acc.x += wk[k] * v.x;
          acc.y += wk[k] * v.y;
          acc.z += wk[k] * v.z;
          acc.w += wk[k] * v.w;
        }
        if (ok)
          *reinterpret_cast<float4*>(orow + c * 4) =
              make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
      }
    }
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 5) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
  }
}

}  // namespace

bool umma_supported(const Ctx* c) {
  const int G = c->cfg.num_q_heads / c->cfg.num_kv_heads;
  return c->cfg.head_dim == kD && c->cfg.page_size == kP && G >= 4 && G <= 16;
}

int umma_max_beams(const Ctx* c) {
  const int G = c->cfg.num_q_heads / c->cfg.num_kv_heads;
  return std::min(32, kRows / G);
}

cudaError_t launch_attention_umma(Ctx* c, const GroupDesc* groups_d, int n_groups, int splits,
                                  int layer_begin, int n_layers, int n_call, const __nv_bfloat16* q,
                                  float scale, float* out, cudaStream_t st) {
  UParams p;
  p.tables = c->buf.block_tables;
  p.lens = c->buf.seq_lens;
  p.q = q;
  p.out = out;
  p.groups = groups_d;
  p.status = c->buf.status;
  p.layer_begin = layer_begin;
  p.n_call = n_call;
  p.Hq = c->cfg.num_q_heads;
  p.Hkv = c->cfg.num_kv_heads;
  p.G = p.Hq / p.Hkv;
  p.maxB = c->cfg.max_beams;
  p.maxP = c->cfg.max_pages_per_beam;
  p.splits = splits;
  p.num_pages = c->cfg.num_pages;
  p.scale_log2 = scale * 1.4426950408889634f;
  static bool attr_done = false;
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(k_tree_umma, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
    if (e != cudaSuccess) return e;
    cudaFuncSetAttribute(k_tree_umma, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
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
  cudaError_t e = cudaLaunchKernelEx(&cfg, k_tree_umma, c->tmap_k, c->tmap_v, p);
  c->launches++;
  return e;
}

}  // namespace tts
