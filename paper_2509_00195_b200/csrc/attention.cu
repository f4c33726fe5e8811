// Prefix-shared (tree / cascade) decode attention for sm_100a.
//
// What it computes: for every active beam b of the call, layer l and q head h
// (kv head h / G, ledger C10), o = softmax_j(scale q.K_j) V_j over all len_b
// tokens of the beam (ledger C11) -- the textbook attention the oracle writes
// out in fp64.  How: the beams of a request are in DFS order (PAPER.md P:394
// "grouping beams spawned from the same parent ... preserving the relative
// order of the parent beams"; ledger C5), so the beams that share a KV page
// form a contiguous run.  One CTA owns (layer, kv head, beam group): a
// producer warp walks the group's block-table rows position by position,
// emits one work item per DISTINCT page (page id + member-beam bitmask) and
// stages it into a shared-memory ring with TMA (cp.async.bulk.tensor, 128-B
// swizzle) -- each shared page is read from HBM once per group and used by
// every beam and GQA head of the group that references it (the reuse Dynamic
// Prefix-Aware Scheduling creates).  Consumer warps each own 16
// query rows (bpt = 16 / G beams x G heads) and run S = Q K^T and O += P V on
// tensor cores (bf16 Q.K, fp16 P.V with V kept in fp16 in the pool; fp32
// accumulate) with an fp32 online softmax (SURVEY ledger C14: a bf16 P fails
// the 2e-3 bar, fp16 P with fp16 V does not).  Output is fp32 (ledger C13).
#include "tts_internal.cuh"

namespace tts {
namespace {

constexpr int kP = 16;  // page size (tokens)

struct AttnParams {
  const int32_t* tables;
  const int32_t* lens;
  const __nv_bfloat16* q;
  float* out;
  const GroupDesc* groups;
  int32_t* status;
  int layer_begin;
  int n_call;
  int Hq, Hkv, G, maxB, maxP;
  int64_t num_pages;
  float scale_log2;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 10000000;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(bar),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int x, int y,
                                            uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(bar)
      : "memory");
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                        uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}

__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                          uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}

__device__ __forceinline__ void mma_bf16(float (&c)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void mma_f16(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t pack_f16(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

__device__ __forceinline__ float2 unpack_bf16(uint32_t u) {
  __nv_bfloat162 v = *reinterpret_cast<__nv_bfloat162*>(&u);
  return __bfloat1622float2(v);
}

// Byte offset of 16-B chunk `c` of token row `r` inside a [P][D] tile written
// by TMA with SWIZZLE_128B in boxes of 64 columns (128 B rows).
template <int D>
__device__ __forceinline__ uint32_t swz(int r, int c) {
  return (uint32_t)((c >> 3) * (kP * 128) + r * 128 + (((c & 7) ^ (r & 7)) << 4));
}

template <int D>
struct Ring {
  static constexpr int kTileBytes = kP * D * 2;
  static constexpr int kSlotBytes = 2 * kTileBytes;  // K + V
};

// ---------------------------------------------------------------------------
template <int D, int NCONS, int NS>
__global__ void __launch_bounds__((NCONS + 1) * 32)
    k_tree_attn(const __grid_constant__ CUtensorMap tmk, const __grid_constant__ CUtensorMap tmv,
                AttnParams p) {
  extern __shared__ uint8_t smem_raw[];
  constexpr int kSlot = Ring<D>::kSlotBytes;
  constexpr int kTile = Ring<D>::kTileBytes;
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  uint8_t* base_ptr = smem_raw + (base - smem_u32(smem_raw));
  int4* meta = reinterpret_cast<int4*>(base_ptr + NS * kSlot);
  uint64_t* bars = reinterpret_cast<uint64_t*>(meta + NS);  // full[NS], empty[NS]
  int32_t* tbl = reinterpret_cast<int32_t*>(bars + 2 * NS);  // [32][33] page ids

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (*(volatile int32_t*)p.status) return;

  const GroupDesc g = p.groups[blockIdx.x];
  const int kh = blockIdx.y;
  const int lrel = blockIdx.z;
  const int layer = p.layer_begin + lrel;

  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(smem_u32(&bars[i]), 1);
      mbar_init(smem_u32(&bars[NS + i]), NCONS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == NCONS) {
    // ======================= producer warp =======================
    const bool act = lane < g.nbeams && ((g.active >> lane) & 1u);
    const int len = act ? p.lens[(int64_t)g.req * p.maxB + g.beam0 + lane] : 0;
    const int np = (len + kP - 1) / kP;
    const int64_t layer_rows = ((int64_t)layer * p.num_pages) * p.Hkv;
    int slot = 0;
    uint32_t phase = 0;
    for (int i0 = 0; i0 < g.max_npages; i0 += 32) {
      // stage the page ids of positions [i0, i0+32) for every beam of the group
      __syncwarp();
      for (int b = 0; b < g.nbeams; ++b) {
        const bool ab = (g.active >> b) & 1u;
        const int lb = __shfl_sync(0xffffffffu, len, b);
        const int npb = (lb + kP - 1) / kP;
        int32_t v = -1;
        if (ab && i0 + lane < npb)
          v = p.tables[((int64_t)g.req * p.maxB + g.beam0 + b) * p.maxP + i0 + lane];
        tbl[b * 33 + lane] = v;
      }
      __syncwarp();
      const int iend = min(32, g.max_npages - i0);
      for (int ii = 0; ii < iend; ++ii) {
        const int i = i0 + ii;
        const bool has = act && i < np;
        const int page = has ? tbl[lane * 33 + ii] : -1;
        const uint32_t hmask = __ballot_sync(0xffffffffu, has);
        const uint32_t below = hmask & ((1u << lane) - 1u);
        const int prev = below ? 31 - __clz(below) : lane;
        const int prev_page = __shfl_sync(0xffffffffu, page, prev);
        const bool start = has && (below == 0 || prev_page != page);
        uint32_t smask = __ballot_sync(0xffffffffu, start);
        while (smask) {
          const int s0 = __ffs(smask) - 1;
          smask &= smask - 1;
          const int s1 = smask ? __ffs(smask) - 1 : 32;
          const uint32_t hi_mask = s1 >= 32 ? 0xffffffffu : ((1u << s1) - 1u);
          const uint32_t members = hmask & hi_mask & ~((1u << s0) - 1u);
          const int pg = __shfl_sync(0xffffffffu, page, s0);
          const int ln = __shfl_sync(0xffffffffu, len, s0);
          if (lane == 0) {
            const int ntok = min(kP, ln - i * kP);
            mbar_wait(smem_u32(&bars[NS + slot]), phase ^ 1u);
            meta[slot] = make_int4(pg, (int)members, ntok, i);
            const uint32_t full = smem_u32(&bars[slot]);
            mbar_expect_tx(full, (uint32_t)kSlot);
            const int y = (int)((layer_rows + (int64_t)pg * p.Hkv + kh) * kP);
            const uint32_t dk = base + slot * kSlot;
#pragma unroll
            for (int x = 0; x < D / 64; ++x) {
              tma_load_2d(dk + x * (kP * 128), &tmk, x * 64, y, full);
              tma_load_2d(dk + kTile + x * (kP * 128), &tmv, x * 64, y, full);
            }
          }
          if (++slot == NS) {
            slot = 0;
            phase ^= 1u;
          }
        }
      }
    }
    if (lane == 0) {
      mbar_wait(smem_u32(&bars[NS + slot]), phase ^ 1u);
      meta[slot] = make_int4(-1, 0, 0, 0);
      mbar_arrive(smem_u32(&bars[slot]));
    }
    return;
  }

  // ======================= consumer warps =======================
  const int G = p.G;
  const int bpt = 16 / G;  // beams per 16-row tile
  const int gq = lane >> 2, tq = lane & 3;
  const int b_first = warp * bpt;  // group-local beam index of row 0
  int rbeam[2], rhead[2];
  bool rvalid[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int r = gq + 8 * h;
    const int bl = r / G;
    rbeam[h] = b_first + bl;
    rhead[h] = kh * G + r % G;
    rvalid[h] = (r < bpt * G) && rbeam[h] < g.nbeams && ((g.active >> rbeam[h]) & 1u);
  }
  uint32_t my_mask = 0;
  for (int b = b_first; b < b_first + bpt && b < g.nbeams; ++b)
    if ((g.active >> b) & 1u) my_mask |= 1u << b;

  // Q fragments (A operand, 16 rows x D), straight from global.
  uint32_t qa[D / 16][4];
  {
    const uint32_t* qrow[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t off =
          ((((int64_t)lrel * p.n_call + g.call_idx) * p.maxB + g.beam0 + (rvalid[h] ? rbeam[h] : 0)) *
               p.Hq +
           rhead[h]) *
          D;
      qrow[h] = reinterpret_cast<const uint32_t*>(p.q + off);
    }
#pragma unroll
    for (int ks = 0; ks < D / 16; ++ks) {
      qa[ks][0] = rvalid[0] ? qrow[0][(ks * 16 + 2 * tq) / 2] : 0u;
      qa[ks][1] = rvalid[1] ? qrow[1][(ks * 16 + 2 * tq) / 2] : 0u;
      qa[ks][2] = rvalid[0] ? qrow[0][(ks * 16 + 8 + 2 * tq) / 2] : 0u;
      qa[ks][3] = rvalid[1] ? qrow[1][(ks * 16 + 8 + 2 * tq) / 2] : 0u;
    }
  }

  float o[D / 8][4];
#pragma unroll
  for (int i = 0; i < D / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m0 = -1e30f, m1 = -1e30f, l0 = 0.f, l1 = 0.f;

  // per-lane ldmatrix row offsets
  const int mi = lane >> 3, rr = lane & 7;
  int slot = 0;
  uint32_t phase = 0;
  while (true) {
    mbar_wait(smem_u32(&bars[slot]), phase);
    const int4 mt = meta[slot];
    if (mt.x < 0) break;
    const uint32_t members = (uint32_t)mt.y;
    if (members & my_mask) {
      const bool in0 = rvalid[0] && ((members >> rbeam[0]) & 1u);
      const bool in1 = rvalid[1] && ((members >> rbeam[1]) & 1u);
      const int ntok = mt.z;
      const uint32_t kt = base + slot * kSlot;
      const uint32_t vt = kt + kTile;
      float s[2][4];
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) s[nt][0] = s[nt][1] = s[nt][2] = s[nt][3] = 0.f;
#pragma unroll
      for (int ks = 0; ks < D / 16; ++ks) {
        uint32_t b00, b01, b10, b11;
        ldsm_x4(kt + swz<D>((mi >> 1) * 8 + rr, ks * 2 + (mi & 1)), b00, b01, b10, b11);
        mma_bf16(s[0], qa[ks], b00, b01);
        mma_bf16(s[1], qa[ks], b10, b11);
      }
      // scale into the log2 domain, mask, online softmax (rows gq and gq+8)
      float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int col = nt * 8 + 2 * tq + e;
          const bool cv = col < ntok;
          s[nt][e] = (in0 && cv) ? s[nt][e] * p.scale_log2 : -INFINITY;
          s[nt][2 + e] = (in1 && cv) ? s[nt][2 + e] * p.scale_log2 : -INFINITY;
          mx0 = fmaxf(mx0, s[nt][e]);
          mx1 = fmaxf(mx1, s[nt][2 + e]);
        }
      }
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
      mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
      mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
      const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);
      const float a0 = exp2f(m0 - mn0), a1 = exp2f(m1 - mn1);
      m0 = mn0;
      m1 = mn1;
      float ps[2][4];
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        ps[nt][0] = exp2f(s[nt][0] - mn0);
        ps[nt][1] = exp2f(s[nt][1] - mn0);
        ps[nt][2] = exp2f(s[nt][2] - mn1);
        ps[nt][3] = exp2f(s[nt][3] - mn1);
      }
      l0 = l0 * a0 + (ps[0][0] + ps[0][1] + ps[1][0] + ps[1][1]);
      l1 = l1 * a1 + (ps[0][2] + ps[0][3] + ps[1][2] + ps[1][3]);
      if (__any_sync(0xffffffffu, a0 != 1.f || a1 != 1.f)) {
#pragma unroll
        for (int i = 0; i < D / 8; ++i) {
          o[i][0] *= a0;
          o[i][1] *= a0;
          o[i][2] *= a1;
          o[i][3] *= a1;
        }
      }
      // P as the A operand (k = 16 tokens) in fp16; V is fp16 in the pool
      uint32_t pa[4];
      pa[0] = pack_f16(ps[0][0], ps[0][1]);
      pa[1] = pack_f16(ps[0][2], ps[0][3]);
      pa[2] = pack_f16(ps[1][0], ps[1][1]);
      pa[3] = pack_f16(ps[1][2], ps[1][3]);
      // token slots >= ntok of a partial page are zero-filled in the pool; the
      // mask below keeps a stale slot from ever reaching O regardless
      uint32_t vm_a = 0xffffffffu, vm_b = 0xffffffffu;
      if (ntok < kP) {
        vm_a = (2 * tq < ntok ? 0x0000ffffu : 0u) | (2 * tq + 1 < ntok ? 0xffff0000u : 0u);
        vm_b = (8 + 2 * tq < ntok ? 0x0000ffffu : 0u) | (9 + 2 * tq < ntok ? 0xffff0000u : 0u);
      }
#pragma unroll
      for (int dp = 0; dp < D / 16; ++dp) {
        uint32_t v0, v1, v2, v3;
        ldsm_x4_t(vt + swz<D>((mi & 1) * 8 + rr, 2 * dp + (mi >> 1)), v0, v1, v2, v3);
        v0 &= vm_a;
        v1 &= vm_b;
        v2 &= vm_a;
        v3 &= vm_b;
        mma_f16(o[2 * dp], pa, v0, v1);
        mma_f16(o[2 * dp + 1], pa, v2, v3);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(smem_u32(&bars[NS + slot]));
    if (++slot == NS) {
      slot = 0;
      phase ^= 1u;
    }
  }

  // epilogue: reduce l over the quad, normalise, store fp32 rows
  l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
  l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
  const float inv0 = 1.f / l0, inv1 = 1.f / l1;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    if (!rvalid[h]) continue;
    const float inv = h ? inv1 : inv0;
    float* orow = p.out + ((((int64_t)lrel * p.n_call + g.call_idx) * p.maxB + g.beam0 + rbeam[h]) *
                               p.Hq +
                           rhead[h]) *
                              D;
#pragma unroll
    for (int i = 0; i < D / 8; ++i) {
      float2 v = make_float2(o[i][2 * h] * inv, o[i][2 * h + 1] * inv);
      *reinterpret_cast<float2*>(orow + i * 8 + 2 * tq) = v;
    }
  }
}

template <int D, int NCONS, int NS>
cudaError_t launch_t(Ctx* c, const GroupDesc* groups_d, int n_groups, int layer_begin,
                     int n_layers, int n_call, const __nv_bfloat16* q, float scale, float* out,
                     cudaStream_t st) {
  AttnParams p;
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
  p.num_pages = c->cfg.num_pages;
  p.scale_log2 = scale * 1.4426950408889634f;
  const size_t smem = 1024 + NS * Ring<D>::kSlotBytes + NS * 16 + 2 * NS * 8 + 32 * 33 * 4;
  auto kern = k_tree_attn<D, NCONS, NS>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid(n_groups, p.Hkv, n_layers);
  kern<<<grid, (NCONS + 1) * 32, smem, st>>>(c->tmap_k, c->tmap_v, p);
  c->launches++;
  return cudaGetLastError();
}

template <int D>
cudaError_t launch_d(Ctx* c, const GroupDesc* groups_d, int n_groups, int ncons, int layer_begin,
                     int n_layers, int n_call, const __nv_bfloat16* q, float scale, float* out,
                     cudaStream_t st) {
  switch (ncons) {
    case 1: return launch_t<D, 1, 8>(c, groups_d, n_groups, layer_begin, n_layers, n_call, q, scale, out, st);
    case 2: return launch_t<D, 2, 8>(c, groups_d, n_groups, layer_begin, n_layers, n_call, q, scale, out, st);
    case 4: return launch_t<D, 4, 12>(c, groups_d, n_groups, layer_begin, n_layers, n_call, q, scale, out, st);
    default: return launch_t<D, 8, 12>(c, groups_d, n_groups, layer_begin, n_layers, n_call, q, scale, out, st);
  }
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                              CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                              CUtensorMapFloatOOBfill);

}  // namespace

bool make_tensor_maps(Ctx* c) {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
      fn == nullptr)
    return false;
  EncodeFn enc = reinterpret_cast<EncodeFn>(fn);
  const tts_config_t& g = c->cfg;
  cuuint64_t rows = (cuuint64_t)g.num_layers * g.num_pages * g.num_kv_heads * g.page_size;
  cuuint64_t dims[2] = {(cuuint64_t)g.head_dim, rows};
  cuuint64_t strides[1] = {(cuuint64_t)g.head_dim * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)g.page_size};
  cuuint32_t es[2] = {1, 1};
  CUresult r1 = enc(&c->tmap_k, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, c->buf.k_pool, dims, strides, box,
                    es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CUresult r2 = enc(&c->tmap_v, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, c->buf.v_pool, dims, strides, box,
                    es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  c->tmap_ok = (r1 == CUDA_SUCCESS && r2 == CUDA_SUCCESS);
  // 3D view: x = 64 columns (128 B), y = token rows, z = the two 64-column halves
  cuuint64_t dims3[3] = {64, rows, 2};
  cuuint64_t strides3[2] = {(cuuint64_t)g.head_dim * 2, 128};
  cuuint32_t box3[3] = {64, (cuuint32_t)g.page_size, 2};
  cuuint32_t es3[3] = {1, 1, 1};
  c->tmap3_ok = false;
  if (g.head_dim == 128) {
    CUresult r3 = enc(&c->tmap3_k, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, c->buf.k_pool, dims3, strides3, box3, es3,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    CUresult r4 = enc(&c->tmap3_v, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, c->buf.v_pool, dims3, strides3, box3, es3,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    c->tmap3_ok = (r3 == CUDA_SUCCESS && r4 == CUDA_SUCCESS);
  }
  return c->tmap_ok;
}

cudaError_t launch_attention(Ctx* c, const GroupDesc* groups_d, int n_groups, int group_beams,
                             int layer_begin, int n_layers, int n_call, const __nv_bfloat16* q,
                             float scale, float* out, cudaStream_t st) {
  if (n_groups == 0 || n_layers == 0) return cudaSuccess;
  const int G = c->cfg.num_q_heads / c->cfg.num_kv_heads;
  const int bpt = 16 / G;
  const int ncons = (group_beams + bpt - 1) / bpt;
  if (c->cfg.head_dim == 64)
    return launch_d<64>(c, groups_d, n_groups, ncons, layer_begin, n_layers, n_call, q, scale, out, st);
  return launch_d<128>(c, groups_d, n_groups, ncons, layer_begin, n_layers, n_call, q, scale, out, st);
}

}  // namespace tts
