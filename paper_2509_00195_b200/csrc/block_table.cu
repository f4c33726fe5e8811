// Paged, prefix-shared block table with a refcounted lowest-free-page
// allocator, and PRM top-K selection + M-way fork with eager copy-on-write.
//
// PAPER.md 3.1: the verification stage keeps "the top-K
// candidates globally with a static branching factor" and replicates them
// ("Top-scoring paths are then replicated to spawn the next set of active
// beams"); siblings are grouped and the parents' order preserved
// (P:394).  The paper is silent on paging; the canonical rules are SURVEY.md
// 8(c) ledger C5-C8 (lowest free id first, releases before allocations,
// (request, beam) order, ref = number of live tables containing the page,
// eager CoW of partially filled last pages).  All integer results are
// order-independent (atomics only commute), so they are bit-exact against the
// sequential oracle.
#include <cub/block/block_scan.cuh>
#include <cub/block/block_reduce.cuh>

#include <cstring>

#include "tts_internal.cuh"

namespace tts {
namespace {

struct DevState {
  __nv_bfloat16* k_pool;
  __nv_bfloat16* v_pool;
  int32_t* tables;
  int32_t* lens;
  int32_t* ref;
  uint32_t* bitmap;
  int32_t* status;
  int32_t L, Hkv, d, P, maxB, maxP;
  int64_t num_pages;
  int64_t nwords;
};

DevState dev_state(const Ctx* c) {
  DevState s;
  s.k_pool = (__nv_bfloat16*)c->buf.k_pool;
  s.v_pool = (__nv_bfloat16*)c->buf.v_pool;
  s.tables = c->buf.block_tables;
  s.lens = c->buf.seq_lens;
  s.ref = c->buf.refcounts;
  s.bitmap = c->buf.free_bitmap;
  s.status = c->buf.status;
  s.L = c->cfg.num_layers;
  s.Hkv = c->cfg.num_kv_heads;
  s.d = c->cfg.head_dim;
  s.P = c->cfg.page_size;
  s.maxB = c->cfg.max_beams;
  s.maxP = c->cfg.max_pages_per_beam;
  s.num_pages = c->cfg.num_pages;
  s.nwords = (c->cfg.num_pages + 31) / 32;
  return s;
}

__device__ __forceinline__ int64_t row_base(const DevState& s, int req, int beam) {
  return ((int64_t)req * s.maxB + beam) * s.maxP;
}

// ---------------------------------------------------------------------------
__global__ void k_init_state(DevState s) {
  int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t p = tid; p < s.num_pages; p += stride) s.ref[p] = 0;
  for (int64_t w = tid; w < s.nwords; w += stride) {
    int64_t lo = w * 32;
    int64_t n = s.num_pages - lo;
    s.bitmap[w] = n >= 32 ? 0xFFFFFFFFu : ((1u << n) - 1u);
  }
  if (tid < 4) s.status[tid] = 0;
}

__global__ void k_fill_i32(int32_t* p, int64_t n, int32_t v) {
  int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (int64_t i = tid; i < n; i += (int64_t)gridDim.x * blockDim.x) p[i] = v;
}

// ---------------------------------------------------------------------------
// Lowest-free-page allocator: one CTA hands out the n lowest free page ids, in
// ascending order, to the n items in item order (ledger C7).  All-or-nothing:
// on exhaustion it sets the sticky status and changes nothing.
constexpr int kAllocThreads = 1024;
constexpr int kAllocInline = 64;
struct AllocInline {
  AllocItem it[kAllocInline];
};

// items: device list, or null when the (<= kAllocInline) items are in `inl`
__global__ void __launch_bounds__(kAllocThreads) k_alloc(DevState s, const AllocItem* items,
                                                         const __grid_constant__ AllocInline inl,
                                                         int n_items, int32_t* pages_out,
                                                         CowCopy* cow_out) {
  using Scan = cub::BlockScan<int, kAllocThreads>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int s_total;
  if (*(volatile int32_t*)s.status) return;
  const int tid = threadIdx.x;
  const int64_t chunk = (s.nwords + kAllocThreads - 1) / kAllocThreads;
  const int64_t w0 = tid * chunk;
  const int64_t w1 = min(w0 + chunk, s.nwords);
  int cnt = 0;
  for (int64_t w = w0; w < w1; ++w) cnt += __popc(s.bitmap[w]);
  int base, total;
  Scan(tmp).ExclusiveSum(cnt, base, total);
  if (tid == 0) s_total = total;
  __syncthreads();
  if (s_total < n_items) {
    if (tid == 0) s.status[0] = TTS_ERR_OUT_OF_PAGES;
    return;
  }
  int rank = base;
  for (int64_t w = w0; w < w1 && rank < n_items; ++w) {
    uint32_t bits = s.bitmap[w];
    uint32_t taken = 0;
    while (bits && rank < n_items) {
      int b = __ffs(bits) - 1;
      pages_out[rank++] = (int32_t)(w * 32 + b);
      taken |= 1u << b;
      bits &= bits - 1;
    }
    if (taken) s.bitmap[w] &= ~taken;
  }
  __syncthreads();
  for (int k = tid; k < n_items; k += kAllocThreads) {
    const AllocItem it = items ? items[k] : inl.it[k];
    int32_t p = pages_out[k];
    int32_t old = s.tables[it.entry];
    s.tables[it.entry] = p;
    s.ref[p] = 1;
    if (it.cow) {
      atomicSub(&s.ref[old], 1);
      cow_out[k] = CowCopy{old, p, it.ntok, 0};
    }
  }
}

// Prompt pages were allocated into beam 0's row; share them with every beam.
__global__ void k_broadcast_prompt(DevState s, int req, int n_beams, int npg) {
  if (*(volatile int32_t*)s.status) return;
  int i = blockIdx.x * blockDim.x + threadIdx.x;  // over (beam, page) pairs
  if (i >= n_beams * npg) return;
  int b = i / npg, pg = i % npg;
  int32_t p = s.tables[row_base(s, req, 0) + pg];
  if (b == 0)
    s.ref[p] = n_beams;
  else
    s.tables[row_base(s, req, b) + pg] = p;
}

// Write prompt K/V [L][prompt][Hkv][d] into the prompt pages (16-B vectors);
// the slots after the last prompt token of a partial last page are zeroed.
__global__ void k_write_prompt(DevState s, int req, int prompt_len, const uint4* __restrict__ k,
                               const uint4* __restrict__ v) {
  if (*(volatile int32_t*)s.status) return;
  const int vec_per_row = s.d / 8;
  const int rem = prompt_len % s.P;
  const int tail = rem ? s.P - rem : 0;
  const int64_t n = (int64_t)s.L * prompt_len * s.Hkv * vec_per_row;
  const int64_t nz = (int64_t)s.L * tail * s.Hkv * vec_per_row;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n + nz;
       i += (int64_t)gridDim.x * blockDim.x) {
    const bool zero = i >= n;
    const int64_t ii = zero ? i - n : i;
    const int span = zero ? tail : prompt_len;
    int64_t r = ii / vec_per_row;
    int e = (int)(ii % vec_per_row);
    int kh = (int)(r % s.Hkv);
    int64_t r2 = r / s.Hkv;
    int j = (int)(r2 % span) + (zero ? prompt_len : 0);
    int l = (int)(r2 / span);
    int32_t page = s.tables[row_base(s, req, 0) + j / s.P];
    int64_t dst = ((((int64_t)l * s.num_pages + page) * s.Hkv + kh) * s.P + j % s.P) * vec_per_row + e;
    reinterpret_cast<uint4*>(s.k_pool)[dst] = zero ? make_uint4(0, 0, 0, 0) : k[ii];
    reinterpret_cast<uint4*>(s.v_pool)[dst] = zero ? make_uint4(0, 0, 0, 0) : v_to_pool(v[ii], s.status);
  }
}

// CoW: copy the first ntok token slots of every (layer, kv head) of src -> dst
// and zero the remaining slots of dst.
__global__ void k_cow_copy(DevState s, const CowCopy* items) {
  if (*(volatile int32_t*)s.status) return;
  CowCopy it = items[blockIdx.x];
  const int l = blockIdx.y;
  const int vec_per_row = s.d / 8;
  const int per_head = s.P * vec_per_row;
  const int n = s.Hkv * per_head;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    int kh = i / per_head;
    int off = i % per_head;  // contiguous within the head's P x d slab
    int64_t src = (((int64_t)l * s.num_pages + it.src) * s.Hkv + kh) * s.P * vec_per_row + off;
    int64_t dst = (((int64_t)l * s.num_pages + it.dst) * s.Hkv + kh) * s.P * vec_per_row + off;
    const bool copy = off < it.ntok * vec_per_row;
    reinterpret_cast<uint4*>(s.k_pool)[dst] =
        copy ? reinterpret_cast<const uint4*>(s.k_pool)[src] : make_uint4(0, 0, 0, 0);
    reinterpret_cast<uint4*>(s.v_pool)[dst] =
        copy ? reinterpret_cast<const uint4*>(s.v_pool)[src] : make_uint4(0, 0, 0, 0);
  }
}

// Append: slot items (call_idx, req, beam, pos) -> write k/v [L][n_call][maxB][Hkv][d]
// at token pos of the beam; lens[req][beam] = pos + 1.  The first token of a
// fresh page also zeroes the page's other slots.
__global__ void k_append_write(DevState s, const int4* __restrict__ slots, int n_call,
                               const uint4* __restrict__ k, const uint4* __restrict__ v) {
  if (*(volatile int32_t*)s.status) return;
  int4 it = slots[blockIdx.x];
  const int l = blockIdx.y;
  const int call = it.x, req = it.y, beam = it.z, pos = it.w;
  const int vec_per_row = s.d / 8;
  const int n = s.Hkv * vec_per_row;
  const int rows = (pos % s.P == 0) ? s.P : 1;  // fresh page: write slot 0, zero slots 1..P-1
  int32_t page = s.tables[row_base(s, req, beam) + pos / s.P];
  for (int i = threadIdx.x; i < n * rows; i += blockDim.x) {
    const int slot_off = i / n, r2 = i % n;
    int kh = r2 / vec_per_row, e = r2 % vec_per_row;
    int64_t dst = ((((int64_t)l * s.num_pages + page) * s.Hkv + kh) * s.P + pos % s.P + slot_off) * vec_per_row + e;
    if (slot_off == 0) {
      int64_t src = ((((int64_t)l * n_call + call) * s.maxB + beam) * s.Hkv + kh) * vec_per_row + e;
      reinterpret_cast<uint4*>(s.k_pool)[dst] = k[src];
      reinterpret_cast<uint4*>(s.v_pool)[dst] = v_to_pool(v[src], s.status);
    } else {
      reinterpret_cast<uint4*>(s.k_pool)[dst] = make_uint4(0, 0, 0, 0);
      reinterpret_cast<uint4*>(s.v_pool)[dst] = make_uint4(0, 0, 0, 0);
    }
  }
  if (l == 0 && threadIdx.x == 0) s.lens[(int64_t)req * s.maxB + beam] = pos + 1;
}

// ---------------------------------------------------------------------------
// Selection (a6): one CTA per request.  Orderable key (ledger C4): NaN lowest,
// -0 == +0, then index ascending.  rank_i = #{j : key_j beats key_i}; the K
// lowest ranks survive; survivors sorted by index via a block scan.
constexpr int kSelThreads = 1024;

__device__ __forceinline__ uint64_t order_key(float f, int i) {
  uint32_t u;
  if (isnan(f)) {
    u = 0u;
  } else {
    if (f == 0.0f) f = 0.0f;
    uint32_t b = __float_as_uint(f);
    u = (b & 0x80000000u) ? ~b : (b | 0x80000000u);
  }
  return ((uint64_t)u << 32) | (uint64_t)(0xFFFFFFFFu - (uint32_t)i);
}

__global__ void __launch_bounds__(kSelThreads) k_select(DevState s, const int32_t* reqs,
                                                       const float* scores, int N, int M,
                                                       int32_t* parent_ws, int32_t* parent_out) {
  using Scan = cub::BlockScan<int, kSelThreads>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ uint64_t keys[1024];
  __shared__ int32_t surv[1024];
  if (*(volatile int32_t*)s.status) return;
  const int call = blockIdx.x;
  const int tid = threadIdx.x;
  const int K = N / M;
  uint64_t my = 0;
  if (tid < N) {
    my = order_key(scores[(int64_t)call * s.maxB + tid], tid);
    keys[tid] = my;
  }
  __syncthreads();
  int flag = 0;
  if (tid < N) {
    int rank = 0;
    for (int j = 0; j < N; ++j) rank += keys[j] > my;
    flag = rank < K;
  }
  int pos;
  Scan(tmp).ExclusiveSum(flag, pos);
  if (flag) surv[pos] = tid;
  __syncthreads();
  if (tid < N) {
    int32_t par = surv[tid / M];
    parent_ws[(int64_t)call * s.maxB + tid] = par;
    if (parent_out) parent_out[(int64_t)call * s.maxB + tid] = par;
  }
  (void)reqs;
}

// Selection variants (ledger C23/C24): one CTA per request.
//   policy 1, diverse (DVTS): subtree s = beams [s n, (s+1) n), n = N / param;
//     its best beam (the orderable key above) spawns the n children of subtree s.
//   policy 2, dynamic branching: the K = N / param survivors of beam search,
//     child counts 1 + floor(q_i) + (largest-remainder extra), q_i = (N - K)
//     w_i / sum(w) in fp64 (the sum in survivor order, by one thread, the way
//     the oracle adds), w = score if finite and > 0 else 0 (all 0 -> equal).
// parent_ws / parent_out as k_select.
__global__ void __launch_bounds__(kSelThreads) k_select_policy(DevState s, const float* scores, int N, int policy,
                                                               int param, int32_t* parent_ws, int32_t* parent_out) {
  using Scan = cub::BlockScan<int, kSelThreads>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ uint64_t keys[1024];
  __shared__ int32_t surv[1024];
  __shared__ int32_t cnt[1024];
  __shared__ double frac[1024];
  __shared__ double wsum;
  if (*(volatile int32_t*)s.status) return;
  const int call = blockIdx.x;
  const int tid = threadIdx.x;
  uint64_t my = 0;
  if (tid < N) {
    my = order_key(scores[(int64_t)call * s.maxB + tid], tid);
    keys[tid] = my;
  }
  __syncthreads();
  int32_t par = 0;
  if (policy == 1) {
    const int n = N / param;
    if (tid < param) {  // one thread per subtree: its best beam
      int best = tid * n;
      for (int i = tid * n + 1; i < (tid + 1) * n; ++i)
        if (keys[i] > keys[best]) best = i;
      surv[tid] = best;
    }
    __syncthreads();
    if (tid < N) par = surv[tid / n];
  } else {
    const int K = N / param;
    int flag = 0;
    if (tid < N) {
      int rank = 0;
      for (int j = 0; j < N; ++j) rank += keys[j] > my;
      flag = rank < K;
    }
    int pos;
    Scan(tmp).ExclusiveSum(flag, pos);
    if (flag) surv[pos] = tid;
    __syncthreads();
    if (tid == 0) {
      double w = 0.0;
      for (int i = 0; i < K; ++i) {
        const double x = (double)scores[(int64_t)call * s.maxB + surv[i]];
        w += (isfinite(x) && x > 0.0) ? x : 0.0;
      }
      wsum = w;
    }
    __syncthreads();
    int c = 0;
    if (tid < K) {
      const double x = (double)scores[(int64_t)call * s.maxB + surv[tid]];
      double wi = (isfinite(x) && x > 0.0) ? x : 0.0, W = wsum;
      if (W == 0.0) {
        wi = 1.0;
        W = (double)K;
      }
      const double q = __dmul_rn((double)(N - K), wi);
      const double qq = __ddiv_rn(q, W);
      const double fl = floor(qq);
      c = 1 + (int)fl;
      frac[tid] = qq - fl;
      cnt[tid] = c;
    }
    int csum;
    {
      int tot;
      Scan(tmp).ExclusiveSum(c, csum, tot);
      __syncthreads();
      if (tid == 0) wsum = (double)(N - tot);  // children still to place
    }
    __syncthreads();
    const int rest = (int)wsum;
    if (tid < K) {  // rank by (fraction desc, survivor index asc)
      int rank = 0;
      const double f = frac[tid];
      for (int j = 0; j < K; ++j) rank += frac[j] > f || (frac[j] == f && j < tid);
      if (rank < rest) cnt[tid] = c + 1;
    }
    __syncthreads();
    int off, c2 = tid < K ? cnt[tid] : 0;
    Scan(tmp).ExclusiveSum(c2, off);
    if (tid < K)
      for (int k = 0; k < c2; ++k) {
        parent_ws[(int64_t)call * s.maxB + off + k] = surv[tid];
        if (parent_out) parent_out[(int64_t)call * s.maxB + off + k] = surv[tid];
      }
    return;
  }
  if (tid < N) {
    parent_ws[(int64_t)call * s.maxB + tid] = par;
    if (parent_out) parent_out[(int64_t)call * s.maxB + tid] = par;
  }
}

// Fork, step A: new rows into tmp (child c <- old row parent[c]); refcounts
// recounted by -1 per old-row entry and +1 per new-row entry (commuting
// atomics).  Old rows [0, n_old), new rows [0, n_new); n_old > n_new when
// migrated lineages were imported into spare slots (multi-GPU, a8).
__global__ void k_fork_count(DevState s, const int32_t* reqs, const int32_t* parent, int n_old, int n_new,
                             int32_t* tmp_tables, int32_t* tmp_lens, const int32_t* new_lens) {
  if (*(volatile int32_t*)s.status) return;
  const int call = blockIdx.y;
  const int b = blockIdx.x;  // old row b and/or new row c = b
  const int req = reqs[call];
  if (b < n_old) {
    const int len_old = s.lens[(int64_t)req * s.maxB + b];
    const int np_old = (len_old + s.P - 1) / s.P;
    const int32_t* old_row = s.tables + row_base(s, req, b);
    for (int i = threadIdx.x; i < np_old; i += blockDim.x) atomicSub(&s.ref[old_row[i]], 1);
  }
  if (b < n_new) {
    const int32_t par = parent[(int64_t)call * s.maxB + b];
    // (a truncating fork -- speculative beam extension -- keeps only the first
    // new_lens[b] tokens of the parent row)
    const int len_par = new_lens ? new_lens[b] : s.lens[(int64_t)req * s.maxB + par];
    const int np_new = (len_par + s.P - 1) / s.P;
    const int32_t* par_row = s.tables + row_base(s, req, par);
    int32_t* new_row = tmp_tables + row_base(s, req, b);
    for (int i = threadIdx.x; i < np_new; i += blockDim.x) {
      int32_t p = par_row[i];
      new_row[i] = p;
      atomicAdd(&s.ref[p], 1);
    }
    if (threadIdx.x == 0) tmp_lens[(int64_t)req * s.maxB + b] = len_par;
  }
}

// Speculative branches (f1): row dst[i] = a copy of row src[i] of request req
// (table entries, length), one more reference on every page; a partially
// filled last page is then replaced by a copy (k_alloc cow items, C6).
__global__ void k_branch_rows(DevState s, int req, const int32_t* __restrict__ src, const int32_t* __restrict__ dst) {
  if (*(volatile int32_t*)s.status) return;
  const int i = blockIdx.x;
  const int a = src[i], b = dst[i];
  const int len = s.lens[(int64_t)req * s.maxB + a];
  const int np = (len + s.P - 1) / s.P;
  const int32_t* from = s.tables + row_base(s, req, a);
  int32_t* to = s.tables + row_base(s, req, b);
  for (int k = threadIdx.x; k < np; k += blockDim.x) {
    const int32_t p = from[k];
    to[k] = p;
    atomicAdd(&s.ref[p], 1);
  }
  if (threadIdx.x == 0) s.lens[(int64_t)req * s.maxB + b] = len;
}

// Zero token slots [ntok, P) of a row's page (every layer, kv head): the kept
// last page of a truncated row holds no stale tokens past the row's length.
// items: (req, row, page position, ntok).
__global__ void k_zero_tail(DevState s, const int4* items) {
  if (*(volatile int32_t*)s.status) return;
  const int4 q = items[blockIdx.x];
  const int l = blockIdx.y;
  struct {
    int32_t dst, ntok;
  } it{s.tables[row_base(s, q.x, q.y) + q.z], q.w};
  const int vec_per_row = s.d / 8;
  const int per_head = s.P * vec_per_row;
  for (int i = threadIdx.x; i < s.Hkv * per_head; i += blockDim.x) {
    const int kh = i / per_head, off = i % per_head;
    if (off < it.ntok * vec_per_row) continue;
    const int64_t dst = (((int64_t)l * s.num_pages + it.dst) * s.Hkv + kh) * s.P * vec_per_row + off;
    reinterpret_cast<uint4*>(s.k_pool)[dst] = make_uint4(0, 0, 0, 0);
    reinterpret_cast<uint4*>(s.v_pool)[dst] = make_uint4(0, 0, 0, 0);
  }
}

// Fork, step B: release pages of the old rows whose refcount reached 0.
__global__ void k_fork_free(DevState s, const int32_t* reqs, int n_old) {
  if (*(volatile int32_t*)s.status) return;
  const int call = blockIdx.y;
  const int b = blockIdx.x;
  if (b >= n_old) return;
  const int req = reqs[call];
  const int len_old = s.lens[(int64_t)req * s.maxB + b];
  const int np_old = (len_old + s.P - 1) / s.P;
  const int32_t* old_row = s.tables + row_base(s, req, b);
  for (int i = threadIdx.x; i < np_old; i += blockDim.x) {
    int32_t p = old_row[i];
    if (s.ref[p] == 0) atomicOr(&s.bitmap[p >> 5], 1u << (p & 31));
  }
}

// Fork, step C: install the new rows and lengths; spare rows [n_new, n_old) emptied.
__global__ void k_fork_commit(DevState s, const int32_t* reqs, int n_old, int n_new, const int32_t* tmp_tables,
                              const int32_t* tmp_lens) {
  if (*(volatile int32_t*)s.status) return;
  const int call = blockIdx.y;
  const int b = blockIdx.x;
  const int req = reqs[call];
  const int64_t li = (int64_t)req * s.maxB + b;
  if (b >= n_new) {
    if (b < n_old && threadIdx.x == 0) s.lens[li] = 0;
    return;
  }
  const int len = tmp_lens[li];
  const int np = (len + s.P - 1) / s.P;
  const int32_t* src = tmp_tables + row_base(s, req, b);
  int32_t* dst = s.tables + row_base(s, req, b);
  for (int i = threadIdx.x; i < np; i += blockDim.x) dst[i] = src[i];
  __syncthreads();
  if (threadIdx.x == 0) s.lens[li] = len;
}

// Lineage export (migration, a8): the beam's len tokens of every layer as a
// contiguous bf16 buffer [2 (K, V)][L][len][Hkv][d].  One block per (token, layer).
__global__ void k_lineage_export(DevState s, int req, int beam, int len, int t0, uint4* __restrict__ buf) {
  if (*(volatile int32_t*)s.status) return;
  const int t = t0 + blockIdx.x, l = blockIdx.y;
  const int vpr = s.d / 8, n = s.Hkv * vpr;
  const int32_t page = s.tables[row_base(s, req, beam) + t / s.P];
  const int64_t plane = (int64_t)s.L * (len - t0) * n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int kh = i / vpr, e = i % vpr;
    const int64_t src = ((((int64_t)l * s.num_pages + page) * s.Hkv + kh) * s.P + t % s.P) * vpr + e;
    const int64_t dst = (((int64_t)l * (len - t0) + (t - t0)) * s.Hkv + kh) * vpr + e;
    buf[dst] = reinterpret_cast<const uint4*>(s.k_pool)[src];
    buf[plane + dst] = reinterpret_cast<const uint4*>(s.v_pool)[src];
  }
}

// Lineage import: write the buffer into the beam's freshly allocated pages and
// set its length (the pages were allocated by k_alloc into the row first).
__global__ void k_lineage_import(DevState s, int req, int beam, int len, int t0, const uint4* __restrict__ buf) {
  if (*(volatile int32_t*)s.status) return;
  const int t = t0 + blockIdx.x, l = blockIdx.y;  // t < ceil(len / P) * P: slots past len are zeroed
  const int vpr = s.d / 8, n = s.Hkv * vpr;
  const int32_t page = s.tables[row_base(s, req, beam) + t / s.P];
  const int64_t plane = (int64_t)s.L * (len - t0) * n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int kh = i / vpr, e = i % vpr;
    const int64_t dst = ((((int64_t)l * s.num_pages + page) * s.Hkv + kh) * s.P + t % s.P) * vpr + e;
    const int64_t src = (((int64_t)l * (len - t0) + (t - t0)) * s.Hkv + kh) * vpr + e;
    reinterpret_cast<uint4*>(s.k_pool)[dst] = t < len ? buf[src] : make_uint4(0, 0, 0, 0);
    reinterpret_cast<uint4*>(s.v_pool)[dst] = t < len ? buf[plane + src] : make_uint4(0, 0, 0, 0);
  }
  if (t == t0 && l == 0 && threadIdx.x == 0) s.lens[(int64_t)req * s.maxB + beam] = len;
}

// Row `beam` of request req takes the first m page entries of local row
// `share` (one more reference each): the shared prefix of an imported
// lineage (f4, cross-GPU deduplication).
__global__ void k_share_prefix(DevState s, int req, int beam, int share, int m) {
  if (*(volatile int32_t*)s.status) return;
  const int32_t* from = s.tables + row_base(s, req, share);
  int32_t* to = s.tables + row_base(s, req, beam);
  for (int k = threadIdx.x; k < m; k += blockDim.x) {
    const int32_t p = from[k];
    to[k] = p;
    atomicAdd(&s.ref[p], 1);
  }
}

// Release a request: -1 per entry, then free the pages that reached 0.
__global__ void k_release_count(DevState s, int req) {
  if (*(volatile int32_t*)s.status) return;
  const int b = blockIdx.x;
  const int len = s.lens[(int64_t)req * s.maxB + b];
  const int np = (len + s.P - 1) / s.P;
  const int32_t* row = s.tables + row_base(s, req, b);
  for (int i = threadIdx.x; i < np; i += blockDim.x) atomicSub(&s.ref[row[i]], 1);
}

__global__ void k_release_free(DevState s, int req) {
  if (*(volatile int32_t*)s.status) return;
  const int b = blockIdx.x;
  const int64_t li = (int64_t)req * s.maxB + b;
  const int len = s.lens[li];
  const int np = (len + s.P - 1) / s.P;
  const int32_t* row = s.tables + row_base(s, req, b);
  for (int i = threadIdx.x; i < np; i += blockDim.x) {
    int32_t p = row[i];
    if (s.ref[p] == 0) atomicOr(&s.bitmap[p >> 5], 1u << (p & 31));
  }
}

__global__ void k_zero_lens(DevState s, int req) {
  if (*(volatile int32_t*)s.status) return;
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < s.maxB) s.lens[(int64_t)req * s.maxB + b] = 0;
}

// Stats: mark[p] = max valid tokens of p over active beams (ledger C22).
__global__ void k_stats_mark(DevState s, const GroupDesc* groups, int32_t* mark) {
  if (*(volatile int32_t*)s.status) return;
  GroupDesc g = groups[blockIdx.x];
  for (int bi = 0; bi < g.nbeams; ++bi) {
    if (!((g.active >> bi) & 1u)) continue;
    const int beam = g.beam0 + bi;
    const int len = s.lens[(int64_t)g.req * s.maxB + beam];
    const int np = (len + s.P - 1) / s.P;
    const int32_t* row = s.tables + row_base(s, g.req, beam);
    for (int i = threadIdx.x; i < np; i += blockDim.x)
      atomicMax(&mark[row[i]], min(s.P, len - i * s.P));
  }
}

__global__ void k_stats_reduce(DevState s, int32_t* mark, int64_t* accum, int64_t logical) {
  using Red = cub::BlockReduce<long long, 1024>;
  __shared__ typename Red::TempStorage tmp;
  long long sum = 0;
  for (int64_t p = blockIdx.x * 1024 + threadIdx.x; p < s.num_pages; p += (int64_t)gridDim.x * 1024) {
    sum += mark[p];
    mark[p] = 0;
  }
  long long tot = Red(tmp).Sum(sum);
  if (threadIdx.x == 0) {
    atomicAdd((unsigned long long*)&accum[0], (unsigned long long)tot);
    if (blockIdx.x == 0) atomicAdd((unsigned long long*)&accum[1], (unsigned long long)logical);
  }
}

}  // namespace

// ---------------------------------------------------------------------------
cudaError_t launch_init_state(Ctx* c, cudaStream_t st) {
  DevState s = dev_state(c);
  k_init_state<<<c->num_sms * 4, 256, 0, st>>>(s);
  c->launches++;
  int64_t ntab = (int64_t)c->cfg.max_requests * c->cfg.max_beams * c->cfg.max_pages_per_beam;
  k_fill_i32<<<c->num_sms * 4, 256, 0, st>>>(s.tables, ntab, -1);
  k_fill_i32<<<c->num_sms, 256, 0, st>>>(s.lens, (int64_t)c->cfg.max_requests * c->cfg.max_beams, 0);
  k_fill_i32<<<c->num_sms * 4, 256, 0, st>>>(c->ws_mark, c->cfg.num_pages, 0);
  c->launches += 3;
  return cudaGetLastError();
}

cudaError_t launch_alloc(Ctx* c, const AllocItem* items_d, int n_items, cudaStream_t st) {
  if (n_items <= 0) return cudaSuccess;
  static const AllocInline none{};
  k_alloc<<<1, kAllocThreads, 0, st>>>(dev_state(c), items_d, none, n_items, c->ws_pages, c->ws_cow);
  c->launches++;
  return cudaGetLastError();
}

cudaError_t launch_alloc_host(Ctx* c, const AllocItem* items_h, int n_items, cudaStream_t st) {
  if (n_items <= 0) return cudaSuccess;
  if (n_items > kAllocInline) {
    cudaError_t e;
    void* d = upload(c, items_h, (size_t)n_items * sizeof(AllocItem), st, &e);
    if (e != cudaSuccess) return e;
    return launch_alloc(c, (const AllocItem*)d, n_items, st);
  }
  AllocInline inl;
  std::memcpy(inl.it, items_h, (size_t)n_items * sizeof(AllocItem));
  k_alloc<<<1, kAllocThreads, 0, st>>>(dev_state(c), nullptr, inl, n_items, c->ws_pages, c->ws_cow);
  c->launches++;
  return cudaGetLastError();
}

cudaError_t launch_broadcast_prompt(Ctx* c, int req, int n_beams, int npg, cudaStream_t st) {
  int n = n_beams * npg;
  if (n == 0) return cudaSuccess;
  k_broadcast_prompt<<<(n + 255) / 256, 256, 0, st>>>(dev_state(c), req, n_beams, npg);
  c->launches++;
  return cudaGetLastError();
}

cudaError_t launch_write_prompt(Ctx* c, int req, int prompt_len, const __nv_bfloat16* k,
                                const __nv_bfloat16* v, cudaStream_t st) {
  if (prompt_len == 0) return cudaSuccess;
  k_write_prompt<<<c->num_sms * 4, 256, 0, st>>>(dev_state(c), req, prompt_len, (const uint4*)k,
                                                 (const uint4*)v);
  c->launches++;
  return cudaGetLastError();
}

cudaError_t launch_cow_copy(Ctx* c, int n_items, cudaStream_t st) {
  if (n_items == 0) return cudaSuccess;
  dim3 grid(n_items, c->cfg.num_layers);
  k_cow_copy<<<grid, 256, 0, st>>>(dev_state(c), c->ws_cow);
  c->launches++;
  return cudaGetLastError();
}

cudaError_t launch_append_write(Ctx* c, const int32_t* slots_d, int n_slots, int n_call,
                                const __nv_bfloat16* k, const __nv_bfloat16* v, cudaStream_t st) {
  if (n_slots == 0) return cudaSuccess;
  dim3 grid(n_slots, c->cfg.num_layers);
  const int threads = 128;
  k_append_write<<<grid, threads, 0, st>>>(dev_state(c), (const int4*)slots_d, n_call,
                                           (const uint4*)k, (const uint4*)v);
  c->launches++;
  return cudaGetLastError();
}

cudaError_t launch_select(Ctx* c, const int32_t* reqs_d, int n_req, const float* scores, int N,
                          int M, int32_t* parent_out, cudaStream_t st) {
  k_select<<<n_req, kSelThreads, 0, st>>>(dev_state(c), reqs_d, scores, N, M, c->ws_parent,
                                          parent_out);
  c->launches++;
  return cudaGetLastError();
}

cudaError_t launch_select_policy(Ctx* c, int n_req, const float* scores, int N, int policy, int param,
                                 int32_t* parent_out, cudaStream_t st) {
  k_select_policy<<<n_req, kSelThreads, 0, st>>>(dev_state(c), scores, N, policy, param, c->ws_parent, parent_out);
  c->launches++;
  return cudaGetLastError();
}

cudaError_t launch_fork_tables(Ctx* c, const int32_t* reqs_d, int n_req, int n_old, int n_new, cudaStream_t st,
                               const int32_t* new_lens_d) {
  DevState s = dev_state(c);
  dim3 grid(n_old > n_new ? n_old : n_new, n_req);
  k_fork_count<<<grid, 128, 0, st>>>(s, reqs_d, c->ws_parent, n_old, n_new, c->ws_tmp_tables, c->ws_tmp_lens,
                                     new_lens_d);
  k_fork_free<<<grid, 128, 0, st>>>(s, reqs_d, n_old);
  k_fork_commit<<<grid, 128, 0, st>>>(s, reqs_d, n_old, n_new, c->ws_tmp_tables, c->ws_tmp_lens);
  c->launches += 3;
  return cudaGetLastError();
}

cudaError_t launch_branch_rows(Ctx* c, int req, const int32_t* src_d, const int32_t* dst_d, int n, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  k_branch_rows<<<n, 128, 0, st>>>(dev_state(c), req, src_d, dst_d);
  c->launches++;
  return cudaGetLastError();
}

cudaError_t launch_zero_tail(Ctx* c, const int32_t* items_d, int n, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  k_zero_tail<<<dim3(n, c->cfg.num_layers), 256, 0, st>>>(dev_state(c), (const int4*)items_d);
  c->launches++;
  return cudaGetLastError();
}

cudaError_t launch_lineage_export(Ctx* c, int req, int beam, int len, void* buf, cudaStream_t st, int t0) {
  if (len - t0 <= 0) return cudaSuccess;
  k_lineage_export<<<dim3(len - t0, c->cfg.num_layers), 128, 0, st>>>(dev_state(c), req, beam, len, t0,
                                                                      (uint4*)buf);
  c->launches++;
  return cudaGetLastError();
}

cudaError_t launch_lineage_import(Ctx* c, int req, int beam, int len, const void* buf, cudaStream_t st, int t0) {
  const int P = c->cfg.page_size;
  if ((len + P - 1) / P * P - t0 <= 0) return cudaSuccess;
  k_lineage_import<<<dim3((len + P - 1) / P * P - t0, c->cfg.num_layers), 128, 0, st>>>(dev_state(c), req, beam,
                                                                                       len, t0, (const uint4*)buf);
  c->launches++;
  return cudaGetLastError();
}

cudaError_t launch_share_prefix(Ctx* c, int req, int beam, int share, int m, cudaStream_t st) {
  if (m <= 0) return cudaSuccess;
  k_share_prefix<<<1, 256, 0, st>>>(dev_state(c), req, beam, share, m);
  c->launches++;
  return cudaGetLastError();
}

cudaError_t launch_select_global(Ctx* c, const float* scores_all, int N, int M, int32_t* parent_out,
                                 cudaStream_t st) {
  k_select<<<1, kSelThreads, 0, st>>>(dev_state(c), nullptr, scores_all, N, M, parent_out, parent_out);
  c->launches++;
  return cudaGetLastError();
}

cudaError_t launch_release(Ctx* c, int req, int n_beams, cudaStream_t st) {
  DevState s = dev_state(c);
  k_release_count<<<n_beams, 128, 0, st>>>(s, req);
  k_release_free<<<n_beams, 128, 0, st>>>(s, req);
  k_zero_lens<<<(c->cfg.max_beams + 255) / 256, 256, 0, st>>>(s, req);
  c->launches += 3;
  return cudaGetLastError();
}

cudaError_t launch_stats(Ctx* c, const GroupDesc* groups_d, int n_groups, int64_t* accum,
                         int64_t logical, cudaStream_t st) {
  DevState s = dev_state(c);
  if (n_groups > 0) {
    k_stats_mark<<<n_groups, 256, 0, st>>>(s, groups_d, c->ws_mark);
    c->launches++;
  }
  int blocks = (int)std::min<int64_t>((c->cfg.num_pages + 1023) / 1024, (int64_t)c->num_sms * 2);
  if (blocks < 1) blocks = 1;
  k_stats_reduce<<<blocks, 1024, 0, st>>>(s, c->ws_mark, accum, logical);
  c->launches++;
  return cudaGetLastError();
}

}  // namespace tts
