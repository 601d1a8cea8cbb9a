// attention.cu — causal GQA prefill attention on tcgen05/TMEM with the RadixMLP
// attention boundary fused into its loads.
//
// Reference boundary (model.py:368-383): scatter Q/K/V from the N' compact
// rows to the N original rows, exact causal softmax attention per sequence
// (model.py:228-265, scale 1/sqrt(hd), GQA contiguous grouping), gather the
// output back to N' rows.  Here nothing is scattered: by SURVEY finding 2 the
// compact rows of sequence s are its suffix [lcp_s, L_s), so
//   * queries stay compact: query i of s is compact row cu_q[s] + i at
//     position lcp_s + i (bottom-right-aligned causal mask);
//   * keys/values are read in place from the compact QKV buffer through the
//     plan's scatter map: key j of s is compact row scatter[cu[s] + j];
//   * the output is written directly in compact layout.
// Plain (no-dedup) mode is the same kernel with scatter == NULL, cu_q == cu.
//
// Persistent CTAs (one per SM) walk the (sequence, kv head) work items; each
// item is every 128-row query block of that sequence/head, and all roles run
// one continuous software pipeline over (item, query block, key tile) steps,
// so the next item's loads overlap the current item's tail.  13 warps:
//   warps 0-3   softmax: row t of S per thread (TMEM lane t), online softmax,
//               P (bf16) -> smem, O rescale when the running max moves
//   warps 4-7   epilogue: O / l -> bf16 -> global (compact rows)
//   warps 8-11  loaders: cp.async 16-byte gathers of Q (2 buffers) and K/V
//               (3-stage ring) into the 128-byte-swizzled UMMA layouts
//   warp  12    TMEM allocator + MMA issuer:
//               S = Q K^T   (M=128 rows = group heads x queries, N=64 keys, K=hd)
//               O += P V    (M=128, N=hd, K=64 keys; V read MN-major, no transpose)
//               S and O are double-buffered in TMEM (S(t+1) overlaps softmax(t),
//               block b+1 accumulates while block b drains).
#include "common.cuh"

namespace rdx {
namespace attn {

constexpr int BQ = 128;        // tile rows (group heads x queries)
constexpr int BKEY = 64;       // keys per K/V tile
constexpr int kThreads = 416;  // 13 warps
constexpr int P_BYTES = BQ * BKEY * 2;     // 16 KB: 128 rows x 128 B
constexpr uint32_t TMEM_COLS = 512;        // S[2]: cols 0 / 64, O[2]: cols 128 / 256 (HDP each)
constexpr uint32_t S_COL = 0, O_COL = 128;

// HDP = head dim padded to a whole number of 64-element (128 B) swizzle atoms;
// the runtime head dim (16..HDP) is zero-padded in smem, which adds nothing to
// Q K^T and only produces ignored output columns in P V.
template <int HDP>
struct Tile {
  static constexpr int HALVES = HDP / 64;
  static constexpr int CHUNKS = HDP / 8;            // 16-byte chunks per row
  static constexpr int Q_BYTES = BQ * HDP * 2;      // HALVES x 128 rows x 128 B
  static constexpr int KV_BYTES = BKEY * HDP * 2;   // HALVES x 64 keys x 128 B
  static constexpr int NS = 3;                      // K/V ring stages
  static constexpr int SMEM = 2 * Q_BYTES + NS * 2 * KV_BYTES + P_BYTES + 1024 + 256;
  // kind::f16, bf16 in, fp32 acc; S: A K-major, B K-major.  PV: A K-major, B MN-major.
  static constexpr uint32_t IDESC_S = umma_idesc_bf16(BQ, BKEY);
  static constexpr uint32_t IDESC_PV = umma_idesc_bf16(BQ, HDP) | (1u << 16);
};

__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr & 0x3FFFFu) >> 4);
  d |= static_cast<uint64_t>((lbo_bytes >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo_bytes >> 4) & 0x3FFFu) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(2) << 61;
  return d;
}

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
      "%14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
      "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
      "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])), "r"(__float_as_uint(v[8])),
      "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
      "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
      "r"(__float_as_uint(v[15])), "r"(__float_as_uint(v[16])), "r"(__float_as_uint(v[17])),
      "r"(__float_as_uint(v[18])), "r"(__float_as_uint(v[19])), "r"(__float_as_uint(v[20])),
      "r"(__float_as_uint(v[21])), "r"(__float_as_uint(v[22])), "r"(__float_as_uint(v[23])),
      "r"(__float_as_uint(v[24])), "r"(__float_as_uint(v[25])), "r"(__float_as_uint(v[26])),
      "r"(__float_as_uint(v[27])), "r"(__float_as_uint(v[28])), "r"(__float_as_uint(v[29])),
      "r"(__float_as_uint(v[30])), "r"(__float_as_uint(v[31]))
      : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// 16-byte async global -> shared copy (L2 only); src_bytes = 0 zero-fills.
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
// Arrive on `bar` once every prior cp.async of this thread has landed.
__device__ __forceinline__ void cp_async_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

struct Args {
  const __nv_bfloat16* qkv;  // [rows, ld] compact (or full, plain mode)
  int64_t ld;                // elements
  const int32_t* scatter;    // [N] original -> compact row; NULL = identity (plain mode)
  const int32_t* cu;         // [B+1] original offsets
  const int32_t* cu_q;       // [B+1] query-row offsets (= cu in plain mode)
  __nv_bfloat16* out;        // [rows_q, ld_out]
  int64_t ld_out;
  int nseq, heads, kv_heads, hd;
  float scale_log2;          // softmax scale * log2(e)
  unsigned long long* trace; // optional per-CTA event timestamps (RDX_ATTN_TRACE), else NULL
};

#define RDX_TRACE(slot)                                                                     \
  do {                                                                                      \
    if (a.trace && blockIdx.x < 4096 && (slot) < 64) {                                      \
      unsigned long long _t;                                                                \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_t));                                \
      a.trace[static_cast<size_t>(blockIdx.x) * 64 + (slot)] = _t;                          \
    }                                                                                       \
  } while (0)

// 16-byte chunk c of a head row -> swizzled smem offset in a
// [halves][rows][128 B] tile (half stride = rows * 128).
__device__ __forceinline__ uint32_t sw_off(int row, int c, int rows) {
  const int half = c >> 3, cc = c & 7;
  return half * rows * 128 + row * 128 + ((cc ^ (row & 7)) << 4);
}

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Work item geometry (identical in every role).
struct Item {
  int s, g, k0, L, q0, qlen, lcp, n_mb;
};

__device__ __forceinline__ bool load_item(const Args& a, int item, int qpt, Item& it) {
  it.s = item / a.kv_heads;
  it.g = item % a.kv_heads;
  it.k0 = a.cu[it.s];
  it.L = a.cu[it.s + 1] - it.k0;
  it.q0 = a.cu_q[it.s];
  it.qlen = a.cu_q[it.s + 1] - it.q0;
  it.lcp = it.L - it.qlen;
  it.n_mb = (it.qlen + qpt - 1) / qpt;
  return it.qlen > 0;
}

// key tiles of query block mb: keys [0, lcp + min(qlen, (mb+1)*qpt))
__device__ __forceinline__ int tiles_of(const Item& it, int mb, int qpt) {
  return (it.lcp + min(it.qlen, (mb + 1) * qpt) + BKEY - 1) / BKEY;
}

template <int HDP>
__global__ void __launch_bounds__(kThreads, 1) attention_kernel(Args a, int n_items) {
  using T = Tile<HDP>;
  constexpr int Q_BYTES = T::Q_BYTES, KV_BYTES = T::KV_BYTES, CH = T::CHUNKS, NS = T::NS;
  constexpr int HD = HDP;  // smem row width (elements)
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;  // 1024-aligned for the SWIZZLE_128B atoms
  uint8_t* sQ0 = smem;
  uint8_t* sKV0 = smem + 2 * Q_BYTES;  // stage i: K at sKV0 + i*2*KV_BYTES, V right after
  uint8_t* sP = sKV0 + NS * 2 * KV_BYTES;
  float* sL = reinterpret_cast<float*>(sP + P_BYTES);  // [2][128] row sums for the epilogue
  uint64_t* bars = reinterpret_cast<uint64_t*>(sL + 256);
  uint64_t* q_full = bars + 0;            // [2]
  uint64_t* q_free = bars + 2;            // [2]
  uint64_t* kv_full = bars + 4;           // [NS]
  uint64_t* kv_free = bars + 4 + NS;      // [NS]
  uint64_t* s_full = bars + 4 + 2 * NS;   // [2]
  uint64_t* s_free = bars + 6 + 2 * NS;   // [2]
  uint64_t* p_full = bars + 8 + 2 * NS;
  uint64_t* pv_done = bars + 9 + 2 * NS;
  uint64_t* o_full = bars + 10 + 2 * NS;  // [2]
  uint64_t* o_free = bars + 12 + 2 * NS;  // [2]
  uint64_t* l_full = bars + 14 + 2 * NS;  // [2]
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 16 + 2 * NS);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int group = a.heads / a.kv_heads;
  const int qpt = BQ / group;  // queries per tile

  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&q_full[i], 128);
      mbar_init(&q_free[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&s_free[i], 128);
      mbar_init(&o_full[i], 1);
      mbar_init(&o_free[i], 128);
      mbar_init(&l_full[i], 128);
    }
    for (int i = 0; i < NS; ++i) {
      mbar_init(&kv_full[i], 128);
      mbar_init(&kv_free[i], 1);
    }
    mbar_init(p_full, 128);
    mbar_init(pv_done, 1);
    fence_mbar_init();
  }
  if (warp == 12) {
    tmem_alloc(tmem_holder, TMEM_COLS);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  if (threadIdx.x == 0) RDX_TRACE(0);

  if (warp >= 8 && warp < 12) {
    // ---------------------------------------------------------------- loaders
    // cp.async (LDGSTS) 16-byte copies that arrive on the stage barrier when
    // they land: several tiles in flight without register staging.
    const int t = threadIdx.x - 256;  // 0..127
    constexpr int KCH = CH / 2;       // chunks per thread per K (or V) row
    const int kr = t >> 1, kc0 = (t & 1) * KCH;
    int step = 0, blk = 0;
    Item it;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
      if (!load_item(a, item, qpt, it)) continue;
      const int64_t kcol = static_cast<int64_t>(a.heads) * a.hd + static_cast<int64_t>(it.g) * a.hd;
      const int64_t vcol = kcol + static_cast<int64_t>(a.kv_heads) * a.hd;
      for (int mb = 0; mb < it.n_mb; ++mb, ++blk) {
        const int qb = blk & 1;
        if (blk >= 2) mbar_wait(&q_free[qb], ((blk >> 1) - 1) & 1);
        const uint32_t sq = smem_u32(sQ0 + qb * Q_BYTES);
#pragma unroll
        for (int k = 0; k < CH; ++k) {
          const int idx = t + k * 128;
          const int r = idx / CH, c = idx % CH;
          const int hh = r / qpt, qi = mb * qpt + (r - hh * qpt);
          const bool ok = qi < it.qlen && c * 8 < a.hd;
          const __nv_bfloat16* src = ok ? a.qkv + static_cast<int64_t>(it.q0 + qi) * a.ld +
                                              static_cast<int64_t>(it.g * group + hh) * a.hd + c * 8
                                        : a.qkv;
          cp_async16(sq + sw_off(r, c, BQ), src, ok ? 16u : 0u);
        }
        cp_async_arrive(&q_full[qb]);
        const int n_kt = tiles_of(it, mb, qpt);
        for (int kt = 0; kt < n_kt; ++kt, ++step) {
          const int st = step % NS;
          if (step >= NS) mbar_wait(&kv_free[st], ((step / NS) - 1) & 1);
          const uint32_t sk = smem_u32(sKV0 + st * 2 * KV_BYTES), sv = sk + KV_BYTES;
          const int j = kt * BKEY + kr;
          const bool ok = j < it.L;
          const int64_t row =
              !ok ? 0 : (a.scatter ? static_cast<int64_t>(__ldg(a.scatter + it.k0 + j)) : static_cast<int64_t>(it.k0 + j));
          const __nv_bfloat16* base = a.qkv + row * a.ld;
#pragma unroll
          for (int k = 0; k < KCH; ++k) {
            const int c = kc0 + k;
            const bool cok = ok && c * 8 < a.hd;
            const uint32_t off = sw_off(kr, c, BKEY);
            cp_async16(sk + off, cok ? base + kcol + c * 8 : a.qkv, cok ? 16u : 0u);
            cp_async16(sv + off, cok ? base + vcol + c * 8 : a.qkv, cok ? 16u : 0u);
          }
          cp_async_arrive(&kv_full[st]);
        }
      }
    }
  } else if (warp == 12) {
    // ---------------------------------------------------------------- MMA issuer
    if (lane == 0) {
      const uint32_t pa = smem_u32(sP);
      int step = 0, blk = 0;
      int prev_stage = -1, prev_blk = -1, prev_last = 0, prev_first = 0;
      auto issue_pv = [&](int pstep) {
        if (prev_first && prev_blk >= 2) mbar_wait(&o_free[prev_blk & 1], ((prev_blk >> 1) - 1) & 1);
        mbar_wait(p_full, pstep & 1);
        tc_fence_after();
        const uint32_t va = smem_u32(sKV0 + prev_stage * 2 * KV_BYTES) + KV_BYTES;
        const uint32_t o = tmem + O_COL + (prev_blk & 1) * 128;
#pragma unroll
        for (int kk = 0; kk < BKEY / 16; ++kk)
          umma_bf16(o, sdesc(pa + kk * 32, 16, 1024), sdesc(va + kk * 2048, BKEY * 128, 1024), T::IDESC_PV,
                    (prev_first && kk == 0) ? 0u : 1u);
        umma_commit(&kv_free[prev_stage]);
        umma_commit(pv_done);
        if (prev_last) umma_commit(&o_full[prev_blk & 1]);
      };
      Item it;
      for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
        if (!load_item(a, item, qpt, it)) continue;
        for (int mb = 0; mb < it.n_mb; ++mb, ++blk) {
          const int qb = blk & 1;
          mbar_wait(&q_full[qb], (blk >> 1) & 1);
          fence_proxy_async_smem();  // cp.async (generic proxy) writes -> tcgen05 operand reads
          tc_fence_after();
          const uint32_t qa = smem_u32(sQ0 + qb * Q_BYTES);
          const int n_kt = tiles_of(it, mb, qpt);
          for (int kt = 0; kt < n_kt; ++kt, ++step) {
            const int st = step % NS;
            mbar_wait(&kv_full[st], (step / NS) & 1);
            if (step < 8) RDX_TRACE(8 + step * 7 + 0);
            if (step >= 2) mbar_wait(&s_free[step & 1], ((step >> 1) - 1) & 1);
            if (step < 8) RDX_TRACE(8 + step * 7 + 1);
            fence_proxy_async_smem();
            tc_fence_after();
            const uint32_t ka = smem_u32(sKV0 + st * 2 * KV_BYTES);
            const uint32_t sacc = tmem + S_COL + (step & 1) * 64;
#pragma unroll
            for (int kk = 0; kk < HD / 16; ++kk)
              umma_bf16(sacc, sdesc(qa + (kk >> 2) * (BQ * 128) + (kk & 3) * 32, 16, 1024),
                        sdesc(ka + (kk >> 2) * (BKEY * 128) + (kk & 3) * 32, 16, 1024), T::IDESC_S,
                        kk > 0 ? 1u : 0u);
            umma_commit(&s_full[step & 1]);
            if (kt == n_kt - 1) umma_commit(&q_free[qb]);  // last S of this block reads Q(qb)
            if (prev_stage >= 0) issue_pv(step - 1);        // PV(step-1) overlaps S(step)
            prev_stage = st;
            prev_blk = blk;
            prev_first = kt == 0;
            prev_last = kt == n_kt - 1;
          }
        }
      }
      if (prev_stage >= 0) issue_pv(step - 1);
    }
  } else if (warp < 4) {
    // ---------------------------------------------------------------- softmax (row t)
    const int t = threadIdx.x;  // 0..127 == TMEM lane
    const uint32_t lane_base = tmem + (static_cast<uint32_t>(warp * 32) << 16);
    int step = 0, blk = 0;
    Item it;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
      if (!load_item(a, item, qpt, it)) continue;
      for (int mb = 0; mb < it.n_mb; ++mb, ++blk) {
        const int qi = mb * qpt + (t % qpt);
        const int pos = it.lcp + qi;                       // keys 0..pos visible
        const int pos_min = __reduce_min_sync(0xffffffffu, pos);
        const uint32_t o_base = lane_base + O_COL + (blk & 1) * 128;
        float m_run = -INFINITY, l_run = 0.f;
        const int n_kt = tiles_of(it, mb, qpt);
        for (int kt = 0; kt < n_kt; ++kt, ++step) {
          const uint32_t s_base = lane_base + S_COL + (step & 1) * 64;
          mbar_wait(&s_full[step & 1], (step >> 1) & 1);
          if (t == 0 && step < 8) RDX_TRACE(8 + step * 7 + 3);
          tc_fence_after();
          float sv[64];
          tmem_ld32p(s_base, sv);
          tmem_ld32p(s_base + 32, sv + 32);
          tmem_wait_ld();
          tc_fence_before();
          mbar_arrive(&s_free[step & 1]);  // S buffer may be overwritten by S(step + 2)
          const bool diag = kt * BKEY + BKEY - 1 > pos_min;  // warp-uniform: some key masked
          float mx[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) mx[u] = -INFINITY;
          if (diag) {
#pragma unroll
            for (int j = 0; j < 64; ++j) {
              sv[j] = (kt * BKEY + j <= pos) ? sv[j] * a.scale_log2 : -INFINITY;
              mx[j & 7] = fmaxf(mx[j & 7], sv[j]);
            }
          } else {
#pragma unroll
            for (int j = 0; j < 64; ++j) {
              sv[j] *= a.scale_log2;
              mx[j & 7] = fmaxf(mx[j & 7], sv[j]);
            }
          }
          const float mt = fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])),
                                 fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7])));
          const float m_new = fmaxf(m_run, mt);
          const float m_use = m_new == -INFINITY ? 0.f : m_new;
          const float alpha = ex2(m_run - m_use);
          m_run = m_new;
          float ls[8];
          uint32_t pw[32];
#pragma unroll
          for (int u = 0; u < 8; ++u) ls[u] = 0.f;
#pragma unroll
          for (int j = 0; j < 64; j += 2) {
            const float p0 = ex2(sv[j] - m_use), p1 = ex2(sv[j + 1] - m_use);
            ls[(j >> 1) & 7] += p0 + p1;
            pw[j >> 1] = pack_bf16x2(p0, p1);
          }
          l_run = l_run * alpha +
                  (((ls[0] + ls[1]) + (ls[2] + ls[3])) + ((ls[4] + ls[5]) + (ls[6] + ls[7])));
          if (t == 0 && step < 8) RDX_TRACE(8 + step * 7 + 4);
          if (step > 0) {
            // PV(step - 1) done: O may be rescaled and P overwritten
            mbar_wait(pv_done, (step - 1) & 1);
            if (t == 0 && step < 8) RDX_TRACE(8 + step * 7 + 5);
            tc_fence_after();
            if (kt > 0 && __any_sync(0xffffffffu, alpha != 1.f)) {
#pragma unroll
              for (int c = 0; c < HD; c += 32) {
                float ov[32];
                tmem_ld32p(o_base + c, ov);
                tmem_wait_ld();
#pragma unroll
                for (int j = 0; j < 32; ++j) ov[j] *= alpha;
                tmem_st32(o_base + c, ov);
              }
              tmem_wait_st();
            }
          }
          const uint32_t prow = smem_u32(sP) + t * 128;
#pragma unroll
          for (int c = 0; c < 8; ++c)
            st_shared_v4(prow + ((c ^ (t & 7)) << 4), pw[4 * c], pw[4 * c + 1], pw[4 * c + 2], pw[4 * c + 3]);
          fence_proxy_async_smem();
          tc_fence_before();
          mbar_arrive(p_full);
          if (t == 0 && step < 8) RDX_TRACE(8 + step * 7 + 6);
        }
        if (blk >= 2) mbar_wait(&o_free[blk & 1], ((blk >> 1) - 1) & 1);  // epilogue of blk-2 read sL
        sL[(blk & 1) * 128 + t] = l_run;
        mbar_arrive(&l_full[blk & 1]);
      }
    }
  } else {
    // ---------------------------------------------------------------- epilogue (warps 4-7)
    const int t = (warp & 3) * 32 + lane;  // TMEM lane of this thread's row
    const uint32_t lane_base = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16);
    int blk = 0;
    Item it;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
      if (!load_item(a, item, qpt, it)) continue;
      for (int mb = 0; mb < it.n_mb; ++mb, ++blk) {
        const int hh = t / qpt, qi = mb * qpt + (t - hh * qpt);
        const uint32_t o_base = lane_base + O_COL + (blk & 1) * 128;
        mbar_wait(&o_full[blk & 1], (blk >> 1) & 1);
        mbar_wait(&l_full[blk & 1], (blk >> 1) & 1);
        tc_fence_after();
        const float l = sL[(blk & 1) * 128 + t];
        const float inv = l > 0.f ? 1.f / l : 0.f;
        const bool valid = qi < it.qlen;
        __nv_bfloat16* orow = a.out + static_cast<int64_t>(it.q0 + (valid ? qi : 0)) * a.ld_out +
                              static_cast<int64_t>(it.g * group + hh) * a.hd;
#pragma unroll
        for (int c = 0; c < HD; c += 32) {
          if (c < a.hd) {
            float ov[32];
            tmem_ld32p(o_base + c, ov);
            tmem_wait_ld();
            if (valid) {
#pragma unroll
              for (int j = 0; j < 32; j += 8)
                if (c + j < a.hd)
                  st_global_v4(orow + c + j, pack_bf16x2(ov[j] * inv, ov[j + 1] * inv),
                               pack_bf16x2(ov[j + 2] * inv, ov[j + 3] * inv),
                               pack_bf16x2(ov[j + 4] * inv, ov[j + 5] * inv),
                               pack_bf16x2(ov[j + 6] * inv, ov[j + 7] * inv));
            }
          }
        }
        tc_fence_before();
        mbar_arrive(&o_free[blk & 1]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 12) {
    tc_fence_after();
    tmem_dealloc(tmem, TMEM_COLS);
  }
}

unsigned long long* g_trace = nullptr;  // debug: RDX_ATTN_TRACE=1 allocates 4096 x 64 timestamps

template <int HDP>
int launch(const Args& a, int64_t grid, cudaStream_t st) {
  static bool attr_set = false;
  if (!attr_set) {
    RDX_CUDA_TRY(cudaFuncSetAttribute(attention_kernel<HDP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      Tile<HDP>::SMEM));
    attr_set = true;
  }
  const int64_t ctas = grid < num_sms() ? grid : num_sms();
  attention_kernel<HDP><<<static_cast<unsigned>(ctas), kThreads, Tile<HDP>::SMEM, st>>>(a, static_cast<int>(grid));
  RDX_LAUNCH_CHECK();
  return RDX_OK;
}

}  // namespace attn
}  // namespace rdx

extern "C" int rdx_attention_trace(void* host_out, size_t bytes) {
  using namespace rdx::attn;
  if (!g_trace) {
    if (cudaMalloc(&g_trace, 4096 * 64 * 8) != cudaSuccess) return RDX_ERR_CUDA;
    cudaMemset(g_trace, 0, 4096 * 64 * 8);
    return RDX_OK;
  }
  if (host_out) cudaMemcpy(host_out, g_trace, bytes < 4096 * 64 * 8 ? bytes : 4096 * 64 * 8, cudaMemcpyDeviceToHost);
  return RDX_OK;
}

extern "C" int rdx_attention(const void* qkv_bf16, int64_t ld_qkv, const int32_t* scatter, const int32_t* cu,
                             const int32_t* cu_q, int64_t n_seqs, int32_t max_q_len, int32_t heads, int32_t kv_heads,
                             int32_t head_dim, float softmax_scale, void* out_bf16, int64_t ld_out, void* stream) {
  using namespace rdx;
  using namespace rdx::attn;
  if (head_dim <= 0 || head_dim > 128 || head_dim % 8) return RDX_ERR_UNSUPPORTED;
  if (kv_heads <= 0 || heads % kv_heads || (BQ % (heads / kv_heads))) return RDX_ERR_SHAPE_MISMATCH;
  if ((ld_qkv % 8) || (ld_out % 8)) return RDX_ERR_SHAPE_MISMATCH;
  if (n_seqs <= 0 || max_q_len <= 0) return RDX_OK;
  if (!qkv_bf16 || !cu || !cu_q || !out_bf16) return RDX_ERR_INVALID_ARGUMENT;
  Args a;
  a.qkv = static_cast<const __nv_bfloat16*>(qkv_bf16);
  a.ld = ld_qkv;
  a.scatter = scatter;
  a.cu = cu;
  a.cu_q = cu_q;
  a.out = static_cast<__nv_bfloat16*>(out_bf16);
  a.ld_out = ld_out;
  a.nseq = static_cast<int>(n_seqs);
  a.heads = heads;
  a.kv_heads = kv_heads;
  a.hd = head_dim;
  a.scale_log2 = softmax_scale * 1.4426950408889634f;
  a.trace = g_trace;
  const int64_t grid = n_seqs * kv_heads;
  if (grid >= (int64_t(1) << 31)) return RDX_ERR_CAPACITY_EXCEEDED;
  return head_dim <= 64 ? launch<64>(a, grid, as_stream(stream)) : launch<128>(a, grid, as_stream(stream));
}
