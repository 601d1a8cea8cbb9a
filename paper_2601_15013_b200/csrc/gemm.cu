// gemm.cu — persistent warp-specialised tcgen05/TMEM GEMM for sm_100a with the
// fused RadixMLP epilogues (model.py:352-399 on the compact rows).
//
//   acc[m, n] = sum_k A[m, k] * B[n, k]        A: activations [M, K] bf16
//                                              B: weight [N, K] bf16 ([out, in])
// CG = 1: one CTA per 128 x BN tile, tcgen05.mma.cta_group::1 (M = 128).
// CG = 2: a CTA pair (cluster of 2) per 256 x BN tile, tcgen05.mma.cta_group::2
//         (M = 256): each CTA stages its 128 rows of A and BN/2 rows of B, the
//         leader issues the MMA for both, so per-SM operand traffic drops by a
//         third versus CG = 1 at the same accumulator size.
// CTA = 6 warps:
//   warp 0      TMA producer (one lane): A/B k-blocks -> smem ring
//   warp 1      TMEM allocator + MMA issuer (one lane, leader CTA)
//   warps 2..5  epilogue: tcgen05.ld -> fused op -> swizzled smem box ->
//               TMA store (bf16 / fp32) or TMA reduce-add (fp32 residual)
// Pipelines: smem full/empty mbarriers (TMA <-> MMA), two TMEM accumulator
// buffers with full/empty mbarriers (MMA <-> epilogue), static persistent
// tile schedule (M fastest).  Each output row depends only on its own A row:
// no split-K and an M-independent tile shape, so compact and full forwards
// give bit-identical rows (the reference's _mm rule, model.py:124-144).
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <type_traits>

#include "common.cuh"

namespace rdx {
namespace gemm {

constexpr int BM = 128;  // rows per CTA
constexpr int BK = 64;   // 64 bf16 = 128 B = one SWIZZLE_128B atom row
constexpr int kEpiWarps = 8;   // 2 per TMEM lane quarter, each owning half of the tile's columns
constexpr int kThreads = 64 + 32 * kEpiWarps;

// Debug build (-DRDX_GEMM_STATS_BUILD): clock64 wait / busy counters per role,
// read with rdx_gemm_debug_stats.  [0] MMA waits on tempty, [1] MMA waits on
// full stages, [2] MMA loop total, [3] epilogue waits on tfull (sum over warps),
// [4] epilogue busy (tfull seen -> accumulator released), [5] epilogue tiles.
#ifdef RDX_GEMM_STATS_BUILD
__device__ unsigned long long g_gemm_stats[8];
// %globaltimer landmarks of one launch (ns): [0] first CTA entry (min), [1] last CTA entry,
// [2] last CTA past its prologue, [3] first MMA operand stage ready (min), [4] last MMA
// commit (max), [5] last epilogue warp done (max), [6] last CTA exit (max)
__device__ unsigned long long g_gemm_times[8];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define GTIME_MIN(k) atomicMin(&g_gemm_times[k], gtimer())
#define GTIME_MAX(k) atomicMax(&g_gemm_times[k], gtimer())
#define GST_WAIT(slot, ...)                 \
  do {                                      \
    const long long _t = clock64();         \
    __VA_ARGS__;                            \
    slot += clock64() - _t;                 \
  } while (0)
#else
#define GTIME_MIN(k) do {} while (0)
#define GTIME_MAX(k) do {} while (0)
#define GST_WAIT(slot, ...) __VA_ARGS__
#endif

constexpr int kSwigluUnit = 64;     // gate/up interleave unit (columns)
constexpr int kEpiBoxBytes = 4096;  // staging box: 32 rows x 32 cols (bf16: 64 B rows, f32: 128 B rows)

struct EpiParams {
  const float* qn;
  const float* kn;
  const float2* rope;
  int rope_ps;  // float2 stride between column pairs: 1 = row-major [M][hd/2], 32 = lane-blocked
  const uint32_t* rope_pos;  // non-null: (cos, sin) computed in the epilogue from positions
  double rope_theta;
  int hd, q_dim, kv_dim;
  float eps;
  // fused RMSNorm of the A rows: acc row m *= rsqrt(sum_t row_ss[m*ss_parts+t] / norm_dim + norm_eps)
  const float* row_ss;
  int ss_parts;
  float inv_norm_dim, norm_eps;
  // RDX_EPI_RESID_NORM: h (fp32, in/out), hb = bf16(h_new), ss_out = per-64-column partial sum of h_new^2
  float* h;
  int64_t ldh;
  __nv_bfloat16* hb;
  int64_t ldhb;
  float* ss_out;
  int ss_out_parts;
  // Column partition (cp_ncol > 0): each row block is cut into cp_ncol column tiles of
  // cp_wide (where bit c of cp_mask is set) or cp_narrow columns, multiples of 32 that
  // sum to N.  Chosen on the host when the tile count is only a few rounds of the
  // persistent grid, so the rounds stay balanced (see choose_colpart).
  int cp_ncol, cp_wide, cp_narrow;
  uint32_t cp_mask;
  // chained A (rdx_rmsnorm_rows_after with ready_ctr): A rows of 32-row slab s are ready
  // once a_ready[s] >= a_ready_use * rows(s); the producer waits per tile instead of the
  // launch waiting for the whole norm grid (programmatic dependent without griddepcontrol.wait)
  const uint32_t* a_ready;
  uint32_t a_ready_use;
  // RDX_EPI_RESID_F32 with a completion counter: tiles in row-block-major order, and
  // per 32-row slab the number of columns whose stores have completed
  uint32_t* done_ctr;
  // tile raster: groups of group_m row blocks, row block fastest inside a group
  // (group_m = 1: row-block-major; >= m_tiles: column-block-major)
  int group_m;
};

constexpr int kNormGroup = 64;  // columns per partial sum of squares (RDX_EPI_RESID_NORM)

// rsqrt(mean of squares + eps) of row r from its partial sums (fixed order: deterministic).
__device__ __forceinline__ float row_rstd(const EpiParams& ep, int64_t r) {
  const float* p = ep.row_ss + r * ep.ss_parts;
  float s = 0.f;
  for (int t = 0; t < ep.ss_parts; ++t) s += __ldg(p + t);
  return rsqrtf(s * ep.inv_norm_dim + ep.norm_eps);
}

template <int BN, int CG, int EPI>
struct Cfg {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_ROWS = BN / CG;
  static constexpr int B_BYTES = B_ROWS * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  // RESID_NORM warps stage two fp32 boxes (h in/out) and two bf16 boxes (hb out)
  static constexpr int EPI_WARP_BYTES = EPI == RDX_EPI_RESID_NORM ? 2 * kEpiBoxBytes + 2 * 2048 : 2 * kEpiBoxBytes;
  static constexpr int EPI_BYTES = kEpiWarps * EPI_WARP_BYTES;
  // QKV only: q/k-norm weights (2 x 128 fp32) and the RoPE inverse frequencies (64 x (hi, lo)
  // fp32).  Other epilogues keep none, which leaves an SM room for a small rmsnorm block
  // beside the GEMM CTA (its 1 KB per-block reservation included).
  static constexpr int AUX_BYTES = EPI == RDX_EPI_QKV ? 1536 : 0;
  static constexpr int BAR_BYTES = 512;
  static constexpr int BUDGET = 227 * 1024 - 1024 - BAR_BYTES - EPI_BYTES - AUX_BYTES;
  static constexpr int STAGES = (BUDGET / STAGE_BYTES) > 8 ? 8 : (BUDGET / STAGE_BYTES);
  static constexpr int SMEM = 1024 + STAGES * STAGE_BYTES + EPI_BYTES + AUX_BYTES + BAR_BYTES;
  static constexpr uint32_t IDESC = umma_idesc_bf16(BM * CG, BN);
  static constexpr uint32_t IDESC_HALF = umma_idesc_bf16(BM * CG, BN / 2);
  static constexpr uint32_t IDESC_QUARTER = umma_idesc_bf16(BM * CG, BN / 4);
  static constexpr uint32_t TMEM_COLS = 2 * BN;
  static_assert(STAGES >= 3, "pipeline too shallow");
};

// ------------------------------------------------------------------ epilogue plumbing
// Each epilogue warp owns kEpiWarpBytes of staging smem, used as a ring of
// TMA-store boxes (32 rows x 32 columns): four 2 KB boxes for bf16 outputs,
// two 4 KB boxes for fp32, so a warp keeps 3 (1) stores in flight.
constexpr int kEpiWarpBytes = 2 * kEpiBoxBytes;

template <int NB>
struct EpiWarp {
  uint8_t* base;
  int cur;
  int lane;
  int32_t row0;     // first global row of this warp's 32-row slab
  uint64_t* lbar;   // RESID_NORM: two TMA-load barriers (one per fp32 box)
  uint32_t lphase;  // their phase bits
};

template <int NB>
__device__ __forceinline__ uint32_t epi_acquire(EpiWarp<NB>& e) {
  if (e.lane == 0) bulk_wait_read<NB - 1>();  // the box written NB emits ago has been read by its TMA store
  __syncwarp();
  return smem_u32(e.base + e.cur * (kEpiWarpBytes / NB));
}

template <int NB>
__device__ __forceinline__ void epi_issue(EpiWarp<NB>& e, const CUtensorMap* map, int32_t c0, bool reduce_add) {
  fence_proxy_async_smem();
  __syncwarp();
  if (e.lane == 0) {
    const uint8_t* box = e.base + e.cur * (kEpiWarpBytes / NB);
    if (reduce_add) tma_reduce_add_2d(map, box, c0, e.row0);
    else tma_store_2d(map, box, c0, e.row0);
    bulk_commit();
  }
  e.cur = (e.cur + 1) % NB;
}

// 32 bf16 columns of this lane's row -> 64 B row of a SWIZZLE_64B box -> TMA store at (c0, row0).
template <int NB>
__device__ __forceinline__ void emit_bf16x32(EpiWarp<NB>& e, const float* v, const CUtensorMap* map, int32_t c0) {
  uint32_t w[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) w[j] = pack_bf16x2(v[2 * j], v[2 * j + 1]);
  const uint32_t base = epi_acquire(e) + e.lane * 64;
  const int sw = (e.lane >> 1) & 3;
#pragma unroll
  for (int j = 0; j < 4; ++j) st_shared_v4(base + ((j ^ sw) << 4), w[4 * j], w[4 * j + 1], w[4 * j + 2], w[4 * j + 3]);
  epi_issue(e, map, c0, false);
}

// Two 32-column bf16 boxes behind one proxy fence and one bulk group.  Used by
// the QKV epilogue (HD >= 64), which then emits only pairs: with every group two
// boxes, the two ring slots about to be written (the 4th and 3rd most recent) are
// free once at most one group is still being read.
template <int NB>
__device__ __forceinline__ void emit_bf16x32_pair(EpiWarp<NB>& e, const float* v1, int32_t c1, const float* v2,
                                                  int32_t c2, const CUtensorMap* map) {
  static_assert(NB == 4, "pair emits assume a ring of four boxes");
  if (e.lane == 0) bulk_wait_read<1>();
  __syncwarp();
  const int sw = (e.lane >> 1) & 3;
#pragma unroll
  for (int b = 0; b < 2; ++b) {
    const float* v = b ? v2 : v1;
    uint32_t w[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) w[j] = pack_bf16x2(v[2 * j], v[2 * j + 1]);
    const uint32_t base = smem_u32(e.base + ((e.cur + b) % NB) * (kEpiWarpBytes / NB)) + e.lane * 64;
#pragma unroll
    for (int j = 0; j < 4; ++j) st_shared_v4(base + ((j ^ sw) << 4), w[4 * j], w[4 * j + 1], w[4 * j + 2], w[4 * j + 3]);
  }
  fence_proxy_async_smem();
  __syncwarp();
  if (e.lane == 0) {
    tma_store_2d(map, e.base + e.cur * (kEpiWarpBytes / NB), c1, e.row0);
    tma_store_2d(map, e.base + ((e.cur + 1) % NB) * (kEpiWarpBytes / NB), c2, e.row0);
    bulk_commit();
  }
  e.cur = (e.cur + 2) % NB;
}

// 32 fp32 columns -> 128 B row of a SWIZZLE_128B box -> TMA store or reduce-add.
template <int NB>
__device__ __forceinline__ void emit_f32x32(EpiWarp<NB>& e, const float* v, const CUtensorMap* map, int32_t c0,
                                            bool reduce_add) {
  const uint32_t base = epi_acquire(e) + e.lane * 128;
#pragma unroll
  for (int j = 0; j < 8; ++j)
    st_shared_v4(base + ((j ^ (e.lane & 7)) << 4), __float_as_uint(v[4 * j]), __float_as_uint(v[4 * j + 1]),
                 __float_as_uint(v[4 * j + 2]), __float_as_uint(v[4 * j + 3]));
  epi_issue(e, map, c0, reduce_add);
}

// packed fp32 pairs (FFMA2 / FMUL2 / FADD2 on sm_100a): IEEE-identical to the scalar ops
__device__ __forceinline__ uint64_t p2(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void up2(uint64_t r, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}
__device__ __forceinline__ uint64_t fma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t mul2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t add2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
constexpr uint64_t kNeg2 = 0x8000000080000000ULL;

// (cos, sin) of pos * inv_freq for two columns at once: the same operations as
// rope_cs below on packed pairs (identical bits), MUFU sin/cos per element.
__device__ __forceinline__ void rope_cs2(uint64_t pos2, float4 f, float& c0, float& s0, float& c1, float& s1) {
  const uint64_t ghi = p2(f.x, f.z), glo = p2(f.y, f.w);
  const uint64_t t = mul2(pos2, ghi);
  uint64_t e = fma2(pos2, ghi, t ^ kNeg2);
  e = fma2(pos2, glo, e);
  float t0, t1;
  up2(t, t0, t1);
  const uint64_t r = mul2(add2(add2(t, p2(-rintf(t0), -rintf(t1))), e), p2(6.283185307179586f, 6.283185307179586f));
  float r0, r1;
  up2(r, r0, r1);
  __sincosf(r0, &s0, &c0);
  __sincosf(r1, &s1, &c1);
}

// (cos, sin) of pos * inv_freq for one column.  g = inv_freq / (2*pi) in fp64,
// kept as an fp32 (hi, lo) pair; the angle in turns is pos*g_hi (exact FMA
// residual) + pos*g_lo, its integer part drops out exactly, and MUFU sin/cos run
// on the remaining [-1/2, 1/2] turn.  |error| < 1e-6 rad against the fp64 angle
// for positions < 2^20, far below the bf16 output rounding.
__device__ __forceinline__ void rope_cs(float pos, float ghi, float glo, float& c, float& s) {
  const float t = pos * ghi;
  float e = fmaf(pos, ghi, -t);
  e = fmaf(pos, glo, e);
  const float r = (t - rintf(t)) + e;  // t - rint(t) is exact
  __sincosf(r * 6.283185307179586f, &s, &c);
}

// RoPE on a (first-half, second-half) pair of 32-column slices of a normalised head:
// x1 = cols [c, c+32), x2 = cols [c+H, c+H+32) of a head of width 2H (model.py:363-365).
// cs = this lane's (cos, sin) of column c; column c + j sits at cs + j * ps (j even).
__device__ __forceinline__ void rope_pair32(float* x1, float* x2, const float* w1, const float* w2, float inv,
                                            const float2* __restrict__ cs, int ps) {
#pragma unroll
  for (int j = 0; j < 32; j += 2) {
    const float4 t = __ldg(reinterpret_cast<const float4*>(cs + j * ps));
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const float c = u ? t.z : t.x, s = u ? t.w : t.y;
      const float a = x1[j + u] * inv * w1[j + u];
      const float b = x2[j + u] * inv * w2[j + u];
      x1[j + u] = a * c - b * s;
      x2[j + u] = b * c + a * s;
    }
  }
}

// QKV epilogue for this warp's column range [c_lo, c_hi) of the tile (multiple of HD).
template <int HD, int NB>
__device__ __forceinline__ void qkv_cols(EpiWarp<NB>& e, uint32_t taddr, int64_t n0, int c_lo, int c_hi, int64_t N,
                                         const EpiParams& ep, const float* s_qn, const float* s_kn,
                                         const float2* rope_row, const CUtensorMap* map, float rs, float pos) {
  if constexpr (HD >= 64) {
    constexpr int H = HD / 2;
#pragma unroll 1
    for (int h0 = c_lo; h0 < c_hi; h0 += HD) {
      const int64_t col0 = n0 + h0;
      if (col0 >= N) break;
      const int kind = col0 < ep.q_dim ? 0 : (col0 < ep.q_dim + ep.kv_dim ? 1 : 2);
      if (kind == 2) {
#pragma unroll 1
        for (int c = 0; c < HD; c += 64) {
          float v[64];
          tmem_ld32p(taddr + h0 + c, v);
          tmem_ld32p(taddr + h0 + c + 32, v + 32);
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 64; ++j) v[j] *= rs;
          emit_bf16x32_pair(e, v, static_cast<int32_t>(col0 + c), v + 32, static_cast<int32_t>(col0 + c + 32), map);
        }
        continue;
      }
      const float* w = kind == 0 ? s_qn : s_kn;
      float ss;
      {
        // sum of squares of the head row: two TMEM loads per wait, packed FFMA2 into
        // two running sums; (v * rs)^2 = rs^2 * v^2
        uint64_t ss2 = 0ULL;
#pragma unroll
        for (int c = 0; c < HD; c += 64) {
          float v[64];
          tmem_ld32p(taddr + h0 + c, v);
          tmem_ld32p(taddr + h0 + c + 32, v + 32);
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 64; j += 2) {
            const uint64_t x = p2(v[j], v[j + 1]);
            ss2 = fma2(x, x, ss2);
          }
        }
        float s0, s1;
        up2(ss2, s0, s1);
        ss = (s0 + s1) * (rs * rs);
      }
      const float inv = rsqrtf(ss / static_cast<float>(HD) + ep.eps) * rs;  // x1/x2 below are unscaled
#pragma unroll 1
      for (int c = 0; c < H; c += 32) {
        float x1[32], x2[32];
        tmem_ld32p(taddr + h0 + c, x1);
        tmem_ld32p(taddr + h0 + H + c, x2);
        if (ep.rope_pos) {  // (cos, sin) from the position; the math overlaps the TMEM loads
          float cs[32], sn[32];
          const uint32_t fq = smem_u32(s_qn + 256);
          const uint64_t pos2 = p2(pos, pos);
#pragma unroll
          for (int j = 0; j < 32; j += 2)
            rope_cs2(pos2, ld_shared_f4(fq + 8 * (c + j)), cs[j], sn[j], cs[j + 1], sn[j + 1]);
          tmem_wait_ld();
          const uint32_t ws = smem_u32(w);
          const uint64_t inv2 = p2(inv, inv);
#pragma unroll
          for (int j = 0; j < 32; j += 4) {
            const float4 w1 = ld_shared_f4(ws + 4 * (c + j));
            const float4 w2 = ld_shared_f4(ws + 4 * (H + c + j));
#pragma unroll
            for (int u = 0; u < 4; u += 2) {
              // a = x1 * inv * w1, b = x2 * inv * w2 (same order as the scalar form)
              const uint64_t a = mul2(mul2(p2(x1[j + u], x1[j + u + 1]), inv2), u ? p2(w1.z, w1.w) : p2(w1.x, w1.y));
              const uint64_t b = mul2(mul2(p2(x2[j + u], x2[j + u + 1]), inv2), u ? p2(w2.z, w2.w) : p2(w2.x, w2.y));
              const uint64_t c2 = p2(cs[j + u], cs[j + u + 1]), s2 = p2(sn[j + u], sn[j + u + 1]);
              up2(fma2(a, c2, mul2(b, s2) ^ kNeg2), x1[j + u], x1[j + u + 1]);  // a*c - b*s
              up2(fma2(b, c2, mul2(a, s2)), x2[j + u], x2[j + u + 1]);          // b*c + a*s
            }
          }
        } else {
          tmem_wait_ld();
          rope_pair32(x1, x2, w + c, w + H + c, inv, rope_row + c * ep.rope_ps, ep.rope_ps);
        }
        emit_bf16x32_pair(e, x1, static_cast<int32_t>(col0 + c), x2, static_cast<int32_t>(col0 + H + c), map);
      }
    }
  } else {
    // HD in {16, 32}: 32-column chunks hold whole heads (HD = 32) or two heads (HD = 16).
#pragma unroll 1
    for (int c0 = c_lo; c0 < c_hi; c0 += 32) {
      const int64_t colc = n0 + c0;
      if (colc >= N) break;
      float x[32];
      tmem_ld32p(taddr + c0, x);
      tmem_wait_ld();
#pragma unroll
      for (int j = 0; j < 32; ++j) x[j] *= rs;
#pragma unroll
      for (int h = 0; h < 32; h += HD) {
        const int64_t col0 = colc + h;
        const int kind = col0 < ep.q_dim ? 0 : (col0 < ep.q_dim + ep.kv_dim ? 1 : 2);
        if (kind < 2 && col0 < N) {
          const float* w = kind == 0 ? s_qn : s_kn;
          float ss = 0.f;
#pragma unroll
          for (int j = 0; j < HD; ++j) ss += x[h + j] * x[h + j];
          const float inv = rsqrtf(ss / static_cast<float>(HD) + ep.eps);
          constexpr int H = HD / 2;
#pragma unroll
          for (int j = 0; j < H; ++j) {
            const float2 cs = __ldg(rope_row + (j & ~1) * ep.rope_ps + (j & 1));
            const float a = x[h + j] * inv * w[j];
            const float b = x[h + j + H] * inv * w[j + H];
            x[h + j] = a * cs.x - b * cs.y;
            x[h + j + H] = b * cs.x + a * cs.y;
          }
        }
      }
      emit_bf16x32(e, x, map, static_cast<int32_t>(colc));
    }
  }
}

// RDX_EPI_RESID_NORM: TMA loads of the warp's first two 32-column h chunks, issued
// before the accumulator wait so their latency overlaps the mainloop.
template <int NB>
__device__ __forceinline__ void resid_norm_prefetch(EpiWarp<NB>& e, const CUtensorMap* map, int64_t c0, int64_t N) {
  if (e.lane == 0 && c0 < N) {
    bulk_wait_read<0>();  // the previous tile's stores are done reading the boxes
    mbar_arrive_expect_tx(&e.lbar[0], 2 * kEpiBoxBytes);
    tma_load_3d(map, e.base, &e.lbar[0], 0, e.row0, static_cast<int32_t>(c0 / 32));
  }
}

// This warp: 32 rows (lane quarter) x columns [ch*BN/2, (ch+1)*BN/2) of the tile.
// All of the warp's accumulator columns are read from TMEM with one wait,
// then transformed in registers and emitted box by box.
template <int BN, int EPI, int NB>
// hw = columns per warp of this tile (BN/2, or BN/4 for a split tail tile),
// n0 = the tile's first output-space column.
__device__ __forceinline__ void epilogue_tile(EpiWarp<NB>& e, uint32_t taddr, int ch, int c_lo, int hw, int64_t gm_lane,
                                              int64_t M, int64_t n0, int64_t N, const EpiParams& ep,
                                              const float* s_qn, const float* s_kn, const CUtensorMap* map,
                                              const CUtensorMap* map_hb, float rs) {
  constexpr int HALF = BN / 2;  // hw <= HALF; c_lo = ch * hw except in a column partition
  float v[HALF];
  if constexpr (EPI == RDX_EPI_SWIGLU) {
    // warp ch owns outputs [ch*hw/2, (ch+1)*hw/2) of the tile's width/2: output o of
    // pair p = o/64 reads gate column p*128 + o%64 and up column +64
#pragma unroll
    for (int q = 0; q < HALF / 2; q += 32) {
      if (q < hw / 2) {
        const int o = ch * (hw / 2) + q;
        const int gcol = (o / kSwigluUnit) * 2 * kSwigluUnit + o % kSwigluUnit;
        tmem_ld32p(taddr + gcol, v + q);
        tmem_ld32p(taddr + gcol + kSwigluUnit, v + HALF / 2 + q);
      }
    }
  } else if constexpr (EPI != RDX_EPI_QKV) {
#pragma unroll
    for (int c = 0; c < HALF; c += 32)
      if (c < hw) tmem_ld32p(taddr + c_lo + c, v + c);
  }
  const int64_t r_clamped = gm_lane < M ? gm_lane : (M > 0 ? M - 1 : 0);
  if constexpr (EPI != RDX_EPI_QKV) tmem_wait_ld();
  if constexpr (EPI == RDX_EPI_RESID_NORM) {
    // 64-column steps: one 8 KB TMA load of h (two stacked 32x32 fp32 swizzled boxes,
    // 3-D map), each lane adds its accumulator row, writes h_new back into the box and
    // bf16(h_new) into a 4 KB 32x64 bf16 box, and both go out as one TMA store each;
    // the sum of h_new^2 over the 64 columns goes to ss_out.  Step 0's load was issued
    // before the accumulator wait (resid_norm_prefetch); later steps reuse the boxes
    // once the previous step's stores have read them.
    uint8_t* fb8 = e.base;
    uint8_t* bb8 = e.base + 2 * kEpiBoxBytes;
#pragma unroll
    for (int g = 0; g < HALF / 64; ++g) {
      const int64_t col = n0 + c_lo + 64 * g;
      if (64 * g >= hw || col >= N) break;
      if (g > 0 && e.lane == 0) {
        bulk_wait_read<0>();
        mbar_arrive_expect_tx(&e.lbar[0], 2 * kEpiBoxBytes);
        tma_load_3d(map, fb8, &e.lbar[0], 0, e.row0, static_cast<int32_t>(col / 32));
      }
      mbar_wait(&e.lbar[0], e.lphase & 1);
      e.lphase ^= 1u;
      float ssp = 0.f;
      const uint32_t bb = smem_u32(bb8) + e.lane * 128;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const uint32_t fb = smem_u32(fb8) + c * kEpiBoxBytes + e.lane * 128;
        uint32_t w[16];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint32_t addr = fb + ((j ^ (e.lane & 7)) << 4);
          float4 hv = ld_shared_f4(addr);
          const float* a = v + 64 * g + 32 * c + 4 * j;
          hv.x += a[0];
          hv.y += a[1];
          hv.z += a[2];
          hv.w += a[3];
          ssp += hv.x * hv.x + hv.y * hv.y + hv.z * hv.z + hv.w * hv.w;
          st_shared_v4(addr, __float_as_uint(hv.x), __float_as_uint(hv.y), __float_as_uint(hv.z), __float_as_uint(hv.w));
          w[2 * j] = pack_bf16x2(hv.x, hv.y);
          w[2 * j + 1] = pack_bf16x2(hv.z, hv.w);
        }
        // bf16 row of 128 B = 8 chunks of 16 B; this c fills chunks 4c .. 4c+3
#pragma unroll
        for (int j = 0; j < 4; ++j)
          st_shared_v4(bb + (((4 * c + j) ^ (e.lane & 7)) << 4), w[4 * j], w[4 * j + 1], w[4 * j + 2], w[4 * j + 3]);
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (e.lane == 0) {
        tma_store_3d(map, fb8, 0, e.row0, static_cast<int32_t>(col / 32));
        tma_store_2d(map_hb, bb8, static_cast<int32_t>(col), e.row0);
        bulk_commit();
      }
      if (gm_lane < M) ep.ss_out[gm_lane * ep.ss_out_parts + col / kNormGroup] = ssp;
    }
  } else if constexpr (EPI == RDX_EPI_STORE_BF16 || EPI == RDX_EPI_STORE_F32 || EPI == RDX_EPI_RESID_F32) {
#pragma unroll
    for (int c = 0; c < HALF; c += 32) {
      if (c < hw && n0 + c_lo + c < N) {
        if constexpr (EPI == RDX_EPI_STORE_BF16) emit_bf16x32(e, v + c, map, static_cast<int32_t>(n0 + c_lo + c));
        else emit_f32x32(e, v + c, map, static_cast<int32_t>(n0 + c_lo + c), EPI == RDX_EPI_RESID_F32);
      }
    }
  } else if constexpr (EPI == RDX_EPI_SWIGLU) {
    const int64_t nout = N / 2;
#pragma unroll
    for (int q = 0; q < HALF / 2; q += 32) {
      const int64_t ocol = n0 / 2 + ch * (hw / 2) + q;
      if (q < hw / 2 && ocol < nout) {
        float* g = v + q;
        const float* u = v + HALF / 2 + q;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float gj = g[j] * rs;
          g[j] = __fdividef(gj, 1.f + __expf(-gj)) * (u[j] * rs);
        }
        emit_bf16x32(e, g, map, static_cast<int32_t>(ocol));
      }
    }
  } else if constexpr (EPI == RDX_EPI_QKV) {
    // chunked: TMEM loads interleaved with the norm / RoPE math and the stores
    // row-major: row r at r * hd/2; blocked: ((r/32) * hd/4 * 32 + r%32) float4s
    const float2* rope_row = ep.rope_ps == 1 ? ep.rope + r_clamped * (ep.hd >> 1)
                                             : ep.rope + 2 * ((r_clamped >> 5) * (ep.hd >> 2) * 32 + (r_clamped & 31));
    // a split tail tile narrower than two heads (hw < hd, hd >= 64): the ch = 0 warp
    // takes its whole width (whole heads), the ch = 1 warp has nothing to do
    const bool whole = hw % ep.hd != 0 && ep.hd > 32;
    const int lo = whole ? (ch ? 2 * hw : 0) : c_lo;
    const int c_hi = whole ? 2 * hw : c_lo + hw;
    const float pos = ep.rope_pos ? static_cast<float>(__ldg(ep.rope_pos + r_clamped)) : 0.f;
    switch (ep.hd) {
      case 128: qkv_cols<128>(e, taddr, n0, lo, c_hi, N, ep, s_qn, s_kn, rope_row, map, rs, pos); break;
      case 64: qkv_cols<64>(e, taddr, n0, lo, c_hi, N, ep, s_qn, s_kn, rope_row, map, rs, pos); break;
      case 32: qkv_cols<32>(e, taddr, n0, lo, c_hi, N, ep, s_qn, s_kn, rope_row, map, rs, pos); break;
      default: qkv_cols<16>(e, taddr, n0, lo, c_hi, N, ep, s_qn, s_kn, rope_row, map, rs, pos); break;
    }
  }
}

// Tensor maps and scalar arguments of one GEMM ("job") of a launch.
struct alignas(64) JobMaps {
  CUtensorMap a, b, b2, b4, c, d;  // A, B (full / half or wide / quarter or narrow boxes), output, RESID_NORM bf16 out
};
struct JobArgs {
  int64_t N, K, tail_start;
  int split;
  EpiParams ep;
};
// staging boxes per epilogue warp: four 2 KB bf16 boxes or two 4 KB fp32 boxes
__host__ __device__ constexpr int nb_of(int epi) {
  return (epi == RDX_EPI_STORE_F32 || epi == RDX_EPI_RESID_F32 || epi == RDX_EPI_RESID_NORM) ? 2 : 4;
}

// ------------------------------------------------------------------ the kernel
// Per-warp epilogue state carried across tiles (and across the two jobs of a pair).
struct EpiCtx {
  uint32_t tmem_base, tempty_leader0;
  uint64_t *tfull, *tempty;
  const float* s_norm;
  uint32_t rank;
  int q, ch, lane;
  int acc;
  uint32_t acc_phase;
  long long st_w, st_b;
  long long n_t;
};

// One output tile of one job in this epilogue warp: wait for the accumulator, the fused
// epilogue (EP), release the accumulator, publish slab counters (done_ctr of a residual
// GEMM; `dep` = job 0 of a pair: the output columns job 1 waits for).
template <int BN, int CG, int EP, int NB>
__device__ __forceinline__ void epi_job_tile(EpiWarp<NB>& e, EpiCtx& x, const JobArgs& J, const JobMaps& MP,
                                             uint32_t* dep, int64_t M, int64_t m_blk, int64_t n0, int width) {
  const EpiParams& ej = J.ep;
  const int64_t N = J.N;
  const int lane = x.lane, ch = x.ch;
  e.row0 = static_cast<int32_t>(m_blk * (BM * CG) + x.rank * BM + x.q * 32);
  // row scale of the fused RMSNorm: its loads overlap the wait for the accumulator
  const int64_t gm = e.row0 + lane;
  const float rs = ej.row_ss ? row_rstd(ej, gm < M ? gm : (M > 0 ? M - 1 : 0)) : 1.f;
  if constexpr (EP == RDX_EPI_RESID_NORM) resid_norm_prefetch(e, &MP.c, n0 + ch * (width / 2), N);
  GST_WAIT(x.st_w, mbar_wait(&x.tfull[x.acc], x.acc_phase));
  const long long st_tb = clock64();
  tc_fence_after();
  const uint32_t taddr = x.tmem_base + x.acc * BN + (static_cast<uint32_t>(x.q * 32) << 16);
  // this warp's columns: halves of the tile, or in a column partition (widths in
  // 32-column boxes, possibly odd) the first ceil(boxes/2) boxes and the rest
  int c_lo = ch * (width / 2), hw = width / 2;
  if (ej.cp_ncol > 0) {
    const int w0 = ((width / 32 + 1) / 2) * 32;
    c_lo = ch ? w0 : 0;
    hw = ch ? width - w0 : w0;
  }
  epilogue_tile<BN, EP, NB>(e, taddr, ch, c_lo, hw, gm, M, n0, N, ej, x.s_norm, x.s_norm + 128, &MP.c, &MP.d, rs);
  tc_fence_before();
  __syncwarp();
  if (lane == 0) {
    if constexpr (CG == 2) mbar_arrive_cluster(x.tempty_leader0 + x.acc * 8);
    else mbar_arrive(&x.tempty[x.acc]);
  }
  x.acc ^= 1;
  if (x.acc == 0) x.acc_phase ^= 1;
  if constexpr (EP == RDX_EPI_RESID_F32) {
    if (ej.done_ctr && lane == 0 && e.row0 < M) {  // slabs past M do not exist
      // this warp's reduce-adds are complete and visible: publish its columns of the slab
      const int64_t c0 = n0 + c_lo;
      const int64_t cols = N - c0 < hw ? (N - c0 > 0 ? N - c0 : 0) : hw;
      bulk_wait_all();
      asm volatile("fence.proxy.async.global;" ::: "memory");
      __threadfence();
      atomicAdd(ej.done_ctr + (e.row0 >> 5), static_cast<uint32_t>(cols));
    }
  }
  if (dep && lane == 0 && e.row0 < M) {
    // job 1 of the pair reads these rows: publish this warp's output columns once its stores landed
    const int64_t nout = EP == RDX_EPI_SWIGLU ? N / 2 : N;
    const int64_t c0 = EP == RDX_EPI_SWIGLU ? (n0 + c_lo) / 2 : n0 + c_lo;
    const int64_t w_out = EP == RDX_EPI_SWIGLU ? hw / 2 : hw;
    const int64_t cols = nout - c0 < w_out ? (nout - c0 > 0 ? nout - c0 : 0) : w_out;
    bulk_wait_all();
    asm volatile("fence.proxy.async.global;" ::: "memory");
    __threadfence();
    atomicAdd(dep + (e.row0 >> 5), static_cast<uint32_t>(cols));
  }
  x.st_b += clock64() - st_tb;
  ++x.n_t;
}

// One launch runs one GEMM (EPI2 < 0) or two dependent GEMMs sharing M, BN and CG
// (EPI2 >= 0, rdx_gemm_pair: the MLP's gate|up -> down).  Job 1's tiles follow job 0's
// in every CTA's static schedule; a job-1 tile's producer waits until job 0 has written
// all dep_cols output columns of its A rows (per-32-row-slab counters in `dep`), so job
// 1's first tiles overlap job 0's last epilogues and one launch prologue is saved.
template <int BN, int EPI, int CG, int EPI2>
__global__ void __launch_bounds__(kThreads, 1)
gemm_kernel(const __grid_constant__ JobMaps mp0, const __grid_constant__ JobMaps mp1, int64_t M,
            const __grid_constant__ JobArgs j0, const __grid_constant__ JobArgs j1, uint32_t* dep, uint32_t dep_cols) {
  using C = Cfg<BN, CG, EPI>;
  static_assert(EPI2 < 0 || Cfg<BN, CG, EPI2 < 0 ? EPI : EPI2>::SMEM == C::SMEM, "paired jobs share one smem layout");
  const EpiParams& ep = j0.ep;  // job 0's epilogue parameters (prologue uses)
  constexpr int STAGES = C::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* epi_smem = smem + STAGES * C::STAGE_BYTES;
  float* s_norm = reinterpret_cast<float*>(epi_smem + C::EPI_BYTES);
  uint64_t* full = reinterpret_cast<uint64_t*>(epi_smem + C::EPI_BYTES + C::AUX_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* eload = tempty + 2;  // [kEpiWarps][2] epilogue TMA-load barriers (RESID_NORM)
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(eload + 2 * kEpiWarps);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    GTIME_MIN(0);
    GTIME_MAX(1);
  }
  const uint32_t rank = CG == 2 ? cluster_ctarank() : 0;
  const int64_t unit = CG == 2 ? (blockIdx.x >> 1) : blockIdx.x;
  const int64_t n_units = CG == 2 ? (gridDim.x >> 1) : gridDim.x;
  const int64_t m_tiles = (M + BM * CG - 1) / (BM * CG);
  auto n_tiles_of = [&](const JobArgs& J) -> int64_t {
    return J.ep.cp_ncol > 0 ? J.ep.cp_ncol : (J.N + BN - 1) / BN;
  };
  // Tail split: the tiles of the last partial round (from tail_start on) run as
  // `split` narrower tiles each (width BN/split), so r leftover tiles occupy
  // ceil(split*r/units)/split of a round instead of a whole one.  No split-K:
  // every output element is still one CTA's full K reduction -> same bits.
  auto num_tiles_of = [&](const JobArgs& J) -> int64_t {
    return J.tail_start + J.split * (m_tiles * n_tiles_of(J) - J.tail_start);
  };
  const int64_t nt0 = num_tiles_of(j0);
  const int64_t num_tiles = nt0 + (EPI2 >= 0 ? num_tiles_of(j1) : 0);
  // job of a schedule index and the tile index inside that job
  auto job_of = [&](int64_t tile, int64_t& t) -> int {
    if (EPI2 >= 0 && tile >= nt0) {
      t = tile - nt0;
      return 1;
    }
    t = tile;
    return 0;
  };
  auto decode = [&](const JobArgs& J, int64_t t, int64_t& m_blk, int64_t& n0, int& width) {
    const EpiParams& ej = J.ep;
    const int64_t n_tiles = n_tiles_of(J);
    int64_t f = t;
    int part = 0;
    width = BN;
    if (t >= J.tail_start) {
      f = J.tail_start + (t - J.tail_start) / J.split;
      part = static_cast<int>((t - J.tail_start) % J.split);
      width = BN / J.split;
    }
    // grouped raster: the tiles running at once cover ~group_m row blocks x a few column
    // blocks, so both A rows and B columns are re-read from L2 rather than HBM
    const int64_t gsz = static_cast<int64_t>(ej.group_m) * n_tiles;
    const int64_t g = f / gsz, r = f - g * gsz;
    const int64_t g_rows = m_tiles - g * ej.group_m < ej.group_m ? m_tiles - g * ej.group_m : ej.group_m;
    m_blk = g * ej.group_m + r % g_rows;
    const int cblk = static_cast<int>(r / g_rows);
    if (ej.cp_ncol > 0) {
      const bool wide = (ej.cp_mask >> cblk) & 1u;
      width = wide ? ej.cp_wide : ej.cp_narrow;
      n0 = static_cast<int64_t>(cblk) * ej.cp_narrow +
           static_cast<int64_t>(__popc(ej.cp_mask & ((1u << cblk) - 1u))) * (ej.cp_wide - ej.cp_narrow);
    } else {
      n0 = static_cast<int64_t>(cblk) * BN + part * width;
    }
  };

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&mp0.a);
    tma_prefetch_desc(&mp0.b);
    tma_prefetch_desc(&mp0.b2);
    tma_prefetch_desc(&mp0.b4);
    tma_prefetch_desc(&mp0.c);
    if constexpr (EPI2 >= 0) {
      tma_prefetch_desc(&mp1.a);
      tma_prefetch_desc(&mp1.b);
      tma_prefetch_desc(&mp1.b2);
      tma_prefetch_desc(&mp1.b4);
      tma_prefetch_desc(&mp1.c);
    }
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], kEpiWarps * CG);
    }
    for (int i = 0; i < 2 * kEpiWarps; ++i) mbar_init(&eload[i], 1);
    fence_mbar_init();
  }
  if (warp == 1) {
    if constexpr (CG == 2) {
      tmem_alloc_cg2(tmem_holder, C::TMEM_COLS);
      tmem_relinquish_cg2();
    } else {
      tmem_alloc(tmem_holder, C::TMEM_COLS);
      tmem_relinquish();
    }
  }
  if constexpr (EPI == RDX_EPI_QKV) {
    for (int i = threadIdx.x; i < ep.hd; i += blockDim.x) {
      s_norm[i] = ep.qn[i];
      s_norm[128 + i] = ep.kn[i];
    }
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (CG == 2) cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  if (threadIdx.x == 0) GTIME_MAX(2);
  // everything above overlapped the previous kernel's tail (PDL); inputs from here on.
  // A chained consumer does not wait for its predecessor grid: it waits per tile on the
  // norm's ready counters (producer below); weights and outputs have no other producer.
  if (!ep.a_ready) pdl_wait();
  pdl_launch_dependents();

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t tile = unit; tile < num_tiles; tile += n_units) {
        int64_t m_blk, n0, lt;
        int width;
        const int job = job_of(tile, lt);
        const JobArgs& J = job ? j1 : j0;
        const JobMaps& MP = job ? mp1 : mp0;
        decode(J, lt, m_blk, n0, width);
        const int kblocks = static_cast<int>((J.K + BK - 1) / BK);
        // B rows this CTA stages: width / CG (1, 1/2 or 1/4 of B_ROWS, or a column-partition width)
        const int b_rows = width / CG;
        const int32_t m0 = static_cast<int32_t>(m_blk * (BM * CG) + rank * BM);
        const int32_t nb0 = static_cast<int32_t>(n0 + rank * b_rows);
        const uint32_t bytes = C::A_BYTES + static_cast<uint32_t>(b_rows) * (BK * 2);
        if (job == 1 && m0 < M) {
          // job 1's A rows are job 0's output: wait until every column of them is written
#ifdef RDX_GEMM_STATS_BUILD
          const long long dw0 = clock64();
#endif
          const int64_t r_hi = (m0 + BM < M ? m0 + BM : M) - 1;
          for (int64_t slab = m0 >> 5; slab <= (r_hi >> 5); ++slab) {
            unsigned ns = 32;
            uint32_t spins = 0;
            while (ld_acquire_u32(dep + slab) < dep_cols) {
              __nanosleep(ns);
              ns = ns < 512 ? 2 * ns : ns;
              if (++spins > (1u << 24)) {  // ~8 s: job 0 never completed these rows
                atomicCAS(&g_device_status, 0, static_cast<int>(RDX_ERR_DEVICE_TIMEOUT));
                break;
              }
            }
          }
          asm volatile("fence.proxy.async.global;" ::: "memory");  // TMA-written rows -> TMA reads
#ifdef RDX_GEMM_STATS_BUILD
          atomicAdd(&g_gemm_stats[6], static_cast<unsigned long long>(clock64() - dw0));
          atomicAdd(&g_gemm_stats[7], 1ull);
#endif
        }
        if (job == 0 && ep.a_ready && m0 < M) {
          const int64_t r_hi = (m0 + BM < M ? m0 + BM : M) - 1;
          for (int64_t slab = m0 >> 5; slab <= (r_hi >> 5); ++slab) {
            const uint32_t rows = static_cast<uint32_t>(M - slab * 32 < 32 ? M - slab * 32 : 32);
            const uint32_t want = ep.a_ready_use * rows;
            unsigned ns = 64;
            uint32_t spins = 0;
            while (ld_acquire_u32(ep.a_ready + slab) < want) {
              __nanosleep(ns);
              ns = ns < 1024 ? 2 * ns : ns;
              if (++spins > (1u << 23)) {  // ~8 s: the norm never published these rows
                atomicCAS(&g_device_status, 0, static_cast<int>(RDX_ERR_DEVICE_TIMEOUT));
                break;
              }
            }
          }
          // the rows were written by generic-proxy stores of another grid: order this
          // thread's acquire before its async-proxy (TMA) reads of them
          asm volatile("fence.proxy.async.global;" ::: "memory");
        }
        const CUtensorMap* mapb;
        if (J.ep.cp_ncol > 0) {
          mapb = width == J.ep.cp_wide ? &MP.b2 : &MP.b4;  // boxes of cp_wide / cp_narrow rows (host)
        } else {
          const int div = BN / width;  // 1, 2 or 4
          mapb = div == 1 ? &MP.b : (div == 2 ? &MP.b2 : &MP.b4);
        }
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * C::STAGE_BYTES;
          uint8_t* sb = sa + C::A_BYTES;
          if constexpr (CG == 2) {
            const uint32_t bar = mapa_shared(smem_u32(&full[stage]), 0);
            if (rank == 0) mbar_arrive_expect_tx(&full[stage], 2 * bytes);
            tma_load_2d_cg2(&MP.a, sa, bar, kb * BK, m0);
            tma_load_2d_cg2(mapb, sb, bar, kb * BK, nb0);
          } else {
            mbar_arrive_expect_tx(&full[stage], bytes);
            tma_load_2d(&MP.a, sa, &full[stage], kb * BK, m0);
            tma_load_2d(mapb, sb, &full[stage], kb * BK, nb0);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {  // whole warp walks the schedule; one elected lane issues
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      long long st_te = 0, st_fu = 0;
      const long long st_t0 = clock64();
      for (int64_t tile = unit; tile < num_tiles; tile += n_units) {
        int64_t m_blk, n0, lt;
        int width;
        const int job = job_of(tile, lt);
        const JobArgs& J = job ? j1 : j0;
        decode(J, lt, m_blk, n0, width);
        const int kblocks = static_cast<int>((J.K + BK - 1) / BK);
        const uint32_t idesc = J.ep.cp_ncol > 0 ? umma_idesc_bf16(BM * CG, width)
                               : (width == BN ? C::IDESC : (width == BN / 2 ? C::IDESC_HALF : C::IDESC_QUARTER));
        GST_WAIT(st_te, mbar_wait(&tempty[acc], acc_phase ^ 1));
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < kblocks; ++kb) {
          GST_WAIT(st_fu, mbar_wait(&full[stage], phase));
#ifdef RDX_GEMM_STATS_BUILD
          if (kb == 0 && tile == unit && lane == 0) GTIME_MIN(3);
#endif
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * C::STAGE_BYTES);
          const uint64_t da = umma_sdesc_sw128(sa);
          const uint64_t db = umma_sdesc_sw128(sa + C::A_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            // +32 B per K=16 step inside the 128 B swizzle atom (encoded >> 4)
            if constexpr (CG == 2) umma_bf16_cg2_elect(d_tmem, da + 2 * k, db + 2 * k, idesc, (kb | k) != 0);
            else umma_bf16_elect(d_tmem, da + 2 * k, db + 2 * k, idesc, (kb | k) != 0);
          }
          if constexpr (CG == 2) umma_commit_cg2_mc_elect(&empty[stage], 0x3);
          else umma_commit_elect(&empty[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if constexpr (CG == 2) umma_commit_cg2_mc_elect(&tfull[acc], 0x3);
        else umma_commit_elect(&tfull[acc]);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
#ifdef RDX_GEMM_STATS_BUILD
      if (lane == 0) {
        GTIME_MAX(4);
        atomicAdd(&g_gemm_stats[0], static_cast<unsigned long long>(st_te));
        atomicAdd(&g_gemm_stats[1], static_cast<unsigned long long>(st_fu));
        atomicAdd(&g_gemm_stats[2], static_cast<unsigned long long>(clock64() - st_t0));
      }
#endif
      (void)st_te;
      (void)st_fu;
      (void)st_t0;
    }
  } else {
    const int ew = warp - 2;
    const int q = warp & 3;  // TMEM lane quarter accessible to this warp
    const int ch = ew >> 2;  // column half of the tile
    if constexpr (EPI == RDX_EPI_QKV) {
      if (ep.rope_pos) {
        // inv_freq_i = theta^(-2i/hd) in fp64 (model.py:165-172), in turns (/ 2 pi), as an fp32
        // (hi, lo) pair.  Computed here by the epilogue warps while the first tile's mainloop
        // runs (fp64 pow costs ~1.2 us; in the prologue it delayed every launch by that much).
        for (int i = threadIdx.x - 64; i < ep.hd / 2; i += 32 * kEpiWarps) {
          const double f = pow(ep.rope_theta, -2.0 * i / static_cast<double>(ep.hd)) * 0.15915494309189533577;
          const float hi = static_cast<float>(f);
          s_norm[256 + 2 * i] = hi;
          s_norm[256 + 2 * i + 1] = static_cast<float>(f - static_cast<double>(hi));
        }
        named_bar_sync(1, 32 * kEpiWarps);
      }
    }
    constexpr int E2 = EPI2 < 0 ? EPI : EPI2;
    EpiWarp<nb_of(EPI)> e;
    e.base = epi_smem + ew * C::EPI_WARP_BYTES;
    e.lbar = eload + 2 * ew;
    e.lphase = 0;
    e.cur = 0;
    e.lane = lane;
    const uint32_t tempty_leader0 = CG == 2 ? mapa_shared(smem_u32(&tempty[0]), 0) : smem_u32(&tempty[0]);
    EpiCtx x{tmem_base, tempty_leader0, tfull, tempty, s_norm, rank, q, ch, lane, 0, 0u, 0, 0};
    // job 0's tiles, then (paired launch) job 1's: in every CTA's static schedule all job-0
    // tiles come first, so two loops with concrete epilogue types (no job-generic code)
    int64_t tile = unit;
    for (; tile < nt0; tile += n_units) {
      int64_t m_blk, n0;
      int width;
      decode(j0, tile, m_blk, n0, width);
      epi_job_tile<BN, CG, EPI>(e, x, j0, mp0, EPI2 >= 0 ? dep : nullptr, M, m_blk, n0, width);
    }
    if constexpr (EPI2 >= 0) {
      if (lane == 0) bulk_wait_all();  // the staging ring changes box layout: drain job 0's stores
      __syncwarp();
      EpiWarp<nb_of(E2)> e2;  // job 1's staging ring (same smem, its own box layout)
      e2.base = e.base;
      e2.lbar = e.lbar;
      e2.lphase = 0;
      e2.cur = 0;
      e2.lane = lane;
      for (; tile < num_tiles; tile += n_units) {
        int64_t m_blk, n0;
        int width;
        decode(j1, tile - nt0, m_blk, n0, width);
        epi_job_tile<BN, CG, E2>(e2, x, j1, mp1, nullptr, M, m_blk, n0, width);
      }
    }
    long long st_w = x.st_w, st_b = x.st_b, n_t = x.n_t;
    if (lane == 0) bulk_wait_all();
#ifdef RDX_GEMM_STATS_BUILD
    if (lane == 0) {
      GTIME_MAX(5);
      atomicAdd(&g_gemm_stats[3], static_cast<unsigned long long>(st_w));
      atomicAdd(&g_gemm_stats[4], static_cast<unsigned long long>(st_b));
      atomicAdd(&g_gemm_stats[5], static_cast<unsigned long long>(n_t));
    }
#endif
    (void)st_w;
    (void)st_b;
    (void)n_t;
  }

  tc_fence_before();
  __syncthreads();
  if constexpr (CG == 2) cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    if constexpr (CG == 2) tmem_dealloc_cg2(tmem_base, C::TMEM_COLS);
    else tmem_dealloc(tmem_base, C::TMEM_COLS);
  }
  if (threadIdx.x == 0) GTIME_MAX(6);
}

// ---------------------------------------------------------------- host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

// 2-D row-major map: inner = columns (elements), outer = rows, box = box_inner x box_outer, 128B swizzle.
int make_map(CUtensorMap* map, CUtensorMapDataType dt, int esize, const void* ptr, int64_t inner, int64_t outer,
             int64_t ld_elems, int box_inner, int box_outer,
             CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return RDX_ERR_UNSUPPORTED;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(outer)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld_elems) * esize};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(box_inner), static_cast<cuuint32_t>(box_outer)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, dt, 2, const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? RDX_OK : RDX_ERR_INVALID_ARGUMENT;
}

// 3-D view [blocks][outer][inner] of a row-major matrix whose column blocks of
// `inner` elements are stacked: dims {inner, outer, blocks}, strides {ld, inner}
// (bytes), 128B swizzle; a {inner, box_outer, box_blocks} box lands in smem as
// box_blocks consecutive [box_outer][inner] swizzled boxes.
int make_map_3d(CUtensorMap* map, CUtensorMapDataType dt, int esize, const void* ptr, int64_t inner, int64_t outer,
                int64_t blocks, int64_t ld_elems, int box_inner, int box_outer, int box_blocks) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return RDX_ERR_UNSUPPORTED;
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(outer),
                        static_cast<cuuint64_t>(blocks)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(ld_elems) * esize, static_cast<cuuint64_t>(inner) * esize};
  cuuint32_t box[3] = {static_cast<cuuint32_t>(box_inner), static_cast<cuuint32_t>(box_outer),
                       static_cast<cuuint32_t>(box_blocks)};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, dt, 3, const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? RDX_OK : RDX_ERR_INVALID_ARGUMENT;
}

// RDX_GEMM_GROUP_M (env) / rdx_gemm_debug_group_m: row blocks per raster group (0 = default).
int g_group_m = -1;
int group_m_setting() {
  if (g_group_m == -1) {  // unset: read the environment once
    const char* e = getenv("RDX_GEMM_GROUP_M");
    g_group_m = e ? atoi(e) : 0;
  }
  return g_group_m;
}

// Row blocks per raster group for K >= 8192 (the C4 down projection, K = 12288): a
// 16-row-block group of A is 100 MB there and does not stay L2-resident next to B.
// RDX_GEMM_GROUP_M_BIGK (env) / rdx_gemm_debug_group_m_bigk for A/B runs.
int g_group_m_bigk = -1;
int group_m_bigk_setting() {
  if (g_group_m_bigk == -1) {
    const char* e = getenv("RDX_GEMM_GROUP_M_BIGK");
    g_group_m_bigk = e ? atoi(e) : 16;
    if (g_group_m_bigk <= 0) g_group_m_bigk = 16;
  }
  return g_group_m_bigk;
}

// RDX_GEMM_TAIL_SPLIT=0 (env) or rdx_gemm_debug_tail_split(0) disables the tail split (A/B runs).
int g_tail_split = -1;
bool tail_split_enabled() {
  if (g_tail_split < 0) {
    const char* e = getenv("RDX_GEMM_TAIL_SPLIT");
    g_tail_split = (e && e[0] == '0') ? 0 : 1;
  }
  return g_tail_split == 1;
}

// RDX_GEMM_COLPART=0 (env) or rdx_gemm_debug_colpart(0) disables the column partition (A/B runs).
int g_colpart = -1;
int g_pair = -1;  // RDX_GEMM_PAIR / rdx_gemm_debug_pair
bool pair_enabled() {
  if (g_pair < 0) {
    const char* e = getenv("RDX_GEMM_PAIR");
    g_pair = (e && e[0] == '0') ? 0 : 1;
  }
  return g_pair == 1;
}
int g_last_cp_ncol = 0;  // debug query (rdx_gemm_debug_colpart(-1))
bool colpart_enabled() {
  if (g_colpart < 0) {
    const char* e = getenv("RDX_GEMM_COLPART");
    g_colpart = (e && e[0] == '0') ? 0 : 1;
  }
  return g_colpart == 1;
}

// Column partition for few-round launches (the C2 o_proj / down shape: M = 7024 ->
// 28 pair row blocks x 4 column tiles of 256 = 112 tiles on 74 CTA pairs, 1.51 rounds
// run as 2).  Candidates cut N into ncol column tiles whose widths are multiples of 32
// (<= BN, as equal as possible: `wide` tiles 32 columns wider than the rest) and place
// the wide ones at every bit pattern; each is scored by the makespan of the kernel's
// static round-robin schedule (tile t -> unit t % units, in the kernel's raster order)
// with a per-tile cost of (width + kTileFixed) columns (A is streamed per tile whatever
// its width; kTileFixed fitted to the measured 128- vs 256-wide pair tiles).  Still no
// split-K: each output element is one CTA's full K reduction, same bits.
constexpr int kTileFixed = 100;
struct ColPart {
  int ncol, wide_w, narrow_w;
  uint32_t mask;
};

double sched_makespan(int64_t m_tiles, int ncol, const int* widths, int group_m, int64_t units, int64_t offset = 0,
                      double head = 0.0) {
  double load[1024];
  if (units > 1024) return 1e30;
  // a preceding job of `offset` (mod units) leftover tiles of cost `head` on units [0, offset)
  for (int64_t u = 0; u < units; ++u) load[u] = u < offset ? head : 0.0;
  const int64_t tiles = m_tiles * ncol;
  for (int64_t t = 0; t < tiles; ++t) {
    const int64_t gsz = static_cast<int64_t>(group_m) * ncol;
    const int64_t g = t / gsz, r = t - g * gsz;
    const int64_t g_rows = m_tiles - g * group_m < group_m ? m_tiles - g * group_m : group_m;
    load[(t + offset) % units] += widths[r / g_rows] + kTileFixed;
  }
  double mx = 0.0;
  for (int64_t u = 0; u < units; ++u) mx = load[u] > mx ? load[u] : mx;
  return mx;
}

bool choose_colpart(int64_t m_tiles, int64_t n, int bn, int group_m, int64_t units, int64_t tail_rem,
                    int tail_split, ColPart* out, int64_t offset = 0, double head = 0.0) {
  if (n % 32 || n > 32 * 256) return false;
  const int64_t tiles = m_tiles * ((n + bn - 1) / bn);
  if (tiles > 6 * units || tiles <= units / 2) return false;
  // baseline: bn-wide tiles, the last round possibly split (as the kernel runs it)
  const int n_tiles = static_cast<int>((n + bn - 1) / bn);
  double base;
  {
    int w[64];
    for (int c = 0; c < n_tiles; ++c) w[c] = bn;
    base = sched_makespan(m_tiles, n_tiles, w, group_m, units, offset, head);
    if (tail_split > 1 && tail_rem > 0 && offset == 0) {  // full rounds + the split tail's rounds
      const double full = static_cast<double>(tiles / units) * (bn + kTileFixed);
      const int64_t narrow = tail_split * tail_rem;
      base = full + static_cast<double>((narrow + units - 1) / units) * (bn / tail_split + kTileFixed);
    }
  }
  struct Key {
    int64_t m_tiles, n, units, offset;
    int bn, group_m;
    ColPart cp;
    bool ok;
  };
  static Key cache[16];
  static int cache_n = 0;
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  for (int i = 0; i < cache_n; ++i) {
    const Key& k = cache[i];
    if (k.m_tiles == m_tiles && k.n == n && k.units == units && k.bn == bn && k.group_m == group_m &&
        k.offset == offset) {
      *out = k.cp;
      return k.ok;
    }
  }
  const int boxes = static_cast<int>(n / 32);
  double best = base * 0.97;  // adopt only a predicted gain of >= 3 %
  ColPart bestcp{0, 0, 0, 0};
  for (int ncol = n_tiles; ncol <= n_tiles + 3 && ncol <= 32; ++ncol) {
    const int nar = boxes / ncol, wide = boxes % ncol;
    if (32 * (nar + (wide ? 1 : 0)) > bn || nar < 2) continue;
    // every placement of the wide tiles (ncol <= 8 keeps this at most 70 patterns)
    const uint32_t lim = ncol <= 12 ? (1u << ncol) : 0u;
    for (uint32_t mask = 0; mask < lim; ++mask) {
      if (__builtin_popcount(mask) != wide) continue;
      int w[32];
      for (int c = 0; c < ncol; ++c) w[c] = 32 * (nar + ((mask >> c) & 1u));
      const double ms = sched_makespan(m_tiles, ncol, w, group_m, units, offset, head);
      if (ms < best - 1e-9) {
        best = ms;
        bestcp = ColPart{ncol, 32 * (nar + 1), 32 * nar, mask};
      }
    }
  }
  const bool ok = bestcp.ncol > 0;
  Key k{m_tiles, n, units, offset, bn, group_m, bestcp, ok};
  if (cache_n < 16) cache[cache_n++] = k;
  else cache[(m_tiles + n) & 15] = k;
  *out = bestcp;
  return ok;
}

// Tensor maps, epilogue parameters and static schedule (raster, tail split or column
// partition) of one GEMM; *grid_units = CTA units (pairs when CG = 2) it wants.
// pair_role: 0 = a stand-alone launch; 1 = job 0 of a pair (row-block-major raster so its
// early row blocks finish first, no tail split: job 1's tiles fill its last round);
// 2 = job 1 of a pair, whose tiles continue job 0's round-robin from unit `offset`.
template <int BN, int EPI, int CG>
int prepare_job(const rdx_gemm_args& a, JobMaps* maps, JobArgs* job, int64_t* grid_units, int pair_role = 0,
                int64_t offset = 0) {
  using C = Cfg<BN, CG, EPI>;
  std::memset(maps, 0, sizeof(*maps));
  CUtensorMap &ma = maps->a, &mb = maps->b, &mb2 = maps->b2, &mb4 = maps->b4, &mc = maps->c, &md = maps->d;
  int st = make_map(&ma, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, a.a, a.k, a.m, a.lda, BK, BM);
  if (st) return st;
  st = make_map(&mb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, a.b, a.k, a.n, a.ldb, BK, C::B_ROWS);
  if (st) return st;
  st = make_map(&mb2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, a.b, a.k, a.n, a.ldb, BK, C::B_ROWS / 2);
  if (st) return st;
  st = make_map(&mb4, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, a.b, a.k, a.n, a.ldb, BK, C::B_ROWS / 4);
  if (st) return st;
  if (EPI == RDX_EPI_RESID_NORM) {
    // [col blocks of 32][rows][32 cols] view: a box of {32, 32, 2} = two stacked swizzled 32x32 boxes
    st = make_map_3d(&mc, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, a.out, 32, a.m, a.n / 32, a.ldo, 32, 32, 2);
  } else if (EPI == RDX_EPI_STORE_F32 || EPI == RDX_EPI_RESID_F32) {
    st = make_map(&mc, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, a.out, a.n, a.m, a.ldo, 32, 32);
  } else {
    const int64_t ncols = EPI == RDX_EPI_SWIGLU ? a.n / 2 : a.n;
    st = make_map(&mc, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, a.out, ncols, a.m, a.ldo, 32, 32,
                  CU_TENSOR_MAP_SWIZZLE_64B);
  }
  if (st) return st;
  if (EPI == RDX_EPI_RESID_NORM) {
    st = make_map(&md, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, a.out_bf16, a.n, a.m, a.ldo_bf16, 64, 32);
    if (st) return st;
  }
  EpiParams& ep = job->ep;
  std::memset(&ep, 0, sizeof(ep));
  ep.qn = a.q_norm_w;
  ep.kn = a.k_norm_w;
  ep.rope = reinterpret_cast<const float2*>(a.rope_table);
  ep.rope_ps = a.rope_blocked ? 32 : 1;
  ep.rope_pos = a.rope_pos;
  ep.rope_theta = a.rope_theta;
  ep.hd = a.head_dim;
  ep.q_dim = a.q_heads * a.head_dim;
  ep.kv_dim = a.kv_heads * a.head_dim;
  ep.eps = a.eps;
  ep.row_ss = a.row_ss;
  ep.ss_parts = a.ss_parts;
  ep.inv_norm_dim = a.norm_dim > 0 ? 1.f / static_cast<float>(a.norm_dim) : 0.f;
  ep.norm_eps = a.norm_eps;
  ep.h = static_cast<float*>(a.out);
  ep.ldh = a.ldo;
  ep.hb = static_cast<__nv_bfloat16*>(a.out_bf16);
  ep.ldhb = a.ldo_bf16;
  ep.ss_out = a.ss_out;
  ep.ss_out_parts = static_cast<int>(a.n / kNormGroup);
  ep.done_ctr = EPI == RDX_EPI_RESID_F32 ? a.done_ctr : nullptr;
  ep.a_ready = a.a_ready;
  ep.a_ready_use = a.a_ready_use;
  {
    const int64_t m_tiles = (a.m + BM * CG - 1) / (BM * CG);
    // Default raster: with many row blocks (C3/C4 scale: A = M x K no longer fits L2)
    // groups of 16 row blocks keep each group's A rows L2-resident while the group
    // walks the column blocks, so A is read from HBM once and B m_tiles/16 times
    // (measured: C3 step +10.5 %, C4 +13 % over column-block-major; 8, 24, 32 and a
    // K-scaled group size (A rows of a group ~48 MB) were equal or slower).  Few row blocks (C2): the legacy orders (row-block-major when a
    // completion counter is attached).
    int gm = group_m_setting();
    if (gm <= 0) gm = m_tiles >= 64 ? (a.k >= 8192 ? group_m_bigk_setting() : 16)
                                     : ((ep.done_ctr || ep.a_ready || pair_role == 1) ? 1 : static_cast<int>(m_tiles));
    ep.group_m = static_cast<int>(gm < m_tiles ? gm : m_tiles);
  }
  const int64_t tiles = ((a.m + BM * CG - 1) / (BM * CG)) * ((a.n + BN - 1) / BN);
  const int64_t units_max = num_sms() / CG;
  const int64_t units = tiles < units_max ? tiles : units_max;
  // tail split (see gemm_kernel): pick the factor s in {1, 2} that minimises the
  // last round's length ceil(s*rem/units)/s, subject to each narrow tile keeping
  // whole epilogue units per warp (64-column SwiGLU pairs, whole heads, 64-column
  // norm groups, 32-column boxes)
  const int64_t rem = tiles % units;
  int split = 1;
  if (BN == 256 && rem > 0 && tail_split_enabled() && pair_role == 0) {
    double best = 1.0;
    for (int sf : {2}) {  // quarters measured slower: a narrow tile still streams the full A tile
      const int w = BN / sf;
      bool ok = (w / 2) % 32 == 0;
      if (EPI == RDX_EPI_SWIGLU) ok = ok && w % (2 * kSwigluUnit) == 0;
      // QKV: each warp needs whole heads; a tile of one head width goes to the ch = 0 warps
      if (EPI == RDX_EPI_QKV) ok = ok && a.head_dim > 0 && ((w / 2) % a.head_dim == 0 || (a.head_dim > 32 && w % a.head_dim == 0));
      if (EPI == RDX_EPI_RESID_NORM) ok = ok && (w / 2) % kNormGroup == 0;
      const double len = static_cast<double>((sf * rem + units - 1) / units) / sf;
      if (ok && len < best - 1e-9) {
        best = len;
        split = sf;
      }
    }
  }
  int64_t tail_start = split > 1 ? tiles - rem : tiles;
  ep.cp_ncol = ep.cp_wide = ep.cp_narrow = 0;
  ep.cp_mask = 0;
  if constexpr (EPI == RDX_EPI_RESID_F32 || EPI == RDX_EPI_STORE_BF16 || EPI == RDX_EPI_STORE_F32) {
    ColPart cp;
    const int64_t m_tiles = (a.m + BM * CG - 1) / (BM * CG);
    if (colpart_enabled() && choose_colpart(m_tiles, a.n, BN, ep.group_m, units_max, rem, split, &cp,
                                            pair_role == 2 ? offset % units_max : 0,
                                            pair_role == 2 ? static_cast<double>(BN + kTileFixed) : 0.0)) {
      ep.cp_ncol = cp.ncol;
      ep.cp_wide = cp.wide_w;
      ep.cp_narrow = cp.narrow_w;
      ep.cp_mask = cp.mask;
      split = 1;
      tail_start = m_tiles * cp.ncol;
      // B boxes of the two widths (per CTA: width / CG rows) in the tmB2 / tmB4 slots
      int st2 = make_map(&mb2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, a.b, a.k, a.n, a.ldb, BK, cp.wide_w / CG);
      if (st2) return st2;
      st2 = make_map(&mb4, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, a.b, a.k, a.n, a.ldb, BK, cp.narrow_w / CG);
      if (st2) return st2;
    }
  }
  *grid_units = ep.cp_ncol > 0 ? units_max : units;
  g_last_cp_ncol = ep.cp_ncol;
  job->N = a.n;
  job->K = a.k;
  job->tail_start = tail_start;
  job->split = split;
  return RDX_OK;
}

template <int BN, int EPI, int CG, int EPI2>
int launch_jobs(const JobMaps& mp0, const JobMaps& mp1, int64_t m, const JobArgs& j0, const JobArgs& j1,
                uint32_t* dep, uint32_t dep_cols, int64_t grid_units, cudaStream_t stream) {
  using C = Cfg<BN, CG, EPI>;
  auto kern = gemm_kernel<BN, EPI, CG, EPI2>;
  static bool attr_set = false;
  if (!attr_set) {
    RDX_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    if (CG == 2) RDX_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 0));
    attr_set = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(grid_units * CG));  // persistent: at most one CTA per SM
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = (pdl_enabled() || j0.ep.a_ready) ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  RDX_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, mp0, mp1, m, j0, j1, dep, dep_cols));
  return RDX_OK;
}

template <int BN, int EPI, int CG>
int launch(const rdx_gemm_args& a, cudaStream_t stream) {
  JobMaps mp0, mp1;
  JobArgs j0, j1;
  int64_t units = 0;
  if (int st = prepare_job<BN, EPI, CG>(a, &mp0, &j0, &units)) return st;
  std::memset(&mp1, 0, sizeof(mp1));
  std::memset(&j1, 0, sizeof(j1));
  return launch_jobs<BN, EPI, CG, -1>(mp0, mp1, a.m, j0, j1, nullptr, 0, units, stream);
}

template <int EPI>
int dispatch(const rdx_gemm_args& a, int bn, int cg, cudaStream_t s) {
  if (cg == 2) return bn == 256 ? launch<256, EPI, 2>(a, s) : launch<128, EPI, 2>(a, s);
  if constexpr (EPI == RDX_EPI_RESID_NORM) {
    return launch<128, EPI, 1>(a, s);  // the 1-CTA 256-wide tile leaves too few stages next to its staging boxes
  } else {
    return bn == 256 ? launch<256, EPI, 1>(a, s) : launch<128, EPI, 1>(a, s);
  }
}

template <int BN, int CG>
int launch_mlp_pair(const rdx_gemm_args& g, const rdx_gemm_args& d, uint32_t* dep, cudaStream_t stream) {
  JobMaps mp0, mp1;
  JobArgs j0, j1;
  int64_t u0 = 0, u1 = 0;
  if (int st = prepare_job<BN, RDX_EPI_SWIGLU, CG>(g, &mp0, &j0, &u0, 1)) return st;
  const int64_t nt0 = j0.tail_start + j0.split * (((g.m + BM * CG - 1) / (BM * CG)) *
                                                  (j0.ep.cp_ncol > 0 ? j0.ep.cp_ncol : (g.n + BN - 1) / BN) -
                                                  j0.tail_start);
  if (int st = prepare_job<BN, RDX_EPI_RESID_F32, CG>(d, &mp1, &j1, &u1, 2, nt0)) return st;
  const int64_t units_max = num_sms() / CG;
  int64_t units = u0 > u1 ? u0 : u1;
  units = units < units_max ? units : units_max;
  return launch_jobs<BN, RDX_EPI_SWIGLU, CG, RDX_EPI_RESID_F32>(mp0, mp1, g.m, j0, j1, dep,
                                                                  static_cast<uint32_t>(g.n / 2), units, stream);
}

// Pick (CG, BN) minimising tile rounds x per-tile cost.  A 1-CTA tile streams
// a third more operand bytes per FLOP than the pair tile, hence the penalty.
// RDX_GEMM_SHAPE="cg,bn" (env) pins the choice for experiments.
int g_forced_cg = -1, g_forced_bn = -1;  // RDX_GEMM_SHAPE / rdx_gemm_debug_shape

void choose_shape(const rdx_gemm_args& a, int* bn_out, int* cg_out) {
  int& forced_cg = g_forced_cg;
  int& forced_bn = g_forced_bn;
  if (forced_cg < 0) {
    forced_cg = 0;
    if (const char* e = getenv("RDX_GEMM_SHAPE")) {
      int c = 0, n = 0;
      if (sscanf(e, "%d,%d", &c, &n) == 2 && (c == 1 || c == 2) && (n == 128 || n == 256)) {
        forced_cg = c;
        forced_bn = n;
      }
    }
  }
  int best_bn = 256, best_cg = a.m > BM ? 2 : 1;
  double best_cost = 1e30;
  for (int cg : {2, 1}) {
    if (cg == 2 && a.m <= BM) continue;
    for (int bn : {256, 128}) {
      if (a.block_n && bn != a.block_n) continue;
      if (a.epi == RDX_EPI_QKV && ((bn / 2) % a.head_dim) && a.head_dim > 32) continue;
      const int64_t tiles = ((a.m + BM * cg - 1) / (BM * cg)) * ((a.n + bn - 1) / bn);
      const int64_t units = num_sms() / cg;
      // a partial last round costs about a quarter of a full one per missing tile
      // (measured: the few busy SMs clock up under the power cap), so rounds are
      // counted fractionally plus a 0.25 penalty on the idle share
      const double frac = static_cast<double>(tiles) / static_cast<double>(units);
      const double rounds = frac + 0.25 * (static_cast<double>((tiles + units - 1) / units) - frac);
      const double cost = rounds * (bn + 64) * (cg == 1 ? 1.15 : 1.0);
      if (cost < best_cost) {
        best_cost = cost;
        best_bn = bn;
        best_cg = cg;
      }
    }
  }
  if (forced_cg > 0 && (forced_cg == 1 || a.m > BM)) {
    const bool ok = !(a.epi == RDX_EPI_QKV && ((forced_bn / 2) % a.head_dim) && a.head_dim > 32);
    if (ok && (!a.block_n || a.block_n == forced_bn)) {
      best_cg = forced_cg;
      best_bn = forced_bn;
    }
  }
  *bn_out = best_bn;
  *cg_out = best_cg;
}

}  // namespace gemm
}  // namespace rdx

extern "C" int rdx_gemm(const rdx_gemm_args* args, void* stream) {
  using namespace rdx;
  using namespace rdx::gemm;
  if (!args) return RDX_ERR_INVALID_ARGUMENT;
  const rdx_gemm_args& a = *args;
  if (a.m < 0 || a.n <= 0 || a.k <= 0) return RDX_ERR_SHAPE_MISMATCH;
  if (a.m == 0) return RDX_OK;
  if ((a.k % 8) || (a.lda % 8) || (a.ldb % 8) || a.lda < a.k || a.ldb < a.k) return RDX_ERR_SHAPE_MISMATCH;
  if (a.m >= (int64_t(1) << 31) || a.n >= (int64_t(1) << 31)) return RDX_ERR_CAPACITY_EXCEEDED;
  if (!a.a || !a.b || !a.out) return RDX_ERR_INVALID_ARGUMENT;
  if ((reinterpret_cast<uintptr_t>(a.a) | reinterpret_cast<uintptr_t>(a.b) | reinterpret_cast<uintptr_t>(a.out)) &
      15)
    return RDX_ERR_INVALID_ARGUMENT;
  if (a.block_n != 0 && a.block_n != 128 && a.block_n != 256) return RDX_ERR_INVALID_ARGUMENT;
  int bn = 256, cg = 1;
  if (a.epi == RDX_EPI_QKV && (a.head_dim <= 0 || a.head_dim % 16 || a.head_dim > 128))
    return RDX_ERR_SHAPE_MISMATCH;
  if (a.row_ss && (a.ss_parts <= 0 || a.norm_dim <= 0)) return RDX_ERR_INVALID_ARGUMENT;
  // slab completion counters exist only on the residual reduce-add epilogue
  if (a.done_ctr && a.epi != RDX_EPI_RESID_F32) return RDX_ERR_INVALID_ARGUMENT;
  choose_shape(a, &bn, &cg);
  cudaStream_t s = as_stream(stream);
  switch (a.epi) {
    case RDX_EPI_STORE_BF16:
      if (a.ldo % 8 || a.ldo < a.n) return RDX_ERR_SHAPE_MISMATCH;
      return dispatch<RDX_EPI_STORE_BF16>(a, bn, cg, s);
    case RDX_EPI_STORE_F32:
      if (a.ldo % 4 || a.ldo < a.n) return RDX_ERR_SHAPE_MISMATCH;
      return dispatch<RDX_EPI_STORE_F32>(a, bn, cg, s);
    case RDX_EPI_RESID_F32:
      if (a.ldo % 4 || a.ldo < a.n) return RDX_ERR_SHAPE_MISMATCH;
      return dispatch<RDX_EPI_RESID_F32>(a, bn, cg, s);
    case RDX_EPI_RESID_NORM:
      if (a.n % kNormGroup || a.ldo % 4 || a.ldo < a.n || a.ldo_bf16 % 8 || a.ldo_bf16 < a.n) return RDX_ERR_SHAPE_MISMATCH;
      if (!a.out_bf16 || !a.ss_out || (reinterpret_cast<uintptr_t>(a.out_bf16) & 15)) return RDX_ERR_INVALID_ARGUMENT;
      return dispatch<RDX_EPI_RESID_NORM>(a, bn, cg, s);
    case RDX_EPI_SWIGLU:
      if (a.n % (2 * kSwigluUnit) || a.ldo % 8 || a.ldo < a.n / 2) return RDX_ERR_SHAPE_MISMATCH;
      return dispatch<RDX_EPI_SWIGLU>(a, bn, cg, s);
    case RDX_EPI_QKV: {
      if (a.head_dim > 32 && (bn / 2) % a.head_dim) return RDX_ERR_SHAPE_MISMATCH;
      if (a.n != static_cast<int64_t>(a.q_heads + 2 * a.kv_heads) * a.head_dim) return RDX_ERR_SHAPE_MISMATCH;
      if (!a.q_norm_w || !a.k_norm_w) return RDX_ERR_INVALID_ARGUMENT;
      if (a.rope_pos) {
        if ((a.head_dim != 64 && a.head_dim != 128) || !(a.rope_theta > 0.0)) return RDX_ERR_INVALID_ARGUMENT;
      } else if (!a.rope_table) {
        return RDX_ERR_INVALID_ARGUMENT;
      }
      if (a.ldo % 8 || a.ldo < a.n) return RDX_ERR_SHAPE_MISMATCH;
      return dispatch<RDX_EPI_QKV>(a, bn, cg, s);
    }
    default:
      return RDX_ERR_INVALID_ARGUMENT;
  }
}

// Checks of rdx_gemm shared by rdx_gemm_pair (RDX_OK or the status rdx_gemm returns).
namespace rdx {
namespace gemm {
int validate_common(const rdx_gemm_args& a) {
  if (a.m < 0 || a.n <= 0 || a.k <= 0) return RDX_ERR_SHAPE_MISMATCH;
  if ((a.k % 8) || (a.lda % 8) || (a.ldb % 8) || a.lda < a.k || a.ldb < a.k) return RDX_ERR_SHAPE_MISMATCH;
  if (a.m >= (int64_t(1) << 31) || a.n >= (int64_t(1) << 31)) return RDX_ERR_CAPACITY_EXCEEDED;
  if (!a.a || !a.b || !a.out) return RDX_ERR_INVALID_ARGUMENT;
  if ((reinterpret_cast<uintptr_t>(a.a) | reinterpret_cast<uintptr_t>(a.b) | reinterpret_cast<uintptr_t>(a.out)) & 15)
    return RDX_ERR_INVALID_ARGUMENT;
  if (a.block_n != 0 && a.block_n != 128 && a.block_n != 256) return RDX_ERR_INVALID_ARGUMENT;
  if (a.row_ss && (a.ss_parts <= 0 || a.norm_dim <= 0)) return RDX_ERR_INVALID_ARGUMENT;
  if (a.done_ctr && a.epi != RDX_EPI_RESID_F32) return RDX_ERR_INVALID_ARGUMENT;
  return RDX_OK;
}
}  // namespace gemm
}  // namespace rdx

extern "C" int rdx_gemm_pair(const rdx_gemm_args* first, const rdx_gemm_args* second, uint32_t* dep_ctr,
                             void* stream) {
  using namespace rdx;
  using namespace rdx::gemm;
  if (!first || !second) return RDX_ERR_INVALID_ARGUMENT;
  const rdx_gemm_args &g = *first, &d = *second;
  if (int st = validate_common(g)) return st;
  if (int st = validate_common(d)) return st;
  if (g.epi != RDX_EPI_SWIGLU || d.epi != RDX_EPI_RESID_F32) return RDX_ERR_UNSUPPORTED;
  if (g.m != d.m || d.a != g.out || d.lda != g.ldo || d.k != g.n / 2 || d.a_ready) return RDX_ERR_SHAPE_MISMATCH;
  if (g.n % (2 * kSwigluUnit) || g.ldo % 8 || g.ldo < g.n / 2) return RDX_ERR_SHAPE_MISMATCH;
  if (d.ldo % 4 || d.ldo < d.n) return RDX_ERR_SHAPE_MISMATCH;
  if (!dep_ctr) return RDX_ERR_INVALID_ARGUMENT;
  if (g.m == 0) return RDX_OK;
  int bn0 = 256, cg0 = 1, bn1 = 256, cg1 = 1;
  choose_shape(g, &bn0, &cg0);
  choose_shape(d, &bn1, &cg1);
  cudaStream_t s = as_stream(stream);
  // One launch pays off when the MLP is a few rounds of tiles (C2: +3.9 % per step); at C3/C4
  // scale (>= 64 pair row blocks, grouped raster) a launch boundary is noise and measured
  // neutral / -2 %, so those shapes (and pairs that want different tile shapes) run as two
  // stream-ordered launches (dep_ctr unused).
  const bool few_rounds = (g.m + 2 * BM - 1) / (2 * BM) < 64;
  if (!pair_enabled() || !few_rounds || bn0 != bn1 || cg0 != cg1 || bn0 != 256 || cg0 != 2) {
    if (int st = rdx_gemm(first, stream)) return st;
    return rdx_gemm(second, stream);
  }
  return launch_mlp_pair<256, 2>(g, d, dep_ctr, s);
}

// RDX_GEMM_PAIR=0 (env) or rdx_gemm_debug_pair(0): rdx_gemm_pair runs two launches (A/B).
extern "C" int rdx_gemm_debug_pair(int on) {
  const int prev = rdx::gemm::pair_enabled() ? 1 : 0;
  rdx::gemm::g_pair = on ? 1 : 0;
  return prev;
}

// Debug: switch the GEMM tail split on (1) / off (0); returns the previous setting.
extern "C" int rdx_gemm_debug_stats(unsigned long long* out8, int reset) {
#ifdef RDX_GEMM_STATS_BUILD
  // reset >= 2: out8 receives the %globaltimer landmarks (g_gemm_times) instead
  if (out8 && cudaMemcpyFromSymbol(out8, reset >= 2 ? rdx::gemm::g_gemm_times : rdx::gemm::g_gemm_stats,
                                   sizeof(unsigned long long) * 8) != cudaSuccess)
    return RDX_ERR_CUDA;
  if (reset) {
    const unsigned long long z[8] = {};
    unsigned long long zt[8] = {};
    zt[0] = zt[3] = ~0ULL;  // min slots
    if (cudaMemcpyToSymbol(rdx::gemm::g_gemm_stats, z, sizeof(z)) != cudaSuccess) return RDX_ERR_CUDA;
    if (cudaMemcpyToSymbol(rdx::gemm::g_gemm_times, zt, sizeof(zt)) != cudaSuccess) return RDX_ERR_CUDA;
  }
  return RDX_OK;
#else
  (void)out8;
  (void)reset;
  return RDX_ERR_UNSUPPORTED;
#endif
}

extern "C" int rdx_gemm_debug_group_m(int group_m) {
  const int prev = rdx::gemm::group_m_setting();
  rdx::gemm::g_group_m = group_m < 0 ? 0 : group_m;
  return prev;
}

extern "C" int rdx_gemm_debug_group_m_bigk(int group_m) {
  const int prev = rdx::gemm::group_m_bigk_setting();
  rdx::gemm::g_group_m_bigk = group_m <= 0 ? 16 : group_m;
  return prev;
}

extern "C" int rdx_gemm_debug_shape(int cg, int block_n) {
  using namespace rdx::gemm;
  if (cg == 0) {
    g_forced_cg = 0;  // automatic choice
    return RDX_OK;
  }
  if ((cg != 1 && cg != 2) || (block_n != 128 && block_n != 256)) return RDX_ERR_INVALID_ARGUMENT;
  g_forced_cg = cg;
  g_forced_bn = block_n;
  return RDX_OK;
}

extern "C" int rdx_gemm_debug_colpart(int on) {
  if (on < 0) return rdx::gemm::g_last_cp_ncol;  // query: column tiles of the last launch (0 = no partition)
  const int prev = rdx::gemm::colpart_enabled() ? 1 : 0;
  rdx::gemm::g_colpart = on ? 1 : 0;
  return prev;
}

extern "C" int rdx_gemm_debug_tail_split(int on) {
  const int prev = rdx::gemm::tail_split_enabled() ? 1 : 0;
  rdx::gemm::g_tail_split = on ? 1 : 0;
  return prev;
}

int rdx::take_device_status_gemm(int* out, cudaStream_t st) { return take_device_status(out, st); }
