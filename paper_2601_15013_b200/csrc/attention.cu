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
// Tiling.  A query tile is 128 rows = (GQA group heads) x (128 / group
// queries) of one (sequence, kv head), so one S MMA serves the whole group
// against one K tile.  A work unit is a PAIR of consecutive query tiles
// (h = 0, 1) of one (sequence, kv head); both stream the same 128-key K/V
// tiles, which are loaded once.  Units are walked longest-first by
// persistent CTAs (one per SM) in one continuous pipeline across units.
//
// TMEM (512 columns): S_h at [128h, 128h+128) fp32, with P_h (bf16 pairs)
// written back over its first 64 columns; O_h at [256+128h, ...).  The P V
// product reads P straight from TMEM (tcgen05.mma A-from-TMEM), so P never
// touches shared memory.  The MMA issue order per key tile j is
//     PV_0(j)  S_0(j+1)  PV_1(j)  S_1(j+1)
// so the tensor pipe works on one tile while the other tile's softmax runs.
// Softmax keeps a stale running max unless the tile max exceeds it by more
// than 2^8 (exact: the final O / l uses the same max), so O is rescaled in
// TMEM only on the rare large jumps.
//
// Loads.  One loader warp.  Q tiles: one TMA box per (group head, 64-column
// half).  K/V tiles: a 128-key tile whose compact rows form one contiguous
// run (always in plain layout and for long shared prefixes) is one TMA box
// per half; otherwise each 16-key group that is a contiguous run is one
// 16-row box and the other groups use TMA gather4 (4 arbitrary rows per
// instruction).  Head dims that are not a multiple of 64 fall back to
// cp.async 16-byte copies.  Short units (few key tiles) double-buffer Q so
// the next unit's Q streams in while the current one computes.
//
// 16 warps (setmaxnreg re-balances registers toward the softmax groups):
//   warps 0-3    softmax of query tile 0 (row t = TMEM lane t)
//   warps 4-7    softmax of query tile 1
//   warp  8      loader
//   warps 9-12   epilogue: O_h / l -> bf16 compact rows (TMEM lane quarters 1,2,3,0)
//   warp  13     TMEM allocator + MMA issuer (warp-uniform, elect.sync issue)
//   warps 14-15  idle (complete the warpgroup for setmaxnreg)
#include <cstdlib>
#include <cstring>

#include "common.cuh"

namespace rdx {
namespace attn {

constexpr int BQ = 128;        // rows per query tile (group heads x queries)
constexpr int BK = 128;        // keys per K/V tile
constexpr int kThreads = 512;  // 16 warps
constexpr int kLoaderWarp = 8, kMmaWarp = 13;
constexpr uint32_t TMEM_COLS = 512;
constexpr uint32_t O_COL = 256;
constexpr float kRescaleThreshold = 8.0f;  // log2 units: rescale O only when the max grows by > 2^8
#ifndef RDX_ATTN_EMU
#define RDX_ATTN_EMU 0x00u
#endif
constexpr uint32_t kEmulated = RDX_ATTN_EMU;  // pairs (mod 8) whose exp2 runs on the FMA pipe (bitmask)
constexpr int kShortUnitTiles = 4;         // <= this many key tiles per unit: double-buffered Q
constexpr int kRing = 8;                   // unit descriptors the scheduler warp runs ahead
constexpr int kUnitWords = 12;             // ints per ring entry (Unit + its index)
constexpr int kSchedWarp = 14;             // walks this CTA's units and publishes the valid ones
constexpr int kUnitConsumers = 14;         // warps that read each entry: softmax 8, loader, epilogue 4, MMA

// NQB = Q buffers per query tile, NSLOT = K/V ring slots (K and V tiles alternate).
template <int HDP, int NQB, int NSLOT, int BKT = BK>
struct Tile {
  static constexpr int HALVES = HDP / 64;
  static constexpr int CH = HDP / 8;               // 16-byte chunks per row
  static constexpr int Q_BYTES = BQ * HDP * 2;     // HALVES x 128 rows x 128 B
  static constexpr int T_BYTES = BKT * HDP * 2;    // one K or V tile
  static constexpr int T_OFF = 2 * NQB * Q_BYTES;
  static constexpr int L_OFF = T_OFF + NSLOT * T_BYTES;  // fp32 [2 h][2 slots][128] row sums
  static constexpr int BAR_OFF = L_OFF + 2 * 2 * BQ * 4;
  static constexpr int RING_OFF = BAR_OFF + 512;               // unit ring (scheduler warp -> roles)
  static constexpr int SMEM = RING_OFF + kRing * kUnitWords * 4 + 2 * kRing * 8;
  static_assert(SMEM <= 232448, "shared memory budget");
  static constexpr uint32_t IDESC_S = umma_idesc_bf16(BQ, BKT);
  static constexpr uint32_t IDESC_S_HALF = umma_idesc_bf16(BQ, BKT / 2);  // a short last key tile
  static constexpr uint32_t IDESC_PV = umma_idesc_bf16(BQ, HDP) | (1u << 16);  // B (V) MN-major
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

// Warp-collective tcgen05 issue (every lane runs the asm with warp-uniform
// operands; elect.sync picks the issuing lane, always the same one, so the
// commits track that lane's MMAs).
__device__ __forceinline__ void umma_ss_elect(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                              uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred e, p;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// D[tmem] (+)= A[tmem] * B[smem]: A = P in TMEM, bf16 pairs per 32-bit column.
__device__ __forceinline__ void umma_ts_elect(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                              uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred e, p;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void commit_elect(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar))
      : "memory");
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
__device__ __forceinline__ void tmem_st16u(uint32_t taddr, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
      "%14, %15, %16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
      "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
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
template <uint32_t N>
__device__ __forceinline__ void setmaxnreg_inc() {
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(N));
}
template <uint32_t N>
__device__ __forceinline__ void setmaxnreg_dec() {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(N));
}
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Packed fp32 pairs (FFMA2 / FADD2 on sm_100).
__device__ __forceinline__ uint64_t f2pack(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void f2unpack(uint64_t r, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

// 2^x for a pair on the FMA pipe: x = j + f with j = rint(x), f in [-1/2, 1/2];
// 2^f by a degree-3 fit (max relative error 7.7e-5, far below bf16's 2^-9),
// 2^j added to the exponent field.  x is clamped at -126 (result ~1e-38, i.e.
// zero at bf16 weight precision; -126 keeps the biased exponent >= 0 for
// 2^f < 1); inputs are <= 8 (lazy max).
__device__ __forceinline__ uint64_t exp2_poly2(uint64_t x) {
  float x0, x1;
  f2unpack(x, x0, x1);
  const uint64_t xc = f2pack(fmaxf(x0, -126.f), fmaxf(x1, -126.f));
  const uint64_t t = fadd2(xc, f2pack(12582912.f, 12582912.f));  // 1.5 * 2^23: rint into the low bits
  const uint64_t j = fadd2(t, f2pack(-12582912.f, -12582912.f));
  const uint64_t f = ffma2(j, f2pack(-1.f, -1.f), xc);
  uint64_t p = ffma2(f2pack(0.05508868f, 0.05508868f), f, f2pack(0.24260405f, 0.24260405f));
  p = ffma2(p, f, f2pack(0.69327623f, 0.69327623f));
  p = ffma2(p, f, f2pack(0.99992895f, 0.99992895f));
  float p0, p1, t0, t1;
  f2unpack(p, p0, p1);
  f2unpack(t, t0, t1);
  const uint32_t r0 = __float_as_uint(p0) + (__float_as_uint(t0) << 23);
  const uint32_t r1 = __float_as_uint(p1) + (__float_as_uint(t1) << 23);
  return f2pack(__uint_as_float(r0), __uint_as_float(r1));
}

// TMA gather4: rows r0..r3 (64 columns each, box {64, 1}) -> 4 consecutive 128-byte smem rows.
__device__ __forceinline__ void tma_gather4(const CUtensorMap* map, uint32_t dst, uint64_t* bar, int32_t col,
                                            int32_t r0, int32_t r1, int32_t r2, int32_t r3) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
      : "memory");
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
  int group, qpt;            // heads / kv_heads, queries per tile (BQ / group)
  int max_pairs;             // query-tile pairs of the longest query range
  int n_units;               // max_pairs * nseq * kv_heads
  int use_tma;               // head_dim % 64 == 0: whole 128-byte column boxes, TMA tile loads
  int bk;                    // keys per K/V tile of the launched variant (64 or 128)
  int split_tail;            // deal a short last round as single-query-tile half units
  float scale_log2;          // softmax scale * log2(e)
  unsigned long long* stats; // debug (RDX_ATTN_STATS_BUILD + RDX_ATTN_STATS=1): summed clocks per role
  uint32_t* trace;           // debug: event log of CTA trace_cta [count, (clock, code) x 4096]
  int trace_cta;             // debug: which CTA the event log follows (RDX_ATTN_TRACE_CTA, default 0)
  unsigned long long* cta_times;  // debug: per CTA [start, end, units] (globaltimer ns)
};

// Stats slots (summed over CTAs): see rdx_attention_debug_stats.
enum { ST_MMA_TFULL, ST_MMA_PFULL, ST_MMA_QFULL, ST_MMA_OFREE, ST_MMA_TOTAL, ST_SM_SFULL, ST_SM_TOTAL,
       ST_EPI_WAIT, ST_LD_FREE, ST_LD_TOTAL, ST_SM_RESCALE, ST_MMA_ISSUE, ST_EPI_TOTAL, ST_SM_EXP, ST_N };
#ifndef RDX_ATTN_STATS_BUILD
#define RDX_ATTN_STATS_BUILD 0  // 1: per-role clock counters (debug builds only)
#endif
#define RDX_STATS_ON (RDX_ATTN_STATS_BUILD && a.stats)
#define RDX_TWAIT(bar, par, acc)       \
  do {                                 \
    if (RDX_STATS_ON) {                \
      const long long _t0 = clock64(); \
      mbar_wait(bar, par);             \
      acc += clock64() - _t0;          \
    } else {                           \
      mbar_wait(bar, par);             \
    }                                  \
  } while (0)

// Debug event log of CTA 0 (stats builds): code = role << 12 | event << 8 | payload.
// Events go to a per-thread local buffer (no atomics on the timed path) and
// are flushed to a.trace when the role finishes.
struct EvLog {
  uint32_t tm[96], code[96];
  int n;
};
#define RDX_EV(role, ev, payload)                                                    \
  do {                                                                               \
    if (RDX_STATS_ON && a.trace && blockIdx.x == a.trace_cta && evl.n < 96) {        \
      evl.tm[evl.n] = static_cast<uint32_t>(clock64());                              \
      evl.code[evl.n] = ((role) << 12) | ((ev) << 8) | ((payload) & 0xFF);           \
      ++evl.n;                                                                       \
    }                                                                                \
  } while (0)
#define RDX_EV_FLUSH()                                                               \
  do {                                                                               \
    if (RDX_STATS_ON && a.trace && blockIdx.x == a.trace_cta && evl.n > 0) {         \
      const uint32_t _b = atomicAdd(a.trace, static_cast<uint32_t>(evl.n));          \
      for (int _i = 0; _i < evl.n; ++_i)                                             \
        if (_b + _i < 4096) {                                                        \
          a.trace[2 + 2 * (_b + _i)] = evl.tm[_i];                                   \
          a.trace[3 + 2 * (_b + _i)] = evl.code[_i];                                 \
        }                                                                            \
    }                                                                                \
  } while (0)

// 16-byte chunk c of a head row -> swizzled smem offset in a
// [halves][rows][128 B] tile (half stride = rows * 128).
__device__ __forceinline__ uint32_t sw_off(int row, int c, int rows) {
  const int half = c >> 3, cc = c & 7;
  return half * rows * 128 + row * 128 + ((cc ^ (row & 7)) << 4);
}

// Unit geometry (identical in every role).  Units are ordered pair-index
// descending so the longest key ranges are scheduled first.
struct Unit {
  int s, g, k0, L, q0, qlen, lcp, mb0;
  int nkt0, nkt1;  // key tiles of query tile h (0 = tile absent)
};

__device__ __forceinline__ void unit_geometry(const Args& a, int u, int k0, int k1, int q0, int q1, Unit& it) {
  const int per = a.nseq * a.kv_heads;
  const int pair = a.max_pairs - 1 - u / per;
  const int rem = u - (u / per) * per;
  it.s = rem / a.kv_heads;
  it.g = rem - it.s * a.kv_heads;
  it.k0 = k0;
  it.L = k1 - k0;
  it.q0 = q0;
  it.qlen = q1 - q0;
  it.lcp = it.L - it.qlen;
  it.mb0 = 2 * pair;
  const int mb1 = it.mb0 + 1;
  it.nkt0 = it.mb0 * a.qpt < it.qlen ? (it.lcp + min(it.qlen, (it.mb0 + 1) * a.qpt) + a.bk - 1) / a.bk : 0;
  it.nkt1 = mb1 * a.qpt < it.qlen ? (it.lcp + min(it.qlen, (mb1 + 1) * a.qpt) + a.bk - 1) / a.bk : 0;
}

// Work distribution.  The valid units (a query-tile pair that exists) are
// numbered densely in (pair level descending, sequence, kv head) order -- the
// longest key ranges first -- and dealt to the CTAs in snake order (round r
// gives dense unit r*G + c to CTA c when r is even, r*G + G-1-c when odd), so
// every CTA gets the same number of units up to one, heavy ones spread evenly.
// Each CTA's scheduler warp walks the (level, sequence) grid 32 sequences per
// step (one L2 round trip for cu_q), picks out its own units, publishes them
// into a shared-memory ring (kRing entries, full/empty mbarriers) and ends with
// a sentinel (u = n_units).  Every role reads its next unit from the ring, so no
// role ever waits on global loads to find its work.
struct Ring {
  int* units;          // [kRing][kUnitWords]
  uint64_t* full;      // [kRing], 1 arrival (scheduler)
  uint64_t* empty;     // [kRing], kUnitConsumers arrivals
};

__device__ __forceinline__ void sched_units(const Args& a, const Ring& r, int lane) {
  int k = 0;
  const int G = static_cast<int>(gridDim.x), c = static_cast<int>(blockIdx.x);
  auto publish = [&](int u, const Unit& it) {
    const int slot = k % kRing;
    if (k >= kRing) mbar_wait(&r.empty[slot], ((k / kRing) - 1) & 1);
    if (lane == 0) {
      int* e = r.units + slot * kUnitWords;
      e[0] = u; e[1] = it.s; e[2] = it.g; e[3] = it.k0; e[4] = it.L; e[5] = it.q0; e[6] = it.qlen;
      e[7] = it.lcp; e[8] = it.mb0; e[9] = it.nkt0; e[10] = it.nkt1;
      mbar_arrive(&r.full[slot]);  // release: the entry is visible to the waiters
    }
    __syncwarp();
    ++k;
  };
  // Tail split: when the last partial round holds rem units and 2 rem <= G, those units
  // (the shortest: dense order is longest first) are dealt as 2 rem single-query-tile
  // half units, one per CTA, so the slowest CTAs run n/G + 1/2 units instead of n/G + 1
  // (C2: 512 units on 148 CTAs = 3 rounds + 68 -> 136 halves).  Needs the valid-unit
  // count first: one pass of ballots over the (pair level, sequence) grid.
  int64_t base = INT64_MAX;
  if (a.split_tail) {
    int64_t n_full = 0;
    for (int pair = a.max_pairs - 1; pair >= 0; --pair)
      for (int s0 = 0; s0 < a.nseq; s0 += 32) {
        const int sq = s0 + lane;
        bool ok = false;
        if (sq < a.nseq) ok = 2 * pair * a.qpt < __ldg(a.cu_q + sq + 1) - __ldg(a.cu_q + sq);
        n_full += static_cast<int64_t>(__popc(__ballot_sync(0xffffffffu, ok))) * a.kv_heads;
      }
    const int64_t rem = n_full % G;
    if (rem > 0 && 2 * rem <= G) base = n_full - rem;
  }
  int64_t dense = 0;  // dense index of the first unit of the current chunk
  for (int pair = a.max_pairs - 1; pair >= 0; --pair) {
    for (int s0 = 0; s0 < a.nseq; s0 += 32) {
      const int sq = s0 + lane;
      int k0 = 0, k1 = 0, q0 = 0, q1 = 0;
      bool ok = false;
      if (sq < a.nseq) {
        q0 = __ldg(a.cu_q + sq);
        q1 = __ldg(a.cu_q + sq + 1);
        ok = 2 * pair * a.qpt < q1 - q0;  // query tile 0 of the pair exists
        if (ok) {
          k0 = __ldg(a.cu + sq);
          k1 = __ldg(a.cu + sq + 1);
        }
      }
      const uint32_t bits = __ballot_sync(0xffffffffu, ok);
      const int64_t cnt = static_cast<int64_t>(__popc(bits)) * a.kv_heads;
      // one unit (or half unit) of dense index d in this chunk: geometry + publish
      auto emit = [&](int64_t d, int half) {
        const int e = static_cast<int>(d - dense);
        const int nth = e / a.kv_heads;  // nth valid sequence of the chunk
        int l = 0;
        uint32_t b = bits;
        for (int i = 0; i < nth; ++i) b &= b - 1;
        l = __ffs(b) - 1;
        Unit it;
        const int qa = __shfl_sync(0xffffffffu, q0, l), qb = __shfl_sync(0xffffffffu, q1, l);
        const int ka = __shfl_sync(0xffffffffu, k0, l), kb = __shfl_sync(0xffffffffu, k1, l);
        const int g = e - nth * a.kv_heads;
        const int u = (a.max_pairs - 1 - pair) * (a.nseq * a.kv_heads) + (s0 + l) * a.kv_heads + g;
        unit_geometry(a, u, ka, kb, qa, qb, it);
        if (half == 0) {  // the pair's first query tile alone
          it.nkt1 = 0;
        } else if (half == 1) {  // its second query tile alone, as tile h = 0
          if (it.nkt1 == 0) return;  // the pair has no second tile: nothing to run
          it.mb0 += 1;
          it.nkt0 = it.nkt1;
          it.nkt1 = 0;
        }
        publish(u, it);
      };
      // this CTA's dense indices in [dense, min(dense + cnt, base)): one candidate per snake round
      for (int64_t rd = dense / G; rd * G < dense + cnt; ++rd) {
        const int64_t d = rd * G + ((rd & 1) ? (G - 1 - c) : c);
        if (d < dense || d >= dense + cnt || d >= base) continue;
        emit(d, -1);
      }
      // the tail's half units: half k = 2 (d - base) + h goes to CTA k mod G
      for (int64_t d = dense > base ? dense : base; d < dense + cnt; ++d) {
        const int64_t k0 = 2 * (d - base);
        if (k0 % G == c) emit(d, 0);
        if ((k0 + 1) % G == c) emit(d, 1);
      }
      dense += cnt;
    }
  }
  Unit none;
  none.nkt0 = none.nkt1 = 0;
  none.s = none.g = none.k0 = none.L = none.q0 = none.qlen = none.lcp = none.mb0 = 0;
  publish(a.n_units, none);  // sentinel
  if (RDX_STATS_ON && a.cta_times && lane == 0) a.cta_times[3 * blockIdx.x + 2] = static_cast<unsigned long long>(k - 1);
}

// Entry k of the ring (blocking until published); the calling warp releases the slot.
__device__ __forceinline__ int ring_unit(const Ring& r, int k, Unit& it, int lane) {
  const int slot = k % kRing;
  mbar_wait(&r.full[slot], (k / kRing) & 1);
  const int* e = r.units + slot * kUnitWords;
  const int u = e[0];
  it.s = e[1]; it.g = e[2]; it.k0 = e[3]; it.L = e[4]; it.q0 = e[5]; it.qlen = e[6];
  it.lcp = e[7]; it.mb0 = e[8]; it.nkt0 = e[9]; it.nkt1 = e[10];
  __syncwarp();
  if (lane == 0) mbar_arrive(&r.empty[slot]);
  return u;
}

template <int HDP, int NQB, int NSLOT, uint32_t EMU, int BKT>
__global__ void __launch_bounds__(kThreads, 1)
attention_kernel(const __grid_constant__ CUtensorMap map_kv, const __grid_constant__ CUtensorMap map_q,
                 const __grid_constant__ CUtensorMap map_g4, const __grid_constant__ CUtensorMap map_r16, Args a) {
  using T = Tile<HDP, NQB, NSLOT, BKT>;
  constexpr bool DB = BKT == 64;  // 64-key S tiles, two S buffers per query tile
  constexpr int Q_BYTES = T::Q_BYTES, T_BYTES = T::T_BYTES, CH = T::CH;
  extern __shared__ __align__(1024) uint8_t smem[];  // dynamic smem starts 1024-aligned (no static smem)
  // the swizzled tiles need a 1024-byte aligned base (no room for slack: T::SMEM is
  // at the 227 KB limit).  Uniform check: every thread leaves, none waits on a barrier
  // that will never complete; rdx_device_status reports it.
  if (smem_u32(smem) & 1023u) {
    if (threadIdx.x == 0) atomicCAS(&g_device_status, 0, static_cast<int>(RDX_ERR_DEVICE_TIMEOUT));
    return;
  }
  uint8_t* sQ = smem;                                // [2 h][NQB][Q_BYTES]
  uint8_t* sT = smem + T::T_OFF;                     // [NSLOT][T_BYTES]
  float* sL = reinterpret_cast<float*>(smem + T::L_OFF);  // [2 h][2][128]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + T::BAR_OFF);
  uint64_t* q_full = bars + 0;                   // [2][NQB]
  uint64_t* q_free = bars + 2 * NQB;             // [2][NQB]
  uint64_t* t_full = bars + 4 * NQB;             // [NSLOT]
  uint64_t* t_free = t_full + NSLOT;             // [NSLOT]
  uint64_t* s_full = t_free + NSLOT;             // [2 h][2 S buffers] ([h][0] when single-buffered)
  uint64_t* p_full = s_full + 4;                 // [2 h][2] by P parity ([h][0] when single-buffered)
  uint64_t* o_full = p_full + 4;                 // [2]
  uint64_t* o_free = o_full + 2;                 // [2]
  uint64_t* l_full = o_free + 2;                 // [2 h][2 slots]: one barrier per sL slot, so the
                                                 // softmax can never run two phases ahead of a waiter
  uint64_t* pv_done = l_full + 4;                // [2 h]: PV_h(j) done, j < last (DB: O rescale may follow)
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(pv_done + 2);
  Ring ring;
  ring.units = reinterpret_cast<int*>(smem + T::RING_OFF);
  ring.full = reinterpret_cast<uint64_t*>(smem + T::RING_OFF + kRing * kUnitWords * 4);
  ring.empty = ring.full + kRing;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int i = 0; i < 2 * NQB; ++i) {
      mbar_init(&q_full[i], 32);
      mbar_init(&q_free[i], 1);
    }
    for (int i = 0; i < NSLOT; ++i) {
      mbar_init(&t_full[i], 32);
      mbar_init(&t_free[i], 1);
    }
    for (int i = 0; i < 4; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 128);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&pv_done[i], 1);
      mbar_init(&o_full[i], 1);
      mbar_init(&o_free[i], 128);
      mbar_init(&l_full[2 * i], 128);
      mbar_init(&l_full[2 * i + 1], 128);
    }
    for (int i = 0; i < kRing; ++i) {
      mbar_init(&ring.full[i], 1);
      mbar_init(&ring.empty[i], kUnitConsumers);
    }
    fence_mbar_init();
  }
  if (warp == kMmaWarp) {
    tmem_alloc(tmem_holder, TMEM_COLS);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  // barrier init + TMEM alloc overlapped the previous kernel's tail (PDL); inputs from here on
  pdl_wait();
  pdl_launch_dependents();
  if (RDX_STATS_ON && a.cta_times && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.cta_times[3 * blockIdx.x] = t;
  }

  if (warp >= 8) {
    setmaxnreg_dec<80>();
    if (warp == kLoaderWarp) {
      // ---------------------------------------------------------------- loader (one warp)
      long long st_free = 0;
      const long long st_t0 = clock64();
      EvLog evl;
      evl.n = 0;
      int q_cnt0 = 0, q_cnt1 = 0;
      uint32_t seq = 0;  // K/V ring sequence number (K and V tiles alternate)
      Unit it;
      for (int k = 0; ring_unit(ring, k, it, lane) < a.n_units; ++k) {
        // Q tiles of this unit
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (!(h ? it.nkt1 : it.nkt0)) continue;
          int& q_cnt = h ? q_cnt1 : q_cnt0;
          const int qb = q_cnt % NQB;
          if (q_cnt >= NQB) RDX_TWAIT(&q_free[h * NQB + qb], ((q_cnt / NQB) - 1) & 1, st_free);
          uint8_t* dstq = sQ + (h * NQB + qb) * Q_BYTES;
          uint64_t* bar = &q_full[h * NQB + qb];
          const int mb = it.mb0 + h;
          if (a.use_tma) {
            if (lane == 0) {
              mbar_arrive_expect_tx(bar, Q_BYTES);
              for (int hh = 0; hh < a.group; ++hh)
#pragma unroll
                for (int half = 0; half < T::HALVES; ++half)
                  tma_load_2d(&map_q, dstq + half * (BQ * 128) + hh * a.qpt * 128, bar,
                              (it.g * a.group + hh) * a.hd + half * 64, it.q0 + mb * a.qpt);
            } else {
              mbar_arrive(bar);
            }
          } else {
            const uint32_t sq = smem_u32(dstq);
#pragma unroll 4
            for (int k = 0; k < 4 * CH; ++k) {
              const int idx = lane + k * 32;
              const int r = idx / CH, c = idx % CH;
              const int hh = r / a.qpt, qi = mb * a.qpt + (r - hh * a.qpt);
              const bool ok = qi < it.qlen && c * 8 < a.hd;
              const __nv_bfloat16* src = ok ? a.qkv + static_cast<int64_t>(it.q0 + qi) * a.ld +
                                                  static_cast<int64_t>(it.g * a.group + hh) * a.hd + c * 8
                                            : a.qkv;
              cp_async16(sq + sw_off(r, c, BQ), src, ok ? 16u : 0u);
            }
            cp_async_arrive(bar);
          }
          ++q_cnt;
        }
        const int32_t kcol = a.heads * a.hd + it.g * a.hd;
        const int32_t vcol = kcol + a.kv_heads * a.hd;
        const int nkt = max(it.nkt0, it.nkt1);
        // rows of keys 4*lane .. 4*lane+3 of tile j (-1 past the sequence end)
        const bool ld_lane = 4 * lane < BKT;  // lanes holding keys of the tile (all 32 for 128-key tiles)
        auto key_rows = [&](int j, int (&r)[4]) {
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int key = j * BKT + 4 * lane + i;
            r[i] = (!ld_lane || key >= it.L) ? -1 : (a.scatter ? __ldg(a.scatter + it.k0 + key) : it.k0 + key);
          }
        };
        int rn[4];
        key_rows(0, rn);
#pragma unroll 1
        for (int j = 0; j < nkt; ++j) {
          int r[4] = {rn[0], rn[1], rn[2], rn[3]};
          if (j + 1 < nkt) key_rows(j + 1, rn);  // prefetch the next tile's rows
          const int row0 = __shfl_sync(0xffffffffu, r[0], 0);
          bool run = true;
#pragma unroll
          for (int i = 0; i < 4; ++i) run = run && (r[i] < 0 || r[i] == row0 + 4 * lane + i);
          const bool contiguous = __all_sync(0xffffffffu, run);
          // 16-key groups (lanes 4g..4g+3) that are contiguous runs of compact rows
          const int grow0 = __shfl_sync(0xffffffffu, r[0], lane & ~3);
          bool grun = true;
#pragma unroll
          for (int i = 0; i < 4; ++i) grun = grun && (r[i] < 0 || r[i] == grow0 + 4 * (lane & 3) + i);
          const uint32_t gbits = __ballot_sync(0xffffffffu, grun);
          const bool group_run = ((gbits >> (lane & ~3)) & 0xFu) == 0xFu && grow0 >= 0;
#pragma unroll
          for (int kv = 0; kv < 2; ++kv, ++seq) {
            const uint32_t slot = seq % NSLOT;
            if (seq >= NSLOT) RDX_TWAIT(&t_free[slot], ((seq / NSLOT) - 1) & 1, st_free);
            uint8_t* dst = sT + slot * T_BYTES;
            uint64_t* bar = &t_full[slot];
            const int32_t col = kv ? vcol : kcol;
            if (a.use_tma) {
              if (lane == 0) mbar_arrive_expect_tx(bar, T_BYTES);
              if (contiguous) {
                if (lane == 0) {
#pragma unroll
                  for (int half = 0; half < T::HALVES; ++half)
                    tma_load_2d(&map_kv, dst + half * (BKT * 128), bar, col + half * 64, row0);
                }
              } else if (!ld_lane) {
              } else if (group_run) {
                // one 16-row box per contiguous 16-key group, issued by the group's first lane
                if ((lane & 3) == 0) {
#pragma unroll
                  for (int half = 0; half < T::HALVES; ++half)
                    tma_load_2d(&map_r16, dst + half * (BKT * 128) + 4 * lane * 128, bar, col + half * 64, grow0);
                }
              } else {
#pragma unroll
                for (int half = 0; half < T::HALVES; ++half)
                  tma_gather4(&map_g4, smem_u32(dst + half * (BKT * 128) + 4 * lane * 128), bar, col + half * 64,
                              max(r[0], 0), max(r[1], 0), max(r[2], 0), max(r[3], 0));
              }
              if (lane != 0) mbar_arrive(bar);
              if (lane == 0) RDX_EV(0, 1 + kv, (j & 15) | (contiguous ? 0x80 : (group_run ? 0x40 : 0)));
            } else {
              const uint32_t st = smem_u32(dst);
#pragma unroll
              for (int i = 0; i < (ld_lane ? 4 : 0); ++i) {
#pragma unroll
                for (int c = 0; c < CH; ++c) {
                  const bool ok = r[i] >= 0 && c * 8 < a.hd;
                  cp_async16(st + sw_off(4 * lane + i, c, BKT),
                             a.qkv + static_cast<int64_t>(ok ? r[i] : 0) * a.ld + col + c * 8, ok ? 16u : 0u);
                }
              }
              cp_async_arrive(bar);
            }
          }
        }
      }
      if (lane == 0) RDX_EV_FLUSH();
      if (RDX_STATS_ON && lane == 0) {
        atomicAdd(a.stats + ST_LD_FREE, static_cast<unsigned long long>(st_free));
        atomicAdd(a.stats + ST_LD_TOTAL, static_cast<unsigned long long>(clock64() - st_t0));
      }
    } else if (warp == kMmaWarp) {
      // ---------------------------------------------------------------- MMA issuer (whole warp)
      long long st_t = 0, st_p = 0, st_q = 0, st_o = 0, st_iss = 0;
      const long long st_t0 = clock64();
      EvLog evl;
      evl.n = 0;
      int s_cnt0 = 0, s_cnt1 = 0;  // S tiles issued per h (== P tiles consumed)
      int o_cnt0 = 0, o_cnt1 = 0;  // units finished per h
      int q_cnt0 = 0, q_cnt1 = 0;  // Q tiles consumed per h
      uint32_t gt = 0;             // global key-tile counter (K at seq 2gt, V at 2gt+1)

      // half: every row of the query tile sees fewer than BKT/2 keys of this tile (a short
      // last tile): S with N = BKT/2 and only the first half of PV (the rest of P is zero).
      // S columns the softmax never reads and PV terms that are all exactly zero: same O.
      auto issue_S = [&](int h, int nkt_h, int j, uint32_t tile, bool half = false) {
        int& q_cnt = h ? q_cnt1 : q_cnt0;
        const int qb = q_cnt % NQB;
        if (j == 0) RDX_TWAIT(&q_full[h * NQB + qb], (q_cnt / NQB) & 1, st_q);
        const uint32_t kslot = (2 * tile) % NSLOT;
        if (!a.use_tma) fence_proxy_async_smem();  // cp.async (generic proxy) writes -> tcgen05 operand reads
        tc_fence_after();
        const uint32_t qa = smem_u32(sQ + (h * NQB + qb) * Q_BYTES), ka = smem_u32(sT + kslot * T_BYTES);
        const uint32_t sacc = tmem + h * 128;
        const uint64_t qd = sdesc(qa, 16, 1024), kd = sdesc(ka, 16, 1024);  // + (byte offset >> 4) per step
        const long long st_i0 = RDX_STATS_ON ? clock64() : 0;
#pragma unroll
        for (int kk = 0; kk < HDP / 16; ++kk)
          umma_ss_elect(sacc, qd + (((kk >> 2) * (BQ * 128) + (kk & 3) * 32) >> 4),
                        kd + (((kk >> 2) * (BKT * 128) + (kk & 3) * 32) >> 4), half ? T::IDESC_S_HALF : T::IDESC_S,
                        kk > 0 ? 1u : 0u);
        commit_elect(&s_full[2 * h]);
        if (lane == 0) RDX_EV(1, 1, h * 16 + j);  // MMA: S_h(j) issued
        if (RDX_STATS_ON) st_iss += clock64() - st_i0;
        if (h) ++s_cnt1; else ++s_cnt0;
        if (j == nkt_h - 1) {
          commit_elect(&q_free[h * NQB + qb]);
          ++q_cnt;
        }
      };
      auto issue_PV = [&](int h, int nkt_h, int j, uint32_t tile, bool half = false) {
        int& o_cnt = h ? o_cnt1 : o_cnt0;
        const int s_cnt = h ? s_cnt1 : s_cnt0;
        // P_h(j) is published in two halves (keys [0, BKT/2) on p_full[2h+1], the rest on
        // p_full[2h]): the first half's MMAs run while the softmax exponentiates the second.
        // Same K = 16 MMA sequence into O as one batch, so the same bits.
        RDX_TWAIT(&p_full[2 * h + 1], (s_cnt - 1) & 1, st_p);
        if (lane == 0) RDX_EV(1, 2, h * 16 + j);  // MMA: P_h(j) first half seen
        if (j == 0 && o_cnt > 0) RDX_TWAIT(&o_free[h], (o_cnt - 1) & 1, st_o);
        if (!a.use_tma) fence_proxy_async_smem();
        tc_fence_after();
        const uint32_t va = smem_u32(sT + ((2 * tile + 1) % NSLOT) * T_BYTES);
        const uint32_t o = tmem + O_COL + h * 128, pa = tmem + h * 128;
        const uint64_t vd = sdesc(va, BKT * 128, 1024);
        const long long st_i0 = RDX_STATS_ON ? clock64() : 0;
#pragma unroll
        for (int kk = 0; kk < BKT / 32; ++kk)
          umma_ts_elect(o, pa + kk * 8, vd + ((kk * 2048) >> 4), T::IDESC_PV, (j > 0 || kk > 0) ? 1u : 0u);
        RDX_TWAIT(&p_full[2 * h], (s_cnt - 1) & 1, st_p);  // second half (waited even when unused: parity)
        tc_fence_after();
        if (!half) {
#pragma unroll
          for (int kk = BKT / 32; kk < BKT / 16; ++kk)
            umma_ts_elect(o, pa + kk * 8, vd + ((kk * 2048) >> 4), T::IDESC_PV, 1u);
        }
        if (RDX_STATS_ON) st_iss += clock64() - st_i0;
        if (j == nkt_h - 1) {
          commit_elect(&o_full[h]);
          ++o_cnt;
        }
      };
      auto wait_tile = [&](uint32_t seqno) { RDX_TWAIT(&t_full[seqno % NSLOT], (seqno / NSLOT) & 1, st_t); };

      if constexpr (DB) {
        // 64-key S tiles, two S buffers per query tile: S_h(j+2) goes into the buffer
        // PV_h(j) has just read, so S runs two key tiles ahead of the softmax and the
        // softmax never waits for its S behind its own P (the single-buffered chain).
        int sc[2] = {0, 0};  // S tiles issued per h (buffer sc & 1)
        int pc[2] = {0, 0};  // P tiles consumed per h (p_full[h][pc & 1], P(k) sits in buffer k & 1)
        int oc[2] = {0, 0};  // units finished per h
        int qc[2] = {0, 0};  // Q tiles consumed per h
        int kread = 0;       // next ring entry
        struct It {
          int u, j, n0, n1, nall;
        };
        auto fetch = [&](It& x) {
          Unit tmp;
          x.u = ring_unit(ring, kread++, tmp, lane);
          x.j = 0;
          x.n0 = tmp.nkt0;
          x.n1 = tmp.nkt1;
          x.nall = max(tmp.nkt0, tmp.nkt1);
        };
        auto advance = [&](const It& x, It& y) {
          if (x.u >= a.n_units) {
            y = x;
          } else if (x.j + 1 < x.nall) {
            y = x;
            ++y.j;
          } else {
            fetch(y);
          }
        };
        auto issue_S2 = [&](int h, const It& x, uint32_t tile) {
          const int nkt = h ? x.n1 : x.n0;
          if (x.j >= nkt) return;
          const int qb = qc[h] % NQB;
          if (x.j == 0) RDX_TWAIT(&q_full[h * NQB + qb], (qc[h] / NQB) & 1, st_q);
          if (!a.use_tma) fence_proxy_async_smem();
          tc_fence_after();
          const uint32_t qa = smem_u32(sQ + (h * NQB + qb) * Q_BYTES);
          const uint32_t ka = smem_u32(sT + ((2 * tile) % NSLOT) * T_BYTES);
          const int b = sc[h] & 1;
          const uint32_t sacc = tmem + h * 128 + b * 64;
          const uint64_t qd = sdesc(qa, 16, 1024), kd = sdesc(ka, 16, 1024);
          const long long st_i0 = RDX_STATS_ON ? clock64() : 0;
#pragma unroll
          for (int kk = 0; kk < HDP / 16; ++kk)
            umma_ss_elect(sacc, qd + (((kk >> 2) * (BQ * 128) + (kk & 3) * 32) >> 4),
                          kd + (((kk >> 2) * (BKT * 128) + (kk & 3) * 32) >> 4), T::IDESC_S, kk > 0 ? 1u : 0u);
          commit_elect(&s_full[2 * h + b]);
          if (lane == 0) RDX_EV(1, 1, h * 16 + (x.j & 15));  // MMA: S_h(j) issued
          if (RDX_STATS_ON) st_iss += clock64() - st_i0;
          ++sc[h];
          if (x.j == nkt - 1) {
            commit_elect(&q_free[h * NQB + qb]);
            ++qc[h];
          }
        };
        auto issue_PV2 = [&](int h, const It& x, uint32_t tile) {
          const int nkt = h ? x.n1 : x.n0;
          if (x.j >= nkt) return;
          const int b = pc[h] & 1;
          RDX_TWAIT(&p_full[2 * h + b], (pc[h] >> 1) & 1, st_p);
          if (lane == 0) RDX_EV(1, 2, h * 16 + (x.j & 15));  // MMA: P_h(j) seen
          ++pc[h];
          if (x.j == 0 && oc[h] > 0) RDX_TWAIT(&o_free[h], (oc[h] - 1) & 1, st_o);
          if (!a.use_tma) fence_proxy_async_smem();
          tc_fence_after();
          const uint32_t va = smem_u32(sT + ((2 * tile + 1) % NSLOT) * T_BYTES);
          const uint32_t o = tmem + O_COL + h * 128, pa = tmem + h * 128 + b * 64;
          const uint64_t vd = sdesc(va, BKT * 128, 1024);
          const long long st_i0 = RDX_STATS_ON ? clock64() : 0;
#pragma unroll
          for (int kk = 0; kk < BKT / 16; ++kk)
            umma_ts_elect(o, pa + kk * 8, vd + ((kk * 2048) >> 4), T::IDESC_PV, (x.j > 0 || kk > 0) ? 1u : 0u);
          if (RDX_STATS_ON) st_iss += clock64() - st_i0;
          if (x.j == nkt - 1) {
            commit_elect(&o_full[h]);
            ++oc[h];
          } else {
            commit_elect(&pv_done[h]);  // the softmax of tile j + 1 may rescale O after this
          }
        };
        auto wait_tile2 = [&](uint32_t seqno) { RDX_TWAIT(&t_full[seqno % NSLOT], (seqno / NSLOT) & 1, st_t); };
        It cur, n1, n2;
        uint32_t gt = 0;  // iteration (key tile) counter: K at ring seq 2gt, V at 2gt + 1
        fetch(cur);
        if (cur.u < a.n_units) {
          wait_tile2(0);
          issue_S2(0, cur, 0);
          issue_S2(1, cur, 0);
          commit_elect(&t_free[0]);
        }
        advance(cur, n1);
        if (n1.u < a.n_units) {
          wait_tile2(2);
          issue_S2(0, n1, 1);
          issue_S2(1, n1, 1);
          commit_elect(&t_free[2 % NSLOT]);
        }
        advance(n1, n2);
        while (cur.u < a.n_units) {
          const bool nx = n2.u < a.n_units;
          wait_tile2(2 * gt + 1);  // V(cur)
          if (lane == 0) RDX_EV(1, 4, cur.j & 15);  // MMA: V(cur) resident
          issue_PV2(0, cur, gt);
          if (nx) {
            wait_tile2(2 * (gt + 2));  // K(cur + 2)
            if (lane == 0) RDX_EV(1, 3, n2.j & 15);  // MMA: K(cur + 2) resident
            issue_S2(0, n2, gt + 2);
          }
          issue_PV2(1, cur, gt);
          commit_elect(&t_free[(2 * gt + 1) % NSLOT]);  // V(cur) consumed by both PV
          if (nx) {
            issue_S2(1, n2, gt + 2);
            commit_elect(&t_free[(2 * (gt + 2)) % NSLOT]);  // K(cur + 2) consumed by both S
          }
          cur = n1;
          n1 = n2;
          advance(n1, n2);
          ++gt;
        }
      } else {
        Unit tmp, pre;
        // keys visible to the last row of query tile h of a unit: tile j is short when
        // khi - j * BKT <= BKT / 2 (only 128-key tiles; the 64-key ones never split)
        auto khi = [&](const Unit& u, int h) { return u.lcp + min(u.qlen, (u.mb0 + h + 1) * a.qpt); };
        auto short_tile = [&](int kh, int j) { return BKT == 128 && kh - j * BKT <= BKT / 2; };
        int kcur = 0;  // ring entry of the current unit
        int ucur = ring_unit(ring, 0, tmp, lane);
        int c0 = tmp.nkt0, c1 = tmp.nkt1, call = max(tmp.nkt0, tmp.nkt1);  // key tiles of the current unit
        int ck0 = khi(tmp, 0), ck1 = khi(tmp, 1);
        int jcur = 0;
        int upre = a.n_units;  // the unit after the current one, fetched while S/softmax of this one run
        if (ucur < a.n_units) {
          wait_tile(2 * gt);
          if (c0 > 0) issue_S(0, c0, 0, gt, short_tile(ck0, 0));
          if (c1 > 0) issue_S(1, c1, 0, gt, short_tile(ck1, 0));
          commit_elect(&t_free[(2 * gt) % NSLOT]);  // both S of tile 0 issued: K slot free when done
          upre = ring_unit(ring, kcur + 1, pre, lane);
        }
        while (ucur < a.n_units) {
          int unxt = ucur, jnxt = jcur + 1, n0 = c0, n1 = c1, nall = call, nk0 = ck0, nk1 = ck1;
          if (jnxt >= call) {
            unxt = upre;
            jnxt = 0;
            n0 = pre.nkt0;
            n1 = pre.nkt1;
            nall = max(pre.nkt0, pre.nkt1);
            nk0 = khi(pre, 0);
            nk1 = khi(pre, 1);
          }
          const bool has_next = unxt < a.n_units;
          const uint32_t tnext = gt + 1;
          wait_tile(2 * gt + 1);  // V(cur)
          if (jcur < c0) issue_PV(0, c0, jcur, gt, short_tile(ck0, jcur));
          if (has_next) {
            wait_tile(2 * tnext);  // K(next)
            if (jnxt < n0) issue_S(0, n0, jnxt, tnext, short_tile(nk0, jnxt));
          }
          if (jcur < c1) issue_PV(1, c1, jcur, gt, short_tile(ck1, jcur));
          commit_elect(&t_free[(2 * gt + 1) % NSLOT]);  // V(cur) consumed by both PV
          if (has_next) {
            if (jnxt < n1) issue_S(1, n1, jnxt, tnext, short_tile(nk1, jnxt));
            commit_elect(&t_free[(2 * tnext) % NSLOT]);  // K(next) consumed by both S
          }
          const bool switched = unxt != ucur;
          ucur = unxt;
          jcur = jnxt;
          c0 = n0;
          c1 = n1;
          ck0 = nk0;
          ck1 = nk1;
          call = nall;
          ++gt;
          // new current unit: its S tiles are issued; the entry after it is already in the ring
          if (switched) {
            ++kcur;
            if (ucur < a.n_units) upre = ring_unit(ring, kcur + 1, pre, lane);
          }
        }
      }
      if (lane == 0) RDX_EV_FLUSH();
      if (RDX_STATS_ON && lane == 0) {
        atomicAdd(a.stats + ST_MMA_TFULL, static_cast<unsigned long long>(st_t));
        atomicAdd(a.stats + ST_MMA_PFULL, static_cast<unsigned long long>(st_p));
        atomicAdd(a.stats + ST_MMA_QFULL, static_cast<unsigned long long>(st_q));
        atomicAdd(a.stats + ST_MMA_OFREE, static_cast<unsigned long long>(st_o));
        atomicAdd(a.stats + ST_MMA_ISSUE, static_cast<unsigned long long>(st_iss));
        atomicAdd(a.stats + ST_MMA_TOTAL, static_cast<unsigned long long>(clock64() - st_t0));
      }
    } else if (warp == kSchedWarp) {
      sched_units(a, ring, lane);
    } else if (warp >= 9 && warp <= 12) {
      // ---------------------------------------------------------------- epilogue: O_h / l -> bf16 compact rows
      const int q4 = warp & 3;            // TMEM lane quarter of this warp
      const int t = q4 * 32 + lane;       // tile row == TMEM lane
      const uint32_t lane_base = tmem + (static_cast<uint32_t>(q4 * 32) << 16);
      long long st_w = 0;
      const long long st_t0 = clock64();
      EvLog evl;
      evl.n = 0;
      int cnt0 = 0, cnt1 = 0;
      Unit it;
      for (int k = 0; ring_unit(ring, k, it, lane) < a.n_units; ++k) {
#pragma unroll 1
        for (int h = 0; h < 2; ++h) {
          if (!(h ? it.nkt1 : it.nkt0)) continue;
          int& cnt = h ? cnt1 : cnt0;
          const int mb = it.mb0 + h;
          const int hh = t / a.qpt, qi = mb * a.qpt + (t - hh * a.qpt);
          RDX_TWAIT(&l_full[2 * h + (cnt & 1)], (cnt >> 1) & 1, st_w);
          RDX_TWAIT(&o_full[h], cnt & 1, st_w);
          if (t == 0) RDX_EV(3, 1, h);  // epilogue: O_h ready
          tc_fence_after();
          const float l = sL[(h * 2 + (cnt & 1)) * BQ + t];
          const float inv = l > 0.f ? 1.f / l : 0.f;
          const bool valid = qi < it.qlen;
          __nv_bfloat16* orow = a.out + static_cast<int64_t>(it.q0 + (valid ? qi : 0)) * a.ld_out +
                                static_cast<int64_t>(it.g * a.group + hh) * a.hd;
          const uint32_t o_addr = lane_base + O_COL + h * 128;
#pragma unroll
          for (int c = 0; c < HDP; c += 32) {
            if (c < a.hd) {
              float ov[32];
              tmem_ld32p(o_addr + c, ov);
              tmem_wait_ld();
              if (valid) {
#pragma unroll
                for (int e = 0; e < 32; e += 8)
                  if (c + e < a.hd)
                    st_global_v4(orow + c + e, pack_bf16x2(ov[e] * inv, ov[e + 1] * inv),
                                 pack_bf16x2(ov[e + 2] * inv, ov[e + 3] * inv),
                                 pack_bf16x2(ov[e + 4] * inv, ov[e + 5] * inv),
                                 pack_bf16x2(ov[e + 6] * inv, ov[e + 7] * inv));
              }
            }
          }
          tc_fence_before();
          mbar_arrive(&o_free[h]);
          if (t == 0) RDX_EV(3, 2, h);  // epilogue: O_h stored
          ++cnt;
        }
      }
      if (t == 0) RDX_EV_FLUSH();
      if (RDX_STATS_ON && t == 0) {
        atomicAdd(a.stats + ST_EPI_WAIT, static_cast<unsigned long long>(st_w));
        atomicAdd(a.stats + ST_EPI_TOTAL, static_cast<unsigned long long>(clock64() - st_t0));
      }
    }
  } else {
    // ---------------------------------------------------------------- softmax (query tile h, row t)
    setmaxnreg_inc<176>();
    const int h = warp >> 2;
    const int t = threadIdx.x & 127;  // row of the tile == TMEM lane
    const uint32_t lane_base = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16);
    const uint32_t s_addr = lane_base + h * 128;
    const uint32_t o_addr = lane_base + O_COL + h * 128;
    int s_cnt = 0, u_cnt = 0, pv_cnt = 0;
    long long st_s = 0, st_resc = 0, st_exp = 0;
    const long long st_t0 = clock64();
    EvLog evl;
    evl.n = 0;
    Unit it;
    for (int k = 0; ring_unit(ring, k, it, lane) < a.n_units; ++k) {
      const int nkt_h = h ? it.nkt1 : it.nkt0;
      if (!nkt_h) continue;
      const int mb = it.mb0 + h;
      const int hh = t / a.qpt, qi = mb * a.qpt + (t - hh * a.qpt);
      // keys 0..pos visible; rows past the query range (never stored) see key 0 only
      const int pos = qi < it.qlen ? it.lcp + qi : 0;
      const int pos_min = __reduce_min_sync(0xffffffffu, pos);
      const int pos_max = __reduce_max_sync(0xffffffffu, pos);
      float m_run = -INFINITY, l_run = 0.f;
#pragma unroll 1
      for (int j = 0; j < nkt_h; ++j, ++s_cnt) {
        // S_h(j): buffer s_cnt & 1 when double-buffered
        const uint32_t s_cur = DB ? s_addr + (s_cnt & 1) * 64 : s_addr;
        if constexpr (DB) RDX_TWAIT(&s_full[2 * h + (s_cnt & 1)], (s_cnt >> 1) & 1, st_s);
        else RDX_TWAIT(&s_full[2 * h], s_cnt & 1, st_s);
        if (t == 0) RDX_EV(2, 1, h * 16 + j);  // softmax: S_h(j) ready
        tc_fence_after();
        const int kbase = j * BKT;
        // warp-uniform column classes of this tile (32-column chunks): chunks at or past
        // vis_warp are masked for every row of the warp (never loaded, max'ed or exp'ed);
        // chunks below lo_vis are visible for every row (no per-element mask)
        const int vis_warp = pos_max - kbase + 1;
        const int lo_vis = pos_min - kbase + 1;
        float sv[BKT];
#pragma unroll
        for (int c = 0; c < BKT; c += 32)
          if (c < vis_warp) tmem_ld32p(s_cur + c, sv + c);
        tmem_wait_ld();
        if (t == 0) RDX_EV(2, 3, static_cast<int>(sv[0] != 12345.f));  // softmax: S in registers
        const int nvis = pos - kbase + 1;  // visible keys of this row in the tile
        float mx[8];
#pragma unroll
        for (int u8 = 0; u8 < 8; ++u8) mx[u8] = -INFINITY;
#pragma unroll
        for (int c0 = 0; c0 < BKT; c0 += 32) {
          if (c0 >= vis_warp) continue;  // whole chunk masked for the warp (column 0 is always visible)
          if (c0 + 32 > lo_vis) {         // the diagonal crosses this chunk: per-element mask
#pragma unroll
            for (int c = c0; c < c0 + 32; ++c) sv[c] = c < nvis ? sv[c] : -INFINITY;
          }
#pragma unroll
          for (int c = c0; c < c0 + 32; ++c) mx[c & 7] = fmaxf(mx[c & 7], sv[c]);
        }
        const float mt = fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])),
                               fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7]))) * a.scale_log2;
        const bool need = mt > m_run + kRescaleThreshold;
        bool resc_o = false;  // DB: O_h rescaled by alpha once PV_h(j-1) has completed
        float alpha_o = 1.f;
        if (__any_sync(0xffffffffu, need)) {
          const float m_new = need ? mt : m_run;
          const float alpha = ex2(m_run - m_new);  // 0 on the first tile (m_run = -inf)
          if (DB && j > 0) {
            resc_o = true;
            alpha_o = alpha;
          } else if (j > 0) {
            if (RDX_STATS_ON) ++st_resc;
            // O_h holds PV_h(0..j-1): complete, since S_h(j) was issued after PV_h(j-1)
#pragma unroll 1
            for (int c = 0; c < HDP; c += 32) {
              float ov[32];
              tmem_ld32p(o_addr + c, ov);
              tmem_wait_ld();
#pragma unroll
              for (int e = 0; e < 32; ++e) ov[e] *= alpha;
              tmem_st32(o_addr + c, ov);
            }
          }
          l_run *= alpha;
          m_run = m_new;
        }
        const long long st_b = RDX_STATS_ON ? clock64() : 0;
        if (t == 0) RDX_EV(2, 4, h * 16 + j);  // softmax: max done
        const uint64_t scale2 = f2pack(a.scale_log2, a.scale_log2), negm2 = f2pack(-m_run, -m_run);
        uint64_t ls[4] = {0, 0, 0, 0};  // pairs of fp32 partial row sums (+0.0f bits)
#pragma unroll
        for (int c = 0; c < BKT; c += 32) {
          uint32_t pw[16];
          if (c >= vis_warp) {
#pragma unroll
            for (int e = 0; e < 16; ++e) pw[e] = 0u;
            tmem_st16u(s_cur + c / 2, pw);
            if (!DB && c == BKT / 2 - 32) {  // first half of P_h(j) complete (see below)
              tmem_wait_st();
              tc_fence_before();
              mbar_arrive(&p_full[2 * h + 1]);
            }
            continue;
          }
#pragma unroll
          for (int e = 0; e < 32; e += 2) {
            const uint64_t x = ffma2(f2pack(sv[c + e], sv[c + e + 1]), scale2, negm2);
            uint64_t p;
            if (EMU & (1u << ((e >> 1) & 7))) {
              p = exp2_poly2(x);  // FMA-pipe exp2: offloads the MUFU unit
            } else {
              float x0, x1;
              f2unpack(x, x0, x1);
              p = f2pack(ex2(x0), ex2(x1));
            }
            ls[(e >> 1) & 3] = fadd2(ls[(e >> 1) & 3], p);
            float p0, p1;
            f2unpack(p, p0, p1);
            pw[e >> 1] = pack_bf16x2(p0, p1);
          }
          tmem_st16u(s_cur + c / 2, pw);  // P over the first BKT / 2 columns of S_h
          if (!DB && c == BKT / 2 - 32) {
            // first half of P_h(j) complete: its PV MMAs may start (p_full[2h+1])
            tmem_wait_st();
            tc_fence_before();
            mbar_arrive(&p_full[2 * h + 1]);
          }
        }
        {
          float s0, s1;
          f2unpack(fadd2(fadd2(ls[0], ls[1]), fadd2(ls[2], ls[3])), s0, s1);
          l_run += s0 + s1;
        }
        if (t == 0) RDX_EV(2, 5, static_cast<int>(l_run != 12345.f));  // softmax: exp + P stores issued
        if constexpr (DB) {
          if (j > 0) {
            // PV_h(j-1) is still in flight behind S_h(j+1): wait for it (lockstep, one
            // phase per tile) before O_h may be rescaled for this tile's new max
            RDX_TWAIT(&pv_done[h], pv_cnt & 1, st_s);
            ++pv_cnt;
            if (__any_sync(0xffffffffu, resc_o)) {
              if (RDX_STATS_ON) ++st_resc;
              tc_fence_after();
#pragma unroll 1
              for (int c = 0; c < HDP; c += 32) {
                float ov[32];
                tmem_ld32p(o_addr + c, ov);
                tmem_wait_ld();
#pragma unroll
                for (int e = 0; e < 32; ++e) ov[e] *= alpha_o;
                tmem_st32(o_addr + c, ov);
              }
            }
          }
        }
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(&p_full[DB ? 2 * h + (s_cnt & 1) : 2 * h]);
        if (t == 0) RDX_EV(2, 2, h * 16 + j);  // softmax: P_h(j) published
        if (RDX_STATS_ON) st_exp += clock64() - st_b;
      }
      // hand the row sum to the epilogue warps (slot u_cnt & 1: the epilogue of
      // unit u_cnt - 2 finished before PV_h(u_cnt - 1) could start)
      sL[(h * 2 + (u_cnt & 1)) * BQ + t] = l_run;
      mbar_arrive(&l_full[2 * h + (u_cnt & 1)]);
      ++u_cnt;
    }
    if (t == 0) RDX_EV_FLUSH();
    if (RDX_STATS_ON && t == 0) {
      atomicAdd(a.stats + ST_SM_SFULL, static_cast<unsigned long long>(st_s));
      atomicAdd(a.stats + ST_SM_RESCALE, static_cast<unsigned long long>(st_resc));
      atomicAdd(a.stats + ST_SM_EXP, static_cast<unsigned long long>(st_exp));
      atomicAdd(a.stats + ST_SM_TOTAL, static_cast<unsigned long long>(clock64() - st_t0));
    }
  }
  tc_fence_before();
  __syncthreads();
  if (RDX_STATS_ON && a.cta_times && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.cta_times[3 * blockIdx.x + 1] = t;
  }
  if (warp == kMmaWarp) {
    tc_fence_after();
    tmem_dealloc(tmem, TMEM_COLS);
  }
}

unsigned long long* g_stats = nullptr;  // debug counters (RDX_ATTN_STATS=1)
int g_attn_bk64 = 1;                    // rdx_attention_debug_bk64 (AND-ed with RDX_ATTN_BK64=1)
int g_attn_split = 0;                   // rdx_attention_debug_split: 2 = half units forced on
unsigned long long* g_cta_times = nullptr;  // debug per-CTA [start, end, units]
uint32_t* g_trace = nullptr;            // debug event log of CTA 0 (RDX_ATTN_STATS=1)

template <int HDP, int NQB, int NSLOT, uint32_t EMU, int BKT = BK>
int launch(Args a, int64_t qkv_rows, cudaStream_t st) {
  using T = Tile<HDP, NQB, NSLOT, BKT>;
  auto kern = attention_kernel<HDP, NQB, NSLOT, EMU, BKT>;
  a.bk = BKT;
  static bool attr_set = false;
  if (!attr_set) {
    RDX_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, T::SMEM));
    attr_set = true;
  }
  CUtensorMap map_kv, map_q, map_g4, map_r16;
  std::memset(&map_r16, 0, sizeof(map_r16));
  std::memset(&map_kv, 0, sizeof(map_kv));
  std::memset(&map_q, 0, sizeof(map_q));
  std::memset(&map_g4, 0, sizeof(map_g4));
  if (a.use_tma) {
    int e = gemm::make_map(&map_kv, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, a.qkv, a.ld, qkv_rows, a.ld, 64, BKT,
                           CU_TENSOR_MAP_SWIZZLE_128B);
    if (e) return e;
    e = gemm::make_map(&map_q, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, a.qkv, a.ld, qkv_rows, a.ld, 64, a.qpt,
                       CU_TENSOR_MAP_SWIZZLE_128B);
    if (e) return e;
    e = gemm::make_map(&map_g4, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, a.qkv, a.ld, qkv_rows, a.ld, 64, 1,
                       CU_TENSOR_MAP_SWIZZLE_128B);
    if (e) return e;
    e = gemm::make_map(&map_r16, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, a.qkv, a.ld, qkv_rows, a.ld, 64, 16,
                       CU_TENSOR_MAP_SWIZZLE_128B);
    if (e) return e;
  }
  const int ctas = a.n_units < num_sms() ? a.n_units : num_sms();
  return launch_pdl(kern, dim3(static_cast<unsigned>(ctas)), dim3(kThreads), T::SMEM, st, map_kv, map_q, map_g4,
                    map_r16, a);
}

}  // namespace attn
}  // namespace rdx

extern "C" int rdx_attention(const void* qkv_bf16, int64_t ld_qkv, int64_t qkv_rows, const int32_t* scatter,
                             const int32_t* cu, const int32_t* cu_q, int64_t n_seqs, int32_t max_q_len,
                             int32_t max_k_len, int32_t heads, int32_t kv_heads, int32_t head_dim,
                             float softmax_scale, void* out_bf16, int64_t ld_out, void* stream) {
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
  a.group = heads / kv_heads;
  a.qpt = BQ / a.group;
  const int64_t tiles = (static_cast<int64_t>(max_q_len) + a.qpt - 1) / a.qpt;
  a.max_pairs = static_cast<int>((tiles + 1) / 2);
  const int64_t units = static_cast<int64_t>(a.max_pairs) * n_seqs * kv_heads;
  if (units >= (int64_t(1) << 31)) return RDX_ERR_CAPACITY_EXCEEDED;
  a.n_units = static_cast<int>(units);
  a.scale_log2 = softmax_scale * 1.4426950408889634f;
  a.use_tma = (head_dim % 64 == 0) && (reinterpret_cast<uintptr_t>(qkv_bf16) % 16 == 0) && qkv_rows > 0 &&
              qkv_rows < (int64_t(1) << 31) && ld_qkv < (int64_t(1) << 31);
  a.stats = nullptr;
  a.trace = nullptr;
  a.trace_cta = 0;
  // off by default: measured slower at C2 (35.5 vs 34.8 us suffix, 38.8 vs 32.5 us on the
  // literal configs[1] shape): the counting pass delays every CTA's first unit and a lone
  // query tile loses the two-tile ping-pong that hides its softmax
  static const int split_env = [] {
    const char* v = std::getenv("RDX_ATTN_SPLIT");
    return v && v[0] == '1' ? 1 : 0;
  }();
  a.split_tail = split_env || g_attn_split == 2;
  a.cta_times = nullptr;
  if (const char* e = std::getenv("RDX_ATTN_STATS")) {
    if (e[0] == '1') {
      if (!g_stats) {
        RDX_CUDA_TRY(cudaMalloc(&g_stats, ST_N * sizeof(unsigned long long)));
        RDX_CUDA_TRY(cudaMemset(g_stats, 0, ST_N * sizeof(unsigned long long)));
      }
      a.stats = g_stats;
      if (!g_trace) RDX_CUDA_TRY(cudaMalloc(&g_trace, (2 + 2 * 4096) * sizeof(uint32_t)));
      RDX_CUDA_TRY(cudaMemsetAsync(g_trace, 0, 2 * sizeof(uint32_t), as_stream(stream)));
      a.trace = g_trace;
      if (const char* tc = std::getenv("RDX_ATTN_TRACE_CTA")) a.trace_cta = atoi(tc);
      if (!g_cta_times) RDX_CUDA_TRY(cudaMalloc(&g_cta_times, 3 * 1024 * sizeof(unsigned long long)));
      a.cta_times = g_cta_times;
    }
  }
  // short units (few key tiles): double-buffer Q; long units: deeper K/V ring
  const bool short_units = max_k_len > 0 && (max_k_len + BK - 1) / BK <= kShortUnitTiles;
  cudaStream_t s = as_stream(stream);
  if (head_dim <= 64)
    return short_units ? launch<64, 2, 4, kEmulated>(a, qkv_rows, s) : launch<64, 1, 6, kEmulated>(a, qkv_rows, s);
  // short suffix-query units at head_dim 128: 64-key tiles with double-buffered S when enabled
  // (RDX_ATTN_BK64=1 / rdx_attention_debug_bk64(1)).  Off by default: it gains 1 % at C2 (35.1 vs
  // 35.5 us) but the plain layout is faster on 128-key tiles (43.8 vs 46.8 us), and different key
  // tiles change the online-softmax order, so suffix and plain attention (RadixMLP on vs off)
  // would no longer give bit-identical rows.
  static const int bk64 = [] {
    const char* v = std::getenv("RDX_ATTN_BK64");
    return v && v[0] == '1' ? 1 : 0;
  }();
  if (short_units && scatter && (bk64 || g_attn_bk64 == 2)) return launch<128, 2, 6, kEmulated, 64>(a, qkv_rows, s);
  return short_units ? launch<128, 2, 3, kEmulated>(a, qkv_rows, s) : launch<128, 1, 4, kEmulated>(a, qkv_rows, s);
}

// Debug: copy (and reset) the summed per-role clock counters of every launch
// since the last call; n >= ST_N slots (order: enum ST_* above).
extern "C" int rdx_attention_debug_stats(unsigned long long* host, int n) {
  using namespace rdx::attn;
  if (!g_stats) return RDX_ERR_INVALID_ARGUMENT;
  const int m = n < ST_N ? n : ST_N;
  RDX_CUDA_TRY(cudaMemcpy(host, g_stats, m * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
  RDX_CUDA_TRY(cudaMemset(g_stats, 0, ST_N * sizeof(unsigned long long)));
  return RDX_OK;
}

// Debug: per-CTA [start ns, end ns, units] of the last launch (stats builds), n_ctas entries.
extern "C" int rdx_attention_debug_cta_times(unsigned long long* host, int n_ctas) {
  using namespace rdx::attn;
  if (!g_cta_times || n_ctas <= 0 || n_ctas > 1024) return RDX_ERR_INVALID_ARGUMENT;
  RDX_CUDA_TRY(cudaMemcpy(host, g_cta_times, 3 * n_ctas * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
  return RDX_OK;
}

// Debug: copy the CTA-0 event log of the last launch (RDX_ATTN_STATS=1 builds
// with RDX_ATTN_STATS_BUILD): [count, (clock, code) x min(count, 4096)].
extern "C" int rdx_attention_debug_trace(uint32_t* host, int n_words) {
  using namespace rdx::attn;
  if (!g_trace || n_words < 2) return RDX_ERR_INVALID_ARGUMENT;
  const int m = n_words < 2 + 2 * 4096 ? n_words : 2 + 2 * 4096;
  RDX_CUDA_TRY(cudaMemcpy(host, g_trace, m * sizeof(uint32_t), cudaMemcpyDeviceToHost));
  return RDX_OK;
}

int rdx::take_device_status_attention(int* out, cudaStream_t st) { return take_device_status(out, st); }

// Debug: the 64-key double-buffered-S variant for short units on (1) / off (0) for A/B
// runs; returns the previous setting.
extern "C" int rdx_attention_debug_bk64(int on) {
  const int prev = rdx::attn::g_attn_bk64 == 2 ? 1 : 0;
  rdx::attn::g_attn_bk64 = on ? 2 : 0;  // 2 = forced on for this process
  return prev;
}

// Debug: deal a short last round of attention units as single-query-tile half units
// (1) or not (0, the default); returns the previous setting.
extern "C" int rdx_attention_debug_split(int on) {
  const int prev = rdx::attn::g_attn_split == 2 ? 1 : 0;
  rdx::attn::g_attn_split = on ? 2 : 0;
  return prev;
}
