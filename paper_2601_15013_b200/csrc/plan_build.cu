// plan_build.cu — GPU prefix-trie planner, bit-exact to the reference trie.
//
// Reference: pkg/src/radix_compact/trie.py:73-148 (_build_indices /
// build_plan).  The reference walks a trie sequence by sequence; a node is a
// (parent, key = (pos << 32) ^ tok) pair and compact ids are node creation
// order.  Two facts make a flat data-parallel formulation exact:
//
//  (1) token i maps to the same compact row as token j  <=>  the (tok, pos)
//      paths from their sequence starts are identical (trie.py:3-4);
//  (2) once a sequence creates a node, every later node of that sequence is
//      new (its parent has no children yet, trie.py:100-118), so the compact
//      rows of sequence s are the contiguous suffix [cu[s] + lcp_s, cu[s+1])
//      and compact ids are ranks in (sequence, depth) order.
//
// Algorithm (one persistent launch, phases split by grid-wide barriers):
//   P0  validate cu; seg[i] (binary search); m_i = mix(tok, pos, depth, seed)
//   P1  global inclusive scan of m (wrapping u64 adds) -> P; block sums
//   P2  path hash H_i = P_i - P_{start(s)-1} (exact in Z/2^64); insert H_i
//       into an open-addressing table, atomicMin(index) -> first occurrence
//   P3  rep_i = table[H_i]; verify by induction over depth:
//         tok/pos/depth(rep_i) == tok/pos/depth(i)  and
//         depth == 0  or  rep_{i-1} == rep_{rep_i - 1}
//       which proves path(rep_i) == path(i) for every i (so the hash
//       partition equals the trie partition); any failure re-runs the whole
//       build with a new seed on the GPU.  lcp_s = min{depth : rep_i == i}.
//   P4  cu_q = exclusive scan of (L_s - lcp_s); N' = cu_q[B]
//   P5  scatter[i] = cu_q[s_r] + depth - lcp_{s_r} (r = rep_i);
//       gather[cid] = i and compact_positions[cid] = pos[i] for representatives.
#include <climits>
#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace rdx {
namespace {

constexpr int kPlanThreads = 512;
constexpr int kPlanWarps = kPlanThreads / 32;
constexpr int kMaxAttempts = 4;
constexpr int kTokensPerBlockTarget = 512;
constexpr int64_t kSingleCtaTokens = 1024;  // up to here one CTA beats a cooperative grid (launch + grid barriers)
// Up to here the grid is ONE thread-block cluster (<= 16 CTAs on one GPC): the phase
// barriers are hardware cluster barriers (barrier.cluster, release/acquire at cluster
// scope, which orders the global-memory phases too) instead of cooperative grid syncs,
// which cost microseconds each.  Beyond it: the cooperative grid (512 tokens per CTA).
constexpr int64_t kClusterTokens = 65536;

enum PlanMode { kSingle = 0, kCluster = 1, kGrid = 2 };
// cu is staged in shared memory (per CTA) when it has at most this many entries: the
// per-token sequence lookups (binary search, starts) then cost no L2 round trips.
constexpr int64_t kSmemCu = 4096;

__device__ __forceinline__ uint64_t fmix64(uint64_t k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdULL;
  k ^= k >> 33;
  k *= 0xc4ceb9fe1a85ec53ULL;
  k ^= k >> 33;
  return k;
}

__device__ __forceinline__ uint64_t token_element(uint32_t tok, uint32_t pos, uint32_t depth,
                                                  uint64_t seed) {
  const uint64_t key = (static_cast<uint64_t>(pos) << 32) | tok;
  return fmix64(fmix64(key ^ seed) + static_cast<uint64_t>(depth) * 0x9E3779B97F4A7C15ULL +
                (seed >> 7));
}

// last s with cu[s] <= i (skips empty sequences)
__device__ __forceinline__ uint32_t find_seq(const int64_t* __restrict__ cu, int64_t nseq, int64_t i) {
  int64_t lo = 0, hi = nseq;  // answer in [0, nseq-1]
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (cu[mid] <= i) lo = mid; else hi = mid;
  }
  return static_cast<uint32_t>(lo);
}

struct PlanScratch {
  uint64_t* P;          // [N]
  uint32_t* seg;        // [N]
  uint32_t* rep;        // [N]
  uint32_t* slot;       // [N]
  uint64_t* keys;       // [T]
  uint32_t* vals;       // [T]
  uint64_t* block_sums; // [max_grid]
  int32_t* lcp;         // [B]
  uint32_t* flags;      // [kMaxAttempts + 4]: per-attempt failure, validation bits
  uint64_t table_mask;
};

struct PlanArgs {
  const uint32_t* tok;
  const uint32_t* pos;
  const int64_t* cu;
  int64_t nseq;
  int64_t n;
  uint32_t flags;
  uint32_t* gather;
  uint32_t* scatter;
  uint32_t* cpos;
  int32_t* cu_q;
  int32_t* lcp_out;
  uint32_t* info;
};

// u64 block-wide exclusive scan of one value per thread; returns the exclusive
// prefix and writes the block total.
__device__ uint64_t block_exclusive_scan_u64(uint64_t v, uint64_t* warp_tot, uint64_t& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint64_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[warp] = x;
  __syncthreads();
  if (warp == 0) {
    uint64_t t = lane < kPlanWarps ? warp_tot[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    if (lane < kPlanWarps) warp_tot[lane] = t;  // inclusive warp prefix
  }
  __syncthreads();
  const uint64_t warp_prefix = warp == 0 ? 0 : warp_tot[warp - 1];
  total = warp_tot[kPlanWarps - 1];
  __syncthreads();
  return warp_prefix + x - v;
}

__device__ uint64_t block_sum_u64(uint64_t v, uint64_t* warp_tot) {
  uint64_t total;
  block_exclusive_scan_u64(v, warp_tot, total);
  return total;
}

// kSingle = one CTA (small batches): phases are separated by __syncthreads and
// the launch is an ordinary one; kCluster = the grid is one cluster (cluster
// barriers); kGrid = cooperative launch (grid barriers).
template <int MODE>
__global__ void __launch_bounds__(kPlanThreads)
plan_build_kernel(PlanArgs a, PlanScratch s) {
  struct Sync {
    __device__ void sync() {
      if constexpr (MODE == kSingle) {
        __syncthreads();
      } else if constexpr (MODE == kCluster) {
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
      } else {
        cg::this_grid().sync();
      }
    }
  } grid;
  __shared__ uint64_t warp_tot[kPlanWarps];
  __shared__ uint32_t s_vmax;
  if (threadIdx.x == 0) s_vmax = 0;

  const int64_t n = a.n;
  const int64_t nseq = a.nseq;
  const int64_t nthreads = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t gtid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
  const int64_t c_lo = min(n, chunk * blockIdx.x);
  const int64_t c_hi = min(n, c_lo + chunk);
  const uint64_t tmask = s.table_mask;
  const uint32_t* __restrict__ tok = a.tok;
  const uint32_t* __restrict__ pos = a.pos;
  extern __shared__ int64_t s_cu[];  // [nseq + 1] when staged (dynamic smem sized by the launch)
  const int64_t* __restrict__ cu = a.cu;
  if (nseq + 1 <= kSmemCu) {
    for (int64_t q = threadIdx.x; q <= nseq; q += blockDim.x) s_cu[q] = a.cu[q];
    __syncthreads();
    cu = s_cu;
  }

  // ---- validation of cu (device-side mirror of ragged.validate_batch) ----
  // bit0 start!=0, bit1 decrease, bit2 empty, bit3 end!=n.  With cu staged in shared
  // memory every block checks all of it itself (no grid barrier); otherwise the blocks
  // split the check and meet at two grid barriers.  The attempt flags are cleared here
  // and first set in P3, three grid barriers later.
  const bool staged = nseq + 1 <= kSmemCu;
  if (!staged && gtid == 0) s.flags[kMaxAttempts] = 0;
  if (gtid == 0)
    for (int t = 0; t < kMaxAttempts; ++t) s.flags[t] = 0;
  if (!staged) grid.sync();
  {
    __shared__ uint32_t s_bits;
    if (threadIdx.x == 0) s_bits = 0;
    __syncthreads();
    uint32_t bits = 0;
    if (staged ? threadIdx.x == 0 : gtid == 0) {
      if (cu[0] != 0) bits |= 1u;
      if (cu[nseq] != n) bits |= 8u;
    }
    const int64_t q0 = staged ? threadIdx.x : gtid, qs = staged ? static_cast<int64_t>(blockDim.x) : nthreads;
    for (int64_t q = q0; q < nseq; q += qs) {
      const int64_t d = cu[q + 1] - cu[q];
      if (d < 0) bits |= 2u;
      if (d == 0 && !(a.flags & RDX_PLAN_ALLOW_EMPTY)) bits |= 4u;
    }
    bits = __reduce_or_sync(0xffffffffu, bits);
    if (bits && (threadIdx.x & 31) == 0) atomicOr(staged ? &s_bits : &s.flags[kMaxAttempts], bits);
    if (staged) __syncthreads();
    else grid.sync();
    bits = staged ? s_bits : *((volatile uint32_t*)&s.flags[kMaxAttempts]);
    if (bits) {
      if (gtid == 0) {
        uint32_t st = (bits & 1u) ? RDX_ERR_BOUNDARY_MISMATCH
                      : (bits & 2u) ? RDX_ERR_NON_MONOTONE_OFFSETS
                      : (bits & 4u) ? RDX_ERR_NON_MONOTONE_OFFSETS
                                    : RDX_ERR_BOUNDARY_MISMATCH;
        a.info[0] = 0;
        a.info[1] = st;
        a.info[2] = 0;
        a.info[3] = 0;
      }
      return;  // uniform across the grid
    }
  }

  for (int attempt = 0; attempt < kMaxAttempts; ++attempt) {
    const uint64_t seed = 0x243F6A8885A308D3ULL * static_cast<uint64_t>(2 * attempt + 1) + 0x13198A2E03707344ULL;
    // ---- P0: clear table, seg ids, elements, block sums, lcp init ----
    for (uint64_t t = gtid; t <= tmask; t += nthreads) {
      s.keys[t] = 0;
      s.vals[t] = 0xFFFFFFFFu;
    }
    for (int64_t q = gtid; q < nseq; q += nthreads) s.lcp[q] = static_cast<int32_t>(cu[q + 1] - cu[q]);
    uint64_t local = 0;
    for (int64_t i = c_lo + threadIdx.x; i < c_hi; i += blockDim.x) {
      const uint32_t sq = find_seq(cu, nseq, i);
      const uint32_t depth = static_cast<uint32_t>(i - cu[sq]);
      const uint64_t m = token_element(tok[i], pos[i], depth, seed);
      s.seg[i] = sq;
      s.P[i] = m;
      local += m;
    }
    {
      const uint64_t tot = block_sum_u64(local, warp_tot);
      if (threadIdx.x == 0) s.block_sums[blockIdx.x] = tot;
    }
    grid.sync();

    // ---- P1: inclusive scan of P over the whole batch ----
    {
      uint64_t off_part = 0;
      for (int b = threadIdx.x; b < static_cast<int>(blockIdx.x); b += blockDim.x) off_part += s.block_sums[b];
      uint64_t carry = block_sum_u64(off_part, warp_tot);
      for (int64_t base = c_lo; base < c_hi; base += blockDim.x) {
        const int64_t i = base + threadIdx.x;
        const uint64_t v = i < c_hi ? s.P[i] : 0;
        uint64_t tile_total;
        const uint64_t ex = block_exclusive_scan_u64(v, warp_tot, tile_total);
        if (i < c_hi) s.P[i] = carry + ex + v;
        carry += tile_total;
      }
    }
    grid.sync();

    // ---- P2: path hashes into the first-occurrence table.  Only tokens whose path
    // differs from the same depth of the previous sequence are inserted (the first
    // occurrence of a path always is one); long shared prefixes then cost one insert
    // per node instead of B contending atomics, the other tokens look their key up in P3.
    auto Pm = [&](int64_t x) -> uint64_t { return x < 0 ? 0ULL : s.P[x]; };
    for (int64_t i = gtid; i < n; i += nthreads) {
      const uint32_t sq = s.seg[i];
      const int64_t st = cu[sq];
      const uint64_t h = s.P[i] - Pm(st - 1);
      bool insert = true;
      if (sq > 0) {
        const int64_t pst = cu[sq - 1];
        if (i - st < st - pst) insert = (Pm(pst + (i - st)) - Pm(pst - 1)) != h;
      }
      uint32_t slot = 0xFFFFFFFFu;
      if (insert) {
        uint64_t key = fmix64(h ^ seed);
        if (key == 0) key = 1;
        uint64_t t = key & tmask;
        while (true) {
          const unsigned long long prev =
              atomicCAS(reinterpret_cast<unsigned long long*>(&s.keys[t]), 0ULL,
                        static_cast<unsigned long long>(key));
          if (prev == 0ULL || prev == key) break;
          t = (t + 1) & tmask;
        }
        atomicMin(&s.vals[t], static_cast<uint32_t>(i));
        slot = static_cast<uint32_t>(t);
      }
      s.slot[i] = slot;
    }
    grid.sync();

    // ---- P3: representatives (lookups for non-inserted tokens) + inductive verification
    // (rep is a function of the key, so rep(i-1) == rep(rep_i - 1) <=> H_{i-1} == H_{rep_i - 1})
    // + lcp (warp-aggregated atomicMin: one per sequence run of a warp) ----
    {
      uint32_t fail = 0;
      for (int64_t i0 = gtid - (threadIdx.x & 31); i0 < n; i0 += nthreads) {  // warp-uniform trip count
        const int64_t i = i0 + (threadIdx.x & 31);
        const bool live = i < n;
        uint32_t si = 0xFFFFFFFFu;
        int32_t mine = INT_MAX;
        if (live) {
          si = s.seg[i];
          const int64_t st = cu[si];
          const int64_t di = i - st;
          const uint64_t pst1 = Pm(st - 1);
          uint64_t t = s.slot[i];
          bool lost = false;
          if (t == 0xFFFFFFFFu) {
            uint64_t key = fmix64((s.P[i] - pst1) ^ seed);
            if (key == 0) key = 1;
            t = key & tmask;
            while (true) {
              const uint64_t k = s.keys[t];
              if (k == key) break;
              if (k == 0ULL) {  // unreachable unless hashes collided: new seed
                lost = true;
                break;
              }
              t = (t + 1) & tmask;
            }
          }
          const uint32_t r = lost ? static_cast<uint32_t>(i) : s.vals[t];
          s.rep[i] = r;
          if (lost) fail = 1;
          if (r == static_cast<uint32_t>(i)) {
            mine = static_cast<int32_t>(di);
          } else {
            const uint32_t sr = s.seg[r];
            const int64_t sst = cu[sr];
            bool ok = (tok[r] == tok[i]) && (pos[r] == pos[i]) && (static_cast<int64_t>(r) - sst == di);
            if (ok && di > 0) ok = (s.P[i - 1] - pst1) == (s.P[r - 1] - Pm(sst - 1));
            if (!ok) fail = 1;
          }
        }
        const unsigned grp = __match_any_sync(0xffffffffu, si);
        const int32_t mn = __reduce_min_sync(grp, mine);
        if (live && mn != INT_MAX && static_cast<int>(threadIdx.x & 31) == __ffs(grp) - 1)
          atomicMin(&s.lcp[si], mn);
      }
      if (__syncthreads_or(fail) && threadIdx.x == 0) atomicOr(&s.flags[attempt], 1u);
    }
    grid.sync();
    if (*((volatile uint32_t*)&s.flags[attempt]) != 0) continue;  // re-run with a new seed

    // ---- P4: cu_q.  Few sequences (cu staged, <= 1024): every block scans them into its
    // own shared copy (no grid barrier before P5); else block 0 alone, then a barrier ----
    const bool local_cuq = staged && nseq <= 1024;
    int32_t* s_cuq = reinterpret_cast<int32_t*>(s_cu + nseq + 1);  // staged layout only
    if (local_cuq || blockIdx.x == 0) {
      uint64_t carry = 0;
      uint32_t vmax = 0;  // longest compact suffix (info[3] = max_q)
      for (int64_t base = 0; base < nseq; base += blockDim.x) {
        const int64_t q = base + threadIdx.x;
        const int32_t lq = q < nseq ? s.lcp[q] : 0;
        const uint64_t v = q < nseq ? static_cast<uint64_t>(cu[q + 1] - cu[q] - lq) : 0;
        vmax = max(vmax, static_cast<uint32_t>(v));
        uint64_t tile_total;
        const uint64_t ex = block_exclusive_scan_u64(v, warp_tot, tile_total);
        if (q < nseq) {
          if (local_cuq) s_cuq[q] = static_cast<int32_t>(carry + ex);
          if (blockIdx.x == 0) {
            a.cu_q[q] = static_cast<int32_t>(carry + ex);
            if (a.lcp_out) a.lcp_out[q] = lq;
          }
        }
        carry += tile_total;
      }
      if (local_cuq && threadIdx.x == 0) s_cuq[nseq] = static_cast<int32_t>(carry);
      if (blockIdx.x != 0) {
        __syncthreads();  // s_cuq complete
      } else {
        vmax = __reduce_max_sync(0xffffffffu, vmax);
        if ((threadIdx.x & 31) == 0) atomicMax(&s_vmax, vmax);
        __syncthreads();
        if (threadIdx.x == 0) {
          a.cu_q[nseq] = static_cast<int32_t>(carry);
          a.info[0] = static_cast<uint32_t>(carry);
          a.info[1] = RDX_OK;
          a.info[2] = static_cast<uint32_t>(attempt + 1);
          a.info[3] = s_vmax;
        }
      }
    }
    if (!local_cuq) grid.sync();

    // ---- P5: emit ----
    for (int64_t i = gtid; i < n; i += nthreads) {
      const uint32_t r = s.rep[i];
      const uint32_t si = s.seg[i];
      const int64_t depth = i - cu[si];
      const uint32_t sr = (r == static_cast<uint32_t>(i)) ? si : s.seg[r];
      const uint32_t cid = static_cast<uint32_t>((local_cuq ? s_cuq[sr] : a.cu_q[sr]) + depth - s.lcp[sr]);
      a.scatter[i] = cid;
      if (r == static_cast<uint32_t>(i)) {
        a.gather[cid] = static_cast<uint32_t>(i);
        a.cpos[cid] = pos[i];
      }
    }
    return;
  }
  if (gtid == 0) {
    a.info[0] = 0;
    a.info[1] = RDX_ERR_HASH_RETRIES;
    a.info[2] = kMaxAttempts;
    a.info[3] = 0;
  }
}

// ---------------------------------------------------------------- cluster-resident planner
// Batches up to kSmMaxCtas * kSmChunkMax tokens (and a staged cu) run as ONE
// thread-block cluster whose whole working set lives in shared memory: each CTA
// owns a contiguous chunk of tokens (tok, pos, seg, path prefix P, slot) and a
// slice of the open-addressing table; the cross-token lookups (P at a sequence
// start and at rep-1, the table itself) are distributed-shared-memory accesses
// (~200 cycles) instead of L2 round trips (the representative's tok/pos are read
// from global memory: a shared prefix's representatives all sit in one CTA), and
// the phases are separated by 4 hardware cluster barriers (the cooperative grid
// version has 4-7 grid barriers and L2 traffic in every phase).  A hash slot is
// one 64-bit word: 48-bit key tag over the 16-bit index of the path's first token.
// Same algorithm and outputs as plan_build_kernel.
constexpr int kSmThreads = 1024;
constexpr int kSmWarps = kSmThreads / 32;
constexpr int kSmPerThread = 4;                               // tokens per thread at most
constexpr int64_t kSmChunkMax = kSmThreads * kSmPerThread;   // tokens per CTA
constexpr int kSmMaxCtas = 16;
constexpr size_t kSmBudget = 227 * 1024 - 2048;               // dynamic smem (static: ~1 KB)

struct SmGeom {
  int64_t chunk;   // tokens per CTA
  int64_t tslots;  // hash slots per CTA
  int64_t tsize;   // tslots * cluster size
  uint32_t off_P, off_slot, off_seg, off_tok, off_pos, off_keys, off_lcp, off_cuq;
  uint32_t bytes;
  unsigned long long* trace;  // debug (rdx_plan_debug_trace): phase timestamps of CTA 0, start of every CTA
};

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Phase barrier of the cluster planner; the one-CTA instance (batches <= 1024 tokens)
// only needs its block barrier.
template <bool kOne>
__device__ __forceinline__ void cl_sync() {
  if constexpr (kOne) {
    __syncthreads();
  } else {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
}

template <int NW>
__device__ uint64_t block_exclusive_scan_u64_w(uint64_t v, uint64_t* warp_tot, uint64_t& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint64_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[warp] = x;
  __syncthreads();
  if (warp == 0) {
    uint64_t t = lane < NW ? warp_tot[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    if (lane < NW) warp_tot[lane] = t;
  }
  __syncthreads();
  const uint64_t warp_prefix = warp == 0 ? 0 : warp_tot[warp - 1];
  total = warp_tot[NW - 1];
  __syncthreads();
  return warp_prefix + x - v;
}

// kOne: the single-CTA instance, every access local (no DSMEM mapping, block barriers).
template <bool kOne>
__global__ void __launch_bounds__(kSmThreads, 1) plan_build_smem_kernel(PlanArgs a, SmGeom g) {
  cg::cluster_group cl = cg::this_cluster();
  const int C = static_cast<int>(cl.num_blocks());
  const int me = static_cast<int>(cl.block_rank());
  extern __shared__ __align__(16) uint8_t sm[];
  int64_t* s_cu = reinterpret_cast<int64_t*>(sm);
  uint64_t* s_P = reinterpret_cast<uint64_t*>(sm + g.off_P);
  uint32_t* s_slot = reinterpret_cast<uint32_t*>(sm + g.off_slot);
  uint32_t* s_seg = reinterpret_cast<uint32_t*>(sm + g.off_seg);
  uint32_t* s_tok = reinterpret_cast<uint32_t*>(sm + g.off_tok);
  uint32_t* s_pos = reinterpret_cast<uint32_t*>(sm + g.off_pos);
  unsigned long long* s_keys = reinterpret_cast<unsigned long long*>(sm + g.off_keys);
  int32_t* s_lcp = reinterpret_cast<int32_t*>(sm + g.off_lcp);
  int32_t* s_cuq = reinterpret_cast<int32_t*>(sm + g.off_cuq);
  __shared__ uint64_t s_wtot[kSmWarps];
  __shared__ uint64_t s_carry[kSmMaxCtas];
  __shared__ uint64_t s_total;
  __shared__ uint32_t s_flags[kMaxAttempts + 1];  // [0] validation bits, [1 + t] attempt t failed (CTA 0's copy counts)
  __shared__ uint32_t s_vmax;

  const int tid = threadIdx.x;
  auto mark = [&](int k) {
    if (g.trace && me == 0 && tid == 0) g.trace[k] = globaltimer_ns();
  };
  if (g.trace && tid == 0) g.trace[16 + me] = globaltimer_ns();
  mark(0);
  const int64_t n = a.n, nseq = a.nseq, chunk = g.chunk;
  const int64_t lo = min(n, static_cast<int64_t>(me) * chunk);
  const int64_t cnt = min(n, lo + chunk) - lo;
  auto owner_of = [&](int64_t x) { return static_cast<int>(x / chunk); };

  // ---- stage cu, tok, pos; validate cu (sequences spread over the cluster) ----
  for (int64_t q = tid; q <= nseq; q += kSmThreads) s_cu[q] = a.cu[q];
  for (int64_t j = tid; j < cnt; j += kSmThreads) {
    s_tok[j] = a.tok[lo + j];
    s_pos[j] = a.pos[lo + j];
  }
  if (tid <= kMaxAttempts) s_flags[tid] = 0;
  if (tid == 0) s_vmax = 0;
  __syncthreads();
  {
    // every CTA validates the whole staged cu itself (<= 8192 entries): no shared-memory
    // traffic between CTAs before the first cluster barrier
    uint32_t bits = 0;  // bit0 start!=0, bit1 decrease, bit2 empty, bit3 end!=n
    if (tid == 0) {
      if (s_cu[0] != 0) bits |= 1u;
      if (s_cu[nseq] != n) bits |= 8u;
    }
    for (int64_t q = tid; q < nseq; q += kSmThreads) {
      const int64_t d = s_cu[q + 1] - s_cu[q];
      if (d < 0) bits |= 2u;
      if (d == 0 && !(a.flags & RDX_PLAN_ALLOW_EMPTY)) bits |= 4u;
    }
    bits = __reduce_or_sync(0xffffffffu, bits);
    if (bits && (tid & 31) == 0) atomicOr(&s_flags[0], bits);
  }
  if (me == 0)
    for (int64_t q = tid; q < nseq; q += kSmThreads) s_lcp[q] = static_cast<int32_t>(s_cu[q + 1] - s_cu[q]);
  // independent of the other CTAs, so done before B1: the first attempt's table clear and
  // the sequence of each own token (a contiguous run per thread, found once; garbage
  // but bounded when cu is invalid, in which case the kernel leaves after B1)
  for (int64_t t = tid; t < g.tslots; t += kSmThreads) s_keys[t] = 0ULL;
  const int per = static_cast<int>((cnt + kSmThreads - 1) / kSmThreads);
  const int64_t j0 = static_cast<int64_t>(tid) * per;
  if (j0 < cnt) {
    uint32_t sq = find_seq(s_cu, nseq, lo + j0);
    for (int u = 0; u < per && j0 + u < cnt; ++u) {
      const int64_t i = lo + j0 + u;
      while (sq + 1 < nseq && s_cu[sq + 1] <= i) ++sq;
      s_seg[j0 + u] = sq;
    }
  }
  mark(1);
  cl_sync<kOne>();  // B1
  mark(2);
  {
    const uint32_t bits = s_flags[0];  // this CTA's own verdict on the whole cu
    if (bits) {
      if (me == 0 && tid == 0) {
        a.info[0] = 0;
        a.info[1] = (bits & 1u) ? RDX_ERR_BOUNDARY_MISMATCH
                    : (bits & 6u) ? RDX_ERR_NON_MONOTONE_OFFSETS
                                  : RDX_ERR_BOUNDARY_MISMATCH;
        a.info[2] = 0;
        a.info[3] = 0;
      }
      cl_sync<kOne>();  // nobody leaves while another CTA may still use this one's shared memory
      return;
    }
  }
  for (int attempt = 0; attempt < kMaxAttempts; ++attempt) {
    const uint64_t seed = 0x243F6A8885A308D3ULL * static_cast<uint64_t>(2 * attempt + 1) + 0x13198A2E03707344ULL;
    // ---- P0: clear the table slice (retries); per-token elements; chunk-local inclusive scan ----
    if (attempt > 0)
      for (int64_t t = tid; t < g.tslots; t += kSmThreads) s_keys[t] = 0ULL;
    if (me == 0 && attempt > 0)
      for (int64_t q = tid; q < nseq; q += kSmThreads) s_lcp[q] = static_cast<int32_t>(s_cu[q + 1] - s_cu[q]);
    {
      uint64_t m[kSmPerThread];
      uint64_t sum = 0;
#pragma unroll
      for (int u = 0; u < kSmPerThread; ++u) {
        m[u] = 0;
        const int64_t j = j0 + u;
        if (u < per && j < cnt) {
          const uint32_t sq = s_seg[j];
          m[u] = token_element(s_tok[j], s_pos[j], static_cast<uint32_t>(lo + j - s_cu[sq]), seed);
          sum += m[u];
        }
      }
      uint64_t tot;
      uint64_t run = block_exclusive_scan_u64_w<kSmWarps>(sum, s_wtot, tot);
#pragma unroll
      for (int u = 0; u < kSmPerThread; ++u) {
        const int64_t j = j0 + u;
        if (u < per && j < cnt) {
          run += m[u];
          s_P[j] = run;
        }
      }
      if (tid == 0) s_total = tot;
    }
    mark(3);
    cl_sync<kOne>();  // B2: chunk prefixes and totals visible, tables clear
    mark(4);
    if (tid < C) s_carry[tid] = kOne ? s_total : *cl.map_shared_rank(&s_total, tid);
    __syncthreads();
    if (tid == 0) {
      uint64_t acc = 0;
      for (int c = 0; c < C; ++c) {
        const uint64_t t = s_carry[c];
        s_carry[c] = acc;
        acc += t;
      }
    }
    __syncthreads();

    // Path prefix P at any token x (own chunk or remote) and the path hash of token x
    // in sequence q: H = P_x - P_{cu[q]-1} (exact in Z/2^64).  Indices fit 32 bits.
    auto P_at = [&](int64_t x) -> uint64_t {
      if (x < 0) return 0ULL;
      const uint32_t o = static_cast<uint32_t>(x) / static_cast<uint32_t>(chunk);
      const uint32_t lx = static_cast<uint32_t>(x) - o * static_cast<uint32_t>(chunk);
      return (kOne ? s_P[lx] : *cl.map_shared_rank(&s_P[lx], o)) + s_carry[o];
    };
    auto key_of = [&](uint64_t h) -> unsigned long long {
      const uint64_t k = fmix64(h ^ seed);
      return k == 0 ? 1ULL : k;
    };
    // A slot is one 64-bit word: the key's top 48 bits (nonzero) over the 16-bit index of
    // the path's first token (cluster batches have <= 65536 tokens).  Claiming an empty
    // slot is one CAS, a repeated key one 64-bit atomicMin (equal high bits: min index),
    // and a lookup one load.  Two paths sharing 48 key bits share a slot; the inductive
    // verification catches that like any other collision (retry with a new seed).
    auto tag_of = [&](unsigned long long key) -> unsigned long long {
      const unsigned long long k48 = key >> 16;
      return k48 == 0 ? 1ULL : k48;
    };
    const uint32_t tsl = static_cast<uint32_t>(g.tslots), tsz = static_cast<uint32_t>(g.tsize);
    auto home = [&](unsigned long long key) -> uint32_t { return static_cast<uint32_t>(__umul64hi(key, tsz)); };

    // ---- P2: insert only the tokens whose path differs from the same depth of the
    // previous sequence (the first occurrence of a path is always such a token: an
    // equal path one sequence earlier would be earlier still).  Reranking batches then
    // insert ~N' distinct keys and the shared prefix costs one insert, not B contending
    // atomics; every other token finds its key in P3 with plain loads. ----
    for (int64_t j = tid; j < cnt; j += kSmThreads) {
      const int64_t i = lo + j;
      const uint32_t sq = s_seg[j];
      const int64_t st = s_cu[sq];
      const uint64_t h = s_P[j] + s_carry[me] - P_at(st - 1);
      bool insert = true;
      if (sq > 0) {
        const int64_t pst = s_cu[sq - 1];
        if (i - st < st - pst) insert = (P_at(pst + (i - st)) - P_at(pst - 1)) != h;
      }
      uint32_t t = 0xFFFFFFFFu;
      if (insert) {
        const unsigned long long key = key_of(h), tag = tag_of(key);
        const unsigned long long word = (tag << 16) | static_cast<unsigned long long>(i);
        t = home(key);
        while (true) {
          const uint32_t o = t / tsl, lt = t - o * tsl;
          unsigned long long* slot = kOne ? &s_keys[lt] : cl.map_shared_rank(&s_keys[lt], o);
          const unsigned long long prev = atomicCAS(slot, 0ULL, word);
          if (prev == 0ULL) break;
          if ((prev >> 16) == tag) {
            // min index by CAS: a 64-bit atomicMin through the cluster-mapped pointer gave
            // wrong minima here (tests/test_plan_gpu.py::test_multilevel_trie_vs_oracle)
            unsigned long long cur = prev;
            while (word < cur) {
              const unsigned long long got = atomicCAS(slot, cur, word);
              if (got == cur) break;
              cur = got;
            }
            break;
          }
          t = t + 1 == tsz ? 0 : t + 1;
        }
      }
      s_slot[j] = t;
    }
    mark(5);
    if (g.trace && tid == 0 && me < 16) g.trace[32 + me] = globaltimer_ns();  // this CTA's P2 end
    cl_sync<kOne>();  // B3: table final
    mark(6);
    auto slot_at = [&](uint32_t t) -> unsigned long long {
      const uint32_t o = t / tsl;
      return kOne ? s_keys[t] : *cl.map_shared_rank(&s_keys[t - o * tsl], o);
    };

    // ---- P3: representatives (table lookups), inductive verification, lcp ----
    // rep(x) is a function of x's key (one slot per key, one first index per slot), so
    // the inductive condition rep(i-1) == rep(rep_i - 1) is H_{i-1} == H_{rep_i - 1}.
    uint32_t rr[kSmPerThread], srr[kSmPerThread];
    uint32_t fail = 0;
#pragma unroll
    for (int u = 0; u < kSmPerThread; ++u) {
      const int64_t j = tid + static_cast<int64_t>(u) * kSmThreads;
      const bool live = j < cnt;
      const int64_t i = lo + j;
      uint32_t si = 0xFFFFFFFFu, r = 0, sr = 0;
      int32_t mine = INT_MAX;
      if (live) {
        si = s_seg[j];
        const int64_t st = s_cu[si];
        const int64_t di = i - st;
        const uint64_t pst1 = P_at(st - 1);
        uint32_t t = s_slot[j];
        bool lost = false;
        unsigned long long w;
        if (t != 0xFFFFFFFFu) {
          w = slot_at(t);
        } else {  // not inserted: find the key
          const unsigned long long key = key_of(s_P[j] + s_carry[me] - pst1), tag = tag_of(key);
          t = home(key);
          while (true) {
            w = slot_at(t);
            if ((w >> 16) == tag) break;
            if (w == 0ULL) {  // cannot happen unless hashes collided: retry with a new seed
              lost = true;
              break;
            }
            t = t + 1 == tsz ? 0 : t + 1;
          }
        }
        if (lost) fail = 1;
        r = lost ? static_cast<uint32_t>(i) : static_cast<uint32_t>(w & 0xFFFFu);
        sr = si;
        if (r == static_cast<uint32_t>(i)) {
          mine = static_cast<int32_t>(di);
        } else {
          // a representative in another CTA: its sequence from this CTA's copy of cu, its
          // token and position from global memory (L1/L2) -- the representatives of a shared
          // prefix all live in one CTA, whose shared memory would otherwise serve every such
          // lookup (C2 18.3 -> 17.4 us, C3 36.0 -> 34.3 us per launch)
          uint32_t rtok, rpos;
          if constexpr (kOne) {  // one CTA: plain shared-memory loads
            sr = s_seg[r];
            rtok = s_tok[r];
            rpos = s_pos[r];
          } else {
            sr = find_seq(s_cu, nseq, r);
            rtok = __ldg(a.tok + r);
            rpos = __ldg(a.pos + r);
          }
          const int64_t sst = s_cu[sr];
          bool ok = (rtok == s_tok[j]) && (rpos == s_pos[j]) &&
                    (static_cast<int64_t>(r) - sst == di);
          if (ok && di > 0) ok = (P_at(i - 1) - pst1) == (P_at(static_cast<int64_t>(r) - 1) - P_at(sst - 1));
          if (!ok) fail = 1;
        }
      }
      rr[u] = r;
      srr[u] = sr;
      // lcp_s = min depth of a token that is its own representative: reduced per warp
      // over the lanes of the same sequence, one remote atomicMin per group
      const unsigned grp = __match_any_sync(0xffffffffu, si);
      const int32_t mn = __reduce_min_sync(grp, mine);
      if (live && mn != INT_MAX && (threadIdx.x & 31) == __ffs(grp) - 1)
        atomicMin(kOne ? &s_lcp[si] : cl.map_shared_rank(&s_lcp[si], 0), mn);
    }
    if (__syncthreads_or(fail) && tid == 0) atomicOr(cl.map_shared_rank(&s_flags[1 + attempt], 0), 1u);
    mark(7);
    if (g.trace && tid == 0 && me < 16) g.trace[48 + me] = globaltimer_ns();  // this CTA's P3 end
    cl_sync<kOne>();  // B4: verification and lcp final
    mark(8);
    if (*reinterpret_cast<volatile uint32_t*>(cl.map_shared_rank(&s_flags[1 + attempt], 0)) != 0) continue;

    // ---- P4: every CTA copies lcp from CTA 0 and scans cu_q itself (no further barrier) ----
    if (me != 0)
      for (int64_t q = tid; q < nseq; q += kSmThreads) s_lcp[q] = *cl.map_shared_rank(&s_lcp[q], 0);
    __syncthreads();
    // done with every other CTA's shared memory: let them leave once P5 is done
    if constexpr (!kOne) asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    {
      uint64_t carry = 0;
      uint32_t vmax = 0;  // longest compact suffix (info[3] = max_q)
      for (int64_t base = 0; base < nseq; base += kSmThreads) {
        const int64_t q = base + tid;
        const uint64_t v = q < nseq ? static_cast<uint64_t>(s_cu[q + 1] - s_cu[q] - s_lcp[q]) : 0;
        vmax = max(vmax, static_cast<uint32_t>(v));
        uint64_t tile_total;
        const uint64_t ex = block_exclusive_scan_u64_w<kSmWarps>(v, s_wtot, tile_total);
        if (q < nseq) {
          s_cuq[q] = static_cast<int32_t>(carry + ex);
          if (me == 0) {
            a.cu_q[q] = static_cast<int32_t>(carry + ex);
            if (a.lcp_out) a.lcp_out[q] = s_lcp[q];
          }
        }
        carry += tile_total;
      }
      if (me == 0) {
        vmax = __reduce_max_sync(0xffffffffu, vmax);
        if ((tid & 31) == 0) atomicMax(&s_vmax, vmax);
        __syncthreads();
      }
      if (tid == 0) {
        s_cuq[nseq] = static_cast<int32_t>(carry);
        if (me == 0) {
          a.cu_q[nseq] = static_cast<int32_t>(carry);
          a.info[0] = static_cast<uint32_t>(carry);
          a.info[1] = RDX_OK;
          a.info[2] = static_cast<uint32_t>(attempt + 1);
          a.info[3] = s_vmax;
        }
      }
    }
    __syncthreads();
    mark(9);
    // ---- P5: emit (own tokens, representatives held in registers since P3) ----
#pragma unroll
    for (int u = 0; u < kSmPerThread; ++u) {
      const int64_t j = tid + static_cast<int64_t>(u) * kSmThreads;
      if (j >= cnt) continue;
      const int64_t i = lo + j;
      const int64_t depth = i - s_cu[s_seg[j]];
      const uint32_t sr = srr[u];
      const uint32_t cid = static_cast<uint32_t>(s_cuq[sr] + depth - s_lcp[sr]);
      a.scatter[i] = cid;
      if (rr[u] == static_cast<uint32_t>(i)) {
        a.gather[cid] = static_cast<uint32_t>(i);
        a.cpos[cid] = s_pos[j];
      }
    }
    mark(10);
    if constexpr (!kOne) asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    mark(11);
    return;
  }
  if (me == 0 && tid == 0) {
    a.info[0] = 0;
    a.info[1] = RDX_ERR_HASH_RETRIES;
    a.info[2] = kMaxAttempts;
    a.info[3] = 0;
  }
  cl_sync<kOne>();
}

// Shared-memory geometry of the cluster planner for (n, nseq) on `ctas` CTAs; false
// when it does not fit (the cooperative grid kernel takes the batch).
bool sm_geometry(int64_t n, int64_t nseq, int ctas, SmGeom* g) {
  if (ctas < 1 || nseq + 1 > 8192 || n > 65536) return false;  // 16-bit token indices in the slots
  const int64_t chunk = (n + ctas - 1) / ctas;
  if (chunk > kSmChunkMax) return false;
  int64_t tslots = (2 * n + ctas - 1) / ctas;
  tslots = tslots < 2 ? 2 : tslots;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const uint32_t o = static_cast<uint32_t>(off);
    off = (off + bytes + 15) & ~static_cast<size_t>(15);
    return o;
  };
  take(8 * static_cast<size_t>(nseq + 1));  // cu at offset 0
  g->off_P = take(8 * static_cast<size_t>(chunk));
  g->off_keys = take(8 * static_cast<size_t>(tslots));
  g->off_slot = take(4 * static_cast<size_t>(chunk));
  g->off_seg = take(4 * static_cast<size_t>(chunk));
  g->off_tok = take(4 * static_cast<size_t>(chunk));
  g->off_pos = take(4 * static_cast<size_t>(chunk));
  g->off_lcp = take(4 * static_cast<size_t>(nseq > 0 ? nseq : 1));
  g->off_cuq = take(4 * static_cast<size_t>(nseq + 1));
  g->bytes = static_cast<uint32_t>(off);
  g->chunk = chunk;
  g->tslots = tslots;
  g->tsize = tslots * ctas;
  return off <= kSmBudget;
}

// Largest cluster the shared-memory planner can be launched as (16 non-portable, else 8).
int sm_cluster_max() {
  static int cached = -1;
  if (cached < 0) {
    cached = 0;
    auto kern = plan_build_smem_kernel<false>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSmBudget)) !=
            cudaSuccess ||
        cudaFuncSetAttribute(plan_build_smem_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(kSmBudget)) != cudaSuccess) {
      cudaGetLastError();
      return cached;
    }
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)
      cudaGetLastError();
    for (int c : {16, 8}) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(c);
      cfg.blockDim = dim3(kSmThreads);
      cfg.dynamicSmemBytes = kSmBudget;
      cudaLaunchAttribute attr;
      attr.id = cudaLaunchAttributeClusterDimension;
      attr.val.clusterDim.x = c;
      attr.val.clusterDim.y = 1;
      attr.val.clusterDim.z = 1;
      cfg.attrs = &attr;
      cfg.numAttrs = 1;
      int nclusters = 0;
      if (cudaOccupancyMaxActiveClusters(&nclusters, kern, &cfg) == cudaSuccess && nclusters > 0) {
        cached = c;
        break;
      }
      cudaGetLastError();
    }
  }
  return cached;
}

// RDX_PLAN_SMEM=0 (env) or rdx_plan_debug_smem(0): route every batch to the L2 planners (A/B, tests).
int g_plan_smem = -1;
unsigned long long* g_plan_trace = nullptr;  // debug: device buffer of >= 32 u64 (rdx_plan_debug_trace)
bool sm_planner_enabled() {
  if (g_plan_smem < 0) {
    const char* e = getenv("RDX_PLAN_SMEM");
    g_plan_smem = (e && e[0] == '0') ? 0 : 1;
  }
  return g_plan_smem == 1;
}

uint64_t table_size(int64_t n) {
  uint64_t t = 64;
  while (t < static_cast<uint64_t>(2 * n)) t <<= 1;
  return t;
}

int max_coop_blocks() {
  static int cached = 0;
  if (cached == 0) {
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, plan_build_kernel<kGrid>, kPlanThreads,
                                                      8 * kSmemCu) !=
        cudaSuccess)
      return 0;
    cached = per_sm * num_sms();
  }
  return cached;
}

// Largest cluster (16, non-portable, else 8) the planner can be launched as; 0 = none.
int cluster_ctas() {
  static int cached = -1;
  if (cached < 0) {
    cached = 0;
    auto kern = plan_build_kernel<kCluster>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
      cudaGetLastError();
    }
    for (int c : {16, 8}) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(c);
      cfg.blockDim = dim3(kPlanThreads);
      cfg.dynamicSmemBytes = 8 * kSmemCu;
      cudaLaunchAttribute attr;
      attr.id = cudaLaunchAttributeClusterDimension;
      attr.val.clusterDim.x = c;
      attr.val.clusterDim.y = 1;
      attr.val.clusterDim.z = 1;
      cfg.attrs = &attr;
      cfg.numAttrs = 1;
      int nclusters = 0;
      if (cudaOccupancyMaxActiveClusters(&nclusters, kern, &cfg) == cudaSuccess && nclusters > 0) {
        cached = c;
        break;
      }
      cudaGetLastError();
    }
  }
  return cached;
}

size_t align_up(size_t x) { return (x + 255) & ~static_cast<size_t>(255); }

size_t carve(int64_t n, int64_t nseq, int max_grid, PlanScratch* s, char* base) {
  const uint64_t t = table_size(n);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    char* p = base ? base + off : nullptr;
    off = align_up(off + bytes);
    return p;
  };
  PlanScratch tmp;
  tmp.P = reinterpret_cast<uint64_t*>(take(8 * static_cast<size_t>(n)));
  tmp.seg = reinterpret_cast<uint32_t*>(take(4 * static_cast<size_t>(n)));
  tmp.rep = reinterpret_cast<uint32_t*>(take(4 * static_cast<size_t>(n)));
  tmp.slot = reinterpret_cast<uint32_t*>(take(4 * static_cast<size_t>(n)));
  tmp.keys = reinterpret_cast<uint64_t*>(take(8 * t));
  tmp.vals = reinterpret_cast<uint32_t*>(take(4 * t));
  tmp.block_sums = reinterpret_cast<uint64_t*>(take(8 * static_cast<size_t>(max_grid)));
  tmp.lcp = reinterpret_cast<int32_t*>(take(4 * static_cast<size_t>(nseq > 0 ? nseq : 1)));
  tmp.flags = reinterpret_cast<uint32_t*>(take(4 * (kMaxAttempts + 4)));
  tmp.table_mask = t - 1;
  if (s) *s = tmp;
  return off;
}

}  // namespace
}  // namespace rdx

extern "C" size_t rdx_plan_scratch_bytes(int64_t n_tokens, int64_t n_seqs) {
  if (n_tokens < 0 || n_seqs < 0) return 0;
  int mg = rdx::max_coop_blocks();
  if (mg <= 0) mg = 4096;
  return rdx::carve(n_tokens, n_seqs, mg, nullptr, nullptr);
}

extern "C" int rdx_plan_build(const uint32_t* tok, const uint32_t* pos, const int64_t* cu,
                              int64_t n_seqs, int64_t n_tokens, uint32_t flags, uint32_t* gather_out,
                              uint32_t* scatter_out, uint32_t* cpos_out, int32_t* cu_q_out,
                              int32_t* lcp_out, uint32_t* info_out, void* scratch,
                              size_t scratch_bytes, void* stream) {
  using namespace rdx;
  if (n_tokens < 0 || n_seqs < 0) return RDX_ERR_INVALID_ARGUMENT;
  if (n_tokens >= (int64_t(1) << 32) - 1) return RDX_ERR_CAPACITY_EXCEEDED;
  if (!cu || !info_out || !cu_q_out) return RDX_ERR_INVALID_ARGUMENT;
  if (n_tokens > 0 && (!tok || !pos || !gather_out || !scatter_out || !cpos_out))
    return RDX_ERR_INVALID_ARGUMENT;
  const int mg = max_coop_blocks();
  if (mg <= 0) return set_cuda_error(cudaGetLastError());
  if (scratch_bytes < carve(n_tokens, n_seqs, mg, nullptr, nullptr) || !scratch)
    return RDX_ERR_INVALID_ARGUMENT;
  PlanScratch s;
  carve(n_tokens, n_seqs, mg, &s, static_cast<char*>(scratch));
  PlanArgs a{tok, pos, cu, n_seqs, n_tokens, flags, gather_out, scatter_out, cpos_out,
             cu_q_out, lcp_out, info_out};
  int64_t want = (n_tokens + kTokensPerBlockTarget - 1) / kTokensPerBlockTarget;
  if (want < 1) want = 1;
  const int grid = static_cast<int>(want < mg ? want : mg);
  void* params[] = {&a, &s};
  // staged cu (int64) + the per-block cu_q copy (int32) of the few-sequence P4 (<= 1024
  // sequences: at most 32 KB either way, under the 48 KB default)
  const size_t dsmem = n_seqs + 1 <= kSmemCu ? static_cast<size_t>((n_seqs <= 1024 ? 12 : 8) * (n_seqs + 1)) : 0;
  // up to 16 x 4096 tokens: the cluster-resident planner (everything in shared memory)
  if (sm_planner_enabled()) {
    const int cmax = sm_cluster_max();
    int ctas = 1;
    while (ctas < cmax && ctas * static_cast<int64_t>(kSmThreads) < n_tokens) ctas *= 2;
    SmGeom g;
    g.trace = g_plan_trace;
    if (cmax > 0 && sm_geometry(n_tokens, n_seqs, ctas, &g)) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(ctas);
      cfg.blockDim = dim3(kSmThreads);
      cfg.dynamicSmemBytes = g.bytes;
      cfg.stream = as_stream(stream);
      cudaLaunchAttribute attr;
      attr.id = cudaLaunchAttributeClusterDimension;
      attr.val.clusterDim.x = ctas;
      attr.val.clusterDim.y = 1;
      attr.val.clusterDim.z = 1;
      cfg.attrs = &attr;
      cfg.numAttrs = 1;
      RDX_CUDA_TRY(cudaLaunchKernelEx(&cfg, ctas == 1 ? plan_build_smem_kernel<true> : plan_build_smem_kernel<false>,
                                      a, g));
      return RDX_OK;
    }
  }
  if (n_tokens <= kSingleCtaTokens) {  // small batch: one CTA, no grid-wide barriers
    plan_build_kernel<kSingle><<<1, kPlanThreads, dsmem, as_stream(stream)>>>(a, s);
    RDX_LAUNCH_CHECK();
    return RDX_OK;
  }
  const int cl = cluster_ctas();
  if (n_tokens <= kClusterTokens && cl > 0) {  // mid-size batch: one cluster, hardware barriers
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cl);
    cfg.blockDim = dim3(kPlanThreads);
    cfg.dynamicSmemBytes = dsmem;
    cfg.stream = as_stream(stream);
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = cl;
    attr.val.clusterDim.y = 1;
    attr.val.clusterDim.z = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    RDX_CUDA_TRY(cudaLaunchKernelEx(&cfg, plan_build_kernel<kCluster>, a, s));
    return RDX_OK;
  }
  RDX_CUDA_TRY(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(plan_build_kernel<kGrid>), dim3(grid),
                                           dim3(kPlanThreads), params, dsmem, as_stream(stream)));
  return RDX_OK;
}

extern "C" int rdx_plan_debug_smem(int on) {
  const int prev = rdx::sm_planner_enabled() ? 1 : 0;
  rdx::g_plan_smem = on ? 1 : 0;
  return prev;
}

extern "C" int rdx_plan_debug_trace(void* buf) {
  rdx::g_plan_trace = static_cast<unsigned long long*>(buf);
  return 0;
}
