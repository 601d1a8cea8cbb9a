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
  // bit0 start!=0, bit1 decrease, bit2 empty, bit3 end!=n
  if (gtid == 0) {
    s.flags[kMaxAttempts] = 0;
    for (int t = 0; t < kMaxAttempts; ++t) s.flags[t] = 0;
  }
  grid.sync();
  {
    uint32_t bits = 0;
    if (gtid == 0) {
      if (cu[0] != 0) bits |= 1u;
      if (cu[nseq] != n) bits |= 8u;
    }
    for (int64_t q = gtid; q < nseq; q += nthreads) {
      const int64_t d = cu[q + 1] - cu[q];
      if (d < 0) bits |= 2u;
      if (d == 0 && !(a.flags & RDX_PLAN_ALLOW_EMPTY)) bits |= 4u;
    }
    if (bits) atomicOr(&s.flags[kMaxAttempts], bits);
  }
  grid.sync();
  {
    const uint32_t bits = *((volatile uint32_t*)&s.flags[kMaxAttempts]);
    if (bits) {
      if (gtid == 0) {
        uint32_t st = (bits & 1u) ? RDX_ERR_BOUNDARY_MISMATCH
                      : (bits & 2u) ? RDX_ERR_NON_MONOTONE_OFFSETS
                      : (bits & 4u) ? RDX_ERR_NON_MONOTONE_OFFSETS
                                    : RDX_ERR_BOUNDARY_MISMATCH;
        a.info[0] = 0;
        a.info[1] = st;
        a.info[2] = 0;
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

    // ---- P2: path hashes into the first-occurrence table ----
    for (int64_t i = gtid; i < n; i += nthreads) {
      const uint32_t sq = s.seg[i];
      const int64_t st = cu[sq];
      const uint64_t h = s.P[i] - (st > 0 ? s.P[st - 1] : 0ULL);
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
      s.slot[i] = static_cast<uint32_t>(t);
    }
    grid.sync();

    // ---- P3: representatives + inductive verification + lcp ----
    {
      uint32_t fail = 0;
      for (int64_t i = gtid; i < n; i += nthreads) {
        const uint32_t r = s.vals[s.slot[i]];
        s.rep[i] = r;
        const uint32_t si = s.seg[i];
        const int64_t di = i - cu[si];
        const uint32_t sr = s.seg[r];
        const int64_t dr = static_cast<int64_t>(r) - cu[sr];
        bool ok = (tok[r] == tok[i]) && (pos[r] == pos[i]) && (dr == di);
        if (ok && di > 0) ok = s.vals[s.slot[i - 1]] == s.vals[s.slot[r - 1]];
        if (!ok) fail = 1;
        if (r == static_cast<uint32_t>(i)) atomicMin(&s.lcp[si], static_cast<int32_t>(di));
      }
      if (__syncthreads_or(fail) && threadIdx.x == 0) atomicOr(&s.flags[attempt], 1u);
    }
    grid.sync();
    if (*((volatile uint32_t*)&s.flags[attempt]) != 0) continue;  // re-run with a new seed

    // ---- P4: cu_q (block 0) ----
    if (blockIdx.x == 0) {
      uint64_t carry = 0;
      for (int64_t base = 0; base < nseq; base += blockDim.x) {
        const int64_t q = base + threadIdx.x;
        const uint64_t v = q < nseq ? static_cast<uint64_t>(cu[q + 1] - cu[q] - s.lcp[q]) : 0;
        uint64_t tile_total;
        const uint64_t ex = block_exclusive_scan_u64(v, warp_tot, tile_total);
        if (q < nseq) {
          a.cu_q[q] = static_cast<int32_t>(carry + ex);
          if (a.lcp_out) a.lcp_out[q] = s.lcp[q];
        }
        carry += tile_total;
      }
      if (threadIdx.x == 0) {
        a.cu_q[nseq] = static_cast<int32_t>(carry);
        a.info[0] = static_cast<uint32_t>(carry);
        a.info[1] = RDX_OK;
        a.info[2] = static_cast<uint32_t>(attempt + 1);
      }
    }
    grid.sync();

    // ---- P5: emit ----
    for (int64_t i = gtid; i < n; i += nthreads) {
      const uint32_t r = s.rep[i];
      const uint32_t si = s.seg[i];
      const int64_t depth = i - cu[si];
      const uint32_t sr = (r == static_cast<uint32_t>(i)) ? si : s.seg[r];
      const uint32_t cid = static_cast<uint32_t>(a.cu_q[sr] + depth - s.lcp[sr]);
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
  }
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
  const size_t dsmem = n_seqs + 1 <= kSmemCu ? static_cast<size_t>(8 * (n_seqs + 1)) : 0;
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
