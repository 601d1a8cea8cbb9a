// rowops.cu — HBM-bound row kernels of the RadixMLP hot path:
//   rdx_gather_rows     gather/scatter of rows (ops.py:50-66), 16-byte vectors
//   rdx_embed_rmsnorm   compact embedding gather + layer-0 RMSNorm (model.py:329-349)
//   rdx_rmsnorm_rows    RMSNorm of (selected) fp32 rows (model.py:147-152)
//   rdx_rope_table      fp64 RoPE tables on compact positions (model.py:165-172)
//   rdx_rerank_scores   last-token reranker read-out (DESIGN.md scoring contract)
//   rdx_transpose_f32_bf16  fp32 [rows, cols] -> bf16 [cols, ld_dst] (zero-padded), the
//                       K-major operands of the tcgen05 dgrad / wgrad GEMMs (training.py)
#include <cstdlib>
#include "common.cuh"

namespace rdx {
namespace {

__device__ __forceinline__ void report(uint32_t* err, uint32_t code) {
  if (err) atomicCAS(err, 0u, code);
}


// One warp per output row; UNROLL independent vector loads in flight per lane.
template <typename V, int UNROLL>
__global__ void __launch_bounds__(256)
gather_rows_kernel(const char* __restrict__ src, int64_t src_rows, int64_t ld_src,
                   const uint32_t* __restrict__ idx, int64_t n_idx, char* __restrict__ dst,
                   int64_t ld_dst, int64_t row_vecs, uint32_t* err) {
  pdl_wait();  // no early trigger: a waiting dependent CTA would crowd out this grid's own blocks
  const int lane = threadIdx.x & 31;
  const int64_t warp0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t j = warp0; j < n_idx; j += nwarps) {
    const uint32_t r = __ldg(idx + j);
    V* d = reinterpret_cast<V*>(dst + j * ld_dst);
    if (static_cast<int64_t>(r) >= src_rows) {
      V z;
      memset(&z, 0, sizeof(V));
      for (int64_t c = lane; c < row_vecs; c += 32) d[c] = z;
      if (lane == 0) report(err, RDX_ERR_INDEX_OUT_OF_RANGE);
      continue;
    }
    const V* s = reinterpret_cast<const V*>(src + static_cast<int64_t>(r) * ld_src);
    for (int64_t c = lane; c < row_vecs; c += 32 * UNROLL) {
      V tmp[UNROLL];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u)
        if (c + u * 32 < row_vecs) tmp[u] = s[c + u * 32];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u)
        if (c + u * 32 < row_vecs) d[c + u * 32] = tmp[u];
    }
  }
}

__device__ __forceinline__ void bf16x8_to_f32(const int4 v, float (&f)[8]) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 t = __bfloat1622float2(h[i]);
    f[2 * i] = t.x;
    f[2 * i + 1] = t.y;
  }
}

// One warp per compact row; d % 8 == 0.
__global__ void __launch_bounds__(256)
embed_rmsnorm_kernel(const uint32_t* __restrict__ tok, const uint32_t* __restrict__ gather,
                     int64_t n_rows, const __nv_bfloat16* __restrict__ embed, int64_t vocab,
                     int64_t d, const float* __restrict__ w, float eps, float* __restrict__ h,
                     __nv_bfloat16* __restrict__ hn, uint32_t* err) {
  pdl_wait();  // no early trigger: a waiting dependent CTA would crowd out this grid's own blocks
  const int lane = threadIdx.x & 31;
  const int64_t warp0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t j = warp0; j < n_rows; j += nwarps) {
    const uint32_t src = gather ? __ldg(gather + j) : static_cast<uint32_t>(j);
    const uint32_t t = __ldg(tok + src);
    float* hrow = h + j * d;
    __nv_bfloat16* orow = hn + j * d;
    if (static_cast<int64_t>(t) >= vocab) {
      for (int64_t c = lane; c < d; c += 32) {
        hrow[c] = 0.f;
        orow[c] = __float2bfloat16(0.f);
      }
      if (lane == 0) report(err, RDX_ERR_INDEX_OUT_OF_RANGE);
      continue;
    }
    const int4* erow = reinterpret_cast<const int4*>(embed + static_cast<int64_t>(t) * d);
    float ss = 0.f;
    for (int64_t c = lane; c < d / 8; c += 32) {
      float f[8];
      bf16x8_to_f32(__ldg(erow + c), f);
#pragma unroll
      for (int i = 0; i < 8; ++i) ss += f[i] * f[i];
      float4* hp = reinterpret_cast<float4*>(hrow + c * 8);
      hp[0] = make_float4(f[0], f[1], f[2], f[3]);
      hp[1] = make_float4(f[4], f[5], f[6], f[7]);
    }
    ss = warp_sum(ss);
    const float inv = rsqrtf(ss / static_cast<float>(d) + eps);
    for (int64_t c = lane; c < d / 8; c += 32) {
      float f[8];
      bf16x8_to_f32(__ldg(erow + c), f);
      const float4* wp = reinterpret_cast<const float4*>(w + c * 8);
      const float4 w0 = __ldg(wp), w1 = __ldg(wp + 1);
      st_global_v4(orow + c * 8, pack_bf16x2(f[0] * inv * w0.x, f[1] * inv * w0.y),
                   pack_bf16x2(f[2] * inv * w0.z, f[3] * inv * w0.w),
                   pack_bf16x2(f[4] * inv * w1.x, f[5] * inv * w1.y),
                   pack_bf16x2(f[6] * inv * w1.z, f[7] * inv * w1.w));
    }
  }
}

// Compact embedding gather for the fused-norm layer stack: h (fp32), hb = bf16(h)
// (= the bf16 embedding row, exactly) and one partial sum of h^2 per 64 columns
// (8 lanes x 8 columns, fixed xor-tree order).  One warp per row; d % 64 == 0.
__global__ void __launch_bounds__(256)
embed_rows_kernel(const uint32_t* __restrict__ tok, const uint32_t* __restrict__ gather, int64_t n_rows,
                  const __nv_bfloat16* __restrict__ embed, int64_t vocab, int64_t d, float* __restrict__ h,
                  __nv_bfloat16* __restrict__ hb, float* __restrict__ ss_out, uint32_t* err) {
  pdl_wait();  // no early trigger: a waiting dependent CTA would crowd out this grid's own blocks
  const int lane = threadIdx.x & 31;
  const int64_t warp0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int64_t parts = d / 64;
  for (int64_t j = warp0; j < n_rows; j += nwarps) {
    const uint32_t src = gather ? __ldg(gather + j) : static_cast<uint32_t>(j);
    const uint32_t t = __ldg(tok + src);
    const bool bad = static_cast<int64_t>(t) >= vocab;
    if (bad && lane == 0) report(err, RDX_ERR_INDEX_OUT_OF_RANGE);
    float* hrow = h + j * d;
    int4* brow = reinterpret_cast<int4*>(hb + j * d);
    const int4* erow = reinterpret_cast<const int4*>(embed + static_cast<int64_t>(bad ? 0 : t) * d);
    for (int64_t c = lane; c < d / 8; c += 32) {  // d/8 is a multiple of 8: groups never straddle the loop
      const int4 raw = bad ? make_int4(0, 0, 0, 0) : __ldg(erow + c);
      float f[8];
      bf16x8_to_f32(raw, f);
      float s = 0.f;
#pragma unroll
      for (int i = 0; i < 8; ++i) s += f[i] * f[i];
      s += __shfl_xor_sync(0xffffffffu, s, 1);
      s += __shfl_xor_sync(0xffffffffu, s, 2);
      s += __shfl_xor_sync(0xffffffffu, s, 4);
      if ((lane & 7) == 0) ss_out[j * parts + c / 8] = s;
      float4* hp = reinterpret_cast<float4*>(hrow + c * 8);
      hp[0] = make_float4(f[0], f[1], f[2], f[3]);
      hp[1] = make_float4(f[4], f[5], f[6], f[7]);
      brow[c] = raw;
    }
  }
}

// One warp per selected row; d % 8 == 0.
__global__ void __launch_bounds__(256)
rmsnorm_rows_kernel(const float* __restrict__ x, int64_t ld_x, const uint32_t* __restrict__ rows,
                    int64_t n_rows, int64_t d, const float* __restrict__ w, float eps,
                    __nv_bfloat16* __restrict__ out, int64_t ld_out) {
  pdl_wait();  // no early trigger: a waiting dependent CTA would crowd out this grid's own blocks
  const int lane = threadIdx.x & 31;
  const int64_t warp0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t j = warp0; j < n_rows; j += nwarps) {
    const int64_t r = rows ? static_cast<int64_t>(__ldg(rows + j)) : j;
    const float4* xr = reinterpret_cast<const float4*>(x + r * ld_x);
    float ss = 0.f;
    for (int64_t c = lane; c < d / 4; c += 32) {
      const float4 v = xr[c];
      ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
    }
    ss = warp_sum(ss);
    const float inv = rsqrtf(ss / static_cast<float>(d) + eps);
    __nv_bfloat16* orow = out + j * ld_out;
    for (int64_t c = lane; c < d / 8; c += 32) {
      const float4 a = xr[2 * c], b = xr[2 * c + 1];
      const float4* wp = reinterpret_cast<const float4*>(w + c * 8);
      const float4 w0 = __ldg(wp), w1 = __ldg(wp + 1);
      st_global_v4(orow + c * 8, pack_bf16x2(a.x * inv * w0.x, a.y * inv * w0.y),
                   pack_bf16x2(a.z * inv * w0.z, a.w * inv * w0.w),
                   pack_bf16x2(b.x * inv * w1.x, b.y * inv * w1.y),
                   pack_bf16x2(b.z * inv * w1.z, b.w * inv * w1.w));
    }
  }
}

// Single pass: the row lives in registers (V float4 per lane, d = 128 * V), one
// HBM read and one write per element.
template <int V>
__global__ void __launch_bounds__(256)
rmsnorm_rows_reg_kernel(const float* __restrict__ x, int64_t ld_x, const uint32_t* __restrict__ rows,
                        int64_t n_rows, const float* __restrict__ w, float eps, __nv_bfloat16* __restrict__ out,
                        int64_t ld_out) {
  pdl_wait();  // no early trigger: a waiting dependent CTA would crowd out this grid's own blocks
  constexpr int D = 128 * V;
  const int lane = threadIdx.x & 31;
  const int64_t warp0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t j = warp0; j < n_rows; j += nwarps) {
    const int64_t r = rows ? static_cast<int64_t>(__ldg(rows + j)) : j;
    const float4* xr = reinterpret_cast<const float4*>(x + r * ld_x);
    float4 v[V];
    float ss = 0.f;
#pragma unroll
    for (int i = 0; i < V; ++i) {
      v[i] = __ldcs(xr + lane + 32 * i);
      ss += v[i].x * v[i].x + v[i].y * v[i].y + v[i].z * v[i].z + v[i].w * v[i].w;
    }
    ss = warp_sum(ss);
    const float inv = rsqrtf(ss / static_cast<float>(D) + eps);
    uint2* orow = reinterpret_cast<uint2*>(out + j * ld_out);
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const float4 g = __ldg(reinterpret_cast<const float4*>(w) + lane + 32 * i);
      orow[lane + 32 * i] = make_uint2(pack_bf16x2(v[i].x * inv * g.x, v[i].y * inv * g.y),
                                       pack_bf16x2(v[i].z * inv * g.z, v[i].w * inv * g.w));
    }
  }
}

// Same math with a two-row software pipeline: the grid is exactly resident (one
// wave) and each warp loads row j + stride while it reduces and writes row j, so
// a row's HBM latency overlaps the previous row's work instead of forming a
// second wave (d <= 2048).
template <int V>
__global__ void __launch_bounds__(256)
rmsnorm_rows_pipe_kernel(const float* __restrict__ x, int64_t ld_x, const uint32_t* __restrict__ rows,
                         int64_t n_rows, const float* __restrict__ w, float eps, __nv_bfloat16* __restrict__ out,
                         int64_t ld_out) {
  pdl_wait();
  constexpr int D = 128 * V;
  const int lane = threadIdx.x & 31;
  const int64_t warp0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  auto load = [&](int64_t j, float4 (&v)[V]) {
    const int64_t r = rows ? static_cast<int64_t>(__ldg(rows + j)) : j;
    const float4* xr = reinterpret_cast<const float4*>(x + r * ld_x);
#pragma unroll
    for (int i = 0; i < V; ++i) v[i] = __ldcs(xr + lane + 32 * i);
  };
  float4 cur[V], nxt[V];
  int64_t j = warp0;
  if (j < n_rows) load(j, cur);
  for (; j < n_rows; j += nwarps) {
    const bool more = j + nwarps < n_rows;
    if (more) load(j + nwarps, nxt);
    float ss = 0.f;
#pragma unroll
    for (int i = 0; i < V; ++i) ss += cur[i].x * cur[i].x + cur[i].y * cur[i].y + cur[i].z * cur[i].z + cur[i].w * cur[i].w;
    ss = warp_sum(ss);
    const float inv = rsqrtf(ss / static_cast<float>(D) + eps);
    uint2* orow = reinterpret_cast<uint2*>(out + j * ld_out);
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const float4 g = __ldg(reinterpret_cast<const float4*>(w) + lane + 32 * i);
      orow[lane + 32 * i] = make_uint2(pack_bf16x2(cur[i].x * inv * g.x, cur[i].y * inv * g.y),
                                       pack_bf16x2(cur[i].z * inv * g.z, cur[i].w * inv * g.w));
    }
    if (more) {
#pragma unroll
      for (int i = 0; i < V; ++i) cur[i] = nxt[i];
    }
  }
}

// rmsnorm of rows still being produced by the preceding residual GEMM (launched as
// its programmatic dependent, no griddepcontrol.wait): row j is read once its
// 32-row slab counter reaches `target` (acquire), in row order, so the blocks that
// land on SMs the GEMM's last round leaves idle work on the row blocks it has
// already finished.

#ifndef RDX_NORM_BACKOFF_MAX
#define RDX_NORM_BACKOFF_MAX 2048  // ns: the slab poller's longest nanosleep
#endif
__device__ unsigned g_norm_backoff_max = RDX_NORM_BACKOFF_MAX;  // rdx_norm_debug_backoff

// W warps per block, one row per warp per step.  ready_ctr != NULL (the chained mode):
// after each step the block publishes its W finished rows on ready_ctr[slab] (release),
// so a consumer GEMM launched as this kernel's programmatic dependent can stream A rows
// as they become ready; the launch trigger fires at entry so that consumer can launch
// (its CTAs start as the producing GEMM's CTAs exit).  The chained grid is one small
// block per SM whose registers fit beside a GEMM CTA (see rdx_rmsnorm_rows_after).
#ifdef RDX_NORM_STATS_BUILD
__device__ unsigned long long g_norm_times[2 * 4096];  // per block: %globaltimer at entry / exit
#endif

template <int V, int W>
__global__ void __launch_bounds__(W * 32)
rmsnorm_rows_after_kernel(const float* __restrict__ x, int64_t ld_x, int64_t n_rows, const float* __restrict__ w,
                          float eps, __nv_bfloat16* __restrict__ out, int64_t ld_out,
                          const uint32_t* __restrict__ done_ctr, uint32_t target, uint32_t* ready_ctr) {
  constexpr int D = 128 * V;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (ready_ctr) pdl_launch_dependents();
#ifdef RDX_NORM_STATS_BUILD
  unsigned long long t_in;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_in));
  if (threadIdx.x == 0 && blockIdx.x < 4096) g_norm_times[2 * blockIdx.x] = t_in;
#endif
  // A block takes W consecutive rows (one per warp) per step.  One thread polls
  // their slab counters (acquire, backing off) so waiting blocks add almost no L2
  // traffic.  No cross-step prefetch: a block must not wait on a later, unfinished
  // row block while it holds rows that are ready.
  for (int64_t base = static_cast<int64_t>(blockIdx.x) * W; base < n_rows; base += static_cast<int64_t>(gridDim.x) * W) {
    if (threadIdx.x == 0) {
      const int64_t last = base + W - 1 < n_rows ? base + W - 1 : n_rows - 1;
      for (int64_t slab = base >> 5; slab <= (last >> 5); ++slab) {
        unsigned ns = 128;
        const unsigned ns_max = g_norm_backoff_max;
        uint32_t spins = 0;
        while (ld_acquire_u32(done_ctr + slab) < target) {
          __nanosleep(ns);
          ns = ns < ns_max ? 2 * ns : ns;
          if (++spins > (1u << 22)) {  // ~8 s: the producing GEMM never completed this slab
            atomicCAS(&g_device_status, 0, static_cast<int>(RDX_ERR_DEVICE_TIMEOUT));  // reported by rdx_device_status
            break;
          }
        }
      }
    }
    __syncthreads();
    const int64_t j = base + warp;
    if (j < n_rows) {
      const float4* xr = reinterpret_cast<const float4*>(x + j * ld_x);
      float4 v[V];
      float ss = 0.f;
#pragma unroll
      for (int i = 0; i < V; ++i) {
        v[i] = __ldcg(xr + lane + 32 * i);
        ss += v[i].x * v[i].x + v[i].y * v[i].y + v[i].z * v[i].z + v[i].w * v[i].w;
      }
      ss = warp_sum(ss);
      const float inv = rsqrtf(ss / static_cast<float>(D) + eps);
      uint2* orow = reinterpret_cast<uint2*>(out + j * ld_out);
#pragma unroll
      for (int i = 0; i < V; ++i) {
        const float4 g = __ldg(reinterpret_cast<const float4*>(w) + lane + 32 * i);
        orow[lane + 32 * i] = make_uint2(pack_bf16x2(v[i].x * inv * g.x, v[i].y * inv * g.y),
                                         pack_bf16x2(v[i].z * inv * g.z, v[i].w * inv * g.w));
      }
    }
    if (ready_ctr) {
      __threadfence();  // this thread's row stores, visible at gpu scope before the publication
      __syncthreads();
      if (threadIdx.x == 0) {
        const int64_t rows = n_rows - base < W ? n_rows - base : W;
        atomicAdd(ready_ctr + (base >> 5), static_cast<uint32_t>(rows));
      }
    }
  }
#ifdef RDX_NORM_STATS_BUILD
  __syncthreads();
  if (threadIdx.x == 0 && blockIdx.x < 4096) {
    unsigned long long t_out;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_out));
    g_norm_times[2 * blockIdx.x + 1] = t_out;
  }
#endif
}

// blocked = 0: table[j][i]; blocked = 1: the QKV epilogue's lane-coalesced layout
// (see rdx_rope_table_blocked): float2 (j, i) at 2*(((j/32)*(half/2) + i/2)*32 + j%32) + i%2.
__global__ void rope_table_kernel(const uint32_t* __restrict__ pos, int64_t n_rows, int half,
                                  double theta, int head_dim, int blocked, float2* __restrict__ table) {
  pdl_wait();  // no early trigger: a waiting dependent CTA would crowd out this grid's own blocks
  const int64_t total = n_rows * half;
  for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t j = t / half;
    const int i = static_cast<int>(t - j * half);
    const double inv_freq = pow(theta, -static_cast<double>(2 * i) / static_cast<double>(head_dim));
    const double ang = static_cast<double>(pos[j]) * inv_freq;
    double sn, cs;
    sincos(ang, &sn, &cs);
    const int64_t o = blocked ? 2 * (((j >> 5) * (half >> 1) + (i >> 1)) * 32 + (j & 31)) + (i & 1) : t;
    table[o] = make_float2(static_cast<float>(cs), static_cast<float>(sn));
  }
}

__global__ void rerank_kernel(const float* __restrict__ logits, int64_t n, int64_t ld, int64_t yes,
                              int64_t no, float* __restrict__ out) {
  pdl_wait();  // no early trigger: a waiting dependent CTA would crowd out this grid's own blocks
  const int64_t b = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (b < n) {
    const float z = logits[b * ld + yes] - logits[b * ld + no];
    out[b] = 1.f / (1.f + __expf(-z));
  }
}

int grid_for_rows(int64_t rows, int warps_per_block) {
  int64_t g = (rows + warps_per_block - 1) / warps_per_block;
  const int64_t cap = static_cast<int64_t>(num_sms()) * 16;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return static_cast<int>(g);
}

// 32x32 tiles through shared memory: coalesced fp32 reads along src rows, coalesced bf16
// writes along dst rows; dst columns [rows, ld_dst) are written as zeros (K padding).
__global__ void __launch_bounds__(256)
transpose_f32_bf16_kernel(const float* __restrict__ src, int64_t rows, int64_t cols, int64_t ld_src,
                          __nv_bfloat16* __restrict__ dst, int64_t ld_dst) {
  __shared__ float tile[32][33];
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * 32, c0 = static_cast<int64_t>(blockIdx.y) * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  for (int i = ty; i < 32; i += 8) {
    const int64_t r = r0 + i, c = c0 + tx;
    tile[i][tx] = (r < rows && c < cols) ? src[r * ld_src + c] : 0.f;
  }
  __syncthreads();
  for (int i = ty; i < 32; i += 8) {
    const int64_t c = c0 + i, r = r0 + tx;  // dst[c][r]
    if (c < cols && r < ld_dst) dst[c * ld_dst + r] = __float2bfloat16_rn(tile[tx][i]);
  }
}

}  // namespace
}  // namespace rdx

extern "C" int rdx_transpose_f32_bf16(const float* src, int64_t rows, int64_t cols, int64_t ld_src, void* dst_bf16,
                                      int64_t ld_dst, void* stream) {
  using namespace rdx;
  if (rows < 0 || cols < 0 || ld_src < cols || ld_dst < rows) return RDX_ERR_SHAPE_MISMATCH;
  if (rows == 0 || cols == 0) return RDX_OK;
  if (!src || !dst_bf16) return RDX_ERR_INVALID_ARGUMENT;
  const dim3 grid(static_cast<unsigned>((ld_dst + 31) / 32), static_cast<unsigned>((cols + 31) / 32));
  transpose_f32_bf16_kernel<<<grid, 256, 0, as_stream(stream)>>>(src, rows, cols, ld_src,
                                                                  static_cast<__nv_bfloat16*>(dst_bf16), ld_dst);
  RDX_LAUNCH_CHECK();
  return RDX_OK;
}

extern "C" int rdx_gather_rows(const void* src, int64_t src_rows, int64_t ld_src_bytes,
                               const uint32_t* idx, int64_t n_idx, void* dst, int64_t ld_dst_bytes,
                               int64_t row_bytes, uint32_t* err_flag, void* stream) {
  using namespace rdx;
  if (n_idx < 0 || src_rows < 0 || row_bytes < 0) return RDX_ERR_INVALID_ARGUMENT;
  if (n_idx == 0 || row_bytes == 0) return RDX_OK;
  if (!src || !idx || !dst) return RDX_ERR_INVALID_ARGUMENT;
  const int grid = grid_for_rows(n_idx, 8);
  const uintptr_t align = reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst) |
                          static_cast<uintptr_t>(ld_src_bytes) | static_cast<uintptr_t>(ld_dst_bytes) |
                          static_cast<uintptr_t>(row_bytes);
  cudaStream_t st = as_stream(stream);
  if ((align & 15) == 0) {
    RDX_LAUNCH_PDL((gather_rows_kernel<int4, 4>), grid, 256, 0, st, 
        static_cast<const char*>(src), src_rows, ld_src_bytes, idx, n_idx, static_cast<char*>(dst),
        ld_dst_bytes, row_bytes / 16, err_flag);
  } else if ((align & 3) == 0) {
    RDX_LAUNCH_PDL((gather_rows_kernel<uint32_t, 8>), grid, 256, 0, st, 
        static_cast<const char*>(src), src_rows, ld_src_bytes, idx, n_idx, static_cast<char*>(dst),
        ld_dst_bytes, row_bytes / 4, err_flag);
  } else {
    RDX_LAUNCH_PDL((gather_rows_kernel<uint8_t, 8>), grid, 256, 0, st, 
        static_cast<const char*>(src), src_rows, ld_src_bytes, idx, n_idx, static_cast<char*>(dst),
        ld_dst_bytes, row_bytes, err_flag);
  }
  RDX_LAUNCH_CHECK();
  return RDX_OK;
}

extern "C" int rdx_embed_rmsnorm(const uint32_t* tok, const uint32_t* gather, int64_t n_rows,
                                 const void* embed_bf16, int64_t vocab, int64_t d, const float* norm_w,
                                 float eps, float* h_out, void* hn_bf16_out, uint32_t* err_flag,
                                 void* stream) {
  using namespace rdx;
  if (n_rows < 0 || d <= 0 || (d % 8) != 0) return RDX_ERR_SHAPE_MISMATCH;
  if (n_rows == 0) return RDX_OK;
  RDX_LAUNCH_PDL(embed_rmsnorm_kernel, grid_for_rows(n_rows, 8), 256, 0, as_stream(stream), 
      tok, gather, n_rows, static_cast<const __nv_bfloat16*>(embed_bf16), vocab, d, norm_w, eps, h_out,
      static_cast<__nv_bfloat16*>(hn_bf16_out), err_flag);
  RDX_LAUNCH_CHECK();
  return RDX_OK;
}

extern "C" int rdx_embed_rows(const uint32_t* tok, const uint32_t* gather, int64_t n_rows, const void* embed_bf16,
                              int64_t vocab, int64_t d, float* h_out, void* hb_out, float* ss_out, uint32_t* err_flag,
                              void* stream) {
  using namespace rdx;
  if (n_rows < 0 || d <= 0 || (d % 64) != 0) return RDX_ERR_SHAPE_MISMATCH;
  if (n_rows == 0) return RDX_OK;
  if (!tok || !embed_bf16 || !h_out || !hb_out || !ss_out) return RDX_ERR_INVALID_ARGUMENT;
  RDX_LAUNCH_PDL(embed_rows_kernel, grid_for_rows(n_rows, 8), 256, 0, as_stream(stream), 
      tok, gather, n_rows, static_cast<const __nv_bfloat16*>(embed_bf16), vocab, d, h_out,
      static_cast<__nv_bfloat16*>(hb_out), ss_out, err_flag);
  RDX_LAUNCH_CHECK();
  return RDX_OK;
}

extern "C" int rdx_rmsnorm_rows(const float* x, int64_t ld_x, const uint32_t* rows, int64_t n_rows,
                                int64_t d, const float* w, float eps, void* out_bf16, int64_t ld_out,
                                void* stream) {
  using namespace rdx;
  if (n_rows < 0 || d <= 0 || (d % 8) != 0 || (ld_x % 4) != 0 || (ld_out % 8) != 0)
    return RDX_ERR_SHAPE_MISMATCH;
  if (n_rows == 0) return RDX_OK;
  const int grid = grid_for_rows(n_rows, 8);
  // pipelined kernels: exactly the resident blocks (one wave), never more than the rows need
  auto pgrid = [&](auto kern) {
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, 0) != cudaSuccess || per_sm < 1) per_sm = 1;
    const int64_t g = static_cast<int64_t>(per_sm) * num_sms();
    return static_cast<int>(g < grid ? g : grid);
  };
  cudaStream_t st = as_stream(stream);
  __nv_bfloat16* o = static_cast<__nv_bfloat16*>(out_bf16);
  const bool aligned = ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(w)) & 15) == 0;
  switch (aligned ? d : 0) {
    case 1024: RDX_LAUNCH_PDL(rmsnorm_rows_pipe_kernel<8>, pgrid(rmsnorm_rows_pipe_kernel<8>), 256, 0, st, x, ld_x, rows, n_rows, w, eps, o, ld_out); break;
    case 2048: RDX_LAUNCH_PDL(rmsnorm_rows_pipe_kernel<16>, pgrid(rmsnorm_rows_pipe_kernel<16>), 256, 0, st, x, ld_x, rows, n_rows, w, eps, o, ld_out); break;
    case 2560: RDX_LAUNCH_PDL(rmsnorm_rows_reg_kernel<20>, grid, 256, 0, st, x, ld_x, rows, n_rows, w, eps, o, ld_out); break;
    case 4096: RDX_LAUNCH_PDL(rmsnorm_rows_reg_kernel<32>, grid, 256, 0, st, x, ld_x, rows, n_rows, w, eps, o, ld_out); break;
    case 512: RDX_LAUNCH_PDL(rmsnorm_rows_reg_kernel<4>, grid, 256, 0, st, x, ld_x, rows, n_rows, w, eps, o, ld_out); break;
    case 256: RDX_LAUNCH_PDL(rmsnorm_rows_reg_kernel<2>, grid, 256, 0, st, x, ld_x, rows, n_rows, w, eps, o, ld_out); break;
    default:
      RDX_LAUNCH_PDL(rmsnorm_rows_kernel, grid, 256, 0, st, x, ld_x, rows, n_rows, d, w, eps, o, ld_out);
  }
  RDX_LAUNCH_CHECK();
  return RDX_OK;
}

namespace rdx {
namespace {
// Warps per block of the (non-chained) rmsnorm_rows_after grid (rdx_norm_debug_warps).  4:
// a 128-thread block fits beside a GEMM CTA (registers; the non-QKV GEMMs leave the shared
// memory for its reservation), so more of the grid is resident before the GEMM exits
// (C2 +0.2-0.3 %, C3 +0.7 %, C4 +0.2 % over 8-warp blocks, scripts/ab_graph.py normw).
int g_norm_warps = 4;

template <int V, int W>
cudaError_t launch_norm_after(cudaLaunchConfig_t& cfg, const float* x, int64_t ld_x, int64_t n_rows, const float* w,
                              float eps, __nv_bfloat16* o, int64_t ld_out, const uint32_t* done_ctr, uint32_t target,
                              uint32_t* ready_ctr) {
  cfg.blockDim = dim3(W * 32);
  return cudaLaunchKernelEx(&cfg, rmsnorm_rows_after_kernel<V, W>, x, ld_x, n_rows, w, eps, o, ld_out, done_ctr,
                            target, ready_ctr);
}
}  // namespace
}  // namespace rdx

extern "C" int rdx_rmsnorm_rows_after(const float* x, int64_t ld_x, int64_t n_rows, int64_t d, const float* w,
                                      float eps, void* out_bf16, int64_t ld_out, const uint32_t* done_ctr,
                                      uint32_t target, uint32_t* ready_ctr, void* stream) {
  using namespace rdx;
  if (n_rows < 0 || d <= 0 || (d % 8) != 0 || (ld_x % 4) != 0 || (ld_out % 8) != 0) return RDX_ERR_SHAPE_MISMATCH;
  if (n_rows == 0) return RDX_OK;
  if (!done_ctr) return RDX_ERR_INVALID_ARGUMENT;
  if (((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(w)) & 15) != 0) return RDX_ERR_UNSUPPORTED;
  __nv_bfloat16* o = static_cast<__nv_bfloat16*>(out_bf16);
  cudaLaunchConfig_t cfg = {};
  // chained: one block per SM, 2-8 warps so its registers fit beside a GEMM CTA (168 x 320);
  // plain: 8 warps, one block per 8 rows (capped)
  static const int chain_grid = [] {  // RDX_NORM_CHAIN_GRID=1: the one-block-per-SM chained grid
    const char* v = std::getenv("RDX_NORM_CHAIN_GRID");
    return v && v[0] == '1' ? 1 : 0;
  }();
  const bool small = ready_ctr && chain_grid;
  const bool w4 = !small && g_norm_warps == 4;
  cfg.gridDim = dim3(static_cast<unsigned>(small ? (n_rows < num_sms() ? n_rows : num_sms())
                                                 : grid_for_rows(n_rows, w4 ? 4 : 8)));
  cfg.stream = as_stream(stream);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // always: it overlaps the GEMM's tail
  static const int pdl = [] {
    const char* v = std::getenv("RDX_NORM_AFTER_PDL");
    return v && v[0] == '0' ? 0 : 1;
  }();
  attr[0].val.programmaticStreamSerializationAllowed = pdl;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e;
#define RDX_NA(V, WCH) (small ? launch_norm_after<V, WCH>(cfg, x, ld_x, n_rows, w, eps, o, ld_out, done_ctr, target, ready_ctr) \
                              : w4 ? launch_norm_after<V, 4>(cfg, x, ld_x, n_rows, w, eps, o, ld_out, done_ctr, target, ready_ctr) \
                                   : launch_norm_after<V, 8>(cfg, x, ld_x, n_rows, w, eps, o, ld_out, done_ctr, target, ready_ctr))
  switch (d) {
    case 256: e = RDX_NA(2, 8); break;
    case 512: e = RDX_NA(4, 8); break;
    case 1024: e = RDX_NA(8, 4); break;
    case 2048: e = RDX_NA(16, 4); break;
    case 2560: e = RDX_NA(20, 2); break;
    case 4096: e = RDX_NA(32, 1); break;  // 197 registers: one warp fits beside a 168 x 320 GEMM CTA
    default: return RDX_ERR_UNSUPPORTED;
  }
#undef RDX_NA
  if (e != cudaSuccess) return set_cuda_error(e);
  RDX_LAUNCH_CHECK();
  return RDX_OK;
}

namespace rdx {
namespace {
int rope_table_launch(const uint32_t* pos, int64_t n_rows, int32_t head_dim, double theta, int blocked,
                      float* table_out, void* stream) {
  const int half = head_dim / 2;
  int64_t total = n_rows * half;
  int64_t g = (total + 255) / 256;
  if (g > num_sms() * 8) g = num_sms() * 8;
  RDX_LAUNCH_PDL(rope_table_kernel, static_cast<int>(g), 256, 0, as_stream(stream), 
      pos, n_rows, half, theta, head_dim, blocked, reinterpret_cast<float2*>(table_out));
  RDX_LAUNCH_CHECK();
  return RDX_OK;
}
}  // namespace
}  // namespace rdx

extern "C" int rdx_rope_table(const uint32_t* pos, int64_t n_rows, int32_t head_dim, double theta,
                              float* table_out, void* stream) {
  using namespace rdx;
  if (head_dim <= 0) return RDX_ERR_SHAPE_MISMATCH;
  if (head_dim % 2) return RDX_ERR_ODD_HEAD_DIM;
  if (n_rows <= 0) return RDX_OK;
  return rope_table_launch(pos, n_rows, head_dim, theta, 0, table_out, stream);
}

extern "C" int rdx_rope_table_blocked(const uint32_t* pos, int64_t n_rows, int32_t head_dim, double theta,
                                      float* table_out, void* stream) {
  using namespace rdx;
  if (head_dim <= 0) return RDX_ERR_SHAPE_MISMATCH;
  if (head_dim % 2) return RDX_ERR_ODD_HEAD_DIM;
  if (head_dim % 4) return RDX_ERR_SHAPE_MISMATCH;
  if (n_rows <= 0) return RDX_OK;
  if (reinterpret_cast<uintptr_t>(table_out) & 15) return RDX_ERR_INVALID_ARGUMENT;
  return rope_table_launch(pos, n_rows, head_dim, theta, 1, table_out, stream);
}

extern "C" int rdx_rerank_scores(const float* logits, int64_t n_rows, int64_t ld, int64_t yes_id,
                                 int64_t no_id, float* scores_out, void* stream) {
  using namespace rdx;
  if (n_rows <= 0) return RDX_OK;
  if (yes_id < 0 || no_id < 0 || yes_id >= ld || no_id >= ld) return RDX_ERR_INDEX_OUT_OF_RANGE;
  RDX_LAUNCH_PDL(rerank_kernel, static_cast<int>((n_rows + 127) / 128), 128, 0, as_stream(stream), 
      logits, n_rows, ld, yes_id, no_id, scores_out);
  RDX_LAUNCH_CHECK();
  return RDX_OK;
}

int rdx::take_device_status_rowops(int* out, cudaStream_t st) { return take_device_status(out, st); }

// Debug: longest nanosleep (ns, 64..16384) of the rmsnorm_rows_after slab pollers; read by
// the kernel at run time (graph replays included).
extern "C" int rdx_norm_debug_backoff(unsigned ns) {
  if (ns < 64 || ns > 16384) return RDX_ERR_INVALID_ARGUMENT;
  RDX_CUDA_TRY(cudaMemcpyToSymbol(rdx::g_norm_backoff_max, &ns, sizeof(ns)));
  return RDX_OK;
}

// Debug: warps per block of the plain rmsnorm_rows_after grid (4 or 8; read at launch).
extern "C" int rdx_norm_debug_warps(int w) {
  if (w != 4 && w != 8) return RDX_ERR_INVALID_ARGUMENT;
  rdx::g_norm_warps = w;
  return RDX_OK;
}

// Debug (-DRDX_NORM_STATS_BUILD): per-block [entry, exit] %globaltimer of the last
// rdx_rmsnorm_rows_after launch, n_blocks <= 4096 entries.
extern "C" int rdx_norm_debug_times(unsigned long long* host, int n_blocks) {
#ifdef RDX_NORM_STATS_BUILD
  if (!host || n_blocks <= 0 || n_blocks > 4096) return RDX_ERR_INVALID_ARGUMENT;
  RDX_CUDA_TRY(cudaMemcpyFromSymbol(host, rdx::g_norm_times, 2 * n_blocks * sizeof(unsigned long long)));
  return RDX_OK;
#else
  (void)host;
  (void)n_blocks;
  return RDX_ERR_UNSUPPORTED;
#endif
}
