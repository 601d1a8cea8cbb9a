// gemm.cu — persistent warp-specialised tcgen05/TMEM GEMM for sm_100a with the
// fused RadixMLP epilogues (model.py:352-399 on the compact rows).
//
//   acc[m, n] = sum_k A[m, k] * B[n, k]        A: activations [M, K] bf16
//                                              B: weight [N, K] bf16 ([out, in])
// CTA = 6 warps:
//   warp 0      TMA producer (one elected lane): A/B k-blocks -> smem ring
//   warp 1      TMEM allocator + MMA issuer (one lane): tcgen05.mma 128xBNx16
//   warps 2..5  epilogue: tcgen05.ld accumulator rows -> fused op -> global
// Pipelines: smem full/empty mbarriers (TMA <-> MMA), two TMEM accumulator
// buffers with full/empty mbarriers (MMA <-> epilogue), static persistent
// tile schedule (tile = blockIdx.x + i * gridDim.x, M fastest).
// Each output row depends only on its own A row: no split-K, M-independent
// tiling, so the compact and the full forward give bit-identical rows
// (the reference's _mm batch-invariance rule, model.py:124-144).
#include <mutex>

#include "common.cuh"

namespace rdx {
namespace gemm {

constexpr int BM = 128;
constexpr int BK = 64;  // 64 bf16 = 128 B = one SWIZZLE_128B atom row
constexpr int kThreads = 192;
constexpr int kSwigluUnit = 64;  // gate/up interleave unit (columns)

struct EpiParams {
  void* out;
  int64_t ldo;
  const float* qn;
  const float* kn;
  const float2* rope;
  int hd, q_dim, kv_dim;
  float eps;
};

template <int BN, int STAGES>
struct Cfg {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256;
  static constexpr uint32_t IDESC = umma_idesc_bf16(BM, BN);
  static constexpr uint32_t TMEM_COLS = 2 * BN;
};

__device__ __forceinline__ void store8_bf16(void* out, int64_t ldo, int64_t gm, int64_t col,
                                            int64_t ncols, const float (&v)[8]) {
  __nv_bfloat16* p = static_cast<__nv_bfloat16*>(out) + gm * ldo + col;
  if (col + 8 <= ncols) {
    st_global_v4(p, pack_bf16x2(v[0], v[1]), pack_bf16x2(v[2], v[3]), pack_bf16x2(v[4], v[5]),
                 pack_bf16x2(v[6], v[7]));
  } else {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (col + j < ncols) p[j] = __float2bfloat16(v[j]);
  }
}

__device__ __forceinline__ void store8_f32(void* out, int64_t ldo, int64_t gm, int64_t col,
                                           int64_t ncols, const float (&v)[8], bool accumulate) {
  float* p = static_cast<float*>(out) + gm * ldo + col;
  if (col + 8 <= ncols) {
    float4* q = reinterpret_cast<float4*>(p);
    float4 a = make_float4(v[0], v[1], v[2], v[3]), b = make_float4(v[4], v[5], v[6], v[7]);
    if (accumulate) {
      const float4 a0 = q[0], b0 = q[1];
      a.x += a0.x; a.y += a0.y; a.z += a0.z; a.w += a0.w;
      b.x += b0.x; b.y += b0.y; b.z += b0.z; b.w += b0.w;
    }
    q[0] = a;
    q[1] = b;
  } else {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (col + j < ncols) p[j] = accumulate ? p[j] + v[j] : v[j];
  }
}

template <int BN, int EPI>
__device__ __forceinline__ void epilogue_tile(uint32_t taddr, int64_t gm, bool row_ok, int64_t n_blk,
                                              int64_t N, const EpiParams& ep) {
  const int64_t gn0 = n_blk * BN;
  if constexpr (EPI == RDX_EPI_STORE_BF16 || EPI == RDX_EPI_STORE_F32 || EPI == RDX_EPI_RESID_F32) {
#pragma unroll 1
    for (int c = 0; c < BN; c += 32) {
      if (gn0 + c >= N) break;
      float v[32];
      tmem_ld32(taddr + c, v);
      tmem_wait_ld();
      if (row_ok) {
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          float w[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) w[j] = v[g * 8 + j];
          const int64_t col = gn0 + c + g * 8;
          if (col < N) {
            if constexpr (EPI == RDX_EPI_STORE_BF16) store8_bf16(ep.out, ep.ldo, gm, col, N, w);
            else store8_f32(ep.out, ep.ldo, gm, col, N, w, EPI == RDX_EPI_RESID_F32);
          }
        }
      }
    }
  } else if constexpr (EPI == RDX_EPI_SWIGLU) {
    // tile columns: [g(64) u(64)] x (BN/128); out col = n_blk*BN/2 + pair*64 + j
    const int64_t nout = N / 2;
#pragma unroll 1
    for (int p = 0; p < BN / (2 * kSwigluUnit); ++p) {
      const int64_t ocol0 = n_blk * (BN / 2) + p * kSwigluUnit;
      if (ocol0 >= nout) break;
#pragma unroll 1
      for (int c = 0; c < kSwigluUnit; c += 32) {
        float g[32], u[32];
        tmem_ld32(taddr + p * 2 * kSwigluUnit + c, g);
        tmem_ld32(taddr + p * 2 * kSwigluUnit + kSwigluUnit + c, u);
        tmem_wait_ld();
        if (row_ok) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            float w[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const float x = g[q * 8 + j];
              w[j] = x / (1.f + __expf(-x)) * u[q * 8 + j];
            }
            store8_bf16(ep.out, ep.ldo, gm, ocol0 + c + q * 8, nout, w);
          }
        }
      }
    }
  } else if constexpr (EPI == RDX_EPI_QKV) {
    const int hd = ep.hd, half = hd >> 1;
#pragma unroll 1
    for (int h0 = 0; h0 < BN; h0 += hd) {
      const int64_t col0 = gn0 + h0;
      if (col0 >= N) break;
      const int kind = col0 < ep.q_dim ? 0 : (col0 < ep.q_dim + ep.kv_dim ? 1 : 2);
      if (kind == 2) {
#pragma unroll 1
        for (int c = 0; c < hd; c += 8) {
          float v[8];
          tmem_ld8(taddr + h0 + c, v);
          tmem_wait_ld();
          if (row_ok) store8_bf16(ep.out, ep.ldo, gm, col0 + c, N, v);
        }
        continue;
      }
      const float* __restrict__ nw = kind == 0 ? ep.qn : ep.kn;
      float ss = 0.f;
#pragma unroll 1
      for (int c = 0; c < hd; c += 8) {
        float v[8];
        tmem_ld8(taddr + h0 + c, v);
        tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 8; ++j) ss += v[j] * v[j];
      }
      const float inv = rsqrtf(ss / static_cast<float>(hd) + ep.eps);
      const float2* __restrict__ rope = ep.rope + (row_ok ? gm : 0) * half;
#pragma unroll 1
      for (int c = 0; c < half; c += 8) {
        float x1[8], x2[8], o1[8], o2[8];
        tmem_ld8(taddr + h0 + c, x1);
        tmem_ld8(taddr + h0 + half + c, x2);
        tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float a = x1[j] * inv * __ldg(nw + c + j);
          const float b = x2[j] * inv * __ldg(nw + half + c + j);
          const float2 cs = __ldg(rope + c + j);
          o1[j] = a * cs.x - b * cs.y;
          o2[j] = b * cs.x + a * cs.y;
        }
        if (row_ok) {
          store8_bf16(ep.out, ep.ldo, gm, col0 + c, N, o1);
          store8_bf16(ep.out, ep.ldo, gm, col0 + half + c, N, o2);
        }
      }
    }
  }
}

template <int BN, int STAGES, int EPI>
__global__ void __launch_bounds__(kThreads, 1)
gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
            int64_t M, int64_t N, int64_t K, EpiParams ep) {
  using C = Cfg<BN, STAGES>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * C::STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t m_tiles = (M + BM - 1) / BM;
  const int64_t n_tiles = (N + BN - 1) / BN;
  const int64_t num_tiles = m_tiles * n_tiles;
  const int kblocks = static_cast<int>((K + BK - 1) / BK);

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 128);
    }
    fence_mbar_init();
  }
  if (warp == 1) {
    tmem_alloc(tmem_holder, C::TMEM_COLS);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        const int32_t m0 = static_cast<int32_t>((tile % m_tiles) * BM);
        const int32_t n0 = static_cast<int32_t>((tile / m_tiles) * BN);
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * C::STAGE_BYTES;
          uint8_t* sb = sa + C::A_BYTES;
          mbar_arrive_expect_tx(&full[stage], C::STAGE_BYTES);
          tma_load_2d(&tmA, sa, &full[stage], kb * BK, m0);
          tma_load_2d(&tmB, sb, &full[stage], kb * BK, n0);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int64_t tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * C::STAGE_BYTES);
          const uint32_t sb = sa + C::A_BYTES;
          const uint64_t da = umma_sdesc_sw128(sa);
          const uint64_t db = umma_sdesc_sw128(sb);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            // +32 B per K=16 step inside the 128 B swizzle atom (encoded >> 4)
            umma_bf16(d_tmem, da + 2 * k, db + 2 * k, C::IDESC, (kb | k) != 0);
          }
          umma_commit(&empty[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit(&tfull[acc]);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else {
    const int q = warp & 3;  // TMEM lane quarter accessible to this warp
    const int row = q * 32 + lane;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int64_t tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      const int64_t m_blk = tile % m_tiles;
      const int64_t n_blk = tile / m_tiles;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t taddr = tmem_base + acc * BN + (static_cast<uint32_t>(q * 32) << 16);
      const int64_t gm = m_blk * BM + row;
      epilogue_tile<BN, EPI>(taddr, gm, gm < M, n_blk, N, ep);
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, C::TMEM_COLS);
  }
}

// ---------------------------------------------------------------- host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

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

int make_map(CUtensorMap* map, const void* ptr, int64_t inner, int64_t outer, int64_t ld_elems,
             int box_outer) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return RDX_ERR_UNSUPPORTED;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(outer)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld_elems) * 2};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(BK), static_cast<cuuint32_t>(box_outer)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box,
                  estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? RDX_OK : RDX_ERR_INVALID_ARGUMENT;
}

template <int BN, int STAGES, int EPI>
int launch(const rdx_gemm_args& a, cudaStream_t stream) {
  using C = Cfg<BN, STAGES>;
  auto kern = gemm_kernel<BN, STAGES, EPI>;
  static bool attr_set = false;
  if (!attr_set) {
    RDX_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    attr_set = true;
  }
  CUtensorMap ma, mb;
  int st = make_map(&ma, a.a, a.k, a.m, a.lda, BM);
  if (st) return st;
  st = make_map(&mb, a.b, a.k, a.n, a.ldb, BN);
  if (st) return st;
  EpiParams ep;
  ep.out = a.out;
  ep.ldo = a.ldo;
  ep.qn = a.q_norm_w;
  ep.kn = a.k_norm_w;
  ep.rope = reinterpret_cast<const float2*>(a.rope_table);
  ep.hd = a.head_dim;
  ep.q_dim = a.q_heads * a.head_dim;
  ep.kv_dim = a.kv_heads * a.head_dim;
  ep.eps = a.eps;
  const int64_t tiles = ((a.m + BM - 1) / BM) * ((a.n + BN - 1) / BN);
  const int grid = static_cast<int>(tiles < num_sms() ? tiles : num_sms());
  kern<<<grid, kThreads, C::SMEM, stream>>>(ma, mb, a.m, a.n, a.k, ep);
  RDX_LAUNCH_CHECK();
  return RDX_OK;
}

template <int EPI>
int dispatch_bn(const rdx_gemm_args& a, int bn, cudaStream_t s) {
  if (bn == 256) return launch<256, 4, EPI>(a, s);
  return launch<128, 6, EPI>(a, s);
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
  if ((reinterpret_cast<uintptr_t>(a.a) | reinterpret_cast<uintptr_t>(a.b) |
       reinterpret_cast<uintptr_t>(a.out)) & 15)
    return RDX_ERR_INVALID_ARGUMENT;
  int bn = a.block_n;
  if (bn == 0) {
    const int64_t m_tiles = (a.m + BM - 1) / BM;
    bn = (m_tiles * ((a.n + 255) / 256) >= 2 * num_sms()) ? 256 : 128;
  }
  if (bn != 128 && bn != 256) return RDX_ERR_INVALID_ARGUMENT;
  cudaStream_t s = as_stream(stream);
  switch (a.epi) {
    case RDX_EPI_STORE_BF16:
      if (a.ldo % 8 || a.ldo < a.n) return RDX_ERR_SHAPE_MISMATCH;
      return dispatch_bn<RDX_EPI_STORE_BF16>(a, bn, s);
    case RDX_EPI_STORE_F32:
      if (a.ldo % 4 || a.ldo < a.n) return RDX_ERR_SHAPE_MISMATCH;
      return dispatch_bn<RDX_EPI_STORE_F32>(a, bn, s);
    case RDX_EPI_RESID_F32:
      if (a.ldo % 4 || a.ldo < a.n) return RDX_ERR_SHAPE_MISMATCH;
      return dispatch_bn<RDX_EPI_RESID_F32>(a, bn, s);
    case RDX_EPI_SWIGLU:
      if (a.n % (2 * kSwigluUnit) || a.ldo % 8 || a.ldo < a.n / 2) return RDX_ERR_SHAPE_MISMATCH;
      return dispatch_bn<RDX_EPI_SWIGLU>(a, bn, s);
    case RDX_EPI_QKV: {
      const int hd = a.head_dim;
      if (hd <= 0 || hd % 16 || hd > 128 || bn % hd) return RDX_ERR_SHAPE_MISMATCH;
      if (a.n != static_cast<int64_t>(a.q_heads + 2 * a.kv_heads) * hd) return RDX_ERR_SHAPE_MISMATCH;
      if (!a.q_norm_w || !a.k_norm_w || !a.rope_table) return RDX_ERR_INVALID_ARGUMENT;
      if (a.ldo % 8 || a.ldo < a.n) return RDX_ERR_SHAPE_MISMATCH;
      return dispatch_bn<RDX_EPI_QKV>(a, bn, s);
    }
    default:
      return RDX_ERR_INVALID_ARGUMENT;
  }
}
