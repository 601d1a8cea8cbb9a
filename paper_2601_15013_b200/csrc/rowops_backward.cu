// rowops_backward.cu — adjoints of the RadixMLP row gather / scatter on the GPU.
//
// Reference: ops.py:69-107 (gather_rows_backward / scatter_rows_backward):
//   out = zeros(n_out, cols);  out[idx[j], :] += grad[j, :]  for j = 0, 1, ...
// with ascending-j accumulation where indices repeat (np.add.at order, the
// reference's single-thread path).  Here the adds for each output row happen
// in exactly that order, so results are bit-identical to np.add.at for fp32
// and fp64 (0 + g_j1 + g_j2 + ... in ascending j):
//   1. stable radix sort of (idx[j], j) by idx            -> j grouped by row, ascending
//   2. segment bounds per output row (first / one-past-last position)
//   3. one warp per output row: sequential sum over its segment, lanes over
//      columns (8-byte / 16-byte vectors), zero rows without entries.
// Out-of-range indices set *err_flag (IndexOutOfRange on the host) and are
// skipped.  Used for the compact-path backward of model.py:456-500.
#include <cub/device/device_radix_sort.cuh>

#include "common.cuh"

namespace rdx {
namespace {

__global__ void iota_check_kernel(const uint32_t* __restrict__ idx, int64_t n, uint32_t n_out,
                                  uint32_t* __restrict__ keys, uint32_t* __restrict__ vals,
                                  uint32_t* __restrict__ err) {
  for (int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; j < n;
       j += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    uint32_t k = idx[j];
    if (k >= n_out) {
      if (err) atomicOr(err, 1u);
      k = n_out;  // sorts past every real row; never summed
    }
    keys[j] = k;
    vals[j] = static_cast<uint32_t>(j);
  }
}

__global__ void fill_u32_kernel(uint32_t* __restrict__ p, int64_t n, uint32_t v) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    p[i] = v;
}

// seg_start[r] / seg_end[r] for every row r present in the sorted keys.
__global__ void segments_kernel(const uint32_t* __restrict__ keys, int64_t n, uint32_t n_out,
                                uint32_t* __restrict__ seg_start, uint32_t* __restrict__ seg_end) {
  for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < n;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint32_t k = keys[p];
    if (k >= n_out) continue;
    if (p == 0 || keys[p - 1] != k) seg_start[k] = static_cast<uint32_t>(p);
    if (p == n - 1 || keys[p + 1] != k) seg_end[k] = static_cast<uint32_t>(p + 1);
  }
}

// One warp per output row; lanes stride over the row in units of V (float2 /
// double / float4 ...).  The j loop is sequential: ascending-j accumulation.
template <typename T, typename V>
__global__ void sum_rows_kernel(const char* __restrict__ grad, int64_t ld_grad, const uint32_t* __restrict__ order,
                                const uint32_t* __restrict__ seg_start, const uint32_t* __restrict__ seg_end,
                                int64_t n_out, char* __restrict__ out, int64_t ld_out, int64_t nvec) {
  constexpr int E = sizeof(V) / sizeof(T);
  const int lane = threadIdx.x & 31;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x >> 5) + (threadIdx.x >> 5); r < n_out; r += warps) {
    const uint32_t b = seg_start[r], e = seg_end[r];
    V* orow = reinterpret_cast<V*>(out + r * ld_out);
    for (int64_t c = lane; c < nvec; c += 32) {
      T acc[E];
#pragma unroll
      for (int u = 0; u < E; ++u) acc[u] = T(0);
      for (uint32_t p = b; p < e; ++p) {
        const V g = __ldg(reinterpret_cast<const V*>(grad + static_cast<int64_t>(order[p]) * ld_grad) + c);
        const T* gv = reinterpret_cast<const T*>(&g);
#pragma unroll
        for (int u = 0; u < E; ++u) acc[u] = acc[u] + gv[u];
      }
      V o;
      T* ov = reinterpret_cast<T*>(&o);
#pragma unroll
      for (int u = 0; u < E; ++u) ov[u] = acc[u];
      orow[c] = o;
    }
  }
}

int grid_for(int64_t n, int per_block) {
  const int64_t want = (n + per_block - 1) / per_block;
  const int64_t cap = static_cast<int64_t>(num_sms()) * 16;
  return static_cast<int>(want < 1 ? 1 : (want < cap ? want : cap));
}

int end_bit_for(uint32_t n_out) {
  int b = 1;
  while (b < 32 && (uint64_t(1) << b) <= n_out) ++b;  // keys are in [0, n_out]
  return b;
}

size_t sort_temp_bytes(int64_t n, uint32_t n_out) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, static_cast<const uint32_t*>(nullptr),
                                  static_cast<uint32_t*>(nullptr), static_cast<const uint32_t*>(nullptr),
                                  static_cast<uint32_t*>(nullptr), static_cast<int>(n), 0, end_bit_for(n_out));
  return bytes;
}

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

}  // namespace
}  // namespace rdx

extern "C" size_t rdx_gather_rows_backward_scratch_bytes(int64_t n_idx, int64_t n_out) {
  using namespace rdx;
  if (n_idx < 0 || n_out < 0 || n_out >= (int64_t(1) << 32) - 1) return 0;
  return 4 * align256(static_cast<size_t>(n_idx) * 4) + 2 * align256(static_cast<size_t>(n_out) * 4) +
         align256(sort_temp_bytes(n_idx, static_cast<uint32_t>(n_out)));
}

extern "C" int rdx_gather_rows_backward(const void* grad, int64_t ld_grad_bytes, const uint32_t* idx, int64_t n_idx,
                                        int64_t n_out, void* out, int64_t ld_out_bytes, int64_t cols,
                                        int32_t dtype, uint32_t* err_flag, void* scratch, size_t scratch_bytes,
                                        void* stream) {
  using namespace rdx;
  if (n_idx < 0 || n_out < 0 || cols < 0) return RDX_ERR_INVALID_ARGUMENT;
  if (dtype != RDX_DTYPE_F32 && dtype != RDX_DTYPE_F64) return RDX_ERR_UNSUPPORTED;
  if (n_idx >= (int64_t(1) << 31) || n_out >= (int64_t(1) << 32) - 1) return RDX_ERR_CAPACITY_EXCEEDED;
  if (n_out == 0 || cols == 0) return RDX_OK;
  const int esz = dtype == RDX_DTYPE_F32 ? 4 : 8;
  if (!out || (n_idx > 0 && (!grad || !idx))) return RDX_ERR_INVALID_ARGUMENT;
  if (scratch_bytes < rdx_gather_rows_backward_scratch_bytes(n_idx, n_out)) return RDX_ERR_INVALID_ARGUMENT;
  cudaStream_t st = as_stream(stream);
  char* s = static_cast<char*>(scratch);
  const size_t a_idx = align256(static_cast<size_t>(n_idx) * 4), a_out = align256(static_cast<size_t>(n_out) * 4);
  uint32_t* keys_in = reinterpret_cast<uint32_t*>(s);
  uint32_t* vals_in = reinterpret_cast<uint32_t*>(s + a_idx);
  uint32_t* keys = reinterpret_cast<uint32_t*>(s + 2 * a_idx);
  uint32_t* order = reinterpret_cast<uint32_t*>(s + 3 * a_idx);
  uint32_t* seg_start = reinterpret_cast<uint32_t*>(s + 4 * a_idx);
  uint32_t* seg_end = reinterpret_cast<uint32_t*>(s + 4 * a_idx + a_out);
  void* temp = s + 4 * a_idx + 2 * a_out;
  size_t temp_bytes = sort_temp_bytes(n_idx, static_cast<uint32_t>(n_out));

  fill_u32_kernel<<<grid_for(n_out, 256), 256, 0, st>>>(seg_start, n_out, 0u);
  fill_u32_kernel<<<grid_for(n_out, 256), 256, 0, st>>>(seg_end, n_out, 0u);
  if (n_idx > 0) {
    iota_check_kernel<<<grid_for(n_idx, 256), 256, 0, st>>>(idx, n_idx, static_cast<uint32_t>(n_out), keys_in,
                                                             vals_in, err_flag);
    if (cub::DeviceRadixSort::SortPairs(temp, temp_bytes, keys_in, keys, vals_in, order, static_cast<int>(n_idx), 0,
                                        end_bit_for(static_cast<uint32_t>(n_out)), st) != cudaSuccess)
      return set_cuda_error(cudaGetLastError());
    segments_kernel<<<grid_for(n_idx, 256), 256, 0, st>>>(keys, n_idx, static_cast<uint32_t>(n_out), seg_start,
                                                           seg_end);
  }
  const int64_t row_bytes = cols * esz;
  const uintptr_t align = reinterpret_cast<uintptr_t>(grad) | reinterpret_cast<uintptr_t>(out) |
                          static_cast<uintptr_t>(ld_grad_bytes) | static_cast<uintptr_t>(ld_out_bytes) |
                          static_cast<uintptr_t>(row_bytes);
  const int grid = grid_for(n_out, 8);
  const char* g = static_cast<const char*>(grad);
  char* o = static_cast<char*>(out);
  if (dtype == RDX_DTYPE_F32) {
    if ((align & 15) == 0)
      sum_rows_kernel<float, float4><<<grid, 256, 0, st>>>(g, ld_grad_bytes, order, seg_start, seg_end, n_out, o,
                                                            ld_out_bytes, row_bytes / 16);
    else
      sum_rows_kernel<float, float><<<grid, 256, 0, st>>>(g, ld_grad_bytes, order, seg_start, seg_end, n_out, o,
                                                           ld_out_bytes, cols);
  } else {
    if ((align & 15) == 0)
      sum_rows_kernel<double, double2><<<grid, 256, 0, st>>>(g, ld_grad_bytes, order, seg_start, seg_end, n_out, o,
                                                              ld_out_bytes, row_bytes / 16);
    else
      sum_rows_kernel<double, double><<<grid, 256, 0, st>>>(g, ld_grad_bytes, order, seg_start, seg_end, n_out, o,
                                                             ld_out_bytes, cols);
  }
  RDX_LAUNCH_CHECK();
  return RDX_OK;
}
