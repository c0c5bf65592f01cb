// K-EXP: dense d x d block-circulant expansion (Lemma 1; Alg. 1 lines 3-6, P:340-343;
// Alg. 2 line 10). Write-bandwidth bound: each source row segment (b, k, i) of m values is read
// once and written to the n output positions (r*m + i, ((r + k) mod n)*m + j), r = 0..n-1, with 128-bit
// streaming (evict-first) stores. In C-LOT mode the source value is S_ij where argmin_ij == k, else 0
// (the lift of eq. optimal_solution_problem_CLOT). Pure placement => bit-exact.
#include <cstdlib>

#include "common.cuh"
#include "internal.h"

namespace cot {

template <typename T, int V>
struct VecT;
template <>
struct VecT<float, 4> {
  using type = float4;
  __device__ static float get(const type& v, int q) { return q == 0 ? v.x : q == 1 ? v.y : q == 2 ? v.z : v.w; }
  __device__ static void set(type& v, int q, float x) {
    if (q == 0) v.x = x; else if (q == 1) v.y = x; else if (q == 2) v.z = x; else v.w = x;
  }
};
template <>
struct VecT<double, 2> {
  using type = double2;
  __device__ static double get(const type& v, int q) { return q == 0 ? v.x : v.y; }
  __device__ static void set(type& v, int q, double x) {
    if (q == 0) v.x = x; else v.y = x;
  }
};
template <typename T>
struct VecT<T, 1> {
  using type = T;
  __device__ static T get(const type& v, int) { return v; }
  __device__ static void set(type& v, int, T x) { v = x; }
};

// Work unit = (b, k, i): one source row segment. Threads of the CTA cover (r, j-vector) pairs.
// Source blocks hold R rows (R = m unsharded); destination row (r, i) is r*R + i with row stride d.
template <typename T, int V>
__global__ void __launch_bounds__(256) k_expand(const T* __restrict__ S, const int32_t* __restrict__ A, int64_t B,
                                                int n, int64_t m, int64_t R, T* __restrict__ out) {
  using VT = typename VecT<T, V>::type;
  const int64_t mv = m / V;            // vectors per row segment
  const int64_t d = (int64_t)n * m;
  const int64_t units = B * n * R;
  const int64_t items = (int64_t)n * mv;
  for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
    const int64_t b = u / (n * R);
    const int64_t rem = u - b * n * R;
    const int k = (int)(rem / R);
    const int64_t i = rem - (int64_t)k * R;
    T* ob = out + b * (int64_t)n * R * d;
    for (int64_t it = threadIdx.x; it < items; it += blockDim.x) {
      const int r = (int)(it / mv);
      const int64_t jv = it - (int64_t)r * mv;
      VT v;
      if (A == nullptr) {
        v = reinterpret_cast<const VT*>(S + ((b * n + k) * R + i) * m)[jv];
      } else {
        const VT sv = reinterpret_cast<const VT*>(S + (b * R + i) * m)[jv];
        const int32_t* ar = A + (b * R + i) * m + jv * V;
#pragma unroll
        for (int q = 0; q < V; ++q) VecT<T, V>::set(v, q, ar[q] == k ? VecT<T, V>::get(sv, q) : T(0));
      }
      const int s = (r + k) % n;        // block (r, s) holds source block (s - r) mod n = k
      VT* dst = reinterpret_cast<VT*>(ob + ((int64_t)r * R + i) * d + (int64_t)s * m) + jv;
      __stcs(dst, v);
    }
  }
}

// Main path (m * sizeof(T) % 16 == 0): the CTA builds the source segment in shared memory, then ONE
// thread issues n TMA bulk stores (cp.async.bulk.global.shared::cta, SASS UBLKCP) of m*sizeof(T) bytes,
// one per destination block; the TMA engine, not the SMs' issue slots, moves the d*d output.
// Two smem slots alternate; bulk-async group accounting guards their reuse.
template <typename T>
__global__ void __launch_bounds__(128) k_expand_bulk(const T* __restrict__ S, const int32_t* __restrict__ A,
                                                     int64_t B, int n, int64_t m, int64_t R, T* __restrict__ out) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int64_t mpad = (m + 31) & ~int64_t(31);
  T* bufs = reinterpret_cast<T*>(smem_raw);
  const int64_t d = (int64_t)n * m;
  const int64_t units = B * n * R;
  const uint32_t seg_bytes = (uint32_t)(m * sizeof(T));
  int slot = 0;
  for (int64_t u = blockIdx.x; u < units; u += gridDim.x, slot ^= 1) {
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    __syncthreads();
    const int64_t b = u / (n * R);
    const int64_t rem = u - b * n * R;
    const int k = (int)(rem / R);
    const int64_t i = rem - (int64_t)k * R;
    T* buf = bufs + slot * mpad;
    if (A == nullptr) {
      const T* src = S + ((b * n + k) * R + i) * m;
      for (int64_t j = threadIdx.x; j < m; j += blockDim.x) buf[j] = __ldg(src + j);
    } else {
      const T* src = S + (b * R + i) * m;
      const int32_t* ar = A + (b * R + i) * m;
      for (int64_t j = threadIdx.x; j < m; j += blockDim.x) buf[j] = (__ldg(ar + j) == k) ? __ldg(src + j) : T(0);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      T* ob = out + b * (int64_t)n * R * d + i * d;
      const uint32_t sbuf = smem_u32(buf);
      for (int r = 0, s = k; r < n; ++r, s = (s + 1 == n) ? 0 : s + 1) {   // block (r, s), s = (r + k) mod n
        T* dst = ob + (int64_t)r * R * d + (int64_t)s * m;
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(sbuf),
                     "r"(seg_bytes)
                     : "memory");
      }
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// Small blocks (C5: n = 16, m = 128, a 512-byte segment per block row): one unit = row i of all n blocks of a
// problem. The n segments are assembled in shared memory twice over (T_0 .. T_{n-1}, T_0 .. T_{n-2}), so every
// row r*R + i of the dense plan -- T_{(s - r) mod n}[i] for s = 0 .. n-1 -- is one contiguous window, written by
// ONE bulk store of d values (n stores of n*m values instead of n^2 stores of m).
template <typename T>
__global__ void __launch_bounds__(256) k_expand_rows(const T* __restrict__ S, const int32_t* __restrict__ A,
                                                     int64_t B, int n, int64_t m, int64_t R, T* __restrict__ out) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* bufs = reinterpret_cast<T*>(smem_raw);
  const int64_t d = (int64_t)n * m;
  const int64_t win = (int64_t)(2 * n - 1) * m;   // elements per slot
  const int64_t units = B * R;
  const uint32_t row_bytes = (uint32_t)(d * sizeof(T));
  int slot = 0;
  for (int64_t u = blockIdx.x; u < units; u += gridDim.x, slot ^= 1) {
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    __syncthreads();
    const int64_t b = u / R, i = u - b * R;
    T* buf = bufs + slot * win;
    for (int64_t idx = threadIdx.x; idx < d; idx += blockDim.x) {
      const int k = (int)(idx / m);
      const int64_t j = idx - (int64_t)k * m;
      T v;
      if (A == nullptr) {
        v = __ldg(S + ((b * n + k) * R + i) * m + j);
      } else {
        const int64_t o = (b * R + i) * m + j;
        v = (__ldg(A + o) == k) ? __ldg(S + o) : T(0);
      }
      buf[idx] = v;
      if (k < n - 1) buf[idx + d] = v;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int r = 0; r < n; ++r) {
        const int start = (n - r) % n;
        T* dst = out + (b * (int64_t)n * R + (int64_t)r * R + i) * d;
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
                     "r"(smem_u32(buf + (int64_t)start * m)), "r"(row_bytes)
                     : "memory");
      }
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// Which kernel launch_expand selects: 2 = k_expand_rows (whole dense rows from shared memory), 1 = k_expand_bulk
// (one segment, n bulk stores), 0 = k_expand (vector stores; ragged m).
int expand_path(int64_t n, int64_t m, int dtype) {
  const size_t esz = dtype == COT_F32 ? 4 : 8;
  const size_t rows_smem = 2 * (size_t)(2 * n - 1) * m * esz;
  if ((m * esz) % 16 == 0 && rows_smem <= 48 * 1024 && !getenv("COT_EXPAND_SEGMENTS")) return 2;
  if ((m * esz) % 16 == 0 && m * esz <= 32768) return 1;
  return 0;
}

cudaError_t launch_expand(const void* S, const int32_t* A, int64_t B, int64_t n, int64_t m, int dtype, void* out,
                          cudaStream_t s, int64_t R) {
  if (R < 0) R = m;
  const int sms = device_sm_count();
  const int64_t units = B * n * R;
  const int grid = (int)(units < (int64_t)sms * 16 ? units : (int64_t)sms * 16);
  const size_t esz = dtype == COT_F32 ? 4 : 8;
  const size_t rows_smem = 2 * (size_t)(2 * n - 1) * m * esz;
  const int path = expand_path(n, m, dtype);
  if (path == 2) {
    const int64_t runits = B * R;
    const int rgrid = (int)(runits < (int64_t)sms * 8 ? runits : (int64_t)sms * 8);
    if (dtype == COT_F32)
      k_expand_rows<float><<<rgrid, 256, rows_smem, s>>>((const float*)S, A, B, (int)n, m, R, (float*)out);
    else
      k_expand_rows<double><<<rgrid, 256, rows_smem, s>>>((const double*)S, A, B, (int)n, m, R, (double*)out);
    return cudaGetLastError();
  }
  if (path == 1) {
    const int64_t mpad = (m + 31) & ~int64_t(31);
    const size_t smem = 2 * mpad * esz;
    cudaError_t e;
    if (dtype == COT_F32) {
      e = cudaFuncSetAttribute(k_expand_bulk<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      k_expand_bulk<float><<<grid, 128, smem, s>>>((const float*)S, A, B, (int)n, m, R, (float*)out);
    } else {
      e = cudaFuncSetAttribute(k_expand_bulk<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      k_expand_bulk<double><<<grid, 128, smem, s>>>((const double*)S, A, B, (int)n, m, R, (double*)out);
    }
    return cudaGetLastError();
  }
  if (dtype == COT_F32) {
    if (m % 4 == 0)
      k_expand<float, 4><<<grid, 256, 0, s>>>((const float*)S, A, B, (int)n, m, R, (float*)out);
    else
      k_expand<float, 1><<<grid, 256, 0, s>>>((const float*)S, A, B, (int)n, m, R, (float*)out);
  } else {
    if (m % 2 == 0)
      k_expand<double, 2><<<grid, 256, 0, s>>>((const double*)S, A, B, (int)n, m, R, (double*)out);
    else
      k_expand<double, 1><<<grid, 256, 0, s>>>((const double*)S, A, B, (int)n, m, R, (double*)out);
  }
  return cudaGetLastError();
}

}  // namespace cot
