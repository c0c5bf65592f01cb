// K-AGG: C-LOT aggregation G_ij = min_k C_ijk with the smallest argmin.
// HBM-streaming: every C element is read once with 128-bit loads (coalesced along j), the k loop is
// unrolled so that 8 independent loads per thread are in flight. Comparisons only => bit-exact.
#include "common.cuh"
#include "internal.h"

namespace cot {

template <typename T, int V>
struct Vec;
template <>
struct Vec<float, 4> {
  using type = float4;
};
template <>
struct Vec<double, 2> {
  using type = double2;
};
template <>
struct Vec<float, 1> {
  using type = float;
};
template <>
struct Vec<double, 1> {
  using type = double;
};
template <>
struct Vec<int, 4> {
  using type = int4;
};
template <>
struct Vec<int, 2> {
  using type = int2;
};
template <>
struct Vec<int, 1> {
  using type = int;
};


template <typename T, int V>
__device__ __forceinline__ T lane(const typename Vec<T, V>::type& v, int q) {
  if constexpr (V == 1) {
    return v;
  } else if constexpr (V == 2) {
    return q == 0 ? v.x : v.y;
  } else {
    return q == 0 ? v.x : (q == 1 ? v.y : (q == 2 ? v.z : v.w));
  }
}
template <typename T, int V>
__device__ __forceinline__ void set_lane(typename Vec<T, V>::type& v, int q, T x) {
  if constexpr (V == 1) {
    v = x;
  } else if constexpr (V == 2) {
    if (q == 0) v.x = x; else v.y = x;
  } else {
    if (q == 0) v.x = x; else if (q == 1) v.y = x; else if (q == 2) v.z = x; else v.w = x;
  }
}

// One thread per V consecutive (i,j) entries of one problem; grid-stride over B*m*m/V groups.
template <typename T, int V>
__global__ void __launch_bounds__(256) k_aggregate(const T* __restrict__ C, int64_t B, int n, int64_t mm,
                                                   T* __restrict__ G, int32_t* __restrict__ A,
                                                   int32_t* __restrict__ nonfinite) {
  using VT = typename Vec<T, V>::type;
  using IT = typename Vec<int, V>::type;
  const int64_t groups = B * mm / V;
  int bad = 0;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < groups; g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = g * V;           // first flat (b, i, j) element
    const int64_t b = e / mm, ij = e - b * mm;
    const VT* src = reinterpret_cast<const VT*>(C + b * n * mm + ij);
    const int64_t kstride = mm / V;
    T best[V];
    int arg[V];
    {
      VT v0 = __ldcs(src);
#pragma unroll
      for (int q = 0; q < V; ++q) {
        best[q] = lane<T, V>(v0, q);
        arg[q] = 0;
        bad += !finite_f(best[q]);
      }
    }
    int k = 1;
    for (; k + 8 <= n; k += 8) {
      VT v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = __ldcs(src + (int64_t)(k + u) * kstride);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
#pragma unroll
        for (int q = 0; q < V; ++q) {
          const T c = lane<T, V>(v[u], q);
          bad += !finite_f(c);
          if (c < best[q]) {   // strict: keeps the smallest k among ties; -0 vs +0 is a tie
            best[q] = c;
            arg[q] = k + u;
          }
        }
      }
    }
    for (; k < n; ++k) {
      VT v = __ldcs(src + (int64_t)k * kstride);
#pragma unroll
      for (int q = 0; q < V; ++q) {
        const T c = lane<T, V>(v, q);
        bad += !finite_f(c);
        if (c < best[q]) {
          best[q] = c;
          arg[q] = k;
        }
      }
    }
    VT gv;
    IT av;
#pragma unroll
    for (int q = 0; q < V; ++q) {
      set_lane<T, V>(gv, q, best[q]);
      set_lane<int, V>(av, q, arg[q]);
    }
    reinterpret_cast<VT*>(G)[g] = gv;
    reinterpret_cast<IT*>(A)[g] = av;
  }
  // one atomic per warp at most
  const unsigned any = __ballot_sync(0xffffffffu, bad != 0);
  if (any) {
    const int tot = warp_sum(bad);
    if ((threadIdx.x & 31) == 0 && nonfinite) atomicAdd(nonfinite, tot);
  }
}

// NEXT-1 (Alg. 2 line 1, in the G-shifted form): S_ij = sum_k exp((G_ij - C_ijk)/eps) in [1, n],
// i.e. K_ij = S_ij exp(-G_ij/eps) (eq. def_Kij) without over/underflow. One streaming pass.
template <typename T, int V>
__global__ void __launch_bounds__(256) k_precompute(const T* __restrict__ C, const T* __restrict__ G, int64_t B,
                                                    int n, int64_t mm, const double* __restrict__ eps,
                                                    T* __restrict__ S) {
  using VT = typename Vec<T, V>::type;
  const int64_t groups = B * mm / V;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < groups; g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = g * V;
    const int64_t b = e / mm, ij = e - b * mm;
    const VT* src = reinterpret_cast<const VT*>(C + b * n * mm + ij);
    const int64_t kstride = mm / V;
    const VT gv = reinterpret_cast<const VT*>(G)[g];
    const double inv_eps = 1.0 / eps[b];
    T gg[V], acc[V];
#pragma unroll
    for (int q = 0; q < V; ++q) {
      gg[q] = lane<T, V>(gv, q);
      acc[q] = T(0);
    }
    for (int k = 0; k < n; ++k) {
      const VT v = __ldcs(src + (int64_t)k * kstride);
#pragma unroll
      for (int q = 0; q < V; ++q) {
        if constexpr (sizeof(T) == 4)
          acc[q] += ex2((gg[q] - lane<T, V>(v, q)) * (float)(COT_LOG2E * inv_eps));
        else
          acc[q] += exp((gg[q] - lane<T, V>(v, q)) * inv_eps);
      }
    }
    VT out;
#pragma unroll
    for (int q = 0; q < V; ++q) set_lane<T, V>(out, q, acc[q]);
    reinterpret_cast<VT*>(S)[g] = out;
  }
}

cudaError_t launch_precompute(const void* C, const void* G, int64_t B, int64_t n, int64_t m, int dtype,
                              const double* eps, void* S, cudaStream_t s) {
  const int64_t mm = m * m;
  const int sms = device_sm_count();
  auto grid_for = [&](int64_t groups) {
    int64_t g = (groups + 255) / 256;
    const int64_t cap = (int64_t)sms * 8;
    return (int)(g < cap ? (g > 0 ? g : 1) : cap);
  };
  if (dtype == COT_F32) {
    if (mm % 4 == 0)
      k_precompute<float, 4><<<grid_for(B * mm / 4), 256, 0, s>>>((const float*)C, (const float*)G, B, (int)n, mm, eps,
                                                                  (float*)S);
    else
      k_precompute<float, 1><<<grid_for(B * mm), 256, 0, s>>>((const float*)C, (const float*)G, B, (int)n, mm, eps,
                                                              (float*)S);
  } else {
    if (mm % 2 == 0)
      k_precompute<double, 2><<<grid_for(B * mm / 2), 256, 0, s>>>((const double*)C, (const double*)G, B, (int)n, mm,
                                                                   eps, (double*)S);
    else
      k_precompute<double, 1><<<grid_for(B * mm), 256, 0, s>>>((const double*)C, (const double*)G, B, (int)n, mm, eps,
                                                               (double*)S);
  }
  return cudaGetLastError();
}

cudaError_t launch_aggregate(const void* C, int64_t B, int64_t n, int64_t m, int dtype, void* G, int32_t* A,
                             int32_t* nonfinite, cudaStream_t s, int64_t R) {
  const int64_t mm = (R < 0 ? m : R) * m;   // elements per block (R rows of m columns)
  if (nonfinite) {
    cudaError_t e = cudaMemsetAsync(nonfinite, 0, sizeof(int32_t), s);
    if (e != cudaSuccess) return e;
  }
  const int sms = device_sm_count();
  auto grid_for = [&](int64_t groups) {
    int64_t g = (groups + 255) / 256;
    const int64_t cap = (int64_t)sms * 8;
    return (int)(g < cap ? (g > 0 ? g : 1) : cap);
  };
  if (dtype == COT_F32) {
    if (mm % 4 == 0) {
      k_aggregate<float, 4><<<grid_for(B * mm / 4), 256, 0, s>>>((const float*)C, B, (int)n, mm, (float*)G, A, nonfinite);
    } else {
      k_aggregate<float, 1><<<grid_for(B * mm), 256, 0, s>>>((const float*)C, B, (int)n, mm, (float*)G, A, nonfinite);
    }
  } else {
    if (mm % 2 == 0) {
      k_aggregate<double, 2><<<grid_for(B * mm / 2), 256, 0, s>>>((const double*)C, B, (int)n, mm, (double*)G, A,
                                                                  nonfinite);
    } else {
      k_aggregate<double, 1><<<grid_for(B * mm), 256, 0, s>>>((const double*)C, B, (int)n, mm, (double*)G, A,
                                                              nonfinite);
    }
  }
  return cudaGetLastError();
}

}  // namespace cot
