// common.cuh — small fp64 vector/matrix helpers and deterministic block primitives (sm_100a).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#define HD __host__ __device__ __forceinline__

namespace tac {

struct v3 { double x, y, z; };
HD v3 mk(double a, double b, double c) { return v3{a, b, c}; }
HD v3 operator+(v3 a, v3 b) { return v3{a.x + b.x, a.y + b.y, a.z + b.z}; }
HD v3 operator-(v3 a, v3 b) { return v3{a.x - b.x, a.y - b.y, a.z - b.z}; }
HD v3 operator-(v3 a) { return v3{-a.x, -a.y, -a.z}; }
HD v3 operator*(double s, v3 a) { return v3{s * a.x, s * a.y, s * a.z}; }
HD v3& operator+=(v3& a, v3 b) { a.x += b.x; a.y += b.y; a.z += b.z; return a; }
HD double dot(v3 a, v3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
HD v3 cross(v3 a, v3 b) { return v3{a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x}; }
HD double comp(v3 a, int i) { return i == 0 ? a.x : (i == 1 ? a.y : a.z); }
HD v3 ld3(const double* p) { return v3{p[0], p[1], p[2]}; }
HD void st3(double* p, v3 a) { p[0] = a.x; p[1] = a.y; p[2] = a.z; }
HD v3 vmin(v3 a, v3 b) { return v3{fmin(a.x, b.x), fmin(a.y, b.y), fmin(a.z, b.z)}; }
HD v3 vmax(v3 a, v3 b) { return v3{fmax(a.x, b.x), fmax(a.y, b.y), fmax(a.z, b.z)}; }

// 3x3 row-major matrices as double[9]
HD v3 mul33(const double* A, v3 v) {
  return v3{A[0] * v.x + A[1] * v.y + A[2] * v.z, A[3] * v.x + A[4] * v.y + A[5] * v.z,
            A[6] * v.x + A[7] * v.y + A[8] * v.z};
}
HD v3 mul33T(const double* A, v3 v) {  // Aᵀ v
  return v3{A[0] * v.x + A[3] * v.y + A[6] * v.z, A[1] * v.x + A[4] * v.y + A[7] * v.z,
            A[2] * v.x + A[5] * v.y + A[8] * v.z};
}
HD double det33(const double* F) {
  return F[0] * (F[4] * F[8] - F[5] * F[7]) - F[1] * (F[3] * F[8] - F[5] * F[6]) + F[2] * (F[3] * F[7] - F[4] * F[6]);
}
HD void inv33(const double* A, double* Ai) {
  double c00 = A[4] * A[8] - A[5] * A[7], c01 = A[5] * A[6] - A[3] * A[8], c02 = A[3] * A[7] - A[4] * A[6];
  double det = A[0] * c00 + A[1] * c01 + A[2] * c02;
  double id = 1.0 / det;
  Ai[0] = c00 * id; Ai[1] = (A[2] * A[7] - A[1] * A[8]) * id; Ai[2] = (A[1] * A[5] - A[2] * A[4]) * id;
  Ai[3] = c01 * id; Ai[4] = (A[0] * A[8] - A[2] * A[6]) * id; Ai[5] = (A[2] * A[3] - A[0] * A[5]) * id;
  Ai[6] = c02 * id; Ai[7] = (A[1] * A[6] - A[0] * A[7]) * id; Ai[8] = (A[0] * A[4] - A[1] * A[3]) * id;
}

// packed upper-triangular index of a symmetric n×n matrix (row-major upper): i <= j
HD int sym_idx(int i, int j, int n) {
  if (i > j) { int t = i; i = j; j = t; }
  return i * n - (i * (i - 1)) / 2 + (j - i);
}

// affine body: position of body-frame point xb under y = (t, A row-major)
HD v3 embed(const double* y, v3 xb) { return v3{y[0], y[1], y[2]} + mul33(y + 3, xb); }

// ------------------------------------------------------------------------------------------
// deterministic block reductions (fixed thread→element assignment and fixed tree)
// ------------------------------------------------------------------------------------------
#ifdef __CUDACC__
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ int warp_sum_i(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// All threads of the block must call; `red` is __shared__ double[32]. Returns the total to all.
__device__ __forceinline__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  double t = (lane < nw) ? red[lane] : 0.0;
  t = warp_sum(t);
  return t;
}
__device__ __forceinline__ double block_max(double v, double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_max(v);
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  double t = (lane < nw) ? red[lane] : -1.0e300;
  return warp_max(t);
}
__device__ __forceinline__ double block_min(double v, double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_min(v);
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  double t = (lane < nw) ? red[lane] : 1.0e300;
  return warp_min(t);
}
__device__ __forceinline__ int block_or(int v, int* red) {
  v = __syncthreads_or(v);
  return v;
}
// Exclusive scan of one int per thread over the block; returns the exclusive prefix; total in *tot.
// `sh` is __shared__ int[33].
__device__ __forceinline__ int block_excl_scan(int v, int* sh, int* tot) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  __syncthreads();
  if (lane == 31) sh[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int s = (lane < nw) ? sh[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < nw) sh[lane] = s;   // inclusive warp totals
  }
  __syncthreads();
  int base = (wid > 0) ? sh[wid - 1] : 0;
  int total = sh[nw - 1];
  __syncthreads();
  *tot = total;
  return base + x - v;
}
#endif

}  // namespace tac
