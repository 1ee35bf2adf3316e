// rpg_fit.cu — K3: the least-squares rational fit (poly::fit_rational,
// polyfit.hpp:337-427) on sm_100a.
//
// The reference forms the m x n sample matrix A (row k = [num monomials(x_k),
// -y_k den monomials(x_k)], polyfit.hpp:139-154), scales its columns to unit
// norm (equilibrate_columns, :219-229) and takes the right singular vector of
// the smallest singular value from Eigen's JacobiSVD (:162-169, :364-367).
// For m up to 10^6 that is an O(m n^2) job dominated by touching A.  Here:
//
//   K3a tsqr_tiles   rows are generated on the fly from (x_k, y_k) into SMEM
//                    tiles; every CTA folds its tiles into a running
//                    upper-triangular R with Householder reflections of the
//                    stacked [R; tile] (A is never materialised in HBM);
//   K3b tsqr_combine the per-CTA R factors are merged pairwise (tree);
//   K3c svd_small    one CTA: column norms of R (= those of A), R S with
//                    S = diag(1/||a_j||) — the R factor of the equilibrated
//                    A S, an exact identity — then a one-sided Jacobi SVD of
//                    R S (singular values and V of A S), the smallest right
//                    singular vector, c = v .* S;
//   K3d den_stats    q_k = den(x_k) . c_den over all samples: the positivity
//                    safeguard's trigger (polyfit.hpp:370-378).
//
// The normal equations (A^T A) are never formed: they would square the
// condition number of these Vandermonde-like matrices and break the
// 1e-10 sigma_1 rank cut (polyfit.hpp:171-177).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "rpg.h"
#include "rpg_fit.h"

namespace rpg_fit {

constexpr int kMaxCols = 64;   // n = |num basis| + |den basis|
constexpr int kTile = 128;     // rows per SMEM tile
constexpr int kFitThreads = 256;
constexpr int kFitWarps = kFitThreads / 32;

struct FitParams {
  int32_t m_lo, m_hi;           // unused by the tree kernels
  int32_t n_vars, nn, nd, n;    // basis sizes
  const double* X;              // m x n_vars
  const double* y;              // m
  const double* w;              // optional row weights (nullptr: 1)
  const uint8_t* exps;          // n x n_vars: numerator basis then denominator basis
  int64_t m;
  int32_t with_y_col;           // 1: append y as column n (TSQR of [V | y])
  int32_t num_only;             // 1: numerator block only (start-vector LS)
};

__device__ __forceinline__ double block_sum_d(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double r = 0.0;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) r += red[i];
  return r;
}

// Folds a tile T (rows x n, column-major with leading dimension ld) into the
// upper-triangular R (n x n, row-major) held in SMEM: Householder QR of the
// stacked [R; T], keeping the new R (LAPACK dlarfg/dlarf conventions).  T is
// destroyed.
__device__ void fold_tile(double* R, double* T, int rows, int ld, int n, double* red,
                          double* wbuf) {
  for (int j = 0; j < n; ++j) {
    double s = 0.0;
    for (int i = threadIdx.x; i < rows; i += blockDim.x) {
      const double t = T[j * ld + i];
      s = fma(t, t, s);
    }
    const double sig2 = block_sum_d(s, red);
    if (sig2 == 0.0) continue;  // column already reduced: H = I
    const double alpha = R[j * n + j];
    const double nrm = sqrt(fma(alpha, alpha, sig2));
    const double beta = alpha >= 0.0 ? -nrm : nrm;
    const double v0 = alpha - beta;
    const double tau = (beta - alpha) / beta;
    const double inv_v0 = 1.0 / v0;
    // w_k = R[j][k] + sum_i v_i T[i][k], v_i = T[i][j] / v0, for k > j
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int k = j + 1 + warp; k < n; k += kFitWarps) {
      double d = 0.0;
      for (int i = lane; i < rows; i += 32) d = fma(T[j * ld + i], T[k * ld + i], d);
      for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
      if (lane == 0) wbuf[k] = fma(d, inv_v0, R[j * n + k]);
    }
    __syncthreads();
    if (threadIdx.x == 0) R[j * n + j] = beta;
    for (int k = j + 1 + (int)threadIdx.x; k < n; k += blockDim.x)
      R[j * n + k] -= tau * wbuf[k];
    const int cols = n - j - 1;
    for (int e = threadIdx.x; e < rows * cols; e += blockDim.x) {
      const int k = j + 1 + e / rows, i = e % rows;
      T[k * ld + i] -= (tau * wbuf[k]) * (T[j * ld + i] * inv_v0);
    }
    __syncthreads();
  }
}

// eval_monomial (polyfit.hpp:96-105) for one sample and exponent row.
__device__ __forceinline__ double monomial(const double* x, const uint8_t* e, int nv) {
  double m = 1.0;
  for (int v = 0; v < nv; ++v) {
    double p = 1.0;
    for (int t = 0; t < e[v]; ++t) p *= x[v];
    m *= p;
  }
  return m;
}

// Builds rows [r0, r0+kTile) of the (optionally weighted) sample matrix into
// T (column-major, ld = kTile); rows past m are zero.
__device__ void build_tile(const FitParams& F, int64_t r0, double* T, const uint8_t* sexps) {
  const int ncols = F.num_only ? F.nn + F.with_y_col : F.n;
  for (int i = threadIdx.x; i < kTile; i += blockDim.x) {
    const int64_t r = r0 + i;
    if (r >= F.m) {
      for (int k = 0; k < ncols; ++k) T[k * kTile + i] = 0.0;
      continue;
    }
    double x[RPG_MAX_VARS];
    for (int v = 0; v < F.n_vars; ++v) x[v] = F.X[r * F.n_vars + v];
    const double yv = F.y[r];
    const double wr = F.w ? F.w[r] : 1.0;
    for (int k = 0; k < F.nn; ++k) {
      const double mo = monomial(x, sexps + k * F.n_vars, F.n_vars);
      T[k * kTile + i] = F.w ? mo / wr : mo;
    }
    if (F.num_only) {
      if (F.with_y_col) T[F.nn * kTile + i] = yv;
      continue;
    }
    for (int k = 0; k < F.nd; ++k) {
      const double mo = monomial(x, sexps + (F.nn + k) * F.n_vars, F.n_vars);
      const double a = -yv * mo;
      T[(F.nn + k) * kTile + i] = F.w ? a / wr : a;
    }
  }
}

// K3a: each CTA folds tiles blockIdx.x, blockIdx.x + gridDim.x, ... into its
// own R (written to Rout[blockIdx.x]).
__global__ void __launch_bounds__(kFitThreads)
tsqr_tiles(const FitParams F, double* __restrict__ Rout) {
  extern __shared__ __align__(16) double fsm[];
  const int ncols = F.num_only ? F.nn + F.with_y_col : F.n;
  double* R = fsm;                        // kMaxCols^2
  double* T = R + kMaxCols * kMaxCols;    // kTile * kMaxCols
  double* red = T + kTile * kMaxCols;     // 32
  double* wbuf = red + 32;                // kMaxCols
  uint8_t* sexps = reinterpret_cast<uint8_t*>(wbuf + kMaxCols);
  for (int e = threadIdx.x; e < F.n * F.n_vars; e += blockDim.x) sexps[e] = F.exps[e];
  for (int e = threadIdx.x; e < ncols * ncols; e += blockDim.x) R[e] = 0.0;
  __syncthreads();
  const int64_t tiles = (F.m + kTile - 1) / kTile;
  for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    build_tile(F, t * kTile, T, sexps);
    __syncthreads();
    fold_tile(R, T, kTile, kTile, ncols, red, wbuf);
  }
  __syncthreads();
  double* out = Rout + (size_t)blockIdx.x * ncols * ncols;
  for (int e = threadIdx.x; e < ncols * ncols; e += blockDim.x) out[e] = R[e];
}

// K3b: R[2b] <- qr([R[2b]; R[2b+1]]).R for b < count/2 (tree level).
__global__ void __launch_bounds__(kFitThreads)
tsqr_combine(double* __restrict__ Rs, int count, int n) {
  extern __shared__ __align__(16) double fsm[];
  double* R = fsm;
  double* T = R + kMaxCols * kMaxCols;
  double* red = T + kMaxCols * kMaxCols;
  double* wbuf = red + 32;
  const int a = 2 * blockIdx.x, b = a + 1;
  if (b >= count) return;
  const double* Ra = Rs + (size_t)a * n * n;
  const double* Rb = Rs + (size_t)b * n * n;
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    R[e] = Ra[e];
    const int i = e / n, k = e % n;  // Rb row-major -> T column-major (ld = n)
    T[k * n + i] = Rb[e];
  }
  __syncthreads();
  fold_tile(R, T, n, n, n, red, wbuf);
  __syncthreads();
  double* out = Rs + (size_t)a * n * n;
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) out[e] = R[e];
}

// One-sided (Hestenes) Jacobi SVD of the n x n matrix M (column-major in
// SMEM): M V = U diag(sigma).  Round-robin pair ordering, one warp per pair.
__device__ void jacobi_svd(double* M, double* V, int n, int* rot_flag) {
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) V[e] = (e / n == e % n) ? 1.0 : 0.0;
  __syncthreads();
  const int np = (n + 1) & ~1;  // even number of slots (slot n is a phantom zero column)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int sweep = 0; sweep < 80; ++sweep) {
    if (threadIdx.x == 0) *rot_flag = 0;
    __syncthreads();
    for (int step = 0; step < np - 1; ++step) {
      for (int pr = warp; pr < np / 2; pr += kFitWarps) {
        // round-robin pairing: slot 0 fixed, others rotate
        int a = pr == 0 ? 0 : 1 + (pr - 1 + step) % (np - 1);
        int b = 1 + (np - 2 - pr + step) % (np - 1);
        if (a > b) { const int t = a; a = b; b = t; }
        if (b >= n) continue;
        double aa = 0, bb = 0, ab = 0;
        for (int i = lane; i < n; i += 32) {
          const double x = M[a * n + i], z = M[b * n + i];
          aa = fma(x, x, aa);
          bb = fma(z, z, bb);
          ab = fma(x, z, ab);
        }
        for (int o = 16; o > 0; o >>= 1) {
          aa += __shfl_xor_sync(0xffffffffu, aa, o);
          bb += __shfl_xor_sync(0xffffffffu, bb, o);
          ab += __shfl_xor_sync(0xffffffffu, ab, o);
        }
        if (ab == 0.0 || fabs(ab) <= 1e-15 * sqrt(aa * bb)) continue;
        const double zeta = (bb - aa) / (2.0 * ab);
        const double t = (zeta >= 0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double cs = 1.0 / sqrt(1.0 + t * t), sn = cs * t;
        for (int i = lane; i < n; i += 32) {
          const double x = M[a * n + i], z = M[b * n + i];
          M[a * n + i] = cs * x - sn * z;
          M[b * n + i] = sn * x + cs * z;
          const double vx = V[a * n + i], vz = V[b * n + i];
          V[a * n + i] = cs * vx - sn * vz;
          V[b * n + i] = sn * vx + cs * vz;
        }
        if (lane == 0) *rot_flag = 1;
      }
      __syncthreads();
    }
    if (*rot_flag == 0) break;
    __syncthreads();
  }
}

// K3c: one CTA.  In: R (n x n row-major).  Out: sigma (n, descending),
// Vs (n x n column-major, columns = right singular vectors of A S, sorted),
// col_scale (n), c (n) = V[:, n-1] .* col_scale.
__global__ void __launch_bounds__(kFitThreads)
svd_small(const double* __restrict__ R, int n, double* __restrict__ sigma,
          double* __restrict__ Vout, double* __restrict__ col_scale,
          double* __restrict__ Uout, int equilibrate) {
  extern __shared__ __align__(16) double fsm[];
  double* M = fsm;                 // n x n column-major
  double* V = M + kMaxCols * kMaxCols;
  double* nrm = V + kMaxCols * kMaxCols;
  int* order = reinterpret_cast<int*>(nrm + kMaxCols);
  int* flag = order + kMaxCols;
  // column norms of R == column norms of A (Q orthonormal)
  for (int k = threadIdx.x; k < n; k += blockDim.x) {
    double s = 0.0;
    for (int i = 0; i <= k; ++i) s = fma(R[i * n + k], R[i * n + k], s);
    const double cn = sqrt(s);
    col_scale[k] = (equilibrate && cn > 0.0) ? 1.0 / cn : 1.0;
    nrm[k] = col_scale[k];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int k = e / n, i = e % n;  // M column k, row i
    M[k * n + i] = R[i * n + k] * nrm[k];
  }
  __syncthreads();
  jacobi_svd(M, V, n, flag);
  for (int k = threadIdx.x; k < n; k += blockDim.x) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s = fma(M[k * n + i], M[k * n + i], s);
    nrm[k] = sqrt(s);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 0; k < n; ++k) order[k] = k;
    for (int a = 1; a < n; ++a) {  // stable insertion sort, descending
      const int v = order[a];
      int b = a - 1;
      while (b >= 0 && nrm[order[b]] < nrm[v]) {
        order[b + 1] = order[b];
        --b;
      }
      order[b + 1] = v;
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int k = e / n, i = e % n;
    const int src = order[k];
    Vout[k * n + i] = V[src * n + i];
    if (Uout) Uout[k * n + i] = nrm[src] > 0.0 ? M[src * n + i] / nrm[src] : 0.0;
  }
  for (int k = threadIdx.x; k < n; k += blockDim.x) sigma[k] = nrm[order[k]];
}

// K3d: den(x_k) . c_den over all samples -> {min q, max q, sum |q|, min |q|}.
__global__ void den_stats(const FitParams F, const double* __restrict__ cden,
                          double* __restrict__ partial) {
  extern __shared__ __align__(16) double fsm[];
  double* red = fsm;
  uint8_t* sexps = reinterpret_cast<uint8_t*>(red + 32);
  for (int e = threadIdx.x; e < F.nd * F.n_vars; e += blockDim.x)
    sexps[e] = F.exps[F.nn * F.n_vars + e];
  __syncthreads();
  double qmin = INFINITY, qmax = -INFINITY, asum = 0.0, amin = INFINITY;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < F.m;
       r += (int64_t)gridDim.x * blockDim.x) {
    double x[RPG_MAX_VARS];
    for (int v = 0; v < F.n_vars; ++v) x[v] = F.X[r * F.n_vars + v];
    double q = 0.0;
    for (int k = 0; k < F.nd; ++k) q = fma(monomial(x, sexps + k * F.n_vars, F.n_vars), cden[k], q);
    qmin = fmin(qmin, q);
    qmax = fmax(qmax, q);
    asum += fabs(q);
    amin = fmin(amin, fabs(q));
  }
  // block reductions (min via -max trick avoided: do four passes)
  double v[4] = {qmin, -qmax, asum, amin};
  for (int j = 0; j < 4; ++j) {
    double t = v[j];
    for (int o = 16; o > 0; o >>= 1) {
      const double u = __shfl_xor_sync(0xffffffffu, t, o);
      t = j == 2 ? t + u : fmin(t, u);
    }
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = t;
    __syncthreads();
    if (threadIdx.x == 0) {
      double r = red[0];
      for (int i = 1; i < (int)(blockDim.x >> 5); ++i) r = j == 2 ? r + red[i] : fmin(r, red[i]);
      partial[blockIdx.x * 4 + j] = r;
    }
  }
}

}  // namespace rpg_fit
