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
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <map>
#include <mutex>
#include <thread>
#include <vector>

#include "rpg.h"
#include "rpg_fit.h"

namespace rpg_fit {

constexpr int kMaxCols = 64;   // n = |num basis| + |den basis|
static_assert(kMaxCols == RPG_FIT_MAX_COLS, "rpg.h RPG_FIT_MAX_COLS");
#ifndef RPG_FIT_KTILE
#define RPG_FIT_KTILE 256
#endif
constexpr int kTile = RPG_FIT_KTILE;  // rows per SMEM tile of the TSQR leaves
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
  const double* Dm;             // optional m x nd raw denominator monomials (den_pass)
  int32_t den01;                // 1: n_vars <= 4 and every denominator exponent <= 1
  int32_t den_lat3;             // 1: 3 variables, denominator basis = monomial_basis({1,1,1})
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

// fold_tile for a leaf tile of exactly blockDim.x rows (thread i owns row
// i): the same Householder arithmetic in the same order — bit-identical —
// with two barriers per column instead of four (column j+1's norm is
// reduced by the threads that just updated it, inside column j's update
// phase) and no per-element index division in the update.
__device__ void fold_tile_leaf(double* R, double* T, int ld, int n, double* red, double* wbuf) {
  const int i = threadIdx.x, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  auto warp_sq = [&](int col) {
    const double t = T[col * ld + i];
    double v = t * t;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[warp] = v;
  };
  warp_sq(0);
  __syncthreads();
  for (int j = 0; j < n; ++j) {
    double sig2 = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) sig2 += red[w];
    if (sig2 == 0.0) {  // column already reduced: H = I
      __syncthreads();  // every thread has read red
      if (j + 1 < n) warp_sq(j + 1);
      __syncthreads();
      continue;
    }
    const double alpha = R[j * n + j];
    const double nrm = sqrt(fma(alpha, alpha, sig2));
    const double beta = alpha >= 0.0 ? -nrm : nrm;
    const double v0 = alpha - beta;
    const double tau = (beta - alpha) / beta;
    const double inv_v0 = 1.0 / v0;
    // w_k = R[j][k] + sum_i v_i T[i][k], v_i = T[i][j] / v0, for k > j:
    // warp per k, two k per pass (independent chains), the lane's rows of
    // column j in registers; per k the row order and shuffle tree of
    // fold_tile.
    constexpr int kRows = kFitThreads / 32;
    double tj[kRows];
#pragma unroll
    for (int rr = 0; rr < kRows; ++rr) tj[rr] = T[j * ld + lane + 32 * rr];
    for (int k = j + 1 + warp; k < n; k += 2 * kFitWarps) {
      const int k2 = k + kFitWarps;
      const bool two = k2 < n;
      const int kk2 = two ? k2 : k;
      double d = 0.0, d2 = 0.0;
#pragma unroll
      for (int rr = 0; rr < kRows; ++rr) {
        d = fma(tj[rr], T[k * ld + lane + 32 * rr], d);
        d2 = fma(tj[rr], T[kk2 * ld + lane + 32 * rr], d2);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        d += __shfl_xor_sync(0xffffffffu, d, o);
        d2 += __shfl_xor_sync(0xffffffffu, d2, o);
      }
      if (lane == 0) {
        wbuf[k] = fma(d, inv_v0, R[j * n + k]);
        if (two) wbuf[k2] = fma(d2, inv_v0, R[j * n + k2]);
      }
    }
    __syncthreads();  // wbuf complete; red read by every thread
    if (i == 0) R[j * n + j] = beta;
    for (int k = j + 1 + i; k < n; k += blockDim.x) R[j * n + k] -= tau * wbuf[k];
    const double vi = T[j * ld + i] * inv_v0;
    int k = j + 1;
    for (; k + 4 <= n; k += 4) {  // four independent updates per pass
      double t[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) t[u] = T[(k + u) * ld + i];
#pragma unroll
      for (int u = 0; u < 4; ++u) t[u] -= (tau * wbuf[k + u]) * vi;
#pragma unroll
      for (int u = 0; u < 4; ++u) T[(k + u) * ld + i] = t[u];
    }
    for (; k < n; ++k) T[k * ld + i] -= (tau * wbuf[k]) * vi;
    if (j + 1 < n) warp_sq(j + 1);
    __syncthreads();
  }
}

// eval_monomial (polyfit.hpp:96-105) for one sample and exponent row.
__device__ __forceinline__ double monomial(const double (&x)[RPG_MAX_VARS], const uint8_t* e, int nv) {
  // Unrolled over the variables so x stays in registers (a runtime index
  // would put it in local memory); the product order is eval_monomial's.
  double m = 1.0;
#pragma unroll
  for (int v = 0; v < RPG_MAX_VARS; ++v) {
    if (v < nv) {
      double p = 1.0;
      for (int t = 0; t < e[v]; ++t) p *= x[v];
      m *= p;
    }
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
#pragma unroll
    for (int v = 0; v < RPG_MAX_VARS; ++v) x[v] = v < F.n_vars ? F.X[r * F.n_vars + v] : 0.0;
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
  double* R = fsm;                        // ncols^2
  double* T = R + ncols * ncols;          // kTile * ncols
  double* red = T + kTile * ncols;        // 32
  double* wbuf = red + 32;                // kMaxCols
  uint8_t* sexps = reinterpret_cast<uint8_t*>(wbuf + kMaxCols);
  for (int e = threadIdx.x; e < F.n * F.n_vars; e += blockDim.x) sexps[e] = F.exps[e];
  for (int e = threadIdx.x; e < ncols * ncols; e += blockDim.x) R[e] = 0.0;
  __syncthreads();
  const int64_t tiles = (F.m + kTile - 1) / kTile;
  for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    build_tile(F, t * kTile, T, sexps);
    __syncthreads();
    if (kTile == kFitThreads) fold_tile_leaf(R, T, kTile, ncols, red, wbuf);
    else fold_tile(R, T, kTile, kTile, ncols, red, wbuf);
  }
  __syncthreads();
  double* out = Rout + (size_t)blockIdx.x * ncols * ncols;
  for (int e = threadIdx.x; e < ncols * ncols; e += blockDim.x) out[e] = R[e];
}

// K3b: one tree level of radix kCombine: Rout[b] <- qr([Rin[kb]; Rin[kb+1];
// ...; Rin[kb+k-1]]).R — the first factor is the running R, the others are
// stacked as one (k-1) n-row tile (fewer, wider levels: each fold costs n
// block-synchronised column steps whatever its height).  Ping-pong buffers.
constexpr int kCombine = 8;

__global__ void __launch_bounds__(kFitThreads)
tsqr_combine(const double* __restrict__ Rs, int count, int n, double* __restrict__ Rout) {
  extern __shared__ __align__(16) double fsm[];
  const int first = kCombine * blockIdx.x;
  const int k = min(kCombine, count - first);  // factors in this group
  const int rows = (k - 1) * n;
  double* R = fsm;
  double* T = R + n * n;                        // rows x n, column-major (ld = rows)
  double* red = T + (size_t)(kCombine - 1) * n * n;
  double* wbuf = red + 32;
  const double* Ra = Rs + (size_t)first * n * n;
  double* out = Rout + (size_t)blockIdx.x * n * n;
  if (k == 1) {
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) out[e] = Ra[e];
    return;
  }
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) R[e] = Ra[e];
  for (int e = threadIdx.x; e < rows * n; e += blockDim.x) {
    const int f = e / (n * n), w = e % (n * n);  // factor f+1, entry (i, col) row-major
    const int i = w / n, col = w % n;
    T[col * rows + f * n + i] = Ra[(size_t)(f + 1) * n * n + w];
  }
  __syncthreads();
  fold_tile(R, T, rows, rows, n, red, wbuf);
  __syncthreads();
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
      for (int pr = warp; pr < np / 2; pr += (int)(blockDim.x >> 5)) {
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
// Threads of svd_small: one warp per rotation pair of a round-robin step.
__host__ __device__ inline int svd_threads(int n) {
  const int pairs = ((n + 1) & ~1) / 2;
  return 32 * (pairs < 8 ? 8 : pairs > 32 ? 32 : pairs);
}

__global__ void __launch_bounds__(1024)
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
#pragma unroll
    for (int v = 0; v < RPG_MAX_VARS; ++v) x[v] = v < F.n_vars ? F.X[r * F.n_vars + v] : 0.0;
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

namespace rpg_fit {

// Final small reductions / normalisation on the device (one warp-sized CTA).
// stats: G x 4 partials of den_stats.  out_flags[0]: safeguard trigger.
__global__ void den_stats_final(const double* __restrict__ partial, int G, int64_t m,
                                int* __restrict__ trigger, double* __restrict__ stats) {
  if (threadIdx.x != 0) return;
  double qmin = INFINITY, nqmax = INFINITY, asum = 0.0, amin = INFINITY;
  for (int g = 0; g < G; ++g) {
    qmin = fmin(qmin, partial[g * 4 + 0]);
    nqmax = fmin(nqmax, partial[g * 4 + 1]);
    asum += partial[g * 4 + 2];
    amin = fmin(amin, partial[g * 4 + 3]);
  }
  const double qmax = -nqmax;
  const double mean_mag = asum / (double)m;
  // polyfit.hpp:375-378
  const bool sign_mixed = qmin < 0.0 && qmax > 0.0;
  const bool pinched = mean_mag > 0.0 && amin < 1e-4 * mean_mag;
  *trigger = (sign_mixed || pinched) ? 1 : 0;
  stats[0] = qmin;
  stats[1] = qmax;
  stats[2] = mean_mag;
  stats[3] = amin;
}

// make_ratfunc_from_coeffs (polyfit.hpp:185-213) + numerical_rank
// (polyfit.hpp:171-177).  status: 0 ok, 1 all-zero vector, 2 zero denominator.
__global__ void fit_finalize(double* __restrict__ c, int nn, int nd, const double* __restrict__ sigma,
                             int nsig, double rank_tol, int* __restrict__ status,
                             int* __restrict__ rank) {
  if (threadIdx.x != 0) return;
  const int n = nn + nd;
  double s = 0.0;
  for (int k = 0; k < n; ++k) s = fma(c[k], c[k], s);
  const double norm = sqrt(s);
  int r = 0;
  if (nsig > 0 && sigma[0] > 0.0)
    for (int i = 0; i < nsig; ++i) r += sigma[i] >= rank_tol * sigma[0];
  *rank = r;
  if (norm == 0.0) {
    *status = 1;
    return;
  }
  for (int k = 0; k < n; ++k) c[k] /= norm;
  int first = -1;
  for (int j = 0; j < nd; ++j)
    if (fabs(c[nn + j]) > 1e-10) {
      first = j;
      break;
    }
  if (first < 0) {
    *status = 2;
    return;
  }
  if (c[nn + first] < 0.0)
    for (int k = 0; k < n; ++k) c[k] = -c[k];
  *status = 0;
}

__global__ void smallest_vector(const double* __restrict__ V, const double* __restrict__ col_scale,
                                int n, double* __restrict__ c) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) c[i] = V[(n - 1) * n + i] * col_scale[i];
}

__global__ void all_finite(const double* __restrict__ a, int64_t count, int* __restrict__ bad) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    if (!isfinite(a[i])) *bad = 1;
}

}  // namespace rpg_fit

namespace rpg_fit {

// ---------------------------------------------------------------------------
// Positivity safeguard (polyfit.hpp:242-311, 369-414) — device kernels.

// Column sums of the denominator monomials: g = Q.colwise().sum() / S_den.
__global__ void den_colsum(const FitParams F, double* __restrict__ partial) {
  extern __shared__ __align__(16) double fsm[];
  double* acc = fsm;  // nd x (blockDim/32)
  uint8_t* sexps = reinterpret_cast<uint8_t*>(acc + kMaxCols * kFitWarps);
  for (int e = threadIdx.x; e < F.nd * F.n_vars; e += blockDim.x)
    sexps[e] = F.exps[F.nn * F.n_vars + e];
  __syncthreads();
  double loc[kMaxCols];
  for (int k = 0; k < F.nd; ++k) loc[k] = 0.0;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < F.m;
       r += (int64_t)gridDim.x * blockDim.x) {
    double x[RPG_MAX_VARS];
#pragma unroll
    for (int v = 0; v < RPG_MAX_VARS; ++v) x[v] = v < F.n_vars ? F.X[r * F.n_vars + v] : 0.0;
    for (int k = 0; k < F.nd; ++k) loc[k] += monomial(x, sexps + k * F.n_vars, F.n_vars);
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  for (int k = 0; k < F.nd; ++k) {
    double t = loc[k];
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (l == 0) acc[k * kFitWarps + w] = t;
  }
  __syncthreads();
  for (int k = threadIdx.x; k < F.nd; k += blockDim.x) {
    double t = 0.0;
    for (int i = 0; i < kFitWarps; ++i) t += acc[k * kFitWarps + i];
    partial[(size_t)blockIdx.x * F.nd + k] = t;
  }
}

// One pass over the samples for the denominator values q_k = D_k . cd
// (cd: raw-coordinate denominator coefficients) at up to kAlphas candidate
// vectors cd + alpha_a * dd: per candidate min q and sum log q; with
// `newton`, for candidate 0 also sum (1/q) D_k and sum (1/q^2) D_k D_k^T.
constexpr int kAlphas = 4;
constexpr int kPassRows = 256;

// Device-side control of the positivity minimizer's Newton / line-search loop
// (positive_den_minimizer, polyfit.hpp:242-311), so the whole loop runs as a
// stream of kernels without a host round trip per iteration.
enum { kMinNewton = 0, kMinLine = 1, kMinDone = 2, kMinFail = 3 };
struct MinCtl {
  int phase, outer, inner, n_alpha;
  double mu, phi0, decrement, alpha;  // alpha: first candidate of the next line pass
  double al[kAlphas];
  long long tail_cycles[2];           // RPG_FIT_TRACE: serial tail time (Newton, line)
  long long newton_parts[3];          // ... of Newton steps: final fold, staging, solve
  int n_steps[2];
  // %globaltimer ns: CTA 0's start of the current step, end of the previous
  // step; summed sample-pass span (start -> last CTA's arrival) and
  // inter-step gap (previous end -> start).
  unsigned long long t_start, t_prev_end, pass_ns, gap_ns, tail_ns, t_arrive, t_first;
};

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// Candidate source of a controlled den_pass: c, dc in equilibrated
// coordinates, S the column scale.
struct CtlSrc {
  const MinCtl* ctl;
  const double* c;
  const double* dc;
  const double* S;
};

// frexp for the running log-sum products: integer exponent split on the
// high word for normal numbers, frexp otherwise (zero, subnormal, inf, NaN).
__device__ __forceinline__ double split_mant(double q, int& e) {
  const int hi = __double2hiint(q);
  const int ex = (hi >> 20) & 0x7ff;
  if (ex > 0 && ex < 0x7ff) {
    e += ex - 1022;
    return __hiloint2double((hi & 0x800fffff) | (1022 << 20), __double2loint(q));
  }
  int e2;
  const double m = frexp(q, &e2);
  e += e2;
  return m;
}

// |v| in [2^-500, 2^500) (biased exponent in [523, 1523)): products of two
// such numbers are normal.
__device__ __forceinline__ bool mid_range(double v) {
  return (unsigned)(((__double2hiint(v) >> 20) & 0x7ff) - 523) < 1000u;
}

// Raw denominator monomials of every sample (m x nd), computed once per fit
// and read by every sample pass of the safeguard instead of recomputed.
__global__ void den_monomials(const FitParams F, double* __restrict__ Dm) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < F.m;
       r += (int64_t)gridDim.x * blockDim.x) {
    double x[RPG_MAX_VARS];
#pragma unroll
    for (int v = 0; v < RPG_MAX_VARS; ++v) x[v] = v < F.n_vars ? F.X[r * F.n_vars + v] : 0.0;
    const int st = F.nd <= 8 ? 8 : F.nd;  // stride 8 (zero-padded) for den_pass<8>
    for (int k = 0; k < st; ++k)
      Dm[r * st + k] = k < F.nd ? monomial(x, F.exps + (size_t)(F.nn + k) * F.n_vars, F.n_vars) : 0.0;
  }
}

// Per-candidate min q and sum log q of the CTA's rows into out[2a], out[2a+1]
// (warp shuffles, then warps 0..7 in order; buf: >= 2 kAlphas kFitWarps
// doubles of SMEM free after the leading barrier).
__device__ __forceinline__ void write_alpha_partials(const double (&qmin)[kAlphas],
                                                     const double (&slog)[kAlphas], double* buf,
                                                     double* out) {
  double t[kAlphas], u[kAlphas];
#pragma unroll
  for (int a = 0; a < kAlphas; ++a) {
    t[a] = qmin[a];
    u[a] = slog[a];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int a = 0; a < kAlphas; ++a) {
      t[a] = fmin(t[a], __shfl_xor_sync(0xffffffffu, t[a], o));
      u[a] += __shfl_xor_sync(0xffffffffu, u[a], o);
    }
  __syncthreads();
  if ((threadIdx.x & 31) == 0) {
#pragma unroll
    for (int a = 0; a < kAlphas; ++a) {
      buf[a * 2 * kFitWarps + (threadIdx.x >> 5)] = t[a];
      buf[a * 2 * kFitWarps + kFitWarps + (threadIdx.x >> 5)] = u[a];
    }
  }
  __syncthreads();
  if (threadIdx.x < kAlphas) {
    const double* b = buf + threadIdx.x * 2 * kFitWarps;
    double mn = b[0], sm = b[kFitWarps];
    for (int i = 1; i < kFitWarps; ++i) {
      mn = fmin(mn, b[i]);
      sm += b[kFitWarps + i];
    }
    out[2 * threadIdx.x] = mn;
    out[2 * threadIdx.x + 1] = sm;
  }
}

// The sample pass for any nd <= NDT (the FMA Gram; nd <= 8 runs
// den_pass8_body unless RPG_FIT_NO_DMMA): per CTA, for each candidate a,
// min q and sum log q over its rows, and with `newton` for candidate 0 also
// sum (1/q) D_k and sum (1/q^2) D_k D_k^T.
template <int NDT>
__device__ __forceinline__ void den_pass_body(const FitParams& F, const double* __restrict__ cd,
                                              const double* __restrict__ dd,
                                              const double* __restrict__ alphas, int n_alpha,
                                              int newton, double* __restrict__ partial,
                                              const CtlSrc& src) {
  extern __shared__ __align__(16) double fsm[];
  const int nd = F.nd;
  if (src.ctl) {
    // Controlled pass: NEWTON = candidate S.*c (with the Newton sums), LINE =
    // S.*c + al[a] (S.*dc) for the pass's candidates; nothing once finished.
    const int ph = src.ctl->phase;
    if (ph >= kMinDone) return;
    newton = ph == kMinNewton;
    n_alpha = newton ? 1 : src.ctl->n_alpha;
  }
  const int ust = nd <= 8 ? 8 : nd;                 // row stride of U and of Dm (den_pass_smem)
  double* U = fsm;                                  // kPassRows x ust (row-major)
  double* cands = U + kPassRows * ust + 32;         // kAlphas x nd
  uint8_t* sexps = reinterpret_cast<uint8_t*>(cands + kAlphas * (nd > 4 ? nd : 4));
  for (int e = threadIdx.x; e < nd * F.n_vars; e += blockDim.x)
    sexps[e] = F.exps[F.nn * F.n_vars + e];
  for (int e = threadIdx.x; e < n_alpha * nd; e += blockDim.x) {
    const int a = e / nd, k = e % nd;
    if (src.ctl) {
      const int j = F.nn + k;
      const double ck = src.S[j] * src.c[j];
      cands[e] = newton ? ck : ck + src.ctl->al[a] * (src.S[j] * src.dc[j]);
    } else {
      cands[e] = dd ? cd[k] + alphas[a] * dd[k] : cd[k];
    }
  }
  __syncthreads();
  double qmin[kAlphas], slog[kAlphas], prod[kAlphas];
  int pexp[kAlphas];
#pragma unroll
  for (int a = 0; a < kAlphas; ++a) {
    qmin[a] = INFINITY;
    slog[a] = 0.0;
    prod[a] = 1.0;
    pexp[a] = 0;
  }
  // Gram accumulators: with nd*nd <= blockDim/2 every entry gets `parts`
  // threads (thread = part * nd*nd + entry); else thread t owns entries t,
  // t + blockDim, ...
  const int parts = (nd * nd <= (int)blockDim.x / 2) ? (int)blockDim.x / (nd * nd) >= 4 ? 4 : 2 : 1;
  const int ne_stride = parts > 1 ? nd * nd : (int)blockDim.x;
  const int part = parts > 1 ? (int)threadIdx.x / (nd * nd) : 0;
  double gacc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) gacc[i] = 0.0;
  double gq = 0.0;  // thread t < nd owns sum (1/q) D[t]
  const int64_t nrow_tiles = (F.m + kPassRows - 1) / kPassRows;
  for (int64_t tile = blockIdx.x; tile < nrow_tiles; tile += gridDim.x) {
    const int64_t r = tile * kPassRows + threadIdx.x;
    const bool valid = threadIdx.x < kPassRows && r < F.m;
    double D[NDT];
    if (valid) {
      if (F.Dm) {
        // Denominator monomials precomputed once per fit (m x ust).
#pragma unroll
        for (int k = 0; k < NDT; ++k) D[k] = k < nd ? F.Dm[r * ust + k] : 0.0;
      } else {
        double x[RPG_MAX_VARS];
#pragma unroll
        for (int v = 0; v < RPG_MAX_VARS; ++v) x[v] = v < F.n_vars ? F.X[r * F.n_vars + v] : 0.0;
#pragma unroll
        for (int k = 0; k < NDT; ++k) D[k] = k < nd ? monomial(x, sexps + k * F.n_vars, F.n_vars) : 0.0;
      }
#pragma unroll
      for (int a = 0; a < kAlphas; ++a) {
        if (a < n_alpha) {
          double q = 0.0;
#pragma unroll
          for (int k = 0; k < NDT; ++k)
            if (k < nd) q = fma(D[k], cands[a * nd + k], q);
          qmin[a] = fmin(qmin[a], q);
          // sum log q as log(prod of mantissas) + (sum of exponents) ln 2:
          // one multiply per row instead of a log (q <= 0 makes it NaN, as
          // the log would; such candidates fail the q > 0 test anyway).
          int e;
          const double mq = frexp(q, &e);
          prod[a] *= mq;
          pexp[a] += e;
        }
      }
    }
#pragma unroll
    for (int a = 0; a < kAlphas; ++a) prod[a] = split_mant(prod[a], pexp[a]);  // keep products in range
    if (newton) {
      __syncthreads();
      if (threadIdx.x < kPassRows) {
        double q = 0.0, qi = 0.0;
        if (valid) {
#pragma unroll
          for (int k = 0; k < NDT; ++k)
            if (k < nd) q = fma(D[k], cands[k], q);
          qi = 1.0 / q;
        }
#pragma unroll
        for (int k = 0; k < NDT; ++k)
          if (k < nd) U[threadIdx.x * ust + k] = valid ? D[k] * qi : 0.0;
      }
      __syncthreads();
      // Gram of the tile's U rows: `parts` threads per entry, each over a
      // contiguous row range with four independent accumulators.
      for (int e = threadIdx.x % ne_stride, i = 0; part < parts && e < nd * nd; e += ne_stride, ++i) {
        const int a = e / nd, b = e % nd;
        const int r0 = part * (kPassRows / parts), r1 = r0 + kPassRows / parts;
        double t0 = 0.0, t1 = 0.0, t2 = 0.0, t3 = 0.0;
        for (int row = r0; row < r1; row += 4) {
          t0 = fma(U[row * ust + a], U[row * ust + b], t0);
          t1 = fma(U[(row + 1) * ust + a], U[(row + 1) * ust + b], t1);
          t2 = fma(U[(row + 2) * ust + a], U[(row + 2) * ust + b], t2);
          t3 = fma(U[(row + 3) * ust + a], U[(row + 3) * ust + b], t3);
        }
        gacc[i] += (t0 + t1) + (t2 + t3);
      }
      if ((int)threadIdx.x < nd) {
        // sum_k (1/q_k) D_k[t] = sum of column t of U
        double t0 = 0.0, t1 = 0.0, t2 = 0.0, t3 = 0.0;
        for (int row = 0; row < kPassRows; row += 4) {
          t0 += U[row * ust + threadIdx.x];
          t1 += U[(row + 1) * ust + threadIdx.x];
          t2 += U[(row + 2) * ust + threadIdx.x];
          t3 += U[(row + 3) * ust + threadIdx.x];
        }
        gq += (t0 + t1) + (t2 + t3);
      }
    }
  }
  if (newton && parts > 1) {
    // Fold the per-part partial Gram entries (thread = part * ne + entry).
    __syncthreads();
    double* P = U;  // reuse: parts x nd*nd
    if (threadIdx.x < parts * nd * nd) P[threadIdx.x] = gacc[0];
    __syncthreads();
    if ((int)threadIdx.x < nd * nd) {
      double t = 0.0;
      for (int q = 0; q < parts; ++q) t += P[q * nd * nd + threadIdx.x];
      gacc[0] = t;
    }
  }
#pragma unroll
  for (int a = 0; a < kAlphas; ++a) slog[a] = fma((double)pexp[a], 0.69314718055994530942, log(prod[a]));
  double* out = partial + (size_t)blockIdx.x * (2 * kAlphas + nd + nd * nd);
  write_alpha_partials(qmin, slog, U + (size_t)parts * nd * nd, out);
  if (newton) {
    if ((int)threadIdx.x < nd) out[2 * kAlphas + threadIdx.x] = gq;
    if (parts > 1) {
      if ((int)threadIdx.x < nd * nd) out[2 * kAlphas + nd + threadIdx.x] = gacc[0];
    } else {
      for (int e = threadIdx.x, i = 0; e < nd * nd; e += blockDim.x, ++i) out[2 * kAlphas + nd + e] = gacc[i];
    }
  }
}

// ---------------------------------------------------------------------------
// The nd <= 8 sample pass (FP64 tensor-core Gram), specialized by where a
// row's denominator monomials come from (den_src):
//   kSrcDm      the precomputed m x 8 array (den_monomials),
//   kSrcLat3    x of 3 variables, denominator basis = monomial_basis({1,1,1})
//               (polyfit.hpp:50-73): 4 multiplies per row,
//   kSrcMask    x of <= 4 variables, 0/1 exponents: bit-mask products,
//   kSrcGeneric x, any exponents: monomial().
// Every source yields monomial()'s bits, so all four give identical sums.
// The row loop is straight-line: the next tile's row is prefetched into the
// row buffer while the current one is consumed, rows past m read row m-1
// and contribute nothing (q -> +inf for the minimum, 1 for the product, 0
// for the Gram).
enum { kSrcDm = 0, kSrcLat3 = 1, kSrcMask = 2, kSrcGeneric = 3 };

template <int SRC>
struct Row8 {
  double v[SRC == kSrcLat3 ? 3 : SRC == kSrcMask ? 4 : 8];
};

template <int SRC>
__device__ __forceinline__ void load_row8(const FitParams& F, int64_t r, Row8<SRC>& b) {
  if constexpr (SRC == kSrcDm) {
    const double2* p = reinterpret_cast<const double2*>(F.Dm + r * 8);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const double2 t = __ldg(p + k);
      b.v[2 * k] = t.x;
      b.v[2 * k + 1] = t.y;
    }
  } else if constexpr (SRC == kSrcLat3) {
    const double* p = F.X + r * 3;
#pragma unroll
    for (int v = 0; v < 3; ++v) b.v[v] = __ldg(p + v);
  } else {
    const int nv = F.n_vars;
    const double* p = F.X + r * nv;
    constexpr int kV = SRC == kSrcMask ? 4 : RPG_MAX_VARS;
#pragma unroll
    for (int v = 0; v < kV; ++v) b.v[v] = v < nv ? __ldg(p + v) : 0.0;
  }
}

template <int SRC>
__device__ __forceinline__ void row_monomials8(const FitParams& F, const Row8<SRC>& b, uint32_t dm4,
                                               const uint8_t* sexps, double (&D)[8]) {
  const int nd = F.nd;
  if constexpr (SRC == kSrcDm) {
#pragma unroll
    for (int k = 0; k < 8; ++k) D[k] = b.v[k];  // zero-padded past nd
  } else if constexpr (SRC == kSrcLat3) {
    // 1, x2, x1, x0, x1x2, x0x2, x0x1, x0x1x2: each product extends a
    // shorter one by its highest variable, as monomial() multiplies
    const double p01 = b.v[0] * b.v[1], p02 = b.v[0] * b.v[2], p12 = b.v[1] * b.v[2];
    D[0] = 1.0;
    D[1] = b.v[2];
    D[2] = b.v[1];
    D[3] = b.v[0];
    D[4] = p12;
    D[5] = p02;
    D[6] = p01;
    D[7] = p01 * b.v[2];
  } else if constexpr (SRC == kSrcMask) {
    // monomial()'s order with the exponent-0 factors (exact multiplies by
    // 1) skipped
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      double mo = 1.0;
#pragma unroll
      for (int v = 0; v < 4; ++v)
        if ((dm4 >> (4 * k + v)) & 1u) mo *= b.v[v];
      D[k] = k < nd ? mo : 0.0;
    }
  } else {
#pragma unroll
    for (int k = 0; k < 8; ++k) D[k] = k < nd ? monomial(b.v, sexps + k * F.n_vars, F.n_vars) : 0.0;
  }
}

// One row's contribution to candidate a: min q and the log-sum's mantissa
// product / exponent (mid-range factors multiply in unsplit; see
// mid_range).  Rows past m pass q = +inf / 1.
__device__ __forceinline__ void accum_q(double q, bool valid, double& qmin, double& prod, int& pexp) {
  qmin = fmin(qmin, valid ? q : INFINITY);
  const double qp = valid ? q : 1.0;
  if (mid_range(qp)) prod *= qp;
  else prod *= split_mant(qp, pexp);
}

template <int SRC, bool DIR>
__device__ __forceinline__ void rows8(const FitParams& F, int64_t nrow_tiles, const double* cands,
                                      const double (&al)[kAlphas], int n_alpha, bool newton,
                                      uint32_t dm4, const uint8_t* sexps, double (&qmin)[kAlphas],
                                      double (&prod)[kAlphas], int (&pexp)[kAlphas], double* U,
                                      double& gmma0, double& gmma1, double& gqv) {
  const int nd = F.nd;
  const int64_t step = (int64_t)gridDim.x * kPassRows, last = F.m - 1;
  int64_t r = (int64_t)blockIdx.x * kPassRows + threadIdx.x;
  Row8<SRC> buf;
  if ((int64_t)blockIdx.x < nrow_tiles) load_row8<SRC>(F, r < last ? r : last, buf);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int64_t tile = blockIdx.x; tile < nrow_tiles; tile += gridDim.x, r += step) {
    const bool valid = r < F.m;
    double D[8];
    row_monomials8<SRC>(F, buf, dm4, sexps, D);
    if (tile + gridDim.x < nrow_tiles) {
      const int64_t rn = r + step;
      load_row8<SRC>(F, rn < last ? rn : last, buf);
    }
    double q0 = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) q0 = fma(D[k], cands[k], q0);
    if constexpr (DIR) {
      // q_a = D.(cd + al_a dd) evaluated as D.cd + al_a (D.dd)
      double qd = 0.0;
#pragma unroll
      for (int k = 0; k < 8; ++k) qd = fma(D[k], cands[8 + k], qd);
#pragma unroll
      for (int a = 0; a < kAlphas; ++a)
        if (a < n_alpha) accum_q(fma(al[a], qd, q0), valid, qmin[a], prod[a], pexp[a]);
    } else {
#pragma unroll
      for (int a = 0; a < kAlphas; ++a)
        if (a < n_alpha) accum_q(q0, valid, qmin[a], prod[a], pexp[a]);
      if (newton) {
        // U = D / q for the Gram U^T U and the column sums, on the FP64
        // tensor cores: warp w folds rows [32w, 32w + 32) in 4-row chunks
        // with mma.m8n8k4 (A = U^T chunk, B = U chunk: lane l supplies
        // U[r0 + l%4][l/4] to both).
        const double qi = 1.0 / q0;
        __syncthreads();
#pragma unroll
        for (int k = 0; k < 8; ++k) U[threadIdx.x * 8 + k] = (valid && k < nd) ? D[k] * qi : 0.0;
        __syncthreads();
#pragma unroll
        for (int cidx = 0; cidx < 8; ++cidx) {
          const double v = U[(warp * 32 + cidx * 4 + (lane & 3)) * 8 + (lane >> 2)];
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                       : "+d"(gmma0), "+d"(gmma1) : "d"(v), "d"(v));
          gqv += v;
        }
      }
    }
#pragma unroll
    for (int a = 0; a < kAlphas; ++a)  // keep the products in range
      if (!mid_range(prod[a])) prod[a] = split_mant(prod[a], pexp[a]);
  }
}

template <int SRC>
__device__ __forceinline__ void den_pass8_body(const FitParams& F, const double* __restrict__ cd,
                                               const double* __restrict__ dd,
                                               const double* __restrict__ alphas, int n_alpha,
                                               int newton, double* __restrict__ partial,
                                               const CtlSrc& src) {
  extern __shared__ __align__(16) double fsm[];
  const int nd = F.nd;
  if (src.ctl) {
    // Controlled pass: NEWTON = candidate S.*c (with the Newton sums), LINE =
    // S.*c + al[a] (S.*dc) for the pass's candidates; nothing once finished.
    const int ph = src.ctl->phase;
    if (ph >= kMinDone) return;
    newton = ph == kMinNewton;
    n_alpha = newton ? 1 : src.ctl->n_alpha;
  }
  double* U = fsm;                        // kPassRows x 8 (row-major, zero-padded)
  double* cands = U + kPassRows * 8 + 32;  // cd[8], dd[8] (den_pass_smem's layout)
  uint8_t* sexps = reinterpret_cast<uint8_t*>(cands + kAlphas * (nd > 4 ? nd : 4));
  if constexpr (SRC == kSrcMask || SRC == kSrcGeneric)
    for (int e = threadIdx.x; e < nd * F.n_vars; e += blockDim.x) sexps[e] = F.exps[F.nn * F.n_vars + e];
  const bool has_dir = src.ctl ? !newton : dd != nullptr;
  double al[kAlphas];
#pragma unroll
  for (int a = 0; a < kAlphas; ++a)
    al[a] = a < n_alpha ? (src.ctl ? src.ctl->al[a] : (alphas ? alphas[a] : 0.0)) : 0.0;
  if (threadIdx.x < 16) {
    const int k = threadIdx.x & 7;
    double v = 0.0;
    if (k < nd) {
      if (threadIdx.x < 8) v = src.ctl ? src.S[F.nn + k] * src.c[F.nn + k] : cd[k];
      else if (has_dir) v = src.ctl ? src.S[F.nn + k] * src.dc[F.nn + k] : dd[k];
    }
    cands[threadIdx.x] = v;
  }
  __syncthreads();
  uint32_t dm4 = 0;
  if constexpr (SRC == kSrcMask) {
#pragma unroll
    for (int k = 0; k < 8; ++k)
#pragma unroll
      for (int v = 0; v < 4; ++v)
        if (k < nd && v < F.n_vars && sexps[k * F.n_vars + v]) dm4 |= 1u << (4 * k + v);
  }
  double qmin[kAlphas], prod[kAlphas], slog[kAlphas];
  int pexp[kAlphas];
#pragma unroll
  for (int a = 0; a < kAlphas; ++a) {
    qmin[a] = INFINITY;
    prod[a] = 1.0;
    pexp[a] = 0;
  }
  double gmma0 = 0.0, gmma1 = 0.0, gqv = 0.0;  // DMMA accumulator fragment, column sums
  const int64_t nrow_tiles = (F.m + kPassRows - 1) / kPassRows;
  if (has_dir)
    rows8<SRC, true>(F, nrow_tiles, cands, al, n_alpha, false, dm4, sexps, qmin, prod, pexp, U, gmma0,
                     gmma1, gqv);
  else
    rows8<SRC, false>(F, nrow_tiles, cands, al, n_alpha, newton, dm4, sexps, qmin, prod, pexp, U, gmma0,
                      gmma1, gqv);
  double* out = partial + (size_t)blockIdx.x * (2 * kAlphas + nd + nd * nd);
  double gram = 0.0, gq = 0.0;
  if (newton) {
    // Fold the 8 warps' fragments (fixed order): thread t holds
    // G[t/4][2(t%4) + {0,1}] of its warp; column sums by column t/4.
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    gqv += __shfl_xor_sync(0xffffffffu, gqv, 1);
    gqv += __shfl_xor_sync(0xffffffffu, gqv, 2);
    __syncthreads();
    double* Pm = U;  // 8 warps x (64 Gram + 8 column sums)
    Pm[warp * 72 + (lane >> 2) * 8 + 2 * (lane & 3)] = gmma0;
    Pm[warp * 72 + (lane >> 2) * 8 + 2 * (lane & 3) + 1] = gmma1;
    if ((lane & 3) == 0) Pm[warp * 72 + 64 + (lane >> 2)] = gqv;
    __syncthreads();
    if (threadIdx.x < 72) {
      double t = 0.0;
      for (int w = 0; w < kFitWarps; ++w) t += Pm[w * 72 + threadIdx.x];
      if (threadIdx.x < 64) gram = t;
      else gq = t;
    }
  }
#pragma unroll
  for (int a = 0; a < kAlphas; ++a) {
    // normalized as after the per-tile split of every tile (CTAs past the
    // last tile never split: prod 1, exponent 0)
    if ((int64_t)blockIdx.x < nrow_tiles) prod[a] = split_mant(prod[a], pexp[a]);
    slog[a] = fma((double)pexp[a], 0.69314718055994530942, log(prod[a]));
  }
  write_alpha_partials(qmin, slog, U + 72 * kFitWarps, out);
  if (newton) {
    const int t = threadIdx.x;
    if (t < 64 && (t >> 3) < nd && (t & 7) < nd) out[2 * kAlphas + nd + (t >> 3) * nd + (t & 7)] = gram;
    if (t >= 64 && t < 64 + nd) out[2 * kAlphas + (t - 64)] = gq;
  }
}

// Sums the per-block partials of den_pass (min for the q minima).
template <int NDT, int SRC = kSrcDm>
__global__ void __launch_bounds__(kFitThreads)
den_pass(const FitParams F, const double* __restrict__ cd, const double* __restrict__ dd,
         const double* __restrict__ alphas, int n_alpha, int newton,
         double* __restrict__ partial /* per block: 2*kAlphas + nd + nd*nd */, CtlSrc src) {
  if constexpr (NDT == 8) den_pass8_body<SRC>(F, cd, dd, alphas, n_alpha, newton, partial, src);
  else den_pass_body<NDT>(F, cd, dd, alphas, n_alpha, newton, partial, src);
}

// Folds G per-block partials (W values each) into out: one thread per
// value, the G loads of a thread independent of each other (issued back to
// back, one L2 round trip for the whole fold instead of one per value), a
// fixed g order (deterministic).
__device__ __forceinline__ void den_pass_reduce(const double* __restrict__ partial, int G, int nd,
                                                double* __restrict__ out, bool newton) {
  const int W = 2 * kAlphas + nd + nd * nd;
  // a non-Newton pass writes only the candidates' (min q, sum log q)
  const int nv = newton ? W : 2 * kAlphas;
  for (int e = threadIdx.x; e < nv; e += blockDim.x) {
    const bool is_min = e < 2 * kAlphas && (e % 2) == 0;
    double t = is_min ? INFINITY : 0.0;
    const double* p = partial + e;
    int g = 0;
    for (; g + 8 <= G; g += 8) {
      double v[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = p[(size_t)(g + i) * W];
#pragma unroll
      for (int i = 0; i < 8; ++i) t = is_min ? fmin(t, v[i]) : t + v[i];
    }
    for (; g < G; ++g) t = is_min ? fmin(t, p[(size_t)g * W]) : t + p[(size_t)g * W];
    out[e] = t;
  }
}

__global__ void den_pass_final(const double* __restrict__ partial, int G, int nd,
                               double* __restrict__ out, const MinCtl* __restrict__ ctl, int newton) {
  if (ctl && ctl->phase >= kMinDone) return;
  den_pass_reduce(partial, G, nd, out, ctl ? ctl->phase == kMinNewton : newton != 0);
}

// ||R S v||^2 for the n x n upper-triangular R (row-major) and scale S.
__device__ double rs_norm2(const double* R, const double* S, const double* v, int n) {
  double acc = 0.0;
  for (int i = 0; i < n; ++i) {
    double t = 0.0;
    for (int k = i; k < n; ++k) t = fma(R[i * n + k], S[k] * v[k], t);
    acc = fma(t, t, acc);
  }
  return acc;
}

// Setup state of the minimizer (min_setup).
struct MinState {
  double mu, phi0, decrement;
  int ok;
};

// Setup: c = start / S, q = Q c must be > 0, rescale so g.c = m, mu.
// pass_out: den_pass of the raw start's denominator (min q at index 0).
__global__ void min_setup(const double* __restrict__ R, const double* __restrict__ S,
                          const double* __restrict__ start, const double* __restrict__ gsum,
                          const double* __restrict__ pass_out, int nn, int nd, int64_t m,
                          double* __restrict__ c, MinState* __restrict__ st) {
  if (threadIdx.x != 0) return;
  const int n = nn + nd;
  for (int k = 0; k < n; ++k) c[k] = start[k] / S[k];
  st->ok = 0;
  if (!(pass_out[0] > 0.0)) return;
  // g = Q.colwise().sum(): den block = S_den .* colsum(D)
  double gc = 0.0;
  for (int k = 0; k < nd; ++k) gc = fma(gsum[k] * S[nn + k], c[nn + k], gc);
  const double s = (double)m / gc;
  if (!(s > 0.0) || !isfinite(s)) return;
  for (int k = 0; k < n; ++k) c[k] *= s;
  const double a2 = rs_norm2(R, S, c, n);
  st->mu = fmax(a2, 1e-30) / (double)m;
  st->ok = 1;
}

// Per-minimizer-call factorization of the Newton matrix's constant part.
// H = 2 H0 + mu M with H0 = S R^T R S fixed for the call and M nonzero only
// on the denominator block, so with u = numerator, v = denominator block:
//   A = 2 H0_uu (Cholesky, explicit inverse), B = 2 H0_uv, F = A^-1 B,
//   Sv0 = 2 H0_vv - B^T F.
// A Newton step then only solves the (nd+1) x (nd+1) Schur system
// [Sv0 + mu M_vv, g_v; g_v^T, 0] (newton_body).  prep layout: ok flag,
// Ainv (nn x nn), B (nn x nd), F (nn x nd), Sv0 (nd x nd).
constexpr int kPrepOk = 0;
__host__ __device__ inline int prep_size(int nn, int nd) {
  return 1 + nn * nn + 2 * nn * nd + nd * nd;
}

// Doubles of SMEM the Newton step's workspace takes ahead of the staged R
// and prep factors: newton_body's KKT system (N x (N+1) + 3n) or
// newton_schur_fast's fixed layout (kSchurWs), whichever is larger.
constexpr int kSchurWs = 504;
__host__ __device__ inline int newton_ws(int n) {
  const int kkt = (n + 1) * (n + 2) + 3 * n;
  return kkt > kSchurWs ? kkt : kSchurWs;
}

__global__ void __launch_bounds__(kFitThreads)
min_prep(const double* __restrict__ R, const double* __restrict__ S, int nn, int nd,
         double* __restrict__ prep) {
  extern __shared__ __align__(16) double fsm[];
  const int n = nn + nd;
  double* H = fsm;              // n x n (2 H0)
  double* L = H + n * n;        // nn x nn Cholesky factor
  __shared__ int ok;
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int a = e / n, b = e % n;
    double h = 0.0;
    for (int i = 0; i <= (a < b ? a : b); ++i) h = fma(R[i * n + a], R[i * n + b], h);
    H[e] = 2.0 * S[a] * S[b] * h;
  }
  for (int e = threadIdx.x; e < nn * nn; e += blockDim.x) L[e] = 0.0;
  if (threadIdx.x == 0) ok = 1;
  __syncthreads();
  // Cholesky of A = H_uu (left-looking, column j by the block)
  for (int j = 0; j < nn; ++j) {
    if (threadIdx.x == 0) {
      double d = H[j * n + j];
      for (int k = 0; k < j; ++k) d -= L[j * nn + k] * L[j * nn + k];
      if (!(d > 0.0) || !isfinite(d)) ok = 0;
      L[j * nn + j] = ok ? sqrt(d) : 1.0;
    }
    __syncthreads();
    for (int i = j + 1 + (int)threadIdx.x; i < nn; i += blockDim.x) {
      double t = H[i * n + j];
      for (int k = 0; k < j; ++k) t -= L[i * nn + k] * L[j * nn + k];
      L[i * nn + j] = t / L[j * nn + j];
    }
    __syncthreads();
  }
  double* Ainv = prep + 1;
  double* B = Ainv + nn * nn;
  double* Fm = B + nn * nd;
  double* Sv0 = Fm + nn * nd;
  if (threadIdx.x == 0) prep[kPrepOk] = ok ? 1.0 : 0.0;
  if (!ok) return;
  // Ainv = (L L^T)^-1, one column per thread (forward then backward solve)
  for (int col = threadIdx.x; col < nn; col += blockDim.x) {
    double z[64];
    for (int i = 0; i < nn; ++i) {
      double t = i == col ? 1.0 : 0.0;
      for (int k = 0; k < i; ++k) t -= L[i * nn + k] * z[k];
      z[i] = t / L[i * nn + i];
    }
    for (int i = nn - 1; i >= 0; --i) {
      double t = z[i];
      for (int k = i + 1; k < nn; ++k) t -= L[k * nn + i] * z[k];
      z[i] = t / L[i * nn + i];
    }
    for (int i = 0; i < nn; ++i) Ainv[i * nn + col] = z[i];
  }
  for (int e = threadIdx.x; e < nn * nd; e += blockDim.x) B[e] = H[(e / nd) * n + nn + (e % nd)];
  __syncthreads();
  for (int e = threadIdx.x; e < nn * nd; e += blockDim.x) {
    const int i = e / nd, j = e % nd;
    double t = 0.0;
    for (int k = 0; k < nn; ++k) t = fma(Ainv[i * nn + k], B[k * nd + j], t);
    Fm[e] = t;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < nd * nd; e += blockDim.x) {
    const int a = e / nd, b = e % nd;
    double t = H[(nn + a) * n + nn + b];
    for (int k = 0; k < nn; ++k) t -= B[k * nd + a] * Fm[k * nd + b];
    Sv0[e] = t;
  }
}

// Newton step: grad = 2 H0 c - mu Q^T(1/q), H = 2 H0 + mu Q^T diag(1/q^2) Q,
// KKT [H g; g^T 0] [dc; l] = [-grad; 0] solved by Gaussian elimination with
// partial pivoting (the reference uses LDLT), decrement = -grad.dc,
// phi0 = ||A_eq c||^2 - mu sum log q.  One CTA.
// ---------------------------------------------------------------------------
// Warp-parallel pieces of the minimizer's serial tail (one CTA of
// kFitThreads threads; R and the Schur factors staged in SMEM).

__device__ __forceinline__ double warp_sum(double t) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  return t;
}

// rows[i] = (R v)[i] = sum_{k >= i} R[i][k] v[k] for the upper-triangular
// R, one thread per row (thread `first` + i), k ascending — the same bits
// for the Newton step's phi0 (v = S c) and the line search's candidates
// (v = S (c + alpha dc)), whichever thread computes a row.
__device__ __forceinline__ void r_rows(const double* R, const double* v, int n, double* rows,
                                       int first) {
  const int i = (int)threadIdx.x - first;
  if (i < 0 || i >= n) return;
  double t = 0.0;
  for (int k = i; k < n; ++k) t = fma(R[i * n + k], v[k], t);
  rows[i] = t;
}

// sum_i rows[i]^2 over n <= 64 rows: one warp, lanes i and i + 32, then the
// shuffle tree (fixed order).  Lane 0 returns it.
__device__ __forceinline__ double sumsq_rows(const double* rows, int n) {
  const int lane = threadIdx.x & 31;
  double t = 0.0;
  if (lane < n) t = rows[lane] * rows[lane];
  if (lane + 32 < n) t = fma(rows[lane + 32], rows[lane + 32], t);
  return warp_sum(t);
}

// Gaussian elimination with partial pivoting (first largest |pivot|) of the
// Schur system [K | rhs] with M = nd + 1 <= 9 rows, one warp: lane r holds
// row r in registers, padded with identity rows up to 9 (they never win a
// pivot of a real column).  On return lane r < M holds x_r; *singular when
// a pivot is zero.
__device__ __forceinline__ double ge9_warp(double (&a)[10], int M, bool* singular) {
  const int lane = threadIdx.x & 31;
  bool sing = false;
#pragma unroll
  for (int col = 0; col < 9; ++col) {
    double v = (lane >= col && lane < 9) ? fabs(a[col]) : -1.0;
    int p = lane;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, v, o);
      const int op = __shfl_xor_sync(0xffffffffu, p, o);
      if (ov > v || (ov == v && op < p)) {
        v = ov;
        p = op;
      }
    }
    if (col < M && v == 0.0) sing = true;
    // swap rows col and p
#pragma unroll
    for (int j = 0; j < 10; ++j) {
      const double from_p = __shfl_sync(0xffffffffu, a[j], p);
      const double from_c = __shfl_sync(0xffffffffu, a[j], col);
      if (lane == col) a[j] = from_p;
      else if (lane == p) a[j] = from_c;
    }
    double prow[10];
#pragma unroll
    for (int j = 0; j < 10; ++j) prow[j] = __shfl_sync(0xffffffffu, a[j], col);
    if (lane > col && lane < 9) {
      const double f = a[col] / prow[col];
#pragma unroll
      for (int j = col + 1; j < 10; ++j) a[j] -= f * prow[j];
    }
  }
  double x = 0.0;  // lane r: x_r after back substitution
#pragma unroll
  for (int r = 8; r >= 0; --r) {
    // t = rhs_r - sum_{j > r} a[r][j] x_j, on lane r
    double t = a[9];
#pragma unroll
    for (int j = r + 1; j < 9; ++j) t -= a[j] * __shfl_sync(0xffffffffu, x, j);
    if (lane == r) x = t / a[r];
  }
  *singular = sing;
  return x;
}

// The Schur-complement Newton step (see min_prep) for nd <= 8, all stages
// warp-parallel: RSc = R S c, H0c = S R^T RSc, grad, t = A^-1 (-grad_u),
// the (nd+1)-square KKT system in one warp's registers, dc, the decrement
// and phi0 = ||R S c||^2 - mu sum log q.  P: the min_prep factors in SMEM.
__device__ void newton_schur_fast(const double* R, const double* __restrict__ S,
                                  const double* __restrict__ gsum,
                                  const double* __restrict__ pass_out,
                                  const double* __restrict__ c, int nn, int nd,
                                  double* __restrict__ dc, const double mu,
                                  MinState* __restrict__ st, const double* P, double* ws) {
  const int n = nn + nd;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  double* RSc = ws;           // 64
  double* grad = ws + 64;     // 64
  double* tu = ws + 128;      // 64
  double* rhs = ws + 192;     // 16
  double* xs = ws + 208;      // 16
  double* cv = ws + 224;      // 64: S .* c
  // One round of global loads for every small input the solve reads more
  // than once (S, the pass sums, gsum); c only for cv.
  double* Ss = ws + 288;      // 64
  double* po = ws + 352;      // <= 2 kAlphas + 8 + 64 = 80
  double* gs = ws + 432;      // 8
  const int W = 2 * kAlphas + nd + nd * nd;
  for (int k = threadIdx.x; k < n; k += blockDim.x) {
    const double sk = S[k];
    Ss[k] = sk;
    cv[k] = sk * c[k];
  }
  for (int e = threadIdx.x; e < W; e += blockDim.x) po[e] = pass_out[e];
  for (int e = threadIdx.x; e < nd; e += blockDim.x) gs[e] = gsum[e];
  __syncthreads();
  S = Ss;
  pass_out = po;
  gsum = gs;
  const double* gq = pass_out + 2 * kAlphas;
  const double* G = gq + nd;
  const double* Ainv = P + 1;
  const double* B = Ainv + nn * nn;
  const double* Fm = B + nn * nd;
  const double* Sv0 = Fm + nn * nd;
  r_rows(R, cv, n, RSc, 0);
  __syncthreads();
  for (int k = warp; k < n; k += nw) {
    double t = 0.0;
    for (int i = lane; i <= k; i += 32) t = fma(R[i * n + k], RSc[i], t);
    t = warp_sum(t);
    if (lane == 0) grad[k] = 2.0 * (S[k] * t) - mu * (k >= nn ? S[k] * gq[k - nn] : 0.0);
  }
  __syncthreads();
  for (int i = warp; i < nn; i += nw) {
    double t = 0.0;
    for (int k = lane; k < nn; k += 32) t = fma(Ainv[i * nn + k], -grad[k], t);
    t = warp_sum(t);
    if (lane == 0) tu[i] = t;
  }
  __syncthreads();
  for (int a = warp; a < nd; a += nw) {
    double t = 0.0;
    for (int k = lane; k < nn; k += 32) t = fma(B[k * nd + a], tu[k], t);
    t = warp_sum(t);
    if (lane == 0) rhs[a] = -grad[nn + a] - t;
  }
  __syncthreads();
  if (warp == 0) {
    const int M = nd + 1;
    // columns 0..nd-1: dv, nd: the multiplier, nd+1..8: identity padding,
    // 9: right-hand side
    double row[10];
#pragma unroll
    for (int j = 0; j < 10; ++j) row[j] = 0.0;
    if (lane < nd) {
      const double sa = S[nn + lane];
#pragma unroll
      for (int b = 0; b < 9; ++b) {
        if (b < nd) row[b] = Sv0[lane * nd + b] + mu * sa * S[nn + b] * G[lane * nd + b];
        else if (b == nd) row[b] = gsum[lane] * sa;
      }
      row[9] = rhs[lane];
    } else if (lane == nd) {
#pragma unroll
      for (int b = 0; b < 8; ++b)
        if (b < nd) row[b] = gsum[b] * S[nn + b];
    } else if (lane < 9) {
#pragma unroll
      for (int b = 0; b < 9; ++b)
        if (b == lane) row[b] = 1.0;
    }
    bool sing;
    const double x = ge9_warp(row, M, &sing);
    if (lane < nd) xs[lane] = x;
    if (lane == 0) st->ok = sing ? 0 : 1;
  }
  __syncthreads();
  double* dcs = ws + 440;     // 64: dc, also kept here for the decrement (440 + 64 = kSchurWs)
  for (int i = threadIdx.x; i < nn; i += blockDim.x) {
    double t = tu[i];
    for (int j = 0; j < nd; ++j) t -= Fm[i * nd + j] * xs[j];
    dc[i] = t;
    dcs[i] = t;
  }
  for (int j = threadIdx.x; j < nd; j += blockDim.x) dc[nn + j] = dcs[nn + j] = xs[j];
  __syncthreads();
  if (warp == 0) {
    double d = 0.0;
    bool fin = true;
    for (int k = lane; k < n; k += 32) {
      fin &= isfinite(dcs[k]);
      d = fma(-grad[k], dcs[k], d);
    }
    d = warp_sum(d);
    fin = __all_sync(0xffffffffu, fin);
    const double a2 = sumsq_rows(RSc, n);
    if (lane == 0) {
      st->ok = (st->ok && fin) ? 1 : 0;
      st->decrement = d;
      st->phi0 = a2 - mu * pass_out[1];
    }
  }
}

__device__ void newton_body(const double* __restrict__ R, const double* __restrict__ S,
                            const double* __restrict__ gsum, const double* __restrict__ pass_out,
                            const double* __restrict__ c, int nn, int nd, double* __restrict__ dc,
                            const double mu, MinState* __restrict__ st,
                            const double* __restrict__ prep = nullptr) {
  extern __shared__ __align__(16) double fsm[];
  const int n = nn + nd, N = n + 1;
  double* K = fsm;                 // N x (N+1) augmented, row-major
  double* H0c = K + N * (N + 1);   // n
  double* RSc = H0c + n;           // n: (R S c)
  double* grad = RSc + n;          // n
  const double* gq = pass_out + 2 * kAlphas;
  const double* G = gq + nd;
  if (prep && prep[kPrepOk] != 0.0 && nd <= 8 && n <= 64) {
    newton_schur_fast(R, S, gsum, pass_out, c, nn, nd, dc, mu, st, prep, K);
    return;
  }
  // RSc = R S c
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    double t = 0.0;
    for (int k = i; k < n; ++k) t = fma(R[i * n + k], S[k] * c[k], t);
    RSc[i] = t;
  }
  __syncthreads();
  // H0 c = S R^T (R S c)
  for (int k = threadIdx.x; k < n; k += blockDim.x) {
    double t = 0.0;
    for (int i = 0; i <= k; ++i) t = fma(R[i * n + k], RSc[i], t);
    H0c[k] = S[k] * t;
  }
  __syncthreads();
  for (int k = threadIdx.x; k < n; k += blockDim.x) {
    double qterm = k >= nn ? S[k] * gq[k - nn] : 0.0;
    grad[k] = 2.0 * H0c[k] - mu * qterm;
  }
  if (prep && prep[kPrepOk] != 0.0 && nd <= 16) {
    // Schur-complement path (min_prep): t = A^-1 (-grad_u),
    // [Sv0 + mu M_vv, g_v; g_v^T, 0][dv; l] = [-grad_v - B^T t; 0],
    // du = t - F dv.
    const double* Ainv = prep + 1;
    const double* B = Ainv + nn * nn;
    const double* Fm = B + nn * nd;
    const double* Sv0 = Fm + nn * nd;
    double* tu = K;             // nn
    double* Ks = tu + nn;       // (nd+1) x (nd+2)
    const int M = nd + 1;
    __syncthreads();
    for (int i = threadIdx.x; i < nn; i += blockDim.x) {
      double t = 0.0;
      for (int k = 0; k < nn; ++k) t = fma(Ainv[i * nn + k], -grad[k], t);
      tu[i] = t;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < nd * nd; e += blockDim.x) {
      const int a = e / nd, b = e % nd;
      Ks[a * (M + 1) + b] = Sv0[e] + mu * S[nn + a] * S[nn + b] * G[a * nd + b];
    }
    for (int a = threadIdx.x; a < nd; a += blockDim.x) {
      double t = -grad[nn + a];
      for (int k = 0; k < nn; ++k) t -= B[k * nd + a] * tu[k];
      const double g = gsum[a] * S[nn + a];
      Ks[a * (M + 1) + nd] = g;
      Ks[nd * (M + 1) + a] = g;
      Ks[a * (M + 1) + M] = t;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      Ks[nd * (M + 1) + nd] = 0.0;
      Ks[nd * (M + 1) + M] = 0.0;
      // (nd+1)-square Gaussian elimination with partial pivoting
      bool sing = false;
      for (int col = 0; col < M; ++col) {
        int p = col;
        for (int r = col + 1; r < M; ++r)
          if (fabs(Ks[r * (M + 1) + col]) > fabs(Ks[p * (M + 1) + col])) p = r;
        if (Ks[p * (M + 1) + col] == 0.0) sing = true;
        if (p != col)
          for (int j = 0; j <= M; ++j) {
            const double t = Ks[col * (M + 1) + j];
            Ks[col * (M + 1) + j] = Ks[p * (M + 1) + j];
            Ks[p * (M + 1) + j] = t;
          }
        for (int r = col + 1; r < M; ++r) {
          const double f = Ks[r * (M + 1) + col] / Ks[col * (M + 1) + col];
          for (int j = col + 1; j <= M; ++j) Ks[r * (M + 1) + j] -= f * Ks[col * (M + 1) + j];
        }
      }
      for (int r = M - 1; r >= 0; --r) {
        double t = Ks[r * (M + 1) + M];
        for (int j = r + 1; j < M; ++j) t -= Ks[r * (M + 1) + j] * Ks[j * (M + 1) + M];
        Ks[r * (M + 1) + M] = t / Ks[r * (M + 1) + r];  // solution stored in the rhs column
      }
      st->ok = sing ? 0 : 1;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nn; i += blockDim.x) {
      double t = tu[i];
      for (int j = 0; j < nd; ++j) t -= Fm[i * nd + j] * Ks[j * (M + 1) + M];
      dc[i] = t;
    }
    for (int j = threadIdx.x; j < nd; j += blockDim.x) dc[nn + j] = Ks[j * (M + 1) + M];
    __syncthreads();
    if (threadIdx.x == 0) {
      bool finite = st->ok != 0;
      double dec = 0.0;
      for (int k = 0; k < n; ++k) {
        finite &= isfinite(dc[k]);
        dec = fma(-grad[k], dc[k], dec);
      }
      st->ok = finite ? 1 : 0;
      st->decrement = dec;
      double a2 = 0.0;
      for (int i = 0; i < n; ++i) a2 = fma(RSc[i], RSc[i], a2);
      st->phi0 = a2 - mu * pass_out[1];
    }
    return;
  }
  // H entries
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int a = e / n, b = e % n;
    double h = 0.0;
    for (int i = 0; i <= (a < b ? a : b); ++i) h = fma(R[i * n + a], R[i * n + b], h);
    h = 2.0 * S[a] * S[b] * h;
    if (a >= nn && b >= nn) h += mu * S[a] * S[b] * G[(a - nn) * nd + (b - nn)];
    K[a * (N + 1) + b] = h;
  }
  for (int a = threadIdx.x; a < n; a += blockDim.x) {
    const double g = a >= nn ? gsum[a - nn] * S[a] : 0.0;
    K[a * (N + 1) + n] = g;
    K[n * (N + 1) + a] = g;
  }
  __syncthreads();
  for (int a = threadIdx.x; a < n; a += blockDim.x) K[a * (N + 1) + N] = -grad[a];
  if (threadIdx.x == 0) {
    K[n * (N + 1) + n] = 0.0;
    K[n * (N + 1) + N] = 0.0;
  }
  __syncthreads();
  __shared__ int singular;
  __shared__ double xs[kMaxCols + 1];
  if (threadIdx.x == 0) singular = 0;
  {
  // Gaussian elimination with partial pivoting: warp 0 picks the pivot (the
  // first row holding the largest |entry|, as a sequential scan would), the
  // multipliers are formed once per row, all threads eliminate.
  __shared__ int piv;
  __shared__ double mult[kMaxCols + 1];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) singular = 0;
  for (int col = 0; col < N; ++col) {
    if (warp == 0) {
      int p = N;
      double best = -1.0;
      for (int r = col + lane; r < N; r += 32) {
        const double v = fabs(K[r * (N + 1) + col]);
        if (v > best) {
          best = v;
          p = r;
        }
      }
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int op = __shfl_xor_sync(0xffffffffu, p, o);
        if (ob > best || (ob == best && op < p)) {
          best = ob;
          p = op;
        }
      }
      if (lane == 0) {
        piv = p;
        if (best == 0.0) singular = 1;
      }
    }
    __syncthreads();
    if (piv != col)
      for (int j = threadIdx.x; j <= N; j += blockDim.x) {
        const double t = K[col * (N + 1) + j];
        K[col * (N + 1) + j] = K[piv * (N + 1) + j];
        K[piv * (N + 1) + j] = t;
      }
    __syncthreads();
    const double d = K[col * (N + 1) + col];
    for (int r = col + 1 + (int)threadIdx.x; r < N; r += blockDim.x) mult[r] = K[r * (N + 1) + col] / d;
    __syncthreads();
    for (int e = threadIdx.x; e < (N - col - 1) * (N - col); e += blockDim.x) {
      const int r = col + 1 + e / (N - col), j = col + 1 + e % (N - col);
      K[r * (N + 1) + j] -= mult[r] * K[col * (N + 1) + j];
    }
    __syncthreads();
  }
  // Back substitution, one warp (lane-split dot products).
  if (warp == 0) {
    for (int r = N - 1; r >= 0; --r) {
      double t = 0.0;
      for (int j = r + 1 + lane; j < N; j += 32) t = fma(K[r * (N + 1) + j], xs[j], t);
      for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
      if (lane == 0) xs[r] = (K[r * (N + 1) + N] - t) / K[r * (N + 1) + r];
      __syncwarp();
    }
  }
  __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double* x = xs;
    bool finite = !singular;
    double dec = 0.0;
    for (int k = 0; k < n; ++k) {
      dc[k] = x[k];
      finite &= isfinite(x[k]);
      dec = fma(-grad[k], x[k], dec);
    }
    st->ok = finite ? 1 : 0;
    st->decrement = dec;
    double a2 = 0.0;
    for (int i = 0; i < n; ++i) a2 = fma(RSc[i], RSc[i], a2);
    st->phi0 = a2 - mu * pass_out[1];
  }
}

// The inner loop ended (no decrement, no acceptable step, or 40 steps):
// mu *= 0.1 and the next outer round (16 rounds).
__device__ __forceinline__ void ctl_end_inner(MinCtl* ctl) {
  ctl->mu *= 0.1;
  ctl->outer += 1;
  ctl->inner = 0;
  ctl->phase = ctl->outer >= 16 ? kMinDone : kMinNewton;
}

// One controlled step after its den_pass (pass_out):
//   NEWTON: the KKT Newton direction (newton_step's algebra); stop the inner
//           loop when the decrement is negligible, else start a line search
//           at alpha = 1;
//   LINE:   phi at the pass's candidates (||R S cn||^2 - mu sum log qn);
//           accept the first (in halving order) with q > 0 and Armijo
//           decrease, else continue halving (the inner loop ends when alpha
//           drops to 1e-18) — polyfit.hpp:279-306.
__device__ __forceinline__ void ctl_step_body(const double* R, const double* __restrict__ S,
                                              const double* __restrict__ gsum,
                                              const double* __restrict__ pass_out,
                                              double* __restrict__ c, int nn, int nd,
                                              double* __restrict__ dc, MinCtl* __restrict__ ctl,
                                              MinState* __restrict__ scratch,
                                              const double* __restrict__ prep) {
  const int ph = ctl->phase;
  if (ph >= kMinDone) return;
  const int n = nn + nd;
  // Stage R (n x n) in SMEM behind newton_body's KKT workspace: every dot
  // product below reads it many times.
  {
    extern __shared__ __align__(16) double fsm[];
    double* Rs = fsm + newton_ws(n);               // behind the Newton step's workspace
    double* Ps = Rs + n * n;                       // the min_prep factors
    __syncthreads();
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) Rs[e] = R[e];
    // the prep factors only when min_prep succeeded (else only the flag is
    // written and newton_body takes the general path)
    const bool stage_prep = prep && ph == kMinNewton && prep[kPrepOk] != 0.0;
    if (stage_prep)
      for (int e = threadIdx.x; e < prep_size(nn, nd); e += blockDim.x) Ps[e] = prep[e];
    __syncthreads();
    R = Rs;
    if (stage_prep) prep = Ps;
  }
  const long long t_staged = clock64();
  if (ph == kMinNewton) {
    newton_body(R, S, gsum, pass_out, c, nn, nd, dc, ctl->mu, scratch, prep);
    __syncthreads();
    if (threadIdx.x == 0) ctl->newton_parts[2] += clock64() - t_staged;
    if (threadIdx.x == 0) {
      if (!scratch->ok) {
        ctl->phase = kMinFail;  // non-finite KKT solution: empty result
      } else if (!(scratch->decrement > 1e-14 * (1.0 + fabs(scratch->phi0)))) {
        ctl_end_inner(ctl);
      } else {
        ctl->phi0 = scratch->phi0;
        ctl->decrement = scratch->decrement;
        ctl->phase = kMinLine;
        ctl->alpha = 1.0;
        int na = 0;
        for (double a = 1.0; na < kAlphas && a > 1e-18; a *= 0.5) ctl->al[na++] = a;
        ctl->n_alpha = na;
      }
    }
    return;
  }
  // LINE: phis of the candidates, one warp each.
  __shared__ double phis[kAlphas];
  __shared__ int accepted;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int na = ctl->n_alpha;
  __shared__ double rows[kAlphas][kMaxCols];
  // ||R S cn||^2 per candidate: the candidate vectors S (c + alpha dc),
  // their rows (r_rows: the Newton step's phi0 rows for alpha = 0), then the
  // fixed-order sum of squares (sumsq_rows) — one thread per (candidate, k)
  // and per (candidate, row).
  __shared__ double cvs[kAlphas][kMaxCols];
  for (int e = threadIdx.x; e < na * n; e += blockDim.x) {
    const int a = e / n, k = e % n;
    cvs[a][k] = S[k] * (c[k] + ctl->al[a] * dc[k]);
  }
  __syncthreads();
  for (int a = 0; a < na; ++a) r_rows(R, cvs[a], n, rows[a], a * n);
  __syncthreads();
  if (warp < na) {
    const double acc = sumsq_rows(rows[warp], n);
    if (lane == 0) phis[warp] = acc - ctl->mu * pass_out[2 * warp + 1];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    accepted = -1;
    for (int a = 0; a < na; ++a)
      if (pass_out[2 * a] > 0.0 && phis[a] <= ctl->phi0 - 1e-4 * ctl->al[a] * ctl->decrement) {
        accepted = a;
        break;
      }
  }
  __syncthreads();
  if (accepted >= 0) {
    const double al = ctl->al[accepted];
    for (int k = threadIdx.x; k < n; k += blockDim.x) c[k] += al * dc[k];
    __syncthreads();
    if (threadIdx.x == 0) {
      ctl->inner += 1;
      if (ctl->inner >= 40) ctl_end_inner(ctl);
      else ctl->phase = kMinNewton;
    }
  } else if (threadIdx.x == 0) {
    const double next = ctl->al[na - 1] * 0.5;
    if (!(next > 1e-18)) {
      ctl_end_inner(ctl);  // no acceptable step: break the inner loop
    } else {
      int k = 0;
      for (double a = next; k < kAlphas && a > 1e-18; a *= 0.5) ctl->al[k++] = a;
      ctl->n_alpha = k;
      ctl->alpha = next;
    }
  }
}

// One whole minimizer step in one launch: every CTA runs its share of the
// controlled sample pass and writes its partial sums; the partials are
// folded in two deterministic levels — the last CTA of each group of
// kStepGroup CTAs (threadfence + per-group counter) reduces its group, the
// last group reducer reduces the group sums — and that CTA applies the
// Newton / line-search update and re-arms the counters.  Every reduction
// follows lane / shuffle order, so the result does not depend on which CTA
// arrives last.  No-op for every CTA once the loop is done.
constexpr int kStepGroup = 32;

#ifndef RPG_FIT_STEP_MINB
#define RPG_FIT_STEP_MINB 2  // min_step CTAs per SM (launch bounds; the pass grid's default)
#endif
template <int NDT, int SRC = kSrcDm>
__global__ void __launch_bounds__(kFitThreads, RPG_FIT_STEP_MINB)
min_step(const FitParams F, CtlSrc src, double* __restrict__ partial, double* __restrict__ pass_out,
         unsigned* __restrict__ counter /* n_groups + 1 */, double* __restrict__ gpart,
         const double* __restrict__ R, const double* __restrict__ S,
         const double* __restrict__ gsum, double* __restrict__ c, double* __restrict__ dc,
         MinCtl* __restrict__ ctl, MinState* __restrict__ scratch, const double* __restrict__ prep) {
  // Programmatic dependent launch (fit_use_pdl): let the next step's grid
  // launch now — its CTAs take the SM slots this grid's CTAs free and wait
  // below — then wait for the previous step's grid to complete (its memory
  // visible).  Both are no-ops without the launch attribute.
  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (src.ctl->phase >= kMinDone) return;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    ctl->t_start = global_ns();
    if (!ctl->t_first) ctl->t_first = ctl->t_start;
  }
  if constexpr (NDT == 8) den_pass8_body<SRC>(F, nullptr, nullptr, nullptr, 1, 1, partial, src);
  else den_pass_body<NDT>(F, nullptr, nullptr, nullptr, 1, 1, partial, src);
  const int W = 2 * kAlphas + F.nd + F.nd * F.nd;
  const int G = gridDim.x, n_groups = (G + kStepGroup - 1) / kStepGroup;
  const int group = blockIdx.x / kStepGroup;
  const int gsize = min(kStepGroup, G - group * kStepGroup);
  __shared__ int last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(counter + group, 1u) == (unsigned)gsize - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  const bool newton_pass = src.ctl->phase == kMinNewton;  // only the tail below changes it
  den_pass_reduce(partial + (size_t)group * kStepGroup * W, gsize, F.nd, gpart + (size_t)group * W,
                  newton_pass);
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    counter[group] = 0u;
    last = atomicAdd(counter + n_groups, 1u) == (unsigned)n_groups - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  const long long t0 = clock64();
  const int ph = ctl->phase;
  if (threadIdx.x == 0) {
    const unsigned long long ts = ctl->t_start;
    ctl->t_arrive = global_ns();
    ctl->pass_ns += ctl->t_arrive - ts;
    if (ctl->t_prev_end) ctl->gap_ns += ts - ctl->t_prev_end;
  }
  den_pass_reduce(gpart, n_groups, F.nd, pass_out, ph == kMinNewton);
  __syncthreads();
  if (threadIdx.x == 0 && ph == kMinNewton) ctl->newton_parts[0] += clock64() - t0;
  ctl_step_body(R, S, gsum, pass_out, c, F.nn, F.nd, dc, ctl, scratch, prep);
  __syncthreads();
  if (threadIdx.x == 0) {
    counter[n_groups] = 0u;
    ctl->tail_cycles[ph == kMinNewton ? 0 : 1] += clock64() - t0;
    ctl->n_steps[ph == kMinNewton ? 0 : 1] += 1;
    ctl->t_prev_end = global_ns();
    ctl->tail_ns += ctl->t_prev_end - ctl->t_arrive;
  }
}

__global__ void to_raw(const double* __restrict__ c, const double* __restrict__ S, int n,
                       double* __restrict__ raw, int* __restrict__ finite) {
  if (threadIdx.x != 0) return;
  int f = 1;
  for (int k = 0; k < n; ++k) {
    raw[k] = c[k] * S[k];
    f &= isfinite(raw[k]) ? 1 : 0;
  }
  *finite = f;
}

// Row weights of the reweighted rounds: max(1, |y_k|) * qprev_k.
__global__ void row_weights(const FitParams F, const double* __restrict__ cd,
                            double* __restrict__ w) {
  extern __shared__ __align__(16) double fsm[];
  uint8_t* sexps = reinterpret_cast<uint8_t*>(fsm);
  for (int e = threadIdx.x; e < F.nd * F.n_vars; e += blockDim.x)
    sexps[e] = F.exps[F.nn * F.n_vars + e];
  __syncthreads();
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < F.m;
       r += (int64_t)gridDim.x * blockDim.x) {
    double x[RPG_MAX_VARS];
#pragma unroll
    for (int v = 0; v < RPG_MAX_VARS; ++v) x[v] = v < F.n_vars ? F.X[r * F.n_vars + v] : 0.0;
    double q = 0.0;
    for (int k = 0; k < F.nd; ++k) q = fma(monomial(x, sexps + k * F.n_vars, F.n_vars), cd[k], q);
    w[r] = fmax(1.0, fabs(F.y[r])) * q;
  }
}

// Start vector of the safeguard from the SVD of R_v (the R factor of the
// numerator-only matrix V) and z = (Q_v^T y)[0:nn]: start[0:nn] =
// sum_{i<rank} W_i (u_i . z) / sigma_i, start[nn] = 1 (polyfit.hpp:382-395).
__global__ void start_vector(const double* __restrict__ Wv, const double* __restrict__ Uv,
                             const double* __restrict__ sig, const double* __restrict__ z,
                             int nn, int nd, double rank_tol, double* __restrict__ start) {
  if (threadIdx.x != 0) return;
  int rank = 0;
  if (nn > 0 && sig[0] > 0.0)
    for (int i = 0; i < nn; ++i) rank += sig[i] >= rank_tol * sig[0];
  for (int k = 0; k < nn + nd; ++k) start[k] = 0.0;
  for (int i = 0; i < rank; ++i) {
    double uty = 0.0;
    for (int j = 0; j < nn; ++j) uty = fma(Uv[i * nn + j], z[j], uty);
    const double f = uty / sig[i];
    for (int k = 0; k < nn; ++k) start[k] = fma(Wv[i * nn + k], f, start[k]);
  }
  start[nn] = 1.0;
}

// 1 / column norms of an R factor (equilibrate_columns, polyfit.hpp:219-229).
__global__ void col_scale_from_R(const double* __restrict__ R, int n, double* __restrict__ S) {
  for (int k = threadIdx.x; k < n; k += blockDim.x) {
    double t = 0.0;
    for (int i = 0; i <= k; ++i) t = fma(R[i * n + k], R[i * n + k], t);
    const double cn = sqrt(t);
    S[k] = cn > 0.0 ? 1.0 / cn : 1.0;
  }
}

__global__ void sum_partials(const double* __restrict__ partial, int G, int width,
                             double* __restrict__ out) {
  for (int k = threadIdx.x; k < width; k += blockDim.x) {
    double t = 0.0;
    for (int g = 0; g < G; ++g) t += partial[(size_t)g * width + k];
    out[k] = t;
  }
}

// Splits the (nn+1) x (nn+1) R factor of [V | y] into R_v and z.
__global__ void split_vy(const double* __restrict__ Rvy, int nn, double* __restrict__ Rv,
                         double* __restrict__ z) {
  const int N = nn + 1;
  for (int e = threadIdx.x; e < nn * nn; e += blockDim.x) Rv[e] = Rvy[(e / nn) * N + (e % nn)];
  for (int j = threadIdx.x; j < nn; j += blockDim.x) z[j] = Rvy[j * N + nn];
}

}  // namespace rpg_fit

// ---------------------------------------------------------------------------
// Host orchestration + C ABI.

namespace {

using namespace rpg_fit;

int fset_err(char* err, size_t errlen, int code, const char* fmt, ...) {
  if (err && errlen) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(err, errlen, fmt, ap);
    va_end(ap);
  }
  return code;
}

std::vector<std::vector<int>> basis(const int32_t* bounds, int nv) {
  std::vector<std::vector<int>> tuples{{}};
  for (int v = 0; v < nv; ++v) {
    std::vector<std::vector<int>> next;
    for (const auto& t : tuples)
      for (int e = 0; e <= bounds[v]; ++e) {
        next.push_back(t);
        next.back().push_back(e);
      }
    tuples.swap(next);
  }
  std::stable_sort(tuples.begin(), tuples.end(), [](const std::vector<int>& a, const std::vector<int>& b) {
    int ga = 0, gb = 0;
    for (int x : a) ga += x;
    for (int x : b) gb += x;
    if (ga != gb) return ga < gb;
    return a < b;
  });
  return tuples;
}

// Scratch buffers are stream-ordered allocations on the fit's stream
// (cudaMallocAsync from the device's pool, kept cached between calls): no
// device-wide synchronization per buffer, unlike cudaMalloc / cudaFree.
thread_local cudaStream_t g_fit_stream = nullptr;

cudaError_t fit_malloc(void** p, size_t bytes) {
  return g_fit_stream ? cudaMallocAsync(p, bytes, g_fit_stream) : cudaMalloc(p, bytes);
}

// RPG_FIT_PDL=0: minimizer steps launch without programmatic dependent
// launch (each step's grid then starts only after the previous completes).
static bool fit_use_pdl() {
  static const bool on = [] {
    const char* e = getenv("RPG_FIT_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

// RPG_FIT_NO_DMMA=1: the sample passes of nd <= 8 denominators use the
// generic kernels (Gram of D/q with FMA chains) instead of the
// register-resident nd = 8 path with the FP64 tensor-core Gram
// (mma.m8n8k4.f64) — the A/B switch behind DESIGN.md's DMMA measurement.
inline bool fit_use_dmma() {
  static const bool on = [] {
    const char* e = getenv("RPG_FIT_NO_DMMA");
    return e == nullptr || e[0] == '\0' || e[0] == '0';
  }();
  return on;
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) only ever raised, under a
// lock: concurrent fits (rpg_fit_rational_multi) with different column
// counts must not lower the limit under another thread's launch.
cudaError_t raise_smem_attr(const void* fn, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> cur;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  size_t& c = cur[{fn, dev}];
  if (bytes <= c) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) c = bytes;
  return e;
}

struct DevBuf {
  void* p = nullptr;
  ~DevBuf() {
    if (!p) return;
    if (g_fit_stream) cudaFreeAsync(p, g_fit_stream);
    else cudaFree(p);
  }
  template <class T>
  T* as() const { return static_cast<T*>(p); }
};

#define FCUDA(expr)                                                                   \
  do {                                                                                \
    cudaError_t e_ = (expr);                                                          \
    if (e_ != cudaSuccess)                                                            \
      return fset_err(err, errlen, RPG_E_CUDA, "%s: %s", #expr, cudaGetErrorString(e_)); \
  } while (0)

size_t tsqr_smem(int ncols) {
  return sizeof(double) * ((size_t)ncols * ncols + (size_t)kTile * ncols + 32 + kMaxCols) +
         (size_t)kMaxCols * RPG_MAX_VARS + 16;
}

// R factor (n x n, row-major, in *Rdev) of the sample matrix described by F.
int tsqr(const FitParams& F, int ncols, int sms, DevBuf* Rbuf, cudaStream_t s, char* err,
         size_t errlen) {
  const int64_t tiles = (F.m + kTile - 1) / kTile;
  const size_t sm1 = tsqr_smem(ncols);
  int per_sm = 1;
  FCUDA(raise_smem_attr(reinterpret_cast<const void*>(tsqr_tiles), sm1));
  FCUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tsqr_tiles, kFitThreads, sm1));
  int G = (int)std::min<int64_t>(tiles, (int64_t)std::max(1, std::min(per_sm, 4)) * sms);
  if (G < 1) G = 1;
  FCUDA(fit_malloc((void**)&Rbuf->p, sizeof(double) * (size_t)G * ncols * ncols));
  tsqr_tiles<<<G, kFitThreads, sm1, s>>>(F, Rbuf->as<double>());
  FCUDA(cudaGetLastError());
  const size_t sm2 = sizeof(double) * ((size_t)kCombine * ncols * ncols + 32 + kMaxCols);
  FCUDA(raise_smem_attr(reinterpret_cast<const void*>(tsqr_combine), sm2));
  // Tree over the G factors, one launch per level, ping-ponging between
  // Rbuf and tmp; the root ends in Rbuf.
  int count = G;
  DevBuf tmp;
  FCUDA(fit_malloc((void**)&tmp.p, sizeof(double) * (size_t)G * ncols * ncols));
  double* in = Rbuf->as<double>();
  double* outb = tmp.as<double>();
  while (count > 1) {
    const int next = (count + kCombine - 1) / kCombine;
    tsqr_combine<<<next, kFitThreads, sm2, s>>>(in, count, ncols, outb);
    FCUDA(cudaGetLastError());
    std::swap(in, outb);
    count = next;
  }
  if (in != Rbuf->as<double>())
    FCUDA(cudaMemcpyAsync(Rbuf->p, in, sizeof(double) * (size_t)ncols * ncols,
                          cudaMemcpyDeviceToDevice, s));
  return RPG_OK;
}

}  // namespace

// Where the nd <= 8 sample passes take a row's denominator monomials from.
static int den_src(const FitParams& F) {
  if (F.Dm) return kSrcDm;
  if (F.den_lat3) return kSrcLat3;
  if (F.den01) return kSrcMask;
  return kSrcGeneric;
}

using DenPassFn = void (*)(const FitParams, const double*, const double*, const double*, int, int,
                           double*, CtlSrc);
static DenPassFn den_pass8_fn(int src) {
  switch (src) {
    case kSrcDm: return den_pass<8, kSrcDm>;
    case kSrcLat3: return den_pass<8, kSrcLat3>;
    case kSrcMask: return den_pass<8, kSrcMask>;
    default: return den_pass<8, kSrcGeneric>;
  }
}

size_t den_pass_smem(const FitParams& F) {
  const size_t ust = F.nd <= 8 ? 8 : (size_t)F.nd;
  return sizeof(double) * ((size_t)kPassRows * ust + 32 + kAlphas * (size_t)std::max(F.nd, 4)) +
         (size_t)F.nd * RPG_MAX_VARS + 16;
}

struct Pass {
  DevBuf part, out;
  int G = 0, nd = 0;
};

int run_den_pass(const FitParams& F, const double* cd, const double* dd, const double* alphas,
                 int n_alpha, int newton, int sms, Pass* P, cudaStream_t s, char* err,
                 size_t errlen, CtlSrc src = CtlSrc{nullptr, nullptr, nullptr, nullptr}) {
  const int W = 2 * kAlphas + F.nd + F.nd * F.nd;
  if (!P->part.p) {
    const int64_t tiles = (F.m + kPassRows - 1) / kPassRows;
    // CTAs per SM of the sample passes (RPG_FIT_PASS_CTAS overrides: more
    // CTAs hide the pass's latency, fewer shorten the serial partial
    // reduction of the fused minimizer step).
    static const int per_sm = [] {
      const char* e = getenv("RPG_FIT_PASS_CTAS");
      return e ? std::max(1, atoi(e)) : RPG_FIT_STEP_MINB;  // min_step's launch bounds
    }();
    P->G = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, (int64_t)per_sm * sms));
    P->nd = F.nd;
    FCUDA(fit_malloc((void**)&P->part.p, sizeof(double) * (size_t)P->G * W));
    FCUDA(fit_malloc((void**)&P->out.p, sizeof(double) * W));
  }
  const size_t sm = den_pass_smem(F);
  if (F.nd <= 8 && fit_use_dmma()) {
    const DenPassFn fn = den_pass8_fn(den_src(F));
    FCUDA(raise_smem_attr(reinterpret_cast<const void*>(fn), sm));
    fn<<<P->G, kFitThreads, sm, s>>>(F, cd, dd, alphas, n_alpha, newton, P->part.as<double>(), src);
  } else {
    FCUDA(raise_smem_attr(reinterpret_cast<const void*>(den_pass<kMaxCols>), sm));
    den_pass<kMaxCols><<<P->G, kFitThreads, sm, s>>>(F, cd, dd, alphas, n_alpha, newton,
                                                     P->part.as<double>(), src);
  }
  FCUDA(cudaGetLastError());
  den_pass_final<<<1, 256, 0, s>>>(P->part.as<double>(), P->G, F.nd, P->out.as<double>(), src.ctl, newton);
  return RPG_OK;
}

// positive_den_minimizer (polyfit.hpp:242-311).  R, S: R factor and column
// scale of the (weighted) sample matrix; gsum: column sums of the raw
// denominator monomials; start (raw coordinates).  *found = 0 when the
// reference would return an empty vector.
int minimizer(const FitParams& F, const double* R, const double* S, const double* gsum,
              const double* start, double* out_raw, int* found, int sms, cudaStream_t s,
              char* err, size_t errlen) {
  const int nn = F.nn, nd = F.nd, n = F.n;
  *found = 0;
  const auto t_begin = std::chrono::steady_clock::now();
  DevBuf c, dc, cd, st, fin;
  FCUDA(fit_malloc((void**)&c.p, sizeof(double) * n));
  FCUDA(fit_malloc((void**)&dc.p, sizeof(double) * n));
  FCUDA(fit_malloc((void**)&cd.p, sizeof(double) * nd));
  FCUDA(fit_malloc((void**)&st.p, sizeof(MinState)));
  FCUDA(fit_malloc((void**)&fin.p, sizeof(int)));
  Pass P;
  // q of the start vector: Q (start / S) = D start_den.
  FCUDA(cudaMemcpyAsync(cd.p, start + nn, sizeof(double) * nd, cudaMemcpyDeviceToDevice, s));
  int rc = run_den_pass(F, cd.as<double>(), nullptr, nullptr, 1, 0, sms, &P, s, err, errlen);
  if (rc) return rc;
  min_setup<<<1, 32, 0, s>>>(R, S, start, gsum, P.out.as<double>(), nn, nd, F.m, c.as<double>(),
                             st.as<MinState>());
  MinState hs;
  FCUDA(cudaMemcpyAsync(&hs, st.p, sizeof(hs), cudaMemcpyDeviceToHost, s));
  FCUDA(cudaStreamSynchronize(s));
  if (!hs.ok) return RPG_OK;
  // newton_body's KKT workspace + the staged R (ctl_step_body)
  const size_t smk = sizeof(double) * ((size_t)newton_ws(n) + (size_t)n * n + (size_t)prep_size(nn, nd));
  DevBuf ctlb;
  FCUDA(fit_malloc((void**)&ctlb.p, sizeof(MinCtl)));
  MinCtl hc{};
  hc.phase = kMinNewton;
  hc.mu = hs.mu;
  hc.n_alpha = 1;
  FCUDA(cudaMemcpyAsync(ctlb.p, &hc, sizeof(hc), cudaMemcpyHostToDevice, s));
  MinCtl* dctl = ctlb.as<MinCtl>();
  const int n_groups = (P.G + kStepGroup - 1) / kStepGroup;
  const int Wp = 2 * kAlphas + nd + nd * nd;
  DevBuf counter, gpart;
  FCUDA(fit_malloc((void**)&counter.p, sizeof(unsigned) * (n_groups + 1)));
  FCUDA(cudaMemsetAsync(counter.p, 0, sizeof(unsigned) * (n_groups + 1), s));
  FCUDA(fit_malloc((void**)&gpart.p, sizeof(double) * (size_t)n_groups * Wp));
  const size_t smstep = std::max(smk, den_pass_smem(F));
  using MinStepFn = void (*)(const FitParams, CtlSrc, double*, double*, unsigned*, double*, const double*,
                            const double*, const double*, double*, double*, MinCtl*, MinState*,
                            const double*);
  MinStepFn step_fn = min_step<kMaxCols>;
  if (F.nd <= 8 && fit_use_dmma()) {
    switch (den_src(F)) {
      case kSrcDm: step_fn = min_step<8, kSrcDm>; break;
      case kSrcLat3: step_fn = min_step<8, kSrcLat3>; break;
      case kSrcMask: step_fn = min_step<8, kSrcMask>; break;
      default: step_fn = min_step<8, kSrcGeneric>; break;
    }
  }
  FCUDA(raise_smem_attr(reinterpret_cast<const void*>(step_fn), smstep));
  // Constant-block factorization for the Schur-complement Newton solve.
  DevBuf prepb;
  FCUDA(fit_malloc((void**)&prepb.p, sizeof(double) * (size_t)prep_size(nn, nd)));
  const size_t smp = sizeof(double) * ((size_t)n * n + (size_t)nn * nn);
  FCUDA(raise_smem_attr(reinterpret_cast<const void*>(min_prep), smp));
  min_prep<<<1, kFitThreads, smp, s>>>(R, S, nn, nd, prepb.as<double>());
  FCUDA(cudaGetLastError());
  const CtlSrc src{dctl, c.as<double>(), dc.as<double>(), S};
  // Steps (controlled den_pass + reduction + Newton-or-line update) are
  // enqueued in chunks; the host only polls the phase between chunks.
  // Bound: 16 outer x 40 inner x (1 Newton + <= 15 line passes).
  constexpr int kChunk = 24;
  const auto t_loop = std::chrono::steady_clock::now();
  for (int done = 0, steps = 0; !done && steps < 16 * 40 * 16; steps += kChunk) {
    for (int i = 0; i < kChunk; ++i) {
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(P.G);
      cfg.blockDim = dim3(kFitThreads);
      cfg.dynamicSmemBytes = smstep;
      cfg.stream = s;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = attr;
      cfg.numAttrs = fit_use_pdl() ? 1 : 0;
      FCUDA(cudaLaunchKernelEx(&cfg, step_fn, F,
                               src, P.part.as<double>(), P.out.as<double>(), counter.as<unsigned>(),
                               gpart.as<double>(), R, S, gsum, c.as<double>(), dc.as<double>(), dctl,
                               st.as<MinState>(), (const double*)prepb.as<double>()));
    }
    FCUDA(cudaGetLastError());
    FCUDA(cudaMemcpyAsync(&hc, ctlb.p, sizeof(hc), cudaMemcpyDeviceToHost, s));
    FCUDA(cudaStreamSynchronize(s));
    done = hc.phase >= kMinDone;
    if (done && getenv("RPG_FIT_TRACE"))
      fprintf(stderr, "[rpg_fit] minimizer wall %.3f ms = %.1f us per step\n",
              std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_begin).count(),
              1e3 * std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_begin).count() /
                  std::max(1, hc.n_steps[0] + hc.n_steps[1]));
    if (done && getenv("RPG_FIT_TRACE"))
      fprintf(stderr,
              "[rpg_fit] minimizer: %d Newton + %d line steps, phase %d, outer %d; serial tail "
              "%.1f / %.1f us per Newton / line step\n",
              hc.n_steps[0], hc.n_steps[1], hc.phase, hc.outer,
              hc.n_steps[0] ? hc.tail_cycles[0] / 1965.0 / hc.n_steps[0] : 0.0,
              hc.n_steps[1] ? hc.tail_cycles[1] / 1965.0 / hc.n_steps[1] : 0.0);
    if (done && getenv("RPG_FIT_TRACE") && hc.n_steps[0])
      fprintf(stderr, "[rpg_fit]   Newton tail: final fold %.1f us, solve %.1f us (rest: staging, control)\n",
              hc.newton_parts[0] / 1965.0 / hc.n_steps[0], hc.newton_parts[2] / 1965.0 / hc.n_steps[0]);
    if (done && getenv("RPG_FIT_TRACE") && hc.n_steps[0] + hc.n_steps[1] > 1)
      fprintf(stderr, "[rpg_fit]   host setup %.3f ms; device span first step -> last step end %.3f ms\n",
              std::chrono::duration<double, std::milli>(t_loop - t_begin).count(),
              1e-6 * (hc.t_prev_end - hc.t_first));
    if (done && getenv("RPG_FIT_TRACE") && hc.n_steps[0] + hc.n_steps[1] > 1)
      fprintf(stderr, "[rpg_fit]   per step: sample pass %.1f us, tail %.1f us, inter-step gap %.1f us\n",
              1e-3 * hc.pass_ns / (hc.n_steps[0] + hc.n_steps[1]),
              1e-3 * hc.tail_ns / (hc.n_steps[0] + hc.n_steps[1]),
              1e-3 * hc.gap_ns / (hc.n_steps[0] + hc.n_steps[1] - 1));
  }
  if (hc.phase == kMinFail) return RPG_OK;
  to_raw<<<1, 32, 0, s>>>(c.as<double>(), S, n, out_raw, fin.as<int>());
  int f = 0;
  FCUDA(cudaMemcpyAsync(&f, fin.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  FCUDA(cudaStreamSynchronize(s));
  *found = f;
  return RPG_OK;
}

// The positivity safeguard (polyfit.hpp:369-414).  c: in = the unconstrained
// candidate (raw coordinates), out = the refined vector when one is found.
int rpg_fit_safeguard(const FitParams& F0, const double* R, const double* S, double* c,
                      double rank_tol, int sms, cudaStream_t s, char* err, size_t errlen,
                      rpg_fit_trace* trace) {
  const int nn = F0.nn, nd = F0.nd, n = F0.n;
  // The sample passes read precomputed denominator monomials.
  DevBuf dm;
  FitParams F = F0;
  // RPG_FIT_DM=1 forces the precomputed monomials, RPG_FIT_DM=0 forbids
  // them; by default they are skipped when the pass recomputes them from x
  // by bit masks (den01, no HBM pass over an m x 8 array).
  static const char* dm_env = getenv("RPG_FIT_DM");
  static const bool no_dm_env = getenv("RPG_FIT_NO_DM") != nullptr;
  const bool use_dm = !no_dm_env && (dm_env ? dm_env[0] == '1' : !(F0.den01 && nd <= 8));
  if (use_dm && fit_malloc((void**)&dm.p, sizeof(double) * (size_t)F0.m * (nd <= 8 ? 8 : nd)) == cudaSuccess) {
    den_monomials<<<(int)std::min<int64_t>((F0.m + 255) / 256, 8LL * sms), 256, 0, s>>>(
        F0, dm.as<double>());
    FCUDA(cudaGetLastError());
    F.Dm = dm.as<double>();
  } else {
    cudaGetLastError();  // out of memory: recompute the monomials per pass
  }
  DevBuf gpart, gsum, Rvy, Rv, z, sv, Wv, Uv, dummy, start, refined, next, w, Rw, Sw;
  // column sums of the raw denominator monomials
  const int G = std::max(1, std::min<int>((int)((F.m + 255) / 256), 2 * sms));
  FCUDA(fit_malloc((void**)&gpart.p, sizeof(double) * (size_t)G * nd));
  FCUDA(fit_malloc((void**)&gsum.p, sizeof(double) * nd));
  const size_t smc = sizeof(double) * kMaxCols * kFitWarps + (size_t)kMaxCols * RPG_MAX_VARS + 16;
  FCUDA(raise_smem_attr(reinterpret_cast<const void*>(den_colsum), smc));
  den_colsum<<<G, kFitThreads, smc, s>>>(F, gpart.as<double>());
  sum_partials<<<1, 64, 0, s>>>(gpart.as<double>(), G, nd, gsum.as<double>());
  // start vector: least squares of the numerator basis against y, from a
  // QR of [V | y] of its own.  (The leading block of A's R is the same QR
  // in exact arithmetic, but the start vector's rank truncation and the
  // minimizer it seeds are sensitive to its rounding on rank-deficient C4
  // metrics — r02aa: coal_mem_insts_per_thread parted from O3 at stage 1.)
  FitParams Fv = F;
  Fv.num_only = 1;
  Fv.with_y_col = 1;
  int rc = tsqr(Fv, nn + 1, sms, &Rvy, s, err, errlen);
  if (rc) return rc;
  FCUDA(fit_malloc((void**)&Rv.p, sizeof(double) * nn * nn));
  FCUDA(fit_malloc((void**)&z.p, sizeof(double) * nn));
  split_vy<<<1, 128, 0, s>>>(Rvy.as<double>(), nn, Rv.as<double>(), z.as<double>());
  FCUDA(fit_malloc((void**)&sv.p, sizeof(double) * nn));
  FCUDA(fit_malloc((void**)&Wv.p, sizeof(double) * nn * nn));
  FCUDA(fit_malloc((void**)&Uv.p, sizeof(double) * nn * nn));
  FCUDA(fit_malloc((void**)&dummy.p, sizeof(double) * nn));
  const size_t sm3 = sizeof(double) * (2 * (size_t)kMaxCols * kMaxCols + kMaxCols) + sizeof(int) * (kMaxCols + 4);
  svd_small<<<1, svd_threads(nn), sm3, s>>>(Rv.as<double>(), nn, sv.as<double>(), Wv.as<double>(),
                                        dummy.as<double>(), Uv.as<double>(), 0);
  FCUDA(fit_malloc((void**)&start.p, sizeof(double) * n));
  start_vector<<<1, 32, 0, s>>>(Wv.as<double>(), Uv.as<double>(), sv.as<double>(), z.as<double>(),
                                nn, nd, rank_tol, start.as<double>());
  FCUDA(fit_malloc((void**)&refined.p, sizeof(double) * n));
  FCUDA(fit_malloc((void**)&next.p, sizeof(double) * n));
  int found = 0;
  rc = minimizer(F, R, S, gsum.as<double>(), start.as<double>(), refined.as<double>(), &found, sms,
                 s, err, errlen);
  if (rc) return rc;
  auto record = [&](const double* dvec) -> int {
    if (!trace || trace->n_stages >= RPG_FIT_TRACE_STAGES) return RPG_OK;
    FCUDA(cudaMemcpyAsync(trace->stage_coef[trace->n_stages], dvec, sizeof(double) * n,
                          cudaMemcpyDeviceToHost, s));
    FCUDA(cudaStreamSynchronize(s));
    ++trace->n_stages;
    return RPG_OK;
  };
  if (trace) trace->stop_reason = found ? RPG_FIT_STOP_ROUNDS : RPG_FIT_STOP_FIRST_EMPTY;
  if (found && (rc = record(refined.as<double>()))) return rc;
  FCUDA(fit_malloc((void**)&w.p, sizeof(double) * (size_t)F.m));
  FCUDA(fit_malloc((void**)&Sw.p, sizeof(double) * n));
  DevBuf cdp;
  FCUDA(fit_malloc((void**)&cdp.p, sizeof(double) * nd));
  Pass P;
  for (int round = 0; found && round < 3; ++round) {
    FCUDA(cudaMemcpyAsync(cdp.p, refined.as<double>() + nn, sizeof(double) * nd,
                          cudaMemcpyDeviceToDevice, s));
    rc = run_den_pass(F, cdp.as<double>(), nullptr, nullptr, 1, 0, sms, &P, s, err, errlen);
    if (rc) return rc;
    double qmin = 0.0;
    FCUDA(cudaMemcpyAsync(&qmin, P.out.p, sizeof(double), cudaMemcpyDeviceToHost, s));
    FCUDA(cudaStreamSynchronize(s));
    if (trace) trace->round_qmin[round] = qmin;
    if (!(qmin > 0.0)) {
      if (trace) trace->stop_reason = RPG_FIT_STOP_QMIN;
      break;
    }
    const size_t smw = (size_t)kMaxCols * RPG_MAX_VARS + 16;
    row_weights<<<G, 256, smw, s>>>(F, cdp.as<double>(), w.as<double>());
    FitParams Fw = F;
    Fw.w = w.as<double>();
    DevBuf Rwb;
    rc = tsqr(Fw, n, sms, &Rwb, s, err, errlen);
    if (rc) return rc;
    col_scale_from_R<<<1, 64, 0, s>>>(Rwb.as<double>(), n, Sw.as<double>());
    int f2 = 0;
    rc = minimizer(F, Rwb.as<double>(), Sw.as<double>(), gsum.as<double>(), refined.as<double>(),
                   next.as<double>(), &f2, sms, s, err, errlen);
    if (rc) return rc;
    if (!f2) {
      if (trace) trace->stop_reason = RPG_FIT_STOP_EMPTY;
      break;
    }
    FCUDA(cudaMemcpyAsync(refined.p, next.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
    if ((rc = record(refined.as<double>()))) return rc;
  }
  if (found) FCUDA(cudaMemcpyAsync(c, refined.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
  FCUDA(cudaStreamSynchronize(s));
  return RPG_OK;
}

extern "C" int rpg_fit_rational(const double* X, const double* y, int64_t m, int32_t n_vars,
                                const int32_t* num_bounds, const int32_t* den_bounds,
                                double rank_tol, int32_t device, double* coef_out,
                                double* sigma_out, int32_t* rank_out, int32_t* truncated_out,
                                double* residual_out, int32_t* safeguard_out, char* err,
                                size_t errlen) {
  return rpg_fit_rational_traced(X, y, m, n_vars, num_bounds, den_bounds, rank_tol, device,
                                 coef_out, sigma_out, rank_out, truncated_out, residual_out,
                                 safeguard_out, nullptr, err, errlen);
}

namespace {
// One fit.  X: host samples (uploaded on this fit's stream), or dX: the
// same samples already resident on `device` (rpg_fit_rational_multi shares
// one upload between concurrent fits).
int fit_impl(const double* X, const double* dXs, const double* y, int64_t m, int32_t n_vars,
             const int32_t* num_bounds, const int32_t* den_bounds, double rank_tol,
             int32_t device, double* coef_out, double* sigma_out, int32_t* rank_out,
             int32_t* truncated_out, double* residual_out, int32_t* safeguard_out,
             rpg_fit_trace* trace, char* err, size_t errlen) {
  if (trace) {
    *trace = rpg_fit_trace{};
    trace->stop_reason = RPG_FIT_STOP_NO_SAFEGUARD;
  }
  if (m <= 0 || !(X || dXs) || !y) return fset_err(err, errlen, RPG_E_INVALID, "fit_rational: no samples");
  if (n_vars < 1 || n_vars > RPG_MAX_VARS || !num_bounds || !den_bounds)
    return fset_err(err, errlen, RPG_E_INVALID, "fit_rational: bad variable count");
  for (int v = 0; v < n_vars; ++v)
    if (num_bounds[v] < 0 || den_bounds[v] < 0)
      return fset_err(err, errlen, RPG_E_INVALID, "negative degree bound");
  const auto nb = basis(num_bounds, n_vars), db = basis(den_bounds, n_vars);
  const int nn = (int)nb.size(), nd = (int)db.size(), n = nn + nd;
  if (n > kMaxCols)
    return fset_err(err, errlen, RPG_E_INVALID,
                    "fit_rational: %d coefficients exceed the GPU fit's limit of %d", n, kMaxCols);
  std::vector<uint8_t> exps((size_t)n * n_vars);
  for (int k = 0; k < nn; ++k)
    for (int v = 0; v < n_vars; ++v) exps[(size_t)k * n_vars + v] = (uint8_t)nb[k][v];
  for (int k = 0; k < nd; ++k)
    for (int v = 0; v < n_vars; ++v) exps[(size_t)(nn + k) * n_vars + v] = (uint8_t)db[k][v];

  FCUDA(cudaSetDevice(device));
  cudaStream_t s;
  FCUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  struct StreamGuard {
    cudaStream_t s;
    ~StreamGuard() {
      cudaStreamSynchronize(s);
      g_fit_stream = nullptr;
      cudaStreamDestroy(s);
    }
  } sg{s};
  {
    // Keep freed scratch cached in the device's default pool between fits.
    static thread_local int pool_device = -1;
    if (pool_device != device) {
      cudaMemPool_t pool;
      if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t keep = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
      }
      pool_device = device;
    }
  }
  g_fit_stream = s;
  int sms = 148;
  FCUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  DevBuf dX, dy, dexps, dR, dsig, dV, dscale, dc, dpart, dflags, dstats, dU;
  if (!dXs) {
    FCUDA(fit_malloc((void**)&dX.p, sizeof(double) * (size_t)m * n_vars));
    FCUDA(cudaMemcpyAsync(dX.p, X, sizeof(double) * (size_t)m * n_vars, cudaMemcpyHostToDevice, s));
  }
  FCUDA(fit_malloc((void**)&dy.p, sizeof(double) * (size_t)m));
  FCUDA(fit_malloc((void**)&dexps.p, exps.size()));
  FCUDA(cudaMemcpyAsync(dy.p, y, sizeof(double) * (size_t)m, cudaMemcpyHostToDevice, s));
  FCUDA(cudaMemcpyAsync(dexps.p, exps.data(), exps.size(), cudaMemcpyHostToDevice, s));
  FCUDA(fit_malloc((void**)&dflags.p, sizeof(int) * 8));
  FCUDA(cudaMemsetAsync(dflags.p, 0, sizeof(int) * 8, s));

  FitParams F{};
  F.n_vars = n_vars;
  F.nn = nn;
  F.nd = nd;
  F.n = n;
  F.X = dXs ? dXs : dX.as<double>();
  F.y = dy.as<double>();
  F.w = nullptr;
  F.exps = dexps.as<uint8_t>();
  F.m = m;
  F.den01 = n_vars <= 4;
  for (size_t e = (size_t)nn * n_vars; e < exps.size(); ++e)
    if (exps[e] > 1) F.den01 = 0;
  {
    // monomial_basis({1, 1, 1}) (polyfit.hpp:50-73), the den_pass kSrcLat3 order
    static const uint8_t lat3[8][3] = {{0, 0, 0}, {0, 0, 1}, {0, 1, 0}, {1, 0, 0},
                                       {0, 1, 1}, {1, 0, 1}, {1, 1, 0}, {1, 1, 1}};
    F.den_lat3 = n_vars == 3 && nd == 8;
    for (int k = 0; F.den_lat3 && k < 8; ++k)
      for (int v = 0; v < 3; ++v)
        if (exps[(size_t)(nn + k) * 3 + v] != lat3[k][v]) F.den_lat3 = 0;
  }
  // RPG_FIT_TRACE=1: per-phase wall times on stderr (profiling aid).
  const bool phase_trace = getenv("RPG_FIT_TRACE") != nullptr;
  auto t_prev = std::chrono::steady_clock::now();
  auto phase = [&](const char* name) {
    if (!phase_trace) return;
    cudaStreamSynchronize(s);
    const auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "[rpg_fit] %-12s %9.3f ms\n", name,
            std::chrono::duration<double, std::milli>(now - t_prev).count());
    t_prev = now;
  };
  phase("upload");
  int rc = tsqr(F, n, sms, &dR, s, err, errlen);
  if (rc) return rc;
  phase("tsqr");
  // Non-finite entries of A propagate into R (svd, polyfit.hpp:163).
  all_finite<<<1, 256, 0, s>>>(dR.as<double>(), (int64_t)n * n, dflags.as<int>() + 4);
  FCUDA(fit_malloc((void**)&dsig.p, sizeof(double) * n));
  FCUDA(fit_malloc((void**)&dV.p, sizeof(double) * n * n));
  FCUDA(fit_malloc((void**)&dscale.p, sizeof(double) * n));
  FCUDA(fit_malloc((void**)&dc.p, sizeof(double) * n));
  const size_t sm3 = sizeof(double) * (2 * (size_t)kMaxCols * kMaxCols + kMaxCols) + sizeof(int) * (kMaxCols + 4);
  FCUDA(raise_smem_attr(reinterpret_cast<const void*>(svd_small), sm3));
  svd_small<<<1, svd_threads(n), sm3, s>>>(dR.as<double>(), n, dsig.as<double>(), dV.as<double>(),
                                        dscale.as<double>(), nullptr, 1);
  FCUDA(cudaGetLastError());
  smallest_vector<<<1, 64, 0, s>>>(dV.as<double>(), dscale.as<double>(), n, dc.as<double>());
  if (trace) {
    FCUDA(cudaMemcpyAsync(trace->stage_coef[0], dc.p, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
    trace->n_stages = 1;
  }
  // Safeguard trigger statistics.
  const int G = std::max(1, std::min<int>((int)((m + 255) / 256), 4 * sms));
  FCUDA(fit_malloc((void**)&dpart.p, sizeof(double) * 4 * G));
  FCUDA(fit_malloc((void**)&dstats.p, sizeof(double) * 4));
  const size_t sm4 = sizeof(double) * 32 + (size_t)kMaxCols * RPG_MAX_VARS + 16;
  den_stats<<<G, 256, sm4, s>>>(F, dc.as<double>() + nn, dpart.as<double>());
  den_stats_final<<<1, 32, 0, s>>>(dpart.as<double>(), G, m, dflags.as<int>() + 0,
                                   dstats.as<double>());
  int flags[8];
  FCUDA(cudaMemcpyAsync(flags, dflags.p, sizeof(flags), cudaMemcpyDeviceToHost, s));
  FCUDA(cudaStreamSynchronize(s));
  if (flags[4]) return fset_err(err, errlen, RPG_E_FIT, "svd: matrix has non-finite entries");
  const int trigger = flags[0];
  phase("svd+stats");
  if (trigger) {
    rc = rpg_fit_safeguard(F, dR.as<double>(), dscale.as<double>(), dc.as<double>(), rank_tol,
                           sms, s, err, errlen, trace);
    if (rc) return rc;
    phase("safeguard");
  }
  const int nsig = (int)std::min<int64_t>(m, n);
  fit_finalize<<<1, 32, 0, s>>>(dc.as<double>(), nn, nd, dsig.as<double>(), nsig, rank_tol,
                                dflags.as<int>() + 1, dflags.as<int>() + 2);
  FCUDA(cudaMemcpyAsync(flags, dflags.p, sizeof(flags), cudaMemcpyDeviceToHost, s));
  std::vector<double> sig(n);
  FCUDA(cudaMemcpyAsync(sig.data(), dsig.p, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
  if (coef_out)
    FCUDA(cudaMemcpyAsync(coef_out, dc.p, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
  FCUDA(cudaStreamSynchronize(s));
  if (flags[1] == 1) return fset_err(err, errlen, RPG_E_FIT, "all-zero coefficient vector");
  if (flags[1] == 2)
    return fset_err(err, errlen, RPG_E_FIT, "recovered denominator is identically zero");
  if (sigma_out) std::copy(sig.begin(), sig.begin() + nsig, sigma_out);
  if (rank_out) *rank_out = flags[2];
  if (truncated_out) *truncated_out = flags[2] < n - 1;
  if (residual_out) *residual_out = nsig >= n ? sig[n - 1] : 0.0;
  if (safeguard_out) *safeguard_out = trigger;
  return RPG_OK;
}

}  // namespace

extern "C" int rpg_fit_rational_traced(const double* X, const double* y, int64_t m, int32_t n_vars,
                                       const int32_t* num_bounds, const int32_t* den_bounds,
                                       double rank_tol, int32_t device, double* coef_out,
                                       double* sigma_out, int32_t* rank_out,
                                       int32_t* truncated_out, double* residual_out,
                                       int32_t* safeguard_out, rpg_fit_trace* trace, char* err,
                                       size_t errlen) {
  return fit_impl(X, nullptr, y, m, n_vars, num_bounds, den_bounds, rank_tol, device, coef_out,
                  sigma_out, rank_out, truncated_out, residual_out, safeguard_out, trace, err,
                  errlen);
}

// Several fits over one sample set (pipe::fit_all_metrics' loop, pipeline.hpp:
// 145-184): X is uploaded once, then every job runs on its own host thread and
// CUDA stream, so one fit's serial phases (the minimizer's per-step tail,
// host polls) overlap the others' sample passes.  Each job's outcome is what
// rpg_fit_rational returns for it alone (the fits are deterministic and
// independent).
extern "C" int rpg_fit_rational_multi(const double* X, int64_t m, int32_t n_vars,
                                      rpg_fit_job* jobs, int32_t n_jobs, double rank_tol,
                                      int32_t device, char* err, size_t errlen) {
  if (m <= 0 || !X) return fset_err(err, errlen, RPG_E_INVALID, "fit_rational: no samples");
  if (n_vars < 1 || n_vars > RPG_MAX_VARS)
    return fset_err(err, errlen, RPG_E_INVALID, "fit_rational: bad variable count");
  if (n_jobs < 0 || (n_jobs > 0 && !jobs))
    return fset_err(err, errlen, RPG_E_INVALID, "rpg_fit_rational_multi: bad job list");
  if (n_jobs == 0) return RPG_OK;
  FCUDA(cudaSetDevice(device));
  cudaStream_t s;
  FCUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  double* dX = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&dX, sizeof(double) * (size_t)m * n_vars, s);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(dX, X, sizeof(double) * (size_t)m * n_vars, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) {
    if (dX) cudaFreeAsync(dX, s);
    cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
    return fset_err(err, errlen, RPG_E_CUDA, "rpg_fit_rational_multi: %s", cudaGetErrorString(e));
  }
  std::vector<std::thread> th;
  for (int32_t k = 0; k < n_jobs; ++k)
    th.emplace_back([&, k] {
      rpg_fit_job& J = jobs[k];
      J.message[0] = 0;
      cudaSetDevice(device);
      J.status = fit_impl(nullptr, dX, J.y, m, n_vars, J.num_bounds, J.den_bounds, rank_tol,
                          device, J.coef_out, J.sigma_out, J.rank_out, J.truncated_out,
                          J.residual_out, J.safeguard_out, J.trace, J.message, sizeof J.message);
    });
  for (auto& t : th) t.join();
  cudaFreeAsync(dX, s);
  cudaStreamSynchronize(s);
  cudaStreamDestroy(s);
  return RPG_OK;
}
