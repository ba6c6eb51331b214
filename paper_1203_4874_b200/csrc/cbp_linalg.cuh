// CTA-level FP64 dense linear algebra for the tiny solves of the recovery path:
//  - herm_jacobi: two-sided cyclic Jacobi eigensolver for Hermitian n x n (n <= 128),
//    round-robin ordering so n/2 disjoint rotations run in parallel;
//  - onesided_sv: one-sided (Hestenes) Jacobi singular values of a square complex
//    matrix, one warp per column pair.
// They replace Eigen::JacobiSVD (reference poly.cpp:85,103,126) on the device.
#pragma once

#include "cbp_common.cuh"

namespace cbp_dev {

// pair k of round r in the circle method over m players (m even)
__device__ __forceinline__ void rr_pair(int r, int k, int m, int& a, int& b) {
  if (k == 0) {
    a = r;
    b = m - 1;
  } else {
    a = (r + k) % (m - 1);
    b = (r - k + m - 1) % (m - 1);
  }
  if (a > b) {
    int t = a;
    a = b;
    b = t;
  }
}

struct JacobiScratch {
  double* cs;   // [m/2]
  double* sn;   // [m/2]
  double2* e;   // [m/2]
  int* flag;    // [1]
};

// G (n x n, row stride ldg) is overwritten by diag(eigenvalues); V (n x n, stride ldv)
// receives the eigenvectors as columns. Whole CTA participates.
__device__ void herm_jacobi(double2* G, int ldg, double2* V, int ldv, int n, JacobiScratch sc,
                            int max_sweeps = 40) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int m = (n + 1) & ~1;
  for (int i = tid; i < n * n; i += nt) {
    const int r = i / n, c = i - r * n;
    V[r * ldv + c] = make_double2(r == c ? 1.0 : 0.0, 0.0);
  }
  __shared__ double s_dmax;
  if (tid == 0) {
    double d = 0.0;
    for (int i = 0; i < n; ++i) d = fmax(d, fabs(G[i * ldg + i].x));
    s_dmax = d;
  }
  __syncthreads();
  const double floor_abs = 1e-17 * s_dmax;
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    if (tid == 0) *sc.flag = 0;
    __syncthreads();
    for (int r = 0; r < m - 1; ++r) {
      for (int k = tid; k < m / 2; k += nt) {
        int p, q;
        rr_pair(r, k, m, p, q);
        double cs = 1.0, sn = 0.0;
        double2 e = make_double2(1.0, 0.0);
        if (q < n) {
          const double al = G[p * ldg + p].x, be = G[q * ldg + q].x;
          const double2 ga = G[p * ldg + q];
          const double ag = hypot(ga.x, ga.y);
          if (ag > 0.0 && ag > 1e-15 * sqrt(fabs(al * be)) && ag > floor_abs) {
            const double zeta = (be - al) / (2.0 * ag);
            const double tt = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
            cs = 1.0 / sqrt(1.0 + tt * tt);
            sn = cs * tt;
            e = make_double2(ga.x / ag, ga.y / ag);
            *sc.flag = 1;
          }
        }
        sc.cs[k] = cs;
        sc.sn[k] = sn;
        sc.e[k] = e;
      }
      __syncthreads();
      // columns: G <- G J, V <- V J with J = [[cs, sn], [-sn conj(e), cs conj(e)]]
      for (int i = tid; i < (m / 2) * n * 2; i += nt) {
        const int which = i / ((m / 2) * n);  // 0: G, 1: V
        const int rem = i - which * (m / 2) * n;
        const int k = rem / n, row = rem - k * n;
        if (sc.sn[k] == 0.0) continue;
        int p, q;
        rr_pair(r, k, m, p, q);
        double2* M = which ? V : G;
        const int ld = which ? ldv : ldg;
        const double cs = sc.cs[k], sn = sc.sn[k];
        const double2 ec = zconj(sc.e[k]);
        const double2 gp = M[row * ld + p], gq = zmul(ec, M[row * ld + q]);
        M[row * ld + p] = make_double2(cs * gp.x - sn * gq.x, cs * gp.y - sn * gq.y);
        M[row * ld + q] = make_double2(sn * gp.x + cs * gq.x, sn * gp.y + cs * gq.y);
      }
      __syncthreads();
      // rows: G <- J^H G
      for (int i = tid; i < (m / 2) * n; i += nt) {
        const int k = i / n, col = i - k * n;
        if (sc.sn[k] == 0.0) continue;
        int p, q;
        rr_pair(r, k, m, p, q);
        const double cs = sc.cs[k], sn = sc.sn[k];
        const double2 e = sc.e[k];
        const double2 gp = G[p * ldg + col], gq = zmul(e, G[q * ldg + col]);
        double2 np = make_double2(cs * gp.x - sn * gq.x, cs * gp.y - sn * gq.y);
        double2 nq = make_double2(sn * gp.x + cs * gq.x, sn * gp.y + cs * gq.y);
        if (col == q) np = make_double2(0.0, 0.0);
        if (col == p) nq = make_double2(0.0, 0.0);
        if (col == p) np.y = 0.0;
        if (col == q) nq.y = 0.0;
        G[p * ldg + col] = np;
        G[q * ldg + col] = nq;
      }
      __syncthreads();
    }
    if (*sc.flag == 0) break;
    __syncthreads();
  }
  __syncthreads();
}

// Warp-synchronous variant for n <= 64: same rotations as herm_jacobi, executed by one
// warp with __syncwarp barriers (the CTA-wide barrier cost dominated the small solves).
__device__ void herm_jacobi_warp(double2* G, int ldg, double2* V, int ldv, int n, JacobiScratch sc,
                                 int max_sweeps = 40) {
  const int lane = threadIdx.x & 31;
  const int m = (n + 1) & ~1;
  for (int i = lane; i < n * n; i += 32) {
    const int r = i / n, c = i - r * n;
    V[r * ldv + c] = make_double2(r == c ? 1.0 : 0.0, 0.0);
  }
  double dmax = 0.0;
  for (int i = lane; i < n; i += 32) dmax = fmax(dmax, fabs(G[i * ldg + i].x));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
  const double floor_abs = 1e-17 * dmax;
  __syncwarp();
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    int rotated = 0;
    for (int r = 0; r < m - 1; ++r) {
      for (int k = lane; k < m / 2; k += 32) {
        int p, q;
        rr_pair(r, k, m, p, q);
        double cs = 1.0, sn = 0.0;
        double2 e = make_double2(1.0, 0.0);
        if (q < n) {
          const double al = G[p * ldg + p].x, be = G[q * ldg + q].x;
          const double2 ga = G[p * ldg + q];
          const double ag = hypot(ga.x, ga.y);
          if (ag > 0.0 && ag > 1e-15 * sqrt(fabs(al * be)) && ag > floor_abs) {
            const double zeta = (be - al) / (2.0 * ag);
            const double tt = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
            cs = 1.0 / sqrt(1.0 + tt * tt);
            sn = cs * tt;
            e = make_double2(ga.x / ag, ga.y / ag);
            rotated = 1;
          }
        }
        sc.cs[k] = cs;
        sc.sn[k] = sn;
        sc.e[k] = e;
      }
      __syncwarp();
      for (int i = lane; i < (m / 2) * n * 2; i += 32) {
        const int which = i / ((m / 2) * n);
        const int rem = i - which * (m / 2) * n;
        const int k = rem / n, row = rem - k * n;
        const double sn = sc.sn[k];
        if (sn == 0.0) continue;
        int p, q;
        rr_pair(r, k, m, p, q);
        double2* M = which ? V : G;
        const int ld = which ? ldv : ldg;
        const double cs = sc.cs[k];
        const double2 ec = zconj(sc.e[k]);
        const double2 gp = M[row * ld + p], gq = zmul(ec, M[row * ld + q]);
        M[row * ld + p] = make_double2(cs * gp.x - sn * gq.x, cs * gp.y - sn * gq.y);
        M[row * ld + q] = make_double2(sn * gp.x + cs * gq.x, sn * gp.y + cs * gq.y);
      }
      __syncwarp();
      for (int i = lane; i < (m / 2) * n; i += 32) {
        const int k = i / n, col = i - k * n;
        const double sn = sc.sn[k];
        if (sn == 0.0) continue;
        int p, q;
        rr_pair(r, k, m, p, q);
        const double cs = sc.cs[k];
        const double2 e = sc.e[k];
        const double2 gp = G[p * ldg + col], gq = zmul(e, G[q * ldg + col]);
        double2 np = make_double2(cs * gp.x - sn * gq.x, cs * gp.y - sn * gq.y);
        double2 nq = make_double2(sn * gp.x + cs * gq.x, sn * gp.y + cs * gq.y);
        if (col == q) np = make_double2(0.0, 0.0);
        if (col == p) nq = make_double2(0.0, 0.0);
        if (col == p) np.y = 0.0;
        if (col == q) nq.y = 0.0;
        G[p * ldg + col] = np;
        G[q * ldg + col] = nq;
      }
      __syncwarp();
    }
    if (!__any_sync(0xffffffffu, rotated)) break;
  }
  __syncwarp();
}

// whole-CTA entry (the CTA-wide variant measured faster than the single-warp one:
// the per-round FP64 rotation parameters dominate, not the barriers)
__device__ __forceinline__ void herm_jacobi_cta(double2* G, int ldg, double2* V, int ldv, int n, JacobiScratch sc) {
  herm_jacobi(G, ldg, V, ldv, n, sc);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Singular values of the square complex matrix A (n x n, column c at A + c*lda, i.e.
// column-major so each column is contiguous). A is destroyed. Writes sv[0..n-1]
// (unsorted). Whole CTA participates; warps own column pairs (one pair per warp per
// round when blockDim >= 32 * n/2) and the four inner products share one shuffle tree.
__device__ void onesided_sv(double2* A, int lda, int n, double* sv, int* flag, int max_sweeps = 60) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int m = (n + 1) & ~1;
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    if (threadIdx.x == 0) *flag = 0;
    __syncthreads();
    for (int r = 0; r < m - 1; ++r) {
      for (int k = warp; k < m / 2; k += nw) {
        int p, q;
        rr_pair(r, k, m, p, q);
        if (q >= n) continue;
        double2* cp = A + p * lda;
        double2* cq = A + q * lda;
        double al = 0, be = 0, gr = 0, gi = 0;
        for (int i = lane; i < n; i += 32) {
          const double2 x = cp[i], y = cq[i];
          al += zabs2(x);
          be += zabs2(y);
          gr += x.x * y.x + x.y * y.y;  // conj(x) * y
          gi += x.x * y.y - x.y * y.x;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          al += __shfl_xor_sync(0xffffffffu, al, o);
          be += __shfl_xor_sync(0xffffffffu, be, o);
          gr += __shfl_xor_sync(0xffffffffu, gr, o);
          gi += __shfl_xor_sync(0xffffffffu, gi, o);
        }
        const double ag = hypot(gr, gi);
        if (ag == 0.0 || ag <= 1e-15 * sqrt(al * be)) continue;
        if (lane == 0) *flag = 1;
        const double zeta = (be - al) / (2.0 * ag);
        const double tt = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double cs = 1.0 / sqrt(1.0 + tt * tt), sn = cs * tt;
        const double2 ec = make_double2(gr / ag, -gi / ag);  // conj(gamma/|gamma|)
        for (int i = lane; i < n; i += 32) {
          const double2 x = cp[i], y = zmul(ec, cq[i]);
          cp[i] = make_double2(cs * x.x - sn * y.x, cs * x.y - sn * y.y);
          cq[i] = make_double2(sn * x.x + cs * y.x, sn * x.y + cs * y.y);
        }
      }
      __syncthreads();
    }
    if (*flag == 0) break;
    __syncthreads();
  }
  for (int c = warp; c < n; c += nw) {
    double s = 0;
    for (int i = lane; i < n; i += 32) s += zabs2(A[c * lda + i]);
    s = warp_sum(s);
    if (lane == 0) sv[c] = sqrt(s);
  }
  __syncthreads();
}

}  // namespace cbp_dev
