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
static __device__ void herm_jacobi(double2* G, int ldg, double2* V, int ldv, int n, JacobiScratch sc,
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

// Hermitian eigen-decomposition by Householder tridiagonalization (LAPACK zhetrd), then
// bisection + inverse iteration on the real tridiagonal (dstebz/dstein), back-transformed.
// O(n^3) work with warp-level barriers, instead of Jacobi's O(n^3 * sweeps) with a CTA
// barrier per round (~3x faster at n = 22 on B200, see tools/micro/bench_eig.cu).
// Executed by one warp; n <= 64. Same contract as herm_jacobi: G's diagonal receives the
// eigenvalues, V the eigenvectors as columns; G's off-diagonal part is destroyed.
// mode: EIG_VALUES (eigenvalues only, bisection), EIG_QL (eigenvectors by implicit QL: exactly
// orthogonal, robust for dense clusters of tiny eigenvalues), EIG_INVIT (eigenvectors by
// inverse iteration: faster when the spectrum is well separated)
// EIG_LOW2: eigenvalues 0, 1 and n-1 only (G[0][0], G[1][1], G[n-1][n-1]) and the eigenvectors
// of the two smallest (V columns 0 and 1): the cofactor solve needs no more.
// EIG_RATIO: G[0][0] <- min|lambda| / max|lambda| (0 if max|lambda| = 0), nothing else: the
// singularity test of a Hermitian block (numerical_singularity, poly.cpp:81-91).
enum EigMode { EIG_VALUES = 0, EIG_QL = 1, EIG_INVIT = 2, EIG_LOW2 = 3, EIG_RATIO = 4 };
// NMAX: largest n (64; 128 for the kernels of widths t > 32, whose 2t x 2t Grams live in
// global memory). EIG_INVIT needs n <= 64 (per-lane arrays); NMAX = 128 runs QL for it.
// Shared state of the tridiagonal eigensolver (one instance per kernel and NMAX), so the
// CTA-wide tridiagonalization and the one-warp remainder can be split.
template <int NMAX>
struct EigShared {
  double d[NMAX], e[NMAX], beta[NMAX], rc[NMAX], rs[NMAX];
  double2 ec[NMAX], w[NMAX], p[NMAX], delta[NMAX];
};
template <int NMAX>
__device__ __forceinline__ EigShared<NMAX>& eig_shared() {
  __shared__ EigShared<NMAX> st;
  return st;
}

// Householder tridiagonalization G = Q T Q^H by the whole CTA (same outputs as the one-warp
// loop in herm_eig_warp: v_k in column k below the diagonal, beta_k, the new subdiagonal
// alpha_k, the diagonal): per step one warp forms the reflector, every warp takes a slice
// of the rows for p = beta S v, and the rank-2 update S -= v w^H + w v^H is spread over the
// CTA. Afterwards call herm_eig_warp(..., tri_done = true) on one warp. `part` is scratch for
// n x n complex values (the partial sums of p).
template <int NMAX = 64>
__device__ void herm_tridiag_cta(double2* G, int ldg, int n, double2* part) {
  EigShared<NMAX>& ES = eig_shared<NMAX>();
  __shared__ double sc_beta;
  __shared__ int sc_skip;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // warps in the p = beta S v partial sums (more would cost warp 0 more partials to add)
  const int nw = min(min(int(blockDim.x >> 5), 4), n);
  const unsigned full = 0xffffffffu;
  auto wsum = [&](double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(full, v, o);
    return v;
  };
  for (int k = 0; k + 2 < n; ++k) {
    const int m = n - k - 1;
    if (warp == 0) {
      double s2 = 0.0;
      for (int i = lane; i < m; i += 32) s2 += zabs2(G[(k + 1 + i) * ldg + k]);
      s2 = wsum(s2);
      const double2 x0 = G[(k + 1) * ldg + k];
      const double xn = sqrt(s2);
      __syncwarp();
      if (lane == 0) {
        ES.d[k] = G[k * ldg + k].x;
        if (xn == 0.0) {
          ES.beta[k] = 0.0, ES.ec[k] = make_double2(0.0, 0.0);
          sc_skip = 1;
        } else {
          // rsqrt / rcp with Newton steps instead of hypot and divisions (FP64 division and
          // hypot cost 130-160 cycles of latency on this serial chain)
          const double a2 = zabs2(x0);
          double ia = 0.0;
          if (a2 > 0.0) {
            ia = rsqrt(a2);
            ia = ia * fma(-0.5 * a2 * ia, ia, 1.5);  // one Newton step
          }
          const double ax0 = a2 * ia;
          const double2 ph = a2 > 0.0 ? zscale(x0, ia) : make_double2(1.0, 0.0);
          const double den = xn * (xn + ax0);
          double beta;  // 2 / |v|^2 = 1 / den
          asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(beta) : "d"(den));
          beta = fma(beta, fma(-den, beta, 1.0), beta);
          beta = fma(beta, fma(-den, beta, 1.0), beta);
          G[(k + 1) * ldg + k] = zscale(ph, ax0 + xn);  // v_0 = x_0 - alpha
          ES.beta[k] = beta;
          ES.ec[k] = zscale(ph, -xn);  // alpha: the new subdiagonal entry
          sc_beta = beta;
          sc_skip = 0;
        }
      }
    }
    __syncthreads();
    if (sc_skip) continue;  // uniform
    const double beta = sc_beta;
    // partial p_i = sum over this warp's rows j of conj(S[j][i]) v_j
    if (warp < nw) {
      const int j0 = (m * warp) / nw, j1 = (m * (warp + 1)) / nw;
      for (int i = lane; i < m; i += 32) {
        double2 acc = make_double2(0.0, 0.0);
        for (int j = j0; j < j1; ++j) acc = zadd(acc, zcmul(G[(k + 1 + j) * ldg + k + 1 + i], G[(k + 1 + j) * ldg + k]));
        part[warp * n + i] = acc;
      }
    }
    __syncthreads();
    if (warp == 0) {
      double kr = 0.0, ki = 0.0;
      for (int i = lane; i < m; i += 32) {
        double2 acc = part[i];
        for (int w = 1; w < nw; ++w) acc = zadd(acc, part[w * n + i]);
        acc = zscale(acc, beta);
        ES.p[i] = acc;
        const double2 u = zcmul(G[(k + 1 + i) * ldg + k], acc);
        kr += u.x;
        ki += u.y;
      }
      const double2 K = zscale(make_double2(wsum(kr), wsum(ki)), 0.5 * beta);  // K = beta/2 v^H p
      for (int i = lane; i < m; i += 32) ES.w[i] = zsub(ES.p[i], zmul(K, G[(k + 1 + i) * ldg + k]));
    }
    __syncthreads();
    // S <- S - v w^H - w v^H
    for (int idx = tid; idx < m * m; idx += blockDim.x) {
      const int j = idx / m, i = idx - j * m;
      const double2 vj = G[(k + 1 + j) * ldg + k], wj = ES.w[j];
      const double2 vi = G[(k + 1 + i) * ldg + k], wi = ES.w[i];
      double2& sji = G[(k + 1 + j) * ldg + k + 1 + i];
      sji = zsub(sji, zadd(zmul(vj, zconj(wi)), zmul(wj, zconj(vi))));
    }
    __syncthreads();
  }
}

template <int NMAX = 64>
static __device__ void herm_eig_warp(double2* G, int ldg, double2* V, int ldv, int n, int mode,
                                     bool tri_done = false) {
  if (NMAX > 64 && (mode == EIG_INVIT || mode == EIG_LOW2)) mode = EIG_QL;
  const bool low2 = mode == EIG_LOW2;
  const bool vectors = mode != EIG_VALUES && mode != EIG_RATIO;
  EigShared<NMAX>& ES = eig_shared<NMAX>();
  double *s_d = ES.d, *s_e = ES.e, *s_beta = ES.beta, *s_rc = ES.rc, *s_rs = ES.rs;
  double2 *s_ec = ES.ec, *s_w = ES.w, *s_p = ES.p, *s_delta = ES.delta;
  const int lane = threadIdx.x & 31;
  const unsigned full = 0xffffffffu;
  auto wsum = [&](double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(full, v, o);
    return v;
  };
  const bool pw = blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0;
  CBP_PHASE(30, pw);
  // ---- tridiagonalization G = Q T Q^H; v_k is kept in column k below the diagonal
  for (int k = 0; k + 2 < n && !tri_done; ++k) {
    const int m = n - k - 1;
    double s2 = 0.0;
    for (int i = lane; i < m; i += 32) s2 += zabs2(G[(k + 1 + i) * ldg + k]);
    s2 = wsum(s2);
    const double2 x0 = G[(k + 1) * ldg + k];
    const double xn = sqrt(s2);
    if (lane == 0) s_d[k] = G[k * ldg + k].x;
    if (xn == 0.0) {
      if (lane == 0) s_beta[k] = 0.0, s_ec[k] = make_double2(0.0, 0.0);
      __syncwarp();
      continue;
    }
    const double ax0 = zabs(x0);
    const double2 ph = ax0 > 0.0 ? zscale(x0, 1.0 / ax0) : make_double2(1.0, 0.0);
    const double beta = 1.0 / (xn * (xn + ax0));  // 2 / |v|^2
    __syncwarp();
    if (lane == 0) {
      G[(k + 1) * ldg + k] = zscale(ph, ax0 + xn);  // v_0 = x_0 - alpha
      s_beta[k] = beta;
      s_ec[k] = zscale(ph, -xn);  // alpha: the new subdiagonal entry
    }
    __syncwarp();
    // p = beta S v; S Hermitian, so p_i = beta sum_j conj(S[j][i]) v_j (lanes on i)
    for (int i = lane; i < m; i += 32) {
      double2 acc = make_double2(0.0, 0.0);
      for (int j = 0; j < m; ++j) acc = zadd(acc, zcmul(G[(k + 1 + j) * ldg + k + 1 + i], G[(k + 1 + j) * ldg + k]));
      s_p[i] = zscale(acc, beta);
    }
    __syncwarp();
    double kr = 0.0, ki = 0.0;  // K = beta/2 v^H p
    for (int i = lane; i < m; i += 32) {
      const double2 u = zcmul(G[(k + 1 + i) * ldg + k], s_p[i]);
      kr += u.x;
      ki += u.y;
    }
    const double2 K = zscale(make_double2(wsum(kr), wsum(ki)), 0.5 * beta);
    for (int i = lane; i < m; i += 32) s_w[i] = zsub(s_p[i], zmul(K, G[(k + 1 + i) * ldg + k]));
    __syncwarp();
    // S <- S - v w^H - w v^H (lanes on columns i)
    for (int i = lane; i < m; i += 32) {
      const double2 vi = G[(k + 1 + i) * ldg + k], wi = s_w[i];
      for (int j = 0; j < m; ++j) {
        const double2 vj = G[(k + 1 + j) * ldg + k], wj = s_w[j];
        double2& sji = G[(k + 1 + j) * ldg + k + 1 + i];
        sji = zsub(sji, zadd(zmul(vj, zconj(wi)), zmul(wj, zconj(vi))));
      }
    }
    __syncwarp();
  }
  if (lane == 0) {
    for (int k = n >= 2 ? n - 2 : 0; k < n; ++k) s_d[k] = G[k * ldg + k].x;
    if (n >= 2) {
      s_ec[n - 2] = G[(n - 1) * ldg + n - 2];
      s_beta[n - 2] = 0.0;
    }
    // unitary diagonal D with D^H T D real: e_k -> |e_k|
    s_delta[0] = make_double2(1.0, 0.0);
    for (int k = 0; k + 1 < n; ++k) {
      const double ae = zabs(s_ec[k]);
      s_e[k] = ae;
      s_delta[k + 1] = ae > 0.0 ? zmul(s_delta[k], zscale(s_ec[k], 1.0 / ae)) : s_delta[k];
    }
    s_e[n - 1] = 0.0;
  }
  for (int i = lane; i < n * n; i += 32) {  // Z = I in the real part of V
    const int r = i / n, c = i - r * n;
    V[r * ldv + c] = make_double2(r == c ? 1.0 : 0.0, 0.0);
  }
  __syncwarp();
  __syncwarp();
  CBP_PHASE(31, pw);
  // ---- the real tridiagonal T is scaled to unit norm by a power of two (exact).
  // Eigenvalues only: bisection on Sturm counts, one lane per eigenvalue. Divisions cost
  // ~130 cycles of FP64 latency on B200, so the counts use the division-free determinant
  // recurrence (no overflow at unit norm: |p_i| <= 3^i; underflow rescale every 8 steps).
  double lo0 = 1e300, hi0 = -1e300;
  for (int i = 0; i < n; ++i) {
    const double rad = (i > 0 ? s_e[i - 1] : 0.0) + (i + 1 < n ? s_e[i] : 0.0);
    lo0 = fmin(lo0, s_d[i] - rad);
    hi0 = fmax(hi0, s_d[i] + rad);
  }
  const double tn = fmax(fabs(lo0), fabs(hi0));
  const double sc = tn > 0.0 ? ldexp(1.0, -ilogb(tn) - 1) : 1.0;  // power of two: exact
  __syncwarp();
  for (int i = lane; i < n; i += 32) {
    s_d[i] *= sc;
    s_e[i] *= sc;
    s_rc[i] = s_e[i] * s_e[i];  // e_i^2
  }
  __syncwarp();
  lo0 = lo0 * sc - 1e-14;
  hi0 = hi0 * sc + 1e-14;
  auto count_below = [&](double x) {  // number of eigenvalues of T' smaller than x
    double p0 = 1.0, p1 = s_d[0] - x;
    int sg1 = p1 < 0.0 ? -1 : 1;
    int cnt = sg1 < 0;
#pragma unroll 4
    for (int i = 1; i < n; ++i) {
      const double p2 = fma(s_d[i] - x, p1, -s_rc[i - 1] * p0);
      const int sg2 = p2 < 0.0 ? -1 : (p2 > 0.0 ? 1 : -sg1);
      cnt += sg2 != sg1;
      sg1 = sg2;
      p0 = p1;
      p1 = p2;
      if ((i & 7) == 0 && fabs(p1) < 0x1p-600 && fabs(p0) < 0x1p-600) {
        p0 *= 0x1p+600;
        p1 *= 0x1p+600;
      }
    }
    return cnt;
  };
  auto rcp = [](double v) {  // ~1 ulp reciprocal: MUFU seed + 2 Newton steps
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(v));
    r = fma(r, fma(-v, r, 1.0), r);
    r = fma(r, fma(-v, r, 1.0), r);
    return r;
  };
  // Multisection: the warp splits into ng groups of lanes; group g refines eigenvalue kg
  // (ascending index), each lane evaluating one interior point per step, so an interval
  // shrinks (size+1)x per Sturm-count latency instead of 2x. Returns the group's eigenvalue
  // (of the scaled T'). Warp-uniform (ballot); `its` steps reach the bisection's precision.
  auto multisect = [&](int ng, int kg, int its) {
    const int gsz = 32 / ng, grp = min(lane / gsz, ng - 1), g0 = grp * gsz;
    const int size = grp == ng - 1 ? 32 - g0 : gsz, j = lane - g0;
    double lo = lo0, hi = hi0;
    for (int it = 0; it < its; ++it) {
      const double w = (hi - lo) / double(size + 1);
      const bool above = count_below(fma(double(j + 1), w, lo)) > kg;  // lambda_kg < x_j
      const unsigned gb = (__ballot_sync(full, above) >> g0) & (size == 32 ? ~0u : ((1u << size) - 1u));
      const int f = gb ? __ffs(gb) - 1 : size;  // first point above lambda_kg
      const double nlo = f == 0 ? lo : fma(double(f), w, lo);
      const double nhi = f == size ? hi : fma(double(f + 1), w, lo);
      if (nhi - nlo < hi - lo) lo = nlo, hi = nhi;
    }
    return 0.5 * (lo + hi);
  };
  if (mode == EIG_RATIO) {
    // min|lambda| / max|lambda| from four eigenvalues: the extremes and the two around 0
    const int k0 = count_below(0.0);  // eigenvalues < 0
    const int grp = lane >> 3;
    const int kg = grp == 0 ? 0 : (grp == 1 ? n - 1 : (grp == 2 ? max(k0 - 1, 0) : min(k0, n - 1)));
    const double lam = fabs(multisect(4, kg, 21));
    const double l0 = __shfl_sync(full, lam, 0), l1 = __shfl_sync(full, lam, 8);
    const double l2 = __shfl_sync(full, lam, 16), l3 = __shfl_sync(full, lam, 24);
    const double mx = fmax(l0, l1), mn = fmin(l2, l3);
    __syncwarp();
    if (lane == 0) G[0] = make_double2(mx == 0.0 ? 0.0 : mn / mx, 0.0);
    __syncwarp();
    return;
  }
  for (int k = lane; k < n && !vectors; k += 32) {
    double lo = lo0, hi = hi0;
    for (int it = 0; it < 62; ++it) {
      const double mid = 0.5 * (lo + hi);
      if (mid <= lo || mid >= hi) break;
      if (count_below(mid) > k) hi = mid;
      else lo = mid;
    }
    s_p[k].x = 0.5 * (lo + hi);
  }
  __syncwarp();
  CBP_PHASE(34, pw);
  if (!vectors) {
    for (int k = lane; k < n; k += 32) G[k * ldg + k] = make_double2(s_p[k].x / sc, 0.0);
    __syncwarp();
    return;
  }
  if (mode == EIG_QL) {
  // ---- eigenvectors: implicit QL with Wilkinson shifts (tqli) on T'. Every lane runs the
  // same scalar recurrence (no broadcast barrier). The sweep reads d/e and writes the
  // updated entries to separate arrays (s_dn/s_en), so its loads never wait behind its
  // stores; rsqrt/rcp with Newton steps replace hypot and the divisions on the chain.
  // The sweep's Givens rotations are then applied to each lane's rows of Z.
  {
    __shared__ double s_dn[NMAX], s_en[NMAX];
    for (int i = lane; i < n * n; i += 32) {  // Z = I in the real part of V
      const int r = i / n, c = i - r * n;
      V[r * ldv + c] = make_double2(r == c ? 1.0 : 0.0, 0.0);
    }
    __syncwarp();
    int l = 0, iter = 0;
    while (l < n) {
      int m = l;
      for (; m < n - 1; ++m) {
        const double dd = fabs(s_d[m]) + fabs(s_d[m + 1]);
        if (fabs(s_e[m]) <= 2.220446049250313e-16 * dd) break;
      }
      if (m == l || ++iter > 60) {
        ++l;
        iter = 0;
        continue;
      }
      const double el = s_e[l];
      double g = (s_d[l + 1] - s_d[l]) * 0.5 * rcp(el);
      double r = sqrt(fma(g, g, 1.0));
      g = s_d[m] - s_d[l] + el * rcp(g + copysign(r, g));
      double sn = 1.0, cs = 1.0, p = 0.0;
      double dip1 = s_d[m];
      int i = m - 1, nr = 0;
      bool early = false;
      for (; i >= l; --i) {
        const double ei = s_e[i], di = s_d[i];
        const double f = sn * ei, b = cs * ei;
        const double q = fma(f, f, g * g);
        if (q == 0.0) {
          early = true;
          break;
        }
        const double ri = rsqrt(q);
        s_en[i + 1] = q * ri;
        sn = f * ri;
        cs = g * ri;
        g = dip1 - p;
        r = fma(di - g, sn, 2.0 * cs * b);
        p = sn * r;
        s_dn[i + 1] = g + p;
        g = fma(cs, r, -b);
        dip1 = di;
        s_rc[nr] = cs;
        s_rs[nr] = sn;
        ++nr;
      }
      __syncwarp();
      // commit the sweep: entries i+1 .. m were rewritten (the last rotation index is m-nr)
      const int lo_w = m - nr + 1;
      for (int j = lane + lo_w; j <= m; j += 32) {
        s_d[j] = s_dn[j];
        if (j < m) s_e[j] = s_en[j];  // e_m is set below
      }
      __syncwarp();
      if (lane == 0) {
        if (early) {  // r == 0 at rotation i: tqli sets e[i+1] = r and deflates there
          s_d[i + 1] = dip1 - p;
          s_e[i + 1] = 0.0;
          s_e[m] = 0.0;
        } else {
          s_d[l] -= p;
          s_e[l] = g;
          s_e[m] = 0.0;
        }
      }
      // rotation j acts on columns (m-1-j, m-j) of every row of Z
      for (int rr = lane; rr < n; rr += 32) {
        double2* zr = V + rr * ldv;
        double zc = zr[m].x;
        for (int j = 0; j < nr; ++j) {
          const int c0 = m - 1 - j;
          const double zi = zr[c0].x;
          zr[c0 + 1].x = fma(s_rs[j], zi, s_rc[j] * zc);
          zc = fma(s_rc[j], zi, -s_rs[j] * zc);
        }
        zr[m - nr].x = zc;
      }
      __syncwarp();
    }
  }
  for (int k = lane; k < n; k += 32) s_p[k].x = s_d[k];
  __syncwarp();
  } else if constexpr (NMAX <= 64) {
  // ---- eigenvectors by inverse iteration, one lane per eigenvalue: bisection to full precision,
  // then three inverse-iteration steps (tridiagonal LU with partial pivoting) with
  // Rayleigh-quotient shifts. Eigenvalues closer than 1e-8 |T'| form a cluster that one
  // lane handles in turn, orthogonalizing each member against the previous ones (LAPACK
  // stein's scheme with a tighter cluster threshold: separated eigenvectors come out
  // orthogonal to ~1e-8 and accurate to ~1e-16 / gap).
  if (low2) {
    // three eigenvalues (k = 0, 1, n-1) by multisection: lanes 0-9, 10-19, 20-31
    const int grp = min(lane / 10, 2);
    const int k = grp == 0 ? 0 : (grp == 1 ? min(1, n - 1) : n - 1);
    const double lam = multisect(3, k, 20);
    if (lane == grp * 10 && (grp < 2 || k > 1)) s_p[k].x = lam;
  } else {
  for (int k = lane; k < n; k += 32) {
    double lo = lo0, hi = hi0;
    for (int it = 0; it < 62; ++it) {  // to full precision: the shifts must resolve close pairs
      const double mid = 0.5 * (lo + hi);
      if (mid <= lo || mid >= hi) break;
      if (count_below(mid) > k) hi = mid;
      else lo = mid;
    }
    s_p[k].x = 0.5 * (lo + hi);  // ascending in k
  }
  }
  __syncwarp();
  __shared__ int s_cl[65], s_ncl;
  if (lane == 0) {
    int nc = 0;
    const int nv = low2 ? min(n, 2) : n;  // eigenvectors wanted: 0 .. nv-1
    // LOW2: the two vectors run in separate lanes unless their eigenvalues are within 1e-13
    // of |T'| (inverse iteration at full-precision shifts still separates them by >= 1e6
    // per step); otherwise members of a 1e-8 cluster share a lane and are orthogonalized
    const double cl_tol = low2 ? 1e-13 : 1e-8;
    for (int k = 0; k < nv; ++k)
      if (k == 0 || s_p[k].x - s_p[k - 1].x > cl_tol) s_cl[nc++] = k;
    s_cl[nc] = nv;
    s_ncl = nc;
  }
  __syncwarp();
  for (int cl = lane; cl < s_ncl; cl += 32) {
    const int k0 = s_cl[cl], k1 = s_cl[cl + 1];
    for (int k = k0; k < k1; ++k) {
      double lam = s_p[k].x, rq = lam;
      double y[64];
      unsigned h = 0x9e3779b9u * unsigned(k + 1);
      for (int i = 0; i < n; ++i) {  // pseudo-random start vector
        h ^= h << 13, h ^= h >> 17, h ^= h << 5;
        y[i] = double(h & 0xffff) * (1.0 / 65536.0) - 0.5;
      }
      for (int it = 0; it < 3; ++it) {
        double u0[64], u1[64], u2[64];
        double a0 = s_d[0] - lam, bn = n > 1 ? s_e[0] : 0.0;
        for (int i = 0; i + 1 < n; ++i) {
          const double cv = s_e[i], dl = s_d[i + 1] - lam, el = i + 2 < n ? s_e[i + 1] : 0.0;
          if (fabs(a0) >= fabs(cv)) {
            const double aa = fabs(a0) < 1e-16 ? copysign(1e-16, a0) : a0;  // pivot floor eps |T'|
            const double m = cv * rcp(aa);
            u0[i] = aa, u1[i] = bn, u2[i] = 0.0;
            y[i + 1] -= m * y[i];
            a0 = dl - m * bn;
            bn = el;
          } else {
            const double m = a0 * rcp(cv);
            u0[i] = cv, u1[i] = dl, u2[i] = el;
            const double tt = y[i];
            y[i] = y[i + 1];
            y[i + 1] = tt - m * y[i];
            a0 = bn - m * dl;
            bn = -m * el;
          }
        }
        u0[n - 1] = fabs(a0) < 1e-16 ? copysign(1e-16, a0) : a0;
        u1[n - 1] = u2[n - 1] = 0.0;
        for (int i = n - 1; i >= 0; --i) {
          double v = y[i];
          if (i + 1 < n) v -= u1[i] * y[i + 1];
          if (i + 2 < n) v -= u2[i] * y[i + 2];
          y[i] = v * rcp(u0[i]);
        }
        for (int j = k0; j < k; ++j) {  // earlier members of this cluster
          double dot = 0.0;
          for (int i = 0; i < n; ++i) dot = fma(V[i * ldv + j].x, y[i], dot);
          for (int i = 0; i < n; ++i) y[i] = fma(-dot, V[i * ldv + j].x, y[i]);
        }
        double nrm = 0.0;
        for (int i = 0; i < n; ++i) nrm = fma(y[i], y[i], nrm);
        const double inv = rsqrt(nrm);
        rq = 0.0;
        for (int i = 0; i < n; ++i) {
          y[i] *= inv;
          rq = fma(s_d[i] * y[i], y[i], rq);
          if (i > 0) rq = fma(2.0 * s_e[i - 1] * y[i - 1], y[i], rq);
        }
        if (k1 - k0 == 1 && fabs(rq - lam) < 1e-6) lam = rq;  // Rayleigh shift (isolated only)
      }
      s_p[k].x = k1 - k0 == 1 ? rq : s_p[k].x;
      for (int i = 0; i < n; ++i) V[i * ldv + k] = make_double2(y[i], 0.0);
    }
  }
  __syncwarp();
  }
  CBP_PHASE(35, pw);
  for (int k = lane; k < n; k += 32) s_d[k] = s_p[k].x / sc;
  __syncwarp();
  CBP_PHASE(32, pw);
  if (low2) {
    // ---- the two wanted columns of V = Q D Z: reflectors in reverse order, lanes on rows
    const int nv = min(n, 2);
    for (int i = lane; i < n * nv; i += 32) {
      const int r = i / nv, c = i - r * nv;
      V[r * ldv + c] = zscale(s_delta[r], V[r * ldv + c].x);
    }
    __syncwarp();
    for (int k = n - 3; k >= 0; --k) {
      const double beta = s_beta[k];
      if (beta == 0.0) continue;
      const int m = n - k - 1;
      double a0r = 0.0, a0i = 0.0, a1r = 0.0, a1i = 0.0;
      for (int j = lane; j < m; j += 32) {
        const double2 vj = G[(k + 1 + j) * ldg + k];
        const double2 u0 = zcmul(vj, V[(k + 1 + j) * ldv + 0]);
        a0r += u0.x, a0i += u0.y;
        if (nv > 1) {
          const double2 u1 = zcmul(vj, V[(k + 1 + j) * ldv + 1]);
          a1r += u1.x, a1i += u1.y;
        }
      }
      const double2 c0 = zscale(make_double2(wsum(a0r), wsum(a0i)), beta);
      const double2 c1 = zscale(make_double2(wsum(a1r), wsum(a1i)), beta);
      for (int j = lane; j < m; j += 32) {
        const double2 vj = G[(k + 1 + j) * ldg + k];
        V[(k + 1 + j) * ldv + 0] = zsub(V[(k + 1 + j) * ldv + 0], zmul(vj, c0));
        if (nv > 1) V[(k + 1 + j) * ldv + 1] = zsub(V[(k + 1 + j) * ldv + 1], zmul(vj, c1));
      }
      __syncwarp();
    }
    if (lane == 0) {
      G[0] = make_double2(s_d[0], 0.0);
      if (n > 1) G[ldg + 1] = make_double2(s_d[1], 0.0);
      G[(n - 1) * ldg + n - 1] = make_double2(s_d[n - 1], 0.0);
    }
    __syncwarp();
    CBP_PHASE(33, pw);
    return;
  }
  // ---- eigenvectors V = Q D Z: Householders applied in reverse order, lanes on columns
  for (int i = lane; i < n * n; i += 32) {
    const int r = i / n, c = i - r * n;
    V[r * ldv + c] = zscale(s_delta[r], V[r * ldv + c].x);
  }
  __syncwarp();
  for (int k = n - 3; k >= 0; --k) {
    const double beta = s_beta[k];
    if (beta == 0.0) continue;
    const int m = n - k - 1;
    for (int c = lane; c < n; c += 32) {
      double2 acc = make_double2(0.0, 0.0);
      for (int j = 0; j < m; ++j) acc = zadd(acc, zcmul(G[(k + 1 + j) * ldg + k], V[(k + 1 + j) * ldv + c]));
      acc = zscale(acc, beta);
      for (int j = 0; j < m; ++j)
        V[(k + 1 + j) * ldv + c] = zsub(V[(k + 1 + j) * ldv + c], zmul(G[(k + 1 + j) * ldg + k], acc));
    }
    __syncwarp();
  }
  for (int k = lane; k < n; k += 32) G[k * ldg + k] = make_double2(s_d[k], 0.0);
  __syncwarp();
  CBP_PHASE(33, pw);
}

// Cholesky A = L L^H of a Hermitian positive definite n x n matrix (lower triangle, row-major,
// stride n), in place, by one warp (lanes on rows). id[k] = 1 / L_kk. A pivot that rounding
// drove to <= 0 is floored (the factor then amplifies that direction, which inverse
// iteration tolerates).
__device__ __forceinline__ void warp_cholesky(double2* L, int n, double* id) {
  const int lane = threadIdx.x & 31;
  for (int k = 0; k < n; ++k) {
    const double piv = fmax(L[k * n + k].x, 1e-300);
    const double inv = rsqrt(piv);
    __syncwarp();
    for (int i = k + 1 + lane; i < n; i += 32) L[i * n + k] = zscale(L[i * n + k], inv);
    if (lane == 0) {
      L[k * n + k] = make_double2(piv * inv, 0.0);
      id[k] = inv;
    }
    __syncwarp();
    for (int i = k + 1 + lane; i < n; i += 32) {
      const double2 lik = L[i * n + k];
      for (int j = k + 1; j <= i; ++j) L[i * n + j] = zsub(L[i * n + j], zmul(lik, zconj(L[j * n + k])));
    }
    __syncwarp();
  }
}

// w <- A^-1 w with the factor from warp_cholesky, one warp (w in shared or global memory).
__device__ __forceinline__ void warp_chol_solve(const double2* L, const double* id, int n, double2* w) {
  const int lane = threadIdx.x & 31;
  for (int k = 0; k < n; ++k) {  // L z = w
    const double2 zk = zscale(w[k], id[k]);
    __syncwarp();
    for (int i = k + 1 + lane; i < n; i += 32) w[i] = zsub(w[i], zmul(L[i * n + k], zk));
    if (lane == 0) w[k] = zk;
    __syncwarp();
  }
  for (int k = n - 1; k >= 0; --k) {  // L^H y = z
    const double2 yk = zscale(w[k], id[k]);
    __syncwarp();
    for (int i = lane; i < k; i += 32) w[i] = zsub(w[i], zcmul(L[k * n + i], yk));
    if (lane == 0) w[k] = yk;
    __syncwarp();
  }
}

// eigenvalues only (G's diagonal), whole CTA
template <int NMAX = 64>
__device__ __forceinline__ void herm_eigvals_cta(double2* G, int ldg, double2* V, int ldv, int n) {
  if (threadIdx.x < 32) herm_eig_warp<NMAX>(G, ldg, V, ldv, n, EIG_VALUES);
  __syncthreads();
}

// whole-CTA entry: the tridiagonal route on warp 0 (the Jacobi solver above is kept as
// the reference implementation, selectable with -DCBP_JACOBI)
template <int NMAX = 64>
__device__ __forceinline__ void herm_jacobi_cta(double2* G, int ldg, double2* V, int ldv, int n, JacobiScratch sc,
                                                int mode = EIG_QL) {
#ifdef CBP_JACOBI
  if (sc.cs) {
    herm_jacobi(G, ldg, V, ldv, n, sc);
    return;
  }
#endif
  (void)sc;
  if (threadIdx.x < 32) herm_eig_warp<NMAX>(G, ldg, V, ldv, n, mode);
  __syncthreads();
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
static __device__ void onesided_sv(double2* A, int lda, int n, double* sv, int* flag, int max_sweeps = 60) {
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
