// Times herm_eig_warp (cbp_linalg.cuh) on a rank-deficient 22x22 complex Gram (the k_solve
// shape) and checks the residual |G V - V diag(d)| (profiling aid). Build:
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -DCBP_PHASES -I../../paper_1203_4874_b200/csrc
//        -I../../include bench_eig.cu -o bench_eig
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>
#include "cbp_linalg.cuh"
namespace cbp_dev {
__device__ unsigned long long g_phase[64];
}
using namespace cbp_dev;
__global__ void keig(const double2* G0, double2* Gout, double2* V, int n, unsigned long long* t) {
  __shared__ double2 G[32 * 32], Vs[32 * 32];
  for (int i = threadIdx.x; i < n * n; i += blockDim.x) G[i] = G0[i];
  __syncthreads();
  unsigned long long t0 = clock64();
  herm_jacobi_cta(G, n, Vs, n, n, JacobiScratch{}, EIG_MODE);
  unsigned long long t1 = clock64();
  for (int i = threadIdx.x; i < n * n; i += blockDim.x) Gout[i] = G[i], V[i] = Vs[i];
  if (threadIdx.x == 0) t[0] = t1 - t0;
}
int main() {
  for (int n : {22, 25, 20}) {
    std::mt19937_64 rng(1);
    std::normal_distribution<double> N;
    const int R = 1940;
    std::vector<double> Ar(R * n), Ai(R * n);
    for (auto& v : Ar) v = N(rng);
    for (auto& v : Ai) v = n == 25 ? 0.0 : N(rng);
    // rank deficiency: remove the component along a random unit x
    std::vector<double> xr(n), xi(n);
    double nx = 0;
    for (int j = 0; j < n; ++j) xr[j] = N(rng), xi[j] = n == 25 ? 0.0 : N(rng), nx += xr[j] * xr[j] + xi[j] * xi[j];
    nx = std::sqrt(nx);
    for (int j = 0; j < n; ++j) xr[j] /= nx, xi[j] /= nx;
    for (int r = 0; r < R; ++r) {
      double sr = 0, si = 0;  // (A x)_r
      for (int j = 0; j < n; ++j) {
        sr += Ar[r * n + j] * xr[j] - Ai[r * n + j] * xi[j];
        si += Ar[r * n + j] * xi[j] + Ai[r * n + j] * xr[j];
      }
      for (int j = 0; j < n; ++j) {  // A -= (A x) x^H
        Ar[r * n + j] -= sr * xr[j] + si * xi[j];
        Ai[r * n + j] -= si * xr[j] - sr * xi[j];
      }
    }
    std::vector<double2> G(n * n);
    if (n == 20) {  // clustered spectrum: U diag(l) U^H, l with exact and near duplicates
      std::vector<double> Ur(n * n), Ui(n * n);
      for (auto& v : Ur) v = N(rng);
      for (auto& v : Ui) v = N(rng);
      for (int c = 0; c < n; ++c) {  // Gram-Schmidt on columns
        for (int j = 0; j < c; ++j) {
          double dr = 0, di = 0;
          for (int r = 0; r < n; ++r) {
            dr += Ur[r * n + j] * Ur[r * n + c] + Ui[r * n + j] * Ui[r * n + c];
            di += Ur[r * n + j] * Ui[r * n + c] - Ui[r * n + j] * Ur[r * n + c];
          }
          for (int r = 0; r < n; ++r) {
            Ur[r * n + c] -= dr * Ur[r * n + j] - di * Ui[r * n + j];
            Ui[r * n + c] -= dr * Ui[r * n + j] + di * Ur[r * n + j];
          }
        }
        double nn = 0;
        for (int r = 0; r < n; ++r) nn += Ur[r * n + c] * Ur[r * n + c] + Ui[r * n + c] * Ui[r * n + c];
        nn = std::sqrt(nn);
        for (int r = 0; r < n; ++r) Ur[r * n + c] /= nn, Ui[r * n + c] /= nn;
      }
      double l[20] = {0, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1 + 1e-9, 1 + 2e-9, 2, 2, 2, 3, 3 + 1e-7, 5, 5, 7};
      for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
          double gr = 0, gi = 0;
          for (int k = 0; k < n; ++k) {  // U_ik l_k conj(U_jk)
            gr += l[k] * (Ur[i * n + k] * Ur[j * n + k] + Ui[i * n + k] * Ui[j * n + k]);
            gi += l[k] * (Ui[i * n + k] * Ur[j * n + k] - Ur[i * n + k] * Ui[j * n + k]);
          }
          G[i * n + j] = make_double2(gr, gi);
        }
    } else
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        double gr = 0, gi = 0;  // sum conj(A_ri) A_rj
        for (int r = 0; r < R; ++r) {
          gr += Ar[r * n + i] * Ar[r * n + j] + Ai[r * n + i] * Ai[r * n + j];
          gi += Ar[r * n + i] * Ai[r * n + j] - Ai[r * n + i] * Ar[r * n + j];
        }
        G[i * n + j] = make_double2(gr, gi);
      }
    double2 *dG, *dGo, *dV;
    unsigned long long* dt;
    cudaMalloc(&dG, 16 * n * n); cudaMalloc(&dGo, 16 * n * n); cudaMalloc(&dV, 16 * n * n); cudaMalloc(&dt, 8);
    cudaMemcpy(dG, G.data(), 16 * n * n, cudaMemcpyHostToDevice);
    for (int rep = 0; rep < 3; ++rep) keig<<<1, 32>>>(dG, dGo, dV, n, dt);
    cudaDeviceSynchronize();
    unsigned long long cyc, ph[64];
    cudaMemcpy(&cyc, dt, 8, cudaMemcpyDeviceToHost);
    cudaMemcpyFromSymbol(ph, g_phase, sizeof(ph));
    std::vector<double2> Go(n * n), V(n * n);
    cudaMemcpy(Go.data(), dGo, 16 * n * n, cudaMemcpyDeviceToHost);
    cudaMemcpy(V.data(), dV, 16 * n * n, cudaMemcpyDeviceToHost);
    double res = 0, nrm = 0, lmin = 1e300;
    for (int i = 0; i < n; ++i) {
      for (int c = 0; c < n; ++c) {
        double pr = 0, pi = 0;
        for (int k = 0; k < n; ++k) {
          pr += G[i * n + k].x * V[k * n + c].x - G[i * n + k].y * V[k * n + c].y;
          pi += G[i * n + k].x * V[k * n + c].y + G[i * n + k].y * V[k * n + c].x;
        }
        const double l = Go[c * n + c].x;
        pr -= l * V[i * n + c].x, pi -= l * V[i * n + c].y;
        res += pr * pr + pi * pi;
        nrm += G[i * n + c].x * G[i * n + c].x + G[i * n + c].y * G[i * n + c].y;
      }
      lmin = std::fmin(lmin, std::fabs(Go[i * n + i].x));
    }
    double orth = 0;
    for (int a = 0; a < n; ++a)
      for (int b = 0; b < n; ++b) {
        double dr = 0, di = 0;
        for (int r = 0; r < n; ++r) {
          dr += V[r * n + a].x * V[r * n + b].x + V[r * n + a].y * V[r * n + b].y;
          di += V[r * n + a].x * V[r * n + b].y - V[r * n + a].y * V[r * n + b].x;
        }
        if (a == b) dr -= 1;
        orth = std::fmax(orth, std::sqrt(dr * dr + di * di));
      }
    printf("  orthogonality max |V^H V - I| = %.2e\n", orth);
    printf("n=%d: %llu cycles (%.1f us at 1.965 GHz); tridiag %.1f us, bisect+invit %.1f, mgs %.1f, (unused %.1f), back %.1f us; rel resid %.2e, min|l| %.3e\n",
           n, cyc, cyc / 1965.0, (ph[31] - ph[30]) / 1e3, (ph[34] - ph[31]) / 1e3, (ph[35] - ph[34]) / 1e3,
           (ph[32] - ph[35]) / 1e3, (ph[33] - ph[32]) / 1e3,
           std::sqrt(res / nrm), lmin);
  }
  return 0;
}
