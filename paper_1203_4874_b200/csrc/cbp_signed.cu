// Width estimation for signed content (reference decoder.cpp:65-82, fft.cpp:217-240).
//
// When a luma has a negative sample the DC sums are not the maximum-energy slices, so the
// reference takes axis_spectrum_half of both lumas (an r2c DFT of every column for z1,
// of every row for z2, at the exact frame length, which is not 2/3/5/7-smooth in general:
// 1090 = 2*5*109), picks the frequency with the largest joint energy (first maximum) and
// runs the Bezout width search on that complex slice pair.
//
// Device version, in FP64: the energies come from a tiled DFT-as-matrix-product over the
// frame (twiddles from an exact table, luma computed in the loads), reduced in a fixed
// order; only the picked frequency's slices are then formed, written over the DC slices
// so k_width_blocks / k_width_pick run unchanged (complex blocks take the Jacobi SVD path).
// Frames without a negative sample exit at the first instruction.
#include <algorithm>

#include "cbp_recover.cuh"

namespace cbp_dev {

namespace {

constexpr int TS = 32;  // output tile edge; 256 threads, 4 outputs each

__device__ __forceinline__ bool signed_frame(const RecoverArgs& a, int b) {
  const cbp_kernel_slot* slot = a.slots + b;
  return slot->status == 0 && slot->width == 0 && (a.flags[b] & 1);
}

__device__ __forceinline__ const float* stream_base(const RecoverArgs& a, int b, int q) {
  return (q ? a.prv : a.pub) + size_t(b) * a.channels * size_t(a.rows) * a.ld;
}

}  // namespace

// roots[k] = exp(-2 pi i k / rows) for k < rows, then exp(-2 pi i k / cols) for k < cols
__global__ void k_spec_roots(RecoverArgs a) {
  pdl_enter();
  bool any = false;  // nothing to do for a batch of nonnegative frames (the common case)
  for (int b = 0; b < a.batch && !any; ++b) any = signed_frame(a, b);
  if (!any) return;
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < a.rows) a.roots[k] = zroot(k, a.rows);
  if (k < a.cols) a.roots[a.rows + k] = zroot(k, a.cols);
}

// z1: F_q(i, n) = sum_m W_M^{i m} luma_q(m, n), i <= M/2. Per tile: partial energies
// sum_n |F|^2 for the tile's 32 frequencies. grid (ceil(N/32), ceil(H1/32), batch*2).
__device__ __forceinline__ bool any_signed(const RecoverArgs& a) {
  for (int b = 0; b < a.batch; ++b)
    if (signed_frame(a, b)) return true;
  return false;
}

// Persistent grid over tiles (x fastest, then y, then frame*2+stream): a batch without
// signed frames costs one flag scan per CTA instead of ~10^4 empty CTAs.
__global__ void __launch_bounds__(256) k_spec_energy_z1(RecoverArgs a) {
  pdl_enter();
  if (!any_signed(a)) return;
  const int M = a.rows, N = a.cols, H1 = M / 2 + 1;
  const int tx = (N + TS - 1) / TS, ty = (H1 + TS - 1) / TS;
  for (int tile = blockIdx.x; tile < tx * ty * a.batch * 2; tile += gridDim.x) {
  const int bz = tile / (tx * ty), rem = tile - bz * (tx * ty);
  const int by = rem / tx, bx = rem - by * tx;
  const int b = bz >> 1, q = bz & 1;
  if (!signed_frame(a, b)) continue;
  __shared__ double Ls[TS][TS + 1];
  __shared__ double2 Ws[TS][TS + 1];
  const int n0 = bx * TS, i0 = by * TS;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t plane = size_t(M) * a.ld;
  const float* base = stream_base(a, b, q);
  const double2* root = a.roots;
  double2 acc[4] = {};
  for (int m0 = 0; m0 < M; m0 += TS) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int r = w + 8 * k;
      const int m = m0 + r, n = n0 + lane, i = i0 + r, mm = m0 + lane;
      Ls[r][lane] = (m < M && n < N) ? luma_at(base, plane, a.channels, size_t(m) * a.ld + n) : 0.0;
      Ws[r][lane] = (i < H1 && mm < M) ? root[(long(i) * mm) % M] : make_double2(0.0, 0.0);
    }
    __syncthreads();
#pragma unroll 8
    for (int mm = 0; mm < TS; ++mm) {
      const double x = Ls[mm][lane];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const double2 wv = Ws[w + 8 * k][mm];
        acc[k].x = fma(wv.x, x, acc[k].x);
        acc[k].y = fma(wv.y, x, acc[k].y);
      }
    }
    __syncthreads();
  }
  const int ntn = (N + TS - 1) / TS;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int i = i0 + w + 8 * k;
    double e = zabs2(acc[k]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
    if (lane == 0 && i < H1) a.epart[((size_t(b) * 2 + q) * ntn + bx) * H1 + i] = e;
  }
  }
}

// z2: F_q(m, j) = sum_n luma_q(m, n) W_N^{j n}, j <= N/2. Per tile: partial energies
// sum_m |F|^2 for the tile's 32 frequencies. grid (ceil(H2/32), ceil(M/32), batch*2).
__global__ void __launch_bounds__(256) k_spec_energy_z2(RecoverArgs a) {
  pdl_enter();
  if (!any_signed(a)) return;
  const int M = a.rows, N = a.cols, H2 = N / 2 + 1;
  const int tx = (H2 + TS - 1) / TS, ty = (M + TS - 1) / TS;
  for (int tile = blockIdx.x; tile < tx * ty * a.batch * 2; tile += gridDim.x) {
  const int bz = tile / (tx * ty), rem = tile - bz * (tx * ty);
  const int by = rem / tx, bx = rem - by * tx;
  const int b = bz >> 1, q = bz & 1;
  if (!signed_frame(a, b)) continue;
  __shared__ double Ls[TS][TS + 1];
  __shared__ double2 Ws[TS][TS + 1];
  __shared__ double Es[8][TS];
  const int j0 = bx * TS, m0 = by * TS;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t plane = size_t(M) * a.ld;
  const float* base = stream_base(a, b, q);
  const double2* root = a.roots + M;
  double2 acc[4] = {};
  for (int nb = 0; nb < N; nb += TS) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int r = w + 8 * k;
      const int m = m0 + r, n = nb + lane, nn = nb + r, j = j0 + lane;
      Ls[r][lane] = (m < M && n < N) ? luma_at(base, plane, a.channels, size_t(m) * a.ld + n) : 0.0;
      Ws[r][lane] = (j < H2 && nn < N) ? root[(long(j) * nn) % N] : make_double2(0.0, 0.0);
    }
    __syncthreads();
#pragma unroll 8
    for (int nn = 0; nn < TS; ++nn) {
      const double2 wv = Ws[nn][lane];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const double x = Ls[w + 8 * k][nn];
        acc[k].x = fma(wv.x, x, acc[k].x);
        acc[k].y = fma(wv.y, x, acc[k].y);
      }
    }
    __syncthreads();
  }
  Es[w][lane] = zabs2(acc[0]) + zabs2(acc[1]) + zabs2(acc[2]) + zabs2(acc[3]);
  __syncthreads();
  const int ntm = (M + TS - 1) / TS;
  if (w == 0 && j0 + lane < H2) {
    double e = 0.0;
    for (int ww = 0; ww < 8; ++ww) e += Es[ww][lane];
    a.epart[((size_t(b) * 2 + q) * ntm + by) * H2 + j0 + lane] = e;
  }
  __syncthreads();  // Es is rewritten by the next tile
  }
}

// Per (frame, axis): joint energies in a fixed order, first maximum (Eigen maxCoeff),
// then the picked slice of both lumas into slices[b][axis][q][0][*]. grid (batch, 2).
__global__ void __launch_bounds__(512) k_spec_pick(RecoverArgs a) {
  pdl_enter();
  const int b = blockIdx.x, axis = blockIdx.y;
  if (!signed_frame(a, b)) return;
  const int M = a.rows, N = a.cols;
  const int H = axis == 0 ? M / 2 + 1 : N / 2 + 1;
  const int nt = axis == 0 ? (N + TS - 1) / TS : (M + TS - 1) / TS;
  const double* ep = a.epart + (axis == 0 ? 0 : a.epart_z2);
  __shared__ double bv[512];
  __shared__ int bi[512];
  double best = -1.0;
  int pick = 0;
  for (int i = threadIdx.x; i < H; i += blockDim.x) {
    double e = 0.0;
    for (int q = 0; q < 2; ++q)
      for (int tl = 0; tl < nt; ++tl) e += ep[((size_t(b) * 2 + q) * nt + tl) * H + i];
    if (e > best) best = e, pick = i;  // i ascends per thread: keeps the first maximum
  }
  bv[threadIdx.x] = best;
  bi[threadIdx.x] = pick;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      const double o = bv[threadIdx.x + s];
      const int oi = bi[threadIdx.x + s];
      if (o > bv[threadIdx.x] || (o == bv[threadIdx.x] && oi < bi[threadIdx.x])) {
        bv[threadIdx.x] = o;
        bi[threadIdx.x] = oi;
      }
    }
    __syncthreads();
  }
  pick = bi[0];
  const size_t plane = size_t(M) * a.ld;
  for (int q = 0; q < 2; ++q) {
    const float* base = stream_base(a, b, q);
    double2* out = a.slices + slice_offset(a, b, axis, q, 0);
    if (axis == 0) {  // p[n] = sum_m W_M^{pick m} luma(m, n)
      for (int n = threadIdx.x; n < N; n += blockDim.x) {
        double re = 0.0, im = 0.0;
        int idx = 0;
        for (int m = 0; m < M; ++m) {
          const double x = luma_at(base, plane, a.channels, size_t(m) * a.ld + n);
          re = fma(a.roots[idx].x, x, re);
          im = fma(a.roots[idx].y, x, im);
          idx += pick;
          if (idx >= M) idx -= M;
        }
        out[n] = make_double2(re, im);
      }
    } else {  // p[m] = sum_n luma(m, n) W_N^{pick n}
      const double2* rootN = a.roots + M;
      for (int m = threadIdx.x; m < M; m += blockDim.x) {
        double re = 0.0, im = 0.0;
        int idx = 0;
        for (int n = 0; n < N; ++n) {
          const double x = luma_at(base, plane, a.channels, size_t(m) * a.ld + n);
          re = fma(rootN[idx].x, x, re);
          im = fma(rootN[idx].y, x, im);
          idx += pick;
          if (idx >= N) idx -= N;
        }
        out[m] = make_double2(re, im);
      }
    }
  }
}

size_t signed_energy_doubles(int batch, int rows, int cols) {
  const size_t z1 = size_t(batch) * 2 * ((cols + TS - 1) / TS) * (rows / 2 + 1);
  const size_t z2 = size_t(batch) * 2 * ((rows + TS - 1) / TS) * (cols / 2 + 1);
  return z1 + z2;
}

cudaError_t launch_signed_slices(const RecoverArgs& a, cudaStream_t s) {
  const int M = a.rows, N = a.cols;
  launch_chain(k_spec_roots, a.chain != 0, dim3((std::max(M, N) + 255) / 256), dim3(256), 0, s, a);
  const int t1 = ((N + TS - 1) / TS) * ((M / 2 + 1 + TS - 1) / TS) * a.batch * 2;
  const int t2 = ((N / 2 + 1 + TS - 1) / TS) * ((M + TS - 1) / TS) * a.batch * 2;
  launch_chain(k_spec_energy_z1, a.chain != 0, dim3(std::min(t1, 148 * 4)), dim3(256), 0, s, a);
  launch_chain(k_spec_energy_z2, a.chain != 0, dim3(std::min(t2, 148 * 4)), dim3(256), 0, s, a);
  launch_chain(k_spec_pick, a.chain != 0, dim3(a.batch, 2), dim3(512), 0, s, a);
  return cudaGetLastError();
}

}  // namespace cbp_dev
