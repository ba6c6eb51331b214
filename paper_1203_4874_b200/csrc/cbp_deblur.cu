// Regularised frequency-domain deconvolution (reference decoder.cpp:184-214,
// make_deblur_plan + run_deblur; fft.cpp:242-270 r2c/c2r):
//
//   latent = crop_{(Mb-t+1) x (Nb-t+1)} IFFT2( FFT2(pad(B1)) * conj(K) / (|K|^2 + eps) )
//
// on the Gr x Gc = friendly_size(Mb) x friendly_size(Nb) grid. Three passes per plane:
//   A  row r2c (half-length complex FFT + split), rows < Mb only      HBM in  -> L2 X
//   B  column FFT, Wiener filter with K computed on the fly from the
//      t x t weights (no Gr x Gc kernel spectrum is ever stored),
//      inverse column FFT, rows < Mb-t+1 kept                           L2 X -> L2 X
//   C  row c2r, 1/(Gr*Gc) folded into the filter, crop                 L2 X -> HBM out
// The row-major grid halves the column axis where column-major FFTW halves rows
// (fft.cpp:45); the arithmetic is the same transform.
#include <cstdlib>

#include "cbp_deblur.cuh"
#include "cbp_fft.cuh"

namespace cbp_dev {

// ---------------------------------------------------------------- pass A
// grid (ceil(Mb / rows_per_cta), planes); smem 2 * rows_per_cta * L float2.
__global__ void __launch_bounds__(256) k_rows_forward(DeblurArgs a) {
  extern __shared__ float2 smem[];
  const int rpc = a.rows_per_cta;
  const int L = a.even ? a.Gc / 2 : a.Gc;  // complex transform length
  const int lp = L;                          // smem row pitch
  float2* buf0 = smem;
  float2* buf1 = smem + size_t(rpc) * lp;
  const int p = blockIdx.y;
  const int r0 = blockIdx.x * rpc;
  const int nrows = min(rpc, a.Mb - r0);
  const float* src = a.in + size_t(p) * a.in_plane + size_t(r0) * a.in_ld;

  // load (zero padded to the grid)
  for (int idx = threadIdx.x; idx < rpc * L; idx += blockDim.x) {
    const int s = idx / L, k = idx - s * L;
    float2 z = make_float2(0.f, 0.f);
    if (s < nrows) {
      const float* row = src + size_t(s) * a.in_ld;
      if (a.even) {
        const int n0 = 2 * k;
        if (n0 < a.Nb) z.x = __ldcs(row + n0);
        if (n0 + 1 < a.Nb) z.y = __ldcs(row + n0 + 1);
      } else if (k < a.Nb) {
        z.x = __ldcs(row + k);
      }
    }
    buf0[s * lp + k] = z;
  }
  __syncthreads();
  float2* res = fft_run<false, false>(buf0, buf1, a.plan_row, rpc, lp, 1, a.tw_row);
  // split into the half spectrum X[0..Gc/2] (fft.cpp:242-255 r2c)
  const int H = a.Hc;
  for (int idx = threadIdx.x; idx < nrows * H; idx += blockDim.x) {
    const int k = idx / nrows, s = idx - k * nrows;  // rows fastest: XT[k][r0 + s]
    float2 x;
    if (a.even) {
      const float2 zk = res[s * lp + (k == L ? 0 : k)];
      const float2 zc = cconj(res[s * lp + (k == 0 ? 0 : L - k)]);
      const float2 e = cscale(cadd(zk, zc), 0.5f);
      const float2 d = csub(zk, zc);
      const float2 o = make_float2(0.5f * d.y, -0.5f * d.x);  // -i/2 * d
      x = cadd(e, cmul(__ldg(&a.tw_post[k]), o));
    } else {
      x = res[s * lp + k];
    }
    a.X[size_t(p) * a.x_plane + size_t(k) * a.xp + r0 + s] = x;
  }
}

// ---------------------------------------------------------------- pass B
// grid (ceil(Hc / W), planes); smem 2 * Gr * W float2 + W * t float2.
template <int W>
__global__ void __launch_bounds__(256) k_cols_filter(DeblurArgs a) {
  extern __shared__ float2 smem[];
  const int p = blockIdx.y;
  const cbp_kernel_slot* slot = a.slot + deblur_slot_index(a, p);
  if (slot->status != 0) return;
  const int t = slot->width;
  const int M = a.Mb - t + 1;
  const int Gr = a.Gr;
  const int v0 = blockIdx.x * W;
  float2* buf0 = smem;
  float2* buf1 = smem + size_t(Gr) * W;
  float2* S = smem + size_t(2) * Gr * W;  // S[s*t + a] = sum_b w[a][b] exp(-2 pi i v b / Gc)
  float2* X = a.X + size_t(p) * a.x_plane;

  for (int idx = threadIdx.x; idx < W * t; idx += blockDim.x) {
    const int s = idx / t, ai = idx - s * t;
    const int v = v0 + s;
    double re = 0.0, im = 0.0;
    for (int bj = 0; bj < t; ++bj) {
      const double w = slot->weights[ai * t + bj];
      double sn, cs;
      sincospi(-2.0 * double((long(v) * bj) % a.Gc) / double(a.Gc), &sn, &cs);
      re = fma(w, cs, re);
      im = fma(w, sn, im);
    }
    S[idx] = make_float2(float(re), float(im));
  }
  for (int idx = threadIdx.x; idx < Gr * W; idx += blockDim.x) {
    const int s = idx / Gr, u = idx - s * Gr;  // column v = v0 + s is contiguous in XT
    const int v = v0 + s;
    float2 x = make_float2(0.f, 0.f);
    if (u < a.Mb && v < a.Hc) x = X[size_t(v) * a.xp + u];
    buf0[u * W + s] = x;
  }
  __syncthreads();
  float2* res = fft_run<false, true>(buf0, buf1, a.plan_col, W, 1, W, a.tw_col);
  float2* other = res == buf0 ? buf1 : buf0;
  // Wiener filter: conj(K)/(|K|^2+eps) * 1/(Gr*Gc)  (decoder.cpp:209-211, fft.cpp:268)
  const float eps = float(slot->epsilon);
  const float scale = float(1.0 / (double(Gr) * double(a.Gc)));
  for (int idx = threadIdx.x; idx < Gr * W; idx += blockDim.x) {
    const int u = idx / W, s = idx - u * W;
    const float2* Ss = S + s * t;
    float2 k = make_float2(0.f, 0.f);
    int ti = 0;
    for (int ai = 0; ai < t; ++ai) {
      const float2 w = __ldg(&a.tw_col[ti]), sv = Ss[ai];
      k.x = fmaf(sv.x, w.x, fmaf(-sv.y, w.y, k.x));
      k.y = fmaf(sv.x, w.y, fmaf(sv.y, w.x, k.y));
      ti += u;
      if (ti >= Gr) ti -= Gr;
    }
    const float den = fmaf(k.x, k.x, fmaf(k.y, k.y, eps));
    const float f = scale / den;
    const float2 h = make_float2(k.x * f, -k.y * f);
    res[idx] = cmul(res[idx], h);
  }
  __syncthreads();
  res = fft_run<true, true>(res, other, a.plan_col, W, 1, W, a.tw_col);
  for (int idx = threadIdx.x; idx < M * W; idx += blockDim.x) {
    const int s = idx / M, u = idx - s * M;
    const int v = v0 + s;
    if (v < a.Hc) X[size_t(v) * a.xp + u] = res[u * W + s];
  }
}

// ---------------------------------------------------------------- pass C
// grid (ceil(Mb / rows_per_cta), planes); rows >= Mb-t+1 exit.
__global__ void __launch_bounds__(256) k_rows_inverse(DeblurArgs a) {
  extern __shared__ float2 smem[];
  const int p = blockIdx.y;
  const cbp_kernel_slot* slot = a.slot + deblur_slot_index(a, p);
  if (slot->status != 0) return;
  const int t = slot->width;
  const int M = a.Mb - t + 1, N = a.Nb - t + 1;
  const int rpc = a.rows_per_cta;
  const int r0 = blockIdx.x * rpc;
  if (r0 >= M) return;
  const int nrows = min(rpc, M - r0);
  const int L = a.even ? a.Gc / 2 : a.Gc;
  const int lp = L;
  float2* buf0 = smem;
  float2* buf1 = smem + size_t(rpc) * lp;
  const float2* Y = a.X + size_t(p) * a.x_plane + r0;  // XT[k][r0 + s]
  for (int idx = threadIdx.x; idx < rpc * L; idx += blockDim.x) {
    const int s = idx / L, k = idx - s * L;
    float2 z = make_float2(0.f, 0.f);
    if (s < nrows) {
      const float2* row = Y + s;  // element k of row r0+s at row[k * xp]
      if (a.even) {  // inverse split (fft.cpp:257-270 c2r)
        const float2 A = row[size_t(k) * a.xp];
        const float2 B = cconj(row[size_t(L - k) * a.xp]);
        const float2 e = cadd(A, B);
        const float2 o = cmul(csub(A, B), cconj(__ldg(&a.tw_post[k])));
        z = make_float2(e.x - o.y, e.y + o.x);  // e + i*o
      } else {
        z = k <= L / 2 ? row[size_t(k) * a.xp] : cconj(row[size_t(L - k) * a.xp]);
      }
    }
    buf0[s * lp + k] = z;
  }
  __syncthreads();
  float2* res = fft_run<true, false>(buf0, buf1, a.plan_row, rpc, lp, 1, a.tw_row);
  float* dst = a.out + size_t(p) * a.out_plane + size_t(r0) * a.out_ld;
  for (int idx = threadIdx.x; idx < nrows * N; idx += blockDim.x) {
    const int s = idx / N, n = idx - s * N;
    float x;
    if (a.even) {
      const float2 z = res[s * lp + (n >> 1)];
      x = (n & 1) ? z.y : z.x;
    } else {
      x = res[s * lp + n].x;
    }
    __stcs(dst + size_t(s) * a.out_ld + n, x);
  }
}

// ------------------------------------------------------------------ host side
static size_t smem_rows(const DeblurArgs& a) {
  const int L = a.even ? a.Gc / 2 : a.Gc;
  return size_t(2) * a.rows_per_cta * L * sizeof(float2);
}

int deblur_col_width(int Gr, int t_max) {
  // largest W with 2*Gr*W*8 + W*t*8 <= ~112 KB (two CTAs per SM)
  for (int W : {8, 4, 2, 1})
    if ((size_t(2) * Gr * W + size_t(W) * t_max) * sizeof(float2) <= 112 * 1024) return W;
  return 1;
}

static size_t smem_cols(const DeblurArgs& a, int W) {
  return (size_t(2) * a.Gr * W + size_t(W) * CBP_MAX_WIDTH) * sizeof(float2);
}

cudaError_t launch_deblur_pass(const DeblurArgs& a, int planes, int pass, cudaStream_t stream) {
  static const bool force_generic = getenv("CBP_GENERIC_FFT") != nullptr;
  if (!force_generic && launch_deblur_pass_ct(a, planes, pass, stream)) return cudaGetLastError();
  CBP_ONCE_PER_DEVICE({
    cudaFuncSetAttribute(k_rows_forward, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_rows_inverse, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_cols_filter<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    cudaFuncSetAttribute(k_cols_filter<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    cudaFuncSetAttribute(k_cols_filter<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    cudaFuncSetAttribute(k_cols_filter<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  });
  dim3 ga((a.Mb + a.rows_per_cta - 1) / a.rows_per_cta, planes);
  if (pass == 0) {
    k_rows_forward<<<ga, 256, smem_rows(a), stream>>>(a);
  } else if (pass == 1) {
    const int W = a.col_width;
    dim3 gb((a.Hc + W - 1) / W, planes);
    switch (W) {
      case 8: k_cols_filter<8><<<gb, 256, smem_cols(a, 8), stream>>>(a); break;
      case 4: k_cols_filter<4><<<gb, 256, smem_cols(a, 4), stream>>>(a); break;
      case 2: k_cols_filter<2><<<gb, 256, smem_cols(a, 2), stream>>>(a); break;
      default: k_cols_filter<1><<<gb, 256, smem_cols(a, 1), stream>>>(a); break;
    }
  } else {
    k_rows_inverse<<<ga, 256, smem_rows(a), stream>>>(a);
  }
  return cudaGetLastError();
}

}  // namespace cbp_dev
