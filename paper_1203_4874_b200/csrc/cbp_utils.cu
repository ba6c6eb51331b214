// C ABI: the polynomial and transform utilities of the reference's public headers that the
// decode path uses internally (poly.hpp:30-55, fft.hpp:9-13), as stand-alone device calls:
//   cbp_bezout_leading_block   bezout_leading_block (poly.cpp:66-79)
//   cbp_numerical_singularity  numerical_singularity (poly.cpp:81-91)
//   cbp_homogeneous_lsq        homogeneous_lsq (poly.cpp:123-130)
//   cbp_fft2                   fft2 / ifft2 (fft.cpp:170-195), FP64 complex, any size
// Complex arrays are interleaved (re, im) FP64 in host memory, matrices row-major. The calls
// stage their operands through context workspaces and synchronize the stream. None of them
// is on the hot path (decode_frame runs the fused versions inside its kernels); they exist
// so reference callers of these functions link against the B200 build unchanged.
#include <cmath>
#include <cstring>
#include <vector>

#include "cbp_ctx.cuh"
#include "cbp_linalg.cuh"

using namespace cbp_dev;
using namespace cbp_host;

namespace {

// B[i][j] = sum_{k=0}^{min(i,j)} p[i+j+1-k] q[k] - q[i+j+1-k] p[k] (poly.cpp:72-77)
__global__ void k_bezout(const double2* p, int lp, const double2* q, int lq, int size, double2* out) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= size * size) return;
  const int i = idx / size, j = idx - i * size;
  double2 s = make_double2(0.0, 0.0);
  for (int k = 0; k <= min(i, j); ++k) {
    const int h = i + j + 1 - k;
    const double2 ph = h < lp ? p[h] : make_double2(0.0, 0.0), qk = k < lq ? q[k] : make_double2(0.0, 0.0);
    const double2 qh = h < lq ? q[h] : make_double2(0.0, 0.0), pk = k < lp ? p[k] : make_double2(0.0, 0.0);
    s = zadd(s, zsub(zmul(ph, qk), zmul(qh, pk)));
  }
  out[idx] = s;
}

// One-sided (Hestenes) Jacobi SVD of A (rows x n, column-major: column c at A + c*rows, in
// global memory), rows >= n, with the right singular vectors accumulated in V (n x n,
// column-major). Column norms of the rotated A are the singular values (Eigen's JacobiSVD
// computes the same factorization two-sidedly; both reach high relative accuracy). One CTA.
__global__ void __launch_bounds__(256) k_svd_onesided(double2* A, int rows, int n, double2* V, double* sv) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __shared__ int flag;
  if (V)
    for (int i = threadIdx.x; i < n * n; i += blockDim.x) V[i] = make_double2((i % (n + 1)) == 0 ? 1.0 : 0.0, 0.0);
  const int m = (n + 1) & ~1;
  __syncthreads();
  for (int sweep = 0; sweep < 80; ++sweep) {
    if (threadIdx.x == 0) flag = 0;
    __syncthreads();
    for (int r = 0; r < m - 1; ++r) {
      for (int k = warp; k < m / 2; k += nw) {
        int p, q;
        rr_pair(r, k, m, p, q);
        if (q >= n) continue;
        double2* cp = A + size_t(p) * rows;
        double2* cq = A + size_t(q) * rows;
        double al = 0, be = 0, gr = 0, gi = 0;
        for (int i = lane; i < rows; i += 32) {
          const double2 x = cp[i], y = cq[i];
          al += zabs2(x);
          be += zabs2(y);
          gr += x.x * y.x + x.y * y.y;  // conj(x) y
          gi += x.x * y.y - x.y * y.x;
        }
        al = warp_sum(al);
        be = warp_sum(be);
        gr = warp_sum(gr);
        gi = warp_sum(gi);
        const double ag = hypot(gr, gi);
        if (ag == 0.0 || ag <= 1e-16 * sqrt(al * be)) continue;
        if (lane == 0) flag = 1;
        const double zeta = (be - al) / (2.0 * ag);
        const double tt = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double cs = 1.0 / sqrt(1.0 + tt * tt), sn = cs * tt;
        const double2 ec = make_double2(gr / ag, -gi / ag);  // conj(gamma / |gamma|)
        for (int i = lane; i < rows; i += 32) {
          const double2 x = cp[i], y = zmul(ec, cq[i]);
          cp[i] = make_double2(cs * x.x - sn * y.x, cs * x.y - sn * y.y);
          cq[i] = make_double2(sn * x.x + cs * y.x, sn * x.y + cs * y.y);
        }
        if (V) {
          double2* vp = V + size_t(p) * n;
          double2* vq = V + size_t(q) * n;
          for (int i = lane; i < n; i += 32) {
            const double2 x = vp[i], y = zmul(ec, vq[i]);
            vp[i] = make_double2(cs * x.x - sn * y.x, cs * x.y - sn * y.y);
            vq[i] = make_double2(sn * x.x + cs * y.x, sn * x.y + cs * y.y);
          }
        }
      }
      __syncthreads();
    }
    if (flag == 0) break;
    __syncthreads();
  }
  for (int c = warp; c < n; c += nw) {
    double s = 0;
    for (int i = lane; i < rows; i += 32) s += zabs2(A[size_t(c) * rows + i]);
    s = warp_sum(s);
    if (lane == 0) sv[c] = sqrt(s);
  }
}

// direct DFT along one axis with an exact twiddle table w[k] = exp(-2 pi i k / L):
// out[u][v] (row-major rows x cols) = sum_m in[m][v] w^(u m) (axis 0) or sum_n in[u][n] w^(v n)
__global__ void k_dft_axis(const double2* in, int rows, int cols, int axis, const double2* w, int inverse,
                           double2* out) {
  const size_t idx = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= size_t(rows) * cols) return;
  const int u = int(idx / cols), v = int(idx - size_t(u) * cols);
  const int L = axis == 0 ? rows : cols, f = axis == 0 ? u : v;
  double2 acc = make_double2(0.0, 0.0);
  long e = 0;
  for (int m = 0; m < L; ++m) {
    double2 wk = w[e];
    if (inverse) wk.y = -wk.y;
    const double2 x = axis == 0 ? in[size_t(m) * cols + v] : in[size_t(u) * cols + m];
    acc = zadd(acc, zmul(x, wk));
    e += f;
    if (e >= L) e -= L;
  }
  out[idx] = acc;
}

__global__ void k_roots(double2* w, int L) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < L) w[k] = zroot(k, L);
}

__global__ void k_scale(double2* x, size_t n, double s) {
  const size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) x[i] = zscale(x[i], s);
}

bool all_zero(const double* v, int n) {
  for (int i = 0; i < 2 * n; ++i)
    if (v[i] != 0.0) return false;
  return true;
}

template <class T>
T* ws_of(cbp_ctx* ctx, int id, size_t count) {
  return static_cast<T*>(workspace(ctx, id, count * sizeof(T)));
}

// transposes a row-major complex matrix (host) into column-major device staging
int upload_colmajor(cbp_ctx* ctx, const double* a, int rows, int cols, double2* dev, cudaStream_t s) {
  std::vector<double2> h(size_t(rows) * cols);
  for (int r = 0; r < rows; ++r)
    for (int c = 0; c < cols; ++c) h[size_t(c) * rows + r] = make_double2(a[2 * (size_t(r) * cols + c)], a[2 * (size_t(r) * cols + c) + 1]);
  return cuda_check(ctx, cudaMemcpyAsync(dev, h.data(), h.size() * sizeof(double2), cudaMemcpyHostToDevice, s),
                    "operand upload");
}

}  // namespace

extern "C" {

int cbp_bezout_leading_block(cbp_ctx* ctx, const double* p, int np, const double* q, int nq, int size,
                             double* out, void* stream) {
  cbp_host::DeviceGuard device_guard(ctx);
  cbp_host::StreamOrder stream_order(ctx, stream);
  if (!ctx || !out || np < 0 || nq < 0) return CBP_INVALID_ARGUMENT;
  if (size < 1) return set_error(ctx, CBP_INVALID_ARGUMENT, "bezout block size must be >= 1");
  if (np == 0 || nq == 0 || all_zero(p, np) || all_zero(q, nq))
    return set_error(ctx, CBP_DEGENERATE_INPUT, "bezout of an all-zero polynomial");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  double2* d = ws_of<double2>(ctx, WS_MISC, size_t(np) + nq + size_t(size) * size);
  if (!d) return set_error(ctx, CBP_CUDA_ERROR, "workspace allocation failed");
  cudaMemcpyAsync(d, p, sizeof(double2) * np, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(d + np, q, sizeof(double2) * nq, cudaMemcpyHostToDevice, s);
  double2* o = d + np + nq;
  k_bezout<<<(size * size + 127) / 128, 128, 0, s>>>(d, np, d + np, nq, size, o);
  ++ctx->launches;
  cudaMemcpyAsync(out, o, sizeof(double2) * size * size, cudaMemcpyDeviceToHost, s);
  return cuda_check(ctx, cudaStreamSynchronize(s), "bezout_leading_block");
}

int cbp_numerical_singularity(cbp_ctx* ctx, const double* m, int n, double tau, int* singular, double* ratio,
                              void* stream) {
  cbp_host::DeviceGuard device_guard(ctx);
  cbp_host::StreamOrder stream_order(ctx, stream);
  if (!ctx || !m || !singular || !ratio) return CBP_INVALID_ARGUMENT;
  if (n < 1) return set_error(ctx, CBP_INVALID_ARGUMENT, "singularity test needs a square matrix");
  if (!(tau > 0.0 && tau < 1.0)) return set_error(ctx, CBP_INVALID_ARGUMENT, "tau must lie in (0,1)");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  double2* A = ws_of<double2>(ctx, WS_MISC, size_t(n) * n + n);
  if (!A) return set_error(ctx, CBP_CUDA_ERROR, "workspace allocation failed");
  double* sv = reinterpret_cast<double*>(A + size_t(n) * n);
  int st = upload_colmajor(ctx, m, n, n, A, s);
  if (st) return st;
  k_svd_onesided<<<1, 256, 0, s>>>(A, n, n, nullptr, sv);
  ++ctx->launches;
  std::vector<double> h(n);
  cudaMemcpyAsync(h.data(), sv, sizeof(double) * n, cudaMemcpyDeviceToHost, s);
  if ((st = cuda_check(ctx, cudaStreamSynchronize(s), "numerical_singularity"))) return st;
  double smax = 0.0, smin = INFINITY;
  for (double v : h) smax = std::fmax(smax, v), smin = std::fmin(smin, v);
  if (smax == 0.0) {  // poly.cpp:87
    *singular = 1;
    *ratio = 0.0;
    return 0;
  }
  *ratio = smin / smax;
  *singular = *ratio < tau;
  return 0;
}

int cbp_homogeneous_lsq(cbp_ctx* ctx, const double* a, int rows, int cols, double* x, void* stream) {
  cbp_host::DeviceGuard device_guard(ctx);
  cbp_host::StreamOrder stream_order(ctx, stream);
  if (!ctx || !a || !x) return CBP_INVALID_ARGUMENT;
  if (!(rows >= cols && cols >= 1))
    return set_error(ctx, CBP_INVALID_ARGUMENT, "homogeneous system needs rows >= cols");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  double2* A = ws_of<double2>(ctx, WS_MISC, size_t(rows) * cols + size_t(cols) * cols + cols);
  if (!A) return set_error(ctx, CBP_CUDA_ERROR, "workspace allocation failed");
  double2* V = A + size_t(rows) * cols;
  double* sv = reinterpret_cast<double*>(V + size_t(cols) * cols);
  int st = upload_colmajor(ctx, a, rows, cols, A, s);
  if (st) return st;
  k_svd_onesided<<<1, 256, 0, s>>>(A, rows, cols, V, sv);
  ++ctx->launches;
  std::vector<double> hs(cols);
  std::vector<double2> hv(size_t(cols) * cols);
  cudaMemcpyAsync(hs.data(), sv, sizeof(double) * cols, cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(hv.data(), V, sizeof(double2) * hv.size(), cudaMemcpyDeviceToHost, s);
  if ((st = cuda_check(ctx, cudaStreamSynchronize(s), "homogeneous_lsq"))) return st;
  // the right singular vector of the smallest singular value; ties go to the highest
  // column index, like the last column of Eigen's descending order
  int kmin = 0;
  for (int k = 1; k < cols; ++k)
    if (hs[k] <= hs[kmin]) kmin = k;
  const double2* v = hv.data() + size_t(kmin) * cols;
  // normalize_phase (poly.cpp:18-23): largest |x_i| (first index) real positive
  int im = 0;
  double best = -1.0;
  for (int i = 0; i < cols; ++i) {
    const double mag = std::hypot(v[i].x, v[i].y);
    if (mag > best) best = mag, im = i;
  }
  const double ma = std::hypot(v[im].x, v[im].y);
  double rr = 1.0, ri = 0.0;
  if (ma > 0.0) rr = v[im].x / ma, ri = -v[im].y / ma;
  for (int i = 0; i < cols; ++i) {
    x[2 * i] = v[i].x * rr - v[i].y * ri;
    x[2 * i + 1] = v[i].x * ri + v[i].y * rr;
  }
  return 0;
}

int cbp_fft2(cbp_ctx* ctx, const double* in, int rows, int cols, int inverse, double* out, void* stream) {
  cbp_host::DeviceGuard device_guard(ctx);
  cbp_host::StreamOrder stream_order(ctx, stream);
  if (!ctx || !in || !out) return CBP_INVALID_ARGUMENT;
  if (rows < 1 || cols < 1) return set_error(ctx, CBP_INVALID_ARGUMENT, "fft2 needs a nonempty matrix");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t n = size_t(rows) * cols;
  double2* X = ws_of<double2>(ctx, WS_MISC, 2 * n + rows + cols);
  if (!X) return set_error(ctx, CBP_CUDA_ERROR, "workspace allocation failed");
  double2* Y = X + n;
  double2* wr = Y + n;
  double2* wc = wr + rows;
  cudaMemcpyAsync(X, in, sizeof(double2) * n, cudaMemcpyHostToDevice, s);
  k_roots<<<(rows + 127) / 128, 128, 0, s>>>(wr, rows);
  k_roots<<<(cols + 127) / 128, 128, 0, s>>>(wc, cols);
  const unsigned g = unsigned((n + 127) / 128);
  k_dft_axis<<<g, 128, 0, s>>>(X, rows, cols, 0, wr, inverse, Y);
  k_dft_axis<<<g, 128, 0, s>>>(Y, rows, cols, 1, wc, inverse, X);
  ctx->launches += 4;
  if (inverse) {  // fft.cpp:193: 1 / (rows * cols)
    k_scale<<<g, 128, 0, s>>>(X, n, 1.0 / (double(rows) * double(cols)));
    ++ctx->launches;
  }
  cudaMemcpyAsync(out, X, sizeof(double2) * n, cudaMemcpyDeviceToHost, s);
  return cuda_check(ctx, cudaStreamSynchronize(s), "fft2");
}

}  // extern "C"
