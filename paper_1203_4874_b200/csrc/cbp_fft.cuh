// Shared-memory mixed-radix Stockham FFT (FP32 data, FP64-accurate twiddle tables).
//
// Replaces the FFTW plans of the reference (core/src/fft.cpp:23-109, 242-270) for the
// 2/3/5/7-smooth grids chosen by friendly_size (fft.cpp:272-280). One CTA transforms a
// set of sequences resident in shared memory; each Stockham stage reads R inputs with
// stride n/R, applies twiddles from a global exp(-2*pi*i*k/n) table (L1-resident) and
// an in-register radix-R DFT, and writes the self-sorted output to the other buffer.
#pragma once

#include "cbp_common.cuh"
#include "cbp_roots.cuh"

namespace cbp_dev {

constexpr int kMaxStages = 24;

struct FftPlan {
  int n;
  int nst;
  int radix[kMaxStages];
};

// cos/sin(2*pi*m/R), m = 0..R-1, for the odd radices (exact float roundings).
template <int R>
struct OddRoots;
template <>
struct OddRoots<3> {
  __device__ static float c(int m) { return m == 0 ? 1.0f : -0.5f; }
  __device__ static float s(int m) { return m == 0 ? 0.0f : (m == 1 ? 0.866025403784438647f : -0.866025403784438647f); }
};
template <>
struct OddRoots<5> {
  __device__ static float c(int m) {
    const float t[5] = {1.0f, 0.309016994374947424f, -0.809016994374947424f, -0.809016994374947424f,
                        0.309016994374947424f};
    return t[m];
  }
  __device__ static float s(int m) {
    const float t[5] = {0.0f, 0.951056516295153572f, 0.587785252292473129f, -0.587785252292473129f,
                        -0.951056516295153572f};
    return t[m];
  }
};
template <>
struct OddRoots<7> {
  __device__ static float c(int m) {
    const float t[7] = {1.0f, 0.623489801858733531f, -0.222520933956314404f, -0.900968867902419126f,
                        -0.900968867902419126f, -0.222520933956314404f, 0.623489801858733531f};
    return t[m];
  }
  __device__ static float s(int m) {
    const float t[7] = {0.0f, 0.781831482468029809f, 0.974927912181823607f, 0.433883739117558120f,
                        -0.433883739117558120f, -0.974927912181823607f, -0.781831482468029809f};
    return t[m];
  }
};
template <>
struct OddRoots<9> {
  __device__ static float c(int m) {
    const float t[9] = {1.0f, 0.766044443118978035f, 0.173648177666930349f, -0.5f,
                        -0.939692620785908384f, -0.939692620785908384f, -0.5f,
                        0.173648177666930349f, 0.766044443118978035f};
    return t[m];
  }
  __device__ static float s(int m) {
    const float t[9] = {0.0f, 0.642787609686539326f, 0.984807753012208059f, 0.866025403784438647f,
                        0.342020143325668733f, -0.342020143325668733f, -0.866025403784438647f,
                        -0.984807753012208059f, -0.642787609686539326f};
    return t[m];
  }
};

// y_k = sum_j v_j exp(-+2*pi*i*j*k/R): INV=false uses the negative exponent (fft.hpp:9-10).
template <int R, bool INV>
__device__ __forceinline__ void dft_odd(float2* v) {
  constexpr int H = (R - 1) / 2;
  float2 a[H], b[H];
#pragma unroll
  for (int j = 1; j <= H; ++j) {
    a[j - 1] = cadd(v[j], v[R - j]);
    b[j - 1] = csub(v[j], v[R - j]);
  }
  float2 y0 = v[0];
#pragma unroll
  for (int j = 0; j < H; ++j) y0 = cadd(y0, a[j]);
  float2 out[R];
  out[0] = y0;
#pragma unroll
  for (int k = 1; k <= H; ++k) {
    float2 re = v[0];
    float2 im = make_float2(0.f, 0.f);
#pragma unroll
    for (int j = 1; j <= H; ++j) {
      const int m = (j * k) % R;
      const float c = OddRoots<R>::c(m), s = OddRoots<R>::s(m);
      re.x = fmaf(a[j - 1].x, c, re.x);
      re.y = fmaf(a[j - 1].y, c, re.y);
      im.x = fmaf(b[j - 1].x, s, im.x);
      im.y = fmaf(b[j - 1].y, s, im.y);
    }
    // forward: y_k = re - i*im, y_{R-k} = re + i*im
    if (!INV) {
      out[k] = make_float2(re.x + im.y, re.y - im.x);
      out[R - k] = make_float2(re.x - im.y, re.y + im.x);
    } else {
      out[k] = make_float2(re.x - im.y, re.y + im.x);
      out[R - k] = make_float2(re.x + im.y, re.y - im.x);
    }
  }
#pragma unroll
  for (int k = 0; k < R; ++k) v[k] = out[k];
}

template <bool INV>
__device__ __forceinline__ void dft4(float2& v0, float2& v1, float2& v2, float2& v3) {
  float2 a = cadd(v0, v2), b = csub(v0, v2), c = cadd(v1, v3), d = csub(v1, v3);
  // forward: -i*d ; inverse: +i*d
  float2 jd = INV ? make_float2(-d.y, d.x) : make_float2(d.y, -d.x);
  v0 = cadd(a, c);
  v2 = csub(a, c);
  v1 = cadd(b, jd);
  v3 = csub(b, jd);
}

// smallest factor used to split a composite radix R = A * B in registers
template <int R>
struct Split {
  static constexpr int A = (R % 9 == 0 && R != 9) ? 9 : (R % 8 == 0 && R != 8) ? 8 : (R % 4 == 0 && R != 4) ? 4
                         : (R % 7 == 0 && R != 7) ? 7 : (R % 5 == 0 && R != 5) ? 5 : (R % 3 == 0 && R != 3) ? 3
                         : (R % 2 == 0 && R != 2) ? 2 : R;
  static constexpr int B = R / A;
};

template <int R, bool INV>
__device__ __forceinline__ void dft(float2* v);

// x * W_R^m (W_R = exp(-+2 pi i / R)) for a compile-time m; quarter turns are swaps and
// sign flips instead of a full complex product
template <int R, bool INV>
__device__ __forceinline__ float2 twiddle_const(float2 x, int m) {
  if (m == 0) return x;
  if (2 * m == R) return make_float2(-x.x, -x.y);
  if (4 * m == R) return INV ? make_float2(-x.y, x.x) : make_float2(x.y, -x.x);      // -+i
  if (4 * m == 3 * R) return INV ? make_float2(x.y, -x.x) : make_float2(-x.y, x.x);  // +-i
  const float2 w = make_float2(Root<R>::re(m), INV ? -Root<R>::im(m) : Root<R>::im(m));
  return cmul(x, w);
}

// Composite in-register DFT, R = A*B (four-step): A-point DFTs of the B strided
// subsequences, twiddles W_R^{b*ka} (compile-time constants, cbp_roots.cuh), then B-point
// DFTs; output in natural order.
template <int R, bool INV>
__device__ __forceinline__ void dft_composite(float2* v) {
  constexpr int A = Split<R>::A, B = Split<R>::B;
  float2 z[B][A];
#pragma unroll
  for (int b = 0; b < B; ++b)
#pragma unroll
    for (int a = 0; a < A; ++a) z[b][a] = v[b + B * a];
#pragma unroll
  for (int b = 0; b < B; ++b) dft<A, INV>(z[b]);
#pragma unroll
  for (int b = 1; b < B; ++b)
#pragma unroll
    for (int ka = 1; ka < A; ++ka) z[b][ka] = twiddle_const<R, INV>(z[b][ka], (b * ka) % R);
#pragma unroll
  for (int ka = 0; ka < A; ++ka) {
    float2 t[B];
#pragma unroll
    for (int b = 0; b < B; ++b) t[b] = z[b][ka];
    dft<B, INV>(t);
#pragma unroll
    for (int kb = 0; kb < B; ++kb) v[ka + A * kb] = t[kb];
  }
}

template <int R, bool INV>
__device__ __forceinline__ void dft(float2* v) {
  if constexpr (R == 1) {
  } else if constexpr (R == 2) {
    float2 a = v[0], b = v[1];
    v[0] = cadd(a, b);
    v[1] = csub(a, b);
  } else if constexpr (R == 4) {
    dft4<INV>(v[0], v[1], v[2], v[3]);
  } else if constexpr (R == 8) {
    float2 e0 = v[0], e1 = v[2], e2 = v[4], e3 = v[6];
    float2 o0 = v[1], o1 = v[3], o2 = v[5], o3 = v[7];
    dft4<INV>(e0, e1, e2, e3);
    dft4<INV>(o0, o1, o2, o3);
    const float c = 0.707106781186547524f;
    // o_k *= w8^k, w8 = exp(-+2*pi*i/8)
    float2 t1, t2, t3;
    if (!INV) {
      t1 = make_float2(c * (o1.x + o1.y), c * (o1.y - o1.x));
      t2 = make_float2(o2.y, -o2.x);
      t3 = make_float2(c * (o3.y - o3.x), -c * (o3.x + o3.y));
    } else {
      t1 = make_float2(c * (o1.x - o1.y), c * (o1.x + o1.y));
      t2 = make_float2(-o2.y, o2.x);
      t3 = make_float2(-c * (o3.x + o3.y), c * (o3.x - o3.y));
    }
    v[0] = cadd(e0, o0);
    v[4] = csub(e0, o0);
    v[1] = cadd(e1, t1);
    v[5] = csub(e1, t1);
    v[2] = cadd(e2, t2);
    v[6] = csub(e2, t2);
    v[3] = cadd(e3, t3);
    v[7] = csub(e3, t3);
  } else if constexpr (R == 3 || R == 5 || R == 7) {
    dft_odd<R, INV>(v);
  } else {
    dft_composite<R, INV>(v);
  }
}

// One Stockham stage over nseq sequences; element k of sequence s lives at
// buf[s*sp + k*es]. SEQ_FAST maps consecutive threads to consecutive sequences
// (column strips, es = nseq) instead of consecutive butterflies (rows, es = 1).
template <int R, bool INV, bool SEQ_FAST>
__device__ __forceinline__ void stockham_stage(const float2* __restrict__ in, float2* __restrict__ out,
                                               int n, int ns, int nseq, int sp, int es,
                                               const float2* __restrict__ tw) {
  const int nb = n / R;
  const int step = n / (ns * R);
  const int total = nb * nseq;
  for (int b = threadIdx.x; b < total; b += blockDim.x) {
    int s, j;
    if (SEQ_FAST) {
      s = b % nseq;
      j = b / nseq;
    } else {
      j = b % nb;
      s = b / nb;
    }
    const int k = j % ns;
    const float2* src = in + s * sp;
    float2 v[R];
#pragma unroll
    for (int i = 0; i < R; ++i) v[i] = src[(j + i * nb) * es];
    if (k != 0) {
#pragma unroll
      for (int i = 1; i < R; ++i) {
        float2 w = __ldg(&tw[i * k * step]);
        if (INV) w.y = -w.y;
        v[i] = cmul(v[i], w);
      }
    }
    dft<R, INV>(v);
    const int base = (j - k) * R + k;
    float2* dst = out + s * sp;
#pragma unroll
    for (int i = 0; i < R; ++i) dst[(base + i * ns) * es] = v[i];
  }
}

// Runs the whole plan; data starts in `a`, `b` is scratch. Returns the buffer that
// holds the result. Contains __syncthreads() (call from the whole CTA).
template <bool INV, bool SEQ_FAST>
__device__ float2* fft_run(float2* a, float2* b, const FftPlan& plan, int nseq, int sp, int es,
                          const float2* __restrict__ tw) {
  int ns = 1;
  for (int st = 0; st < plan.nst; ++st) {
    const int r = plan.radix[st];
    switch (r) {
      case 2: stockham_stage<2, INV, SEQ_FAST>(a, b, plan.n, ns, nseq, sp, es, tw); break;
      case 3: stockham_stage<3, INV, SEQ_FAST>(a, b, plan.n, ns, nseq, sp, es, tw); break;
      case 4: stockham_stage<4, INV, SEQ_FAST>(a, b, plan.n, ns, nseq, sp, es, tw); break;
      case 5: stockham_stage<5, INV, SEQ_FAST>(a, b, plan.n, ns, nseq, sp, es, tw); break;
      case 7: stockham_stage<7, INV, SEQ_FAST>(a, b, plan.n, ns, nseq, sp, es, tw); break;
      case 8: stockham_stage<8, INV, SEQ_FAST>(a, b, plan.n, ns, nseq, sp, es, tw); break;
      case 9: stockham_stage<9, INV, SEQ_FAST>(a, b, plan.n, ns, nseq, sp, es, tw); break;
      default: break;
    }
    __syncthreads();
    float2* t = a;
    a = b;
    b = t;
    ns *= r;
  }
  return a;
}

}  // namespace cbp_dev
