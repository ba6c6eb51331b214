// Compile-time-planned in-place shared-memory FFT for the production grid sizes.
//
// Mixed-radix Cooley-Tukey with radices (R_1, ..., R_m), N = prod R_s, P_s = R_1...R_s.
// Stage s combines R_s sub-transforms of length P_{s-1}: butterfly (block, k) touches
// positions block*P_s + k + i*P_{s-1}, i < R_s, and writes its outputs back to the same
// positions, so a stage needs one barrier and only one butterfly in registers.
//  - DIT (twiddle, then DFT_R; s = 1..m) maps digit-reversed input to natural output.
//  - DIF (DFT_R, then twiddle; s = m..1) maps natural input to digit-reversed output.
// Digit reversal: pos(n) = (n mod R_m) * N/R_m + pos'(n / R_m) (pos' over R_1..R_{m-1}).
// Element n of sequence q lives at buf[q*SP + pos*ES]. Twiddles come from per-stage
// tables in butterfly order (stage_twiddles() on the host), stages in DIT order.
#pragma once

#include "cbp_fft.cuh"

namespace cbp_dev {

template <int... Rs>
struct Radices {};

template <int... Rs>
struct RadixProduct;
template <>
struct RadixProduct<> {
  static constexpr int value = 1;
};
template <int R, int... Rs>
struct RadixProduct<R, Rs...> {
  static constexpr int value = R * RadixProduct<Rs...>::value;
};

// ------------------------------------------------- bulk copies (TMA, no tensor map)
// One elected thread moves a whole contiguous run (size a multiple of 16 bytes, 16-byte
// aligned ends) between global and shared memory; loads complete on an mbarrier.
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_init_fence() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// generic-proxy accesses to shared memory before async-proxy (bulk copy) accesses
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(dst), "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
// the bulk stores of all committed groups have finished reading shared memory
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }

// pos over (R_1..R_m): peel R_m (the last template argument) by recursion on the list.
template <int... Rs>
struct LastRadix;
template <int R>
struct LastRadix<R> {
  static constexpr int value = R;
};
template <int R, int... Rest>
struct LastRadix<R, Rest...> {
  static constexpr int value = LastRadix<Rest...>::value;
};

template <class Done, class Todo>
struct DropLast;
template <int... Ds, int R>
struct DropLast<Radices<Ds...>, Radices<R>> {
  using type = Radices<Ds...>;
};
template <int... Ds, int R, int R2, int... Rest>
struct DropLast<Radices<Ds...>, Radices<R, R2, Rest...>> {
  using type = typename DropLast<Radices<Ds..., R>, Radices<R2, Rest...>>::type;
};

template <class Rs>
struct Pos;
template <>
struct Pos<Radices<>> {
  __device__ __forceinline__ static int get(int) { return 0; }
};
template <int R0, int... Rest>
struct Pos<Radices<R0, Rest...>> {
  static constexpr int Rm = LastRadix<R0, Rest...>::value;
  static constexpr int N = RadixProduct<R0, Rest...>::value;
  using Head = typename DropLast<Radices<>, Radices<R0, Rest...>>::type;
  __device__ __forceinline__ static int get(int n) { return (n % Rm) * (N / Rm) + Pos<Head>::get(n / Rm); }
};

// inverse of Pos<R_1..R_m>: the digit reversal for the reversed radix list
template <class Done, class Todo>
struct Reverse;
template <int... Ds>
struct Reverse<Radices<Ds...>, Radices<>> {
  using type = Radices<Ds...>;
};
template <int... Ds, int R, int... Rest>
struct Reverse<Radices<Ds...>, Radices<R, Rest...>> {
  using type = typename Reverse<Radices<R, Ds...>, Radices<Rest...>>::type;
};
template <class Rs>
using InvPos = Pos<typename Reverse<Radices<>, Rs>::type>;

// NSEQ sequences of length N; element position p of sequence q at buf[q*SP + p*ES].
// SEQ_FAST: consecutive threads walk sequences first (column strips).
// Twiddle table layout of a plan (stage_twiddles() on the host, DIT stage order): stage s
// holds (R_s - 1) * N / R_s entries; stage 1 (PP = 1) has no twiddles, so the used part of
// the table starts at TwUsed::offset and has TwUsed::count entries.
template <int N, class Rs>
struct TwTotal;
template <int N>
struct TwTotal<N, Radices<>> {
  static constexpr int value = 0;
};
template <int N, int R, int... Rest>
struct TwTotal<N, Radices<R, Rest...>> {
  static constexpr int value = (R - 1) * (N / R) + TwTotal<N, Radices<Rest...>>::value;
};
template <int N, class Rs>
struct TwUsed;
template <int N, int R1, int... Rest>
struct TwUsed<N, Radices<R1, Rest...>> {
  static constexpr int offset = (R1 - 1) * (N / R1);
  static constexpr int count = TwTotal<N, Radices<R1, Rest...>>::value - offset;
};

// TWS: the stage twiddle table lives in shared memory (plain loads instead of __ldg).
template <int N, int NSEQ, int SP, int ES, int NT, bool SEQ_FAST, bool TWS = false>
struct FftIP {
  __device__ __forceinline__ static float2 ldtw(const float2* p) {
    if constexpr (TWS) return *p;
    else return __ldg(p);
  }
  static_assert(!SEQ_FAST || NT % NSEQ == 0, "threads must split evenly over sequences");

  // DIT = false: DIF stage (DFT, then twiddle); true: DIT stage (twiddle, then DFT).
  // twst: this stage's twiddles in butterfly order, twst[(i-1)*NB + b] = W_{PS}^{i*(b % PP)},
  // so a warp's twiddle loads are contiguous.
  // MASK (first DIF stage only): input element n of a sequence holds floats 2n, 2n+1 of a
  // real row of nf valid floats; floats >= nf are read as zero, so the tile's row tails
  // (and any rows past the frame, whose outputs are discarded) need no zeroing.
  // FENCE: every thread orders its shared-memory writes before later async-proxy (bulk
  // copy) reads of them, ahead of the stage's closing barrier
  template <bool DIT, bool INV, int R, int PP, bool MASK = false, bool FENCE = false>
  __device__ __forceinline__ static void stage(float2* buf, const float2* __restrict__ twst, int nf = 0) {
    constexpr int NB = N / R;
    static_assert(!MASK || (!DIT && PP > 1), "masked loads: first DIF stage of a multi-stage plan");
    // Butterfly g of the CTA: sequence q, butterfly b. SEQ_FAST: consecutive threads take
    // consecutive sequences of one butterfly; otherwise butterflies are numbered flat over
    // (sequence, butterfly), so idle lanes gather in whole idle warps at the end.
    constexpr int NG = NSEQ * NB;
#pragma unroll 2
    for (int g = threadIdx.x; g < NG; g += NT) {
      const int q = SEQ_FAST ? g % NSEQ : g / NB;
      const int b = SEQ_FAST ? g / NSEQ : g - q * NB;
      float2* sb = buf + q * SP;
      if constexpr (PP == 1 && ES == 1 && R % 2 == 0 && SP % 2 == 0) {
        // contiguous butterflies: 16-byte accesses keep the stride-R pattern conflict-free
        float4* p4 = reinterpret_cast<float4*>(sb + b * R);
        float2 v[R];
#pragma unroll
        for (int j = 0; j < R / 2; ++j) {
          const float4 x = p4[j];
          v[2 * j] = make_float2(x.x, x.y);
          v[2 * j + 1] = make_float2(x.z, x.w);
        }
        dft<R, INV>(v);
#pragma unroll
        for (int j = 0; j < R / 2; ++j) p4[j] = make_float4(v[2 * j].x, v[2 * j].y, v[2 * j + 1].x, v[2 * j + 1].y);
      } else {
        const int k = PP > 1 ? b % PP : 0;
        const int base = (b - k) * R + k;  // block * PS + k
        float2 v[R];
#pragma unroll
        for (int i = 0; i < R; ++i) {
          v[i] = sb[(base + i * PP) * ES];
          if constexpr (MASK) {
            const int n2 = 2 * (base + i * PP);
            if (n2 >= nf) v[i] = make_float2(0.f, 0.f);
            else if (n2 + 1 == nf) v[i].y = 0.f;
          }
        }
        if (DIT && PP > 1) {
#pragma unroll
          for (int i = 1; i < R; ++i) {
            float2 w = ldtw(&twst[(i - 1) * NB + b]);
            if (INV) w.y = -w.y;
            v[i] = cmul(v[i], w);
          }
        }
        dft<R, INV>(v);
        if (!DIT && PP > 1) {
#pragma unroll
          for (int i = 1; i < R; ++i) {
            float2 w = ldtw(&twst[(i - 1) * NB + b]);
            if (INV) w.y = -w.y;
            v[i] = cmul(v[i], w);
          }
        }
#pragma unroll
        for (int i = 0; i < R; ++i) sb[(base + i * PP) * ES] = v[i];
      }
    }
    if constexpr (FENCE) fence_proxy_async();
    __syncthreads();
  }

  template <bool INV, int PP, bool FENCE = false>
  __device__ __forceinline__ static void dit_impl(float2*, const float2*, Radices<>) {}
  template <bool INV, int PP, bool FENCE = false, int R, int... Rest>
  __device__ __forceinline__ static void dit_impl(float2* buf, const float2* tw, Radices<R, Rest...>) {
    stage<true, INV, R, PP, false, FENCE && sizeof...(Rest) == 0>(buf, tw);
    dit_impl<INV, PP * R, FENCE>(buf, tw + (R - 1) * (N / R), Radices<Rest...>{});
  }
  template <bool INV, int PP>
  __device__ __forceinline__ static void dif_impl(float2*, const float2*, Radices<>) {}
  template <bool INV, int PP, int R, int... Rest>
  __device__ __forceinline__ static void dif_impl(float2* buf, const float2* tw, Radices<R, Rest...>) {
    dif_impl<INV, PP * R>(buf, tw + (R - 1) * (N / R), Radices<Rest...>{});
    stage<false, INV, R, PP>(buf, tw);
  }

  // Filtered round trip x -> DIT_inv(H .* DIF_fwd(x)) split so that the last DIF stage, the
  // element-wise product with H and the first DIT stage run as ONE register-resident step:
  // both stages have radix R_1 and PP = 1 (no twiddles) and touch the same R_1 contiguous
  // slots, so the spectrum of a butterfly never goes back to shared memory between them.
  // H is butterfly-major: element i of butterfly b of sequence q at hbuf[q*SP + i*NB + b]
  // (conflict-free: a warp reads consecutive words).
  //   dif_head: DIF stages R_m..R_2;  filter_stage: DFT_R1, * H, IDFT_R1;  dit_tail: R_2..R_m.
  template <int R1, int... Rest>
  __device__ __forceinline__ static void dif_head(float2* buf, const float2* tw, Radices<R1, Rest...>) {
    dif_impl<false, R1>(buf, tw + (R1 - 1) * (N / R1), Radices<Rest...>{});
  }
  // dif_head whose first stage reads elements n >= nf/2 (rows past the column) as zeros
  template <int R1, int... Rest>
  __device__ __forceinline__ static void dif_head_masked(float2* buf, const float2* tw, int nf, Radices<R1, Rest...>) {
    static_assert(sizeof...(Rest) > 0, "masked head needs a second radix");
    dif_impl_m<false, R1>(buf, tw + (R1 - 1) * (N / R1), nf, Radices<Rest...>{});
  }
  // FENCE: the last stage fences every writer before its barrier (the tile then leaves
  // shared memory by bulk copies)
  template <bool FENCE = false, int R1, int... Rest>
  __device__ __forceinline__ static void dit_tail(float2* buf, const float2* tw, Radices<R1, Rest...>) {
    dit_impl<true, R1, FENCE>(buf, tw + (R1 - 1) * (N / R1), Radices<Rest...>{});
  }
  template <int R1, int... Rest>
  __device__ __forceinline__ static void filter_stage(float2* buf, const float2* hbuf, Radices<R1, Rest...>) {
    constexpr int R = R1, NB = N / R, NG = NSEQ * NB;
#pragma unroll 1
    for (int g = threadIdx.x; g < NG; g += NT) {
      const int q = SEQ_FAST ? g % NSEQ : g / NB;
      const int b = SEQ_FAST ? g / NSEQ : g - q * NB;
      float2* sb = buf + q * SP + b * R * ES;
      const float2* hb = hbuf + q * SP + b;
      float2 v[R];
#pragma unroll
      for (int i = 0; i < R; ++i) v[i] = sb[i * ES];
      dft<R, false>(v);
#pragma unroll
      for (int i = 0; i < R; ++i) v[i] = cmul(v[i], hb[i * NB]);
      dft<R, true>(v);
#pragma unroll
      for (int i = 0; i < R; ++i) sb[i * ES] = v[i];
    }
    __syncthreads();
  }

  // filter_stage with H read from global memory (L2) in butterfly-major order: element i of
  // butterfly b of sequence q at hg[q*hsp + i*NB + b], so a warp's loads are contiguous.
  // Sequences q >= nq (absent columns) reuse sequence nq-1's filter (never stored).
  template <int R1, int... Rest>
  __device__ __forceinline__ static void filter_stage_g(float2* buf, const float2* __restrict__ hg, size_t hsp,
                                                        int nq, Radices<R1, Rest...>) {
    constexpr int R = R1, NB = N / R, NG = NSEQ * NB;
#pragma unroll 1
    for (int g = threadIdx.x; g < NG; g += NT) {
      const int q = SEQ_FAST ? g % NSEQ : g / NB;
      const int b = SEQ_FAST ? g / NSEQ : g - q * NB;
      float2* sb = buf + q * SP + b * R * ES;
      const float2* hb = hg + size_t(min(q, nq - 1)) * hsp + b;
      float2 v[R];
#pragma unroll
      for (int i = 0; i < R; ++i) v[i] = sb[i * ES];
      dft<R, false>(v);
#pragma unroll
      for (int i = 0; i < R; ++i) v[i] = cmul(v[i], __ldg(hb + i * NB));
      dft<R, true>(v);
#pragma unroll
      for (int i = 0; i < R; ++i) sb[i * ES] = v[i];
    }
    __syncthreads();
  }

  template <bool INV, int PP, int R, int... Rest>
  __device__ __forceinline__ static void dif_impl_m(float2* buf, const float2* tw, int nf, Radices<R, Rest...>) {
    if constexpr (sizeof...(Rest) == 0) {
      stage<false, INV, R, PP, true>(buf, tw, nf);
    } else {
      dif_impl_m<INV, PP * R>(buf, tw + (R - 1) * (N / R), nf, Radices<Rest...>{});
      stage<false, INV, R, PP>(buf, tw);
    }
  }
  // dif() of real rows with nf valid floats per row (element n = floats 2n, 2n+1); the
  // contents of the tile beyond them are ignored
  template <bool INV, int... Rs>
  __device__ __forceinline__ static void dif_masked(float2* buf, const float2* tw, int nf, Radices<Rs...>) {
    static_assert(RadixProduct<Rs...>::value == N, "radix plan does not multiply to N");
    dif_impl_m<INV, 1>(buf, tw, nf, Radices<Rs...>{});
  }

  // digit-reversed input -> natural output. Contains __syncthreads (whole CTA).
  template <bool INV, int... Rs>
  __device__ __forceinline__ static void dit(float2* buf, const float2* tw, Radices<Rs...> r) {
    static_assert(RadixProduct<Rs...>::value == N, "radix plan does not multiply to N");
    dit_impl<INV, 1>(buf, tw, r);
  }
  // natural input -> digit-reversed output.
  template <bool INV, int... Rs>
  __device__ __forceinline__ static void dif(float2* buf, const float2* tw, Radices<Rs...> r) {
    static_assert(RadixProduct<Rs...>::value == N, "radix plan does not multiply to N");
    dif_impl<INV, 1>(buf, tw, r);
  }
};

}  // namespace cbp_dev
