// Compile-time-planned deconvolution passes for the production grids (1080p, 4K,
// 640x480, 256x256 configs of BASELINE.json). Same math as cbp_deblur.cu (reference
// decoder.cpp:187-214); grids without a specialisation use the runtime-planned kernels.
//
// Each pass is a persistent kernel: a CTA walks tiles (plane x row group, or plane x
// column strip) with stride gridDim.x and keeps two tile buffers in shared memory;
// the next tile's global->shared copies (cp.async, zero-filled outside the frame) are
// in flight while the current tile is transformed, so HBM/L2 latency overlaps the FFT.
#include <cstdlib>
#include <cstring>
#include <vector>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "cbp_deblur.cuh"
#include "cbp_fft_ct.cuh"

namespace cbp_dev {

template <class Rs>
struct RadixCount;
template <int... Rs>
struct RadixCount<Radices<Rs...>> {
  static constexpr int value = sizeof...(Rs);
};


// PIPE: persistent CTAs with a double-buffered cp.async prefetch of the next tile;
// otherwise one tile per CTA and latency is hidden by many resident CTAs.
// MINB: resident CTAs per SM the register allocation must allow (__launch_bounds__).
// HD (columns): read the filter straight from L2 in the multiply instead of staging it.
// RTW (rows): the split twiddles tw_post and the used stage twiddles are copied to shared
// memory per CTA and the digit reversal pos(k) is computed (no pos table).
template <int L_, int RPC_, class Rs, int NT_, bool PIPE_ = true, int MINB_ = 1, bool RTW_ = false>
struct RowPlan {
  static constexpr bool RTW = RTW_;
  static constexpr int TWN = RTW_ ? L_ / 2 + 1 + TwUsed<L_, Rs>::count : 0;  // shared float2 entries
  static constexpr int L = L_;
  // pass A row stride in the tile: rows 2j and 2j + 2 (read by one split warp) fall 16 banks
  // apart only if the stride is 4 (mod 8) complex values, so L = 0 (mod 8) is padded
  static constexpr int SPA = L_ % 8 == 0 ? L_ + 4 : L_;
  static constexpr int RPC = RPC_;
  static constexpr int NT = NT_;
  static constexpr bool PIPE = PIPE_;
  static constexpr int MINB = MINB_;
  using R = Rs;
};
template <int G_, int W_, class Rs, int NT_, bool PIPE_ = true, int MINB_ = 1, bool HD_ = false>
struct ColPlan {
  static constexpr int G = G_;
  static constexpr int W = W_;
  static constexpr int NT = NT_;
  static constexpr bool PIPE = PIPE_;
  static constexpr int MINB = MINB_;
  static constexpr bool HD = HD_;
  using R = Rs;
};

// RTW: copy tw_post[0..L/2] and the used stage twiddles into tws; returns the stage table
// base to hand to FftIP (offset so that the plan's own indices land in the copy).
template <class P>
__device__ __forceinline__ const float2* stage_row_twiddles(const DeblurArgs& a, float2* tws) {
  constexpr int L = P::L, NP = L / 2 + 1;
  using U = TwUsed<L, typename P::R>;
  for (int i = threadIdx.x; i < NP; i += P::NT) tws[i] = __ldg(&a.tw_post[i]);
  for (int i = threadIdx.x; i < U::count; i += P::NT) tws[NP + i] = __ldg(&a.twst_row[U::offset + i]);
  return tws + NP - U::offset;
}

__device__ __forceinline__ const cbp_kernel_slot* plane_slot(const DeblurArgs& a, int p) {
  return a.slot + deblur_slot_index(a, p);
}

// The half spectrum lives transposed in HBM/L2: XT[v][u] (v < Hc columns, u < Mb rows,
// pitch xp = Mb rounded to 4), so a column strip is contiguous for pass B and a group of
// 4 rows is one 32-byte sector per frequency for passes A and C.

// ------------------------------------------------------------ pass A (rows r2c)
// Row s of a tile holds z[m] = (x[2m], x[2m+1]); the forward DIF leaves Z[k] in slot pos(k);
// the r2c split handles the pair (k, L-k) in one thread: X[k] = e + W^k o,
// X[L-k] = conj(e - W^k o), e = (Z[k] + conj Z[L-k])/2, o = -i (Z[k] - conj Z[L-k])/2.
// BULK: the input rows arrive by bulk copies (one per row, TMA engine, completion on an
// mbarrier; rows 16-byte aligned with a pitch >= Nb rounded to 4); threads then zero the
// row tails Nb..2L-1 and the rows beyond Mb.
template <class P, bool BULK = false>
__global__ void __launch_bounds__(P::NT, P::MINB) k_rows_forward_ct(DeblurArgs a, int planes) {
  constexpr int NT = P::NT;
  constexpr int L = P::L, RPC = P::RPC, SPA = P::SPA, TILE = RPC * SPA;
  using R = typename P::R;
  using FFT = FftIP<L, RPC, SPA, 1, NT, false, P::RTW>;
  static_assert(!BULK || (P::PIPE && L % 2 == 0), "bulk rows need two buffers and 16-byte row starts");
  extern __shared__ __align__(16) float2 sm[];
  short* pos = reinterpret_cast<short*>(sm + (P::PIPE ? 2 : 1) * TILE);
  float2* tws = sm + (P::PIPE ? 2 : 1) * TILE;  // RTW: [tw_post][stage twiddles]
  const float2* twst = a.twst_row;
  const float2* twp = a.tw_post;
  if constexpr (P::RTW) {
    twst = stage_row_twiddles<P>(a, tws);
    twp = tws;
  } else {
    for (int i = threadIdx.x; i < L; i += NT) pos[i] = short(Pos<R>::get(i));
  }
  auto posk = [&](int k) { return P::RTW ? Pos<R>::get(k) : int(pos[k]); };
  const int groups = (a.Mb + RPC - 1) / RPC;
  const int total = planes * groups;
  const bool v16 = a.in_vec4 && (L % 2 == 0);
  __shared__ __align__(8) unsigned long long bar[2];
  unsigned ph = 0u;  // mbarrier phase bits of buffers 0, 1 (a register, not an indexed array)
  const unsigned row_bytes = unsigned((a.Nb + 3) & ~3) * 4u;  // 16-byte multiple, within the pitch
  if constexpr (BULK) {
    if (threadIdx.x == 0) {
      mbar_init(&bar[0], 1);
      mbar_init(&bar[1], 1);
      mbar_init_fence();
    }
  }
  __syncthreads();  // pos table / staged twiddles, barriers
  auto issue_bulk = [&](int tile, float2* dst, unsigned long long* b) {  // thread 0
    const int p = tile / groups, r0 = (tile - p * groups) * RPC;
    const float* src = a.in + size_t(p) * a.in_plane + size_t(r0) * a.in_ld;
    const int nr = min(RPC, a.Mb - r0);
    fence_proxy_async();
    mbar_expect_tx(b, unsigned(nr) * row_bytes);
    for (int s = 0; s < nr; ++s) bulk_g2s(dst + s * SPA, src + size_t(s) * a.in_ld, row_bytes, b);
  };
  auto issue = [&](int tile, float2* dst) {
    const int p = tile / groups, r0 = (tile - p * groups) * RPC;
    const float* src = a.in + size_t(p) * a.in_plane + size_t(r0) * a.in_ld;
#pragma unroll
    for (int s = 0; s < RPC; ++s) {
      const bool ok = r0 + s < a.Mb;
      const float* row = src + size_t(s) * a.in_ld;
      float2* d = dst + s * SPA;
      if (v16) {
        const int full = ok ? a.Nb / 4 : 0;  // whole 16-byte chunks inside the row
#pragma unroll 1
        for (int c = threadIdx.x; c < L / 2; c += NT) {
          int bytes = c < full ? 16 : (ok ? min(max((a.Nb - 4 * c) * 4, 0), 16) : 0);
          cp_async16(d + 2 * c, bytes ? row + 4 * c : a.in, bytes);
        }
      } else {
#pragma unroll 1
        for (int m = threadIdx.x; m < L; m += NT) {
          const int bytes = ok ? min(max((a.Nb - 2 * m) * 4, 0), 8) : 0;
          cp_async8(d + m, bytes ? row + 2 * m : a.in, bytes);
        }
      }
    }
  };
  int tile = blockIdx.x;
  if constexpr (BULK) {
    if (tile < total && threadIdx.x == 0) issue_bulk(tile, sm, &bar[0]);
  } else {
    if (tile < total) issue(tile, sm);
    cp_async_commit();
  }
  // dynamic tiles: after its first (static) tile a CTA takes the next one from a counter,
  // so CTAs that start late (SMs still held by another stream's kernels) take fewer tiles
  unsigned* const ctr = BULK && a.tile_ctr ? a.tile_ctr + 0 : nullptr;
  __shared__ int s_next[2];
  for (int it = 0; tile < total; ++it) {
    float2* cur = sm + (P::PIPE ? (it & 1) * TILE : 0);
    int next = tile + gridDim.x;
    if (ctr && threadIdx.x == 0) {  // only thread 0 uses `next` before the loop-end barrier
      next = int(gridDim.x + atomicAdd(ctr, 1u));
      s_next[it & 1] = next;
    }
    if constexpr (BULK) {
      const int cb = it & 1;
      if (next < total && threadIdx.x == 0) issue_bulk(next, sm + (cb ^ 1) * TILE, &bar[cb ^ 1]);
      // every thread observes the rows' arrival; the first DIF stage reads floats >= Nb
      // (row tails, stale rows past the frame) as zeros, so no zeroing and no barrier
      mbar_wait(&bar[cb], (ph >> cb) & 1u);
      ph ^= 1u << cb;
      if (!(a.dbg & 1)) FFT::template dif_masked<false>(cur, twst, a.Nb, R{});
    } else {
      if (P::PIPE && next < total) issue(next, sm + ((it + 1) & 1) * TILE);
      cp_async_commit();
      cp_async_wait<1>();
      __syncthreads();
      if (!(a.dbg & 1)) FFT::template dif<false>(cur, twst, R{});
    }
    const int p = tile / groups, r0 = (tile - p * groups) * RPC;
    float2* XT = a.X + size_t(p) * a.x_plane + r0;
    const int nrows = min(RPC, a.Mb - r0);
    // one thread per frequency pair (k, L-k) and row pair (2j, 2j+1): 16-byte stores
    constexpr int NPAIR = L / 2 + 1, HALF = RPC / 2;
#pragma unroll 1
    for (int idx = threadIdx.x; idx < NPAIR * HALF; idx += NT) {
      const int k = idx / HALF, j = idx - k * HALF;
      if (2 * j >= nrows) continue;
      const int pk = posk(k), pc = posk(k == 0 ? 0 : L - k);
      const float2 w = P::RTW ? twp[k] : __ldg(&twp[k]);
      float2 xk[2], xc[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const float2* z = cur + (2 * j + h) * SPA;
        const float2 zk = z[pk], zc = cconj(z[pc]);
        const float2 e = cscale(cadd(zk, zc), 0.5f);
        const float2 d = csub(zk, zc);
        const float2 wo = cmul(w, make_float2(0.5f * d.y, -0.5f * d.x));  // W^k * (-i/2) d
        xk[h] = cadd(e, wo);
        xc[h] = cconj(csub(e, wo));
      }
      float2* dk = XT + size_t(k) * a.xp + 2 * j;
      float2* dc = XT + size_t(L - k) * a.xp + 2 * j;
      if (2 * j + 1 < nrows) {
        *reinterpret_cast<float4*>(dk) = make_float4(xk[0].x, xk[0].y, xk[1].x, xk[1].y);
        if (L - k != k) *reinterpret_cast<float4*>(dc) = make_float4(xc[0].x, xc[0].y, xc[1].x, xc[1].y);
      } else {
        dk[0] = xk[0];
        if (L - k != k) dc[0] = xc[0];
      }
    }
    __syncthreads();
    tile = ctr ? s_next[it & 1] : tile + gridDim.x;
  }
  if constexpr (!BULK) cp_async_wait<0>();
}

// ----------------------------------------------- pass B (columns + Wiener filter)
// Column v of XT is contiguous: 16-byte copies into a [column][row] tile; the forward DIF
// leaves spectrum row u in slot pos(u), where the filter table (k_wiener_h) already stores
// H(u, v), so the filter is an element-wise product; the inverse DIT restores natural rows.
template <class P>
__global__ void __launch_bounds__(P::NT, P::MINB) k_cols_filter_ct(DeblurArgs a, int planes) {
  constexpr int NT = P::NT;
  constexpr int G = P::G, W = P::W, GP = ((G + 11) / 16) * 16 + 4, TILE = GP * W;  // padded: sequences on distinct banks
  constexpr int NBUF = P::PIPE ? 2 : 1;
  using R = typename P::R;
  using FFT = FftIP<G, W, GP, 1, NT, false>;
  extern __shared__ __align__(16) float2 sm[];
  float2* Hs = sm + NBUF * TILE;
  const int strips = (a.Hc + W - 1) / W;
  const int total = planes * strips;
  auto issue = [&](int tile, float2* dst) {
    const int p = tile / strips, v0 = (tile - p * strips) * W;
    const float2* XT = a.X + size_t(p) * a.x_plane;
#pragma unroll
    for (int s = 0; s < W; ++s) {
      const bool ok = v0 + s < a.Hc;
      const float2* col = XT + size_t(v0 + s) * a.xp;
      for (int c = threadIdx.x; c < GP / 2; c += NT) {
        const int bytes = ok ? min(max((a.Mb - 2 * c) * 8, 0), 16) : 0;
        cp_async16(dst + s * GP + 2 * c, bytes ? col + 2 * c : a.X, bytes);
      }
    }
  };
  int tile = blockIdx.x;
  if (tile < total) issue(tile, sm);
  cp_async_commit();
  for (int it = 0; tile < total; tile += gridDim.x, ++it) {
    float2* cur = sm + (P::PIPE ? (it & 1) * TILE : 0);
    const int p = tile / strips, v0 = (tile - p * strips) * W;
    const int f = deblur_slot_index(a, p);
    const cbp_kernel_slot* slot = a.slot + f;
    const int status = slot->status;
    cp_async_wait<0>();
    __syncthreads();
    if (status == 0 && !P::HD) {  // filter strip in flight during the forward transform
      const float2* Ht = a.H + size_t(f) * a.h_frame;
#pragma unroll
      for (int s = 0; s < W; ++s) {
        const bool ok = v0 + s < a.Hc;
        const float2* hcol = Ht + size_t(v0 + s) * a.hp;
        for (int c = threadIdx.x; c < GP / 2; c += NT) {
          const int bytes = ok ? min(max((G - 2 * c) * 8, 0), 16) : 0;
          cp_async16(Hs + s * GP + 2 * c, bytes ? hcol + 2 * c : a.H, bytes);
        }
      }
    }
    cp_async_commit();
    const int next = tile + gridDim.x;
    if (P::PIPE && next < total) issue(next, sm + ((it + 1) & 1) * TILE);
    cp_async_commit();
    if (status == 0) {  // uniform over the CTA; fused filter stage (see k_cols_filter_bulk)
      const int t = slot->width;
      FFT::dif_head(cur, a.twst_col, R{});
      if constexpr (P::HD) {
        FFT::filter_stage_g(cur, a.H + size_t(f) * a.h_frame + size_t(v0) * a.hp, a.hp, min(W, a.Hc - v0), R{});
      } else {
        cp_async_wait<1>();
        __syncthreads();  // filter strip (copied by all threads) visible
        FFT::filter_stage(cur, Hs, R{});
      }
      FFT::dit_tail(cur, a.twst_col, R{});
      const int M = a.Mb - t + 1;
      float2* XT = a.X + size_t(p) * a.x_plane;
#pragma unroll
      for (int s = 0; s < W; ++s) {
        if (v0 + s >= a.Hc) break;
        float2* col = XT + size_t(v0 + s) * a.xp;
        const float4* src = reinterpret_cast<const float4*>(cur + s * GP);
        for (int c = threadIdx.x; c < M / 2; c += NT) reinterpret_cast<float4*>(col)[c] = src[c];
        if ((M & 1) && threadIdx.x == 0) col[M - 1] = cur[s * GP + M - 1];
      }
    }
    __syncthreads();
  }
  cp_async_wait<0>();
}

// Pass B with bulk copies (TMA engine): one thread moves each column strip in (a single
// copy per column, completion on an mbarrier), the filter strip likewise, and the filtered
// columns back out (bulk stores, drained before the buffer is refilled). Needs an even
// Mb (16-byte multiple column runs); the first DIF stage reads rows Mb..G-1 as zeros.
template <class P>
__global__ void __launch_bounds__(P::NT, P::MINB) k_cols_filter_bulk(DeblurArgs a, int planes) {
  constexpr int NT = P::NT;
  constexpr int G = P::G, W = P::W, GP = ((G + 11) / 16) * 16 + 4, TILE = GP * W;
  constexpr int HB = ((G + 1) / 2) * 2;  // filter run: G rounded up to an even count (16-byte multiple)
  using R = typename P::R;
  using FFT = FftIP<G, W, GP, 1, NT, false>;
  static_assert(P::PIPE, "bulk pass B keeps two tile buffers");
  // HD: the filter is read from L2 in the fused stage (butterfly-major table, hpos from
  // column_slots(..., bmajor)); otherwise a filter strip is staged in shared memory
  extern __shared__ __align__(16) float2 sm[];
  float2* Hs = sm + 2 * TILE;
  __shared__ __align__(8) unsigned long long bar[3];  // tile buffers 0, 1; filter strip
  const int strips = (a.Hc + W - 1) / W;
  const int total = planes * strips;
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_init(&bar[2], 1);
    mbar_init_fence();
  }
  __syncthreads();
  // planes in reverse order: pass A wrote the last planes most recently, so the first strips
  // read here still sit in L2 (and pass C, in forward order, starts on the planes this pass
  // wrote last)
  auto plane_of = [&](int tile) { return planes - 1 - tile / strips; };
  auto issue = [&](int tile, float2* dst, unsigned long long* b) {  // thread 0
    const int p = plane_of(tile), v0 = (tile % strips) * W;
    const float2* XT = a.X + size_t(p) * a.x_plane;
    const int nc = min(W, a.Hc - v0);
    fence_proxy_async();
    mbar_expect_tx(b, unsigned(nc) * unsigned(a.Mb) * 8u);
    for (int s = 0; s < nc; ++s) bulk_g2s(dst + s * GP, XT + size_t(v0 + s) * a.xp, unsigned(a.Mb) * 8u, b);
  };
  unsigned ph = 0u, phh = 0u;  // phase bits of buffers 0, 1; filter strip
  int tile = blockIdx.x;
  if (tile < total && threadIdx.x == 0) issue(tile, sm, &bar[0]);
  // dynamic tiles: after its first (static) tile a CTA takes the next one from a counter,
  // so CTAs that start late (SMs still held by another stream's kernels) take fewer tiles
  unsigned* const ctr = a.tile_ctr ? a.tile_ctr + 1 : nullptr;
  __shared__ int s_next[2];
  for (int it = 0; tile < total; ++it) {
    const int cb = it & 1;
    float2* cur = sm + cb * TILE;
    const int p = plane_of(tile), v0 = (tile % strips) * W;
    const int f = deblur_slot_index(a, p);
    const cbp_kernel_slot* slot = a.slot + f;
    const int status = slot->status;
    mbar_wait(&bar[cb], (ph >> cb) & 1u);  // every thread observes the strip's arrival
    ph ^= 1u << cb;
    const int nc = min(W, a.Hc - v0);
    if (!P::HD && status == 0 && threadIdx.x == 0) {  // filter strip in flight during the forward transform
      const float2* Ht = a.H + size_t(f) * a.h_frame;
      fence_proxy_async();
      mbar_expect_tx(&bar[2], unsigned(nc) * unsigned(HB) * 8u);
      for (int s = 0; s < nc; ++s) bulk_g2s(Hs + s * GP, Ht + size_t(v0 + s) * a.hp, unsigned(HB) * 8u, &bar[2]);
    }
    int next = tile + gridDim.x;
    if (ctr && threadIdx.x == 0) {  // only thread 0 uses `next` before the loop-end barrier
      next = int(gridDim.x + atomicAdd(ctr, 1u));
      s_next[it & 1] = next;
    }
    if (next < total) {  // prefetch into the other buffer (its last bulk stores drained first)
      float2* nb = sm + (cb ^ 1) * TILE;
      if (threadIdx.x == 0) {
        bulk_wait_read();
        issue(next, nb, &bar[cb ^ 1]);
      }
    }
    if (status == 0) {  // uniform over the CTA
      // fused: DIF head, (last DIF stage, filter, first DIT stage) in registers, DIT tail
      const int t = slot->width;
      // rows Mb..G-1 read as zeros by the first stage; absent columns (v >= Hc) hold stale
      // data whose results are never stored
      FFT::dif_head_masked(cur, a.twst_col, 2 * a.Mb, R{});
      if constexpr (P::HD) {
        FFT::filter_stage_g(cur, a.H + size_t(f) * a.h_frame + size_t(v0) * a.hp, a.hp, nc, R{});
      } else {
        mbar_wait(&bar[2], phh);  // every thread observes the filter strip's arrival
        phh ^= 1u;
        FFT::filter_stage(cur, Hs, R{});
      }
      FFT::template dit_tail<true>(cur, a.twst_col, R{});  // every writer fences before the last barrier
      const int M = a.Mb - t + 1;  // even: Mb even, t odd
      if (threadIdx.x == 0) {
        float2* XT = a.X + size_t(p) * a.x_plane;
        for (int s = 0; s < nc; ++s) bulk_s2g(XT + size_t(v0 + s) * a.xp, cur + s * GP, unsigned(M) * 8u);
        bulk_commit();
      }
    }
    __syncthreads();
    tile = ctr ? s_next[it & 1] : tile + gridDim.x;
  }
  if (threadIdx.x == 0) bulk_wait_all();
}

// ------------------------------------------------- pass C (rows c2r + crop)
// Tile layout [slot][s] (RPC rows interleaved): one frequency of RPC consecutive rows is
// one 32-byte chunk of XT, copied straight into its digit-reversed slot pos(k) (X[L] into
// the spare slot L). The pairwise c2r split works slot to slot in place, the inverse DIT
// leaves z[n] in natural order, so each thread stores z[n] of all RPC rows.
template <class P, bool TMA = false>
__global__ void __launch_bounds__(P::NT, P::MINB) k_rows_inverse_ct(DeblurArgs a, int planes,
                                                                     const __grid_constant__ CUtensorMap tmap) {
  constexpr int NT = P::NT;
  constexpr int L = P::L, RPC = P::RPC, H = L + 1, TILE = ((H * RPC + 15) & ~15);  // 128-byte buffers
  static_assert(RPC % 2 == 0, "16-byte copies carry two rows");
  using R = typename P::R;
  using FFT = FftIP<L, RPC, 1, RPC, NT, true, P::RTW>;
  extern __shared__ __align__(128) float2 sm_c[];  // TMA tile destinations: 128-byte aligned
  float2* const sm = sm_c;
  // after the tiles: RTW ? [tw_post][stage twiddles] : pos table (DIT input slot of z[n]); then barriers
  constexpr int AUX = P::RTW ? P::TWN : (L + 3) / 4;
  short* pos = reinterpret_cast<short*>(sm + (P::PIPE ? 2 : 1) * TILE);
  float2* tws = sm + (P::PIPE ? 2 : 1) * TILE;
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(sm + (P::PIPE ? 2 : 1) * TILE + AUX);
  const float2* twst = a.twst_row;
  const float2* twp = a.tw_post;
  if constexpr (P::RTW) {
    twst = stage_row_twiddles<P>(a, tws);
    twp = tws;
  } else {
    for (int i = threadIdx.x; i < L; i += NT) pos[i] = short(Pos<R>::get(i));
  }
  auto posk = [&](int k) { return P::RTW ? Pos<R>::get(k) : int(pos[k]); };
  __syncthreads();
  const int groups = (a.Mb + RPC - 1) / RPC;
  const int total = planes * groups;
  auto rows_of = [&](int p) {
    const cbp_kernel_slot* sl = plane_slot(a, p);
    return sl->status == 0 ? a.Mb - sl->width + 1 : 0;  // failed frames: nothing to write
  };
  auto issue = [&](int tile, float2* dst) {
    const int p = tile / groups, r0 = (tile - p * groups) * RPC;
    const int M = rows_of(p);
    const float2* XT = a.X + size_t(p) * a.x_plane + r0;
    constexpr int HALF = RPC / 2;
    for (int idx = threadIdx.x; idx < H * HALF; idx += NT) {
      const int k = idx / HALF, j = idx - k * HALF;
      const int rows_left = M - r0 - 2 * j;
      const int bytes = rows_left >= 2 ? 16 : (rows_left == 1 ? 8 : 0);
      const int slot = k < L ? posk(k) : L;
      cp_async16(dst + slot * RPC + 2 * j, bytes ? XT + size_t(k) * a.xp + 2 * j : a.X, bytes);
    }
  };
  // TMA: one tensor copy per tile. The map views XT as (row u, digit d_1, ..., digit d_m,
  // plane), the frequency k split into the radix digits of the column order, so the box
  // lands with frequency k in slot pos(k) (a digit reversal is a transpose of the digit
  // axes); X[L] goes to the spare slot by a bulk copy (clipped to the pitch).
  unsigned ph = 0u;  // mbarrier phase bits of buffers 0, 1 (a register, not an indexed array)
  constexpr int NRAD = RadixCount<R>::value;
  if constexpr (TMA) {
    if (threadIdx.x == 0) {
      mbar_init(&bar[0], 1);
      mbar_init(&bar[1], 1);
      mbar_init_fence();
    }
    __syncthreads();
  }
  auto issue_tma = [&](int tile, float2* dst, unsigned long long* b) {  // thread 0
    const int p = tile / groups, r0 = (tile - p * groups) * RPC;
    const unsigned tail = unsigned(min(RPC, a.xp - r0)) * 8u;
    fence_proxy_async();
    mbar_expect_tx(b, unsigned(RPC) * L * 8u + tail);
    const unsigned d = smem_u32(dst), bb = smem_u32(b);
    const unsigned long long tm = reinterpret_cast<unsigned long long>(&tmap);
    if constexpr (NRAD == 2)
      asm volatile(
          "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];\n"
          ::"r"(d), "l"(tm), "r"(r0), "r"(0), "r"(0), "r"(p), "r"(bb) : "memory");
    else
      asm volatile(
          "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];\n"
          ::"r"(d), "l"(tm), "r"(r0), "r"(0), "r"(0), "r"(0), "r"(p), "r"(bb) : "memory");
    bulk_g2s(dst + L * RPC, a.X + size_t(p) * a.x_plane + size_t(L) * a.xp + r0, tail, b);
  };
  int tile = blockIdx.x;
  if constexpr (TMA) {
    if (tile < total && threadIdx.x == 0) issue_tma(tile, sm, &bar[0]);
  } else {
    if (tile < total) issue(tile, sm);
    cp_async_commit();
  }
  // dynamic tiles: after its first (static) tile a CTA takes the next one from a counter,
  // so CTAs that start late (SMs still held by another stream's kernels) take fewer tiles
  unsigned* const ctr = TMA && a.tile_ctr ? a.tile_ctr + 2 : nullptr;
  int* const s_next = reinterpret_cast<int*>(bar + 2);  // dynamic smem: static smem would break the 128-byte TMA alignment
  for (int it = 0; tile < total; ++it) {
    float2* cur = sm + (P::PIPE ? (it & 1) * TILE : 0);
    int next = tile + gridDim.x;
    if (ctr && threadIdx.x == 0) {  // only thread 0 uses `next` before the loop-end barrier
      next = int(gridDim.x + atomicAdd(ctr, 1u));
      s_next[it & 1] = next;
    }
    if constexpr (TMA) {
      const int cb = it & 1;
      if (next < total && threadIdx.x == 0) issue_tma(next, sm + (cb ^ 1) * TILE, &bar[cb ^ 1]);
      mbar_wait(&bar[cb], (ph >> cb) & 1u);  // every thread observes the tile's arrival: no barrier
      ph ^= 1u << cb;
    } else {
      if (P::PIPE && next < total) issue(next, sm + ((it + 1) & 1) * TILE);
      cp_async_commit();
      cp_async_wait<1>();
      __syncthreads();
    }
    const int p = tile / groups, r0 = (tile - p * groups) * RPC;
    const int M = rows_of(p);
    const int nrows = min(RPC, M - r0);
    if (nrows > 0) {
      // inverse split in place (fft.cpp:257-270 c2r), one thread per frequency pair (k, L-k)
      // and row pair: 16-byte shared-memory accesses
      constexpr int NP = L / 2 + 1, HALF = RPC / 2;
#pragma unroll 1
      for (int idx = threadIdx.x; idx < NP * HALF; idx += NT) {
        const int k = idx / HALF, j = idx - k * HALF;
        float4* pa = reinterpret_cast<float4*>(cur + posk(k) * RPC + 2 * j);
        float4* pb = reinterpret_cast<float4*>(cur + (k == 0 ? L : posk(L - k)) * RPC + 2 * j);
        const float4 A4 = *pa, B4 = *pb;
        const float2 w = cconj(P::RTW ? twp[k] : __ldg(&twp[k]));
        const float2 wm = make_float2(-w.x, w.y);  // conj(tw_post[L-k]) = -tw_post[k]
        float2 r1[2], r2[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const float2 A = h ? make_float2(A4.z, A4.w) : make_float2(A4.x, A4.y);
          const float2 B = h ? make_float2(B4.z, B4.w) : make_float2(B4.x, B4.y);
          const float2 e1 = cadd(A, cconj(B));
          const float2 o1 = cmul(csub(A, cconj(B)), w);
          r1[h] = make_float2(e1.x - o1.y, e1.y + o1.x);
          const float2 e2 = cadd(B, cconj(A));
          const float2 o2 = cmul(csub(B, cconj(A)), wm);
          r2[h] = make_float2(e2.x - o2.y, e2.y + o2.x);
        }
        *pa = make_float4(r1[0].x, r1[0].y, r1[1].x, r1[1].y);
        if (k != 0 && 2 * k != L) *pb = make_float4(r2[0].x, r2[0].y, r2[1].x, r2[1].y);
      }
      __syncthreads();
      if (!(a.dbg & 1)) FFT::template dit<true>(cur, twst, R{});  // slot -> natural order
      const int N = a.Nb - (a.Mb - M);  // Nb - t + 1
      float* dst = a.out + size_t(p) * a.out_plane + size_t(r0) * a.out_ld;
      if (a.out_vec2 && N % 2 == 0) {
        // consecutive threads read consecutive 16-byte chunks (conflict-free shared loads):
        // chunk f holds rows 2c, 2c+1 of column n (f = n * RPC/2 + c); each store instruction
        // still writes 128-byte runs of two rows
        constexpr int CH = RPC / 2;
        const int nf = (N / 2) * CH;
        for (int f = threadIdx.x; f < nf; f += NT) {
          const int n = f / CH, s2 = 2 * (f - n * CH);
          const float4 z = reinterpret_cast<const float4*>(cur)[f];
          if (s2 < nrows) __stcs(reinterpret_cast<float2*>(dst + size_t(s2) * a.out_ld) + n, make_float2(z.x, z.y));
          if (s2 + 1 < nrows)
            __stcs(reinterpret_cast<float2*>(dst + size_t(s2 + 1) * a.out_ld) + n, make_float2(z.z, z.w));
        }
      } else {
        for (int s = 0; s < nrows; ++s)
          for (int n = threadIdx.x; n < N; n += NT) {
            const float2 z = cur[(n >> 1) * RPC + s];
            __stcs(dst + size_t(s) * a.out_ld + n, (n & 1) ? z.y : z.x);
          }
      }
    }
    __syncthreads();
    tile = ctr ? s_next[it & 1] : tile + gridDim.x;
  }
  if constexpr (!TMA) cp_async_wait<0>();
}

// --------------------------------------------- Wiener filter tables (per slot)
// S[f][v][a] = sum_b w[a][b] exp(-2 pi i v b / Gc)  (FP64)
__global__ void k_wiener_s(DeblurArgs a, int frames) {
  pdl_enter();
  const int f = blockIdx.y;
  const cbp_kernel_slot* slot = a.slot + f;
  if (slot->status != 0) return;
  const int t = slot->width;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= a.Hc * t) return;
  const int v = idx / t, ai = idx - v * t;
  double re = 0.0, im = 0.0;
  // powers of W_Gc^v by recurrence from one sincos (drift ~t ulp, far below the FP32 table)
  const double2 wv = zroot(v, a.Gc);
  double2 p = make_double2(1.0, 0.0);
  for (int bj = 0; bj < t; ++bj) {
    const double w = slot->weights[ai * t + bj];
    re = fma(w, p.x, re);
    im = fma(w, p.y, im);
    p = zmul(p, wv);
  }
  a.S[size_t(f) * a.s_frame + idx] = make_double2(re, im);
}

// H[f][u][v] = conj(K)/(|K|^2 + eps) / (Gr*Gc), K(u,v) = sum_a S[v][a] exp(-2 pi i u a / Gr)
// in FP64 (decoder.cpp:209-211, fft.cpp:268). A thread owns WH_U table slots (rows u, at a
// stride of the block size so stores stay coalesced) and WH_V consecutive v: per tap a it
// reads WH_V values of S (shared-memory broadcasts) and updates WH_U x WH_V accumulators,
// the powers of W_Gr^u advancing by one complex product per slot (recurrence from one
// sincos; drift ~t ulp, far below the float2 the table is stored in).
// grid (ceil(Gr / (128 WH_U)), ceil(Hc / WH_V), frames).
#ifndef CBP_WH_V
#define CBP_WH_V 8
#endif
#ifndef CBP_WH_U
#define CBP_WH_U 1
#endif
constexpr int WH_V = CBP_WH_V, WH_U = CBP_WH_U;
__global__ void __launch_bounds__(128) k_wiener_h(DeblurArgs a, int frames) {
  __shared__ double2 Ss[WH_V * CBP_MAX_WIDTH];
  pdl_enter();
  const int f = blockIdx.z;
  const cbp_kernel_slot* slot = a.slot + f;
  if (slot->status != 0) return;
  const int t = slot->width;
  const int v0 = blockIdx.y * WH_V;
  const double2* S = a.S + size_t(f) * a.s_frame;
  for (int i = threadIdx.x; i < WH_V * t; i += blockDim.x) {
    const int vv = i / t, ai = i - vv * t;
    Ss[ai * WH_V + vv] = v0 + vv < a.Hc ? S[size_t(v0 + vv) * t + ai] : make_double2(0.0, 0.0);
  }
  __syncthreads();
  // thread = table slots su (consecutive threads, consecutive addresses); u = the row whose
  // filter value the column plan expects there (inverse of a.hpos, stored after it)
  const int su0 = blockIdx.x * blockDim.x * WH_U + threadIdx.x;
  if (su0 >= a.Gr) return;
  double2 wu[WH_U], w[WH_U];
  bool live[WH_U];
#pragma unroll
  for (int k = 0; k < WH_U; ++k) {
    const int su = su0 + k * blockDim.x;
    live[k] = su < a.Gr;
    const int u = live[k] ? (a.hpos ? int(a.hpos[a.Gr + su]) : su) : 0;
    wu[k] = zroot(u, a.Gr);
    w[k] = make_double2(1.0, 0.0);
  }
  double2 acc[WH_U][WH_V];
#pragma unroll
  for (int k = 0; k < WH_U; ++k)
#pragma unroll
    for (int vv = 0; vv < WH_V; ++vv) acc[k][vv] = make_double2(0.0, 0.0);
  for (int ai = 0; ai < t; ++ai) {
    double2 sv[WH_V];
#pragma unroll
    for (int vv = 0; vv < WH_V; ++vv) sv[vv] = Ss[ai * WH_V + vv];
#pragma unroll
    for (int k = 0; k < WH_U; ++k) {
#pragma unroll
      for (int vv = 0; vv < WH_V; ++vv) acc[k][vv] = zadd(acc[k][vv], zmul(sv[vv], w[k]));
      w[k] = zmul(w[k], wu[k]);
    }
  }
  const double sc = 1.0 / (double(a.Gr) * double(a.Gc));
  const double eps = slot->epsilon;
  // transposed table HT[v][slot(u)]: slot(u) = pos(u) of the column plan (a.hpos), so pass B
  // multiplies element-wise in its DIF output order
#pragma unroll
  for (int k = 0; k < WH_U; ++k) {
    if (!live[k]) continue;
    float2* H = a.H + size_t(f) * a.h_frame + su0 + k * blockDim.x;
#pragma unroll
    for (int vv = 0; vv < WH_V; ++vv) {
      const int v = v0 + vv;
      if (v < a.Hc) {
        // reciprocal by MUFU seed + two Newton steps (~1 ulp; the table is stored in FP32)
        // instead of an IEEE division per entry, which dominated the kernel's instructions
        const double den = acc[k][vv].x * acc[k][vv].x + acc[k][vv].y * acc[k][vv].y + eps;
        double r;
        asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(den));
        r = fma(r, fma(-den, r, 1.0), r);
        r = fma(r, fma(-den, r, 1.0), r);
        const double g = sc * r;
        H[size_t(v) * a.hp] = make_float2(float(acc[k][vv].x * g), float(-acc[k][vv].y * g));
      }
    }
  }
}

cudaError_t launch_wiener_tables(const DeblurArgs& a, int frames, cudaStream_t s) {
  dim3 g1((a.Hc * CBP_MAX_WIDTH + 255) / 256, frames);
  launch_chain(k_wiener_s, a.chain != 0, g1, dim3(256), 0, s, a, frames);
  dim3 g2((a.Gr + 128 * WH_U - 1) / (128 * WH_U), (a.Hc + WH_V - 1) / WH_V, frames);
  launch_chain(k_wiener_h, a.chain != 0, g2, dim3(128), 0, s, a, frames);
  return cudaGetLastError();
}

// --------------------------------------------------------------- dispatch
// Persistent grid: resident CTAs per SM x (SMs - a.sm_reserve). The reserve leaves whole
// SMs to kernels of other streams (cbp_set_sm_reserve: the recovery chain of the next
// epoch overlaps the deconvolution in the video pipelines).
template <class K>
int resident_per_sm(K kernel, int nt, size_t smem) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, nt, smem);
  return per_sm < 1 ? 1 : per_sm;
}
__host__ inline int persistent_grid(int per_sm, int sms, int reserve, int total) {
  const int g = (sms - (reserve > 0 && reserve < sms ? reserve : 0)) * per_sm;
  return total < g ? total : g;
}

// Tensor map for pass C's tile loads: XT viewed as (u, d_1, ..., d_m, plane) with frequency
// k = sum_i d_i N/(R_1...R_i), i.e. the slot order of the DIT input; box (RPC, R_1, ..., R_m, 1).
static PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &f, 12000, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }();
  return fn;
}

bool ct_radices(int n, bool column, std::vector<int>& r);

template <class P>
bool rows_inverse_tmap(const DeblurArgs& a, int planes, CUtensorMap* map) {
  std::vector<int> rad;
  ct_radices(P::L, false, rad);
  auto enc = tmap_encoder();
  if (!enc || rad.size() + 2 > 5 || (a.xp * 8) % 16 || (size_t(a.x_plane) * 8) % 16 ||
      reinterpret_cast<uintptr_t>(a.X) % 16)
    return false;
  cuuint64_t dims[5], strides[4];
  cuuint32_t box[5], estr[5];
  const int rank = int(rad.size()) + 2;
  dims[0] = cuuint64_t(a.Mb);
  box[0] = P::RPC;
  size_t step = P::L;  // frequency stride of digit i: N / (R_1 ... R_i)
  for (size_t i = 0; i < rad.size(); ++i) {
    step /= rad[i];
    dims[i + 1] = cuuint64_t(rad[i]);
    box[i + 1] = cuuint32_t(rad[i]);
    strides[i] = cuuint64_t(step * a.xp * 8);
  }
  dims[rank - 1] = cuuint64_t(planes);
  box[rank - 1] = 1;
  strides[rank - 2] = cuuint64_t(size_t(a.x_plane) * 8);
  for (int i = 0; i < rank; ++i) estr[i] = 1;
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, cuuint32_t(rank), const_cast<float2*>(a.X), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <class P>
void launch_rows(const DeblurArgs& a, int planes, bool inverse, cudaStream_t s) {
  constexpr int NB = P::PIPE ? 2 : 1;
  const size_t smA = NB * size_t(P::RPC) * P::SPA * sizeof(float2) +
                     (P::RTW ? size_t(P::TWN) * sizeof(float2) : P::L * sizeof(short));
  const size_t smC = NB * size_t(((P::L + 1) * P::RPC + 15) & ~15) * sizeof(float2) +
                     size_t(P::RTW ? P::TWN : (P::L + 3) / 4) * sizeof(float2) + 3 * sizeof(unsigned long long);
  // per-device launch configuration, set up once per device (thread-safe: call_once)
  struct Cfg {
    int pA = 0, pC = 0, pAb = 0, pCt = 0, sms = 0;
  };
  static Cfg cfgs[kMaxDevices];
  Cfg& c = cfgs[current_device()];
  constexpr bool kBulk = P::PIPE && P::L % 2 == 0;
  CBP_ONCE_PER_DEVICE({
    cudaDeviceGetAttribute(&c.sms, cudaDevAttrMultiProcessorCount, current_device());
    cudaFuncSetAttribute(k_rows_forward_ct<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smA));
    cudaFuncSetAttribute(k_rows_inverse_ct<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smC));
    c.pA = resident_per_sm(k_rows_forward_ct<P>, P::NT, smA);
    c.pC = resident_per_sm(k_rows_inverse_ct<P>, P::NT, smC);
    if constexpr (kBulk) {
      cudaFuncSetAttribute(k_rows_forward_ct<P, kBulk>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smA));
      c.pAb = resident_per_sm(k_rows_forward_ct<P, kBulk>, P::NT, smA);
    }
    if constexpr (P::PIPE) {
      cudaFuncSetAttribute(k_rows_inverse_ct<P, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smC));
      c.pCt = resident_per_sm(k_rows_inverse_ct<P, true>, P::NT, smC);
    }
  });
  const int pA = c.pA, pC = c.pC, pAb = c.pAb, pCt = c.pCt, sms = c.sms;
  (void)pAb;
  (void)pCt;
  const int total = planes * ((a.Mb + P::RPC - 1) / P::RPC);
  if (inverse) {
    CUtensorMap map;
    if constexpr (P::PIPE) {
      static const bool tma = !getenv("CBP_NO_BULK");
      if (tma && rows_inverse_tmap<P>(a, planes, &map)) {
        k_rows_inverse_ct<P, true><<<persistent_grid(pCt, sms, a.sm_reserve, total), P::NT, smC, s>>>(a, planes, map);
        return;
      }
    }
    memset(&map, 0, sizeof(map));
    k_rows_inverse_ct<P><<<P::PIPE ? persistent_grid(pC, sms, a.sm_reserve, total) : total, P::NT, smC, s>>>(a, planes,
                                                                                                              map);
    return;
  }
  if constexpr (kBulk) {
    static const bool bulk = !getenv("CBP_NO_BULK");
    // 16-byte aligned rows whose pitch holds Nb rounded up to 4 floats
    if (bulk && a.in_vec4 && a.in_ld >= ((a.Nb + 3) & ~3)) {
      k_rows_forward_ct<P, kBulk><<<persistent_grid(pAb, sms, a.sm_reserve, total), P::NT, smA, s>>>(a, planes);
      return;
    }
  }
  k_rows_forward_ct<P><<<P::PIPE ? persistent_grid(pA, sms, a.sm_reserve, total) : total, P::NT, smA, s>>>(a, planes);
}

template <class P>
void launch_cols(const DeblurArgs& a, int planes, cudaStream_t s) {
  constexpr int GP = ((P::G + 11) / 16) * 16 + 4;
  const size_t sm = ((P::PIPE ? 2 : 1) + (P::HD ? 0 : 1)) * size_t(GP) * P::W * sizeof(float2);
  struct Cfg {
    int pB = 0, pT = 0, sms = 0;
  };
  static Cfg cfgs[kMaxDevices];
  Cfg& c = cfgs[current_device()];
  CBP_ONCE_PER_DEVICE({
    cudaDeviceGetAttribute(&c.sms, cudaDevAttrMultiProcessorCount, current_device());
    cudaFuncSetAttribute(k_cols_filter_ct<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
    c.pB = resident_per_sm(k_cols_filter_ct<P>, P::NT, sm);
    if constexpr (P::PIPE) {
      cudaFuncSetAttribute(k_cols_filter_bulk<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
      c.pT = resident_per_sm(k_cols_filter_bulk<P>, P::NT, sm);
    }
  });
  const int pB = c.pB, pT = c.pT, sms = c.sms;
  (void)pT;
  const int total = planes * ((a.Hc + P::W - 1) / P::W);
  if constexpr (P::PIPE) {
    static const bool bulk = !getenv("CBP_NO_BULK");
    // column runs of Mb complex values are 16-byte multiples; HD reads a butterfly-major H
    if (bulk && a.Mb % 2 == 0 && (!P::HD || a.h_bmajor)) {
      k_cols_filter_bulk<P><<<persistent_grid(pT, sms, a.sm_reserve, total), P::NT, sm, s>>>(a, planes);
      return;
    }
  }
  k_cols_filter_ct<P><<<P::PIPE ? persistent_grid(pB, sms, a.sm_reserve, total) : total, P::NT, sm, s>>>(a, planes);
}

// Radix plans in DIT order; the first (contiguous-butterfly) radix is odd so its strided
// shared-memory accesses are bank-conflict free. Large radices run in registers.
#ifndef CBP_RTW972
#define CBP_RTW972 1
#endif
using Row972 = RowPlan<972, 4, Radices<27, 36>, 160, true, 3, CBP_RTW972>;  // 1080p: Gc = 1944
using Row972a = RowPlan<972, 4, Radices<27, 36>, 160, true, 1>;
using Row972c = RowPlan<972, 4, Radices<27, 36>, 160, false, 4>;
#ifndef CBP_ROW1944_RPC
#define CBP_ROW1944_RPC 4
#endif
// 4K: Gc = 3888. Four rows per tile (one CTA of 512 threads per SM): a tile then writes whole
// 32-byte XT sectors (4 rows of one frequency); with two rows per tile every pass-A store was
// a half sector (pass A 41.4 -> 26.8 us per 4K plane)
#ifndef CBP_ROW1944_NT
#define CBP_ROW1944_NT (CBP_ROW1944_RPC == 4 ? 512 : 256)
#endif
#ifndef CBP_ROW1944_PIPE
#define CBP_ROW1944_PIPE true
#endif
#ifndef CBP_ROW1944_MINB
#define CBP_ROW1944_MINB 1
#endif
#ifndef CBP_ROW1944_RTW
#define CBP_ROW1944_RTW false
#endif
// radices (27, 9, 8): the last radix 8 makes the digit-reversal stride N/8 = 243 odd, so the
// split steps' pos(k) accesses of consecutive frequencies spread over the banks (with
// (27, 8, 9) the stride 216 put every fourth frequency on one bank: 45% of the passes' shared
// wavefronts were conflicts)
using Row1944 = RowPlan<1944, CBP_ROW1944_RPC, Radices<27, 9, 8>, CBP_ROW1944_NT, CBP_ROW1944_PIPE, CBP_ROW1944_MINB,
                        CBP_ROW1944_RTW>;
#ifndef CBP_C2_ROWS
#define CBP_C2_ROWS 0
#endif
#if CBP_C2_ROWS == 1
using Row324 = RowPlan<324, 8, Radices<27, 12>, 96, true, 4, true>;
#elif CBP_C2_ROWS == 2
using Row324 = RowPlan<324, 8, Radices<27, 12>, 128, true, 3, true>;
#elif CBP_C2_ROWS == 3
using Row324 = RowPlan<324, 4, Radices<27, 12>, 64, true, 6, true>;
#elif CBP_C2_ROWS == 4
using Row324 = RowPlan<324, 8, Radices<27, 12>, 224>;
#else
// 640x480: Gc = 648. 8 rows per tile on 3 warps (the 96 radix-27 butterflies of a tile, one
// per thread), 3 CTAs per SM, stage twiddles in shared memory: 0.67 -> 0.55 us (A) and
// 0.66 -> 0.50 us (C) per plane against 7 warps per tile, 1 CTA per SM
using Row324 = RowPlan<324, 8, Radices<27, 12>, 96, true, 3, true>;
#endif
using Row135 = RowPlan<135, 8, Radices<27, 5>, 224>;       // 256x256: Gc = 270
using Col1120 = ColPlan<1120, 4, Radices<35, 32>, 160, true, 3, true>;  // 1080p: Gr = 1120, filter from L2
using Col1120a = ColPlan<1120, 4, Radices<35, 32>, 160, true, 2>;        // staged filter strip
using Col1120c = ColPlan<1120, 4, Radices<35, 32>, 160, false, 4, true>;
#ifndef CBP_COL2187_W
#define CBP_COL2187_W 2
#endif
#ifndef CBP_COL2187_NT
#define CBP_COL2187_NT 256
#endif
#ifndef CBP_COL2187_MINB
#define CBP_COL2187_MINB 1
#endif
#ifndef CBP_COL2187_HD
#define CBP_COL2187_HD false
#endif
using Col2187 = ColPlan<2187, CBP_COL2187_W, Radices<27, 9, 9>, CBP_COL2187_NT, true, CBP_COL2187_MINB,
                        CBP_COL2187_HD>;  // 4K: Gr = 2187
#ifndef CBP_C2_COLS
#define CBP_C2_COLS 0
#endif
#if CBP_C2_COLS == 1
using Col490 = ColPlan<490, 8, Radices<35, 14>, 288, true, 2>;
#elif CBP_C2_COLS == 2
using Col490 = ColPlan<490, 8, Radices<35, 14>, 160, true, 3, true>;
#elif CBP_C2_COLS == 3
using Col490 = ColPlan<490, 8, Radices<35, 14>, 128, true, 3>;
#elif CBP_C2_COLS == 4
using Col490 = ColPlan<490, 8, Radices<14, 35>, 288, true, 2>;
#else
// 640x480: Gr = 490. 8 columns per strip on 4 warps (the 112 radix-35 butterflies of the
// fused filter stage fit one round), filter read from L2, 3 CTAs per SM: 0.91 -> 0.82 us per
// plane against 9 warps per strip, 2 CTAs per SM with a staged filter strip
using Col490 = ColPlan<490, 8, Radices<35, 14>, 128, true, 3, true>;
#endif
using Col270 = ColPlan<270, 8, Radices<27, 10>, 224>;      // 256x256: Gr = 270

// Radix plans of the specialisations above (host mirror; DIT stage order).
bool ct_radices(int n, bool column, std::vector<int>& r) {
  if (column) {
    switch (n) {
      case 1120: r = {35, 32}; return true;
      case 2187: r = {27, 9, 9}; return true;
      case 490:
        if (CBP_C2_COLS == 4) r = {14, 35};
        else r = {35, 14};
        return true;
      case 270: r = {27, 10}; return true;
    }
    return false;
  }
  switch (n) {
    case 972: r = {27, 36}; return true;
    case 1944: r = {27, 9, 8}; return true;
    case 324: r = {27, 12}; return true;
    case 135: r = {27, 5}; return true;
  }
  return false;
}

// digit-reversal slot of element n for a radix list (host mirror of Pos<>::get)
int ct_pos(const std::vector<int>& rad, int n) {
  int pos = 0, N = 1;
  for (int r : rad) N *= r;
  for (size_t m = rad.size(); m-- > 0;) {  // Pos<R_1..R_m>: last radix first
    const int r = rad[m];
    N /= r;
    pos += (n % r) * N;
    n /= r;
  }
  return pos;
}

bool deblur_has_ct(int Gr, int Gc, int pass) {
  if (pass == 1) return Gr == 1120 || Gr == 2187 || Gr == 490 || Gr == 270;
  if (Gc % 2) return false;
  const int L = Gc / 2;
  return L == 972 || L == 1944 || L == 324 || L == 135;
}

bool launch_deblur_pass_ct(const DeblurArgs& a, int planes, int pass, cudaStream_t s) {
  if (!deblur_has_ct(a.Gr, a.Gc, pass)) return false;
  if (pass == 0 && !a.in_vec2) return false;  // cp.async 8-byte copies need aligned rows
  if (pass == 1) {
    if (!a.H || !a.twst_col) return false;
    switch (a.Gr) {
      case 1120:
        if (a.variant == 1) launch_cols<Col1120a>(a, planes, s);
        else if (a.variant == 3) launch_cols<Col1120c>(a, planes, s);
        else launch_cols<Col1120>(a, planes, s);
        return true;
      case 2187: launch_cols<Col2187>(a, planes, s); return true;
      case 490: launch_cols<Col490>(a, planes, s); return true;
      case 270: launch_cols<Col270>(a, planes, s); return true;
    }
    return false;
  }
  if (!a.twst_row) return false;
  const bool inv = pass == 2;
  switch (a.Gc / 2) {
    case 972:
      if (a.variant == 1) launch_rows<Row972a>(a, planes, inv, s);
      else if (a.variant == 3) launch_rows<Row972c>(a, planes, inv, s);
      else launch_rows<Row972>(a, planes, inv, s);
      return true;
    case 1944: launch_rows<Row1944>(a, planes, inv, s); return true;
    case 324: launch_rows<Row324>(a, planes, inv, s); return true;
    case 135: launch_rows<Row135>(a, planes, inv, s); return true;
  }
  return false;
}


// ------------------------------------------------ fused persistent deconvolution
// One persistent launch runs passes A, B and C of a whole batch, each SM in one role: the
// first CTA to start on an SM claims a role for the SM (A, B, C in a 4:5:4 pattern, the
// passes' relative costs), so an SM only ever runs one pass's code (one pass's instruction
// stream stays in the SM's instruction cache; the union of the three thrashed it) and the
// row roles keep their twiddles in shared memory. Each role takes its items (A and C: row
// tiles, B: column strips) in plane order from its own queue; an item waits for its
// producer plane's completion counter (B(p): all A(p) tiles; C(p): all B(p) strips; A(p):
// all C(p - ring) tiles, whose spectrum slot it reuses). Deadlock-free while every role has
// a running CTA (the first three SMs take A, B, C): the oldest unfinished plane-pass is
// always ready and at the head of its queue. The half spectrum lives in a ring of `ring`
// plane slots (ring x 8.5 MB at 1080p), so it stays L2-resident between the passes.
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;\n" ::: "memory");
}
// the producers of plane p for a role-`role` item have completed (writes visible to TMA)
__device__ __forceinline__ bool fused_ready(const FusedCtl& f, int role, int p) {
  bool ok = true;
  if (role == 0) ok = p < f.ring || ld_acquire(f.done + 2 * f.planes + p - f.ring) >= unsigned(f.nC);
  else if (role == 1) ok = ld_acquire(f.done + p) >= unsigned(f.nA);
  else ok = ld_acquire(f.done + f.planes + p) >= unsigned(f.nB);
  if (ok) fence_proxy_async_global();
  return ok;
}
__device__ __forceinline__ void fused_publish(const FusedCtl& f, int role, int p) {
  fence_proxy_async_global();
  __threadfence();
  atomicAdd(f.done + role * f.planes + p, 1u);
}

template <class PR, class PC>
struct FusedPlan {
  static_assert(PR::NT == PC::NT, "one CTA shape for all three passes");
  static constexpr int NT = PR::NT;
  static constexpr int L = PR::L, RPC = PR::RPC, SPA = PR::SPA;
  static constexpr int G = PC::G, W = PC::W, GP = ((G + 11) / 16) * 16 + 4;
  static constexpr int TILE_A = RPC * SPA, TILE_B = GP * W, TILE_C = ((L + 1) * RPC + 15) & ~15;
  static constexpr int BUFR = ((TILE_A > TILE_C ? TILE_A : TILE_C) + 15) & ~15;  // rows: 128-byte multiple
  static constexpr int BUFB = (TILE_B + 15) & ~15;
  static constexpr int TWN = L / 2 + 1 + TwUsed<L, typename PR::R>::count;  // staged row twiddles
  static constexpr int ROWS_F2 = 2 * BUFR + TWN, COLS_F2 = 2 * BUFB;
  static constexpr int F2 = ROWS_F2 > COLS_F2 ? ROWS_F2 : COLS_F2;
  static constexpr size_t SMEM = size_t(F2) * sizeof(float2) + 64;  // + 2 mbarriers, role
};

template <class PR, class PC>
__global__ void __launch_bounds__(PR::NT, PR::MINB) k_deblur_fused(DeblurArgs a, FusedCtl f,
                                                                   const __grid_constant__ CUtensorMap tmap) {
  using FP = FusedPlan<PR, PC>;
  constexpr int NT = FP::NT, L = FP::L, RPC = FP::RPC, SPA = FP::SPA;
  constexpr int W = FP::W, GP = FP::GP;
  using RR = typename PR::R;
  using RC = typename PC::R;
  using FFTA = FftIP<L, RPC, SPA, 1, NT, false, true>;
  using FFTB = FftIP<FP::G, W, GP, 1, NT, false>;
  using FFTC = FftIP<L, RPC, 1, RPC, NT, true, true>;
  constexpr int NRAD = RadixCount<RR>::value;
  extern __shared__ __align__(128) float2 smf[];
  // barriers and broadcast slots in dynamic shared memory: static shared variables would
  // shift the dynamic region off the 128-byte alignment the tensor copies need
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(smf + FP::F2);
  int* s_role = reinterpret_cast<int*>(bar + 2);
  unsigned* s_item = reinterpret_cast<unsigned*>(bar + 3);
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_init_fence();
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    volatile int* slot = f.sm_role + (smid % unsigned(f.nsm));
    const int old = atomicCAS(f.sm_role + (smid % unsigned(f.nsm)), -1, -2);
    int role;
    if (old == -1) {  // first CTA on this SM: A, B, C, A, B, C, A, B, C, A, B, C, B
      const unsigned k = atomicAdd(f.ticket + 3, 1u) % 13u;
      role = k == 12 ? 1 : int(k % 3);
      __threadfence();
      *slot = role;
    } else {
      role = old;
      while (role < 0) role = *slot;
    }
    *s_role = role;
  }
  __syncthreads();
  const int role = *s_role;
  const int BUF = role == 1 ? FP::BUFB : FP::BUFR;
  const int nper = role == 0 ? f.nA : (role == 1 ? f.nB : f.nC);
  const unsigned total = unsigned(nper) * unsigned(f.planes);
  // row roles: split and stage twiddles in shared memory (RTW), after the two tile buffers
  const float2* twst = a.twst_row;
  const float2* twp = a.tw_post;
  if (role != 1) {
    float2* tws = smf + 2 * FP::BUFR;
    twst = stage_row_twiddles<PR>(a, tws);
    twp = tws;
  }
  const unsigned row_bytes = unsigned((a.Nb + 3) & ~3) * 4u;
  auto xt = [&](int p) { return a.X + size_t(p % f.ring) * a.x_plane; };
  auto rows_of = [&](int p) {
    const cbp_kernel_slot* sl = plane_slot(a, p);
    return sl->status == 0 ? a.Mb - sl->width + 1 : 0;
  };
  // thread 0: loads of item (p, idx) of this role into buffer b (its producers completed)
  auto issue = [&](int p, int idx, int b) {
    float2* dst = smf + b * BUF;
    unsigned long long* mb = &bar[b];
    fence_proxy_async();
    if (role == 0) {
      const int r0 = idx * RPC;
      const float* src = a.in + size_t(p) * a.in_plane + size_t(r0) * a.in_ld;
      const int nr = min(RPC, a.Mb - r0);
      mbar_expect_tx(mb, unsigned(nr) * row_bytes);
      for (int s = 0; s < nr; ++s) bulk_g2s(dst + s * SPA, src + size_t(s) * a.in_ld, row_bytes, mb);
    } else if (role == 1) {
      const int v0 = idx * W, nc = min(W, a.Hc - v0);
      const float2* XT = xt(p);
      mbar_expect_tx(mb, unsigned(nc) * unsigned(a.Mb) * 8u);
      for (int s = 0; s < nc; ++s) bulk_g2s(dst + s * GP, XT + size_t(v0 + s) * a.xp, unsigned(a.Mb) * 8u, mb);
    } else {
      const int r0 = idx * RPC, slot = p % f.ring;
      const unsigned tail = unsigned(min(RPC, a.xp - r0)) * 8u;
      mbar_expect_tx(mb, unsigned(RPC) * L * 8u + tail);
      const unsigned d = smem_u32(dst), bb = smem_u32(mb);
      const unsigned long long tm = reinterpret_cast<unsigned long long>(&tmap);
      if constexpr (NRAD == 2)
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];\n"
            ::"r"(d), "l"(tm), "r"(r0), "r"(0), "r"(0), "r"(slot), "r"(bb) : "memory");
      else
        asm volatile(
            "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];\n"
            ::"r"(d), "l"(tm), "r"(r0), "r"(0), "r"(0), "r"(0), "r"(slot), "r"(bb) : "memory");
      bulk_g2s(dst + L * RPC, xt(p) + size_t(L) * a.xp + r0, tail, mb);
    }
  };
  // thread 0 state: the plane of a pass-B strip whose bulk stores are not yet published
  int pend_b = -1;
  auto flush_b = [&](int keep) {
    if (pend_b < 0) return;
    if (keep) asm volatile("cp.async.bulk.wait_group 1;\n" ::: "memory");
    else bulk_wait_all();
    fused_publish(f, 1, pend_b);
    pend_b = -1;
  };
  unsigned cur = 0;
  if (threadIdx.x == 0) {
    cur = atomicAdd(f.ticket + role, 1u);
    if (cur < total) {
      while (!fused_ready(f, role, int(cur / nper))) __nanosleep(256);
      issue(int(cur / nper), int(cur % nper), 0);
    }
    *s_item = cur;
  }
  __syncthreads();
  cur = *s_item;
  unsigned ph = 0u;  // mbarrier phase bits of buffers 0, 1
  for (int it = 0; cur < total; ++it) {
    const int cb = it & 1;
    float2* buf = smf + cb * BUF;
    unsigned nxt = total;
    bool issued = false;
    if (threadIdx.x == 0) {
      nxt = atomicAdd(f.ticket + role, 1u);
      if (nxt < total && fused_ready(f, role, int(nxt / nper))) {
        bulk_wait_read();  // the other buffer's bulk stores (a pass-B strip) have left shared memory
        issue(int(nxt / nper), int(nxt % nper), cb ^ 1);
        issued = true;
      }
    }
    mbar_wait(&bar[cb], (ph >> cb) & 1u);  // every thread observes the tile's arrival
    ph ^= 1u << cb;
    const int p = int(cur / nper), idx = int(cur % nper);
    int b_commit = 0;  // thread 0: this item committed a bulk-store group
    if (role == 0) {
      // ---- pass A: forward row FFTs of RPC rows, r2c split into XT (see k_rows_forward_ct)
      FFTA::template dif_masked<false>(buf, twst, a.Nb, RR{});
      const int r0 = idx * RPC;
      float2* XT = xt(p) + r0;
      const int nrows = min(RPC, a.Mb - r0);
      constexpr int NPAIR = L / 2 + 1, HALF = RPC / 2;
#pragma unroll 1
      for (int q = threadIdx.x; q < NPAIR * HALF; q += NT) {
        const int k = q / HALF, j = q - k * HALF;
        if (2 * j >= nrows) continue;
        const int pk = Pos<RR>::get(k), pc = Pos<RR>::get(k == 0 ? 0 : L - k);
        const float2 w = twp[k];
        float2 xk[2], xc[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const float2* z = buf + (2 * j + h) * SPA;
          const float2 zk = z[pk], zc = cconj(z[pc]);
          const float2 e = cscale(cadd(zk, zc), 0.5f);
          const float2 d = csub(zk, zc);
          const float2 wo = cmul(w, make_float2(0.5f * d.y, -0.5f * d.x));
          xk[h] = cadd(e, wo);
          xc[h] = cconj(csub(e, wo));
        }
        float2* dk = XT + size_t(k) * a.xp + 2 * j;
        float2* dc = XT + size_t(L - k) * a.xp + 2 * j;
        if (2 * j + 1 < nrows) {
          *reinterpret_cast<float4*>(dk) = make_float4(xk[0].x, xk[0].y, xk[1].x, xk[1].y);
          if (L - k != k) *reinterpret_cast<float4*>(dc) = make_float4(xc[0].x, xc[0].y, xc[1].x, xc[1].y);
        } else {
          dk[0] = xk[0];
          if (L - k != k) dc[0] = xc[0];
        }
      }
    } else if (role == 1) {
      // ---- pass B: column DIF, fused filter stage (H from L2), DIT (see k_cols_filter_bulk)
      const int v0 = idx * W, nc = min(W, a.Hc - v0);
      const int fs = deblur_slot_index(a, p);
      const cbp_kernel_slot* slot = a.slot + fs;
      if (slot->status == 0) {  // uniform over the CTA
        const int t = slot->width;
        FFTB::dif_head_masked(buf, a.twst_col, 2 * a.Mb, RC{});
        FFTB::filter_stage_g(buf, a.H + size_t(fs) * a.h_frame + size_t(v0) * a.hp, a.hp, nc, RC{});
        FFTB::template dit_tail<true>(buf, a.twst_col, RC{});  // every writer fences before the last barrier
        if (threadIdx.x == 0) {
          const int M = a.Mb - t + 1;  // even: Mb even, t odd
          float2* XT = xt(p);
          for (int s2 = 0; s2 < nc; ++s2) bulk_s2g(XT + size_t(v0 + s2) * a.xp, buf + s2 * GP, unsigned(M) * 8u);
          bulk_commit();
          b_commit = 1;
        }
      }
    } else {
      // ---- pass C: c2r split, inverse row DIT, crop (see k_rows_inverse_ct)
      const int r0 = idx * RPC;
      const int M = rows_of(p);
      const int nrows = min(RPC, M - r0);
      if (nrows > 0) {
        constexpr int NP = L / 2 + 1, HALF = RPC / 2;
#pragma unroll 1
        for (int q = threadIdx.x; q < NP * HALF; q += NT) {
          const int k = q / HALF, j = q - k * HALF;
          float4* pa = reinterpret_cast<float4*>(buf + Pos<RR>::get(k) * RPC + 2 * j);
          float4* pb = reinterpret_cast<float4*>(buf + (k == 0 ? L : Pos<RR>::get(L - k)) * RPC + 2 * j);
          const float4 A4 = *pa, B4 = *pb;
          const float2 w = cconj(twp[k]);
          const float2 wm = make_float2(-w.x, w.y);
          float2 r1[2], r2[2];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const float2 A = h ? make_float2(A4.z, A4.w) : make_float2(A4.x, A4.y);
            const float2 B = h ? make_float2(B4.z, B4.w) : make_float2(B4.x, B4.y);
            const float2 e1 = cadd(A, cconj(B));
            const float2 o1 = cmul(csub(A, cconj(B)), w);
            r1[h] = make_float2(e1.x - o1.y, e1.y + o1.x);
            const float2 e2 = cadd(B, cconj(A));
            const float2 o2 = cmul(csub(B, cconj(A)), wm);
            r2[h] = make_float2(e2.x - o2.y, e2.y + o2.x);
          }
          *pa = make_float4(r1[0].x, r1[0].y, r1[1].x, r1[1].y);
          if (k != 0 && 2 * k != L) *pb = make_float4(r2[0].x, r2[0].y, r2[1].x, r2[1].y);
        }
        __syncthreads();
        FFTC::template dit<true>(buf, twst, RR{});
        const int N = a.Nb - (a.Mb - M);
        float* dst = a.out + size_t(p) * a.out_plane + size_t(r0) * a.out_ld;
        if (a.out_vec2 && N % 2 == 0) {
          constexpr int CH = RPC / 2;
          const int nf = (N / 2) * CH;
          for (int q = threadIdx.x; q < nf; q += NT) {
            const int n = q / CH, s2 = 2 * (q - n * CH);
            const float4 z = reinterpret_cast<const float4*>(buf)[q];
            if (s2 < nrows) __stcs(reinterpret_cast<float2*>(dst + size_t(s2) * a.out_ld) + n, make_float2(z.x, z.y));
            if (s2 + 1 < nrows)
              __stcs(reinterpret_cast<float2*>(dst + size_t(s2 + 1) * a.out_ld) + n, make_float2(z.z, z.w));
          }
        } else {
          for (int s2 = 0; s2 < nrows; ++s2)
            for (int n = threadIdx.x; n < N; n += NT) {
              const float2 z = buf[(n >> 1) * RPC + s2];
              __stcs(dst + size_t(s2) * a.out_ld + n, (n & 1) ? z.y : z.x);
            }
        }
      }
    }
    fence_proxy_async();  // shared-memory accesses of this item before the buffer's next bulk fill
    __syncthreads();      // all threads' stores of this item issued
    if (threadIdx.x == 0) {
      if (role == 1) {
        flush_b(b_commit);  // the previous strip's stores (this strip's own group may still run)
        pend_b = p;
      } else {
        fused_publish(f, role, p);
      }
      if (nxt < total && !issued) {
        flush_b(0);  // never wait while holding unpublished work
        while (!fused_ready(f, role, int(nxt / nper))) __nanosleep(128);
        bulk_wait_read();
        issue(int(nxt / nper), int(nxt % nper), cb ^ 1);
      }
      *s_item = nxt;
    }
    __syncthreads();
    cur = *s_item;
  }
  if (threadIdx.x == 0) flush_b(0);
}

template <class PR, class PC>
bool launch_fused_impl(const DeblurArgs& a, const FusedCtl& f, cudaStream_t s) {
  using FP = FusedPlan<PR, PC>;
  struct Cfg {
    int per_sm = 0, sms = 0;
  };
  static Cfg cfgs[kMaxDevices];
  Cfg& c = cfgs[current_device()];
  CBP_ONCE_PER_DEVICE({
    cudaDeviceGetAttribute(&c.sms, cudaDevAttrMultiProcessorCount, current_device());
    cudaFuncSetAttribute(k_deblur_fused<PR, PC>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(FP::SMEM));
    c.per_sm = resident_per_sm(k_deblur_fused<PR, PC>, FP::NT, FP::SMEM);
  });
  CUtensorMap map;
  if (!rows_inverse_tmap<PR>(a, f.ring, &map)) return false;
  const int grid = persistent_grid(c.per_sm, c.sms, a.sm_reserve, 1 << 30);
  k_deblur_fused<PR, PC><<<grid, FP::NT, FP::SMEM, s>>>(a, f, map);
  return true;
}

// Items per plane of the fused plan for this grid, or false if the grid has none.
bool deblur_fused_shape(const DeblurArgs& a, int& nA, int& nB, int& nC) {
  if (a.Gr == 1120 && a.Gc == 1944) {
    nA = nC = (a.Mb + Row972::RPC - 1) / Row972::RPC;
    nB = (a.Hc + Col1120::W - 1) / Col1120::W;
    return true;
  }
  return false;
}

bool launch_deblur_fused(const DeblurArgs& a, const FusedCtl& f, cudaStream_t s) {
  // bulk row loads need 16-byte rows with a pitch of Nb rounded to 4; bulk column copies an even Mb
  if (!a.in_vec4 || a.in_ld < ((a.Nb + 3) & ~3) || a.Mb % 2 || !a.h_bmajor || !a.H || !a.twst_col || !a.twst_row)
    return false;
  if (a.Gr == 1120 && a.Gc == 1944) return launch_fused_impl<Row972, Col1120>(a, f, s);
  return false;
}

}  // namespace cbp_dev
