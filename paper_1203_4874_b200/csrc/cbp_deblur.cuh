// Launch interface of the three-pass deconvolution (see cbp_deblur.cu).
#pragma once

#include <vector>

#include "cbp_fft.cuh"

namespace cbp_dev {

struct DeblurArgs {
  const float* in;  // blurred planes: plane p at in + p*in_plane, rows of in_ld floats
  size_t in_plane;
  int in_ld;
  float* out;  // latent planes
  size_t out_plane;
  int out_ld;
  float2* X;  // transposed half spectrum XT[v][u]: plane p at X + p*x_plane, column v at v*xp
  size_t x_plane;
  int xp;     // pitch of one spectrum column (>= Mb, multiple of 4)
  int Mb, Nb;       // blurred plane extent
  int Gr, Gc, Hc;   // grid and half-spectrum width Gc/2+1
  int even;         // Gc even: half-length complex row transform
  int rows_per_cta; // pass A/C rows per CTA
  int in_vec2;      // input rows 8-byte aligned (float2 loads)
  int out_vec2;     // output rows 8-byte aligned (float2 stores)
  int in_vec4;      // input rows 16-byte aligned (16-byte cp.async)
  int dbg;          // experiment switches (CBP_DEBLUR_DBG): 1 skip FFT stages, 2 skip filter
  int variant;      // kernel configuration variant (CBP_FFT_VARIANT), 0 = default
  int col_width;    // pass B columns per CTA
  int sm_reserve;   // SMs the persistent passes leave free (cbp_set_sm_reserve)
  int chain;        // programmatic dependent launch of the Wiener table kernels
  const cbp_kernel_slot* slot;
  int slot_per_frame;  // 1: slot[p / channels]; 0: slot[0] for every plane
  int channels;
  FftPlan plan_row;  // length Gc/2 (even) or Gc
  FftPlan plan_col;  // length Gr
  const float2* tw_row;   // exp(-2 pi i k / plan_row.n)
  const float2* tw_post;  // exp(-2 pi i k / Gc), k <= Gc/2
  const float2* tw_col;   // exp(-2 pi i k / Gr)
  const float2* twst_row; // per-stage twiddles of the specialised row plan (or null)
  const float2* twst_col; // per-stage twiddles of the specialised column plan (or null)
  double2* S;             // per-slot column kernel transforms S[v][a] (k_wiener_s)
  size_t s_frame;         // S stride per slot
  float2* H;              // per-slot Wiener filter HT[v][slot(u)] (pitch hp), scaled by 1/(Gr*Gc)
  size_t h_frame;         // H stride per slot
  int hp;                 // H column pitch (>= Gr, multiple of 4)
  const short* hpos;      // slot(u) of the column plan's DIF output, or null (natural order)
  unsigned* tile_ctr;     // 3 dynamic-tile counters (passes A, B, C), zeroed per launch group, or null
  int h_bmajor;           // hpos is butterfly-major (i*NB + b for slot b*R1 + i): bulk pass B reads H from L2
  int frames_per_slot;    // slot_per_frame: frame f uses slot f / frames_per_slot (>= 1)
  int frame0;             // launch group's first frame when its slot indices are global
};

// kernel slot (and Wiener table) index of plane p
__host__ __device__ inline int deblur_slot_index(const DeblurArgs& a, int p) {
  return a.slot_per_frame ? (a.frame0 + p / a.channels) / (a.frames_per_slot > 0 ? a.frames_per_slot : 1) : 0;
}

int deblur_col_width(int Gr, int t_max);
// pass 0: rows forward (A), 1: columns + filter (B), 2: rows inverse + crop (C)
cudaError_t launch_deblur_pass(const DeblurArgs& a, int planes, int pass, cudaStream_t stream);
// compile-time-planned passes (cbp_deblur_ct.cu); false if the grid has no specialisation
bool launch_deblur_pass_ct(const DeblurArgs& a, int planes, int pass, cudaStream_t stream);
bool deblur_has_ct(int Gr, int Gc, int pass);
bool ct_radices(int n, bool column, std::vector<int>& r);
int ct_pos(const std::vector<int>& rad, int n);
struct FusedCtl {
  unsigned* ticket;  // [0..2]: queue heads of roles A, B, C; [3]: role counter (zeroed per launch)
  unsigned* done;    // [0, P): A tiles done per plane, [P, 2P): B strips, [2P, 3P): C tiles
  int* sm_role;      // [nsm]: role claimed by the first CTA on each SM (-1 per launch)
  int nsm;
  int planes, ring;
  int nA, nB, nC;    // items per plane of each pass
};

// Fused persistent deconvolution (cbp_deblur_ct.cu): items per plane of each pass for this
// grid (false: no fused plan), and the launch (false: this geometry cannot use it)
bool deblur_fused_shape(const DeblurArgs& a, int& nA, int& nB, int& nC);
bool launch_deblur_fused(const DeblurArgs& a, const FusedCtl& f, cudaStream_t stream);
// Wiener filter tables of `frames` slots: S (column transforms) then H (cbp_deblur_ct.cu)
cudaError_t launch_wiener_tables(const DeblurArgs& a, int frames, cudaStream_t s);

}  // namespace cbp_dev
