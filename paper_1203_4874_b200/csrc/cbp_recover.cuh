// Kernel-recovery stages of decode_frame (reference decoder.cpp:280-361) on the device.
#pragma once

#include "cbp_common.cuh"

namespace cbp_dev {

// Device-side geometry of one decode batch and the workspace layout.
struct RecoverArgs {
  int chain;  // programmatic dependent launch of the small recovery kernels (cbp_set_launch_chaining)
  const float* pub;
  const float* prv;
  int batch, channels, rows, cols, ld;  // blurred geometry (Mb = rows, Nb = cols)
  cbp_kernel_slot* slots;               // [batch]
  int* flags;                           // [batch]: bit0 negative luma sample seen
  int t_max;                            // upper bound of t over the batch
  int lmax;                             // max(rows, cols)
  // fold workspaces
  double* part;       // Z1 partials [batch][2][part_stride]: [row block][t][cols]
  size_t part_stride;
  int fold_rh;        // target rows per fold block (fold_plan)
  double* part2;      // Z2 partials [batch][2][ncb][t_max][rows]
  int ncb;            // column strips of the fold (256 columns)
  double2* slices;    // [batch][2 axes][2 streams][t_max][lmax]
  // solve outputs
  double2* values;    // [batch][2 axes][t_max][t_max]
  double* gaps;       // [batch][2 axes][t_max]
  int* slice_status;  // [batch][2 axes][t_max]: 0 ok, CBP_REASON_GAP / _VANISHING_COFACTOR
  double2* scratch;   // [batch][2 axes][t_max][lmax + t_max] residual vectors
  // width search
  double* ratios;     // [batch][2][nsizes]
  double2* roots;     // signed content: exp(-2 pi i k / rows) then exp(-2 pi i k / cols)
  double* epart;      // signed content: per-tile energy partials, z1 then z2 (at epart_z2)
  size_t epart_z2;
  int search_min, search_max, nsizes;
  double tau;
  int trust_hint;
  // config
  double gap_threshold, max_imag_energy, negative_weight_tol;
  int has_epsilon;
  double epsilon;
  // kernels wider than the shared-memory solvers (t > kSmemMaxWidth): per-CTA scratch for
  // the 2t x 2t Grams and eigenvectors in global memory (L2-resident), wide_ctas CTAs
  double2* wide;
  size_t wide_stride;  // double2 elements per CTA
  int wide_ctas;
};

// widest kernel whose solve / composition scratch lives in shared memory; wider ones (up to
// the reference's 63, decoder.cpp:32-33,305-306) run the same code on global scratch
constexpr int kSmemMaxWidth = 31;
constexpr int kWideMaxWidth = 63;
// double2 elements of global scratch one wide CTA needs (solve and compose at t = 63)
size_t wide_scratch_elems();

__host__ __device__ inline size_t slice_offset(const RecoverArgs& a, int b, int axis, int q, int i) {
  return ((size_t(b) * 2 + axis) * 2 + q) * size_t(a.t_max) * a.lmax + size_t(i) * a.lmax;
}

struct HintChunk {
  static constexpr int kMax = 1024;
  int first, count;
  int hint[kMax];
};
cudaError_t launch_init_slots(const RecoverArgs& a, const int* hints_host, cudaStream_t s);
// t_fixed > 0 folds with that t (1 = DC sums); otherwise with slots[b].width.
cudaError_t launch_fold(const RecoverArgs& a, int t_fixed, cudaStream_t s);
void fold_plan(int batch, int rows, int cols, int t_max, int& ncb, int& rh, size_t& part_stride);
cudaError_t launch_width(const RecoverArgs& a, cudaStream_t s);
// signed content (decoder.cpp:65-82): replaces the DC slices of frames with a negative
// luma sample by the maximum-energy axis_spectrum_half slices (cbp_signed.cu)
cudaError_t launch_signed_slices(const RecoverArgs& a, cudaStream_t s);
size_t signed_energy_doubles(int batch, int rows, int cols);
cudaError_t launch_solve(const RecoverArgs& a, cudaStream_t s);
cudaError_t launch_compose(const RecoverArgs& a, cudaStream_t s);
// validation residual (decoder.cpp:367-376) of the latent against the public frame
cudaError_t launch_validate(const RecoverArgs& a, const float* latent, int ld_out, double* part,
                            int ntiles_max, cudaStream_t s);
int validate_tiles(int rows, int cols, int t);  // t: kernel width (sets the tile height)

// Standalone batched cofactor solve for the stage-level C ABI entry.
// (t > kSmemMaxWidth: wide = global scratch of wide_scratch_elems() per problem, else null)
cudaError_t launch_cofactor_batch(const double2* p, int lp, const double2* q, int lq, int batch, int t,
                                  double gap_threshold, double2* k1, double2* k2, double* gaps,
                                  int* status, double2* scratch, double2* wide, cudaStream_t s);
// complete_to_spectrum / resolve_scales / assemble_kernel on one problem (stage entries).
cudaError_t launch_complete(const double2* values, int t, int axis, double2* out, cudaStream_t s);
cudaError_t launch_resolve(const double2* a_values, const double2* b_values, int t, double2* lambda,
                           double2* mu, double* residual, int* status, double* value, double2* wide,
                           cudaStream_t s);
cudaError_t launch_assemble(const double2* a_spec, const double2* b_spec, const double2* lambda,
                            const double2* mu, int t, double max_imag, double neg_tol,
                            cbp_kernel_slot* slot, double2* wide, cudaStream_t s);
// validate_pair (decoder.cpp:380-395): |pub (*) k2 - prv (*) k1| / |pub (*) k2|
cudaError_t launch_validate_pair(const float* pub, const float* prv, int channels, int rows, int cols,
                                 int ld, const double* k1, const double* k2, int t, double* part,
                                 cudaStream_t s);
// encode_frame (encoder.cpp:83-103) and synthetic frames
cudaError_t launch_encode(const float* latent, int planes, int rows, int cols, int ld, const double* k,
                          int t, float* out, int ld_out, cudaStream_t s);
cudaError_t launch_synth(float* out, int planes, int rows, int cols, int ld, unsigned long long seed,
                         cudaStream_t s);

}  // namespace cbp_dev
