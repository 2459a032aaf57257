// Shared declarations of the U-Net apply (unet.cu) and the tcgen05 conv
// kernel (unet_tc.cu).
#pragma once
#include "common.cuh"

namespace mdp {

struct UnetPlan {
  int n, m, q;
  size_t o_xin, o_a1, o_c1, o_c2, o_p2, o_bt, o_d2, o_d1, o_e2, o_e3, o_scr, scr_bytes;
  size_t bytes;
};
UnetPlan unet_plan(int n, int nb, int path);

enum Epilogue { EPI_STORE = 0, EPI_POOL = 1, EPI_HEAD = 2 };

struct HeadArgs {  // dec1 -> head1 -> head2 -> scale (EPI_HEAD)
  const float* w1;
  const float* b1;
  const float* w2;
  const float* b2;
  const int32_t* sel;
  const double* rnorm;
  double* z;
  int64_t ldz;
  int accumulate;  // z += rnorm * y instead of z = rnorm * y
};

// 3x3x3 same-padding conv on tensor cores (tcgen05 kind::tf32).
// w packed by paper_2505_08491_b200.neural.pack_tc.
int tc_conv3(int nb, int S, int cin, int cout, const float4* in, int in_cq, int in_q0, const float* w,
             const float* bias, int relu, float4* out, int out_cq, int out_q0, int epi, const HeadArgs* head,
             void* scratch, size_t scratch_bytes, cudaStream_t st);
// enc1a (2 -> 16) on tensor cores for wide grids (S >= TC_ENC1A_MIN_S); xin from pack_input_kernel mode 1
constexpr int TC_ENC1A_MIN_S = 64;
int tc_enc1a(int nb, int S, const float4* xin, const float* w, const float* bias, float4* out, int out_cq,
             int out_q0, cudaStream_t st);
// transposed conv k=2 s=2 (+ bias, ReLU, TF32 rounding, output-padding
// planes) on tensor cores; w packed [tap][quad][Cout][4] (neural.pack_tconv path 0)
int tc_tconv(int nb, const float4* in, int in_cq, int cin, int cout, int Sin, int op, const float* w,
             const float* bias, float4* out, int out_cq, int out_q0, cudaStream_t st);
// scratch needed by the split-K partial sums of one layer (0 when not split)
size_t tc_conv3_scratch_bytes(int nb, int S, int cin, int cout);

__device__ __forceinline__ float tf32_round(float f) {
  uint32_t u;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(u) : "f"(f));
  return __uint_as_float(u);
}
__device__ __forceinline__ float4 tf32_round4(float4 v) {
  return make_float4(tf32_round(v.x), tf32_round(v.y), tf32_round(v.z), tf32_round(v.w));
}

// output-padding planes (index 2*Sin in any axis): relu(bias), no kernel mass.
// Run by the tail blocks of the tconv launches (one tap group only).
__device__ __forceinline__ void tconv_pad(int Sin, int cout, const float* __restrict__ bias, float4* __restrict__ out,
                          int out_cq, int out_q0, int b, int64_t t0, int64_t stride, int round_tf32) {
  const int So = 2 * Sin + 1, E = 2 * Sin;
  const int64_t nvo = (int64_t)So * So * So;
  const int64_t nplane = nvo - (int64_t)E * E * E;
  const int64_t total = nplane * (cout / 4);
  for (int64_t t = t0; t < total; t += stride) {
    int64_t k = t % nplane;
    const int q = t / nplane;
    // enumerate the voxels with max(X,Y,Z) == E: Z == E plane, then Y == E, then X == E
    int X, Y, Z;
    if (k < (int64_t)So * So) {
      Z = E; Y = k / So; X = k % So;
    } else if ((k -= (int64_t)So * So) < (int64_t)E * So) {
      Z = k / So; Y = E; X = k % So;
    } else {
      k -= (int64_t)E * So;
      Z = k / E; Y = k % E; X = E;
    }
    float4 r = bias ? make_float4(fmaxf(bias[4 * q], 0.f), fmaxf(bias[4 * q + 1], 0.f), fmaxf(bias[4 * q + 2], 0.f),
                                  fmaxf(bias[4 * q + 3], 0.f))
                    : make_float4(0.f, 0.f, 0.f, 0.f);
    if (round_tf32) r = tf32_round4(r);
    out[((int64_t)b * out_cq + out_q0 + q) * nvo + ((int64_t)Z * So + Y) * So + X] = r;
  }
}

// head1 (32 -> 16, ReLU) and head2 (16 -> 1) of one voxel (neural.py:352-353);
// d = the 32 dec1 activations as stored (bias, ReLU, TF32-rounded).  Shared by
// the fused conv epilogue, the split-K reduce and the unfused head kernel so
// every path sums in the same order.
__device__ __forceinline__ float head_eval(const float* d, const float* __restrict__ w1,
                                           const float* __restrict__ b1, const float* __restrict__ w2,
                                           const float* __restrict__ b2) {
  float h[16];
#pragma unroll
  for (int c = 0; c < 16; ++c) h[c] = b1[c];
#pragma unroll
  for (int q = 0; q < 8; ++q)
#pragma unroll
    for (int c = 0; c < 16; ++c)
      h[c] += w1[c * 32 + 4 * q] * d[4 * q] + w1[c * 32 + 4 * q + 1] * d[4 * q + 1] +
              w1[c * 32 + 4 * q + 2] * d[4 * q + 2] + w1[c * 32 + 4 * q + 3] * d[4 * q + 3];
  float y = b2[0];
#pragma unroll
  for (int c = 0; c < 16; ++c) y += w2[c] * fmaxf(h[c], 0.f);
  return y;
}

}  // namespace mdp
