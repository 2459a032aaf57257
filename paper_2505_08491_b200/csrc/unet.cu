// CNN preconditioner apply: the three-level U-Net of neural.py:342-472 on
// float32 activations in a channel-quad-blocked layout
//     act[((b * CQ + cq) * S + z) * S * S + y * S + x]  (float4 = 4 channels)
// so a concat is a quad range (neural.py:323-328 costs nothing) and every
// warp access is a contiguous run of 16-byte quads.
//
// Two conv paths share this orchestration:
//   path 0  tcgen05 TF32 implicit GEMM (unet_tc.cu) -- the product path
//   path 1  CUDA-core FP32 direct conv (this file)   -- the check path used
//           by the parity tests to localise tensor-core errors
// enc1a (Cin=2), the stride-2 transposed convs and the 1x1 heads are
// memory-bound and run on CUDA cores in both paths.
#include <stdlib.h>

#include "common.cuh"
#include "unet_layout.cuh"

namespace mdp {

// ---------------------------------------------------------------------------
// input pack: xin[b][v] = (r_s[v] / ||r_s||, d_s[v])   (training.py:312-318)
__global__ void pack_input_kernel(const int32_t* sel, const double* __restrict__ r, int64_t ld,
                                  const double* __restrict__ rnorm, const double* __restrict__ dist,
                                  int64_t ldd, float2* __restrict__ xin, int64_t nvox, int S, int shifted) {
  MDP_PDL_ENTER();
  const int b = blockIdx.y;
  const int s = sys_of(sel, b);
  double nr = rnorm[b];
  double den = nr != 0.0 ? nr : 1.0;
  if (shifted) {
    // tensor-core enc1a (tc_enc1a): quad of voxel x = (r, d)[x] | (r, d)[x+1] (zero past the row end), TF32-rounded
    float4* x4 = reinterpret_cast<float4*>(xin);
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t v0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v0 < nvox; v0 += 4 * stride) {
      double ra[4], rb[4], da[4], db[4];  // sixteen loads in flight per thread before the divisions
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int64_t v = v0 + k * stride;
        const bool in = v < nvox;
        const bool nxt = in && (int)(v % S) + 1 < S;
        ra[k] = in ? r[s * ld + v] : 0.0;
        rb[k] = nxt ? r[s * ld + v + 1] : 0.0;
        da[k] = in ? dist[s * ldd + v] : 0.0;
        db[k] = nxt ? dist[s * ldd + v + 1] : 0.0;
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int64_t v = v0 + k * stride;
        if (v >= nvox) break;
        const bool nxt = (int)(v % S) + 1 < S;
        const double r0 = ra[k] / den, r1 = nxt ? rb[k] / den : 0.0;
        x4[b * nvox + v] = tf32_round4(make_float4((float)r0, (float)da[k], (float)r1, (float)db[k]));
      }
    }
    return;
  }
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nvox;
       v += (int64_t)gridDim.x * blockDim.x) {
    double rv = r[s * ld + v] / den;
    xin[b * nvox + v] = make_float2((float)rv, (float)dist[s * ldd + v]);
  }
}

// enc1a: 3x3x3 conv 2 -> 16, bias, ReLU (neural.py:343); w [16][2][27].
// One thread = VX x-adjacent voxels (2 on large grids: weights and neighbour
// columns shared; 1 on small, latency-bound grids: twice the threads).  The
// weights are transposed in shared memory to [tap][ch][16], so one (tap,
// channel) is four 16-byte broadcast loads feeding 16 VX FMAs (a scalar load
// per FMA made this kernel LSU-bound); the neighbour columns of one z-plane
// are loaded before their FMAs.
template <int VX>
__global__ void __launch_bounds__(128) enc1a_kernel(const float2* __restrict__ xin, int S,
                                                     const float* __restrict__ w,
                                                     const float* __restrict__ bias,
                                                     float4* __restrict__ out, int round_tf32) {
  MDP_PDL_ENTER();
  __shared__ float4 ws4[27 * 2 * 4];  // [tap][ch][16 channels as 4 float4]
  __shared__ float bs[16];
  float* wsf = reinterpret_cast<float*>(ws4);
  for (int t = threadIdx.x; t < 16 * 54; t += blockDim.x) {
    const int c = t / 54, ch = (t / 27) % 2, tap = t % 27;  // w[(c * 2 + ch) * 27 + tap]
    wsf[(tap * 2 + ch) * 16 + c] = w[t];
  }
  for (int t = threadIdx.x; t < 16; t += blockDim.x) bs[t] = bias ? bias[t] : 0.f;
  __syncthreads();
  const int b = blockIdx.y;
  const int SX = (S + VX - 1) / VX;  // voxel groups per x-row
  const int64_t nvox = (int64_t)S * S * S;
  const int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (u >= (int64_t)SX * S * S) return;
  const int x = VX * (int)(u % SX), y = (u / SX) % S, z = u / ((int64_t)SX * S);
  float acc[VX][16];
#pragma unroll
  for (int k = 0; k < VX; ++k)
#pragma unroll
    for (int c = 0; c < 16; ++c) acc[k][c] = bs[c];
  const float2* xb = xin + b * nvox;
#pragma unroll
  for (int dz = 0; dz < 3; ++dz) {
    // columns x-1 .. x+VX of rows y-1 .. y+1; out-of-domain neighbours are exact
    // zeros (same sums as skipping the tap)
    float2 in[3][VX + 2];
    const int zz = z + dz - 1;
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      const int yy = y + r - 1;
      const bool rok = zz >= 0 && yy >= 0 && zz < S && yy < S;
#pragma unroll
      for (int k = 0; k < VX + 2; ++k) {
        const int xx = x + k - 1;
        in[r][k] = rok && xx >= 0 && xx < S ? __ldg(xb + ((int64_t)zz * S + yy) * S + xx) : make_float2(0.f, 0.f);
      }
    }
#pragma unroll
    for (int t = 0; t < 9; ++t) {
      const int tap = dz * 9 + t, r = t / 3, kx = t % 3;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float4 w0 = ws4[(tap * 2 + 0) * 4 + q], w1 = ws4[(tap * 2 + 1) * 4 + q];
#pragma unroll
        for (int k = 0; k < VX; ++k) {
          const float2 a = in[r][kx + k];
          acc[k][4 * q + 0] += w0.x * a.x + w1.x * a.y;
          acc[k][4 * q + 1] += w0.y * a.x + w1.y * a.y;
          acc[k][4 * q + 2] += w0.z * a.x + w1.z * a.y;
          acc[k][4 * q + 3] += w0.w * a.x + w1.w * a.y;
        }
      }
    }
  }
  const int64_t v = ((int64_t)z * S + y) * S + x;
#pragma unroll
  for (int k = 0; k < VX; ++k) {
    if (x + k >= S) break;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      float4 o = make_float4(fmaxf(acc[k][4 * q], 0.f), fmaxf(acc[k][4 * q + 1], 0.f), fmaxf(acc[k][4 * q + 2], 0.f),
                             fmaxf(acc[k][4 * q + 3], 0.f));
      if (round_tf32) o = tf32_round4(o);
      out[((int64_t)b * 4 + q) * nvox + v + k] = o;
    }
  }
}

// Direct 3x3x3 conv, one thread per output voxel x 16 output channels.
// w packed [cout/16][cin][27][16]; input quads [in_q0, in_q0 + cin/4) of a
// CQin-quad tensor, output quads [out_q0, +4) per group of a CQout tensor.
__global__ void __launch_bounds__(128) conv3_direct_kernel(const float4* __restrict__ in, int in_cq,
                                                            int in_q0, int cin, int S,
                                                            const float* __restrict__ w,
                                                            const float* __restrict__ bias, int relu,
                                                            float4* __restrict__ out, int out_cq,
                                                            int out_q0) {
  MDP_PDL_ENTER();
  extern __shared__ float wsh[];  // [32 cin][27][16] chunk
  const int g = blockIdx.y;       // cout group of 16
  const int b = blockIdx.z;
  const int64_t nvox = (int64_t)S * S * S;
  const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const bool live = v < nvox;
  const int x = live ? v % S : 0, y = live ? (v / S) % S : 0, z = live ? v / ((int64_t)S * S) : 0;
  float acc[16];
#pragma unroll
  for (int c = 0; c < 16; ++c) acc[c] = bias ? bias[g * 16 + c] : 0.f;
  const float* wg = w + (int64_t)g * cin * 27 * 16;
  for (int c0 = 0; c0 < cin; c0 += 32) {
    const int cc = min(32, cin - c0);
    __syncthreads();
    for (int t = threadIdx.x; t < cc * 27 * 16; t += blockDim.x) wsh[t] = wg[(int64_t)c0 * 27 * 16 + t];
    __syncthreads();
    if (!live) continue;
    for (int q = 0; q < cc / 4; ++q) {
      const float4* ib = in + ((int64_t)b * in_cq + in_q0 + c0 / 4 + q) * nvox;
      for (int dz = 0; dz < 3; ++dz) {
        int zz = z + dz - 1;
        if (zz < 0 || zz >= S) continue;
        for (int dy = 0; dy < 3; ++dy) {
          int yy = y + dy - 1;
          if (yy < 0 || yy >= S) continue;
          for (int dx = 0; dx < 3; ++dx) {
            int xx = x + dx - 1;
            if (xx < 0 || xx >= S) continue;
            float4 a = __ldg(ib + ((int64_t)zz * S + yy) * S + xx);
            const float* wt = wsh + ((4 * q) * 27 + (dz * 3 + dy) * 3 + dx) * 16;
#pragma unroll
            for (int c = 0; c < 16; ++c)
              acc[c] += a.x * wt[c] + a.y * wt[27 * 16 + c] + a.z * wt[2 * 27 * 16 + c] + a.w * wt[3 * 27 * 16 + c];
          }
        }
      }
    }
  }
  if (!live) return;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    float4 o = make_float4(acc[4 * q], acc[4 * q + 1], acc[4 * q + 2], acc[4 * q + 3]);
    if (relu) o = make_float4(fmaxf(o.x, 0.f), fmaxf(o.y, 0.f), fmaxf(o.z, 0.f), fmaxf(o.w, 0.f));
    out[((int64_t)b * out_cq + out_q0 + g * 4 + q) * nvox + v] = o;
  }
}

// 2x2x2 max pool with floor (neural.py:275-290)
__global__ void maxpool_kernel(const float4* __restrict__ in, int in_cq, int S, int cq,
                               float4* __restrict__ out, int out_cq, int out_q0, int nb) {
  MDP_PDL_ENTER();
  const int M = S / 2;
  const int64_t mv = (int64_t)M * M * M;
  const int64_t total = (int64_t)nb * cq * mv;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t v = t % mv;
    int64_t bq = t / mv;
    int q = bq % cq, b = bq / cq;
    int x = v % M, y = (v / M) % M, z = v / ((int64_t)M * M);
    const float4* ib = in + ((int64_t)b * in_cq + q) * S * S * S;
    float4 m = make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
    for (int d = 0; d < 8; ++d) {
      float4 a = ib[((int64_t)(2 * z + (d >> 2)) * S + 2 * y + ((d >> 1) & 1)) * S + 2 * x + (d & 1)];
      m.x = fmaxf(m.x, a.x); m.y = fmaxf(m.y, a.y); m.z = fmaxf(m.z, a.z); m.w = fmaxf(m.w, a.w);
    }
    out[((int64_t)b * out_cq + out_q0 + q) * mv + v] = m;
  }
}

// Transposed conv k=2 s=2 (neural.py:215-246) + bias + ReLU, output size
// 2*Sin+op.  One block = one kernel tap (a,b,c) x 16 output channels over a
// run of input voxels: the tap's weights (Cin x 16) sit in shared memory and
// each input quad is read once, coalesced.  w packed [cout/16][cin][8][16].
__global__ void __launch_bounds__(128) tconv_kernel(const float4* __restrict__ in, int in_cq, int cin,
                                                     int Sin, int op, const float* __restrict__ w,
                                                     const float* __restrict__ bias,
                                                     float4* __restrict__ out, int out_cq, int out_q0,
                                                     int round_tf32, int nmain) {
  MDP_PDL_ENTER();
  __shared__ float4 wsh[128 * 4];  // [cin][16] for this tap
  const int tap = blockIdx.y & 7, g = blockIdx.y >> 3, b = blockIdx.z;
  if ((int)blockIdx.x >= nmain) {  // tail blocks: the output-padding planes
    if (blockIdx.y == 0)
      tconv_pad(Sin, (int)(gridDim.y / 8) * 16, bias, out, out_cq, out_q0, b,
                (blockIdx.x - nmain) * (int64_t)blockDim.x + threadIdx.x, (int64_t)(gridDim.x - nmain) * blockDim.x,
                round_tf32);
    return;
  }
  const float* wg = w + (size_t)g * cin * 8 * 16;
  for (int t = threadIdx.x; t < cin * 4; t += blockDim.x) {
    const int ci = t >> 2, c4 = t & 3;
    const float* src = wg + ((size_t)ci * 8 + tap) * 16 + 4 * c4;
    wsh[t] = make_float4(src[0], src[1], src[2], src[3]);
  }
  __syncthreads();
  const int So = 2 * Sin + op;
  const int64_t nvo = (int64_t)So * So * So, nvi = (int64_t)Sin * Sin * Sin;
  const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (v >= nvi) return;
  const int x = v % Sin, y = (v / Sin) % Sin, z = v / ((int64_t)Sin * Sin);
  float acc[16];
#pragma unroll
  for (int c = 0; c < 16; ++c) acc[c] = bias ? bias[g * 16 + c] : 0.f;
  constexpr int QB = 8;  // input quads loaded per batch (cin/4 is a multiple of 8 here)
  for (int q0 = 0; q0 < cin / 4; q0 += QB) {
    float4 a[QB];
#pragma unroll
    for (int j = 0; j < QB; ++j) a[j] = __ldg(in + ((int64_t)b * in_cq + q0 + j) * nvi + v);
#pragma unroll
    for (int j = 0; j < QB; ++j) {
      const float av[4] = {a[j].x, a[j].y, a[j].z, a[j].w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
#pragma unroll
        for (int c4 = 0; c4 < 4; ++c4) {
          const float4 wv = wsh[(4 * (q0 + j) + e) * 4 + c4];
          acc[4 * c4] += av[e] * wv.x;
          acc[4 * c4 + 1] += av[e] * wv.y;
          acc[4 * c4 + 2] += av[e] * wv.z;
          acc[4 * c4 + 3] += av[e] * wv.w;
        }
      }
    }
  }
  const int X = 2 * x + (tap & 1), Y = 2 * y + ((tap >> 1) & 1), Z = 2 * z + (tap >> 2);
  const int64_t o = ((int64_t)Z * So + Y) * So + X;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    float4 r = make_float4(fmaxf(acc[4 * q], 0.f), fmaxf(acc[4 * q + 1], 0.f), fmaxf(acc[4 * q + 2], 0.f),
                           fmaxf(acc[4 * q + 3], 0.f));
    if (round_tf32) r = tf32_round4(r);
    out[((int64_t)b * out_cq + out_q0 + g * 4 + q) * nvo + o] = r;
  }
}

// heads: d1 (32 ch) -> head1 (16, ReLU) -> head2 (1) -> z = ||r|| * y (float64)
__global__ void __launch_bounds__(128) head_kernel(const float4* __restrict__ d1, int S,
                                                    const float* __restrict__ w1, const float* __restrict__ b1,
                                                    const float* __restrict__ w2, const float* __restrict__ b2,
                                                    const int32_t* sel, const double* __restrict__ rnorm,
                                                    double* __restrict__ z, int64_t ldz, int accumulate) {
  MDP_PDL_ENTER();
  __shared__ float ws[16 * 32 + 16 + 16 + 1];
  for (int t = threadIdx.x; t < 512; t += blockDim.x) ws[t] = w1[t];
  for (int t = threadIdx.x; t < 16; t += blockDim.x) {
    ws[512 + t] = b1[t];
    ws[528 + t] = w2[t];
  }
  if (threadIdx.x == 0) ws[544] = b2[0];
  __syncthreads();
  const int b = blockIdx.y;
  const int64_t nvox = (int64_t)S * S * S;
  const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (v >= nvox) return;
  float d[32];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const float4 a = __ldg(d1 + ((int64_t)b * 8 + q) * nvox + v);
    d[4 * q] = a.x; d[4 * q + 1] = a.y; d[4 * q + 2] = a.z; d[4 * q + 3] = a.w;
  }
  const float y = head_eval(d, ws, ws + 512, ws + 528, ws + 544);
  double* zp = z + sys_of(sel, b) * ldz + v;
  *zp = accumulate ? *zp + rnorm[b] * (double)y : rnorm[b] * (double)y;
}

// ---------------------------------------------------------------------------

static int direct_conv(int nb, int S, int cin, int cout, const float4* in, int in_cq, int in_q0,
                       const float* w, const float* bias, int relu, float4* out, int out_cq, int out_q0,
                       cudaStream_t st) {
  MDP_REQUIRE(cin % 4 == 0 && cout % 16 == 0, "direct conv needs cin%%4==0, cout%%16==0");
  const int64_t nvox = (int64_t)S * S * S;
  const int smem = 32 * 27 * 16 * 4;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(conv3_direct_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  dim3 grid(ceil_div(nvox, 128), cout / 16, nb);
  ::mdp::launch_k(conv3_direct_kernel, grid, 128, smem, st, in, in_cq, in_q0, cin, S, w, bias, relu, out, out_cq, out_q0);
  MDP_LAUNCH_CHECK("conv3_direct_kernel");
  return MDP_OK;
}

static int launch_pool(const float4* in, int in_cq, int S, int cq, float4* out, int out_cq, int out_q0, int nb,
                       cudaStream_t st) {
  int64_t M = S / 2;
  int64_t total = (int64_t)nb * cq * M * M * M;
  int bx = ceil_div(total, 256);
  bx = bx > 8 * sm_count() ? 8 * sm_count() : bx;
  ::mdp::launch_k(maxpool_kernel, bx, 256, 0, st, in, in_cq, S, cq, out, out_cq, out_q0, nb);
  MDP_LAUNCH_CHECK("maxpool_kernel");
  return MDP_OK;
}

static int launch_tconv(int nb, const float4* in, int in_cq, int cin, int cout, int Sin, int op, const float* w,
                        const float* bias, float4* out, int out_cq, int out_q0, int round_tf32,
                        cudaStream_t st) {
  MDP_REQUIRE(cin <= 128 && cin % 32 == 0 && cout % 16 == 0, "tconv needs cin<=128, cin%%32==0, cout%%16==0");
  const int64_t nvi = (int64_t)Sin * Sin * Sin;
  const int nmain = ceil_div(nvi, 128);
  int npad = 0;
  if (op) {
    const int So = 2 * Sin + 1;
    const int64_t per_item = ((int64_t)So * So * So - 8 * nvi) * (cout / 4);
    npad = ceil_div(per_item, 128);
    npad = npad > 64 ? 64 : npad;
  }
  dim3 grid(nmain + npad, 8 * (cout / 16), nb);
  ::mdp::launch_k(tconv_kernel, grid, 128, 0, st, in, in_cq, cin, Sin, op, w, bias, out, out_cq, out_q0, round_tf32, nmain);
  MDP_LAUNCH_CHECK("tconv_kernel");
  return MDP_OK;
}

// A/B switch: MDP_ENC1A_TC=0 keeps enc1a on CUDA cores at every size
static bool enc1a_cuda_cores() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("MDP_ENC1A_TC");
    v = (e && e[0] == '0') ? 1 : 0;
  }
  return v == 1;
}

UnetPlan unet_plan(int n, int nb, int path) {
  UnetPlan p;
  p.n = n;
  p.m = n / 2;
  p.q = p.m / 2;
  const int64_t N = (int64_t)n * n * n, M = (int64_t)p.m * p.m * p.m, Q = (int64_t)p.q * p.q * p.q;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += (bytes + 255) & ~(size_t)255;
    return o;
  };
  p.o_xin = take((size_t)nb * N * sizeof(float4));  // float2 (r, d), or the x-shifted quads of tc_enc1a
  p.o_a1 = take((size_t)nb * 4 * N * 16);
  p.o_c1 = take((size_t)nb * 16 * N * 16);
  p.o_c2 = take((size_t)nb * 32 * M * 16);
  p.o_p2 = take((size_t)nb * 32 * Q * 16);
  p.o_bt = take((size_t)nb * 32 * Q * 16);
  p.o_d2 = take((size_t)nb * 16 * M * 16);
  // path 0 fuses the heads into dec1's epilogue (no d1 tensor) and the pools
  // into enc2/enc3; path 1 keeps d1 and the full-resolution pre-pool tensors
  if (path == 1) {
    p.o_d1 = take((size_t)nb * 8 * N * 16);
    p.o_e2 = take((size_t)nb * 16 * N * 16);
    p.o_e3 = take((size_t)nb * 32 * M * 16);
    p.o_scr = p.scr_bytes = 0;
  } else {
    p.o_d1 = p.o_e2 = p.o_e3 = 0;
    size_t scr = 0;
    const int shp[6][3] = {{n, 16, 32}, {n, 32, 64}, {p.m, 64, 128}, {p.q, 128, 128}, {p.m, 128, 64}, {n, 64, 32}};
    for (auto& L : shp) {
      size_t b = tc_conv3_scratch_bytes(nb, L[0], L[1], L[2]);
      scr = b > scr ? b : scr;
    }
    p.scr_bytes = scr;
    p.o_scr = scr ? take(scr) : 0;
  }
  p.bytes = off;
  return p;
}

}  // namespace mdp

using namespace mdp;

extern "C" size_t mdp_unet_workspace_bytes(int32_t n, int32_t nb, int32_t path) {
  return unet_plan(n, nb, path).bytes;
}

extern "C" size_t mdp_conv3_scratch_bytes(int32_t nb, int32_t S, int32_t cin, int32_t cout) {
  return tc_conv3_scratch_bytes(nb, S, cin, cout);
}

extern "C" int mdp_conv3_layer(int32_t path, int32_t nb, int32_t S, int32_t cin, int32_t cout, const float* in,
                               int32_t in_cq, int32_t in_q0, const float* w, const float* bias, int32_t relu,
                               float* out, int32_t out_cq, int32_t out_q0, int32_t pool, void* scratch,
                               size_t scratch_bytes, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (path == 1) {
    MDP_REQUIRE(!pool, "direct path conv layer has no fused pool");
    return direct_conv(nb, S, cin, cout, (const float4*)in, in_cq, in_q0, w, bias, relu, (float4*)out, out_cq,
                       out_q0, st);
  }
  return tc_conv3(nb, S, cin, cout, (const float4*)in, in_cq, in_q0, w, bias, relu, (float4*)out, out_cq, out_q0,
                  pool ? EPI_POOL : EPI_STORE, nullptr, scratch, scratch_bytes, st);
}

extern "C" int mdp_unet_apply(const mdp_unet* net, int32_t nb, const int32_t* sel, const double* r, int64_t ld,
                              const double* rnorm, const double* dist, int64_t ldd, double* z, int64_t ldz,
                              void* workspace, size_t ws_bytes, void* stream) {
  MDP_REQUIRE(net != nullptr, "null network descriptor");
  const int n = net->n;
  MDP_REQUIRE(n >= 8, "spatial size must be at least 8, got %d", n);
  if (nb == 0) return MDP_OK;
  const int path = net->path;
  UnetPlan P = unet_plan(n, nb, path);
  MDP_REQUIRE(ws_bytes >= P.bytes, "workspace too small: %zu < %zu", ws_bytes, P.bytes);
  cudaStream_t st = (cudaStream_t)stream;
  char* ws = (char*)workspace;
  float2* xin = (float2*)(ws + P.o_xin);
  float4* a1 = (float4*)(ws + P.o_a1);
  float4* c1 = (float4*)(ws + P.o_c1);
  float4* c2 = (float4*)(ws + P.o_c2);
  float4* p2 = (float4*)(ws + P.o_p2);
  float4* bt = (float4*)(ws + P.o_bt);
  float4* d2 = (float4*)(ws + P.o_d2);
  float4* d1 = (float4*)(ws + P.o_d1);
  const int m = P.m, q = P.q;
  const int op2 = m - 2 * q, op1 = n - 2 * m;
  const int64_t N = (int64_t)n * n * n;
  const int tf = path == 0;  // round stored activations to TF32 on the tensor-core path
  int rc;
  // wide grids on the tensor-core path: enc1a as a K = 8 MMA per (dy, halo plane) over x-shifted input quads
  const int tc_enc = path == 0 && n >= TC_ENC1A_MIN_S && !enc1a_cuda_cores();

  {
    int bx = ceil_div(N, 256);
    bx = bx > 8 * sm_count() ? 8 * sm_count() : bx;
    ::mdp::launch_k(pack_input_kernel, dim3(bx, nb), 256, 0, st, sel, r, ld, rnorm, dist, ldd, xin, N, n, tc_enc);
    MDP_LAUNCH_CHECK("pack_input_kernel");
  }
  if (tc_enc) {
    if ((rc = tc_enc1a(nb, n, (const float4*)xin, net->w[0], net->b[0], a1, 4, 0, st))) return rc;
  } else if (n >= 64)  // wide grids: two voxels per thread; small latency-bound grids: one
    ::mdp::launch_k(enc1a_kernel<2>, dim3(ceil_div((int64_t)((n + 1) / 2) * n * n, 128), nb), 128, 0, st, xin, n,
                    net->w[0], net->b[0], a1, tf);
  else
    ::mdp::launch_k(enc1a_kernel<1>, dim3(ceil_div((int64_t)n * n * n, 128), nb), 128, 0, st, xin, n, net->w[0],
                    net->b[0], a1, tf);
  MDP_LAUNCH_CHECK("enc1a_kernel");

  if (path == 1) {
    float4* e2 = (float4*)(ws + P.o_e2);
    float4* e3 = (float4*)(ws + P.o_e3);
    if ((rc = direct_conv(nb, n, 16, 32, a1, 4, 0, net->w[1], net->b[1], 1, c1, 16, 8, st))) return rc;
    if ((rc = direct_conv(nb, n, 32, 64, c1, 16, 8, net->w[2], nullptr, 1, e2, 16, 0, st))) return rc;
    if ((rc = launch_pool(e2, 16, n, 16, c2, 32, 16, nb, st))) return rc;
    if ((rc = direct_conv(nb, m, 64, 128, c2, 32, 16, net->w[3], nullptr, 1, e3, 32, 0, st))) return rc;
    if ((rc = launch_pool(e3, 32, m, 32, p2, 32, 0, nb, st))) return rc;
    if ((rc = direct_conv(nb, q, 128, 128, p2, 32, 0, net->w[4], nullptr, 1, bt, 32, 0, st))) return rc;
    if ((rc = launch_tconv(nb, bt, 32, 128, 64, q, op2, net->w[5], nullptr, c2, 32, 0, 0, st))) return rc;
    if ((rc = direct_conv(nb, m, 128, 64, c2, 32, 0, net->w[6], net->b[6], 1, d2, 16, 0, st))) return rc;
    if ((rc = launch_tconv(nb, d2, 16, 64, 32, m, op1, net->w[7], net->b[7], c1, 16, 0, 0, st))) return rc;
    if ((rc = direct_conv(nb, n, 64, 32, c1, 16, 0, net->w[8], net->b[8], 1, d1, 8, 0, st))) return rc;
  } else {
    if ((rc = tc_conv3(nb, n, 16, 32, a1, 4, 0, net->w[1], net->b[1], 1, c1, 16, 8, EPI_STORE, nullptr, ws + P.o_scr, P.scr_bytes, st)))
      return rc;
    if ((rc = tc_conv3(nb, n, 32, 64, c1, 16, 8, net->w[2], nullptr, 1, c2, 32, 16, EPI_POOL, nullptr, ws + P.o_scr, P.scr_bytes, st)))
      return rc;
    if ((rc = tc_conv3(nb, m, 64, 128, c2, 32, 16, net->w[3], nullptr, 1, p2, 32, 0, EPI_POOL, nullptr, ws + P.o_scr, P.scr_bytes, st)))
      return rc;
    if ((rc = tc_conv3(nb, q, 128, 128, p2, 32, 0, net->w[4], nullptr, 1, bt, 32, 0, EPI_STORE, nullptr, ws + P.o_scr, P.scr_bytes, st)))
      return rc;
    if ((rc = tc_tconv(nb, bt, 32, 128, 64, q, op2, net->w[5], nullptr, c2, 32, 0, st))) return rc;
    if ((rc = tc_conv3(nb, m, 128, 64, c2, 32, 0, net->w[6], net->b[6], 1, d2, 16, 0, EPI_STORE, nullptr, ws + P.o_scr, P.scr_bytes, st)))
      return rc;
    if ((rc = tc_tconv(nb, d2, 16, 64, 32, m, op1, net->w[7], net->b[7], c1, 16, 0, st))) return rc;
    // dec1 with head1 -> head2 -> ||r|| scaling fused into its epilogue
    HeadArgs H{net->w[9], net->b[9], net->w[10], net->b[10], sel, rnorm, z, ldz, net->accumulate};
    return tc_conv3(nb, n, 64, 32, c1, 16, 0, net->w[8], net->b[8], 1, nullptr, 0, 0, EPI_HEAD, &H, ws + P.o_scr,
                    P.scr_bytes, st);
  }
  ::mdp::launch_k(head_kernel, dim3(ceil_div(N, 128), nb), 128, 0, st, d1, n, net->w[9], net->b[9], net->w[10], net->b[10],
                                                          sel, rnorm, z, ldz, net->accumulate);
  MDP_LAUNCH_CHECK("head_kernel");
  return MDP_OK;
}
