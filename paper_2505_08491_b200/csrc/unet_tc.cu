// 3x3x3 same-padding convolution as an implicit GEMM on the 5th-generation
// tensor cores (tcgen05.mma kind::tf32, FP32 accumulate in TMEM), replacing
// neural.conv3d's im2col + BLAS GEMM (neural.py:60-154).
//
// Tile = brick of ZP x 16 x 8 output voxels (z, y, x) of one batch item;
// each z-plane is one M = 128 MMA row block, N = Cout, K = 27 taps x Cin.
//
// A operand: the brick plus its 1-voxel halo, (ZP+2) x 18 x 10 voxels x 32
// channels, is fetched ONCE per 32-channel chunk by a single 4-D TMA box
// (inner row = a 10-voxel x-run of one channel quad, 160 B) from the
// channel-quad-blocked activation tensor, with TMA's out-of-bounds
// zero fill providing the same-padding.  The box lands in shared memory as
// [quad][z][y][x][4 floats], which is exactly the K-major no-swizzle UMMA
// canonical layout (core matrix = 8 consecutive x-voxels x 16 B): every
// tap's operand is the same buffer viewed through a descriptor whose start
// address is shifted by (dz*18*10 + dy*10 + dx) * 16 bytes, LBO = one quad
// plane, SBO = one halo y-line.  No im2col is ever materialised and each
// activation is read from L2 once per brick instead of 27 times.
//
// B operand: weights pre-packed per (chunk, tap) as [quad][Cout][4 floats]
// (K-major no-swizzle) and streamed with 1-D bulk copies.
//
// Warp roles (384 threads): w0 weight (bulk) producer, w3 halo (TMA)
// producer, w1 MMA issuer, w2 TMEM allocator, w4..w11 epilogue (TMEM -> registers -> bias/ReLU/TF32 round ->
// global, optional fused 2x2x2 max-pool).  Two TMEM accumulator buffers let
// the epilogue of tile t overlap the MMAs of tile t+1.
#include <cuda.h>
#include <stdlib.h>
#include <string.h>

#include "async.cuh"
#include "unet_layout.cuh"

namespace mdp {
namespace tc {

using namespace ::mdp::async;

// Brick = ZP x 16 x 8 output voxels; ZP (output z-planes per brick) is a
// kernel template parameter: 2, or 4 for wide grids of Cout <= 64 layers
// (half the weight traffic per voxel, halo overhead 1.5x instead of 2x).
constexpr int BY = 16, BX = 8;
constexpr int HY = BY + 2, HX = BX + 2;
template <int ZP>
struct Brick {
  static constexpr int HZ = ZP + 2;
  static constexpr int QUAD_BYTES = HZ * HY * HX * 16;  // one quad plane of the halo brick
};

// Optional clock64 trace of CTA 0 (build with -DCONV_TRACE; tools/conv_trace.py): per tile the
// cycles at which each role passed its waits, for the launch whose (cin, cout) was selected.
#ifdef CONV_TRACE
__device__ long long g_trace[16 + 6 * 48 * 4];
__device__ int g_trace_sel[2];
#define TR(slot, ti, k)                                                                              \
  do {                                                                                               \
    if (blockIdx.x == 0 && (ti) < 48 && A.cin == g_trace_sel[0] && A.cout == g_trace_sel[1])         \
      g_trace[16 + ((slot) * 48 + (ti)) * 4 + (k)] = clock64();                                      \
  } while (0)
#else
#define TR(slot, ti, k) do { } while (0)
#endif

struct ConvArgs {
  int nb, S, cin, cout, cqc, nchunk;
  int nsplit, ncol;  // output channels split over nsplit CTAs of ncol each (small layers)
  int ksplit, cps;   // input-channel chunks split over ksplit CTAs of cps chunks (small layers)
  float4* partial;   // ksplit > 1: raw FP32 partial sums [ks][item][Cout/4][S^3]
  int tx, ty, tz, ntiles;
  int in_cq, in_q0;
  const float* w;
  const float* bias;
  int relu, epi;
  float4* out;
  int out_cq, out_q0, Sout;
  uint32_t a_bytes, b_bytes;
  int na, nbs;
  int resident;  // 1: the whole filter (27 taps, one chunk) stays in shared memory
  int tps;       // taps (fold: (dy,dx) units) per weight stage (one mbarrier handshake per stage)
  int fold;      // Cout == 32: the 3 z-taps of one (dy,dx) are one N = 3*32 weight block (see issue_stage_fold)
  uint32_t tmem_cols;
  int tail_wait;      // row-remainder launch: a programmatic dependent of the main launch that does NOT wait for it
                      // before working (same input, disjoint output rows) but before it exits (see tc_conv3)
  int perm, zoff;     // perm: the tensor map's dims are (x, z, y): the kernel's 16-line axis is the physical z and
                      // its plane axis the physical y, planes starting at zoff (remainder rows of odd grids)
  int pair;           // enc1a (Cin = 2): x-shifted input quads, one K = 8 MMA per (dy, halo plane) (see issue_stage_pair)
  const float* wraw;  // pair: the raw [16][2][27] filter, packed into shared memory by the kernel itself
  HeadArgs head;
};

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                            int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

// UMMA shared-memory descriptor, K-major, no swizzle (SM100 version 1).
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

// Start-address offset (16-byte units) of tap t's shifted view of the halo brick.
__host__ __device__ constexpr uint32_t tap_off16(int t) {
  return (uint32_t)(((t / 9) * HY + (t / 3) % 3) * HX + t % 3);
}

// Issue one weight stage: TPS taps x 2 K-steps (16-channel chunk = 2 x K8) x ZP
// z-planes, fully unrolled.  Descriptors are built once per stage; every MMA
// only adds compile-time constants to the 14-bit start-address fields
// (addresses < 256 KB, no carry), so the single issuing thread spends a few
// instructions per MMA instead of rebuilding 64-bit descriptors.
template <int TPS, int ZP>
__device__ __forceinline__ void issue_stage(uint32_t a_lo, uint32_t a_hi, uint32_t b_lo, uint32_t b_hi,
                                            uint32_t b_tap16, uint32_t b_ks16, uint32_t dcol, uint32_t ncol,
                                            uint32_t idesc, uint32_t& accf) {
  constexpr uint32_t Q16 = Brick<ZP>::QUAD_BYTES / 16;
#pragma unroll
  for (int tt = 0; tt < TPS; ++tt) {
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
      const uint64_t bd = ((uint64_t)b_hi << 32) | (b_lo + tt * b_tap16 + ks * b_ks16);
#pragma unroll
      for (int zp = 0; zp < ZP; ++zp) {  // one accumulator per z-plane
        const uint32_t off = tap_off16(tt) + (uint32_t)(zp * HY * HX) + (uint32_t)(ks * 2 * Q16);
        const uint64_t ad = ((uint64_t)a_hi << 32) | (a_lo + off);
        mma_tf32(dcol + zp * ncol, ad, bd, idesc, accf);
      }
      accf = 1u;
    }
  }
}

// Start-address offset (16-byte units) of (dy,dx) unit u's view of halo plane 0.
__host__ __device__ constexpr uint32_t unit_off16(int u) { return (uint32_t)((u / 3) * HX + u % 3); }

// z-tap fold (Cout <= 64 layers, A-operand-read bound at small N): for one
// (dy,dx) shift, halo plane hp feeds output planes zp in [hp-2, hp] through
// z-tap dz = hp - zp, so one A read serves up to three output planes with
// N = ndz * ncol.  Weights per unit are [quad][dz][ncol][4], so a dz range is
// a contiguous N range; accumulators are stored descending in zp (plane zp at
// column (ZP-1-zp)*ncol) so every MMA's D is one contiguous range.  The first
// MMAs of a tile (accumulate = 0) must initialise every accumulator exactly
// once: ZP = 2 starts with hp = 1 (planes 0-1); ZP = 4 with hp = 3 (planes
// 1-3) and hp = 0 (plane 0).
template <int ZP>
__device__ __forceinline__ constexpr int fold_hp(int h) {
  return ZP == 2 ? (h == 0 ? 1 : (h == 1 ? 0 : h)) : (h == 0 ? 3 : (h == 1 ? 0 : (h <= 3 ? h - 1 : h)));
}

template <int TPS, int ZP>
__device__ __forceinline__ void issue_stage_fold(uint32_t a_lo, uint32_t a_hi, uint32_t b_lo, uint32_t b_hi,
                                                 uint32_t b_unit16, uint32_t b_ks16, uint32_t dcol, uint32_t ncol,
                                                 const uint32_t* idesc_n, uint32_t& accf) {
  constexpr uint32_t Q16 = Brick<ZP>::QUAD_BYTES / 16;
  constexpr int NINIT = ZP == 2 ? 1 : 2;
  const uint32_t acc0 = accf;
#pragma unroll
  for (int tt = 0; tt < TPS; ++tt) {
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
#pragma unroll
      for (int h = 0; h < ZP + 2; ++h) {
        const int hp = fold_hp<ZP>(h);
        const int zlo = hp - 2 > 0 ? hp - 2 : 0, zhi = hp < ZP - 1 ? hp : ZP - 1;
        const int ndz = zhi - zlo + 1, dz_lo = hp - zhi;
        const uint32_t aoff = unit_off16(tt) + (uint32_t)(hp * HY * HX) + (uint32_t)(ks * 2 * Q16);
        const uint64_t ad = ((uint64_t)a_hi << 32) | (a_lo + aoff);
        const uint64_t bd = ((uint64_t)b_hi << 32) | (b_lo + tt * b_unit16 + ks * b_ks16 + dz_lo * ncol);
        const uint32_t a = (tt == 0 && ks == 0 && h < NINIT) ? acc0 : 1u;
        mma_tf32(dcol + (uint32_t)(ZP - 1 - zhi) * ncol, ad, bd, idesc_n[ndz - 1], a);
      }
    }
  }
  accf = 1u;
}

// enc1a (Cin = 2 -> 16): the input quad of voxel x is (r[x], d[x], r[x+1], d[x+1]), so with
// LBO = 16 B (the next x-voxel) one K = 8 step reads (r,d)[x-1], (r,d)[x], (r,d)[x], (r,d)[x+1]:
// all three dx taps of one (dz,dy) (weight slots 2-3 are zero).  With the z-tap fold the whole
// 54-term filter is 3 (dy) x (ZP+2) (halo planes) MMAs per brick; the layer is store-bound.
template <int ZP>
__device__ __forceinline__ void issue_stage_pair(uint32_t a_lo, uint32_t a_hi, uint32_t b_lo, uint32_t b_hi,
                                                 uint32_t b_unit16, uint32_t dcol, uint32_t ncol,
                                                 const uint32_t* idesc_n, uint32_t& accf) {
  constexpr int NINIT = ZP == 2 ? 1 : 2;
  const uint32_t acc0 = accf;
#pragma unroll
  for (int tt = 0; tt < 3; ++tt) {
#pragma unroll
    for (int h = 0; h < ZP + 2; ++h) {
      const int hp = fold_hp<ZP>(h);
      const int zlo = hp - 2 > 0 ? hp - 2 : 0, zhi = hp < ZP - 1 ? hp : ZP - 1;
      const int ndz = zhi - zlo + 1, dz_lo = hp - zhi;
      const uint64_t ad = ((uint64_t)a_hi << 32) | (a_lo + (uint32_t)(tt * HX + hp * HY * HX));
      const uint64_t bd = ((uint64_t)b_hi << 32) | (b_lo + tt * b_unit16 + dz_lo * ncol);
      mma_tf32(dcol + (uint32_t)(ZP - 1 - zhi) * ncol, ad, bd, idesc_n[ndz - 1], (tt == 0 && h < NINIT) ? acc0 : 1u);
    }
  }
  accf = 1u;
}

// One elected lane of a converged warp.  Unlike `lane == 0`, the compiler knows a single thread
// runs the guarded code, so descriptors move to uniform registers without a per-MMA
// ELECT / R2UR.BROADCAST / BRA.U.ANY waterfall loop (measured: ~70-110 -> cycles per issued MMA).
__device__ __forceinline__ bool elect_one() {
  uint32_t pred;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "elect.sync _|p, 0xffffffff;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}\n"
      : "=r"(pred));
  return pred != 0;
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

template <int ZP>
__device__ __forceinline__ void decode_tile(const ConvArgs& A, int tile, int& b, int& x0, int& y0, int& z0,
                                            int& n0, int& ks) {
  n0 = (tile % A.nsplit) * A.ncol;
  tile /= A.nsplit;
  ks = tile % A.ksplit;
  tile /= A.ksplit;
  int ix = tile % A.tx;
  int t = tile / A.tx;
  int iy = t % A.ty;
  t /= A.ty;
  int iz = t % A.tz;
  b = t / A.tz;
  x0 = ix * BX;
  y0 = iy * BY;
  z0 = iz * ZP + A.zoff;
}

template <int ZP>
__global__ void __launch_bounds__(384, 1) conv3_tc_kernel(const __grid_constant__ CUtensorMap tmap,
                                                          const __grid_constant__ CUtensorMap wmap,
                                                          const ConvArgs A) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;
  uint8_t* sB = sA + (size_t)A.na * A.a_bytes;
  uint64_t* bars = (uint64_t*)(sB + (size_t)A.nbs * A.b_bytes);
  uint64_t* a_full = bars;
  uint64_t* a_empty = a_full + A.na;
  uint64_t* b_full = a_empty + A.na;
  uint64_t* b_empty = b_full + A.nbs;
  uint64_t* t_full = b_empty + A.nbs;
  uint64_t* t_empty = t_full + 2;
  uint32_t* tmem_slot = (uint32_t*)(t_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#ifdef CONV_TRACE
  if (threadIdx.x == 0 && blockIdx.x == 0 && A.cin == g_trace_sel[0] && A.cout == g_trace_sel[1]) g_trace[0] = clock64();
#endif
  if (warp == 0 && lane == 0) {
    for (int i = 0; i < A.na; ++i) {
      mbar_init(&a_full[i], 1);
      mbar_init(&a_empty[i], 1);
    }
    for (int i = 0; i < A.nbs; ++i) {
      mbar_init(&b_full[i], 1);
      mbar_init(&b_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&t_full[i], 1);
      mbar_init(&t_empty[i], 256);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmap) : "memory");
    if (A.nsplit > 1) asm volatile("prefetch.tensormap [%0];" ::"l"(&wmap) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(A.tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_slot;
  // prologue (barriers, TMEM, tensor-map prefetch) overlapped with the previous grid; the
  // weights are never written on the device, so their producer (warp 0) streams the first
  // stages without waiting for it either
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (warp != 0 && !A.tail_wait) asm volatile("griddepcontrol.wait;" ::: "memory");
  const int nunits = A.pair ? 3 : (A.fold ? 9 : 27);

  if (warp == 3) {
    if (lane == 0) {  // ---------------- A producer: halo bricks, one TMA box per 32-channel chunk
      int as = 0, ap = 0, ti = 0;
      for (int tile = blockIdx.x; tile < A.ntiles; tile += gridDim.x, ++ti) {
        int b, x0, y0, z0, n0, ks;
        decode_tile<ZP>(A, tile, b, x0, y0, z0, n0, ks);
        for (int c = ks * A.cps; c < (ks + 1) * A.cps; ++c) {
          mbar_wait(&a_empty[as], ap ^ 1);
          if (c == ks * A.cps) TR(0, ti, 0);
          mbar_expect_tx(&a_full[as], A.a_bytes);
          // inner box row = 10 voxels x 4 channels (160 B); coordinate -4 floats = voxel x0-1
          tma_load_4d(sA + (size_t)as * A.a_bytes, &tmap, &a_full[as], 4 * (x0 - 1), y0 - 1, z0 - 1,
                      b * A.in_cq + A.in_q0 + c * A.cqc);
          if (++as == A.na) { as = 0; ap ^= 1; }
        }
      }
    }
  } else if (warp == 0 && A.pair) {
    // ---------------- pair mode: the 54 x 16 filter is packed here as [dy][kq][dz][cout][4]
    // (kq 0 = (w(dx0,r), w(dx0,d), 0, 0), kq 1 = (w(dx1,r), w(dx1,d), w(dx2,r), w(dx2,d))), TF32-rounded
    float* wb = reinterpret_cast<float*>(sB);
    for (int t = lane; t < 3 * 2 * 3 * 16 * 4; t += 32) {
      const int e = t & 3, c = (t >> 2) & 15, dz = (t >> 6) % 3, kq = ((t >> 6) / 3) & 1, dy = (t >> 6) / 6;
      const int ch = e & 1, dx = kq == 0 ? 0 : 1 + (e >> 1);
      const float v = (kq == 0 && e >= 2) ? 0.f : A.wraw[(c * 2 + ch) * 27 + (dz * 3 + dy) * 3 + dx];
      wb[t] = tf32_round(v);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) mbar_arrive(&b_full[0]);
  } else if (warp == 0) {
    if (lane == 0) {  // ---------------- B producer: weight tiles per (chunk, tap)
      int bs = 0, bp = 0;
      for (int tile = blockIdx.x; tile < A.ntiles; tile += gridDim.x) {
        if (A.resident && tile != (int)blockIdx.x) break;  // resident filter: loaded once
        int b, x0, y0, z0, n0, ks;
        decode_tile<ZP>(A, tile, b, x0, y0, z0, n0, ks);
        for (int c = ks * A.cps; c < (ks + 1) * A.cps; ++c) {
          // packed weights [chunk][tap][quad][cout][4] (fold: [chunk][dydx][quad][dz][cout][4]);
          // a stage holds tps consecutive units: one contiguous copy when the
          // CTA owns every output channel, else one per (tap, quad)
          const size_t tap_floats = (size_t)A.cqc * A.cout * 4 * (A.fold ? 3 : 1);
          const float* wc = A.w + (size_t)c * nunits * tap_floats;
          for (int t0 = 0; t0 < nunits; t0 += A.tps) {
            mbar_wait(&b_empty[bs], bp ^ 1);
            mbar_expect_tx(&b_full[bs], A.b_bytes);
            uint8_t* dst = sB + (size_t)bs * A.b_bytes;
            const float* src = wc + (size_t)t0 * tap_floats;
            if (A.nsplit == 1) {
              bulk_load(dst, src, A.b_bytes, &b_full[bs]);
            } else {
              // this CTA's ncol output channels of tps taps x cqc quads: one 2-D TMA box
              // (rows = (chunk, tap, quad), columns = this n-slice) lands as [tap][quad][ncol][4]
              tma_load_2d(dst, &wmap, &b_full[bs], n0 * 4, (c * nunits + t0) * A.cqc * (A.fold ? 3 : 1));
            }
            if (++bs == A.nbs) { bs = 0; bp ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (elect_one()) {  // ---------------- MMA issuer
      const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(A.ncol >> 3) << 17) |
                             ((uint32_t)(128 >> 4) << 24);
      const uint32_t lbo_a = A.pair ? 16u : Brick<ZP>::QUAD_BYTES, sbo_a = HX * 16;
      const uint32_t lbo_b = A.ncol * 16 * (A.fold ? 3 : 1), sbo_b = 128;
      uint32_t idesc_n[3];  // fold: N = 1, 2, 3 x ncol
      for (int k = 0; k < 3; ++k) idesc_n[k] = (idesc & ~(0x3Fu << 17)) | ((uint32_t)(((k + 1) * A.ncol) >> 3) << 17);
      const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
      int as = 0, ap = 0, bs = 0, bp = 0, li = 0;
      for (int tile = blockIdx.x; tile < A.ntiles; tile += gridDim.x, ++li) {
        const int buf = li & 1;
        mbar_wait(&t_empty[buf], ((li >> 1) & 1) ^ 1);
        fence_after();
        TR(1, li, 0);
        const uint32_t dcol = tmem + (uint32_t)(buf * ZP * A.ncol);
        uint32_t accf = 0u;  // the tile's first MMA overwrites the accumulator
        for (int c = 0; c < A.cps; ++c) {
          mbar_wait(&a_full[as], ap);
          fence_after();
          if (c == 0) TR(1, li, 1);
          const uint32_t abase = a0 + as * A.a_bytes;
          for (int t0 = 0; t0 < nunits; t0 += A.tps) {
            if (!A.resident || li == 0) {
              mbar_wait(&b_full[bs], bp);
              fence_after();
            }
            const uint64_t ad0 = umma_desc(abase + (A.fold ? unit_off16(t0) : tap_off16(t0)) * 16u, lbo_a, sbo_a);
            const uint64_t bd0 = umma_desc(b0 + bs * A.b_bytes, lbo_b, sbo_b);
            const uint32_t a_lo = (uint32_t)ad0, a_hi = (uint32_t)(ad0 >> 32);
            const uint32_t b_lo = (uint32_t)bd0, b_hi = (uint32_t)(bd0 >> 32);
            const uint32_t b_tap16 = (uint32_t)(A.cqc * A.ncol * (A.fold ? 3 : 1));  // one unit's weights / 16 B
            const uint32_t b_ks16 = (uint32_t)(2 * A.ncol * (A.fold ? 3 : 1));         // (2 * lbo_b) / 16
            if (A.pair) {
              issue_stage_pair<ZP>(a_lo, a_hi, b_lo, b_hi, 6u * A.ncol, dcol, A.ncol, idesc_n, accf);
            } else if (A.fold) {
              switch (A.tps) {
                case 9: issue_stage_fold<9, ZP>(a_lo, a_hi, b_lo, b_hi, b_tap16, b_ks16, dcol, A.ncol, idesc_n, accf); break;
                case 3: issue_stage_fold<3, ZP>(a_lo, a_hi, b_lo, b_hi, b_tap16, b_ks16, dcol, A.ncol, idesc_n, accf); break;
                default: issue_stage_fold<1, ZP>(a_lo, a_hi, b_lo, b_hi, b_tap16, b_ks16, dcol, A.ncol, idesc_n, accf); break;
              }
            } else {
              switch (A.tps) {
                case 27: issue_stage<27, ZP>(a_lo, a_hi, b_lo, b_hi, b_tap16, b_ks16, dcol, A.ncol, idesc, accf); break;
                case 9: issue_stage<9, ZP>(a_lo, a_hi, b_lo, b_hi, b_tap16, b_ks16, dcol, A.ncol, idesc, accf); break;
                case 3: issue_stage<3, ZP>(a_lo, a_hi, b_lo, b_hi, b_tap16, b_ks16, dcol, A.ncol, idesc, accf); break;
                default: issue_stage<1, ZP>(a_lo, a_hi, b_lo, b_hi, b_tap16, b_ks16, dcol, A.ncol, idesc, accf); break;
              }
            }
            if (!A.resident) mma_commit(&b_empty[bs]);
            if (++bs == A.nbs) { bs = 0; bp ^= 1; }
          }
          mma_commit(&a_empty[as]);
          if (++as == A.na) { as = 0; ap ^= 1; }
        }
        mma_commit(&t_full[buf]);
        TR(1, li, 2);
      }
    }
  } else if (warp >= 4) {  // ---------------- epilogue
    // 8 warps: warp w reads TMEM lane quarter w % 4; the two warps of a quarter split the
    // brick's (plane, 16-column group) items by parity (the epilogue is a dependent
    // instruction chain per warp: ncu showed the store-heavy layers bound by it at 4 warps)
    const int ew = (warp - 4) & 3, eh = (warp - 4) >> 2;
    const int row = ew * 32 + lane;
    const int ly = row >> 3, lx = row & 7;
    const uint32_t lane_addr = (uint32_t)(ew * 32) << 16;
    const int S = A.S;
    const int64_t S3 = (int64_t)S * S * S;
    const int So = A.Sout;
    const int64_t So3 = (int64_t)So * So * So;
    int li = 0;
    for (int tile = blockIdx.x; tile < A.ntiles; tile += gridDim.x, ++li) {
      const int buf = li & 1;
      int b, x0, y0, z0, n0, ks;
      decode_tile<ZP>(A, tile, b, x0, y0, z0, n0, ks);
      mbar_wait(&t_full[buf], (li >> 1) & 1);
      fence_after();
      if (lane == 0 && ew == 0) TR(2 + eh, li, 0);
      const uint32_t dcol = tmem + lane_addr + (uint32_t)(buf * ZP * A.ncol);
      const int q0 = A.out_q0 + n0 / 4;
      const int gx = x0 + lx, gy0 = y0 + ly;  // gy0: coordinate along the kernel's 16-line axis
      auto zcol = [&](int zp) { return (uint32_t)((A.fold ? ZP - 1 - zp : zp) * A.ncol); };
      if (A.ksplit > 1) {  // raw partial sums; conv_split_reduce_kernel finishes the layer
#pragma unroll
        for (int zp = 0; zp < ZP; ++zp) {
          const int gz = z0 + zp, gy = gy0;
          const bool ok = gx < S && gy < S && gz < S;
          for (int cg = 0; cg < A.ncol / 16; ++cg) {
            if (((zp * (A.ncol / 16) + cg) & 1) != eh) continue;
            float v[16];
            tmem_ld16(dcol + zcol(zp) + cg * 16, v);
            if (ok) {
#pragma unroll
              for (int q = 0; q < 4; ++q)
                A.partial[(((int64_t)ks * A.nb + b) * (A.cout / 4) + n0 / 4 + cg * 4 + q) * S3 +
                          ((int64_t)gz * S + gy) * S + gx] =
                    make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
            }
          }
        }
      } else if (A.epi == EPI_HEAD) {  // dec1 (ncol == cout == 32) -> head1 -> head2 -> ||r|| * y
        const HeadArgs& H = A.head;
        const int sys = sys_of(H.sel, b);
        const double rn = H.rnorm[b];
#pragma unroll
        for (int zp = 0; zp < ZP; ++zp) {
          if ((zp & 1) != eh) continue;
          const int gz = A.perm ? gy0 : z0 + zp, gy = A.perm ? z0 + zp : gy0;  // physical (y, z)
          const bool ok = gx < S && gy < S && gz < S;
          float v[32];
          tmem_ld16(dcol + zcol(zp), v);
          tmem_ld16(dcol + zcol(zp) + 16, v + 16);
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            float m = v[i];
            if (A.bias) m += A.bias[i];
            if (A.relu) m = fmaxf(m, 0.f);
            v[i] = tf32_round(m);
          }
          if (ok) {
            const float y = head_eval(v, H.w1, H.b1, H.w2, H.b2);
            double* zp = H.z + sys * H.ldz + ((int64_t)gz * S + gy) * S + gx;
            *zp = H.accumulate ? *zp + rn * (double)y : rn * (double)y;
          }
        }
      } else if (A.epi == EPI_POOL) {
        const int px = gx >> 1, py = gy0 >> 1;
#pragma unroll
        for (int pp = 0; pp < ZP / 2; ++pp) {  // pooled plane from output planes 2pp, 2pp+1
          const int pz = (z0 >> 1) + pp;
          const bool writer = ((lane & 1) == 0) && ((ly & 1) == 0) && px < So && py < So && pz < So;
          for (int cg = 0; cg < A.ncol / 16; ++cg) {
            if (((pp * (A.ncol / 16) + cg) & 1) != eh) continue;
            float v0[16], v1[16];
            tmem_ld16(dcol + zcol(2 * pp) + cg * 16, v0);
            tmem_ld16(dcol + zcol(2 * pp + 1) + cg * 16, v1);
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              float m = fmaxf(v0[i], v1[i]);
              m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 1));
              m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 8));
              if (A.bias) m += A.bias[n0 + cg * 16 + i];
              if (A.relu) m = fmaxf(m, 0.f);
              v0[i] = tf32_round(m);
            }
            if (writer) {
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                float4 o = make_float4(v0[4 * q], v0[4 * q + 1], v0[4 * q + 2], v0[4 * q + 3]);
                A.out[((int64_t)b * A.out_cq + q0 + cg * 4 + q) * So3 + ((int64_t)pz * So + py) * So + px] = o;
              }
            }
          }
        }
      } else {
#pragma unroll
        for (int zp = 0; zp < ZP; ++zp) {
          const int gz = A.perm ? gy0 : z0 + zp, gy = A.perm ? z0 + zp : gy0;  // physical (y, z)
          const bool ok = gx < S && gy < S && gz < S;
          for (int cg = 0; cg < A.ncol / 16; ++cg) {
            if (((zp * (A.ncol / 16) + cg) & 1) != eh) continue;
            float v[16];
            tmem_ld16(dcol + zcol(zp) + cg * 16, v);
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              float m = v[i];
              if (A.bias) m += A.bias[n0 + cg * 16 + i];
              if (A.relu) m = fmaxf(m, 0.f);
              v[i] = tf32_round(m);
            }
            if (ok) {
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                float4 o = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
                A.out[((int64_t)b * A.out_cq + q0 + cg * 4 + q) * S3 + ((int64_t)gz * S + gy) * S + gx] = o;
              }
            }
          }
        }
      }
      fence_before();
      if (lane == 0 && ew == 0) TR(2 + eh, li, 1);
      mbar_arrive(&t_empty[buf]);
    }
  }
  __syncwarp();
  fence_before();
  __syncthreads();
  fence_after();
  if (warp == 2) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(A.tmem_cols));
  }
  // the remainder launch ran beside the main launch's tail; it may only COMPLETE after it, so that the next
  // kernel in the stream (which waits for this grid) sees both
  if (A.tail_wait) asm volatile("griddepcontrol.wait;" ::: "memory");
#ifdef CONV_TRACE
  if (threadIdx.x == 0 && blockIdx.x == 0 && A.cin == g_trace_sel[0] && A.cout == g_trace_sel[1]) g_trace[1] = clock64();
#endif
}

// Fixed-order sum of the ksplit partials + bias + ReLU (+ 2x2x2 max pool) +
// TF32 rounding into the output slot (deterministic: the split count depends
// on the layer shape, never on the batch).
__global__ void conv_split_reduce_kernel(const float4* __restrict__ part, int ksplit, int nb, int cq, int S,
                                         const float* __restrict__ bias, int relu, int pool, float4* __restrict__ out,
                                         int out_cq, int out_q0) {
  MDP_PDL_ENTER();
  const int So = pool ? S / 2 : S;
  const int64_t S3 = (int64_t)S * S * S, So3 = (int64_t)So * So * So;
  const int64_t total = (int64_t)nb * cq * So3;
  const int64_t kstride = (int64_t)nb * cq * S3;
  // pool: 8 lanes per output quad, one 2x2x2 window voxel each (the split-K sums
  // run in parallel; the max over the window is exact in any order); the loop
  // trip count is warp-uniform so the shuffles see all 32 lanes
  const int wlog = pool ? 3 : 0;
  const int lane = threadIdx.x & 31;
  const int64_t items = total << wlog;
  for (int64_t t0 = blockIdx.x * (int64_t)blockDim.x + (threadIdx.x - lane); t0 < items;
       t0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = t0 + lane;
    const bool live = t < items;
    const int64_t o = live ? t >> wlog : 0;
    const int d = pool ? (int)(t & 7) : 0;
    const int64_t v = o % So3;
    const int64_t bq = o / So3;
    const int q = bq % cq, b = bq / cq;
    const int x = v % So, y = (v / So) % So, z = v / ((int64_t)So * So);
    const int xx = pool ? 2 * x + (d & 1) : x, yy = pool ? 2 * y + ((d >> 1) & 1) : y, zz = pool ? 2 * z + (d >> 2) : z;
    const int64_t vi = ((int64_t)zz * S + yy) * S + xx;
    const float4* pp = part + ((int64_t)b * cq + q) * S3 + vi;
    float4 m = make_float4(0.f, 0.f, 0.f, 0.f);
    if (live) {
      m = pp[0];
#pragma unroll 4
      for (int k = 1; k < ksplit; ++k) {
        const float4 p = pp[k * kstride];
        m.x += p.x; m.y += p.y; m.z += p.z; m.w += p.w;
      }
    }
    if (pool) {
#pragma unroll
      for (int off = 1; off < 8; off <<= 1) {
        m.x = fmaxf(m.x, __shfl_xor_sync(0xffffffffu, m.x, off));
        m.y = fmaxf(m.y, __shfl_xor_sync(0xffffffffu, m.y, off));
        m.z = fmaxf(m.z, __shfl_xor_sync(0xffffffffu, m.z, off));
        m.w = fmaxf(m.w, __shfl_xor_sync(0xffffffffu, m.w, off));
      }
    }
    if (!live || d != 0) continue;
    const float4 bb = bias ? make_float4(bias[4 * q], bias[4 * q + 1], bias[4 * q + 2], bias[4 * q + 3])
                           : make_float4(0.f, 0.f, 0.f, 0.f);
    m.x += bb.x; m.y += bb.y; m.z += bb.z; m.w += bb.w;
    if (relu) m = make_float4(fmaxf(m.x, 0.f), fmaxf(m.y, 0.f), fmaxf(m.z, 0.f), fmaxf(m.w, 0.f));
    out[((int64_t)b * out_cq + out_q0 + q) * So3 + v] = tf32_round4(m);
  }
}

// EPI_HEAD after split-K: fixed-order partial sum of the 32 dec1 channels of
// one voxel + bias + ReLU + TF32 rounding, then the heads and ||r|| scaling.
__global__ void conv_split_reduce_head_kernel(const float4* __restrict__ part, int ksplit, int nb, int S,
                                              const float* __restrict__ bias, int relu, const HeadArgs H) {
  MDP_PDL_ENTER();
  const int64_t S3 = (int64_t)S * S * S;
  const int64_t total = (int64_t)nb * S3;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = t % S3;
    const int b = t / S3;
    float d[32];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      float4 acc = part[((int64_t)b * 8 + q) * S3 + v];
      for (int k = 1; k < ksplit; ++k) {
        const float4 p = part[(((int64_t)k * nb + b) * 8 + q) * S3 + v];
        acc.x += p.x; acc.y += p.y; acc.z += p.z; acc.w += p.w;
      }
      const float a[4] = {acc.x, acc.y, acc.z, acc.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float m = a[e];
        if (bias) m += bias[4 * q + e];
        if (relu) m = fmaxf(m, 0.f);
        d[4 * q + e] = tf32_round(m);
      }
    }
    const float y = head_eval(d, H.w1, H.b1, H.w2, H.b2);
    double* zp = H.z + sys_of(H.sel, b) * H.ldz + v;
    *zp = H.accumulate ? *zp + H.rnorm[b] * (double)y : H.rnorm[b] * (double)y;
  }
}

// ---------------------------------------------------------------------------
// Transposed conv k=2 s=2 (neural.py:215-246) as tcgen05 GEMMs: every output
// voxel takes exactly one tap, so per tap it is [input voxels x Cin] x [Cin x
// Cout].  Persistent CTAs, one group of tg taps each: the group's weights
// ([tap][quad][Cout][4]) are loaded once; a producer warp streams 128-voxel
// M-tiles (cin/4 quad rows of 2 KB, 1-D bulk copies, already K-major core
// matrices of 8 voxels x 16 B) into a double buffer; one thread issues a
// K-chain per tap into the tile's TMEM buffer (double-buffered); four
// epilogue warps scatter each tap's row to output voxel (2x+a, 2y+b, 2z+c)
// while the next tile's MMAs run.  Tail blocks write the output-padding planes.
struct TconvArgs {
  const float4* in;
  int in_cq, cin, cout, Sin, op, tg, nmain, nb, ntiles, ncta;
  const float* w;
  const float* bias;
  float4* out;
  int out_cq, out_q0;
  uint32_t a_bytes, b_bytes, tmem_cols;
};

__global__ void __launch_bounds__(320, 1) tconv_tc_kernel(const TconvArgs T) {
  MDP_PDL_ENTER();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const int grp = blockIdx.y;
  if ((int)blockIdx.x >= T.ncta) {  // tail blocks: output-padding planes
    if (grp == 0)
      for (int b = 0; b < T.nb; ++b)
        tconv_pad(T.Sin, T.cout, T.bias, T.out, T.out_cq, T.out_q0, b,
                  (blockIdx.x - T.ncta) * (int64_t)blockDim.x + threadIdx.x,
                  (int64_t)(gridDim.x - T.ncta) * blockDim.x, 1);
    return;
  }
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sB = smem;
  uint8_t* sA = sB + T.b_bytes;  // two A buffers
  uint64_t* bfull = (uint64_t*)(sA + 2 * (size_t)T.a_bytes);
  uint64_t* afull = bfull + 1;
  uint64_t* aempty = afull + 2;
  uint64_t* tfull = aempty + 2;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = (uint32_t*)(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int Sin = T.Sin;
  const int64_t nvi = (int64_t)Sin * Sin * Sin;
  const int nq = T.cin / 4;
  if (threadIdx.x == 0) {
    mbar_init(bfull, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&afull[i], 1);
      mbar_init(&aempty[i], 1);
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], blockDim.x - 64);  // every epilogue thread (4 or 8 warps) arrives
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(T.tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tstride = (uint32_t)(T.tg * T.cout);  // TMEM columns per tile buffer
  if (warp == 0) {
    if (lane == 0) {  // ---- producer: weights once, then the voxel rows of each tile
      mbar_expect_tx(bfull, T.b_bytes);
      bulk_load(sB, T.w + (size_t)grp * T.tg * T.cin * T.cout, T.b_bytes, bfull);
      int it = 0;
      for (int tile = blockIdx.x; tile < T.ntiles; tile += T.ncta, ++it) {
        const int buf = it & 1;
        mbar_wait(&aempty[buf], ((it >> 1) & 1) ^ 1);
        const int b = tile / T.nmain;
        const int64_t v0 = (int64_t)(tile % T.nmain) * 128;
        const uint32_t rowb = (uint32_t)(nvi - v0 < 128 ? nvi - v0 : 128) * 16u;
        mbar_expect_tx(&afull[buf], rowb * nq);
        uint8_t* dst = sA + (size_t)buf * T.a_bytes;
        for (int q = 0; q < nq; ++q)
          bulk_load(dst + (size_t)q * 2048, T.in + ((int64_t)b * T.in_cq + q) * nvi + v0, rowb, &afull[buf]);
      }
    }
  } else if (warp == 1) {
    if (elect_one()) {  // ---- MMA issuer
      const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(T.cout >> 3) << 17) |
                             ((uint32_t)(128 >> 4) << 24);
      const uint32_t b0 = smem_u32(sB);
      mbar_wait(bfull, 0);
      int it = 0;
      for (int tile = blockIdx.x; tile < T.ntiles; tile += T.ncta, ++it) {
        const int buf = it & 1;
        mbar_wait(&afull[buf], (it >> 1) & 1);
        mbar_wait(&tempty[buf], ((it >> 1) & 1) ^ 1);
        fence_after();
        const uint32_t a0 = smem_u32(sA + (size_t)buf * T.a_bytes);
        const uint32_t d0 = tmem + (uint32_t)buf * tstride;
        for (int t = 0; t < T.tg; ++t)
          for (int ks = 0; ks < nq / 2; ++ks) {
            const uint64_t ad = umma_desc(a0 + ks * 2 * 2048, 2048, 128);
            const uint64_t bd = umma_desc(b0 + (uint32_t)((t * nq + 2 * ks) * T.cout * 16), T.cout * 16, 128);
            mma_tf32(d0 + (uint32_t)(t * T.cout), ad, bd, idesc, ks > 0 ? 1u : 0u);
          }
        mma_commit(&aempty[buf]);  // voxel rows reusable once these MMAs have read them
        mma_commit(&tfull[buf]);
      }
    }
  } else {  // ---- epilogue warps 2..5: TMEM lanes 32 (warp % 4) ..
    const int quarter = warp & 3;
    // 8 epilogue warps (wide inputs): warps 2-5 / 6-9, the two warps of a TMEM lane quarter split the tile's
    // items by parity (65^3: both transposed convs 36 -> 28 us); small inputs launch 4 (33^3: 16 vs 18 us with 8)
    const bool two = blockDim.x > 192;
    const int eh = (warp - 2) >> 2;
    const int row = quarter * 32 + lane;
    const uint32_t lane_addr = (uint32_t)(quarter * 32) << 16;
    const int So = 2 * Sin + T.op;
    const int64_t nvo = (int64_t)So * So * So;
    int it = 0;
    for (int tile = blockIdx.x; tile < T.ntiles; tile += T.ncta, ++it) {
      const int buf = it & 1;
      const int b = tile / T.nmain;
      const int64_t v = (int64_t)(tile % T.nmain) * 128 + row;
      const bool live = v < nvi;
      const int x = live ? (int)(v % Sin) : 0, y = live ? (int)((v / Sin) % Sin) : 0,
                z = live ? (int)(v / ((int64_t)Sin * Sin)) : 0;
      mbar_wait(&tfull[buf], (it >> 1) & 1);
      fence_after();
      const uint32_t d0 = tmem + lane_addr + (uint32_t)buf * tstride;
      if (T.tg >= 2) {
        // taps t, t + 1 differ in a only: output voxels 2x and 2x + 1 are the two 16-byte halves of
        // one 32-byte run, written back to back so L2 sees both halves of a sector together
        for (int t = 0; t < T.tg; t += 2) {
          const int tap = grp * T.tg + t;
          const int64_t o = ((int64_t)(2 * z + (tap >> 2)) * So + 2 * y + ((tap >> 1) & 1)) * So + 2 * x;
          for (int cg = 0; cg < T.cout / 16; ++cg) {
            if (two && (((t >> 1) * (T.cout / 16) + cg) & 1) != eh) continue;
            float r0[16], r1[16];
            tmem_ld16(d0 + (uint32_t)(t * T.cout + cg * 16), r0);
            tmem_ld16(d0 + (uint32_t)((t + 1) * T.cout + cg * 16), r1);
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const float bi = T.bias ? T.bias[cg * 16 + i] : 0.f;
              r0[i] = tf32_round(fmaxf(r0[i] + bi, 0.f));
              r1[i] = tf32_round(fmaxf(r1[i] + bi, 0.f));
            }
            if (live)
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                float4* dst = T.out + ((int64_t)b * T.out_cq + T.out_q0 + cg * 4 + q) * nvo + o;
                dst[0] = make_float4(r0[4 * q], r0[4 * q + 1], r0[4 * q + 2], r0[4 * q + 3]);
                dst[1] = make_float4(r1[4 * q], r1[4 * q + 1], r1[4 * q + 2], r1[4 * q + 3]);
              }
          }
        }
        fence_before();
        mbar_arrive(&tempty[buf]);
        continue;
      }
      for (int t = 0; t < T.tg; ++t) {
        const int tap = grp * T.tg + t;
        const int64_t o = ((int64_t)(2 * z + (tap >> 2)) * So + 2 * y + ((tap >> 1) & 1)) * So + 2 * x + (tap & 1);
        for (int cg = 0; cg < T.cout / 16; ++cg) {
          if (two && ((t * (T.cout / 16) + cg) & 1) != eh) continue;
          float r[16];
          tmem_ld16(d0 + (uint32_t)(t * T.cout + cg * 16), r);
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            float m = r[i];
            if (T.bias) m += T.bias[cg * 16 + i];
            r[i] = tf32_round(fmaxf(m, 0.f));
          }
          if (live)
#pragma unroll
            for (int q = 0; q < 4; ++q)
              T.out[((int64_t)b * T.out_cq + T.out_q0 + cg * 4 + q) * nvo + o] =
                  make_float4(r[4 * q], r[4 * q + 1], r[4 * q + 2], r[4 * q + 3]);
        }
      }
      fence_before();
      mbar_arrive(&tempty[buf]);
    }
  }
  __syncwarp();
  fence_before();
  __syncthreads();
  fence_after();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(T.tmem_cols));
}

}  // namespace tc
}  // namespace mdp
#ifdef CONV_TRACE
extern "C" int mdp_conv_trace_select(int cin, int cout) {
  int sel[2] = {cin, cout};
  cudaMemset(nullptr, 0, 0);
  static long long zero[16 + 6 * 48 * 4] = {0};
  cudaMemcpyToSymbol(mdp::tc::g_trace, zero, sizeof(zero));
  return (int)cudaMemcpyToSymbol(mdp::tc::g_trace_sel, sel, sizeof(sel));
}
extern "C" int mdp_conv_trace_read(long long* host) {
  return (int)cudaMemcpyFromSymbol(host, mdp::tc::g_trace, sizeof(long long) * (16 + 6 * 48 * 4));
}
#endif
namespace mdp {
namespace tc {

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFn)p;
  }
  return fn;
}

}  // namespace tc

// Split decisions for one layer shape (shared by the launch and the workspace plan).
static void tc_split(int nb, int S, int cin, int cout, int& nsplit, int& ksplit) {
  using namespace tc;
  const int tiles_item = ceil_div(S, BX) * ceil_div(S, BY) * ceil_div(S, 2);  // decided on 2-plane bricks
  const int nchunk = cin / 16;
#ifndef CONV_MIN_NCOL
#define CONV_MIN_NCOL 32  // narrowest output-channel slice of a split-N CTA (A/B: 64 is 1.2% faster at cfg2 but moves the cfg1 early residual history to 2.5e-4 of the reference)
#endif
  nsplit = 1;
  while (nb * tiles_item * nsplit < sm_count() && cout / (2 * nsplit) >= CONV_MIN_NCOL) nsplit *= 2;
  // split-K only from the per-item shape so the FP32 summation order (hence
  // the result) is independent of the batch size
  int nsplit_item = 1;
  while (tiles_item * nsplit_item < sm_count() && cout / (2 * nsplit_item) >= CONV_MIN_NCOL) nsplit_item *= 2;
  ksplit = 1;
#ifndef CONV_SPLITK
#define CONV_SPLITK 1
#endif
#ifndef CONV_SPLITK_WAVES
#define CONV_SPLITK_WAVES 1  // target CTAs = waves x SMs
#endif
  const int want = (CONV_SPLITK_WAVES * sm_count() + tiles_item * nsplit_item - 1) / (tiles_item * nsplit_item);
  if (CONV_SPLITK && tiles_item * nsplit_item * 2 <= sm_count())
    for (int k = nchunk; k >= 2; --k)
      if (nchunk % k == 0 && k <= want) {
        ksplit = k;
        break;
      }
}

static void conv3_smem_attr() {
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(tc::conv3_tc_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(227 * 1024));
    cudaFuncSetAttribute(tc::conv3_tc_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(227 * 1024));
    attr_set = true;
  }
}

size_t tc_conv3_scratch_bytes(int nb, int S, int cin, int cout) {
  int ns, ks;
  tc_split(nb, S, cin, cout, ns, ks);
  return ks > 1 ? (size_t)ks * nb * cout * S * S * S * sizeof(float) : 0;
}

int tc_conv3(int nb, int S, int cin, int cout, const float4* in, int in_cq, int in_q0, const float* w,
             const float* bias, int relu, float4* out, int out_cq, int out_q0, int epi, const HeadArgs* head,
             void* scratch, size_t scratch_bytes, cudaStream_t st) {
  using namespace tc;
  MDP_REQUIRE(cin % 16 == 0 && cin >= 16, "tc conv needs cin multiple of 16, got %d", cin);
  MDP_REQUIRE(cout % 16 == 0 && cout >= 16 && cout <= 128, "tc conv needs cout in {16..128} step 16, got %d",
              cout);
  MDP_REQUIRE(epi == EPI_STORE || epi == EPI_POOL || epi == EPI_HEAD, "epilogue %d not supported by tc conv", epi);
  MDP_REQUIRE(epi != EPI_HEAD || (cout == 32 && head != nullptr), "fused head needs cout == 32 and head weights");
  EncodeTiledFn enc = encode_fn();
  MDP_REQUIRE(enc != nullptr, "cuTensorMapEncodeTiled unavailable");
  ConvArgs A{};
  A.nb = nb;
  A.S = S;
  A.cin = cin;
  A.cout = cout;
  A.cqc = 4;  // 16-channel chunks: a 46 KB halo per stage leaves room for deep multi-tap weight stages
  A.nchunk = cin / (4 * A.cqc);
  // floor pooling (neural.py:275-290) never reads output plane / row / column
  // 2*(S/2): pooled layers only compute [0, 2*(S/2))^3 (S = 33: 128 instead of
  // 255 bricks, one round on 148 SMs); halo loads still see the full input
  const int Sc = epi == EPI_POOL ? 2 * (S / 2) : S;
  A.tx = ceil_div(Sc, BX);
  A.ty = ceil_div(Sc, BY);
  // small layers (few bricks): split the output channels over CTAs (down to
  // 32 per CTA) and, if still short of the SM count, the input chunks
  tc_split(nb, S, cin, cout, A.nsplit, A.ksplit);
  A.ncol = cout / A.nsplit;
  // Grids of 2^k + 1 points: the last y-row alone would cost a whole 16-line tile row (+12% bricks at
  // 129^3, +25% at 65^3).  Rows [16 floor(S/16), S) are computed by a second launch of the same kernel on a
  // tensor map with y and z exchanged (and the dy <-> dz permuted weight copy behind the first one): there
  // the 16-line axis runs along z and the 1-2 left-over rows are the plane axis.  Per-item shape only.
  static const int rem_env = [] { const char* e = getenv("MDP_CONV_REMAINDER"); return e ? atoi(e) : 1; }();
  static const int rem_min = [] { const char* e = getenv("MDP_CONV_REMAINDER_MIN"); return e ? atoi(e) : 4; }();
  const int yrem = S % BY;
  // (only where the main grid is several rounds deep per item: the second launch costs ~15 us of its own;
  // measured 129^3 forward -2.1%, 65^3 x 16 -7.7% (cfg3 solve +5.8%), one 65^3 item +3%, 33^3 +17%: the
  // threshold of 4 bricks per SM takes 65^3 in -- its use is the batched multi-query solve -- and leaves 33^3 out)
  const bool split_rows = rem_env && cout <= 64 && epi != EPI_POOL && A.nsplit == 1 && A.ksplit == 1 &&
                          yrem >= 1 && yrem <= 2 &&
                          (int64_t)A.tx * (S / BY) * ceil_div(S, 4) >= rem_min * (int64_t)sm_count();
  if (split_rows) A.ty = S / BY;
  // z-tap fold for Cout <= 64 (weights packed [chunk][dydx][quad][dz][Cout][4]);
  // 4-plane bricks when the layer still has >= 2 bricks per SM with them
  A.fold = cout <= 64;
  // decided from the per-item shape only (like split-K): the brick depth sets the
  // FP32 accumulation order, so batched == serial stays bitwise (training.py:322-338)
  const int zp = (A.fold && A.ksplit == 1 && (int64_t)A.tx * A.ty * ceil_div(Sc, 4) >= 2 * sm_count()) ? 4 : 2;
  A.tz = ceil_div(Sc, zp);
  // likewise the plane remainder of 4-plane bricks (S = 4 k + 1: the last brick of every column would
  // carry one useful plane of four): planes [4 floor(S/4), S) go to a third, 2-plane launch
  const int zrem = S % 4;
  const bool split_planes = split_rows && zp == 4 && zrem >= 1 && zrem <= 2;
  if (split_planes) A.tz = S / 4;
  const int spatial = nb * A.tx * A.ty * A.tz;
  A.cps = A.nchunk / A.ksplit;
  A.ntiles = spatial * A.nsplit * A.ksplit;
  A.partial = (float4*)scratch;
  if (A.ksplit > 1)
    MDP_REQUIRE(scratch && scratch_bytes >= tc_conv3_scratch_bytes(nb, S, cin, cout),
                "split-K conv needs %zu bytes of scratch", tc_conv3_scratch_bytes(nb, S, cin, cout));
  A.in_cq = in_cq;
  A.in_q0 = in_q0;
  A.w = w;
  A.bias = bias;
  A.relu = relu;
  A.epi = epi;
  A.out = out;
  A.out_cq = out_cq;
  A.out_q0 = out_q0;
  A.Sout = epi == EPI_POOL ? S / 2 : S;
  A.a_bytes = (uint32_t)A.cqc * (zp == 4 ? Brick<4>::QUAD_BYTES : Brick<2>::QUAD_BYTES);
  A.na = 2;
  const size_t budget = 227 * 1024 - 2048 - 1024;
  const int nunits = A.fold ? 9 : 27;
  const size_t tap_bytes = (size_t)A.cqc * A.ncol * 16 * (A.fold ? 3 : 1);  // one weight unit
  A.resident = 0;
  int nbs = 0;
  if (A.cps == 1 && A.ksplit == 1 && (size_t)A.na * A.a_bytes + nunits * tap_bytes <= budget) {
    A.resident = 1;  // e.g. enc1b: the 27-tap filter fits next to the halo double buffer
    A.tps = nunits;
    nbs = 1;
  } else {
    // as many taps per stage as leave >= 3 stages: each barrier handshake must
    // cover enough MMA work to hide its ~500-cycle round trip
    const int opts[3] = {9, 3, 1};
    for (int o = 0; o < 3 && nbs == 0; ++o) {
      A.tps = opts[o];
      int k = (int)((budget - (size_t)A.na * A.a_bytes) / (tap_bytes * A.tps));
      if (k >= 3 || (o == 2 && k >= 2)) nbs = k > 8 ? 8 : k;
    }
  }
  A.b_bytes = (uint32_t)(tap_bytes * A.tps);
  A.nbs = nbs;
  MDP_REQUIRE((size_t)A.na * A.a_bytes + (size_t)nbs * A.b_bytes <= budget, "tc conv tile does not fit smem");
  uint32_t cols = 32;
  while (cols < (uint32_t)(2 * zp * A.ncol)) cols <<= 1;
  MDP_REQUIRE(cols <= 512, "conv accumulators need %u TMEM columns", cols);
  A.tmem_cols = cols;
  if (head) A.head = *head;

  // 4-D view of the quad-blocked activations: (x * 4 + channel, y, z, item * CQ + quad);
  // the innermost box row is a whole 10-voxel x-run (160 B) of one quad
  CUtensorMap map;
  cuuint64_t gdim[4] = {(cuuint64_t)4 * S, (cuuint64_t)S, (cuuint64_t)S, (cuuint64_t)nb * in_cq};
  cuuint64_t gstride[3] = {(cuuint64_t)16 * S, (cuuint64_t)16 * S * S, (cuuint64_t)16 * S * S * S};
  cuuint32_t box[4] = {4 * HX, HY, (cuuint32_t)(zp + 2), (cuuint32_t)A.cqc};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, (void*)in, gdim, gstride, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  MDP_REQUIRE(r == CUDA_SUCCESS, "cuTensorMapEncodeTiled failed (%d) for S=%d cin=%d", (int)r, S, cin);

  // weights as a 2-D tensor (row = (chunk, tap, quad), Cout*4 floats per row) for
  // the split-N case: one TMA box per weight stage instead of one copy per (tap, quad)
  CUtensorMap wmap;
  memset(&wmap, 0, sizeof(wmap));
  if (A.nsplit > 1) {
    // rows: (chunk, tap, quad), or with the fold (chunk, dydx, quad, dz) -- 27 x cqc per chunk either way
    cuuint64_t wdim[2] = {(cuuint64_t)cout * 4, (cuuint64_t)A.nchunk * 27 * A.cqc};
    cuuint64_t wstride[1] = {(cuuint64_t)cout * 16};
    cuuint32_t wbox[2] = {(cuuint32_t)A.ncol * 4, (cuuint32_t)(A.tps * A.cqc * (A.fold ? 3 : 1))};
    cuuint32_t westr[2] = {1, 1};
    CUresult rw = enc(&wmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)w, wdim, wstride, wbox, westr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    MDP_REQUIRE(rw == CUDA_SUCCESS, "cuTensorMapEncodeTiled failed (%d) for the weights", (int)rw);
  }

  const size_t smem = 1024 + (size_t)A.na * A.a_bytes + (size_t)nbs * A.b_bytes + 2048;
  conv3_smem_attr();
  MDP_REQUIRE(smem <= 227 * 1024, "tc conv needs %zu bytes of shared memory", smem);
  int grid = A.ntiles < sm_count() ? A.ntiles : sm_count();
  if (zp == 4)
    ::mdp::launch_k(conv3_tc_kernel<4>, grid, 384, smem, st, map, wmap, A);
  else
    ::mdp::launch_k(conv3_tc_kernel<2>, grid, 384, smem, st, map, wmap, A);
  MDP_LAUNCH_CHECK("conv3_tc_kernel");
  if (split_rows) {
    ConvArgs B = A;
    B.perm = 1;
    B.zoff = (S / BY) * BY;
    B.ty = ceil_div(S, BY);  // 16-line tiles along the physical z
    B.tz = 1;                // the 1-2 left-over rows as the planes of a 2-plane brick
    B.ntiles = nb * B.tx * B.ty * B.tz;
    B.w = w + (size_t)cin * cout * 27;  // the dy <-> dz permuted pack (neural.pack_conv)
    B.a_bytes = (uint32_t)B.cqc * Brick<2>::QUAD_BYTES;
    CUtensorMap pmap;
    cuuint64_t pstride[3] = {(cuuint64_t)16 * S * S, (cuuint64_t)16 * S, (cuuint64_t)16 * S * S * S};
    cuuint32_t pbox[4] = {4 * HX, HY, 4, (cuuint32_t)B.cqc};
    CUresult rp = enc(&pmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, (void*)in, gdim, pstride, pbox, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    MDP_REQUIRE(rp == CUDA_SUCCESS, "cuTensorMapEncodeTiled failed (%d) for the row remainder of S=%d", (int)rp, S);
    const size_t smem2 = 1024 + (size_t)B.na * B.a_bytes + (size_t)nbs * B.b_bytes + 2048;
    const int grid2 = B.ntiles < sm_count() ? B.ntiles : sm_count();
    static const int overlap = [] { const char* e = getenv("MDP_CONV_REMAINDER_OVERLAP"); return e ? atoi(e) : 1; }();
    if (overlap) {
      // its CTAs take the SMs the main launch's last round leaves idle (4488 bricks on 148 SMs: a
      // one-brick tail on 70% of them)
      B.tail_wait = 1;
      ::mdp::launch_k_dependent(conv3_tc_kernel<2>, grid2, 384, smem2, st, pmap, wmap, B);
    } else {
      ::mdp::launch_k(conv3_tc_kernel<2>, grid2, 384, smem2, st, pmap, wmap, B);
    }
    MDP_LAUNCH_CHECK("conv3_tc_kernel (row remainder)");
    if (split_planes) {
      ConvArgs C = A;  // normal orientation, rows below the row remainder, the last 1-2 planes
      C.zoff = (S / 4) * 4;
      C.tz = 1;
      C.ntiles = nb * C.tx * C.ty * C.tz;
      C.a_bytes = (uint32_t)C.cqc * Brick<2>::QUAD_BYTES;
      C.tail_wait = overlap ? 1 : 0;
      CUtensorMap zmap;
      CUresult rz = enc(&zmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, (void*)in, gdim, gstride, pbox, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      MDP_REQUIRE(rz == CUDA_SUCCESS, "cuTensorMapEncodeTiled failed (%d) for the plane remainder of S=%d", (int)rz, S);
      const int grid3 = C.ntiles < sm_count() ? C.ntiles : sm_count();
      if (overlap)
        ::mdp::launch_k_dependent(conv3_tc_kernel<2>, grid3, 384, smem2, st, zmap, wmap, C);
      else
        ::mdp::launch_k(conv3_tc_kernel<2>, grid3, 384, smem2, st, zmap, wmap, C);
      MDP_LAUNCH_CHECK("conv3_tc_kernel (plane remainder)");
    }
  }
  if (A.ksplit > 1 && epi == EPI_HEAD) {
    const int64_t total = (int64_t)nb * S * S * S;
    int bx = ceil_div(total, 128);
    bx = bx > 8 * sm_count() ? 8 * sm_count() : bx;
    ::mdp::launch_k(conv_split_reduce_head_kernel, bx, 128, 0, st, A.partial, A.ksplit, nb, S, bias, relu, A.head);
    MDP_LAUNCH_CHECK("conv_split_reduce_head_kernel");
  } else if (A.ksplit > 1) {
    const int pool = epi == EPI_POOL;
    const int So = pool ? S / 2 : S;
    const int64_t total = (int64_t)nb * (cout / 4) * So * So * So * (pool ? 8 : 1);
    int bx = ceil_div(total, 128);  // 128-thread blocks: small layers spread over more SMs
    bx = bx > 8 * sm_count() ? 8 * sm_count() : bx;
    ::mdp::launch_k(conv_split_reduce_kernel, bx, 128, 0, st, A.partial, A.ksplit, nb, cout / 4, S, bias, relu, pool, out,
                                                 out_cq, out_q0);
    MDP_LAUNCH_CHECK("conv_split_reduce_kernel");
  }
  return MDP_OK;
}

// enc1a on tensor cores (wide grids): xin = x-shifted input quads (pack_input_kernel mode 1),
// w = the raw [16][2][27] filter; output 16 channels, bias, ReLU, TF32 rounding.
int tc_enc1a(int nb, int S, const float4* xin, const float* w, const float* bias, float4* out, int out_cq,
             int out_q0, cudaStream_t st) {
  using namespace tc;
  EncodeTiledFn enc = encode_fn();
  MDP_REQUIRE(enc != nullptr, "cuTensorMapEncodeTiled unavailable");
  ConvArgs A{};
  A.nb = nb;
  A.S = S;
  A.cin = 4;
  A.cout = A.ncol = 16;
  A.cqc = 1;
  A.nchunk = A.cps = 1;
  A.nsplit = A.ksplit = 1;
  A.tx = ceil_div(S, BX);
  A.ty = ceil_div(S, BY);
  A.fold = 1;
  A.pair = 1;
  A.wraw = w;
  // brick depth from the per-item shape only (batched == serial bitwise)
  const int zp = (int64_t)A.tx * A.ty * ceil_div(S, 4) >= 2 * sm_count() ? 4 : 2;
  A.tz = ceil_div(S, zp);
  A.ntiles = nb * A.tx * A.ty * A.tz;
  A.in_cq = 1;
  A.in_q0 = 0;
  A.bias = bias;
  A.relu = 1;
  A.epi = EPI_STORE;
  A.out = out;
  A.out_cq = out_cq;
  A.out_q0 = out_q0;
  A.Sout = S;
  A.a_bytes = (uint32_t)(zp == 4 ? Brick<4>::QUAD_BYTES : Brick<2>::QUAD_BYTES);
  A.na = 4;
  A.resident = 1;
  A.tps = 3;
  A.nbs = 1;
  A.b_bytes = 3 * 2 * 3 * 16 * 16;
  A.tmem_cols = 128;  // 2 buffers x 4 planes x 16 columns
  CUtensorMap map, wmap;
  memset(&wmap, 0, sizeof(wmap));
  cuuint64_t gdim[4] = {(cuuint64_t)4 * S, (cuuint64_t)S, (cuuint64_t)S, (cuuint64_t)nb};
  cuuint64_t gstride[3] = {(cuuint64_t)16 * S, (cuuint64_t)16 * S * S, (cuuint64_t)16 * S * S * S};
  cuuint32_t box[4] = {4 * HX, HY, (cuuint32_t)(zp + 2), 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, (void*)xin, gdim, gstride, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  MDP_REQUIRE(r == CUDA_SUCCESS, "cuTensorMapEncodeTiled failed (%d) for enc1a S=%d", (int)r, S);
  const size_t smem = 1024 + (size_t)A.na * A.a_bytes + A.b_bytes + 2048;
  conv3_smem_attr();
  int grid = A.ntiles < sm_count() ? A.ntiles : sm_count();
  if (zp == 4)
    ::mdp::launch_k(conv3_tc_kernel<4>, grid, 384, smem, st, map, wmap, A);
  else
    ::mdp::launch_k(conv3_tc_kernel<2>, grid, 384, smem, st, map, wmap, A);
  MDP_LAUNCH_CHECK("conv3_tc_kernel (enc1a)");
  return MDP_OK;
}

int tc_tconv(int nb, const float4* in, int in_cq, int cin, int cout, int Sin, int op, const float* w,
             const float* bias, float4* out, int out_cq, int out_q0, cudaStream_t st) {
  using namespace tc;
  MDP_REQUIRE(cin % 8 == 0 && cin <= 128 && cout % 16 == 0 && cout <= 128, "tc tconv needs cin%%8==0 (<=128), "
              "cout%%16==0 (<=128), got %d/%d", cin, cout);
  TconvArgs T{};
  T.in = in;
  T.in_cq = in_cq;
  T.cin = cin;
  T.cout = cout;
  T.Sin = Sin;
  T.op = op;
  T.w = w;
  T.bias = bias;
  T.out = out;
  T.out_cq = out_cq;
  T.out_q0 = out_q0;
  T.nb = nb;
  T.a_bytes = (uint32_t)cin * 128 * 4;
  const int64_t nvi = (int64_t)Sin * Sin * Sin;
  T.nmain = ceil_div(nvi, 128);
  T.ntiles = T.nmain * nb;
  // taps per CTA: weights + two voxel-row buffers in shared memory, two TMEM
  // tile buffers; on small grids fewer taps per CTA for parallelism
  const size_t budget = 200 * 1024;
  int tg = 8;
  while (tg > 1 && (2 * (size_t)T.a_bytes + (size_t)tg * cin * cout * 4 > budget || 2 * tg * cout > 512)) tg >>= 1;
  while (tg > 1 && (int64_t)T.ntiles * (8 / tg) < 2 * sm_count()) tg >>= 1;
  T.tg = tg;
  T.b_bytes = (uint32_t)(tg * cin * cout * 4);
  uint32_t cols = 32;
  while (cols < (uint32_t)(2 * tg * cout)) cols <<= 1;
  T.tmem_cols = cols;
  const int groups = 8 / tg;
  int ncta = sm_count() / groups;
  ncta = ncta < 1 ? 1 : (ncta > T.ntiles ? T.ntiles : ncta);
  T.ncta = ncta;
  int npad = 0;
  if (op) {
    const int So = 2 * Sin + 1;
    const int64_t per_item = ((int64_t)So * So * So - 8 * nvi) * (cout / 4);
    npad = ceil_div(per_item, 192);
    npad = npad > 64 ? 64 : npad;
  }
  const size_t smem = 1024 + (size_t)T.b_bytes + 2 * (size_t)T.a_bytes + 128;
  MDP_REQUIRE(smem <= 227 * 1024, "tc tconv needs %zu bytes of shared memory", smem);
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(tconv_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(227 * 1024));
    attr_set = true;
  }
  dim3 grid(ncta + npad, groups, 1);
  ::mdp::launch_k(tconv_tc_kernel, grid, Sin >= 32 ? 320 : 192, smem, st, T);
  MDP_LAUNCH_CHECK("tconv_tc_kernel");
  return MDP_OK;
}

}  // namespace mdp
