// 3x3x3 same-padding convolution as an implicit GEMM on the 5th-generation
// tensor cores (tcgen05.mma kind::tf32, FP32 accumulate in TMEM), replacing
// neural.conv3d's im2col + BLAS GEMM (neural.py:60-154).
//
// Tile = brick of ZP x 16 x 8 output voxels (z, y, x) of one batch item;
// each z-plane is one M = 128 MMA row block, N = Cout, K = 27 taps x Cin.
//
// A operand: the brick plus its 1-voxel halo, (ZP+2) x 18 x 10 voxels x 32
// channels, is fetched ONCE per 32-channel chunk by a single 5-D TMA box
// from the channel-quad-blocked activation tensor, with TMA's out-of-bounds
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
// Warp roles (256 threads): w0 TMA/bulk producer, w1 MMA issuer, w2 TMEM
// allocator, w4..w7 epilogue (TMEM -> registers -> bias/ReLU/TF32 round ->
// global, optional fused 2x2x2 max-pool).  Two TMEM accumulator buffers let
// the epilogue of tile t overlap the MMAs of tile t+1.
#include <cuda.h>

#include "unet_layout.cuh"

namespace mdp {
namespace tc {

constexpr int ZP = 2, BY = 16, BX = 8;
constexpr int HZ = ZP + 2, HY = BY + 2, HX = BX + 2;
constexpr int HROWS = HZ * HY * HX;  // 720 halo voxels per quad plane
constexpr int QUAD_BYTES = HROWS * 16;

struct ConvArgs {
  int nb, S, cin, cout, cqc, nchunk;
  int tx, ty, tz, ntiles;
  int in_cq, in_q0;
  const float* w;
  const float* bias;
  int relu, epi;
  float4* out;
  int out_cq, out_q0, Sout;
  uint32_t a_bytes, b_bytes;
  int na, nbs;
  uint32_t tmem_cols;
  HeadArgs head;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
  }
}

__device__ __forceinline__ void tma_load_5d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                            int c2, int c3, int c4) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
      : "memory");
}

__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
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

__device__ __forceinline__ void decode_tile(const ConvArgs& A, int tile, int& b, int& x0, int& y0, int& z0) {
  int ix = tile % A.tx;
  int t = tile / A.tx;
  int iy = t % A.ty;
  t /= A.ty;
  int iz = t % A.tz;
  b = t / A.tz;
  x0 = ix * BX;
  y0 = iy * BY;
  z0 = iz * ZP;
}

__global__ void __launch_bounds__(256, 1) conv3_tc_kernel(const __grid_constant__ CUtensorMap tmap,
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
      mbar_init(&t_empty[i], 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmap) : "memory");
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
  const int ntaps = 27;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- producer
      int as = 0, ap = 0, bs = 0, bp = 0;
      for (int tile = blockIdx.x; tile < A.ntiles; tile += gridDim.x) {
        int b, x0, y0, z0;
        decode_tile(A, tile, b, x0, y0, z0);
        for (int c = 0; c < A.nchunk; ++c) {
          mbar_wait(&a_empty[as], ap ^ 1);
          mbar_expect_tx(&a_full[as], A.a_bytes);
          tma_load_5d(sA + (size_t)as * A.a_bytes, &tmap, &a_full[as], 0, x0 - 1, y0 - 1, z0 - 1,
                      b * A.in_cq + A.in_q0 + c * A.cqc);
          if (++as == A.na) { as = 0; ap ^= 1; }
          const float* wc = A.w + (size_t)c * ntaps * (A.b_bytes / 4);
          for (int t = 0; t < ntaps; ++t) {
            mbar_wait(&b_empty[bs], bp ^ 1);
            mbar_expect_tx(&b_full[bs], A.b_bytes);
            bulk_load(sB + (size_t)bs * A.b_bytes, wc + (size_t)t * (A.b_bytes / 4), A.b_bytes, &b_full[bs]);
            if (++bs == A.nbs) { bs = 0; bp ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- MMA issuer
      const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(A.cout >> 3) << 17) |
                             ((uint32_t)(128 >> 4) << 24);
      const uint32_t lbo_a = QUAD_BYTES, sbo_a = HX * 16;
      const uint32_t lbo_b = A.cout * 16, sbo_b = 128;
      const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
      int as = 0, ap = 0, bs = 0, bp = 0, li = 0;
      for (int tile = blockIdx.x; tile < A.ntiles; tile += gridDim.x, ++li) {
        const int buf = li & 1;
        mbar_wait(&t_empty[buf], ((li >> 1) & 1) ^ 1);
        fence_after();
        const uint32_t dcol = tmem + (uint32_t)(buf * ZP * A.cout);
        for (int c = 0; c < A.nchunk; ++c) {
          mbar_wait(&a_full[as], ap);
          fence_after();
          const uint32_t abase = a0 + as * A.a_bytes;
          for (int t = 0; t < ntaps; ++t) {
            mbar_wait(&b_full[bs], bp);
            fence_after();
            const int dz = t / 9, dy = (t / 3) % 3, dx = t % 3;
            const uint32_t bbase = b0 + bs * A.b_bytes;
            for (int ks = 0; ks < A.cqc / 2; ++ks) {
              const uint64_t bd = umma_desc(bbase + 2 * ks * lbo_b, lbo_b, sbo_b);
#pragma unroll
              for (int zp = 0; zp < ZP; ++zp) {
                const uint32_t off = (uint32_t)(((zp + dz) * HY + dy) * HX + dx) * 16u;
                const uint64_t ad = umma_desc(abase + 2 * ks * lbo_a + off, lbo_a, sbo_a);
                mma_tf32(dcol + zp * A.cout, ad, bd, idesc, (c | t | ks) != 0);
              }
            }
            mma_commit(&b_empty[bs]);
            if (++bs == A.nbs) { bs = 0; bp ^= 1; }
          }
          mma_commit(&a_empty[as]);
          if (++as == A.na) { as = 0; ap ^= 1; }
        }
        mma_commit(&t_full[buf]);
      }
    }
  } else if (warp >= 4) {  // ---------------- epilogue
    const int ew = warp - 4;
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
      int b, x0, y0, z0;
      decode_tile(A, tile, b, x0, y0, z0);
      mbar_wait(&t_full[buf], (li >> 1) & 1);
      fence_after();
      const uint32_t dcol = tmem + lane_addr + (uint32_t)(buf * ZP * A.cout);
      const int gx = x0 + lx, gy = y0 + ly;
      if (A.epi == EPI_POOL) {
        const int px = gx >> 1, py = gy >> 1, pz = z0 >> 1;
        const bool writer = ((lane & 1) == 0) && ((ly & 1) == 0) && px < So && py < So && pz < So;
        for (int cg = 0; cg < A.cout / 16; ++cg) {
          float v0[16], v1[16];
          tmem_ld16(dcol + cg * 16, v0);
          tmem_ld16(dcol + A.cout + cg * 16, v1);
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            float m = fmaxf(v0[i], v1[i]);
            m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 1));
            m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 8));
            if (A.bias) m += A.bias[cg * 16 + i];
            if (A.relu) m = fmaxf(m, 0.f);
            v0[i] = tf32_round(m);
          }
          if (writer) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              float4 o = make_float4(v0[4 * q], v0[4 * q + 1], v0[4 * q + 2], v0[4 * q + 3]);
              A.out[((int64_t)b * A.out_cq + A.out_q0 + cg * 4 + q) * So3 + ((int64_t)pz * So + py) * So + px] = o;
            }
          }
        }
      } else {
#pragma unroll
        for (int zp = 0; zp < ZP; ++zp) {
          const int gz = z0 + zp;
          const bool ok = gx < S && gy < S && gz < S;
          for (int cg = 0; cg < A.cout / 16; ++cg) {
            float v[16];
            tmem_ld16(dcol + zp * A.cout + cg * 16, v);
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              float m = v[i];
              if (A.bias) m += A.bias[cg * 16 + i];
              if (A.relu) m = fmaxf(m, 0.f);
              v[i] = tf32_round(m);
            }
            if (ok) {
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                float4 o = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
                A.out[((int64_t)b * A.out_cq + A.out_q0 + cg * 4 + q) * S3 + ((int64_t)gz * S + gy) * S + gx] = o;
              }
            }
          }
        }
      }
      fence_before();
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
}

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

int tc_conv3(int nb, int S, int cin, int cout, const float4* in, int in_cq, int in_q0, const float* w,
             const float* bias, int relu, float4* out, int out_cq, int out_q0, int epi, const HeadArgs* head,
             cudaStream_t st) {
  using namespace tc;
  MDP_REQUIRE(cin % 8 == 0 && cin >= 8, "tc conv needs cin multiple of 8, got %d", cin);
  MDP_REQUIRE(cout % 16 == 0 && cout >= 16 && cout <= 128, "tc conv needs cout in {16..128} step 16, got %d",
              cout);
  MDP_REQUIRE(epi == EPI_STORE || epi == EPI_POOL, "epilogue %d not supported by tc conv", epi);
  EncodeTiledFn enc = encode_fn();
  MDP_REQUIRE(enc != nullptr, "cuTensorMapEncodeTiled unavailable");
  ConvArgs A{};
  A.nb = nb;
  A.S = S;
  A.cin = cin;
  A.cout = cout;
  A.cqc = cin >= 32 ? 8 : cin / 4;
  A.nchunk = cin / (4 * A.cqc);
  A.tx = ceil_div(S, BX);
  A.ty = ceil_div(S, BY);
  A.tz = ceil_div(S, ZP);
  A.ntiles = nb * A.tx * A.ty * A.tz;
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
  A.a_bytes = (uint32_t)A.cqc * QUAD_BYTES;
  A.b_bytes = (uint32_t)A.cqc * cout * 16;
  A.na = 2;
  const size_t budget = 227 * 1024 - 2048;
  int nbs = 6;
  while (nbs > 2 && (size_t)A.na * A.a_bytes + (size_t)nbs * A.b_bytes > budget) --nbs;
  A.nbs = nbs;
  MDP_REQUIRE((size_t)A.na * A.a_bytes + (size_t)nbs * A.b_bytes <= budget, "tc conv tile does not fit smem");
  uint32_t cols = 32;
  while (cols < (uint32_t)(2 * ZP * cout)) cols <<= 1;
  A.tmem_cols = cols;
  if (head) A.head = *head;

  CUtensorMap map;
  cuuint64_t gdim[5] = {4, (cuuint64_t)S, (cuuint64_t)S, (cuuint64_t)S, (cuuint64_t)nb * in_cq};
  cuuint64_t gstride[4] = {16, (cuuint64_t)16 * S, (cuuint64_t)16 * S * S, (cuuint64_t)16 * S * S * S};
  cuuint32_t box[5] = {4, HX, HY, HZ, (cuuint32_t)A.cqc};
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, (void*)in, gdim, gstride, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  MDP_REQUIRE(r == CUDA_SUCCESS, "cuTensorMapEncodeTiled failed (%d) for S=%d cin=%d", (int)r, S, cin);

  const size_t smem = 1024 + (size_t)A.na * A.a_bytes + (size_t)nbs * A.b_bytes + 1024;
  static size_t attr_set = 0;
  if (attr_set < smem) {
    cudaFuncSetAttribute(conv3_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(227 * 1024));
    attr_set = 227 * 1024;
  }
  int grid = A.ntiles < sm_count() ? A.ntiles : sm_count();
  conv3_tc_kernel<<<grid, 256, smem, st>>>(map, A);
  MDP_LAUNCH_CHECK("conv3_tc_kernel");
  return MDP_OK;
}

}  // namespace mdp
