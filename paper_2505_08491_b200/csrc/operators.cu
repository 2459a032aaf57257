// Coupled 3D-1D system operators, float64, matrix-free.
//
// K00 (assembly.py:122-125) is applied as the Kronecker sum of 1D P1
// operators: K00 = kO (Mz My Kx + Mz Ky Mx + Kz My Mx) +
// sO Mz My Mx, evaluated by sum factorisation in a 2.5D tile: an x-y tile
// of one z-plane staged in shared memory, the z-direction carried in
// registers over three planes, so x is read from HBM once.
//
// The coupling (assembly.py:322-345) uses the index sets of Pi = T, Psi, W:
//   s_q  = W_q ((T x3)_q - (Psi D x1)_q)            pi_gather
//   y3  += w T^T s      (pull over touched nodes)   pi_scatter
//   y1   = K11 x1 - w D Psi^T s                     oned_apply
// which equals full_operator(s) @ x.
#include <stdlib.h>

#include "async.cuh"
#include "common.cuh"

namespace mdp {

struct Line1D {
  // 3-point rows of the assembled 1D P1 stiffness (1/h tridiag(-1,2,-1),
  // 1 at the ends) and mass (h/6 tridiag(1,4,1), 2 at the ends).
  double kd_in, kd_end, ko, md_in, md_end, mo;
};

__host__ __device__ inline Line1D make_line(double h) {
  Line1D c;
  c.kd_in = 2.0 / h;
  c.kd_end = 1.0 / h;
  c.ko = -1.0 / h;
  c.md_in = 4.0 * h / 6.0;
  c.md_end = 2.0 * h / 6.0;
  c.mo = h / 6.0;
  return c;
}

__device__ __forceinline__ double kdiag(const Line1D& c, int i, int n) {
  return (i == 0 || i == n - 1) ? c.kd_end : c.kd_in;
}
__device__ __forceinline__ double mdiag(const Line1D& c, int i, int n) {
  return (i == 0 || i == n - 1) ? c.md_end : c.md_in;
}
__device__ __forceinline__ bool on_boundary(int i, int j, int k, int n) {
  return i == 0 || j == 0 || k == 0 || i == n - 1 || j == n - 1 || k == n - 1;
}

// s_q = W_q ((T x3)_q - (Psi D x1)_q): one warp per quadrature row, lanes
// over the row's (point, corner) entries (8 for the centreline, up to 64
// for the 8-point ring average), warp-shuffle reduction.  Entries on
// eliminated (Dirichlet) cube nodes are dropped from T at build time.
__device__ __forceinline__ void gather_rows(const mdp_problem& P, int s, int w0, int wstride,
                                            const double* __restrict__ x3, const double* __restrict__ x1,
                                            int64_t ld, double* __restrict__ s_out) {
  const int lane = threadIdx.x & 31;
  for (int q = P.q_start[s] + w0; q < P.q_start[s + 1]; q += wstride) {
    double acc = 0.0;
    if (x3) {
      const double* xp = x3 + (int64_t)s * ld;
      for (int k = P.t_ptr[q] + lane; k < P.t_ptr[q + 1]; k += 32) acc += P.t_val[k] * __ldg(xp + P.t_col[k]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) {
      if (x1) {
        const double* xp = x1 + (int64_t)s * ld;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          int col = P.psi_col[2 * q + e];
          if (col >= 0) acc -= P.psi_val[2 * q + e] * xp[col];
        }
      }
      s_out[q] = P.wq[q] * acc;
    }
  }
}

__device__ double g_zero_row[32];  // zero page: out-of-domain rows read from here

// Warp-per-row-pair stencil: lane l owns column i = i0 - 1 + l (30 output
// columns per warp, lanes 0 and 31 are the x halo), the warp owns rows j,
// j+1 and marches z in [z0, z1).  Per plane each lane holds rows j-1..j+2
// of its column in registers (two planes of loads in flight), takes its
// x-neighbours by shuffle, forms the in-plane sum factorisation
// P = kO (My Kx + Ky Mx) x + sO My Mx x, R = kO My Mx x for both rows
// (the x products of the shared rows are reused) and carries P, R over
// three planes: y = Mz P + Kz R.  No shared memory, no barriers; rows
// outside the domain or on eliminated (Dirichlet) cube nodes read a zero
// page through a pointer that does not advance.  Optional fused Jacobi
// epilogue out = xin + omega (r - y) / diag(C) (coupling correction follows
// in the pull).
#ifndef STENCIL_PF
#define STENCIL_PF 2  // planes of loads in flight per warp (tools/stencil_sweep.py A/B)
#endif
#ifndef STENCIL_UNROLL
#define STENCIL_UNROLL 1
#endif
#ifndef STENCIL_ROWS
#define STENCIL_ROWS 2  // output rows per warp
#endif

struct GatherArgs {  // optional Pi gather folded into the stencil launch
  const double* x3;
  const double* x1;
  double* s_out;
  int nblk;  // v3 launch: blocks given to the gather
};

template <bool JAC, bool GATHER>
__global__ void __launch_bounds__(128) stencil_kernel(const mdp_problem P, const int32_t* sel,
                                                       const double* __restrict__ x, int64_t ldx,
                                                       double* __restrict__ y, int64_t ldy, int zchunk,
                                                       const double* __restrict__ jr, double omega,
                                                       const GatherArgs G) {
  MDP_PDL_ENTER();
  constexpr int RY = STENCIL_ROWS, NR = RY + 2, PF = STENCIL_PF, UNR = STENCIL_UNROLL;
  const int n = P.n;
  const int s = sys_of(sel, blockIdx.z);
  if (GATHER && blockIdx.y == gridDim.y - 1) {  // independent of the stencil: runs alongside it
    gather_rows(P, s, blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), gridDim.x * (blockDim.x >> 5), G.x3, G.x1,
                ldx, G.s_out);
    return;
  }
  const double* xp = x + (int64_t)s * ldx;
  double* yp = y + (int64_t)s * ldy;
  const int lane = threadIdx.x & 31;
  const int tiles_x = (n + 29) / 30;
  const int wrow = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int j = (wrow / tiles_x) * RY;
  if (j >= n) return;
  const int i = (wrow % tiles_x) * 30 - 1 + lane;
  const int z0 = blockIdx.y * zchunk;
  const int z1 = min(n, z0 + zchunk);
  if (z0 >= n) return;
  const bool dir = P.bc3d != 0;
  const Line1D c = make_line(P.h);
  const double kO = P.k_omega, sO = P.sigma_omega;
  const int64_t nn = (int64_t)n * n;
  const bool colok = i >= 0 && i < n && !(dir && (i == 0 || i == n - 1));
  // per-row pointers at plane z0-1 and their per-plane step (0 for zero-page rows)
  const double* ptr[NR];
  int64_t step[NR];
#pragma unroll
  for (int a = 0; a < NR; ++a) {
    const int jj = j - 1 + a;
    const bool ok = colok && jj >= 0 && jj < n && !(dir && (jj == 0 || jj == n - 1));
    ptr[a] = ok ? xp + (int64_t)(z0 - 1) * nn + (int64_t)jj * n + i : g_zero_row + lane;
    step[a] = ok ? nn : 0;
  }
  // plane kk contributes values iff it lies inside and is not an eliminated face
  auto plane_ok = [&](int kk) { return kk >= 0 && kk < n && !(dir && (kk == 0 || kk == n - 1)); };
  auto load = [&](int kk, double* v) {
    const bool pok = plane_ok(kk);
#pragma unroll
    for (int a = 0; a < NR; ++a) {
      v[a] = pok ? __ldg(ptr[a]) : 0.0;
      ptr[a] += step[a];
    }
  };
  const bool out_lane = lane >= 1 && lane <= 30 && i < n;
  const int ic = i < 0 ? 0 : (i >= n ? n - 1 : i);
  const double kdx = kdiag(c, ic, n), mdx = mdiag(c, ic, n);
  double kdy[RY], mdy[RY];
  bool rok[RY], colb[RY];
#pragma unroll
  for (int r = 0; r < RY; ++r) {
    const int jr_ = j + r < n ? j + r : n - 1;
    kdy[r] = kdiag(c, jr_, n);
    mdy[r] = mdiag(c, jr_, n);
    rok[r] = out_lane && j + r < n;
    colb[r] = dir && (i == 0 || i == n - 1 || j + r == 0 || j + r == n - 1);
  }
  double* yrow = yp + (int64_t)z0 * nn + (int64_t)j * n + i;  // output (z0, j, i)
  const double* xrow = xp + (int64_t)z0 * nn + (int64_t)j * n + i;
  int64_t goff = (int64_t)s * ldy + (int64_t)z0 * nn + (int64_t)j * n + i;
  // register ring: q[0] = plane kk, q[1..PF] = the next PF planes (loads in flight)
  double q[PF + 1][NR];
#pragma unroll
  for (int p = 0; p < PF; ++p)
    if (z0 - 1 + p <= z1) load(z0 - 1 + p, q[p]);
  double* cur = q[0];
  double Pm[RY], P0[RY], Rm[RY], R0[RY];
#pragma unroll
  for (int r = 0; r < RY; ++r) Pm[r] = P0[r] = Rm[r] = R0[r] = 0.0;
  // unrolled by the ring / recurrence periods so the plane rotation is register
  // renaming, not moves (the kernel is issue-bound)
#pragma unroll UNR
  for (int kk = z0 - 1; kk <= z1; ++kk) {
    if (kk + PF <= z1) load(kk + PF, q[PF]);
    double kx[NR], mx[NR];
#pragma unroll
    for (int a = 0; a < NR; ++a) {
      const double lr = __shfl_up_sync(0xffffffffu, cur[a], 1) + __shfl_down_sync(0xffffffffu, cur[a], 1);
      kx[a] = c.ko * lr + kdx * cur[a];
      mx[a] = c.mo * lr + mdx * cur[a];
    }
    const int ko = kk - 1;
    const bool emit = ko >= z0;
    const double kd = kdiag(c, ko < 0 ? 0 : ko, n), md = mdiag(c, ko < 0 ? 0 : ko, n);
    const bool planeb = dir && (ko == 0 || ko == n - 1);
#pragma unroll
    for (int r = 0; r < RY; ++r) {
      const double msum = mx[r] + mx[r + 2];
      const double c1 = c.mo * (kx[r] + kx[r + 2]) + mdy[r] * kx[r + 1];
      const double c2 = c.ko * msum + kdy[r] * mx[r + 1];
      const double c3 = c.mo * msum + mdy[r] * mx[r + 1];
      const double Pn = kO * (c1 + c2) + sO * c3;
      const double Rn = kO * c3;
      if (emit && rok[r]) {
        double out = c.mo * (Pm[r] + Pn) + md * P0[r] + c.ko * (Rm[r] + Rn) + kd * R0[r];
        if (colb[r] || planeb) out = xrow[r * n];
        if (JAC) out = xrow[r * n] + (omega * (jr[goff + r * n] - out)) / P.diag_c[goff + r * n];
        yrow[r * n] = out;
      }
      Pm[r] = P0[r]; P0[r] = Pn;
      Rm[r] = R0[r]; R0[r] = Rn;
    }
    if (emit) {
      yrow += nn;
      xrow += nn;
      goff += nn;
    }
#pragma unroll
    for (int p = 0; p < PF; ++p)
#pragma unroll
      for (int a = 0; a < NR; ++a) q[p][a] = q[p + 1][a];
  }
}

// ---------------------------------------------------------------------------
// Folded Kronecker coefficients of the v3 stencil below.  With
// S = lr_{j-1} + lr_{j+1}, T = v_{j-1} + v_{j+1} (lr = x_{i-1} + x_{i+1}):
//   U = mo P + ko R = b1 S + b2 T + rho (b3 lr_j + b4 v_j)
//   C = md P + kd R = c1 S + c2 T + rho (c3 lr_j + c4 v_j)
//   y_k = U_{k-1} + U_{k+1} + sigma_k C_k
// (P, R as in v1; every 1D end-row diagonal is half the interior one, so
// Neumann end rows / end planes only scale the centre terms by 0.5: rho per
// row, sigma per plane).  One fixed expression per node (batched == serial).
struct StencilCoef {
  double b1, b2, b3, b4, c1, c2, c3, c4;
};

__device__ __forceinline__ StencilCoef stencil_coef(const Line1D& c, double kO, double sO, double kdx, double mdx) {
  // interior y / z diagonals; x diagonals per lane
  const double mo = c.mo, ko = c.ko, mdy = c.md_in, kdy = c.kd_in, mdz = c.md_in, kdz = c.kd_in;
  // P = pA A + pB B + pc cc + pd dd, R = rB B + rd dd with A = Kx(row j-1 + row j+1),
  // B = Mx(rows j-1 + j+1), cc = Kx row j, dd = Mx row j
  const double pA = kO * mo, pB = kO * ko + sO * mo, pc = kO * mdy, pd = kO * kdy + sO * mdy;
  const double rB = kO * mo, rd = kO * mdy;
  // U = mo P + ko R, C = mdz P + kdz R
  const double uA = mo * pA, uB = mo * pB + ko * rB, uc = mo * pc, ud = mo * pd + ko * rd;
  const double cA = mdz * pA, cB = mdz * pB + kdz * rB, cc = mdz * pc, cd = mdz * pd + kdz * rd;
  // A = ko S + kdx T, B = mo S + mdx T, cc = ko lr + kdx v, dd = mo lr + mdx v
  StencilCoef k;
  k.b1 = uA * ko + uB * mo;
  k.b2 = uA * kdx + uB * mdx;
  k.b3 = uc * ko + ud * mo;
  k.b4 = uc * kdx + ud * mdx;
  k.c1 = cA * ko + cB * mo;
  k.c2 = cA * kdx + cB * mdx;
  k.c3 = cc * ko + cd * mo;
  k.c4 = cc * kdx + cd * mdx;
  return k;
}

// ---------------------------------------------------------------------------
// Stencil v3: the v2 arithmetic fed by an asynchronous shared-memory plane
// pipeline.  A block owns one band of RY output rows (one consumer warp per
// 32-column tile) over a z-chunk; rows j-1..j+RY of one plane are
// contiguous in HBM, so a producer warp moves each plane's band with ONE
// cp.async.bulk into a ring of kSt3 shared-memory stages (full / empty
// mbarriers): the bytes in flight no longer depend on registers or on the
// per-warp scoreboard depth (v1/v2 were latency-bound: 22% DRAM throughput,
// long-scoreboard stalls).  Consumers read a column and both x-neighbours
// from the stage (no shuffles, every lane produces an output), zero the
// contributions of absent / eliminated neighbours by 0/1 masks, and carry
// the z-recurrence in registers (6-step unroll = register renaming).  Out-of-
// domain planes are copied from the nearest plane and masked, so the stage
// never holds non-finite garbage.
constexpr int kSt3 = 6;  // stages; equals the unroll so slots are compile-time

// Optional trace of three stencil blocks (first / middle / last slot) of the launch (build with
// -DST3_TRACE; tools/stencil_trace.py): %globaltimer at block entry and after the ring is set up,
// then per plane step the clock64 at which consumer warp 0 saw the stage full and finished the step.
#ifdef ST3_TRACE
__device__ long long g_st3_trace[3 * 64];
__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define ST3_TR(which, k) \
  do { if ((which) >= 0 && threadIdx.x == 0) g_st3_trace[(which) * 64 + (k)] = ((k) == 0 || (k) == 3) ? gtimer() : clock64(); } while (0)
#else
#define ST3_TR(which, k) do { } while (0)
#endif

template <int N, int RY, bool JAC, bool DIR, bool EDGE>
__device__ __forceinline__ void stencil3_consumer(const mdp_problem& P, double* __restrict__ yp,
                                                  const double* __restrict__ jrp, const double* __restrict__ dgp,
                                                  double omega, int n, int i, int j, int z0, int z1,
                                                  const StencilCoef& K, const double* stg, int sw, int swj,
                                                  uint64_t* full, uint64_t* empty, int r_lo, int r_hi, int trc,
                                                  const double* __restrict__ xgp, bool lastcol) {
  using namespace async;
  constexpr int NR = RY + 2;
  // Dirichlet cube with n = 32 t + 1 columns (plain stencil): the band runs t consumer warps and the lane of
  // column n - 2 also writes column n - 1, an eliminated identity node (y = x), instead of a further warp
  // with one live column
  const bool lc_lane = DIR && lastcol && i == n - 2;
  const int lane = threadIdx.x & 31;
  const int nn = n * n;
  const bool col_in = i < n;
  const int ic = col_in ? i : n - 1;  // clamped column (reads stay inside the stage)
  // neighbour masks: absent (outside) or eliminated (Dirichlet face) columns contribute 0
  // (as 0/1 factors: selects instead of the two FP64 operations measured 6-10% slower per step --
  // the step is a latency chain, not FP64-issue bound)
  const double mL = (ic - 1 >= (DIR ? 1 : 0)) ? 1.0 : 0.0;
  const double mR = (ic + 1 <= (DIR ? n - 2 : n - 1)) ? 1.0 : 0.0;
  int roff[NR];
  double rmask[NR];
#pragma unroll
  for (int a = 0; a < NR; ++a) {
    const int jj = j - 1 + a;
    const int jc = jj < r_lo ? r_lo : (jj > r_hi ? r_hi : jj);
    roff[a] = (jc - r_lo) * n + ic;
    rmask[a] = (jj >= 0 && jj < n && !(DIR && (jj == 0 || jj == n - 1))) ? 1.0 : 0.0;
  }
  double rho[RY];
  bool rout[RY], rbnd[RY];
#pragma unroll
  for (int r = 0; r < RY; ++r) {
    const int jr_ = j + r;
    rho[r] = (EDGE && !DIR && (jr_ == 0 || jr_ == n - 1)) ? 0.5 : 1.0;
    rout[r] = col_in && (!EDGE || jr_ < n);
    rbnd[r] = DIR && (i == 0 || i == n - 1 || jr_ == 0 || jr_ == n - 1);
  }
  const int obase = j * n + i;
  double U[3][RY], Cc[2][RY], X[2][RY];  // X: raw centre values of the last two planes
#pragma unroll
  for (int r = 0; r < RY; ++r) U[0][r] = U[1][r] = U[2][r] = Cc[0][r] = Cc[1][r] = X[0][r] = X[1][r] = 0.0;
  const int nsteps = z1 - z0 + 2;
  for (int s0 = 0; s0 < nsteps; s0 += kSt3) {
    const uint32_t par = (uint32_t)((s0 / kSt3) & 1);
#pragma unroll
    for (int u = 0; u < kSt3; ++u) {
      const int st = s0 + u;
      if (st >= nsteps) break;
      const int k = z0 - 1 + st;
      const int kc = k < 0 ? 0 : (k > n - 1 ? n - 1 : k);  // plane the producer copied
      const bool pok = k >= 0 && k < n && !(DIR && (k == 0 || k == n - 1));
      mbar_wait(&full[u], par);
      if (st < 24) ST3_TR(trc, 4 + 2 * st);
      const double* b = stg + (size_t)u * (sw + 2 * swj) + ((kc * nn + r_lo * n) & 1);
      double c[NR], lr[NR];
#pragma unroll
      for (int a = 0; a < NR; ++a) {
        c[a] = b[roff[a]];
        lr[a] = fma(mL, b[roff[a] - 1], mR * b[roff[a] + 1]);
      }
      // Jacobi epilogue operands of the plane emitted in this step (k - 1): the
      // producer staged r and diag(C) of this band beside the x plane
      double jv[JAC ? RY : 1], dv[JAC ? RY : 1];
      if (JAC) {
        const double* jb = stg + (size_t)u * (sw + 2 * swj) + sw + (((k - 1) * nn + j * n) & 1) + ic;
#pragma unroll
        for (int r = 0; r < RY; ++r) {
          jv[r] = jb[r * n];
          dv[r] = jb[swj + r * n];
        }
      }
      if (!JAC && DIR && lc_lane && k >= z0 && k < z1) {
        // column n - 1 of plane k needs no recurrence: y = x there, and the raw value sits in this stage
        // (the right neighbour of this lane's column)
#pragma unroll
        for (int r = 0; r < RY; ++r) {
          if (EDGE && j + r >= n) continue;
          yp[(int64_t)k * nn + (int64_t)(j + r) * n + (n - 1)] = b[roff[r + 1] + 1];
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[u]);
      double* xc = X[u % 2];
#pragma unroll
      for (int r = 0; r < RY; ++r) xc[r] = c[r + 1];
      if (EDGE) {
#pragma unroll
        for (int a = 0; a < NR; ++a) {
          c[a] *= rmask[a];
          lr[a] *= rmask[a];
        }
      }
      const double vm = pok ? 1.0 : 0.0;
      double* Un = U[u % 3];
      const double* Um = U[(u + 1) % 3];
      double* Cn = Cc[u % 2];
      const double* Ck = Cc[(u + 1) % 2];
      const double* xo = X[(u + 1) % 2];  // raw x of the output plane k-1
      const int ko = k - 1;
      const bool emit = ko >= z0;
      const double sig = (!DIR && (ko == 0 || ko == n - 1)) ? 0.5 : 1.0;
      const bool pbnd = DIR && (ko == 0 || ko == n - 1);
      double* yrow = yp + (ko * nn + obase);
#pragma unroll
      for (int r = 0; r < RY; ++r) {
        // the centre column of the centre row: Dirichlet-eliminated centres only feed
        // outputs that are overridden below
        const double Sx = lr[r] + lr[r + 2];
        const double T = c[r] + c[r + 2];
        double un = fma(K.b2, T, K.b1 * Sx);
        double cn = fma(K.c2, T, K.c1 * Sx);
        if (EDGE && !DIR) {
          un = fma(rho[r], fma(K.b4, c[r + 1], K.b3 * lr[r + 1]), un);
          cn = fma(rho[r], fma(K.c4, c[r + 1], K.c3 * lr[r + 1]), cn);
        } else {
          un = fma(K.b4, c[r + 1], fma(K.b3, lr[r + 1], un));
          cn = fma(K.c4, c[r + 1], fma(K.c3, lr[r + 1], cn));
        }
        un *= vm;
        cn *= vm;
        double out = DIR ? (Um[r] + un) + Ck[r] : fma(sig, Ck[r], Um[r] + un);
        if (DIR && (rbnd[r] || pbnd)) out = xo[r];
        if (emit && rout[r]) {
          if (JAC) out = xo[r] + (omega * (jv[r] - out)) / dv[r];
          yrow[r * n] = out;
        }
        Un[r] = un;
        Cn[r] = cn;
      }
      if (st < 24) ST3_TR(trc, 5 + 2 * st);
    }
  }
  ST3_TR(trc, 3);
}

#ifndef STENCIL3_MINB
#define STENCIL3_MINB 1  // lifts the compiler's 128-register choice (129^3 x 8: 2.8 -> 3.6 TB/s)
#endif
// 193^3 runs 8 warps per block: at 150 registers only ONE block fits an SM, at 128 (a few bytes of
// spills) two do: K00 stencil 193^3 x 8 0.72 -> 0.86 of HBM, coupled SpMV 0.63 -> 0.74 (the Jacobi
// variant spills ~400 B at 128 and loses, so it keeps its registers).  The 6-warp blocks of 129^3 already hold
// two; squeezing a third in (112 registers) costs more in spills than the occupancy returns.
template <int N, int RY, bool JAC, bool LC = false>
__global__ void __maxnreg__((N == 129 && LC) ? 136 : ((N > 160 && N <= 224 && !JAC) ? 128 : 255)) stencil3_kernel(const mdp_problem P, const int32_t* sel,
                                                        const double* __restrict__ x, int64_t ldx,
                                                        double* __restrict__ y, int64_t ldy, int zchunk,
                                                        const double* __restrict__ jr, double omega,
                                                        const GatherArgs G) {
  using namespace async;
  // launched as a programmatic dependent: everything up to the ring set-up (barrier init, zeroing the
  // stages) touches shared memory only and runs before the wait on the previous grid
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  constexpr int NR = RY + 2;
  const int n = N > 0 ? N : P.n;
  // grid (x: block slot, y: system): slots [0, gx) run the Pi gather (first in
  // launch order, alongside the first stencil blocks), then one slot per
  // (band, z-chunk)
  const int s = sys_of(sel, blockIdx.y);
  const int gx = G.s_out ? G.nblk : 0;
  if ((int)blockIdx.x < gx) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    gather_rows(P, s, blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), gx * (blockDim.x >> 5), G.x3, G.x1, ldx,
                G.s_out);
    return;
  }
  extern __shared__ __align__(16) unsigned char smem3[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem3);
  uint64_t* empty = full + kSt3;
  // stage: one pad double in front (x-neighbour reads of column -1 stay in range), then the band
  double* stg = reinterpret_cast<double*>(smem3 + 16 * kSt3) + 2;
  const int sw = (NR * n + 4 + 1) & ~1;  // x-band stride in doubles (16-byte multiple)
  const int swj = JAC ? ((RY * n + 3) & ~1) : 0;  // r / diag(C) bands of the emitted plane (Jacobi epilogue)
  const int sws = sw + 2 * swj;              // whole stage
  // (plain stencil only: the Jacobi sweep would need r at that node ahead of its stage -- a global load
  // per step on the critical path cost it 35% -- and keeps the extra warp)
  // LC: chosen by the launcher for batches of plain stencils (a single system's coupled SpMV, with the gather
  // folded into this launch, measured 2 us slower with it; at 129^3 the instantiation is capped at 136
  // registers so that three 5-warp blocks fit an SM)
  constexpr bool lastcol = LC && !JAC;
  const int tiles_x = lastcol ? (n - 1) / 32 : (n + 31) / 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int bands = (n + RY - 1) / RY;
  const int slot = blockIdx.x - gx;
  const int j = (slot % bands) * RY;
  const int z0 = (slot / bands) * zchunk;
  const int z1 = min(n, z0 + zchunk);
  if (j >= n || z0 >= n) return;  // gather-slice width / chunk rounding (touches no memory)
  const bool dir = P.bc3d != 0;
  int trc = -1;
#ifdef ST3_TRACE
  {
    const int nslots = gridDim.x - gx;
    trc = blockIdx.y != 0 ? -1 : (slot == 0 ? 0 : (slot == nslots / 2 ? 1 : (slot == nslots - 1 ? 2 : -1)));
    ST3_TR(trc, 0);
    ST3_TR(trc, 2);
  }
#endif
  if (threadIdx.x == 0) {
    for (int t = 0; t < kSt3; ++t) {
      mbar_init(&full[t], 1);
      mbar_init(&empty[t], tiles_x);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // zero the ring once: neighbour reads past a band's copied bytes (masked
  // by 0) must see finite values
  for (int t = threadIdx.x; t < kSt3 * sws + 2; t += blockDim.x) stg[t - 2] = 0.0;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes before the async-proxy copies
  asm volatile("griddepcontrol.wait;" ::: "memory");  // x (and r, for the Jacobi sweep) come from the previous grid
  __syncthreads();
  ST3_TR(trc, 1);
  const double* xp = x + (int64_t)s * ldx;
  const int r_lo = j - 1 < 0 ? 0 : j - 1;
  const int r_hi = j + RY > n - 1 ? n - 1 : j + RY;
  const int nsteps = z1 - z0 + 2;
  if (warp == tiles_x) {  // producer: one bulk copy per plane (planes outside the domain: the nearest one)
    if (lane == 0) {
      const int nn = n * n;
      const uint32_t cnt = (uint32_t)(r_hi - r_lo + 1) * n;
      const uint32_t cntj = (uint32_t)(min(RY, n - j)) * n;
      const double* jsrc = JAC ? jr + (int64_t)s * ldy : nullptr;
      const double* dsrc = JAC ? P.diag_c + (int64_t)s * ldy : nullptr;
      for (int st = 0; st < nsteps; ++st) {
        const int slot = st % kSt3;
        if (st >= kSt3) mbar_wait(&empty[slot], (uint32_t)(((st / kSt3) - 1) & 1));
        int k = z0 - 1 + st;
        const int ko = k - 1;  // plane emitted at this step (from z0 on)
        k = k < 0 ? 0 : (k > n - 1 ? n - 1 : k);
        const int e0 = k * nn + r_lo * n;
        const int sh = e0 & 1;
        const uint32_t bytes = ((cnt + sh) * 8 + 15) & ~15u;
        if (JAC && ko >= z0) {
          const int ej = ko * nn + j * n;
          const int shj = ej & 1;
          const uint32_t bj = ((cntj + shj) * 8 + 15) & ~15u;
          mbar_expect_tx(&full[slot], bytes + 2 * bj);
          bulk_load(stg + (size_t)slot * sws + sw, jsrc + (ej - shj), bj, &full[slot]);
          bulk_load(stg + (size_t)slot * sws + sw + swj, dsrc + (ej - shj), bj, &full[slot]);
        } else {
          mbar_expect_tx(&full[slot], bytes);
        }
        bulk_load(stg + (size_t)slot * sws, xp + (e0 - sh), bytes, &full[slot]);
      }
    }
    return;
  }
  const int i = warp * 32 + lane;
  const Line1D c = make_line(P.h);
  const int ic = i >= n ? n - 1 : i;
  const double half = (!dir && (ic == 0 || ic == n - 1)) ? 0.5 : 1.0;
  const StencilCoef K = stencil_coef(c, P.k_omega, P.sigma_omega, half * c.kd_in, half * c.md_in);
  double* yp = y + (int64_t)s * ldy;
  const double* jrp = JAC ? jr + (int64_t)s * ldy : nullptr;
  const double* dgp = JAC ? P.diag_c + (int64_t)s * ldy : nullptr;
  const int lo = dir ? 1 : 0, hi = dir ? n - 2 : n - 1;
  const bool edge = (j - 1 < lo) || (j + RY > hi);
#define MDP_ST3(D, E) \
  stencil3_consumer<N, RY, JAC, D, E>(P, yp, jrp, dgp, omega, n, i, j, z0, z1, K, stg, sw, swj, full, empty, r_lo, r_hi, trc, \
                                      xp, lastcol)
  if (dir) {
    if (edge) MDP_ST3(true, true); else MDP_ST3(true, false);
  } else {
    if (edge) MDP_ST3(false, true); else MDP_ST3(false, false);
  }
#undef MDP_ST3
}

struct CopyArgs {  // optional copy slice of the gather launch: dst_s[0..n) = src_s[0..n)
  const double* src;
  double* dst;
  int64_t n;
  int gblocks;  // blocks [0, gblocks) gather, the rest copy
};

__global__ void __launch_bounds__(256) pi_gather_kernel(const mdp_problem P, const int32_t* sel,
                                                         const double* __restrict__ x3,
                                                         const double* __restrict__ x1, int64_t ld,
                                                         double* __restrict__ s_out, const CopyArgs CP) {
  MDP_PDL_ENTER();
  const int s = sys_of(sel, blockIdx.y);
  const int gb = CP.dst ? CP.gblocks : gridDim.x;
  if ((int)blockIdx.x >= gb) {
    const double* a = CP.src + s * ld;
    double* d = CP.dst + s * ld;
    for (int64_t e = (blockIdx.x - gb) * (int64_t)blockDim.x + threadIdx.x; e < CP.n;
         e += (int64_t)(gridDim.x - gb) * blockDim.x)
      d[e] = a[e];
    return;
  }
  gather_rows(P, s, blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), gb * (blockDim.x >> 5), x3, x1, ld, s_out);
}

// y3[u] += alpha w_s (T^T s)[u] (/ div[u] when div is given: the Jacobi
// coupling correction): 8 lanes per touched free node, no atomics
__device__ __forceinline__ void pull_rows(const mdp_problem& P, int s, int g0, int gstride,
                                          const double* __restrict__ sv, double alpha, double* __restrict__ y3,
                                          int64_t ld, const double* __restrict__ div) {
  const int sub = threadIdx.x & 7;
  const int ucount = P.u_start[s + 1] - P.u_start[s];
  // launch-invariant list data of this group's first node, fetched BEFORE the grid dependency wait (the
  // kernel is launched as a programmatic dependent: its launch latency and this DRAM round trip overlap
  // the stencil's tail); s and y3 are only touched after the wait
  int q_first = 0, node_first = 0;
  double v_first = 0.0;
  if (g0 < ucount) {
    const int u0 = P.u_start[s] + g0;
    node_first = P.u_node[u0];
    if (P.ell_q && sub < P.ell_w) {
      q_first = P.ell_q[(int64_t)u0 * P.ell_w + sub];
      v_first = P.ell_val[(int64_t)u0 * P.ell_w + sub];
    }
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  // the 8-lane groups of a warp iterate together (shuffles need all lanes)
  const int gfirst = g0 - ((threadIdx.x & 31) >> 3);
  for (int it = 0; gfirst + it * gstride < ucount; ++it) {
    const int base = g0 + it * gstride;
    const int u = P.u_start[s] + base;
    const bool live = base < ucount;
    double acc = 0.0;
    // the read-modify-write operand (and the divisor) are fetched ahead of the entry loads: their
    // DRAM round trip overlaps the list's instead of following the reduction
    int64_t g = 0;
    double yv = 0.0, dv = 1.0;
    if (live && sub == 0) {
      g = (int64_t)s * ld + (it == 0 ? node_first : P.u_node[u]);
      yv = y3[g];
      if (div) dv = div[g];
    }
    if (live)
      if (P.ell_q) {  // fixed-width rows: the entry loads depend on u only
        const int64_t b = (int64_t)u * P.ell_w;
        if (it == 0) {
          if (sub < P.ell_w) acc += v_first * sv[q_first];
          for (int k = sub + 8; k < P.ell_w; k += 8) acc += P.ell_val[b + k] * sv[P.ell_q[b + k]];
        } else {
          for (int k = sub; k < P.ell_w; k += 8) acc += P.ell_val[b + k] * sv[P.ell_q[b + k]];
        }
        // rows wider than the table continue in the CSR list (lane = entry index mod 8 either way)
        for (int k = P.u_ptr[u] + P.ell_w + sub; k < P.u_ptr[u + 1]; k += 8) acc += P.u_val[k] * sv[P.u_q[k]];
      } else {
        for (int k = P.u_ptr[u] + sub; k < P.u_ptr[u + 1]; k += 8) acc += P.u_val[k] * sv[P.u_q[k]];
      }
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (live && sub == 0) {
      if (div)
        y3[g] = yv - (-alpha * (P.wc[s] * acc)) / dv;
      else
        y3[g] = yv + alpha * P.wc[s] * acc;
    }
  }
}

// y1 = K11 x1 - w D Psi^T s: 4 lanes per 1D row
__device__ __forceinline__ void oned_rows(const mdp_problem& P, int s, int g0, int gstride,
                                          const double* __restrict__ x1, const double* __restrict__ sv,
                                          double* __restrict__ y1, int64_t ld) {
  const int sub = threadIdx.x & 3;
  const int rcount = P.r1_start[s + 1] - P.r1_start[s];
  const double* xp = x1 + (int64_t)s * ld;
  const int gfirst = g0 - ((threadIdx.x & 31) >> 2);
  for (int it = 0; gfirst + it * gstride < rcount; ++it) {
    const int base = g0 + it * gstride;
    const int r = P.r1_start[s] + base;
    const bool live = base < rcount;
    double a = 0.0, b = 0.0;
    if (live) {
      for (int k = P.k_ptr[r] + sub; k < P.k_ptr[r + 1]; k += 4) a += P.k_val[k] * xp[P.k_col[k]];
      for (int k = P.p_ptr[r] + sub; k < P.p_ptr[r + 1]; k += 4) b += P.p_val[k] * sv[P.p_q[k]];
    }
#pragma unroll
    for (int o = 2; o > 0; o >>= 1) {
      a += __shfl_xor_sync(0xffffffffu, a, o);
      b += __shfl_xor_sync(0xffffffffu, b, o);
    }
    if (live && sub == 0) y1[(int64_t)s * ld + base] = a - P.wc[s] * b;
  }
}

// Second phase of the coupled / reduced SpMV and of the Jacobi sweep in one
// launch: blocks [0, bpull) pull T^T s into y3, the rest form the 1D rows.
__global__ void __launch_bounds__(256) coupling_phase2_kernel(const mdp_problem P, const int32_t* sel, int bpull,
                                                               const double* __restrict__ sv, double alpha,
                                                               double* __restrict__ y3, int64_t ld,
                                                               const double* __restrict__ div,
                                                               const double* __restrict__ x1,
                                                               double* __restrict__ y1) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int s = sys_of(sel, blockIdx.y);
  if ((int)blockIdx.x < bpull) {
    pull_rows(P, s, blockIdx.x * (blockDim.x >> 3) + (threadIdx.x >> 3), bpull * (blockDim.x >> 3), sv, alpha, y3,
              ld, div);  // waits on the previous grid after its list prologue
  } else if (y1) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int b = blockIdx.x - bpull, nb = gridDim.x - bpull;
    oned_rows(P, s, b * (blockDim.x >> 2) + (threadIdx.x >> 2), nb * (blockDim.x >> 2), x1, sv, y1, ld);
  }
}

// x_out = x + (omega (r - Cx)) / diag  (Cx in tmp); x == NULL means x = 0 and Cx = 0
__global__ void jacobi_update_kernel(const mdp_problem P, const int32_t* sel, const double* __restrict__ r,
                                     const double* __restrict__ x, const double* __restrict__ cx,
                                     double* __restrict__ xo, double omega) {
  MDP_PDL_ENTER();
  const int s = sys_of(sel, blockIdx.y);
  const int64_t n3 = (int64_t)P.n * P.n * P.n;
  const int64_t base = (int64_t)s * P.ld;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n3;
       i += (int64_t)gridDim.x * blockDim.x) {
    double d = P.diag_c[base + i];
    if (x) {
      xo[base + i] = x[base + i] + (omega * (r[base + i] - cx[base + i])) / d;
    } else {
      xo[base + i] = (omega * r[base + i]) / d;
    }
  }
}

// min over segments of |p - (a + clip((p-a).ab / ab.ab, 0, 1) ab)|
__global__ void __launch_bounds__(256) distance_kernel(int n, const double* __restrict__ seg, int nseg,
                                                        double* __restrict__ out) {
  MDP_PDL_ENTER();
  __shared__ double sh[256 * 6];
  const int64_t n3 = (int64_t)n * n * n;
  const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const double h = 1.0 / (n - 1);
  double px = 0, py = 0, pz = 0;
  if (v < n3) {
    px = (double)(v % n) * h;
    py = (double)((v / n) % n) * h;
    pz = (double)(v / ((int64_t)n * n)) * h;
  }
  double best = INFINITY;
  for (int e0 = 0; e0 < nseg; e0 += 256) {
    const int ne = min(256, nseg - e0);
    __syncthreads();
    for (int t = threadIdx.x; t < ne * 6; t += blockDim.x) sh[t] = seg[(int64_t)e0 * 6 + t];
    __syncthreads();
    for (int e = 0; e < ne; ++e) {
      const double ax = sh[6 * e], ay = sh[6 * e + 1], az = sh[6 * e + 2];
      const double bx = sh[6 * e + 3] - ax, by = sh[6 * e + 4] - ay, bz = sh[6 * e + 5] - az;
      const double dx = px - ax, dy = py - ay, dz = pz - az;
      double t = (dx * bx + dy * by + dz * bz) / (bx * bx + by * by + bz * bz);
      t = fmin(fmax(t, 0.0), 1.0);
      const double qx = px - (ax + t * bx), qy = py - (ay + t * by), qz = pz - (az + t * bz);
      best = fmin(best, sqrt(qx * qx + qy * qy + qz * qz));
    }
  }
  if (v < n3) out[v] = best;
}

static int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}

template <int N, int RY>
static void launch_stencil3_attr() {
  static bool attr = false;  // opt in to > 48 KB dynamic shared memory once per instantiation
  if (!attr) {
    cudaFuncSetAttribute(stencil3_kernel<N, RY, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(stencil3_kernel<N, RY, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(stencil3_kernel<N, RY, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
}

template <int N, int RY>
static void launch_stencil3_t(dim3 grid, int threads, size_t smem, cudaStream_t st, const mdp_problem* p,
                              const int32_t* sel, const double* x, int64_t ldx, double* y, int64_t ldy, int zchunk,
                              const double* jr, double omega, const GatherArgs& G, bool lastcol) {
  launch_stencil3_attr<N, RY>();
  static const int dep = env_int("MDP_STENCIL_PDL", 1);
  if (!jr && lastcol) {
    if (dep)
      ::mdp::launch_k_dependent(stencil3_kernel<N, RY, false, true>, grid, threads, smem, st, *p, sel, x, ldx, y, ldy,
                                zchunk, jr, omega, G);
    else
      ::mdp::launch_k(stencil3_kernel<N, RY, false, true>, grid, threads, smem, st, *p, sel, x, ldx, y, ldy, zchunk, jr,
                      omega, G);
  } else if (jr) {
    if (dep)
      ::mdp::launch_k_dependent(stencil3_kernel<N, RY, true>, grid, threads, smem, st, *p, sel, x, ldx, y, ldy, zchunk,
                                jr, omega, G);
    else
      ::mdp::launch_k(stencil3_kernel<N, RY, true>, grid, threads, smem, st, *p, sel, x, ldx, y, ldy, zchunk, jr, omega,
                      G);
  } else {
    if (dep)
      ::mdp::launch_k_dependent(stencil3_kernel<N, RY, false>, grid, threads, smem, st, *p, sel, x, ldx, y, ldy, zchunk,
                                jr, omega, G);
    else
      ::mdp::launch_k(stencil3_kernel<N, RY, false>, grid, threads, smem, st, *p, sel, x, ldx, y, ldy, zchunk, jr,
                      omega, G);
  }
}

// resident blocks per SM of one instantiation at this launch shape (registers AND shared memory;
// the 156-register consumer holds 129^3 to 2 blocks of 192 threads per SM, not the 5 its ring would allow)
template <int N, int RY>
static int stencil3_blocks_per_sm(int threads, size_t smem, bool jac, int n, bool lc) {
  static int cache[3][2] = {{0, 0}, {0, 0}, {0, 0}};  // [plain | Jacobi | plain last-column] -> (n, blocks)
  int* c = cache[jac ? 1 : (lc ? 2 : 0)];
  const int key = n * 2048 + threads;
  if (c[0] == key && c[1] > 0) return c[1];
  launch_stencil3_attr<N, RY>();
  int nb = 0;
  cudaError_t e =
      jac  ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, stencil3_kernel<N, RY, true>, threads, smem)
      : lc ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, stencil3_kernel<N, RY, false, true>, threads, smem)
           : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, stencil3_kernel<N, RY, false>, threads, smem);
  if (e != cudaSuccess || nb < 1) {
    cudaGetLastError();
    nb = 1;
  }
  c[0] = key;
  c[1] = nb;
  return nb;
}

// v3 launch: one block per (RY-row band, z-chunk, system): tiles_x consumer
// warps + 1 producer warp, S shared-memory plane stages
static int launch_stencil3(const mdp_problem* p, int32_t nsel, const int32_t* sel, const double* x, int64_t ldx,
                           double* y, int64_t ldy, cudaStream_t st, const double* jr, double omega,
                           const GatherArgs* g) {
  const int n = p->n;
  static const int ry_env = env_int("MDP_STENCIL_RY", 0);
  const int RY = ry_env == 2 || ry_env == 4 || ry_env == 8 ? ry_env : (n <= 48 ? 2 : 4);
  const int S = kSt3;
  const bool lastcol = jr == nullptr && nsel >= 2 && p->bc3d != 0 && n > 32 && ((n - 1) & 31) == 0;  // see stencil3_consumer
  const int tiles_x = lastcol ? (n - 1) / 32 : ceil_div(n, 32);
  const int bands = ceil_div(n, RY);
  const int threads = 32 * (tiles_x + 1);
  const size_t sw = (size_t)(((RY + 2) * n + 4 + 1) & ~1);
  const size_t swj = jr ? (size_t)((RY * n + 3) & ~1) : 0;  // Jacobi: r and diag(C) bands ride in the stage
  const size_t smem = 16 * (size_t)S + (size_t)S * (sw + 2 * swj) * 8 + 32;
  MDP_REQUIRE(smem <= 200 * 1024, "stencil stage ring of %zu bytes exceeds shared memory (n = %d, RY = %d)", smem, n, RY);
  // z-chunks.  A block's life is a serial chain: ring set-up + the first DRAM round trip (~3.5 plane
  // steps' worth, traced) and then one step per plane of its chunk plus 2 halo planes; blocks run in waves
  // of (resident blocks per SM) x SMs.  Pick the chunk count that minimises waves x chain length.
  int per_sm = 1;
#define MDP_ST3O(NN, R) per_sm = stencil3_blocks_per_sm<NN, R>(threads, smem, jr != nullptr, n, lastcol)
  if (RY == 2) {
    switch (n) {
      case 17: MDP_ST3O(17, 2); break;
      case 33: MDP_ST3O(33, 2); break;
      default: MDP_ST3O(0, 2); break;
    }
  } else if (RY == 8) {
    MDP_ST3O(0, 8);
  } else {
    switch (n) {
      case 65: MDP_ST3O(65, 4); break;
      case 129: MDP_ST3O(129, 4); break;
      case 193: MDP_ST3O(193, 4); break;
      default: MDP_ST3O(0, 4); break;
    }
  }
#undef MDP_ST3O
  const int64_t slots = (int64_t)per_sm * sm_count();
  const int minlen = n <= 48 ? 2 : 8;
  const int zmax = n / minlen > 1 ? n / minlen : 1;
  int zch = 1;
  double best = 1e300;
  for (int c = 1; c <= zmax; ++c) {
    const int len = ceil_div(n, c);
    // chunks beyond ~40 planes lose in the coupled / Jacobi launches (few long blocks: the dependent
    // phase-2 launch waits on the slowest; profiles/r02_stencil_stream.txt)
    if (len > 40 && c < zmax) continue;
    const int64_t blocks = (int64_t)bands * ceil_div(n, len) * nsel;
    const double cost = (double)ceil_div(blocks, slots) * (3.5 + len + 2);
    if (cost < best - 1e-9) {
      best = cost;
      zch = c;
    }
  }
  int zchunk = ceil_div(n, zch);
  static const int forced = env_int("MDP_STENCIL_ZCHUNK", 0);
  if (forced > 0) zchunk = forced < n ? forced : n;
  zch = ceil_div(n, zchunk);
  const bool gat = g != nullptr && p->qmax > 0;
  GatherArgs G = gat ? *g : GatherArgs{nullptr, nullptr, nullptr, 0};
  if (gat) G.nblk = ceil_div(p->qmax, (tiles_x + 1) * 2);  // ~2 quadrature rows per warp
  dim3 grid(G.nblk + bands * zch, nsel);
#define MDP_ST3L(NN, R) \
  launch_stencil3_t<NN, R>(grid, threads, smem, st, p, sel, x, ldx, y, ldy, zchunk, jr, omega, G, lastcol)
  if (RY == 2) {
    switch (n) {
      case 17: MDP_ST3L(17, 2); break;
      case 33: MDP_ST3L(33, 2); break;
      default: MDP_ST3L(0, 2); break;
    }
  } else if (RY == 8) {
    MDP_ST3L(0, 8);
  } else {
    switch (n) {
      case 65: MDP_ST3L(65, 4); break;
      case 129: MDP_ST3L(129, 4); break;
      case 193: MDP_ST3L(193, 4); break;
      default: MDP_ST3L(0, 4); break;
    }
  }
#undef MDP_ST3L
  MDP_LAUNCH_CHECK("stencil3_kernel");
  return MDP_OK;
}

static int launch_stencil(const mdp_problem* p, int32_t nsel, const int32_t* sel, const double* x,
                          int64_t ldx, double* y, int64_t ldy, cudaStream_t st, const double* jr = nullptr,
                          double omega = 0.0, const GatherArgs* g = nullptr) {
  static const int version = env_int("MDP_STENCIL_V", 3);  // 1: the v1 kernel (A/B)
  if (version == 3 && ceil_div(p->n, 32) <= 7) return launch_stencil3(p, nsel, sel, x, ldx, y, ldy, st, jr, omega, g);
  const int n = p->n;
  const int64_t warps = (int64_t)ceil_div(n, 30) * ceil_div(n, STENCIL_ROWS);  // (x-tile, row group) per plane
  int bx = ceil_div(warps, 4);
  // z-chunks: enough warps to fill the machine; chunks of >= 16 planes when the
  // problem is large, down to 4 planes when it is latency-bound anyway
  int64_t want = (int64_t)48 * 4 * sm_count();
  int zch = ceil_div(want, warps * nsel);
  // (latency-bound small grids: 2-plane chunks measured 3% faster in-solve at 33^3)
  const int zmin_len = warps * nsel * (n / 16) >= want ? 16 : (n <= 48 ? 2 : 4);
  const int zmax = n <= 48 ? ceil_div(n, zmin_len) : (n / zmin_len > 1 ? n / zmin_len : 1);
  zch = zch < 1 ? 1 : (zch > zmax ? zmax : zch);
  int zchunk = ceil_div(n, zch);
  {
    static int forced = -1;  // MDP_STENCIL_ZCHUNK: tuning experiments only (tools/stencil_sweep.py)
    if (forced < 0) {
      const char* e = getenv("MDP_STENCIL_ZCHUNK");
      forced = e ? atoi(e) : 0;
    }
    if (forced > 0) zchunk = forced < n ? forced : n;
  }
  zch = ceil_div(n, zchunk);
  const bool gat = g != nullptr && p->qmax > 0;
  if (gat) bx = bx > ceil_div(p->qmax, 4) ? bx : ceil_div(p->qmax, 4);  // one warp per Pi row in the gather slice
  dim3 grid(bx, zch + (gat ? 1 : 0), nsel);
  GatherArgs G = gat ? *g : GatherArgs{nullptr, nullptr, nullptr, 0};
  if (jr) {
    if (gat)
      ::mdp::launch_k(stencil_kernel<true, true>, grid, 128, 0, st, *p, sel, x, ldx, y, ldy, zchunk, jr, omega, G);
    else
      ::mdp::launch_k(stencil_kernel<true, false>, grid, 128, 0, st, *p, sel, x, ldx, y, ldy, zchunk, jr, omega, G);
  } else {
    if (gat)
      ::mdp::launch_k(stencil_kernel<false, true>, grid, 128, 0, st, *p, sel, x, ldx, y, ldy, zchunk, jr, omega, G);
    else
      ::mdp::launch_k(stencil_kernel<false, false>, grid, 128, 0, st, *p, sel, x, ldx, y, ldy, zchunk, jr, omega, G);
  }
  MDP_LAUNCH_CHECK("stencil_kernel");
  return MDP_OK;
}

static int launch_gather(const mdp_problem* p, int32_t nsel, const int32_t* sel, const double* x3,
                         const double* x1, int64_t ld, double* s, cudaStream_t st,
                         const double* csrc = nullptr, double* cdst = nullptr, int64_t cn = 0) {
  const int gb = p->qmax > 0 ? ceil_div(p->qmax, 8) : 0;
  int cb = 0;
  if (cdst && cn > 0) {
    cb = ceil_div(cn, 256);
    cb = cb > 4 * sm_count() ? 4 * sm_count() : cb;
  }
  if (gb + cb == 0) return MDP_OK;
  dim3 grid(gb + cb, nsel);
  const CopyArgs CP{csrc, cb ? cdst : nullptr, cn, gb};
  ::mdp::launch_k(pi_gather_kernel, grid, 256, 0, st, *p, sel, x3, x1, ld, s, CP);
  MDP_LAUNCH_CHECK("pi_gather_kernel");
  return MDP_OK;
}

// pull T^T s into y3 (and, with y1, the 1D rows) in one launch
static int launch_phase2(const mdp_problem* p, int32_t nsel, const int32_t* sel, const double* s, double alpha,
                         double* y3, int64_t ld, cudaStream_t st, const double* div, const double* x1,
                         double* y1) {
  const int bpull = p->umax > 0 ? ceil_div(p->umax, 32) : 0;
  const int boned = (y1 && p->r1max > 0) ? ceil_div(p->r1max, 64) : 0;
  if (bpull + boned == 0) return MDP_OK;
  dim3 grid(bpull + boned, nsel);
  static const int dep = env_int("MDP_PHASE2_PDL", 1);
  if (dep)
    ::mdp::launch_k_dependent(coupling_phase2_kernel, grid, 256, 0, st, *p, sel, bpull, s, alpha, y3, ld, div, x1, y1);
  else
    ::mdp::launch_k(coupling_phase2_kernel, grid, 256, 0, st, *p, sel, bpull, s, alpha, y3, ld, div, x1, y1);
  MDP_LAUNCH_CHECK("coupling_phase2_kernel");
  return MDP_OK;
}

static int validate(const mdp_problem* p, int32_t nsel) {
  MDP_REQUIRE(p != nullptr, "null problem descriptor");
  MDP_REQUIRE(p->n >= 2, "grid needs at least 2 points per edge, got %d", p->n);
  MDP_REQUIRE(nsel >= 0 && nsel <= p->nsys, "nsel %d out of range (nsys %d)", nsel, p->nsys);
  MDP_REQUIRE(p->ld >= (int64_t)p->n * p->n * p->n, "vector stride too small");
  return MDP_OK;
}

// Stencil launch + the Pi gather s = W (T x3 - Psi D x1).  Small grids: the gather rides in the
// stencil launch (first blocks; one launch fewer on a latency-bound step).  Wide grids: gather blocks
// inside the stencil launch inherit its footprint (150 registers, a stage ring: 2 blocks per SM), so
// their dependent-load chains hold stencil slots at 12 warps per SM; for batches of wide grids the
// gather is its own launch of light blocks ahead of the stencil (129^3 x 64 coupled SpMV 594 -> 513 us,
// 65^3 x 16 52 -> 44 us; one 129^3 system is 1 us faster folded; MDP_GATHER_MODE=0/1 forces either).
static int stencil_and_gather(const mdp_problem* p, int32_t nsel, const int32_t* sel, const double* x, int64_t ldx,
                              double* y, int64_t ldy, cudaStream_t st, const double* jr, double omega,
                              const GatherArgs& g) {
  static const int mode = env_int("MDP_GATHER_MODE", -1);
  const bool separate = mode >= 0 ? mode == 1 : (p->n >= 65 && nsel >= 4);
  if (!separate) return launch_stencil(p, nsel, sel, x, ldx, y, ldy, st, jr, omega, &g);
  if (int rc = launch_gather(p, nsel, sel, g.x3, g.x1, ldx, g.s_out, st)) return rc;
  return launch_stencil(p, nsel, sel, x, ldx, y, ldy, st, jr, omega, nullptr);
}

}  // namespace mdp

using namespace mdp;

extern "C" int mdp_distance_field(int32_t n, const double* seg, int32_t nseg, double* out, void* stream) {
  MDP_REQUIRE(n >= 2 && nseg >= 1, "distance field needs n>=2 and at least one segment");
  const int64_t n3 = (int64_t)n * n * n;
  ::mdp::launch_k(distance_kernel, ceil_div(n3, 256), 256, 0, (cudaStream_t)stream, n, seg, nseg, out);
  MDP_LAUNCH_CHECK("distance_kernel");
  return MDP_OK;
}

extern "C" int mdp_stencil_apply(const mdp_problem* p, int32_t nsel, const int32_t* sel,
                                 const double* x3, int64_t ldx, double* y3, int64_t ldy,
                                 void* stream) {
  if (int rc = validate(p, nsel)) return rc;
  if (nsel == 0) return MDP_OK;
  return launch_stencil(p, nsel, sel, x3, ldx, y3, ldy, (cudaStream_t)stream);
}

extern "C" int mdp_pi_gather(const mdp_problem* p, int32_t nsel, const int32_t* sel,
                             const double* x3, const double* x1, int64_t ld, double* s,
                             void* stream) {
  if (int rc = validate(p, nsel)) return rc;
  if (nsel == 0) return MDP_OK;
  return launch_gather(p, nsel, sel, x3, x1, ld, s, (cudaStream_t)stream);
}

extern "C" int mdp_pi_gather_copy(const mdp_problem* p, int32_t nsel, const int32_t* sel, const double* x3,
                                  const double* x1, int64_t ld, double* s, const double* csrc, double* cdst,
                                  int64_t cn, void* stream) {
  if (int rc = validate(p, nsel)) return rc;
  MDP_REQUIRE(csrc && cdst && cn >= 0, "gather+copy needs a source and a destination");
  if (nsel == 0) return MDP_OK;
  return launch_gather(p, nsel, sel, x3, x1, ld, s, (cudaStream_t)stream, csrc, cdst, cn);
}

extern "C" int mdp_pi_scatter(const mdp_problem* p, int32_t nsel, const int32_t* sel,
                              const double* s, double alpha, double* y3, int64_t ld,
                              void* stream) {
  if (int rc = validate(p, nsel)) return rc;
  if (nsel == 0) return MDP_OK;
  return launch_phase2(p, nsel, sel, s, alpha, y3, ld, (cudaStream_t)stream, nullptr, nullptr, nullptr);
}

extern "C" int mdp_coupled_spmv(const mdp_problem* p, int32_t nsel, const int32_t* sel,
                                const double* x, double* y, double* s_work, void* stream) {
  if (int rc = validate(p, nsel)) return rc;
  if (nsel == 0) return MDP_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t n3 = (int64_t)p->n * p->n * p->n;
  // launch 1: stencil y3 = K00 x3 with the Pi gather s = W (T x3 - Psi D x1) alongside;
  // launch 2: y3 += w T^T s and y1 = K11 x1 - w D Psi^T s
  GatherArgs g{x, x + n3, s_work};
  int rc;
  if ((rc = stencil_and_gather(p, nsel, sel, x, p->ld, y, p->ld, st, nullptr, 0.0, g))) return rc;
  return launch_phase2(p, nsel, sel, s_work, 1.0, y, p->ld, st, nullptr, x + n3, y + n3);
}

extern "C" int mdp_reduced_spmv(const mdp_problem* p, int32_t nsel, const int32_t* sel,
                                const double* x3, double* y3, double* s_work, void* stream) {
  if (int rc = validate(p, nsel)) return rc;
  if (nsel == 0) return MDP_OK;
  cudaStream_t st = (cudaStream_t)stream;
  GatherArgs g{x3, nullptr, s_work};
  int rc;
  if ((rc = stencil_and_gather(p, nsel, sel, x3, p->ld, y3, p->ld, st, nullptr, 0.0, g))) return rc;
  return launch_phase2(p, nsel, sel, s_work, 1.0, y3, p->ld, st, nullptr, nullptr, nullptr);
}

extern "C" int mdp_jacobi_sweep(const mdp_problem* p, int32_t nsel, const int32_t* sel,
                                const double* r, const double* x, double* x_out, double omega,
                                double* tmp, double* s_work, void* stream) {
  if (int rc = validate(p, nsel)) return rc;
  MDP_REQUIRE(p->diag_c != nullptr, "jacobi sweep needs diag(C) in the problem descriptor");
  if (nsel == 0) return MDP_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (x) {
    // fused sweep: s = W T x; out = x + omega (r - K00 x) / d in the stencil
    // epilogue; then out -= omega w (T^T s) / d at the touched nodes
    GatherArgs g{x, nullptr, s_work};
    int rc;
    if ((rc = stencil_and_gather(p, nsel, sel, x, p->ld, x_out, p->ld, st, r, omega, g))) return rc;
    return launch_phase2(p, nsel, sel, s_work, -omega, x_out, p->ld, st, p->diag_c, nullptr, nullptr);
  }
  (void)tmp;
  const int64_t n3 = (int64_t)p->n * p->n * p->n;
  int bx = ceil_div(n3, 256);
  bx = bx > 4096 ? 4096 : bx;
  ::mdp::launch_k(jacobi_update_kernel, dim3(bx, nsel), 256, 0, st, *p, sel, r, x, tmp, x_out, omega);
  MDP_LAUNCH_CHECK("jacobi_update_kernel");
  return MDP_OK;
}

#ifdef ST3_TRACE
extern "C" int mdp_st3_trace_read(long long* host) {
  return (int)cudaMemcpyFromSymbol(host, mdp::g_st3_trace, sizeof(long long) * 3 * 64);
}
#endif
