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

// One CTA: TX x TY columns of one system, z in [z0, z1).
template <int TX, int TY>
__global__ void __launch_bounds__(TX* TY) stencil_kernel(const mdp_problem P, const int32_t* sel,
                                                         const double* __restrict__ x, int64_t ldx,
                                                         double* __restrict__ y, int64_t ldy,
                                                         int zchunk) {
  __shared__ double xs[TY + 2][TX + 2];
  __shared__ double sa[TY + 2][TX];
  __shared__ double sb[TY + 2][TX];
  const int n = P.n;
  const int s = sys_of(sel, blockIdx.z);
  const double* xp = x + (int64_t)s * ldx;
  double* yp = y + (int64_t)s * ldy;
  const int tiles_x = (n + TX - 1) / TX;
  const int i0 = (blockIdx.x % tiles_x) * TX;
  const int j0 = (blockIdx.x / tiles_x) * TY;
  const int z0 = blockIdx.y * zchunk;
  const int z1 = min(n, z0 + zchunk);
  if (z0 >= n) return;
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * TX + tx;
  const int i = i0 + tx, j = j0 + ty;
  const bool dir = P.bc3d != 0;
  const Line1D c = make_line(P.h);
  const double kO = P.k_omega, sO = P.sigma_omega;
  const int64_t nn = (int64_t)n * n;

  double Pm = 0.0, P0 = 0.0, Rm = 0.0, R0 = 0.0;
  for (int kk = z0 - 1; kk <= z1; ++kk) {
    double Pn = 0.0, Rn = 0.0;
    const bool plane_ok = (kk >= 0 && kk < n);
    if (plane_ok) {
      for (int t = tid; t < (TY + 2) * (TX + 2); t += TX * TY) {
        int ly = t / (TX + 2), lx = t - ly * (TX + 2);
        int gi = i0 + lx - 1, gj = j0 + ly - 1;
        double v = 0.0;
        if (gi >= 0 && gi < n && gj >= 0 && gj < n) {
          if (!(dir && on_boundary(gi, gj, kk, n))) v = __ldg(xp + kk * nn + (int64_t)gj * n + gi);
        }
        xs[ly][lx] = v;
      }
      __syncthreads();
      for (int t = tid; t < (TY + 2) * TX; t += TX * TY) {
        int ly = t / TX, lx = t - ly * TX;
        int gi = i0 + lx;
        double kd = kdiag(c, gi, n), md = mdiag(c, gi, n);
        double a = c.ko * xs[ly][lx] + kd * xs[ly][lx + 1] + c.ko * xs[ly][lx + 2];
        double b = c.mo * xs[ly][lx] + md * xs[ly][lx + 1] + c.mo * xs[ly][lx + 2];
        sa[ly][lx] = a;
        sb[ly][lx] = b;
      }
      __syncthreads();
      double kd = kdiag(c, j, n), md = mdiag(c, j, n);
      double c1 = c.mo * sa[ty][tx] + md * sa[ty + 1][tx] + c.mo * sa[ty + 2][tx];
      double c2 = c.ko * sb[ty][tx] + kd * sb[ty + 1][tx] + c.ko * sb[ty + 2][tx];
      double c3 = c.mo * sb[ty][tx] + md * sb[ty + 1][tx] + c.mo * sb[ty + 2][tx];
      Pn = kO * (c1 + c2) + sO * c3;
      Rn = kO * c3;
    }
    const int ko = kk - 1;  // output plane
    if (ko >= z0 && ko < z1 && i < n && j < n) {
      double kd = kdiag(c, ko, n), md = mdiag(c, ko, n);
      double out = c.mo * Pm + md * P0 + c.mo * Pn + c.ko * Rm + kd * R0 + c.ko * Rn;
      int64_t idx = ko * nn + (int64_t)j * n + i;
      if (dir && on_boundary(i, j, ko, n)) out = xp[idx];
      yp[idx] = out;
    }
    Pm = P0; P0 = Pn;
    Rm = R0; R0 = Rn;
  }
}

// s_q = W_q ((T x3)_q - (Psi D x1)_q): one warp per quadrature row, lanes
// over the row's (point, corner) entries (8 for the centreline, up to 64
// for the 8-point ring average), warp-shuffle reduction.  Entries on
// eliminated (Dirichlet) cube nodes are dropped from T at build time.
__global__ void __launch_bounds__(256) pi_gather_kernel(const mdp_problem P, const int32_t* sel,
                                                         const double* __restrict__ x3,
                                                         const double* __restrict__ x1, int64_t ld,
                                                         double* __restrict__ s_out) {
  const int s = sys_of(sel, blockIdx.y);
  const int lane = threadIdx.x & 31;
  const int q = P.q_start[s] + blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (q >= P.q_start[s + 1]) return;
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

// y3[u] += alpha w_s (T^T s)[u]: 8 lanes per touched free node, no atomics
__global__ void __launch_bounds__(256) pi_pull_kernel(const mdp_problem P, const int32_t* sel,
                                                       const double* __restrict__ sv, double alpha,
                                                       double* __restrict__ y3, int64_t ld) {
  const int s = sys_of(sel, blockIdx.y);
  const int sub = threadIdx.x & 7;
  const int u = P.u_start[s] + blockIdx.x * (blockDim.x >> 3) + (threadIdx.x >> 3);
  const bool live = u < P.u_start[s + 1];
  double acc = 0.0;
  if (live)
    for (int k = P.u_ptr[u] + sub; k < P.u_ptr[u + 1]; k += 8) acc += P.u_val[k] * sv[P.u_q[k]];
#pragma unroll
  for (int o = 4; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (live && sub == 0) y3[(int64_t)s * ld + P.u_node[u]] += alpha * P.wc[s] * acc;
}

// y1 = K11 x1 - w D Psi^T s: 4 lanes per 1D row
__global__ void __launch_bounds__(256) oned_kernel(const mdp_problem P, const int32_t* sel,
                                                    const double* __restrict__ x1, const double* __restrict__ sv,
                                                    double* __restrict__ y1, int64_t ld) {
  const int s = sys_of(sel, blockIdx.y);
  const int sub = threadIdx.x & 3;
  const int r = P.r1_start[s] + blockIdx.x * (blockDim.x >> 2) + (threadIdx.x >> 2);
  const bool live = r < P.r1_start[s + 1];
  const double* xp = x1 + (int64_t)s * ld;
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
  if (live && sub == 0) y1[(int64_t)s * ld + (r - P.r1_start[s])] = a - P.wc[s] * b;
}

// x_out = x + (omega (r - Cx)) / diag  (Cx in tmp); x == NULL means x = 0 and Cx = 0
__global__ void jacobi_update_kernel(const mdp_problem P, const int32_t* sel, const double* __restrict__ r,
                                     const double* __restrict__ x, const double* __restrict__ cx,
                                     double* __restrict__ xo, double omega) {
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

static int launch_stencil(const mdp_problem* p, int32_t nsel, const int32_t* sel, const double* x,
                          int64_t ldx, double* y, int64_t ldy, cudaStream_t st) {
  const int n = p->n;
  constexpr int TX = 32, TY = 8;
  int tiles = ceil_div(n, TX) * ceil_div(n, TY);
  int want = 6 * sm_count();
  int zch = ceil_div(want, (int64_t)tiles * nsel);
  zch = zch < 1 ? 1 : (zch > n ? n : zch);
  int zchunk = ceil_div(n, zch);
  zch = ceil_div(n, zchunk);
  dim3 grid(tiles, zch, nsel), block(TX, TY);
  stencil_kernel<TX, TY><<<grid, block, 0, st>>>(*p, sel, x, ldx, y, ldy, zchunk);
  MDP_LAUNCH_CHECK("stencil_kernel");
  return MDP_OK;
}

static int launch_gather(const mdp_problem* p, int32_t nsel, const int32_t* sel, const double* x3,
                         const double* x1, int64_t ld, double* s, cudaStream_t st) {
  if (p->qmax <= 0) return MDP_OK;
  dim3 grid(ceil_div(p->qmax, 8), nsel);
  pi_gather_kernel<<<grid, 256, 0, st>>>(*p, sel, x3, x1, ld, s);
  MDP_LAUNCH_CHECK("pi_gather_kernel");
  return MDP_OK;
}

static int launch_pull(const mdp_problem* p, int32_t nsel, const int32_t* sel, const double* s,
                       double alpha, double* y3, int64_t ld, cudaStream_t st) {
  if (p->umax <= 0) return MDP_OK;
  dim3 grid(ceil_div(p->umax, 32), nsel);
  pi_pull_kernel<<<grid, 256, 0, st>>>(*p, sel, s, alpha, y3, ld);
  MDP_LAUNCH_CHECK("pi_pull_kernel");
  return MDP_OK;
}

static int launch_oned(const mdp_problem* p, int32_t nsel, const int32_t* sel, const double* x1,
                       const double* s, double* y1, int64_t ld, cudaStream_t st) {
  if (p->r1max <= 0) return MDP_OK;
  dim3 grid(ceil_div(p->r1max, 64), nsel);
  oned_kernel<<<grid, 256, 0, st>>>(*p, sel, x1, s, y1, ld);
  MDP_LAUNCH_CHECK("oned_kernel");
  return MDP_OK;
}

static int validate(const mdp_problem* p, int32_t nsel) {
  MDP_REQUIRE(p != nullptr, "null problem descriptor");
  MDP_REQUIRE(p->n >= 2, "grid needs at least 2 points per edge, got %d", p->n);
  MDP_REQUIRE(nsel >= 0 && nsel <= p->nsys, "nsel %d out of range (nsys %d)", nsel, p->nsys);
  MDP_REQUIRE(p->ld >= (int64_t)p->n * p->n * p->n, "vector stride too small");
  return MDP_OK;
}

}  // namespace mdp

using namespace mdp;

extern "C" int mdp_distance_field(int32_t n, const double* seg, int32_t nseg, double* out, void* stream) {
  MDP_REQUIRE(n >= 2 && nseg >= 1, "distance field needs n>=2 and at least one segment");
  const int64_t n3 = (int64_t)n * n * n;
  distance_kernel<<<ceil_div(n3, 256), 256, 0, (cudaStream_t)stream>>>(n, seg, nseg, out);
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

extern "C" int mdp_pi_scatter(const mdp_problem* p, int32_t nsel, const int32_t* sel,
                              const double* s, double alpha, double* y3, int64_t ld,
                              void* stream) {
  if (int rc = validate(p, nsel)) return rc;
  if (nsel == 0) return MDP_OK;
  return launch_pull(p, nsel, sel, s, alpha, y3, ld, (cudaStream_t)stream);
}

extern "C" int mdp_coupled_spmv(const mdp_problem* p, int32_t nsel, const int32_t* sel,
                                const double* x, double* y, double* s_work, void* stream) {
  if (int rc = validate(p, nsel)) return rc;
  if (nsel == 0) return MDP_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t n3 = (int64_t)p->n * p->n * p->n;
  int rc;
  if ((rc = launch_gather(p, nsel, sel, x, x + n3, p->ld, s_work, st))) return rc;
  if ((rc = launch_stencil(p, nsel, sel, x, p->ld, y, p->ld, st))) return rc;
  if ((rc = launch_pull(p, nsel, sel, s_work, 1.0, y, p->ld, st))) return rc;
  return launch_oned(p, nsel, sel, x + n3, s_work, y + n3, p->ld, st);
}

extern "C" int mdp_reduced_spmv(const mdp_problem* p, int32_t nsel, const int32_t* sel,
                                const double* x3, double* y3, double* s_work, void* stream) {
  if (int rc = validate(p, nsel)) return rc;
  if (nsel == 0) return MDP_OK;
  cudaStream_t st = (cudaStream_t)stream;
  int rc;
  if ((rc = launch_gather(p, nsel, sel, x3, nullptr, p->ld, s_work, st))) return rc;
  if ((rc = launch_stencil(p, nsel, sel, x3, p->ld, y3, p->ld, st))) return rc;
  return launch_pull(p, nsel, sel, s_work, 1.0, y3, p->ld, st);
}

extern "C" int mdp_jacobi_sweep(const mdp_problem* p, int32_t nsel, const int32_t* sel,
                                const double* r, const double* x, double* x_out, double omega,
                                double* tmp, double* s_work, void* stream) {
  if (int rc = validate(p, nsel)) return rc;
  MDP_REQUIRE(p->diag_c != nullptr, "jacobi sweep needs diag(C) in the problem descriptor");
  if (nsel == 0) return MDP_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (x) {
    int rc = mdp_reduced_spmv(p, nsel, sel, x, tmp, s_work, stream);
    if (rc) return rc;
  }
  const int64_t n3 = (int64_t)p->n * p->n * p->n;
  int bx = ceil_div(n3, 256);
  bx = bx > 4096 ? 4096 : bx;
  jacobi_update_kernel<<<dim3(bx, nsel), 256, 0, st>>>(*p, sel, r, x, tmp, x_out, omega);
  MDP_LAUNCH_CHECK("jacobi_update_kernel");
  return MDP_OK;
}
