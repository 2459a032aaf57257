/*
 * mdp_b200.h -- C ABI of the B200 (sm_100a) hot path of the neural-
 * preconditioned FGMRES solve for coupled 3D-1D systems (arXiv 2505.08491,
 * reference package `mdprec` at /root/reference/pkg/src/mdprec).
 *
 * Conventions
 *   - Every pointer in a call or descriptor is DEVICE memory unless marked
 *     [host].  Callers own all memory; kernels never allocate.
 *   - Every function returns 0 on success, MDP_EINVAL on a bad argument, or
 *     MDP_ECUDA on a CUDA launch/runtime error; mdp_last_error() describes it
 *     (thread-local).
 *   - `stream` is a cudaStream_t passed as void*.
 *   - Batched calls act on `nsel` systems listed in `sel` ([nsel] int32,
 *     device); sel == NULL means systems 0..nsel-1.  Full vectors of system s
 *     start at s*ld (3D part [0,n^3), 1D part [n^3, n^3+n1[s]), zero padding
 *     up to ld).
 *   - All system arithmetic is float64; the CNN computes in float32 with
 *     TF32 tensor-core products (tcgen05) and float32 accumulation.
 *
 * Each entry point names the reference interface it replaces.
 */
#ifndef MDP_B200_H
#define MDP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MDP_OK 0
#define MDP_EINVAL 1001
#define MDP_ECUDA 1002
#define MDP_EPIVOT 1003

/* ------------------------------------------------------------------ */
/* Coupled problem descriptor (batched over systems that share the grid).
 * Built on the host by paper_2505_08491_b200.assembly from the index sets
 * of assemble_coupled_system (assembly.py:306-348).                      */
typedef struct mdp_problem {
  int32_t n;            /* grid points per edge (geometry.py:27-43)        */
  int32_t nsys;         /* systems in the batch                             */
  int32_t bc3d;         /* 0: Neumann (reference), 1: homogeneous Dirichlet */
  int32_t pad0;
  int64_t ld;           /* per-system stride of full vectors                */
  double h, k_omega, sigma_omega;
  const double* wc;     /* [nsys] coupling weight w (assembly.py:48-51)     */
  const int32_t* n1;    /* [nsys] 1D unknowns                               */
  /* quadrature rows q (2 per 1D element, assembly.py:218-222), global ids */
  const int32_t* q_start;  /* [nsys+1]                                       */
  const int32_t* t_ptr;    /* [Qtot+1] row pointers of Pi = T (CSR)          */
  const int32_t* t_col;    /* local 3D node                                  */
  const double* t_val;
  const int32_t* psi_col;  /* [2*Qtot] local 1D node, -1 if Dirichlet (D)    */
  const double* psi_val;   /* [2*Qtot]                                       */
  const double* wq;        /* [Qtot] Gauss weights L_e/2 (W)                 */
  /* Pi^T as a pull over the touched (free) 3D nodes                        */
  const int32_t* u_start;  /* [nsys+1]                                       */
  const int32_t* u_node;   /* [Utot] local 3D node                           */
  const int32_t* u_ptr;    /* [Utot+1]                                       */
  const int32_t* u_q;      /* global quadrature row                          */
  const double* u_val;
  /* 1D rows: K11 after elimination (CSR) and D Psi^T W-free pull          */
  const int32_t* r1_start; /* [nsys+1] global 1D row offsets                 */
  const int32_t* k_ptr;    /* [R1tot+1]                                      */
  const int32_t* k_col;    /* local 1D node                                  */
  const double* k_val;
  const int32_t* p_ptr;    /* [R1tot+1] Psi^T rows (empty on Dirichlet rows) */
  const int32_t* p_q;      /* global quadrature row                          */
  const double* p_val;
  const double* diag_c;    /* [nsys*ld] diag(C) for Jacobi (or NULL)        */
  int32_t qmax, umax, r1max, pad1; /* per-system maxima (launch shapes)      */
  /* optional ELL copy of the head of the pull list: the first ell_w entries of
   * touched node u at [u*ell_w, (u+1)*ell_w), padded with value 0 (no
   * row-pointer load on the pull's dependent-load chain); entries beyond
   * ell_w are read from u_ptr / u_q / u_val.  NULL: use only u_ptr / u_q / u_val */
  const int32_t* ell_q;
  const double* ell_val;
  int32_t ell_w, pad2;
} mdp_problem;

/* y = A x, A = [K00 + w M00, w M01; w M10, K11 + w M11]
 * replaces full_operator(s) @ x (assembly.py:370-374) via krylov.spmv
 * (krylov.py:64-69).  s_work: [Qtot] scratch. */
int mdp_coupled_spmv(const mdp_problem* p, int32_t nsel, const int32_t* sel,
                     const double* x, double* y, double* s_work, void* stream);

/* y3 = C x3, C = K00 + w M00; replaces reduced_operator(s) @ x
 * (assembly.py:351-353).  x3/y3 use stride p->ld. */
int mdp_reduced_spmv(const mdp_problem* p, int32_t nsel, const int32_t* sel,
                     const double* x3, double* y3, double* s_work, void* stream);

/* Stencil part only: y3 = K00 x3 (assembly.py:122-125, Kronecker form). */
int mdp_stencil_apply(const mdp_problem* p, int32_t nsel, const int32_t* sel,
                      const double* x3, int64_t ldx, double* y3, int64_t ldy, void* stream);

/* Pi gather: s_q = W_q ( (T x3)_q - (Psi D x1)_q ); x3 or x1 may be NULL.
 * Replaces the T @ x3 product inside M00/M01 (assembly.py:324-326). */
int mdp_pi_gather(const mdp_problem* p, int32_t nsel, const int32_t* sel,
                  const double* x3, const double* x1, int64_t ld, double* s, void* stream);

/* The gather above plus, in the same launch, cdst_s[0..cn) = csrc_s[0..cn) (stride
 * ld): the block preconditioner's r0 copy ahead of its coupling term
 * (harness.py:391). */
int mdp_pi_gather_copy(const mdp_problem* p, int32_t nsel, const int32_t* sel, const double* x3,
                       const double* x1, int64_t ld, double* s, const double* csrc, double* cdst, int64_t cn,
                       void* stream);

/* Pi^T scatter (as a deterministic pull): y3[u] += alpha*w_s * (T^T s)[u].
 * Replaces T.T @ v (assembly.py:324-326). */
int mdp_pi_scatter(const mdp_problem* p, int32_t nsel, const int32_t* sel,
                   const double* s, double alpha, double* y3, int64_t ld, void* stream);

/* Weighted Jacobi sweep on C, fused: x_out = x + omega (r - C x) / diag(C),
 * replaces krylov.jacobi_smooth (krylov.py:290-299).  x may be NULL (x=0,
 * no SpMV).  tmp: [nsys*ld] scratch. */
int mdp_jacobi_sweep(const mdp_problem* p, int32_t nsel, const int32_t* sel,
                     const double* r, const double* x, double* x_out, double omega,
                     double* tmp, double* s_work, void* stream);

/* Distance of every grid node to the nearest of nseg segments
 * seg[e] = (ax, ay, az, bx, by, bz); replaces geometry.distance_field
 * (geometry.py:293-303), the CNN's second input channel. */
int mdp_distance_field(int32_t n, const double* seg, int32_t nseg, double* out, void* stream);

/* ------------------------------------------------------------------ */
/* ILU(0) of the 1D block A11 (krylov.py:188-284).                       */

/* [host] In-place ILU(0) on a sorted CSR matrix; returns -1 on success or
 * the zero-pivot row (krylov.py:188-216).  diag_pos [n] must be filled. */
int64_t mdp_ilu0_factor_host(int64_t n, const int64_t* indptr, const int64_t* indices,
                             double* data, const int64_t* diag_pos);

/* [host] Level schedule of the forward (L) and backward (U) sweeps:
 * fills perm_f/perm_b [n] and lev_f/lev_b [n+1]; returns number of levels
 * through nlev_f/nlev_b. */
int mdp_ilu0_levels_host(int64_t n, const int64_t* indptr, const int64_t* indices,
                         const int64_t* diag_pos, int32_t* perm_f, int32_t* lev_f,
                         int32_t* nlev_f, int32_t* perm_b, int32_t* lev_b, int32_t* nlev_b);

typedef struct mdp_ilu {
  int32_t nsys, lev_stride; /* level arrays are [nsys][lev_stride]       */
  const int32_t* row_start;  /* [nsys+1] global row offset                 */
  const int32_t* ptr;        /* [Rtot+1] global CSR pointers               */
  const int32_t* col;        /* local column                               */
  const double* val;         /* combined L\U factor                        */
  const int32_t* diag;       /* [Rtot] global position of the diagonal     */
  const int32_t* lev_f;      /* level boundaries (local row counts)        */
  const int32_t* perm_f;     /* [Rtot] local rows ordered by level         */
  const int32_t* lev_b;
  const int32_t* perm_b;
  const int32_t* nlev_f;     /* [nsys]                                     */
  const int32_t* nlev_b;     /* [nsys]                                     */
  int32_t max_rows, max_nnz; /* per-system maxima (shared-memory staging)  */
  const int32_t* perm;       /* optional [Rtot] symmetric permutation: the factor is
                                of P A P^T, z = P^T (LU)^-1 P r (NULL: identity) */
} mdp_ilu;

/* z1 = (LU)^-1 r1, bitwise equal to krylov.ilu0_apply (krylov.py:219-233,
 * 270-276).  r/z point at the 1D parts; stride ld.  With perm set (a
 * fill-free leaf-first order of the tree-structured A11) the same sweeps are
 * the exact solve of one_d="direct" (harness.py:356-358). */
int mdp_ilu0_apply(const mdp_ilu* f, int32_t nsel, const int32_t* sel,
                   const double* r, double* z, int64_t ld, void* stream);

/* ------------------------------------------------------------------ */
/* Krylov vector kernels (krylov.py:88-182).  V is [nsys][kmax+1][ld].   */

/* Fused Arnoldi orthogonalisation of w against V[0..nv[s]), replaces the MGS
 * loop krylov.py:138-141.  Writes hcol[s][0..kmax] = projection coefficients,
 * hcol[s][kmax+1] = ||w_final||, and V[s][nv[s]] = w_final/||w_final||
 * (vnext, also copied to vcur when non-NULL).  work: scratch of
 * mdp_arnoldi_work_bytes().
 * gram != NULL ([nsys][kmax+1][kmax+1], owned by the caller, indexed by system
 * id): modified Gram-Schmidt from one pass of dot products.  The reference's
 * sequential projections h_m = V_m.(w - sum_{c<m} h_c V_c) equal the solution
 * of the unit lower triangular system (I + L) h = V^T w with L the strictly
 * lower part of V^T V; row nv of L (the new vector against the old ones) is
 * produced by the update pass of the same step, so V is read twice per step
 * (dots; update + Gram row + norm) and the step is three launches.  A cycle
 * must run its steps nv = 1, 2, ... in order (each step writes row nv).
 * gram == NULL: CGS2 (two classical passes, three reads of V, four launches). */
size_t mdp_arnoldi_work_bytes(int32_t nsel, int32_t kmax, int64_t n);
int mdp_arnoldi(int32_t nsel, const int32_t* sel, double* V, int64_t ldv_sys, int64_t ldv_vec,
                const int32_t* nv, int32_t kmax, double* w, int64_t ldw, int64_t n,
                double* hcol, double* vcur, int64_t ldc, double* gram, void* work, void* stream);

/* out[i] = ||x_s||_2 for the selected systems (two-stage deterministic). */
int mdp_norms(int32_t nsel, const int32_t* sel, const double* x, int64_t ldx, int64_t n,
              double* out, void* work, void* stream);

/* y_s = alpha_s * x_s  (alpha_s = num[i]/den[i] when den != NULL: exact
 * division like the reference's w / h_next). */
int mdp_scale(int32_t nsel, const int32_t* sel, const double* x, int64_t ldx,
              const double* num, const double* den, double* y, int64_t ldy, int64_t n,
              void* stream);

/* x_s += sum_{k<cnt[i]} Z_s[k] * y[i][k]  (krylov.py:168-172). */
int mdp_basis_update(int32_t nsel, const int32_t* sel, double* x, int64_t ldx, const double* Z,
                     int64_t ldz_sys, int64_t ldz_vec, const int32_t* cnt, const double* y,
                     int32_t ystride, int64_t n, void* stream);

/* r = b - y and rn[i] = ||r||  (krylov.py:110-111, 173-174). */
int mdp_residual(int32_t nsel, const int32_t* sel, const double* b, const double* y, double* r,
                 int64_t ld, int64_t n, double* rn, void* work, void* stream);

/* y = a*x + b*y elementwise over n for all selected systems. */
int mdp_axpby(int32_t nsel, const int32_t* sel, double a, const double* x, double b, double* y,
              int64_t ld, int64_t n, void* stream);

/* dst[dst_off[i]] <- src (per-system gather/scatter of one vector). */
int mdp_copy_vec(int32_t nsel, const int32_t* sel, const double* src, int64_t lds,
                 double* dst, int64_t ldd, const int32_t* dst_slot, int64_t slot_stride,
                 int64_t n, void* stream);

/* Device-side Hessenberg work of the fixed-step inner FGMRES
 * (harness.py:385-387: restart = maxit = m, tol = 1e-300), the same
 * arithmetic as krylov.py:142-172.  State per selection index i:
 * H [(k+1) x k], cs, sn [k], g [k+1], flag (0 ok, 1 breakdown, 2 lucky
 * breakdown, 4 zero rhs -- flagged systems are re-solved by the host path). */
int mdp_fixed_init(int32_t nsel, int32_t k, const double* beta, double* H, double* cs, double* sn,
                   double* g, double* flag, void* stream);
/* Fused launches of the same arithmetic (fewer kernels per inner solve):
 * start  = V0 = b / beta, vcur = V0, and mdp_fixed_init;
 * arnoldi_givens = mdp_arnoldi followed by mdp_givens_step(j) in its last kernel;
 * finish = mdp_backsub(m) + x = sum_k y_k Z_k written into x (no fill / copy). */
int mdp_fixed_start(int32_t nsel, const int32_t* sel, int32_t k, const double* b, int64_t ldb,
                    const double* beta, double* v0, int64_t ldv, double* vcur, int64_t ldc, int64_t n,
                    double* H, double* cs, double* sn, double* g, double* flag, double* jac_out,
                    double omega, const double* diag, void* stream);
int mdp_arnoldi_givens(int32_t nsel, const int32_t* sel, double* V, int64_t ldv_sys, int64_t ldv_vec,
                       const int32_t* nv, int32_t kmax, double* w, int64_t ldw, int64_t n, double* hcol,
                       double* vcur, int64_t ldc, double* gram, void* work, int32_t j, double* H, double* cs, double* sn,
                       double* g, double* flag, double* jac_out, double omega, const double* diag,
                       void* stream);
/* (jac_out != NULL: also jac_out_s = (omega vcur_s) / diag_s, stride ldc -- the first
 * weighted-Jacobi sweep from zero of the next smoothed preconditioner apply) */
int mdp_fixed_finish(int32_t nsel, const int32_t* sel, int32_t k, int32_t m, const double* Z, int64_t ldz_sys,
                     int64_t ldz_vec, double* x, int64_t ldx, int64_t n, double* H, double* g, double* flag,
                     void* stream);
int mdp_givens_step(int32_t nsel, int32_t k, int32_t j, const double* hcol, double* H, double* cs,
                    double* sn, double* g, double* flag, void* stream);
int mdp_backsub(int32_t nsel, int32_t k, int32_t m, const double* H, const double* g,
                const double* flag, double* y, void* stream);
/* dst_s <- src_s[slot[i]] (gather one vector out of a per-system slot array). */
int mdp_copy_slot(int32_t nsel, const int32_t* sel, const double* src, int64_t lds, const int32_t* slot,
                  int64_t slot_stride, double* dst, int64_t ldd, int64_t n, void* stream);
/* y_s[0..n) = v */
int mdp_fill(int32_t nsel, const int32_t* sel, double* y, int64_t ld, int64_t n, double v, void* stream);

/* ------------------------------------------------------------------ */
/* Geometric multigrid baseline (krylov.py:302-387): the V-cycle pieces on
 * host-built Galerkin CSR levels (int32 ptr/col, float64 val), one system.   */

/* xo = x + (omega (r - A x)) / d; x == NULL: xo = (omega r) / d (jacobi_smooth, krylov.py:289-299) */
int mdp_csr_jacobi(int32_t n, const int32_t* ptr, const int32_t* col, const double* val, const double* d,
                   const double* r, const double* x, double* xo, double omega, void* stream);
/* res = r - A x */
int mdp_csr_residual(int32_t n, const int32_t* ptr, const int32_t* col, const double* val, const double* r,
                     const double* x, double* res, void* stream);
/* y = A x (accumulate: y += A x) -- also the restriction P^T and prolongation P */
int mdp_csr_spmv(int32_t n, const int32_t* ptr, const int32_t* col, const double* val, const double* x,
                 double* y, int32_t accumulate, void* stream);
/* y = M x, M dense n x n row-major (the inverted coarsest Galerkin matrix) */
int mdp_dense_matvec(int32_t n, const double* M, const double* x, double* y, void* stream);

/* ------------------------------------------------------------------ */
/* CNN preconditioner (neural.py:423-472, training.py:290-338).          */

typedef struct mdp_unet {
  int32_t n;        /* spatial size (points per edge)                      */
  int32_t path;     /* 0: tcgen05 TF32 implicit GEMM, 1: CUDA-core FP32 check path */
  const float* w[11];  /* packed weights, ARCHITECTURE order (path 0:
                          TF32-rounded, 3x3x3 layers with Cout <= 64 as
                          [chunk][dydx][quad][dz][Cout][4] FOLLOWED by the same pack of
                          the filter with dy and dz exchanged (the row-remainder launch
                          of odd grids reads it at offset Cin*Cout*27 floats), Cout = 128
                          as [chunk][tap][quad][Cout][4], enc1a raw [16][2][27],
                          transposed convs [tap][quad][Cout][4]; as written by
                          paper_2505_08491_b200.neural.pack_conv / pack_tconv) */
  const float* b[11];  /* biases (NULL where the layer has none)           */
  int32_t accumulate;  /* 1: z_s += scale_i * U(..) (fused z + z_net of the
                          smoothed apply, training.py:305-311); 0: z_s = ...  */
  int32_t reserved;
} mdp_unet;

size_t mdp_unet_workspace_bytes(int32_t n, int32_t nb, int32_t path);

/* z_s = scale_i * U([r_s * inv_i | d_s]) for the nb selected systems,
 * where inv_i = 1/||r_s|| (1 when zero) and scale_i = ||r_s||; rnorm [nb]
 * holds ||r_s||.  Replaces apply_neural / apply_batched's forward
 * (training.py:312-319, 331-338).  r, z: stride ld; dist: stride ldd. */
int mdp_unet_apply(const mdp_unet* net, int32_t nb, const int32_t* sel, const double* r,
                   int64_t ld, const double* rnorm, const double* dist, int64_t ldd, double* z,
                   int64_t ldz, void* workspace, size_t ws_bytes, void* stream);

/* Single-layer entry points used by the parity tests (float32 C4-blocked
 * activations [b][C/4][S][S][S][4]; w packed as in mdp_unet.w). */
int mdp_conv3_layer(int32_t path, int32_t nb, int32_t S, int32_t cin, int32_t cout,
                    const float* in, int32_t in_cq, int32_t in_q0, const float* w, const float* bias,
                    int32_t relu, float* out, int32_t out_cq, int32_t out_q0, int32_t pool,
                    void* scratch, size_t scratch_bytes, void* stream);
/* Scratch bytes mdp_conv3_layer (path 0) needs for split-K partial sums. */
size_t mdp_conv3_scratch_bytes(int32_t nb, int32_t S, int32_t cin, int32_t cout);

/* ------------------------------------------------------------------ */
const char* mdp_last_error(void);
int mdp_version(void);
/* Number of kernels this library has launched in the process. */
long long mdp_launch_count(void);
int mdp_device_sm_count(void);

#ifdef __cplusplus
}
#endif
#endif /* MDP_B200_H */
