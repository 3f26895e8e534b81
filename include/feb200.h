/*
 * feb200.h -- C ABI of libfeb200.so: batched finite-element weak-form
 * evaluation on NVIDIA B200 (sm_100a).
 *
 * The operations are those of arXiv 2107.04121:
 *   - Alg. 2 "eval_matrix": per-cell matrices, the derivative of
 *     the form w.r.t. the DOF vector, M[c] = sum_q detw(q) dF/du;
 *   - Alg. 1 "eval_residual": per-cell residuals, the action of
 *     the form on a DOF vector, r[c] = sum_q detw(q) F;
 *   - the gather of the cell DOFs through the connectivity ("the mesh cell
 *     connectivity is used to index the DOF vector") and the
 *     scatter-add of cell residuals into the global vector (the assembly the
 *     paper leaves to SfePy);
 *   - the reference mapping: J = dx/dxi, det J, J^-1 at every quadrature
 *     point, with the quadrature weight folded into det ("The
 *     quadrature weights are incorporated in the element reference mapping
 *     Jacobian"; Tab. 4 "v.det"), and physical gradients
 *     du/dx_j = du/dxi_k J^-1_kj.
 * Arguments follow the paper's statement of the problem:
 * cells (connectivity), node coordinates, Lagrange order, quadrature,
 * material values per quadrature point and the evaluation mode.
 *
 * Conventions:
 *   - reference cell [0,1]^3, Gauss-Legendre rule with q1d points per axis;
 *   - tensor-product Lagrange basis of order p on equispaced nodes i/p;
 *   - lexicographic x-fastest numbering of element vertices (v = a+2b+4c),
 *     element nodes (k = i + (p+1)(j + (p+1) l)) and quadrature points
 *     (q = a + q1d (b + q1d c));
 *   - trilinear geometry from the 8 vertices;
 *   - element-local DOF index a*n_b + k (component-major, Eq. fe1b P:491-526,
 *     'crdse' / 'cresf' layouts P:991); global vectors node-major
 *     [n_nodes][D] (Eq. fe1c);
 *   - every array row-major with the cell axis outermost (layout 'cqgvd0',
 *     P:927-929).
 *
 * Memory: every pointer argument is a DEVICE pointer (cudaMalloc'ed or a
 * torch CUDA tensor) on the current device, unless stated otherwise.
 * Ownership: inputs are read only and never retained after the call returns;
 * fe_create_mesh_geometry copies what the handle keeps.  Outputs are
 * caller-allocated.  A handle is immutable after creation, so concurrent
 * evaluations on different streams are safe.
 * Streams: `stream` is a cudaStream_t passed as void* (NULL = legacy default
 * stream).  Evaluation calls are asynchronous on that stream.
 * Errors: every call returns an fe_status; no C++ exception or abort crosses
 * the ABI.  fe_last_error() gives a thread-local message; asynchronous kernel
 * faults surface as FE_ERR_CUDA on a later call or at stream synchronisation.
 */
#ifndef FEB200_H
#define FEB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  FE_OK = 0,
  FE_ERR_INVALID_ARG = 1, /* null pointer, negative or mismatched size, bad range */
  FE_ERR_UNSUPPORTED = 2, /* order / q1d / form / dtype / material kind not built */
  FE_ERR_DEGENERATE = 3,  /* det J <= 0 at some quadrature point; see fe_last_error_element */
  FE_ERR_CUDA = 4,        /* CUDA runtime error; message has cudaGetErrorString */
  FE_ERR_OOM = 5          /* device allocation failed */
} fe_status;

/* Weak forms (Tab. 2 of the paper; BASELINE configs). */
typedef enum {
  FE_FORM_DIFFUSION = 0,      /* int kappa grad v . grad u, scalar (weak Laplacian '0.i,0.i') */
  FE_FORM_MASS = 1,           /* int rho v u, scalar */
  FE_FORM_VECTOR_MASS = 2,    /* int rho v_i u_i, D = 3 (vector dot product 'i,i'; Eq. fe3c) */
  FE_FORM_MASS_DIFFUSION = 3, /* int rho v u + kappa grad v . grad u, scalar (BASELINE config 4) */
  FE_FORM_ELASTICITY = 4,     /* int e(v)^T D e(u), D = 3, Voigt via Psg */
  FE_FORM_CONVECTIVE = 5,     /* int v_i (du_i/dx_j) u_j, D = 3 (Eq. fe2); matrix = Eq. fe4 */
  FE_FORM_WEIGHTED_DOT = 6,   /* int v_i M_ij u_j, D = 3 ('ij,i,j'); M per qp: material a =
                               * M[E][n_q][3][3] row-major, kind FE_MAT_PER_QP; matrix orders 1-2 */
  FE_FORM_DIVERGENCE = 7      /* int dv_i/dx_i, D = 3 ('i.i'): a linear form -- residual mode
                               * (u is read but does not enter) and eval mode (int div u);
                               * no trial variable, so no matrix mode; no material (mat may be NULL) */
} fe_form;

typedef enum { FE_F64 = 0, FE_F32 = 1 } fe_dtype;

/* Material description.  Arrays have the element type of the call's dtype and
 * are indexed by the GLOBAL element index (also for element sub-ranges).
 *   DIFFUSION       PER_QP: a = kappa[E][n_q]
 *   MASS, VEC_MASS  PER_QP: a = rho[E][n_q]
 *   MASS_DIFFUSION  PER_QP: a = rho[E][n_q], b = kappa[E][n_q]
 *   ELASTICITY      PER_ELEM: a = lambda[E], b = mu[E];
 *                   PER_QP:   a = lambda[E][n_q], b = mu[E][n_q];
 *                   FULL_D:   a = D[E][n_q][6][6] (Voigt xx,yy,zz,xy,xz,yz,
 *                             engineering shears; 'cqIK' operand),
 *                             read as given by every mode (DESIGN.md reading
 *                             23).  A non-symmetric D gives a non-symmetric K.
 *                             At p = 2 matrix mode runs the pipelined kernel
 *                             (which derives K_ba = K_ab^T) and checks the
 *                             symmetry of D (to 8 ulps) on the device while
 *                             it loads D; for a non-symmetric D the general
 *                             9-block kernel then recomputes K (same stream,
 *                             no host synchronisation)
 *   CONVECTIVE      unused (kind ignored)                                  */
typedef enum { FE_MAT_PER_QP = 0, FE_MAT_PER_ELEM = 1, FE_MAT_FULL_D = 2 } fe_material_kind;

typedef struct {
  int32_t kind;  /* fe_material_kind */
  const void *a;
  const void *b;
} fe_material;

typedef struct fe_mesh fe_mesh;

typedef struct {
  int32_t order, q1d, nb, nq;
  int64_t n_vertices, n_elems, n_nodes;
  double min_det_j; /* min over cells and qps of det J (unweighted), from the create-time check */
} fe_info;

/* Create the immutable mesh handle (SYNCHRONOUS on `stream`).
 *   coords   [n_vertices][3] fp64, vertex coordinates
 *   conn     [n_elems][8] int32, vertex ids of each hexahedron (v = a+2b+4c)
 *   order    Lagrange order p of the field (1..4 on the GPU)
 *   q1d      Gauss points per axis (must be p+1 on the GPU)
 *   n_nodes  number of global field nodes (order-p lattice nodes)
 *   dof_conn [n_elems][(p+1)^3] int32 global node of each element node, or
 *            NULL when order == 1 (then dof_conn = conn and n_nodes = n_vertices)
 * Copies coords / conn / dof_conn into library-owned device memory, builds the
 * reference tables (Gauss-Legendre, Lagrange values and derivatives), and
 * checks det J > 0 at every (cell, qp): FE_ERR_DEGENERATE otherwise, with the
 * first offending cell in fe_last_error_element() (SPEC "degenerate-cell
 * error naming the cell").  Connectivity entries out of range give
 * FE_ERR_INVALID_ARG.  *out is set only on FE_OK. */
fe_status fe_create_mesh_geometry(int64_t n_vertices, const double *coords, int64_t n_elems,
                                  const int32_t *conn, int32_t order, int32_t q1d,
                                  int64_t n_nodes, const int32_t *dof_conn, void *stream,
                                  fe_mesh **out);

/* Release the handle and its device memory, stream-ordered: the memory is returned
 * (cudaFreeAsync) after the work already queued on `stream`; the device is NOT
 * synchronised.  Work on other streams that uses the handle must be ordered
 * before this call by the caller (events), as for any stream-ordered free.
 * NULL is a no-op. */
fe_status fe_destroy_mesh(fe_mesh *mesh, void *stream);

/* Sizes of the handle (host struct). */
fe_status fe_mesh_info(const fe_mesh *mesh, fe_info *info);

/* Element matrices, Alg. 2, of cells [elem_begin, elem_end):
 *   K[e - elem_begin][ndof][ndof], ndof = D n_b, row = test (a, k), column =
 *   trial (b, l), local index a*n_b + k.  K is overwritten.
 *   state_u: CONVECTIVE only, the linearisation state [n_nodes][3]; the
 *   matrix is the Newton tangent of Eq. fe4 (both terms).  NULL otherwise.
 * FE_F64: orders scalar forms 1-4, vector forms
 * (VECTOR_MASS, ELASTICITY, CONVECTIVE, WEIGHTED_DOT) 1-3 (order 3 through the
 * dense tensor-core kernel); other combinations FE_ERR_UNSUPPORTED.  DIVERGENCE has no matrix
 * mode (FE_ERR_UNSUPPORTED).  FE_F32 (DIFFUSION, MASS, MASS_DIFFUSION at order 1, 2; default
 * matrix implementation): fp32 coefficient arrays and fp32 K, the contraction in fp64 and K
 * rounded once (within 1e-5 of the fp64 oracle, reading 15). */
fe_status fe_eval_element_matrices(const fe_mesh *mesh, int32_t form, int32_t dtype,
                                   const fe_material *mat, const void *state_u,
                                   int64_t elem_begin, int64_t elem_end, void *K, void *stream);

/* Residuals, Alg. 1, of cells [elem_begin, elem_end) for the
 * global DOF vector u [n_nodes][D]:
 *   r_elem  (nullable) [elem_end - elem_begin][ndof], overwritten;
 *   r_global(nullable) [n_nodes][D], ACCUMULATED (+=): the caller zeroes it.
 * The scatter-add into r_global is fused into the kernel (fp atomics; the
 * atomic order is the only run-to-run difference).  For the CONVECTIVE form
 * the residual is c(v, u, u) with the same u.  FE_F32 is built for
 * DIFFUSION, MASS and MASS_DIFFUSION (fp32 data, geometry from fp64
 * coordinates). */
fe_status fe_eval_residual(const fe_mesh *mesh, int32_t form, int32_t dtype,
                           const fe_material *mat, const void *u, int64_t elem_begin,
                           int64_t elem_end, void *r_elem, void *r_global, void *stream);

/* ---- Fused residual + interface-plane exchange over peer memory ----
 * Residual mode (FE_F64, the sum-factorised kernels) whose fused scatter also adds
 * the contribution to every node n in a window's [node_begin, node_end) at
 * dst[(n - node_begin + dst_node_offset) * D + a] with system-scope fp64 atomics.
 * dst is any device pointer valid in the caller's context -- typically the
 * neighbouring rank's residual vector opened with fe_ipc_open (NVLink peer
 * memory), so the z-slab interface planes are summed inside the residual
 * kernel with no separate collective.  The caller orders the ranks: every
 * rank's r_global is zeroed before any rank's kernel starts, and no rank reads
 * its vector before every rank's kernel has finished (a device-side barrier).
 * 0..2 windows; FE_ERR_UNSUPPORTED with FE_OPT_RESIDUAL_IMPL = 2 (dense). */
typedef struct {
  int64_t node_begin, node_end;   /* local node range of the window */
  double *dst;                    /* device (or peer-mapped) vector [..][D] */
  int64_t dst_node_offset;        /* node index in dst of node_begin */
} fe_peer_window;
fe_status fe_eval_residual_peer(const fe_mesh *mesh, int32_t form, const fe_material *mat,
                                const double *u, int64_t elem_begin, int64_t elem_end,
                                double *r_elem, double *r_global, const fe_peer_window *windows,
                                int32_t n_windows, void *stream);

/* CUDA IPC helpers for the peer windows: fe_ipc_alloc allocates `bytes` of
 * device memory on the current device (cudaMalloc) and returns its 64-byte IPC
 * handle; fe_ipc_open maps another process's handle into this process (peer
 * access enabled lazily; the same device or an NVLink peer); fe_ipc_close /
 * fe_ipc_free release them. */
fe_status fe_ipc_alloc(int64_t bytes, void **dev_ptr, unsigned char handle[64]);
fe_status fe_ipc_free(void *dev_ptr);
fe_status fe_ipc_open(const unsigned char handle[64], void **dev_ptr);
fe_status fe_ipc_close(void *dev_ptr);

/* Matrix mode and residual mode of a LINEAR scalar form (DIFFUSION, MASS,
 * MASS_DIFFUSION; order 1 or 2) in ONE pass: the element matrices K as in
 * fe_eval_element_matrices, and from the same K_e the residual r_e = K_e u_e
 * (Alg. 1 for a bilinear form, which is exactly K_e u_e up to rounding; oracle
 * pin P8) with the fused scatter-add of fe_eval_residual (r_elem nullable and
 * overwritten, r_global nullable and ACCUMULATED).  For a Newton-type step that
 * needs both, this avoids the second geometry / contraction pass.  FE_F64 only;
 * FE_ERR_UNSUPPORTED for other forms / orders. */
fe_status fe_eval_matrix_residual(const fe_mesh *mesh, int32_t form, int32_t dtype,
                                  const fe_material *mat, const void *u, int64_t elem_begin,
                                  int64_t elem_end, void *K, void *r_elem, void *r_global,
                                  void *stream);

/* 'eval' mode ("the integral value in case all variables passed to
 * the evaluation function have associated DOFs"): the form with the test
 * function replaced by the field u itself, over cells [elem_begin, elem_end):
 *   value += sum_e int_e F(u, u)  (= sum_e u_e . r_e(u): u^T K u for the
 *   bilinear forms, c(u, u, u) for the convective form).
 * `value` is ONE device double, ACCUMULATED (+=; the caller zeroes it); fp
 * atomics make the summation order (and the last bits) run-dependent.
 * u has the element type of dtype; the sum is accumulated in fp64. */
fe_status fe_eval_scalar(const fe_mesh *mesh, int32_t form, int32_t dtype, const fe_material *mat,
                         const void *u, int64_t elem_begin, int64_t elem_end, double *value,
                         void *stream);

/* Cauchy stress at the quadrature points (Tab. 2 'IK,s(k:l)->K'), an
 * "evaluated only" form (no test variable):
 *   sigma[e - elem_begin][q][I] = sum_K D_IK(e, q) eps_K(u)(q),  I, K in Voigt order
 *   (xx, yy, zz, xy, xz, yz), eps with engineering shears (du0/dx1 + du1/dx0, ...).
 * u: device double [n_nodes][3] (interleaved components, as in residual mode);
 * mat: the elasticity material (FE_MAT_PER_QP / FE_MAT_PER_ELEM lambda, mu, or
 * FE_MAT_FULL_D); sigma: device double [elem_end - elem_begin][n_q][6], caller
 * owned, overwritten.  FE_F64 only; orders 1..4 (the mesh's q1d = order + 1).
 * Deterministic (no atomics). */
fe_status fe_eval_stress(const fe_mesh *mesh, const fe_material *mat, const double *u,
                         int64_t elem_begin, int64_t elem_end, double *sigma, void *stream);

/* The Cauchy stress in the paper's 'eval' mode, "returning the integral value":
 * per cell, sigma_int[e - elem_begin][I] = int_e sigma_I dx = sum_q w_q det J_q sigma[e][q][I]
 * (the domain integral is the sum over cells).  Arguments as fe_eval_stress; sigma_int
 * [elem_end - elem_begin][6] fp64, caller owned, overwritten.  Deterministic (fixed qp order,
 * no atomics). */
fe_status fe_eval_stress_integral(const fe_mesh *mesh, const fe_material *mat, const double *u,
                                  int64_t elem_begin, int64_t elem_end, double *sigma_int,
                                  void *stream);

/* ---- Element-kind grouping ---------------------------
 * One evaluation call covers cells of one kind (order); a p-/hp-mixed mesh is
 * evaluated group by group.  fe_group_cells is a stable GPU sort of the cell
 * ids by kind: perm (device int64 [n_cells], caller owned) lists the cells of
 * kind 0 in ascending id order, then kind 1, ...; offsets (HOST int64
 * [n_kinds + 1]) gives group g = perm[offsets[g] .. offsets[g+1]).  kind:
 * device int32 [n_cells], values in [0, n_kinds) else FE_ERR_INVALID_ARG.
 * Synchronises `stream` (offsets are returned on the host). */
fe_status fe_group_cells(const int32_t *kind, int64_t n_cells, int32_t n_kinds, int64_t *perm,
                         int64_t *offsets, void *stream);

/* Gather rows in grouped order: out[i][j] = in[row_ptr[perm[i]] + j] for
 * i < n, j < width (row_ptr NULL: fixed stride, in[perm[i] * width + j]).
 * All pointers device; out caller owned [n][width].  Used for the per-group
 * conn / dof_conn / material blocks of a mixed mesh (ragged per-cell arrays
 * are addressed through row_ptr). */
fe_status fe_gather_rows_i32(const int32_t *in, const int64_t *row_ptr, int32_t width,
                             const int64_t *perm, int64_t n, int32_t *out, void *stream);
fe_status fe_gather_rows_f64(const double *in, const int64_t *row_ptr, int32_t width,
                             const int64_t *perm, int64_t n, double *out, void *stream);

/* ---- Mixed velocity-pressure forms (Tab. 2) ----------------------
 * The mesh handle is the velocity space Q_pv (vector, D = 3, its dof_conn and
 * n_nodes); an fe_field is a scalar pressure space Q_pp on the same cells,
 * 1 <= pp <= pv, evaluated at the mesh's quadrature points (one rule for both,
 * DESIGN.md reading 19).  Element-local velocity DOFs are component-major
 * a * n_bv + k (reading 9); pressure DOFs are l = 0..n_bp-1 (lexicographic).
 *   Stokes coupling            ('i.i,0', v, p): int (dv_i/dx_i) p
 *   transposed Stokes coupling ('i.i,0', u, q): int q (du_i/dx_i)           */
typedef struct fe_field fe_field;

/* Create the pressure space: order pp (1..mesh order), n_nodes pressure nodes,
 * dof_conn [n_elems][(pp+1)^3] int32 (host or device; copied, range-checked
 * against n_nodes -> FE_ERR_INVALID_ARG).  The field keeps a pointer to `mesh`,
 * which must outlive it.  Pairs built: (pv, pp) in (1,1) (2,1) (2,2) (3,2)
 * (3,3) (4,3) (4,4); others FE_ERR_UNSUPPORTED. */
fe_status fe_create_field(const fe_mesh *mesh, int32_t order, int64_t n_nodes,
                          const int32_t *dof_conn, void *stream, fe_field **out);
/* Stream-ordered release, as fe_destroy_mesh. */
fe_status fe_destroy_field(fe_field *field, void *stream);

/* Matrix mode of the coupling over cells [elem_begin, elem_end):
 *   transposed = 0: B[e'][a*n_bv + k][l] = int dphi_k/dx_a psi_l   (test v, trial p)
 *   transposed = 1: C[e'][l][a*n_bv + k] = the same entries         (test q, trial u)
 * out: device double, caller owned, overwritten. */
fe_status fe_eval_coupling_matrices(const fe_mesh *mesh, const fe_field *pressure,
                                    int32_t transposed, int64_t elem_begin, int64_t elem_end,
                                    double *out, void *stream);

/* Residual mode:
 *   transposed = 0: input x = pressure p [n_p];        r_elem [E'][3 n_bv],
 *                   r_v = int dphi_k/dx_a p_h, r_global velocity-shaped [n_v][3]
 *   transposed = 1: input x = velocity u [n_v][3];     r_elem [E'][n_bp],
 *                   r_q = int psi_l div u_h,  r_global pressure-shaped [n_p]
 * r_elem nullable (overwritten), r_global nullable (ACCUMULATED, fp atomics). */
fe_status fe_eval_coupling_residual(const fe_mesh *mesh, const fe_field *pressure,
                                    int32_t transposed, const double *x, int64_t elem_begin,
                                    int64_t elem_end, double *r_elem, double *r_global,
                                    void *stream);

/* 'eval' mode: value += int p_h div u_h over the cells (one device
 * double, ACCUMULATED; the caller zeroes it). */
fe_status fe_eval_coupling_scalar(const fe_mesh *mesh, const fe_field *pressure, const double *u,
                                  const double *p, int64_t elem_begin, int64_t elem_end,
                                  double *value, void *stream);

/* Scatter-add of cell residuals (standalone assembly):
 *   r_global[dof_conn[e][k] * ncomp + a] += r_elem[e - elem_begin][a * n_b + k]
 * for e in [elem_begin, elem_end).  ncomp in {1, 3}. */
fe_status fe_assemble_vector(const fe_mesh *mesh, int32_t dtype, int32_t ncomp,
                             int64_t elem_begin, int64_t elem_end, const void *r_elem,
                             void *r_global, void *stream);

/* ---- Global sparse matrix (CSR) assembly (the assembly the paper
 * leaves to SfePy).  A CSR object holds the sparsity pattern of the
 * global matrix for `ncomp` components per node with the interleaved numbering
 * dof = node * ncomp + a (Eq. fe1c); rows are sorted by column.  It keeps a
 * pointer to `mesh`, which must outlive it. */
typedef struct fe_csr fe_csr;

/* Build the pattern on the GPU (SYNCHRONOUS on `stream`): node pairs of every
 * cell, sort + unique, row pointers, and a cell-to-position map for assembly.
 * ncomp in {1, 3}.  Memory: ~12 B per (cell, node, node) pair during setup. */
fe_status fe_create_csr(const fe_mesh *mesh, int32_t ncomp, void *stream, fe_csr **out);

/* n_rows = n_nodes * ncomp; nnz = number of stored entries. Either pointer may be NULL. */
fe_status fe_csr_info(const fe_csr *csr, int64_t *n_rows, int64_t *nnz);

/* Device arrays owned by the CSR object: row_ptr[n_rows + 1] (int64), col_idx[nnz] (int32). */
fe_status fe_csr_arrays(const fe_csr *csr, const int64_t **row_ptr, const int32_t **col_idx);

/* Copy the pattern into caller buffers (device or host) on `stream` (asynchronous). */
fe_status fe_csr_copy_arrays(const fe_csr *csr, int64_t *row_ptr, int32_t *col_idx, void *stream);

/* values[nnz] (fp64, device) += the element matrices K[e - elem_begin][ndof][ndof] of
 * cells [elem_begin, elem_end) (the layout fe_eval_element_matrices writes), with
 * fp atomics: the caller zeroes `values`; summation order is run-dependent.  With the
 * environment variable FEB200_CSR_IMPL=gather (p <= 2) a row-owner kernel without atomics
 * is used instead: each node row sums its incident cells in ascending cell order, so the
 * result is bitwise reproducible (slower on B200: 1.9 vs 1.1 ms for C2).  (The variable is read
 * at library load only; fe_set_option(FE_OPT_CSR_IMPL, 1) selects it at run time.) */
fe_status fe_assemble_matrix(const fe_csr *csr, const double *K, int64_t elem_begin,
                             int64_t elem_end, double *values, void *stream);

/* Release the CSR object, stream-ordered as fe_destroy_mesh.  NULL is a no-op. */
fe_status fe_destroy_csr(fe_csr *csr, void *stream);

/* Test mode: materialise the geometry of step a1 (fp64):
 *   detw[E][n_q] = w_q det J,  jinv[E][n_q][3][3] = J^-1 (row-major).
 * Either pointer may be NULL. */
fe_status fe_geometry(const fe_mesh *mesh, double *detw, double *jinv, void *stream);

/* Thread-local message of the last failing call ("" if none). */
const char *fe_last_error(void);

/* Cell index attached to the last FE_ERR_DEGENERATE (-1 if none). */
int64_t fe_last_error_element(void);

/* Number of kernels this library launched since load (all threads). */
int64_t fe_launch_count(void);

/* ---- Process-wide implementation options ------------------------------------
 * Alternative kernels kept as measured baselines and test hooks.  Defaults are
 * read ONCE, when the library is loaded, from the environment variables named
 * below (FE_OPT_* = 0 when unset); afterwards only fe_set_option changes them
 * (no per-launch getenv).  Values are relaxed atomics: set them while no
 * evaluation is in flight on another thread.  Out-of-range values give
 * FE_ERR_INVALID_ARG.
 *   FE_OPT_MATRIX_IMPL   (FEB200_MATRIX_IMPL = sf1 | dense)  0 default (sum-factorised,
 *                        warp-specialised pipelines where built), 1 single-stage
 *                        sum-factorised kernels, 2 dense DMMA kernels
 *   FE_OPT_RESIDUAL_IMPL (FEB200_RESIDUAL_IMPL = sf | dense) 0 default (register-resident
 *                        kernels at p = 2, sum-factorised otherwise), 1 shared-memory
 *                        sum-factorised kernels for every form, 2 dense DMMA kernels
 *   FE_OPT_CSR_IMPL      (FEB200_CSR_IMPL = gather)          0 fp64 atomics, 1 atomic-free
 *                        row-owner gather (bitwise reproducible, p <= 2)
 *   FE_OPT_MAX_CTAS      (FEB200_MAX_CTAS = n)               0 no cap, else the grid cap of
 *                        the persistent kernels (test hook: many batches per CTA) */
typedef enum {
  FE_OPT_MATRIX_IMPL = 0,
  FE_OPT_RESIDUAL_IMPL = 1,
  FE_OPT_CSR_IMPL = 2,
  FE_OPT_MAX_CTAS = 3,
  FE_OPT_COUNT = 4
} fe_option;
fe_status fe_set_option(int32_t option, int64_t value);
fe_status fe_get_option(int32_t option, int64_t *value);

#ifdef __cplusplus
}
#endif

#endif /* FEB200_H */
