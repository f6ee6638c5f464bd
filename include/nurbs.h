/*
 * nurbs.h — C ABI of libnurbs_b200: the data-parallel hot path of NURBS-Diff
 * (Prasad et al., arXiv 2104.14547) as hand-written sm_100a CUDA.
 *
 * Citations: "P:n" = line n of the paper text; "R<k>" = reading k of
 * DESIGN.md §3 (how a garbled or silent passage is interpreted).
 *
 * WHAT IS COMPUTED
 *   Forward (Eq.2, Eq.3, §3.1.2 steps 1-3 P:138-140, Alg.1):
 *     S(u_a, v_b) = sum_i sum_j N_i^p(u_a) N_j^q(v_b) w_ij P_ij / sum_i sum_j N_i^p(u_a) N_j^q(v_b) w_ij
 *     on the tensor grid u[0..n_u) x v[0..n_v) for each of B surfaces (R1: double-sum
 *     denominator). FindSpan with the half-open interval of P:138 (R2, R3, R4), Cox-de Boor
 *     (Eq.4) on the p+1 non-zero functions, homogeneous sum and rational
 *     divide.
 *   Backward (Eq.8, Eq.9, Eq.10, Alg.2):
 *     grad_ctrl[k][i][j] = (dL/dx, dL/dy, dL/dz, dL/dw)_ij = sum over points of
 *     grad_out . dS/dP_ij and grad_out . dS/dw_ij, i.e. J^T (dL/dS). Computed as a
 *     deterministic transposed banded reduction (no atomics; bitwise repeatable).
 *     Knot gradients are identically zero by the paper's definition (§3.2.2, R14).
 *   Curves: the same with the v-direction removed.
 *
 * LAYOUT (all fp32, C-contiguous, row-major)
 *   ctrl      [B][n][m][4]   Cartesian control points and weights (x, y, z, w), w > 0.
 *   U         [n+p+1]  (knots_batched = 0)  or [B][n+p+1]  (knots_batched = 1); same for V.
 *             Non-decreasing, U[p] < U[n]; the domain is [U[p], U[n]] (R6).
 *   u, v      [n_u], [n_v] parameter samples, non-decreasing (the meshgrid of Alg.1, R8),
 *             inside the domain. Shared by all B surfaces.
 *   out       [B][n_u][n_v][3]  u-major (R17).
 *   grad_out  [B][n_u][n_v][3]  dL/dS.
 *   grad_ctrl [B][n][m][4]  OVERWRITTEN (not accumulated).
 *   grad_U    [n+p+1] or [B][n+p+1] (nullable) — zero-filled; likewise grad_V.
 *   Curves: ctrl [B][n][4], U [n+p+1] or [B][n+p+1], u [n_u], out/grad_out [B][n_u][3];
 *           the shape must have m = 1, q = 0 (n_v is ignored).
 *
 * OWNERSHIP AND EXECUTION
 *   Every tensor pointer is a DEVICE pointer the caller allocates, owns and keeps alive
 *   until the work queued on `stream` (a cudaStream_t passed as void*, NULL = legacy default
 *   stream) has completed. Calls enqueue kernels and return immediately; they never
 *   allocate, free or synchronize, except where stated (nurbs_validate and nurbs_tables
 *   validate synchronously). Calls are stateless and reentrant across streams.
 *   Pointers should be 16-byte aligned; otherwise (or if n_v is not a multiple of 4) the
 *   kernels take a slower non-TMA path with identical results.
 *
 * ERRORS
 *   Every call returns NURBS_OK (0) or an error code; nothing is enqueued on error.
 *   Shape checks always run on the host. Data checks (knots, parameters, weights live on
 *   the device) run in nurbs_validate / nurbs_tables, and inside fwd/bwd when the
 *   environment variable NURBS_CHECK=1 (then those calls synchronize). Unchecked, invalid
 *   data (out-of-domain or unsorted samples, decreasing knots) gives wrong values but never
 *   out-of-bounds access: spans are clamped into [p, n-1] and into each tile's band, and the
 *   rolling row window only moves forward. Tables must come from nurbs_tables for the same
 *   shape (checked mode verifies their header; the Python binding checks their shape).
 *   nurbs_last_error_detail() returns a thread-local message naming the offending value.
 */
#ifndef NURBS_B200_H
#define NURBS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NURBS_MAX_DEGREE 5
#define NURBS_ABI_VERSION 1

enum {
    NURBS_OK = 0,
    NURBS_E_ARG = 1,          /* null pointer, negative size, n <= p, bad curve shape     */
    NURBS_E_UNSUPPORTED = 2,  /* degree outside 1..NURBS_MAX_DEGREE                       */
    NURBS_E_KNOTS = 3,        /* knots decreasing, or empty domain U[p] == U[n]           */
    NURBS_E_DOMAIN = 4,       /* a parameter outside [U[p], U[n]]                  */
    NURBS_E_WEIGHT = 5,       /* a weight w <= 0 (R15) or non-finite input                */
    NURBS_E_UNSORTED = 6,     /* u or v not non-decreasing                                */
    NURBS_E_CUDA = 7,         /* a CUDA runtime error (detail names it)                   */
    NURBS_E_WORKSPACE = 8,    /* workspace NULL or smaller than nurbs_*_workspace_bytes   */
    NURBS_E_TABLES = 9        /* tables given with knots_batched = 1, or (checked mode) a table
                                 header that does not match the call's shape */
};

typedef struct {
    int32_t B;              /* batch of surfaces (or curves)                              */
    int32_t n, m;           /* control-point COUNTS in u, v (curve: m = 1)   (R6)         */
    int32_t p, q;           /* degrees 1..NURBS_MAX_DEGREE (curve: q = 0)                 */
    int32_t n_u, n_v;       /* parameter samples; the grid is n_u x n_v (curve: n_v unused)*/
    int32_t knots_batched;  /* 0: U, V shared by the batch; 1: one knot vector per item   */
} nurbs_shape;

/* ---------------------------------------------------------------------------------------
 * Span/basis tables — the "pre-compute the knot spans and basis functions during the
 * initialization of the NURBS layer" of P:171 (and the stored u_span, N_i of Alg.1).
 * Valid for one (shape.n, m, p, q, n_u, n_v), one knot pair U, V (knots_batched must be 0)
 * and one sample pair u, v. `tables` is caller-allocated DEVICE memory of
 * nurbs_tables_bytes(shape) bytes, 16-byte aligned. nurbs_tables validates U, V, u, v
 * (synchronizing once) and fills the tables on `stream`. Passing tables to fwd/bwd is
 * optional (NULL = compute spans and bases in-kernel); results are identical.
 * For curves pass the curve shape (m = 1, q = 0) and V = v = NULL.
 * --------------------------------------------------------------------------------------- */
size_t nurbs_tables_bytes(const nurbs_shape* shape);
int    nurbs_tables(const nurbs_shape* shape, const float* U, const float* V,
                    const float* u, const float* v, void* tables, void* stream);

/* ---------------------------------------------------------------------------------------
 * Surfaces. nurbs_surface_fwd: Eq.3 on the grid. nurbs_surface_bwd: J^T grad_out
 * (Eq.8/9/10), grad_ctrl overwritten, grad_U/grad_V zero-filled if non-NULL.
 * The backward needs a DEVICE workspace of nurbs_surface_bwd_workspace_bytes(shape) bytes
 * (0 is possible: then workspace may be NULL) for the fixed-order cross-tile reduction.
 * --------------------------------------------------------------------------------------- */
int    nurbs_surface_fwd(const nurbs_shape* shape, const float* ctrl,
                         const float* U, const float* V, const float* u, const float* v,
                         const void* tables, float* out, void* stream);
int    nurbs_surface_bwd(const nurbs_shape* shape, const float* ctrl,
                         const float* U, const float* V, const float* u, const float* v,
                         const void* tables, const float* grad_out,
                         float* grad_ctrl, float* grad_U, float* grad_V,
                         void* workspace, size_t ws_bytes, void* stream);
size_t nurbs_surface_bwd_workspace_bytes(const nurbs_shape* shape);

/* Diagnostic: the launch plan of the backward / fitting step for `shape` (a pure function of
 * the shape, which is what makes results bitwise repeatable; the forward, which has no
 * reduction, picks its own row blocks by a wave model). Writes plan[0..5] = K (knot spans
 * of u per row block), row blocks, column blocks (128 samples of v each), control rows per
 * band, 1 if one tile per surface (no cross-tile reduction) else 0, CTAs per launch
 * (saturated at INT32_MAX). Curves (m = 1, q = 0) are planned as one row of the grid.
 * Host only; returns NURBS_E_ARG for NULL or an invalid shape. */
int    nurbs_grid_plan(const nurbs_shape* shape, int32_t plan[6]);

/* ---------------------------------------------------------------------------------------
 * Parametric derivatives (Eq.7 P:196-209 and its v analogue) and unit normals
 * (the offsetting input of §4.3) on the grid:
 *     S_u = (NR_u w - NR w_u) / w^2,  S_v likewise,  n = S_u x S_v / |S_u x S_v|.
 * out (nullable) receives S, out_u / out_v receive S_u / S_v, normals (nullable) receives n;
 * all [B][n_u][n_v][3]. Spans and bases are computed in-kernel (no tables).
 * --------------------------------------------------------------------------------------- */
int    nurbs_surface_derivs(const nurbs_shape* shape, const float* ctrl,
                            const float* U, const float* V, const float* u, const float* v,
                            float* out, float* out_u, float* out_v, float* normals, void* stream);

/* ---------------------------------------------------------------------------------------
 * Fused fitting step (the surface-fitting loop of §4.2, with Eq.14):
 * one SGD iteration of  L = mean over the n_u x n_v x B points of |S - T|^2  (R20) with
 * respect to the control points and weights, in place:
 *     S = f(ctrl) (Eq.3);  loss = L;  dL/dS = 2 (S - T) / N;  grad_ctrl = J^T dL/dS (Eq.8/9);
 *     ctrl <- ctrl - lr * grad_ctrl   (x, y, z and w; knots fixed).
 * target [B][n_u][n_v][3]; ctrl [B][n][m][4] is read and updated; grad_ctrl [B][n][m][4]
 * receives the gradient at the pre-update ctrl; loss is a DEVICE float receiving L at the
 * pre-update ctrl. S is never written to HBM (the forward and backward are one kernel).
 * Workspace: nurbs_surface_fit_workspace_bytes(shape) bytes (never 0). Deterministic.
 * --------------------------------------------------------------------------------------- */
int    nurbs_surface_fit_step(const nurbs_shape* shape, float* ctrl,
                              const float* U, const float* V, const float* u, const float* v,
                              const void* tables, const float* target, float lr,
                              float* grad_ctrl, float* loss,
                              void* workspace, size_t ws_bytes, void* stream);
size_t nurbs_surface_fit_workspace_bytes(const nurbs_shape* shape);

/* ---------------------------------------------------------------------------------------
 * True knot gradients (NEXT-4). The paper defines dL/dU = dL/dV = 0 (§3.2.2), which is
 * what nurbs_surface_bwd / nurbs_curve_bwd return. These calls return the same grad_ctrl and,
 * in grad_U / grad_V (nullable: that direction is skipped), the derivative of L with respect
 * to every knot: the A2.2 basis differentiated along the 2p knots it reads, at each
 * sample's span (spans held fixed: the derivative exists where no sample sits on a knot):
 *     dL/dU_k = sum_points g . dS/dU_k,   dS/dU_k = (dNR W - NR dW) / W^2   (Eq.7's form).
 * Shared knots (knots_batched = 0) give ONE gradient summed over the B surfaces; batched knots
 * one per surface. u / v must be non-decreasing (the grid); U, V, u, v may not be NULL even
 * with tables. Workspace: nurbs_*_bwd_knots_workspace_bytes(shape) bytes (never 0).
 * Deterministic (fixed-order sums). Curves: grad_U receives the curve's knot gradient.
 * Asynchronous on `stream`: the column-direction assembly runs on an internal per-device
 * helper stream forked from and joined back into `stream` with events (CUDA-graph capturable).
 * When the rows direction has >= 16 samples per knot span the row weights are formed as span
 * moments; the result is the same derivative up to rounding.
 * --------------------------------------------------------------------------------------- */
int    nurbs_surface_bwd_knots(const nurbs_shape* shape, const float* ctrl,
                               const float* U, const float* V, const float* u, const float* v,
                               const void* tables, const float* grad_out,
                               float* grad_ctrl, float* grad_U, float* grad_V,
                               void* workspace, size_t ws_bytes, void* stream);
size_t nurbs_surface_bwd_knots_workspace_bytes(const nurbs_shape* shape);
int    nurbs_curve_bwd_knots(const nurbs_shape* shape, const float* ctrl, const float* U,
                             const float* u, const void* tables, const float* grad_out,
                             float* grad_ctrl, float* grad_U,
                             void* workspace, size_t ws_bytes, void* stream);
size_t nurbs_curve_bwd_knots_workspace_bytes(const nurbs_shape* shape);

/* ---------------------------------------------------------------------------------------
 * Paired (scattered) parameter points (NEXT-1): point t of surface k is evaluated at its own
 * (u, v) = uv[k][t] — S(u, v) anywhere in the domain with the per-point span and
 * basis of Alg.1, the same Eq.3 sum and Eq.8/9 gradient as the grid calls.
 *   shape.n_u = N (points per surface), shape.n_v must be 1; tables are not used.
 *   uv        [B][N][2]  (u, v) pairs in any order, each inside the domain (no sorting needed).
 *   out       [B][N][3];  grad_out [B][N][3];  grad_ctrl [B][n][m][4] OVERWRITTEN;
 *   grad_U / grad_V nullable, zero-filled.
 * The backward sorts each CTA's points by knot cell in shared memory and reduces in a fixed
 * order: deterministic, no atomics. It needs (n-p)(m-q) <= 65535 knot cells and a control
 * net small enough for its shared-memory reduction (about n*m <= 1400 for p = q = 3),
 * otherwise it returns NURBS_E_UNSUPPORTED. Workspace: nurbs_surface_points_bwd_workspace_bytes.
 * nurbs_validate_points is the checked mode (knots, every (u, v) in the domain, weights);
 * it SYNCHRONIZES. NURBS_CHECK=1 runs it inside fwd/bwd.
 * --------------------------------------------------------------------------------------- */
int    nurbs_surface_points_fwd(const nurbs_shape* shape, const float* ctrl,
                                const float* U, const float* V, const float* uv,
                                float* out, void* stream);
int    nurbs_surface_points_bwd(const nurbs_shape* shape, const float* ctrl,
                                const float* U, const float* V, const float* uv,
                                const float* grad_out, float* grad_ctrl,
                                float* grad_U, float* grad_V,
                                void* workspace, size_t ws_bytes, void* stream);
size_t nurbs_surface_points_bwd_workspace_bytes(const nurbs_shape* shape);
int    nurbs_validate_points(const nurbs_shape* shape, const float* ctrl, const float* U,
                             const float* V, const float* uv, void* stream);

/* ---------------------------------------------------------------------------------------
 * Curves: shape.m = 1, shape.q = 0. Same semantics as the surface calls.
 * --------------------------------------------------------------------------------------- */
int    nurbs_curve_fwd(const nurbs_shape* shape, const float* ctrl, const float* U,
                       const float* u, const void* tables, float* out, void* stream);
int    nurbs_curve_bwd(const nurbs_shape* shape, const float* ctrl, const float* U,
                       const float* u, const void* tables, const float* grad_out,
                       float* grad_ctrl, float* grad_U,
                       void* workspace, size_t ws_bytes, void* stream);
size_t nurbs_curve_bwd_workspace_bytes(const nurbs_shape* shape);

/* ---------------------------------------------------------------------------------------
 * Multi-GPU point sharding. When one surface's parameter
 * rows are sharded over ranks, each rank's backward returns a PARTIAL gradient (the Eq.8/9
 * sums of P:215/P:222 over its own points); the full gradient is their sum. After an
 * all-gather of the partials, nurbs_sum_partials adds them in ascending part order:
 *   out[k] = ((parts[0][k] + parts[1][k]) + parts[2][k]) + ... ,  k < n
 * so the result is bitwise repeatable for a fixed number of parts (an NCCL all-reduce's
 * summation order depends on its algorithm and protocol). parts: DEVICE [n_parts][n] fp32;
 * out: DEVICE [n] fp32 (may alias parts[0]); asynchronous on `stream`. NURBS_E_ARG for
 * n_parts < 1, n < 0 or NULL pointers (n = 0 is a no-op).
 * --------------------------------------------------------------------------------------- */
int    nurbs_sum_partials(const float* parts, int32_t n_parts, int64_t n, float* out, void* stream);

/* ---------------------------------------------------------------------------------------
 * Checked mode. nurbs_validate checks every data precondition (knots non-decreasing and
 * non-empty domain, u/v sorted and inside the domain, weights > 0 and finite) on `stream`
 * and SYNCHRONIZES; returns the first error found. Curves: V = v = NULL with the curve shape.
 * --------------------------------------------------------------------------------------- */
int         nurbs_validate(const nurbs_shape* shape, const float* ctrl, const float* U,
                           const float* V, const float* u, const float* v, void* stream);
const char* nurbs_strerror(int status);

/* Path selection (process-wide; defaults from the environment variables NURBS_NO_TMA /
 * NURBS_TC at first use). NURBS_PATH_NO_TMA: stream out / dL/dS with per-thread global
 * accesses instead of TMA (results bitwise identical). NURBS_PATH_TC: run the surface backward
 * on the tcgen05 tensor cores (3xTF32) where it applies (p = q = 3, m <= 32);
 * results equal the SIMT backward's within rounding, not bitwise. Returns the previous flags.
 * Not for use while other threads launch. */
#define NURBS_PATH_NO_TMA 1
#define NURBS_PATH_TC     2
int         nurbs_set_path_flags(int flags);
const char* nurbs_last_error_detail(void);
int         nurbs_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* NURBS_B200_H */
