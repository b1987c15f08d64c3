/*
 * srwcr.h -- C ABI of the B200-native SRWCR hot path (arXiv 1804.05061).
 *
 * The library evaluates, once per quasi-Newton iteration, the spatially
 * region-weighted correlation ratio D (Eq 9; Table I) between a
 * fixed image F (the model image A) and the moving image M warped by a cubic
 * B-spline free-form deformation T(x; Phi) (Eq 17) used as the
 * estimated image B = M(T(x)) ("moving-as-B"), together with its analytic
 * gradient dD/dPhi (Eq 15-17 P:180-190 with Eq 27).  It minimises
 * C = D + w_p C_p (Eq 1) via srwcr_register.
 *
 * "P:NNN" cites line NNN of the paper text; readings where the paper is silent or
 * garbled are numbered c1..c18 in DESIGN.md s3.
 *
 * Conventions shared by every entry point
 *   - Volumes: fp32, x-fastest, [Nz][Ny][Nx]; Nz == 1 means 2-D (reading c16).
 *   - Intensities are normalised to [0, L] with L = intensity_bins - 1
 *     unless srwcr_options.inputs_normalized == 1 (reading c1 gives the formula).
 *   - Control lattice: spacing delta = control_spacing_mm / spacing_mm voxels per
 *     axis (fp64), G = floor((N-1)/delta) + 4 nodes per axis, node j at voxel
 *     coordinate (j-1)*delta (Eq 17 indices shifted by +1, reading c15).  In 2-D
 *     the z axis has G = 1 and no displacement component.
 *   - Spatial bins (regions, Eq 7): spatial_bins[i] = k cells per axis,
 *     Delta = N/k, K = k+3 regions per axis (reading c14); k = 0 (or the z axis in
 *     2-D) is a degenerate axis with K = 4, weights (1,0,0,0): one real region.
 *   - Params / gradient: fp64 SoA [ndim][Gz][Gy][Gx], displacements in voxels,
 *     0 = identity.  ndim = 3 (2 in 2-D).
 *   - Pointers marked "host or device" are classified with
 *     cudaPointerGetAttributes; device pointers are the fast path.
 *   - Every call returns a status and never throws.  srwcr_last_error() gives the
 *     message of the last failing call on that context.  After SRWCR_ECUDA the
 *     context is poisoned and every later call returns SRWCR_ESTATE.
 *   - Thread-compatible: one caller at a time per context; distinct contexts are
 *     independent.
 */
#ifndef SRWCR_H
#define SRWCR_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct srwcr_ctx srwcr_ctx; /* opaque; owns all its device memory */

typedef enum {
    SRWCR_OK = 0,
    SRWCR_EINVAL = -1,      /* bad argument; the message names it */
    SRWCR_ENOMEM = -2,      /* host or device allocation failed */
    SRWCR_ECUDA = -3,       /* CUDA runtime error (context poisoned) */
    SRWCR_ENCCL = -4,       /* NCCL error or NCCL library not loadable */
    SRWCR_EDEGENERATE = -5, /* no region passed the retention test (reading c12) */
    SRWCR_ENOTSUP = -6,     /* option not supported by this build */
    SRWCR_ESTATE = -7,      /* context poisoned by an earlier CUDA error, or call out of order */
    SRWCR_ENONFINITE = -8   /* srwcr_register: cost or gradient not finite */
} srwcr_status;

typedef struct {
    int32_t struct_size;       /* = sizeof(srwcr_options); set by srwcr_default_options */
    int32_t orientation;       /* 0 = moving image is the estimated image B (Eq 18-19/27).
                                  1 = moving image is the model image A (Eq 20-21, App. II Eq 31;
                                  readings c4, c23); above ~64 bins its per-item slot
                                  tables need fewer warps per CTA (slower); other values
                                  SRWCR_EINVAL */
    int32_t inputs_normalized; /* 1: fixed/moving already in [0, L]; 0: min-max normalise */
    int32_t device;            /* CUDA device ordinal */
    int32_t nranks, rank;      /* z-slab decomposition: rank r owns slab srwcr_plan_slab(r) */
    const void *nccl_id;       /* 128-byte ncclUniqueId (broadcast by the caller): the library
                                  all-reduces over NCCL (any nranks >= 1); NULL with nranks > 1:
                                  caller-driven exchange (srwcr_eval_begin/end) */
    double eps_mass;           /* region retained iff p(r) > eps_mass ... (reading c12) */
    double eps_sigma;          /* ... and sigma_r^2 > eps_sigma (bin^2)                  */
    int32_t moment_shift;      /* 1 (default): per-fixed-bin shift of the accumulated moments
                                  estimated at Phi = 0; 0: shift = bin index.  Exact algebra
                                  either way; it only conditions the fp32 partial sums. */
    int32_t use_graph;         /* 1 (default): srwcr_eval with device params (and device or NULL
                                  grad) on one rank replays a CUDA graph of the
                                  evaluation captured on first use for that pointer pair
                                  (re-captured when a pointer changes); 0: ordinary launches */
    int32_t grad_exchange;     /* z-slabs over NCCL (nccl_id set): 0 (default):
                                  all-reduce of the int64 gradient, every rank gets the full
                                  gradient; 1: halo exchange -- rank k sends its partial on the
                                  node layers rank k+1 owns (ncclSend/Recv, 3 layers per
                                  component when slabs follow control cells) and gets the
                                  gradient on ITS OWNED layers only, zero elsewhere
                                  (srwcr_grad_layers; the rank gradients sum / concatenate to
                                  the full one, bitwise the all-reduce's on the owned layers):
                                  for a caller-side optimizer sharded by layers.  3-D fast-path
                                  configurations only (SRWCR_ENOTSUP otherwise), slabs at least
                                  as thick as the 4 taps (SRWCR_EINVAL); srwcr_register
                                  refuses it (its L-BFGS is replicated) */
} srwcr_options;

/* Fills *opt with defaults: orientation 0, inputs_normalized 0, device 0, nranks 1,
 * rank 0, nccl_id NULL, eps_mass 1e-12, eps_sigma 1e-6, moment_shift 1, use_graph 1, grad_exchange 0. */
srwcr_status srwcr_default_options(srwcr_options *opt);

/* Create a context: copies F and M (host or device; the caller may free them on
 * return), normalises them, builds the per-axis B-spline tables (Eq 8, Eq 17),
 * accumulates the static fixed-image counts N[r][a] = sum_x w_r(x) h(a - F(x))
 * (Eq 3; they do not depend on Phi) and estimates the per-bin moment shifts
 * with one identity pass.  (An evaluation is 6 kernels on the context's stream,
 * replayed as one CUDA graph when options.use_graph applies.)
 *   dims[3]            Nx, Ny, Nz (Nz = 1: 2-D); each >= 1, Nx, Ny >= 2, Nx Ny Nz < 2^31
 *   spacing_mm[3]      voxel spacing (> 0)
 *   intensity_bins     L + 1, in [2, 128] (paper: L = 31), both orientations
 *   spatial_bins[3]    k cells per axis (>= 0; 0 = one region on that axis)
 *   control_spacing_mm[3]  control-node spacing (> 0); paper: delta = [5,5,5]
 *   opt                NULL = defaults
 * Returns SRWCR_EINVAL on bad geometry, SRWCR_EDEGENERATE if no region can be
 * retained even at Phi = 0 is NOT an error here (it is reported by srwcr_eval). */
srwcr_status srwcr_create(srwcr_ctx **out, const float *fixed, const float *moving,
                          const int64_t dims[3], const double spacing_mm[3], int32_t intensity_bins,
                          const int32_t spatial_bins[3], const double control_spacing_mm[3],
                          const srwcr_options *opt);

/* Number of parameters n = ndim * Gx * Gy * Gz and the control grid (Gx, Gy, Gz). */
srwcr_status srwcr_num_params(const srwcr_ctx *ctx, int64_t *n, int64_t grid_dims[3]);

/* One SRWCR evaluation at params (host or device, fp64, layout above):
 *   *value = D (Eq 9) on return (host pointer);
 *   grad   = dD/dPhi (host or device, fp64, same layout as params), or NULL for the
 *            value only.  With nranks > 1 every rank passes the same params and gets
 *            the same D and the full gradient (grad_exchange = 1: the gradient on its
 *            owned node layers, zero elsewhere).
 * Returns SRWCR_EDEGENERATE (value = 0, grad = 0) if no region is retained. */
srwcr_status srwcr_eval(srwcr_ctx *ctx, const double *params, double *value, double *grad);

/* Caller-driven exchange (nranks > 1 and nccl_id == NULL), the same kernels as
 * srwcr_eval split at the two exchange points of the z-slab decomposition:
 *   srwcr_eval_begin  uploads params and runs pass 1 on this rank's slab; the
 *                     rank-partial statistics are then in the buffer given by
 *                     srwcr_stats_buffer (device, fp64, `count` values) which the
 *                     caller must sum over ranks in place (e.g. an all-reduce);
 *   srwcr_eval_end    combines and runs pass 2 on this rank's slab; grad receives
 *                     this rank's PARTIAL gradient, which the caller sums over ranks.
 *                     It first waits for all work on the device (cudaDeviceSynchronize), so
 *                     the caller's writes of the summed statistics on any stream -- or a
 *                     pageable cudaMemcpy, whose DMA may still be in flight when it returns --
 *                     have landed. */
srwcr_status srwcr_eval_begin(srwcr_ctx *ctx, const double *params);
srwcr_status srwcr_stats_buffer(srwcr_ctx *ctx, double **dev_ptr, size_t *count);
srwcr_status srwcr_eval_end(srwcr_ctx *ctx, double *value, double *grad);

/* z-slab of rank `rank` out of `nranks` for a volume of nz slices: [*z0, *z1).
 * Host-only (no GPU needed).  Slabs split the slices as evenly as possible. */
srwcr_status srwcr_plan_slab(int64_t nz, int32_t nranks, int32_t rank, int64_t *z0, int64_t *z1);

/* Node-layer plan of the z-slab gradient (the halo exchange; Eq 17: voxel
 * slice z feeds control layers cbz[z] .. cbz[z] + 3).  Host-only (no GPU needed).
 *   nz, nranks, rank  as srwcr_plan_slab (nz >= nranks)
 *   cbz[nz]           tap base of every slice on the control lattice, non-decreasing,
 *                     in [0, gz) (srwcr_debug_dump SRWCR_DUMP_CTRL_TAPS, z part)
 *   gz                control layers Gz
 *   out[5]            t0, t1: layers [t0, t1) the rank's slab touches (its gradient
 *                     partial is zero outside them); o0, o1: layers [o0, o1) the rank owns
 *                     (o0 = t0, 0 for rank 0; o1 = t0 of rank + 1, gz for the last rank);
 *                     r1: rank - 1's partial is non-zero on the owned layers [o0, r1)
 *                     (r1 = o0 for rank 0).  The rank sends [o1, t1) to rank + 1.
 * SRWCR_EINVAL on bad arguments or when some rank's touched layers reach past its upper
 * neighbour's owned range (slabs thinner than the taps: use fewer ranks). */
srwcr_status srwcr_plan_layers(int64_t nz, int32_t nranks, int32_t rank, const int32_t *cbz, int64_t gz,
                               int64_t out[5]);
/* srwcr_plan_layers of the context's own rank (3-D; SRWCR_ENOTSUP for 2-D or an invalid plan). */
srwcr_status srwcr_grad_layers(const srwcr_ctx *ctx, int64_t out[5]);

/* Bending energy C_p of the FFD (the constraint of Eq 1; Rueckert et
 * al. [26]; reading c19 of DESIGN.md):
 *   C_p = (1/V) sum_voxels sum_c [u_c,xx^2 + u_c,yy^2 + u_c,zz^2
 *                                 + 2u_c,xy^2 + 2u_c,xz^2 + 2u_c,yz^2]
 * V = Nx*Ny*Nz, derivatives in voxel coordinates (u in voxels), x,y terms only in
 * 2-D.  Evaluated on the device as phi . H phi / V with H the separable sum of
 * 1-D B-spline derivative Gram matrices (banded, 7 diagonals).
 *   params  fp64 [ndim][Gz][Gy][Gx], host or device pointer (read only)
 *   value   out: C_p (host pointer, required)
 *   grad    out (nullable): dC_p/dphi, host or device, same layout (overwritten)
 * Deterministic (no atomics).  Errors: EINVAL (NULL ctx/params/value), ECUDA. */
srwcr_status srwcr_bending(srwcr_ctx *ctx, const double *params, double *value, double *grad);

/* L-BFGS registration of C = D + w_p * C_p (Eq 1).  params_inout is a
 * host fp64 array (layout above): the start point on entry, the result on return
 * (the last accepted iterate, also on a line-search failure).
 * cfg may be NULL for defaults (srwcr_default_lbfgs_config); report may be NULL;
 * when given, each must carry struct_size = sizeof(its type) (EINVAL otherwise).
 * Algorithm (reading c20): two-loop recursion with m corrections, initial step
 * 1/||g|| then 1 with the y.s/y.y initial-Hessian scaling; backtracking line search
 * (x0.5 on an Armijo failure with constant ftol, x2.1 on a curvature failure with
 * constant wolfe -- the regular Wolfe condition); each trial first runs the value
 * only (pass 1 + combine) and computes the gradient (pass 2) only once the Armijo
 * test passes; pairs with y.s <= 0 are not stored.  Stops when (a) ||g|| <=
 * epsilon * max(1, ||phi||), (b) the spread (max - min) of C over the last
 * stable_window accepted iterates is < stable_tol * max(|C|, 1e-12) ("stable within
 * the last 20 steps"), (c) max_iter iterations, (d) the line search fails.
 * With nranks > 1 every rank runs the same replicated loop (all reductions are
 * deterministic, so the iterates stay identical across ranks).
 * Errors: EINVAL, ESTATE (caller-driven exchange mode), EDEGENERATE, ECUDA, and
 * SRWCR_ENONFINITE when C or the gradient is not finite. */
typedef struct {
    int32_t struct_size;
    int32_t m;                 /* number of corrections (paper: 5) */
    int32_t max_iter;          /* paper: 200/200/120 per resolution level */
    int32_t max_linesearch;    /* trials per iteration (default 20) */
    double w_p;                /* penalty weight (paper: 0.1 mono-modal, 30 multi-modal) */
    double ftol, wolfe;        /* Armijo and curvature constants (defaults 1e-4, 0.9) */
    int32_t stable_window;     /* stop when C is stable over this many iterates (paper: 20) */
    int32_t verbose;           /* 1: one line per iteration on stderr */
    double stable_tol;         /* default 1e-5 */
    double epsilon;            /* gradient-norm test (default 0 = off; P:226 names only
                                  the stability and iteration rules) */
} srwcr_lbfgs_config;

typedef struct {
    int32_t struct_size;
    int32_t iterations, evaluations, status; /* status: 0 converged (gradient test), 1 stable
                                                (C stable over the window), 2 max_iter,
                                                3 line search failed */
    int32_t gradient_evaluations;
    double initial_cost, final_cost;         /* C = D + w_p C_p */
    double final_value, final_penalty;       /* D and C_p at the result */
    double grad_norm;                        /* ||dC/dphi|| at the result */
} srwcr_register_report;

srwcr_status srwcr_default_lbfgs_config(srwcr_lbfgs_config *cfg);
srwcr_status srwcr_register(srwcr_ctx *ctx, double *params_inout, const srwcr_lbfgs_config *cfg,
                            srwcr_register_report *report);

/* ---- multi-resolution registration utilities (backward
 * warping, "the multi-resolution strategy and the concatenation of three isotropic control
 * grids").  Not on the SRWCR hot path.  Fields are fp32 [3][Nz][Ny][Nx] (component x, y,
 * z; displacements in voxels of the volume they belong to); volumes fp32 [Nz][Ny][Nx].
 *
 * srwcr_field: the dense FFD displacement u(x) at params (Eq 17 taps, the fp32 arithmetic of
 *   the passes).  params host or device; field host or device (written).  Errors: EINVAL,
 *   ECUDA, ESTATE.
 * The context-free functions below take DEVICE pointers only (EINVAL otherwise) and run
 * on `stream` (a cudaStream_t, NULL = default stream); they return ECUDA on a launch
 * error and do not synchronise:
 *   srwcr_resample        out(x) = vol(x + u(x)), trilinear, positions clamped per axis to
 *                         [0, N-1] (readings c1-c3)
 *   srwcr_compose         out(x) = u(x) + U(x + u(x)): the backward warp by u followed by U
 *                         (out must not alias U or u)
 *   srwcr_downsample2     2x pyramid: out voxel i = mean of voxels 2i, 2i+1 per axis (the
 *                         last one repeated at an odd edge; a 1-slice z axis stays 1);
 *                         out dims = ceil(dims / 2)
 *   srwcr_upsample2_field fine field u_f(x) = 2 u_c((x - 1/2) / 2) (trilinear, clamped)
 */
srwcr_status srwcr_field(srwcr_ctx *ctx, const double *params, float *field);
srwcr_status srwcr_resample(const float *vol, const int64_t dims[3], const float *field, float *out, void *stream);
srwcr_status srwcr_compose(const float *U, const float *u, const int64_t dims[3], float *out, void *stream);
srwcr_status srwcr_downsample2(const float *vol, const int64_t dims[3], float *out, void *stream);
srwcr_status srwcr_upsample2_field(const float *coarse, const int64_t coarse_dims[3], float *fine,
                                   const int64_t fine_dims[3], void *stream);

/* Debug / parity dumps (copied to host memory `out` of `bytes` bytes).
 *   SRWCR_DUMP_FIXED, _MOVING   normalised volumes, fp32 [Nz][Ny][Nx]
 *   SRWCR_DUMP_A0               fixed-image bin a0 = min(floor F, L-1) per voxel, int16
 *   SRWCR_DUMP_CTRL_TAPS        per axis x,y,z: int32 tap base per voxel index (Nx+Ny+Nz values)
 *   SRWCR_DUMP_SPAT_TAPS        same for the spatial-bin lattice
 *   SRWCR_DUMP_N                static weighted counts N[r][a], fp64 [R][L+1]
 *   SRWCR_DUMP_SQ               S[r][a], Q[r][a] of the last pass 1 (unshifted), fp64 [2][R][L+1]
 *   SRWCR_DUMP_REGIONS          per region {p(r), sigma_r^2, mu_r, 1-CR_r, retained, Z}, fp64 [R][6]
 *   SRWCR_DUMP_COEFS            alpha[R], beta[R], gamma[R][L+1] (fp32) of the last combine
 *   SRWCR_DUMP_WARPED           pass 1's per-voxel (m, dM/dy_x, dM/dy_y, dM/dy_z) of this rank's
 *                               z-slab after the last evaluation, fp32 [z1-z0][Ny][Nx][4]: the warped
 *                               moving intensity m = M(T(x)) that decides the dynamic Parzen bin
 *                               n(m) = min(floor m, L-1) (Eq 5) -- for the fp32-vs-fp64 bin
 *                               mismatch report
 *   SRWCR_DUMP_DDM              per-voxel dD/dm of the last pass 2 is not stored: ENOTSUP
 * `bytes` must be at least the size given by srwcr_debug_size. */
enum {
    SRWCR_DUMP_FIXED = 1, SRWCR_DUMP_MOVING = 2, SRWCR_DUMP_A0 = 3, SRWCR_DUMP_CTRL_TAPS = 4,
    SRWCR_DUMP_SPAT_TAPS = 5, SRWCR_DUMP_N = 6, SRWCR_DUMP_SQ = 7, SRWCR_DUMP_REGIONS = 8,
    SRWCR_DUMP_COEFS = 9, SRWCR_DUMP_WARPED = 10
};
srwcr_status srwcr_debug_size(const srwcr_ctx *ctx, int32_t what, size_t *bytes);
srwcr_status srwcr_debug_dump(srwcr_ctx *ctx, int32_t what, void *out, size_t bytes);

/* Kernel-launch counters and the last eval's per-pass device times (ms, CUDA events
 * on the library stream; only filled when timing is enabled with srwcr_set_timing). */
typedef struct {
    int64_t launches_total;     /* kernels launched by this context since creation */
    int32_t launches_per_eval;  /* kernels in one srwcr_eval (graph nodes that are kernels) */
    float ms_pass1, ms_combine, ms_pass2, ms_total;  /* pass 1 = the k_pass1 launch alone */
    int32_t warps_per_cta;      /* decomposition chosen at create */
    int32_t slot_capacity;      /* max distinct fixed bins of one work item */
    int32_t voxels_per_lane;    /* 1 or 2 along x */
    int32_t items;              /* CTAs per pass on this rank */
    float ms_prep;              /* params -> fp32 and tap-window max kernels before pass 1 */
    int32_t warps_per_cta2, items2;  /* pass 2's decomposition */
    int32_t exact_voxels;       /* voxels of the last eval's pass 2 decided in fp64 (k_exact_fix) */
    int32_t exact_capacity;     /* list capacity; more fall back to a scan of the slab */
    int32_t pipe_items1;        /* host-buffer srwcr_eval: pass-1 items started after the first
                                   part of the params upload (0: not pipelined) */
    int32_t pipe_items2;        /* pass-2 items after which the final gradient layers go back
                                   while the rest run (0: not pipelined) */
    int32_t fast_path;          /* 1: the round-2 passes of srwcr_fast.cuh evaluate (coarse
                                   spatial lattice, orientation 0, 3-D); 0: round-1 passes */
    int32_t fast_items;         /* work items (CTAs) of the fast passes on this rank */
    int32_t fast_warps;         /* warps per CTA of the fast passes */
    int32_t fast_slots;         /* line-table slot stride (max fixed bins of an item + 2) */
} srwcr_stats;
srwcr_status srwcr_set_timing(srwcr_ctx *ctx, int32_t enable);
srwcr_status srwcr_get_stats(const srwcr_ctx *ctx, srwcr_stats *out);

/* The CUDA stream all work of this context is issued on (a cudaStream_t). */
srwcr_status srwcr_stream(const srwcr_ctx *ctx, void **stream);

const char *srwcr_last_error(const srwcr_ctx *ctx);
void srwcr_destroy(srwcr_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif /* SRWCR_H */
