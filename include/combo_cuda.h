/*
 * combo_cuda.h -- C-ABI of the B200-native ComBo Lippmann-Schwinger hot path.
 *
 * Drop-in boundary for the reference library's solver / material API
 * (/root/reference/proj). Every entry point returns an int status (0 = OK,
 * negative = error, mapped onto the reference exception types of
 * include/combo/errors.hpp:11-55); none throws or aborts. Plain pointers and
 * sizes only. Pointers passed to operator-level calls may live on the host or
 * on the device (COMBO_MEM_HOST / COMBO_MEM_DEVICE); host arrays are borrowed
 * for the duration of the call.
 *
 * Reference interface each group replaces:
 *   combo_solve ................. solve()                    src/solver.cpp:286-346, solver.hpp:68-69
 *   combo_stress_sweep .......... stress_sweep()             src/cell_material.cpp:104-168
 *   combo_phase_averages ........ recover_phase_fields() + phase_averages()  src/postprocess.cpp:13-106
 *   combo_recover_composites .... recover_phase_fields() per composite       src/postprocess.cpp:13-36
 *   combo_tangent_matvec ........ stress_sweep(tangents45) + tangent_matvec()  cell_material.cpp:170-194
 *   combo_tangent45 / _matvec45 . pack45 tangents / tangent_matvec (API compat) cell_material.cpp:86-102,170-194
 *   combo_project ............... GreenOperator::project()   src/green.cpp:133-151
 *   combo_fft_forward ........... Fft3::forward()            src/fft.cpp:52
 *   combo_dfmg_stress ........... dfmg_stress()              src/dfmg.cpp:128-176
 *   combo_dfmg_tangent_matvec ... dfmg_tangent_pass + dfmg_tangent_matvec  dfmg.cpp:178-253
 *   combo_bind_materials ........ CellMaterials::CellMaterials src/cell_material.cpp:12-55
 *   combo_coarsen ............... coarsen()                  src/combo_grid.cpp:28-71
 *   combo_laplace_weights ....... laplace_weights(direct)    src/normals.cpp:25-52
 *   combo_normals ............... compute_normals()          src/normals.cpp:211-256
 *   combo_generate .............. generate_*()               src/image.cpp:57-227 (+ seeded config generators)
 *   combo_laminate_solve ........ finite_strain_solve()      src/laminate.cpp:158-272
 */
#ifndef COMBO_CUDA_H_
#define COMBO_CUDA_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------ status codes */
#define COMBO_OK 0
#define COMBO_ERR_CONFIG_INVALID -1      /* ConfigInvalid                   */
#define COMBO_ERR_INADMISSIBLE_MACRO -2  /* InadmissibleMacroState          */
#define COMBO_ERR_LOAD_PATH_FAILED -3    /* LoadPathFailed (solve reports it in the report, returns OK) */
#define COMBO_ERR_SINGULAR -4            /* SingularMatrix                  */
#define COMBO_ERR_NON_DIVIDING_FACTOR -5 /* NonDividingFactor               */
#define COMBO_ERR_BAD_SHAPE -6           /* BadShapeSpec                    */
#define COMBO_ERR_CUDA -10
#define COMBO_ERR_NCCL -11
#define COMBO_ERR_OOM -12
#define COMBO_ERR_BAD_ARGUMENT -13
#define COMBO_ERR_STATE -14 /* call order, e.g. sweep before bind */

#define COMBO_MEM_HOST 0
#define COMBO_MEM_DEVICE 1

/* enums mirror the reference */
#define COMBO_LAW_NEO_HOOKEAN 0 /* materials.hpp:87-101 */
#define COMBO_LAW_LINEAR 1      /* materials.hpp:103-115 */
#define COMBO_GREEN_CONTINUOUS 0 /* green.hpp:12 */
#define COMBO_GREEN_ROTATED 1
#define COMBO_GREEN_STAGGERED 2
#define COMBO_SCHEME_BASIC 0 /* solver.hpp:15 */
#define COMBO_SCHEME_NEWTON_CG 1
#define COMBO_EVAL_PER_CELL 0 /* solver.hpp:16 */
#define COMBO_EVAL_DFMG 1
#define COMBO_NORMAL_BARYCENTER 0 /* normals.hpp:31 */
#define COMBO_NORMAL_SECOND_MOMENT 1
#define COMBO_CENTER_WEIGHTED_CENTROID 0 /* normals.hpp:32 */
#define COMBO_CENTER_BOXEL 1

typedef struct combo_ctx combo_ctx;
typedef struct combo_report combo_report;

/* NeoHookeanParams (materials.hpp:14-21) given directly as (lambda, mu), or
 * LinearElasticParams (materials.hpp:23-29) as a Mandel 6x6 (row major). */
typedef struct combo_law {
  int kind;
  double lambda;
  double mu;
  double c6[36];
} combo_law;

/* LaminateOptions (laminate.hpp:72-79) */
typedef struct combo_laminate_opts {
  double tol_abs;
  double tol_rel;
  double stress_floor; /* 0 -> 1e-12 * max(hi, 1e-12) as cell_material.cpp:50-54 */
  int max_iter;
  int back_projection;
  double c_min;
} combo_laminate_opts;

/* SolverConfig (solver.hpp:18-32) + a bounded-LS-iteration hook for benches */
typedef struct combo_solver_cfg {
  int scheme;
  int green;
  int eval;
  double tol_equilibrium;
  int max_outer;
  double cg_tol;
  int cg_max;
  int load_steps;
  int max_bisections;
  int threads; /* ignored (reference: OpenMP threads) */
  int verbose;
  long long max_ls_iterations; /* 0 = unlimited */
} combo_solver_cfg;

/* SweepStats (cell_material.hpp:76-84) */
typedef struct combo_sweep_stats {
  int64_t inadmissible_cells;
  int64_t laminate_failures;
  int64_t back_projections;
  int64_t laminate_iter_max;
} combo_sweep_stats;

/* PhaseAverages (postprocess.hpp:27-35) + RecoveredFields::max_resolve_iterations */
typedef struct combo_phase_avg {
  double pbar[9];
  double pbar_plus[9];
  double pbar_minus[9];
  double c_plus;  /* inclusion volume fraction as represented */
  int32_t has_plus;
  int32_t has_minus;
  int32_t max_resolve_iterations;
} combo_phase_avg;

/* NormalStats (normals.hpp:39-43) */
typedef struct combo_normal_stats {
  int64_t composite;
  int64_t degenerate_fallbacks;
  int64_t too_few_fallbacks;
} combo_normal_stats;

/* StepReport (solver.hpp:34-46) summary; histories via combo_report_* */
typedef struct combo_step_info {
  double t_start, t_end;
  double fbar[9];
  int converged;
  int outer_iters;
  int cg_breakdowns;
  int line_search_cuts;
  int n_residuals;
  combo_sweep_stats sweep;
  double seconds;
  int64_t ls_basic, ls_residual, ls_cg, ls_trial; /* LS iterations by type */
} combo_step_info;

/* ---------------------------------------------------------------- lifecycle */
int combo_ctx_create(int device, combo_ctx** out);
/* one process driving ndev GPUs: rank q of the axis-0 slab
 * decomposition on devices[q], NCCL clique from ncclCommInitAll; bind /
 * solve / project take and return whole-grid arrays as on one GPU. */
int combo_ctx_create_multi(int ndev, const int* devices, combo_ctx** out);
int combo_ctx_destroy(combo_ctx* ctx);
const char* combo_last_error(const combo_ctx* ctx);
const char* combo_version(void);
/* number of this library's kernels launched so far on ctx (bench evidence) */
int combo_kernel_launches(const combo_ctx* ctx, int64_t* count);
int combo_synchronize(combo_ctx* ctx);
/* CUDA-event timing of every kernel launch on ctx's stream (bench roofline):
 * enable clears the records; json = {"tag": {"launches", "ms", "bytes"}} with
 * bytes the algorithmic HBM bytes of those launches. */
int combo_profile_enable(combo_ctx* ctx, int enable);
const char* combo_profile_json(combo_ctx* ctx);

/* ------------------------------------------------------------ preprocessing */
/* shape: 0 sphere(r), 1 octahedron(r), 2 fiber(axis, r, length),
 * 3 cross_ply(r, pitch, layers), 4 fiber_pack(seed, count, r, length, spread),
 * 5 slab(axis, fraction), 10 rsa_spheres(seed, rmin_vox, rmax_vox, phi),
 * 11 rsa_fibers_z(seed, r_vox, phi), 12 boolean_ellipsoids(seed, amin_vox, amax_vox, phi).
 * out: dims[0]*dims[1]*dims[2] bytes (host or device per mem). */
int combo_generate(combo_ctx* ctx, int shape, const int64_t dims[3], const double lengths[3],
                   const double* params, int nparams, uint8_t* out, int mem);
int combo_coarsen(combo_ctx* ctx, const uint8_t* img, const int64_t dims[3], const int64_t factors[3],
                  uint8_t* kind, double* c_plus, int64_t* count_plus, int mem);
int combo_laplace_weights(combo_ctx* ctx, const uint8_t* img, const int64_t dims[3],
                          const double lengths[3], double* w, int mem);
int combo_normals(combo_ctx* ctx, const uint8_t* img, const int64_t dims[3], const double lengths[3],
                  const int64_t factors[3], const uint8_t* kind, int method, int centering,
                  int min_interface_voxels, double* normal3, uint8_t* flags, combo_normal_stats* stats,
                  int mem);
/* Slab (plane-window) forms for the multi-GPU decomposition (no reference
 * counterpart: the reference builds whole images, image.cpp:57-86):
 * combo_generate_planes writes fine planes [plane0, plane0 + nplanes)
 * (mod dims[0]) of the image combo_generate would produce for dims -- the
 * same voxels bit for bit -- into out [nplanes][dims[1]][dims[2]]; `seed`
 * is the full 64-bit generator seed of the seeded shapes 4, 10, 11, 12
 * (their params[0] is ignored; combo_generate passes uint64(params[0])).
 * combo_normals_slab computes the normals of boxel planes [bp0, bp0 + nbp)
 * from an image window of planes [img0, img0 + img_planes) (mod dims[0])
 * holding those boxels' fine planes plus one halo plane on each side (the
 * Laplace stencil, normals.cpp:39-46); kind / normal3 / flags hold the nbp
 * boxel planes. combo_coarsen needs no halo: pass the slab's fine planes. */
int combo_generate_planes(combo_ctx* ctx, int shape, const int64_t dims[3], const double lengths[3],
                          const double* params, int nparams, uint64_t seed, int64_t plane0, int64_t nplanes,
                          uint8_t* out, int mem);
int combo_normals_slab(combo_ctx* ctx, const uint8_t* img, int64_t img0, int64_t img_planes,
                       const int64_t dims[3], const double lengths[3], const int64_t factors[3], int64_t bp0,
                       int64_t nbp, const uint8_t* kind, int method, int centering, int min_interface_voxels,
                       double* normal3, uint8_t* flags, combo_normal_stats* stats, int mem);

/* ------------------------------------------------------- slab decomposition */
/* Multi-GPU layout of SURVEY.md 8e (the reference is single-process OpenMP,
 * parallel.hpp:19; these calls have no reference counterpart): R ranks own
 * contiguous slabs of n1/R planes along axis 0 (R must divide n1 and n2);
 * the FFT transposes slab <-> pencil with one all-to-all per direction and
 * all scalar reductions combine per-chunk partials in global order, so every
 * result is bitwise independent of R. Call before combo_bind_materials /
 * combo_set_grid; bind / solve / project then take whole-grid arrays.
 *
 * combo_ctx_set_virtual_ranks: R ranks hosted by this context on its device
 *   (test harness for the decomposition; outputs gathered in slab order).
 * combo_ctx_set_ranks: one rank per process; nccl_id = 128 bytes from
 *   combo_nccl_unique_id on rank 0, broadcast by the caller. F_out / P_out
 *   / project outputs then hold this rank's slab [9][n1/R * n2 * n3]. */
int combo_nccl_unique_id(void* nccl_id128);
int combo_ctx_set_virtual_ranks(combo_ctx* ctx, int nranks);
int combo_ctx_set_ranks(combo_ctx* ctx, int nranks, int rank, const void* nccl_id128);
int combo_ctx_ranks(const combo_ctx* ctx, int* nranks, int* rank, int* local_ranks, int64_t* i0,
                    int64_t* ni);
/* Layout introspection (host only): spectrum row offset (complex units) of
 * (c, i, j) on the slab side (side 0: i local plane, j global column) or the
 * pencil side (side 1: i global plane, j local column) of rank `rank`; cell
 * range [beg, end) of reduction chunk `block` of a slab of `nplanes` planes
 * (chunks never straddle planes, so partials are rank-count invariant). */
int combo_slab_row(const int64_t dims[3], int nranks, int rank, int side, int64_t c, int64_t i, int64_t j,
                   int64_t* off);
int combo_chunk_range(const int64_t dims[3], int64_t nplanes, int64_t block, int64_t* beg, int64_t* end,
                      int64_t* nblocks);

/* ------------------------------------------------------------------ binding */
/* SimGrid (field.hpp:16-28) for operator calls that need no materials
 * (combo_project); combo_bind_materials sets it too. */
int combo_set_grid(combo_ctx* ctx, const int64_t dims[3], const double lengths[3]);
/* CellMaterials(grid, matrix, inclusion, combo, lam) from a coarse grid:
 * kind (0 matrix, 1 inclusion, 2 composite), c_plus and normal3 per boxel. */
int combo_bind_materials(combo_ctx* ctx, const int64_t dims[3], const double lengths[3],
                         const uint8_t* kind, const double* c_plus, const double* normal3,
                         const combo_law* matrix, const combo_law* inclusion, int combo,
                         const combo_laminate_opts* lam, int mem);
/* the same from this process's slabs only (one rank per process: its n1/R
 * boxel planes; emulated ranks: the whole grid), e.g. built per slab with
 * combo_generate_planes / combo_coarsen / combo_normals_slab */
int combo_bind_materials_slab(combo_ctx* ctx, const int64_t dims[3], const double lengths[3],
                              const uint8_t* kind, const double* c_plus, const double* normal3,
                              const combo_law* matrix, const combo_law* inclusion, int combo,
                              const combo_laminate_opts* lam, int mem);
/* number of bindings made on ctx so far (a CellMaterials handle records it
 * and refuses to run once another binding replaced its materials) */
int combo_bind_generation(const combo_ctx* ctx, int64_t* gen);
int combo_composite_cells(const combo_ctx* ctx, int64_t* count);
int combo_stress_floor(const combo_ctx* ctx, double* floor);
/* warm starts (jump vectors) per composite id, 3 doubles each */
int combo_get_warm_starts(combo_ctx* ctx, double* warm3, int mem);
int combo_set_warm_starts(combo_ctx* ctx, const double* warm3, int mem);
/* CellMaterials::reset_warm_starts (cell_material.cpp:64-66) */
int combo_reset_warm_starts(combo_ctx* ctx);
/* the cudaStream_t all of ctx's kernels run on (for external CUDA events) */
int combo_get_stream(combo_ctx* ctx, void** stream);
int combo_spectrum_bounds(combo_ctx* ctx, const double fbar[9], double* lo, double* hi);

/* --------------------------------------------------------------- operators */
int combo_stress_sweep(combo_ctx* ctx, const double* F, double* P, combo_sweep_stats* stats, int mem);
int combo_tangent_matvec(combo_ctx* ctx, const double* F, const double* x, double* y, int mem);
/* post-solve: re-solve every composite laminate at F from its warm start
 * (read only) and form the volume-weighted phase averages */
int combo_phase_averages(combo_ctx* ctx, const double* F, combo_phase_avg* out, int mem);
/* recover_phase_fields() per composite cell (src/postprocess.cpp:13-36), the
 * inputs of interface_tractions() (src/postprocess.cpp:114-141): for composite
 * id q < combo_composite_cells(): cell[q] (flat boxel index), f_plus /
 * f_minus [9][ncomp] (component-major F+ / F-), traction [3][ncomp]
 * (LaminateResult::traction, src/laminate.cpp:266). Buffers are host or
 * device memory per `mem`. */
int combo_recover_composites(combo_ctx* ctx, const double* F, int64_t* cell, double* f_plus, double* f_minus,
                             double* traction, int mem);
int combo_tangent45(combo_ctx* ctx, const double* F, double* t45, int mem);
int combo_tangent45_matvec(combo_ctx* ctx, const double* t45, const double* x, double* y, int mem);
int combo_project(combo_ctx* ctx, int green_kind, const double* in, double* out, int mem);
int combo_fft_forward(combo_ctx* ctx, const int64_t dims[3], int ncomp, const double* in,
                      double* out_interleaved, int mem);
int combo_dfmg_stress(combo_ctx* ctx, const double* F, double* P, combo_sweep_stats* stats, int mem);
int combo_dfmg_tangent_matvec(combo_ctx* ctx, const double* F, const double* x, double* y, int mem);
int combo_dfmg_get_warm_starts(combo_ctx* ctx, double* warm3, int mem);
/* single laminate solve (laminate.cpp:158-272) on the device, for tests.
 * istate: converged, iterations, back_projections, inadmissible */
int combo_laminate_solve(combo_ctx* ctx, const double fbox[9], const combo_law* plus,
                         const combo_law* minus, const double normal[3], double c_plus,
                         const double a0[3], const combo_laminate_opts* lam, double p9[9],
                         double a3[3], int istate[4]);

/* ------------------------------------------------------------------- solver */
/* solve(cm, fbar, cfg): F_out / P_out nullable (9*N, component major).
 * Returns COMBO_OK with report->success = 0 on LoadPathFailed (solver.cpp:332-336). */
int combo_solve(combo_ctx* ctx, const double fbar[9], const combo_solver_cfg* cfg, double* F_out,
                double* P_out, double pbar[9], combo_report** report, int mem);
int combo_report_summary(const combo_report* r, int* success, int* bisections, int* nsteps,
                         double* alpha, double* seconds_total, int64_t* ls_total);
int combo_report_step(const combo_report* r, int step, combo_step_info* info);
/* residual / P-bar histories of a step (n = info.n_residuals) */
int combo_report_step_history(const combo_report* r, int step, double* residuals, double* pbar9,
                              int* cg_iters);
const char* combo_report_json(const combo_report* r);
int combo_report_free(combo_report* r);

#ifdef __cplusplus
}
#endif
#endif /* COMBO_CUDA_H_ */
