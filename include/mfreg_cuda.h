/*
 * mfreg_cuda.h — C ABI of the B200-native NGF + curvature derivative hot path
 * (paper_1804_10541_b200/libmfreg_cuda.so).
 *
 * Drop-in boundary for the reference C++ library mfreg (/root/reference/proj).
 * The reference has no FFI; its public surface is the C++ API in
 * include/mfreg/<name>.hpp. Each entry point below names the reference declaration
 * it replaces (file:line under /root/reference/proj/include/mfreg/). Plain
 * pointers and sizes only; no C++ or torch types cross this boundary.
 *
 * Conventions (same as the reference):
 *  - fields are fp64, x fastest (grid.hpp:63); 3-vectors are component-major
 *    (all x, all y, all z; ngf.cpp:75-77);
 *  - `where` = MFREG_CU_HOST: pointers are host memory, copied in/out per call;
 *    `where` = MFREG_CU_DEVICE: pointers are CUDA device memory on the current
 *    device, nothing crosses PCIe;
 *  - errors are returned as status codes; MFREG_CU_EINVAL corresponds to the
 *    reference's std::invalid_argument (same message text, retrievable with
 *    mfreg_cu_last_error), MFREG_CU_ELOGIC to std::logic_error;
 *  - mode MFREG_CU_PARITY reproduces the reference bit for bit (same operation
 *    order, no FMA, 4096-chunk reductions, closed-form Gauss-Newton Hv);
 *    MFREG_CU_FAST uses tree reductions and the factored Hv
 *    2h dT^T dr^T dr dT (max-rel <= 1e-9 vs the reference, tests/test_gpu_parity.py).
 */
#ifndef MFREG_CUDA_H
#define MFREG_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MFREG_CU_OK 0
#define MFREG_CU_EINVAL 1 /* std::invalid_argument in the reference */
#define MFREG_CU_ELOGIC 2 /* std::logic_error */
#define MFREG_CU_ECUDA 3  /* CUDA runtime / launch failure */
#define MFREG_CU_EOTHER 4

#define MFREG_CU_HOST 0
#define MFREG_CU_DEVICE 1

#define MFREG_CU_PARITY 0
#define MFREG_CU_FAST 1
#define MFREG_CU_FAST32 2 /* fused kernels on single-precision image state (tolerance 1e-4) */

#define MFREG_CU_LBFGS 0       /* mfreg::Method::Lbfgs (multilevel.hpp:36) */
#define MFREG_CU_GAUSS_NEWTON 1 /* mfreg::Method::GaussNewton */

/* mfreg::GridDesc (grid.hpp:50-120) without the kind tag: each call states
 * whether it expects a cell-centred image grid or a nodal deformation grid. */
typedef struct {
    int64_t m[3];
    double h[3];
} mfreg_cu_grid;

/* mfreg::OptimizerConfig (optimizer.hpp:145-155), field for field. */
typedef struct {
    int max_iters;
    double c1;
    double beta;
    int max_backtracks;
    int cg_max_iters;
    double cg_rel_tol;
    int h0_max_iters;
    double h0_rel_tol;
    int lbfgs_history;
    double gamma;
    double tol_rel_j;
    double tol_grad;
    double tol_step;
} mfreg_cu_opt_config;

/* mfreg::IterationRecord (optimizer.hpp:22-30). */
typedef struct {
    int iter;
    int cg_iters;
    double j;
    double distance;
    double regularizer;
    double grad_norm;
    double step;
} mfreg_cu_iter_record;

/* mfreg::MultilevelConfig (multilevel.hpp:38-45) + execution mode. */
typedef struct {
    int levels;
    int64_t deform_ratio;
    double tau;
    double rho;
    double alpha;
    int method;
    int mode;
    mfreg_cu_opt_config opt;
} mfreg_cu_ml_config;

typedef struct mfreg_cu_ngf mfreg_cu_ngf;             /* NgfPrecomp + NgfWorkspace (ngf.hpp:21-37) */
typedef struct mfreg_cu_objective mfreg_cu_objective; /* mfreg::Objective (optimizer.hpp:53-106) */

/* ---- runtime -------------------------------------------------------------- */
const char* mfreg_cu_last_error(void);
int mfreg_cu_version(void);
int mfreg_cu_device_count(int* n);
int mfreg_cu_set_device(int device);
int mfreg_cu_synchronize(void);
/* high-water mark of the library's live device allocations (bytes) since load or the last
 * reset (reset != 0 restarts it at the current level); the CLI's peak-derivative-buffer-bytes
 * (the reference reports its host scratch peak, counters.hpp:30-47) */
int mfreg_cu_device_memory_peak(int reset, int64_t* bytes);
/* kernel launches issued by this library since load (for launch accounting) */
int64_t mfreg_cu_launch_count(void);

/* ---- grids (grid.hpp:131-146; multilevel.hpp:31-33) ------------------------ */
int mfreg_cu_make_deform_grid(const mfreg_cu_grid* image, const int64_t points[3], mfreg_cu_grid* out);
int mfreg_cu_deformation_grid_for(const mfreg_cu_grid* image, int64_t ratio, mfreg_cu_grid* out);

/* ---- grid transfer (transfer.hpp:22-30) ------------------------------------ */
int mfreg_cu_transfer_apply(const mfreg_cu_grid* nodal, const mfreg_cu_grid* image, const double* y, double* out,
                            int where);
int mfreg_cu_transfer_apply_transpose(const mfreg_cu_grid* nodal, const mfreg_cu_grid* image, const double* w,
                                      double* out, int where);

/* ---- image (volume.hpp:18-56) ---------------------------------------------- */
int mfreg_cu_sample_deformed(const mfreg_cu_grid* image, const double* tpl, const double* points, int64_t n,
                             double* values, double* partials, int where);
int mfreg_cu_downsample(const mfreg_cu_grid* image, const double* v, double* out, mfreg_cu_grid* out_grid,
                        int where);

/* ---- curvature (curvature.hpp:13-31), nodal grid ---------------------------- */
int mfreg_cu_laplacian_apply(const mfreg_cu_grid* nodal, const double* u_comp, double* out, int where);
int mfreg_cu_curvature_value(const mfreg_cu_grid* nodal, const double* u, double* out, int mode, int where);
int mfreg_cu_curvature_gradient(const mfreg_cu_grid* nodal, const double* u, double* out, int where);
int mfreg_cu_curvature_hessian_vec(const mfreg_cu_grid* nodal, const double* p, double* out, int where);

/* ---- NGF distance (ngf.hpp:26-85) ------------------------------------------- */
/* make_ngf_precomp(reference, rho) + empty workspace */
int mfreg_cu_ngf_create(const double* ref, const mfreg_cu_grid* image, double tau, double rho, int mode, int where,
                        mfreg_cu_ngf** out);
int mfreg_cu_ngf_destroy(mfreg_cu_ngf* ngf);
/* populate_ngf_workspace(ws, tpl, points, pre, params, g) */
int mfreg_cu_ngf_populate(mfreg_cu_ngf* ngf, const double* tpl, const double* points, int where);
/* ngf_value(ws, g) */
int mfreg_cu_ngf_value(mfreg_cu_ngf* ngf, double* out);
/* ngf_gradient(ws, pre, g, out), out length 3m */
int mfreg_cu_ngf_gradient(mfreg_cu_ngf* ngf, double* out, int where);
/* ngf_hessian_vec(p, ws, pre, g, out), image-grid p and out, length 3m */
int mfreg_cu_ngf_hessian_vec(mfreg_cu_ngf* ngf, const double* p, double* out, int where);
/* workspace fields: values (m), partials (3m), residual, inv1, inv2 (m each),
 * rho_hat (7m, direction-major in kAllDirs order = ngf_rho(i, k)); any may be NULL */
int mfreg_cu_ngf_workspace(mfreg_cu_ngf* ngf, double* values, double* partials, double* residual, double* inv1,
                           double* inv2, double* rho_hat, int where);

/* ---- Objective (optimizer.hpp:53-106) --------------------------------------- */
int mfreg_cu_objective_create(const double* ref, const double* tpl, const mfreg_cu_grid* image,
                              const mfreg_cu_grid* deform, double tau, double rho, double alpha, int mode, int where,
                              mfreg_cu_objective** out);
int mfreg_cu_objective_destroy(mfreg_cu_objective* obj);
int mfreg_cu_objective_dof(mfreg_cu_objective* obj, int64_t* dof);
int mfreg_cu_objective_min_spacing(mfreg_cu_objective* obj, double* out);
int mfreg_cu_objective_identity(mfreg_cu_objective* obj, double* out, int where);
/* Objective::eval(y, grad): grad may be NULL (value only) */
int mfreg_cu_objective_eval(mfreg_cu_objective* obj, const double* y, double* grad, int where, double* j);
/* last_distance() / last_regularizer() */
int mfreg_cu_objective_last(mfreg_cu_objective* obj, double* distance, double* regularizer);
/* Bench support (no reference counterpart): average device time in ms, CUDA events on
 * the launching stream, of one fast-mode image-pass kernel: which = 0 GN Hv pass
 * (operand = p), 1 eval pass, 2 warp (operand = y); flush_bytes > 0 writes a scratch
 * buffer of that size before every launch (L2 flush, outside the timed interval). */
int mfreg_cu_objective_profile_kernel(mfreg_cu_objective* obj, int which, const double* operand, int reps,
                                      long long flush_bytes, double* ms);
/* Objective::gn_hessian_vec(p, q) at the last evaluated iterate */
int mfreg_cu_objective_gn_hessian_vec(mfreg_cu_objective* obj, const double* p, double* q, int where);
/* Objective::seed_hessian_vec(p, gamma, q) */
int mfreg_cu_objective_seed_hessian_vec(mfreg_cu_objective* obj, const double* p, double gamma, double* q,
                                        int where);

/* vec_dot(a, b) (optimizer.cpp:12-19) over the dof the objective owns (all of
 * them, or the owned nodal planes of a z-slab objective) */
int mfreg_cu_objective_dot(mfreg_cu_objective* obj, const double* a, const double* b, int where, double* out);

/* ---- z-slab decomposition (multi-GPU) --------------------------
 * No reference counterpart: the reference parallelises one address space with
 * OpenMP (parallel.hpp:22-55); this splits the image z axis across processes.
 * table[r*7 + 0..6] = zlo, zhi (image planes [zlo, zhi) of rank r), own_lo, own_hi
 * (owned nodal planes), need_lo, need_hi (nodal operand planes read; the halo
 * comes from ranks r-1 / r+1), bnd (P^T planes [own_hi, own_hi + bnd) shared with
 * rank r+1, which adds them). Pure host computation. */
int mfreg_cu_slab_partition(const mfreg_cu_grid* image, const mfreg_cu_grid* deform, int nranks, int32_t* table);
/* the same for parity-mode slabs (MFREG_CU_PARITY): their operand halo also covers the warp of
 * the image planes of the nodal slab below own_lo, whose per-voxel terms the rank recomputes so
 * that each owned node's P^T gather runs complete (bnd is then unused) */
int mfreg_cu_slab_partition_mode(const mfreg_cu_grid* image, const mfreg_cu_grid* deform, int nranks, int mode,
                                 int32_t* table);
/* Objective over one slab (fast mode): ref/tpl are the whole volume (replicated);
 * slab = {zlo, zhi, own_lo, own_hi} from the partition. eval / gn_hessian_vec
 * return this rank's contributions: D and alpha S of its planes (via
 * mfreg_cu_objective_last) and the nodal result on [min(own_lo, .), own_hi + bnd). */
int mfreg_cu_objective_create_slab(const double* ref, const double* tpl, const mfreg_cu_grid* image,
                                   const mfreg_cu_grid* deform, double tau, double rho, double alpha,
                                   const int32_t slab[4], int where, mfreg_cu_objective** out);

/* ---- z slabs in the library (csrc/slab.cu): one rank per GPU --------
 * A communicator carries the plane exchanges (ncclSend/ncclRecv) and the scalar
 * all-gathers (ncclAllGather); scalars are summed in rank order, so every rank holds
 * identical J / dot products and takes identical solver branches. */
typedef struct mfreg_cu_comm mfreg_cu_comm;
typedef struct mfreg_cu_slab mfreg_cu_slab;
/* ncclGetUniqueId on one rank; every rank passes the same 128 bytes to create_nccl */
int mfreg_cu_comm_nccl_unique_id(unsigned char out[128]);
/* NCCL communicator of `nranks` on the calling thread's current device (libnccl.so.2 is
 * loaded at run time) */
int mfreg_cu_comm_create_nccl(const unsigned char id[128], int nranks, int rank, mfreg_cu_comm** out);
/* `nranks` in-process communicators (out[0..nranks)) for ranks running as threads of one
 * process, on one or several devices (device copies + host barriers) */
int mfreg_cu_comm_create_local(int nranks, mfreg_cu_comm** out);
int mfreg_cu_comm_destroy(mfreg_cu_comm* comm);
int mfreg_cu_comm_rank(mfreg_cu_comm* comm, int* rank, int* size);
/* this rank's share of Objective (optimizer.hpp:53-106): ref / tpl are the whole volume
 * (replicated), the slab is slab_partition_mode(image, deform, size, mode)[rank].
 * mode MFREG_CU_FAST: fused kernels, scalars within the fast-mode tolerance of one GPU;
 * MFREG_CU_PARITY: J, gradient, GN Hv and every vec_dot bitwise equal to the one-GPU parity
 * objective (the reference's 4096-chunk sums and red-black P^T order across ranks) */
int mfreg_cu_slab_create(mfreg_cu_comm* comm, const double* ref, const double* tpl, const mfreg_cu_grid* image,
                         const mfreg_cu_grid* deform, double tau, double rho, double alpha, int mode, int where,
                         mfreg_cu_slab** out);
int mfreg_cu_slab_destroy(mfreg_cu_slab* slab);
/* zlo, zhi, own_lo, own_hi, need_lo, need_hi, bnd of this rank */
int mfreg_cu_slab_info(mfreg_cu_slab* slab, int32_t info[7]);
int mfreg_cu_slab_identity(mfreg_cu_slab* slab, double* out_dev);
/* Objective::eval on device vectors (full length 3 m^y, owned planes valid; the halo planes
 * of y are overwritten): the global J on every rank; grad valid on the owned planes */
int mfreg_cu_slab_eval(mfreg_cu_slab* slab, double* y_dev, double* grad_dev, double* j);
int mfreg_cu_slab_last(mfreg_cu_slab* slab, double* distance, double* regularizer);
/* Objective::gn_hessian_vec, q valid on the owned planes (p's halo planes overwritten) */
int mfreg_cu_slab_gn_hessian_vec(mfreg_cu_slab* slab, double* p_dev, double* q_dev);
/* vec_dot over the whole (sharded) vector, identical on every rank */
int mfreg_cu_slab_dot(mfreg_cu_slab* slab, const double* a_dev, const double* b_dev, double* out);
/* every rank's owned planes into v (the whole vector on every rank) */
int mfreg_cu_slab_gather(mfreg_cu_slab* slab, double* v_dev);
/* gauss_newton_minimize / lbfgs_minimize, sharded and device-resident; y_out gathered */
int mfreg_cu_slab_minimize(mfreg_cu_slab* slab, int method, const double* y0_dev, const mfreg_cu_opt_config* cfg,
                           double* y_out_dev, mfreg_cu_iter_record* trace, int cap, int* ntrace,
                           int* line_search_failed);
/* register_multilevel over z slabs (fast or parity mode, cfg->mode): every level sharded over
 * the communicator (levels too thin for the slab halo run replicated); result on every rank */
int mfreg_cu_slab_register_multilevel(mfreg_cu_comm* comm, const double* ref, const double* tpl,
                                      const mfreg_cu_grid* image, const mfreg_cu_ml_config* cfg, double* y_out,
                                      mfreg_cu_grid* deform_out, mfreg_cu_iter_record* trace, int cap, int* level_iters,
                                      int* line_search_failed, int where);

/* ---- solvers (optimizer.hpp:123-166) ---------------------------------------- */
/* cg_solve on the objective's GN operator (op = 0) or seed operator (op = 1, gamma) */
int mfreg_cu_cg_solve(mfreg_cu_objective* obj, int op, double gamma, const double* b, int max_iters, double rel_tol,
                      double* x, int* iters, double* relres, int* breakdown, int where);
/* lbfgs_minimize / gauss_newton_minimize; trace holds up to `cap` records */
int mfreg_cu_minimize(mfreg_cu_objective* obj, int method, const double* y0, const mfreg_cu_opt_config* cfg,
                      double* y_out, mfreg_cu_iter_record* trace, int cap, int* ntrace, int* line_search_failed,
                      int where);

/* ---- multilevel (multilevel.hpp:20-64) -------------------------------------- */
int mfreg_cu_prolong(const mfreg_cu_grid* coarse, const mfreg_cu_grid* fine, const double* y_coarse, double* y_fine,
                     int where);
/* register_multilevel(reference, tpl, cfg): y_out sized from the finest
 * deformation grid (deformation_grid_for(image, ratio)); traces packed coarsest
 * level first, level_iters[levels] records per level, ls_failed[levels]. */
int mfreg_cu_register_multilevel(const double* ref, const double* tpl, const mfreg_cu_grid* image,
                                 const mfreg_cu_ml_config* cfg, double* y_out, mfreg_cu_grid* deform_out,
                                 mfreg_cu_iter_record* trace, int cap, int* level_iters, int* line_search_failed,
                                 int where);

/* register_multilevel with the per-level results of multilevel.hpp:47-51: level_image_grids /
 * level_deform_grids [levels] (coarsest first) and, when level_y is non-NULL, every level's
 * final deformation concatenated coarsest first (3 * count(level deform grid) each; at most
 * level_y_cap doubles, else MFREG_CU_EINVAL). */
int mfreg_cu_register_multilevel_ex(const double* ref, const double* tpl, const mfreg_cu_grid* image,
                                    const mfreg_cu_ml_config* cfg, double* y_out, mfreg_cu_grid* deform_out,
                                    mfreg_cu_iter_record* trace, int cap, int* level_iters, int* line_search_failed,
                                    mfreg_cu_grid* level_image_grids, mfreg_cu_grid* level_deform_grids,
                                    double* level_y, int64_t level_y_cap, int where);

/* ---- drop-in API: the rest of the reference's public surface (csrc/api.cu) ----------
 * All computed on the GPU in the reference's operation order (bitwise in parity). */

/* vec_dot / vec_inf_norm (optimizer.hpp:18-20; optimizer.cpp:12-29): the exact
 * 4096-element chunked sum of the reference; vec_norm = sqrt(vec_dot(a, a)) */
int mfreg_cu_vec_dot(const double* a, const double* b, int64_t n, int where, double* out);
int mfreg_cu_vec_inf_norm(const double* a, int64_t n, int where, double* out);
/* make_transfer_plan (transfer.hpp:22; transfer.cpp:11-47): base[k], rem[k] over the image
 * axes concatenated (m_x, then m_y, then m_z entries); either may be NULL */
int mfreg_cu_transfer_plan(const mfreg_cu_grid* nodal, const mfreg_cu_grid* image, int64_t* base, double* rem);
/* discrete_gradient (volume.hpp:50-51; volume.cpp:96-109) at the voxels idx[0..n) (host
 * array; NULL = every voxel in order) -> out6[6k..6k+5] (backward x,y,z, forward x,y,z) */
int mfreg_cu_discrete_gradient(const mfreg_cu_grid* image, const double* v, const int64_t* idx, int64_t n,
                               double* out6, int where);
/* eps_norm (volume.hpp:53; volume.cpp:115-121) of n 6-vectors */
int mfreg_cu_eps_norm(const double* g6, int64_t n, double eps, double* out, int where);
/* laplacian(u_comp, g, i) (curvature.hpp:13; curvature.cpp:9-21) at the nodes idx[0..n) (host array) */
int mfreg_cu_laplacian_at(const mfreg_cu_grid* nodal, const double* u_comp, const int64_t* idx, int64_t n, double* out,
                          int where);
/* nodal_interpolate(comp, g, p) (multilevel.hpp:28-29; multilevel.cpp:51-76) at n points
 * (x, y, z interleaved) */
int mfreg_cu_nodal_interpolate(const mfreg_cu_grid* nodal, const double* comp, const double* pts, int64_t n,
                               double* out, int where);
/* make_ngf_precomp (ngf.hpp:26; ngf.cpp:167-183): ref_grads [m][6], ref_norms [m] */
int mfreg_cu_ngf_precomp(const double* ref, const mfreg_cu_grid* image, double rho, double* ref_grads,
                         double* ref_norms, int where);
/* NgfWorkspace::tpl_grads [m][6] of the last mfreg_cu_ngf_populate (ngf.cpp:195-201) */
int mfreg_cu_ngf_tpl_grads(mfreg_cu_ngf* ngf, double* tpl_grads, int where);
/* make_offset_table (ngf.hpp:67-85; ngf.cpp:267-300): entries grouped by linear kappa,
 * ascending; pairs (a, b) as Dir values, flattened entry by entry (<= 25 entries, 49 pairs);
 * MFREG_CU_ELOGIC on the closed-form mismatch, as the reference */
int mfreg_cu_offset_table(const mfreg_cu_grid* image, int* nentries, int64_t* kappa, int* npairs, int* pairs);
/* armijo_search (optimizer.hpp:138-139; optimizer.cpp:156-175) on a host phi(eta); phi sets
 * *err != 0 to abort (MFREG_CU_EOTHER) */
int mfreg_cu_armijo_search(double (*phi)(void* ctx, double eta, int* err), void* ctx, double f0, double gdotd,
                           double c1, double beta, int max_backtracks, double eta0, double* eta, int* accepted,
                           int* descent, double* f_new);

/* A host-defined mfreg::Problem (optimizer.hpp:36-48) as C callbacks. Vectors passed to the
 * callbacks are host memory of length n; a callback returns 0 on success. alpha,
 * last_distance and last_regularizer may be NULL (0.0, the Problem defaults). */
typedef struct {
    void* ctx;
    int (*eval)(void* ctx, const double* y, double* grad /* NULL: value only */, double* j);
    int (*gn_hessian_vec)(void* ctx, const double* p, double* q);
    int (*seed_hessian_vec)(void* ctx, const double* p, double gamma, double* q);
    double (*min_spacing)(void* ctx);
    double (*alpha)(void* ctx);
    double (*last_distance)(void* ctx);
    double (*last_regularizer)(void* ctx);
} mfreg_cu_problem_ops;
/* lbfgs_minimize / gauss_newton_minimize (optimizer.hpp:162-165) on a host Problem: the
 * solver loops run device-resident (vectors in HBM, exact chunked reductions), the
 * problem's operators are called back on host copies */
int mfreg_cu_problem_minimize(const mfreg_cu_problem_ops* ops, int64_t n, int method, const double* y0,
                              const mfreg_cu_opt_config* cfg, double* y_out, mfreg_cu_iter_record* trace, int cap,
                              int* ntrace, int* line_search_failed, int where);
/* cg_solve(apply, b, cfg) (optimizer.hpp:123; optimizer.cpp:113-154): apply =
 * ops->gn_hessian_vec (op 0) or ops->seed_hessian_vec with gamma (op 1) */
int mfreg_cu_problem_cg_solve(const mfreg_cu_problem_ops* ops, int64_t n, int op, double gamma, const double* b,
                              int max_iters, double rel_tol, double* x, int* iters, double* relres, int* breakdown,
                              int where);

/* ---- synthetic inputs (synthetic.hpp:13-44) --------------------------------- */
int mfreg_cu_make_phantom(const mfreg_cu_grid* image, double* out, int where);
/* warp_with(vol, make_sinusoid_warp(extent(image), max_amp, seed)) */
int mfreg_cu_warp_sinusoid(const mfreg_cu_grid* image, const double* vol, double max_amp, uint64_t seed, double* out,
                           int where);
int mfreg_cu_scale(int64_t n, double a, double* x, int where);


/* ---- volume / deformation / landmark files (reference io.hpp).
 * File-format errors map to MFREG_CU_EOTHER with the reference's std::runtime_error text. */

/* io::read_volume (io.cpp:111-164): MetaImage (MET_SHORT/USHORT/FLOAT/DOUBLE, LOCAL or
 * sibling raw). Fills `grid`; `data` (count() doubles, host or device) may be NULL to
 * query the grid (all checks still run). Elements are converted to fp64 on the GPU. */
int mfreg_cu_read_volume(const char* path, mfreg_cu_grid* grid, double* data, int where);
/* io::write_volume (io.cpp:166-188): MET_DOUBLE, LOCAL payload, byte-identical files */
int mfreg_cu_write_volume(const char* path, const mfreg_cu_grid* grid, const double* data, int where);
/* io::write_deformation (io.cpp:200-229): raw doubles + "<path>.meta" sidecar; n = length of y */
int mfreg_cu_write_deformation(const char* path, const double* y, int64_t n, const mfreg_cu_grid* nodal, int where);
/* io::read_deformation_grid (io.cpp:231-253) */
int mfreg_cu_read_deformation_grid(const char* path, mfreg_cu_grid* nodal);
/* io::read_deformation (io.cpp:255-274): y = 3 * nodal.count() doubles */
int mfreg_cu_read_deformation(const char* path, const mfreg_cu_grid* nodal, double* y, int where);
/* io::read_landmarks (io.cpp:276-303): up to `cap` physical points (x, y, z interleaved)
 * into `out` (host, may be NULL); *count = number of landmarks in the file */
int mfreg_cu_read_landmarks(const char* path, const double spacing[3], double* out, int64_t cap, int64_t* count);
/* io::landmark_error (io.cpp:305-348): fixed/moving are host (x, y, z) triples; y (length ny)
 * host or device; per-landmark errors on the GPU, mean / stddev in landmark order */
int mfreg_cu_landmark_error(const double* fixed, int64_t n_fixed, const double* moving, int64_t n_moving,
                            const double* y, int64_t ny, const mfreg_cu_grid* nodal, int where, double* mean,
                            double* stddev, int64_t* count);
/* mfreg CLI `warp` (tools/mfreg_cli.cpp:112-135) without the file IO: out = vol(P y) on the
 * volume's grid (transfer_apply + sample_deformed, reference order); extents must match */
int mfreg_cu_warp_volume(const double* vol, const mfreg_cu_grid* image, const double* y, const mfreg_cu_grid* nodal,
                         double* out, int where);

#ifdef __cplusplus
}
#endif

#endif /* MFREG_CUDA_H */
