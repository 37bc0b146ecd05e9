/*
 * fvb.h -- C ABI of libfvb.so, the B200 (sm_100a) batched multi-patch
 * finite-volume (Rusanov, compressible Euler) time step.
 *
 * Plain pointers and sizes only; every pointer argument named *_dev is a
 * device pointer (cudaMalloc / torch CUDA tensor storage), `stream` is a
 * cudaStream_t (NULL = legacy default stream).  All calls are asynchronous
 * on `stream` unless stated otherwise.  Return value: 0 on success, a
 * negative FVB_E* code otherwise; fvb_last_error() then holds a one-line
 * message for the calling thread.
 *
 * Batch layout (device): SoA over cells, the reference's Layout.SOA
 * (pkg/src/patchbench/patchdata.py:163-165):
 *     value(k, patch, cell) = base[k*T*M + patch*M + lin(cell)]
 * with lin = sum_k (c_k + shift) * m^k (coordinate 0 fastest,
 * patchdata.py:122-129), M = m^d, m = p+2 / shift 1 for the haloed input and
 * m = p / shift 0 for the interior output.  k runs over the N = d+2
 * unknowns (rho, rho*u_0..u_{d-1}, E) (equations.py:1-9).
 *
 * Threading: any host thread may call any entry point.  State the library
 * keeps per stream (the fused flavour's reduction slot, cached plans and
 * their scratch, the transfer engines) is keyed by (device, stream), and for
 * cudaStreamPerThread additionally by the calling thread.  Launches on one
 * stream are ordered; destroy a stream only after synchronising it (a new
 * stream may reuse the handle).  Independent launches on different streams
 * over disjoint batches may run concurrently.
 *
 * Which reference interface each entry point replaces is cited per
 * function (paths relative to /root/reference/pkg/src/patchbench/).
 */
#ifndef FVB_H
#define FVB_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Realisation flavours (executors.py:61-65 Realization, GPU variants). */
enum fvb_flavour {
    FVB_FUSED = 0,   /* patch-wise / nested-parallel: one fused kernel (run_patchwise, executors.py:390-445) */
    FVB_CASCADE = 1, /* batched / sequence of for-loops: one kernel per step (run_batched, executors.py:312-382) */
    FVB_GRAPH = 2    /* task graph: CUDA Graph over the per-step kernels following the lifted
                        per-patch DAG (run_taskgraph, executors.py:453-535; kernelgraph.py:215-247) */
};

/* Batch layouts (patchdata.py:49-58, codes as _LAYOUT_CODES patchdata.py:57;
 * offsets patchdata.py:142-168).  M = (p+2)^d haloed / p^d interior cells:
 *   FVB_LAYOUT_AOS    (patch*M + lin)*N + k
 *   FVB_LAYOUT_SOA    k*T*M + patch*M + lin          (fvb_step's layout)
 *   FVB_LAYOUT_AOSOA  patch*N*M + k*M + lin                                  */
enum fvb_layout { FVB_LAYOUT_AOS = 0, FVB_LAYOUT_SOA = 1, FVB_LAYOUT_AOSOA = 2 };

/* Error codes. */
#define FVB_OK 0
#define FVB_EINVAL -1     /* bad shape / parameter: ValueError (patchdata.py:69-75, microkernels.py:63-67) */
#define FVB_ELIMIT -2     /* patch too large for the fused kernel: WorkgroupLimitError (executors.py:402-408) */
#define FVB_ECUDA -3      /* CUDA runtime error: RuntimeError */
#define FVB_EINVALID_STATE -4 /* check mode found rho <= 0 or p <= 0: InvalidStateError (equations.py:64-73) */

/* Library version string, e.g. "fvb 0.1.0 sm_100a". */
const char* fvb_version(void);

/* Message for the last failed call on this thread ("" if none). */
const char* fvb_last_error(void);

/*
 * One batched time step (the hot path).  Replaces the executor call inside
 * run_launch (bench.py:236-246): run_sequential / run_batched /
 * run_patchwise / run_taskgraph (executors.py:219, :312, :390, :453) on
 * SoA field views.  Reads q_in_dev (N*T*(p+2)^d doubles, never written) and
 * writes q_out_dev (N*T*p^d doubles).  With with_reduction != 0 the maximal
 * eigenvalue of the updated solution, max over cells and axes of
 * max_eigenvalue(Q_new, axis) (neutral 0.0, executors.py:58), is written to
 * lam_dev[0] (one double, device) and, if lam_patch_dev != NULL, the
 * per-patch maxima to lam_patch_dev[0..T).  The library zeroes both first.
 * dt/h is formed once in double precision (microkernels.py:179).
 * FVB_CASCADE / FVB_GRAPH use a cached scratch arena per (d, p, T, stream)
 * owned by the library (pooled semantics, memory.py:105-137); FVB_GRAPH
 * instantiates its graph on first use and replays it afterwards.
 */
int fvb_step(int flavour, int dim, int p, int64_t T, const double* q_in_dev, double* q_out_dev,
             double dt, double h, double gamma, int with_reduction, double* lam_dev,
             double* lam_patch_dev, void* stream);

/*
 * Plan objects (explicit form of the cached arena / graph above).
 * fvb_plan_create allocates scratch for `flavour` at (dim, p, T); for
 * FVB_GRAPH `chunks` splits the batch into that many independent per-chunk
 * step chains (the reference's per-patch DAG lifted to patch chunks;
 * chunks = T reproduces one node chain per patch).  fvb_plan_execute is
 * fvb_step on the plan's buffers; fvb_plan_graph_nodes reports the node
 * count of the instantiated graph (ExecutionTrace.launch_count analog,
 * executors.py:528-534).
 */
typedef struct fvb_plan fvb_plan;
int fvb_plan_create(int flavour, int dim, int p, int64_t T, int chunks, fvb_plan** out);
int fvb_plan_execute(fvb_plan* plan, const double* q_in_dev, double* q_out_dev, double dt,
                     double h, double gamma, int with_reduction, double* lam_dev,
                     double* lam_patch_dev, void* stream);
int fvb_plan_graph_nodes(const fvb_plan* plan, int64_t* nodes);
int fvb_plan_kernel_launches(const fvb_plan* plan, int with_reduction, int64_t* launches);
int fvb_plan_destroy(fvb_plan* plan);
/*
 * fvb_step on batch arrays in any layout (both arrays in `layout`): the
 * run_patchwise / run_batched / run_taskgraph operator contract on
 * FlatFieldViews of any Layout (executors.py:312-320, :390-399, :453-462;
 * patchdata.py:293-315).  Results are bit-identical across layouts.
 */
int fvb_step_layout(int flavour, int layout, int dim, int p, int64_t T, const double* q_in_dev,
                    double* q_out_dev, double dt, double h, double gamma, int with_reduction,
                    double* lam_dev, double* lam_patch_dev, void* stream);

/*
 * fvb_step_layout with a DEVICE-resident time step: the kernels read *dt_dev
 * and form dt/h on the device (the same IEEE quotient as the host path), so
 * a multi-step loop -- step, eigenvalue, fvb_admissible_dt_dev, halo
 * refresh -- runs without host synchronisation and can be captured into a
 * CUDA graph (builder addition for SURVEY 8f row f2; the reference performs
 * one step with a host dt, TimeStepContext microkernels.py:54-67).
 */
int fvb_step_dt(int flavour, int layout, int dim, int p, int64_t T, const double* q_in_dev,
                double* q_out_dev, const double* dt_dev, double h, double gamma, int with_reduction,
                double* lam_dev, double* lam_patch_dev, void* stream);

/*
 * Local time stepping (builder addition for SURVEY 8f row f2; the paper's
 * motivation for per-patch eigenvalues): every patch
 * advances with its own time step dt_patch_dev[patch] (T doubles, device),
 * e.g. cfl*h/lam_patch of the previous step.  Each patch's result is
 * bit-identical to a one-patch fvb_step with that dt.
 */
int fvb_step_lts(int flavour, int layout, int dim, int p, int64_t T, const double* q_in_dev,
                 double* q_out_dev, const double* dt_patch_dev, double h, double gamma,
                 int with_reduction, double* lam_dev, double* lam_patch_dev, void* stream);

/* Batch layout a plan executes on (default FVB_LAYOUT_SOA). */
int fvb_plan_set_layout(fvb_plan* plan, int layout);

/*
 * Re-layout a batch array (haloed = input extent): src in src_layout ->
 * dst in dst_layout, T patches (the layout-changing gather of
 * memory.py:240-251 on the device).  src and dst must not overlap.
 */
int fvb_relayout(int dim, int p, int64_t T, int haloed, int src_layout, int dst_layout,
                 const double* src_dev, double* dst_dev, void* stream);

/* Release every cached arena / graph created by fvb_step (memory.py:231-237)
 * and the fused flavour's per-stream reduction slots. */
int fvb_release_all(void);

/*
 * Largest p the fused flavour supports for `dim` (shared-memory bound; the
 * analog of the reference's workgroup limit (p+2)^d <= 1024,
 * executors.py:402-408), and the dynamic shared memory one fused CTA uses.
 */
int fvb_fused_limit(int dim, int* max_p);
int fvb_fused_smem_bytes(int dim, int p, int64_t* bytes);

/*
 * Launch tuning of the fused kernels (builder addition; no reference
 * counterpart -- results never depend on it, only speed):
 *   FVB_TUNE_PENCIL_VARIANT  launch shape of the 2D kernels: 0 = default (p = 3
 *                            SoA: the tile kernel; tensor-map TMA rows where
 *                            p | 32 and the batch is SoA / AoSoA; else the
 *                            cp.async ring, AoS cells by 16-byte unknown
 *                            pairs), 2 / 3 / 4 / 7 = tile-kernel shapes,
 *                            6 = no tile kernel, 8 = cp.async ring only,
 *                            9 = AoS by 8-byte copies
 *   FVB_TUNE_SLAB_VARIANT    launch shape of the 3D plane-walk kernel: 0 = default
 *                            (p = 8: one warp per patch, tensor-map planes,
 *                            every layout), 5 = the slot kernel
 *   FVB_TUNE_REDUCE_FILTER   eigenvalue reduction without per-patch maxima:
 *                            -1 = per-kernel default, 0 = exhaustive, 1 = filtered
 *                            (filtered only where the physics has the hook)
 * Initial values come from the environment variables of the same names.
 */
enum fvb_tuning { FVB_TUNE_PENCIL_VARIANT = 0, FVB_TUNE_SLAB_VARIANT = 1, FVB_TUNE_REDUCE_FILTER = 2 };
int fvb_set_tuning(int key, int value);
int fvb_get_tuning(int key, int* value);

/*
 * Physics policy of every step kernel (csrc/physics.cuh): the device twin of
 * the reference's user microkernels -- flux and max_eigenvalue, opaque user
 * code the executors call but never alter (equations.py:11-12, :60-107,
 * microkernels.py:10-13).  The kernels are templates over the policy; these
 * two are compiled in:
 *   FVB_PHYSICS_EULER        compressible Euler + the optional hooks
 *                            (fast-path certification, reduce filter): default
 *   FVB_PHYSICS_EULER_PLAIN  the same closure stated as the reference's three
 *                            functions only, plain IEEE double (no hooks)
 * Both give the reference's bits.  Process-wide; a plan records the physics
 * selected when it is created (cached fvb_step plans are keyed by it).
 * Initial value from the environment variable FVB_PHYSICS.
 */
enum fvb_physics { FVB_PHYSICS_EULER = 0, FVB_PHYSICS_EULER_PLAIN = 1 };
int fvb_set_physics(int physics);
int fvb_get_physics(int* physics);

/*
 * Seeded synthetic field, bit-identical to init_field (bench.py:107-133):
 * 64-bit LCG (MMIX constants, bench.py:89-104), draws per haloed cell in
 * canonical patch / cell order, rho, u_0..u_{d-1}, p, converted to conserved
 * variables.  Fills patches [patch_begin, patch_begin + T_local) of a
 * T_total-patch stream into a T_local-patch SoA batch (jump-ahead per cell,
 * so shards of a multi-GPU run reproduce the single-stream bits).
 */
int fvb_init_field(int dim, int p, int64_t T_local, int64_t patch_begin, uint64_t seed,
                   double gamma, double* q_in_dev, void* stream);

/*
 * Layout transforms between the reference's scattered per-patch AoS arrays
 * (concatenated in patch order: ((patch*M + lin)*N + k), memory.py:60-64)
 * and the device SoA batch: gather_patches (memory.py:240-251) and
 * scatter_results (memory.py:254-265).  `haloed` selects m = p+2 or p.
 */
int fvb_aos_to_soa(int dim, int p, int64_t T, int haloed, const double* aos_dev, double* soa_dev,
                   void* stream);
int fvb_soa_to_aos(int dim, int p, int64_t T, int haloed, const double* soa_dev, double* aos_dev,
                   void* stream);

/*
 * Device microkernel probe: applies the device domain functions (the
 * equations.py:77-107 twins in euler.cuh) to `count` AoS states, writing
 * flux(q, axis) (count*N) and max_eigenvalue(q, axis) (count).  policy 0
 * evaluates in IEEE double; policy 1 the way the fused kernels do (XReal
 * fast paths, IEEE redo when one leaves its range).  Used by the parity
 * tests of the user-function interface.
 */
int fvb_eval_microkernels(int dim, int64_t count, int axis, double gamma, int policy,
                          const double* q_dev, double* flux_dev, double* lambda_dev, void* stream);

/*
 * Fast-path probe (test support for csrc/realx.cuh): quot = a/b and
 * root = sqrt(a) as the kernels' XReal fast paths compute them, flags bit 0
 * / bit 1 set where the division / square root left its proven range (the
 * kernels then recompute in IEEE).  Where a flag is clear the value must
 * equal IEEE a/b / sqrt(a) bit for bit.
 */
int fvb_probe_fastmath(int64_t count, const double* a_dev, const double* b_dev, double* quot_dev,
                       double* root_dev, int32_t* flags_dev, void* stream);

/*
 * RCP64H scaling probe (test support): counts, over every 20-bit high
 * mantissa and every biased exponent in [e_lo, e_hi], the x for which the
 * refined fast-path reciprocal of 2x differs from half that of x (the
 * kernels rely on it being 0 over the certified range of rho).
 */
int fvb_probe_rcp_scaling(int e_lo, int e_hi, int64_t* mismatches_dev, void* stream);

/*
 * Admissibility check over a batch (check=True mode, equations.py:64-73):
 * writes the number of cells with rho <= 0 or pressure <= 0 (NaN counts as
 * inadmissible, like the reference's `not rho > 0.0`) to bad_count_dev[0]
 * (one int64, device).  Only the states the reference's step evaluates are
 * checked: haloed != 0 -> the union of the flux ranges of the input (cells
 * with at most one halo coordinate; corner halo cells are never read,
 * microkernels.py:138, :153), haloed == 0 -> the interior output cells the
 * reduce evaluates (microkernels.py:190).  SoA batch.
 */
int fvb_check_admissible(int dim, int p, int64_t T, int haloed, double gamma, const double* q_dev,
                         int64_t* bad_count_dev, void* stream);

/* The same check on a batch in any layout, or (tab_dev != NULL, q_dev
 * ignored) on per-patch AoS arrays addressed through a device table of T
 * pointers (SHARED mode). */
int fvb_check_admissible_ex(int dim, int p, int64_t T, int haloed, int layout, double gamma,
                            const double* q_dev, const double* const* tab_dev, int64_t* bad_count_dev,
                            void* stream);

/*
 * Halo refresh for a multi-step run (builder addition, SURVEY §8f row f2;
 * the reference stops after one step): the T = px*py*pz patches
 * form a periodic Cartesian grid (patch index ix + px*(iy + py*iz); pz = 1
 * for d = 2).  Every haloed cell of every patch receives the interior value
 * it overlaps -- its own patch's or a neighbour's -- read from the interior
 * SoA output of the previous step (interior_dev, N*T*p^d) and written to the
 * haloed SoA input of the next (haloed_dev, N*T*(p+2)^d).
 */
int fvb_refresh_halos(int dim, int p, int px, int py, int pz, const double* interior_dev,
                      double* haloed_dev, void* stream);

/*
 * ---- Transfer modes over independently allocated host patches (SURVEY §8f
 * row f1; memory.py:162-265, bench.py:209-259) ----
 *
 * A ScatteredPatchSet is T per-patch AoS arrays (memory.py:60-64): the
 * haloed input of patch t is N*(p+2)^d doubles at in_ptr[t], its interior
 * output N*p^d doubles at out_ptr[t].  The GPU addresses them in place when
 * they are device-addressable host memory (pinned / registered, UVA).
 */

/* Registration handle of host ranges (opaque). */
typedef struct fvb_pin fvb_pin;

/* Make `count` host arrays of `nbytes` each device-addressable: the
 * page-merged spans are registered (cudaHostRegister, mapped + portable)
 * unless already known; registrations are refcounted and shared between
 * handles.  Host call.  Keep registrations of heap arrays short (the
 * Python layer registers per launch): a pageable cudaMemcpy of any other
 * buffer that starts inside a registered page and runs past it fails with
 * cudaErrorInvalidValue (measured, driver 580). */
int fvb_host_pin(const uint64_t* host_ptrs, int64_t count, int64_t nbytes, fvb_pin** out);
/* Announce a caller-pinned block (cudaHostAlloc / torch pin_memory) as
 * device-addressable (nothing is registered). */
int fvb_host_note_pinned(const void* base, int64_t nbytes, fvb_pin** out);
/* Drop a handle (unregisters ranges no other handle holds). */
int fvb_host_unpin(fvb_pin* handle);
/* *first_bad = index of the first array not inside known device-addressable
 * host memory, or -1 if all are. */
int fvb_host_accessible(const uint64_t* host_ptrs, int64_t count, int64_t nbytes, int64_t* first_bad);

/* Gather (memory.py:240-251): per-patch AoS input arrays [t0, t1) of a
 * device table of pointers -> the device batch (T patches) in `layout`.
 * Scatter (memory.py:254-265): batch interior output [t0, t1) in `layout`
 * -> per-patch AoS output arrays.  Zero-copy when the arrays are host
 * memory: the SMs read / write them over PCIe. */
int fvb_gather_table(int dim, int p, int64_t T, int64_t t0, int64_t t1, const double* const* tab_dev,
                     int layout, double* batch_dev, void* stream);
int fvb_scatter_table(int dim, int p, int64_t T, int64_t t0, int64_t t1, int layout,
                      const double* batch_dev, double* const* tab_dev, void* stream);

/*
 * The step over per-patch AoS arrays addressed through device pointer
 * tables -- SHARED mode: compute in place on the scattered allocations, no
 * batch buffers (memory.py:162-228, ScatteredFieldView patchdata.py:318-334).
 */
int fvb_step_table(int flavour, int dim, int p, int64_t T, const double* const* in_tab_dev,
                   double* const* out_tab_dev, double dt, double h, double gamma, int with_reduction,
                   double* lam_dev, double* lam_patch_dev, void* stream);

/*
 * The step over the patch range [t0, t1) of a batch of T patches (the
 * chunks of a pipelined launch).  zero_outputs != 0 zeroes lam_dev and
 * lam_patch_dev[t0..t1) first; otherwise the launch max-accumulates into
 * them.  Not for FVB_GRAPH (whole batches).
 */
int fvb_step_range(int flavour, int layout, int dim, int p, int64_t T, int64_t t0, int64_t t1,
                   const double* q_in_dev, double* q_out_dev, double dt, double h, double gamma,
                   int with_reduction, int zero_outputs, double* lam_dev, double* lam_patch_dev,
                   void* stream);

/* Plan execution with all options: pointer tables (in_tab/out_tab, q_* NULL),
 * patch range (t1 < 0: the whole batch), zeroing as fvb_step_range. */
int fvb_plan_execute_ex(fvb_plan* plan, const double* q_in_dev, double* q_out_dev,
                        const double* const* in_tab_dev, double* const* out_tab_dev, int64_t t0, int64_t t1,
                        int zero_outputs, double dt, double h, double gamma, int with_reduction,
                        double* lam_dev, double* lam_patch_dev, void* stream);

/* Sizes of the cascade / graph temporaries per axis (the reference's
 * ScratchArrays, microkernels.py:70-112, tight to the flux range): flux
 * N*T*(p+2)*p^(d-1) doubles, wave speed T*(p+2)*p^(d-1) doubles. */
int fvb_scratch_doubles(int dim, int p, int64_t T, int64_t* flux_doubles, int64_t* lambda_doubles);

/* A plan over caller-owned temporaries (flux_dev[a], lambda_dev[a] for
 * a < dim; arena buffers, memory.py:162-228).  FVB_FUSED needs none (NULL). */
int fvb_plan_create_ext(int flavour, int dim, int p, int64_t T, int chunks, double* const* flux_dev,
                        double* const* lambda_dev, fvb_plan** out);

/*
 * One launch of run_launch (bench.py:209-259) over per-patch host arrays
 * (host tables in_tab_host / out_tab_host of T addresses; SHARED needs them
 * inside device-addressable memory, fvb_host_pin).  Synchronous on `stream`.
 *   batch_in_dev == batch_out_dev == NULL: SHARED -- the step runs in place
 *     on the arrays (fvb_step_table semantics, AoS).
 *   else COPY / POOLED -- gather into the batch (`layout`), step, scatter
 *     back, pipelined over chunks of chunk_patches patches (0: ~64 MB of
 *     input per chunk) on three streams so PCIe reads, the step and PCIe
 *     writes of different chunks overlap.  Arrays that are one contiguous
 *     range in patch order inside one pinned allocation / registration
 *     (pinned blocks) move by DMA on the copy engines (staging chunk +
 *     device permutation); arrays outside device-addressable memory are
 *     host-staged (host memcpy into pinned chunks + DMA); other addressable
 *     arrays by zero-copy table kernels.  FVB_GRAPH moves chunks but runs
 *     one whole-batch step.
 * plan: the cascade / graph plan (its temporaries); NULL for FVB_FUSED.
 * *reduced_out = max(0, max eigenvalue) (0 without reduction);
 * *compute_seconds_out = device time of the step kernels.
 */
int fvb_launch_table(int flavour, int layout, int dim, int p, int64_t T, const uint64_t* in_tab_host,
                     const uint64_t* out_tab_host, double* batch_in_dev, double* batch_out_dev,
                     fvb_plan* plan, double dt, double h, double gamma, int with_reduction,
                     double* lam_patch_dev, int64_t chunk_patches, double* reduced_out,
                     double* compute_seconds_out, void* stream);

/* fvb_admissible_dt on the device: *dt_dev = cfl * h / *lam_dev (one thread). */
int fvb_admissible_dt_dev(const double* lam_dev, double h, double cfl, double* dt_dev, void* stream);

/*
 * Admissible time step from the reduced eigenvalue (builder addition; the
 * reference stops at the eigenvalue):  dt = cfl * h / lambda,
 * evaluated in IEEE double as written.  Host function.
 */
double fvb_admissible_dt(double lambda, double h, double cfl);

#ifdef __cplusplus
}
#endif

#endif /* FVB_H */
