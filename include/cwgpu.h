/*
 * cwgpu.h -- C ABI of the B200-native DAETI monodomain hot path.
 *
 * This is the drop-in boundary for the reference solver "cardwave"
 * (/root/reference/proj/core). The reference has no C ABI or plugin registry;
 * its replaceable seam is the C++ API of proj/core. Every entry point below
 * states which reference interface it replaces. Plain pointers and sizes only:
 * no C++ or torch types cross this boundary. The C++ drop-in classes with the
 * reference's exact signatures (cardwave::gpu::StrangIntegrator,
 * cardwave::gpu::run_simulation, cardwave::gpu::diffusion_substep) are in
 * include/cardwave_gpu.hpp, header-only over this ABI.
 *
 * Status codes mirror the reference exception taxonomy and the CLI exit codes
 * (errors.hpp:11-32, tools/main.cpp:322-331):
 *   CWG_OK 0, CWG_EVALIDATION 2 (ValidationError), CWG_EINSTABILITY 3
 *   (InstabilityError, node + time in cwg_error), CWG_EIO 4 (IoError),
 *   CWG_ECUDA 5 (CUDA / NCCL failure; no reference equivalent).
 *
 * Threading: one host thread per context; every call is stream-ordered on the
 * context's stream. Nothing here falls back to the CPU: without a usable
 * sm_100 device cwg_create fails with CWG_ECUDA.
 */
#ifndef CWGPU_H
#define CWGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CWG_ABI_VERSION 1

enum {
  CWG_OK = 0,
  CWG_EVALIDATION = 2,
  CWG_EINSTABILITY = 3,
  CWG_EIO = 4,
  CWG_ECUDA = 5
};

/* Cell models, by the reference registry names (ionic.cpp:59-70). The passive
 * model is an extension (non-excitable scar tissue, BASELINE config 3). */
enum {
  CWG_MODEL_ALIEV_PANFILOV = 0, /* "aliev-panfilov"   aliev_panfilov.cpp */
  CWG_MODEL_ORD_ENDO = 1,       /* "ohara2011-endo"   ohara_rudy_2011.cpp */
  CWG_MODEL_ORD_EPI = 2,        /* "ohara2011-epi" */
  CWG_MODEL_ORD_MID = 3,        /* "ohara2011-mid" */
  CWG_MODEL_MACCANNELL = 4,     /* "maccannell2007"   maccannell_2007.cpp */
  CWG_MODEL_PASSIVE = 5         /* "passive" (extension) */
};

/* Scheme (splitting.hpp:19) */
enum { CWG_OST = 0, CWG_OSTAR = 1, CWG_DAETI = 2 };

/* Operator storage chosen on the device. */
enum {
  CWG_OP_AUTO = 0,      /* stencil-2D when the CSR is a regular-sheet 9-point operator, else CSR */
  CWG_OP_CSR = 1,       /* generic CSR row loop, ascending columns (fem.cpp:201-206) */
  CWG_OP_STENCIL2D = 2, /* per-node 9 coefficients taken verbatim from the CSR */
  CWG_OP_STRUCT3D = 3,  /* extension: structured 3D slab, per-layer tables (see cwg_problem.s3d) */
  CWG_OP_SHEET2D = 4    /* regular sheet assembled on the device (see cwg_problem.sheet2d) */
};

typedef struct cwg_ctx cwg_ctx;

/* InstabilityError payload (errors.hpp:18-26) */
typedef struct {
  int code;       /* CWG_* */
  int64_t node;   /* lowest offending node (global index), -1 if none */
  double t_ms;    /* reaction: failing sub-step time t + j*dt/k; diffusion: outer step time */
  int phase;      /* 1 reaction, 2 diffusion, 0 none */
  char msg[256];
} cwg_error;

/* Structured 3D slab operator (EXTENSION): (nx+1) x (ny+1) x
 * (nz+1) nodes, spacing h, node index = (iy*(nz+1) + iz)*(nx+1) + ix.
 * Coefficients are the trilinear-hex / 2x2x2-Gauss element integrals computed
 * on the reference element per z-layer (fibre angle per layer, rotating in
 * the x-y plane), with row-sum lumped mass. */
typedef struct {
  int64_t nx, ny, nz; /* element counts */
  double h;           /* cm */
  double d_long, rho; /* D_l, D_t = rho * D_l */
  const double* fiber_angle_of_layer; /* nz element layers, radians */
} cwg_struct3d;

/* Regular sheet whose operator is assembled ON THE DEVICE (replaces the host
 * path build_diffusion_field fem.cpp:21-51 -> assemble fem.cpp:112-176 ->
 * gershgorin_step fem.cpp:178-192 for meshes made by build_regular_sheet,
 * mesh.cpp:72-98): node (ix, iy) at (ix h, iy h) with index iy (nx+1) + ix,
 * element (ex, ey) = ey nx + ex. Lumped mass and off-diagonal entries are
 * bit-identical to the reference's; a diagonal entry sums its four element
 * contributions in ascending element index and can differ from the
 * reference's std::sort order by 1-2 ulp. */
typedef struct {
  int64_t nx, ny;             /* element counts */
  double h;                   /* cm */
  double fiber_angle;         /* radians, uniform (cos/sin taken on the host) */
  double d0_myocyte, d0_fibrotic, rho;
  const int32_t* node_tags;   /* [n] host, 1 = fibroblast (assign_fibrosis, mesh.cpp:100-122); NULL = none */
  const double* elem_scale;   /* [nx ny] host, D multiplier (extension, 0 = scar); NULL = 1 */
} cwg_sheet2d;

/* Everything StrangIntegrator/run_simulation consume (splitting.hpp:83-94,
 * fem.hpp:23-32, ionic.hpp:39-55, stimulus.hpp:35-50), flattened. */
typedef struct {
  /* ---- AssembledOperator (fem.hpp:23-32) */
  int64_t n;                  /* rows = nodes */
  const int64_t* row_ptr;     /* n+1 (ignored for CWG_OP_STRUCT3D) */
  const int64_t* col;         /* nnz, ascending per row */
  const double* val;          /* nnz */
  const double* lumped_mass;  /* n */
  double dt_s;                /* Gershgorin step (fem.cpp:178-192) */
  int op_kind;                /* CWG_OP_* */
  int64_t grid_nx1, grid_ny1; /* regular-sheet node counts (x fastest); 0 = unknown */
  const cwg_struct3d* s3d;    /* for CWG_OP_STRUCT3D */

  /* ---- models (SimulationSetup::models) and NodeStateArray::model_of_node */
  int n_models;
  const int* model_kind;        /* [n_models] CWG_MODEL_* */
  const uint8_t* model_of_node; /* [n] */
  const double* gkr_scale;      /* [n] optional per-node ORd GKr multiplier (extension); NULL = 1 */

  /* ---- ProtocolIndex (stimulus.hpp:35-50), flattened: entries + per-node id lists */
  int n_stim;
  const double* stim_t_start;
  const double* stim_duration;
  const double* stim_amplitude;
  const double* stim_period;      /* NaN = single shot */
  const int32_t* stim_node_ptr;   /* [n+1] or NULL when n_stim == 0 */
  const int32_t* stim_ids;        /* entry ids per node, in protocol order */

  /* ---- probes / detector (SimulationSetup) */
  int n_probes;
  const int64_t* probes;
  double lat_threshold_mv;
  double map_interval_ms;

  /* ---- SchemeConfig (splitting.hpp:24-35) */
  int scheme;
  double dt_ms;
  double t_end_ms;
  int k0_up, k0_down;
  int strict_substeps;
  double record_interval_ms;

  /* ---- placement */
  int device;     /* CUDA ordinal */
  int rank, world;                 /* y-slab decomposition; world = 1 for single GPU */
  const unsigned char* nccl_id;    /* 128-byte ncclUniqueId (world > 1) */

  /* ---- appended (ABI: older callers that zero-initialise the struct are unaffected) */
  const cwg_sheet2d* sheet2d; /* for CWG_OP_SHEET2D (row_ptr/col/val/lumped_mass/dt_s ignored) */
} cwg_problem;

/* StrangIntegrator ctor (splitting.cpp:74-93): validates, uploads the operator,
 * stimulus tables and model lists, derives dt_eff, plan and k_max. */
int cwg_create(const cwg_problem* prob, cwg_ctx** out, cwg_error* err);
/* StrangIntegrator destructor (splitting.hpp:101-127): frees the device context. */
void cwg_destroy(cwg_ctx* ctx);

/* No reference counterpart (stream plumbing): use an external CUDA stream
 * (e.g. torch's current stream); NULL = own stream. cwg_stream returns it. */
int cwg_set_stream(cwg_ctx* ctx, void* cuda_stream);
void* cwg_stream(cwg_ctx* ctx);

/* make_initial_state (splitting.cpp:183-217) result upload / final_state
 * download. AoS host layout s[i*stride+q] (NodeStateArray::s); the device keeps
 * the states column-wise in groups of four (csrc/common.cuh sidx).
 * For world > 1 the arrays are the GLOBAL arrays; each rank copies its slab. */
int cwg_upload_state(cwg_ctx* ctx, const double* v, const double* s_aos, int stride,
                     const double* last_dvdt);
/* SimulationResult::final_state (splitting.cpp:292) / the state advance()
 * mutates in place (splitting.cpp:171-181): device SoA -> host AoS. */
int cwg_download_state(cwg_ctx* ctx, double* v, double* s_aos, int stride, double* last_dvdt);
/* make_initial_state (splitting.cpp:183-217) from the models' rest states
 * directly on the device (no host arrays; for 10^8-node slabs). last_dvdt = 0,
 * V = rest V. */
int cwg_init_rest_state(cwg_ctx* ctx);
/* Reconfigure the scheme of an existing context -- cli_compare
 * (runner.cpp:254-324) runs OST / OSTAR / DAETI on one prepared problem, so
 * the device-resident operator, stimulus, probes and model bins are kept
 * while dt_eff, l, dt_ad (and dt/m), k_max, n_steps and the record cadences
 * are recomputed exactly as by cwg_create; cached graphs are dropped.
 * Upload the initial state and call cwg_run_begin afterwards. */
int cwg_set_scheme(cwg_ctx* ctx, int scheme, double dt_ms, double t_end_ms, int k0_up, int k0_down,
                   int strict_substeps, cwg_error* err);
/* Testing hook for the multi-GPU decomposition on ONE device: contexts
 * created with world = N, rank r, no NCCL id and CWG_LOOPBACK=1 in the
 * environment skip the communicator; this call runs steps [first,
 * first+count) of all N ranks interleaved on rank 0's stream, copying the
 * one-row (2D) / one-plane (3D) halos between the ranks' V buffers before
 * every diffusion sub-step exactly where halo_exchange's ncclSend/ncclRecv
 * would. Everything but the transport (slab kernels, offsets, failure keys,
 * recording) runs as on N GPUs. Call cwg_run_begin on each rank first. */
int cwg_loopback_steps(cwg_ctx* const* ranks, int world, int64_t first, int64_t count);
/* No reference counterpart (testing hook of the peer-memory transport): link
 * loopback rank contexts the way NCCL ranks are linked over IPC at creation
 * (PeerLink: each diffusion launch stores the neighbours' halo rows into their
 * V buffers and paces itself on launch counters). cwg_loopback_steps then runs
 * the peer-memory data path instead of copying halos. */
int cwg_loopback_link(cwg_ctx* const* ranks, int world);

/* Asynchronous V snapshot for on_snapshot (splitting.cpp:267-277): enqueue,
 * after the steps issued so far, a device-side copy of V and of the failure
 * record, then their transfer to host_v[global node] on a side stream; the
 * solver stream continues with the next steps meanwhile. host_v must stay
 * valid until cwg_snapshot_wait returns (pinned or cwg_host_register-ed
 * memory makes the copy asynchronous). One snapshot in flight per context.
 * cwg_snapshot_wait blocks until host_v is complete; it returns
 * CWG_EINSTABILITY (err filled as by cwg_run_sync) when the run had already
 * failed at the snapshot point, so no snapshot later than the reference's
 * throw is ever delivered. (world > 1: synchronous, the failure agreement is
 * a collective.) */
int cwg_snapshot_begin(cwg_ctx* ctx, double* host_v);
/* Completes cwg_snapshot_begin (see above; splitting.cpp:276-277 delivery). */
int cwg_snapshot_wait(cwg_ctx* ctx, cwg_error* err);
/* No reference counterpart (host memory plumbing): cudaHostRegister /
 * cudaHostUnregister for caller-owned buffers (e.g. the std::vector handed
 * to on_snapshot). */
int cwg_host_register(void* p, size_t bytes);
int cwg_host_unregister(void* p);

/* No reference counterpart (host memory plumbing): pinned staging for
 * host<->device copies (e2e path); returns host pointers owned by ctx of the
 * sizes of the local slab. */
int cwg_pinned_buffers(cwg_ctx* ctx, double** v, double** s_aos, double** last_dvdt);

/* StrangIntegrator::advance (splitting.cpp:171-181): one outer step at t_ms.
 * Synchronous: returns CWG_EINSTABILITY with the reference's node/time. */
int cwg_advance(cwg_ctx* ctx, double t_ms, int64_t step_index, int64_t n_steps, cwg_error* err);

/* run_simulation (splitting.cpp:219-294) split into stream-ordered pieces:
 *   cwg_run_begin   records traces/maps at t = 0 and resets counters;
 *   cwg_run_steps   enqueues steps [first, first+count) incl. the record /
 *                   map cadence (CUDA-graph replay; no host sync);
 *   cwg_run_sync    waits and reports the first InstabilityError, if any.
 * cwg_run = begin + all steps + sync. */
int cwg_run_begin(cwg_ctx* ctx);
int cwg_run_steps(cwg_ctx* ctx, int64_t first, int64_t count);
int cwg_run_sync(cwg_ctx* ctx, cwg_error* err);
int cwg_run(cwg_ctx* ctx, cwg_error* err);

/* SimulationResult pieces (splitting.hpp:64-75) */
typedef struct {
  double dt_effective, dt_s, dt_ad;
  int l, k_max_global;
  int64_t n_steps, steps_per_record, steps_per_map, n_samples;
  int64_t n_local, node_begin; /* this rank's slab */
  int op_kind;                 /* resolved CWG_OP_* */
} cwg_info;
/* dt_effective / plan / k_max_global (splitting.hpp:108-110) and the
 * SimulationResult scalars (splitting.hpp:64-75) */
int cwg_get_info(cwg_ctx* ctx, cwg_info* info);
/* k_histogram (splitting.hpp:111): cumulative, index k */
int cwg_get_khist(cwg_ctx* ctx, int64_t* out, int len);
/* SimulationResult::traces (splitting.hpp:64-75; recorded at splitting.cpp:271-275) */
int cwg_get_traces(cwg_ctx* ctx, double* t_ms, double* v /* [probe][sample] */);
/* SimulationResult lat_map / apd90_map = ActivationDetector::lat / apd90
 * (postprocess.hpp:45-46, postprocess.cpp:68-90); this rank's slab */
int cwg_get_maps(cwg_ctx* ctx, double* lat, uint8_t* lat_valid, double* apd90, uint8_t* apd_valid);
/* The global SimulationResult::final_state (AoS, any stride >= the model
 * list's) and lat_map / apd90_map (splitting.cpp:286-293) on EVERY rank of a
 * y-slab run: each rank's owned slab is broadcast to all ranks over NCCL
 * (world > 1); world == 1: the plain download. Arrays are global-size;
 * any pointer may be NULL. Collective for world > 1 (call on all ranks). */
int cwg_gather_result(cwg_ctx* ctx, double* v, double* s_aos, int stride, double* last_dvdt, double* lat,
                      uint8_t* lat_valid, double* apd90, uint8_t* apd_valid);
/* No reference counterpart (runtime): return the device blocks cached by
 * destroyed contexts to CUDA (contexts reuse them for allocations of the
 * same size; at most 32 GiB is kept; CWG_POOL=0 disables caching). */
void cwg_trim_pool(void);
/* reaction / diffusion / recording device time (ms, CUDA events) of the last
 * cwg_advance calls (TimingBreakdown, splitting.hpp:57-62) */
int cwg_get_timing(cwg_ctx* ctx, double* reaction_ms, double* diffusion_ms, double* recording_ms);
/* No reference counterpart (measurement): kernel launches issued by this
 * context so far (for the bench's gpu_launches). */
int64_t cwg_launch_count(cwg_ctx* ctx);

/* Benchmark driver (bench.py; the role of the reference's BM_strang_step,
 * bench_core.cpp:70-75): enqueue steps [first, first+count) one at a
 * time, each preceded by an (untimed) write of flush_bytes to a scratch
 * buffer that evicts L2, and bracketed by CUDA events on the context stream.
 * split_phases = 0: each middle step is one single-step CUDA graph (the
 * production launch path), step_ms[i] = the step; split_phases = 1: direct
 * launches with an extra event between the reaction kernels (step A) and
 * the diffusion sub-steps + recording: react_ms[i], diff_ms[i];
 * split_phases = 2: the step graph without event nodes, events recorded on
 * the stream around its launch (react_ms[i] = the step, diff_ms[i] = the
 * cost of one more stream event record). */
int cwg_bench_steps(cwg_ctx* ctx, int64_t first, int64_t count, int64_t flush_bytes, int split_phases,
                    double* step_ms, double* react_ms, double* diff_ms);
/* Reaction node-updates (rates evaluations) so far = sum_k k * khist[k]
 * (the reference's k_histogram, splitting.hpp:111, weighted by k). */
int64_t cwg_reaction_evals(cwg_ctx* ctx);

/* No reference counterpart (diagnostics): with CWG_REACT_TRACE set in the
 * environment, every reaction launch stamps %globaltimer per block (slot 15:
 * block start, slot 0: the block's reaction done; 16 slots per block, at most
 * 4096 blocks, overwritten by the next launch). Copies the first n slots of
 * the last launch's stamps. Returns CWG_EVALIDATION when tracing is off. */
int cwg_react_trace(uint64_t* out, int n);

/* No reference counterpart (measurement): FP64 peak of this device, a
 * DFMA-chain kernel at full occupancy, CUDA-event timed. Returns TFLOP/s
 * (2 flops per DFMA) or < 0 on error. */
double cwg_fp64_peak_tflops(int device, double seconds);

/* pace_to_steady_state (ionic.cpp:122-165, ionic.hpp:74), batched: n
 * independent single cells of one model kind, request i paced with
 * cycle_ms[i] / amplitude[i] / duration_ms[i] for n_beats beats, forward Euler
 * at dt = stable_step / 2, one device thread per request. Outputs (host
 * buffers, any may be NULL): state_out [n][state_count+1] end-diastolic
 * [V, s...] of the final beat, apd90_out [n][n_beats] (NaN: no AP),
 * max_rel_out [n] (change between the last two end-diastolic states),
 * status_out [n] (CWG_OK / CWG_EINSTABILITY), fail_t_out [n].
 * Validation as the reference (n_beats >= 1, cycle > 0). Returns
 * CWG_EINSTABILITY, with err filled from the lowest failing request like the
 * reference's InstabilityError (node -1, t = beat * cycle + t_in_beat), when
 * any request diverged; the other requests' outputs are still written. */
int cwg_pace_cells(int model_kind, int64_t n, const double* cycle_ms, const double* amplitude,
                   const double* duration_ms, int n_beats, double* state_out, double* apd90_out,
                   double* max_rel_out, int* status_out, double* fail_t_out, int device, cwg_error* err);

/* ThresholdOptions (stimulus.hpp:60-67) */
typedef struct {
  double duration_ms;    /* 1.0 */
  double upper_factor;   /* 1000.0 */
  double initial_guess;  /* 1.0 mV/ms */
  double rel_tol;        /* 0.05 */
  double window_ms;      /* 50.0 */
  double dt_ms;          /* 0.05 */
} cwg_threshold_options;

/* diastolic_threshold (stimulus.cpp:115-157) on the device: bisection over
 * the amplitude of a single-shot stimulus on stim_nodes, each probe a fixed-
 * step monodomain run from rest (reaction with k = 1 at dt = min(opt.dt,
 * dt0/2, dt_s), then one diffusion sub-step of dt) that propagates when V at
 * the node farthest from the stimulus (>= 1 cm) exceeds 0 mV within the
 * window. prob supplies the 2D operator, ONE model and the device; its scheme
 * and stimulus fields are ignored. coords_xy: [n][2] node coordinates. */
int cwg_diastolic_threshold(const cwg_problem* prob, const double* coords_xy, const int64_t* stim_nodes,
                            int64_t n_stim, const cwg_threshold_options* opt, double* threshold,
                            int64_t* probe_node, cwg_error* err);

/* diffusion_substep (fem.cpp:194-207): standalone out = v - dt/m * K v on the
 * device, host in/out, bit-identical to the reference. */
int cwg_diffusion_substep(int64_t n, const int64_t* row_ptr, const int64_t* col, const double* val,
                          const double* lumped_mass, const double* v, double dt_sub, double* out,
                          int device, cwg_error* err);

/* CellModel::rates (ionic.hpp:33) batched on the device: v[n], s_aos[n*ns],
 * i_stim[n] -> dv[n], ds_aos[n*ns]. For tests and single-cell tooling. */
int cwg_rates(int model_kind, int64_t n, const double* v, const double* s_aos, const double* i_stim,
              double* dv, double* ds_aos, int device, cwg_error* err);

/* Model metadata: CellModel::state_count (ionic.hpp:23), stable_step
 * (ionic.hpp:28), rest_state (ionic.hpp:26) */
int cwg_model_state_count(int model_kind);
double cwg_model_stable_step(int model_kind);
int cwg_model_rest_state(int model_kind, double* out /* state_count+1 */);
int cwg_model_kind_from_name(const char* name); /* -1 if unknown (make_model, ionic.cpp:59) */

/* Adaptation rules (splitting.cpp:48-72), host-side, exported for parity tests */
int cwg_reaction_substeps(double dvdt_prev, int scheme, int k0_up, int k0_down, int k_max); /* splitting.cpp:48-54 */
int cwg_diffusion_substeps(double dt, double dt_s, int strict, int scheme, int* l, double* dt_ad); /* :56-67 */
int cwg_k_max_for(double dt, int model_kind);                                                /* :69-72 */

/* assemble (fem.cpp:112-176) + gershgorin_step (fem.cpp:178-192) of a
 * regular sheet on `device` (see cwg_sheet2d). Outputs may be NULL; CSR in
 * the reference's layout (ascending columns): row_ptr [n+1], col / val
 * [cwg_sheet2d_nnz], lumped_mass [n], dt_s. Validation failures carry the
 * reference's messages (first failing element / node, as its loops throw). */
int64_t cwg_sheet2d_nnz(const cwg_sheet2d* g);
int cwg_sheet2d_assemble(const cwg_sheet2d* g, int device, int64_t* row_ptr, int64_t* col, double* val,
                         double* lumped_mass, double* dt_s, cwg_error* err);

/* No reference counterpart (new: the reference is single-process OpenMP):
 * y-slab plan for world ranks over ny1 node rows,
 * [row_begin, row_end) owned rows, balanced by node count. No GPU needed. */
int cwg_slab_plan(int64_t ny1, int world, int rank, int64_t* row_begin, int64_t* row_end);

/* No reference counterpart: library version string. */
const char* cwg_version(void);
/* No reference counterpart (the reference throws): message of the last failed
 * call on this host thread ("" if none). */
const char* cwg_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* CWGPU_H */
