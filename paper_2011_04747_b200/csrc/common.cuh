// Shared device-side definitions of the cwgpu kernels (sm_100a).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace cwg {

constexpr unsigned kFull = 0xffffffffu;
constexpr unsigned long long kNoError = ~0ull;
constexpr long long kNoSeq = 0x7fffffffffffffffll;  // ErrRec::seq before any failure
// doubles of slack after every V buffer: the 3D diffusion kernel's 16-byte
// aligned row copies may run up to 2 nodes past a row (diffuse.cu S3R_COPY)
constexpr long long kVPad = 128;

// Error record, one per context. key = node << 22 | k << 11 | j (reaction) or
// node << 22 (diffusion); atomicMin gives the reference's "lowest node"
// (splitting.cpp:129-140, :162-166). seq = program-order event id of the
// first failing event (atomicMin, kNoSeq before any failure); kernels of
// later events skip their work so the state stays exactly where the
// reference would have thrown.
// The failing launch also records its V buffers and fused depth T, so the
// host can put V exactly where the reference stops (later events skip their
// work without writing): the reaction's in-place V, a diffusion launch's
// output, or -- for a launch that fused T sub-steps and failed in sub-step
// q < T-1 -- a replay of q+1 sub-steps from its (untouched) input.
struct ErrRec {
  unsigned long long key;
  long long seq;
  int phase;  // 1 reaction, 2 diffusion
  int T;      // sub-steps fused by the failing launch (1: unfused / reaction)
  const double* vin;
  double* vout;
};

// Flattened ProtocolIndex (stimulus.hpp:35-50)
struct StimDev {
  const int32_t* node_ptr;  // local node -> [begin, end) into ids; nullptr when no stimulus
  const int32_t* ids;
  const double* t0;
  const double* dur;
  const double* amp;
  const double* per;  // NaN: single shot
};

// ProtocolIndex::current (stimulus.cpp:33-45), same comparisons and fmod.
__device__ __forceinline__ double stim_current(const StimDev& st, int p0, int p1, double t) {
  double sum = 0.0;
  for (int q = p0; q < p1; ++q) {
    const int e = __ldg(st.ids + q);
    const double t0 = __ldg(st.t0 + e);
    if (t < t0) continue;
    const double per = __ldg(st.per + e);
    if (per == per) {  // periodic
      if (fmod(__dsub_rn(t, t0), per) < __ldg(st.dur + e)) sum = __dadd_rn(sum, __ldg(st.amp + e));
    } else if (t < __dadd_rn(t0, __ldg(st.dur + e))) {
      sum = __dadd_rn(sum, __ldg(st.amp + e));
    }
  }
  return sum;
}

// reaction_substeps (splitting.cpp:48-54)
__device__ __forceinline__ int substeps(double dvdt, int scheme, int k0_up, int k0_down, int kmax) {
  if (scheme == 0) return 1;  // OST
  const int k0 = dvdt > 0.0 ? k0_up : k0_down;
  const double raw = __dadd_rn(static_cast<double>(k0), floor(fabs(dvdt)));
  const int k = raw > static_cast<double>(kmax) ? kmax : static_cast<int>(raw);
  return k < 1 ? 1 : k;
}

// Exact forward-Euler update x + h*d (no contraction: splitting.cpp:126-127).
__device__ __forceinline__ double fe(double x, double h, double d) {
  return __dadd_rn(x, __dmul_rn(h, d));
}

struct ReactArgs {
  double* v;            // local V (current buffer)
  double* S;            // SoA states, S[q*pitch + i]
  long long pitch;
  double* last;         // last_dvdt
  const int32_t* list;  // position -> local node (nullptr: dense range)
  long long first;      // dense range start
  long long count;      // positions
  StimDev stim;
  const double* gkr;    // per-node GKr scale or nullptr
  double dt;            // dt_eff
  double t_fixed;       // caller-supplied t (StrangIntegrator::advance) when use_t_fixed
  int use_t_fixed;
  const long long* clock;  // device step base
  long long step_off;      // step = *clock + step_off
  int scheme, k0_up, k0_down, kmax;
  unsigned long long* khist;  // [kmax_global + 1]
  int khist_len;
  ErrRec* err;
  long long evs;        // events per step (seq = step*evs + ev)
  int ev;
  unsigned int* counter;  // work counter (self-resetting)
  unsigned int* done;     // finished-block counter (self-resetting)
  long long node_offset;  // local -> global node index
  unsigned long long* trace;  // diagnostics (CWG_REACT_TRACE): per block 16 globaltimer slots, or nullptr
  int preclaim;         // claim a finishing lane's next node one trip ahead (react.cuh)
};

struct DiffArgs {
  const double* vin;
  double* vout;
  long long n;  // local rows (owned)
  long long halo;  // owned row 0 is at vin[halo] (multi-GPU y-slab halo)
  double dt_sub;
  ErrRec* err;
  const long long* clock;
  long long step_off;
  long long evs;
  int ev;
  long long node_offset;
};

__device__ __forceinline__ long long cur_seq(const long long* clock, long long step_off, long long evs,
                                             int ev) {
  return (*clock + step_off) * evs + ev;
}

// True when a STRICTLY earlier event already failed: skip the work (state
// frozen at the throw). Only seq decides: a failure of the current event
// (written concurrently by this launch) carries seq == the current seq and
// never makes a block skip, so every block of a launch agrees (an earlier
// event's record was complete at its kernel boundary).
// err == nullptr: an unchecked launch (diastolic_threshold probe runs, whose
// diffusion has no NaN scan, stimulus.cpp:106) -- never skips, never records.
__device__ __forceinline__ bool earlier_failure(const ErrRec* err, long long seq) {
  if (!err) return false;
  const volatile ErrRec* e = err;
  return e->seq < seq;
}

__device__ __forceinline__ void record_failure(ErrRec* err, unsigned long long key, long long seq, int phase,
                                               int T, const double* vin, double* vout) {
  if (!err) return;
  atomicMin(reinterpret_cast<unsigned long long*>(&err->seq), static_cast<unsigned long long>(seq));  // seq >= 0
  atomicMin(&err->key, key);
  // all failing threads of this event write the same values
  err->phase = phase;
  err->T = T;
  err->vin = vin;
  err->vout = vout;
}

struct Stencil2D {
  const double* coef;
  long long cpitch;
  const double* cm;
  long long w;          // nodes per row
  long long rows;       // owned rows
  long long row_begin;  // global index of owned row 0
  long long ny1;        // global rows
  // Local layouts: V has hrows_v halo rows each side of the owned rows (owned
  // row r at (r + hrows_v) * w); coef / cm cover hrows_c rows each side (owned
  // row r at (r + hrows_c) * w). One GPU: 1 / 0. Multi-rank fused diffusion:
  // H / H, so halo points can be advanced through the fused sub-steps.
  long long hrows_v = 1;
  long long hrows_c = 0;
};

// Structured 3D slab (EXTENSION): per-class 27-point coefficients
struct Struct3D {
  const double* coef;  // [n_classes][27]
  const double* cm;    // [n_classes] dt_sub / m
  long long nx1, nz1, plane;  // plane = nx1 * nz1 nodes per y-plane
  long long planes;           // owned y-planes
  long long row_begin;        // global y of owned plane 0
  long long ny1;
  int ychunk = 16;            // y-planes marched per block (launch_diffuse_struct3d)
};

struct CsrDev {
  const long long* row_ptr;
  const long long* col;
  const double* val;
  const double* cm;
};

struct DetDev {
  double *prev_v, *v_rest, *max_slope, *t_max_slope, *v_peak, *lat, *apd;
  unsigned char *phase, *has_lat, *has_apd;
  double threshold;
};

// single-cell pacing batch (react.cuh: pace_kernel)
struct PaceArgs {
  long long n;
  int n_beats;
  double dt;
  const double* cycle;
  const double* amp;
  const double* dur;
  const double* rest;  // [NS + 1]: V, states
  double* state_out;   // [n][NS + 1]
  double* apd_out;     // [n][n_beats]
  double* prev_out;    // [n][NS + 1] scratch: end-diastolic state of beat n_beats - 2
  double* maxrel_out;  // [n]
  int* status_out;     // [n]: 0 ok, 2 non-finite V, 3 |V| > 1000 mV
  int* beat_out;       // [n]: failing beat
  double* fail_t_out;  // [n]: beat * cycle + t_in_beat at the failure
};

}  // namespace cwg
