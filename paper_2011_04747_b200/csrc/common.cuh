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

// State layout: columns in groups of four, S[(q / 4) * 4 * pitch + 4 * i + (q & 3)] -- node i's states
// q .. q + 3 (q a multiple of 4) sit side by side, so a lane moves them with one 32-byte access (sm_100's
// LDG/STG.256) and a warp's 32 consecutive nodes with one contiguous 1 KB one: a quarter of the load/store
// instructions of one column per state.
constexpr int kStateGroup = 4;
__host__ __device__ __forceinline__ long long sidx(int q, long long i, long long pitch) {
  return static_cast<long long>(q >> 2) * 4 * pitch + 4 * i + (q & 3);
}
__device__ __forceinline__ void ld_state4(const double* p, double& a, double& b, double& c, double& d) {
  asm volatile("ld.global.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
}
__device__ __forceinline__ void st_state4(double* p, double a, double b, double c, double d) {
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d) : "memory");
}

struct ReactArgs {
  double* v;            // local V (current buffer)
  double* S;            // grouped-column states, S[sidx(q, i, pitch)]
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

// Peer-memory halo link of a y-slab rank (multi-GPU without NCCL on the data
// path): a diffusion launch stores the rows/planes its neighbours need straight
// into their V buffers over NVLink (IPC-mapped), and the ranks pace each other
// with launch counters: every halo-writing launch first waits until both
// neighbours completed as many such launches as this rank (their data for it
// is in place and they no longer read the buffers it is about to write), and
// its last block publishes the new count into the neighbours' memory
// (release/acquire at system scope). Loopback contexts on one device link the
// same way (cwg_loopback_link), which is how the data path is tested.
struct PeerLink {
  int on = 0;
  long long w = 0;     // nodes per row / plane
  long long rows = 0;  // owned rows / planes
  // this rank's owned row r (0-based) -> lo_dst[p][r*w + x] (neighbour rank-1's upper halo rows) for
  // rows r < H; row rows-j -> hi_dst[p][-j*w + x] (rank+1's lower halo) for j <= H; p = buffer parity
  double* lo_dst[2] = {nullptr, nullptr};
  double* hi_dst[2] = {nullptr, nullptr};
  unsigned long long* wait_lo = nullptr;  // local: launches completed by rank-1 (written by it)
  unsigned long long* wait_hi = nullptr;  // local: launches completed by rank+1
  unsigned long long* post_lo = nullptr;  // remote: rank-1's wait_hi
  unsigned long long* post_hi = nullptr;  // remote: rank+1's wait_lo
  unsigned long long* count = nullptr;    // local: halo-writing launches this rank completed
  unsigned* blocks_done = nullptr;        // local: block arrivals of the running launch
  long long lim = 1;                      // halo rows a neighbour keeps (2D: hrows_v; 3D: one plane)
};

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Block entry of a halo-writing launch: wait for the neighbours (bounded; a
// neighbour that never arrives traps instead of hanging the device).
__device__ __forceinline__ void peer_wait(const PeerLink& pl) {
  if (!pl.on) return;
  if (threadIdx.x == 0) {
    const unsigned long long need = *reinterpret_cast<volatile unsigned long long*>(pl.count);
    for (long long it = 0;; ++it) {
      const bool lo = !pl.wait_lo || ld_acquire_sys(pl.wait_lo) >= need;
      const bool hi = !pl.wait_hi || ld_acquire_sys(pl.wait_hi) >= need;
      if (lo && hi) break;
      if (it > (1ll << 28)) __trap();  // minutes: a rank is gone (trap instead of hanging the device)
      __nanosleep(64);
    }
    asm volatile("fence.proxy.async.global;" ::: "memory");  // the peers' stores before our bulk copies
  }
  __syncthreads();
}

// Block exit: after this block's peer stores; the last block publishes the count.
__device__ __forceinline__ void peer_post(const PeerLink& pl) {
  if (!pl.on) return;
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned prev;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(pl.blocks_done) : "memory");
    if (prev == gridDim.x * gridDim.y * gridDim.z - 1) {  // (the fused 2D kernel has a 2D grid)
      *pl.blocks_done = 0u;
      const unsigned long long n = *pl.count + 1;
      *pl.count = n;
      __threadfence_system();
      if (pl.post_lo) st_release_sys(pl.post_lo, n);
      if (pl.post_hi) st_release_sys(pl.post_hi, n);
    }
  }
}

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
  PeerLink pl;      // peer-memory halo stores (multi-GPU P2P transport), off by default
  int out_par = 0;  // parity (index in the context's V pair) of vout
};

// this rank's output value of owned row `r`, column offset `xo` (within the row / plane) to the
// neighbours that keep it as a halo row: rows r < lim go down, rows r >= rows - lim go up
__device__ __forceinline__ void peer_store(const DiffArgs& a, long long r, long long xo, double val) {
  const PeerLink& pl = a.pl;
  if (!pl.on) return;
  if (r < pl.lim && pl.lo_dst[a.out_par]) pl.lo_dst[a.out_par][r * pl.w + xo] = val;
  if (r >= pl.rows - pl.lim && pl.hi_dst[a.out_par]) pl.hi_dst[a.out_par][(r - pl.rows) * pl.w + xo] = val;
}

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
