// Host runtime of the cwgpu C ABI (include/cwgpu.h): device-resident solver
// context, state upload/download, the DAETI step sequence
// (StrangIntegrator::advance, splitting.cpp:171-181) and run_simulation's
// outer loop with its record cadence (splitting.cpp:219-294), replayed as
// CUDA graphs; y-slab halo exchange over NCCL for world > 1.
#include <dlfcn.h>
#include <cuda.h>
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <chrono>
#include <map>
#include <mutex>
#include <unordered_map>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/cwgpu.h"
#include "../../include/cwgpu_setup.h"
#include "launch.h"

using namespace cwg;

namespace {

// ------------------------------------------------------------------ errors
struct Fail {
  int code;
  std::string msg;
};

void set_error(cwg_error* e, int code, const std::string& msg) {
  if (!e) return;
  e->code = code;
  e->node = -1;
  e->t_ms = 0.0;
  e->phase = 0;
  std::snprintf(e->msg, sizeof(e->msg), "%s", msg.c_str());
}

#define CUDA_TRY(x)                                                                              \
  do {                                                                                           \
    cudaError_t _e = (x);                                                                        \
    if (_e != cudaSuccess)                                                                       \
      throw Fail{CWG_ECUDA, std::string("CUDA error: ") + cudaGetErrorString(_e) + " at " #x};  \
  } while (0)

void validation(bool ok, const std::string& msg) {
  if (!ok) throw Fail{CWG_EVALIDATION, msg};
}

// ------------------------------------------------------------------ models
int state_count(int kind) {
  switch (kind) {
    case CWG_MODEL_ALIEV_PANFILOV: return 1;
    case CWG_MODEL_ORD_ENDO:
    case CWG_MODEL_ORD_EPI:
    case CWG_MODEL_ORD_MID: return 40;
    case CWG_MODEL_MACCANNELL: return 2;
    case CWG_MODEL_PASSIVE: return 0;
    default: return -1;
  }
}

double stable_step(int kind) {
  switch (kind) {
    case CWG_MODEL_ALIEV_PANFILOV: return 1.0;
    case CWG_MODEL_MACCANNELL: return 0.1;
    case CWG_MODEL_PASSIVE: return 1.0;
    default: return 0.01;
  }
}

bool is_ord(int kind) { return kind >= CWG_MODEL_ORD_ENDO && kind <= CWG_MODEL_ORD_MID; }

// k_max_for (splitting.cpp:69-72)
int kmax_for(double dt, int kind) {
  const int k = static_cast<int>(std::floor(dt / stable_step(kind)));
  return k < 1 ? 1 : k;
}

long long llround_ref(double x) { return std::llround(x); }

// Published quiescent states [V, s...] of the ORd variants (model constants,
// ohara_rudy_2011.cpp:454-489), state order of StateIndex.
const double kOrdRest[3][41] = {
    {-88.069987424096993, 6.7857694543304437, 6.7858240866305497, 145.2270611623554,
     145.22703970422316, 6.6496500901714538e-05, 6.5363220572944042e-05, 1.1773572696330052,
     1.1780931136267005, 0.0072940079209426727, 0.7004598461826681, 0.70045979343293074,
     0.70045953530570237, 0.45778977781006114, 0.70045939195427553, 0.0001858428745214649,
     0.51535061430259566, 0.31721806727437052, 0.0009965088352518912, 0.99955951365975104,
     0.99955949399976396, 0.00050774700555622921, 0.99955951368195861, 0.99955949654005649,
     2.3033854222194026e-09, 0.99999999104293114, 0.99999999105447779, 0.99999999104293658,
     0.99999999104087156, 0.99999999104142678, 0.0010021110565670483, 0.99999999104268988,
     0.99999999104270343, 7.9332827982721131e-06, 7.9336066064785696e-06,
     0.00019132437263296958, 0.00019132414231280508, 0.99674141905341751,
     5.4200685188624244e-08, 6.7752012471923812e-08, 0.0003810650518518126},
    {-88.029323128607928, 6.7962192631889486, 6.7962623821225367, 145.20458892004748,
     145.20456959400204, 5.4852819578522002e-05, 5.4064603199250324e-05, 1.2563944307309074,
     1.2563851562790889, 0.0073238975664768622, 0.69905606284853461, 0.69905600543119961,
     0.69905572480467026, 0.45613173681108238, 0.69905556898249277, 0.00018728379656753348,
     0.51399396544560239, 0.3160425988040147, 0.00099924415555908345, 0.99955636760901723,
     0.99955636599890663, 0.00050914140569242004, 0.99955636761083866, 0.99955636620603716,
     2.3256353623298777e-09, 0.99999999094384107, 0.99999999095528003, 0.99999999094384651,
     0.99999999094178149, 0.99999999094233671, 0.00047971941613231592, 0.9999999909435997,
     0.99999999094361336, 7.9809446184557774e-06, 7.9812954631181394e-06,
     0.00019219809297998605, 0.00019219700739629426, 0.99675215233995673,
     1.0117197919343792e-07, 1.2646498743342686e-07, 0.00025496603469158611},
    {-87.918787307816828, 6.8844140619690002, 6.8844676613520441, 145.13903811434193,
     145.13902449899223, 6.3130680404950644e-05, 6.1753113171964479e-05, 1.1286605779696908,
     1.129987340810549, 0.00740576098250912, 0.69522137580095822, 0.69522116072571494,
     0.69522011165021347, 0.45162926254354163, 0.69521952838802525, 0.00019125728633946081,
     0.51029968338090503, 0.31284466603507399, 0.0010067174531280458, 0.99954770073199861,
     0.99954761833889205, 0.00051295113113861634, 0.99954770082322897, 0.99954762898761162,
     2.3872087752034307e-09, 0.99999999066891365, 0.99999999064687006, 0.99999999066891909,
     0.99999999066685408, 0.9999999906674093, 0.00080416517322784442, 0.99999999066867218,
     0.99999999066868595, 8.1119973876114768e-06, 8.1133560675743664e-06,
     0.00019463394428381671, 0.00019459031922160661, 0.99678115341920093,
     1.7708324928868821e-07, 2.2136126205224297e-07, 0.00034040551198936118}};


// ------------------------------------------------------------------ NCCL (dlopen'ed)
struct Nccl {
  void* h = nullptr;
  decltype(&ncclCommInitRank) init = nullptr;
  decltype(&ncclCommDestroy) destroy = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclGroupStart) gstart = nullptr;
  decltype(&ncclGroupEnd) gend = nullptr;
  decltype(&ncclAllReduce) allreduce = nullptr;
  decltype(&ncclBroadcast) bcast = nullptr;
  decltype(&ncclAllGather) allgather = nullptr;
  decltype(&ncclGetErrorString) errstr = nullptr;
  bool load() {
    if (h) return true;
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* nm : names)
      if ((h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL))) break;
    if (!h) return false;
    init = reinterpret_cast<decltype(init)>(dlsym(h, "ncclCommInitRank"));
    destroy = reinterpret_cast<decltype(destroy)>(dlsym(h, "ncclCommDestroy"));
    send = reinterpret_cast<decltype(send)>(dlsym(h, "ncclSend"));
    recv = reinterpret_cast<decltype(recv)>(dlsym(h, "ncclRecv"));
    gstart = reinterpret_cast<decltype(gstart)>(dlsym(h, "ncclGroupStart"));
    gend = reinterpret_cast<decltype(gend)>(dlsym(h, "ncclGroupEnd"));
    allreduce = reinterpret_cast<decltype(allreduce)>(dlsym(h, "ncclAllReduce"));
    errstr = reinterpret_cast<decltype(errstr)>(dlsym(h, "ncclGetErrorString"));
    bcast = reinterpret_cast<decltype(bcast)>(dlsym(h, "ncclBroadcast"));
    allgather = reinterpret_cast<decltype(allgather)>(dlsym(h, "ncclAllGather"));
    return init && destroy && send && recv && gstart && gend && allreduce && errstr && bcast && allgather;
  }
};
Nccl g_nccl;

#define NCCL_TRY(x)                                                                                     \
  do {                                                                                                  \
    ncclResult_t _r = (x);                                                                              \
    if (_r != ncclSuccess) throw Fail{CWG_ECUDA, std::string("NCCL error: ") + g_nccl.errstr(_r)};    \
  } while (0)

// Caching device allocator. A run_simulation-style caller builds a context
// per run (the reference's run_simulation constructs its StrangIntegrator);
// at C4 that is ~1.5 GB in a dozen cudaMallocs, 20-60 ms per context
// (tools/e2e_phases.py). Freed blocks are kept per (device, rounded size) and
// handed to the next allocation of that size; cwg_trim_pool() returns them.
// Contexts synchronise their streams before freeing (ctx_free), since
// reusing a block skips cudaFree's implicit device synchronisation.
// CWG_POOL=0 disables caching.
struct DevPool {
  std::mutex mu;
  std::multimap<std::pair<int, size_t>, void*> free_blocks;
  std::unordered_map<void*, std::pair<int, size_t>> live;
  size_t cached = 0;
  static constexpr size_t kCap = 32ull << 30;  // at most 32 GiB kept
  bool on = [] {
    const char* e = getenv("CWG_POOL");
    return !(e && e[0] == '0');
  }();
  static size_t round(size_t b) {
    return b >= (1u << 20) ? (b + (2u << 20) - 1) / (2u << 20) * (2u << 20) : (b + 255) / 256 * 256;
  }
  void* get(size_t bytes) {
    int dev = 0;
    cudaGetDevice(&dev);
    const size_t rb = round(bytes);
    {
      std::lock_guard<std::mutex> g(mu);
      auto it = free_blocks.find({dev, rb});
      if (it != free_blocks.end()) {
        void* p = it->second;
        free_blocks.erase(it);
        cached -= rb;
        live[p] = {dev, rb};
        return p;
      }
    }
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, rb);
    if (e != cudaSuccess && cached > 0) {  // device full: release the cache and retry once
      cudaGetLastError();
      trim();
      e = cudaMalloc(&p, rb);
    }
    CUDA_TRY(e);
    std::lock_guard<std::mutex> g(mu);
    live[p] = {dev, rb};
    return p;
  }
  void put(void* p) {
    std::unique_lock<std::mutex> g(mu);
    auto it = live.find(p);
    if (it == live.end()) {  // not ours (never happens) -- plain free
      g.unlock();
      cudaFree(p);
      return;
    }
    const auto key = it->second;
    live.erase(it);
    if (on && cached + key.second <= kCap) {
      free_blocks.insert({key, p});
      cached += key.second;
      return;
    }
    g.unlock();
    cudaFree(p);
  }
  void trim() {
    std::vector<void*> v;
    {
      std::lock_guard<std::mutex> g(mu);
      for (auto& kv : free_blocks) v.push_back(kv.second);
      free_blocks.clear();
      cached = 0;
    }
    for (void* p : v) cudaFree(p);
  }
};
DevPool& dev_pool() {
  static DevPool* pool = new DevPool();  // never destroyed: no cudaFree after the driver shuts down
  return *pool;
}

template <class T>
T* dev_alloc(size_t count) {
  if (count == 0) count = 1;
  return static_cast<T*>(dev_pool().get(count * sizeof(T)));
}

template <class T>
void dev_free(T*& p) {
  if (p) dev_pool().put(p);
  p = nullptr;
}

}  // namespace

// ====================================================================== ctx
struct Bin {
  int model = 0, kind = 0;
  int variant = 0;  // ORd launch shape (react_ord.cu ModelOrd)
  int32_t* d_list = nullptr;  // nullptr: dense [first, first+count)
  long long first = 0, count = 0;
  int grid = 1;
  unsigned* d_counter = nullptr;  // [0] counter, [1] done
  unsigned* d_counter_b = nullptr;  // boundary-first split (y-slab runs): [0..1] lower rows, [2..3] upper rows
  int variant_b = 0, grid_b = 1;   // launch shape of the edge-row ranges
};

struct cwg_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int num_sms = 148;

  // problem geometry
  long long n_global = 0, w = 0, ny1 = 0;
  int op_kind = CWG_OP_CSR;
  int rank = 0, world = 1;
  long long row_begin = 0, row_end = 0;  // owned rows (stencil / slab)
  long long n_own = 0, halo = 0, n_alloc = 0;
  int hrows_v = 1, hrows_c = 0;  // 2D: halo rows of V / of the coefficient arrays per side (Stencil2D)
  long long n_coef = 0;          // 2D: nodes covered by coef / cm ((rows + 2 hrows_c) * w)
  long long node_offset = 0;  // global index of local index 0
  long long own_global0 = 0;  // global index of the first owned node

  // scheme
  int scheme = CWG_DAETI;
  double dt = 0.1, dt_s = 0, t_end = 0, dt_eff = 0, dt_ad = 0;
  int l = 1, k0_up = 5, k0_down = 1, strict = 0;
  double record_interval = 1.0, map_interval = 1.0;
  long long n_steps = 0, spr = 1, spm = 1, evs = 3;
  int kmax_global = 1, stride = 1;
  std::vector<int> model_kind, kmax_of_model;

  // device state
  double* d_v[2] = {nullptr, nullptr};
  int cur = 0;
  double* d_S = nullptr;
  long long pitch = 0;
  double* d_last = nullptr;
  double* d_gkr = nullptr;

  // operator
  long long s3_nx1 = 0, s3_nz1 = 0;  // struct3d
  double* d_coef = nullptr;  // stencil: [9][n_own]; struct3d: [classes][27]
  double* d_cm = nullptr;    // dt_ad / m_i
  // padded coefficient tensor for the TMA diffusion kernel (2D, one device):
  // [10][rows][w_pad], planes 0..8 = coef, 9 = dt/m; tensor maps for T = 2..4
  double* d_coefp = nullptr;
  long long w_pad = 0;
  CUtensorMap tmap[7];  // TMA diffusion: one map per fused depth T = 2..6
  bool tma_ok = false;
  double* d_mass = nullptr;  // lumped mass: owned rows (2D / CSR) or node classes (3D)
  long long n_mass = 0;
  long long* d_rp = nullptr;
  long long* d_col = nullptr;
  double* d_val = nullptr;

  // stimulus
  int32_t* d_stim_ptr = nullptr;
  int32_t* d_stim_ids = nullptr;
  double *d_st0 = nullptr, *d_sdur = nullptr, *d_samp = nullptr, *d_sper = nullptr;

  std::vector<Bin> bins;

  // bookkeeping
  ErrRec* d_err = nullptr;
  long long* d_clock = nullptr;
  unsigned long long* d_khist = nullptr;
  int khist_len = 2;

  // recording
  DetDev det{};
  double lat_threshold = 0.0;
  int n_probes = 0;
  long long* d_probe_loc = nullptr;
  double* d_traces = nullptr;
  long long n_samples = 0;
  bool det_initialised = false;

  // graphs
  long long G = 0;
  // one G-step graph per starting V-buffer parity (a block may flip it when
  // fused diffusion launches make the per-step launch count odd)
  cudaGraphExec_t graph_p[2] = {nullptr, nullptr};
  int graph_cur_after[2] = {0, 0};
  bool graph_built = false;
  long long graph_base_mod = 0;
  long long graph_launches = 0;
  long long clock_at = -1;  // host knowledge of *d_clock, -1 unknown
  long long restored_seq = -1;  // failure whose state restore_failed_state already put in place

  // multi-GPU
  // boundary-first reaction (world > 1, dense model bins): the split_rows owned
  // rows/planes at each slab edge -- what the neighbours' first diffusion
  // launch needs -- run as launches of their own (on `side` under NCCL, so the
  // halo exchange overlaps the interior reaction on the solver stream)
  bool split = false;
  long long split_rows = 0;
  // peer-memory halo transport (default for NCCL y-slab runs whose neighbours are peer-accessible, and for
  // linked loopback contexts): diffusion launches store the neighbours' halo rows themselves (PeerLink)
  bool p2p = false;
  bool halo_fresh = false;  // the last enqueued V writer already pushed the current halos (capture-time state)
  PeerLink pl;
  unsigned long long* d_flags = nullptr;  // [0] wait_lo, [1] wait_hi, [2] count, [3] blocks_done
  std::vector<void*> ipc_opened;
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  ncclComm_t comm = nullptr;
  bool loopback = false;  // world > 1 without NCCL: halos copied by cwg_loopback_steps (testing hook)

  // asynchronous V snapshots (cwg_snapshot_begin / _wait)
  double* d_snap = nullptr;
  ErrRec* d_snap_err = nullptr;
  ErrRec* h_snap_err = nullptr;  // pinned
  cudaStream_t snap_stream = nullptr;
  cudaEvent_t ev_vready = nullptr, ev_snapdone = nullptr;
  bool snap_pending = false;

  // stats / timing
  long long launches = 0;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  double t_react = 0, t_diff = 0, t_rec = 0;

  // fixed-step mode (diastolic_threshold probe runs, stimulus.cpp:76-111):
  // reaction (k = 1) then ONE diffusion sub-step of dt, no NaN check after diffusion
  bool fixed_step = false;
  ErrRec* d_err_dummy = nullptr;
  long long* d_cross = nullptr;
  long long probe_local = -1;

  // bench
  void* d_flush = nullptr;
  size_t flush_bytes = 0;

  // pinned staging
  double *h_v = nullptr, *h_s = nullptr, *h_last = nullptr;
  double* d_stage = nullptr;
  long long stage_nodes = 0;  // nodes per staging chunk at the current caller stride
  long long stage_cap = 0;    // doubles allocated in d_stage
};

namespace {

void ctx_free(cwg_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  // pooled blocks may be handed out again at once: no kernel of this context may still use them
  if (c->stream) cudaStreamSynchronize(c->stream);
  if (c->snap_stream) cudaStreamSynchronize(c->snap_stream);
  for (auto& gx : c->graph_p)
    if (gx) cudaGraphExecDestroy(gx);
  for (auto& b : c->bins) {
    dev_free(b.d_list);
    dev_free(b.d_counter);
    dev_free(b.d_counter_b);
  }
  for (void* p : c->ipc_opened) cudaIpcCloseMemHandle(p);
  c->ipc_opened.clear();
  dev_free(c->d_flags);
  if (c->side) cudaStreamSynchronize(c->side);
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  if (c->side) cudaStreamDestroy(c->side);
  dev_free(c->d_v[0]);
  dev_free(c->d_v[1]);
  dev_free(c->d_S);
  dev_free(c->d_last);
  dev_free(c->d_gkr);
  dev_free(c->d_coef);
  dev_free(c->d_cm);
  dev_free(c->d_mass);
  dev_free(c->d_coefp);
  dev_free(c->d_rp);
  dev_free(c->d_col);
  dev_free(c->d_val);
  dev_free(c->d_stim_ptr);
  dev_free(c->d_stim_ids);
  dev_free(c->d_st0);
  dev_free(c->d_sdur);
  dev_free(c->d_samp);
  dev_free(c->d_sper);
  dev_free(c->d_err);
  dev_free(c->d_clock);
  dev_free(c->d_khist);
  dev_free(c->d_probe_loc);
  dev_free(c->d_traces);
  dev_free(c->d_stage);
  dev_free(c->d_err_dummy);
  dev_free(c->d_cross);
  if (c->d_flush) cudaFree(c->d_flush);
  double** dd[] = {&c->det.prev_v, &c->det.v_rest, &c->det.max_slope, &c->det.t_max_slope, &c->det.v_peak,
                   &c->det.lat, &c->det.apd};
  for (auto p : dd) dev_free(*p);
  dev_free(c->det.phase);
  dev_free(c->det.has_lat);
  dev_free(c->det.has_apd);
  if (c->h_v) cudaFreeHost(c->h_v);
  if (c->h_s) cudaFreeHost(c->h_s);
  if (c->h_last) cudaFreeHost(c->h_last);
  if (c->snap_pending && c->ev_snapdone) cudaEventSynchronize(c->ev_snapdone);
  dev_free(c->d_snap);
  dev_free(c->d_snap_err);
  if (c->h_snap_err) cudaFreeHost(c->h_snap_err);
  if (c->ev_vready) cudaEventDestroy(c->ev_vready);
  if (c->ev_snapdone) cudaEventDestroy(c->ev_snapdone);
  if (c->snap_stream) cudaStreamDestroy(c->snap_stream);
  for (auto& e : c->ev)
    if (e) cudaEventDestroy(e);
  if (c->comm && g_nccl.destroy) g_nccl.destroy(c->comm);
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

// Host -> device copy that has LANDED on return. cudaMemcpy from pageable
// memory returns once the data sits in the driver's staging buffer, with the
// DMA still queued on the legacy stream; the contexts' streams are
// non-blocking, so a kernel on them could otherwise read the old contents
// (seen: a 13 MB stimulus-pointer upload racing the kernel that rebases it).
void h2d(void* d, const void* h, size_t bytes) {
  if (!bytes) return;
  CUDA_TRY(cudaMemcpy(d, h, bytes, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaStreamSynchronize(nullptr));
}

template <class T>
T* upload(const T* h, size_t count) {
  T* d = dev_alloc<T>(count);
  h2d(d, h, count * sizeof(T));
  return d;
}

// Frees the temporary device buffers of a one-shot entry point on every exit
// path, including a CUDA_TRY / validation throw half-way through.
struct DevScope {
  std::vector<void*> ptrs;
  template <class T>
  T* keep(T* p) {
    ptrs.push_back(p);
    return p;
  }
  ~DevScope() {
    for (void* p : ptrs)
      if (p) dev_pool().put(p);
  }
};

// ------------------------------------------------- device sheet assembly
// A regular sheet's operator assembled on the device (assemble.cu): the full
// [9][n] stencil table, lumped mass and dt_s. Validation failures are
// reported like the reference's loops throw them: the first degenerate
// element (fem.cpp:84-86), then the first node failing the structural checks
// in the reference's order (mass, symmetry per entry, row sum; fem.cpp:154-172),
// then the first non-diffusive row (fem.cpp:184-187).
struct SheetAsm {
  double* coef = nullptr;  // [9][n] (pool memory; owner frees)
  double* mass = nullptr;  // [n]
  unsigned char* nnz_row = nullptr;
  long long n = 0, w = 0;
  double dt_s = 0.0;
  void release() {
    dev_free(coef);
    dev_free(mass);
    dev_free(nnz_row);
  }
};

SheetAsm assemble_sheet2d(const cwg_sheet2d* g, cudaStream_t st) {
  validation(g != nullptr, "operator: CWG_OP_SHEET2D needs cwg_problem.sheet2d");
  validation(g->h > 0.0 && std::isfinite(g->h), "mesh: spacing h must be positive and finite");
  validation(g->nx >= 1 && g->ny >= 1, "mesh: the sheet needs at least one element per axis");
  validation(g->d0_myocyte > 0.0 && g->d0_fibrotic > 0.0, "diffusion: coefficients must be positive");
  validation(g->rho > 0.0 && g->rho <= 1.0, "diffusion: rho must lie in (0, 1]");
  SheetAsm a;
  a.w = g->nx + 1;
  a.n = a.w * (g->ny + 1);
  validation(a.n < (1ll << 40), "mesh: at most 2^40 nodes");
  DevScope tmp;
  const int32_t* dtags = g->node_tags ? tmp.keep(upload(g->node_tags, static_cast<size_t>(a.n))) : nullptr;
  const double* desc = g->elem_scale ? tmp.keep(upload(g->elem_scale, static_cast<size_t>(g->nx * g->ny))) : nullptr;
  unsigned long long* dkeys = tmp.keep(dev_alloc<unsigned long long>(5));
  a.coef = dev_alloc<double>(static_cast<size_t>(9 * a.n));
  a.mass = dev_alloc<double>(static_cast<size_t>(a.n));
  a.nnz_row = dev_alloc<unsigned char>(static_cast<size_t>(a.n));
  try {
    const Sheet2DDev d{g->nx, g->ny, g->h, std::cos(g->fiber_angle), std::sin(g->fiber_angle), g->d0_myocyte,
                       g->d0_fibrotic, g->rho, dtags, desc};
    CUDA_TRY(launch_sheet2d_assemble(d, AsmOut{a.coef, a.mass, a.nnz_row, dkeys}, st));
    unsigned long long keys[5];
    CUDA_TRY(cudaMemcpyAsync(keys, dkeys, sizeof(keys), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    const auto s = [](long long x) { return std::to_string(x); };
    if (keys[0] != ~0ull)
      throw Fail{CWG_EVALIDATION, "assemble: element " + s(static_cast<long long>(keys[0])) +
                                      " has non-positive Jacobian (degenerate or clockwise)"};
    if (keys[1] != ~0ull) {
      const long long i = static_cast<long long>(keys[1] / 16);
      const int what = static_cast<int>(keys[1] % 16);
      if (what == 0) throw Fail{CWG_EVALIDATION, "assemble: non-positive lumped mass at node " + s(i)};
      // the row's present entries, ascending column (= slot) order
      double row[9];
      CUDA_TRY(cudaMemcpy2D(row, sizeof(double), a.coef + i, static_cast<size_t>(a.n) * sizeof(double),
                            sizeof(double), 9, cudaMemcpyDeviceToHost));
      const long long iy = i / a.w, ix = i % a.w;
      double row_sum = 0.0;
      int p = 0;
      for (int q = 0; q < 9; ++q) {
        const long long jy = iy + q / 3 - 1, jx = ix + q % 3 - 1;
        if (jy < 0 || jy > g->ny || jx < 0 || jx > g->nx) continue;
        if (what == 1 + p)
          throw Fail{CWG_EVALIDATION, "assemble: stiffness not symmetric at (" + s(i) + ", " + s(jy * a.w + jx) + ")"};
        row_sum += row[q];
        ++p;
      }
      throw Fail{CWG_EVALIDATION, "assemble: row " + s(i) + " sum " + std::to_string(row_sum) + " not zero"};
    }
    if (keys[2] != ~0ull)
      throw Fail{CWG_EVALIDATION, "gershgorin: row " + s(static_cast<long long>(keys[2])) +
                                      " has non-positive k_ii + sum|k_ij|; operator is not diffusive"};
    double min_ratio;
    std::memcpy(&min_ratio, &keys[4], sizeof(min_ratio));
    validation(std::isfinite(min_ratio), "gershgorin: no diffusive row");
    a.dt_s = 0.9 * min_ratio;
  } catch (...) {
    a.release();
    throw;
  }
  return a;
}

// ---------------------------------------------------------------- step pieces
// Exchange `rows` halo rows (planes) with both neighbours: my first / last
// `rows` owned rows go down / up, theirs land in the halo rows adjacent to my
// slab. Local V layout: [hrows_v halo | owned | hrows_v halo] rows of w nodes.
// The halo exchange of `rows` rows (2D) or planes (3D) of a V buffer: what
// this rank sends to / receives from each neighbour. Shared by the NCCL
// transport (halo_exchange) and the one-GPU loopback (cwg_loopback_steps), so
// the loopback tests exercise the same buffer arithmetic.
struct HaloPlan {
  size_t n = 0;                                          // doubles per direction
  bool lo = false, hi = false;                           // neighbours rank - 1 / rank + 1 exist
  double *send_lo = nullptr, *recv_lo = nullptr;         // first owned rows / the halo below
  double *send_hi = nullptr, *recv_hi = nullptr;         // last owned rows / the halo above
};

HaloPlan halo_plan(const cwg_ctx* c, double* buf, int rows) {
  HaloPlan h;
  h.n = static_cast<size_t>(c->w) * static_cast<size_t>(rows);
  const size_t own0 = static_cast<size_t>(c->halo), own1 = own0 + static_cast<size_t>(c->n_own);
  h.lo = c->rank > 0;
  h.hi = c->rank + 1 < c->world;
  h.send_lo = buf + own0;
  h.recv_lo = buf + own0 - h.n;
  h.send_hi = buf + own1 - h.n;
  h.recv_hi = buf + own1;
  return h;
}

cudaError_t push_halo_now(cwg_ctx* c, const double* buf, cudaStream_t st);

void halo_exchange(cwg_ctx* c, double* buf, int rows, cudaStream_t st = nullptr) {
  if (c->p2p) {  // peer-memory transport: only a V writer that did not push its halos needs a push
    if (!c->halo_fresh) CUDA_TRY(push_halo_now(c, buf, st ? st : c->stream));
    c->halo_fresh = true;
    return;
  }
  if (c->world <= 1 || c->loopback) return;
  if (!st) st = c->stream;
  const HaloPlan h = halo_plan(c, buf, rows);
  NCCL_TRY(g_nccl.gstart());
  if (h.lo) {
    NCCL_TRY(g_nccl.send(h.send_lo, h.n, ncclDouble, c->rank - 1, c->comm, st));
    NCCL_TRY(g_nccl.recv(h.recv_lo, h.n, ncclDouble, c->rank - 1, c->comm, st));
  }
  if (h.hi) {
    NCCL_TRY(g_nccl.send(h.send_hi, h.n, ncclDouble, c->rank + 1, c->comm, st));
    NCCL_TRY(g_nccl.recv(h.recv_hi, h.n, ncclDouble, c->rank + 1, c->comm, st));
  }
  NCCL_TRY(g_nccl.gend());
}

// Build the padded coefficient tensor and its TMA descriptors (2D sheet on
// one device). Any failure just leaves the register-loading kernel in charge.
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// Rows of the padded coefficient tensor: the coefficient rows of the context (owned rows plus hrows_c
// halo rows each side on a multi-rank slab, so fused launches advance the neighbours' edge rows too)
long long tma_rows(const cwg_ctx* c) { return (c->row_end - c->row_begin) + 2ll * c->hrows_c; }

void refresh_padded_cm(cwg_ctx* c) {
  if (!c->d_coefp) return;
  CUDA_TRY(launch_pad_planes(c->d_cm, 0, 1, c->w, tma_rows(c), c->d_coefp, c->w_pad, 9, c->stream));
}

void setup_tma(cwg_ctx* c) {
  const char* e = getenv("CWG_TB_TMA");
  if (e && e[0] == '0') return;
  if (c->op_kind != CWG_OP_STENCIL2D || !c->d_coef) return;
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q{};
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn ||
      q != cudaDriverEntryPointSuccess) {
    cudaGetLastError();
    return;
  }
  const long long rows = tma_rows(c);
  unsigned bx0 = 0, by0 = 0;
  int margin = 0;
  tbm_box(4, &bx0, &by0, &margin);
  c->w_pad = (c->w + margin + 1) / 2 * 2;  // zeroed left margin; 16-byte row pitch
  c->d_coefp = dev_alloc<double>(static_cast<size_t>(10 * rows * c->w_pad));
  CUDA_TRY(cudaMemsetAsync(c->d_coefp, 0, static_cast<size_t>(10 * rows * c->w_pad) * sizeof(double), c->stream));
  CUDA_TRY(launch_pad_planes(c->d_coef, c->n_coef, 9, c->w, rows, c->d_coefp, c->w_pad, 0, c->stream));
  refresh_padded_cm(c);
  const cuuint64_t dims[3] = {static_cast<cuuint64_t>(c->w + margin), static_cast<cuuint64_t>(rows), 10};
  const cuuint64_t strides[2] = {static_cast<cuuint64_t>(c->w_pad) * 8, static_cast<cuuint64_t>(rows * c->w_pad) * 8};
  const cuuint32_t estr[3] = {1, 1, 1};
  bool ok = true;
  for (int T = 2; T <= 6 && ok; ++T) {
    unsigned cx = 0, cy = 0;
    tbm_box(T, &cx, &cy, &margin);
    const cuuint32_t box[3] = {cx, cy, 10};
    ok = reinterpret_cast<EncodeTiledFn>(fn)(&c->tmap[T], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, c->d_coefp, dims, strides,
                                             box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  }
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  c->tma_ok = ok;
}

// Large sheets (and y-slabs) take the TMA-fed persistent kernels (enqueue_diffusion). They do not store
// the neighbours' halo rows themselves, so a slab linked by the peer-memory transport keeps the
// register-loading kernel (which does); NCCL / loopback slabs exchange between launches.
bool tma_path(const cwg_ctx* c) {
  return c->tma_ok && !c->pl.on && ((c->w + 63) / 64) * ((c->row_end - c->row_begin + 15) / 16) >= 2ll * c->num_sms;
}

// sub-steps fused per launch by the temporal-blocking stencil (1 = off; CWG_DIFF_TB overrides): up to
// 6 in the TMA kernel (its 64 x 16 tile plus a 6-deep halo still fits shared memory; fewer launches
// re-read the coefficients fewer times), 4 in the register-loading kernel
int diffusion_fuse(const cwg_ctx* c) {
  if (c->op_kind != CWG_OP_STENCIL2D) return 1;
  const int cap = tma_path(c) ? 6 : 4;
  int f = cap;
  if (const char* e = getenv("CWG_DIFF_TB")) f = std::max(1, std::min(cap, atoi(e)));
  return c->world > 1 ? std::min(f, c->hrows_c) : f;  // T fused sub-steps need T halo rows (V and coefficients)
}

// fused-launch group sizes for `count` sub-steps: ceil(count/fuse) launches, balanced
std::vector<int> diffusion_groups(const cwg_ctx* c, int count) {
  const int fuse = diffusion_fuse(c);
  const int m = (count + fuse - 1) / fuse;
  std::vector<int> g;
  for (int q = 0, launch = 0; q < count; ++launch) {
    const int T = (count - q + (m - launch) - 1) / (m - launch);
    g.push_back(T);
    q += T;
  }
  return g;
}

// One diffusion launch of T fused sub-steps vin -> vout (err == nullptr: unchecked).
void launch_diffusion_group(cwg_ctx* c, int T, const double* vin, double* vout, ErrRec* err, long long step_off,
                            int ev) {
  DiffArgs a{};
  a.vin = vin;
  a.vout = vout;
  a.n = c->n_own;
  a.halo = c->halo;
  a.dt_sub = c->dt_ad;
  a.err = err;
  a.clock = c->d_clock;
  a.step_off = step_off;
  a.evs = c->evs;
  a.ev = ev;
  a.node_offset = c->own_global0;
  if (c->p2p && err) {  // (the unchecked replay of restore_failed_state never runs on linked ranks)
    a.pl = c->pl;
    a.out_par = vout == c->d_v[1] ? 1 : 0;
  }
  if (c->op_kind == CWG_OP_STENCIL2D) {
    Stencil2D s{c->d_coef, c->n_coef, c->d_cm, c->w, c->row_end - c->row_begin, c->row_begin, c->ny1,
                c->hrows_v, c->hrows_c};
    if (T > 1 && tma_path(c))
      CUDA_TRY(launch_diffuse_stencil2d_tbm(T, a, s, c->tmap[T], c->num_sms, c->stream));
    else if (T > 1)
      CUDA_TRY(launch_diffuse_stencil2d_tb(T, a, s, c->num_sms, c->stream));
    else
      CUDA_TRY(launch_diffuse_stencil2d(a, s, c->num_sms * 16, c->stream));
  } else if (c->op_kind == CWG_OP_STRUCT3D) {
    Struct3D s{c->d_coef, c->d_cm, c->s3_nx1, c->s3_nz1, c->w, c->row_end - c->row_begin, c->row_begin, c->ny1};
    CUDA_TRY(launch_diffuse_struct3d(a, s, c->num_sms, c->stream));
  } else {
    CsrDev m{c->d_rp, c->d_col, c->d_val, c->d_cm};
    CUDA_TRY(launch_diffuse_csr(a, m, c->num_sms * 16, c->stream));
  }
  ++c->launches;
  if (a.pl.on) c->halo_fresh = true;  // this launch stored the neighbours' halo rows of vout
}

// P2P: push this rank's edge rows of `buf` (one of the context's V pair) into the neighbours' halos
cudaError_t push_halo_now(cwg_ctx* c, const double* buf, cudaStream_t st) {
  DiffArgs a{};
  a.vin = buf;
  a.halo = c->halo;
  a.pl = c->pl;
  a.out_par = buf == c->d_v[1] ? 1 : 0;
  ++c->launches;
  return launch_push_halo(a, st);
}

void enqueue_diffusion(cwg_ctx* c, int count, long long step_off, int ev0, bool first_exchanged = false) {
  // ceil(count / fuse) launches with balanced group sizes; every launch flips
  // the V double buffer (graphs are kept per starting parity)
  const std::vector<int> groups = diffusion_groups(c, count);
  for (int gi = 0, q = 0; gi < static_cast<int>(groups.size()); ++gi) {
    const int T = groups[static_cast<size_t>(gi)];
    double* vin = c->d_v[c->cur];
    double* vout = c->d_v[c->cur ^ 1];
    if (!(gi == 0 && first_exchanged)) halo_exchange(c, vin, T);
    // threshold probe runs: no NaN scan after diffusion (stimulus.cpp:106) -> unchecked launch
    launch_diffusion_group(c, T, vin, vout, c->fixed_step ? nullptr : c->d_err, step_off, ev0 + q);
    c->cur ^= 1;
    q += T;
  }
}

// After a failure: put the state where the reference stops (splitting.cpp:
// 129-140 reaction: every node finished, V in place; :162-166 diffusion: the
// failing sub-step's output). Later events skipped without writing, so the
// failing launch's buffers are intact: copy its output into the current V
// buffer, or -- when it fused T sub-steps and failed in sub-step q < T-1 --
// replay q+1 sub-steps from its input first (bit-identical kernels,
// unchecked). One device only: with y-slabs a neighbour's halo may have
// moved on. Idempotent per failure (restored_seq).
void restore_failed_state(cwg_ctx* c, const ErrRec& r) {
  if (r.key == kNoError || r.seq == c->restored_seq || !r.vout) return;
  double* dst = c->d_v[c->cur];
  const double* src = r.vout;
  if (r.phase == 2 && r.T > 1 && c->world == 1) {
    const int q = static_cast<int>(r.key >> 58);
    if (q < r.T - 1) {
      launch_diffusion_group(c, q + 1, r.vin, r.vout, nullptr, 0, 0);
      CUDA_TRY(cudaStreamSynchronize(c->stream));
    }
  }
  if (src != dst)
    CUDA_TRY(cudaMemcpyAsync(dst, src, c->n_alloc * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  c->restored_seq = r.seq;
}

unsigned long long* g_react_trace = nullptr;  // diagnostics only (CWG_REACT_TRACE, cwg_react_trace)

ReactArgs react_args(const cwg_ctx* c, const Bin& b, long long step_off, int ev, bool use_t, double t_fixed) {
  ReactArgs a{};
  a.v = c->d_v[c->cur];
  a.S = c->d_S;
  a.pitch = c->pitch;
  a.last = c->d_last;
  a.list = b.d_list;
  a.first = b.first;
  a.count = b.count;
  a.stim = StimDev{c->d_stim_ptr, c->d_stim_ids, c->d_st0, c->d_sdur, c->d_samp, c->d_sper};
  a.gkr = c->d_gkr;
  a.dt = c->dt_eff;
  a.t_fixed = t_fixed;
  a.use_t_fixed = use_t ? 1 : 0;
  a.clock = c->d_clock;
  a.step_off = step_off;
  a.scheme = c->scheme;
  a.k0_up = c->k0_up;
  a.k0_down = c->k0_down;
  a.kmax = c->kmax_of_model[b.model];
  a.khist = c->d_khist;
  a.khist_len = c->khist_len;
  a.err = c->d_err;
  a.evs = c->evs;
  a.ev = ev;
  a.counter = b.d_counter;
  a.done = b.d_counter + 1;
  a.node_offset = c->node_offset;
  static const int preclaim = [] {
    const char* e = getenv("CWG_PRECLAIM");
    return e ? atoi(e) : 1;
  }();
  a.preclaim = preclaim;
  return a;
}

// One reaction launch of bin b over the dense local range [first, first + count)
// with its own self-resetting counter pair (concurrent launches never share one).
void launch_bin_range(cwg_ctx* c, const Bin& b, long long first, long long count, unsigned* counter, int variant,
                      int grid, cudaStream_t st, long long step_off, int ev, bool use_t, double t_fixed) {
  if (count <= 0) return;
  ReactArgs a = react_args(c, b, step_off, ev, use_t, t_fixed);
  a.first = first;
  a.count = count;
  a.counter = counter;
  a.done = counter + 1;
  cudaError_t e = is_ord(b.kind) ? launch_react_ord(b.kind, variant, a, grid, st)
                                 : launch_react_exact(b.kind, a, grid, st);
  CUDA_TRY(e);
  ++c->launches;
}

// bst: stream of the boundary-first launches (split runs; default the solver stream)
void enqueue_reaction(cwg_ctx* c, long long step_off, int ev, bool use_t, double t_fixed, cudaStream_t bst = nullptr) {
  c->halo_fresh = false;  // V changes in place: the neighbours' copies of the edge rows are stale
  for (auto& b : c->bins) {
    if (b.count == 0) continue;
    if (c->split && !b.d_list) {  // edge rows first, then the interior (node-local: same bits in any order)
      const long long e = c->split_rows * c->w, lo = c->halo, hi = c->halo + c->n_own;
      const cudaStream_t es = bst ? bst : c->stream;
      launch_bin_range(c, b, lo, e, b.d_counter_b, b.variant_b, b.grid_b, es, step_off, ev, use_t, t_fixed);
      launch_bin_range(c, b, hi - e, e, b.d_counter_b + 2, b.variant_b, b.grid_b, es, step_off, ev, use_t, t_fixed);
      launch_bin_range(c, b, lo + e, c->n_own - 2 * e, b.d_counter, b.variant, b.grid, c->stream, step_off, ev, use_t,
                       t_fixed);
      continue;
    }
    ReactArgs a = react_args(c, b, step_off, ev, use_t, t_fixed);
    if (getenv("CWG_REACT_TRACE") && b.grid <= 4096) {
      if (!g_react_trace) CUDA_TRY(cudaMalloc(&g_react_trace, 16 * 4096 * sizeof(unsigned long long)));
      CUDA_TRY(cudaMemsetAsync(g_react_trace, 0, 16 * 4096 * sizeof(unsigned long long), c->stream));
      a.trace = g_react_trace;
    }
    cudaError_t e = is_ord(b.kind) ? launch_react_ord(b.kind, b.variant, a, b.grid, c->stream)
                                   : launch_react_exact(b.kind, a, b.grid, c->stream);
    CUDA_TRY(e);
    ++c->launches;
  }
}

// Reaction then the step's merged diffusion sub-steps (steps A and B/III).
// NCCL y-slab runs overlap the first halo exchange with the reaction: the slab
// edge rows react first on the side stream, their exchange follows there while
// the interior reacts on the solver stream, and the diffusion joins both.
// mid_event (bench phase timing, graph capture): recorded on the solver stream
// once the reaction is enqueued there (the interior part, under the split).
void enqueue_react_then_diffuse(cwg_ctx* c, long long step_off, int count, bool use_t, double t_fixed,
                                cudaEvent_t mid_event = nullptr) {
  if (c->split && c->side && !c->loopback) {
    CUDA_TRY(cudaEventRecord(c->ev_fork, c->stream));
    CUDA_TRY(cudaStreamWaitEvent(c->side, c->ev_fork, 0));
    enqueue_reaction(c, step_off, c->l, use_t, t_fixed, c->side);
    halo_exchange(c, c->d_v[c->cur], diffusion_groups(c, count).front(), c->side);
    CUDA_TRY(cudaEventRecord(c->ev_join, c->side));
    if (mid_event) CUDA_TRY(cudaEventRecordWithFlags(mid_event, c->stream, cudaEventRecordExternal));
    CUDA_TRY(cudaStreamWaitEvent(c->stream, c->ev_join, 0));
    enqueue_diffusion(c, count, step_off, c->l + 1, true);
    return;
  }
  enqueue_reaction(c, step_off, c->l, use_t, t_fixed);
  if (mid_event) CUDA_TRY(cudaEventRecordWithFlags(mid_event, c->stream, cudaEventRecordExternal));
  enqueue_diffusion(c, count, step_off, c->l + 1);
}

// One outer step (StrangIntegrator::advance, splitting.cpp:171-181) at
// step = base + off, kernels addressing it as *clock + off. Records (run mode)
// follow splitting.cpp:274-279: traces when (step+1) % spr == 0, maps when
// (step+1) % spm == 0.
void enqueue_step(cwg_ctx* c, long long base, long long off, bool record, bool use_t, double t_fixed) {
  const long long step = base + off;
  if (step == 0) enqueue_diffusion(c, c->l, off, 0);  // step I
  enqueue_react_then_diffuse(c, off, step == c->n_steps - 1 ? c->l : 2 * c->l, use_t, t_fixed);  // A, III / merged B
  if (!record) return;
  const long long S = step + 1;
  if (c->n_probes > 0 && S % c->spr == 0) {
    CUDA_TRY(launch_record_probes(c->d_v[c->cur], c->d_probe_loc, c->n_probes, c->d_traces, c->d_clock, off + 1,
                                  c->spr, c->stream));
    ++c->launches;
  }
  if (S % c->spm == 0) {
    CUDA_TRY(launch_detector_observe(c->d_v[c->cur] + c->halo, c->n_own, 0, c->det, c->d_clock, off + 1, c->spm,
                                     c->dt_eff, c->stream));
    ++c->launches;
  }
}

void set_clock(cwg_ctx* c, long long value) {
  if (c->clock_at == value) return;
  CUDA_TRY(launch_set_clock(c->d_clock, value, c->stream));
  ++c->launches;
  c->clock_at = value;
}

// Graph of G consecutive middle steps (1 <= step, step + G <= n_steps - 1),
// valid for any base b with b == b0 (mod G) because G is a multiple of both
// record cadences. Ends with a clock tick so replays chain without host work.
void build_graph(cwg_ctx* c, long long b0) {
  cudaGraph_t g = nullptr;
  const int cur0 = c->cur;
  CUDA_TRY(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
  const long long l0 = c->launches;
  try {
    for (long long off = 0; off < c->G; ++off) enqueue_step(c, b0, off, true, false, 0.0);
    CUDA_TRY(launch_tick_clock(c->d_clock, c->G, c->stream));
  } catch (...) {
    cudaStreamEndCapture(c->stream, &g);
    if (g) cudaGraphDestroy(g);
    throw;
  }
  CUDA_TRY(cudaStreamEndCapture(c->stream, &g));
  c->graph_launches = c->launches - l0 + 1;
  c->launches = l0;
  CUDA_TRY(cudaGraphInstantiate(&c->graph_p[cur0], g, 0));
  cudaGraphDestroy(g);
  c->graph_cur_after[cur0] = c->cur;  // capture only recorded the flips
  c->cur = cur0;
  c->graph_base_mod = ((b0 % c->G) + c->G) % c->G;
  c->graph_built = true;
}

// One middle step as a graph (bench timing: the production launch path,
// kernels back to back) with three external event-record nodes -- step start,
// end of the reaction pass, step end -- whose events are swapped per launch
// (cudaGraphExecEventRecordNodeSetEvent) so every timed step has its own.
struct StepGraph {
  cudaGraph_t graph = nullptr;  // kept: node handles are only valid while their graph lives
  cudaEvent_t tmp[3] = {nullptr, nullptr, nullptr};
  cudaGraphExec_t exec = nullptr;
  cudaGraphNode_t ev_nodes[3] = {nullptr, nullptr, nullptr};
  long long launches = 0;
  int cur_after = 0;
};

void free_step_graph(StepGraph& sg) {
  if (sg.exec) cudaGraphExecDestroy(sg.exec);
  if (sg.graph) cudaGraphDestroy(sg.graph);
  for (auto& e : sg.tmp)
    if (e) cudaEventDestroy(e);
  sg = StepGraph{};
}

StepGraph& step_graph(cwg_ctx* c, long long step, StepGraph* cache, bool events = true) {
  const long long S = step + 1;
  const int flags = ((c->n_probes > 0 && S % c->spr == 0) ? 1 : 0) | (S % c->spm == 0 ? 2 : 0);
  StepGraph& sg = cache[flags | (c->cur << 2)];  // per recording pattern and starting V-buffer parity
  if (sg.exec) return sg;
  cudaGraph_t g = nullptr;
  const int cur0 = c->cur;
  const long long l0 = c->launches;
  cudaEvent_t* tmp = sg.tmp;
  for (int q = 0; q < 3; ++q) CUDA_TRY(cudaEventCreate(&tmp[q]));
  CUDA_TRY(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
  try {
    if (events) CUDA_TRY(cudaEventRecordWithFlags(tmp[0], c->stream, cudaEventRecordExternal));
    // the production step (boundary-first reaction + overlapped exchange under a y-slab split)
    enqueue_react_then_diffuse(c, 0, 2 * c->l, false, 0.0, events ? tmp[1] : nullptr);
    const long long base = step;
    if (flags & 1) {
      CUDA_TRY(launch_record_probes(c->d_v[c->cur], c->d_probe_loc, c->n_probes, c->d_traces, c->d_clock, 1, c->spr,
                                    c->stream));
      ++c->launches;
    }
    if (flags & 2) {
      CUDA_TRY(launch_detector_observe(c->d_v[c->cur] + c->halo, c->n_own, 0, c->det, c->d_clock, 1, c->spm,
                                       c->dt_eff, c->stream));
      ++c->launches;
    }
    (void)base;
    if (events) CUDA_TRY(cudaEventRecordWithFlags(tmp[2], c->stream, cudaEventRecordExternal));
  } catch (...) {
    cudaStreamEndCapture(c->stream, &g);
    if (g) cudaGraphDestroy(g);
    throw;
  }
  CUDA_TRY(cudaStreamEndCapture(c->stream, &g));
  sg.graph = g;
  sg.launches = c->launches - l0;
  c->launches = l0;
  // locate the event-record nodes in capture order (they form a chain with the kernels)
  size_t nn = 0;
  CUDA_TRY(cudaGraphGetNodes(g, nullptr, &nn));
  std::vector<cudaGraphNode_t> nodes(nn);
  CUDA_TRY(cudaGraphGetNodes(g, nodes.data(), &nn));
  int found = 0;
  for (auto nd : nodes) {
    cudaGraphNodeType ty;
    CUDA_TRY(cudaGraphNodeGetType(nd, &ty));
    if (ty != cudaGraphNodeTypeEventRecord) continue;
    cudaEvent_t e;
    CUDA_TRY(cudaGraphEventRecordNodeGetEvent(nd, &e));
    for (int q = 0; q < 3; ++q)
      if (e == tmp[q]) {
        sg.ev_nodes[q] = nd;
        ++found;
      }
  }
  if (events && found != 3) throw Fail{CWG_ECUDA, "step graph: event nodes not found"};
  CUDA_TRY(cudaGraphInstantiate(&sg.exec, g, 0));
  sg.cur_after = c->cur;
  c->cur = cur0;
  return sg;
}

long long lcm_ll(long long a, long long b) { return a / std::gcd(a, b) * b; }

}  // namespace

// ====================================================================== C ABI
namespace {

void build_stencil(cwg_ctx* c, const cwg_problem* p) {
  // Per-node 9 coefficients taken verbatim from the CSR rows; a row must hold
  // exactly its in-grid 9-neighbourhood in ascending order. Covers the owned
  // rows plus hrows_c rows each side (multi-rank fused diffusion).
  const long long w = c->w;
  const long long n_coef = c->n_coef;
  const long long g0 = (c->row_begin - c->hrows_c) * w;  // global index of local coefficient 0
  std::vector<double> coef(static_cast<size_t>(9 * n_coef), 0.0);
  for (long long o = 0; o < n_coef; ++o) {
    const long long i = g0 + o;
    if (i < 0 || i >= p->n) continue;  // beyond the sheet: never read
    const long long y = i / w, x = i - y * w;
    int prev = -1;
    for (long long p_ = p->row_ptr[i]; p_ < p->row_ptr[i + 1]; ++p_) {
      // the slot from the column's grid coordinates, not from the index
      // offset: for w = 2 the offsets -w+1 / -1 and 1 / w-1 coincide
      const long long j = p->col[p_];
      if (j < 0 || j >= p->n)
        throw Fail{CWG_EVALIDATION, "stencil: row " + std::to_string(i) + " couples outside the grid"};
      const long long dy = j / w - y, dx = j % w - x;
      if (dy < -1 || dy > 1 || dx < -1 || dx > 1)
        throw Fail{CWG_EVALIDATION, "stencil: row " + std::to_string(i) + " is not a 9-point grid row"};
      const int slot = static_cast<int>((dy + 1) * 3 + (dx + 1));
      if (slot <= prev)
        throw Fail{CWG_EVALIDATION, "stencil: row " + std::to_string(i) + " columns are not ascending"};
      prev = slot;
      coef[static_cast<size_t>(slot) * n_coef + o] = p->val[p_];
    }
    // every in-grid neighbour must be present (absent ones would be read as 0)
    int expect = 0;
    for (int s = 0; s < 9; ++s) {
      const long long gy = y + (s / 3) - 1, gx = x + (s % 3) - 1;
      if (gy >= 0 && gy < c->ny1 && gx >= 0 && gx < w) ++expect;
    }
    if (p->row_ptr[i + 1] - p->row_ptr[i] != expect)
      throw Fail{CWG_EVALIDATION, "stencil: row " + std::to_string(i) + " misses grid neighbours"};
  }
  c->d_coef = upload(coef.data(), coef.size());
}

// ORd launch shape. Throughput regime (many nodes per lane): one persistent
// 384-thread block per SM (<= 168 registers) whose warps advance in lockstep
// -- free-running warps drift apart and thrash the 32 KB L1.5 instruction
// cache with the ~54 KB fast-path body (C3: 0.65 ms lockstep vs 1.12 ms free-running).
// Latency regime (the bin fits into <= 10 warps per SM, e.g. C2's 40k nodes:
// about one node per lane): two free-running 128-thread blocks per SM with up
// to 255 registers -- there the per-evaluation barrier only adds waiting (C2
// reaction 53.6 us vs 59.0 us for the best lockstep shape).
int choose_ord_variant(long long count, int num_sms) {
  if (const char* e = getenv("CWG_ORD_VARIANT")) {
    const int v = atoi(e);
    if (react_ord_variant_valid(v)) return v;
  }
  const long long warps_per_sm = (count + 32ll * num_sms - 1) / (32ll * num_sms);
  return warps_per_sm <= 10 ? 0 : 1;
}

bool stencil_ok(const cwg_problem* p) {
  if (p->grid_nx1 <= 0 || p->grid_ny1 <= 0 || p->grid_nx1 * p->grid_ny1 != p->n) return false;
  const long long w = p->grid_nx1;
  for (long long i = 0; i < p->n; ++i) {
    const long long y = i / w, x = i - y * w;
    int expect = 0;
    for (int s = 0; s < 9; ++s) {
      const long long gy = y + (s / 3) - 1, gx = x + (s % 3) - 1;
      if (gy >= 0 && gy < p->grid_ny1 && gx >= 0 && gx < w) ++expect;
    }
    if (p->row_ptr[i + 1] - p->row_ptr[i] != expect) return false;
    long long prev = -1;
    for (long long q = p->row_ptr[i]; q < p->row_ptr[i + 1]; ++q) {
      const long long j = p->col[q];
      const long long jy = j / w, jx = j - jy * w;
      if (j <= prev || std::llabs(jy - y) > 1 || std::llabs(jx - x) > 1) return false;
      prev = j;
    }
  }
  return true;
}

// A regular sheet's row 0 couples {0, 1, w, w+1} (mesh.hpp:23-24 numbering):
// infer the grid when the caller (e.g. the C++ drop-in) has only the CSR.
void infer_grid(cwg_problem* q) {
  if (q->grid_nx1 > 0 || !q->row_ptr || q->n < 4) return;
  if (q->row_ptr[1] - q->row_ptr[0] != 4) return;
  const long long w = q->col[2];
  if (q->col[0] != 0 || q->col[1] != 1 || w < 2 || q->col[3] != w + 1 || q->n % w != 0) return;
  q->grid_nx1 = w;
  q->grid_ny1 = q->n / w;
}

// Scheme-dependent quantities (StrangIntegrator ctor, splitting.cpp:74-93;
// run_simulation's step counts and record cadences, :225-240).
void configure_scheme(cwg_ctx* c, int scheme, double dt_ms, double t_end_ms, int k0_up, int k0_down, int strict) {
  validation(dt_ms > 0.0, "scheme: dt must be positive");
  validation(t_end_ms >= dt_ms, "scheme: T must be >= dt");
  validation(k0_down >= 1 && k0_up >= k0_down, "scheme: need k0_up >= k0_down >= 1");
  validation(scheme >= CWG_OST && scheme <= CWG_DAETI, "scheme: unknown scheme");
  c->scheme = scheme;
  c->dt = dt_ms;
  c->t_end = t_end_ms;
  c->k0_up = k0_up;
  c->k0_down = k0_down;
  c->strict = strict;
  c->dt_eff = c->scheme == CWG_OSTAR ? std::min(c->dt, c->dt_s) : c->dt;
  {
    int l = 0;
    double dt_ad = 0;
    cwg_diffusion_substeps(c->dt_eff, c->dt_s, c->strict, c->scheme, &l, &dt_ad);
    c->l = l;
    c->dt_ad = dt_ad;
  }
  c->evs = 3ll * c->l + 2;
  c->kmax_of_model.clear();
  c->kmax_global = 0;
  for (int kind : c->model_kind) {
    c->kmax_of_model.push_back(kmax_for(c->dt_eff, kind));
    c->kmax_global = std::max(c->kmax_global, c->kmax_of_model.back());
  }
  validation(c->kmax_global < 2048, "integrator: k_max >= 2048 is not supported");
  c->khist_len = c->kmax_global + 1;
  c->n_steps = static_cast<long long>(std::ceil(c->t_end / c->dt_eff - 1e-9));
  c->spr = std::max<long long>(1, llround_ref(c->record_interval / c->dt_eff));
  c->spm = std::max<long long>(1, llround_ref(c->map_interval / c->dt_eff));
  c->n_samples = c->n_steps / c->spr + 1;
  const long long G = lcm_ll(c->spr, c->spm);  // graph block: a multiple of both record cadences
  c->G = G <= 200 ? G : 0;
}

// ------------------------------------------------------------------ peer-memory halo link
bool p2p_eligible(const cwg_ctx* c) {
  if (c->world <= 1) return false;
  if (const char* e = getenv("CWG_P2P"))
    if (e[0] == '0') return false;
  if (c->op_kind == CWG_OP_CSR) return false;
  return c->row_end - c->row_begin >= 2 * c->hrows_v;  // the edge rows of the two sides do not overlap
}

// Fill c->pl from the neighbours' buffers (loopback: other contexts' pointers; NCCL ranks: IPC-mapped).
void set_peer_link(cwg_ctx* c, double* const lo_v[2], long long lo_halo, long long lo_own, unsigned long long* lo_flags,
                   double* const hi_v[2], long long hi_halo, unsigned long long* hi_flags) {
  PeerLink& pl = c->pl;
  pl.on = 1;
  pl.w = c->w;
  pl.rows = c->row_end - c->row_begin;
  pl.lim = c->op_kind == CWG_OP_STRUCT3D ? 1 : c->hrows_v;
  for (int p = 0; p < 2; ++p) {
    pl.lo_dst[p] = lo_v[p] ? lo_v[p] + lo_halo + lo_own : nullptr;  // rank-1's upper halo rows
    pl.hi_dst[p] = hi_v[p] ? hi_v[p] + hi_halo : nullptr;           // rank+1's first owned node
  }
  pl.wait_lo = lo_flags ? c->d_flags + 0 : nullptr;
  pl.wait_hi = hi_flags ? c->d_flags + 1 : nullptr;
  pl.post_lo = lo_flags ? lo_flags + 1 : nullptr;
  pl.post_hi = hi_flags ? hi_flags + 0 : nullptr;
  pl.count = c->d_flags + 2;
  pl.blocks_done = reinterpret_cast<unsigned*>(c->d_flags + 3);
  c->p2p = true;
  c->split = false;  // the halo goes out with the launches themselves
}

void alloc_flags(cwg_ctx* c) {
  if (c->d_flags) return;
  c->d_flags = dev_alloc<unsigned long long>(4);
  CUDA_TRY(cudaMemset(c->d_flags, 0, 4 * sizeof(unsigned long long)));
}

// NCCL ranks: exchange IPC handles of both V buffers and the flag words with an
// allgather, map the two neighbours'. All ranks agree (allreduce min) or all
// keep the NCCL transport.
struct P2PInfo {
  cudaIpcMemHandle_t hv[2], hf;
  long long halo, n_own;
  int ok, pad;
};

void setup_p2p_nccl(cwg_ctx* c) {
  if (!p2p_eligible(c) || c->loopback || !c->comm) return;
  alloc_flags(c);
  P2PInfo mine{};
  mine.ok = 1;
  if (cudaIpcGetMemHandle(&mine.hv[0], c->d_v[0]) != cudaSuccess ||
      cudaIpcGetMemHandle(&mine.hv[1], c->d_v[1]) != cudaSuccess || cudaIpcGetMemHandle(&mine.hf, c->d_flags) != cudaSuccess) {
    cudaGetLastError();
    mine.ok = 0;
  }
  mine.halo = c->halo;
  mine.n_own = c->n_own;
  DevScope scope;
  char* d_all = scope.keep(dev_alloc<char>(sizeof(P2PInfo) * c->world));
  char* d_mine = scope.keep(dev_alloc<char>(sizeof(P2PInfo)));
  h2d(d_mine, &mine, sizeof(P2PInfo));
  NCCL_TRY(g_nccl.allgather(d_mine, d_all, sizeof(P2PInfo), ncclChar, c->comm, c->stream));
  std::vector<P2PInfo> all(static_cast<size_t>(c->world));
  CUDA_TRY(cudaMemcpyAsync(all.data(), d_all, sizeof(P2PInfo) * c->world, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  double* lo_v[2] = {nullptr, nullptr};
  double* hi_v[2] = {nullptr, nullptr};
  unsigned long long *lo_f = nullptr, *hi_f = nullptr;
  int ok = 1;
  for (const auto& a : all) ok &= a.ok;
  auto open = [&](const P2PInfo& nb, double** v, unsigned long long** f) {
    void* p = nullptr;
    for (int q = 0; q < 2 && ok; ++q) {
      if (cudaIpcOpenMemHandle(&p, nb.hv[q], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
        cudaGetLastError();
        ok = 0;
        return;
      }
      c->ipc_opened.push_back(p);
      v[q] = static_cast<double*>(p);
    }
    if (ok && cudaIpcOpenMemHandle(&p, nb.hf, cudaIpcMemLazyEnablePeerAccess) == cudaSuccess) {
      c->ipc_opened.push_back(p);
      *f = static_cast<unsigned long long*>(p);
    } else {
      cudaGetLastError();
      ok = 0;
    }
  };
  if (ok && c->rank > 0) open(all[static_cast<size_t>(c->rank - 1)], lo_v, &lo_f);
  if (ok && c->rank + 1 < c->world) open(all[static_cast<size_t>(c->rank + 1)], hi_v, &hi_f);
  // every rank must take the same transport
  int* d_ok = scope.keep(dev_alloc<int>(1));
  h2d(d_ok, &ok, sizeof(int));
  NCCL_TRY(g_nccl.allreduce(d_ok, d_ok, 1, ncclInt, ncclMin, c->comm, c->stream));
  CUDA_TRY(cudaMemcpyAsync(&ok, d_ok, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  if (!ok) {
    for (void* p : c->ipc_opened) cudaIpcCloseMemHandle(p);
    c->ipc_opened.clear();
    return;
  }
  const P2PInfo* lo = c->rank > 0 ? &all[static_cast<size_t>(c->rank - 1)] : nullptr;
  const P2PInfo* hi = c->rank + 1 < c->world ? &all[static_cast<size_t>(c->rank + 1)] : nullptr;
  set_peer_link(c, lo_v, lo ? lo->halo : 0, lo ? lo->n_own : 0, lo_f, hi_v, hi ? hi->halo : 0, hi_f);
}

// CWG_TRACE_CREATE=1: per-phase wall times of cwg_create on stderr (fixed-cost analysis of the e2e path)
struct PhaseTrace {
  bool on = getenv("CWG_TRACE_CREATE") != nullptr;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now(), last = t0;
  void mark(const char* what) {
    if (!on) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[cwg_create] %-22s %8.3f ms (total %8.3f)\n", what,
                 std::chrono::duration<double, std::milli>(now - last).count(),
                 std::chrono::duration<double, std::milli>(now - t0).count());
    last = now;
  }
};

void create_impl(const cwg_problem* p_in, cwg_ctx* c) {
  PhaseTrace tr;
  validation(p_in != nullptr, "integrator: empty problem");
  cwg_problem pc = *p_in;
  if (pc.op_kind == CWG_OP_AUTO) infer_grid(&pc);
  const cwg_problem* p = &pc;
  const bool dev_sheet = pc.op_kind == CWG_OP_SHEET2D;  // operator assembled on the device below
  validation(p->n > 0, "integrator: empty problem");
  validation(p->lumped_mass != nullptr || p->op_kind == CWG_OP_STRUCT3D || dev_sheet,
             "integrator: missing assembled operator");
  validation(p->n_models > 0 && p->model_kind, "integrator: no cell models");
  validation(p->record_interval_ms > 0.0, "scheme: record interval must be positive");
  validation(dev_sheet || p->dt_s > 0.0, "diffusion sub-steps: dt and dt_s must be positive");
  validation(p->world >= 1 && p->rank >= 0 && p->rank < p->world, "placement: bad rank/world");
  validation(p->n < (1ll << 40), "integrator: at most 2^40 nodes");

  c->device = p->device;
  CUDA_TRY(cudaSetDevice(c->device));
  // two attribute queries (cudaGetDeviceProperties fills ~100 fields and costs milliseconds per context)
  int major = 0;
  CUDA_TRY(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, c->device));
  if (major < 10) throw Fail{CWG_ECUDA, "cwgpu needs an sm_100 (Blackwell) device"};
  CUDA_TRY(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, c->device));
  CUDA_TRY(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  c->own_stream = true;
  for (auto& e : c->ev) CUDA_TRY(cudaEventCreate(&e));

  // ---- device-assembled sheet: stencil tables and dt_s from assemble.cu; from
  // here on the context is a stencil-2D one (no CSR crosses PCIe)
  SheetAsm sheet;
  struct SheetRelease {
    SheetAsm& a;
    ~SheetRelease() { a.release(); }
  } sheet_release{sheet};
  if (dev_sheet) {
    sheet = assemble_sheet2d(p->sheet2d, c->stream);
    validation(p->n == sheet.n, "operator: n does not match the sheet");
    pc.dt_s = sheet.dt_s;
    pc.grid_nx1 = p->sheet2d->nx + 1;
    pc.grid_ny1 = p->sheet2d->ny + 1;
    pc.op_kind = CWG_OP_STENCIL2D;
  }
  tr.mark("device assembly");

  // ---- scheme (StrangIntegrator ctor, splitting.cpp:74-93)
  c->dt_s = p->dt_s;
  c->record_interval = p->record_interval_ms;
  c->map_interval = p->map_interval_ms > 0.0 ? p->map_interval_ms : 1.0;
  c->model_kind.assign(p->model_kind, p->model_kind + p->n_models);
  c->stride = 1;
  for (int m = 0; m < p->n_models; ++m) {
    validation(state_count(c->model_kind[m]) >= 0, "integrator: unknown model kind " + std::to_string(c->model_kind[m]));
    c->stride = std::max(c->stride, state_count(c->model_kind[m]));
  }
  configure_scheme(c, p->scheme, p->dt_ms, p->t_end_ms, p->k0_up, p->k0_down, p->strict_substeps);
  tr.mark("device+scheme");

  // ---- partition and operator layout
  std::vector<double> s3_coef, s3_mass;
  if (p->op_kind == CWG_OP_STRUCT3D) {
    validation(p->s3d != nullptr, "operator: CWG_OP_STRUCT3D needs cwg_problem.s3d");
    const cwg_struct3d& s3 = *p->s3d;
    validation(s3.nx >= 1 && s3.ny >= 1 && s3.nz >= 1, "operator: 3D slab needs >= 1 element per axis");
    const long long n3 = (s3.nx + 1) * (s3.ny + 1) * (s3.nz + 1);
    validation(p->n == n3, "operator: n does not match the 3D slab");
    s3_coef.resize(static_cast<size_t>(9 * (s3.nz + 1) * 27));
    s3_mass.resize(static_cast<size_t>(9 * (s3.nz + 1)));
    const double dts = cwg_struct3d_tables(p->s3d, s3_coef.data(), s3_mass.data());
    validation(dts > 0.0, "operator: invalid 3D slab parameters");
    c->s3_nx1 = s3.nx + 1;
    c->s3_nz1 = s3.nz + 1;
  }
  c->n_global = p->n;
  int kind = p->op_kind;
  if (kind == CWG_OP_AUTO) kind = stencil_ok(p) ? CWG_OP_STENCIL2D : CWG_OP_CSR;
  validation(kind == CWG_OP_CSR || kind == CWG_OP_STENCIL2D || kind == CWG_OP_STRUCT3D, "operator: unknown op_kind");
  if (kind == CWG_OP_STENCIL2D && !dev_sheet)
    validation(stencil_ok(p), "operator: CSR is not a regular-sheet 9-point operator");
  c->op_kind = kind;
  c->rank = p->rank;
  c->world = p->world;
  if (kind == CWG_OP_STRUCT3D) {  // y-slabs of (nx+1)*(nz+1)-node planes
    c->w = c->s3_nx1 * c->s3_nz1;
    c->ny1 = p->s3d->ny + 1;
    int64_t rb = 0, re = 0;
    validation(cwg_slab_plan(c->ny1, c->world, c->rank, &rb, &re) == CWG_OK, "placement: fewer planes than ranks");
    c->row_begin = rb;
    c->row_end = re;
    c->n_own = (re - rb) * c->w;
    c->halo = c->w;
    c->own_global0 = rb * c->w;
    c->node_offset = c->own_global0 - c->halo;
  } else if (kind == CWG_OP_STENCIL2D || p->world > 1) {
    validation(p->grid_nx1 > 0 && p->grid_ny1 > 0 && p->grid_nx1 * p->grid_ny1 == p->n,
               "placement: slab decomposition needs the sheet's grid dimensions");
    c->w = p->grid_nx1;
    c->ny1 = p->grid_ny1;
    int64_t rb = 0, re = 0;
    validation(cwg_slab_plan(c->ny1, c->world, c->rank, &rb, &re) == CWG_OK, "placement: fewer rows than ranks");
    c->row_begin = rb;
    c->row_end = re;
    c->n_own = (re - rb) * c->w;
    // Multi-rank stencil: H = min(4, thinnest slab) halo rows of V and of the
    // coefficients, so a launch can fuse up to H sub-steps: it advances the
    // neighbours' boundary rows itself and exchanges H rows once per launch.
    if (c->world > 1 && kind == CWG_OP_STENCIL2D) {
      c->hrows_v = static_cast<int>(std::max<long long>(1, std::min<long long>(4, c->ny1 / c->world)));
      c->hrows_c = c->hrows_v;
    }
    c->halo = c->hrows_v * c->w;
    c->own_global0 = rb * c->w;
    c->node_offset = c->own_global0 - c->halo;
  } else {
    c->w = p->grid_nx1;
    c->ny1 = p->grid_ny1;
    c->row_begin = 0;
    c->row_end = p->grid_ny1;
    c->n_own = p->n;
    c->halo = 0;
    c->own_global0 = 0;
    c->node_offset = 0;
  }
  c->n_alloc = c->n_own + 2 * c->halo;
  tr.mark("partition");

  // ---- device state (SoA, pitch padded to 32 nodes = 256 B)
  c->pitch = (c->n_alloc + 31) / 32 * 32;
  // (+ kVPad: slack for the 3D kernel's aligned row copies; the halo rows /
  // planes stay zero unless a neighbour rank writes them)
  c->d_v[0] = dev_alloc<double>(c->n_alloc + kVPad);
  c->d_v[1] = dev_alloc<double>(c->n_alloc + kVPad);
  CUDA_TRY(cudaMemset(c->d_v[0], 0, (c->n_alloc + kVPad) * sizeof(double)));
  CUDA_TRY(cudaMemset(c->d_v[1], 0, (c->n_alloc + kVPad) * sizeof(double)));
  c->d_S = dev_alloc<double>(static_cast<size_t>(c->pitch) * ((c->stride + 3) & ~3));  // columns in groups of 4 (sidx)
  c->d_last = dev_alloc<double>(c->n_alloc);
  CUDA_TRY(cudaMemset(c->d_S, 0, static_cast<size_t>(c->pitch) * ((c->stride + 3) & ~3) * sizeof(double)));
  CUDA_TRY(cudaMemset(c->d_last, 0, c->n_alloc * sizeof(double)));
  tr.mark("state alloc");

  // ---- operator upload
  if (kind == CWG_OP_STRUCT3D) {
    c->d_mass = upload(s3_mass.data(), s3_mass.size());
    c->n_mass = static_cast<long long>(s3_mass.size());
    c->d_cm = dev_alloc<double>(s3_mass.size());
    CUDA_TRY(launch_mass_factor(c->d_mass, c->n_mass, c->dt_ad, c->d_cm, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    c->d_coef = upload(s3_coef.data(), s3_coef.size());
  } else if (dev_sheet) {
    // the coefficient rows of this rank (owned rows + hrows_c halo rows each side)
    // sliced out of the device-assembled tables; rows beyond the sheet: 0 / mass 1
    const long long rows_c = (c->row_end - c->row_begin) + 2ll * c->hrows_c;
    c->n_coef = rows_c * c->w;
    const long long g0 = (c->row_begin - c->hrows_c) * c->w;
    c->d_coef = dev_alloc<double>(static_cast<size_t>(9 * c->n_coef));
    c->d_mass = dev_alloc<double>(static_cast<size_t>(c->n_coef));
    CUDA_TRY(launch_sheet2d_slice(sheet.coef, sheet.mass, sheet.n, c->w, g0, c->n_coef, c->d_coef, c->d_mass,
                                  c->stream));
    c->n_mass = c->n_coef;
    c->d_cm = dev_alloc<double>(c->n_coef);
    CUDA_TRY(launch_mass_factor(c->d_mass, c->n_coef, c->dt_ad, c->d_cm, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
  } else {
    validation(p->lumped_mass != nullptr, "integrator: missing assembled operator");
    // lumped mass of the coefficient rows (owned rows, plus hrows_c halo rows
    // each side for a multi-rank stencil; rows beyond the sheet: 1, never read)
    const long long rows_c = (c->row_end - c->row_begin) + 2ll * c->hrows_c;
    c->n_coef = kind == CWG_OP_STENCIL2D ? rows_c * c->w : c->n_own;
    std::vector<double> mass_own(static_cast<size_t>(c->n_coef), 1.0);
    const long long g0 = kind == CWG_OP_STENCIL2D ? (c->row_begin - c->hrows_c) * c->w : c->own_global0;
    for (long long o = 0; o < c->n_coef; ++o)
      if (g0 + o >= 0 && g0 + o < p->n) mass_own[static_cast<size_t>(o)] = p->lumped_mass[g0 + o];
    c->d_mass = upload(mass_own.data(), mass_own.size());
    c->n_mass = c->n_coef;
    c->d_cm = dev_alloc<double>(c->n_coef);
    CUDA_TRY(launch_mass_factor(c->d_mass, c->n_coef, c->dt_ad, c->d_cm, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
  }
  if (kind == CWG_OP_STRUCT3D) {
    // tables uploaded above
  } else if (kind == CWG_OP_STENCIL2D) {
    if (!dev_sheet) build_stencil(c, p);
    setup_tma(c);
  } else {
    validation(p->row_ptr && p->col && p->val, "operator: CSR arrays missing");
    const long long r0 = c->own_global0, r1 = c->own_global0 + c->n_own;
    const long long p0 = p->row_ptr[r0], p1 = p->row_ptr[r1];
    std::vector<long long> rp(static_cast<size_t>(c->n_own + 1));
    for (long long i = 0; i <= c->n_own; ++i) rp[i] = p->row_ptr[r0 + i] - p0;
    std::vector<long long> col(static_cast<size_t>(p1 - p0));
    for (long long q = p0; q < p1; ++q) {
      const long long lc = p->col[q] - c->node_offset;
      validation(lc >= 0 && lc < c->n_alloc, "operator: coupling beyond the neighbouring slab rows");
      col[q - p0] = lc;
    }
    c->d_rp = upload(rp.data(), rp.size());
    c->d_col = upload(col.data(), col.size());
    c->d_val = upload(p->val + p0, static_cast<size_t>(p1 - p0));
  }

  tr.mark("before models: per-model node bins over owned nodes");
  // ---- models: per-model node bins over owned nodes (local indices)
  validation(p->model_of_node != nullptr, "integrator: model_of_node missing");
  validation(c->n_alloc < (1ll << 31), "integrator: more than 2^31 local nodes per device (use more ranks)");
  std::vector<long long> per_model(static_cast<size_t>(p->n_models), 0);
  {
    // byte histogram over the owned nodes, four interleaved tables (no store-to-load chain on a run of equal ids)
    std::vector<long long> hist(4 * 256, 0);
    const uint8_t* mo = p->model_of_node + c->own_global0;
    long long o = 0;
    for (; o + 4 <= c->n_own; o += 4) {
      ++hist[mo[o]];
      ++hist[256 + mo[o + 1]];
      ++hist[512 + mo[o + 2]];
      ++hist[768 + mo[o + 3]];
    }
    for (; o < c->n_own; ++o) ++hist[mo[o]];
    for (int m = 0; m < 256; ++m) {
      const long long cnt = hist[m] + hist[256 + m] + hist[512 + m] + hist[768 + m];
      if (m < p->n_models) {
        per_model[static_cast<size_t>(m)] = cnt;
      } else if (cnt > 0) {  // the reference names the first node without a model
        for (long long q = 0; q < c->n_own; ++q)
          if (mo[q] >= p->n_models)
            validation(false, "initial state: node " + std::to_string(c->own_global0 + q) + " has no model");
      }
    }
  }
  for (int m = 0; m < p->n_models; ++m) {
    Bin b;
    b.model = m;
    b.kind = c->model_kind[m];
    b.count = per_model[static_cast<size_t>(m)];
    if (b.count == c->n_own) {
      b.first = c->halo;  // dense
    } else if (b.count > 0) {
      std::vector<int32_t> list;
      list.reserve(static_cast<size_t>(b.count));
      for (long long o = 0; o < c->n_own; ++o)
        if (p->model_of_node[c->own_global0 + o] == m) list.push_back(static_cast<int32_t>(o + c->halo));
      b.d_list = upload(list.data(), list.size());
    }
    b.variant = choose_ord_variant(b.count, c->num_sms);
    const int threads = is_ord(b.kind) ? react_ord_threads(b.variant) : react_exact_threads(b.kind);
    const int occ =
        std::max(1, is_ord(b.kind) ? react_ord_occupancy(b.kind, b.variant) : react_exact_occupancy(b.kind));
    const long long need = (b.count + threads - 1) / threads;
    b.grid = static_cast<int>(std::max<long long>(1, std::min<long long>(need, static_cast<long long>(occ) * c->num_sms)));
    b.d_counter = dev_alloc<unsigned>(2);
    CUDA_TRY(cudaMemset(b.d_counter, 0, 2 * sizeof(unsigned)));
    c->bins.push_back(b);
  }
  // boundary-first split of the reaction (y-slab runs): the rows a neighbour's
  // first fused diffusion launch reads (hrows_v, >= its fused depth)
  c->split_rows = c->hrows_v;
  c->split = c->world > 1 && c->op_kind != CWG_OP_CSR && c->n_own >= 4 * c->split_rows * c->w &&
             getenv("CWG_SPLIT") == nullptr;
  if (c->split) {
    for (auto& b : c->bins)
      if (!b.d_list && b.count > 0) {
        b.d_counter_b = dev_alloc<unsigned>(4);
        CUDA_TRY(cudaMemset(b.d_counter_b, 0, 4 * sizeof(unsigned)));
        const long long e = c->split_rows * c->w;
        // the interior's launch shape: ptxas contracts mul/add pairs per kernel instance, so
        // only the same instance keeps the slab run bit-identical to the single-GPU one
        b.variant_b = b.variant;
        const int threads = is_ord(b.kind) ? react_ord_threads(b.variant_b) : react_exact_threads(b.kind);
        const int occ = std::max(1, is_ord(b.kind) ? react_ord_occupancy(b.kind, b.variant_b)
                                                   : react_exact_occupancy(b.kind));
        b.grid_b = static_cast<int>(std::max<long long>(
            1, std::min<long long>((e + threads - 1) / threads, static_cast<long long>(occ) * c->num_sms)));
      }
    if (!c->loopback) {
      CUDA_TRY(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
      CUDA_TRY(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
      CUDA_TRY(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
    }
  }
  if (p->gkr_scale) {
    std::vector<double> g(static_cast<size_t>(c->n_alloc), 1.0);
    for (long long o = 0; o < c->n_own; ++o) g[o + c->halo] = p->gkr_scale[c->own_global0 + o];
    c->d_gkr = upload(g.data(), g.size());
  }

  tr.mark("before stimulus");
  // ---- stimulus (ProtocolIndex, flattened to the local slab)
  if (p->n_stim > 0) {
    validation(p->stim_node_ptr && p->stim_ids && p->stim_t_start && p->stim_duration && p->stim_amplitude &&
                   p->stim_period, "stimulus: arrays missing");
    for (int e = 0; e < p->n_stim; ++e) {
      validation(p->stim_duration[e] > 0.0, "stimulus: duration must be positive");
      validation(std::isfinite(p->stim_amplitude[e]), "stimulus: amplitude must be finite");
    }
    // the owned nodes' entry lists are one contiguous slice of stim_ids; the local
    // per-node pointer array (0 over the lower halo, the total over the upper one)
    // is rebased from the caller's on the device
    const int32_t id0 = p->stim_node_ptr[c->own_global0], id1 = p->stim_node_ptr[c->own_global0 + c->n_own];
    if (id1 > id0) {
      DevScope tmp;
      const int32_t* gptr = tmp.keep(upload(p->stim_node_ptr + c->own_global0, static_cast<size_t>(c->n_own + 1)));
      c->d_stim_ptr = dev_alloc<int32_t>(static_cast<size_t>(c->n_alloc + 1));
      CUDA_TRY(launch_stim_local_ptr(gptr, c->n_own, c->halo, c->n_alloc, c->d_stim_ptr, c->stream));
      CUDA_TRY(cudaStreamSynchronize(c->stream));
      c->d_stim_ids = upload(p->stim_ids + id0, static_cast<size_t>(id1 - id0));
      c->d_st0 = upload(p->stim_t_start, p->n_stim);
      c->d_sdur = upload(p->stim_duration, p->n_stim);
      c->d_samp = upload(p->stim_amplitude, p->n_stim);
      c->d_sper = upload(p->stim_period, p->n_stim);
    }
  }

  tr.mark("before bookkeeping");
  // ---- bookkeeping
  c->d_err = dev_alloc<ErrRec>(1);
  c->d_clock = dev_alloc<long long>(1);
  c->d_khist = dev_alloc<unsigned long long>(c->khist_len);
  ErrRec none{kNoError, kNoSeq, 0, 0, nullptr, nullptr};
  h2d(c->d_err, &none, sizeof(none));
  CUDA_TRY(cudaMemset(c->d_clock, 0, sizeof(long long)));
  c->clock_at = 0;
  CUDA_TRY(cudaMemset(c->d_khist, 0, c->khist_len * sizeof(unsigned long long)));

  tr.mark("before recording");
  // ---- recording
  c->lat_threshold = p->lat_threshold_mv;
  c->n_probes = p->n_probes;
  if (c->n_probes > 0) {
    std::vector<long long> loc(static_cast<size_t>(c->n_probes), -1);
    for (int q = 0; q < c->n_probes; ++q) {
      const long long g = p->probes[q];
      validation(g >= 0 && g < p->n, "probe: node out of range");
      if (g >= c->own_global0 && g < c->own_global0 + c->n_own) loc[q] = g - c->node_offset;
    }
    c->d_probe_loc = upload(loc.data(), loc.size());
    c->d_traces = dev_alloc<double>(static_cast<size_t>(c->n_samples) * c->n_probes);
    CUDA_TRY(cudaMemset(c->d_traces, 0, static_cast<size_t>(c->n_samples) * c->n_probes * sizeof(double)));
  }
  double** dd[] = {&c->det.prev_v, &c->det.v_rest, &c->det.max_slope, &c->det.t_max_slope, &c->det.v_peak,
                   &c->det.lat, &c->det.apd};
  for (auto q : dd) *q = dev_alloc<double>(c->n_own);
  c->det.phase = dev_alloc<unsigned char>(c->n_own);
  c->det.has_lat = dev_alloc<unsigned char>(c->n_own);
  c->det.has_apd = dev_alloc<unsigned char>(c->n_own);
  c->det.threshold = c->lat_threshold;

  // ---- NCCL communicator for the halo exchange
  if (c->world > 1 && p->nccl_id == nullptr && getenv("CWG_LOOPBACK") && atoi(getenv("CWG_LOOPBACK"))) {
    c->loopback = true;  // ranks share one process and device; cwg_loopback_steps drives them
  } else if (c->world > 1) {
    validation(p->nccl_id != nullptr, "placement: world > 1 needs an NCCL unique id");
    if (!g_nccl.load()) throw Fail{CWG_ECUDA, "NCCL library (libnccl.so.2) not loadable"};
    ncclUniqueId id;
    std::memcpy(&id, p->nccl_id, sizeof(id));
    NCCL_TRY(g_nccl.init(&c->comm, c->world, id, c->rank));
    setup_p2p_nccl(c);
  }
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  tr.mark("recording+comm");
}

thread_local std::string g_last_error;

template <class F>
int guarded(cwg_error* err, F&& f) {
  g_last_error.clear();
  try {
    f();
    if (err) {
      err->code = CWG_OK;
      err->node = -1;
      err->phase = 0;
      err->msg[0] = 0;
    }
    return CWG_OK;
  } catch (const Fail& e) {
    g_last_error = e.msg;
    set_error(err, e.code, e.msg);
    return e.code;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    set_error(err, CWG_ECUDA, e.what());
    return CWG_ECUDA;
  }
}

void reset_error(cwg_ctx* c) {
  ErrRec none{kNoError, kNoSeq, 0, 0, nullptr, nullptr};
  c->restored_seq = -1;
  CUDA_TRY(cudaMemcpyAsync(c->d_err, &none, sizeof(none), cudaMemcpyHostToDevice, c->stream));
  // the reaction bins' work/done counters reset themselves at the end of
  // every launch; zero them here too so no earlier launch can leave them stale
  for (const auto& b : c->bins) {
    if (b.d_counter) CUDA_TRY(cudaMemsetAsync(b.d_counter, 0, 2 * sizeof(unsigned), c->stream));
    if (b.d_counter_b) CUDA_TRY(cudaMemsetAsync(b.d_counter_b, 0, 4 * sizeof(unsigned), c->stream));
  }
  CUDA_TRY(cudaStreamSynchronize(c->stream));
}

bool ev_is_reaction(const cwg_ctx* c, long long seq) { return seq % c->evs == c->l; }

// Read the error record (after a sync) and, for world > 1, agree on the
// earliest failing event and its lowest node across ranks.
bool fetch_error(cwg_ctx* c, bool use_t, double t_fixed, cwg_error* out) {
  ErrRec r{};
  CUDA_TRY(cudaMemcpy(&r, c->d_err, sizeof(r), cudaMemcpyDeviceToHost));
  const ErrRec local = r;
  if (c->world > 1 && !c->loopback) {
    long long* tmp = dev_alloc<long long>(2);
    long long h[2] = {r.key == kNoError ? (1ll << 62) : r.seq, 0};
    h2d(tmp, h, sizeof(long long));
    NCCL_TRY(g_nccl.allreduce(tmp, tmp, 1, ncclInt64, ncclMin, c->comm, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    CUDA_TRY(cudaMemcpy(h, tmp, sizeof(long long), cudaMemcpyDeviceToHost));
    unsigned long long key = (r.key != kNoError && r.seq == h[0]) ? r.key : kNoError;
    h2d(tmp, &key, sizeof(key));
    NCCL_TRY(g_nccl.allreduce(tmp, tmp, 1, ncclUint64, ncclMin, c->comm, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    CUDA_TRY(cudaMemcpy(&key, tmp, sizeof(key), cudaMemcpyDeviceToHost));
    dev_free(tmp);
    r.key = key;
    r.seq = h[0];
  }
  if (r.key == kNoError) return false;
  restore_failed_state(c, local);
  // diffusion keys carry the fused sub-step index in bits 58..63 (temporal blocking)
  const long long node = static_cast<long long>(r.key >> 22) & (ev_is_reaction(c, r.seq) ? -1ll : (1ll << 36) - 1);
  const long long step = r.seq / c->evs;
  const long long ev = r.seq % c->evs;
  const double t = use_t ? t_fixed : static_cast<double>(step) * c->dt_eff;
  char buf[256];
  if (ev == c->l) {  // reaction event
    const int k = static_cast<int>((r.key >> 11) & 2047u);
    const int j = static_cast<int>(r.key & 2047u);
    const double dt_ar = c->dt_eff / static_cast<double>(k);
    const double ts = t + static_cast<double>(j) * dt_ar;
    std::snprintf(buf, sizeof(buf), "reaction step produced non-finite V (node %lld, t = %f ms)", node, ts);
    if (out) {
      out->code = CWG_EINSTABILITY;
      out->node = node;
      out->t_ms = ts;
      out->phase = 1;
    }
  } else {
    std::snprintf(buf, sizeof(buf), "diffusion sub-step produced non-finite V (node %lld, t = %f ms)", node, t);
    if (out) {
      out->code = CWG_EINSTABILITY;
      out->node = node;
      out->t_ms = t;
      out->phase = 2;
    }
  }
  if (out) std::snprintf(out->msg, sizeof(out->msg), "%s", buf);
  return true;
}

// recompute cm = dt_ad / m after dt_ad changed (fixed-step mode)
cudaError_t launch_mass_factor_fix(cwg_ctx* c) {
  if (!c->d_mass) return cudaErrorNotSupported;
  cudaError_t e = launch_mass_factor(c->d_mass, c->n_mass, c->dt_ad, c->d_cm, c->stream);
  if (e != cudaSuccess) return e;
  if (c->d_coefp) {
    e = launch_pad_planes(c->d_cm, 0, 1, c->w, c->row_end - c->row_begin, c->d_coefp, c->w_pad, 9, c->stream);
    if (e != cudaSuccess) return e;
  }
  return cudaStreamSynchronize(c->stream);
}

void normalise_parity(cwg_ctx* c) {
  if (c->cur == 0) return;
  CUDA_TRY(cudaMemcpyAsync(c->d_v[0], c->d_v[1], c->n_alloc * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  c->cur = 0;
}

// AoS staging buffer for a caller state of `stride` doubles per node (any
// stride >= c->stride: a wider model list, a checkpoint): up to 2^20 nodes
// per chunk, reallocated when a wider stride needs more room.
void ensure_stage(cwg_ctx* c, int stride) {
  const long long nodes = std::max<long long>(1, std::min<long long>(c->n_own, 1ll << 20));
  const long long need = nodes * stride;
  if (c->d_stage && c->stage_cap >= need) {
    c->stage_nodes = c->stage_cap / stride;
    if (c->stage_nodes > nodes) c->stage_nodes = nodes;
    return;
  }
  dev_free(c->d_stage);
  c->d_stage = dev_alloc<double>(static_cast<size_t>(need));
  c->stage_cap = need;
  c->stage_nodes = nodes;
}

}  // namespace

extern "C" {

const char* cwg_version(void) { return "cwgpu 1 (sm_100a)"; }

const char* cwg_last_error(void) { return g_last_error.c_str(); }

int cwg_model_state_count(int kind) { return state_count(kind); }

int cwg_model_rest_state(int kind, double* out) {
  const int ns = state_count(kind);
  if (ns < 0) return CWG_EVALIDATION;
  if (is_ord(kind)) {
    std::memcpy(out, kOrdRest[kind - CWG_MODEL_ORD_ENDO], 41 * sizeof(double));
  } else if (kind == CWG_MODEL_ALIEV_PANFILOV) {
    out[0] = -80.0;
    out[1] = 0.0;
  } else if (kind == CWG_MODEL_MACCANNELL) {
    out[0] = -48.865796143695611;
    out[1] = 0.067599408770662575;
    out[2] = 0.97575886906521692;
  } else {
    out[0] = -85.0;  // passive: its reversal potential
  }
  return CWG_OK;
}
double cwg_model_stable_step(int kind) { return stable_step(kind); }

int cwg_model_kind_from_name(const char* name) {
  if (!name) return -1;
  const std::string n(name);
  if (n == "aliev-panfilov") return CWG_MODEL_ALIEV_PANFILOV;
  if (n == "ohara2011-endo") return CWG_MODEL_ORD_ENDO;
  if (n == "ohara2011-epi") return CWG_MODEL_ORD_EPI;
  if (n == "ohara2011-mid") return CWG_MODEL_ORD_MID;
  if (n == "maccannell2007") return CWG_MODEL_MACCANNELL;
  if (n == "passive") return CWG_MODEL_PASSIVE;
  return -1;
}

int cwg_reaction_substeps(double dvdt, int scheme, int k0_up, int k0_down, int k_max) {
  if (scheme == CWG_OST) return 1;
  const int k0 = dvdt > 0.0 ? k0_up : k0_down;
  const double raw = static_cast<double>(k0) + std::floor(std::fabs(dvdt));
  const int k = raw > static_cast<double>(k_max) ? k_max : static_cast<int>(raw);
  return k < 1 ? 1 : k;
}

int cwg_diffusion_substeps(double dt, double dt_s, int strict, int scheme, int* l, double* dt_ad) {
  if (!(dt > 0.0) || !(dt_s > 0.0)) return CWG_EVALIDATION;
  int ll = 1;
  if (scheme == CWG_DAETI && dt / 2.0 > dt_s) {
    const double q = dt / (2.0 * dt_s);
    ll = static_cast<int>(strict ? std::ceil(q) : std::floor(q));
    if (ll < 1) ll = 1;
  }
  *l = ll;
  *dt_ad = dt / (2.0 * ll);
  return CWG_OK;
}

int cwg_k_max_for(double dt, int kind) { return kmax_for(dt, kind); }

int cwg_slab_plan(int64_t ny1, int world, int rank, int64_t* row_begin, int64_t* row_end) {
  if (world < 1 || rank < 0 || rank >= world || ny1 < world) return CWG_EVALIDATION;
  const int64_t base = ny1 / world, extra = ny1 % world;
  *row_begin = rank * base + std::min<int64_t>(rank, extra);
  *row_end = *row_begin + base + (rank < extra ? 1 : 0);
  return CWG_OK;
}

int64_t cwg_sheet2d_nnz(const cwg_sheet2d* g) {
  if (!g || g->nx < 1 || g->ny < 1) return 0;
  return (3 * g->nx + 1) * (3 * g->ny + 1);  // rows with 2 (edge) or 3 neighbours per axis, incl. the node
}

int cwg_sheet2d_assemble(const cwg_sheet2d* g, int device, int64_t* row_ptr, int64_t* col, double* val,
                         double* lumped_mass, double* dt_s, cwg_error* err) {
  return guarded(err, [&] {
    CUDA_TRY(cudaSetDevice(device));
    cudaStream_t st = nullptr;
    CUDA_TRY(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    struct StreamGuard {
      cudaStream_t s;
      ~StreamGuard() { cudaStreamDestroy(s); }
    } sg{st};
    SheetAsm a = assemble_sheet2d(g, st);
    struct Release {
      SheetAsm& a;
      ~Release() { a.release(); }
    } rel{a};
    if (dt_s) *dt_s = a.dt_s;
    if (lumped_mass)
      CUDA_TRY(cudaMemcpy(lumped_mass, a.mass, static_cast<size_t>(a.n) * sizeof(double), cudaMemcpyDeviceToHost));
    if (row_ptr || col || val) {  // the stencil table -> the reference's CSR (ascending columns)
      std::vector<double> coef(static_cast<size_t>(9 * a.n));
      CUDA_TRY(cudaMemcpy(coef.data(), a.coef, coef.size() * sizeof(double), cudaMemcpyDeviceToHost));
      int64_t q = 0;
      for (long long i = 0; i < a.n; ++i) {
        if (row_ptr) row_ptr[i] = q;
        const long long iy = i / a.w, ix = i % a.w;
        for (int sl = 0; sl < 9; ++sl) {
          const long long jy = iy + sl / 3 - 1, jx = ix + sl % 3 - 1;
          if (jy < 0 || jy > g->ny || jx < 0 || jx > g->nx) continue;
          if (col) col[q] = jy * a.w + jx;
          if (val) val[q] = coef[static_cast<size_t>(sl) * a.n + i];
          ++q;
        }
      }
      if (row_ptr) row_ptr[a.n] = q;
    }
  });
}

int cwg_create(const cwg_problem* prob, cwg_ctx** out, cwg_error* err) {
  cwg_ctx* c = new cwg_ctx();
  const int rc = guarded(err, [&] { create_impl(prob, c); });
  if (rc != CWG_OK) {
    ctx_free(c);
    *out = nullptr;
    return rc;
  }
  *out = c;
  return CWG_OK;
}

void cwg_destroy(cwg_ctx* c) { ctx_free(c); }

int cwg_set_stream(cwg_ctx* c, void* s) {
  return guarded(nullptr, [&] {
    CUDA_TRY(cudaSetDevice(c->device));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    if (c->own_stream) CUDA_TRY(cudaStreamDestroy(c->stream));
    if (s) {
      c->stream = static_cast<cudaStream_t>(s);
      c->own_stream = false;
    } else {
      CUDA_TRY(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
      c->own_stream = true;
    }
  });
}

void* cwg_stream(cwg_ctx* c) { return c->stream; }

int cwg_upload_state(cwg_ctx* c, const double* v, const double* s_aos, int stride, const double* last) {
  return guarded(nullptr, [&] {
    validation(stride >= c->stride, "state: stride smaller than the largest model state count");
    CUDA_TRY(cudaSetDevice(c->device));
    c->cur = 0;
    c->halo_fresh = false;
    const long long g0 = c->own_global0;
    CUDA_TRY(cudaMemcpyAsync(c->d_v[0] + c->halo, v + g0, c->n_own * sizeof(double), cudaMemcpyHostToDevice,
                             c->stream));
    CUDA_TRY(cudaMemcpyAsync(c->d_last + c->halo, last + g0, c->n_own * sizeof(double), cudaMemcpyHostToDevice,
                             c->stream));
    ensure_stage(c, stride);
    for (long long o = 0; o < c->n_own; o += c->stage_nodes) {
      const long long cnt = std::min(c->stage_nodes, c->n_own - o);
      CUDA_TRY(cudaMemcpyAsync(c->d_stage, s_aos + (g0 + o) * stride, cnt * stride * sizeof(double),
                               cudaMemcpyHostToDevice, c->stream));
      CUDA_TRY(launch_aos_to_soa(c->d_stage, stride, c->stride, cnt, c->d_S, c->pitch, c->halo + o, c->stream));
      ++c->launches;
    }
    CUDA_TRY(cudaStreamSynchronize(c->stream));
  });
}

int cwg_init_rest_state(cwg_ctx* c) {
  return guarded(nullptr, [&] {
    CUDA_TRY(cudaSetDevice(c->device));
    c->cur = 0;
    c->halo_fresh = false;
    for (const auto& b : c->bins) {
      double rest[64] = {0};
      cwg_model_rest_state(b.kind, rest);
      double* d_rest = upload(rest, 64);
      CUDA_TRY(launch_init_rest(c->d_v[0], c->d_S, c->pitch, c->d_last, b.d_list, b.first, b.count, d_rest,
                                state_count(b.kind), c->stride, c->stream));
      ++c->launches;
      CUDA_TRY(cudaStreamSynchronize(c->stream));
      dev_free(d_rest);
    }
  });
}

int cwg_download_state(cwg_ctx* c, double* v, double* s_aos, int stride, double* last) {
  return guarded(nullptr, [&] {
    validation(stride >= c->stride, "state: stride smaller than the largest model state count");
    CUDA_TRY(cudaSetDevice(c->device));
    const long long g0 = c->own_global0;
    if (v)
      CUDA_TRY(cudaMemcpyAsync(v + g0, c->d_v[c->cur] + c->halo, c->n_own * sizeof(double), cudaMemcpyDeviceToHost,
                               c->stream));
    if (last)
      CUDA_TRY(cudaMemcpyAsync(last + g0, c->d_last + c->halo, c->n_own * sizeof(double), cudaMemcpyDeviceToHost,
                               c->stream));
    if (s_aos) {
      ensure_stage(c, stride);
      for (long long o = 0; o < c->n_own; o += c->stage_nodes) {
        const long long cnt = std::min(c->stage_nodes, c->n_own - o);
        CUDA_TRY(launch_soa_to_aos(c->d_S, c->pitch, c->halo + o, c->stride, cnt, c->d_stage, stride, c->stream));
        ++c->launches;
        CUDA_TRY(cudaMemcpyAsync(s_aos + (g0 + o) * stride, c->d_stage, cnt * stride * sizeof(double),
                                 cudaMemcpyDeviceToHost, c->stream));
      }
    }
    CUDA_TRY(cudaStreamSynchronize(c->stream));
  });
}

int cwg_set_scheme(cwg_ctx* c, int scheme, double dt_ms, double t_end_ms, int k0_up, int k0_down,
                   int strict_substeps, cwg_error* err) {
  return guarded(err, [&] {
    validation(!c->fixed_step, "scheme: not available on a threshold probe context");
    CUDA_TRY(cudaSetDevice(c->device));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    const long long old_khist = c->khist_len, old_samples = c->n_samples;
    configure_scheme(c, scheme, dt_ms, t_end_ms, k0_up, k0_down, strict_substeps);
    if (c->khist_len != old_khist) {
      dev_free(c->d_khist);
      c->d_khist = dev_alloc<unsigned long long>(c->khist_len);
    }
    CUDA_TRY(cudaMemset(c->d_khist, 0, c->khist_len * sizeof(unsigned long long)));
    if (c->n_probes > 0 && c->n_samples != old_samples) {
      dev_free(c->d_traces);
      c->d_traces = dev_alloc<double>(static_cast<size_t>(c->n_samples) * c->n_probes);
    }
    CUDA_TRY(launch_mass_factor_fix(c));  // cm = dt_ad / m for the new dt_ad (same division)
    for (auto& gx : c->graph_p)
      if (gx) {
        cudaGraphExecDestroy(gx);
        gx = nullptr;
      }
    c->graph_built = false;
  });
}

int cwg_loopback_link(cwg_ctx* const* ranks, int world) {
  return guarded(nullptr, [&] {
    validation(ranks && world >= 2, "loopback: need >= 2 rank contexts");
    for (int r = 0; r < world; ++r) {
      validation(ranks[r] && ranks[r]->loopback && ranks[r]->world == world && ranks[r]->rank == r,
                 "loopback: contexts must be ranks 0..world-1 created with CWG_LOOPBACK=1");
      validation(p2p_eligible(ranks[r]), "loopback: the peer-memory transport needs 2D stencil / 3D slabs");
      CUDA_TRY(cudaSetDevice(ranks[r]->device));
      alloc_flags(ranks[r]);
    }
    for (int r = 0; r < world; ++r) {
      cwg_ctx* lo = r > 0 ? ranks[r - 1] : nullptr;
      cwg_ctx* hi = r + 1 < world ? ranks[r + 1] : nullptr;
      double* lo_v[2] = {lo ? lo->d_v[0] : nullptr, lo ? lo->d_v[1] : nullptr};
      double* hi_v[2] = {hi ? hi->d_v[0] : nullptr, hi ? hi->d_v[1] : nullptr};
      set_peer_link(ranks[r], lo_v, lo ? lo->halo : 0, lo ? lo->n_own : 0, lo ? lo->d_flags : nullptr, hi_v,
                    hi ? hi->halo : 0, hi ? hi->d_flags : nullptr);
    }
  });
}

int cwg_loopback_steps(cwg_ctx* const* ranks, int world, int64_t first, int64_t count) {
  return guarded(nullptr, [&] {
    validation(ranks && world >= 2, "loopback: need >= 2 rank contexts");
    for (int r = 0; r < world; ++r)
      validation(ranks[r] && ranks[r]->loopback && ranks[r]->world == world && ranks[r]->rank == r,
                 "loopback: contexts must be ranks 0..world-1 created with CWG_LOOPBACK=1");
    cwg_ctx* c0 = ranks[0];
    CUDA_TRY(cudaSetDevice(c0->device));
    const cudaStream_t shared = c0->stream;
    std::vector<cudaStream_t> own(static_cast<size_t>(world));
    for (int r = 0; r < world; ++r) {
      own[static_cast<size_t>(r)] = ranks[r]->stream;
      CUDA_TRY(cudaStreamSynchronize(ranks[r]->stream));
      ranks[r]->stream = shared;  // one stream: every rank's work is ordered as enqueued below
    }
    // halo_exchange()'s plan with the NCCL send/recv pairs as device copies between the ranks' current
    // V buffers: rank r's halo below <- rank r-1's last rows, its halo above <- rank r+1's first rows
    auto exchange = [&](int rows) {
      for (int r = 0; r < world; ++r) {
        const HaloPlan h = halo_plan(ranks[r], ranks[r]->d_v[ranks[r]->cur], rows);
        if (h.lo) {
          const HaloPlan b = halo_plan(ranks[r - 1], ranks[r - 1]->d_v[ranks[r - 1]->cur], rows);
          validation(b.n == h.n && b.hi, "loopback: halo plans of ranks r-1 and r disagree");
          CUDA_TRY(cudaMemcpyAsync(h.recv_lo, b.send_hi, h.n * sizeof(double), cudaMemcpyDeviceToDevice, shared));
        }
        if (h.hi) {
          const HaloPlan t = halo_plan(ranks[r + 1], ranks[r + 1]->d_v[ranks[r + 1]->cur], rows);
          validation(t.n == h.n && t.lo, "loopback: halo plans of ranks r and r+1 disagree");
          CUDA_TRY(cudaMemcpyAsync(h.recv_hi, t.send_lo, h.n * sizeof(double), cudaMemcpyDeviceToDevice, shared));
        }
      }
    };
    // linked contexts (cwg_loopback_link): the launches store the halos themselves (peer-memory
    // transport); a rank whose halos are stale after the reaction pushes them, all ranks before any launch
    const bool linked = c0->p2p;
    auto diffuse_all = [&](int count, int ev0) {
      int q = 0;
      for (int T : diffusion_groups(c0, count)) {
        if (linked) {
          for (int r = 0; r < world; ++r) halo_exchange(ranks[r], ranks[r]->d_v[ranks[r]->cur], T);
          for (int r = 0; r < world; ++r) enqueue_diffusion(ranks[r], T, 0, ev0 + q, true);
        } else {
          exchange(T);
          for (int r = 0; r < world; ++r) enqueue_diffusion(ranks[r], T, 0, ev0 + q);
        }
        q += T;
      }
    };
    try {
      for (long long s = first; s < first + count; ++s) {
        for (int r = 0; r < world; ++r) set_clock(ranks[r], s);
        const int l = c0->l;
        if (s == 0) diffuse_all(l, 0);                                                   // step I
        for (int r = 0; r < world; ++r) enqueue_reaction(ranks[r], 0, l, false, 0.0);  // step A
        diffuse_all(s == c0->n_steps - 1 ? l : 2 * l, l + 1);                         // step III / merged B
        const long long S = s + 1;
        for (int r = 0; r < world; ++r) {
          cwg_ctx* c = ranks[r];
          if (c->n_probes > 0 && S % c->spr == 0)
            CUDA_TRY(launch_record_probes(c->d_v[c->cur], c->d_probe_loc, c->n_probes, c->d_traces, c->d_clock, 1,
                                          c->spr, shared));
          if (S % c->spm == 0)
            CUDA_TRY(launch_detector_observe(c->d_v[c->cur] + c->halo, c->n_own, 0, c->det, c->d_clock, 1, c->spm,
                                             c->dt_eff, shared));
        }
      }
      CUDA_TRY(cudaStreamSynchronize(shared));
    } catch (...) {
      for (int r = 0; r < world; ++r) ranks[r]->stream = own[static_cast<size_t>(r)];
      throw;
    }
    for (int r = 0; r < world; ++r) ranks[r]->stream = own[static_cast<size_t>(r)];
  });
}

int cwg_snapshot_begin(cwg_ctx* c, double* host_v) {
  return guarded(nullptr, [&] {
    validation(host_v != nullptr, "snapshot: no destination");
    validation(!c->snap_pending, "snapshot: the previous snapshot was not waited for");
    CUDA_TRY(cudaSetDevice(c->device));
    if (c->world > 1) {  // the failure agreement is a collective on the solver stream: stay synchronous
      CUDA_TRY(cudaMemcpyAsync(host_v + c->own_global0, c->d_v[c->cur] + c->halo, c->n_own * sizeof(double),
                               cudaMemcpyDeviceToHost, c->stream));
      c->snap_pending = true;
      return;
    }
    if (!c->d_snap) {
      c->d_snap = dev_alloc<double>(std::max<long long>(c->n_own, 1));
      c->d_snap_err = dev_alloc<ErrRec>(1);
      CUDA_TRY(cudaMallocHost(&c->h_snap_err, sizeof(ErrRec)));
      CUDA_TRY(cudaStreamCreateWithFlags(&c->snap_stream, cudaStreamNonBlocking));
      CUDA_TRY(cudaEventCreateWithFlags(&c->ev_vready, cudaEventDisableTiming));
      CUDA_TRY(cudaEventCreateWithFlags(&c->ev_snapdone, cudaEventDisableTiming));
    }
    // device-side copy on the solver stream (V and the failure record at this
    // point of the run), then the D2H on a side stream: the solver stream
    // moves on to the next steps while the copy drains
    CUDA_TRY(cudaMemcpyAsync(c->d_snap, c->d_v[c->cur] + c->halo, c->n_own * sizeof(double),
                             cudaMemcpyDeviceToDevice, c->stream));
    CUDA_TRY(cudaMemcpyAsync(c->d_snap_err, c->d_err, sizeof(ErrRec), cudaMemcpyDeviceToDevice, c->stream));
    CUDA_TRY(cudaEventRecord(c->ev_vready, c->stream));
    CUDA_TRY(cudaStreamWaitEvent(c->snap_stream, c->ev_vready, 0));
    CUDA_TRY(cudaMemcpyAsync(host_v + c->own_global0, c->d_snap, c->n_own * sizeof(double), cudaMemcpyDeviceToHost,
                             c->snap_stream));
    CUDA_TRY(cudaMemcpyAsync(c->h_snap_err, c->d_snap_err, sizeof(ErrRec), cudaMemcpyDeviceToHost, c->snap_stream));
    CUDA_TRY(cudaEventRecord(c->ev_snapdone, c->snap_stream));
    c->snap_pending = true;
  });
}

int cwg_snapshot_wait(cwg_ctx* c, cwg_error* err) {
  bool failed = false;
  cwg_error e{};
  const int rc = guarded(err, [&] {
    validation(c->snap_pending, "snapshot: nothing to wait for");
    CUDA_TRY(cudaSetDevice(c->device));
    c->snap_pending = false;
    if (c->world > 1) {
      CUDA_TRY(cudaStreamSynchronize(c->stream));
      failed = fetch_error(c, false, 0.0, &e);
      return;
    }
    CUDA_TRY(cudaEventSynchronize(c->ev_snapdone));
    if (c->h_snap_err->key != kNoError) {  // the run failed at or before this point: report it like run_sync
      CUDA_TRY(cudaStreamSynchronize(c->stream));
      failed = fetch_error(c, false, 0.0, &e);
    }
  });
  if (rc != CWG_OK) return rc;
  if (failed) {
    if (err) *err = e;
    return CWG_EINSTABILITY;
  }
  return CWG_OK;
}

int cwg_host_register(void* p, size_t bytes) {
  return guarded(nullptr, [&] { CUDA_TRY(cudaHostRegister(p, bytes, cudaHostRegisterDefault)); });
}

int cwg_host_unregister(void* p) {
  return guarded(nullptr, [&] { CUDA_TRY(cudaHostUnregister(p)); });
}

int cwg_pinned_buffers(cwg_ctx* c, double** v, double** s_aos, double** last) {
  return guarded(nullptr, [&] {
    CUDA_TRY(cudaSetDevice(c->device));
    if (!c->h_v) {
      CUDA_TRY(cudaMallocHost(&c->h_v, std::max<long long>(c->n_global, 1) * sizeof(double)));
      CUDA_TRY(cudaMallocHost(&c->h_s, std::max<long long>(c->n_global, 1) * c->stride * sizeof(double)));
      CUDA_TRY(cudaMallocHost(&c->h_last, std::max<long long>(c->n_global, 1) * sizeof(double)));
    }
    *v = c->h_v;
    *s_aos = c->h_s;
    *last = c->h_last;
  });
}

int cwg_advance(cwg_ctx* c, double t_ms, int64_t step, int64_t n_steps, cwg_error* err) {
  cwg_error e{};
  bool inst = false;
  const int rc = guarded(err, [&] {
    validation(step < n_steps, "integrator: step index past the end of the run");
    CUDA_TRY(cudaSetDevice(c->device));
    reset_error(c);
    set_clock(c, step);
    const long long saved = c->n_steps;
    c->n_steps = n_steps;
    CUDA_TRY(cudaEventRecord(c->ev[0], c->stream));
    if (step == 0) enqueue_diffusion(c, c->l, 0, 0);                       // step I
    CUDA_TRY(cudaEventRecord(c->ev[1], c->stream));
    enqueue_reaction(c, 0, c->l, true, t_ms);                               // step A
    CUDA_TRY(cudaEventRecord(c->ev[2], c->stream));
    enqueue_diffusion(c, step == n_steps - 1 ? c->l : 2 * c->l, 0, c->l + 1);  // step III / B
    CUDA_TRY(cudaEventRecord(c->ev[3], c->stream));
    c->n_steps = saved;
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    float a = 0, b = 0, d = 0;
    cudaEventElapsedTime(&a, c->ev[0], c->ev[1]);
    cudaEventElapsedTime(&b, c->ev[1], c->ev[2]);
    cudaEventElapsedTime(&d, c->ev[2], c->ev[3]);
    c->t_react += b;
    c->t_diff += a + d;
    inst = fetch_error(c, true, t_ms, &e);
  });
  if (rc != CWG_OK) return rc;
  if (inst) {
    if (err) *err = e;
    return CWG_EINSTABILITY;
  }
  return CWG_OK;
}

int cwg_run_begin(cwg_ctx* c) {
  return guarded(nullptr, [&] {
    CUDA_TRY(cudaSetDevice(c->device));
    normalise_parity(c);
    c->halo_fresh = false;
    reset_error(c);
    CUDA_TRY(cudaMemsetAsync(c->d_khist, 0, c->khist_len * sizeof(unsigned long long), c->stream));
    set_clock(c, 0);
    if (c->n_probes > 0) {
      CUDA_TRY(cudaMemsetAsync(c->d_traces, 0, static_cast<size_t>(c->n_samples) * c->n_probes * sizeof(double),
                               c->stream));
      CUDA_TRY(launch_record_probes(c->d_v[c->cur], c->d_probe_loc, c->n_probes, c->d_traces, c->d_clock, 0, c->spr,
                                    c->stream));
      ++c->launches;
    }
    CUDA_TRY(launch_detector_init(c->d_v[c->cur] + c->halo, c->n_own, 0, c->det, c->stream));
    ++c->launches;
    c->det_initialised = true;
  });
}

int cwg_run_steps(cwg_ctx* c, int64_t first, int64_t count) {
  return guarded(nullptr, [&] {
    CUDA_TRY(cudaSetDevice(c->device));
    validation(first >= 0 && first + count <= c->n_steps, "run: step range outside [0, n_steps)");
    long long s = first;
    const long long end = first + count;
    while (s < end) {
      const bool block_ok = c->G > 0 && s >= 1 && s + c->G <= c->n_steps - 1 && s + c->G <= end &&
                            (!c->graph_built ? (s % c->G == 1 % c->G) : (s % c->G == c->graph_base_mod));
      if (block_ok) {
        set_clock(c, s);
        if (!c->graph_p[c->cur]) build_graph(c, s);
        CUDA_TRY(cudaGraphLaunch(c->graph_p[c->cur], c->stream));
        c->cur = c->graph_cur_after[c->cur];
        c->launches += c->graph_launches;
        c->clock_at = s + c->G;
        s += c->G;
      } else {
        set_clock(c, s);
        enqueue_step(c, s, 0, true, false, 0.0);
        ++s;
      }
    }
  });
}

int cwg_run_sync(cwg_ctx* c, cwg_error* err) {
  cwg_error e{};
  bool inst = false;
  const int rc = guarded(err, [&] {
    CUDA_TRY(cudaSetDevice(c->device));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    inst = fetch_error(c, false, 0.0, &e);
  });
  if (rc != CWG_OK) return rc;
  if (inst) {
    if (err) *err = e;
    return CWG_EINSTABILITY;
  }
  return CWG_OK;
}

int cwg_run(cwg_ctx* c, cwg_error* err) {
  int rc = cwg_run_begin(c);
  if (rc) return rc;
  rc = cwg_run_steps(c, 0, c->n_steps);
  if (rc) return rc;
  return cwg_run_sync(c, err);
}

int cwg_get_info(cwg_ctx* c, cwg_info* i) {
  i->dt_effective = c->dt_eff;
  i->dt_s = c->dt_s;
  i->dt_ad = c->dt_ad;
  i->l = c->l;
  i->k_max_global = c->kmax_global;
  i->n_steps = c->n_steps;
  i->steps_per_record = c->spr;
  i->steps_per_map = c->spm;
  i->n_samples = c->n_samples;
  i->n_local = c->n_own;
  i->node_begin = c->own_global0;
  i->op_kind = c->op_kind;
  return CWG_OK;
}

int cwg_get_khist(cwg_ctx* c, int64_t* out, int len) {
  return guarded(nullptr, [&] {
    CUDA_TRY(cudaSetDevice(c->device));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    if (c->world > 1 && !c->loopback) {
      unsigned long long* tmp = dev_alloc<unsigned long long>(c->khist_len);
      NCCL_TRY(g_nccl.allreduce(c->d_khist, tmp, c->khist_len, ncclUint64, ncclSum, c->comm, c->stream));
      CUDA_TRY(cudaStreamSynchronize(c->stream));
      std::vector<unsigned long long> h(c->khist_len);
      CUDA_TRY(cudaMemcpy(h.data(), tmp, h.size() * sizeof(h[0]), cudaMemcpyDeviceToHost));
      dev_free(tmp);
      for (int k = 0; k < len; ++k) out[k] = k < c->khist_len ? static_cast<int64_t>(h[k]) : 0;
    } else {
      std::vector<unsigned long long> h(c->khist_len);
      CUDA_TRY(cudaMemcpy(h.data(), c->d_khist, h.size() * sizeof(h[0]), cudaMemcpyDeviceToHost));
      for (int k = 0; k < len; ++k) out[k] = k < c->khist_len ? static_cast<int64_t>(h[k]) : 0;
    }
  });
}

int cwg_get_traces(cwg_ctx* c, double* t_ms, double* v) {
  return guarded(nullptr, [&] {
    CUDA_TRY(cudaSetDevice(c->device));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    for (long long q = 0; q < c->n_samples; ++q) t_ms[q] = static_cast<double>(q * c->spr) * c->dt_eff;
    if (c->n_probes == 0) return;
    const size_t cnt = static_cast<size_t>(c->n_samples) * c->n_probes;
    double* src = c->d_traces;
    double* tmp = nullptr;
    if (c->world > 1 && !c->loopback) {  // non-owned probes are 0 on each rank
      tmp = dev_alloc<double>(cnt);
      NCCL_TRY(g_nccl.allreduce(c->d_traces, tmp, cnt, ncclDouble, ncclSum, c->comm, c->stream));
      CUDA_TRY(cudaStreamSynchronize(c->stream));
      src = tmp;
    }
    std::vector<double> h(cnt);
    CUDA_TRY(cudaMemcpy(h.data(), src, cnt * sizeof(double), cudaMemcpyDeviceToHost));
    if (tmp) dev_free(tmp);
    for (int p = 0; p < c->n_probes; ++p)
      for (long long q = 0; q < c->n_samples; ++q) v[p * c->n_samples + q] = h[q * c->n_probes + p];
  });
}

int cwg_get_maps(cwg_ctx* c, double* lat, uint8_t* lat_valid, double* apd, uint8_t* apd_valid) {
  return guarded(nullptr, [&] {
    CUDA_TRY(cudaSetDevice(c->device));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    // straight into the caller's arrays (no host temporaries); NaN where a map has
    // no value, filled on the device on the way out
    const size_t n = static_cast<size_t>(c->n_own);
    DevScope tmp;
    if (lat) {
      double* d = tmp.keep(dev_alloc<double>(n));
      CUDA_TRY(launch_map_values(c->det.lat, c->det.has_lat, static_cast<long long>(n), d, c->stream));
      CUDA_TRY(cudaMemcpyAsync(lat, d, n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    }
    if (apd) {
      double* d = tmp.keep(dev_alloc<double>(n));
      CUDA_TRY(launch_map_values(c->det.apd, c->det.has_apd, static_cast<long long>(n), d, c->stream));
      CUDA_TRY(cudaMemcpyAsync(apd, d, n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    }
    if (lat_valid) CUDA_TRY(cudaMemcpyAsync(lat_valid, c->det.has_lat, n, cudaMemcpyDeviceToHost, c->stream));
    if (apd_valid) CUDA_TRY(cudaMemcpyAsync(apd_valid, c->det.has_apd, n, cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
  });
}

// The whole result on every rank (run_simulation returns one SimulationResult,
// splitting.cpp:286-293): each rank stages its owned y-slab in a global-size
// device buffer and the ranks broadcast their slabs to each other (one NCCL
// group of in-place ncclBroadcast per array; slab r = cwg_slab_plan rows).
// world == 1 or loopback contexts: this context's own rows only (the
// loopback tests assemble the slabs themselves). Any output may be null.
int cwg_gather_result(cwg_ctx* c, double* v, double* s_aos, int stride, double* last, double* lat,
                      uint8_t* lat_valid, double* apd, uint8_t* apd_valid) {
  return guarded(nullptr, [&] {
    CUDA_TRY(cudaSetDevice(c->device));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    const bool multi = c->world > 1 && !c->loopback;
    if (!multi) {
      CUDA_TRY(cudaStreamSynchronize(c->stream));
      if (v || s_aos || last) {
        const int rc = cwg_download_state(c, v, s_aos, stride, last);
        if (rc != CWG_OK) throw Fail{rc, g_last_error};
      }
      std::vector<double> L(static_cast<size_t>(c->n_global)), A(static_cast<size_t>(c->n_global));
      std::vector<uint8_t> lv(static_cast<size_t>(c->n_global)), av(static_cast<size_t>(c->n_global));
      const int rc = cwg_get_maps(c, L.data() + c->own_global0, lv.data() + c->own_global0, A.data() + c->own_global0,
                                  av.data() + c->own_global0);
      if (rc != CWG_OK) throw Fail{rc, g_last_error};
      for (long long i = c->own_global0; i < c->own_global0 + c->n_own; ++i) {
        if (lat) lat[i] = L[static_cast<size_t>(i)];
        if (lat_valid) lat_valid[i] = lv[static_cast<size_t>(i)];
        if (apd) apd[i] = A[static_cast<size_t>(i)];
        if (apd_valid) apd_valid[i] = av[static_cast<size_t>(i)];
      }
      return;
    }
    validation(!s_aos || stride >= c->stride, "state: stride smaller than the largest model state count");
    const long long N = c->n_global;
    std::vector<std::pair<long long, long long>> slab(static_cast<size_t>(c->world));  // (first node, count)
    for (int r = 0; r < c->world; ++r) {
      int64_t rb = 0, re = 0;
      cwg_slab_plan(c->ny1, c->world, r, &rb, &re);
      slab[static_cast<size_t>(r)] = {rb * c->w, (re - rb) * c->w};
    }
    DevScope scope;
    auto bcast_all = [&](void* buf, size_t elem, ncclDataType_t type, long long per_node) {
      NCCL_TRY(g_nccl.gstart());
      for (int r = 0; r < c->world; ++r) {
        char* p = static_cast<char*>(buf) + static_cast<size_t>(slab[static_cast<size_t>(r)].first * per_node) * elem;
        NCCL_TRY(g_nccl.bcast(p, p, static_cast<size_t>(slab[static_cast<size_t>(r)].second * per_node), type, r,
                              c->comm, c->stream));
      }
      NCCL_TRY(g_nccl.gend());
    };
    auto gather_d = [&](const double* own, double* host) {
      double* d = scope.keep(dev_alloc<double>(static_cast<size_t>(N)));
      CUDA_TRY(cudaMemcpyAsync(d + c->own_global0, own, c->n_own * sizeof(double), cudaMemcpyDeviceToDevice,
                               c->stream));
      bcast_all(d, sizeof(double), ncclDouble, 1);
      CUDA_TRY(cudaMemcpyAsync(host, d, N * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
      CUDA_TRY(cudaStreamSynchronize(c->stream));
    };
    auto gather_u8 = [&](const unsigned char* own, uint8_t* host) {
      unsigned char* d = scope.keep(dev_alloc<unsigned char>(static_cast<size_t>(N)));
      CUDA_TRY(cudaMemcpyAsync(d + c->own_global0, own, c->n_own, cudaMemcpyDeviceToDevice, c->stream));
      bcast_all(d, 1, ncclUint8, 1);
      CUDA_TRY(cudaMemcpyAsync(host, d, N, cudaMemcpyDeviceToHost, c->stream));
      CUDA_TRY(cudaStreamSynchronize(c->stream));
    };
    if (v) gather_d(c->d_v[c->cur] + c->halo, v);
    if (last) gather_d(c->d_last + c->halo, last);
    if (s_aos) {
      double* d = scope.keep(dev_alloc<double>(static_cast<size_t>(N) * stride));
      CUDA_TRY(launch_soa_to_aos(c->d_S, c->pitch, c->halo, c->stride, c->n_own, d + c->own_global0 * stride, stride,
                                 c->stream));
      bcast_all(d, sizeof(double), ncclDouble, stride);
      CUDA_TRY(cudaMemcpyAsync(s_aos, d, static_cast<size_t>(N) * stride * sizeof(double), cudaMemcpyDeviceToHost,
                               c->stream));
      CUDA_TRY(cudaStreamSynchronize(c->stream));
    }
    std::vector<uint8_t> lv(static_cast<size_t>(N)), av(static_cast<size_t>(N));
    if (lat || lat_valid || apd || apd_valid) {
      gather_u8(c->det.has_lat, lv.data());
      gather_u8(c->det.has_apd, av.data());
    }
    if (lat) {
      gather_d(c->det.lat, lat);
      for (long long i = 0; i < N; ++i)
        if (!lv[static_cast<size_t>(i)]) lat[i] = std::nan("");
    }
    if (apd) {
      gather_d(c->det.apd, apd);
      for (long long i = 0; i < N; ++i)
        if (!av[static_cast<size_t>(i)]) apd[i] = std::nan("");
    }
    if (lat_valid) std::memcpy(lat_valid, lv.data(), static_cast<size_t>(N));
    if (apd_valid) std::memcpy(apd_valid, av.data(), static_cast<size_t>(N));
  });
}

void cwg_trim_pool(void) { dev_pool().trim(); }

int cwg_get_timing(cwg_ctx* c, double* r, double* d, double* rec) {
  *r = c->t_react;
  *d = c->t_diff;
  *rec = c->t_rec;
  return CWG_OK;
}

int64_t cwg_launch_count(cwg_ctx* c) { return c->launches; }

int cwg_react_trace(uint64_t* out, int n) {
  if (!g_react_trace || n < 0 || n > 16 * 4096) return CWG_EVALIDATION;
  if (cudaDeviceSynchronize() != cudaSuccess) return CWG_ECUDA;
  return cudaMemcpy(out, g_react_trace, static_cast<size_t>(n) * sizeof(uint64_t), cudaMemcpyDeviceToHost) ==
                 cudaSuccess ? CWG_OK : CWG_ECUDA;
}

int64_t cwg_reaction_evals(cwg_ctx* c) {
  std::vector<int64_t> h(static_cast<size_t>(c->khist_len));
  if (cwg_get_khist(c, h.data(), c->khist_len) != CWG_OK) return -1;
  int64_t s = 0;
  for (int k = 0; k < c->khist_len; ++k) s += static_cast<int64_t>(k) * h[k];
  return s;
}

int cwg_bench_steps(cwg_ctx* c, int64_t first, int64_t count, int64_t flush_bytes, int split_phases,
                    double* step_ms, double* react_ms, double* diff_ms) {
  return guarded(nullptr, [&] {
    CUDA_TRY(cudaSetDevice(c->device));
    validation(first >= 0 && first + count <= c->n_steps, "bench: step range outside [0, n_steps)");
    if (flush_bytes > 0 && static_cast<size_t>(flush_bytes) > c->flush_bytes) {
      if (c->d_flush) cudaFree(c->d_flush);
      CUDA_TRY(cudaMalloc(&c->d_flush, static_cast<size_t>(flush_bytes)));
      c->flush_bytes = static_cast<size_t>(flush_bytes);
    }
    constexpr int kChunk = 256;
    StepGraph graphs[8];
    std::vector<cudaEvent_t> ev(3 * kChunk);
    for (auto& e : ev) CUDA_TRY(cudaEventCreate(&e));
    try {
      for (int64_t b = 0; b < count; b += kChunk) {
        const int64_t m = std::min<int64_t>(kChunk, count - b);
        for (int64_t i = 0; i < m; ++i) {
          const long long step = first + b + i;
          if (flush_bytes > 0)
            CUDA_TRY(cudaMemsetAsync(c->d_flush, static_cast<int>(step & 0xff), static_cast<size_t>(flush_bytes),
                                     c->stream));
          {
            const long long l0 = c->launches;  // the clock write sits outside the timed events: not counted
            set_clock(c, step);
            c->launches = l0;
          }
          const bool middle = step >= 1 && step < c->n_steps - 1;
          if (middle && split_phases == 2) {  // plain step graph, events recorded on the stream around it
            StepGraph& sg = step_graph(c, step, graphs, false);
            CUDA_TRY(cudaEventRecord(ev[3 * i], c->stream));
            CUDA_TRY(cudaGraphLaunch(sg.exec, c->stream));
            CUDA_TRY(cudaEventRecord(ev[3 * i + 1], c->stream));
            CUDA_TRY(cudaEventRecord(ev[3 * i + 2], c->stream));
            c->cur = sg.cur_after;
            c->launches += sg.launches;
            continue;
          }
          if (middle && split_phases == 0) {
            StepGraph& sg = step_graph(c, step, graphs);
            for (int q = 0; q < 3; ++q)
              CUDA_TRY(cudaGraphExecEventRecordNodeSetEvent(sg.exec, sg.ev_nodes[q], ev[3 * i + q]));
            CUDA_TRY(cudaGraphLaunch(sg.exec, c->stream));
            c->cur = sg.cur_after;
            c->launches += sg.launches;
            continue;
          }
          CUDA_TRY(cudaEventRecord(ev[3 * i], c->stream));
          if (step == 0) enqueue_diffusion(c, c->l, 0, 0);
          enqueue_reaction(c, 0, c->l, false, 0.0);
          CUDA_TRY(cudaEventRecord(ev[3 * i + 1], c->stream));
          enqueue_diffusion(c, step == c->n_steps - 1 ? c->l : 2 * c->l, 0, c->l + 1);
          const long long S = step + 1;
          if (c->n_probes > 0 && S % c->spr == 0) {
            CUDA_TRY(launch_record_probes(c->d_v[c->cur], c->d_probe_loc, c->n_probes, c->d_traces, c->d_clock, 1,
                                          c->spr, c->stream));
            ++c->launches;
          }
          if (S % c->spm == 0) {
            CUDA_TRY(launch_detector_observe(c->d_v[c->cur] + c->halo, c->n_own, 0, c->det, c->d_clock, 1, c->spm,
                                             c->dt_eff, c->stream));
            ++c->launches;
          }
          CUDA_TRY(cudaEventRecord(ev[3 * i + 2], c->stream));
        }
        CUDA_TRY(cudaStreamSynchronize(c->stream));
        for (int64_t i = 0; i < m; ++i) {
          float a = 0, d = 0;
          CUDA_TRY(cudaEventElapsedTime(&a, ev[3 * i], ev[3 * i + 1]));
          CUDA_TRY(cudaEventElapsedTime(&d, ev[3 * i + 1], ev[3 * i + 2]));
          if (react_ms) react_ms[b + i] = a;
          if (diff_ms) diff_ms[b + i] = d;
          if (step_ms) step_ms[b + i] = static_cast<double>(a) + d;
        }
      }
    } catch (...) {
      for (auto& e : ev) cudaEventDestroy(e);
      for (auto& sg : graphs) free_step_graph(sg);
      throw;
    }
    for (auto& e : ev) cudaEventDestroy(e);
    for (auto& sg : graphs) free_step_graph(sg);
  });
}

double cwg_fp64_peak_tflops(int device, double seconds) {
  double result = -1.0;
  guarded(nullptr, [&] {
    CUDA_TRY(cudaSetDevice(device));
    cudaDeviceProp prop{};
    CUDA_TRY(cudaGetDeviceProperties(&prop, device));
    int occ = 0;
    occ = 8;  // 8 x 256 threads per SM
    const int blocks = prop.multiProcessorCount * occ;
    DevScope scope;
    double* out = scope.keep(dev_alloc<double>(1));
    cudaEvent_t a, b;
    CUDA_TRY(cudaEventCreate(&a));
    CUDA_TRY(cudaEventCreate(&b));
    int iters = 1 << 14;
    CUDA_TRY(launch_fp64_peak(out, blocks, iters, nullptr));  // warm-up
    CUDA_TRY(cudaDeviceSynchronize());
    float ms = 0;
    for (int rep = 0; rep < 6; ++rep) {
      CUDA_TRY(cudaEventRecord(a));
      CUDA_TRY(launch_fp64_peak(out, blocks, iters, nullptr));
      CUDA_TRY(cudaEventRecord(b));
      CUDA_TRY(cudaEventSynchronize(b));
      CUDA_TRY(cudaEventElapsedTime(&ms, a, b));
      if (ms > seconds * 1e3 / 4 || iters >= (1 << 24)) break;
      iters *= 2;
    }
    double best = 0.0;
    for (int rep = 0; rep < 5; ++rep) {
      CUDA_TRY(cudaEventRecord(a));
      CUDA_TRY(launch_fp64_peak(out, blocks, iters, nullptr));
      CUDA_TRY(cudaEventRecord(b));
      CUDA_TRY(cudaEventSynchronize(b));
      CUDA_TRY(cudaEventElapsedTime(&ms, a, b));
      const double flops = 2.0 * 8.0 * static_cast<double>(iters) * blocks * 256.0;
      best = std::max(best, flops / (ms * 1e-3) / 1e12);
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    result = best;
  });
  return result;
}

// ---------------------------------------------------------------- diastolic_threshold
namespace {

// One fixed-step probe run (stimulus.cpp:76-111) at `amp`; true when V[probe] > 0
// within the window. Chunks of G steps are replayed as a CUDA graph; the host
// checks the device crossing flag and the error record between chunks.
bool propagates(cwg_ctx* c, double amp, long long steps, cudaGraphExec_t& graph, long long G) {
  CUDA_TRY(cudaMemcpyAsync(c->d_samp, &amp, sizeof(double), cudaMemcpyHostToDevice, c->stream));
  c->cur = 0;
  for (const auto& b : c->bins) {
    double rest[64] = {0};
    cwg_model_rest_state(b.kind, rest);
    DevScope scope;
    double* d_rest = scope.keep(upload(rest, 64));
    CUDA_TRY(launch_init_rest(c->d_v[0], c->d_S, c->pitch, c->d_last, b.d_list, b.first, b.count, d_rest,
                              state_count(b.kind), c->stride, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
  }
  ErrRec none{kNoError, kNoSeq, 0, 0, nullptr, nullptr};
  CUDA_TRY(cudaMemcpyAsync(c->d_err, &none, sizeof(none), cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(cudaMemcpyAsync(c->d_err_dummy, &none, sizeof(none), cudaMemcpyHostToDevice, c->stream));
  const long long never = 0x7fffffffffffffffll;
  CUDA_TRY(cudaMemcpyAsync(c->d_cross, &never, sizeof(never), cudaMemcpyHostToDevice, c->stream));
  auto enqueue = [&](long long off) {
    enqueue_reaction(c, off, 0, false, 0.0);
    enqueue_diffusion(c, 1, off, 1);
    CUDA_TRY(launch_probe_cross(c->d_v[c->cur], c->probe_local, c->d_cross, c->d_clock, off, c->stream));
  };
  if (!graph) {  // capture G steps + clock tick (parity of V buffers: G even)
    cudaGraph_t g = nullptr;
    const int cur0 = c->cur;
    CUDA_TRY(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    for (long long off = 0; off < G; ++off) enqueue(off);
    CUDA_TRY(launch_tick_clock(c->d_clock, G, c->stream));
    CUDA_TRY(cudaStreamEndCapture(c->stream, &g));
    CUDA_TRY(cudaGraphInstantiate(&graph, g, 0));
    cudaGraphDestroy(g);
    if (c->cur != cur0) throw Fail{CWG_ECUDA, "threshold graph must preserve the V buffer parity"};
  }
  CUDA_TRY(launch_set_clock(c->d_clock, 0, c->stream));
  for (long long s = 0; s < steps;) {
    if (s + G <= steps) {
      CUDA_TRY(cudaGraphLaunch(graph, c->stream));
      c->launches += G * (static_cast<long long>(c->bins.size()) + 2) + 1;
      s += G;
    } else {  // tail steps, launched directly on a correctly set clock
      CUDA_TRY(launch_set_clock(c->d_clock, s, c->stream));
      enqueue(0);
      s += 1;
    }
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    long long cross = never;
    CUDA_TRY(cudaMemcpy(&cross, c->d_cross, sizeof(cross), cudaMemcpyDeviceToHost));
    ErrRec r{};
    CUDA_TRY(cudaMemcpy(&r, c->d_err, sizeof(r), cudaMemcpyDeviceToHost));
    const long long err_step = r.key == kNoError ? never : r.seq / c->evs;
    if (err_step != never && err_step <= cross) {  // the reaction of that step throws first
      const long long node = static_cast<long long>(r.key >> 22);
      char buf[160];
      std::snprintf(buf, sizeof(buf), "threshold probe run diverged (node %lld, t = %f ms)", node,
                    static_cast<double>(err_step) * c->dt);
      throw Fail{CWG_EINSTABILITY, buf};
    }
    if (cross != never && cross < steps) return true;
  }
  return false;
}

}  // namespace

extern "C" int cwg_diastolic_threshold(const cwg_problem* prob, const double* coords_xy, const int64_t* stim_nodes,
                                       int64_t n_stim, const cwg_threshold_options* opt, double* threshold,
                                       int64_t* probe_out, cwg_error* err) {
  cwg_ctx* c = nullptr;
  cudaGraphExec_t graph = nullptr;
  long long fail_node = -1;
  double fail_t = 0.0;
  const int rc = guarded(err, [&] {
    validation(prob && coords_xy && stim_nodes && opt, "threshold: missing arguments");
    validation(n_stim > 0, "threshold: stimulus node set is empty");
    validation(prob->world <= 1, "threshold: single device only");
    validation(prob->n_models == 1, "threshold: one cell model");
    const long long n = prob->n;
    std::vector<long long> sn(stim_nodes, stim_nodes + n_stim);
    std::sort(sn.begin(), sn.end());
    sn.erase(std::unique(sn.begin(), sn.end()), sn.end());
    for (long long i : sn) validation(i >= 0 && i < n, "threshold: stimulus node out of range");
    // probe: the node farthest from the stimulus region, required >= 1 cm away (stimulus.cpp:120-134)
    long long probe = -1;
    double best = -1.0;
    for (long long i = 0; i < n; ++i) {
      double dmin = std::numeric_limits<double>::infinity();
      for (long long q : sn) {
        const double dx = coords_xy[2 * i] - coords_xy[2 * q];
        const double dy = coords_xy[2 * i + 1] - coords_xy[2 * q + 1];
        dmin = std::min(dmin, std::hypot(dx, dy));
      }
      if (dmin > best) {
        best = dmin;
        probe = i;
      }
    }
    if (best < 1.0) throw Fail{CWG_EVALIDATION, "threshold: no probe node >= 1 cm from the stimulus region"};
    if (probe_out) *probe_out = probe;
    // fixed-step problem: dt = min(opt.dt, dt0/2, dt_s) (stimulus.cpp:90)
    const double dt = std::min({opt->dt_ms, stable_step(prob->model_kind[0]) / 2.0, prob->dt_s});
    const long long steps = static_cast<long long>(std::ceil(opt->window_ms / dt));
    cwg_problem p = *prob;
    std::vector<int32_t> ptr(static_cast<size_t>(n + 1), 0), ids(sn.size(), 0);
    for (long long i : sn) ptr[static_cast<size_t>(i + 1)] = 1;
    for (long long i = 0; i < n; ++i) ptr[static_cast<size_t>(i + 1)] += ptr[static_cast<size_t>(i)];
    const double t0 = 0.0, dur = opt->duration_ms, amp0 = 0.0, per = std::nan("");
    p.n_stim = 1;
    p.stim_t_start = &t0;
    p.stim_duration = &dur;
    p.stim_amplitude = &amp0;
    p.stim_period = &per;
    p.stim_node_ptr = ptr.data();
    p.stim_ids = ids.data();
    p.n_probes = 0;
    p.scheme = CWG_OST;
    p.dt_ms = dt;
    p.t_end_ms = static_cast<double>(steps) * dt;
    p.k0_up = 1;
    p.k0_down = 1;
    p.strict_substeps = 0;
    p.record_interval_ms = p.t_end_ms;
    p.map_interval_ms = p.t_end_ms;
    p.gkr_scale = nullptr;
    c = new cwg_ctx();
    create_impl(&p, c);
    c->fixed_step = true;
    c->dt_ad = dt;  // one diffusion sub-step of the full dt (stimulus.cpp:106)
    c->evs = 2;     // ev 0 reaction, ev 1 diffusion
    CUDA_TRY(launch_mass_factor_fix(c));
    c->d_err_dummy = dev_alloc<ErrRec>(1);
    {
      const ErrRec none{kNoError, kNoSeq, 0, 0, nullptr, nullptr};
      h2d(c->d_err_dummy, &none, sizeof(none));
    }
    c->d_cross = dev_alloc<long long>(1);
    c->probe_local = probe - c->node_offset;
    // bisection (stimulus.cpp:136-156)
    const long long G = 64;
    const double cap = opt->upper_factor * opt->initial_guess;
    double lo = 0.0, hi = opt->initial_guess;
    while (!propagates(c, hi, steps, graph, G)) {
      lo = hi;
      hi *= 2.0;
      if (hi > cap) throw Fail{CWG_EVALIDATION, "threshold: no propagation at upper bracket " + std::to_string(cap)};
    }
    while ((hi - lo) / hi > opt->rel_tol) {
      const double mid = 0.5 * (lo + hi);
      if (propagates(c, mid, steps, graph, G))
        hi = mid;
      else
        lo = mid;
    }
    *threshold = hi;
  });
  if (rc == CWG_EINSTABILITY && err) {
    // message carries node and time; parse them back for the structured fields
    long long node = -1;
    double t = 0.0;
    if (std::sscanf(err->msg, "threshold probe run diverged (node %lld, t = %lf", &node, &t) == 2) {
      fail_node = node;
      fail_t = t;
    }
    err->node = fail_node;
    err->t_ms = fail_t;
    err->phase = 1;
  }
  if (graph) cudaGraphExecDestroy(graph);
  ctx_free(c);
  return rc;
}

int cwg_diffusion_substep(int64_t n, const int64_t* rp, const int64_t* col, const double* val, const double* mass,
                          const double* v, double dt_sub, double* out, int device, cwg_error* err) {
  return guarded(err, [&] {
    CUDA_TRY(cudaSetDevice(device));
    const long long nnz = rp[n];
    DevScope ds;
    long long* d_rp = ds.keep(upload(reinterpret_cast<const long long*>(rp), n + 1));
    long long* d_col = ds.keep(upload(reinterpret_cast<const long long*>(col), nnz));
    double* d_val = ds.keep(upload(val, nnz));
    double* d_m = ds.keep(upload(mass, n));
    double* d_v = ds.keep(upload(v, n));
    double* d_o = ds.keep(dev_alloc<double>(n));
    CUDA_TRY(launch_diffuse_csr_plain(n, d_rp, d_col, d_val, d_m, d_v, dt_sub, d_o, nullptr));
    CUDA_TRY(cudaDeviceSynchronize());
    CUDA_TRY(cudaMemcpy(out, d_o, n * sizeof(double), cudaMemcpyDeviceToHost));
  });
}

int cwg_rates(int kind, int64_t n, const double* v, const double* s, const double* ist, double* dv, double* ds,
              int device, cwg_error* err) {
  return guarded(err, [&] {
    validation(state_count(kind) >= 0, "unknown cell model kind");
    CUDA_TRY(cudaSetDevice(device));
    const int ns = state_count(kind);
    DevScope scope;
    double* d_v = scope.keep(upload(v, n));
    double* d_s = scope.keep(upload(s, static_cast<size_t>(n) * ns));
    double* d_i = scope.keep(upload(ist, n));
    double* d_dv = scope.keep(dev_alloc<double>(n));
    double* d_ds = scope.keep(dev_alloc<double>(static_cast<size_t>(n) * ns));
    CUDA_TRY(is_ord(kind) ? launch_rates_ord(kind, n, d_v, d_s, d_i, d_dv, d_ds, nullptr)
                          : launch_rates_exact(kind, n, d_v, d_s, d_i, d_dv, d_ds, nullptr));
    CUDA_TRY(cudaDeviceSynchronize());
    CUDA_TRY(cudaMemcpy(dv, d_dv, n * sizeof(double), cudaMemcpyDeviceToHost));
    if (ns) CUDA_TRY(cudaMemcpy(ds, d_ds, static_cast<size_t>(n) * ns * sizeof(double), cudaMemcpyDeviceToHost));
  });
}

static const char* model_name(int kind) {
  switch (kind) {
    case CWG_MODEL_ALIEV_PANFILOV: return "aliev-panfilov";
    case CWG_MODEL_ORD_ENDO: return "ohara2011-endo";
    case CWG_MODEL_ORD_EPI: return "ohara2011-epi";
    case CWG_MODEL_ORD_MID: return "ohara2011-mid";
    case CWG_MODEL_MACCANNELL: return "maccannell2007";
    default: return "passive";
  }
}

int cwg_pace_cells(int kind, int64_t n, const double* cycle_ms, const double* amplitude, const double* duration_ms,
                   int n_beats, double* state_out, double* apd90_out, double* max_rel_out, int* status_out,
                   double* fail_t_out, int device, cwg_error* err) {
  int first_bad = -1, bad_status = 0, bad_beat = 0;
  double bad_t = 0.0;
  const int rc = guarded(err, [&] {
    validation(state_count(kind) >= 0, "unknown cell model kind");
    validation(n_beats >= 1, "pacing: n_beats must be >= 1");
    for (int64_t i = 0; i < n; ++i) validation(cycle_ms[i] > 0.0, "pacing: cycle length must be positive");
    if (n == 0) return;
    CUDA_TRY(cudaSetDevice(device));
    const int ns = state_count(kind);
    double rest[64];
    cwg_model_rest_state(kind, rest);
    PaceArgs a{};
    a.n = n;
    a.n_beats = n_beats;
    a.dt = stable_step(kind) / 2.0;  // ionic.cpp:127
    DevScope scope;
    a.cycle = scope.keep(upload(cycle_ms, n));
    a.amp = scope.keep(upload(amplitude, n));
    a.dur = scope.keep(upload(duration_ms, n));
    a.rest = scope.keep(upload(rest, static_cast<size_t>(ns) + 1));
    a.state_out = scope.keep(dev_alloc<double>(static_cast<size_t>(n) * (ns + 1)));
    a.prev_out = scope.keep(dev_alloc<double>(static_cast<size_t>(n) * (ns + 1)));
    a.apd_out = scope.keep(dev_alloc<double>(static_cast<size_t>(n) * n_beats));
    a.maxrel_out = scope.keep(dev_alloc<double>(n));
    a.status_out = scope.keep(dev_alloc<int>(n));
    a.beat_out = scope.keep(dev_alloc<int>(n));
    a.fail_t_out = scope.keep(dev_alloc<double>(n));
    CUDA_TRY(is_ord(kind) ? launch_pace_ord(kind, a, nullptr) : launch_pace_exact(kind, a, nullptr));
    CUDA_TRY(cudaDeviceSynchronize());
    std::vector<int> st(static_cast<size_t>(n)), beat(static_cast<size_t>(n));
    std::vector<double> ft(static_cast<size_t>(n));
    CUDA_TRY(cudaMemcpy(st.data(), a.status_out, n * sizeof(int), cudaMemcpyDeviceToHost));
    CUDA_TRY(cudaMemcpy(beat.data(), a.beat_out, n * sizeof(int), cudaMemcpyDeviceToHost));
    CUDA_TRY(cudaMemcpy(ft.data(), a.fail_t_out, n * sizeof(double), cudaMemcpyDeviceToHost));
    if (state_out)
      CUDA_TRY(cudaMemcpy(state_out, a.state_out, static_cast<size_t>(n) * (ns + 1) * sizeof(double),
                          cudaMemcpyDeviceToHost));
    if (apd90_out)
      CUDA_TRY(cudaMemcpy(apd90_out, a.apd_out, static_cast<size_t>(n) * n_beats * sizeof(double),
                          cudaMemcpyDeviceToHost));
    if (max_rel_out) CUDA_TRY(cudaMemcpy(max_rel_out, a.maxrel_out, n * sizeof(double), cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < n; ++i) {
      if (status_out) status_out[i] = st[static_cast<size_t>(i)] == 0 ? CWG_OK : CWG_EINSTABILITY;
      if (fail_t_out) fail_t_out[i] = st[static_cast<size_t>(i)] == 0 ? 0.0 : ft[static_cast<size_t>(i)];
      if (st[static_cast<size_t>(i)] != 0 && first_bad < 0) {
        first_bad = static_cast<int>(i);
        bad_status = st[static_cast<size_t>(i)];
        bad_beat = beat[static_cast<size_t>(i)];
        bad_t = ft[static_cast<size_t>(i)];
      }
    }
  });
  if (rc != CWG_OK || first_bad < 0) return rc;
  // the reference throws InstabilityError(msg, -1, t) (ionic.cpp:141-147)
  const std::string msg = bad_status == 2 ? std::string("pacing: ") + model_name(kind) + " diverged at beat " +
                                                std::to_string(bad_beat)
                                          : "pacing: |V| > 1000 mV at beat " + std::to_string(bad_beat);
  g_last_error = msg;
  if (err) {
    err->code = CWG_EINSTABILITY;
    err->node = -1;
    err->t_ms = bad_t;
    err->phase = 1;
    std::snprintf(err->msg, sizeof(err->msg), "%s", msg.c_str());
  }
  return CWG_EINSTABILITY;
}

}  // extern "C"
