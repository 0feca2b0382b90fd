// The reaction pass (StrangIntegrator::reaction_step, splitting.cpp:95-155) as
// one sm_100a kernel template per cell model.
//
// Work distribution ("lane refill"): each lane owns one node at a time and
// runs that node's k forward-Euler sub-steps; every loop trip is ONE rates()
// evaluation for every busy lane, so the expensive model code always runs
// warp-converged. A lane whose node finished its k sub-steps (or went
// non-finite) writes the node back and takes the next node position from a
// global counter with one warp-aggregated atomicAdd. Adaptive k therefore
// costs no divergence: a warp never waits for its slowest node (the
// reference's per-node k, splitting.cpp:116, makes the order of nodes
// irrelevant to the results, so the dynamic schedule stays bit-deterministic).
//
// State columns are stored in groups of four (common.cuh sidx); the needy
// lanes of one refill get consecutive node positions, so their 32-byte
// accesses coalesce.
#pragma once

#include "common.cuh"

namespace cwg {

// kSync (M::kBlockSync): the warps of the (single, persistent) block on an SM
// advance one rates() evaluation per loop trip in lockstep (one
// __syncthreads_or per trip). The ORd fast-path body is ~54 KB of SASS, larger than the
// 32 KB L1.5 instruction cache; warps that drift to different PCs thrash it
// (ncu: ~35% of stall cycles were instruction fetch). In lockstep every
// fetched line serves all warps.
// Launch shapes opt in to the one-trip-ahead claim (M::kPreclaim): it helps
// the latency regime (C2 reaction 53.2 -> 52.3 us) but adds spills to the
// 168-register lockstep shape (C3 +1.1%, C4 -0.6%).
template <class M>
__host__ __device__ constexpr bool preclaim_of() {
  if constexpr (requires { M::kPreclaim; }) return M::kPreclaim;
  return false;
}

template <class M>
__device__ __forceinline__ void react_body(const ReactArgs& a, unsigned* shist) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  const long long step = *a.clock + a.step_off;
  const double t = a.use_t_fixed ? a.t_fixed : static_cast<double>(step) * a.dt;  // splitting.cpp:270
  const long long seq = step * a.evs + a.ev;

  int node = -1;  // local node index (< 2^31: a rank holds at most ~2.7e8 ORd nodes in 180 GB)
  bool open = true;  // may still receive work
  int k = 0, j = 0, p0 = 0, p1 = 0;
  double h = 0.0, v = 0.0, dv = 0.0, g = 1.0;
  double s[M::NS > 0 ? M::NS : 1];  // the lane's node states (registers)

  // First round: position = global thread index (no atomic: ~1,200 warps
  // claiming from one counter at once serialise in L2; ncu put 4% of the C2
  // kernel's stall samples on that claim). Refills then take positions
  // nthreads, nthreads + 1, ... from the counter, claimed one trip ahead:
  // lanes that will finish their node in this trip (j + 1 == k) claim their
  // next position before the evaluation, so the atomic's round trip hides
  // behind it (shapes with M::kPreclaim; CWG_PRECLAIM=0 claims at refill
  // time instead).
  const unsigned nthreads = gridDim.x * blockDim.x;
  bool first = true;
  long long nxt = -1;  // pre-claimed next position, -1: none
  while (true) {
    const bool need = node < 0 && open;
    const bool need_claim = need && nxt < 0;
    const unsigned m = __ballot_sync(kFull, need_claim);
    long long pos = nxt;
    if (m) {
      const int leader = __ffs(m) - 1;
      unsigned base = 0;
      if (first) {
        base = blockIdx.x * blockDim.x + (threadIdx.x & ~31u);
      } else {
        if (lane == leader) base = atomicAdd(a.counter, static_cast<unsigned>(__popc(m))) + nthreads;
        base = __shfl_sync(kFull, base, leader);
      }
      if (need_claim) pos = static_cast<long long>(base) + __popc(m & lt);  // first trip: m is full, so + lane
    }
    first = false;
    if (need) {
      nxt = -1;
      {
        if (pos < a.count) {
          node = a.list ? __ldg(a.list + pos) : static_cast<int>(a.first + pos);
          v = a.v[node];
          const double last = a.last[node];
          k = substeps(last, a.scheme, a.k0_up, a.k0_down, a.kmax);
          h = a.dt / static_cast<double>(k);  // dt_ar (splitting.cpp:117)
          j = 0;
          dv = 0.0;
          {
            const double* sp = a.S + 4ll * node;  // column group q / 4 at sp + (q & ~3) * pitch (sidx)
#pragma unroll
            for (int q = 0; q + 3 < M::NS; q += 4) ld_state4(sp + q * a.pitch, s[q], s[q + 1], s[q + 2], s[q + 3]);
#pragma unroll
            for (int q = M::NS & ~3; q < M::NS; ++q) s[q] = sp[(q & ~3) * a.pitch + (q & 3)];
          }
          if (a.stim.node_ptr) {
            p0 = __ldg(a.stim.node_ptr + node);
            p1 = __ldg(a.stim.node_ptr + node + 1);
          }
          if (M::kUsesGkr) g = a.gkr ? __ldg(a.gkr + node) : 1.0;
          atomicAdd(shist + k, 1u);
        } else {
          open = false;
        }
      }
    }
    if (preclaim_of<M>() && a.preclaim) {
      const bool want = node >= 0 && j + 1 == k && open;
      const unsigned m2 = __ballot_sync(kFull, want);
      if (m2) {
        const int leader = __ffs(m2) - 1;
        unsigned base = 0;
        if (lane == leader) base = atomicAdd(a.counter, static_cast<unsigned>(__popc(m2))) + nthreads;
        base = __shfl_sync(kFull, base, leader);
        if (want) nxt = static_cast<long long>(base) + __popc(m2 & lt);
      }
    }
    if (M::kBlockSync) {
      if (!__syncthreads_or(node >= 0)) break;
    } else if (!__any_sync(kFull, node >= 0)) {
      break;
    }
    if (node >= 0) {
      const double ts = __dadd_rn(t, __dmul_rn(static_cast<double>(j), h));  // t + j*dt_ar, never contracted
      const double ist = p1 > p0 ? stim_current(a.stim, p0, p1, ts) : 0.0;
      M::advance(v, s, ist, g, h, dv);
      ++j;
      const bool bad = !isfinite(v);
      if (bad) {
        const unsigned long long key = (static_cast<unsigned long long>(node + a.node_offset) << 22) |
                                       (static_cast<unsigned long long>(k) << 11) |
                                       static_cast<unsigned long long>(j - 1);
        record_failure(a.err, key, seq, 1, 1, a.v, a.v);
      }
      if (bad || j == k) {
        a.v[node] = v;
        a.last[node] = dv;  // dv at the start of the last sub-step (splitting.cpp:143)
        {
          double* sp = a.S + 4ll * node;
#pragma unroll
          for (int q = 0; q + 3 < M::NS; q += 4) st_state4(sp + q * a.pitch, s[q], s[q + 1], s[q + 2], s[q + 3]);
#pragma unroll
          for (int q = M::NS & ~3; q < M::NS; ++q) sp[(q & ~3) * a.pitch + (q & 3)] = s[q];
        }
        node = -1;
      }
    }
  }
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

template <class M>
__global__ void __launch_bounds__(M::kThreads, M::kMinBlocks) react_kernel(ReactArgs a) {
  extern __shared__ __align__(16) unsigned shist[];
  if (a.trace && threadIdx.x == 0) a.trace[blockIdx.x * 16 + 15] = gtimer();  // block start
  // A strictly earlier event failed: skip the work (uniform across the grid,
  // common.cuh earlier_failure) but still arrive on `done` below, so the
  // self-resetting work counter is reset by the last block either way.
  const bool skip = earlier_failure(a.err, (*a.clock + a.step_off) * a.evs + a.ev);
  if (!skip) {
    for (int i = threadIdx.x; i < a.khist_len; i += blockDim.x) shist[i] = 0u;
    if constexpr (requires { M::block_init(); }) M::block_init();  // e.g. the exp table (fastmath.cuh)
    __syncthreads();
    react_body<M>(a, shist);
    __syncthreads();
    for (int i = threadIdx.x; i < a.khist_len; i += blockDim.x)
      if (shist[i]) atomicAdd(a.khist + i, static_cast<unsigned long long>(shist[i]));
  }
  if (a.trace && threadIdx.x == 0) a.trace[blockIdx.x * 16] = gtimer();  // block's reaction done
  if (threadIdx.x == 0) {
    // acq_rel: this block's claims happen before its arrival; the last block
    // to arrive sees every block's claims before it resets the counters
    unsigned prev;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(a.done) : "memory");
    if (prev == gridDim.x - 1) {  // last block out resets the work counter for the next launch
      *a.counter = 0u;
      *a.done = 0u;
    }
  }
}

}  // namespace cwg

namespace cwg {

// ---------------------------------------------------------------------------
// Single-cell pacing to steady state (pace_to_steady_state, ionic.cpp:122-165),
// batched: one thread per request (model kind fixed per launch; cycle length,
// amplitude and duration per request). Forward Euler at dt = dt0 / 2 through
// the same M::advance as the reaction pass; per-beat APD90 markers
// (BeatMarkers, ionic.cpp:86-118) with the reference's operation order, every
// product and sum rounded explicitly so the TU's contraction setting does not
// matter.
// ---------------------------------------------------------------------------

template <class M>
__global__ void __launch_bounds__(64) pace_kernel(PaceArgs a) {
  if constexpr (requires { M::block_init(); }) M::block_init();
  __syncthreads();
  const long long r = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (r >= a.n) return;
  constexpr int NS = M::NS > 0 ? M::NS : 1;
  double s[NS];
  double v = a.rest[0];
#pragma unroll
  for (int q = 0; q < M::NS; ++q) s[q] = a.rest[1 + q];
  const double cycle = a.cycle[r], amp = a.amp[r], dur = a.dur[r], dt = a.dt;
  const long long spb = llround(cycle / dt);
  const double inf = __longlong_as_double(0x7ff0000000000000ll), nan = __longlong_as_double(0x7ff8000000000000ll);
  a.status_out[r] = 0;
  for (int beat = 0; beat < a.n_beats; ++beat) {
    const double v_rest = v;
    double max_slope = -inf, t_max = nan, v_peak = -inf, apd = nan;
    bool closed = false;
    double v_prev = v;
    for (long long i = 0; i < spb; ++i) {
      const double t_in = __dmul_rn(static_cast<double>(i), dt);
      const double ist = t_in < dur ? amp : 0.0;
      double dv;
      M::advance(v, s, ist, 1.0, dt, dv);
      if (!isfinite(v) || fabs(v) > 1000.0) {
        a.status_out[r] = isfinite(v) ? 3 : 2;
        a.beat_out[r] = beat;
        a.fail_t_out[r] = __dadd_rn(__dmul_rn(static_cast<double>(beat), cycle), t_in);
        return;
      }
      if (!closed) {
        const double t = __dadd_rn(t_in, dt);
        const double slope = __ddiv_rn(__dsub_rn(v, v_prev), dt);
        if (slope > max_slope) {
          max_slope = slope;
          t_max = t;
        }
        if (v > v_peak) v_peak = v;
        if (isfinite(t_max) && v_peak > 0.0) {
          const double v90 = __dsub_rn(v_peak, __dmul_rn(0.9, __dsub_rn(v_peak, v_rest)));
          if (v < v90 && __dsub_rn(v_peak, v_rest) > 20.0) {
            apd = __dsub_rn(t, t_max);
            closed = true;
          }
        }
      }
      v_prev = v;
    }
    a.apd_out[r * a.n_beats + beat] = apd;
    if (beat == a.n_beats - 2) {
      double* pv = a.prev_out + r * (M::NS + 1);
      pv[0] = v;
#pragma unroll
      for (int q = 0; q < M::NS; ++q) pv[1 + q] = s[q];
    }
  }
  double* out = a.state_out + r * (M::NS + 1);
  out[0] = v;
#pragma unroll
  for (int q = 0; q < M::NS; ++q) out[1 + q] = s[q];
  double max_rel = 0.0;
  if (a.n_beats >= 2) {
    const double* pv = a.prev_out + r * (M::NS + 1);
    for (int k = 0; k <= M::NS; ++k) {
      const double e = out[k], p = pv[k];
      const double scale = fmax(fabs(p), fabs(e));
      if (scale > 1e-12) max_rel = fmax(max_rel, __ddiv_rn(fabs(__dsub_rn(e, p)), scale));
    }
  }
  a.maxrel_out[r] = max_rel;
}

template <class M>
cudaError_t launch_pace_t(const PaceArgs& a, cudaStream_t st) {
  if (a.n == 0) return cudaSuccess;
  pace_kernel<M><<<static_cast<unsigned>((a.n + 63) / 64), 64, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace cwg
