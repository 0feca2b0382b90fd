// Two-warp ORd reaction kernel for the latency regime (small meshes such as
// BASELINE config 2, where one node per lane leaves ~8 warps per SM and every
// warp stalls on its dependent FP64 chains).
//
// Each node is evaluated by a lane PAIR: lane l of warp A (group A: INa, INaL,
// Ito, ICaL and their 24 gates) and lane l of warp B (group B: IKr, IKs, IK1,
// NaCa, NaK, background currents, then the SR fluxes, concentrations and V).
// Different warps may run different code without SIMT divergence; they meet at
// two per-pair named barriers per rates() evaluation:
//   B publishes V + the concentrations A needs  --bar-->  A and B evaluate
//   their groups; A publishes its 5 currents    --bar-->  B finishes the step.
// Warp B owns the node (refill, stimulus, k, failure record, write-back of V,
// last_dvdt and its 16 states); warp A writes back its 24 gates when B moves
// its lane to a new node. Arithmetic is exactly that of step() (same pieces,
// same order), so results equal the one-warp kernel's.
#pragma once

#include "react.cuh"

namespace cwg {

constexpr int kPairWarps = 8;  // 4 pairs per 256-thread block

struct PairShm {
  double cur[5][32];  // A -> B: i_na(+INaL), i_to, i_cal, i_cana, i_cak
  double sh[7][32];   // B -> A: V, nai, ki, cass, nass, kss, CaMKt
  double hh[32];      // B -> A: dt_ar = dt / k of the lane's node
  long long node[32]; // B -> A: lane's node (-1 none)
  int status;         // B -> A: 1 = pair finished
  int pad;
};

__device__ __forceinline__ void pair_bar(int id) { asm volatile("bar.sync %0, 64;" ::"r"(id) : "memory"); }

// group A state indices (ord::StateIndex)
__device__ __forceinline__ constexpr int a_state(int q) {
  // INa/INaL gates M..HLP (8..16), Ito A..ISP (17..22), ICaL D..FCAFP (23..31)
  return 8 + q;
}
constexpr int kNA = 24;   // group A states: indices 8..31
constexpr int kB0 = 32;   // group B gates XRF..CAMKT (32..39) + concentrations 0..7

template <int CT>
__global__ void __launch_bounds__(kPairWarps * 32, 2) react_pair_kernel(ReactArgs a) {
  extern __shared__ __align__(16) unsigned shist[];
  PairShm* pshm = reinterpret_cast<PairShm*>(shist + ((a.khist_len + 3) & ~3));
  {
    const long long seq = (*a.clock + a.step_off) * a.evs + a.ev;
    if (earlier_failure(a.err, seq)) return;
  }
  for (int i = threadIdx.x; i < a.khist_len; i += blockDim.x) shist[i] = 0u;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pid = warp >> 1;
  const bool roleB = warp & 1;
  PairShm& P = pshm[pid];
  if (roleB && lane == 0) P.status = 0;
  exp_table_init();
  __syncthreads();

  const long long step = *a.clock + a.step_off;
  const double t = a.use_t_fixed ? a.t_fixed : static_cast<double>(step) * a.dt;
  const long long seq = step * a.evs + a.ev;
  const unsigned lt = (1u << lane) - 1u;

  long long node = -1;
  bool open = true;
  int k = 0, j = 0, p0 = 0, p1 = 0;
  double h = 0.0, v = 0.0, dv = 0.0, g = 1.0;
  double s[ord::NSTATE];  // each role touches only its own indices (+ the shared copies for A)

  while (true) {
    // ---------------------------------------------------------------- B: refill + publish
    if (roleB) {
      const bool need = node < 0 && open;
      const unsigned m = __ballot_sync(kFull, need);
      if (m) {
        const int leader = __ffs(m) - 1;
        unsigned base = 0;
        if (lane == leader) base = atomicAdd(a.counter, static_cast<unsigned>(__popc(m)));
        base = __shfl_sync(kFull, base, leader);
        if (need) {
          const long long pos = static_cast<long long>(base) + __popc(m & lt);
          if (pos < a.count) {
            node = a.list ? static_cast<long long>(__ldg(a.list + pos)) : a.first + pos;
            v = a.v[node];
            k = substeps(a.last[node], a.scheme, a.k0_up, a.k0_down, a.kmax);
            h = a.dt / static_cast<double>(k);
            j = 0;
            dv = 0.0;
#pragma unroll
            for (int q = 0; q < 8; ++q) s[q] = a.S[q * a.pitch + node];
#pragma unroll
            for (int q = kB0; q < ord::NSTATE; ++q) s[q] = a.S[q * a.pitch + node];
            if (a.stim.node_ptr) {
              p0 = __ldg(a.stim.node_ptr + node);
              p1 = __ldg(a.stim.node_ptr + node + 1);
            }
            g = a.gkr ? __ldg(a.gkr + node) : 1.0;
            atomicAdd(shist + k, 1u);
          } else {
            open = false;
          }
        }
      }
      P.node[lane] = node;
      if (node >= 0) {
        P.hh[lane] = h;
        P.sh[0][lane] = v;
        P.sh[1][lane] = s[ord::NAI];
        P.sh[2][lane] = s[ord::KI];
        P.sh[3][lane] = s[ord::CASS];
        P.sh[4][lane] = s[ord::NASS];
        P.sh[5][lane] = s[ord::KSS];
        P.sh[6][lane] = s[ord::CAMKT];
      }
      const bool any = __any_sync(kFull, node >= 0);
      if (lane == 0) P.status = any ? 0 : 1;
    }
    pair_bar(pid + 1);
    // ---------------------------------------------------------------- A: follow B's assignment
    if (!roleB) {
      const long long nb = P.node[lane];
      if (nb != node) {
        if (node >= 0) {  // B finished this lane's previous node: write back group A gates
#pragma unroll
          for (int q = 0; q < kNA; ++q) a.S[a_state(q) * a.pitch + node] = s[a_state(q)];
        }
        node = nb;
        if (node >= 0) {
#pragma unroll
          for (int q = 0; q < kNA; ++q) s[a_state(q)] = a.S[a_state(q) * a.pitch + node];
        }
      }
      if (node >= 0) {
        h = P.hh[lane];
        v = P.sh[0][lane];
        s[ord::NAI] = P.sh[1][lane];
        s[ord::KI] = P.sh[2][lane];
        s[ord::CASS] = P.sh[3][lane];
        s[ord::NASS] = P.sh[4][lane];
        s[ord::KSS] = P.sh[5][lane];
        s[ord::CAMKT] = P.sh[6][lane];
      }
    }
    if (P.status) break;  // uniform across the pair (written before the barrier)
    // ---------------------------------------------------------------- evaluate
    const bool fast = fabs(v) <= 130.0;
    ord::CurA ca{};
    ord::CurB cb{};
    ord::Pro pr{};
    if (node >= 0) {
      if (fast)
        pr = ord::prologue<CT, true>(v, s);
      else
        pr = ord::prologue<CT, false>(v, s);
      if (!roleB) {
        ca = fast ? ord::group_a<CT, false, true>(v, s, nullptr, pr, h)
                  : ord::group_a<CT, false, false>(v, s, nullptr, pr, h);
        P.cur[0][lane] = ca.i_na;
        P.cur[1][lane] = ca.i_to;
        P.cur[2][lane] = ca.i_cal;
        P.cur[3][lane] = ca.i_cana;
        P.cur[4][lane] = ca.i_cak;
      } else {
        cb = fast ? ord::group_b<CT, false, true>(v, s, nullptr, pr, h, g)
                  : ord::group_b<CT, false, false>(v, s, nullptr, pr, h, g);
      }
    }
    pair_bar(pid + 1);
    if (roleB && node >= 0) {
      ca.i_na = P.cur[0][lane];
      ca.i_to = P.cur[1][lane];
      ca.i_cal = P.cur[2][lane];
      ca.i_cana = P.cur[3][lane];
      ca.i_cak = P.cur[4][lane];
      const double ts = __dadd_rn(t, __dmul_rn(static_cast<double>(j), h));  // t + j*dt_ar
      const double ist = p1 > p0 ? stim_current(a.stim, p0, p1, ts) : 0.0;
      ord::finish<CT, false>(v, s, nullptr, pr, ca, cb, ist, h, dv);
      ++j;
      const bool bad = !isfinite(v);
      if (bad) {
        const unsigned long long key = (static_cast<unsigned long long>(node + a.node_offset) << 22) |
                                       (static_cast<unsigned long long>(k) << 11) |
                                       static_cast<unsigned long long>(j - 1);
        record_failure(a.err, key, seq, 1);
      }
      if (bad || j == k) {
        a.v[node] = v;
        a.last[node] = dv;
#pragma unroll
        for (int q = 0; q < 8; ++q) a.S[q * a.pitch + node] = s[q];
#pragma unroll
        for (int q = kB0; q < ord::NSTATE; ++q) a.S[q * a.pitch + node] = s[q];
        node = -1;
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < a.khist_len; i += blockDim.x)
    if (shist[i]) atomicAdd(a.khist + i, static_cast<unsigned long long>(shist[i]));
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned prev = atomicAdd(a.done, 1u);
    if (prev == gridDim.x - 1) {
      *a.counter = 0u;
      *a.done = 0u;
      __threadfence();
    }
  }
}

}  // namespace cwg
