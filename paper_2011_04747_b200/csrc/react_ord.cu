// O'Hara-Rudy 2011 reaction kernels (ohara_rudy_2011.cpp:85-444) for sm_100a.
//
// The model is FP64-pipe bound (libdevice exp/log/expm1 are DFMA polynomials,
// IEEE reciprocals are MUFU.RCP64H + DFMA Newton steps). This formulation is
// mathematically identical to the reference but spends fewer FP64
// instructions per evaluation:
//   * division by a constant  -> multiplication by its (compile-time) reciprocal;
//   * gates integrate (x_inf - x) * rate with rate = 1/tau taken directly
//     where tau is written as 1/(a e^u + b e^w) (no division at all);
//   * 1/(1 + a/x) style terms are rewritten as x/(x + a) (one reciprocal);
//   * e^x, e^2x, expm1(2x) for the GHK terms derive from one expm1(x); the
//     reciprocal-pair exponentials (tff, tfcaf) share one exp;
//   * pow(x, 2|3|8) are products, pow(3.8e-5/cai, 1.4) is one fexp(log);
//   * Nernst potentials log(c_o / c_i) = log(c_o) - log(c_i) (no reciprocal);
//   * every reciprocal is the MUFU seed + one cubic Newton step (3 DFMA,
//     faithful, fastmath.cuh rcp_nc / rcp_g) instead of __drcp_rn's 5;
//   * on the fast path: exponentials whose slopes are commensurate come from
//     one another (e^((v+70)/20) gives the (v+70)/5, (v+20)/10, (v-10)/10 and
//     (v-50)/20 terms by products), rates 1 / (c + 1 / s) are s / (c s + 1),
//     coefficients a e^u ride in the exponent as e^(u + log a), and the NCX /
//     INaK cycle algebra is factored (tools/refill_cost_probe.py, DESIGN.md
//     3.1: ~100 FP64 instructions fewer per evaluation).
// It therefore agrees with the reference to rounding, not bitwise; the parity
// contract for ORd is max|dV| <= 1e-6 mV (tests/test_gpu_parity.py), which
// the survey's +-1-ulp experiment shows is met with ~8 orders of margin.
//
// Register pressure: every gate is forward-Euler-updated in place right after
// the last current that reads its old value (exact FE semantics: each gate's
// derivative depends only on V and itself), so old and new gate values are
// never live together; concentrations, which every current reads, are updated
// last. The FE update itself (x + h*dx) is never contracted.
#include <cstdlib>

#include "fastmath.cuh"
#include "launch.h"
#include "react.cuh"

namespace cwg {
namespace ord {

constexpr double F = 96485.0;
constexpr double RT = 8314.0 * 310.0;
constexpr double RTF = RT / F;
constexpr double FRT = F / RT;
constexpr double NAO = 140.0, CAO = 1.8, KO = 5.4;
constexpr double VCELL = 1000.0 * 3.14 * 0.0011 * 0.0011 * 0.01;
constexpr double AGEO = 2.0 * 3.14 * 0.0011 * 0.0011 + 2.0 * 3.14 * 0.0011 * 0.01;
constexpr double ACAP = 2.0 * AGEO;
constexpr double VMYO = 0.68 * VCELL, VNSR = 0.0552 * VCELL, VJSR = 0.0048 * VCELL, VSS = 0.02 * VCELL;

// Concentration-dependent reciprocals and logs: on the fast path (FP: |V| <= 130
// mV AND every concentration in the range conc_ok() checks) each argument is
// provably a normal, finite, positive number, so the unchecked forms give the
// same bits as the checked ones without a branch per call; otherwise the
// checked forms keep IEEE special values (the abort step depends on them).
template <bool FP>
__device__ __forceinline__ double crcp(double x) { return FP ? rcp_nc(x) : rcp_g(x); }
template <bool FP>
__device__ __forceinline__ double clog(double x) { return FP ? flog_nc(x) : flog(x); }

// FP = true ("fast" evaluation, taken when |V| <= 130 mV): every exponent
// argument that depends on V alone is then provably < 708 in magnitude and
// every V-dependent denominator is a normal positive number, so those calls
// use the branch-free fexp_nc / rcp_nc. Concentration-dependent reciprocals
// and exponentials always use the checked forms (they can reach 0 / Inf /
// NaN while a node blows up, where IEEE semantics decide the abort step).
// s (v + a) / b written as fma(v, s / b, s a / b) with both constants folded:
// one FP64 instruction per exponent argument instead of an add and a multiply
// (absolute error ~ulp(a / b), i.e. a few ulp of the exponential near x = 0)
__device__ __forceinline__ double lin(double v, double slope, double offset) { return fma(v, slope, offset); }
template <bool FP>
__device__ __forceinline__ double vexp(double x) { return FP ? fexp_nc(x) : fexp(x); }
template <bool FP>
__device__ __forceinline__ double vrcp(double x) { return FP ? rcp_nc(x) : rcp_g(x); }
template <bool FP>
__device__ __forceinline__ double sigm(double u) { return vrcp<FP>(1.0 + vexp<FP>(u)); }  // 1/(1+e^u)
template <bool FP, int N>
__device__ __forceinline__ void vexp_n(double (&x)[N]) {
  if (FP) {
    fexp_nc_n(x);
  } else {
#pragma unroll
    for (int i = 0; i < N; ++i) x[i] = fexp(x[i]);
  }
}
template <bool FP, int N>
__device__ __forceinline__ void vrcp_n(double (&x)[N]) {
  if (FP) {
    rcp_nc_n(x);
  } else {
#pragma unroll
    for (int i = 0; i < N; ++i) x[i] = rcp_g(x[i]);
  }
}

template <int CT>  // 0 endo, 1 epi, 2 mid (ohara_rudy_2011.cpp:86-87 celltype_)
struct Var {
  static constexpr bool epi = CT == 1, mid = CT == 2;
  static constexpr double gnal = 0.0075 * (epi ? 0.6 : 1.0);
  static constexpr double gto = 0.02 * ((epi || mid) ? 4.0 : 1.0);
  static constexpr double pca = 0.0001 * (epi ? 1.2 : (mid ? 2.5 : 1.0));
  static constexpr double gkr = 0.046 * (epi ? 1.3 : (mid ? 0.8 : 1.0));
  static constexpr double gks = 0.0034 * (epi ? 1.4 : 1.0);
  static constexpr double gk1 = 0.1908 * (epi ? 1.2 : (mid ? 1.3 : 1.0));
  static constexpr double gncx = 0.0008 * (epi ? 1.1 : (mid ? 1.4 : 1.0));
  static constexpr double pnak = 30.0 * (epi ? 0.9 : (mid ? 0.7 : 1.0));
  static constexpr double gkb = 0.003 * (epi ? 0.6 : 1.0);
  static constexpr double jrel = mid ? 1.7 : 1.0;
  static constexpr double jup = epi ? 1.3 : 1.0;
  static constexpr double cmdn = 0.05 * (epi ? 1.3 : 1.0);
};

// x / expm1(x) given em = expm1(x) (ohara_rudy_2011.cpp:67-70)
template <bool FP>
__device__ __forceinline__ double xem1(double x, double em) {
  const bool small = fabs(x) < 1e-8;
  const double r = vrcp<FP>(small ? 1.0 + 0.5 * x : em);  // one reciprocal for both branches
  return small ? r : x * r;
}

struct NcxShared {
  double hna, hca6, h8, h9;  // hca6 = 6e4 / hca
};

// Na/Ca exchanger flux for one compartment (ohara_rudy_2011.cpp:264-300)
template <bool FP>
__device__ __forceinline__ double ncx(double na, double ca, const NcxShared& c) {
  constexpr double h10 = 12.5 + 1.0 + NAO / 15.0 * (1.0 + NAO / 5.0);
  constexpr double h11 = NAO * NAO / (h10 * 15.0 * 5.0);
  constexpr double k1 = 1.0 / h10 * CAO * 1.5e6;
  constexpr double k2 = 5.0e3, k5 = 5.0e3;
  const double r1 = crcp<FP>(1.0 + na * (1.0 / 88.12) * (1.0 + c.hna));
  const double r4 = crcp<FP>(1.0 + na * (1.0 / 15.0) * (1.0 + na * (1.0 / 5.0)));
  const double k3pp = c.h8 * 5.0e3;
  const double k3 = c.h9 * 6.0e4 + k3pp;
  const double k4pp = (na * (5.0e3 / 88.12)) * c.hna * r1;  // h2 k4pp_rate, h2 = na hna / 88.12 r1
  const double k4 = r1 * c.hca6 + k4pp;                     // h3 wca = r1 / hca, times 6e4
  const double k6 = r4 * (ca * 1.5e6);
  const double k7 = (na * na) * (6.0e4 / (75.0 * 5.0e3)) * r4 * k4pp;  // h5 h2 wna, h5 = na^2 / 75 r4
  const double k8 = c.h8 * h11 * 6.0e4;
  const double x1 = k2 * k4 * (k7 + k6) + k5 * k7 * (k2 + k3);
  const double x2 = k1 * k7 * (k4 + k5) + k4 * k6 * (k1 + k8);
  const double x3 = k1 * k3 * (k7 + k6) + k8 * k6 * (k2 + k3);
  const double x4 = k2 * k8 * (k4 + k5) + k3 * k5 * (k1 + k8);
  const double ca2 = ca * ca;
  const double j_na = 3.0 * (x4 * k7 - x1 * k8) + x3 * k4pp - x2 * k3pp;
  const double j_ca = x2 * k2 - x1 * k1;
  if (FP)  // allo / (x1 + .. + x4) with one reciprocal of the product (ca2 <= 1e20, the sum <= ~1e25 on the fast path)
    return ca2 * crcp<FP>((ca2 + 150.0e-6 * 150.0e-6) * (x1 + x2 + x3 + x4)) * (j_na + 2.0 * j_ca);
  const double rt = crcp<FP>(x1 + x2 + x3 + x4);
  const double allo = ca2 * crcp<FP>(ca2 + 150.0e-6 * 150.0e-6);
  return allo * rt * (j_na + 2.0 * j_ca);
}

// State indices (StateIndex, ohara_rudy_2011.cpp:18-26)
enum {
  NAI, NASS, KI, KSS, CAI, CASS, CANSR, CAJSR, M, HF, HS, J, HSP, JP, ML, HL, HLP, A, IF, IS, AP, IFP, ISP,
  D, FF, FS, FCAF, FCAS, JCA, NCA, FFP, FCAFP, XRF, XRS, XS1, XS2, XK1, JRELNP, JRELP, CAMKT, NSTATE
};

// State FE updates (SA: register array or shared-memory column).
// Output policy: R = false integrates in place; R = true only reports dx
// (CellModel::rates semantics, for cwg_rates).
#ifndef CWG_ORD_FMA_UPDATE
#define CWG_ORD_FMA_UPDATE 1
#endif
// x += h * dx. With CWG_ORD_FMA_UPDATE the update is one fused multiply-add
// (the exact x + h dx rounded once, where the reference rounds h dx first):
// one FP64 instruction and one dependent step fewer per state; the membrane
// potential keeps the reference's two roundings (fe, react.cuh).
template <bool R, class SA>
__device__ __forceinline__ void put(SA s, double* ds, int i, double h, double d) {
  if (R) ds[i] = d;
  else s[i] = CWG_ORD_FMA_UPDATE ? fma(h, d, s[i]) : fe(s[i], h, d);
}
// gate: x += h * (x_inf - x) * rate, as x + (x_inf - x) (h rate) in one FMA
template <bool R, class SA>
__device__ __forceinline__ void gate(SA s, double* ds, int i, double h, double xinf, double rate) {
  if (R || !CWG_ORD_FMA_UPDATE) put<R>(s, ds, i, h, (xinf - s[i]) * rate);
  else s[i] = fma(xinf - s[i], h * rate, s[i]);
}

// The evaluation is split into composable pieces (prologue, group A: INa,
// INaL, Ito, ICaL; group B: IKr, IKs, IK1, NaCa, NaK, background; finish:
// fluxes, concentrations, V); step() chains them in one thread. (A two-warp
// variant that ran groups A and B in different warps was measured slower and
// dropped; the split keeps each piece's live ranges short.)
struct Pro {
  double ena, ek, eks, camk_b, camkt, fk, nfk, vfrt, e1, e2, xq1, xq2;
};
struct CurA {
  double i_na, i_to, i_cal, i_cana, i_cak;  // i_na includes INaL
  double e70;                                // e^((v+70)/20), reused by IKs (group B) on the fast path
};
struct CurB {
  double i_k, inaca_i, inaca_ss, i_nak, i_kb, i_nab, i_cab, i_pca;
};

// reversal potentials, CaMK, GHK driving terms (reads nai, ki, cass, CaMKt)
template <int CT, bool FP, class SA>
__device__ __forceinline__ Pro prologue(double v, SA s) {
  Pro p;
  const double nai = s[NAI], ki = s[KI], cass = s[CASS];
  // log(a / x) = log(a) - log(x): no reciprocal (log 140, log 5.4, log(5.4 + 0.01833 * 140))
  p.ena = RTF * (4.941642422609304 - clog<FP>(nai));
  p.ek = RTF * (1.6863989535702288 - clog<FP>(ki));
  p.eks = RTF * (2.0752075911477745 - clog<FP>(ki + 0.01833 * nai));
  p.camkt = s[CAMKT];
  p.camk_b = 0.05 * (1.0 - p.camkt) * cass * crcp<FP>(cass + 0.0015);
  const double camk_a = p.camk_b + p.camkt;
  p.fk = camk_a * crcp<FP>(camk_a + 0.15);
  p.nfk = 1.0 - p.fk;
  p.vfrt = v * FRT;
  const double vfrt = p.vfrt;
  // ---------------- GHK driving terms (one expm1 for e^x, e^2x, expm1(2x))
  const double em1 = expm1(vfrt);
  p.e1 = em1 + 1.0;
  p.e2 = p.e1 * p.e1;
  const double em2 = em1 * (em1 + 2.0);
  p.xq1 = xem1<FP>(vfrt, em1);
  p.xq2 = xem1<FP>(2.0 * vfrt, em2);

  return p;
}

// group A: INa, INaL, Ito, ICaL/ICaNa/ICaK and their 24 gates (reads nass, kss, cass)
template <int CT, bool R, bool FP, class SA>
__device__ __forceinline__ CurA group_a(double v, SA s, double* ds, const Pro& pr, double h) {
  using P = Var<CT>;
  const double ena = pr.ena, ek = pr.ek, fk = pr.fk, nfk = pr.nfk;
  const double e1 = pr.e1, e2 = pr.e2, xq1 = pr.xq1, xq2 = pr.xq2;
  const double nass = s[NASS], kss = s[KSS], cass = s[CASS];
  CurA o;
  // ---------------- INa + INaL: the 14 V-dependent exponentials in one batch
  double i_na;
  {
    // a e^u = e^(u + log a): the rate coefficients ride in the exponents' offsets (LN_x = log x)
    constexpr double LN_6_765 = 1.9117622616227514, LN_8_552 = 2.146165173722744, LN_1_432em5 = -11.153853396431774;
    constexpr double LN_6_149 = 1.8162894669713328, LN_0_009794 = -4.625985325702011, LN_0_3343 = -1.0957164855560841;
    constexpr double LN_0_02136 = -3.846235264890143, LN_0_3052 = -1.186787979571835;
    double e[12] = {lin(v, -1.0 / (9.871), -(39.57) / (9.871)),   lin(v, 1.0 / (34.77), (11.64) / (34.77) + LN_6_765),  lin(v, -1.0 / (5.955), -(77.42) / (5.955) + LN_8_552),
                    lin(v, 1.0 / (6.086), (82.90) / (6.086)),    lin(v, -1.0 / (6.285), -(1.196) / (6.285) + LN_1_432em5), lin(v, 1.0 / (20.27), (0.5096) / (20.27) + LN_6_149),
                    lin(v, -1.0 / (28.05), -(17.95) / (28.05) + LN_0_009794),   lin(v, 1.0 / (56.66), (5.730) / (56.66) + LN_0_3343),  lin(v, -1.0 / (8.281), -(100.6) / (8.281) + LN_0_02136),
                    lin(v, 1.0 / (38.45), (0.9941) / (38.45) + LN_0_3052),   lin(v, -1.0 / (5.264), -(42.85) / (5.264)), lin(v, 1.0 / (7.488), (87.61) / (7.488))};
    vexp_n<FP>(e);
    // e^((v+89.1)/6.086) = e^((v+82.9)/6.086) e^(6.2/6.086), e^((v+93.81)/7.488) = e^((v+87.61)/7.488) e^(6.2/7.488)
    const double e_hp = FP ? e[3] * 2.7696792380394113 : vexp<FP>(lin(v, 1.0 / (6.086), (89.1) / (6.086)));
    const double e_hlp = FP ? e[11] * 2.288717124596482 : vexp<FP>(lin(v, 1.0 / (7.488), (93.81) / (7.488)));
    // 1 / (2.038 + 1 / s) = s / (2.038 s + 1): one reciprocal instead of two on the fast path
    const double s_j = e[8] + e[9];
    double q[7] = {1.0 + e[0], 1.0 + e[3], 1.0 + e_hp, 1.0 + e[10], 1.0 + e[11], 1.0 + e_hlp,
                   FP ? fma(2.038, s_j, 1.0) : s_j};
    vrcp_n<FP>(q);
    const double m_inf = q[0], h_inf = q[1], hp_inf = q[2];
    const double r_m = e[1] + e[2];
    const double r_hf = e[4] + e[5];
    const double r_hs = e[6] + e[7];
    const double r_j = FP ? s_j * q[6] : vrcp<FP>(2.038 + q[6]);
    const double hmix = 0.99 * s[HF] + (1.0 - 0.99) * s[HS];
    const double hpmix = 0.99 * s[HF] + (1.0 - 0.99) * s[HSP];
    const double m = s[M];
    i_na = 75.0 * (v - ena) * (m * m * m) * (nfk * hmix * s[J] + fk * hpmix * s[JP]);
    gate<R>(s, ds, M, h, m_inf, r_m);
    gate<R>(s, ds, HF, h, h_inf, r_hf);
    gate<R>(s, ds, HS, h, h_inf, r_hs);
    gate<R>(s, ds, J, h, h_inf, r_j);
    gate<R>(s, ds, HSP, h, hp_inf, r_hs * (1.0 / 3.0));
    gate<R>(s, ds, JP, h, h_inf, r_j * (1.0 / 1.46));
    // INaL (tmL = tm)
    const double i_nal = P::gnal * (v - ena) * s[ML] * (nfk * s[HL] + fk * s[HLP]);
    i_na += i_nal;  // INa + INaL travel together into dv and d[nai]
    gate<R>(s, ds, ML, h, q[3], r_m);
    gate<R>(s, ds, HL, h, q[4], 1.0 / 200.0);
    gate<R>(s, ds, HLP, h, q[5], 1.0 / 600.0);
  }

  // ---------------- Ito
  double i_to;
  double e70, e70sq;  // e^((v+70)/20) and its square: ICaL and IKs reuse them on the fast path
  {
    // 11 exponentials; on the fast path two more follow from them: e^((v+100)/29.3814) = K / e[1]
    // (folded into its sigmoid: 1 / (1 + K / e) = e / (e + K)) and e^((v+70)/5) = (e^((v+70)/20))^4
    double e[11] = {lin(v, -1.0 / (14.82), -(-14.34) / (14.82)),     lin(v, -1.0 / (29.3814), -(-18.4099) / (29.3814)),
                    lin(v, 1.0 / (5.711), (43.94) / (5.711)),      lin(v, -1.0 / (100.0), -(100.0) / (100.0) - 0.9331825995443732 /* log 0.3933 */),     lin(v, 1.0 / (16.59), (50.0) / (16.59) - 2.5252287692666044 /* log 0.08004 */),
                    lin(v, -1.0 / (59.05), -(96.52) / (59.05) - 6.5599192837106095 /* log 0.001416 */),     lin(v, 1.0 / (8.079), (114.1) / (8.079) - 17.844067379648372 /* log 1.780e-8 */),
                    lin(v, 1.0 / (151.2), (-213.6) / (151.2)),      lin(v, 1.0 / (15.89), (-167.4) / (15.89)),      lin(v, -1.0 / (0.2154), -(-12.23) / (0.2154)),
                    lin(v, 1.0 / (20.0), (70.0) / (20.0))};
    vexp_n<FP>(e);
    // e^(-(v-24.34)/14.82) = e^(-(v-14.34)/14.82) e^(10/14.82)
    const double e_ap = FP ? e[0] * 1.9635691902911017 : vexp<FP>(lin(v, -1.0 / (14.82), -(-24.34) / (14.82)));
    e70sq = e[10] * e[10];  // e^((v+70)/10), also feeds ICaL below
    const double e_d5 = FP ? e70sq * e70sq : vexp<FP>(lin(v, 1.0 / (5.0), (70.0) / (5.0)));
    e70 = e[10];
    double a_inf, r_a, i_inf, a_if, ap_inf, r_if, r_is, r_dr;
    if (FP) {
      // every 1 / (c + 1 / s) is s / (c s + 1) and the epi / development / recovery factors
      // (a + e) / (1 + e) go into the same denominators: one batch of 9 reciprocals
      const double s_if = e[3] + e[4], s_is = e[5] + e[6];
      const double s_dv = e[8] + e[9], g10 = 1.0 + e[10];
      double d_if = fma(4.562, s_if, 1.0), d_is = fma(23.62, s_is, 1.0);
      double n_if = s_if, n_is = s_is;
      if (P::epi) {  // delta_epi = 1 - 0.95 / (1 + e) = (0.05 + e) / (1 + e)
        const double ge = 1.0 + e_d5, he = 0.05 + e_d5;
        d_if *= he;
        d_is *= he;
        n_if *= ge;
        n_is *= ge;
      }
      // 1 / (dev rec), dev = 1.354 + 1e-4 / s_dv, rec = 1 - 0.5 / (1 + e10) = (0.5 + e10) / (1 + e10)
      double q[9] = {1.0 + e[0], fma(e[1], 1.2089, 1.2089), e[1] + 56.266384148520984, 1.0 + e[2], d_if, d_is,
                     1.0 + e[7], 1.0 + e_ap, fma(1.354, s_dv, 1.0e-4) * (0.5 + e[10])};
      vrcp_n<FP>(q);
      a_inf = q[0];
      r_a = (1.0 / 1.0515) * (q[1] + 3.5 * (q[2] * e[1]));
      i_inf = q[3];
      r_if = n_if * q[4];
      r_is = n_is * q[5];
      a_if = q[6];
      ap_inf = q[7];
      r_dr = (s_dv * g10) * q[8];
    } else {
      double q[11] = {1.0 + e[0], 1.2089 * (1.0 + e[1]),
                      1.0 + vexp<FP>(lin(v, 1.0 / (29.3814), (100.0) / (29.3814))), 1.0 + e[2],
                      e[3] + e[4], e[5] + e[6], 1.0 + e_d5,
                      1.0 + e[7], 1.0 + e_ap, e[8] + e[9], 1.0 + e[10]};
      vrcp_n<FP>(q);
      a_inf = q[0];
      r_a = (1.0 / 1.0515) * (q[1] + 3.5 * q[2]);
      i_inf = q[3];
      double t_if = 4.562 + q[4];
      double t_is = 23.62 + q[5];
      if (P::epi) {
        const double d_epi = 1.0 - 0.95 * q[6];
        t_if *= d_epi;
        t_is *= d_epi;
      }
      a_if = q[7];
      ap_inf = q[8];
      const double dev = 1.354 + 1.0e-4 * q[9];
      const double rec = 1.0 - 0.5 * q[10];
      double r3[3] = {t_if, t_is, dev * rec};
      vrcp_n<FP>(r3);
      r_if = r3[0], r_is = r3[1], r_dr = r3[2];
    }
    const double a_is = 1.0 - a_if;
    const double imix = a_if * s[IF] + a_is * s[IS];
    const double ipmix = a_if * s[IFP] + a_is * s[ISP];
    i_to = P::gto * (v - ek) * (nfk * s[A] * imix + fk * s[AP] * ipmix);
    gate<R>(s, ds, A, h, a_inf, r_a);
    gate<R>(s, ds, IF, h, i_inf, r_if);
    gate<R>(s, ds, IS, h, i_inf, r_is);
    gate<R>(s, ds, AP, h, ap_inf, r_a);
    gate<R>(s, ds, IFP, h, i_inf, r_if * r_dr);
    gate<R>(s, ds, ISP, h, i_inf, r_is * r_dr);
  }

  // ---------------- ICaL, ICaNa, ICaK
  double i_cal, i_cana, i_cak;
  {
    // 7 exponentials; on the fast path e^((v+20)/10) = e^((v+70)/10) e^-5 (Ito's), e^((v-4)/7) = e^(v/7) e^(-4/7)
    // and e^(-(v+5)/4) = (e^(-(v+6)/20))^5 e^(1/4)
    double e[7] = {lin(v, -1.0 / (4.230), -(3.940) / (4.230)), -0.05 * (v + 6.0),          0.09 * (v + 14.0),
                   lin(v, 1.0 / (3.696), (19.58) / (3.696)),  lin(v, 1.0 / (6.0), (5.0) / (6.0)),      lin(v, -1.0 / 3.0, -9.028018815182229 /* log 0.00012 */),
                   lin(v, 1.0 / 7.0, -9.028018815182229)};
    vexp_n<FP>(e);
    const double eff = FP ? e70sq * 0.006737946999085467 : vexp<FP>(lin(v, 1.0 / (10.0), (20.0) / (10.0)));
    const double efc = FP ? e[6] * (0.5647181220077593 / 0.00012) : vexp<FP>(lin(v, 1.0 / (7.0), (-4.0) / (7.0)));
    // e^((v-10)/10) = e^((v+20)/10) e^-3
    const double e_fca = FP ? e70sq * 0.00033546262790251185 : vexp<FP>(lin(v, 1.0 / (10.0), (-10.0) / (10.0)));
    double t_fs;  // 0.000035 e^(-(v+5)/4) + 0.000035 e^((v+5)/6)
    if (FP) {
      const double x2 = e[1] * e[1];
      t_fs = fma((x2 * x2) * e[1], 4.4940889584070944e-05, 0.000035 * e[4]);
    } else {
      t_fs = 0.000035 * vexp<FP>(lin(v, -1.0 / (4.0), -(5.0) / (4.0))) + 0.000035 * e[4];
    }
    double d_inf, f_inf, r_d, r_fs, r_fcas, r_ff, r_fcaf, q_fca;
    if (FP) {
      // 1 / (c + 1 / s) = s / (c s + 1); 1 / (7 + 1 / (a (e + 1 / e))) = a (e^2 + 1) / (7 a (e^2 + 1) + e):
      // one batch of 8 reciprocals instead of 8 + 5 + 2
      const double s_d = e[1] + e[2], s_ca = e[5] + e[6];
      const double w_ff = fma(eff, eff, 1.0), w_fc = fma(efc, efc, 1.0);
      double q[8] = {1.0 + e[0], fma(0.6, s_d, 1.0), 1.0 + e[3], fma(7.0 * 0.0045, w_ff, eff), fma(1000.0, t_fs, 1.0),
                     fma(7.0 * 0.04, w_fc, efc), fma(100.0, s_ca, 1.0), 1.0 + e_fca};
      vrcp_n<FP>(q);
      d_inf = q[0], f_inf = q[2], q_fca = q[7];
      r_d = s_d * q[1];
      r_ff = (0.0045 * w_ff) * q[3];
      r_fs = t_fs * q[4];
      r_fcaf = (0.04 * w_fc) * q[5];
      r_fcas = s_ca * q[6];
    } else {
      double q[8] = {1.0 + e[0], e[1] + e[2], 1.0 + e[3], eff, t_fs, efc,
                     e[5] + e[6], 1.0 + e_fca};
      vrcp_n<FP>(q);
      double q2[5] = {0.6 + q[1], 0.0045 * (q[3] + eff), 1000.0 + q[4], 0.04 * (q[5] + efc), 100.0 + q[6]};
      vrcp_n<FP>(q2);
      double q3[2] = {7.0 + q2[1], 7.0 + q2[3]};
      vrcp_n<FP>(q3);
      d_inf = q[0], f_inf = q[2], q_fca = q[7];
      r_d = q2[0], r_fs = q2[2], r_fcas = q2[4], r_ff = q3[0], r_fcaf = q3[1];
    }
    const double a_fcaf = 0.3 + 0.6 * q_fca;
    const double a_fcas = 1.0 - a_fcaf;
    const double fmix = 0.6 * s[FF] + (1.0 - 0.6) * s[FS];
    const double fcamix = a_fcaf * s[FCAF] + a_fcas * s[FCAS];
    const double fpmix = 0.6 * s[FFP] + (1.0 - 0.6) * s[FS];
    const double fcapmix = a_fcaf * s[FCAFP] + a_fcas * s[FCAS];
    const double jca = s[JCA], nca = s[NCA];
    const double cn = (cass + 0.002) * crcp<FP>(cass);
    const double cn2 = cn * cn;
    const double anca = jca * crcp<FP>(1000.0 + jca * (cn2 * cn2));
    const double phi_cal = 2.0 * F * (cass * e2 - 0.341 * CAO) * xq2;
    const double phi_cana = F * (0.75 * nass * e1 - 0.75 * NAO) * xq1;
    const double phi_cak = F * (0.75 * kss * e1 - 0.75 * KO) * xq1;
    const double g_np = s[D] * (fmix * (1.0 - nca) + jca * fcamix * nca);
    const double g_p = s[D] * (fpmix * (1.0 - nca) + jca * fcapmix * nca);
    const double mixed = nfk * g_np + fk * 1.1 * g_p;  // PCap = 1.1 PCa
    i_cal = P::pca * phi_cal * mixed;
    i_cana = (0.00125 * P::pca) * phi_cana * mixed;
    i_cak = (3.574e-4 * P::pca) * phi_cak * mixed;
    gate<R>(s, ds, D, h, d_inf, r_d);
    gate<R>(s, ds, FF, h, f_inf, r_ff);
    gate<R>(s, ds, FS, h, f_inf, r_fs);
    gate<R>(s, ds, FCAF, h, f_inf, r_fcaf);
    gate<R>(s, ds, FCAS, h, f_inf, r_fcas);
    gate<R>(s, ds, JCA, h, f_inf, 1.0 / 75.0);
    put<R>(s, ds, NCA, h, anca * 1000.0 - jca * nca);
    gate<R>(s, ds, FFP, h, f_inf, r_ff * (1.0 / 2.5));
    gate<R>(s, ds, FCAFP, h, f_inf, r_fcaf * (1.0 / 2.5));
  }

  o.i_na = i_na;
  o.i_to = i_to;
  o.i_cal = i_cal;
  o.i_cana = i_cana;
  o.i_cak = i_cak;
  o.e70 = e70;
  return o;
}

// group B: IKr, IKs, IK1 (5 gates), INaCa, INaK, background currents
template <int CT, bool R, bool FP, class SA>
__device__ __forceinline__ CurB group_b(double v, SA s, double* ds, const Pro& pr, double h, double gkr_scale,
                                         double e70) {
  using P = Var<CT>;
  const double ek = pr.ek, eks = pr.eks, vfrt = pr.vfrt;
  const double e1 = pr.e1, e2 = pr.e2, xq1 = pr.xq1, xq2 = pr.xq2;
  const double nai = s[NAI], nass = s[NASS], ki = s[KI], cai = s[CAI], cass = s[CASS];
  CurB o;
  // ---------------- IKr, IKs, IK1
  double i_k;  // IKr + IKs + IK1
  {
    double e[8] = {lin(v, -1.0 / (6.789), -(8.337) / (6.789)), lin(v, 1.0 / (3.869), (-31.66) / (3.869) - 1.0073101302613237 /* log 0.3652 */), lin(v, -1.0 / (20.38), -(-47.78) / (20.38) - 10.096344411245465 /* log 4.123e-5 */),
                   lin(v, 1.0 / (7.355), (-34.70) / (7.355) - 2.713716222728837 /* log 0.06629 */),  lin(v, -1.0 / (25.94), -(-29.74) / (25.94) - 11.39247931189436 /* log 1.128e-5 */), lin(v, 1.0 / (38.21), (54.81) / (38.21)),
                   lin(v, 1.0 / (75.0), (55.0) / (75.0)),    lin(v, 1.0 / (30.0), (-10.0) / (30.0))};
    vexp_n<FP>(e);
    const double s_xrf = e[1] + e[2], s_xrs = e[3] + e[4];
    double q[5] = {1.0 + e[0], FP ? fma(12.98, s_xrf, 1.0) : s_xrf, FP ? fma(1.865, s_xrs, 1.0) : s_xrs, 1.0 + e[5],
                   (1.0 + e[6]) * (1.0 + e[7])};
    vrcp_n<FP>(q);
    double r_xrf, r_xrs;
    if (FP) {  // 1 / (c + 1 / s) = s / (c s + 1)
      r_xrf = s_xrf * q[1];
      r_xrs = s_xrs * q[2];
    } else {
      double q2[2] = {12.98 + q[1], 1.865 + q[2]};
      vrcp_n<FP>(q2);
      r_xrf = q2[0], r_xrs = q2[1];
    }
    const double xr_inf = q[0], a_xrf = q[3], rkr = q[4];
    const double xrmix = a_xrf * s[XRF] + (1.0 - a_xrf) * s[XRS];
    const double i_kr = (P::gkr * gkr_scale) * xrmix * rkr * (v - ek);  // sqrt(ko/5.4) == 1
    gate<R>(s, ds, XRF, h, xr_inf, r_xrf);
    gate<R>(s, ds, XRS, h, xr_inf, r_xrs);

    // on the fast path e^((v-50)/20) = e^((v+70)/20) e^-6 (Ito's exponential, passed in as e70)
    double f[8] = {lin(v, -1.0 / (8.932), -(11.60) / (8.932)),  lin(v, 1.0 / (17.80), (48.28) / (17.80) - 8.36619031787971 /* log 2.326e-4 */), lin(v, -1.0 / (230.0), -(210.0) / (230.0) - 6.651563873621727 /* log 0.001292 */),
                   lin(v, -1.0 / (31.0), -(66.54) / (31.0) - 3.947650183071297 /* log 0.0193 */),
                   -(v + 2.5538 * KO + 144.59) * (1.0 / (1.5692 * KO + 3.8115)),
                   lin(v, -1.0 / (20.36), -(127.2) / (20.36) - 4.805659046737495 /* log(1/122.2) */),  lin(v, 1.0 / (69.33), (236.8) / (69.33) - 4.805659046737495),  lin(v, 1.0 / (9.493), (105.8 - 2.6 * KO) / (9.493))};
    vexp_n<FP>(f);
    const double s_xs1 = f[1] + f[2];
    double p[4] = {1.0 + f[0], FP ? fma(817.3, s_xs1, 1.0) : s_xs1, 1.0 + f[4], 1.0 + f[7]};
    vrcp_n<FP>(p);
    const double xs_inf = p[0];
    const double r_xs1 = FP ? s_xs1 * p[1] : vrcp<FP>(817.3 + p[1]);
    const double r_xs2 = FP ? fma(e70, 2.4787521766663585e-05, f[3])
                            : 0.01 * vexp<FP>(lin(v, 1.0 / (20.0), (-50.0) / (20.0))) + f[3];
    const double ksca = 1.0 + 0.6 * crcp<FP>(1.0 + vexp<FP>(1.4 * (-10.177924398237888 - clog<FP>(cai))) /* log(3.8e-5) */);
    const double i_ks = P::gks * ksca * s[XS1] * s[XS2] * (v - eks);
    gate<R>(s, ds, XS1, h, xs_inf, r_xs1);
    gate<R>(s, ds, XS2, h, xs_inf, r_xs2);

    const double xk1_inf = p[2];
    const double r_xk1 = f[5] + f[6];
    const double rk1 = p[3];
    const double i_k1 = (P::gk1 * 2.3237900077244502) * rk1 * s[XK1] * (v - ek);  // sqrt(5.4)
    gate<R>(s, ds, XK1, h, xk1_inf, r_xk1);
    i_k = i_kr + i_ks + i_k1;
  }

  // ---------------- INaCa (bulk + subspace)
  double inaca_i, inaca_ss;
  {
    NcxShared c;
    c.hna = vexp<FP>(0.5224 * vfrt);
    c.hca6 = vexp<FP>(fma(vfrt, -0.1670, 11.002099841204238 /* log 6e4 */));  // 6e4 / hca
    if (FP) {  // h9 = 1 / (1 + c (1 + 1 / hna)) = hna / (hna + c (hna + 1)), h8 = c / (same)
      const double r = vrcp<FP>(fma(NAO * (1.0 / 88.12), c.hna + 1.0, c.hna));
      c.h9 = c.hna * r;
      c.h8 = NAO * (1.0 / 88.12) * r;
    } else {
      const double hna_r = vrcp<FP>(c.hna);
      const double r7 = vrcp<FP>(1.0 + NAO * (1.0 / 88.12) * (1.0 + hna_r));
      c.h9 = r7;
      c.h8 = NAO * (1.0 / 88.12) * hna_r * r7;
    }
    inaca_i = (0.8 * P::gncx) * ncx<FP>(nai, cai, c);
    inaca_ss = (0.2 * P::gncx) * ncx<FP>(nass, cass, c);
  }

  // ---------------- INaK
  double i_nak;
  {
    constexpr double rko = KO / 0.3582;
    constexpr double qo = (1.0 + rko) * (1.0 + rko);
    constexpr double b1 = 182.4 * 0.05, a2 = 687.2;
    constexpr double a4 = 639.0 * 9.8 / 1.698e-7 / (1.0 + 9.8 / 1.698e-7);
    constexpr double b3c = 79300.0 * 1.0e-7 / (1.0 + 9.8 / 1.698e-7);
    const double p_hp = 4.2 * crcp<FP>(1.0 + 1.0e-7 / 1.698e-7 + nai * (1.0 / 224.0) + ki * (1.0 / 292.0));
    const double ri = nai * vexp<FP>(fma(vfrt, 0.1550 / 3.0, -2.2053029701874918 /* log(1/9.073) */));   // nai / Knai
    const double ro = vexp<FP>(fma(vfrt, -(1.1550 / 3.0), 1.6173260852831066 /* log(140/27.78) */));  // nao / Knao
    const double rk = ki * 2.0;                                            // ki / 0.5
    const double ci = (1.0 + ri) * (1.0 + ri) * (1.0 + ri), qi = (1.0 + rk) * (1.0 + rk);
    const double co = (1.0 + ro) * (1.0 + ro) * (1.0 + ro);
    const double di = crcp<FP>(ci + qi - 1.0), dco = crcp<FP>(co + qo - 1.0);
    const double a1 = 949.5 * (ri * ri * ri) * di;
    const double b2 = 39.4 * (ro * ro * ro) * dco;
    const double a3 = 1899.0 * (rko * rko) * dco;
    const double b3 = b3c * p_hp;
    const double b4 = 40.0 * (rk * rk) * di;
    // the cycle's state occupancies, each four triple products factored into two
    const double a1a2 = a1 * a2, b3b4 = b3 * b4, b1b4 = b1 * b4, a2a3 = a2 * a3;
    const double a3a4 = a3 * a4, b1b2 = b1 * b2, b2b3 = b2 * b3, a1a4 = a1 * a4;
    const double y1 = a1a2 * (a4 + b3) + b3b4 * (b2 + a2);
    const double y2 = b1b4 * (b2 + a3) + a2a3 * (a1 + b4);
    const double y3 = a3a4 * (a2 + b1) + b1b2 * (b3 + a4);
    const double y4 = b2b3 * (b4 + a1) + a1a4 * (a3 + b2);
    const double ry = crcp<FP>(y1 + y2 + y3 + y4);
    i_nak = P::pnak * ry * (3.0 * (y1 * a3 - y2 * b3) + 2.0 * (y4 * b1 - y3 * a1));
  }

  // ---------------- background currents
  const double i_kb = P::gkb * sigm<FP>(lin(v, -1.0 / (18.34), -(-14.48) / (18.34))) * (v - ek);
  const double i_nab = (3.75e-10 * F) * (nai * e1 - NAO) * xq1;
  const double i_cab = (2.5e-8 * 2.0 * F) * (cai * e2 - 0.341 * CAO) * xq2;
  const double i_pca = 0.0005 * cai * crcp<FP>(0.0005 + cai);

  o.i_k = i_k;
  o.inaca_i = inaca_i;
  o.inaca_ss = inaca_ss;
  o.i_nak = i_nak;
  o.i_kb = i_kb;
  o.i_nab = i_nab;
  o.i_cab = i_cab;
  o.i_pca = i_pca;
  return o;
}

// SR fluxes (Jrel gates need ICaL), CaMKt, buffers, concentrations, dV
template <int CT, bool R, bool FP, class SA>
__device__ __forceinline__ void finish(double& v, SA s, double* ds, const Pro& pr, const CurA& A, const CurB& B,
                                       double ist, double h, double& dv) {
  using P = Var<CT>;
  const double fk = pr.fk, nfk = pr.nfk, camk_b = pr.camk_b, camkt = pr.camkt;
  const double nai = s[NAI], nass = s[NASS], ki = s[KI], kss = s[KSS];
  const double cai = s[CAI], cass = s[CASS], cansr = s[CANSR], cajsr = s[CAJSR];
  const double i_na = A.i_na, i_to = A.i_to, i_cal = A.i_cal, i_cana = A.i_cana, i_cak = A.i_cak;
  const double i_k = B.i_k, inaca_i = B.inaca_i, inaca_ss = B.inaca_ss, i_nak = B.i_nak, i_kb = B.i_kb;
  const double i_nab = B.i_nab, i_cab = B.i_cab, i_pca = B.i_pca;
  // ---------------- SR release / uptake, buffers
  const double jrel = nfk * s[JRELNP] + fk * s[JRELP];
  {
    const double rc = crcp<FP>(cajsr);
    const double rr = 1.5 * rc;
    const double rr2 = rr * rr, rr4 = rr2 * rr2;
    const double gate_rel = crcp<FP>(1.0 + rr4 * rr4);
    const double jrel_inf = (0.5 * 4.75 * P::jrel) * (-i_cal) * gate_rel;
    double r_rel = (cajsr + 0.0123) * (rc * (1.0 / 4.75));  // 1/tau_rel (one reciprocal of cajsr for both)
    double r_relp = r_rel * (1.0 / 1.25);
    r_rel = r_rel > 200.0 ? 200.0 : r_rel;  // tau_rel >= 0.005 (NaN passes through, like the reference)
    r_relp = r_relp > 200.0 ? 200.0 : r_relp;
    gate<R>(s, ds, JRELNP, h, jrel_inf, r_rel);
    gate<R>(s, ds, JRELP, h, jrel_inf * 1.25, r_relp);
    put<R>(s, ds, CAMKT, h, 0.05 * camk_b * (camk_b + camkt) - 0.00068 * camkt);
  }
  const double jup_np = (0.004375 * P::jup) * cai * crcp<FP>(cai + 0.00092);
  const double jup_p = (2.75 * 0.004375 * P::jup) * cai * crcp<FP>(cai + 0.00092 - 0.00017);
  const double j_up = nfk * jup_np + fk * jup_p - (0.0039375 / 15.0) * cansr;
  const double j_tr = (cansr - cajsr) * (1.0 / 100.0);
  const double jd_na = (nass - nai) * 0.5;
  const double jd_k = (kss - ki) * 0.5;
  const double jd_ca = (cass - cai) * 5.0;
  double b_cai, b_cass, b_cajsr;
  {
    const double kc = 0.00238 + cai, kt = 0.0005 + cai;
    const double kc2 = kc * kc, kt2 = kt * kt;
    const double pc = kc2 * kt2;
    b_cai = pc * crcp<FP>(pc + (P::cmdn * 0.00238) * kt2 + (0.07 * 0.0005) * kc2);
    const double kb = 0.00087 + cass, kl = 0.0087 + cass;
    const double kb2 = kb * kb, kl2 = kl * kl;
    const double pb = kb2 * kl2;
    b_cass = pb * crcp<FP>(pb + (0.047 * 0.00087) * kl2 + (1.124 * 0.0087) * kb2);
    const double kq = 0.8 + cajsr;
    const double kq2 = kq * kq;
    b_cajsr = kq2 * crcp<FP>(kq2 + 10.0 * 0.8);
  }

  // ---------------- concentrations (last: every current above read the old values)
  constexpr double cm_myo = ACAP / (F * VMYO), cm_ss = ACAP / (F * VSS);
  put<R>(s, ds, NAI, h, -(i_na + 3.0 * inaca_i + 3.0 * i_nak + i_nab) * cm_myo + jd_na * (VSS / VMYO));
  put<R>(s, ds, NASS, h, -(i_cana + 3.0 * inaca_ss) * cm_ss - jd_na);
  put<R>(s, ds, KI, h, -(i_to + i_k + i_kb - 2.0 * i_nak) * cm_myo + jd_k * (VSS / VMYO));
  put<R>(s, ds, KSS, h, -i_cak * cm_ss - jd_k);
  put<R>(s, ds, CAI, h, b_cai * (-(i_pca + i_cab - 2.0 * inaca_i) * (0.5 * cm_myo) - j_up * (VNSR / VMYO) + jd_ca * (VSS / VMYO)));
  put<R>(s, ds, CASS, h, b_cass * (-(i_cal - 2.0 * inaca_ss) * (0.5 * cm_ss) + jrel * (VJSR / VSS) - jd_ca));
  put<R>(s, ds, CANSR, h, j_up - j_tr * (VJSR / VNSR));
  put<R>(s, ds, CAJSR, h, b_cajsr * (j_tr - jrel));

  dv = -(i_na + i_to + i_cal + i_cana + i_cak + i_k + inaca_i + inaca_ss + i_nak + i_kb + i_nab + i_pca + i_cab) + ist;
  if (!R) v = fe(v, h, dv);
}

// The fast path's precondition on the state (besides |V| <= 130 mV): the eight
// concentrations in [1e-10, 1e10] mM, CaMKt in [0, 1e10] and the jca gate in
// [0, 1e10]. Then every concentration-dependent denominator and log argument
// of the model is a sum or product of bounded positive terms -- normal, finite,
// positive (e.g. 1000 + jca cn^4 >= 1000 with cn <= 2e7; 1 + (1.5/cajsr)^8 <=
// 3e80; the NCX cycle total and the INaK y-sum are positive sums of positive
// rate products) -- so the unchecked reciprocals / logs return exactly the
// checked ones' bits. Physiological values sit orders of magnitude inside.
template <class SA>
__device__ __forceinline__ bool conc_ok(SA s) {
  bool ok = true;
#pragma unroll
  for (int q = NAI; q <= CAJSR; ++q) ok = ok && s[q] >= 1e-10 && s[q] <= 1e10;
  return ok && s[CAMKT] >= 0.0 && s[CAMKT] <= 1e10 && s[JCA] >= 0.0 && s[JCA] <= 1e10;
}

template <int CT, bool R, bool FP, class SA>
__device__ __forceinline__ void step(double& v, SA s, double* ds, double ist, double gkr_scale, double h,
                                     double& dv) {
  const Pro pr = prologue<CT, FP>(v, s);
  const CurA ca = group_a<CT, R, FP>(v, s, ds, pr, h);
  const CurB cb = group_b<CT, R, FP>(v, s, ds, pr, h, gkr_scale, ca.e70);
  finish<CT, R, FP>(v, s, ds, pr, ca, cb, ist, h, dv);
}

// CellModel::rates (no update), for the batched rates entry point / tests
template <int CT>
__device__ void rates(double v, const double* s, double ist, double& dv, double* ds) {
  double tmp[NSTATE];
#pragma unroll
  for (int q = 0; q < NSTATE; ++q) tmp[q] = s[q];
  step<CT, true, false, double*>(v, tmp, ds, ist, 1.0, 0.0, dv);
}

}  // namespace ord

// Launch shapes: 0: 128-thread blocks, 2 per SM (<= 255 regs), warps
// free-running (latency regime default); 1: one persistent 384-thread block
// per SM (<= 168 regs, 12 warps), lockstep (throughput regime default);
// 2 / 7: one persistent 256 / 288-thread lockstep block per SM (alternatives
// for the latency regime, selectable with CWG_ORD_VARIANT). Measured and
// dropped: 512-thread blocks, node states in shared memory, a
// two-warp-per-node split of the rates, a cp.async next-node prefetch,
// free-running 256/288-thread blocks, lockstep in warp groups.
template <int CT, int V = 0>
struct ModelOrd {
  static constexpr int NS = ord::NSTATE;
  // V = 10 / 11: shapes 0 / 1 for runs without a per-node GKr scale (launch_ct picks them when a.gkr is null):
  // the scale is the constant 1 there, two registers fewer in the lane-refill loop
  static constexpr int S = V == 10 ? 0 : (V == 11 ? 1 : V);  // the launch shape
  static constexpr int kThreads = S == 1 ? 384 : (S == 2 ? 256 : (S == 7 ? 288 : 128));
  static constexpr int kMinBlocks = S == 0 ? 2 : 1;
  static constexpr bool kBlockSync = S != 0;
  static constexpr bool kPreclaim = S == 0;  // react.cuh: claim the next node one trip ahead
  static constexpr bool kUsesGkr = V < 10;
  __device__ __forceinline__ static void block_init() { exp_table_init(); }
  template <class SA>
  __device__ __forceinline__ static void advance(double& v, SA s, double ist, double g, double h, double& dv) {
    if (fabs(v) <= 130.0 && ord::conc_ok(s))
      ord::step<CT, false, true>(v, s, nullptr, ist, g, h, dv);
    else
      ord::step<CT, false, false>(v, s, nullptr, ist, g, h, dv);
  }
};

template <int CT>
__global__ void ord_rates_kernel(long long n, const double* v, const double* s, const double* ist, double* dv,
                                 double* ds) {
  exp_table_init();
  __syncthreads();
  const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  double sl[ord::NSTATE], dl[ord::NSTATE];
  for (int q = 0; q < ord::NSTATE; ++q) sl[q] = s[i * ord::NSTATE + q];
  double d;
  ord::rates<CT>(v[i], sl, ist[i], d, dl);
  dv[i] = d;
  for (int q = 0; q < ord::NSTATE; ++q) ds[i * ord::NSTATE + q] = dl[q];
}

template <class M>
static size_t smem_bytes(int khist_len) {
  const size_t hist = static_cast<size_t>((khist_len + 1) & ~1) * sizeof(unsigned);
  return hist;
}

template <class M>
static cudaError_t launch_react_t(const ReactArgs& a, int grid, cudaStream_t st) {
  const size_t smem = smem_bytes<M>(a.khist_len);
  if (smem > 48 * 1024) {
    static std::atomic<uint64_t> attr_done{0};
    const cudaError_t e = ensure_dyn_smem(react_kernel<M>, 200 * 1024, attr_done);
    if (e != cudaSuccess) return e;
  }
  react_kernel<M><<<grid, M::kThreads, smem, st>>>(a);
  return cudaGetLastError();
}

template <class M>
static int occupancy_t() {
  int b = 0;
  const size_t smem = smem_bytes<M>(2048);
  if (smem > 48 * 1024) cudaFuncSetAttribute(react_kernel<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, react_kernel<M>, M::kThreads, smem);
  return b;
}

// Launch-shape variants (see ModelOrd). The host picks one per model bin
// (cwg_host.cu: choose_ord_variant); CWG_ORD_VARIANT overrides for experiments.
#define CWG_ORD_VARIANTS(X) X(0) X(1) X(2) X(7)

bool react_ord_variant_valid(int v) {
  switch (v) {
#define CWG_CASE(n) case n:
    CWG_ORD_VARIANTS(CWG_CASE) return true;
#undef CWG_CASE
    default: return false;
  }
}

template <int CT>
static cudaError_t launch_ct(int variant, const ReactArgs& a, int grid, cudaStream_t st) {
  if (!a.gkr) {  // no per-node GKr scale: the twins with the scale folded to 1
    if (variant == 0) return launch_react_t<ModelOrd<CT, 10>>(a, grid, st);
    if (variant == 1) return launch_react_t<ModelOrd<CT, 11>>(a, grid, st);
  }
  switch (variant) {
#define CWG_CASE(n) case n: return launch_react_t<ModelOrd<CT, n>>(a, grid, st);
    CWG_ORD_VARIANTS(CWG_CASE)
#undef CWG_CASE
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_react_ord(int kind, int variant, const ReactArgs& a, int grid, cudaStream_t st) {
  switch (kind) {
    case 1: return launch_ct<0>(variant, a, grid, st);
    case 2: return launch_ct<1>(variant, a, grid, st);
    case 3: return launch_ct<2>(variant, a, grid, st);
    default: return cudaErrorInvalidValue;
  }
}

int react_ord_threads(int variant) {
  switch (variant) {
#define CWG_CASE(n) case n: return ModelOrd<0, n>::kThreads;
    CWG_ORD_VARIANTS(CWG_CASE)
#undef CWG_CASE
    default: return 0;
  }
}

template <int CT>
static int occ_ct(int variant) {
  switch (variant) {
#define CWG_CASE(n) case n: return occupancy_t<ModelOrd<CT, n>>();
    CWG_ORD_VARIANTS(CWG_CASE)
#undef CWG_CASE
    default: return 0;
  }
}

int react_ord_occupancy(int kind, int variant) {
  switch (kind) {
    case 1: return occ_ct<0>(variant);
    case 2: return occ_ct<1>(variant);
    case 3: return occ_ct<2>(variant);
    default: return 0;
  }
}

cudaError_t launch_pace_ord(int kind, const PaceArgs& a, cudaStream_t st) {
  switch (kind) {
    case 1: return launch_pace_t<ModelOrd<0, 0>>(a, st);
    case 2: return launch_pace_t<ModelOrd<1, 0>>(a, st);
    case 3: return launch_pace_t<ModelOrd<2, 0>>(a, st);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_rates_ord(int kind, long long n, const double* v, const double* s, const double* ist, double* dv,
                             double* ds, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  const int grid = static_cast<int>((n + 127) / 128);
  switch (kind) {
    case 1: ord_rates_kernel<0><<<grid, 128, 0, st>>>(n, v, s, ist, dv, ds); break;
    case 2: ord_rates_kernel<1><<<grid, 128, 0, st>>>(n, v, s, ist, dv, ds); break;
    case 3: ord_rates_kernel<2><<<grid, 128, 0, st>>>(n, v, s, ist, dv, ds); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace cwg
