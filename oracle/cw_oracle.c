/* TEST INFRASTRUCTURE ONLY -- CPU restatement oracle (see cw_oracle.h).
 *
 * Every function restates the reference algorithm it cites, keeping the
 * reference's floating-point evaluation order so that, compiled with
 * -ffp-contract=off against the same libm, the results are bit-identical to
 * the reference (pinned by tests/test_oracle_pins.py). Organisation, naming
 * and data layout are our own.
 */
#include "cw_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ *
 * Aliev-Panfilov (aliev_panfilov.cpp:28-38): u = (V + 80)/100, t/12.9 *
 * ------------------------------------------------------------------ */
static void ap_rates(double v, const double* s, double i_stim, double* dv, double* ds) {
  const double u = (v - (-80.0)) / 100.0;
  const double w = s[0];
  const double du = -8.0 * u * (u - 0.15) * (u - 1.0) - u * w;
  const double eps = 0.002 + 0.2 * w / (u + 0.3);
  const double dw = eps * (-w - 8.0 * u * (u - 0.15 - 1.0));
  *dv = 100.0 / 12.9 * du + i_stim;
  ds[0] = dw / 12.9;
}

/* ------------------------------------------------------------------ *
 * MacCannell 2007 fibroblast (maccannell_2007.cpp:31-70)              *
 * ------------------------------------------------------------------ */
static void mac_rates(double v, const double* s, double i_stim, double* dv, double* ds) {
  const double rtf = 8314.0 * 306.15 / 96485.0;
  const double e_k = rtf * log(5.4 / 129.4349);
  const double e_na = rtf * log(130.0110 / 8.5547);
  const double r = s[0], sg = s[1];

  const double r_inf = 1.0 / (1.0 + exp(-(v + 20.0) / 11.0));
  const double xr = (v + 20.0) / 25.9;
  const double tau_r = 20.3 + 138.0 * exp(-xr * xr);
  const double s_inf = 1.0 / (1.0 + exp((v + 23.0) / 7.0));
  const double xs = (v + 23.0) / 22.7;
  const double tau_s = 1574.0 + 5268.0 * exp(-xs * xs);

  const double i_kv = 0.25 * r * sg * (v - e_k);
  const double vk = v - e_k;
  const double ak1 = 0.1 / (1.0 + exp(0.06 * (vk - 200.0)));
  const double bk1 = (3.0 * exp(0.0002 * (vk + 100.0)) + exp(0.1 * (vk - 10.0))) / (1.0 + exp(-0.5 * vk));
  const double i_k1 = 0.4822 * ak1 / (ak1 + bk1) * vk;
  const double na15 = pow(8.5547, 1.5);
  const double i_nak = 2.002 * 5.4 / (5.4 + 1.0) * na15 / (na15 + pow(11.0, 1.5)) * (v - (-150.0)) /
                       (v - (-200.0));
  const double i_bna = 0.0095 * (v - e_na);

  *dv = -(i_kv + i_k1 + i_nak + i_bna) + i_stim;
  ds[0] = (r_inf - r) / tau_r;
  ds[1] = (s_inf - sg) / tau_s;
}

/* ------------------------------------------------------------------ *
 * Passive, non-excitable membrane (EXTENSION, parity unpinned):       *
 * dV/dt = -g (V - E) + i_stim, no gating states.                      *
 * ------------------------------------------------------------------ */
#define PASSIVE_G 0.01
#define PASSIVE_E (-85.0)
static void passive_rates(double v, double i_stim, double* dv) {
  *dv = -PASSIVE_G * (v - PASSIVE_E) + i_stim;
}

/* ------------------------------------------------------------------ *
 * O'Hara-Rudy 2011 (ohara_rudy_2011.cpp:85-444)                       *
 * State order: concentrations 0..7, gates, CaMKt (StateIndex :18-26). *
 * ------------------------------------------------------------------ */
enum {
  O_NAI, O_NASS, O_KI, O_KSS, O_CAI, O_CASS, O_CANSR, O_CAJSR,
  O_M, O_HF, O_HS, O_J, O_HSP, O_JP, O_ML, O_HL, O_HLP,
  O_A, O_IF, O_IS, O_AP, O_IFP, O_ISP,
  O_D, O_FF, O_FS, O_FCAF, O_FCAS, O_JCA, O_NCA, O_FFP, O_FCAFP,
  O_XRF, O_XRS, O_XS1, O_XS2, O_XK1,
  O_JRELNP, O_JRELP, O_CAMKT, O_COUNT
};

/* Variant multipliers (1.0 where a variant leaves the base value alone;
 * x * 1.0 == x exactly, so one branch-free table reproduces the reference's
 * `if (epi) G *= f` chains bit for bit). */
typedef struct {
  double gnal, gto, pca, gkr, gks, gk1, gncx, pnak, gkb, jrel, jup, cmdn;
  int epi;
} ord_var;

static const ord_var kOrdVar[3] = {
    /* endo */ {1.0, 1.0, 1.0, 1.0, 1.0, 1.0, 1.0, 1.0, 1.0, 1.0, 1.0, 1.0, 0},
    /* epi  */ {0.6, 4.0, 1.2, 1.3, 1.4, 1.2, 1.1, 0.9, 0.6, 1.0, 1.3, 1.3, 1},
    /* mid  */ {1.0, 4.0, 2.5, 0.8, 1.0, 1.3, 1.4, 0.7, 1.0, 1.7, 1.0, 1.0, 0},
};

#define NAO 140.0
#define CAO 1.8
#define KO 5.4
#define FARADAY 96485.0
#define RTF (8314.0 * 310.0 / FARADAY)

/* cell geometry, with the reference code's rounded pi (ohara_rudy_2011.cpp:56-64) */
#define VCELL (1000.0 * 3.14 * 0.0011 * 0.0011 * 0.01)
#define AGEO (2.0 * 3.14 * 0.0011 * 0.0011 + 2.0 * 3.14 * 0.0011 * 0.01)
#define ACAP (2.0 * AGEO)
#define VMYO (0.68 * VCELL)
#define VNSR (0.0552 * VCELL)
#define VJSR (0.0048 * VCELL)
#define VSS (0.02 * VCELL)

static double xexpm1(double x) { /* x / (e^x - 1), ohara_rudy_2011.cpp:67-70 */
  if (fabs(x) < 1e-8) return 1.0 / (1.0 + 0.5 * x);
  return x / expm1(x);
}

static double sig(double num) { return 1.0 / (1.0 + exp(num)); }

/* Na/Ca exchanger for one compartment (ohara_rudy_2011.cpp:264-300) */
static double ncx_flux(double na_in, double ca_in, double hna, double hca) {
  const double h1 = 1.0 + na_in / 88.12 * (1.0 + hna);
  const double h2 = na_in * hna / (88.12 * h1);
  const double h3 = 1.0 / h1;
  const double h4 = 1.0 + na_in / 15.0 * (1.0 + na_in / 5.0);
  const double h5 = na_in * na_in / (h4 * 15.0 * 5.0);
  const double h6 = 1.0 / h4;
  const double h7 = 1.0 + NAO / 88.12 * (1.0 + 1.0 / hna);
  const double h8 = NAO / (88.12 * hna * h7);
  const double h9 = 1.0 / h7;
  const double h10 = 12.5 + 1.0 + NAO / 15.0 * (1.0 + NAO / 5.0);
  const double h11 = NAO * NAO / (h10 * 15.0 * 5.0);
  const double h12 = 1.0 / h10;
  const double k1 = h12 * CAO * 1.5e6;
  const double k2 = 5.0e3;
  const double k3pp = h8 * 5.0e3;
  const double k3 = h9 * 6.0e4 + k3pp;
  const double k4pp = h2 * 5.0e3;
  const double k4 = h3 * 6.0e4 / hca + k4pp;
  const double k5 = 5.0e3;
  const double k6 = h6 * ca_in * 1.5e6;
  const double k7 = h5 * h2 * 6.0e4;
  const double k8 = h8 * h11 * 6.0e4;
  const double x1 = k2 * k4 * (k7 + k6) + k5 * k7 * (k2 + k3);
  const double x2 = k1 * k7 * (k4 + k5) + k4 * k6 * (k1 + k8);
  const double x3 = k1 * k3 * (k7 + k6) + k8 * k6 * (k2 + k3);
  const double x4 = k2 * k8 * (k4 + k5) + k3 * k5 * (k1 + k8);
  const double tot = x1 + x2 + x3 + x4;
  const double e1 = x1 / tot, e2 = x2 / tot, e3 = x3 / tot, e4 = x4 / tot;
  const double q = 150.0e-6 / ca_in;
  const double allo = 1.0 / (1.0 + q * q);
  const double j_na = 3.0 * (e4 * k7 - e1 * k8) + e3 * k4pp - e2 * k3pp;
  const double j_ca = e2 * k2 - e1 * k1;
  return allo * (1.0 * j_na + 2.0 * j_ca);
}

static void ord_rates(int variant, double v, const double* s, double i_stim, double gkr_scale,
                      double* dv, double* ds) {
  const ord_var* P = &kOrdVar[variant];
  const double nai = s[O_NAI], nass = s[O_NASS], ki = s[O_KI], kss = s[O_KSS];
  const double cai = s[O_CAI], cass = s[O_CASS], cansr = s[O_CANSR], cajsr = s[O_CAJSR];

  /* reversal potentials, CaMK */
  const double ena = RTF * log(NAO / nai);
  const double ek = RTF * log(KO / ki);
  const double eks = RTF * log((KO + 0.01833 * NAO) / (ki + 0.01833 * nai));
  const double camk_b = 0.05 * (1.0 - s[O_CAMKT]) / (1.0 + 0.0015 / cass);
  const double camk_a = camk_b + s[O_CAMKT];
  const double fk = 1.0 / (1.0 + 0.15 / camk_a);
  const double vfrt = v * FARADAY / (8314.0 * 310.0);

  /* fast sodium */
  const double m_inf = sig(-(v + 39.57) / 9.871);
  const double tau_m = 1.0 / (6.765 * exp((v + 11.64) / 34.77) + 8.552 * exp(-(v + 77.42) / 5.955));
  const double h_inf = sig((v + 82.90) / 6.086);
  const double tau_hf = 1.0 / (1.432e-5 * exp(-(v + 1.196) / 6.285) + 6.149 * exp((v + 0.5096) / 20.27));
  const double tau_hs = 1.0 / (0.009794 * exp(-(v + 17.95) / 28.05) + 0.3343 * exp((v + 5.730) / 56.66));
  const double h_mix = 0.99 * s[O_HF] + (1.0 - 0.99) * s[O_HS];
  const double tau_j = 2.038 + 1.0 / (0.02136 * exp(-(v + 100.6) / 8.281) + 0.3052 * exp((v + 0.9941) / 38.45));
  const double hp_inf = sig((v + 89.1) / 6.086);
  const double tau_hsp = 3.0 * tau_hs;
  const double hp_mix = 0.99 * s[O_HF] + (1.0 - 0.99) * s[O_HSP];
  const double tau_jp = 1.46 * tau_j;
  const double m_cube = s[O_M] * s[O_M] * s[O_M];
  const double i_na = 75.0 * (v - ena) * m_cube * ((1.0 - fk) * h_mix * s[O_J] + fk * hp_mix * s[O_JP]);

  /* late sodium */
  const double ml_inf = sig(-(v + 42.85) / 5.264);
  const double hl_inf = sig((v + 87.61) / 7.488);
  const double hlp_inf = sig((v + 93.81) / 7.488);
  const double g_nal = 0.0075 * P->gnal;
  const double i_nal = g_nal * (v - ena) * s[O_ML] * ((1.0 - fk) * s[O_HL] + fk * s[O_HLP]);

  /* transient outward */
  const double a_inf = sig(-(v - 14.34) / 14.82);
  const double tau_a = 1.0515 / (1.0 / (1.2089 * (1.0 + exp(-(v - 18.4099) / 29.3814))) +
                                 3.5 / (1.0 + exp((v + 100.0) / 29.3814)));
  const double i_inf = sig((v + 43.94) / 5.711);
  const double d_epi = P->epi ? 1.0 - 0.95 / (1.0 + exp((v + 70.0) / 5.0)) : 1.0;
  const double tau_if = (4.562 + 1.0 / (0.3933 * exp(-(v + 100.0) / 100.0) + 0.08004 * exp((v + 50.0) / 16.59))) * d_epi;
  const double tau_is = (23.62 + 1.0 / (0.001416 * exp(-(v + 96.52) / 59.05) + 1.780e-8 * exp((v + 114.1) / 8.079))) * d_epi;
  const double a_if = sig((v - 213.6) / 151.2);
  const double a_is = 1.0 - a_if;
  const double i_mix = a_if * s[O_IF] + a_is * s[O_IS];
  const double ap_inf = sig(-(v - 24.34) / 14.82);
  const double dev = 1.354 + 1.0e-4 / (exp((v - 167.4) / 15.89) + exp(-(v - 12.23) / 0.2154));
  const double rec = 1.0 - 0.5 / (1.0 + exp((v + 70.0) / 20.0));
  const double tau_ifp = dev * rec * tau_if;
  const double tau_isp = dev * rec * tau_is;
  const double ip_mix = a_if * s[O_IFP] + a_is * s[O_ISP];
  const double g_to = 0.02 * P->gto;
  const double i_to = g_to * (v - ek) * ((1.0 - fk) * s[O_A] * i_mix + fk * s[O_AP] * ip_mix);

  /* L-type calcium (+ Na, K components) */
  const double d_inf = sig(-(v + 3.940) / 4.230);
  const double tau_d = 0.6 + 1.0 / (exp(-0.05 * (v + 6.0)) + exp(0.09 * (v + 14.0)));
  const double f_inf = sig((v + 19.58) / 3.696);
  const double tau_ff = 7.0 + 1.0 / (0.0045 * exp(-(v + 20.0) / 10.0) + 0.0045 * exp((v + 20.0) / 10.0));
  const double tau_fs = 1000.0 + 1.0 / (0.000035 * exp(-(v + 5.0) / 4.0) + 0.000035 * exp((v + 5.0) / 6.0));
  const double f_mix = 0.6 * s[O_FF] + (1.0 - 0.6) * s[O_FS];
  const double tau_fcaf = 7.0 + 1.0 / (0.04 * exp(-(v - 4.0) / 7.0) + 0.04 * exp((v - 4.0) / 7.0));
  const double tau_fcas = 100.0 + 1.0 / (0.00012 * exp(-v / 3.0) + 0.00012 * exp(v / 7.0));
  const double a_fcaf = 0.3 + 0.6 / (1.0 + exp((v - 10.0) / 10.0));
  const double a_fcas = 1.0 - a_fcaf;
  const double fca_mix = a_fcaf * s[O_FCAF] + a_fcas * s[O_FCAS];
  const double fp_mix = 0.6 * s[O_FFP] + (1.0 - 0.6) * s[O_FS];
  const double fcap_mix = a_fcaf * s[O_FCAFP] + a_fcas * s[O_FCAS];
  const double km2n = s[O_JCA] * 1.0;
  const double cn = 1.0 + 0.002 / cass;
  const double anca = 1.0 / (1000.0 / km2n + cn * cn * cn * cn);
  const double phi_cal = 2.0 * FARADAY * (cass * exp(2.0 * vfrt) - 0.341 * CAO) * xexpm1(2.0 * vfrt);
  const double phi_cana = FARADAY * (0.75 * nass * exp(vfrt) - 0.75 * NAO) * xexpm1(vfrt);
  const double phi_cak = FARADAY * (0.75 * kss * exp(vfrt) - 0.75 * KO) * xexpm1(vfrt);
  const double p_ca = 0.0001 * P->pca;
  const double p_cap = 1.1 * p_ca;
  const double p_cana = 0.00125 * p_ca, p_cak = 3.574e-4 * p_ca;
  const double p_canap = 0.00125 * p_cap, p_cakp = 3.574e-4 * p_cap;
  const double nca = s[O_NCA];
  const double g_np = s[O_D] * (f_mix * (1.0 - nca) + s[O_JCA] * fca_mix * nca);
  const double g_p = s[O_D] * (fp_mix * (1.0 - nca) + s[O_JCA] * fcap_mix * nca);
  const double i_cal = (1.0 - fk) * p_ca * phi_cal * g_np + fk * p_cap * phi_cal * g_p;
  const double i_cana = (1.0 - fk) * p_cana * phi_cana * g_np + fk * p_canap * phi_cana * g_p;
  const double i_cak = (1.0 - fk) * p_cak * phi_cak * g_np + fk * p_cakp * phi_cak * g_p;

  /* rapid delayed rectifier */
  const double xr_inf = sig(-(v + 8.337) / 6.789);
  const double tau_xrf = 12.98 + 1.0 / (0.3652 * exp((v - 31.66) / 3.869) + 4.123e-5 * exp(-(v - 47.78) / 20.38));
  const double tau_xrs = 1.865 + 1.0 / (0.06629 * exp((v - 34.70) / 7.355) + 1.128e-5 * exp(-(v - 29.74) / 25.94));
  const double a_xrf = sig((v + 54.81) / 38.21);
  const double a_xrs = 1.0 - a_xrf;
  const double xr_mix = a_xrf * s[O_XRF] + a_xrs * s[O_XRS];
  const double r_kr = 1.0 / (1.0 + exp((v + 55.0) / 75.0)) * 1.0 / (1.0 + exp((v - 10.0) / 30.0));
  const double g_kr = 0.046 * P->gkr * gkr_scale;
  const double i_kr = g_kr * sqrt(KO / 5.4) * xr_mix * r_kr * (v - ek);

  /* slow delayed rectifier */
  const double xs1_inf = sig(-(v + 11.60) / 8.932);
  const double tau_xs1 = 817.3 + 1.0 / (2.326e-4 * exp((v + 48.28) / 17.80) + 0.001292 * exp(-(v + 210.0) / 230.0));
  const double tau_xs2 = 1.0 / (0.01 * exp((v - 50.0) / 20.0) + 0.0193 * exp(-(v + 66.54) / 31.0));
  const double ks_ca = 1.0 + 0.6 / (1.0 + pow(3.8e-5 / cai, 1.4));
  const double g_ks = 0.0034 * P->gks;
  const double i_ks = g_ks * ks_ca * s[O_XS1] * s[O_XS2] * (v - eks);

  /* inward rectifier */
  const double xk1_inf = sig(-(v + 2.5538 * KO + 144.59) / (1.5692 * KO + 3.8115));
  const double tau_xk1 = 122.2 / (exp(-(v + 127.2) / 20.36) + exp((v + 236.8) / 69.33));
  const double r_k1 = sig((v + 105.8 - 2.6 * KO) / 9.493);
  const double g_k1 = 0.1908 * P->gk1;
  const double i_k1 = g_k1 * sqrt(KO) * r_k1 * s[O_XK1] * (v - ek);

  /* Na/Ca exchanger */
  const double hca = exp(0.1670 * vfrt);
  const double hna = exp(0.5224 * vfrt);
  const double g_ncx = 0.0008 * P->gncx;
  const double i_naca_i = 0.8 * g_ncx * ncx_flux(nai, cai, hna, hca);
  const double i_naca_ss = 0.2 * g_ncx * ncx_flux(nass, cass, hna, hca);

  /* Na/K pump */
  const double knai = 9.073 * exp(-0.1550 * vfrt / 3.0);
  const double knao = 27.78 * exp((1.0 - -0.1550) * vfrt / 3.0);
  const double p_hp = 4.2 / (1.0 + 1.0e-7 / 1.698e-7 + nai / 224.0 + ki / 292.0);
  const double ri = nai / knai, rk = ki / 0.5;
  const double ro = NAO / knao, rko = KO / 0.3582;
  const double ci = pow(1.0 + ri, 3.0), qi = pow(1.0 + rk, 2.0);
  const double co = pow(1.0 + ro, 3.0), qo = pow(1.0 + rko, 2.0);
  const double a1 = 949.5 * pow(ri, 3.0) / (ci + qi - 1.0);
  const double b1 = 182.4 * 0.05;
  const double a2 = 687.2;
  const double b2 = 39.4 * pow(ro, 3.0) / (co + qo - 1.0);
  const double a3 = 1899.0 * pow(rko, 2.0) / (co + qo - 1.0);
  const double b3 = 79300.0 * p_hp * 1.0e-7 / (1.0 + 9.8 / 1.698e-7);
  const double a4 = 639.0 * 9.8 / 1.698e-7 / (1.0 + 9.8 / 1.698e-7);
  const double b4 = 40.0 * pow(rk, 2.0) / (ci + qi - 1.0);
  const double y1 = a4 * a1 * a2 + b2 * b4 * b3 + a2 * b4 * b3 + b3 * a1 * a2;
  const double y2 = b2 * b1 * b4 + a1 * a2 * a3 + a3 * b1 * b4 + a2 * a3 * b4;
  const double y3 = a2 * a3 * a4 + b3 * b2 * b1 + b2 * b1 * a4 + a3 * a4 * b1;
  const double y4 = b4 * b3 * b2 + a3 * a4 * a1 + b2 * a4 * a1 + b3 * b2 * a1;
  const double ysum = y1 + y2 + y3 + y4;
  const double f1 = y1 / ysum, f2 = y2 / ysum, f3 = y3 / ysum, f4 = y4 / ysum;
  const double jnak_na = 3.0 * (f1 * a3 - f2 * b3);
  const double jnak_k = 2.0 * (f4 * b1 - f3 * a1);
  const double p_nak = 30.0 * P->pnak;
  const double i_nak = p_nak * (1.0 * jnak_na + 1.0 * jnak_k);

  /* background currents */
  const double x_kb = sig(-(v - 14.48) / 18.34);
  const double g_kb = 0.003 * P->gkb;
  const double i_kb = g_kb * x_kb * (v - ek);
  const double i_nab = 3.75e-10 * FARADAY * (nai * exp(vfrt) - NAO) * xexpm1(vfrt);
  const double i_cab = 2.5e-8 * 2.0 * FARADAY * (cai * exp(2.0 * vfrt) - 0.341 * CAO) * xexpm1(2.0 * vfrt);
  const double i_pca = 0.0005 * cai / (0.0005 + cai);

  /* fluxes and buffering */
  const double jd_na = (nass - nai) / 2.0;
  const double jd_k = (kss - ki) / 2.0;
  const double jd_ca = (cass - cai) / 0.2;
  const double jrel_gate = 1.0 + pow(1.5 / cajsr, 8.0);
  const double jrel_inf = 0.5 * 4.75 * (-i_cal) / jrel_gate * P->jrel;
  double tau_rel = 4.75 / (1.0 + 0.0123 / cajsr);
  if (tau_rel < 0.005) tau_rel = 0.005;
  const double jrelp_inf = 0.5 * (1.25 * 4.75) * (-i_cal) / jrel_gate * P->jrel;
  double tau_relp = (1.25 * 4.75) / (1.0 + 0.0123 / cajsr);
  if (tau_relp < 0.005) tau_relp = 0.005;
  const double j_rel = (1.0 - fk) * s[O_JRELNP] + fk * s[O_JRELP];
  const double jup_np = 0.004375 * cai / (cai + 0.00092) * P->jup;
  const double jup_p = 2.75 * 0.004375 * cai / (cai + 0.00092 - 0.00017) * P->jup;
  const double j_leak = 0.0039375 * cansr / 15.0;
  const double j_up = (1.0 - fk) * jup_np + fk * jup_p - j_leak;
  const double j_tr = (cansr - cajsr) / 100.0;
  const double cmdn = 0.05 * P->cmdn;
  const double kc = 0.00238 + cai, kt = 0.0005 + cai;
  const double b_cai = 1.0 / (1.0 + cmdn * 0.00238 / (kc * kc) + 0.07 * 0.0005 / (kt * kt));
  const double kb = 0.00087 + cass, kl = 0.0087 + cass;
  const double b_cass = 1.0 / (1.0 + 0.047 * 0.00087 / (kb * kb) + 1.124 * 0.0087 / (kl * kl));
  const double kq = 0.8 + cajsr;
  const double b_cajsr = 1.0 / (1.0 + 10.0 * 0.8 / (kq * kq));

  /* gates: (x_inf - x) / tau */
  ds[O_M] = (m_inf - s[O_M]) / tau_m;
  ds[O_HF] = (h_inf - s[O_HF]) / tau_hf;
  ds[O_HS] = (h_inf - s[O_HS]) / tau_hs;
  ds[O_J] = (h_inf - s[O_J]) / tau_j;
  ds[O_HSP] = (hp_inf - s[O_HSP]) / tau_hsp;
  ds[O_JP] = (h_inf - s[O_JP]) / tau_jp;
  ds[O_ML] = (ml_inf - s[O_ML]) / tau_m;
  ds[O_HL] = (hl_inf - s[O_HL]) / 200.0;
  ds[O_HLP] = (hlp_inf - s[O_HLP]) / (3.0 * 200.0);
  ds[O_A] = (a_inf - s[O_A]) / tau_a;
  ds[O_IF] = (i_inf - s[O_IF]) / tau_if;
  ds[O_IS] = (i_inf - s[O_IS]) / tau_is;
  ds[O_AP] = (ap_inf - s[O_AP]) / tau_a;
  ds[O_IFP] = (i_inf - s[O_IFP]) / tau_ifp;
  ds[O_ISP] = (i_inf - s[O_ISP]) / tau_isp;
  ds[O_D] = (d_inf - s[O_D]) / tau_d;
  ds[O_FF] = (f_inf - s[O_FF]) / tau_ff;
  ds[O_FS] = (f_inf - s[O_FS]) / tau_fs;
  ds[O_FCAF] = (f_inf - s[O_FCAF]) / tau_fcaf;
  ds[O_FCAS] = (f_inf - s[O_FCAS]) / tau_fcas;
  ds[O_JCA] = (f_inf - s[O_JCA]) / 75.0;
  ds[O_NCA] = anca * 1000.0 - km2n * nca;
  ds[O_FFP] = (f_inf - s[O_FFP]) / (2.5 * tau_ff);
  ds[O_FCAFP] = (f_inf - s[O_FCAFP]) / (2.5 * tau_fcaf);
  ds[O_XRF] = (xr_inf - s[O_XRF]) / tau_xrf;
  ds[O_XRS] = (xr_inf - s[O_XRS]) / tau_xrs;
  ds[O_XS1] = (xs1_inf - s[O_XS1]) / tau_xs1;
  ds[O_XS2] = (xs1_inf - s[O_XS2]) / tau_xs2;
  ds[O_XK1] = (xk1_inf - s[O_XK1]) / tau_xk1;
  ds[O_JRELNP] = (jrel_inf - s[O_JRELNP]) / tau_rel;
  ds[O_JRELP] = (jrelp_inf - s[O_JRELP]) / tau_relp;
  ds[O_CAMKT] = 0.05 * camk_b * (camk_b + s[O_CAMKT]) - 0.00068 * s[O_CAMKT];

  /* concentrations */
  ds[O_NAI] = -(i_na + i_nal + 3.0 * i_naca_i + 3.0 * i_nak + i_nab) * ACAP / (FARADAY * VMYO) + jd_na * VSS / VMYO;
  ds[O_NASS] = -(i_cana + 3.0 * i_naca_ss) * ACAP / (FARADAY * VSS) - jd_na;
  ds[O_KI] = -(i_to + i_kr + i_ks + i_k1 + i_kb - 2.0 * i_nak) * ACAP / (FARADAY * VMYO) + jd_k * VSS / VMYO;
  ds[O_KSS] = -i_cak * ACAP / (FARADAY * VSS) - jd_k;
  ds[O_CAI] = b_cai * (-(i_pca + i_cab - 2.0 * i_naca_i) * ACAP / (2.0 * FARADAY * VMYO) - j_up * VNSR / VMYO + jd_ca * VSS / VMYO);
  ds[O_CASS] = b_cass * (-(i_cal - 2.0 * i_naca_ss) * ACAP / (2.0 * FARADAY * VSS) + j_rel * VJSR / VSS - jd_ca);
  ds[O_CANSR] = j_up - j_tr * VJSR / VNSR;
  ds[O_CAJSR] = b_cajsr * (j_tr - j_rel);

  *dv = -(i_na + i_nal + i_to + i_cal + i_cana + i_cak + i_kr + i_ks + i_k1 + i_naca_i + i_naca_ss + i_nak + i_kb +
          i_nab + i_pca + i_cab) +
        i_stim;
}

/* rest states (ohara_rudy_2011.cpp:454-489, maccannell_2007.cpp:25-26,
 * aliev_panfilov.cpp:22): the published 17-digit constants */
static const double kRestOrd[3][41] = {
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

int cwo_state_count(int kind) {
  switch (kind) {
    case CWO_AP: return 1;
    case CWO_MAC: return 2;
    case CWO_PASSIVE: return 0;
    default: return O_COUNT;
  }
}

double cwo_stable_step(int kind) {
  switch (kind) {
    case CWO_AP: return 1.0;
    case CWO_MAC: return 0.1;
    case CWO_PASSIVE: return 1.0;
    default: return 0.01;
  }
}

void cwo_rest_state(int kind, double* out) {
  switch (kind) {
    case CWO_AP: out[0] = -80.0; out[1] = 0.0; return;
    case CWO_MAC:
      out[0] = -48.865796143695611; out[1] = 0.067599408770662575; out[2] = 0.97575886906521692;
      return;
    case CWO_PASSIVE: out[0] = PASSIVE_E; return;
    default: memcpy(out, kRestOrd[kind - CWO_ORD_ENDO], sizeof(kRestOrd[0])); return;
  }
}

void cwo_rates(int kind, double v, const double* s, double i_stim, double gkr_scale, double* dv,
               double* ds) {
  switch (kind) {
    case CWO_AP: ap_rates(v, s, i_stim, dv, ds); return;
    case CWO_MAC: mac_rates(v, s, i_stim, dv, ds); return;
    case CWO_PASSIVE: passive_rates(v, i_stim, dv); return;
    default: ord_rates(kind - CWO_ORD_ENDO, v, s, i_stim, gkr_scale, dv, ds); return;
  }
}

void cwo_rates_batch(int kind, int64_t n, const double* v, const double* s, const double* i_stim,
                     double* dv, double* ds) {
  const int ns = cwo_state_count(kind);
  for (int64_t i = 0; i < n; ++i) cwo_rates(kind, v[i], s + i * ns, i_stim[i], 1.0, &dv[i], ds + i * ns);
}

/* ------------------------------------------------------------------ *
 * Single-cell pacing (pace_to_steady_state, ionic.cpp:122-165; euler   *
 * step :74-83; BeatMarkers :86-118). Returns 0, or 1 on validation     *
 * error, 2 on non-finite V, 3 on |V| > 1000 mV (fail_beat / fail_t set). *
 * ------------------------------------------------------------------ */
int cwo_pace(int kind, double cycle_ms, int n_beats, double amp, double dur, double* state_out,
             double* apd_out, double* max_rel, int* fail_beat, double* fail_t) {
  if (n_beats < 1 || !(cycle_ms > 0.0)) return 1;
  const int ns = cwo_state_count(kind);
  const double dt = cwo_stable_step(kind) / 2.0;
  const int64_t spb = llround(cycle_ms / dt);
  double st[64], eds[64], prev[64], ds[64];
  int have_prev = 0;
  cwo_rest_state(kind, st);
  for (int beat = 0; beat < n_beats; ++beat) {
    const double v_rest = st[0];
    double max_slope = -INFINITY, t_max = NAN, v_peak = -INFINITY, apd = NAN;
    int closed = 0;
    double v_prev = st[0];
    for (int64_t i = 0; i < spb; ++i) {
      const double t_in = (double)i * dt;
      const double ist = t_in < dur ? amp : 0.0;
      double dv = 0.0;
      cwo_rates(kind, st[0], st + 1, ist, 1.0, &dv, ds);
      st[0] += dt * dv;
      for (int k = 0; k < ns; ++k) st[1 + k] += dt * ds[k];
      if (!isfinite(st[0]) || fabs(st[0]) > 1000.0) {
        *fail_beat = beat;
        *fail_t = (double)beat * cycle_ms + t_in;
        return isfinite(st[0]) ? 3 : 2;
      }
      if (!closed) {
        const double t = t_in + dt, slope = (st[0] - v_prev) / dt;
        if (slope > max_slope) {
          max_slope = slope;
          t_max = t;
        }
        if (st[0] > v_peak) v_peak = st[0];
        if (isfinite(t_max) && v_peak > 0.0) {
          const double v90 = v_peak - 0.9 * (v_peak - v_rest);
          if (st[0] < v90 && v_peak - v_rest > 20.0) {
            apd = t - t_max;
            closed = 1;
          }
        }
      }
      v_prev = st[0];
    }
    apd_out[beat] = apd;
    if (beat > 0) {
      memcpy(prev, eds, sizeof(double) * (size_t)(ns + 1));
      have_prev = 1;
    }
    memcpy(eds, st, sizeof(double) * (size_t)(ns + 1));
  }
  memcpy(state_out, st, sizeof(double) * (size_t)(ns + 1));
  double mr = 0.0;
  if (have_prev) {
    for (int k = 0; k <= ns; ++k) {
      const double scale = fabs(prev[k]) < fabs(eds[k]) ? fabs(eds[k]) : fabs(prev[k]);
      if (scale > 1e-12) {
        const double r = fabs(eds[k] - prev[k]) / scale;
        if (mr < r) mr = r;
      }
    }
  }
  *max_rel = mr;
  return 0;
}

/* ------------------------------------------------------------------ *
 * Adaptation rules (splitting.cpp:48-72)                               *
 * ------------------------------------------------------------------ */
int cwo_reaction_substeps(double dvdt_prev, int scheme, int k0_up, int k0_down, int k_max) {
  if (scheme == CWO_OST) return 1;
  const double base = dvdt_prev > 0.0 ? (double)k0_up : (double)k0_down;
  const double raw = base + floor(fabs(dvdt_prev));
  if (raw > (double)k_max) return k_max;
  const int k = (int)raw;
  return k < 1 ? 1 : k;
}

int cwo_diffusion_substeps(double dt, double dt_s, int strict, int scheme, int* l, double* dt_ad) {
  if (!(dt > 0.0) || !(dt_s > 0.0)) return 2;
  int ll = 1;
  if (scheme == CWO_DAETI && dt / 2.0 > dt_s) {
    const double q = dt / (2.0 * dt_s);
    ll = (int)(strict ? ceil(q) : floor(q));
    if (ll < 1) ll = 1;
  }
  *l = ll;
  *dt_ad = dt / (2.0 * ll);
  return 0;
}

int cwo_k_max_for(double dt, double stable_step) {
  const int k = (int)floor(dt / stable_step);
  return k < 1 ? 1 : k;
}

/* ------------------------------------------------------------------ *
 * Stimulus (stimulus.cpp:33-45)                                        *
 * ------------------------------------------------------------------ */
double cwo_stim_current(const cwo_protocol* p, int64_t node, double t) {
  double acc = 0.0;
  if (!p) return 0.0;
  for (int32_t q = p->node_ptr[node]; q < p->node_ptr[node + 1]; ++q) {
    const int32_t e = p->ids[q];
    if (t < p->t_start[e]) continue;
    if (!isnan(p->period[e])) {
      if (fmod(t - p->t_start[e], p->period[e]) < p->duration[e]) acc += p->amplitude[e];
    } else if (t < p->t_start[e] + p->duration[e]) {
      acc += p->amplitude[e];
    }
  }
  return acc;
}

/* ------------------------------------------------------------------ *
 * Diffusion sub-step (fem.cpp:194-207)                                 *
 * ------------------------------------------------------------------ */
void cwo_diffusion_substep_csr(int64_t n, const int64_t* row_ptr, const int64_t* col,
                               const double* val, const double* mass, const double* v,
                               double dt_sub, double* out) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    double acc = 0.0;
    for (int64_t q = row_ptr[i]; q < row_ptr[i + 1]; ++q) acc += val[q] * v[col[q]];
    out[i] = v[i] - dt_sub / mass[i] * acc;
  }
}

/* ------------------------------------------------------------------ *
 * Reaction pass (splitting.cpp:95-155)                                 *
 * ------------------------------------------------------------------ */
int64_t cwo_reaction_step(int64_t n, int stride, double* v, double* s, double* last_dvdt,
                          const uint8_t* model_of_node, const int* model_kind, const int* k_max,
                          const double* gkr_scale, const cwo_protocol* prot, int scheme, int k0_up,
                          int k0_down, double dt, double t, int64_t* khist, double* bad_t) {
  int64_t bad = -1;
  double bt = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const int mid = model_of_node[i];
    const int kind = model_kind[mid];
    const int k = cwo_reaction_substeps(last_dvdt[i], scheme, k0_up, k0_down, k_max[mid]);
    khist[k] += 1;
    const double h = dt / (double)k;
    const int ns = cwo_state_count(kind);
    const double g = gkr_scale ? gkr_scale[i] : 1.0;
    double vi = v[i];
    double* si = s + i * stride;
    double dv = 0.0, ds[64];
    for (int j = 0; j < k; ++j) {
      const double ts = t + (double)j * h;
      const double cur = cwo_stim_current(prot, i, ts);
      cwo_rates(kind, vi, si, cur, g, &dv, ds);
      vi += h * dv;
      for (int q = 0; q < ns; ++q) si[q] += h * ds[q];
      if (!isfinite(vi)) {
        if (bad < 0) {
          bad = i;
          bt = ts;
        }
        break;
      }
    }
    v[i] = vi;
    last_dvdt[i] = dv;
  }
  if (bad_t) *bad_t = bt;
  return bad;
}

/* Same pass with the node loop spread over OpenMP threads, as the
 * reference's own `#pragma omp parallel for` (splitting.cpp:104-149): every
 * node is independent, so any schedule gives the same bits; the k-histogram
 * is summed per thread and the lowest failing node wins. */
int64_t cwo_reaction_step_omp(int64_t n, int stride, double* v, double* s, double* last_dvdt,
                              const uint8_t* model_of_node, const int* model_kind, const int* k_max,
                              const double* gkr_scale, const cwo_protocol* prot, int scheme, int k0_up,
                              int k0_down, double dt, double t, int64_t* khist, int khist_len, double* bad_t) {
  int64_t bad = -1;
  double bt = 0.0;
#pragma omp parallel
  {
    int64_t lh[64] = {0};
    int64_t lbad = -1;
    double lbt = 0.0;
#pragma omp for schedule(dynamic, 256)
    for (int64_t i = 0; i < n; ++i) {
      const int mid = model_of_node[i];
      const int kind = model_kind[mid];
      const int k = cwo_reaction_substeps(last_dvdt[i], scheme, k0_up, k0_down, k_max[mid]);
      lh[k] += 1;
      const double h = dt / (double)k;
      const int ns = cwo_state_count(kind);
      const double g = gkr_scale ? gkr_scale[i] : 1.0;
      double vi = v[i];
      double* si = s + i * stride;
      double dv = 0.0, ds[64];
      for (int j = 0; j < k; ++j) {
        const double ts = t + (double)j * h;
        const double cur = cwo_stim_current(prot, i, ts);
        cwo_rates(kind, vi, si, cur, g, &dv, ds);
        vi += h * dv;
        for (int q = 0; q < ns; ++q) si[q] += h * ds[q];
        if (!isfinite(vi)) {
          if (lbad < 0 || i < lbad) {
            lbad = i;
            lbt = ts;
          }
          break;
        }
      }
      v[i] = vi;
      last_dvdt[i] = dv;
    }
#pragma omp critical
    {
      for (int q = 0; q < khist_len && q < 64; ++q) khist[q] += lh[q];
      if (lbad >= 0 && (bad < 0 || lbad < bad)) {
        bad = lbad;
        bt = lbt;
      }
    }
  }
  if (bad_t) *bad_t = bt;
  return bad;
}

/* ------------------------------------------------------------------ *
 * Activation detector (postprocess.cpp:15-66)                          *
 * ------------------------------------------------------------------ */
void cwo_detector_init(cwo_detector* d, int64_t n, double threshold) {
  memset(d, 0, sizeof(*d));
  d->n = n;
  d->threshold = threshold;
  d->first = 1;
  double** arrs[] = {&d->prev_v, &d->v_rest, &d->max_slope, &d->t_max_slope, &d->v_peak, &d->lat, &d->apd};
  for (int a = 0; a < 7; ++a) *arrs[a] = (double*)calloc((size_t)n, sizeof(double));
  d->phase = (uint8_t*)calloc((size_t)n, 1);
  d->has_lat = (uint8_t*)calloc((size_t)n, 1);
  d->has_apd = (uint8_t*)calloc((size_t)n, 1);
}

void cwo_detector_free(cwo_detector* d) {
  free(d->prev_v); free(d->v_rest); free(d->max_slope); free(d->t_max_slope); free(d->v_peak);
  free(d->lat); free(d->apd); free(d->phase); free(d->has_lat); free(d->has_apd);
  memset(d, 0, sizeof(*d));
}

void cwo_detector_observe(cwo_detector* d, double t, const double* v) {
  if (d->first) {
    for (int64_t i = 0; i < d->n; ++i) {
      d->prev_v[i] = v[i];
      d->v_rest[i] = v[i];
      d->max_slope[i] = -INFINITY;
    }
    d->prev_t = t;
    d->first = 0;
    return;
  }
  const double h = t - d->prev_t;
  const double thr = d->threshold;
  for (int64_t i = 0; i < d->n; ++i) {
    if (d->phase[i] == 2) continue;
    const double x = v[i], px = d->prev_v[i];
    const double slope = (x - px) / h;
    if (slope > d->max_slope[i]) {
      d->max_slope[i] = slope;
      d->t_max_slope[i] = d->prev_t + 0.5 * h;
    }
    if (d->phase[i] == 0) {
      if (px < thr && x >= thr) {
        d->lat[i] = d->prev_t + (thr - px) / (x - px) * h;
        d->has_lat[i] = 1;
        d->phase[i] = 1;
        d->v_peak[i] = x;
      } else {
        d->v_rest[i] = x < d->v_rest[i] ? x : d->v_rest[i]; /* std::min(a, b) = b < a ? b : a */
      }
    } else {
      if (d->v_peak[i] < x) d->v_peak[i] = x; /* std::max(a, b) = a < b ? b : a */
      const double v90 = d->v_peak[i] - 0.9 * (d->v_peak[i] - d->v_rest[i]);
      if (px >= v90 && x < v90 && d->v_peak[i] - d->v_rest[i] >= 20.0) {
        const double tc = d->prev_t + (px - v90) / (px - x) * h;
        d->apd[i] = tc - d->t_max_slope[i];
        d->has_apd[i] = 1;
        d->phase[i] = 2;
      }
    }
    d->prev_v[i] = x;
  }
  d->prev_t = t;
}

/* ------------------------------------------------------------------ *
 * 3D slab assembly (EXTENSION; the 3D analogue of fem.cpp:63-176)     *
 * ------------------------------------------------------------------ */
static void hex_integrals(double h, const double D[3][3], double k[8][8], double m[8]) {
  const double g = 0.57735026918962576;
  const double gp[2] = {-g, g};
  for (int a = 0; a < 8; ++a) {
    m[a] = 0.0;
    for (int b = 0; b < 8; ++b) k[a][b] = 0.0;
  }
  const double det = h * h * h / 8.0;
  const double sc = 2.0 / h;
  for (int q = 0; q < 8; ++q) {
    const double xi = gp[q & 1], eta = gp[(q >> 1) & 1], zeta = gp[q >> 2];
    double n[8], gx[8], gy[8], gz[8];
    for (int a = 0; a < 8; ++a) {
      const double sx = (a & 1) ? 1.0 : -1.0, sy = (a & 2) ? 1.0 : -1.0, sz = (a & 4) ? 1.0 : -1.0;
      const double fx = 1.0 + sx * xi, fy = 1.0 + sy * eta, fz = 1.0 + sz * zeta;
      n[a] = 0.125 * fx * fy * fz;
      gx[a] = sc * (0.125 * sx * fy * fz);
      gy[a] = sc * (0.125 * fx * sy * fz);
      gz[a] = sc * (0.125 * fx * fy * sz);
    }
    for (int a = 0; a < 8; ++a) {
      const double dgx = D[0][0] * gx[a] + D[0][1] * gy[a] + D[0][2] * gz[a];
      const double dgy = D[1][0] * gx[a] + D[1][1] * gy[a] + D[1][2] * gz[a];
      const double dgz = D[2][0] * gx[a] + D[2][1] * gy[a] + D[2][2] * gz[a];
      for (int b = 0; b < 8; ++b) k[a][b] += det * (dgx * gx[b] + dgy * gy[b] + dgz * gz[b]);
      m[a] += det * n[a];
    }
  }
}

double cwo_assemble_slab3d(int64_t nx, int64_t ny, int64_t nz, double h, double d_long, double rho,
                           const double* angle_of_layer, int64_t** row_ptr_out, int64_t** col_out,
                           double** val_out, double** mass_out) {
  const int64_t nx1 = nx + 1, ny1 = ny + 1, nz1 = nz + 1, n = nx1 * ny1 * nz1;
  double* acc = (double*)calloc((size_t)n * 27, sizeof(double));
  unsigned char* has = (unsigned char*)calloc((size_t)n * 27, 1);
  double* mass = (double*)calloc((size_t)n, sizeof(double));
  double(*K)[8][8] = (double(*)[8][8])malloc((size_t)nz * sizeof(double[8][8]));
  double(*M)[8] = (double(*)[8])malloc((size_t)nz * sizeof(double[8]));
  for (int64_t ez = 0; ez < nz; ++ez) {
    const double th = angle_of_layer[ez];
    const double f[3] = {cos(th), sin(th), 0.0};
    const double dt = rho * d_long;
    double D[3][3];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        const double ff = f[i] * f[j];
        D[i][j] = d_long * ff + dt * ((i == j ? 1.0 : 0.0) - ff);
      }
    hex_integrals(h, D, K[ez], M[ez]);
  }
  /* element loop in ascending element index e = (ey*nz + ez)*nx + ex */
  for (int64_t ey = 0; ey < ny; ++ey)
    for (int64_t ez = 0; ez < nz; ++ez)
      for (int64_t ex = 0; ex < nx; ++ex)
        for (int a = 0; a < 8; ++a) {
          const int64_t ix = ex + (a & 1), iy = ey + ((a >> 1) & 1), iz = ez + ((a >> 2) & 1);
          const int64_t i = (iy * nz1 + iz) * nx1 + ix;
          mass[i] += M[ez][a];
          for (int b = 0; b < 8; ++b) {
            const int64_t dx = ex + (b & 1) - ix, dy = ey + ((b >> 1) & 1) - iy, dz = ez + ((b >> 2) & 1) - iz;
            const int64_t slot = i * 27 + (dy + 1) * 9 + (dz + 1) * 3 + (dx + 1);
            acc[slot] += K[ez][a][b];
            has[slot] = 1;
          }
        }
  int64_t nnz = 0;
  for (int64_t s = 0; s < n * 27; ++s) nnz += has[s];
  int64_t* rp = (int64_t*)malloc((size_t)(n + 1) * sizeof(int64_t));
  int64_t* col = (int64_t*)malloc((size_t)nnz * sizeof(int64_t));
  double* val = (double*)malloc((size_t)nnz * sizeof(double));
  const int64_t plane = nz1 * nx1;
  int64_t p = 0;
  double min_ratio = INFINITY;
  for (int64_t i = 0; i < n; ++i) {
    rp[i] = p;
    double den = 0.0;
    /* slots in (dy, dz, dx) lexicographic order == ascending column index */
    for (int q = 0; q < 27; ++q) {
      if (!has[i * 27 + q]) continue;
      const int64_t dy = q / 9 - 1, dz = (q / 3) % 3 - 1, dx = q % 3 - 1;
      col[p] = i + dy * plane + dz * nx1 + dx;
      val[p] = acc[i * 27 + q];
      den += q == 13 ? val[p] : fabs(val[p]);
      ++p;
    }
    if (den > 0.0 && mass[i] / den < min_ratio) min_ratio = mass[i] / den;
  }
  rp[n] = p;
  free(acc);
  free(has);
  free(K);
  free(M);
  *row_ptr_out = rp;
  *col_out = col;
  *val_out = val;
  *mass_out = mass;
  return 0.9 * min_ratio;
}

void cwo_free(void* p) { free(p); }

/* Node-class tables of the slab operator, from the oracle's own CSR assembly
 * of a 2 x 2 x nz-element slab: every class (x face 0 / interior / nx, y
 * face likewise, z layer) has a representative row there, and a row's
 * coefficients are sums of its own elements' contributions in ascending
 * element index, whatever the slab's extent in x and y. Layout as the
 * structured operator: cls = (by*3 + bx)*(nz+1) + iz, slot q = (dy+1)*9 +
 * (dz+1)*3 + (dx+1) (absent neighbours 0). Returns dt_s of any slab with
 * nx, ny >= 2 (Gershgorin over the class rows, which are all its rows). */
double cwo_slab3d_classes(int64_t nz, double h, double d_long, double rho, const double* angle_of_layer,
                          double* coef, double* mass_out) {
  int64_t *rp, *col;
  double *val, *mass;
  const double dt_s = cwo_assemble_slab3d(2, 2, nz, h, d_long, rho, angle_of_layer, &rp, &col, &val, &mass);
  const int64_t nz1 = nz + 1, plane = nz1 * 3;
  for (int by = 0; by < 3; ++by)
    for (int bx = 0; bx < 3; ++bx)
      for (int64_t iz = 0; iz < nz1; ++iz) {
        const int64_t cls = (by * 3 + bx) * nz1 + iz;
        const int64_t i = (by * nz1 + iz) * 3 + bx;
        double* cf = coef + cls * 27;
        for (int q = 0; q < 27; ++q) cf[q] = 0.0;
        for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
          /* (dy, dz, dx) from the column's grid coordinates (offsets alone are ambiguous for thin slabs) */
          const int64_t cy = col[p] / plane, cz = (col[p] % plane) / 3, cx = col[p] % 3;
          const int64_t dy = cy - by, dz = cz - iz, dx = cx - bx;
          cf[(dy + 1) * 9 + (dz + 1) * 3 + (dx + 1)] = val[p];
        }
        mass_out[cls] = mass[i];
      }
  free(rp);
  free(col);
  free(val);
  free(mass);
  return dt_s;
}

/* diffusion_substep (fem.cpp:194-207) on the structured slab: the same row
 * sum in ascending column order ((dy, dz, dx) lexicographic for the y-outer
 * numbering) over the present neighbours, then v - dt/m * acc. OpenMP over
 * nodes (fem.cpp:198). */
void cwo_diffusion_substep_slab3d(int64_t nx1, int64_t ny1, int64_t nz1, const double* coef, const double* mass,
                                  const double* v, double dt_sub, double* out) {
  const int64_t plane = nx1 * nz1;
#pragma omp parallel for schedule(static) collapse(2)
  for (int64_t iy = 0; iy < ny1; ++iy)
    for (int64_t iz = 0; iz < nz1; ++iz) {
      const int by = iy == 0 ? 0 : (iy == ny1 - 1 ? 2 : 1);
      for (int64_t ix = 0; ix < nx1; ++ix) {
        const int bx = ix == 0 ? 0 : (ix == nx1 - 1 ? 2 : 1);
        const int64_t cls = (by * 3 + bx) * nz1 + iz;
        const double* cf = coef + cls * 27;
        const int64_t i = iy * plane + iz * nx1 + ix;
        double acc = 0.0;
        for (int dy = -1; dy <= 1; ++dy) {
          if ((dy < 0 && by == 0) || (dy > 0 && by == 2)) continue;
          for (int dz = -1; dz <= 1; ++dz) {
            if ((dz < 0 && iz == 0) || (dz > 0 && iz == nz1 - 1)) continue;
            for (int dx = -1; dx <= 1; ++dx) {
              if ((dx < 0 && bx == 0) || (dx > 0 && bx == 2)) continue;
              acc += cf[(dy + 1) * 9 + (dz + 1) * 3 + (dx + 1)] * v[i + dy * plane + dz * nx1 + dx];
            }
          }
        }
        out[i] = v[i] - dt_sub / mass[cls] * acc;
      }
    }
}

/* MT19937-64 (Matsumoto & Nishimura 2004; the generator behind the
 * reference's std::mt19937_64, mesh.cpp:112): 312-word state, seeded by
 * x_i = 6364136223846793005 * (x_{i-1} ^ (x_{i-1} >> 62)) + i. */
typedef struct {
  uint64_t mt[312];
  int mti;
} cwo_mt64;

static void mt64_seed(cwo_mt64* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i) g->mt[i] = 6364136223846793005ull * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->mti = 312;
}

static uint64_t mt64_next(cwo_mt64* g) {
  const uint64_t A = 0xB5026F5AA96619E9ull, UM = 0xFFFFFFFF80000000ull, LM = 0x7FFFFFFFull;
  if (g->mti >= 312) {
    for (int i = 0; i < 312; ++i) {
      const uint64_t x = (g->mt[i] & UM) | (g->mt[(i + 1) % 312] & LM);
      g->mt[i] = g->mt[(i + 156) % 312] ^ (x >> 1) ^ ((x & 1ull) ? A : 0ull);
    }
    g->mti = 0;
  }
  uint64_t x = g->mt[g->mti++];
  x ^= (x >> 29) & 0x5555555555555555ull;
  x ^= (x << 17) & 0x71D67FFFEDA60000ull;
  x ^= (x << 37) & 0xFFF7EEE000000000ull;
  x ^= x >> 43;
  return x;
}

/* raw outputs (known-answer pin: the C++ standard requires the 10000th output
 * of a default-seeded (5489) mt19937_64 to be 9981545732273789042) */
void cwo_mt64_raw(uint64_t seed, int64_t n, uint64_t* out) {
  cwo_mt64 g;
  mt64_seed(&g, seed);
  for (int64_t k = 0; k < n; ++k) out[k] = mt64_next(&g);
}

/* uniform draws lo + (hi - lo) * ((x >> 11) * 2^-53) for the synthetic configurations */
void cwo_uniform_mt64(uint64_t seed, int64_t n, double lo, double hi, double* out) {
  cwo_mt64 g;
  mt64_seed(&g, seed);
  const double w = hi - lo;
  for (int64_t k = 0; k < n; ++k) out[k] = lo + w * ((double)(mt64_next(&g) >> 11) * 0x1.0p-53);
}
