// Table-based FP64 0.5 ln(x) shared by the IK1 kernels (see wq_fast.cu for
// the table: 16 mantissa bins c_j = 1/mid_j and the double-double
// 0.5 (-ln c_j), so 16 doubles span the 32 shared-memory banks once).
#pragma once
#include "wq_common.cuh"

namespace wq {

// 0.5 ln 2 = HLN2_A + HLN2_B, HLN2_A with 41 significant bits (e*A exact)
constexpr double HLN2_A = 0.3465735902798315;
constexpr double HLN2_B = 1.4117645281515789e-13;

__device__ __forceinline__ double half_ln16(double x, const double* __restrict__ tab) {
  const int hi = __double2hiint(x);
  const int lo = __double2loint(x);
  const int e = (hi >> 20) - 1023;
  const int j = (hi >> 16) & 15;
  const double m = __hiloint2double((hi & 0x000fffff) | 0x3ff00000, lo);
  const double r = fma(m, tab[j], -1.0);  // |r| < 2^-5
  double q = fma(r, 0.5 / 9.0, -0.5 / 8.0);  // degree 9: truncation < 1.1e-19
  q = fma(r, q, 0.5 / 7.0);
  q = fma(r, q, -0.5 / 6.0);
  q = fma(r, q, 0.5 / 5.0);
  q = fma(r, q, -0.5 / 4.0);
  q = fma(r, q, 0.5 / 3.0);
  q = fma(r, q, -0.25);
  const double r2 = r * r;
  const double de = (double)e;
  const double t_hi = fma(de, HLN2_A, tab[16 + j]);
  const double t_lo = fma(de, HLN2_B, tab[32 + j]);
  return t_hi + fma(r, 0.5, fma(r2, q, t_lo));
}


// Accurate-table variant (Tang): c_j (24 significant bits) near 1/mid_j is
// chosen so that 0.5 (-ln c_j) lies within 2.3e-4 ulp of the double stored
// next to it (tools/tang_table.py), so one {c_j, log_j} pair per bin replaces
// the double-double: one 16-byte shared-memory load per logarithm.  The 16
// pairs (256 B) are read in two wavefronts whatever the lanes' bins.  |r| <=
// 0.0304; the degree-10 series truncates below 1.2e-18.
static __device__ const double kTang16[32] = {
    0.9696735143661499, 0.015397923634601744, 0.9141139388084412, 0.04490002788475267,
    0.8648698925971985, 0.0725880982729422,   0.8205273747444153, 0.09890400275873984,
    0.7804121971130371, 0.1239665205229706,   0.7441437840461731, 0.14776050234720728,
    0.7110554575920105, 0.17050242639725907,  0.6809029579162598, 0.1921677411876897,
    0.6530550122261047, 0.2130469539424608,   0.627486526966095,  0.23301653958853463,
    0.6037552952766418, 0.25229315170463756,  0.5818923115730286, 0.270734940016316,
    0.5614768862724304, 0.28859233495151887,  0.5423704385757446, 0.3059030224960531,
    0.5245840549468994, 0.3225748033494321,   0.5081863403320312, 0.33845354349269224};

__device__ __forceinline__ double half_ln16t(double x, const double2* __restrict__ tab) {
  const int hi = __double2hiint(x);
  const int lo = __double2loint(x);
  const int j = (hi >> 16) & 15;
  const double m = __hiloint2double((hi & 0x000fffff) | 0x3ff00000, lo);
  const double2 t = tab[j];
  const double r = fma(m, t.x, -1.0);
  double q = fma(r, -0.5 / 10.0, 0.5 / 9.0);
  q = fma(r, q, -0.5 / 8.0);
  q = fma(r, q, 0.5 / 7.0);
  q = fma(r, q, -0.5 / 6.0);
  q = fma(r, q, 0.5 / 5.0);
  q = fma(r, q, -0.5 / 4.0);
  q = fma(r, q, 0.5 / 3.0);
  q = fma(r, q, -0.25);
  const double r2 = r * r;
  // exponent as a double without I2F: (2^52 + biased e) - (2^52 + 1023), both exact
  const double de = __hiloint2double(0x43300000, hi >> 20) - 4503599627371519.0;
  const double t_hi = fma(de, HLN2_A, t.y);
  return t_hi + fma(r, 0.5, fma(r2, q, de * HLN2_B));
}

// 64-bin accurate table (tools/tang_table.py 64): |r| <= 0.00780, degree-7
// series (truncation < 9e-19).  1 KB: a warp's lanes mostly share a few bins.
static __device__ const double kTang64[128] = {
    0.9922055006027222, 0.003912517642922336,
    0.977015495300293, 0.011626383491470452,
    0.9624148011207581, 0.01915486752713532,
    0.9481599926948547, 0.026616011150742875,
    0.934187114238739, 0.03403926218695702,
    0.9211106896400452, 0.041087532878612915,
    0.9078326225280762, 0.048347626897856974,
    0.8953129053115845, 0.05529100346752097,
    0.8826634287834167, 0.06240565944840471,
    0.8707258105278015, 0.06921407508230953,
    0.859043538570404, 0.07596783655070966,
    0.8476601839065552, 0.08263772501392648,
    0.8366871476173401, 0.08915252830005801,
    0.8258291482925415, 0.09568368455840767,
    0.8152822256088257, 0.10211046829745976,
    0.8049449324607849, 0.1084907053922218,
    0.795027494430542, 0.11468929036823172,
    0.7853490710258484, 0.12081349178647977,
    0.7757850885391235, 0.1269398724574462,
    0.7664577960968018, 0.1329878213626134,
    0.7572845220565796, 0.13900812069804533,
    0.7484667301177979, 0.1448642624253728,
    0.7398455739021301, 0.1506568992387401,
    0.7313272953033447, 0.15644709152165204,
    0.7230793237686157, 0.16211817404277884,
    0.7149736881256104, 0.16775476839479037,
    0.7072440981864929, 0.17318970678491158,
    0.6995078921318054, 0.1786891012036443,
    0.6918871998786926, 0.18416617130351434,
    0.6843928694725037, 0.18961157783669708,
    0.6773003935813904, 0.19482019582898147,
    0.6700306534767151, 0.2002159080929538,
    0.6634669899940491, 0.20513808888762317,
    0.6560558676719666, 0.21075466476510582,
    0.6496248245239258, 0.2156801378862983,
    0.6431455016136169, 0.22069214739275408,
    0.6368311643600464, 0.2256253533209137,
    0.6305492520332336, 0.2305820053971048,
    0.6244571805000305, 0.23543625891002867,
    0.6183585524559021, 0.2403434038987273,
    0.6124482154846191, 0.2451454431425213,
    0.6067626476287842, 0.24980879485811538,
    0.6010132431983948, 0.2545691547089155,
    0.5953637957572937, 0.25929131941880557,
    0.5899803042411804, 0.2638330626408259,
    0.5843999981880188, 0.26858480110308824,
    0.5790656805038452, 0.2731696850061253,
    0.5739985704421997, 0.2775641865922439,
    0.5688543915748596, 0.2820653899666438,
    0.5640321373939514, 0.28632202395624773,
    0.5589823722839355, 0.29081867035002146,
    0.5541883111000061, 0.29512536912944776,
    0.5494123697280884, 0.2994529952989616,
    0.5447152256965637, 0.30374607126929437,
    0.5400892496109009, 0.3080104380116706,
    0.535578191280365, 0.3122041921453436,
    0.531210720539093, 0.31629824964290554,
    0.5267581343650818, 0.32050689193176246,
    0.5225108861923218, 0.32455473027118603,
    0.518248975276947, 0.32864975247187567,
    0.5139580368995667, 0.33280682856646854,
    0.5098555684089661, 0.33681389628516845,
    0.5059772729873657, 0.34063176287405705,
    0.5020620226860046, 0.3445158078774424};

// series and ln 2 constants as constant-bank operands (no per-use register
// materialisation in the unrolled IK1 loops).  q(r) = (r/2 - ln(1+r)/2) / r^2 to degree 4:
// the Taylor coefficients 1/4, -1/6, 1/8, -1/10, 1/12 with the r^5 term -r^5/14
// Chebyshev-economised onto r^3 and r on |r| <= a = 0.0077945 (the table's largest |r|):
// r^5 ~ (20 a^2 r^3 - 5 a^4 r) / 16.  Truncation error of 0.5 ln(1+r): <= 8.7e-18
// absolute (`python tools/tang_table.py 64 series`), one DFMA less per ln.
static __constant__ double kLn64C[6] = {0.08333333333333333, -0.10000542448484374, 0.125,
                                        -0.16666666658427656, 0.25, 0.34657359027997264};

__device__ __forceinline__ double half_ln64t(double x, const double2* __restrict__ tab) {
  const int hi = __double2hiint(x);
  const int lo = __double2loint(x);
  const double m = __hiloint2double((hi & 0x000fffff) | 0x3ff00000, lo);
  const double2 t = tab[(hi >> 14) & 63];
  const double r = fma(m, t.x, -1.0);
  double q = fma(r, kLn64C[0], kLn64C[1]);
  q = fma(r, q, kLn64C[2]);
  q = fma(r, q, kLn64C[3]);
  q = fma(r, q, kLn64C[4]);
  // 0.5 ln x = de (0.5 ln 2) + (t.y + r (0.5 - r q)), 0.5 ln 2 rounded to a double (its
  // error de * 2.8e-17 scales with the result): 8 FP64 operations; max error 1.7e-16 of
  // max(|0.5 ln x|, 1) (exact-rounding emulation, tools/ln_emulate.py)
  const double de = (double)((hi >> 20) - 1023);  // I2F: the conversion pipe is idle here
  const double u = fma(-r, q, 0.5);
  const double w = fma(r, u, t.y);
  return fma(de, kLn64C[5], w);
}

}  // namespace wq
