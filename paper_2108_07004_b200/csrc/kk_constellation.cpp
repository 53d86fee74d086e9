// kk_constellation.cpp -- built-in conventional constellations (host side).
//
// MP 4/8/16/32/64/128-QAM.  The paper prints no coordinates or
// labels; the convention (reading R12) is:
//   square M-QAM : L = sqrt(M) levels per axis, index k = iI*L + iQ,
//                  point (2iI-(L-1)) + i(2iQ-(L-1)), label gray(iI)<<log2(L) | gray(iQ)
//   8-QAM        : 4x2 rectangle, same indexing/labels with (4, 2) levels
//   32 / 128     : cross, from the 8x4 / 16x8 rectangle: points with
//                  |x| > 1.5*Lq - 1 move to x' = sgn(x)(Lq - |y|), y' = sgn(y)(|x| - Li/4)
// normalised to unit mean power.  GS-8 / GS-128 are uploaded by
// the caller.
#include <cmath>
#include <cstdint>
#include <vector>

namespace kk {

static int gray(int i) { return i ^ (i >> 1); }

static void rect(int li, int lq, std::vector<double>& re, std::vector<double>& im, std::vector<int>& lab) {
  int bq = 0;
  while ((1 << bq) < lq) ++bq;
  for (int a = 0; a < li; ++a)
    for (int b = 0; b < lq; ++b) {
      re.push_back(2.0 * a - (li - 1));
      im.push_back(2.0 * b - (lq - 1));
      lab.push_back((gray(a) << bq) | gray(b));
    }
}

static void cross(int li, int lq, std::vector<double>& re, std::vector<double>& im, std::vector<int>& lab) {
  rect(li, lq, re, im, lab);
  const double core = 1.5 * lq - 1.0;
  const double shift = li / 4;
  for (size_t k = 0; k < re.size(); ++k) {
    const double x = re[k], y = im[k];
    if (std::fabs(x) > core) {
      const double sx = x > 0 ? 1.0 : -1.0, sy = y > 0 ? 1.0 : -1.0;
      re[k] = sx * (lq - std::fabs(y));
      im[k] = sy * (std::fabs(x) - shift);
    }
  }
}

// Returns M (>0) and fills pts (2M doubles) / labs, or -1 for formats without a built-in table.
int builtin_constellation(int fmt, std::vector<double>& pts, std::vector<int>& labs) {
  std::vector<double> re, im;
  labs.clear();
  switch (fmt) {
    case 0: rect(2, 2, re, im, labs); break;    // QAM4
    case 1: rect(4, 2, re, im, labs); break;    // QAM8
    case 2: rect(4, 4, re, im, labs); break;    // QAM16
    case 3: cross(8, 4, re, im, labs); break;   // QAM32
    case 4: rect(8, 8, re, im, labs); break;    // QAM64
    case 5: cross(16, 8, re, im, labs); break;  // QAM128
    default: return -1;
  }
  double p = 0;
  for (size_t k = 0; k < re.size(); ++k) p += re[k] * re[k] + im[k] * im[k];
  const double s = 1.0 / std::sqrt(p / re.size());
  pts.resize(2 * re.size());
  for (size_t k = 0; k < re.size(); ++k) {
    pts[2 * k] = re[k] * s;
    pts[2 * k + 1] = im[k] * s;
  }
  return (int)re.size();
}

}  // namespace kk
