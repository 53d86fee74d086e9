// kk_rx.cu -- C ABI (include/kk_rx.h) of the B200-native KK receiver.
//
// Host side: argument validation, constellation / static-EQ / twiddle tables
// (fp64, rounded once to fp32), device scratch, streams and the per-batch
// launch sequence  kk_x2_kernel -> kk_lms_kernel -> kk_apply_kernel.
// With host input the H2D of batch j+1 (copy stream) overlaps the kernels of
// batch j (compute stream), double-buffered device staging.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/kk_rx.h"
// NVTX ranges around every API call (header-only NVTX v3: free when no tool is attached), so
// ncu --nvtx / nsys timelines show the receiver's host-side stages (SURVEY.md 5 "NVTX ranges")
#include <nvtx3/nvToolsExt.h>
#include "kk_internal.h"

namespace {
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace


namespace kk {
int builtin_constellation(int fmt, std::vector<double>& pts, std::vector<int>& labs);
}

using namespace kk;

namespace {
thread_local std::string g_err = "";

kk_status fail(kk_status s, const std::string& msg) {
  g_err = msg;
  return s;
}
}  // namespace

// One in-flight batch of the asynchronous pipeline (kk_rx_submit_batch).
struct AsyncSlot {
  int64_t cap = 0;                          // buffers the scratch below holds
  float2* tails = nullptr;                  // [(cap + 1) * x2h + 64] update-pass x2 tails
  float2* taps = nullptr;                   // [cap][8]
  unsigned long long* d_counts = nullptr;   // [cap][8]
  unsigned long long* h_counts = nullptr;   // pinned [cap][8]
  uint8_t* d_out = nullptr;                 // labels staging (host or NULL output) [cap * n_sym]
  int16_t* d_stage = nullptr;               // host input staging [left + cap*N + right]
  int64_t stage_cap = 0;
  uint8_t* d_pack = nullptr;                // packed-12 input staging [1.5 (left + cap*N + right)]
  int64_t pack_cap = 0;
  uint8_t* h_pin = nullptr;                 // pinned host staging of PAGEABLE host input (bytes)
  size_t pin_bytes = 0;
  int64_t nb = 0, index = 0, n_off0 = 0;
  float dc = 0.f, a_hat = 0.f;              // DC offset hypothesis of the batch (kk_rx_set_dc_offset)
  const int16_t* codes = nullptr;           // device samples of buffer 0 of the batch
  uint8_t* out_dev = nullptr;               // where the chain writes labels
  uint8_t* out_host = nullptr;              // host destination (D2H after the chain) or NULL
  cudaEvent_t ev_done = nullptr, ev_h2d = nullptr, ev_copy = nullptr, ev_zero = nullptr,
              ev_chain = nullptr;
  cudaEvent_t ev_t[4] = {nullptr, nullptr, nullptr, nullptr};  // timing: LMS start/end, chain start/end
  bool timed_lms = false, timed_chain = false;
  int state = 0;                            // 0 free, 1 LMS issued + chain deferred, 2 chain issued
};

struct kk_rx {
  int device = 0;
  int64_t N = 0, n_sym = 0, L = 0;
  int nsub = 0, K = 0, m = 0, bits_per = 0, max_batch = 16;
  int64_t left = 0, right = 0;
  int steps_per_buf = 0, pre_first = 0, pre_steps = 0;
  int64_t x2h = 0;
  float dc = 0, vmin = 1, a_hat = 0, mu = 1e-3f, tau = 0;
  double cspr_lin = 1.0;                   // c = 10^(CSPR/10), for A_hat of a new DC offset
  int prek_h = -1;                         // pre-KK equaliser half length (-1: off)
  float prek[2 * PKH + 1] = {0};
  double prek_sum = 0.0;
  int mode = 0;
  uint32_t tb_mod = 0, s32 = 0;
  int64_t P = 0, ref_offset = 0, stream_index = 0;
  int64_t tone_bin = 0;
  bool has_pattern = false;
  uint32_t dump = 0;
  int grid_chain = 0;
  // constant tables
  float2 *d_tw = nullptr, *d_tw512 = nullptr, *d_H = nullptr, *d_pts = nullptr, *d_winit = nullptr;
  float2* d_lmslut = nullptr;
  float lms_lcx = 0, lms_lcy = 0, lms_linv = 0;
  uint32_t* d_lut = nullptr;
  // work counters of the dynamically scheduled chain launches (ring, zeroed per launch)
  // and the monotone tail-step counter of the async pipeline
  unsigned long long* d_ctr = nullptr;
  int ctr_next = 0;
  static constexpr int CTR_POOL = 4096;  // dynamic-schedule work counters (use_dyn)
  unsigned long long tail_done_target = 0;
  bool dyn_sched = true;
  unsigned long long* d_dbg = nullptr;     // KKRX_PHASE_TIMING diagnostics
  // asynchronous pipeline
#ifndef KK_NSLOT
#define KK_NSLOT 3
#endif
  static constexpr int NSLOT = KK_NSLOT;  // batches in flight: LMS(j) | chain(j-1) queued | chain(j-2) running
  AsyncSlot aslot[NSLOT];
  int a_next = 0, a_deferred = -1;
  int a_order[NSLOT] = {};       // slots with an issued chain, oldest first
  int a_norder = 0;
  std::vector<kk_rx_counts> a_counts;      // harvested per-buffer counters since the last sync
  cudaStream_t h2d_stream = nullptr, unpack_stream = nullptr, aux_stream = nullptr;
  cudaEvent_t ev_in = nullptr;
  int64_t a_launches = 0;
  int64_t a_paged = 0;  // submissions whose pageable host input went through a slot's pinned staging
  DecLut lut{};
  uint8_t *d_lab = nullptr, *d_pattern = nullptr;
  // per-chunk scratch (grown on demand to the largest chunk seen)
  int64_t cap = 0;                       // buffers
  float2* d_tails = nullptr;             // [cap + 1][x2h]  update-pass tails of x2
  float2* d_taps = nullptr;              // [cap * nsub][8]
  unsigned long long* d_counts = nullptr;  // [cap][8]
  unsigned long long* h_counts = nullptr;  // pinned [cap][8]
  uint8_t* d_out = nullptr;              // labels staging for host outputs [cap * n_sym]
  // full x2 (sub_block < buffer or debug), max_batch buffers
  float2* d_x2full = nullptr;            // x2 index -x2h .. max_batch*N/2
  float2* d_es = nullptr;                // debug E_s [max_batch * N]
  // host-input staging (double-buffered, max_batch buffers each)
  int16_t* d_stage[2] = {nullptr, nullptr};
  cudaStream_t stream = nullptr, copy_stream = nullptr;
  bool own_stream = false;
  cudaEvent_t ev_h2d[2] = {nullptr, nullptr}, ev_used[2] = {nullptr, nullptr};
  kk_rx_counts totals{};
  kk_status sticky = KK_OK;
  int64_t last_nb = 0;
  bool last_full = false;                // the last chunk materialised full x2
  int64_t last_launches = 0;
  // per-kernel timing (kk_rx_set_timing): events around each launch slot of a chunk
  bool timing = false;
  cudaEvent_t trace_ref = nullptr;  // KKRX_EVENT_TRACE diagnostics
  // init-time work buffers (train_fir / train_taps / frame_sync), grown on demand, kept
  // until destroy: cudaMalloc/cudaFree per call cost more than the work itself
  void* iw[8] = {};
  size_t iw_cap[8] = {};
  cudaEvent_t ev_t[4] = {nullptr, nullptr, nullptr, nullptr};
  double kernel_ms[3] = {0, 0, 0};
  int64_t kernel_n[3] = {0, 0, 0};
};

#define CK(call)                                                                        \
  do {                                                                                  \
    cudaError_t _e = (call);                                                            \
    if (_e != cudaSuccess) {                                                            \
      if (h) h->sticky = KK_ECUDA;                                                      \
      return fail(KK_ECUDA, std::string(#call) + ": " + cudaGetErrorString(_e));        \
    }                                                                                   \
  } while (0)

static void halo_geometry(int64_t N, int K, int64_t* left, int64_t* right, int* spb, int* i0, int64_t* x2h) {
  const int64_t X2H = 2 * (int64_t)K + 64;
  const int steps = (int)((N + 125) / STEP) + 1;
  int64_t num = N - 2 * X2H - 2944;
  int first = (num >= 0) ? (int)(num / STEP) + 1 : 0;
  if (first > steps) first = steps;
  // GPU grid needs: warm-up window of the first pre-pass step, last step window
  const int64_t gpu_left = N - ((int64_t)STEP * first - 1280);
  const int64_t gpu_right = (int64_t)STEP * steps + 256 - N;
  // method needs (oracle window): 512*ceil((4K+4+101)/512) + 256 and 768
  const int64_t need = 4 * (int64_t)K + 4 + 101;
  const int64_t m_left = 512 * ((need + 511) / 512) + 256;
  // + PKH: the kernel stages PKH extra codes per side (pre-KK equaliser reach)
  *left = std::max(gpu_left, m_left) + PKH;
  *right = std::max<int64_t>(gpu_right, 768) + PKH;
  if (spb) *spb = steps;
  if (i0) *i0 = first;
  if (x2h) *x2h = X2H;
}

// Exact decision look-up table: a G x G grid over the
// constellation's bounding box (+2 d_min).  For each cell R (enlarged by 1e-3 of a
// cell to absorb fp32 index rounding) the candidate list holds every point k with
//   min_{y in R} |y - p_k|^2  <=  min_j max_{y in R} |y - p_j|^2  (+ slack)
// i.e. every point that can be nearest anywhere in R, in ascending index order, so
// argmin over the list == brute-force argmin with the lowest-index tie rule.
// Packed per cell: count in bits 60..63 (15 = brute force), 7-bit indices.
static bool build_lut_g(const std::vector<double>& pts, int m, int G, DecLut& L, std::vector<uint32_t>& cells,
                        int* n_brute) {
  double xmin = 1e300, xmax = -1e300, ymin = 1e300, ymax = -1e300, dmin = 1e300;
  for (int k = 0; k < m; ++k) {
    xmin = std::min(xmin, pts[2 * k]);
    xmax = std::max(xmax, pts[2 * k]);
    ymin = std::min(ymin, pts[2 * k + 1]);
    ymax = std::max(ymax, pts[2 * k + 1]);
    for (int j = 0; j < k; ++j)
      dmin = std::min(dmin, std::hypot(pts[2 * k] - pts[2 * j], pts[2 * k + 1] - pts[2 * j + 1]));
  }
  const double pad = 2.0 * dmin;
  const double span = std::max(xmax - xmin, ymax - ymin) + 2 * pad;
  const float inv = (float)(G / span);
  // origin snapped so that -x0*inv is a half-integer: the kernel's y*inv + (-x0*inv - 1/2 + 2^23)
  // then rounds (single fp32 rounding) to 2^23 + floor((y - x0)*inv)
  const double hx = std::floor(-(xmin - pad) * (double)inv) + 0.5, hy = std::floor(-(ymin - pad) * (double)inv) + 0.5;
  const float x0 = (float)(-hx / (double)inv), y0 = (float)(-hy / (double)inv);
  const double cs = 1.0 / (double)inv;
  cells.assign((size_t)G * G, 0);
  int nb = 0;
  std::vector<double> mind(m);
  for (int cy = 0; cy < G; ++cy)
    for (int cx = 0; cx < G; ++cx) {
      if (cx == 0 || cy == 0 || cx == G - 1 || cy == G - 1) {
        // outer ring: the kernel clamps y into the grid, so these cells also receive every
        // y outside it -> brute force (not counted as crowded)
        cells[(size_t)cy * G + cx] = 1u << 31;
        continue;
      }
      const double e = 1e-3 * cs;
      const double xl = x0 + cx * cs - e, xh = x0 + (cx + 1) * cs + e;
      const double yl = y0 + cy * cs - e, yh = y0 + (cy + 1) * cs + e;
      double U = 1e300;
      for (int k = 0; k < m; ++k) {
        const double px = pts[2 * k], py = pts[2 * k + 1];
        const double dx = std::max(0.0, std::max(xl - px, px - xh)), dy = std::max(0.0, std::max(yl - py, py - yh));
        mind[k] = dx * dx + dy * dy;
        const double fx = std::max(std::fabs(px - xl), std::fabs(px - xh)),
                     fy = std::max(std::fabs(py - yl), std::fabs(py - yh));
        U = std::min(U, fx * fx + fy * fy);
      }
      const double slack = 1e-5 * (1.0 + U);
      uint32_t w = 0;
      int c = 0, first = -1;
      for (int k = 0; k < m && c <= 4; ++k)
        if (mind[k] <= U + slack) {
          if (first < 0) first = k;
          if (c < 4) w |= (uint32_t)k << (7 * c);
          ++c;
        }
      if (c > 4 || c == 0) {
        w = 1u << 31;  // brute force
        ++nb;
      } else {
        for (int q = c; q < 4; ++q) w |= (uint32_t)first << (7 * q);  // pad: duplicates never win a strict <
      }
      cells[(size_t)cy * G + cx] = w;
    }
  L.g = G;
  L.x0 = x0;
  L.y0 = y0;
  L.inv = inv;
  L.cxm = (float)(hx - 0.5 + 8388608.0);
  L.cym = (float)(hy - 0.5 + 8388608.0);
  L.lg = (G == 128) ? 7 : 6;
  *n_brute = nb;
  return true;
}

static void build_lut(const std::vector<double>& pts, int m, DecLut& L, std::vector<uint32_t>& cells) {
  L = DecLut{};
  cells.clear();
  if (m <= 8) return;  // brute force is as cheap as a lookup
  // 64 x 64 cells (16 KB, L2/L1 resident): 1-4 candidates per cell for all built-in / GS formats
  int nb = 0;
  build_lut_g(pts, m, 64, L, cells, &nb);
  if (nb * 200 > 64 * 64) build_lut_g(pts, m, 128, L, cells, &nb);
  if (nb * 200 > 128 * 128) {
    L = DecLut{};  // too crowded for 4-candidate cells: brute force everywhere
    cells.clear();
  }
}

// LMS update-pass look-up table (kk_internal.h "LmsArgs"): for each cell R (enlarged
// by 1e-3 of a cell against fp32 index rounding) the list holds every point k with
//   min_{y in R} |y - p_k|^2  <=  U + tau  (+ slack),   U = min_j max_{y in R} |y - p_j|^2,
// a superset of the points that can be nearest, or within tau of the nearest, somewhere
// in R (since D_k(y) - D_1(y) >= min_R D_k - U).  One point => FAST entry (p_k itself);
// 2..4 points => SLOW entry (NaN, ascending indices, 128-padded); more, or the outer
// ring of cells (which also receives every clamped y outside the grid) => brute force.
static void build_lms_lut(const std::vector<double>& pts, int m, double tau, LmsArgs& la, std::vector<float2>& cells,
                          int* n_fast) {
  const int G = LMS_LUT_G;
  double xmin = 1e300, xmax = -1e300, ymin = 1e300, ymax = -1e300, dmin = 1e300;
  for (int k = 0; k < m; ++k) {
    xmin = std::min(xmin, pts[2 * k]);
    xmax = std::max(xmax, pts[2 * k]);
    ymin = std::min(ymin, pts[2 * k + 1]);
    ymax = std::max(ymax, pts[2 * k + 1]);
    for (int j = 0; j < k; ++j)
      dmin = std::min(dmin, std::hypot(pts[2 * k] - pts[2 * j], pts[2 * k + 1] - pts[2 * j + 1]));
  }
  const double pad = 2.0 * dmin;
  const double span = std::max(xmax - xmin, ymax - ymin) + 2 * pad;
  const float linv = (float)(G / span);
  // half-integer origins: the kernel adds 2^23 - 1/2 to lc, which must stay exact in fp32
  const float lcx = (float)(std::floor(-(xmin - pad) * (double)linv) + 0.5);
  const float lcy = (float)(std::floor(-(ymin - pad) * (double)linv) + 0.5);
  la.linv = linv;
  la.lcx = lcx;
  la.lcy = lcy;
  const double cs = 1.0 / (double)linv;
  cells.assign((size_t)G * G, make_float2(0.f, 0.f));
  std::vector<double> mind(m);
  int nf = 0;
  const uint32_t nan_bits = 0x7fc00000u;
  for (int cy = 0; cy < G; ++cy)
    for (int cx = 0; cx < G; ++cx) {
      float2 ent;
      std::memcpy(&ent.x, &nan_bits, 4);
      uint32_t w = LMS_BRUTE;
      if (cx > 0 && cy > 0 && cx < G - 1 && cy < G - 1) {
        const double e = 1e-3 * cs;
        const double xl = (cx - (double)lcx) * cs - e, xh = (cx + 1 - (double)lcx) * cs + e;
        const double yl = (cy - (double)lcy) * cs - e, yh = (cy + 1 - (double)lcy) * cs + e;
        double U = 1e300;
        for (int k = 0; k < m; ++k) {
          const double px = pts[2 * k], py = pts[2 * k + 1];
          const double dx = std::max(0.0, std::max(xl - px, px - xh)), dy = std::max(0.0, std::max(yl - py, py - yh));
          mind[k] = dx * dx + dy * dy;
          const double fx = std::max(std::fabs(px - xl), std::fabs(px - xh)),
                       fy = std::max(std::fabs(py - yl), std::fabs(py - yh));
          U = std::min(U, fx * fx + fy * fy);
        }
        const double lim = U + tau + 1e-5 * (1.0 + U);
        int cnt = 0, first = -1;
        uint32_t lw = 0x80808080u;
        for (int k = 0; k < m; ++k)
          if (mind[k] <= lim) {
            if (cnt < 4) lw = (lw & ~(0xffu << (8 * cnt))) | ((uint32_t)k << (8 * cnt));
            if (first < 0) first = k;
            ++cnt;
          }
        if (cnt == 1) {
          ent = make_float2((float)pts[2 * first], (float)pts[2 * first + 1]);
          ++nf;
          cells[(size_t)cy * G + cx] = ent;
          continue;
        }
        if (cnt >= 2 && cnt <= 4) w = lw;
      }
      std::memcpy(&ent.y, &w, 4);
      cells[(size_t)cy * G + cx] = ent;
    }
  if (n_fast) *n_fast = nf;
}

// S4 with the downconversion moved behind the LTI filter:
//   x2[m] = e^{i theta_{2m}} sum_i h'_i D[2m - i],  h'_i = h_i e^{-2 pi i tb i / N}
// Hs = DFT_1024(h' placed circularly) / 1024, fp64, rounded once (reading R16).
static void eq_spectrum(const float* fir, int64_t tone_bin, int64_t buffer_len, float2* Hs) {
  int64_t tbn = tone_bin % buffer_len;
  if (tbn < 0) tbn += buffer_len;
  std::vector<std::complex<double>> hp(203);
  for (int t = 0; t < 203; ++t) {
    const int64_t i = t - 101;
    int64_t ph = (tbn * i) % buffer_len;
    if (ph < 0) ph += buffer_len;
    const double a = -2.0 * M_PI * (double)ph / (double)buffer_len;
    hp[t] = std::complex<double>(fir[2 * t], fir[2 * t + 1]) * std::complex<double>(std::cos(a), std::sin(a));
  }
  for (int k = 0; k < 1024; ++k) {
    std::complex<double> acc = 0;
    for (int t = 0; t < 203; ++t) {
      const int i = t - 101;
      const double a = -2.0 * M_PI * (double)(((int64_t)k * (i + 1024)) % 1024) / 1024.0;
      acc += hp[t] * std::complex<double>(std::cos(a), std::sin(a));
    }
    acc /= 1024.0;
    Hs[k] = make_float2((float)acc.real(), (float)acc.imag());
  }
}

extern "C" {

int kk_rx_abi_version(void) { return KK_RX_ABI_VERSION; }

void kk_rx_params_default(kk_rx_params* p) {
  if (!p) return;
  std::memset(p, 0, sizeof(*p));
  p->tone_bin = 541065;
  p->fir_len = 203;
  p->mu = 1e-3f;
  p->k_update = 4096;
  p->sub_block = 0;
  p->gate_tau = -1.0f;
  p->update_mode = KK_UPD_DD_SOFT;
  p->v_min = 1.0f;
  p->device = -1;
  p->max_batch = 16;
}

const char* kk_rx_last_error(const kk_rx_t*) { return g_err.c_str(); }

int kk_rx_constellation(int fmt, float* points_out, uint8_t* labels_out) {
  std::vector<double> pts;
  std::vector<int> labs;
  const int m = builtin_constellation(fmt, pts, labs);
  if (m < 0) {
    g_err = "format has no built-in table";
    return -1;
  }
  if (points_out)
    for (int k = 0; k < 2 * m; ++k) points_out[k] = (float)pts[k];
  if (labels_out)
    for (int k = 0; k < m; ++k) labels_out[k] = (uint8_t)labs[k];
  return m;
}

int kk_rx_decision_tables(const float* points, int m, float tau, float* lms_cells, float* lms_geom, uint32_t* dec_cells,
                          float* dec_geom) {
  if (!points || m < 2 || m > 128) {
    g_err = "need 2..128 points";
    return -1;
  }
  std::vector<double> pts(2 * m);
  for (int k = 0; k < 2 * m; ++k) pts[k] = points[k];
  LmsArgs la{};
  std::vector<float2> lc;
  build_lms_lut(pts, m, tau > 0.f ? (double)tau : 0.0, la, lc, nullptr);
  if (lms_cells) std::memcpy(lms_cells, lc.data(), lc.size() * sizeof(float2));
  if (lms_geom) {
    lms_geom[0] = la.lcx;
    lms_geom[1] = la.lcy;
    lms_geom[2] = la.linv;
  }
  DecLut L{};
  std::vector<uint32_t> dc;
  build_lut(pts, m, L, dc);
  if (dec_cells && !dc.empty()) std::memcpy(dec_cells, dc.data(), dc.size() * sizeof(uint32_t));
  if (dec_geom) {
    dec_geom[0] = L.x0;
    dec_geom[1] = L.y0;
    dec_geom[2] = L.inv;
    dec_geom[3] = (float)L.g;
  }
  return LMS_LUT_G;
}

kk_status kk_rx_halo_for(int64_t buffer_len, int32_t k_update, int64_t* left, int64_t* right) {
  if (!left || !right || buffer_len <= 0 || k_update <= 0) return fail(KK_EINVAL, "bad arguments");
  halo_geometry(buffer_len, k_update, left, right, nullptr, nullptr, nullptr);
  return KK_OK;
}

kk_status kk_rx_destroy(kk_rx_t* h) {
  if (!h) return KK_OK;
  int cur = 0;
  cudaGetDevice(&cur);
  cudaSetDevice(h->device);
  if (h->stream) cudaStreamSynchronize(h->stream);
  for (cudaStream_t q : {h->aux_stream, h->unpack_stream, h->h2d_stream})
    if (q) cudaStreamSynchronize(q);
  if (h->d_dbg) {
    unsigned long long t[8] = {0};
    cudaMemcpy(t, h->d_dbg, sizeof(t), cudaMemcpyDeviceToHost);
    const double st = t[4] ? (double)t[4] : 1.0;
    std::fprintf(stderr,
                 "KKRX_PHASE_TIMING steps %llu  cycles/step: staging %.0f  H %.0f  E %.0f  A+tail %.0f  |  "
                 "busy/task: H %.0f  E %.0f\n",
                 t[4], t[0] / st, t[1] / st, t[2] / st, t[3] / st, t[5] / st / 3.0, t[6] / st / 4.0);
    cudaFree(h->d_dbg);
  }
  if (h->copy_stream) cudaStreamSynchronize(h->copy_stream);
  void* ptrs[] = {h->d_tw,     h->d_tw512,  h->d_H,      h->d_pts,    h->d_winit,    h->d_lut,
                  h->d_lab,    h->d_pattern, h->d_lmslut, h->d_ctr, h->d_tails, h->d_taps,   h->d_counts,   h->d_out,
                  h->d_x2full, h->d_es,     h->d_stage[0], h->d_stage[1]};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  for (void* q : h->iw)
    if (q) cudaFree(q);
  if (h->trace_ref) cudaEventDestroy(h->trace_ref);
  if (h->h_counts) cudaFreeHost(h->h_counts);
  if (h->h2d_stream) cudaStreamSynchronize(h->h2d_stream);
  for (AsyncSlot& a : h->aslot) {
    void* ap[] = {a.tails, a.taps, a.d_counts, a.d_out, a.d_stage, a.d_pack};
    for (void* q : ap)
      if (q) cudaFree(q);
    if (a.h_counts) cudaFreeHost(a.h_counts);
    if (a.h_pin) cudaFreeHost(a.h_pin);
    for (cudaEvent_t e : {a.ev_done, a.ev_h2d, a.ev_copy, a.ev_zero, a.ev_chain, a.ev_t[0], a.ev_t[1],
                          a.ev_t[2], a.ev_t[3]})
      if (e) cudaEventDestroy(e);
  }
  if (h->ev_in) cudaEventDestroy(h->ev_in);
  if (h->h2d_stream) cudaStreamDestroy(h->h2d_stream);
  if (h->unpack_stream) cudaStreamDestroy(h->unpack_stream);
  if (h->aux_stream) cudaStreamDestroy(h->aux_stream);
  for (int i = 0; i < 2; ++i) {
    if (h->ev_h2d[i]) cudaEventDestroy(h->ev_h2d[i]);
    if (h->ev_used[i]) cudaEventDestroy(h->ev_used[i]);
  }
  for (int i = 0; i < 4; ++i)
    if (h->ev_t[i]) cudaEventDestroy(h->ev_t[i]);
  if (h->copy_stream) cudaStreamDestroy(h->copy_stream);
  if (h->own_stream && h->stream) cudaStreamDestroy(h->stream);
  delete h;
  cudaSetDevice(cur);
  return KK_OK;
}

kk_status kk_rx_create(kk_rx_t** out, int fmt, int sps, int64_t buffer_len, float cspr_db, const kk_rx_params* p) {
  if (!out || !p) return fail(KK_EINVAL, "out and params are required");
  *out = nullptr;
  if (sps != 4) return fail(KK_EINVAL, "sps must be 4 (PAPER l.47: 4 -> 2 samples per symbol)");
  if (buffer_len <= 0 || buffer_len % 512 != 0 || buffer_len > (1LL << 30))
    return fail(KK_EINVAL, "buffer_len must be a positive multiple of 512 and <= 2^30");
  if (!p->fir || p->fir_len != 203) return fail(KK_EINVAL, "fir with fir_len == 203 is required (PAPER l.53)");
  if (p->k_update <= 0) return fail(KK_EINVAL, "k_update must be > 0");
  if (buffer_len < 4 * (int64_t)p->k_update + 3200)
    return fail(KK_EINVAL, "buffer_len must be >= 4*k_update + 3200");
  const int64_t n_sym = buffer_len / 4;
  const int64_t L = p->sub_block > 0 ? p->sub_block : n_sym;
  if (n_sym % L != 0) return fail(KK_EINVAL, "sub_block must divide buffer_len/4");
  if (p->update_mode < 0 || p->update_mode > 2) return fail(KK_EINVAL, "bad update_mode");
  if (p->update_mode == KK_UPD_PILOT && !p->ref_pattern) return fail(KK_EINVAL, "PILOT mode needs ref_pattern");
  if (!(cspr_db > -100.f && cspr_db < 100.f)) return fail(KK_EINVAL, "bad cspr_db");
  if (!(p->dc_offset > 0.f)) return fail(KK_EINVAL, "dc_offset must be > 0");
  if (!(p->v_min > 0.f)) return fail(KK_EINVAL, "v_min must be > 0");
  if (p->max_batch < 0) return fail(KK_EINVAL, "max_batch must be >= 0");
  if (p->pre_fir && (p->pre_fir_len < 1 || p->pre_fir_len > 2 * PKH + 1 || p->pre_fir_len % 2 == 0))
    return fail(KK_EINVAL, "pre_fir_len must be odd and <= 17");

  // constellation
  std::vector<double> pts;
  std::vector<int> labs;
  int m = 0;
  if (p->points) {
    if (!p->labels || p->m < 4 || p->m > 128 || (p->m & (p->m - 1)))
      return fail(KK_EINVAL, "points need labels and a power-of-two m in [4,128]");
    m = p->m;
    pts.resize(2 * m);
    labs.resize(m);
    for (int k = 0; k < 2 * m; ++k) pts[k] = p->points[k];
    for (int k = 0; k < m; ++k) labs[k] = p->labels[k];
  } else {
    if (fmt == KK_GS8 || fmt == KK_GS128 || fmt == KK_CUSTOM)
      return fail(KK_EINVAL, "GS / custom formats need points and labels (PAPER l.53: uploaded)");
    m = builtin_constellation(fmt, pts, labs);
    if (m < 0) return fail(KK_EINVAL, "unknown format");
  }
  if ((fmt == KK_GS8 && m != 8) || (fmt == KK_GS128 && m != 128)) return fail(KK_EINVAL, "m does not match format");
  {
    std::vector<int> seen(m, 0);
    for (int k = 0; k < m; ++k) {
      if (labs[k] < 0 || labs[k] >= m || seen[labs[k]]) return fail(KK_EINVAL, "labels must be a permutation");
      seen[labs[k]] = 1;
    }
  }
  double dmin2 = 1e300;
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < m; ++j)
      if (i != j) {
        const double dx = pts[2 * i] - pts[2 * j], dy = pts[2 * i + 1] - pts[2 * j + 1];
        dmin2 = std::min(dmin2, dx * dx + dy * dy);
      }
  if (!(dmin2 > 0)) return fail(KK_EINVAL, "duplicate constellation points");
  if (p->ref_pattern) {
    if (p->ref_len <= 0) return fail(KK_EINVAL, "ref_len must be > 0");
    for (int64_t i = 0; i < p->ref_len; ++i)
      if (p->ref_pattern[i] >= m) return fail(KK_EINVAL, "ref_pattern holds indices >= m");
  }

  kk_rx* h = new kk_rx();
  int dev = p->device;
  if (dev < 0) {
    if (cudaGetDevice(&dev) != cudaSuccess) {
      delete h;
      return fail(KK_ECUDA, "no CUDA device");
    }
  }
  h->device = dev;
  int cur = 0;
  cudaGetDevice(&cur);
  if (cudaSetDevice(dev) != cudaSuccess) {
    delete h;
    return fail(KK_ECUDA, "cudaSetDevice failed");
  }
  struct Restore {
    int d;
    ~Restore() { cudaSetDevice(d); }
  } restore{cur};

  h->N = buffer_len;
  h->n_sym = n_sym;
  h->L = L;
  h->nsub = (int)(n_sym / L);
  h->K = p->k_update;
  h->m = m;
  h->bits_per = 0;
  while ((1 << h->bits_per) < m) ++h->bits_per;
  h->max_batch = p->max_batch > 0 ? p->max_batch : 16;
  halo_geometry(buffer_len, h->K, &h->left, &h->right, &h->steps_per_buf, &h->pre_first, &h->x2h);
  h->pre_steps = h->steps_per_buf - h->pre_first;
  h->dc = p->dc_offset;
  h->vmin = p->v_min;
  const double c = std::pow(10.0, (double)cspr_db / 10.0);
  h->a_hat = (float)std::sqrt((double)p->dc_offset * c / (1.0 + c));  // reading R6
  h->cspr_lin = c;
  if (p->pre_fir) {
    h->prek_h = (p->pre_fir_len - 1) / 2;
    for (int k = 0; k < p->pre_fir_len; ++k) {
      h->prek[PKH - h->prek_h + k] = p->pre_fir[k];
      h->prek_sum += (double)p->pre_fir[k];
    }
  }
  h->mu = p->mu;
  h->tau = p->gate_tau < 0 ? (float)(dmin2 / 4.0) : p->gate_tau;
  h->mode = p->update_mode;
  int64_t tb = p->tone_bin % buffer_len;
  if (tb < 0) tb += buffer_len;
  h->tb_mod = (uint32_t)tb;
  h->tone_bin = p->tone_bin;
  h->s32 = (uint32_t)((tb * 32) % buffer_len);
  h->has_pattern = p->ref_pattern != nullptr;
  h->P = h->has_pattern ? p->ref_len : 1;
  h->ref_offset = p->ref_offset;
  h->dump = p->debug_dump;

  // tables in fp64, rounded once (reading R16)
  std::vector<float2> tw(1024), tw512(512), Hs(1024), fpts(m), winit(8);
  for (int r = 0; r < 32; ++r)
    for (int l = 0; l < 32; ++l) {
      const double a = -2.0 * M_PI * (double)(r * l) / 1024.0;
      tw[r * 32 + l] = make_float2((float)std::cos(a), (float)std::sin(a));
    }
  for (int r = 0; r < 16; ++r)
    for (int l = 0; l < 32; ++l) {
      const double a = -2.0 * M_PI * (double)(r * l) / 512.0;
      tw512[r * 32 + l] = make_float2((float)std::cos(a), (float)std::sin(a));
    }
  // S4 with the downconversion moved behind the LTI filter:
  //   x2[m] = e^{i theta_{2m}} sum_i h'_i D[2m - i],  h'_i = h_i e^{-2 pi i tb i / N}
  // Hs = DFT_1024(h' placed circularly) / 1024, fp64, rounded once (reading R16).
  eq_spectrum(p->fir, p->tone_bin, buffer_len, Hs.data());
  for (int k = 0; k < m; ++k) fpts[k] = make_float2((float)pts[2 * k], (float)pts[2 * k + 1]);
  if (p->w_init) {
    for (int k = 0; k < 8; ++k) winit[k] = make_float2(p->w_init[2 * k], p->w_init[2 * k + 1]);
  } else {
    for (int k = 0; k < 8; ++k) winit[k] = make_float2(0.f, 0.f);
    winit[1] = make_float2(1.f, 0.f);
  }
  std::vector<uint8_t> lab8(m);
  for (int k = 0; k < m; ++k) lab8[k] = (uint8_t)labs[k];

  auto cleanup_fail = [&](kk_status s, const std::string& msg) {
    kk_rx_destroy(h);
    return fail(s, msg);
  };
#define CKC(call)                                                                             \
  do {                                                                                        \
    cudaError_t _e = (call);                                                                  \
    if (_e != cudaSuccess)                                                                    \
      return cleanup_fail(_e == cudaErrorMemoryAllocation ? KK_ENOMEM : KK_ECUDA,             \
                          std::string(#call) + ": " + cudaGetErrorString(_e));                \
  } while (0)

  if (p->cuda_stream) {
    h->stream = (cudaStream_t)p->cuda_stream;
  } else {
    CKC(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
    h->own_stream = true;
  }
  CKC(cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking));
  for (int i = 0; i < 2; ++i) {
    CKC(cudaEventCreateWithFlags(&h->ev_h2d[i], cudaEventDisableTiming));
    CKC(cudaEventCreateWithFlags(&h->ev_used[i], cudaEventDisableTiming));
  }
  for (int i = 0; i < 4; ++i) CKC(cudaEventCreate(&h->ev_t[i]));
  const int B = h->max_batch;
  CKC(cudaMalloc(&h->d_tw, 1024 * sizeof(float2)));
  CKC(cudaMalloc(&h->d_tw512, 512 * sizeof(float2)));
  CKC(cudaMalloc(&h->d_H, 1024 * sizeof(float2)));
  CKC(cudaMalloc(&h->d_pts, 128 * sizeof(float2)));
  CKC(cudaMalloc(&h->d_winit, 8 * sizeof(float2)));
  CKC(cudaMalloc(&h->d_lab, 128));
  CKC(cudaMalloc(&h->d_pattern, (size_t)h->P));
  if (h->nsub > 1 || (h->dump & (KK_DUMP_ES | KK_DUMP_X2))) {
    CKC(cudaMalloc(&h->d_x2full, (size_t)(h->x2h + (int64_t)B * h->N / 2 + 64) * sizeof(float2)));
  }
  if (h->dump & KK_DUMP_ES) CKC(cudaMalloc(&h->d_es, (size_t)B * h->N * sizeof(float2)));
  CKC(cudaMemcpy(h->d_tw, tw.data(), 1024 * sizeof(float2), cudaMemcpyHostToDevice));
  CKC(cudaMemcpy(h->d_tw512, tw512.data(), 512 * sizeof(float2), cudaMemcpyHostToDevice));
  CKC(cudaMemcpy(h->d_H, Hs.data(), 1024 * sizeof(float2), cudaMemcpyHostToDevice));
  CKC(cudaMemcpy(h->d_pts, fpts.data(), m * sizeof(float2), cudaMemcpyHostToDevice));
  CKC(cudaMemcpy(h->d_winit, winit.data(), 8 * sizeof(float2), cudaMemcpyHostToDevice));
  CKC(cudaMemcpy(h->d_lab, lab8.data(), m, cudaMemcpyHostToDevice));
  if (h->has_pattern) CKC(cudaMemcpy(h->d_pattern, p->ref_pattern, (size_t)h->P, cudaMemcpyHostToDevice));
  {
    std::vector<uint32_t> cells;
    build_lut(pts, m, h->lut, cells);
    if (h->lut.g > 0) {
      CKC(cudaMalloc(&h->d_lut, cells.size() * sizeof(uint32_t)));
      CKC(cudaMemcpy(h->d_lut, cells.data(), cells.size() * sizeof(uint32_t), cudaMemcpyHostToDevice));
      h->lut.cell = h->d_lut;
    }
  }
  {
    // LMS look-up table: tau of the soft gate, 0 for the hard / PILOT modes
    std::vector<float2> cells;
    LmsArgs tmp{};
    const double tau_lut = (h->mode == KK_UPD_DD_SOFT && h->tau > 0.f) ? (double)h->tau : 0.0;
    int nf = 0;
    build_lms_lut(pts, m, tau_lut, tmp, cells, &nf);
    h->lms_lcx = tmp.lcx;
    h->lms_lcy = tmp.lcy;
    h->lms_linv = tmp.linv;
    CKC(cudaMalloc(&h->d_lmslut, cells.size() * sizeof(float2)));
    CKC(cudaMemcpy(h->d_lmslut, cells.data(), cells.size() * sizeof(float2), cudaMemcpyHostToDevice));
  }
  CKC(chain_setup(dev, &h->grid_chain));
  CKC(lms_setup());
  CKC(cudaMalloc(&h->d_ctr, (8 + kk_rx_t::CTR_POOL) * sizeof(unsigned long long)));
  CKC(cudaMemset(h->d_ctr, 0, (8 + kk_rx_t::CTR_POOL) * sizeof(unsigned long long)));
  if (const char* e = std::getenv("KKRX_STATIC_SCHED")) h->dyn_sched = (e[0] == '0');
  if (const char* e = std::getenv("KKRX_PHASE_TIMING")) {
    if (e[0] == '1') {
      CKC(cudaMalloc(&h->d_dbg, 8 * sizeof(unsigned long long)));
      CKC(cudaMemset(h->d_dbg, 0, 8 * sizeof(unsigned long long)));
    }
  }
  CKC(cudaGetLastError());
#undef CKC
  *out = h;
  g_err.clear();
  return KK_OK;
}

kk_status kk_rx_halo(const kk_rx_t* h, int64_t* left, int64_t* right) {
  if (!h || !left || !right) return fail(KK_EINVAL, "bad arguments");
  *left = h->left;
  *right = h->right;
  return KK_OK;
}

kk_status kk_rx_seek(kk_rx_t* h, int64_t buffer_index) {
  if (!h) return fail(KK_EINVAL, "null handle");
  h->stream_index = buffer_index;
  return KK_OK;
}

static bool is_device_ptr(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

// host memory the driver would have to stage itself (neither registered/pinned nor device):
// kk_rx_submit_batch stages it through the slot's pinned buffer instead (page_copy)
static bool is_pageable_ptr(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return at.type == cudaMemoryTypeUnregistered;
}

// pageable -> pinned copy on several host threads (one thread copies at ~10 GB/s; the DMA from
// pinned memory runs at the PCIe rate, ~55 GB/s on the measured B200 host)
static void page_copy(void* dst, const void* src, size_t bytes) {
  const unsigned hw = std::thread::hardware_concurrency();
  const int nt = (int)std::max<size_t>(1, std::min<size_t>({(size_t)(hw ? hw : 1), (size_t)8, bytes >> 24}));
  if (nt <= 1) {
    std::memcpy(dst, src, bytes);
    return;
  }
  std::vector<std::thread> th;
  const size_t chunk = ((bytes + nt - 1) / nt + 63) & ~(size_t)63;
  size_t done = 0;  // bytes handed to threads; the rest (thread creation failed) copied here
  try {
    for (int k = 0; k < nt; ++k) {
      const size_t o = (size_t)k * chunk;
      if (o >= bytes) break;
      const size_t n = std::min(chunk, bytes - o);
      th.emplace_back([=] { std::memcpy(static_cast<uint8_t*>(dst) + o, static_cast<const uint8_t*>(src) + o, n); });
      done = o + n;
    }
  } catch (...) {
  }
  if (done < bytes) std::memcpy(static_cast<uint8_t*>(dst) + done, static_cast<const uint8_t*>(src) + done, bytes - done);
  for (auto& x : th) x.join();
}

static void fill_chain_common(kk_rx_t* h, ChainArgs& ca, const int16_t* codes_dev) {
  ca.N = h->N;
  ca.prek_h = h->prek_h;
  for (int k = 0; k < 2 * PKH + 1; ++k) ca.prek[k] = h->prek[k];
  ca.dbg = h->d_dbg;
  ca.x2h = h->x2h;
  ca.dc = h->dc;
  ca.vmin = h->vmin;
  ca.a_hat = h->a_hat;
  ca.invN = (float)(1.0 / (double)h->N);
  ca.tb_mod = h->tb_mod;
  ca.s32 = h->s32;
  for (int r = 0; r < 16; ++r) {
    const int64_t ph = ((int64_t)h->tb_mod * 32 * r) % h->N;
    const double t = -0.0 + 2.0 * M_PI * (double)ph / (double)h->N;
    ca.rot[r] = make_float2((float)std::cos(t), (float)std::sin(t));
  }
  ca.tw1024 = h->d_tw;
  ca.tw512 = h->d_tw512;
  ca.Hs = h->d_H;
  ca.aligned16 = ((uintptr_t)codes_dev % 16) == 0 && (h->N % 8) == 0;
  ca.n_sym = h->n_sym;
  ca.m = h->m;
  ca.pts = h->d_pts;
  ca.labels = h->d_lab;
  ca.pattern = h->has_pattern ? h->d_pattern : nullptr;
  ca.P = h->P;
  ca.pat_tma = h->has_pattern && (h->P % 16 == 0);
  ca.lut = h->lut;
}

static int64_t seg_steps(const Seg& g) { return (int64_t)g.n_own * (g.i_end - g.i_begin); }

// every chain launch: d * sum(pre-KK taps) per segment (each segment may carry its own d)
static cudaError_t chain_launch(const kk_rx_t* h, ChainArgs& ca, int grid, cudaStream_t st) {
  for (int k = 0; k < ca.nseg; ++k) ca.seg[k].prek_dsum = (float)((double)ca.seg[k].dc * h->prek_sum);
  return launch_chain(ca, grid, st);
}

// dynamic work distribution for one chain launch: a zeroed counter from the ring
// (slot 0 is the async pipeline's tail counter)
static cudaError_t use_dyn(kk_rx_t* h, ChainArgs& ca, cudaStream_t st) {
  if (!h->dyn_sched) {
    ca.work_ctr = nullptr;
    return cudaSuccess;
  }
  // a fresh counter from a pool zeroed ahead of use: each half is re-zeroed (one memset)
  // when the other half starts, CTR_POOL/2 launches after its own last use -- far beyond
  // the launches in flight -- so no per-launch memset sits between chain launches
  const int slot = h->ctr_next++ % kk_rx_t::CTR_POOL;
  if (slot % (kk_rx_t::CTR_POOL / 2) == 0 && h->ctr_next > kk_rx_t::CTR_POOL / 2) {
    const int other = (slot + kk_rx_t::CTR_POOL / 2) % kk_rx_t::CTR_POOL;
    cudaError_t e = cudaMemsetAsync(h->d_ctr + 8 + other, 0, (kk_rx_t::CTR_POOL / 2) * sizeof(unsigned long long), st);
    if (e != cudaSuccess) return e;
  }
  ca.work_ctr = h->d_ctr + 8 + slot;
  return cudaSuccess;
}

static kk_status grow(kk_rx_t* h, int64_t nb) {
  if (nb <= h->cap) return KK_OK;
  void* olds[] = {h->d_tails, h->d_taps, h->d_counts, h->d_out};
  for (void* p : olds)
    if (p) cudaFree(p);
  if (h->h_counts) cudaFreeHost(h->h_counts);
  h->d_tails = nullptr;
  h->d_taps = nullptr;
  h->d_counts = nullptr;
  h->d_out = nullptr;
  h->h_counts = nullptr;
  h->cap = 0;
  CK(cudaMalloc(&h->d_tails, (size_t)((nb + 1) * h->x2h + 64) * sizeof(float2)));
  CK(cudaMalloc(&h->d_taps, (size_t)nb * h->nsub * 8 * sizeof(float2)));
  CK(cudaMalloc(&h->d_counts, (size_t)nb * 8 * sizeof(unsigned long long)));
  CK(cudaMalloc(&h->d_out, (size_t)nb * h->n_sym));
  CK(cudaMallocHost(&h->h_counts, (size_t)nb * 8 * sizeof(unsigned long long)));
  h->cap = nb;
  return KK_OK;
}

// Launch sequence of one chunk of nb buffers:
//  sub_block == buffer (default):  [1] x2 update-pass tails  [2] LMS  [3] fused S1-S7
//  sub_block <  buffer          :  [1] full x2               [2] LMS  [3] apply/decide/count
//  KK_DUMP_*                     :  + a debug full-x2 pass (E_s / x2 for kk_rx_debug_*)
// `out_dev`: where the labels go (the caller's device buffer, or d_out).
static kk_status run_chunk(kk_rx_t* h, const int16_t* codes_dev, int64_t nb, int64_t stream_index, uint8_t* out_dev,
                           bool full) {
  const int64_t Pp = h->P;
  int64_t n_off0 = h->has_pattern ? ((h->ref_offset + (stream_index % Pp) * (h->n_sym % Pp)) % Pp) : 0;
  if (n_off0 < 0) n_off0 += Pp;
  CK(cudaMemsetAsync(h->d_counts, 0, (size_t)nb * 8 * sizeof(unsigned long long), h->stream));
  const int S = h->steps_per_buf;
  const bool fused = h->nsub == 1;
  float2* x2f0 = h->d_x2full ? h->d_x2full + h->x2h : nullptr;  // x2 index 0 of buffer 0
  auto full_pass = [&](int count_clip, float2* es) -> kk_status {
    ChainArgs ca{};
    fill_chain_common(h, ca, codes_dev);
    ca.nseg = 2;
    ca.seg[0] = Seg{-1, 1, h->pre_first, S, SEG_X2_FULL, 0, 0, 0, x2f0, nullptr, nullptr, nullptr, 0, codes_dev, h->dc, h->a_hat};
    ca.seg[1] = Seg{0, (int32_t)nb, 0, S, SEG_X2_FULL, count_clip, 0, 0, x2f0, nullptr, h->d_counts, nullptr, 0, codes_dev, h->dc, h->a_hat};
    ca.es_dump = es;
    ca.total_steps = seg_steps(ca.seg[0]) + seg_steps(ca.seg[1]);
    CK(chain_launch(h, ca, h->grid_chain, h->stream));
    h->last_launches += 1;
    return KK_OK;
  };
  if (h->timing) CK(cudaEventRecord(h->ev_t[0], h->stream));
  // [1] x2: update-pass tails of owners -1 .. nb-2 (chain b reads tail b), or everything
  if (fused) {
    ChainArgs ca{};
    fill_chain_common(h, ca, codes_dev);
    ca.nseg = 1;
    ca.seg[0] = Seg{-1, (int32_t)nb, h->pre_first, S, SEG_X2_TAIL, 0, 0, 0, h->d_tails, nullptr, nullptr, nullptr, 0, codes_dev, h->dc, h->a_hat};
    ca.total_steps = seg_steps(ca.seg[0]);
    CK(chain_launch(h, ca, h->grid_chain, h->stream));
    h->last_launches += 1;
  } else {
    kk_status st = full_pass(1, h->d_es);
    if (st != KK_OK) return st;
  }
  if (h->timing) CK(cudaEventRecord(h->ev_t[1], h->stream));
  // [2] LMS update pass
  {
    LmsArgs la{};
    if (fused) {
      la.x2_b0 = h->d_tails + h->x2h;
      la.x2_stride = h->x2h;
    } else {
      la.x2_b0 = x2f0;
      la.x2_stride = h->N / 2;
    }
    la.lut = h->d_lmslut;
    la.lcx = h->lms_lcx;
    la.lcy = h->lms_lcy;
    la.linv = h->lms_linv;
    la.n_sym = h->n_sym;
    la.L = h->L;
    la.nsub = h->nsub;
    la.nchains = (int32_t)(nb * h->nsub);
    la.K = h->K;
    la.mu = h->mu;
    la.inv_tau = h->tau > 0.f ? 1.0f / h->tau : 0.f;
    la.mode = h->mode;
    la.m = h->m;
    la.pts = h->d_pts;
    la.pattern = h->has_pattern ? h->d_pattern : nullptr;
    la.P = Pp;
    la.n_off0 = n_off0;
    la.w_init = h->d_winit;
    la.taps = h->d_taps;
    la.counts = h->d_counts;
    CK(launch_lms(la, h->stream));
    h->last_launches += 1;
  }
  if (h->timing) CK(cudaEventRecord(h->ev_t[2], h->stream));
  // [3] fused chain (or apply from materialised x2)
  if (fused) {
    ChainArgs ca{};
    fill_chain_common(h, ca, codes_dev);
    ca.nseg = 1;
    ca.seg[0] = Seg{0, (int32_t)nb, 0, S, SEG_APPLY, 1, 0, 0, nullptr, out_dev, h->d_counts, h->d_taps, n_off0, codes_dev, h->dc, h->a_hat};
    ca.total_steps = seg_steps(ca.seg[0]);
    CK(use_dyn(h, ca, h->stream));
    CK(chain_launch(h, ca, h->grid_chain, h->stream));
  } else {
    ApplyArgs aa{};
    aa.x2 = x2f0;
    aa.n_sym = h->n_sym;
    aa.L = h->L;
    aa.nsub = h->nsub;
    aa.total = nb * h->n_sym;
    aa.m = h->m;
    aa.pts = h->d_pts;
    aa.labels = h->d_lab;
    aa.pattern = h->has_pattern ? h->d_pattern : nullptr;
    aa.P = Pp;
    aa.n_off0 = n_off0;
    aa.taps = h->d_taps;
    aa.out = out_dev;
    aa.counts = h->d_counts;
    aa.lut = h->lut;
    CK(launch_apply(aa, h->stream));
  }
  h->last_launches += 1;
  if (h->timing) CK(cudaEventRecord(h->ev_t[3], h->stream));
  if (fused && full) {
    kk_status st = full_pass(0, h->d_es);
    if (st != KK_OK) return st;
  }
  h->last_full = full || !fused;
  return KK_OK;
}

static kk_status finish_counts(kk_rx_t* h, int64_t nb, kk_rx_counts* out_per_buf) {
  for (int64_t b = 0; b < nb; ++b) {
    const unsigned long long* c = h->h_counts + 8 * b;
    kk_rx_counts r{};
    r.bit_errors = c[C_BITERR];
    r.sym_errors = c[C_SYMERR];
    r.bits = h->has_pattern ? (uint64_t)h->n_sym * h->bits_per : 0;
    r.symbols = (uint64_t)h->n_sym;
    r.clipped_samples = c[C_CLIP];
    r.gated_updates = c[C_GATED];
    r.flags = (uint32_t)c[C_FLAGS];
    if (out_per_buf) out_per_buf[b] = r;
    h->totals.bit_errors += r.bit_errors;
    h->totals.sym_errors += r.sym_errors;
    h->totals.bits += r.bits;
    h->totals.symbols += r.symbols;
    h->totals.clipped_samples += r.clipped_samples;
    h->totals.gated_updates += r.gated_updates;
    h->totals.flags |= r.flags;
  }
  return KK_OK;
}

kk_status kk_rx_process_batch(kk_rx_t* h, const int16_t* first, int64_t nbuf, uint8_t* out_symbols,
                              kk_rx_counts* out_per_buf) {
  NvtxRange nvtx_range("kk_rx_process_batch");
  if (!h) return fail(KK_EINVAL, "null handle");
  if (h->sticky != KK_OK) return fail(KK_ESTATE, "handle is in a failed state (previous CUDA error)");
  if (!first || nbuf <= 0) return fail(KK_EINVAL, "need a buffer pointer and nbuf > 0");
  int cur = 0;
  cudaGetDevice(&cur);
  CK(cudaSetDevice(h->device));
  struct Restore {
    int d;
    ~Restore() { cudaSetDevice(d); }
  } restore{cur};
  h->last_launches = 0;
  const bool in_dev = is_device_ptr(first);
  const bool out_dev = out_symbols ? is_device_ptr(out_symbols) : false;
  const bool full = (h->dump & (KK_DUMP_ES | KK_DUMP_X2)) != 0;
  // chunking: device input on the fused path runs the whole call as one chunk
  // (one LMS latency per call); host input, sub_block < buffer and debug dumps
  // use chunks of max_batch buffers.
  const int64_t B = (in_dev && h->nsub == 1 && !full) ? nbuf : std::min<int64_t>(h->max_batch, nbuf);
  kk_status st = grow(h, B);
  if (st != KK_OK) return st;
  const int64_t span_extra = h->left + h->right;
  if (!in_dev) {
    for (int i = 0; i < 2; ++i)
      if (!h->d_stage[i]) {
        cudaError_t e = cudaMalloc(&h->d_stage[i], (size_t)(span_extra + (int64_t)h->max_batch * h->N) * sizeof(int16_t));
        if (e != cudaSuccess) return fail(KK_ENOMEM, "staging allocation failed");
      }
  }
  auto issue_h2d = [&](int64_t j0, int64_t nb, int slot) -> kk_status {
    const int16_t* src = first + j0 * h->N - h->left;
    const size_t bytes = (size_t)(span_extra + nb * h->N) * sizeof(int16_t);
    CK(cudaStreamWaitEvent(h->copy_stream, h->ev_used[slot], 0));
    CK(cudaMemcpyAsync(h->d_stage[slot], src, bytes, cudaMemcpyHostToDevice, h->copy_stream));
    CK(cudaEventRecord(h->ev_h2d[slot], h->copy_stream));
    return KK_OK;
  };
  int64_t j0 = 0;
  int slot = 0;
  if (!in_dev) {
    st = issue_h2d(0, std::min<int64_t>(B, nbuf), 0);
    if (st != KK_OK) return st;
  }
  while (j0 < nbuf) {
    const int64_t nb = std::min<int64_t>(B, nbuf - j0);
    const int16_t* codes;
    if (in_dev) {
      codes = first + j0 * h->N;
    } else {
      CK(cudaStreamWaitEvent(h->stream, h->ev_h2d[slot], 0));
      codes = h->d_stage[slot] + h->left;
    }
    uint8_t* odev = (out_symbols && out_dev) ? out_symbols + j0 * h->n_sym : h->d_out;
    st = run_chunk(h, codes, nb, h->stream_index + j0, odev, full);
    if (st != KK_OK) return st;
    if (!in_dev) {
      CK(cudaEventRecord(h->ev_used[slot], h->stream));
      const int64_t jn = j0 + nb;
      if (jn < nbuf) {
        st = issue_h2d(jn, std::min<int64_t>(B, nbuf - jn), slot ^ 1);
        if (st != KK_OK) return st;
      }
    }
    if (out_symbols && !out_dev) {
      CK(cudaMemcpyAsync(out_symbols + j0 * h->n_sym, h->d_out, (size_t)nb * h->n_sym, cudaMemcpyDeviceToHost,
                         h->stream));
    }
    CK(cudaMemcpyAsync(h->h_counts, h->d_counts, (size_t)nb * 8 * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                       h->stream));
    CK(cudaStreamSynchronize(h->stream));
    if (h->timing) {
      for (int k = 0; k < 3; ++k) {
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, h->ev_t[k], h->ev_t[k + 1]));
        h->kernel_ms[k] += ms;
        h->kernel_n[k] += 1;
      }
    }
    finish_counts(h, nb, out_per_buf ? out_per_buf + j0 : nullptr);
    h->last_nb = nb;
    j0 += nb;
    slot ^= 1;
  }
  h->stream_index += nbuf;
  return KK_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Asynchronous pipeline: batch j's LMS update pass
// (one SM, lane-per-chain kernel, side stream) runs concurrently with the fused
// chain of batch j-1, whose launch also computes batch j's x2 tails first (the LMS
// kernel waits on their completion counter).  The chain of the newest batch is
// deferred to the next submit or to kk_rx_sync.
// ---------------------------------------------------------------------------
static kk_status slot_reserve(kk_rx_t* h, AsyncSlot& a, int64_t nb, bool host_in, bool packed) {
  if (!a.ev_done) {
    CK(cudaEventCreateWithFlags(&a.ev_done, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&a.ev_h2d, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&a.ev_copy, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&a.ev_zero, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&a.ev_chain, cudaEventDisableTiming));
    for (int k = 0; k < 4; ++k) CK(cudaEventCreate(&a.ev_t[k]));
  }
  if (nb > a.cap) {
    void* ap[] = {a.tails, a.taps, a.d_counts, a.d_out};
    for (void* q : ap)
      if (q) cudaFree(q);
    if (a.h_counts) cudaFreeHost(a.h_counts);
    a.tails = nullptr;
    a.taps = nullptr;
    a.d_counts = nullptr;
    a.d_out = nullptr;
    a.h_counts = nullptr;
    a.cap = 0;
    CK(cudaMalloc(&a.tails, (size_t)((nb + 1) * h->x2h + 64) * sizeof(float2)));
    CK(cudaMalloc(&a.taps, (size_t)nb * 8 * sizeof(float2)));
    CK(cudaMalloc(&a.d_counts, (size_t)nb * 8 * sizeof(unsigned long long)));
    CK(cudaMalloc(&a.d_out, (size_t)nb * h->n_sym));
    CK(cudaMallocHost(&a.h_counts, (size_t)nb * 8 * sizeof(unsigned long long)));
    a.cap = nb;
  }
  if ((host_in || packed) && nb > a.stage_cap) {
    if (a.d_stage) cudaFree(a.d_stage);
    a.d_stage = nullptr;
    a.stage_cap = 0;
    CK(cudaMalloc(&a.d_stage, (size_t)(h->left + nb * h->N + h->right) * sizeof(int16_t)));
    a.stage_cap = nb;
  }
  if (packed && nb > a.pack_cap) {
    if (a.d_pack) cudaFree(a.d_pack);
    a.d_pack = nullptr;
    a.pack_cap = 0;
    CK(cudaMalloc(&a.d_pack, (size_t)(h->left + nb * h->N + h->right) * 3 / 2 + 16));
    a.pack_cap = nb;
  }
  return KK_OK;
}

static void slot_harvest(kk_rx_t* h, AsyncSlot& a) {
  // per-kernel device times of this batch (kk_rx_set_timing): [1] LMS pass, [2] chain launch
  float ms = 0.f;
  if (a.timed_lms && cudaEventElapsedTime(&ms, a.ev_t[0], a.ev_t[1]) == cudaSuccess) {
    h->kernel_ms[1] += ms;
    h->kernel_n[1] += 1;
  }
  if (a.timed_chain && cudaEventElapsedTime(&ms, a.ev_t[2], a.ev_t[3]) == cudaSuccess) {
    h->kernel_ms[2] += ms;
    h->kernel_n[2] += 1;
  }
  if (a.timed_chain && h->trace_ref) {
    // KKRX_EVENT_TRACE=1: start/end of every chain launch relative to the first one
    float t0 = 0.f, t1 = 0.f;
    cudaEventElapsedTime(&t0, h->trace_ref, a.ev_t[2]);
    cudaEventElapsedTime(&t1, h->trace_ref, a.ev_t[3]);
    std::fprintf(stderr, "KKRX_EVENT_TRACE chain %9.4f -> %9.4f ms (%.4f)\n", t0, t1, t1 - t0);
  }
  a.timed_lms = a.timed_chain = false;
  for (int64_t b = 0; b < a.nb; ++b) {
    const unsigned long long* c = a.h_counts + 8 * b;
    kk_rx_counts r{};
    r.bit_errors = c[C_BITERR];
    r.sym_errors = c[C_SYMERR];
    r.bits = h->has_pattern ? (uint64_t)h->n_sym * h->bits_per : 0;
    r.symbols = (uint64_t)h->n_sym;
    r.clipped_samples = c[C_CLIP];
    r.gated_updates = c[C_GATED];
    r.flags = (uint32_t)c[C_FLAGS];
    h->a_counts.push_back(r);
    h->totals.bit_errors += r.bit_errors;
    h->totals.sym_errors += r.sym_errors;
    h->totals.bits += r.bits;
    h->totals.symbols += r.symbols;
    h->totals.clipped_samples += r.clipped_samples;
    h->totals.gated_updates += r.gated_updates;
    h->totals.flags |= r.flags;
  }
  a.state = 0;
}

// the fused chain of slot p (APPLY), optionally preceded in the same launch by the
// x2 tails of slot t's batch (a leading SEG_X2_TAIL segment, published via the counter)
constexpr int LMS_WARP_MAX_CHAINS = 60;  // measured crossover (streaming small batches)

static kk_status issue_chain(kk_rx_t* h, int p, int t, const LmsArgs* la) {
  AsyncSlot& ap = h->aslot[p];
  ChainArgs ca{};
  fill_chain_common(h, ca, ap.codes);
  const int S = h->steps_per_buf;
  int ns = 0;
  int grid = h->grid_chain;
  if (t >= 0) {
    AsyncSlot& at = h->aslot[t];
    ca.seg[ns++] = Seg{-1, (int32_t)at.nb, h->pre_first, S, SEG_X2_TAIL, 0, 0, 0, at.tails, nullptr, nullptr,
                       nullptr, 0, at.codes, at.dc, at.a_hat};
    ca.tail_ctr = h->d_ctr;
    ca.aligned16 = ca.aligned16 && ((uintptr_t)at.codes % 16) == 0;
    if (la) {  // batch t's update pass rides along as the last CTAs of this launch
      ca.lms = *la;
      ca.lms_mode = (la->mode == 1) ? 1 : (la->mode == 2 || !(la->inv_tau > 0.f)) ? 2 : 0;
      // few chains: the chain work of the launch is short, so the one-SM lane-per-chain pass
      // (~1.2 ms for 4096 steps) would set the launch time; one warp-per-chain CTA per chain
      // (~0.3 ms, x2 window in shared memory) instead, each joining the chain work afterwards
      ca.lms_warp = (la->nchains <= LMS_WARP_MAX_CHAINS) ? 1 : 0;
      ca.lms_ctas = ca.lms_warp ? la->nchains : lms_lanes_ctas(la->nchains);
    }
  }
  ca.seg[ns++] = Seg{0, (int32_t)ap.nb, 0, S, SEG_APPLY, 1, 0, 0, nullptr, ap.out_dev, ap.d_counts, ap.taps, ap.n_off0,
                     ap.codes, ap.dc, ap.a_hat};
  ca.nseg = ns;
  ca.total_steps = 0;
  for (int k = 0; k < ns; ++k) ca.total_steps += seg_steps(ca.seg[k]);
  {
    const bool d = h->dyn_sched;
    h->dyn_sched = true;  // the tail segment must be grabbed first
    cudaError_t e = use_dyn(h, ca, h->stream);
    h->dyn_sched = d;
    CK(e);
  }
  if (h->timing) CK(cudaEventRecord(ap.ev_t[2], h->stream));
  if (h->timing && !h->trace_ref && std::getenv("KKRX_EVENT_TRACE")) {
    CK(cudaEventCreate(&h->trace_ref));
    CK(cudaEventRecord(h->trace_ref, h->stream));
  }
  CK(chain_launch(h, ca, grid, h->stream));
  if (h->timing) CK(cudaEventRecord(ap.ev_t[3], h->stream));
  ap.timed_chain = h->timing;
  h->a_launches += 1;
  // results back to the host on the auxiliary stream, behind the chain
  CK(cudaEventRecord(ap.ev_chain, h->stream));
  CK(cudaStreamWaitEvent(h->aux_stream, ap.ev_chain, 0));
  if (ap.out_host)
    CK(cudaMemcpyAsync(ap.out_host, ap.out_dev, (size_t)ap.nb * h->n_sym, cudaMemcpyDeviceToHost, h->aux_stream));
  CK(cudaMemcpyAsync(ap.h_counts, ap.d_counts, (size_t)ap.nb * 8 * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                     h->aux_stream));
  CK(cudaEventRecord(ap.ev_done, h->aux_stream));
  ap.state = 2;
  h->a_order[h->a_norder++] = p;
  return KK_OK;
}

// input formats of the submit path
enum { IN_INT16 = 0, IN_PACKED12 = 1 };

static kk_status submit_impl(kk_rx_t* h, const void* first_v, int64_t nbuf, uint8_t* out_symbols, int fmt) {
  NvtxRange nvtx_range("kk_rx_submit_batch");
  const int16_t* first = static_cast<const int16_t*>(first_v);
  const uint8_t* first_b = static_cast<const uint8_t*>(first_v);
  if (!h) return fail(KK_EINVAL, "null handle");
  if (h->sticky != KK_OK) return fail(KK_ESTATE, "handle is in a failed state (previous CUDA error)");
  if (!first || nbuf <= 0) return fail(KK_EINVAL, "need a buffer pointer and nbuf > 0");
  if (h->nsub != 1) return fail(KK_EUNSUPPORTED, "kk_rx_submit_batch needs sub_block == buffer_len/4");
  if (h->dump) return fail(KK_EUNSUPPORTED, "kk_rx_submit_batch does not support debug dumps");
  if (nbuf > 4096) return fail(KK_EINVAL, "nbuf > 4096 per submission");
  int cur = 0;
  cudaGetDevice(&cur);
  CK(cudaSetDevice(h->device));
  struct Restore {
    int d;
    ~Restore() { cudaSetDevice(d); }
  } restore{cur};
  if (!h->h2d_stream) {
    CK(cudaStreamCreateWithFlags(&h->h2d_stream, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&h->unpack_stream, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&h->aux_stream, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&h->ev_in, cudaEventDisableTiming));
  }
  const bool in_dev = is_device_ptr(first_v);
  const bool out_dev = out_symbols ? is_device_ptr(out_symbols) : false;
  const bool packed = fmt == IN_PACKED12;
  if (packed && ((h->left | h->right | h->N) & 7)) return fail(KK_EUNSUPPORTED, "packed-12 input needs halos and N in multiples of 8");
  const int s = h->a_next;
  AsyncSlot& a = h->aslot[s];
  if (a.state == 2) {  // the chain of NSLOT submissions ago (normally finished): wait and harvest
    CK(cudaEventSynchronize(a.ev_done));
    if (h->a_norder > 0 && h->a_order[0] == s) {
      slot_harvest(h, a);
      for (int k = 1; k < h->a_norder; ++k) h->a_order[k - 1] = h->a_order[k];
      h->a_norder -= 1;
    }
  }
  if (a.state != 0) return fail(KK_ESTATE, "async slot busy");
  // grow every slot at once: the pipeline cycles through all NSLOT of them, and device
  // allocations (cudaMalloc synchronises) must not land in a later, steady-state submit
  kk_status st = KK_OK;
  for (int k = 0; k < kk_rx_t::NSLOT; ++k) {
    if (h->aslot[k].state != 0 && k != s) continue;  // in flight: grows when it is next reused
    st = slot_reserve(h, h->aslot[k], nbuf, !in_dev, packed);
    if (st != KK_OK) return st;
  }
  a.nb = nbuf;
  a.index = h->stream_index;
  a.dc = h->dc;
  a.a_hat = h->a_hat;
  const int64_t Pp = h->P;
  int64_t n_off0 = h->has_pattern ? ((h->ref_offset + (h->stream_index % Pp) * (h->n_sym % Pp)) % Pp) : 0;
  if (n_off0 < 0) n_off0 += Pp;
  a.n_off0 = n_off0;
  a.out_dev = (out_symbols && out_dev) ? out_symbols : a.d_out;
  a.out_host = (out_symbols && !out_dev) ? out_symbols : nullptr;
  if (packed) {
    // packed 12-bit samples (host or device) -> packed staging on the copy stream, unpacked
    // there to int16 codes (1.5 instead of 2 bytes per sample cross PCIe)
    const int64_t span = h->left + nbuf * h->N + h->right;
    if (in_dev) CK(cudaEventRecord(h->ev_in, h->stream));  // device input: the caller's stream order
    if (in_dev) CK(cudaStreamWaitEvent(h->h2d_stream, h->ev_in, 0));
    CK(cudaMemcpyAsync(a.d_pack, first_b - h->left * 3 / 2, (size_t)(span * 3 / 2), cudaMemcpyDefault, h->h2d_stream));
    // the unpack runs on its own stream so the next batch's copy follows this one back to
    // back (the copy engine, not the SMs, is the bound); slot reuse is ordered by ev_done
    CK(cudaEventRecord(a.ev_copy, h->h2d_stream));
    CK(cudaStreamWaitEvent(h->unpack_stream, a.ev_copy, 0));
    CK(launch_unpack12(a.d_pack, a.d_stage, span, h->unpack_stream));
    h->a_launches += 1;
    CK(cudaEventRecord(a.ev_h2d, h->unpack_stream));
    CK(cudaStreamWaitEvent(h->stream, a.ev_h2d, 0));
    a.codes = a.d_stage + h->left;
  } else if (in_dev) {
    a.codes = first;
  } else {
    // host input: pinned -> slot staging on the copy stream.  No wait on the compute stream:
    // the data is in host memory, and the slot's previous batch has finished (host wait
    // above), so copies run back to back while earlier batches compute.  The chain launch
    // that first reads the batch (its tails) waits for this copy.  PAGEABLE host memory is
    // first copied by host threads into the slot's pinned buffer (the slot's previous copy
    // finished with its chain, waited for above), so the DMA itself is a pinned transfer.
    const size_t bytes = (size_t)(h->left + nbuf * h->N + h->right) * sizeof(int16_t);
    const void* src = first - h->left;
    if (is_pageable_ptr(src)) {
      if (a.pin_bytes < bytes) {
        if (a.h_pin) cudaFreeHost(a.h_pin);
        a.h_pin = nullptr;
        a.pin_bytes = 0;
        CK(cudaMallocHost(&a.h_pin, bytes));
        a.pin_bytes = bytes;
      }
      page_copy(a.h_pin, src, bytes);
      src = a.h_pin;
      h->a_paged += 1;
    }
    CK(cudaMemcpyAsync(a.d_stage, src, bytes, cudaMemcpyHostToDevice, h->h2d_stream));
    CK(cudaEventRecord(a.ev_h2d, h->h2d_stream));
    CK(cudaStreamWaitEvent(h->stream, a.ev_h2d, 0));
    a.codes = a.d_stage + h->left;
  }
  // counters zeroed off the compute stream (only chain launches sit on it in steady state)
  CK(cudaMemsetAsync(a.d_counts, 0, (size_t)nbuf * 8 * sizeof(unsigned long long), h->aux_stream));
  CK(cudaEventRecord(a.ev_zero, h->aux_stream));
  CK(cudaStreamWaitEvent(h->stream, a.ev_zero, 0));
  LmsArgs la{};
  la.lut = h->d_lmslut;
  la.lcx = h->lms_lcx;
  la.lcy = h->lms_lcy;
  la.linv = h->lms_linv;
  la.x2_b0 = a.tails + h->x2h;
  la.x2_stride = h->x2h;
  la.n_sym = h->n_sym;
  la.L = h->L;
  la.nsub = 1;
  la.nchains = (int32_t)nbuf;
  la.K = h->K;
  la.mu = h->mu;
  la.inv_tau = h->tau > 0.f ? 1.0f / h->tau : 0.f;
  la.mode = h->mode;
  la.m = h->m;
  la.pts = h->d_pts;
  la.pattern = h->has_pattern ? h->d_pattern : nullptr;
  la.P = Pp;
  la.n_off0 = n_off0;
  la.w_init = h->d_winit;
  la.taps = a.taps;
  la.counts = a.d_counts;
  const int p = h->a_deferred;
  if (p < 0) {
    // pipeline empty: the tails of this batch by their own launch, then the update pass
    ChainArgs ca{};
    fill_chain_common(h, ca, a.codes);
    ca.nseg = 1;
    ca.seg[0] = Seg{-1, (int32_t)nbuf, h->pre_first, h->steps_per_buf, SEG_X2_TAIL, 0, 0, 0, a.tails,
                    nullptr, nullptr, nullptr, 0, a.codes, a.dc, a.a_hat};
    ca.total_steps = seg_steps(ca.seg[0]);
    CK(chain_launch(h, ca, h->grid_chain, h->stream));
    // nothing else runs yet: the one-warp-per-chain kernel (lowest latency, many SMs)
    if (h->timing) CK(cudaEventRecord(a.ev_t[0], h->stream));
    CK(launch_lms(la, h->stream));
    if (h->timing) CK(cudaEventRecord(a.ev_t[1], h->stream));
    a.timed_lms = h->timing;
    h->a_launches += 2;
    a.state = 1;
  } else {
    // this batch's tails are the first work items of the chain launch of batch p, and its
    // update pass runs as that launch's last CTAs (waiting on the tail counter)
    h->tail_done_target += (unsigned long long)nbuf * (unsigned long long)h->pre_steps;
    la.wait_ctr = h->d_ctr;
    la.wait_target = h->tail_done_target;
    a.state = 1;
    st = issue_chain(h, p, s, &la);
    if (st != KK_OK) return st;
  }
  h->a_deferred = s;
  h->a_next = (s + 1) % kk_rx::NSLOT;
  h->stream_index += nbuf;
  return KK_OK;
}

extern "C" kk_status kk_rx_submit_batch(kk_rx_t* h, const int16_t* first, int64_t nbuf, uint8_t* out_symbols) {
  return submit_impl(h, first, nbuf, out_symbols, IN_INT16);
}

extern "C" kk_status kk_rx_submit_batch_packed12(kk_rx_t* h, const uint8_t* first, int64_t nbuf,
                                                 uint8_t* out_symbols) {
  return submit_impl(h, first, nbuf, out_symbols, IN_PACKED12);
}

extern "C" kk_status kk_rx_sync(kk_rx_t* h, kk_rx_counts* out_per_buf, int64_t max_out, int64_t* n_out) {
  NvtxRange nvtx_range("kk_rx_sync");
  if (!h) return fail(KK_EINVAL, "null handle");
  if (h->sticky != KK_OK) return fail(KK_ESTATE, "handle is in a failed state (previous CUDA error)");
  int cur = 0;
  cudaGetDevice(&cur);
  CK(cudaSetDevice(h->device));
  struct Restore {
    int d;
    ~Restore() { cudaSetDevice(d); }
  } restore{cur};
  if (h->a_deferred >= 0) {
    kk_status st = issue_chain(h, h->a_deferred, -1, nullptr);
    if (st != KK_OK) return st;
    h->a_deferred = -1;
  }
  CK(cudaStreamSynchronize(h->stream));
  if (h->aux_stream) CK(cudaStreamSynchronize(h->aux_stream));
  for (int k = 0; k < h->a_norder; ++k) slot_harvest(h, h->aslot[h->a_order[k]]);
  h->a_norder = 0;
  const int64_t n = (int64_t)h->a_counts.size();
  if (out_per_buf)
    for (int64_t i = 0; i < n && i < max_out; ++i) out_per_buf[i] = h->a_counts[i];
  if (n_out) *n_out = n;
  h->a_counts.clear();
  return KK_OK;
}


extern "C" kk_status kk_rx_set_dc_offset(kk_rx_t* h, float dc_offset) {
  if (!h) return fail(KK_EINVAL, "null handle");
  if (!(dc_offset > 0.f)) return fail(KK_EINVAL, "dc_offset must be > 0");
  h->dc = dc_offset;
  h->a_hat = (float)std::sqrt((double)dc_offset * h->cspr_lin / (1.0 + h->cspr_lin));  // reading R6
  return KK_OK;
}

// "all measurements are performed multiple times using different DC offset
// values" and the best Q is kept.  Each hypothesis is a full S1-S7 pass over the same
// buffers; the hypotheses run back to back through the streaming pipeline.
extern "C" kk_status kk_rx_set_cspr(kk_rx_t* h, float cspr_db) {
  if (!h) return fail(KK_EINVAL, "null handle");
  if (!(cspr_db > -60.f && cspr_db < 60.f)) return fail(KK_EINVAL, "cspr_db out of range");
  h->cspr_lin = std::pow(10.0, (double)cspr_db / 10.0);
  h->a_hat = (float)std::sqrt((double)h->dc * h->cspr_lin / (1.0 + h->cspr_lin));  // reading R6
  return KK_OK;
}

static bool pipeline_idle(const kk_rx_t* h) {
  if (h->a_deferred >= 0) return false;
  for (const AsyncSlot& a : h->aslot)
    if (a.state != 0) return false;
  return true;
}

// "batched DC-offset (and CSPR-hypothesis) sweep".  Hypothesis k
// runs S1-S7 over the same buffers with DC offset dc_values[k] and, if cspr_db_values is
// given, CSPR cspr_db_values[k] (A_hat = sqrt(d c / (1 + c)), reading R6); the hypotheses go
// back to back through the streaming pipeline (each slot carries its own d and A_hat).
extern "C" kk_status kk_rx_sweep(kk_rx_t* h, const int16_t* first, int64_t nbuf, const float* dc_values,
                                 const float* cspr_db_values, int nd, kk_rx_counts* out_per_hyp, int* best) {
  NvtxRange nvtx_range("kk_rx_sweep");
  if (!h || !first || !dc_values || nd <= 0 || nbuf <= 0) return fail(KK_EINVAL, "bad arguments");
  for (int k = 0; k < nd; ++k) {
    if (!(dc_values[k] > 0.f)) return fail(KK_EINVAL, "dc_values must be > 0");
    if (cspr_db_values && !(cspr_db_values[k] > -60.f && cspr_db_values[k] < 60.f))
      return fail(KK_EINVAL, "cspr_db_values out of range");
  }
  // the caller's submitted-but-unsynced batches would be drained and their counters lost:
  // like train_fir / frame_sync, the sweep needs an idle streaming pipeline
  if (!pipeline_idle(h)) return fail(KK_ESTATE, "kk_rx_sync the streaming pipeline first");
  const float dc0 = h->dc;
  const double c0 = h->cspr_lin;
  const int64_t idx0 = h->stream_index;
  const kk_rx_counts totals0 = h->totals;  // hypothesis passes are not traffic: totals restored below
  kk_status st = KK_OK;
  for (int k = 0; k < nd; ++k) {
    if (cspr_db_values) h->cspr_lin = std::pow(10.0, (double)cspr_db_values[k] / 10.0);
    kk_rx_set_dc_offset(h, dc_values[k]);
    h->stream_index = idx0;
    st = kk_rx_submit_batch(h, first, nbuf, nullptr);
    if (st != KK_OK) break;
  }
  std::vector<kk_rx_counts> per((size_t)nd * nbuf);
  int64_t n = 0;
  if (st == KK_OK) st = kk_rx_sync(h, per.data(), (int64_t)per.size(), &n);
  h->cspr_lin = c0;
  kk_rx_set_dc_offset(h, dc0);
  h->stream_index = idx0 + nbuf;
  h->totals = totals0;
  if (st != KK_OK) return st;
  if (n != (int64_t)nd * nbuf) return fail(KK_ECUDA, "sweep: unexpected result count");
  int kb = 0;
  double ber_b = 2.0;
  for (int k = 0; k < nd; ++k) {
    kk_rx_counts t{};
    for (int64_t b = 0; b < nbuf; ++b) {
      const kk_rx_counts& c = per[(size_t)k * nbuf + b];
      t.bit_errors += c.bit_errors;
      t.sym_errors += c.sym_errors;
      t.bits += c.bits;
      t.symbols += c.symbols;
      t.clipped_samples += c.clipped_samples;
      t.gated_updates += c.gated_updates;
      t.flags |= c.flags;
    }
    if (out_per_hyp) out_per_hyp[k] = t;
    const double ber = t.bits ? (double)t.bit_errors / (double)t.bits : 0.0;
    if (ber < ber_b) {
      ber_b = ber;
      kb = k;
    }
  }
  if (best) *best = kb;
  return KK_OK;
}

extern "C" kk_status kk_rx_dc_sweep(kk_rx_t* h, const int16_t* first, int64_t nbuf, const float* dc_values, int nd,
                                    kk_rx_counts* out_per_dc, int* best) {
  return kk_rx_sweep(h, first, nbuf, dc_values, nullptr, nd, out_per_dc, best);
}


// ---------------------------------------------------------------------------
// Init-time training (NEXT row of SURVEY 8(f))
// ---------------------------------------------------------------------------

// device copy (if needed) of one buffer + halos; returns the device pointer of its sample 0
static kk_status stage_one(kk_rx_t* h, const int16_t* buffer, int16_t** tmp, const int16_t** dev0) {
  *tmp = nullptr;
  if (is_device_ptr(buffer)) {
    *dev0 = buffer;
    return KK_OK;
  }
  const size_t n = (size_t)(h->left + h->N + h->right);
  CK(cudaMalloc(tmp, n * sizeof(int16_t)));
  CK(cudaMemcpyAsync(*tmp, buffer - h->left, n * sizeof(int16_t), cudaMemcpyHostToDevice, h->stream));
  *dev0 = *tmp + h->left;
  return KK_OK;
}

// S1-S4 of one buffer with the debug outputs: x2 (index 0 <-> position 0, x2h samples of
// margin before) and optionally E_s at positions [0, N)
static kk_status one_buffer_stages(kk_rx_t* h, const int16_t* codes, float2* x2_full, float2* es) {
  ChainArgs ca{};
  fill_chain_common(h, ca, codes);
  // the previous buffer's tail (x2 indices [-x2h, 0), from the left halo) and the buffer
  ca.nseg = 2;
  ca.seg[0] = Seg{-1, 1, h->pre_first, h->steps_per_buf, SEG_X2_FULL, 0, 0, 0, x2_full + h->x2h, nullptr, nullptr,
                  nullptr, 0, codes, h->dc, h->a_hat};
  ca.seg[1] = Seg{0, 1, 0, h->steps_per_buf, SEG_X2_FULL, 0, 0, 0, x2_full + h->x2h, nullptr, nullptr, nullptr, 0,
                  codes, h->dc, h->a_hat};
  ca.es_dump = es;
  ca.total_steps = seg_steps(ca.seg[0]) + seg_steps(ca.seg[1]);
  CK(chain_launch(h, ca, h->grid_chain, h->stream));
  return KK_OK;
}

enum { IW_X2 = 0, IW_ES, IW_R, IW_B, IW_SYM, IW_OUT, IW_CVAL, IW_SMALL };
// a cached init-time work buffer of at least `bytes` (nullptr if the allocation fails)
static void* iw_get(kk_rx_t* h, int slot, size_t bytes) {
  if (h->iw_cap[slot] < bytes) {
    if (h->iw[slot]) cudaFree(h->iw[slot]);
    h->iw[slot] = nullptr;
    h->iw_cap[slot] = 0;
    if (cudaMalloc(&h->iw[slot], bytes) != cudaSuccess) return nullptr;
    h->iw_cap[slot] = bytes;
  }
  return h->iw[slot];
}

extern "C" kk_status kk_rx_train_fir(kk_rx_t* h, const int16_t* buffer, const float* symbols, int64_t n_first,
                                     int64_t n_count, double ridge, float* out_fir) {
  NvtxRange nvtx_range("kk_rx_train_fir");
  if (!h || !buffer || !symbols || !out_fir || n_count <= 0) return fail(KK_EINVAL, "bad arguments");
  if (4 * n_first - 101 < 0 || 4 * (n_first + n_count - 1) + 101 >= h->N)
    return fail(KK_EINVAL, "training symbols must satisfy 4*n_first >= 101 and 4*(n_first+n_count-1)+101 < buffer_len");
  if (!pipeline_idle(h)) return fail(KK_ESTATE, "kk_rx_sync the streaming pipeline first");
  CK(cudaSetDevice(h->device));
  int16_t* tmp = nullptr;
  const int16_t* dev0 = nullptr;
  kk_status st = stage_one(h, buffer, &tmp, &dev0);
  if (st != KK_OK) return st;
  auto release = [&]() {
    if (tmp) cudaFree(tmp);
  };
  cudaError_t e = cudaSuccess;
  const int ntap = 203;
  auto* x2 = static_cast<float2*>(iw_get(h, IW_X2, (size_t)(h->x2h + h->N / 2 + 64) * sizeof(float2)));
  auto* es = static_cast<float2*>(iw_get(h, IW_ES, (size_t)h->N * sizeof(float2)));
  auto* sym = static_cast<float2*>(iw_get(h, IW_SYM, (size_t)n_count * sizeof(float2)));
  // GRAM_SPLIT partial planes of R and b (kk_gram_kernel), summed by the solver
  auto* R = static_cast<double2*>(iw_get(h, IW_R, (size_t)GRAM_SPLIT * ntap * ntap * sizeof(double2)));
  auto* b = static_cast<double2*>(iw_get(h, IW_B, (size_t)GRAM_SPLIT * ntap * sizeof(double2)));
  auto* out = static_cast<float*>(iw_get(h, IW_OUT, 2 * ntap * sizeof(float)));
  if (!x2 || !es || !sym || !R || !b || !out) e = cudaErrorMemoryAllocation;
  if (e == cudaSuccess) e = cudaMemcpyAsync(sym, symbols, (size_t)n_count * sizeof(float2), cudaMemcpyHostToDevice, h->stream);
  if (e != cudaSuccess) {
    release();
    return fail(KK_ENOMEM, std::string("kk_rx_train_fir: ") + cudaGetErrorString(e));
  }
  st = one_buffer_stages(h, dev0, x2, es);
  if (st == KK_OK) {
    e = launch_train_fir(es, 4 * n_first, sym, (int)n_count, ntap, ridge, R, b, out, h->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(out_fir, out, 2 * ntap * sizeof(float), cudaMemcpyDeviceToHost, h->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    if (e != cudaSuccess) {
      h->sticky = KK_ECUDA;
      st = fail(KK_ECUDA, std::string("kk_rx_train_fir: ") + cudaGetErrorString(e));
    }
  }
  release();
  return st;
}

// SURVEY 8(f) NEXT row 2, first step of the init-time training: frame synchronisation
// against the known PCG64 pattern (oracle.train.frame_sync).  E_s of one buffer by the
// chain kernel, then kk_fsync_kernel over every cyclic lag of the pattern.
extern "C" kk_status kk_rx_frame_sync(kk_rx_t* h, const int16_t* buffer, int64_t n0, int32_t n_corr, int64_t* n_off,
                                      float* peak, double* peak_to_mean) {
  NvtxRange nvtx_range("kk_rx_frame_sync");
  if (!h || !buffer || !n_off) return fail(KK_EINVAL, "bad arguments");
  if (!h->has_pattern) return fail(KK_EINVAL, "frame synchronisation needs ref_pattern");
  if (n_corr < 16 || n_corr > 8192 || n0 < 0 || 4 * (n0 + (int64_t)n_corr - 1) >= h->N)
    return fail(KK_EINVAL, "need 16 <= n_corr <= 8192, n0 >= 0 and 4*(n0+n_corr-1) < buffer_len");
  if (!pipeline_idle(h)) return fail(KK_ESTATE, "kk_rx_sync the streaming pipeline first");
  CK(cudaSetDevice(h->device));
  int16_t* tmp = nullptr;
  const int16_t* dev0 = nullptr;
  kk_status st = stage_one(h, buffer, &tmp, &dev0);
  if (st != KK_OK) return st;
  auto release = [&]() {
    if (tmp) cudaFree(tmp);
  };
  cudaError_t e = cudaSuccess;
  auto* x2 = static_cast<float2*>(iw_get(h, IW_X2, (size_t)(h->x2h + h->N / 2 + 64) * sizeof(float2)));
  auto* es = static_cast<float2*>(iw_get(h, IW_ES, (size_t)h->N * sizeof(float2)));
  float2* cval = peak ? static_cast<float2*>(iw_get(h, IW_CVAL, (size_t)h->P * sizeof(float2))) : nullptr;
  auto* small = static_cast<unsigned char*>(iw_get(h, IW_SMALL, 256));
  auto* best = reinterpret_cast<unsigned long long*>(small);
  auto* sum2 = reinterpret_cast<double*>(small + 16);
  if (!x2 || !es || (peak && !cval) || !small) e = cudaErrorMemoryAllocation;
  if (e == cudaSuccess) e = cudaMemsetAsync(best, 0, sizeof(unsigned long long), h->stream);
  if (e == cudaSuccess) e = cudaMemsetAsync(sum2, 0, sizeof(double), h->stream);
  if (e != cudaSuccess) {
    release();
    return fail(KK_ENOMEM, std::string("kk_rx_frame_sync: ") + cudaGetErrorString(e));
  }
  st = one_buffer_stages(h, dev0, x2, es);
  if (st == KK_OK) {
    unsigned long long hb = 0;
    double hs = 0.0;
    float2 hc = make_float2(0.f, 0.f);
    e = launch_frame_sync(es, 4 * n0, n_corr, h->d_pattern, h->P, n0, h->d_pts, h->m, best, sum2, cval, h->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&hb, best, sizeof(hb), cudaMemcpyDeviceToHost, h->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&hs, sum2, sizeof(hs), cudaMemcpyDeviceToHost, h->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    const int64_t k = (int64_t)(uint32_t)~(uint32_t)(hb & 0xffffffffull);
    if (e == cudaSuccess && peak) e = cudaMemcpy(&hc, cval + k, sizeof(hc), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) {
      h->sticky = KK_ECUDA;
      st = fail(KK_ECUDA, std::string("kk_rx_frame_sync: ") + cudaGetErrorString(e));
    } else {
      *n_off = k;
      if (peak) {
        peak[0] = hc.x;
        peak[1] = hc.y;
      }
      const double mag = (double)__builtin_bit_cast(float, (uint32_t)(hb >> 32));
      if (peak_to_mean) *peak_to_mean = (hs > 0.0) ? mag / (hs / (double)h->P) : 0.0;
    }
  }
  release();
  return st;
}

extern "C" kk_status kk_rx_set_fir(kk_rx_t* h, const float* fir) {
  if (!h || !fir) return fail(KK_EINVAL, "bad arguments");
  if (!pipeline_idle(h)) return fail(KK_ESTATE, "kk_rx_sync the streaming pipeline first");
  CK(cudaSetDevice(h->device));
  std::vector<float2> Hs(1024);
  eq_spectrum(fir, h->tone_bin, h->N, Hs.data());
  CK(cudaStreamSynchronize(h->stream));
  CK(cudaMemcpy(h->d_H, Hs.data(), 1024 * sizeof(float2), cudaMemcpyHostToDevice));
  return KK_OK;
}

extern "C" kk_status kk_rx_set_w_init(kk_rx_t* h, const float* w) {
  if (!h || !w) return fail(KK_EINVAL, "bad arguments");
  if (!pipeline_idle(h)) return fail(KK_ESTATE, "kk_rx_sync the streaming pipeline first");
  CK(cudaSetDevice(h->device));
  CK(cudaStreamSynchronize(h->stream));
  CK(cudaMemcpy(h->d_winit, w, 8 * sizeof(float2), cudaMemcpyHostToDevice));
  return KK_OK;
}

// PAPER l.53 ("after initial setup and convergence using a training sequence"): the WL
// taps after k_steps LMS steps in PILOT mode (known pattern) from the handle's W_init over
// symbols [0, k_steps) of one buffer (stream position of the handle, as for process).
extern "C" kk_status kk_rx_train_taps(kk_rx_t* h, const int16_t* buffer, int32_t k_steps, float* out_w) {
  NvtxRange nvtx_range("kk_rx_train_taps");
  if (!h || !buffer || !out_w || k_steps <= 0) return fail(KK_EINVAL, "bad arguments");
  if (!h->has_pattern) return fail(KK_EINVAL, "PILOT training needs ref_pattern");
  if (4 * (int64_t)k_steps + 16 > h->N) return fail(KK_EINVAL, "k_steps must fit in the buffer");
  if (!pipeline_idle(h)) return fail(KK_ESTATE, "kk_rx_sync the streaming pipeline first");
  CK(cudaSetDevice(h->device));
  int16_t* tmp = nullptr;
  const int16_t* dev0 = nullptr;
  kk_status st = stage_one(h, buffer, &tmp, &dev0);
  if (st != KK_OK) return st;
  cudaError_t e = cudaSuccess;
  auto* x2 = static_cast<float2*>(iw_get(h, IW_X2, (size_t)(h->x2h + h->N / 2 + 64) * sizeof(float2)));
  auto* small = static_cast<unsigned char*>(iw_get(h, IW_SMALL, 256));
  auto* taps = reinterpret_cast<float2*>(small);                      // 8 float2
  auto* cnt = reinterpret_cast<unsigned long long*>(small + 128);     // 8 counters
  if (!x2 || !small) e = cudaErrorMemoryAllocation;
  if (e == cudaSuccess) e = cudaMemsetAsync(cnt, 0, 8 * sizeof(unsigned long long), h->stream);
  if (e == cudaSuccess) {
    st = one_buffer_stages(h, dev0, x2, nullptr);
    if (st == KK_OK) {
      const int64_t Pp = h->P;
      int64_t idx0 = (h->ref_offset + (h->stream_index % Pp) * (h->n_sym % Pp)) % Pp;
      if (idx0 < 0) idx0 += Pp;
      LmsArgs la{};
      la.lut = h->d_lmslut;
      la.lcx = h->lms_lcx;
      la.lcy = h->lms_lcy;
      la.linv = h->lms_linv;
      // one chain whose K update steps are symbols [0, K): the base is shifted by K symbols
      la.x2_b0 = x2 + h->x2h + 2 * (int64_t)k_steps;
      la.x2_stride = 0;
      la.n_sym = h->n_sym;
      la.L = h->n_sym;
      la.nsub = 1;
      la.nchains = 1;
      la.K = k_steps;
      la.mu = h->mu;
      la.inv_tau = 0.f;
      la.mode = KK_UPD_PILOT;
      la.m = h->m;
      la.pts = h->d_pts;
      la.pattern = h->d_pattern;
      la.P = Pp;
      la.n_off0 = (idx0 + k_steps) % Pp;
      la.w_init = h->d_winit;
      la.taps = taps;
      la.counts = cnt;
      e = launch_lms(la, h->stream);
      if (e == cudaSuccess) e = cudaMemcpyAsync(out_w, taps, 8 * sizeof(float2), cudaMemcpyDeviceToHost, h->stream);
      if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    }
  }
  if (e != cudaSuccess && st == KK_OK) {
    h->sticky = KK_ECUDA;
    st = fail(KK_ECUDA, std::string("kk_rx_train_taps: ") + cudaGetErrorString(e));
  }
  void* ptrs[] = {tmp};
  for (void* q : ptrs)
    if (q) cudaFree(q);
  return st;
}


// ---------------------------------------------------------------------------
// GMI evaluation (NEXT row 4 of SURVEY 8(f)); host-side Gauss-Hermite nodes
// ---------------------------------------------------------------------------
// Gauss-Hermite nodes/weights (weight e^{-t^2}) by Golub-Welsch: eigen-decomposition of
// the symmetric tridiagonal Jacobi matrix (diag 0, off-diag sqrt(k/2)) with implicit QL;
// w_k = sqrt(pi) * v_{0k}^2.
extern "C" int kk_hermgauss(int order, double* nodes, double* weights) {
  if (order < 1 || order > 64 || !nodes || !weights) {
    g_err = "order must be 1..64";
    return -1;
  }
  const int n = order;
  std::vector<double> d(n, 0.0), e(n, 0.0), z((size_t)n * n, 0.0);
  for (int k = 1; k < n; ++k) e[k - 1] = std::sqrt(k / 2.0);
  for (int k = 0; k < n; ++k) z[(size_t)k * n + k] = 1.0;
  for (int l = 0; l < n; ++l) {
    int iter = 0, mm;
    do {
      for (mm = l; mm < n - 1; ++mm) {
        const double dd = std::fabs(d[mm]) + std::fabs(d[mm + 1]);
        if (std::fabs(e[mm]) <= 1e-16 * dd) break;
      }
      if (mm != l) {
        if (iter++ == 60) break;
        double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
        double r = std::hypot(g, 1.0);
        g = d[mm] - d[l] + e[l] / (g + (g >= 0 ? std::fabs(r) : -std::fabs(r)));
        double s = 1.0, c = 1.0, p = 0.0;
        int i;
        for (i = mm - 1; i >= l; --i) {
          double f = s * e[i], b = c * e[i];
          r = std::hypot(f, g);
          e[i + 1] = r;
          if (r == 0.0) {
            d[i + 1] -= p;
            e[mm] = 0.0;
            break;
          }
          s = f / r;
          c = g / r;
          g = d[i + 1] - p;
          r = (d[i] - g) * s + 2.0 * c * b;
          p = s * r;
          d[i + 1] = g + p;
          g = c * r - b;
          for (int k = 0; k < n; ++k) {
            f = z[(size_t)k * n + i + 1];
            z[(size_t)k * n + i + 1] = s * z[(size_t)k * n + i] + c * f;
            z[(size_t)k * n + i] = c * z[(size_t)k * n + i] - s * f;
          }
        }
        if (r == 0.0 && i >= l) continue;
        d[l] -= p;
        e[l] = g;
        e[mm] = 0.0;
      }
    } while (mm != l);
  }
  std::vector<int> ord(n);
  for (int k = 0; k < n; ++k) ord[k] = k;
  std::sort(ord.begin(), ord.end(), [&](int a, int b) { return d[a] < d[b]; });
  for (int k = 0; k < n; ++k) {
    nodes[k] = d[ord[k]];
    const double v = z[ord[k]];  // first component of eigenvector ord[k]
    weights[k] = std::sqrt(M_PI) * v * v;
  }
  return n;
}

extern "C" kk_status kk_gmi_awgn(const float* points, const uint8_t* labels, int m, int n_cand, double snr_db, int order,
                                 double* out_gmi) {
  NvtxRange nvtx_range("kk_gmi_awgn");
  if (!points || !labels || !out_gmi || m < 2 || m > 256 || (m & (m - 1)) || n_cand < 1 || order < 1 || order > 64)
    return fail(KK_EINVAL, "kk_gmi_awgn: bad arguments (m a power of two <= 256, order 1..64)");
  int nb = 0;
  while ((1 << nb) < m) ++nb;
  if (nb > 8) return fail(KK_EINVAL, "kk_gmi_awgn: m > 256");
  std::vector<double> t(order), w(order);
  kk_hermgauss(order, t.data(), w.data());
  std::vector<double2> nodes((size_t)order * order);
  std::vector<double> wts((size_t)order * order);
  for (int a = 0; a < order; ++a)
    for (int b = 0; b < order; ++b) {
      nodes[(size_t)a * order + b] = make_double2(t[a], t[b]);
      wts[(size_t)a * order + b] = w[a] * w[b] / M_PI;
    }
  const double n0 = std::pow(10.0, -snr_db / 10.0);
  const int nq = order * order;
  float2* d_p = nullptr;
  uint8_t* d_l = nullptr;
  double2* d_n = nullptr;
  double *d_w = nullptr, *d_o = nullptr;
  [[maybe_unused]] kk_rx_t* h = nullptr;  // for CK() (no handle here)
  auto release = [&]() {
    void* ptrs[] = {d_p, d_l, d_n, d_w, d_o};
    for (void* q : ptrs)
      if (q) cudaFree(q);
  };
  cudaError_t e = cudaMalloc(&d_p, (size_t)n_cand * m * sizeof(float2));
  if (e == cudaSuccess) e = cudaMalloc(&d_l, (size_t)n_cand * m);
  if (e == cudaSuccess) e = cudaMalloc(&d_n, (size_t)nq * sizeof(double2));
  if (e == cudaSuccess) e = cudaMalloc(&d_w, (size_t)nq * sizeof(double));
  if (e == cudaSuccess) e = cudaMalloc(&d_o, (size_t)n_cand * sizeof(double));
  if (e == cudaSuccess) e = cudaMemcpy(d_p, points, (size_t)n_cand * m * sizeof(float2), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(d_l, labels, (size_t)n_cand * m, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(d_n, nodes.data(), (size_t)nq * sizeof(double2), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(d_w, wts.data(), (size_t)nq * sizeof(double), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = launch_gmi(d_p, d_l, m, nb, d_n, d_w, nq, n0, n_cand, d_o, 0);
  if (e == cudaSuccess) e = cudaMemcpy(out_gmi, d_o, (size_t)n_cand * sizeof(double), cudaMemcpyDeviceToHost);
  release();
  (void)h;
  if (e != cudaSuccess) return fail(KK_ECUDA, std::string("kk_gmi_awgn: ") + cudaGetErrorString(e));
  return KK_OK;
}

extern "C" int64_t kk_rx_async_launches(kk_rx_t* h) {
  if (!h) return 0;
  const int64_t n = h->a_launches;
  h->a_launches = 0;
  return n;
}

extern "C" kk_status kk_rx_pageable_staged(const kk_rx_t* h, int64_t* n) {
  if (!h || !n) return fail(KK_EINVAL, "bad arguments");
  *n = h->a_paged;
  return KK_OK;
}

extern "C" {
kk_status kk_rx_process(kk_rx_t* h, const int16_t* buffer, uint8_t* out_symbols, kk_rx_counts* out_errors) {
  return kk_rx_process_batch(h, buffer, 1, out_symbols, out_errors);
}

kk_status kk_rx_get_taps(kk_rx_t* h, int64_t buf, float* out) {
  if (!h || !out) return fail(KK_EINVAL, "bad arguments");
  if (buf < 0 || buf >= h->last_nb) return fail(KK_EINVAL, "buffer index outside the last batch");
  CK(cudaSetDevice(h->device));
  CK(cudaMemcpy(out, h->d_taps + buf * h->nsub * 8, (size_t)h->nsub * 8 * sizeof(float2), cudaMemcpyDeviceToHost));
  return KK_OK;
}

kk_status kk_rx_totals(const kk_rx_t* h, kk_rx_counts* out) {
  if (!h || !out) return fail(KK_EINVAL, "bad arguments");
  *out = h->totals;
  return KK_OK;
}

kk_status kk_rx_reset_totals(kk_rx_t* h) {
  if (!h) return fail(KK_EINVAL, "null handle");
  h->totals = kk_rx_counts{};
  return KK_OK;
}

kk_status kk_rx_debug_x2(kk_rx_t* h, int64_t first, int64_t count, float* out) {
  if (!h || !out || count < 0) return fail(KK_EINVAL, "bad arguments");
  if (first < -(2 * (int64_t)h->K + 2) || first + count > h->last_nb * h->N / 2)
    return fail(KK_EINVAL, "x2 range outside the last batch");
  CK(cudaSetDevice(h->device));
  if (h->last_full && h->d_x2full) {
    CK(cudaMemcpy(out, h->d_x2full + h->x2h + first, (size_t)count * sizeof(float2), cudaMemcpyDeviceToHost));
    return KK_OK;
  }
  // only the update-pass tails are materialised: [b*N/2 - x2h, b*N/2) for b in [0, nb)
  std::vector<float2> tmp((size_t)count, make_float2(NAN, NAN));
  for (int64_t b = 0; b < h->last_nb; ++b) {
    const int64_t lo = b * h->N / 2 - h->x2h, hi = b * h->N / 2;
    const int64_t a0 = std::max(lo, first), a1 = std::min(hi, first + count);
    if (a1 > a0)
      CK(cudaMemcpy(tmp.data() + (a0 - first), h->d_tails + b * h->x2h + (a0 - lo), (size_t)(a1 - a0) * sizeof(float2),
                    cudaMemcpyDeviceToHost));
  }
  std::memcpy(out, tmp.data(), (size_t)count * sizeof(float2));
  return KK_OK;
}

kk_status kk_rx_debug_es(kk_rx_t* h, int64_t first, int64_t count, float* out) {
  if (!h || !out || count < 0) return fail(KK_EINVAL, "bad arguments");
  if (!h->d_es) return fail(KK_ESTATE, "create with debug_dump & KK_DUMP_ES");
  if (first < 0 || first + count > h->last_nb * h->N) return fail(KK_EINVAL, "range outside the last batch");
  CK(cudaSetDevice(h->device));
  CK(cudaMemcpy(out, h->d_es + first, (size_t)count * sizeof(float2), cudaMemcpyDeviceToHost));
  return KK_OK;
}

int64_t kk_rx_last_launches(const kk_rx_t* h) { return h ? h->last_launches : 0; }

kk_status kk_rx_set_timing(kk_rx_t* h, int on) {
  if (!h) return fail(KK_EINVAL, "null handle");
  h->timing = on != 0;
  for (int k = 0; k < 3; ++k) {
    h->kernel_ms[k] = 0;
    h->kernel_n[k] = 0;
  }
  return KK_OK;
}

kk_status kk_rx_kernel_times(const kk_rx_t* h, double* ms_out, int64_t* n_out) {
  if (!h || !ms_out || !n_out) return fail(KK_EINVAL, "bad arguments");
  for (int k = 0; k < 3; ++k) {
    ms_out[k] = h->kernel_ms[k];
    n_out[k] = h->kernel_n[k];
  }
  return KK_OK;
}

}  // extern "C"
