/* oracle.c — TEST INFRASTRUCTURE ONLY. Plain-C restatement of the CoNet-Rx inference path of the
 * reference (arxiv/paper_2510_12739, proj/core). Each function cites the reference lines it follows.
 * The float loops keep the reference's accumulation order so that, compiled without FP contraction,
 * the restatement is bit-identical to the reference on x86-64 (pinned by tests/test_oracle_pin.py). */
#include "oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static char g_err[512];
const char* orc_last_error(void) { return g_err; }

/* conv2d: kernels.hpp:47-91. Zero "same" padding by skipping out-of-range taps (:71-75); weights
 * [kh,kw,Cin,Cout] (:32); bias first, then accumulate in (dt, df, ci, co) order (:66-83).
 * Extension: dilation (dil_t, dil_f) scales the tap offsets (BASELINE config 3); dil = 1 is the
 * reference loop unchanged. */
void orc_conv2d(const float* x, int64_t B, int64_t T, int64_t F, int64_t Cin, const float* w, int kh, int kw,
                int64_t Cout, const float* bias, int dil_t, int dil_f, float* y) {
  const int64_t oh = kh / 2, ow = kw / 2;
  for (int64_t b = 0; b < B; ++b) {
    const float* xb = x + b * T * F * Cin;
    float* yb = y + b * T * F * Cout;
    for (int64_t to = 0; to < T; ++to)
      for (int64_t fo = 0; fo < F; ++fo) {
        float* yrow = yb + (to * F + fo) * Cout;
        for (int64_t co = 0; co < Cout; ++co) yrow[co] = bias ? bias[co] : 0.0f;
        for (int64_t dt = 0; dt < kh; ++dt) {
          const int64_t ti = to + (dt - oh) * dil_t;
          if (ti < 0 || ti >= T) continue;
          for (int64_t df = 0; df < kw; ++df) {
            const int64_t fi = fo + (df - ow) * dil_f;
            if (fi < 0 || fi >= F) continue;
            const float* xrow = xb + (ti * F + fi) * Cin;
            const float* wbase = w + (dt * kw + df) * Cin * Cout;
            for (int64_t ci = 0; ci < Cin; ++ci) {
              const float xv = xrow[ci];
              const float* wrow = wbase + ci * Cout;
              for (int64_t co = 0; co < Cout; ++co) yrow[co] += xv * wrow[co];
            }
          }
        }
      }
  }
}

/* depthwise_conv2d: kernels.hpp:196-233. */
void orc_dwconv2d(const float* x, int64_t B, int64_t T, int64_t F, int64_t C, const float* w, int kh, int kw,
                  const float* bias, float* y) {
  const int64_t oh = kh / 2, ow = kw / 2;
  for (int64_t b = 0; b < B; ++b) {
    const float* xb = x + b * T * F * C;
    float* yb = y + b * T * F * C;
    for (int64_t to = 0; to < T; ++to)
      for (int64_t fo = 0; fo < F; ++fo) {
        float* yrow = yb + (to * F + fo) * C;
        for (int64_t ci = 0; ci < C; ++ci) yrow[ci] = bias ? bias[ci] : 0.0f;
        for (int64_t dt = 0; dt < kh; ++dt) {
          const int64_t ti = to + dt - oh;
          if (ti < 0 || ti >= T) continue;
          for (int64_t df = 0; df < kw; ++df) {
            const int64_t fi = fo + df - ow;
            if (fi < 0 || fi >= F) continue;
            const float* xrow = xb + (ti * F + fi) * C;
            const float* wrow = w + (dt * kw + df) * C;
            for (int64_t ci = 0; ci < C; ++ci) yrow[ci] += xrow[ci] * wrow[ci];
          }
        }
      }
  }
}

/* relu: kernels.hpp:305-310 */
void orc_relu(const float* x, int64_t n, float* y) {
  for (int64_t i = 0; i < n; ++i) y[i] = x[i] > 0.0f ? x[i] : 0.0f;
}

/* batch_norm eval branch: norms.hpp:65-95. istd in double, scale/shift in float. */
void orc_bn_eval(const float* x, int64_t rows, int64_t C, const float* gamma, const float* beta,
                 const float* rmean, const float* rvar, double eps, float* y) {
  float* scale = (float*)malloc(sizeof(float) * (size_t)C);
  float* shift = (float*)malloc(sizeof(float) * (size_t)C);
  for (int64_t i = 0; i < C; ++i) {
    const float istd = (float)(1.0 / sqrt((double)rvar[i] + eps));
    scale[i] = gamma[i] * istd;
    shift[i] = beta[i] - rmean[i] * scale[i];
  }
  for (int64_t r = 0; r < rows; ++r) {
    const float* xr = x + r * C;
    float* yr = y + r * C;
    for (int64_t i = 0; i < C; ++i) yr[i] = xr[i] * scale[i] + shift[i];
  }
  free(scale);
  free(shift);
}

/* layer_norm: norms.hpp:155-191 (double statistics). */
void orc_layer_norm(const float* x, int64_t rows, int64_t C, const float* gamma, const float* beta, double eps,
                    float* y) {
  for (int64_t r = 0; r < rows; ++r) {
    const float* xr = x + r * C;
    float* yr = y + r * C;
    double sum = 0.0, sq = 0.0;
    for (int64_t i = 0; i < C; ++i) {
      sum += xr[i];
      sq += (double)xr[i] * xr[i];
    }
    const double m = sum / (double)C;
    double v = sq / (double)C - m * m;
    if (v < 0) v = 0;
    const double istd = 1.0 / sqrt(v + eps);
    for (int64_t i = 0; i < C; ++i) yr[i] = (float)(((double)xr[i] - m) * istd * gamma[i] + beta[i]);
  }
}

/* elementwise mul/add: kernels.hpp:323-337 (op: ORC_ADD or ORC_MUL) */
void orc_elementwise(int op, const float* a, const float* b, int64_t n, float* y) {
  if (op == ORC_MUL)
    for (int64_t i = 0; i < n; ++i) y[i] = a[i] * b[i];
  else
    for (int64_t i = 0; i < n; ++i) y[i] = a[i] + b[i];
}

/* concat_channels: kernels.hpp:359-375 */
void orc_concat(const float* a, int64_t ca, const float* b, int64_t cb, int64_t rows, float* y) {
  for (int64_t r = 0; r < rows; ++r) {
    memcpy(y + r * (ca + cb), a + r * ca, sizeof(float) * (size_t)ca);
    memcpy(y + r * (ca + cb) + ca, b + r * cb, sizeof(float) * (size_t)cb);
  }
}

/* Network<float>::forward in eval mode: network.hpp:162-180 (node loop) and :380-420 (dispatch). */
int orc_forward(const int32_t* nodes, int n_nodes, int input_node, int output_node, const float* const* params,
                const int64_t* pdims, const uint8_t* bn_ready, const float* x, int64_t B, int64_t T, int64_t F,
                int64_t C, float* out) {
  const double bn_eps = 1e-5, ln_eps = 1e-5; /* network.hpp:429-431 */
  if (input_node < 0 || output_node < 0) {
    snprintf(g_err, sizeof g_err, "network has no input/output");
    return 1;
  }
  const int32_t* in_node = nodes + (size_t)input_node * ORC_NODE_FIELDS;
  if (in_node[10] != C) {
    snprintf(g_err, sizeof g_err, "network expects %d input channels, got [%lld,%lld,%lld,%lld]", in_node[10],
             (long long)B, (long long)T, (long long)F, (long long)C);
    return 1;
  }
  const int64_t rows = B * T * F;
  float** buf = (float**)calloc((size_t)n_nodes, sizeof(float*));
  int rc = 0;
  for (int i = 0; i < n_nodes && rc == 0; ++i) {
    const int32_t* n = nodes + (size_t)i * ORC_NODE_FIELDS;
    const int op = n[0], in0 = n[1], in1 = n[2], cout = n[10], dil = n[11] > 0 ? n[11] : 1;
    buf[i] = (float*)malloc(sizeof(float) * (size_t)(rows * cout));
    if (i == input_node) {
      memcpy(buf[i], x, sizeof(float) * (size_t)(rows * C));
      continue;
    }
    const int64_t cin = nodes[(size_t)in0 * ORC_NODE_FIELDS + 10];
    const float* a = buf[in0];
    switch (op) {
      case ORC_CONV: {
        const int64_t* d = pdims + 4 * n[3];
        if (d[2] != cin) {
          snprintf(g_err, sizeof g_err, "conv input has %lld channels but weights expect %lld", (long long)cin,
                   (long long)d[2]);
          rc = 1;
          break;
        }
        orc_conv2d(a, B, T, F, cin, params[n[3]], (int)d[0], (int)d[1], d[3], n[4] >= 0 ? params[n[4]] : NULL, 1,
                   dil, buf[i]);
        break;
      }
      case ORC_DWCONV: {
        const int64_t* d = pdims + 4 * n[3];
        orc_dwconv2d(a, B, T, F, cin, params[n[3]], (int)d[0], (int)d[1], n[4] >= 0 ? params[n[4]] : NULL, buf[i]);
        break;
      }
      case ORC_RELU:
        orc_relu(a, rows * cin, buf[i]);
        break;
      case ORC_BN:
        if (!bn_ready[n[9]]) {
          snprintf(g_err, sizeof g_err,
                   "batch norm evaluated in eval mode before any train-mode update; train first or seed the "
                   "running statistics");
          rc = 2;
          break;
        }
        orc_bn_eval(a, rows, cin, params[n[5]], params[n[6]], params[n[7]], params[n[8]], bn_eps, buf[i]);
        break;
      case ORC_LN:
        orc_layer_norm(a, rows, cin, params[n[5]], params[n[6]], ln_eps, buf[i]);
        break;
      case ORC_ADD:
      case ORC_MUL:
        orc_elementwise(op, a, buf[in1], rows * cin, buf[i]);
        break;
      case ORC_CONCAT: {
        const int64_t cb = nodes[(size_t)in1 * ORC_NODE_FIELDS + 10];
        orc_concat(a, cin, buf[in1], cb, rows, buf[i]);
        break;
      }
      default:
        snprintf(g_err, sizeof g_err, "unknown op %d", op);
        rc = 1;
    }
  }
  if (rc == 0) {
    const int64_t oc = nodes[(size_t)output_node * ORC_NODE_FIELDS + 10];
    memcpy(out, buf[output_node], sizeof(float) * (size_t)(rows * oc));
  }
  for (int i = 0; i < n_nodes; ++i) free(buf[i]);
  free(buf);
  return rc;
}

/* ---------------------------------------------------------------------------------------------
 * Rng (rng.hpp:14-69): std::mt19937_64 seeded with splitmix64(seed).
 * ------------------------------------------------------------------------------------------- */
static uint64_t splitmix64(uint64_t x) { /* rng.hpp:59-64 */
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

void orc_rng_seed(orc_rng* r, uint64_t seed) {
  r->mt[0] = splitmix64(seed);
  for (int i = 1; i < 312; ++i) r->mt[i] = 6364136223846793005ull * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->idx = 312;
}

uint64_t orc_rng_u64(orc_rng* r) {
  static const uint64_t UM = 0xFFFFFFFF80000000ull, LM = 0x7FFFFFFFull, A = 0xB5026F5AA96619E9ull;
  if (r->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      const uint64_t y = (r->mt[i] & UM) | (r->mt[(i + 1) % 312] & LM);
      r->mt[i] = r->mt[(i + 156) % 312] ^ (y >> 1) ^ ((y & 1u) ? A : 0u);
    }
    r->idx = 0;
  }
  uint64_t y = r->mt[r->idx++];
  y ^= (y >> 29) & 0x5555555555555555ull;
  y ^= (y << 17) & 0x71D67FFFEDA60000ull;
  y ^= (y << 37) & 0xFFF7EEE000000000ull;
  y ^= (y >> 43);
  return y;
}

double orc_rng_uniform(orc_rng* r) { return (double)(orc_rng_u64(r) >> 11) * 0x1.0p-53; } /* rng.hpp:21 */
int orc_rng_bit(orc_rng* r) { return (int)(orc_rng_u64(r) >> 63); }                        /* rng.hpp:31 */
double orc_rng_normal(orc_rng* r) {                                                         /* rng.hpp:34-39 */
  double u1 = orc_rng_uniform(r);
  double u2 = orc_rng_uniform(r);
  while (u1 <= 0.0) u1 = orc_rng_uniform(r);
  return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.141592653589793238462643383279502884 * u2);
}
uint64_t orc_rng_derive(uint64_t master, uint64_t index) { /* rng.hpp:54-56 */
  return splitmix64(master ^ splitmix64(index + 0x9E3779B97F4A7C15ull));
}

/* ---------------------------------------------------------------------------------------------
 * QAM (qam.cpp:10-52)
 * ------------------------------------------------------------------------------------------- */
static double axis_level(const uint8_t* b, int nbits) { /* qam.cpp:23-30 */
  const double s0 = 1.0 - 2.0 * b[0];
  if (nbits == 1) return s0;
  const double s1 = 1.0 - 2.0 * b[1];
  if (nbits == 2) return s0 * (2.0 - s1);
  const double s2 = 1.0 - 2.0 * b[2];
  return s0 * (4.0 - s1 * (2.0 - s2));
}

int orc_qam_map(const uint8_t* bits, int order, double* re, double* im) {
  int nb;
  double nf;
  switch (order) {
    case 4: nb = 2; nf = sqrt(2.0); break;
    case 16: nb = 4; nf = sqrt(10.0); break;
    case 64: nb = 6; nf = sqrt(42.0); break;
    default: snprintf(g_err, sizeof g_err, "modulation order must be 4, 16 or 64, got %d", order); return 1;
  }
  const int half = nb / 2;
  uint8_t ib[3], qb[3];
  for (int i = 0; i < half; ++i) {
    ib[i] = bits[2 * i];
    qb[i] = bits[2 * i + 1];
  }
  const double inv = 1.0 / nf;
  *re = axis_level(ib, half) * inv;
  *im = axis_level(qb, half) * inv;
  return 0;
}

/* pilot_pattern (pilots.cpp:13-31), generalised to several DM-RS symbols (BASELINE configs place
 * pilots on symbols 2 and 11; PilotConfig holds one, link_config.hpp:9-12). */
int orc_pilot_pattern(int T, int F, const int* symbols, int n_sym, int spacing, uint8_t* mask, double* values) {
  if (spacing < 1 || F < spacing) {
    snprintf(g_err, sizeof g_err, "pilot spacing must fit the subcarrier count");
    return 1;
  }
  memset(mask, 0, (size_t)T * (size_t)F);
  memset(values, 0, sizeof(double) * 2 * (size_t)T * (size_t)F);
  orc_rng rng;
  orc_rng_seed(&rng, 0x50494C4F54ull); /* "PILOT", pilots.cpp:10 */
  for (int s = 0; s < n_sym; ++s) {
    const int t = symbols[s];
    if (t < 0 || t >= T) {
      snprintf(g_err, sizeof g_err, "pilot symbol index out of range");
      return 1;
    }
    for (int f = 0; f < F; f += spacing) {
      uint8_t bits[2];
      bits[0] = (uint8_t)orc_rng_bit(&rng);
      bits[1] = (uint8_t)orc_rng_bit(&rng);
      const size_t idx = (size_t)t * (size_t)F + (size_t)f;
      mask[idx] = 1;
      orc_qam_map(bits, 4, &values[2 * idx], &values[2 * idx + 1]);
    }
  }
  return 0;
}

/* ---------------------------------------------------------------------------------------------
 * Featurize (format_nn_input SPEC.md:221-229 + LS/interpolation SPEC.md:272-289; see oracle.h).
 * Computed in double; the GPU kernel computes in fp32 and is compared with a tolerance.
 * ------------------------------------------------------------------------------------------- */
int orc_featurize(const float* y, int64_t B, int64_t T, int64_t F, int64_t N, const float* pilots,
                  const uint8_t* mask, float* feat) {
  int* psym = (int*)malloc(sizeof(int) * (size_t)T);
  int nps = 0;
  for (int64_t t = 0; t < T; ++t) {
    int any = 0;
    for (int64_t f = 0; f < F; ++f) any |= mask[t * F + f];
    if (any) psym[nps++] = (int)t;
  }
  if (nps == 0) {
    free(psym);
    snprintf(g_err, sizeof g_err, "pilot pattern has no pilots");
    return 1;
  }
  double* hs = (double*)malloc(sizeof(double) * 2 * (size_t)nps * (size_t)F); /* per pilot symbol, F-interp */
  int* pf = (int*)malloc(sizeof(int) * (size_t)F);
  const int C = (int)(6 * N);
  for (int64_t b = 0; b < B; ++b)
    for (int64_t a = 0; a < N; ++a) {
      for (int j = 0; j < nps; ++j) {
        const int s = psym[j];
        int np = 0;
        for (int64_t f = 0; f < F; ++f)
          if (mask[s * F + f]) pf[np++] = (int)f;
        for (int64_t f = 0; f < F; ++f) {
          int k0, k1;
          double w;
          if (f <= pf[0]) {
            k0 = k1 = 0;
            w = 0.0;
          } else if (f >= pf[np - 1]) {
            k0 = k1 = np - 1;
            w = 0.0;
          } else {
            k0 = 0;
            while (pf[k0 + 1] < f) ++k0;
            k1 = k0 + 1;
            w = (double)(f - pf[k0]) / (double)(pf[k1] - pf[k0]);
          }
          double lr[2], li[2];
          for (int q = 0; q < 2; ++q) {
            const int fq = pf[q == 0 ? k0 : k1];
            const size_t yi = (size_t)(((b * T + s) * F + fq) * N + a);
            const double yr = y[2 * yi], yim = y[2 * yi + 1];
            const double xr = pilots[2 * (s * F + fq)], xi = pilots[2 * (s * F + fq) + 1];
            const double den = xr * xr + xi * xi;
            lr[q] = (yr * xr + yim * xi) / den;
            li[q] = (yim * xr - yr * xi) / den;
          }
          hs[2 * ((size_t)j * F + f)] = (1.0 - w) * lr[0] + w * lr[1];
          hs[2 * ((size_t)j * F + f) + 1] = (1.0 - w) * li[0] + w * li[1];
        }
      }
      for (int64_t t = 0; t < T; ++t) {
        int j0, j1;
        double w;
        if (t <= psym[0]) {
          j0 = j1 = 0;
          w = 0.0;
        } else if (t >= psym[nps - 1]) {
          j0 = j1 = nps - 1;
          w = 0.0;
        } else {
          j0 = 0;
          while (psym[j0 + 1] < t) ++j0;
          j1 = j0 + 1;
          w = (double)(t - psym[j0]) / (double)(psym[j1] - psym[j0]);
        }
        for (int64_t f = 0; f < F; ++f) {
          const size_t yi = (size_t)(((b * T + t) * F + f) * N + a);
          float* o = feat + ((b * T + t) * F + f) * C + 6 * a;
          o[0] = y[2 * yi];
          o[1] = y[2 * yi + 1];
          o[2] = pilots[2 * (t * F + f)];
          o[3] = pilots[2 * (t * F + f) + 1];
          o[4] = (float)((1.0 - w) * hs[2 * ((size_t)j0 * F + f)] + w * hs[2 * ((size_t)j1 * F + f)]);
          o[5] = (float)((1.0 - w) * hs[2 * ((size_t)j0 * F + f) + 1] + w * hs[2 * ((size_t)j1 * F + f) + 1]);
        }
      }
    }
  free(psym);
  free(hs);
  free(pf);
  return 0;
}
