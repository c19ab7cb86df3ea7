/* oracle.h — TEST INFRASTRUCTURE ONLY: plain-C restatement of the reference's CoNet-Rx inference
 * path (proj/core of arxiv/paper_2510_12739). Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load it; the product (paper_2510_12739_b200) never does.
 * Pinned against the reference compiled in place (oracle/_ref) by tests/test_oracle_pin.py and
 * against the committed fixtures in tests/golden/. */
#ifndef CNRX_ORACLE_H
#define CNRX_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* LayerOp (network.hpp:17) */
enum { ORC_INPUT = 0, ORC_CONV, ORC_DWCONV, ORC_RELU, ORC_BN, ORC_LN, ORC_ADD, ORC_MUL, ORC_CONCAT };

/* Node record: op,in0,in1,w,b,gamma,beta,rmean,rvar,bn_flag,out_channels,dilation_f (GraphNode,
 * network.hpp:19-26, plus the dilation extension needed by BASELINE config 3). */
#define ORC_NODE_FIELDS 12

void orc_conv2d(const float* x, int64_t B, int64_t T, int64_t F, int64_t Cin, const float* w, int kh, int kw,
                int64_t Cout, const float* bias, int dil_t, int dil_f, float* y);
void orc_dwconv2d(const float* x, int64_t B, int64_t T, int64_t F, int64_t C, const float* w, int kh, int kw,
                  const float* bias, float* y);
void orc_relu(const float* x, int64_t n, float* y);
void orc_bn_eval(const float* x, int64_t rows, int64_t C, const float* gamma, const float* beta,
                 const float* rmean, const float* rvar, double eps, float* y);
void orc_layer_norm(const float* x, int64_t rows, int64_t C, const float* gamma, const float* beta, double eps,
                    float* y);
void orc_elementwise(int op, const float* a, const float* b, int64_t n, float* y);
void orc_concat(const float* a, int64_t ca, const float* b, int64_t cb, int64_t rows, float* y);

/* Graph executor restating Network<float>::forward in eval mode (network.hpp:162-180, :380-420).
 * params[i] points at parameter i's data, pdims[4*i..] its dims (unused trailing dims = 1).
 * bn_ready[flag] must be non-zero for every batch norm (norms.hpp:66-69), else returns 2.
 * Returns 0 on success, 1 on a shape/argument error (message via orc_last_error). */
int orc_forward(const int32_t* nodes, int n_nodes, int input_node, int output_node, const float* const* params,
                const int64_t* pdims, const uint8_t* bn_ready, const float* x, int64_t B, int64_t T, int64_t F,
                int64_t C, float* out);
const char* orc_last_error(void);

/* Rng restatement (rng.hpp:14-69): splitmix64-seeded mt19937_64. */
typedef struct {
  uint64_t mt[312];
  int idx;
} orc_rng;
void orc_rng_seed(orc_rng* r, uint64_t seed);
uint64_t orc_rng_u64(orc_rng* r);
double orc_rng_uniform(orc_rng* r);
int orc_rng_bit(orc_rng* r);
double orc_rng_normal(orc_rng* r);
uint64_t orc_rng_derive(uint64_t master, uint64_t index);

/* Gray QAM map (qam.cpp:10-52). Returns 0 or 1 for an unsupported order. */
int orc_qam_map(const uint8_t* bits, int order, double* re, double* im);

/* Pilot pattern (pilots.cpp:13-31) generalised to n_sym DM-RS symbols: for each listed symbol in
 * order, every `spacing`-th subcarrier from 0 gets a QPSK value from the fixed "PILOT" stream.
 * n_sym == 1 reproduces the reference exactly. values: [T*F] complex (re,im) doubles. */
int orc_pilot_pattern(int T, int F, const int* symbols, int n_sym, int spacing, uint8_t* mask, double* values);

/* Featurize (restated from SPEC.md:221-229 + :272-289, adapted to BASELINE's feature set; the
 * reference's format_nn_input / classic.cpp are missing from the snapshot):
 *   y: [B,T,F,N] complex float (re,im), pilots: [T,F] complex float, mask: [T,F].
 *   ls at pilot REs = y / x_p; interpolate linearly in F within each pilot symbol (nearest beyond the
 *   first/last pilot subcarrier), then linearly in T between pilot symbols (nearest outside).
 *   feat: [B,T,F,6N], per antenna a: [Re y, Im y, Re x_p, Im x_p, Re h_ls, Im h_ls] at 6a+k. */
int orc_featurize(const float* y, int64_t B, int64_t T, int64_t F, int64_t N, const float* pilots,
                  const uint8_t* mask, float* feat);

#ifdef __cplusplus
}
#endif
#endif
