/*
 * flatneat_oracle.c -- TEST INFRASTRUCTURE ONLY (see flatneat_oracle.h).
 *
 * CPU restatement of the reference flatneat hot path, one function per
 * reference function, each citing the file:line it follows
 * (paths relative to /root/reference/proj/include/flatneat/).
 * Compiled without -march and with -ffp-contract=off: every FP64 operation
 * rounds separately, as in the reference Release build.
 */
#include "flatneat_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static const char* errc_name(int c) {
  /* errors.hpp:33-57 */
  static const char* names[] = {
      "unknown_function", "genome_full", "duplicate_key", "duplicate_conn",
      "dangling_endpoint", "key_not_found", "protected_node", "attr_out_of_range",
      "shape_mismatch", "corrupt_row", "cycle_detected", "non_finite_input",
      "non_finite_state", "empty_aggregation", "empty_dataset", "parse_error",
      "version_unsupported", "limits_too_small", "config_error", "eval_error"};
  return (c >= 0 && c < 20) ? names[c] : "unknown";
}

/* ------------------------------------------------------------------------ */
/* RNG  (rng.hpp:19-134)                                                    */
/* ------------------------------------------------------------------------ */

void fo_philox(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
  /* rng.hpp:19-35: Random123 Philox4x32-10 */
  uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
  uint32_t k0 = key_in[0], k1 = key_in[1];
  for (int i = 0; i < 10; ++i) {
    uint64_t a = (uint64_t)0xD2511F53u * c0;
    uint64_t b = (uint64_t)0xCD9E8D57u * c2;
    uint32_t n0 = (uint32_t)(b >> 32) ^ c1 ^ k0;
    uint32_t n1 = (uint32_t)b;
    uint32_t n2 = (uint32_t)(a >> 32) ^ c3 ^ k1;
    uint32_t n3 = (uint32_t)a;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

fo_key fo_key_seed(uint64_t seed) {
  /* rng.hpp:48-56 */
  uint32_t ctr[4] = {(uint32_t)seed, (uint32_t)(seed >> 32), 0x464C4154u, 0x4E454154u};
  uint32_t key[2] = {0x243F6A88u, 0x85A308D3u};
  fo_key k;
  fo_philox(ctr, key, k.w);
  return k;
}

fo_key fo_key_split(fo_key k, uint64_t index) {
  /* rng.hpp:58-66 */
  uint32_t ctr[4] = {(uint32_t)index, (uint32_t)(index >> 32), k.w[2], k.w[3]};
  uint32_t key[2] = {k.w[0], k.w[1]};
  fo_key c;
  fo_philox(ctr, key, c.w);
  return c;
}

void fo_stream_init(fo_stream* s, fo_key k) {
  s->key = k;
  s->block = 0;
  memset(s->buf, 0, sizeof(s->buf));
  s->avail = 0;
}

uint64_t fo_next_u64(fo_stream* s) {
  /* rng.hpp:81-87 and refill 119-128 */
  if (s->avail == 0) {
    uint32_t ctr[4] = {(uint32_t)s->block, (uint32_t)(s->block >> 32),
                       s->key.w[2] ^ 0x9E3779B9u, s->key.w[3]};
    uint32_t key[2] = {s->key.w[0], s->key.w[1]};
    fo_philox(ctr, key, s->buf);
    s->block++;
    s->avail = 4;
  }
  s->avail -= 2;
  uint64_t lo = s->buf[s->avail];
  uint64_t hi = s->buf[s->avail + 1];
  return (hi << 32) | lo;
}

double fo_uniform(fo_stream* s) {
  /* rng.hpp:90-92 */
  return (double)(fo_next_u64(s) >> 11) * 0x1.0p-53;
}

int fo_coin(fo_stream* s, double p) { return fo_uniform(s) < p; } /* rng.hpp:96 */

uint64_t fo_below(fo_stream* s, uint64_t n) {
  /* rng.hpp:99-106 */
  const uint64_t mx = ~(uint64_t)0;
  const uint64_t limit = mx - ((mx % n) + 1) % n;
  uint64_t x = fo_next_u64(s);
  while (x > limit) x = fo_next_u64(s);
  return x % n;
}

static int fo_index(fo_stream* s, int n) { return (int)fo_below(s, (uint64_t)n); }

double fo_normal(fo_stream* s, double mean, double sd) {
  /* rng.hpp:111-116: Box-Muller, no spare; host glibc log/cos */
  const double u1 = 1.0 - fo_uniform(s);
  const double u2 = fo_uniform(s);
  const double r = sqrt(-2.0 * log(u1));
  const double sr = sd * r;
  return mean + sr * cos(6.283185307179586476925286766559 * u2);
}

/* ------------------------------------------------------------------------ */
/* Genome row helpers (genome.hpp:177-231)                                  */
/* ------------------------------------------------------------------------ */

#define NROW(n, r) ((n) + (size_t)(r) * FO_NODE_COLS)
#define CROW(c, r) ((c) + (size_t)(r) * FO_CONN_COLS)

static int node_empty(const double* n, int r) { return isnan(NROW(n, r)[FO_NODE_KEY]); }
static int conn_empty(const double* c, int r) { return isnan(CROW(c, r)[FO_CONN_IN]); }

static int find_node(const fo_shape* sh, const double* n, int key) {
  for (int r = 0; r < sh->max_nodes; ++r)
    if (!node_empty(n, r) && (int)NROW(n, r)[FO_NODE_KEY] == key) return r;
  return -1;
}

static int find_conn(const fo_shape* sh, const double* c, int in, int out) {
  for (int r = 0; r < sh->max_conns; ++r) {
    if (conn_empty(c, r)) continue;
    if ((int)CROW(c, r)[FO_CONN_IN] == in && (int)CROW(c, r)[FO_CONN_OUT] == out) return r;
  }
  return -1;
}

static int first_empty_node(const fo_shape* sh, const double* n) {
  for (int r = 0; r < sh->max_nodes; ++r)
    if (node_empty(n, r)) return r;
  return -1;
}

static int first_empty_conn(const fo_shape* sh, const double* c) {
  for (int r = 0; r < sh->max_conns; ++r)
    if (conn_empty(c, r)) return r;
  return -1;
}

static int is_input(const fo_shape* sh, int key) {
  for (int i = 0; i < sh->num_inputs; ++i)
    if (sh->input_keys[i] == key) return 1;
  return 0;
}

static int is_output(const fo_shape* sh, int key) {
  for (int i = 0; i < sh->num_outputs; ++i)
    if (sh->output_keys[i] == key) return 1;
  return 0;
}

static int fail(char* msg, size_t n, int code, const char* detail) {
  if (msg) snprintf(msg, n, "%s: %s", errc_name(code), detail);
  return 1 + code;
}

/* ------------------------------------------------------------------------ */
/* Transform (network.hpp:122-220) and describe_cycle (network.hpp:73-115)  */
/* ------------------------------------------------------------------------ */

typedef struct { int key, row; } kr_t;

static int kr_cmp(const void* a, const void* b) {
  const kr_t* x = (const kr_t*)a;
  const kr_t* y = (const kr_t*)b;
  if (x->key != y->key) return x->key < y->key ? -1 : 1;
  return x->row < y->row ? -1 : (x->row > y->row);
}

static int row_of_key(const kr_t* k2r, int n, int key) {
  /* network.hpp:57-63: lower_bound on key */
  int lo = 0, hi = n;
  while (lo < hi) {
    int mid = (lo + hi) / 2;
    if (k2r[mid].key < key) lo = mid + 1; else hi = mid;
  }
  if (lo == n || k2r[lo].key != key) return -1;
  return k2r[lo].row;
}

static void describe_cycle(const fo_shape* sh, const double* nodes, const double* conns,
                           const unsigned char* emitted, const int* row_key,
                           char* out, size_t outn) {
  const int N = sh->max_nodes;
  int start = -1;
  for (int r = 0; r < N; ++r)
    if (!node_empty(nodes, r) && !emitted[r] && (start < 0 || row_key[r] < row_key[start]))
      start = r;
  if (start < 0) { snprintf(out, outn, "unlocatable cycle"); return; }
  int* path = (int*)malloc(sizeof(int) * (size_t)(N + 1));
  int* pos = (int*)malloc(sizeof(int) * (size_t)N);
  int plen = 0;
  for (int r = 0; r < N; ++r) pos[r] = -1;
  int at = start;
  for (;;) {
    if (pos[at] >= 0) {
      size_t used = 0;
      out[0] = 0;
      for (int i = pos[at]; i < plen; ++i)
        used += (size_t)snprintf(out + used, used < outn ? outn - used : 0, "%d->", row_key[path[i]]);
      snprintf(out + used, used < outn ? outn - used : 0, "%d", row_key[at]);
      break;
    }
    pos[at] = plen;
    path[plen++] = at;
    int next = -1;
    for (int r = 0; r < sh->max_conns; ++r) {
      if (conn_empty(conns, r)) continue;
      const double* row = CROW(conns, r);
      if (row[FO_CONN_EN] != 1.0) continue;
      if ((int)row[FO_CONN_IN] != row_key[at]) continue;
      for (int rr = 0; rr < N; ++rr) {
        if (node_empty(nodes, rr) || emitted[rr]) continue;
        if (row_key[rr] == (int)row[FO_CONN_OUT]) {
          if (next < 0 || row_key[rr] < row_key[next]) next = rr;
        }
      }
    }
    if (next < 0) { snprintf(out, outn, "unlocatable cycle"); break; }
    at = next;
  }
  free(path);
  free(pos);
}

int fo_transform(const fo_shape* sh, const fo_schema* sc, const double* nodes,
                 const double* conns, fo_net* net) {
  const int N = sh->max_nodes;
  char detail[400];
  int status = 0;
  int* row_key = (int*)malloc(sizeof(int) * (size_t)N);
  kr_t* k2r = (kr_t*)malloc(sizeof(kr_t) * (size_t)N);
  unsigned char* row_is_input = (unsigned char*)calloc((size_t)N, 1);
  unsigned char* emitted = (unsigned char*)calloc((size_t)N, 1);
  int* in_degree = (int*)calloc((size_t)N, sizeof(int));
  double* expanded = (double*)malloc(sizeof(double) * (size_t)N * (size_t)N);
  kr_t* ready = (kr_t*)malloc(sizeof(kr_t) * (size_t)N);
  int nk = 0, populated = 0;
  net->msg[0] = 0;
  net->order_count = 0;
  for (int i = 0; i < N; ++i) net->order[i] = -1;
  for (size_t i = 0; i < (size_t)N * (size_t)N; ++i) expanded[i] = NAN;

  /* :139-152 resolve attributes row by row (activation first, then aggregation) */
  for (int r = 0; r < N; ++r) {
    row_key[r] = -1;
    if (node_empty(nodes, r)) continue;
    const double* row = NROW(nodes, r);
    const int key = (int)row[FO_NODE_KEY];
    row_key[r] = key;
    k2r[nk].key = key; k2r[nk].row = r; ++nk;
    const int act = (int)row[FO_NODE_ACT];
    if (act < 0 || act >= sc->n_act) {
      snprintf(detail, sizeof detail, "activation id %d out of range", act);
      status = fail(net->msg, sizeof net->msg, FO_E_unknown_function, detail);
      goto done;
    }
    const int agg = (int)row[FO_NODE_AGG];
    if (agg < 0 || agg >= sc->n_agg) {
      snprintf(detail, sizeof detail, "aggregation id %d out of range", agg);
      status = fail(net->msg, sizeof net->msg, FO_E_unknown_function, detail);
      goto done;
    }
    ++populated;
  }
  qsort(k2r, (size_t)nk, sizeof(kr_t), kr_cmp);

  /* :155-165 */
  for (int i = 0; i < sh->num_inputs; ++i) {
    const int r = row_of_key(k2r, nk, sh->input_keys[i]);
    if (r < 0) {
      snprintf(detail, sizeof detail, "input key %d", sh->input_keys[i]);
      status = fail(net->msg, sizeof net->msg, FO_E_dangling_endpoint, detail);
      goto done;
    }
    net->input_rows[i] = r;
    row_is_input[r] = 1;
  }
  for (int i = 0; i < sh->num_outputs; ++i) {
    const int r = row_of_key(k2r, nk, sh->output_keys[i]);
    if (r < 0) {
      snprintf(detail, sizeof detail, "output key %d", sh->output_keys[i]);
      status = fail(net->msg, sizeof net->msg, FO_E_dangling_endpoint, detail);
      goto done;
    }
    net->output_rows[i] = r;
  }

  /* :167-183 expanded + in-degree over enabled rows */
  for (int r = 0; r < sh->max_conns; ++r) {
    if (conn_empty(conns, r)) continue;
    const double* row = CROW(conns, r);
    const int src = row_of_key(k2r, nk, (int)row[FO_CONN_IN]);
    const int dst = row_of_key(k2r, nk, (int)row[FO_CONN_OUT]);
    if (src < 0 || dst < 0) {
      snprintf(detail, sizeof detail, "conn (%d, %d)", (int)row[FO_CONN_IN], (int)row[FO_CONN_OUT]);
      status = fail(net->msg, sizeof net->msg, FO_E_dangling_endpoint, detail);
      goto done;
    }
    if (row[FO_CONN_EN] != 1.0) continue;
    expanded[(size_t)src * N + dst] = row[FO_CONN_W];
    ++in_degree[dst];
  }
  /* :184-190 incoming lists, ascending source row */
  {
    int e = 0;
    for (int dst = 0; dst < N; ++dst) {
      net->in_begin[dst] = e;
      for (int src = 0; src < N; ++src) {
        const double w = expanded[(size_t)src * N + dst];
        if (!isnan(w)) {
          net->in_src[e] = src;
          net->in_w[e] = w;
          ++e;
        }
      }
    }
    net->in_begin[N] = e;
  }

  /* :192-214 Kahn, smallest (key,row) first */
  {
    int nready = 0;
    for (int r = 0; r < N; ++r)
      if (row_key[r] >= 0 && in_degree[r] == 0) { ready[nready].key = row_key[r]; ready[nready].row = r; ++nready; }
    while (nready > 0) {
      int best = 0;
      for (int i = 1; i < nready; ++i)
        if (kr_cmp(&ready[i], &ready[best]) < 0) best = i;
      const int r = ready[best].row;
      ready[best] = ready[--nready];
      net->order[net->order_count++] = r;
      emitted[r] = 1;
      for (int dst = 0; dst < N; ++dst) {
        if (isnan(expanded[(size_t)r * N + dst])) continue;
        if (--in_degree[dst] == 0) { ready[nready].key = row_key[dst]; ready[nready].row = dst; ++nready; }
      }
    }
  }
  /* :216-218 */
  if (net->order_count != populated) {
    char cyc[300];
    describe_cycle(sh, nodes, conns, emitted, row_key, cyc, sizeof cyc);
    snprintf(detail, sizeof detail, "cycle %s", cyc);
    status = fail(net->msg, sizeof net->msg, FO_E_cycle_detected, detail);
  }

done:
  free(row_key); free(k2r); free(row_is_input); free(emitted); free(in_degree);
  free(expanded); free(ready);
  return status;
}

static double act_apply(int code, double x) {
  /* functions.hpp:17-21 */
  switch (code) {
    case FO_ACT_IDENTITY: return x;
    case FO_ACT_TANH: return tanh(x);
    case FO_ACT_SIGMOID: return 1.0 / (1.0 + exp(-x));
    case FO_ACT_RELU: return x > 0.0 ? x : 0.0;
    case FO_ACT_SIN: return sin(x);
  }
  return x;
}

int fo_forward(const fo_shape* sh, const fo_schema* sc, const double* nodes,
               const fo_net* net, const double* inputs, double* outputs, double* v) {
  /* network.hpp:238-268 */
  const int N = sh->max_nodes;
  for (int i = 0; i < sh->num_inputs; ++i)
    if (!isfinite(inputs[i])) return 1 + FO_E_non_finite_input;
  for (int r = 0; r < N; ++r) v[r] = NAN;
  unsigned char is_in[1024] = {0};
  if (N > 1024) return 1 + FO_E_limits_too_small;
  for (int i = 0; i < sh->num_inputs; ++i) { v[net->input_rows[i]] = inputs[i]; is_in[net->input_rows[i]] = 1; }
  for (int idx = 0; idx < net->order_count; ++idx) {
    const int r = net->order[idx];
    if (is_in[r]) continue;
    const double* row = NROW(nodes, r);
    const int agg = sc->agg[(int)row[FO_NODE_AGG]];
    const int act = sc->act[(int)row[FO_NODE_ACT]];
    const int b = net->in_begin[r], e = net->in_begin[r + 1];
    double a;
    if (b == e) {
      a = (agg == FO_AGG_PRODUCT) ? 1.0 : 0.0;  /* functions.hpp:44-52 */
    } else if (agg == FO_AGG_SUM || agg == FO_AGG_MEAN) {
      a = 0.0;
      for (int k = b; k < e; ++k) a += net->in_w[k] * v[net->in_src[k]];
      if (agg == FO_AGG_MEAN) a = a / (double)(e - b);
    } else if (agg == FO_AGG_PRODUCT) {
      a = 1.0;
      for (int k = b; k < e; ++k) a *= net->in_w[k] * v[net->in_src[k]];
    } else {
      a = net->in_w[b] * v[net->in_src[b]];
      for (int k = b + 1; k < e; ++k) {
        const double x = net->in_w[k] * v[net->in_src[k]];
        a = x > a ? x : a;
      }
    }
    const double pre = row[FO_NODE_RESP] * a;
    v[r] = act_apply(act, pre + row[FO_NODE_BIAS]);
  }
  for (int o = 0; o < sh->num_outputs; ++o) outputs[o] = v[net->output_rows[o]];
  return 0;
}

/* ------------------------------------------------------------------------ */
/* Distance (ops.hpp:415-473)                                               */
/* ------------------------------------------------------------------------ */

double fo_distance(const fo_shape* sh, const double* n1, const double* c1,
                   const double* n2, const double* c2, const fo_dist_cfg* cfg) {
  double total = 0.0;
  {
    int cn1 = 0, cn2 = 0, matching = 0;
    double sum = 0.0;
    for (int r = 0; r < sh->max_nodes; ++r) if (!node_empty(n2, r)) ++cn2;
    for (int r = 0; r < sh->max_nodes; ++r) {
      if (node_empty(n1, r)) continue;
      ++cn1;
      const double* a = NROW(n1, r);
      const int m = find_node(sh, n2, (int)a[FO_NODE_KEY]);
      if (m < 0) continue;
      ++matching;
      const double* b = NROW(n2, m);
      double d = fabs(a[FO_NODE_BIAS] - b[FO_NODE_BIAS]);
      d = d + fabs(a[FO_NODE_RESP] - b[FO_NODE_RESP]);
      d = d + (a[FO_NODE_AGG] != b[FO_NODE_AGG] ? 1.0 : 0.0);
      d = d + (a[FO_NODE_ACT] != b[FO_NODE_ACT] ? 1.0 : 0.0);
      sum += d / 4.0;
    }
    const int disjoint = (cn1 - matching) + (cn2 - matching);
    int nm = cn1 > cn2 ? cn1 : cn2;
    if (nm < 1) nm = 1;
    const double t = cfg->compatibility_disjoint * (double)disjoint;
    total += t / (double)nm;
    if (matching > 0) {
      const double h = cfg->compatibility_homologous * sum;
      total += h / (double)matching;
    }
  }
  {
    int cn1 = 0, cn2 = 0, matching = 0;
    double sum = 0.0;
    for (int r = 0; r < sh->max_conns; ++r) if (!conn_empty(c2, r)) ++cn2;
    for (int r = 0; r < sh->max_conns; ++r) {
      if (conn_empty(c1, r)) continue;
      ++cn1;
      const double* a = CROW(c1, r);
      const int m = find_conn(sh, c2, (int)a[FO_CONN_IN], (int)a[FO_CONN_OUT]);
      if (m < 0) continue;
      ++matching;
      const double* b = CROW(c2, m);
      sum += fabs(a[FO_CONN_W] - b[FO_CONN_W]) / 1.0;
    }
    const int disjoint = (cn1 - matching) + (cn2 - matching);
    int nm = cn1 > cn2 ? cn1 : cn2;
    if (nm < 1) nm = 1;
    const double t = cfg->compatibility_disjoint * (double)disjoint;
    total += t / (double)nm;
    if (matching > 0) {
      const double h = cfg->compatibility_homologous * sum;
      total += h / (double)matching;
    }
  }
  return total;
}

/* ------------------------------------------------------------------------ */
/* Crossover (ops.hpp:382-407)                                              */
/* ------------------------------------------------------------------------ */

void fo_crossover(const fo_shape* sh, const double* fn, const double* fc,
                  const double* on, const double* oc, fo_key key,
                  double* cn, double* cc) {
  memcpy(cn, fn, sizeof(double) * (size_t)sh->max_nodes * FO_NODE_COLS);
  memcpy(cc, fc, sizeof(double) * (size_t)sh->max_conns * FO_CONN_COLS);
  fo_stream s;
  fo_stream_init(&s, key);
  for (int r = 0; r < sh->max_nodes; ++r) {
    if (node_empty(cn, r)) continue;
    double* row = NROW(cn, r);
    const int m = find_node(sh, on, (int)row[FO_NODE_KEY]);
    if (m < 0) continue;
    const double* theirs = NROW(on, m);
    for (int a = 1; a < FO_NODE_COLS; ++a)
      if (fo_coin(&s, 0.5)) row[a] = theirs[a];
  }
  for (int r = 0; r < sh->max_conns; ++r) {
    if (conn_empty(cc, r)) continue;
    double* row = CROW(cc, r);
    const int m = find_conn(sh, oc, (int)row[FO_CONN_IN], (int)row[FO_CONN_OUT]);
    if (m < 0) continue;
    const double* theirs = CROW(oc, m);
    for (int a = 3; a < FO_CONN_COLS; ++a)
      if (fo_coin(&s, 0.5)) row[a] = theirs[a];
  }
}

/* ------------------------------------------------------------------------ */
/* Structural primitives (ops.hpp:19-111)                                   */
/* ------------------------------------------------------------------------ */

int fo_add_node(const fo_shape* sh, double* nodes, const double row[5]) {
  /* ops.hpp:19-27 */
  const int key = (int)row[FO_NODE_KEY];
  if (find_node(sh, nodes, key) >= 0) return 1 + FO_E_duplicate_key;
  const int r = first_empty_node(sh, nodes);
  if (r < 0) return 1 + FO_E_genome_full;
  memcpy(NROW(nodes, r), row, sizeof(double) * FO_NODE_COLS);
  return 0;
}

int fo_remove_node(const fo_shape* sh, double* nodes, double* conns, int key) {
  /* ops.hpp:30-44 */
  if (is_input(sh, key) || is_output(sh, key)) return 1 + FO_E_protected_node;
  const int r = find_node(sh, nodes, key);
  if (r < 0) return 1 + FO_E_key_not_found;
  for (int a = 0; a < FO_NODE_COLS; ++a) NROW(nodes, r)[a] = NAN;
  for (int c = 0; c < sh->max_conns; ++c) {
    if (conn_empty(conns, c)) continue;
    double* row = CROW(conns, c);
    if ((int)row[FO_CONN_IN] == key || (int)row[FO_CONN_OUT] == key)
      for (int a = 0; a < FO_CONN_COLS; ++a) row[a] = NAN;
  }
  return 0;
}

int fo_add_conn(const fo_shape* sh, const double* nodes, double* conns, const double row[4]) {
  /* ops.hpp:46-58 */
  const int in = (int)row[FO_CONN_IN], out = (int)row[FO_CONN_OUT];
  if (find_node(sh, nodes, in) < 0 || find_node(sh, nodes, out) < 0) return 1 + FO_E_dangling_endpoint;
  if (find_conn(sh, conns, in, out) >= 0) return 1 + FO_E_duplicate_conn;
  const int r = first_empty_conn(sh, conns);
  if (r < 0) return 1 + FO_E_genome_full;
  memcpy(CROW(conns, r), row, sizeof(double) * FO_CONN_COLS);
  return 0;
}

int fo_remove_conn(const fo_shape* sh, double* conns, int in_key, int out_key) {
  /* ops.hpp:60-67 */
  const int r = find_conn(sh, conns, in_key, out_key);
  if (r < 0) return 1 + FO_E_key_not_found;
  for (int a = 0; a < FO_CONN_COLS; ++a) CROW(conns, r)[a] = NAN;
  return 0;
}

int fo_creates_cycle(const fo_shape* sh, const double* conns, int from_key, int to_key) {
  /* ops.hpp:93-111: is from_key reachable from to_key over enabled conns?
   * Restated as a worklist over keys with a visited list; same boolean. */
  if (from_key == to_key) return 1;
  const int C = sh->max_conns;
  int* stack = (int*)malloc(sizeof(int) * (size_t)(C + 1) * 2);
  int* seen = (int*)malloc(sizeof(int) * (size_t)(C + 1) * 2);
  int ns = 0, nseen = 0, hit = 0;
  stack[ns++] = to_key;
  while (ns > 0) {
    const int at = stack[--ns];
    if (at == from_key) { hit = 1; break; }
    int dup = 0;
    for (int i = 0; i < nseen; ++i) if (seen[i] == at) { dup = 1; break; }
    if (dup) continue;
    seen[nseen++] = at;
    for (int r = 0; r < C; ++r) {
      if (conn_empty(conns, r)) continue;
      const double* row = CROW(conns, r);
      if (row[FO_CONN_EN] == 1.0 && (int)row[FO_CONN_IN] == at) stack[ns++] = (int)row[FO_CONN_OUT];
    }
  }
  free(stack);
  free(seen);
  return hit;
}

/* ------------------------------------------------------------------------ */
/* Mutation (ops.hpp:178-374)                                               */
/* ------------------------------------------------------------------------ */

fo_split_plan fo_plan_node_split(const fo_shape* sh, const double* nodes,
                                 const double* conns, fo_key key, const fo_mut_cfg* cfg) {
  /* ops.hpp:196-217 */
  fo_split_plan p = {0, 0, 0};
  if (cfg->node_add <= 0.0) return p;
  fo_stream s;
  fo_stream_init(&s, fo_key_split(key, 0));
  if (!fo_coin(&s, cfg->node_add)) return p;
  int n_en = 0;
  int* en = (int*)malloc(sizeof(int) * (size_t)sh->max_conns);
  for (int r = 0; r < sh->max_conns; ++r)
    if (!conn_empty(conns, r) && CROW(conns, r)[FO_CONN_EN] == 1.0) en[n_en++] = r;
  if (n_en == 0 || first_empty_node(sh, nodes) < 0) { free(en); return p; }
  int free_rows = 0;
  for (int r = 0; r < sh->max_conns && free_rows < 2; ++r)
    if (conn_empty(conns, r)) ++free_rows;
  if (free_rows < 2) { free(en); return p; }
  const int pick = en[fo_index(&s, n_en)];
  free(en);
  p.split = 1;
  p.in_key = (int)CROW(conns, pick)[FO_CONN_IN];
  p.out_key = (int)CROW(conns, pick)[FO_CONN_OUT];
  return p;
}

int fo_apply_node_split(const fo_shape* sh, const fo_schema* sc, double* nodes,
                        double* conns, fo_split_plan plan, int new_key,
                        fo_key key, const fo_mut_cfg* cfg) {
  /* ops.hpp:222-243 */
  if (!plan.split) return 0;
  const int r = find_conn(sh, conns, plan.in_key, plan.out_key);
  if (r < 0) return 0;
  const double old_w = CROW(conns, r)[FO_CONN_W];
  CROW(conns, r)[FO_CONN_EN] = 0.0;
  fo_stream s;
  fo_stream_init(&s, fo_key_split(key, 1));
  double node[5];
  node[0] = (double)new_key;
  node[1] = fo_normal(&s, cfg->bias.init_mean, cfg->bias.init_std);
  node[2] = fo_normal(&s, cfg->response.init_mean, cfg->response.init_std);
  node[3] = (double)sc->default_agg;
  node[4] = (double)sc->default_act;
  int st = fo_add_node(sh, nodes, node);
  if (st) return st;
  const double c1[4] = {(double)plan.in_key, (double)new_key, 1.0, 1.0};
  st = fo_add_conn(sh, nodes, conns, c1);
  if (st) return st;
  const double c2[4] = {(double)new_key, (double)plan.out_key, 1.0, old_w};
  return fo_add_conn(sh, nodes, conns, c2);
}

static int int_cmp(const void* a, const void* b) {
  const int x = *(const int*)a, y = *(const int*)b;
  return (x > y) - (x < y);
}

/* ops.hpp:251-279 */
static int pick_new_conn(const fo_shape* sh, const double* nodes, const double* conns,
                         fo_stream* s, int* from_out, int* to_out) {
  const int N = sh->max_nodes;
  int* keys = (int*)malloc(sizeof(int) * (size_t)N);
  int* targets = (int*)malloc(sizeof(int) * (size_t)N);
  int nk = 0, nt = 0, found = 0;
  for (int r = 0; r < N; ++r)
    if (!node_empty(nodes, r)) keys[nk++] = (int)NROW(nodes, r)[FO_NODE_KEY];
  for (int i = 0; i < nk; ++i)
    if (!is_input(sh, keys[i])) targets[nt++] = keys[i];
  if (nk == 0 || nt == 0) goto out;
  for (int probe = 0; probe < 16; ++probe) {
    const int from = keys[fo_index(s, nk)];
    const int to = targets[fo_index(s, nt)];
    if (find_conn(sh, conns, from, to) < 0 && !fo_creates_cycle(sh, conns, from, to)) {
      *from_out = from; *to_out = to; found = 1; goto out;
    }
  }
  qsort(keys, (size_t)nk, sizeof(int), int_cmp);
  qsort(targets, (size_t)nt, sizeof(int), int_cmp);
  {
    int* cand = (int*)malloc(sizeof(int) * 2 * (size_t)nk * (size_t)nt);
    int nc = 0;
    for (int i = 0; i < nk; ++i)
      for (int j = 0; j < nt; ++j)
        if (find_conn(sh, conns, keys[i], targets[j]) < 0 &&
            !fo_creates_cycle(sh, conns, keys[i], targets[j])) {
          cand[2 * nc] = keys[i]; cand[2 * nc + 1] = targets[j]; ++nc;
        }
    if (nc > 0) {
      const int k = fo_index(s, nc);
      *from_out = cand[2 * k]; *to_out = cand[2 * k + 1]; found = 1;
    }
    free(cand);
  }
out:
  free(keys);
  free(targets);
  return found;
}

static void mutate_scalar(double* v, const fo_attr_mut* m, fo_stream* s) {
  /* ops.hpp:281-289 */
  const double u = fo_uniform(s);
  if (u < m->mutate_rate) {
    *v += fo_normal(s, 0.0, m->mutate_power);
  } else if (u < m->mutate_rate + m->replace_rate) {
    *v = fo_normal(s, m->init_mean, m->init_std);
  }
}

int fo_mutate_rest(const fo_shape* sh, const fo_schema* sc, double* nodes,
                   double* conns, fo_key key, const fo_mut_cfg* cfg) {
  /* ops.hpp:296-361 */
  {
    fo_stream s;
    fo_stream_init(&s, fo_key_split(key, 2));
    if (cfg->conn_add > 0.0 && fo_coin(&s, cfg->conn_add) && first_empty_conn(sh, conns) >= 0) {
      int from, to;
      if (pick_new_conn(sh, nodes, conns, &s, &from, &to)) {
        double row[4];
        row[0] = (double)from; row[1] = (double)to; row[2] = 1.0;
        row[3] = fo_normal(&s, cfg->weight.init_mean, cfg->weight.init_std);
        const int st = fo_add_conn(sh, nodes, conns, row);
        if (st) return st;
      }
    }
  }
  {
    fo_stream s;
    fo_stream_init(&s, fo_key_split(key, 3));
    if (cfg->node_delete > 0.0 && fo_coin(&s, cfg->node_delete)) {
      int* hidden = (int*)malloc(sizeof(int) * (size_t)sh->max_nodes);
      int nh = 0;
      for (int r = 0; r < sh->max_nodes; ++r) {
        if (node_empty(nodes, r)) continue;
        const int k = (int)NROW(nodes, r)[FO_NODE_KEY];
        if (!is_input(sh, k) && !is_output(sh, k)) hidden[nh++] = k;
      }
      int st = 0;
      if (nh > 0) st = fo_remove_node(sh, nodes, conns, hidden[fo_index(&s, nh)]);
      free(hidden);
      if (st) return st;
    }
  }
  {
    fo_stream s;
    fo_stream_init(&s, fo_key_split(key, 4));
    if (cfg->conn_delete > 0.0 && fo_coin(&s, cfg->conn_delete)) {
      int* rows = (int*)malloc(sizeof(int) * (size_t)sh->max_conns);
      int nr = 0;
      for (int r = 0; r < sh->max_conns; ++r) if (!conn_empty(conns, r)) rows[nr++] = r;
      int st = 0;
      if (nr > 0) {
        const int r = rows[fo_index(&s, nr)];
        st = fo_remove_conn(sh, conns, (int)CROW(conns, r)[FO_CONN_IN], (int)CROW(conns, r)[FO_CONN_OUT]);
      }
      free(rows);
      if (st) return st;
    }
  }
  {
    fo_stream s;
    fo_stream_init(&s, fo_key_split(key, 5));
    for (int r = 0; r < sh->max_nodes; ++r) {
      if (node_empty(nodes, r)) continue;
      double* row = NROW(nodes, r);
      if (is_input(sh, (int)row[FO_NODE_KEY])) continue;
      mutate_scalar(&row[FO_NODE_BIAS], &cfg->bias, &s);
      mutate_scalar(&row[FO_NODE_RESP], &cfg->response, &s);
      if (cfg->aggregation_replace_rate > 0.0 && fo_coin(&s, cfg->aggregation_replace_rate))
        row[FO_NODE_AGG] = (double)fo_index(&s, sc->n_agg);
      if (cfg->activation_replace_rate > 0.0 && fo_coin(&s, cfg->activation_replace_rate))
        row[FO_NODE_ACT] = (double)fo_index(&s, sc->n_act);
    }
    for (int r = 0; r < sh->max_conns; ++r) {
      if (conn_empty(conns, r)) continue;
      mutate_scalar(&CROW(conns, r)[FO_CONN_W], &cfg->weight, &s);
    }
  }
  return 0;
}

void fo_innov_init(fo_innov* t, int first_key) {
  t->next_key = first_key;
  t->count = 0;
  t->cap = 64;
  t->pairs = (int*)malloc(sizeof(int) * 3 * (size_t)t->cap);
}

void fo_innov_free(fo_innov* t) { free(t->pairs); t->pairs = NULL; }

int fo_innov_get_or_assign(fo_innov* t, int in_key, int out_key) {
  /* ops.hpp:149-156 */
  for (int i = 0; i < t->count; ++i)
    if (t->pairs[3 * i] == in_key && t->pairs[3 * i + 1] == out_key) return t->pairs[3 * i + 2];
  if (t->count == t->cap) {
    t->cap *= 2;
    t->pairs = (int*)realloc(t->pairs, sizeof(int) * 3 * (size_t)t->cap);
  }
  const int key = t->next_key++;
  t->pairs[3 * t->count] = in_key;
  t->pairs[3 * t->count + 1] = out_key;
  t->pairs[3 * t->count + 2] = key;
  t->count++;
  return key;
}

void fo_innov_next_generation(fo_innov* t) { t->count = 0; } /* ops.hpp:158 */

int fo_mutate(const fo_shape* sh, const fo_schema* sc, double* nodes,
              double* conns, fo_key key, const fo_mut_cfg* cfg, fo_innov* t) {
  /* ops.hpp:363-374.  Value semantics: on error the input is left as is. */
  const size_t nn = (size_t)sh->max_nodes * FO_NODE_COLS, cn = (size_t)sh->max_conns * FO_CONN_COLS;
  double* wn = (double*)malloc(sizeof(double) * nn);
  double* wc = (double*)malloc(sizeof(double) * cn);
  memcpy(wn, nodes, sizeof(double) * nn);
  memcpy(wc, conns, sizeof(double) * cn);
  int st = 0;
  const fo_split_plan plan = fo_plan_node_split(sh, wn, wc, key, cfg);
  if (plan.split) {
    const int new_key = fo_innov_get_or_assign(t, plan.in_key, plan.out_key);
    st = fo_apply_node_split(sh, sc, wn, wc, plan, new_key, key, cfg);
  }
  if (!st) st = fo_mutate_rest(sh, sc, wn, wc, key, cfg);
  if (!st) {
    memcpy(nodes, wn, sizeof(double) * nn);
    memcpy(conns, wc, sizeof(double) * cn);
  }
  free(wn);
  free(wc);
  return st;
}

/* ------------------------------------------------------------------------ */
/* explain_invalid (genome.hpp:364-417)                                     */
/* ------------------------------------------------------------------------ */

static int row_all_nan(const double* row, int n) {
  for (int i = 0; i < n; ++i) if (!isnan(row[i])) return 0;
  return 1;
}
static int row_all_finite(const double* row, int n) {
  for (int i = 0; i < n; ++i) if (!isfinite(row[i])) return 0;
  return 1;
}
static int bsearch_int(const int* a, int n, int k) {
  int lo = 0, hi = n;
  while (lo < hi) { int m = (lo + hi) / 2; if (a[m] < k) lo = m + 1; else hi = m; }
  return lo < n && a[lo] == k;
}
static int pair_cmp(const void* a, const void* b) {
  const int* x = (const int*)a; const int* y = (const int*)b;
  if (x[0] != y[0]) return x[0] < y[0] ? -1 : 1;
  return (x[1] > y[1]) - (x[1] < y[1]);
}

int fo_explain_invalid(const fo_shape* sh, const fo_schema* sc, const double* nodes,
                       const double* conns, char* buf, size_t n) {
  int* keys = (int*)malloc(sizeof(int) * (size_t)sh->max_nodes);
  int* pairs = (int*)malloc(sizeof(int) * 2 * (size_t)sh->max_conns);
  int nk = 0, np = 0, bad = 1;
  for (int r = 0; r < sh->max_nodes; ++r) {
    const double* row = NROW(nodes, r);
    if (row_all_nan(row, 5)) continue;
    if (!row_all_finite(row, 5)) { snprintf(buf, n, "node row %d partially NaN", r); goto out; }
    const double key = row[0];
    if (key < 0 || key != floor(key)) { snprintf(buf, n, "node row %d has non-integral key", r); goto out; }
    const int agg = (int)row[FO_NODE_AGG], act = (int)row[FO_NODE_ACT];
    if (row[FO_NODE_AGG] != floor(row[FO_NODE_AGG]) || agg < 0 || agg >= sc->n_agg) { snprintf(buf, n, "node row %d has bad aggregation id", r); goto out; }
    if (row[FO_NODE_ACT] != floor(row[FO_NODE_ACT]) || act < 0 || act >= sc->n_act) { snprintf(buf, n, "node row %d has bad activation id", r); goto out; }
    keys[nk++] = (int)key;
  }
  qsort(keys, (size_t)nk, sizeof(int), int_cmp);
  for (int i = 1; i < nk; ++i) if (keys[i] == keys[i - 1]) { snprintf(buf, n, "duplicate node key"); goto out; }
  for (int i = 0; i < sh->num_inputs; ++i)
    if (!bsearch_int(keys, nk, sh->input_keys[i])) { snprintf(buf, n, "input key %d missing", sh->input_keys[i]); goto out; }
  for (int i = 0; i < sh->num_outputs; ++i)
    if (!bsearch_int(keys, nk, sh->output_keys[i])) { snprintf(buf, n, "output key %d missing", sh->output_keys[i]); goto out; }
  for (int r = 0; r < sh->max_conns; ++r) {
    const double* row = CROW(conns, r);
    if (row_all_nan(row, 4)) continue;
    if (!row_all_finite(row, 4)) { snprintf(buf, n, "conn row %d partially NaN", r); goto out; }
    const double e = row[FO_CONN_EN];
    if (e != 0.0 && e != 1.0) { snprintf(buf, n, "conn row %d has non-boolean enabled flag", r); goto out; }
    const int in = (int)row[0], o = (int)row[1];
    if (row[0] != floor(row[0]) || row[1] != floor(row[1]) || in < 0 || o < 0) { snprintf(buf, n, "conn row %d has non-integral endpoint", r); goto out; }
    if (!bsearch_int(keys, nk, in) || !bsearch_int(keys, nk, o)) { snprintf(buf, n, "conn row %d references a missing node", r); goto out; }
    pairs[2 * np] = in; pairs[2 * np + 1] = o; ++np;
  }
  qsort(pairs, (size_t)np, 2 * sizeof(int), pair_cmp);
  for (int i = 1; i < np; ++i)
    if (pairs[2 * i] == pairs[2 * i - 2] && pairs[2 * i + 1] == pairs[2 * i - 1]) { snprintf(buf, n, "duplicate connection pair"); goto out; }
  bad = 0;
  if (n) buf[0] = 0;
out:
  free(keys);
  free(pairs);
  return bad;
}

/* ------------------------------------------------------------------------ */
/* Test generator (tests/support/generators.hpp:37-84)                      */
/* ------------------------------------------------------------------------ */

int fo_random_acyclic_genome(fo_stream* s, const fo_schema* sc, const fo_genspec* spec,
                             int max_nodes, int max_conns, double* nodes, double* conns) {
  const int hidden = spec->max_hidden > 0 ? fo_index(s, spec->max_hidden + 1) : 0;
  const int total = spec->num_inputs + spec->num_outputs + hidden;
  int* by_rank = (int*)malloc(sizeof(int) * (size_t)total);
  int nr = 0;
  for (int i = 0; i < spec->num_inputs; ++i) by_rank[nr++] = i;
  int* hk = by_rank + nr;
  for (int h = 0; h < hidden; ++h) hk[h] = spec->num_inputs + spec->num_outputs + h;
  for (int i = hidden - 1; i > 0; --i) {
    const int j = fo_index(s, i + 1);
    const int t = hk[i]; hk[i] = hk[j]; hk[j] = t;
  }
  nr += hidden;
  for (int o = 0; o < spec->num_outputs; ++o) by_rank[nr++] = spec->num_inputs + o;

  for (size_t i = 0; i < (size_t)max_nodes * FO_NODE_COLS; ++i) nodes[i] = NAN;
  for (size_t i = 0; i < (size_t)max_conns * FO_CONN_COLS; ++i) conns[i] = NAN;
  int status = 0;
  /* node rows are generated for every key even if they overflow, to keep
   * the stream in step with the reference (pad happens afterwards). */
  double* tmpn = (double*)malloc(sizeof(double) * FO_NODE_COLS * (size_t)total);
  for (int k = 0; k < total; ++k) {
    double* row = tmpn + (size_t)k * FO_NODE_COLS;
    row[0] = (double)k;
    row[1] = fo_normal(s, 0.0, 1.0);
    const double n = fo_normal(s, 0.0, 1.0);
    const double t = 0.1 * n;
    row[2] = 1.0 + t;
    row[3] = (double)fo_index(s, sc->n_agg);
    row[4] = (double)fo_index(s, sc->n_act);
  }
  int cap = 64, nc = 0;
  double* tmpc = (double*)malloc(sizeof(double) * FO_CONN_COLS * (size_t)cap);
  for (int a = 0; a < total; ++a) {
    for (int b = a + 1; b < total; ++b) {
      const int from = by_rank[a], to = by_rank[b];
      int to_is_input = 0;
      for (int i = 0; i < spec->num_inputs; ++i) if (i == to) to_is_input = 1;
      if (to_is_input) continue;
      if (!fo_coin(s, spec->conn_prob)) continue;
      if (nc == cap) { cap *= 2; tmpc = (double*)realloc(tmpc, sizeof(double) * FO_CONN_COLS * (size_t)cap); }
      double* row = tmpc + (size_t)nc * FO_CONN_COLS;
      row[0] = (double)from;
      row[1] = (double)to;
      row[2] = fo_coin(s, spec->disabled_prob) ? 0.0 : 1.0;
      row[3] = fo_normal(s, 0.0, 1.0);
      ++nc;
    }
  }
  if (total > max_nodes || nc > max_conns) {
    status = 1 + FO_E_genome_full;
  } else {
    memcpy(nodes, tmpn, sizeof(double) * FO_NODE_COLS * (size_t)total);
    memcpy(conns, tmpc, sizeof(double) * FO_CONN_COLS * (size_t)nc);
  }
  free(tmpn);
  free(tmpc);
  free(by_rank);
  return status;
}
