/*
 * mtx_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU implementation of what the synchronous
 * data-parallel SGD step of MaTEx-TensorFlow (arXiv 1704.04560) computes.  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * leg may load it.  It shares no code, header, table or constant generator with
 * the CUDA path (paper_1704_04560_b200/csrc); neither includes the other.
 *
 * Arithmetic is IEEE double (the paper fixes no precision, PAPER.md:436-437,
 * SURVEY.md §8(c) A11) except orc_avg_update_f32, which is the fp32
 * correctly-rounded-FMA definition of the update used for the bit-exact pin.
 * Compile with -O2 -ffp-contract=off and no fast-math so every operation below
 * is exactly the one written.
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n; "S:n" = SPEC.md line n;
 * "A<k>" / "O<k>" = readings listed in DESIGN.md.
 *
 * Parity status per function is stated in DESIGN.md §"Oracle pins"; every
 * function here is pinned (none is "parity unpinned").
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ O1/O2 generator
 * H(key,k): the k-th output of SplitMix64 seeded with key (Steele et al. 2014).
 * Used here only for parameter initialisation (O2); data come in as inputs. */
uint64_t orc_splitmix64(uint64_t key, uint64_t k) {
    uint64_t z = key + (k + 1) * 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* ------------------------------------------------------------------ network description
 * MLP (kind 0): widths d_0..d_L, Z_l = A_{l-1} W_l + b_l, W_l is [d_{l-1}][d_l]
 *   (x.W + b convention), ReLU on hidden layers, softmax-CE on the last.
 * CNN (kind 1, LeNet-style, A7): NHWC input [in_h][in_w][in_c]; each conv layer
 *   is valid/stride-1 k x k with W[kh][kw][ci][co], + bias, ReLU, 2x2/2 max-pool;
 *   then flatten (h,w,c) and fully-connected layers fc_dims (last = classes).
 * Canonical tensor order (O2): W_1, b_1, W_2, b_2, ... (conv first). */
typedef struct {
    int32_t kind;
    int32_t n_dims;
    const int32_t *dims;
    int32_t in_h, in_w, in_c;
    int32_t n_conv;
    const int32_t *conv_k;
    const int32_t *conv_c;
    int32_t n_fc;
    const int32_t *fc_dims;
} orc_net;

#define ORC_MAX_T 64

typedef struct {
    int n;                     /* number of tensors */
    int64_t off[ORC_MAX_T], size[ORC_MAX_T];
    int fan_in[ORC_MAX_T], fan_out[ORC_MAX_T], is_bias[ORC_MAX_T];
    int64_t total;
} orc_tensors;

static void add_tensor(orc_tensors *t, int64_t size, int fi, int fo, int bias) {
    int i = t->n++;
    t->off[i] = t->total;
    t->size[i] = size;
    t->fan_in[i] = fi;
    t->fan_out[i] = fo;
    t->is_bias[i] = bias;
    t->total += size;
}

/* Spatial sizes after conv layer c (valid) and its 2x2/2 pool (floor). */
static void cnn_shapes(const orc_net *m, int c, int *h_in, int *w_in, int *c_in, int *h_conv, int *w_conv,
                       int *h_pool, int *w_pool) {
    int h = m->in_h, w = m->in_w, ch = m->in_c;
    for (int i = 0; i < c; i++) {
        h = (h - m->conv_k[i] + 1) / 2;
        w = (w - m->conv_k[i] + 1) / 2;
        ch = m->conv_c[i];
    }
    *h_in = h; *w_in = w; *c_in = ch;
    *h_conv = h - m->conv_k[c] + 1;
    *w_conv = w - m->conv_k[c] + 1;
    *h_pool = *h_conv / 2;
    *w_pool = *w_conv / 2;
}

static int cnn_flat_dim(const orc_net *m) {
    int hi, wi, ci, hc, wc, hp, wp;
    cnn_shapes(m, m->n_conv - 1, &hi, &wi, &ci, &hc, &wc, &hp, &wp);
    return hp * wp * m->conv_c[m->n_conv - 1];
}

static void enum_tensors(const orc_net *m, orc_tensors *t) {
    memset(t, 0, sizeof(*t));
    if (m->kind == 0) {
        for (int l = 1; l < m->n_dims; l++) {
            add_tensor(t, (int64_t)m->dims[l - 1] * m->dims[l], m->dims[l - 1], m->dims[l], 0);
            add_tensor(t, m->dims[l], 0, 0, 1);
        }
    } else {
        int cin = m->in_c;
        for (int c = 0; c < m->n_conv; c++) {
            int k = m->conv_k[c], co = m->conv_c[c];
            add_tensor(t, (int64_t)k * k * cin * co, k * k * cin, k * k * co, 0);
            add_tensor(t, co, 0, 0, 1);
            cin = co;
        }
        int d = cnn_flat_dim(m);
        for (int f = 0; f < m->n_fc; f++) {
            add_tensor(t, (int64_t)d * m->fc_dims[f], d, m->fc_dims[f], 0);
            add_tensor(t, m->fc_dims[f], 0, 0, 1);
            d = m->fc_dims[f];
        }
    }
}

int64_t orc_param_count(const orc_net *m) {
    orc_tensors t;
    enum_tensors(m, &t);
    return t.total;
}

int orc_tensor_table(const orc_net *m, int64_t *off, int64_t *size) {
    orc_tensors t;
    enum_tensors(m, &t);
    for (int i = 0; i < t.n; i++) { off[i] = t.off[i]; size[i] = t.size[i]; }
    return t.n;
}

/* O2 (A9): Glorot-uniform weights, zero biases, keyed by (seed, 16 + tensor index).
 * u = (H(K(seed,16+t), e) >> 40) * 2^-24 (exact); lim = (float)sqrt(6/(fan_in+fan_out));
 * w = (2u - 1) * lim with one fp32 rounding.  The paper only says an initializer
 * runs; rank r uses seed init_seed + r so that the broadcast
 * is observable. */
void orc_init_params(const orc_net *m, uint64_t seed, float *out) {
    orc_tensors t;
    enum_tensors(m, &t);
    for (int i = 0; i < t.n; i++) {
        float *p = out + t.off[i];
        if (t.is_bias[i]) {
            for (int64_t e = 0; e < t.size[i]; e++) p[e] = 0.0f;
            continue;
        }
        uint64_t key = orc_splitmix64(seed, (uint64_t)(16 + i));
        float lim = (float)sqrt(6.0 / (double)(t.fan_in[i] + t.fan_out[i]));
        for (int64_t e = 0; e < t.size[i]; e++) {
            uint64_t bits = orc_splitmix64(key, (uint64_t)e) >> 40;  /* 24 bits */
            float u = (float)bits * 0x1p-24f;                          /* exact */
            float two_u_minus_1 = 2.0f * u - 1.0f;                     /* exact */
            p[e] = two_u_minus_1 * lim;                                /* one rounding */
        }
    }
}

/* ------------------------------------------------------------------ O4 shard (A10)
 * Global batch window of step t starts at s_t = (t*B) mod n and covers the
 * cyclic positions s_t .. s_t+B-1; rank r owns positions [r*b, (r+1)*b),
 * b = B/P (B mod P == 0, A1; B <= n so a window never repeats a sample).
 * Returned as <= 2 contiguous pieces of sample ids.
 * S:351-368 (balanced partition of each cyclic window). */
int orc_batch_slice(int64_t n, int64_t B, int64_t step, int32_t rank, int32_t P, int64_t begin[2], int64_t len[2]) {
    if (n <= 0 || B <= 0 || B > n || P <= 0 || rank < 0 || rank >= P || B % P != 0 || step < 0) return -1;
    int64_t b = B / P;
    int64_t s = (int64_t)(((__int128)step * B) % n);
    int64_t first = (s + (int64_t)rank * b) % n;
    begin[0] = first;
    begin[1] = 0;
    if (first + b <= n) {
        len[0] = b;
        len[1] = 0;
    } else {
        len[0] = n - first;
        len[1] = b - (n - first);
    }
    return 0;
}

static int64_t shard_sample(int64_t n, int64_t B, int64_t step, int32_t rank, int32_t P, int64_t i) {
    int64_t b = B / P;
    int64_t s = (int64_t)(((__int128)step * B) % n);
    return (s + (int64_t)rank * b + i) % n;
}

/* ------------------------------------------------------------------ O6 loss / dlogits
 * Mean softmax cross-entropy with max subtraction (A8):
 *   m = max_j z_j, S = sum_j exp(z_j - m), l = m + log S - z_y,
 *   dz_j = (exp(z_j - m)/S - [j == y]) / b   (local mean, A1). */
static double softmax_xent_row(const double *z, int C, int y, double inv_b, double *dz) {
    double m = z[0];
    for (int j = 1; j < C; j++) if (z[j] > m) m = z[j];
    double S = 0.0;
    for (int j = 0; j < C; j++) S += exp(z[j] - m);
    double loss = m + log(S) - z[y];
    if (dz) {
        for (int j = 0; j < C; j++) {
            double p = exp(z[j] - m) / S;
            dz[j] = (p - (j == y ? 1.0 : 0.0)) * inv_b;
        }
    }
    return loss;
}

/* ------------------------------------------------------------------ tf32emu
 * The TF32 tier's contractions, emulated: tcgen05 kind::tf32 reads each fp32 operand with its low
 * 13 mantissa bits dropped (reading A12, measured: 1+2^-11+2^-12 -> 1, 1+3*2^-11 -> 1+2^-10).  The
 * operand is first rounded to fp32, the format it is stored in, then truncated; products and sums
 * stay exact-ish (double).  Which contractions the TF32 tier issues on tensor cores (reading A23):
 * the hidden layers' forward (d_l >= 16), dgrad (d_{l-1} >= 16) and weight gradient (d_l > 16),
 * when both widths are multiples of 4; the last layer (softmax head), narrow weight gradients and
 * every bias gradient (column sums) are fp32 CUDA-core arithmetic, i.e. exact here. */
static double tf32_of(double x) {
    float f = (float)x;
    uint32_t u;
    memcpy(&u, &f, 4);
    u &= 0xFFFFE000u;
    memcpy(&f, &u, 4);
    return (double)f;
}

double orc_tf32(double x) { return tf32_of(x); }

/* ------------------------------------------------------------------ MLP O5-O7
 * Local gradient of the mean loss over this rank's shard (b = B/P rows) at the
 * given parameters, written in canonical order into grad (length N); returns
 * the local loss SUM (sum of per-row losses, i ascending).
 *   forward  Z_l = A_{l-1} W_l + b_l (k ascending, bias after the sum, A13);
 *            A_l = max(Z_l, 0) for l < L
 *   backward dW_l = A_{l-1}^T dZ_l, db_l = colsum dZ_l (i ascending);
 *            dZ_{l-1} = (dZ_l W_l^T) .* [A_{l-1} > 0]  (ReLU'(0) = 0, A5)
 * S:44-49 gradient rules; P:298-301 (gradients are the data tokens reduced).
 * If acts != NULL, the hidden/logit activations of layer `acts_layer` are copied
 * out ([b][d_l], post-ReLU for hidden layers, logits for the last). */
static double mlp_local(const orc_net *m, const double *params, const float *X, const int32_t *y, int64_t n,
                        int64_t B, int64_t step, int32_t rank, int32_t P, int64_t b_override, double *grad,
                        int acts_layer, double *acts, int tf32emu) {
    orc_tensors t;
    enum_tensors(m, &t);
    const int L = m->n_dims - 1;
    const int64_t b = b_override > 0 ? b_override : B / P;
    const int *d = m->dims;
    /* tf32emu: which contractions of layer l take TF32 operands (A23, see tf32_of) */
#define AL4(l) (d[(l) - 1] % 4 == 0 && d[(l)] % 4 == 0)
#define FWD_TC(l) (tf32emu && (l) < L && d[(l)] >= 16 && AL4(l))
#define DGRAD_TC(l) (tf32emu && (l) < L && d[(l) - 1] >= 16 && AL4(l))
#define WGRAD_TC(l) (tf32emu && (l) < L && d[(l)] > 16 && AL4(l))
#define OP(tc, x) ((tc) ? tf32_of(x) : (x))
    double **A = calloc((size_t)L + 1, sizeof(double *));
    for (int l = 0; l <= L; l++) A[l] = calloc((size_t)(b * d[l]), sizeof(double));
    for (int64_t i = 0; i < b; i++) {
        int64_t s = b_override > 0 ? i : shard_sample(n, B, step, rank, P, i);
        for (int k = 0; k < d[0]; k++) A[0][i * d[0] + k] = (double)X[s * d[0] + k];
    }
    int dmax = 1;
    for (int l = 0; l <= L; l++) if (d[l] > dmax) dmax = d[l];
    double *acc = malloc(sizeof(double) * (size_t)dmax);
    for (int l = 1; l <= L; l++) {
        const double *W = params + t.off[2 * (l - 1)];
        const double *bias = params + t.off[2 * (l - 1) + 1];
        const int tc = FWD_TC(l);
        for (int64_t i = 0; i < b; i++) {
            for (int j = 0; j < d[l]; j++) acc[j] = 0.0;
            for (int k = 0; k < d[l - 1]; k++) {
                double a = OP(tc, A[l - 1][i * d[l - 1] + k]);
                for (int j = 0; j < d[l]; j++) acc[j] += a * OP(tc, W[(int64_t)k * d[l] + j]);
            }
            for (int j = 0; j < d[l]; j++) {
                double z = acc[j] + bias[j];
                A[l][i * d[l] + j] = (l < L) ? (z > 0.0 ? z : 0.0) : z;
            }
        }
    }
    if (acts) memcpy(acts, A[acts_layer], sizeof(double) * (size_t)(b * d[acts_layer]));
    /* loss + dZ_L */
    const int C = d[L];
    double *dZ = calloc((size_t)(b * C), sizeof(double));
    double loss_sum = 0.0;
    const double inv_b = 1.0 / (double)b;
    for (int64_t i = 0; i < b; i++) {
        int64_t s = b_override > 0 ? i : shard_sample(n, B, step, rank, P, i);
        loss_sum += softmax_xent_row(A[L] + i * C, C, y[s], inv_b, dZ + i * C);
    }
    if (grad) {
        memset(grad, 0, sizeof(double) * (size_t)t.total);
        for (int l = L; l >= 1; l--) {
            double *dW = grad + t.off[2 * (l - 1)];
            double *db = grad + t.off[2 * (l - 1) + 1];
            const double *W = params + t.off[2 * (l - 1)];
            const int tcw = WGRAD_TC(l), tcd = DGRAD_TC(l);
            for (int64_t i = 0; i < b; i++) {
                const double *a = A[l - 1] + i * d[l - 1];
                const double *dz = dZ + i * d[l];
                for (int k = 0; k < d[l - 1]; k++)
                    for (int j = 0; j < d[l]; j++) dW[(int64_t)k * d[l] + j] += OP(tcw, a[k]) * OP(tcw, dz[j]);
                for (int j = 0; j < d[l]; j++) db[j] += dz[j];
            }
            if (l > 1) {
                double *dprev = calloc((size_t)(b * d[l - 1]), sizeof(double));
                for (int64_t i = 0; i < b; i++) {
                    for (int k = 0; k < d[l - 1]; k++) {
                        double s = 0.0;
                        for (int j = 0; j < d[l]; j++)
                            s += OP(tcd, dZ[i * d[l] + j]) * OP(tcd, W[(int64_t)k * d[l] + j]);
                        dprev[i * d[l - 1] + k] = A[l - 1][i * d[l - 1] + k] > 0.0 ? s : 0.0;
                    }
                }
                free(dZ);
                dZ = dprev;
            }
        }
    }
    free(dZ);
    free(acc);
    for (int l = 0; l <= L; l++) free(A[l]);
    free(A);
    return loss_sum;
#undef AL4
#undef FWD_TC
#undef DGRAD_TC
#undef WGRAD_TC
#undef OP
}

/* ------------------------------------------------------------------ CNN O5-O7
 * Per sample n (ascending): for each conv layer c
 *   Y[oh][ow][co] = b[co] + sum_{kh,kw,ci asc} X[oh+kh][ow+kw][ci] W[kh][kw][ci][co]
 *   R = max(Y, 0);  P[ph][pw][co] = max over the 2x2 window of R, argmax = first
 *   maximum in (dh, dw) row-major order with strict '>' (A6)
 * then flatten (h,w,c) (A7) and the MLP head (ReLU between fc layers).
 * Backward: head as in mlp; pool routes dP to its argmax; ReLU mask [R > 0];
 * conv wgrad dW += X (x) dY, db += dY; conv dgrad dX = sum dY W (textbook). */
typedef struct {
    int hi, wi, ci, hc, wc, hp, wp, co, k;
} conv_geom;

static double cnn_local(const orc_net *m, const double *params, const float *X, const int32_t *y, int64_t n,
                        int64_t B, int64_t step, int32_t rank, int32_t P, int64_t b_override, double *grad) {
    orc_tensors t;
    enum_tensors(m, &t);
    const int NC = m->n_conv, NF = m->n_fc;
    const int64_t b = b_override > 0 ? b_override : B / P;
    conv_geom g[8];
    for (int c = 0; c < NC; c++) {
        cnn_shapes(m, c, &g[c].hi, &g[c].wi, &g[c].ci, &g[c].hc, &g[c].wc, &g[c].hp, &g[c].wp);
        g[c].co = m->conv_c[c];
        g[c].k = m->conv_k[c];
    }
    int fd[16];
    fd[0] = cnn_flat_dim(m);
    for (int f = 0; f < NF; f++) fd[f + 1] = m->fc_dims[f];
    const int C = fd[NF];
    const int in_sz = m->in_h * m->in_w * m->in_c;
    if (grad) memset(grad, 0, sizeof(double) * (size_t)t.total);
    double loss_sum = 0.0;
    const double inv_b = 1.0 / (double)b;

    /* per-sample buffers */
    double *xin[9], *R[8], *Pl[8], *dR[8], *dX[9];
    int *arg[8];
    xin[0] = malloc(sizeof(double) * in_sz);
    dX[0] = NULL;
    for (int c = 0; c < NC; c++) {
        R[c] = malloc(sizeof(double) * g[c].hc * g[c].wc * g[c].co);
        dR[c] = malloc(sizeof(double) * g[c].hc * g[c].wc * g[c].co);
        Pl[c] = malloc(sizeof(double) * g[c].hp * g[c].wp * g[c].co);
        arg[c] = malloc(sizeof(int) * g[c].hp * g[c].wp * g[c].co);
        xin[c + 1] = Pl[c];
        dX[c + 1] = malloc(sizeof(double) * g[c].hp * g[c].wp * g[c].co);
    }
    double *Af[16], *dAf[16];
    for (int f = 0; f <= NF; f++) {
        Af[f] = malloc(sizeof(double) * fd[f]);
        dAf[f] = malloc(sizeof(double) * fd[f]);
    }

    for (int64_t i = 0; i < b; i++) {
        int64_t s = b_override > 0 ? i : shard_sample(n, B, step, rank, P, i);
        for (int e = 0; e < in_sz; e++) xin[0][e] = (double)X[s * in_sz + e];
        /* conv stack forward */
        for (int c = 0; c < NC; c++) {
            const conv_geom *G = &g[c];
            const double *W = params + t.off[2 * c];
            const double *bias = params + t.off[2 * c + 1];
            for (int oh = 0; oh < G->hc; oh++)
                for (int ow = 0; ow < G->wc; ow++)
                    for (int co = 0; co < G->co; co++) {
                        double acc = 0.0;
                        for (int kh = 0; kh < G->k; kh++)
                            for (int kw = 0; kw < G->k; kw++)
                                for (int ci = 0; ci < G->ci; ci++)
                                    acc += xin[c][((oh + kh) * G->wi + (ow + kw)) * G->ci + ci] *
                                           W[((kh * G->k + kw) * G->ci + ci) * G->co + co];
                        double z = acc + bias[co];
                        R[c][(oh * G->wc + ow) * G->co + co] = z > 0.0 ? z : 0.0;
                    }
            for (int ph = 0; ph < G->hp; ph++)
                for (int pw = 0; pw < G->wp; pw++)
                    for (int co = 0; co < G->co; co++) {
                        int best = -1;
                        double bv = 0.0;
                        for (int dh = 0; dh < 2; dh++)
                            for (int dw = 0; dw < 2; dw++) {
                                int idx = ((2 * ph + dh) * G->wc + (2 * pw + dw)) * G->co + co;
                                if (best < 0 || R[c][idx] > bv) { best = idx; bv = R[c][idx]; }
                            }
                        Pl[c][(ph * G->wp + pw) * G->co + co] = bv;
                        arg[c][(ph * G->wp + pw) * G->co + co] = best;
                    }
        }
        /* fc head forward */
        memcpy(Af[0], Pl[NC - 1], sizeof(double) * fd[0]);
        for (int f = 1; f <= NF; f++) {
            const double *W = params + t.off[2 * NC + 2 * (f - 1)];
            const double *bias = params + t.off[2 * NC + 2 * (f - 1) + 1];
            for (int j = 0; j < fd[f]; j++) {
                double acc = 0.0;
                for (int k = 0; k < fd[f - 1]; k++) acc += Af[f - 1][k] * W[(int64_t)k * fd[f] + j];
                double z = acc + bias[j];
                Af[f][j] = (f < NF) ? (z > 0.0 ? z : 0.0) : z;
            }
        }
        loss_sum += softmax_xent_row(Af[NF], C, y[s], inv_b, dAf[NF]);
        if (!grad) continue;
        /* fc head backward */
        for (int f = NF; f >= 1; f--) {
            double *dW = grad + t.off[2 * NC + 2 * (f - 1)];
            double *db = grad + t.off[2 * NC + 2 * (f - 1) + 1];
            const double *W = params + t.off[2 * NC + 2 * (f - 1)];
            for (int k = 0; k < fd[f - 1]; k++)
                for (int j = 0; j < fd[f]; j++) dW[(int64_t)k * fd[f] + j] += Af[f - 1][k] * dAf[f][j];
            for (int j = 0; j < fd[f]; j++) db[j] += dAf[f][j];
            for (int k = 0; k < fd[f - 1]; k++) {
                double s2 = 0.0;
                for (int j = 0; j < fd[f]; j++) s2 += dAf[f][j] * W[(int64_t)k * fd[f] + j];
                /* ReLU mask for hidden fc inputs; the flatten input (f==1) is a pool output,
                   whose gradient is routed through the pool below. */
                dAf[f - 1][k] = (f - 1 == 0) ? s2 : (Af[f - 1][k] > 0.0 ? s2 : 0.0);
            }
        }
        memcpy(dX[NC], dAf[0], sizeof(double) * fd[0]);
        /* conv stack backward */
        for (int c = NC - 1; c >= 0; c--) {
            const conv_geom *G = &g[c];
            const double *W = params + t.off[2 * c];
            double *dW = grad + t.off[2 * c];
            double *db = grad + t.off[2 * c + 1];
            int nR = G->hc * G->wc * G->co;
            for (int e = 0; e < nR; e++) dR[c][e] = 0.0;
            for (int e = 0; e < G->hp * G->wp * G->co; e++) dR[c][arg[c][e]] += dX[c + 1][e];
            for (int e = 0; e < nR; e++) if (!(R[c][e] > 0.0)) dR[c][e] = 0.0;  /* dY = dR .* [R > 0] */
            for (int kh = 0; kh < G->k; kh++)
                for (int kw = 0; kw < G->k; kw++)
                    for (int ci = 0; ci < G->ci; ci++)
                        for (int co = 0; co < G->co; co++) {
                            double acc = 0.0;
                            for (int oh = 0; oh < G->hc; oh++)
                                for (int ow = 0; ow < G->wc; ow++)
                                    acc += xin[c][((oh + kh) * G->wi + (ow + kw)) * G->ci + ci] *
                                           dR[c][(oh * G->wc + ow) * G->co + co];
                            dW[((kh * G->k + kw) * G->ci + ci) * G->co + co] += acc;
                        }
            for (int co = 0; co < G->co; co++) {
                double acc = 0.0;
                for (int e = 0; e < G->hc * G->wc; e++) acc += dR[c][e * G->co + co];
                db[co] += acc;
            }
            if (c > 0) {
                /* dX of a conv input that is a pool output; the previous layer routes it. */
                double *dx = dX[c];
                for (int h = 0; h < G->hi; h++)
                    for (int w = 0; w < G->wi; w++)
                        for (int ci = 0; ci < G->ci; ci++) {
                            double acc = 0.0;
                            for (int kh = 0; kh < G->k; kh++)
                                for (int kw = 0; kw < G->k; kw++) {
                                    int oh = h - kh, ow = w - kw;
                                    if (oh < 0 || ow < 0 || oh >= G->hc || ow >= G->wc) continue;
                                    for (int co = 0; co < G->co; co++)
                                        acc += dR[c][(oh * G->wc + ow) * G->co + co] *
                                               W[((kh * G->k + kw) * G->ci + ci) * G->co + co];
                                }
                            dx[(h * G->wi + w) * G->ci + ci] = acc;
                        }
            }
        }
    }
    free(xin[0]);
    for (int c = 0; c < NC; c++) { free(R[c]); free(dR[c]); free(Pl[c]); free(arg[c]); free(dX[c + 1]); }
    for (int f = 0; f <= NF; f++) { free(Af[f]); free(dAf[f]); }
    return loss_sum;
}

/* Local gradient for rank `rank` of P at `step` (O5-O7).  Returns loss sum. */
double orc_local_grad(const orc_net *m, const double *params, const float *X, const int32_t *y, int64_t n,
                      int64_t B, int64_t step, int32_t rank, int32_t P, double *grad) {
    if (m->kind == 0) return mlp_local(m, params, X, y, n, B, step, rank, P, 0, grad, 0, NULL, 0);
    return cnn_local(m, params, X, y, n, B, step, rank, P, 0, grad);
}

/* O5-O7 of the TF32 tier (tf32emu: SURVEY.md §8(c), readings A12/A23) on rank's shard; MLP only
 * (returns NaN for the CNN, whose convolutions are CUDA-core fp32). */
double orc_local_grad_tf32emu(const orc_net *m, const double *params, const float *X, const int32_t *y, int64_t n,
                              int64_t B, int64_t step, int32_t rank, int32_t P, double *grad) {
    if (m->kind != 0) return NAN;
    return mlp_local(m, params, X, y, n, B, step, rank, P, 0, grad, 0, NULL, 1);
}

/* tf32emu forward activations of layer l for an explicit batch. */
void orc_mlp_activations_tf32emu(const orc_net *m, const double *params, const float *X, const int32_t *y,
                                 int64_t b, int layer, double *out) {
    mlp_local(m, params, X, y, b, b, 0, 0, 1, b, NULL, layer, out, 1);
}

/* Same on an explicit batch of b rows X[0..b) (no sharding) -- used by FD checks. */
double orc_batch_grad(const orc_net *m, const double *params, const float *X, const int32_t *y, int64_t b,
                      double *grad) {
    if (m->kind == 0) return mlp_local(m, params, X, y, b, b, 0, 0, 1, b, grad, 0, NULL, 0);
    return cnn_local(m, params, X, y, b, b, 0, 0, 1, b, grad);
}

/* MLP forward activations of layer l for an explicit batch (S:93 worked value). */
void orc_mlp_activations(const orc_net *m, const double *params, const float *X, const int32_t *y, int64_t b,
                         int layer, double *out) {
    mlp_local(m, params, X, y, b, b, 0, 0, 1, b, NULL, layer, out, 0);
}

/* ------------------------------------------------------------------ O9 reduce (A2)
 * G = (((g_0 + g_1) + g_2) + ...) + g_{P-1}: ascending-rank left fold, the
 * allreduce-sum of P:182-184, P:298-306 ("MPI_Allreduce ... averaging gradients"). */
void orc_fold_f64(int32_t P, int64_t N, const double *g, double *G) {
    for (int64_t e = 0; e < N; e++) {
        double s = g[e];
        for (int r = 1; r < P; r++) s = s + g[(int64_t)r * N + e];
        G[e] = s;
    }
}

void orc_fold_f32(int32_t P, int64_t N, const float *g, float *G) {
    for (int64_t e = 0; e < N; e++) {
        float s = g[e];
        for (int r = 1; r < P; r++) s = s + g[(int64_t)r * N + e];
        G[e] = s;
    }
}

/* ------------------------------------------------------------------ O10-O11 average + update
 * gbar = G * fl(1/P) (A3); v <- fma(mu, v, gbar); w <- fma(-lr, v, w) (A4):
 * TF MomentumOptimizer form v = mu v + g, w = w - lr v ("Momentum");
 * plain SGD for mu = 0.  Returns the number of non-finite gbar entries (A17). */
int64_t orc_avg_update_f64(int64_t N, int32_t P, double lr, double mu, const double *G, double *w, double *v) {
    const double invP = 1.0 / (double)P;
    int64_t bad = 0;
    for (int64_t e = 0; e < N; e++) {
        double gbar = G[e] * invP;
        if (!isfinite(gbar)) bad++;
        v[e] = fma(mu, v[e], gbar);
        w[e] = fma(-lr, v[e], w[e]);
    }
    return bad;
}

int64_t orc_avg_update_f32(int64_t N, int32_t P, float lr, float mu, const float *G, float *w, float *v) {
    const float invP = 1.0f / (float)P;
    int64_t bad = 0;
    for (int64_t e = 0; e < N; e++) {
        float gbar = G[e] * invP;
        if (!isfinite(gbar)) bad++;
        v[e] = fmaf(mu, v[e], gbar);
        w[e] = fmaf(-lr, v[e], w[e]);
    }
    return bad;
}
