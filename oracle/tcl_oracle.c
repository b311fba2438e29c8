/*
 * tcl_oracle.c -- plain, slow, obviously-correct fp64 CPU oracle of TCL's Mamba cost model.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2604_12891_b200/) never links, imports or calls it, and shares no code,
 * header or constant with it.
 *
 * Citations: "P:n" = PAPER.md line n (section given); "S:n" = SPEC.md line n;
 * "Rk" = reading k of SURVEY.md §8(c) / DESIGN.md §3.
 *
 * Everything is computed in double precision from the fp32 weight blob and fp32 features
 * (promoted on read).  No blocking, no fusion, no SIMD, no BLAS: every loop is the formula.
 *
 * Forward pass of one candidate (§5.2 "Model Architecture"):
 *   encoder  : three linears with output widths enc_dims (64,128,128 in the paper),
 *              SiLU after the first two (R1)
 *   per layer: h <- h + Mixer(LN_l(h))   (R3; pre-norm residual Mamba block)
 *              Mixer = in_proj -> causal depthwise conv1d (d_conv taps) -> SiLU (R4)
 *                      -> x_proj [dt_r | B | C] -> Delta = softplus(dt_proj(dt_r) + b_dt) (R7)
 *                      -> selective scan with ZOH discretisation (Eqs. 4-5, R5, R6)
 *                      -> D-skip -> gate y * SiLU(z) -> out_proj
 *   final    : LN_f ("normalized again"), masked mean over the T real tokens (R9),
 *              decoder three linears 64,32,1 with SiLU after the first two (R1).
 *
 * Parity-pin status of each function: see the header of tests/test_oracle_pins.py and
 * DESIGN.md §4.  Absolute agreement with the paper's trained model is "parity unpinned"
 * (no weights were released); the pins fix every step's arithmetic instead.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* Same field order as tcl_dims in include/tcl.h (an interface, declared independently). */
typedef struct {
    int32_t d_in, max_len, d_model, n_layer, d_state, d_conv, expand, dt_rank;
    int32_t enc_dims[3];
    int32_t dec_dims[3];
    float ln_eps;
    float dropout_p;
    int32_t precision, disc;
} tclo_dims;

enum { TCLO_DISC_ZOH = 0, TCLO_DISC_EULER_B = 1 };

/* ------------------------------------------------------------------ elementary functions */

/* SiLU(v) = v * sigmoid(v) = v / (1 + e^{-v})  (R1; Mamba's activation) */
double tclo_silu(double v) { return v / (1.0 + exp(-v)); }

/* softplus(v) = log(1 + e^v) (R13).  For v > 0 the algebraically identical
 * v + log1p(e^{-v}) is used so that e^v cannot overflow. */
double tclo_softplus(double v) {
    if (v > 0.0) return v + log1p(exp(-v));
    return log1p(exp(v));
}

/* y = W x + b, W row-major [out][in] (PyTorch nn.Linear layout). b may be NULL. */
static void linear(const float* W, const float* b, int out, int in, const double* x, double* y) {
    for (int o = 0; o < out; ++o) {
        double acc = b ? (double)b[o] : 0.0;
        for (int i = 0; i < in; ++i) acc += (double)W[(size_t)o * in + i] * x[i];
        y[o] = acc;
    }
}

/* LayerNorm over one row of width d (R2): (x - mean) / sqrt(var + eps) * g + b, biased var. */
void tclo_layernorm_row(const double* x, int d, const float* g, const float* b, double eps,
                        double* y) {
    double mean = 0.0;
    for (int i = 0; i < d; ++i) mean += x[i];
    mean /= d;
    double var = 0.0;
    for (int i = 0; i < d; ++i) var += (x[i] - mean) * (x[i] - mean);
    var /= d;
    double rstd = 1.0 / sqrt(var + eps);
    for (int i = 0; i < d; ++i) {
        double v = (x[i] - mean) * rstd;
        y[i] = g ? v * (double)g[i] + (double)b[i] : v;
    }
}

/* Causal depthwise conv1d + SiLU over one candidate ("lightweight depthwise
 * one-dimensional convolution"; R4 conv then SiLU):
 *   c[t][d] = SiLU( b[d] + sum_{k<dc} w[d][k] * x[t-(dc-1)+k][d] ),  x[t'<0] = 0.
 * x, c: [T][di] row-major; w: [di][dc]; tap dc-1 multiplies the current token. */
void tclo_causal_conv_silu(const double* x, int T, int di, int dc, const float* w,
                           const float* b, double* c) {
    for (int t = 0; t < T; ++t)
        for (int d = 0; d < di; ++d) {
            double acc = b ? (double)b[d] : 0.0;
            for (int k = 0; k < dc; ++k) {
                int ts = t - (dc - 1) + k;
                if (ts >= 0) acc += (double)w[(size_t)d * dc + k] * x[(size_t)ts * di + d];
            }
            c[(size_t)t * di + d] = tclo_silu(acc);
        }
}

/* Selective scan over one candidate (Eqs. 4-5 discretised; R5, R6):
 *   s_{-1} = 0;  for t < T, d < di, n < N:
 *     Abar = exp(delta[t][d] * A[d][n])
 *     Bbar = (exp(delta*A) - 1) / A * B[t][n]      (ZOH, default)  |  delta * B[t][n]  (Euler-B)
 *     s[d][n] = Abar * s[d][n] + Bbar * u[t][d]
 *   y[t][d] = sum_n C[t][n] * s[d][n] + Dv[d] * u[t][d]
 * u, delta, y: [T][di]; B, C: [T][N]; A: [di][N] (strictly negative); Dv: [di].
 * (e^{x}-1) is evaluated with expm1, i.e. exactly the definition without cancellation. */
void tclo_ssm_scan(int T, int di, int N, const double* u, const double* delta,
                   const double* A, const double* B, const double* C, const double* Dv,
                   int disc, double* y) {
    double* s = (double*)calloc((size_t)di * N, sizeof(double));
    for (int t = 0; t < T; ++t) {
        for (int d = 0; d < di; ++d) {
            double dt = delta[(size_t)t * di + d];
            double ut = u[(size_t)t * di + d];
            double acc = 0.0;
            for (int n = 0; n < N; ++n) {
                double a = A[(size_t)d * N + n];
                double Abar = exp(dt * a);
                double Bbar = (disc == TCLO_DISC_EULER_B) ? dt * B[(size_t)t * N + n]
                                                          : expm1(dt * a) / a * B[(size_t)t * N + n];
                s[(size_t)d * N + n] = Abar * s[(size_t)d * N + n] + Bbar * ut;
                acc += C[(size_t)t * N + n] * s[(size_t)d * N + n];
            }
            y[(size_t)t * di + d] = acc + Dv[d] * ut;
        }
    }
    free(s);
}

/* ------------------------------------------------------------------ Philox4x32-10 (R17) */
/* Salmon et al. 2011 ("Parallel random numbers: as easy as 1, 2, 3"), the Random123
 * Philox4x32 with 10 rounds: multipliers 0xD2511F53, 0xCD9E8D57; Weyl key increments
 * 0x9E3779B9, 0xBB67AE85.  Pinned by the published known-answer vectors (tests). */
void tclo_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int r = 0; r < 10; ++r) {
        uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* Inverted-dropout multiplier for hidden unit `unit` of `site` (R17):
 *   counter = (unit>>2, token<<2 | site, pass, global index), key = (seed lo, seed hi);
 *   keep iff word[unit & 3] >= floor(p * 2^32); kept units are scaled by 1/(1-p). */
static double dropout_mult(uint64_t seed, double p, uint32_t thr, int unit, int token, int site,
                           int pass, int64_t gidx) {
    uint32_t ctr[4] = {(uint32_t)unit >> 2, ((uint32_t)token << 2) | (uint32_t)site,
                       (uint32_t)pass, (uint32_t)gidx};
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint32_t w[4];
    tclo_philox4x32_10(ctr, key, w);
    return (w[unit & 3] >= thr) ? 1.0 / (1.0 - p) : 0.0;
}

/* ------------------------------------------------------------------ weight blob */
typedef struct {
    const float *W1, *b1, *W2, *b2, *W3, *b3;
} mlp_w;
typedef struct {
    const float *ln_w, *ln_b, *W_in, *w_conv, *b_conv, *W_x, *W_dt, *b_dt, *A_log, *Dv, *W_out;
} layer_w;

/* Canonical order of SURVEY §8(b); returns number of floats consumed. */
static int64_t parse_blob(const tclo_dims* d, const float* w, mlp_w* enc, layer_w* L, const float** lnf_w,
                          const float** lnf_b, mlp_w* dec) {
    const int dm = d->d_model, di = d->expand * d->d_model, N = d->d_state, R = d->dt_rank;
    const float* p = w;
#define TAKE(dst, cnt) do { dst = p; p += (cnt); } while (0)
    TAKE(enc->W1, (int64_t)d->enc_dims[0] * d->d_in); TAKE(enc->b1, d->enc_dims[0]);
    TAKE(enc->W2, (int64_t)d->enc_dims[1] * d->enc_dims[0]); TAKE(enc->b2, d->enc_dims[1]);
    TAKE(enc->W3, (int64_t)d->enc_dims[2] * d->enc_dims[1]); TAKE(enc->b3, d->enc_dims[2]);
    for (int l = 0; l < d->n_layer; ++l) {
        layer_w* q = L ? &L[l] : NULL;
        layer_w dummy;
        if (!q) q = &dummy;
        TAKE(q->ln_w, dm); TAKE(q->ln_b, dm);
        TAKE(q->W_in, (int64_t)2 * di * dm);
        TAKE(q->w_conv, (int64_t)di * d->d_conv); TAKE(q->b_conv, di);
        TAKE(q->W_x, (int64_t)(R + 2 * N) * di);
        TAKE(q->W_dt, (int64_t)di * R); TAKE(q->b_dt, di);
        TAKE(q->A_log, (int64_t)di * N); TAKE(q->Dv, di);
        TAKE(q->W_out, (int64_t)dm * di);
    }
    TAKE(*lnf_w, dm); TAKE(*lnf_b, dm);
    TAKE(dec->W1, (int64_t)d->dec_dims[0] * dm); TAKE(dec->b1, d->dec_dims[0]);
    TAKE(dec->W2, (int64_t)d->dec_dims[1] * d->dec_dims[0]); TAKE(dec->b2, d->dec_dims[1]);
    TAKE(dec->W3, (int64_t)d->dec_dims[2] * d->dec_dims[1]); TAKE(dec->b3, d->dec_dims[2]);
#undef TAKE
    return (int64_t)(p - w);
}

/* Number of fp32 weights in the canonical blob: the sizes parse_blob walks, summed. */
int64_t tclo_weights_count(const tclo_dims* d) {
    const int64_t dm = d->d_model, di = (int64_t)d->expand * d->d_model, N = d->d_state,
                  R = d->dt_rank, din = d->d_in;
    int64_t enc = d->enc_dims[0] * din + d->enc_dims[0] + (int64_t)d->enc_dims[1] * d->enc_dims[0] +
                  d->enc_dims[1] + (int64_t)d->enc_dims[2] * d->enc_dims[1] + d->enc_dims[2];
    int64_t layer = 2 * dm + 2 * di * dm + di * d->d_conv + di + (R + 2 * N) * di + di * R + di +
                    di * N + di + dm * di;
    int64_t dec = d->dec_dims[0] * dm + d->dec_dims[0] + (int64_t)d->dec_dims[1] * d->dec_dims[0] +
                  d->dec_dims[1] + (int64_t)d->dec_dims[2] * d->dec_dims[1] + d->dec_dims[2];
    return enc + d->n_layer * layer + 2 * dm + dec;
}

static int dims_ok(const tclo_dims* d) {
    if (d->d_in < 1 || d->max_len < 1 || d->d_model < 1 || d->n_layer < 0 || d->d_state < 1 ||
        d->d_conv < 1 || d->expand < 1 || d->dt_rank < 1) return 0;
    if (d->enc_dims[2] != d->d_model || d->dec_dims[2] != 1) return 0;
    for (int i = 0; i < 3; ++i) if (d->enc_dims[i] < 1 || d->dec_dims[i] < 1) return 0;
    return 1;
}

/* ------------------------------------------------------------------ forward, one candidate */
/* Dump layout (doubles), written when dump != NULL (per-stage parity checks):
 *   h_enc [T][dm]
 *   per layer l: a [T][dm], x [T][di], z [T][di], u [T][di], dtr [T][R], B [T][N], C [T][N],
 *                delta [T][di], y [T][di], g [T][di], h [T][dm]
 *   pooled [dm], dec_h1 [h1], dec_h2 [h2]
 * Dropout (MC mode) is applied when mc_pass >= 0. */
typedef struct {
    int mc_pass;          /* -1: deterministic forward */
    uint64_t seed;
    int64_t gidx;
} mc_ctx;

/* ---- KB + AC two-column model (§6 Eq. 7; reading R23).
 * The AC's layer i output is h_i = act(W_i h_{i-1} + alpha_i (.) U_i SiLU(V_i h^KB_{i-1} + c_i) + b_i)
 * at every encoder linear, after every Mamba block (act = identity: the lateral joins the
 * residual stream) and at the two hidden decoder layers; h^KB_{i-1} is the KB's input to its own
 * layer i (the features for encoder layer 1).  The KB runs first, deterministic (frozen); its
 * site inputs are recorded and read by the AC column.  Adapter blob, per site in the order
 * enc1, enc2, enc3, layer 0..n_layer-1, dec1, dec2: V [a][in], c [a], U [out][a], alpha [out]. */
typedef struct {
    double *e1, *e2, *hin, *pooled, *dh1;   /* KB site inputs: [T][e1], [T][e2], [n_layer][T][dm], [dm], [h1] */
} kb_rec;
typedef struct {
    const float *V, *c, *U, *alpha;
    int in, out;
} adapter_w;
typedef struct {
    const kb_rec* kb;
    const adapter_w* ad;   /* sites: 0..2 encoder, 3..3+n_layer-1 Mamba blocks, then dec1, dec2 */
    int a;
} lateral_ctx;

/* y[o] += alpha[o] * sum_j U[o][j] SiLU(sum_i V[j][i] hkb[i] + c[j])   (the Eq. 7 lateral term) */
static void lateral_add(const adapter_w* A, int a, const double* hkb, double* y) {
    double* sj = (double*)calloc((size_t)a, sizeof(double));
    for (int j = 0; j < a; ++j) {
        double v = (double)A->c[j];
        for (int i = 0; i < A->in; ++i) v += (double)A->V[(size_t)j * A->in + i] * hkb[i];
        sj[j] = tclo_silu(v);
    }
    for (int o = 0; o < A->out; ++o) {
        double u = 0.0;
        for (int j = 0; j < a; ++j) u += (double)A->U[(size_t)o * a + j] * sj[j];
        y[o] += (double)A->alpha[o] * u;
    }
    free(sj);
}

static int adapter_sites(const tclo_dims* d, int a, const float* blob, adapter_w* out, int64_t* count) {
    const int ins[3] = {d->d_in, d->enc_dims[0], d->enc_dims[1]};
    const int outs[3] = {d->enc_dims[0], d->enc_dims[1], d->d_model};
    const int nsite = 3 + d->n_layer + 2;
    int64_t off = 0;
    for (int s = 0; s < nsite; ++s) {
        int in, o;
        if (s < 3) { in = ins[s]; o = outs[s]; }
        else if (s < 3 + d->n_layer) { in = d->d_model; o = d->d_model; }
        else if (s == 3 + d->n_layer) { in = d->d_model; o = d->dec_dims[0]; }
        else { in = d->dec_dims[0]; o = d->dec_dims[1]; }
        if (out) {
            out[s].in = in; out[s].out = o;
            out[s].V = blob + off;
            out[s].c = blob + off + (int64_t)a * in;
            out[s].U = blob + off + (int64_t)a * in + a;
            out[s].alpha = blob + off + (int64_t)a * in + a + (int64_t)o * a;
        }
        off += (int64_t)a * in + a + (int64_t)o * a + o;
    }
    if (count) *count = off;
    return nsite;
}

int64_t tclo_adapters_count(const tclo_dims* d, int a) {
    int64_t c = 0;
    adapter_sites(d, a, NULL, NULL, &c);
    return c;
}

static double forward_one(const tclo_dims* d, const float* wblob, const float* x_in, int T,
                          const mc_ctx* mc, double* dump, kb_rec* rec, const lateral_ctx* lat) {
    const int dm = d->d_model, di = d->expand * d->d_model, N = d->d_state, R = d->dt_rank;
    const int e1 = d->enc_dims[0], e2 = d->enc_dims[1];
    const int h1 = d->dec_dims[0], h2 = d->dec_dims[1];
    const double eps = (double)d->ln_eps;
    const double p = (double)d->dropout_p;
    const uint32_t thr = (uint32_t)floor(p * 4294967296.0);
    mlp_w enc, dec;
    const float *lnf_w, *lnf_b;
    layer_w* L = (layer_w*)calloc((size_t)(d->n_layer > 0 ? d->n_layer : 1), sizeof(layer_w));
    parse_blob(d, wblob, &enc, L, &lnf_w, &lnf_b, &dec);

    double* h = (double*)calloc((size_t)T * dm, sizeof(double));
    double* xin = (double*)calloc((size_t)d->d_in, sizeof(double));
    double* t1 = (double*)calloc((size_t)(e1 > h1 ? e1 : h1) + 1, sizeof(double));
    double* t2 = (double*)calloc((size_t)(e2 > h2 ? e2 : h2) + 1, sizeof(double));
    double* dp = dump;

    /* encoder */
    for (int t = 0; t < T; ++t) {
        for (int i = 0; i < d->d_in; ++i) xin[i] = (double)x_in[(size_t)t * d->d_in + i];
        linear(enc.W1, enc.b1, e1, d->d_in, xin, t1);
        if (lat) lateral_add(&lat->ad[0], lat->a, xin, t1);                 /* h^KB_0 = the features */
        for (int i = 0; i < e1; ++i) {
            t1[i] = tclo_silu(t1[i]);
            if (mc && mc->mc_pass >= 0) t1[i] *= dropout_mult(mc->seed, p, thr, i, t, 0, mc->mc_pass, mc->gidx);
        }
        if (rec) memcpy(&rec->e1[(size_t)t * e1], t1, sizeof(double) * e1);
        linear(enc.W2, enc.b2, e2, e1, t1, t2);
        if (lat) lateral_add(&lat->ad[1], lat->a, &lat->kb->e1[(size_t)t * e1], t2);
        for (int i = 0; i < e2; ++i) {
            t2[i] = tclo_silu(t2[i]);
            if (mc && mc->mc_pass >= 0) t2[i] *= dropout_mult(mc->seed, p, thr, i, t, 1, mc->mc_pass, mc->gidx);
        }
        if (rec) memcpy(&rec->e2[(size_t)t * e2], t2, sizeof(double) * e2);
        linear(enc.W3, enc.b3, dm, e2, t2, &h[(size_t)t * dm]);
        if (lat) lateral_add(&lat->ad[2], lat->a, &lat->kb->e2[(size_t)t * e2], &h[(size_t)t * dm]);
    }
    if (dp) { memcpy(dp, h, sizeof(double) * T * dm); dp += (size_t)T * dm; }

    double* a = (double*)calloc((size_t)T * dm, sizeof(double));
    double* xz = (double*)calloc((size_t)2 * di, sizeof(double));
    double* x = (double*)calloc((size_t)T * di, sizeof(double));
    double* z = (double*)calloc((size_t)T * di, sizeof(double));
    double* u = (double*)calloc((size_t)T * di, sizeof(double));
    double* dbc = (double*)calloc((size_t)(R + 2 * N), sizeof(double));
    double* dtr = (double*)calloc((size_t)T * R, sizeof(double));
    double* Bm = (double*)calloc((size_t)T * N, sizeof(double));
    double* Cm = (double*)calloc((size_t)T * N, sizeof(double));
    double* delta = (double*)calloc((size_t)T * di, sizeof(double));
    double* A = (double*)calloc((size_t)di * N, sizeof(double));
    double* Dv = (double*)calloc((size_t)di, sizeof(double));
    double* y = (double*)calloc((size_t)T * di, sizeof(double));
    double* g = (double*)calloc((size_t)T * di, sizeof(double));
    double* o = (double*)calloc((size_t)dm, sizeof(double));

    for (int l = 0; l < d->n_layer; ++l) {
        const layer_w* q = &L[l];
        if (rec) memcpy(&rec->hin[(size_t)l * T * dm], h, sizeof(double) * (size_t)T * dm);
        /* pre-norm (R2, R3) and in_proj */
        for (int t = 0; t < T; ++t) {
            tclo_layernorm_row(&h[(size_t)t * dm], dm, q->ln_w, q->ln_b, eps, &a[(size_t)t * dm]);
            linear(q->W_in, NULL, 2 * di, dm, &a[(size_t)t * dm], xz);
            for (int i = 0; i < di; ++i) { x[(size_t)t * di + i] = xz[i]; z[(size_t)t * di + i] = xz[di + i]; }
        }
        /* causal depthwise conv + SiLU (R4) */
        tclo_causal_conv_silu(x, T, di, d->d_conv, q->w_conv, q->b_conv, u);
        /* selection: x_proj -> [dt_r | B | C]; Delta = softplus(W_dt dt_r + b_dt) (R7) */
        for (int t = 0; t < T; ++t) {
            linear(q->W_x, NULL, R + 2 * N, di, &u[(size_t)t * di], dbc);
            for (int r = 0; r < R; ++r) dtr[(size_t)t * R + r] = dbc[r];
            for (int n = 0; n < N; ++n) { Bm[(size_t)t * N + n] = dbc[R + n]; Cm[(size_t)t * N + n] = dbc[R + N + n]; }
            linear(q->W_dt, q->b_dt, di, R, &dtr[(size_t)t * R], &delta[(size_t)t * di]);
            for (int i = 0; i < di; ++i) delta[(size_t)t * di + i] = tclo_softplus(delta[(size_t)t * di + i]);
        }
        /* A = -exp(A_log) (R8) */
        for (int i = 0; i < di * N; ++i) A[i] = -exp((double)q->A_log[i]);
        for (int i = 0; i < di; ++i) Dv[i] = (double)q->Dv[i];
        tclo_ssm_scan(T, di, N, u, delta, A, Bm, Cm, Dv, d->disc, y);
        /* gate y * SiLU(z); out_proj; residual */
        for (int t = 0; t < T; ++t) {
            for (int i = 0; i < di; ++i) g[(size_t)t * di + i] = y[(size_t)t * di + i] * tclo_silu(z[(size_t)t * di + i]);
            linear(q->W_out, NULL, dm, di, &g[(size_t)t * di], o);
            for (int i = 0; i < dm; ++i) h[(size_t)t * dm + i] += o[i];
            /* Eq. 7 at the Mamba-block output (identity activation: joins the residual stream) */
            if (lat) lateral_add(&lat->ad[3 + l], lat->a, &lat->kb->hin[((size_t)l * T + t) * dm], &h[(size_t)t * dm]);
        }
        if (dp) {
#define DUMP(src, cnt) do { memcpy(dp, src, sizeof(double) * (size_t)(cnt)); dp += (cnt); } while (0)
            DUMP(a, (size_t)T * dm); DUMP(x, (size_t)T * di); DUMP(z, (size_t)T * di); DUMP(u, (size_t)T * di);
            DUMP(dtr, (size_t)T * R); DUMP(Bm, (size_t)T * N); DUMP(Cm, (size_t)T * N);
            DUMP(delta, (size_t)T * di); DUMP(y, (size_t)T * di); DUMP(g, (size_t)T * di); DUMP(h, (size_t)T * dm);
        }
    }

    /* final norm, masked mean over the T real tokens (R9), decoder */
    double* pooled = (double*)calloc((size_t)dm, sizeof(double));
    double* f = (double*)calloc((size_t)dm, sizeof(double));
    for (int t = 0; t < T; ++t) {
        tclo_layernorm_row(&h[(size_t)t * dm], dm, lnf_w, lnf_b, eps, f);
        for (int i = 0; i < dm; ++i) pooled[i] += f[i];
    }
    for (int i = 0; i < dm; ++i) pooled[i] /= (double)T;
    if (rec) memcpy(rec->pooled, pooled, sizeof(double) * dm);
    linear(dec.W1, dec.b1, h1, dm, pooled, t1);
    if (lat) lateral_add(&lat->ad[3 + d->n_layer], lat->a, lat->kb->pooled, t1);
    for (int i = 0; i < h1; ++i) {
        t1[i] = tclo_silu(t1[i]);
        if (mc && mc->mc_pass >= 0) t1[i] *= dropout_mult(mc->seed, p, thr, i, 0, 2, mc->mc_pass, mc->gidx);
    }
    if (rec) memcpy(rec->dh1, t1, sizeof(double) * h1);
    linear(dec.W2, dec.b2, h2, h1, t1, t2);
    if (lat) lateral_add(&lat->ad[4 + d->n_layer], lat->a, lat->kb->dh1, t2);
    for (int i = 0; i < h2; ++i) {
        t2[i] = tclo_silu(t2[i]);
        if (mc && mc->mc_pass >= 0) t2[i] *= dropout_mult(mc->seed, p, thr, i, 0, 3, mc->mc_pass, mc->gidx);
    }
    double score;
    linear(dec.W3, dec.b3, 1, h2, t2, &score);
    if (dp) { DUMP(pooled, dm); DUMP(t1, h1); DUMP(t2, h2); }
#undef DUMP

    free(pooled); free(f); free(o); free(g); free(y); free(Dv); free(A); free(delta); free(Cm);
    free(Bm); free(dtr); free(dbc); free(u); free(z); free(x); free(xz); free(a); free(t2);
    free(t1); free(xin); free(h); free(L);
    return score;
}

/* Two-column forward (R23): the frozen KB column (deterministic, site inputs recorded), then the
 * AC column reading them through the lateral adapters; the AC's output is the score.  MC dropout
 * (when mc) applies to the AC column only. */
static double forward_kbac(const tclo_dims* d, const float* kb_w, const float* ac_w, const float* ad_w, int a,
                           const float* x_in, int T, const mc_ctx* mc) {
    const int dm = d->d_model;
    kb_rec rec;
    rec.e1 = (double*)calloc((size_t)T * d->enc_dims[0], sizeof(double));
    rec.e2 = (double*)calloc((size_t)T * d->enc_dims[1], sizeof(double));
    rec.hin = (double*)calloc((size_t)(d->n_layer > 0 ? d->n_layer : 1) * T * dm, sizeof(double));
    rec.pooled = (double*)calloc((size_t)dm, sizeof(double));
    rec.dh1 = (double*)calloc((size_t)d->dec_dims[0], sizeof(double));
    adapter_w* ad = (adapter_w*)calloc((size_t)(5 + d->n_layer), sizeof(adapter_w));
    adapter_sites(d, a, ad_w, ad, NULL);
    (void)forward_one(d, kb_w, x_in, T, NULL, NULL, &rec, NULL);
    lateral_ctx lat = {&rec, ad, a};
    double score = forward_one(d, ac_w, x_in, T, mc, NULL, NULL, &lat);
    free(ad); free(rec.dh1); free(rec.pooled); free(rec.hin); free(rec.e2); free(rec.e1);
    return score;
}

/* Size of the dump of forward_one, in doubles. */
int64_t tclo_dump_size(const tclo_dims* d, int T) {
    const int64_t dm = d->d_model, di = (int64_t)d->expand * d->d_model, N = d->d_state, R = d->dt_rank;
    /* a, x, z, u, dtr, B, C, delta, y, g, h */
    int64_t per_layer = T * dm + 3 * T * di + T * R + 2 * T * N + 3 * T * di + T * dm;
    return T * dm + d->n_layer * per_layer + dm + d->dec_dims[0] + d->dec_dims[1];
}

/* One candidate with the per-stage dump (dump may be NULL). Returns 0 on success. */
int tclo_forward_one(const tclo_dims* d, const float* w, const float* feats_one, int T, double* dump,
                     double* score) {
    if (!dims_ok(d) || T < 1 || T > d->max_len) return -1;
    *score = forward_one(d, w, feats_one, T, NULL, dump, NULL, NULL);
    return 0;
}

/* ------------------------------------------------------------------ batched, threaded */
typedef struct {
    const tclo_dims* d;
    const float* w;
    const float* feats;
    const int32_t* lens;
    int64_t n, begin, step;
    int mc_passes;
    uint64_t seed;
    int64_t index_base;
    double* scores;   /* deterministic mode */
    double* mean;     /* MC mode */
    double* var;
    const float* kb_w;   /* non-NULL: KB + AC two-column model; w is the AC column */
    const float* ad_w;
    int ad_rank;
    int one_pass;        /* >= 0: scores[i] = the score of dropout pass `one_pass` alone */
} job_t;

static void* worker(void* arg) {
    job_t* j = (job_t*)arg;
    const size_t stride = (size_t)j->d->max_len * j->d->d_in;
    for (int64_t i = j->begin; i < j->n; i += j->step) {
        int T = j->lens[i];
        const float* xf = j->feats + (size_t)i * stride;
        if (T < 1 || T > j->d->max_len) {  /* R16: invalid length -> NaN score */
            if (j->scores) j->scores[i] = NAN;
            if (j->mean) { j->mean[i] = NAN; j->var[i] = NAN; }
            continue;
        }
        if (j->one_pass >= 0) {   /* one dropout pass (pins the MC reduction from outside) */
            mc_ctx mc = {j->one_pass, j->seed, j->index_base + i};
            j->scores[i] = forward_one(j->d, j->w, xf, T, &mc, NULL, NULL, NULL);
        } else if (j->mc_passes <= 0) {
            j->scores[i] = j->kb_w ? forward_kbac(j->d, j->kb_w, j->w, j->ad_w, j->ad_rank, xf, T, NULL)
                                   : forward_one(j->d, j->w, xf, T, NULL, NULL, NULL, NULL);
        } else {
            /* Welford over passes; population variance (divide by the number of passes) (R17) */
            double m = 0.0, M2 = 0.0;
            for (int ps = 0; ps < j->mc_passes; ++ps) {
                mc_ctx mc = {ps, j->seed, j->index_base + i};
                double v = j->kb_w ? forward_kbac(j->d, j->kb_w, j->w, j->ad_w, j->ad_rank, xf, T, &mc)
                                   : forward_one(j->d, j->w, xf, T, &mc, NULL, NULL, NULL);
                double delta = v - m;
                m += delta / (double)(ps + 1);
                M2 += delta * (v - m);
            }
            j->mean[i] = m;
            j->var[i] = M2 / (double)j->mc_passes;
        }
    }
    return NULL;
}

static int run_threads(job_t* proto, int nthreads) {
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    pthread_t th[256];
    job_t jobs[256];
    for (int k = 0; k < nthreads; ++k) {
        jobs[k] = *proto;
        jobs[k].begin = k;
        jobs[k].step = nthreads;
        if (nthreads == 1) { worker(&jobs[0]); return 0; }
        pthread_create(&th[k], NULL, worker, &jobs[k]);
    }
    for (int k = 0; k < nthreads; ++k) pthread_join(th[k], NULL);
    return 0;
}

/* scores[i] for candidates i < n; feats [n][max_len][d_in] fp32; lens [n]. */
int tclo_score(const tclo_dims* d, const float* w, const float* feats, const int32_t* lens,
               int64_t n, double* scores, int nthreads) {
    if (!dims_ok(d) || n < 0) return -1;
    job_t j = {d, w, feats, lens, n, 0, 1, 0, 0, 0, scores, NULL, NULL, NULL, NULL, 0, -1};
    return run_threads(&j, nthreads);
}

/* KB + AC two-column scores (R23): kb_w, ac_w canonical blobs, ad_w the adapter blob of rank a. */
int tclo_score_kbac(const tclo_dims* d, const float* kb_w, const float* ac_w, const float* ad_w, int a,
                    const float* feats, const int32_t* lens, int64_t n, double* scores, int nthreads) {
    if (!dims_ok(d) || n < 0 || a < 1) return -1;
    job_t j = {d, ac_w, feats, lens, n, 0, 1, 0, 0, 0, scores, NULL, NULL, kb_w, ad_w, a, -1};
    return run_threads(&j, nthreads);
}

int tclo_score_mc_kbac(const tclo_dims* d, const float* kb_w, const float* ac_w, const float* ad_w, int a,
                       const float* feats, const int32_t* lens, int64_t n, int32_t n_passes, uint64_t seed,
                       int64_t index_base, double* mean, double* var, int nthreads) {
    if (!dims_ok(d) || n < 0 || n_passes < 1 || a < 1) return -1;
    job_t j = {d, ac_w, feats, lens, n, 0, 1, n_passes, seed, index_base, NULL, mean, var, kb_w, ad_w, a, -1};
    return run_threads(&j, nthreads);
}

/* MC-dropout (R17; north-star addition, absent from the paper): mean and population variance
 * of the score over n_passes dropout passes. */
int tclo_score_mc(const tclo_dims* d, const float* w, const float* feats, const int32_t* lens,
                  int64_t n, int32_t n_passes, uint64_t seed, int64_t index_base, double* mean,
                  double* var, int nthreads) {
    if (!dims_ok(d) || n < 0 || n_passes < 1) return -1;
    job_t j = {d, w, feats, lens, n, 0, 1, n_passes, seed, index_base, NULL, mean, var, NULL, NULL, 0, -1};
    return run_threads(&j, nthreads);
}

/* The score of ONE MC-dropout pass `pass` (the same masks tclo_score_mc draws for that pass): the
 * per-pass scores that tclo_score_mc reduces to (mean, population variance).  Used by the pins to
 * check that reduction against numpy's mean / var of these scores. */
int tclo_score_pass(const tclo_dims* d, const float* w, const float* feats, const int32_t* lens,
                    int64_t n, int32_t pass, uint64_t seed, int64_t index_base, double* scores, int nthreads) {
    if (!dims_ok(d) || n < 0 || pass < 0) return -1;
    job_t j = {d, w, feats, lens, n, 0, 1, 0, seed, index_base, scores, NULL, NULL, NULL, NULL, 0, pass};
    return run_threads(&j, nthreads);
}

/* ------------------------------------------------------------------ top-k (R15) */
/* The k best candidates under the total order (score desc, index asc), NaN treated as -inf.
 * Selection by repeated linear scans (obviously correct, O(n k)); k is clamped to n and the
 * slots >= n are filled with (idx -1, score -inf). */
static int better(double a, int64_t ia, double b, int64_t ib) {
    if (isnan(a)) a = -INFINITY;
    if (isnan(b)) b = -INFINITY;
    if (a != b) return a > b;
    return ia < ib;
}

int tclo_topk_f64(const double* scores, int64_t n, int32_t k, int64_t index_base, int64_t* idx,
                  double* top) {
    if (k <= 0 || n < 0) return -1;
    unsigned char* taken = (unsigned char*)calloc((size_t)(n > 0 ? n : 1), 1);
    for (int32_t r = 0; r < k; ++r) {
        int64_t best = -1;
        for (int64_t i = 0; i < n; ++i) {
            if (taken[i]) continue;
            if (best < 0 || better(scores[i], i, scores[best], best)) best = i;
        }
        if (best < 0) { idx[r] = -1; top[r] = -INFINITY; continue; }
        taken[best] = 1;
        idx[r] = index_base + best;
        top[r] = isnan(scores[best]) ? -INFINITY : scores[best];
    }
    free(taken);
    return 0;
}

int tclo_topk_f32(const float* scores, int64_t n, int32_t k, int64_t index_base, int64_t* idx,
                  float* top) {
    if (k <= 0 || n < 0) return -1;
    double* s = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    double* t = (double*)malloc(sizeof(double) * (size_t)k);
    for (int64_t i = 0; i < n; ++i) s[i] = (double)scores[i];
    int rc = tclo_topk_f64(s, n, k, index_base, idx, t);
    for (int32_t r = 0; r < k; ++r) top[r] = (float)t[r];
    free(s); free(t);
    return rc;
}

/* ------------------------------------------------------------------ RDU acquisition (NEXT #1) */
/* One selection round of PAPER.md Algorithm 1 (lines 16-31) with Eqs. 1-3 (§4), reading R21:
 *   f^ = (f - lo) / (hi - lo), lo/hi over pool u labeled predictions ("normalized");
 *        every f^ = 0.5 when hi == lo; non-finite predictions take no part anywhere (never picked,
 *        not counted in the labeled set), their operator still counts toward the budget shares
 *   d_s(i) = min_j |f^_i - f^_j| over the labeled set (Eq. 1); 1 when the labeled set is empty
 *   mu = (f^_i + S) r (Eq. 2); u_s = ((f^_i - mu)^2 + sum_j (f^_j - mu)^2) r (Eq. 3), r = 1/(M+1), with
 *        sum_j (f^_j - mu)^2 = Q - 2 mu S + M mu^2 (S = sum f^_j, Q = sum f^_j^2, running sums)
 *   t_s = f^_i d_s + u_s (line 24); pick argmax t_s, ties: higher f^, then lower index
 *   budget[op] = B_t * count(op) / n_pool (lines 16-19); an operator type whose selected count has
 *        reached its budget is skipped (lines 25-31); the pick joins D_l before the next pick.
 * Where floating point decides the integer pick, this follows the kernel's precision: the scores are
 * evaluated in fp32, one IEEE operation at a time in the order written above (the file is compiled
 * with -ffp-contract=off), and the labeled sums are accumulated sequentially in index order.
 * Returns the number of picks written to out_idx (<= budget_total). */
static float rdu_uncertainty(float fi, float S, float Q, float Mf) {   /* Eqs. 2-3 */
    float m1 = Mf + 1.0f;
    float r = 1.0f / m1;              /* 1/(M+1), once per pick (R21) */
    float mu = (fi + S) * r;
    float a = fi - mu;
    float a2 = a * a;
    float t1 = mu * S;
    float t2 = t1 + t1;
    float t3 = mu * mu;
    float t4 = Mf * t3;
    float b = (Q - t2) + t4;
    return (a2 + b) * r;
}

static float rdu_total_score(float fi, float ds, float S, float Q, float Mf) {   /* line 24 */
    float us = rdu_uncertainty(fi, S, Q, Mf);
    float t5 = fi * ds;
    return t5 + us;
}

/* Eqs. 1-3 + line 24 for already-normalised predictions (fh_pool, fh_lab): the per-candidate scores
 * of the first pick of a round.  Used by the pins (SPEC rdu examples, two-pass variance). */
void tclo_rdu_scores(const float* fh_pool, int64_t n_pool, const float* fh_lab, int64_t n_lab,
                     float* ds, float* us, float* ts) {
    float S = 0.0f, Q = 0.0f, Mf = 0.0f;
    for (int64_t j = 0; j < n_lab; ++j) {
        S = S + fh_lab[j];
        Q = Q + fh_lab[j] * fh_lab[j];
        Mf = Mf + 1.0f;
    }
    for (int64_t i = 0; i < n_pool; ++i) {
        float d = INFINITY;
        for (int64_t j = 0; j < n_lab; ++j) {
            float e = fabsf(fh_pool[i] - fh_lab[j]);
            if (e < d) d = e;
        }
        ds[i] = n_lab > 0 ? d : 1.0f;
        us[i] = rdu_uncertainty(fh_pool[i], S, Q, Mf);
        ts[i] = rdu_total_score(fh_pool[i], ds[i], S, Q, Mf);
    }
}

int64_t tclo_rdu_select(const float* pool, const int32_t* ops, int64_t n_pool, const float* lab,
                        int64_t n_lab, int32_t n_ops, int32_t budget_total, int64_t* out_idx) {
    if (n_pool <= 0 || budget_total <= 0 || n_ops < 1) return 0;
    float lo = INFINITY, hi = -INFINITY;
    for (int64_t i = 0; i < n_pool + n_lab; ++i) {
        float v = i < n_pool ? pool[i] : lab[i - n_pool];
        if (!isfinite(v)) continue;   /* only finite predictions take part (R21) */
        if (v < lo) lo = v;
        if (v > hi) hi = v;
    }
    int flat = !(hi > lo);
    float range = hi - lo;
#define NORM(v) (flat ? 0.5f : (((v) - lo) / range))
    int64_t* count = (int64_t*)calloc((size_t)n_ops, sizeof(int64_t));
    int64_t* sel = (int64_t*)calloc((size_t)n_ops, sizeof(int64_t));
    float* budget = (float*)malloc(sizeof(float) * (size_t)n_ops);
    for (int64_t i = 0; i < n_pool; ++i)
        if (ops[i] >= 0 && ops[i] < n_ops) count[ops[i]]++;
    for (int o = 0; o < n_ops; ++o) budget[o] = (float)((double)budget_total * (double)count[o] / (double)n_pool);
    float S = 0.0f, Q = 0.0f, Mf = 0.0f;
    for (int64_t j = 0; j < n_lab; ++j) {
        if (!isfinite(lab[j])) continue;
        float f = NORM(lab[j]);
        S = S + f;
        Q = Q + f * f;
        Mf = Mf + 1.0f;
    }
    float* fh = (float*)malloc(sizeof(float) * (size_t)n_pool);
    float* ds = (float*)malloc(sizeof(float) * (size_t)n_pool);
    unsigned char* alive = (unsigned char*)malloc((size_t)n_pool);
    for (int64_t i = 0; i < n_pool; ++i) {
        fh[i] = NORM(pool[i]);
        alive[i] = isfinite(pool[i]) && isfinite(fh[i]) && ops[i] >= 0 && ops[i] < n_ops;
        float d = INFINITY;
        for (int64_t j = 0; j < n_lab; ++j) {
            if (!isfinite(lab[j])) continue;
            float e = fabsf(fh[i] - NORM(lab[j]));
            if (e < d) d = e;
        }
        ds[i] = d == INFINITY ? 1.0f : d;   /* empty labeled set: maximal novelty 1 */
    }
    int64_t picks = 0;
    for (int32_t p = 0; p < budget_total; ++p) {
        int64_t best = -1;
        float bts = 0.0f, bf = 0.0f;
        for (int64_t i = 0; i < n_pool; ++i) {
            if (!alive[i] || !((float)sel[ops[i]] < budget[ops[i]])) continue;
            float ts = rdu_total_score(fh[i], ds[i], S, Q, Mf);
            if (best < 0 || ts > bts || (ts == bts && (fh[i] > bf || (fh[i] == bf && i < best)))) {
                best = i;
                bts = ts;
                bf = fh[i];
            }
        }
        if (best < 0) break;
        out_idx[picks++] = best;
        alive[best] = 0;
        sel[ops[best]]++;
        float fs = fh[best];
        S = S + fs;
        Q = Q + fs * fs;
        Mf = Mf + 1.0f;
        for (int64_t i = 0; i < n_pool; ++i) {
            float e = fabsf(fh[i] - fs);
            if (e < ds[i]) ds[i] = e;
        }
    }
#undef NORM
    free(count); free(sel); free(budget); free(fh); free(ds); free(alive);
    return picks;
}

/* ------------------------------------------------------------------ Top-k score (NEXT #4) */
/* PAPER.md Eq. 12 (§7.1.2), reading R22:
 *   Top-k = sum_{m,s} min_latency_{m,s} w_{m,s} / sum_{m,s} min_{i in [1,k]} p_latency_{m,s,i} w_{m,s}
 * Task t (one subgraph s of model m) holds candidates off[t] .. off[t+1]-1 with true latencies lat[]
 * and predicted scores scores[] (larger = better, R14); p_latency_{m,s,i} is the latency of the
 * i-th candidate ranked by predicted score (ties: lower index first, NaN = -inf: R15, the order
 * tclo_topk_f64 defines); k larger than the task clamps to the task size.
 * For each of the n_k values ks[j]: num[j], den[j] (fp64 sums in task order) and out[j] = num/den.
 * Returns 0, or -1 on bad arguments (a task with no candidates, k < 1). */
int tclo_topk_score(const float* scores, const float* lat, const int64_t* off, const float* w,
                    int64_t n_tasks, const int32_t* ks, int32_t n_k, double* out, double* num, double* den) {
    for (int32_t j = 0; j < n_k; ++j) {
        if (ks[j] < 1) return -1;
        num[j] = 0.0;
        den[j] = 0.0;
    }
    for (int64_t t = 0; t < n_tasks; ++t) {
        int64_t T = off[t + 1] - off[t];
        if (T < 1) return -1;
        double minlat = INFINITY;
        double* s = (double*)malloc(sizeof(double) * (size_t)T);
        for (int64_t i = 0; i < T; ++i) {
            s[i] = (double)scores[off[t] + i];
            if ((double)lat[off[t] + i] < minlat) minlat = (double)lat[off[t] + i];
        }
        for (int32_t j = 0; j < n_k; ++j) {
            int32_t k = ks[j] < T ? ks[j] : (int32_t)T;
            int64_t* idx = (int64_t*)malloc(sizeof(int64_t) * (size_t)k);
            double* top = (double*)malloc(sizeof(double) * (size_t)k);
            tclo_topk_f64(s, T, k, 0, idx, top);
            double pmin = INFINITY;
            for (int32_t r = 0; r < k; ++r)
                if ((double)lat[off[t] + idx[r]] < pmin) pmin = (double)lat[off[t] + idx[r]];
            num[j] += minlat * (double)w[t];
            den[j] += pmin * (double)w[t];
            free(idx);
            free(top);
        }
        free(s);
    }
    for (int32_t j = 0; j < n_k; ++j) out[j] = num[j] / den[j];
    return 0;
}
