/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU implementation, in double precision, of
 * the two batch-reduction operations TurboTransformers (arXiv 2010.05680)
 * optimises outside BLAS:
 *
 *   - ApplyMaskAndSoftmax  (PAPER.md l.765 kernel name; l.316 "Softmax
 *     calculates summation and maximum"; l.192 "the short sequence must be
 *     filled with zeros according to the longest sequence")
 *   - AddBiasLayerNorm     (l.316 "LayerNorm calculates the
 *     mean and variance"; Eq. 1 `seq:varience`, l.406-409)
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  The product path
 * (paper_2010_05680_b200/) never includes, links or calls anything here, and
 * this file includes nothing from it: the two share no code.
 *
 * Every loop below is the plain definition, evaluated left to right in double,
 * with no blocking, fusion or reordering.  Readings of the paper where it is
 * silent (mask value, masked axis, eps placement, ...) are DESIGN.md §3 R1-R14.
 *
 * dtype codes: 0 = fp32, 1 = fp16 (IEEE binary16), 2 = bf16 (bfloat16).
 * Storage-dtype inputs are widened EXACTLY to double by the hand-written bit
 * decoders below (no cuda_fp16.h, no compiler half type).
 *
 * Return value of every entry point: 0 ok, -1 bad argument.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define TTO_F32 0
#define TTO_F16 1
#define TTO_BF16 2

/* ---------------------------------------------------------------------------
 * Exact widening of one stored element to double.
 * fp16: 1 sign, 5 exponent (bias 15), 10 mantissa bits (IEEE 754 binary16).
 * bf16: the upper 16 bits of an IEEE binary32.
 * ------------------------------------------------------------------------- */
static double f32_bits_to_double(uint32_t u) {
    float f;
    memcpy(&f, &u, sizeof f);
    return (double)f;
}

static double f16_bits_to_double(uint16_t h) {
    int sign = (h >> 15) & 1;
    int exp = (h >> 10) & 0x1f;
    int man = h & 0x3ff;
    double v;
    if (exp == 0) {
        v = ldexp((double)man, -24); /* subnormal: man * 2^-14 * 2^-10 */
    } else if (exp == 31) {
        v = man ? NAN : INFINITY;
    } else {
        v = ldexp((double)(1024 + man), exp - 25); /* (1 + man/2^10) * 2^(exp-15) */
    }
    return sign ? -v : v;
}

static double bf16_bits_to_double(uint16_t b) {
    return f32_bits_to_double((uint32_t)b << 16);
}

static double load_elem(const void* base, int dtype, int64_t i) {
    if (dtype == TTO_F32) {
        uint32_t u;
        memcpy(&u, (const char*)base + 4 * i, 4);
        return f32_bits_to_double(u);
    } else {
        uint16_t h;
        memcpy(&h, (const char*)base + 2 * i, 2);
        return dtype == TTO_F16 ? f16_bits_to_double(h) : bf16_bits_to_double(h);
    }
}

/* Widen n stored elements to double (exposed so the tests can pin the
 * decoders exhaustively against an independent library). */
int tto_widen(const void* src, int dtype, int64_t n, double* dst) {
    if (n < 0 || (n > 0 && (!src || !dst)) || dtype < 0 || dtype > 2) return -1;
    for (int64_t i = 0; i < n; ++i) dst[i] = load_elem(src, dtype, i);
    return 0;
}

/* ---------------------------------------------------------------------------
 * Masked softmax (§4.1.2 l.315-317; masking l.192, l.576; DESIGN R1-R5)
 *
 * scores: [B, H, Sq, Sk] row-major, storage dtype `dtype`.
 * lengths: int32[B]; L_b = min(max(lengths[b], 0), Sk).
 * out: double [B, H, Sq, Sk].
 *
 *   z_j   = scale * x_j                       (j < L_b)
 *   m     = max_{j < L_b} z_j
 *   s     = sum_{j < L_b} exp(z_j - m)
 *   y_j   = exp(z_j - m) / s                  (j < L_b)
 *   y_j   = +0.0                              (L_b <= j < Sk, padding keys)
 *   L_b == 0: the whole row is +0.0
 * ------------------------------------------------------------------------- */
int tto_softmax_masked(const void* scores, int dtype, const int32_t* lengths,
                       int64_t B, int64_t H, int64_t Sq, int64_t Sk,
                       float scale, double* out) {
    if (B < 0 || H < 0 || Sq < 0 || Sk < 0 || dtype < 0 || dtype > 2) return -1;
    if (B * H * Sq * Sk == 0) return 0;
    if (!scores || !lengths || !out) return -1;
    const double sc = (double)scale;
    for (int64_t b = 0; b < B; ++b) {
        int64_t L = lengths[b];
        if (L < 0) L = 0;
        if (L > Sk) L = Sk;
        for (int64_t h = 0; h < H; ++h) {
            for (int64_t i = 0; i < Sq; ++i) {
                const int64_t row = ((b * H + h) * Sq + i) * Sk;
                double* y = out + row;
                if (L == 0) {
                    for (int64_t j = 0; j < Sk; ++j) y[j] = 0.0;
                    continue;
                }
                double m = -INFINITY;
                for (int64_t j = 0; j < L; ++j) {
                    double z = sc * load_elem(scores, dtype, row + j);
                    if (z > m) m = z;
                }
                double s = 0.0;
                for (int64_t j = 0; j < L; ++j) {
                    s += exp(sc * load_elem(scores, dtype, row + j) - m);
                }
                for (int64_t j = 0; j < L; ++j) {
                    y[j] = exp(sc * load_elem(scores, dtype, row + j) - m) / s;
                }
                for (int64_t j = L; j < Sk; ++j) y[j] = 0.0;
            }
        }
    }
    return 0;
}

/* ---------------------------------------------------------------------------
 * Fused add-bias + residual + LayerNorm (PAPER.md l.299-304 fusion rule,
 * l.765 `AddBiasLayerNorm`; Eq. 1 LHS, l.408; DESIGN R7-R10)
 *
 * x, residual: [rows, hidden]; bias, gamma, beta: [hidden]; all storage dtype.
 * out: double [rows, hidden].
 *
 *   v_k  = (x_k + bias_k) + residual_k
 *   mu   = (1/N) sum_k v_k
 *   var  = (1/N) sum_k (v_k - mu)^2          (population variance, Eq. 1 LHS)
 *   y_k  = (v_k - mu) / sqrt(var + eps) * gamma_k + beta_k
 * ------------------------------------------------------------------------- */
int tto_add_bias_layernorm(const void* x, const void* residual, const void* bias,
                           const void* gamma, const void* beta, int dtype,
                           int64_t rows, int64_t hidden, float eps, double* out) {
    if (rows < 0 || hidden < 0 || dtype < 0 || dtype > 2) return -1;
    if (rows * hidden == 0) return 0;
    if (!x || !residual || !bias || !gamma || !beta || !out) return -1;
    const double N = (double)hidden;
    const double e = (double)eps;
    for (int64_t r = 0; r < rows; ++r) {
        double* y = out + r * hidden;
        /* y doubles as the buffer for v */
        for (int64_t k = 0; k < hidden; ++k) {
            y[k] = (load_elem(x, dtype, r * hidden + k) + load_elem(bias, dtype, k)) +
                   load_elem(residual, dtype, r * hidden + k);
        }
        double sum = 0.0;
        for (int64_t k = 0; k < hidden; ++k) sum += y[k];
        const double mu = sum / N;
        double ss = 0.0;
        for (int64_t k = 0; k < hidden; ++k) ss += (y[k] - mu) * (y[k] - mu);
        const double var = ss / N;
        const double denom = sqrt(var + e);
        for (int64_t k = 0; k < hidden; ++k) {
            y[k] = (y[k] - mu) / denom * load_elem(gamma, dtype, k) + load_elem(beta, dtype, k);
        }
    }
    return 0;
}

/* ---------------------------------------------------------------------------
 * The paper's own one-pass LayerNorm (Eq. 1 RHS, l.408; "simultaneously reduce
 * x and x^2", l.404), in double, variance clamped at 0 (SPEC.md l.355
 * reading).  Kept so the tests can pin Eq. 1's identity against the two-pass
 * definition above; the GPU path does NOT use this formulation (DESIGN R9).
 * Plain LayerNorm: no bias, no residual.
 * ------------------------------------------------------------------------- */
int tto_layernorm_onepass_eq1(const void* x, const void* gamma, const void* beta,
                              int dtype, int64_t rows, int64_t hidden, float eps,
                              double* out) {
    if (rows < 0 || hidden < 0 || dtype < 0 || dtype > 2) return -1;
    if (rows * hidden == 0) return 0;
    if (!x || !gamma || !beta || !out) return -1;
    const double N = (double)hidden;
    for (int64_t r = 0; r < rows; ++r) {
        double s1 = 0.0, s2 = 0.0;
        for (int64_t k = 0; k < hidden; ++k) {
            double v = load_elem(x, dtype, r * hidden + k);
            s1 += v;
            s2 += v * v;
        }
        const double mu = s1 / N;
        double var = s2 / N - mu * mu;
        if (var < 0.0) var = 0.0;
        const double denom = sqrt(var + (double)eps);
        for (int64_t k = 0; k < hidden; ++k) {
            double v = load_elem(x, dtype, r * hidden + k);
            out[r * hidden + k] =
                (v - mu) / denom * load_elem(gamma, dtype, k) + load_elem(beta, dtype, k);
        }
    }
    return 0;
}

/* ---------------------------------------------------------------------------
 * NEXT-2: the element-wise non-GEMM kernels of the fused graph,
 * "fused activation functions and fused transpose operations" (PAPER.md
 * l.304-308; K4/K5 in SURVEY §2.2).
 * ------------------------------------------------------------------------- */

/* out[r, j] = gelu(x[r, j] + bias[j]) over [rows, n], double.
 * approximate = 0: exact GELU, v * Phi(v) = 0.5 v (1 + erf(v / sqrt 2))
 * approximate = 1: tanh form, 0.5 v (1 + tanh(sqrt(2/pi) (v + 0.044715 v^3)))
 * (BERT's definition is the exact form; the tanh form is PyTorch's
 * approximate='tanh'.  DESIGN R17.) */
int tto_add_bias_gelu(const void* x, const void* bias, int dtype, int64_t rows, int64_t n,
                      int approximate, double* out) {
    if (rows < 0 || n < 0 || dtype < 0 || dtype > 2 || approximate < 0 || approximate > 1)
        return -1;
    if (rows * n == 0) return 0;
    if (!x || !bias || !out) return -1;
    const double k = sqrt(2.0 / 3.14159265358979323846);
    for (int64_t r = 0; r < rows; ++r) {
        for (int64_t j = 0; j < n; ++j) {
            const double v = load_elem(x, dtype, r * n + j) + load_elem(bias, dtype, j);
            double y;
            if (approximate)
                y = 0.5 * v * (1.0 + tanh(k * (v + 0.044715 * v * v * v)));
            else
                y = 0.5 * v * (1.0 + erf(v / sqrt(2.0)));
            out[r * n + j] = y;
        }
    }
    return 0;
}

/* QKV split with bias (the "add bias + transpose" after the QKV GEMM):
 * qkv [B*S, 3, H, D] (token-major, the GEMM's output row layout), bias [3, H, D]
 * -> q, k, v, each [B, H, S, D]:
 *   out_t[b, h, s, d] = qkv[(b*S + s), t, h, d] + bias[t, h, d],  t = 0, 1, 2
 * out is double [3, B, H, S, D] (q block, then k, then v). */
int tto_split_qkv_add_bias(const void* qkv, const void* bias, int dtype, int64_t B, int64_t S,
                           int64_t H, int64_t D, double* out) {
    if (B < 0 || S < 0 || H < 0 || D < 0 || dtype < 0 || dtype > 2) return -1;
    if (B * S * H * D == 0) return 0;
    if (!qkv || !bias || !out) return -1;
    const int64_t per = B * H * S * D;
    for (int64_t t = 0; t < 3; ++t)
        for (int64_t b = 0; b < B; ++b)
            for (int64_t h = 0; h < H; ++h)
                for (int64_t s = 0; s < S; ++s)
                    for (int64_t d = 0; d < D; ++d) {
                        const int64_t src = (((b * S + s) * 3 + t) * H + h) * D + d;
                        const int64_t dst = t * per + ((b * H + h) * S + s) * D + d;
                        out[dst] = load_elem(qkv, dtype, src) +
                                   load_elem(bias, dtype, (t * H + h) * D + d);
                    }
    return 0;
}

/* Head merge (the transpose after P.V): in [B, H, S, D] -> out [B*S, H*D]:
 *   out[(b*S + s), h*D + d] = in[b, h, s, d]      (double; exact copy) */
int tto_merge_heads(const void* in, int dtype, int64_t B, int64_t S, int64_t H, int64_t D,
                    double* out) {
    if (B < 0 || S < 0 || H < 0 || D < 0 || dtype < 0 || dtype > 2) return -1;
    if (B * S * H * D == 0) return 0;
    if (!in || !out) return -1;
    for (int64_t b = 0; b < B; ++b)
        for (int64_t s = 0; s < S; ++s)
            for (int64_t h = 0; h < H; ++h)
                for (int64_t d = 0; d < D; ++d)
                    out[((b * S + s) * H + h) * D + d] =
                        load_elem(in, dtype, ((b * H + h) * S + s) * D + d);
    return 0;
}

/* ---------------------------------------------------------------------------
 * NEXT-3: the attention the masked softmax sits in (PAPER.md
 * l.179-182: "the scaled dot-product attention computes the dot products of the
 * query with all keys, and applies a Softmax function to obtain the weights on
 * the values"), with the padding mask of tto_softmax_masked:
 *   q, k, v: [B, H, S, D]; lengths int32[B]; L_b = clamp(lengths[b], 0, S)
 *   p_ij = softmax_j(scale * q_i . k_j) over j < L_b  (tto_softmax_masked)
 *   o_i  = sum_{j < L_b} p_ij v_j                       (o_i = 0 when L_b = 0)
 * out: double [B, H, S, D]. */
int tto_attention(const void* q, const void* k, const void* v, int dtype,
                  const int32_t* lengths, int64_t B, int64_t H, int64_t S, int64_t D,
                  float scale, double* out) {
    if (B < 0 || H < 0 || S < 0 || D < 0 || dtype < 0 || dtype > 2) return -1;
    if (B * H * S * D == 0) return 0;
    if (!q || !k || !v || !lengths || !out) return -1;
    const double sc = (double)scale;
    double* z = (double*)malloc(sizeof(double) * (size_t)S);
    if (!z) return -1;
    for (int64_t b = 0; b < B; ++b) {
        int64_t L = lengths[b];
        if (L < 0) L = 0;
        if (L > S) L = S;
        for (int64_t h = 0; h < H; ++h) {
            const int64_t base = (b * H + h) * S * D;
            for (int64_t i = 0; i < S; ++i) {
                double* o = out + base + i * D;
                for (int64_t d = 0; d < D; ++d) o[d] = 0.0;
                if (L == 0) continue;
                double m = -INFINITY;
                for (int64_t j = 0; j < L; ++j) {
                    double dot = 0.0;
                    for (int64_t d = 0; d < D; ++d)
                        dot += load_elem(q, dtype, base + i * D + d) *
                               load_elem(k, dtype, base + j * D + d);
                    z[j] = sc * dot;
                    if (z[j] > m) m = z[j];
                }
                double s = 0.0;
                for (int64_t j = 0; j < L; ++j) s += exp(z[j] - m);
                for (int64_t j = 0; j < L; ++j) {
                    const double p = exp(z[j] - m) / s;
                    for (int64_t d = 0; d < D; ++d)
                        o[d] += p * load_elem(v, dtype, base + j * D + d);
                }
            }
        }
    }
    free(z);
    return 0;
}
