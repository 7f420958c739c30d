/*
 * m2c_oracle.c -- plain, slow, obviously-correct CPU ORACLE of the M2Cache
 * dynamic sparse mixed-precision FFN decode step (arXiv 2410.14740).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  The
 * product (paper_2410_14740_b200/, libm2c) never links, imports or calls it,
 * and it shares no code, header, table or constant generator with the CUDA
 * path.  Build: gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math -fPIC -shared.
 *
 * Citations: P:L = /root/reference/PAPER.md line L; SURVEY §8(c) O0..O8 are the
 * step definitions this file restates; DESIGN.md "Readings" R1..R12 list every
 * place the paper is silent and the reading taken.
 *
 * Precision: double accumulation everywhere a sum is formed; IEEE fp32 single
 * operations (round-to-nearest-even) exactly where the quantiser definition
 * (O0, reading R4) prescribes fp32; integer predictor arithmetic is exact.
 *
 * Pins (tests/test_oracle_*.py): fp16 conversions vs numpy float16; O0 vs the
 * hand-verified worked examples in tests/golden/quant_examples.txt and closed
 * form invariants; O1-O4 vs python big-integer matmul and exact rationals; O5 vs python sorted();
 * O6 vs numpy float64 dense FFN (100% active, FP16 tier) and gather-matmul;
 * O7 vs an independently written move-to-front list LRU and SPEC's examples.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_EINVAL 1

/* ------------------------------------------------------------------------- */
/* IEEE binary16 <-> binary64 (exact decode; round-to-nearest-even encode).    */
/* ------------------------------------------------------------------------- */
double orc_half_to_double(uint16_t h)
{
    int sign = (h >> 15) & 1;
    int e = (h >> 10) & 0x1f;
    int m = h & 0x3ff;
    double v;
    if (e == 0)
        v = ldexp((double)m, -24); /* subnormal: m * 2^-24 */
    else if (e == 31)
        v = m ? NAN : INFINITY;
    else
        v = ldexp((double)(1024 + m), e - 25); /* (1 + m/1024) * 2^(e-15) */
    return sign ? -v : v;
}

uint16_t orc_double_to_half(double v)
{
    uint16_t sign = signbit(v) ? 0x8000 : 0;
    double a = fabs(v);
    if (isnan(v))
        return (uint16_t)(sign | 0x7e00);
    if (a < ldexp(1.0, -14)) {
        /* subnormal range: units of 2^-24; nearbyint = round half to even */
        double q = nearbyint(ldexp(a, 24));
        return (uint16_t)(sign | (uint16_t)q); /* q == 1024 encodes 2^-14 */
    }
    int ex;
    (void)frexp(a, &ex); /* a = f * 2^ex, f in [0.5, 1) */
    int E = ex - 1;      /* a in [2^E, 2^(E+1)) */
    double r = nearbyint(ldexp(a, 10 - E)); /* in [1024, 2048] */
    if (r == 2048.0) {
        r = 1024.0;
        E += 1;
    }
    if (E > 15)
        return (uint16_t)(sign | 0x7c00);
    return (uint16_t)(sign | (uint16_t)((E + 15) << 10) | (uint16_t)(r - 1024.0));
}

/* fp32 value -> fp16 RNE (float -> double is exact, so a single rounding). */
uint16_t orc_float_to_half(float f) { return orc_double_to_half((double)f); }

/* ------------------------------------------------------------------------- */
/* Tier plan (reading R3): k = floor(pct*F_r/100);              */
/* k16 = floor(k*a16/den), k8 = floor(k*a8/den), k4 = k - k16 - k8.           */
/* The paper's mix is 25% FP16 / 25% INT8 / 50% INT4.                 */
/* ------------------------------------------------------------------------- */
int orc_tier_plan(int32_t F_r, int32_t active_pct, int32_t a16, int32_t a8, int32_t den,
                  int32_t out[4])
{
    if (F_r < 0 || active_pct < 0 || active_pct > 100 || den <= 0 || a16 < 0 || a8 < 0 ||
        a16 + a8 > den)
        return ORC_EINVAL;
    int64_t k = (int64_t)F_r * active_pct / 100;
    int64_t k16 = k * a16 / den;
    int64_t k8 = k * a8 / den;
    out[0] = (int32_t)k;
    out[1] = (int32_t)k16;
    out[2] = (int32_t)k8;
    out[3] = (int32_t)(k - k16 - k8);
    return ORC_OK;
}

/* ------------------------------------------------------------------------- */
/* O0: per-group asymmetric min/max quantisation (reading R4; paper silent:   */
/* P:73 "quantized to a smaller number of bits", P:134 dequantisation "back  */
/* to FP16").  One group = 128 consecutive weights along d.                    */
/* ------------------------------------------------------------------------- */
void orc_quant_group(int bits, const uint16_t *w, int n, uint16_t *scale16, uint8_t *zero,
                     uint8_t *q)
{
    int maxq = (1 << bits) - 1;
    float lo = 0.0f, hi = 0.0f; /* range extended to include 0 */
    for (int j = 0; j < n; j++) {
        float v = (float)orc_half_to_double(w[j]);
        if (v < lo) lo = v;
        if (v > hi) hi = v;
    }
    uint16_t s16;
    if (lo == hi) {
        s16 = 0x3c00; /* 1.0 */
    } else {
        volatile float range = hi - lo;                 /* fl32 */
        volatile float s32 = range / (float)maxq;       /* fl32 */
        s16 = orc_float_to_half(s32);
        if ((s16 & 0x7fff) == 0) s16 = 0x0001;          /* underflow -> 2^-24 */
    }
    float s = (float)orc_half_to_double(s16);
    volatile float zf = -lo / s;                        /* fl32 */
    float zr = nearbyintf(zf);
    int z = (int)zr;
    if (z < 0) z = 0;
    if (z > maxq) z = maxq;
    *scale16 = s16;
    *zero = (uint8_t)z;
    for (int j = 0; j < n; j++) {
        float v = (float)orc_half_to_double(w[j]);
        volatile float t = v / s;                       /* fl32 */
        int qi = (int)nearbyintf(t) + z;
        if (qi < 0) qi = 0;
        if (qi > maxq) qi = maxq;
        q[j] = (uint8_t)qi;
    }
}

/* Record layout:
 *   FP16: gate[d] | up[d] | down[d]  (fp16, 6d bytes)
 *   INT8: q_gate[d] | q_up[d] | q_down[d] (u8) | scales fp16[3G] | zeros u8[3G] | pad16
 *   INT4: nib_gate[d/2] | nib_up[d/2] | nib_down[d/2] (element 2i low nibble, 2i+1 high)
 *         | scales fp16[3G] | zeros u8[3G] | pad16
 *   G = d/128; scales/zeros ordered gate groups, then up groups, then down groups. */
int64_t orc_record_bytes(int bits, int d)
{
    if (d <= 0 || d % 128) return -1;
    int64_t G = d / 128, raw;
    if (bits == 16) raw = 6LL * d;
    else if (bits == 8) raw = 3LL * d + 9 * G;
    else if (bits == 4) raw = 3LL * d / 2 + 9 * G;
    else return -1;
    return (raw + 15) / 16 * 16;
}

int orc_pack(int bits, int d, const uint16_t *gate, const uint16_t *up, const uint16_t *down_t,
             int64_t n0, int64_t n1, uint8_t *out)
{
    int64_t nb = orc_record_bytes(bits, d);
    if (nb < 0 || n1 < n0) return ORC_EINVAL;
    int G = d / 128;
    const uint16_t *mats[3] = {gate, up, down_t};
    uint8_t q[128];
    for (int64_t n = n0; n < n1; n++) {
        uint8_t *rec = out + (n - n0) * nb;
        memset(rec, 0, (size_t)nb);
        if (bits == 16) {
            for (int m = 0; m < 3; m++)
                memcpy(rec + (size_t)m * d * 2, mats[m] + n * d, (size_t)d * 2);
            continue;
        }
        int64_t data_bytes = (bits == 8) ? 3LL * d : 3LL * d / 2;
        uint8_t *scales = rec + data_bytes;
        uint8_t *zeros = scales + 2 * 3 * G;
        for (int m = 0; m < 3; m++) {
            for (int gi = 0; gi < G; gi++) {
                uint16_t s16;
                uint8_t z;
                orc_quant_group(bits, mats[m] + n * d + gi * 128, 128, &s16, &z, q);
                memcpy(scales + 2 * (m * G + gi), &s16, 2);
                zeros[m * G + gi] = z;
                for (int j = 0; j < 128; j++) {
                    int e = gi * 128 + j; /* element index within the vector */
                    if (bits == 8) {
                        rec[(size_t)m * d + e] = q[j];
                    } else {
                        uint8_t *b = rec + (size_t)m * (d / 2) + e / 2;
                        if (e % 2 == 0) *b = (uint8_t)((*b & 0xf0) | q[j]);
                        else *b = (uint8_t)((*b & 0x0f) | (q[j] << 4));
                    }
                }
            }
        }
    }
    return ORC_OK;
}

/* Exact dequantised values of one record: deq = (q - z) * s (exact in double). */
int orc_dequant_record(int bits, int d, const uint8_t *rec, double *gate, double *up,
                       double *down)
{
    double *outs[3] = {gate, up, down};
    int G = d / 128;
    if (orc_record_bytes(bits, d) < 0) return ORC_EINVAL;
    for (int m = 0; m < 3; m++) {
        for (int e = 0; e < d; e++) {
            if (bits == 16) {
                uint16_t h;
                memcpy(&h, rec + ((size_t)m * d + e) * 2, 2);
                outs[m][e] = orc_half_to_double(h);
                continue;
            }
            int64_t data_bytes = (bits == 8) ? 3LL * d : 3LL * d / 2;
            const uint8_t *scales = rec + data_bytes;
            const uint8_t *zeros = scales + 2 * 3 * G;
            int gi = e / 128;
            uint16_t s16;
            memcpy(&s16, scales + 2 * (m * G + gi), 2);
            int z = zeros[m * G + gi];
            int qv;
            if (bits == 8) qv = rec[(size_t)m * d + e];
            else {
                uint8_t b = rec[(size_t)m * (d / 2) + e / 2];
                qv = (e % 2 == 0) ? (b & 0x0f) : (b >> 4);
            }
            outs[m][e] = (double)(qv - z) * orc_half_to_double(s16);
        }
    }
    return ORC_OK;
}

/* ------------------------------------------------------------------------- */
/* O1-O4: exact-integer low-rank predictor (reading R2; paper: "low-rank      */
/* predictor" P:73, Deja Vu score per neuron P:252).                          */
/*   O1  X_j = x_j * 2^24, exact integer (every fp16 is a multiple of 2^-24)  */
/*   O2  h = A X in exact integer arithmetic (|h| < 2^60 for d <= 8192)       */
/*   O3  hq = Q(h), Q(v)_i = sgn(v_i) floor((254|v_i| + M) / (2M)), M = max|v|*/
/*   O4  s = B hq (int32)                                                     */
/* ------------------------------------------------------------------------- */
static int8_t quant_sym_127(int64_t v, int64_t M)
{
    /* sgn(v) * floor((254|v| + M) / (2M)) : round-half-up of 127|v|/M.       */
    /* |v| <= M < 2^60: 254|v| + M would overflow int64, so the quotient is    */
    /* formed from M's multiples: 127|v|/M = q + rem/M, and the rounding       */
    /* compares 2 rem with M (half rounds up).                                 */
    if (M == 0) return 0;
    int64_t a = v < 0 ? -v : v;
    int64_t q = 0, rem = 0;
    /* long division of 127 a by M without overflow: a <= M, so q <= 127 */
    for (int i = 0; i < 127; i++) {
        rem += a;
        if (rem >= M) { rem -= M; q++; }
    }
    if (rem >= M - rem) q++; /* 2 rem >= M  <=>  fraction >= 1/2 */
    return (int8_t)(v < 0 ? -q : q);
}

int orc_predict(int d, int r, int F_r, const uint16_t *x, const int8_t *A, const int8_t *B,
                int64_t *h, int8_t *hq, int32_t *s)
{
    if (d <= 0 || r <= 0 || F_r < 0 || d > 8192) return ORC_EINVAL;
    int64_t *X = (int64_t *)malloc(sizeof(int64_t) * (size_t)d);
    for (int j = 0; j < d; j++) { /* O1 */
        double v = orc_half_to_double(x[j]);
        if (!isfinite(v)) { free(X); return ORC_EINVAL; }
        X[j] = (int64_t)ldexp(v, 24); /* exact: every fp16 is a multiple of 2^-24 */
    }
    int64_t Mh = 0;
    for (int i = 0; i < r; i++) { /* O2 */
        int64_t acc = 0;
        for (int j = 0; j < d; j++) acc += (int64_t)A[(size_t)i * d + j] * X[j];
        h[i] = acc;
        int64_t a = acc < 0 ? -acc : acc;
        if (a > Mh) Mh = a;
    }
    free(X);
    for (int i = 0; i < r; i++) hq[i] = quant_sym_127(h[i], Mh); /* O3 */
    for (int n = 0; n < F_r; n++) { /* O4 */
        int64_t acc = 0;
        for (int i = 0; i < r; i++) acc += (int64_t)B[(size_t)n * r + i] * hq[i];
        s[n] = (int32_t)acc;
    }
    return ORC_OK;
}

/* ------------------------------------------------------------------------- */
/* O5: top-k by (score desc, id asc) (P:253 top-k; tie rule S:182), split by  */
/* rank into FP16 / INT8 / INT4 (P:226, P:254 higher score -> higher          */
/* precision; P:428 25/25/50).                                                */
/* ------------------------------------------------------------------------- */
typedef struct { int32_t s; int32_t n; } sc_t;

static int cmp_score(const void *a, const void *b)
{
    const sc_t *x = (const sc_t *)a, *y = (const sc_t *)b;
    if (x->s != y->s) return x->s > y->s ? -1 : 1;
    return x->n < y->n ? -1 : (x->n > y->n);
}

static int cmp_i32(const void *a, const void *b)
{
    int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
    return x < y ? -1 : (x > y);
}

int orc_select(int F_r, const int32_t *s, const int32_t plan[4], int32_t *rank_list,
               int8_t *tier_of, int32_t *tier_ids)
{
    int k = plan[0], k16 = plan[1], k8 = plan[2], k4 = plan[3];
    if (k < 0 || k > F_r || k16 < 0 || k8 < 0 || k4 < 0 || k16 + k8 + k4 != k)
        return ORC_EINVAL;
    sc_t *v = (sc_t *)malloc(sizeof(sc_t) * (size_t)(F_r > 0 ? F_r : 1));
    for (int n = 0; n < F_r; n++) { v[n].s = s[n]; v[n].n = n; }
    qsort(v, (size_t)F_r, sizeof(sc_t), cmp_score);
    for (int n = 0; n < F_r; n++) tier_of[n] = -1;
    for (int i = 0; i < k; i++) {
        rank_list[i] = v[i].n;
        tier_of[v[i].n] = (int8_t)(i < k16 ? 0 : (i < k16 + k8 ? 1 : 2));
    }
    int off[3] = {0, k16, k16 + k8}, cnt[3] = {0, 0, 0};
    for (int n = 0; n < F_r; n++) /* ascending id within each tier */
        if (tier_of[n] >= 0) { int t = tier_of[n]; tier_ids[off[t] + cnt[t]++] = n; }
    (void)cmp_i32;
    free(v);
    return ORC_OK;
}

/* ------------------------------------------------------------------------- */
/* O6: sparse FFN over the selected neurons (P:69 neuron = row of the first   */
/* FFN matrices + column of the next; P:76 compute only active neurons).      */
/*   g = sum_j Wg_j x_j, u = sum_j Wu_j x_j, a = act(g) * u, yhat += a * Wd.  */
/* recs[t] = packed records of tier t indexed by neuron id (stride nb_t).     */
/* act: 0 = SiLU (LLaMA-2), 1 = ReLU (ReGLU flag, reading R6).                */
/* ------------------------------------------------------------------------- */
int orc_ffn(int d, const int32_t plan[4], const int32_t *tier_ids, const uint8_t *rec16,
            const uint8_t *rec8, const uint8_t *rec4, const uint16_t *x, int act, double *yhat,
            double *a_out)
{
    const uint8_t *recs[3] = {rec16, rec8, rec4};
    const int bits[3] = {16, 8, 4};
    int cnt[3] = {plan[1], plan[2], plan[3]};
    double *wg = (double *)malloc(sizeof(double) * 3 * (size_t)d);
    double *wu = wg + d, *wd = wg + 2 * d;
    double *xd = (double *)malloc(sizeof(double) * (size_t)d);
    for (int j = 0; j < d; j++) { xd[j] = orc_half_to_double(x[j]); yhat[j] = 0.0; }
    int idx = 0;
    for (int t = 0; t < 3; t++) {
        int64_t nb = orc_record_bytes(bits[t], d);
        for (int i = 0; i < cnt[t]; i++, idx++) {
            int32_t n = tier_ids[idx];
            orc_dequant_record(bits[t], d, recs[t] + (size_t)n * nb, wg, wu, wd);
            double g = 0.0, u = 0.0;
            for (int j = 0; j < d; j++) { g += wg[j] * xd[j]; u += wu[j] * xd[j]; }
            double a = (act == 1) ? (g > 0.0 ? g : 0.0) * u : g / (1.0 + exp(-g)) * u;
            if (a_out) a_out[idx] = a;
            for (int j = 0; j < d; j++) yhat[j] += a * wd[j];
        }
    }
    free(wg);
    free(xd);
    return ORC_OK;
}

/* ------------------------------------------------------------------------- */
/* SURVEY 8(d) "oracle timing: an OpenMP variant over neurons on all host      */
/* cores".  The same O2/O4 and O6 arithmetic in the same order per output:    */
/* integer dot products split over rows; a_n split over neurons; yhat_j split */
/* over j with the neuron sum in the serial order -- bit-identical to          */
/* orc_predict / orc_ffn (pinned by tests/test_oracle_ffn.py).  Timing only.   */
/* ------------------------------------------------------------------------- */
int orc_predict_mt(int d, int r, int F_r, const uint16_t *x, const int8_t *A, const int8_t *B,
                   int64_t *h, int8_t *hq, int32_t *s, int nthreads)
{
    if (d <= 0 || r <= 0 || F_r < 0 || d > 8192 || nthreads < 1) return ORC_EINVAL;
    int64_t *X = (int64_t *)malloc(sizeof(int64_t) * (size_t)d);
    for (int j = 0; j < d; j++) {
        double v = orc_half_to_double(x[j]);
        if (!isfinite(v)) { free(X); return ORC_EINVAL; }
        X[j] = (int64_t)ldexp(v, 24);
    }
#pragma omp parallel for num_threads(nthreads) schedule(static)
    for (int i = 0; i < r; i++) {
        int64_t acc = 0;
        for (int j = 0; j < d; j++) acc += (int64_t)A[(size_t)i * d + j] * X[j];
        h[i] = acc;
    }
    free(X);
    int64_t Mh = 0;
    for (int i = 0; i < r; i++) {
        int64_t a = h[i] < 0 ? -h[i] : h[i];
        if (a > Mh) Mh = a;
    }
    for (int i = 0; i < r; i++) hq[i] = quant_sym_127(h[i], Mh);
#pragma omp parallel for num_threads(nthreads) schedule(static)
    for (int n = 0; n < F_r; n++) {
        int64_t acc = 0;
        for (int i = 0; i < r; i++) acc += (int64_t)B[(size_t)n * r + i] * hq[i];
        s[n] = (int32_t)acc;
    }
    return ORC_OK;
}

int orc_ffn_mt(int d, const int32_t plan[4], const int32_t *tier_ids, const uint8_t *rec16,
               const uint8_t *rec8, const uint8_t *rec4, const uint16_t *x, int act, double *yhat,
               int nthreads)
{
    if (nthreads < 1) return ORC_EINVAL;
    const uint8_t *recs[3] = {rec16, rec8, rec4};
    const int bits[3] = {16, 8, 4};
    const int k = plan[1] + plan[2] + plan[3];
    double *xd = (double *)malloc(sizeof(double) * (size_t)d);
    double *a = (double *)malloc(sizeof(double) * (size_t)(k > 0 ? k : 1));
    double *wdall = (double *)malloc(sizeof(double) * (size_t)(k > 0 ? k : 1) * d);
    for (int j = 0; j < d; j++) xd[j] = orc_half_to_double(x[j]);
#pragma omp parallel num_threads(nthreads)
    {
        double *wg = (double *)malloc(sizeof(double) * 2 * (size_t)d);
        double *wu = wg + d;
#pragma omp for schedule(dynamic, 4)
        for (int idx = 0; idx < k; idx++) {
            const int t = idx < plan[1] ? 0 : (idx < plan[1] + plan[2] ? 1 : 2);
            const int64_t nb = orc_record_bytes(bits[t], d);
            orc_dequant_record(bits[t], d, recs[t] + (size_t)tier_ids[idx] * nb, wg, wu,
                               wdall + (size_t)idx * d);
            double g = 0.0, u = 0.0;
            for (int j = 0; j < d; j++) { g += wg[j] * xd[j]; u += wu[j] * xd[j]; }
            a[idx] = (act == 1) ? (g > 0.0 ? g : 0.0) * u : g / (1.0 + exp(-g)) * u;
        }
        free(wg);
#pragma omp for schedule(static)
        for (int j = 0; j < d; j++) {
            double y = 0.0;
            for (int idx = 0; idx < k; idx++) y += a[idx] * wdall[(size_t)idx * d + j];
            yhat[j] = y;
        }
    }
    free(wdall);
    free(a);
    free(xd);
    return ORC_OK;
}

/* O8 stack harness: x_next = fp16_rne(x + fp16_rne(yhat)) (exact sum in double). */
void orc_residual(int d, const uint16_t *x, const double *yhat, uint16_t *y16, uint16_t *x_next)
{
    for (int j = 0; j < d; j++) {
        uint16_t yh = orc_double_to_half(yhat[j]);
        if (y16) y16[j] = yh;
        x_next[j] = orc_double_to_half(orc_half_to_double(x[j]) + orc_half_to_double(yh));
    }
}

/* ------------------------------------------------------------------------- */
/* O7: LRU per (layer, tier) pool ("LRU cache"; P:335 isolated    */
/* contiguous unit).  Step-granular timestamps; victims = smallest            */
/* (last_use, slot) with last_use < t; misses in ascending id (reading R7).   */
/* State: occupant[C] (-1 empty), last[C] (-1 never), slot_of[F_r] (-1).      */
/* R: required ids of this tier, ascending.  Outputs in R's order.            */
/* ------------------------------------------------------------------------- */
typedef struct { int64_t key; int32_t slot; } cand_t;

static int cmp_cand(const void *a, const void *b)
{
    const cand_t *x = (const cand_t *)a, *y = (const cand_t *)b;
    if (x->key != y->key) return x->key < y->key ? -1 : 1;
    return x->slot < y->slot ? -1 : (x->slot > y->slot);
}

int orc_lru_step(int C, int F_r, int32_t *occupant, int32_t *last, int32_t *slot_of, int32_t t,
                 const int32_t *R, int nR, int32_t *slots, uint32_t *hit_bits, int32_t *miss_ids,
                 int32_t *miss_slots, int32_t *n_miss, int32_t *ev_ids, int32_t *ev_slots,
                 int32_t *n_ev)
{
    if (nR > C) return ORC_EINVAL;
    for (int i = 0; i < (nR + 31) / 32; i++) hit_bits[i] = 0;
    int nm = 0;
    for (int i = 0; i < nR; i++) { /* 1. hits */
        int32_t n = R[i];
        if (n < 0 || n >= F_r || (i > 0 && R[i - 1] >= n)) return ORC_EINVAL;
        int32_t sl = slot_of[n];
        if (sl >= 0) {
            last[sl] = t;
            slots[i] = sl;
            hit_bits[i / 32] |= 1u << (i % 32);
        } else {
            slots[i] = -1;
            nm++;
        }
    }
    /* 3. candidates: last < t, sorted by (last, slot) */
    cand_t *cv = (cand_t *)malloc(sizeof(cand_t) * (size_t)(C > 0 ? C : 1));
    int nc = 0;
    for (int sl = 0; sl < C; sl++)
        if (last[sl] < t) { cv[nc].key = last[sl]; cv[nc].slot = sl; nc++; }
    if (nc < nm) { free(cv); return ORC_EINVAL; }
    qsort(cv, (size_t)nc, sizeof(cand_t), cmp_cand);
    int mi = 0, ne = 0;
    for (int i = 0; i < nR; i++) { /* 2+4. misses ascending, paired with candidates */
        if (slots[i] >= 0) continue;
        int32_t n = R[i], sl = cv[mi].slot;
        int32_t old = occupant[sl];
        if (old >= 0) {
            slot_of[old] = -1;
            if (ev_ids) { ev_ids[ne] = old; ev_slots[ne] = sl; }
            ne++;
        }
        occupant[sl] = n;
        slot_of[n] = sl;
        last[sl] = t;
        slots[i] = sl;
        if (miss_ids) { miss_ids[mi] = n; miss_slots[mi] = sl; }
        mi++;
    }
    *n_miss = mi;
    *n_ev = ne;
    free(cv);
    return ORC_OK;
}
