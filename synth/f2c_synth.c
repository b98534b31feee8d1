/*
 * f2c_synth.c -- seeded, counter-based synthetic input generator.
 *
 * Serves both sides (oracle tests and the CUDA path) and holds NONE of the
 * method's arithmetic: it only draws random numbers, normalises generated
 * vectors (part of the input recipe) and rounds them to the
 * input dtype.  Every value is a pure function of (seed, stream, step, row, col),
 * so any row of any step can be regenerated independently and in parallel, and
 * the output is bit-identical for any thread count.
 *
 * RNG: SplitMix64 finaliser used as a keyed hash; Gaussians by fp64 Box-Muller.
 * Identity labels: a keyed Feistel permutation of [0, n_id) with cycle walking,
 * cut into consecutive M-chunks (distinct ids per block, reshuffled per epoch).
 */
#include <math.h>
#include <stdint.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static inline uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static inline uint64_t row_key(uint64_t seed, uint64_t stream, uint64_t step, uint64_t row) {
    uint64_t h = mix64(seed ^ (stream * 0xD6E8FEB86659FD93ull));
    h = mix64(h ^ (step * 0xA0761D6478BD642Full));
    h = mix64(h ^ (row * 0xE7037ED1A0B428DBull));
    return h;
}

/* uniform in (0, 1] with 53 random bits */
static inline double u01(uint64_t r) { return ((double)(r >> 11) + 1.0) * 0x1.0p-53; }

static void gauss_row(uint64_t key, int32_t d, double *out) {
    for (int32_t k = 0; k < d; k += 2) {
        double u1 = u01(mix64(key + (uint64_t)(k + 1) * 0x9E3779B97F4A7C15ull));
        double u2 = u01(mix64(key + (uint64_t)(k + 2) * 0x9E3779B97F4A7C15ull));
        double r = sqrt(-2.0 * log(u1));
        double a = 6.283185307179586476925286766559 * u2;
        out[k] = r * cos(a);
        if (k + 1 < d) out[k + 1] = r * sin(a);
    }
}

/* round-to-nearest-even from double to bf16, returned as the bit pattern */
static inline uint16_t to_bf16(double x) {
    if (x == 0.0) return signbit(x) ? 0x8000u : 0u;
    int e;
    double f = frexp(x, &e); /* x = f * 2^e, 0.5 <= |f| < 1 */
    double q;
    if (e - 1 < -126) {      /* bf16 subnormal range: quantum 2^-133 */
        q = rint(ldexp(x, 133));
        float v = (float)ldexp(q, -133);
        uint32_t w;
        memcpy(&w, &v, 4);
        return (uint16_t)(w >> 16);
    }
    q = rint(f * 256.0); /* 8 significant bits, ties to even (default rounding mode) */
    float v = (float)ldexp(q, e - 8); /* exact in fp32 */
    uint32_t w;
    memcpy(&w, &v, 4);
    return (uint16_t)(w >> 16);
}

static void store_row(const double *v, int32_t d, int32_t dtype, void *dst) {
    if (dtype == 0) {
        uint16_t *o = (uint16_t *)dst;
        for (int32_t k = 0; k < d; ++k) o[k] = to_bf16(v[k]);
    } else {
        float *o = (float *)dst;
        for (int32_t k = 0; k < d; ++k) o[k] = (float)v[k];
    }
}

static void normalise(double *v, int32_t d) {
    double ss = 0.0;
    for (int32_t k = 0; k < d; ++k) ss += v[k] * v[k];
    double inv = 1.0 / sqrt(ss);
    for (int32_t k = 0; k < d; ++k) v[k] *= inv;
}

#define MAXD 4096

/* N(0,1) rows, fp64 (used by tests) */
void syn_gauss(uint64_t seed, uint64_t stream, uint64_t step, int64_t row0, int64_t nrows,
               int32_t d, double *out) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < nrows; ++i)
        gauss_row(row_key(seed, stream, step, (uint64_t)(row0 + i)), d, out + i * d);
}

/* unit-norm rows: normalise(N(0,1)^d) in fp64, then rounded to dtype (0 bf16, 1 f32) */
void syn_unit_rows(uint64_t seed, uint64_t stream, uint64_t step, int64_t row0, int64_t nrows,
                   int32_t d, int32_t dtype, void *out) {
    size_t es = dtype == 0 ? 2 : 4;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < nrows; ++i) {
        double v[MAXD];
        gauss_row(row_key(seed, stream, step, (uint64_t)(row0 + i)), d, v);
        normalise(v, d);
        store_row(v, d, dtype, (char *)out + (size_t)i * d * es);
    }
}

/* paired rows: x = normalise(N(0,1)^d) from (stream_x), g = normalise(x + sigma * n)
 * with n ~ N(0,1)^d from (stream_n); both rounded to dtype. */
void syn_pair_rows(uint64_t seed, uint64_t stream_x, uint64_t stream_n, uint64_t step,
                   int64_t row0, int64_t nrows, int32_t d, double sigma, int32_t dtype,
                   void *x_out, void *g_out) {
    size_t es = dtype == 0 ? 2 : 4;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < nrows; ++i) {
        double v[MAXD], w[MAXD];
        gauss_row(row_key(seed, stream_x, step, (uint64_t)(row0 + i)), d, v);
        normalise(v, d);
        gauss_row(row_key(seed, stream_n, step, (uint64_t)(row0 + i)), d, w);
        for (int32_t k = 0; k < d; ++k) w[k] = v[k] + sigma * w[k];
        normalise(w, d);
        if (x_out) store_row(v, d, dtype, (char *)x_out + (size_t)i * d * es);
        if (g_out) store_row(w, d, dtype, (char *)g_out + (size_t)i * d * es);
    }
}

/* i.i.d. uniform labels in [0, n_id) */
void syn_uniform_labels(uint64_t seed, uint64_t stream, uint64_t step, int64_t row0, int64_t n,
                        int64_t n_id, int64_t *out) {
    for (int64_t i = 0; i < n; ++i) {
        uint64_t r = mix64(row_key(seed, stream, step, (uint64_t)(row0 + i)));
        out[i] = (int64_t)(((unsigned __int128)r * (uint64_t)n_id) >> 64);
    }
}

/* keyed Feistel permutation of [0, n) with cycle walking */
static uint64_t feistel(uint64_t x, uint64_t n, uint64_t key) {
    int bits = 2;
    while ((1ull << bits) < n) bits += 2;
    int half = bits / 2;
    uint64_t mask = (1ull << half) - 1;
    do {
        uint64_t L = x >> half, R = x & mask;
        for (int r = 0; r < 4; ++r) {
            uint64_t F = mix64(key ^ ((uint64_t)r << 56) ^ R) & mask;
            uint64_t nL = R;
            R = L ^ F;
            L = nL;
        }
        x = (L << half) | R;
    } while (x >= n);
    return x;
}

/* identity labels of enqueue block t: M_glob distinct ids.  Blocks are
 * consecutive M_glob-chunks of a per-epoch permutation of [0, n_id); an epoch
 * holds floor(n_id / M_glob) blocks, so no block straddles a reshuffle.
 * Writes rows [row0, row0 + n) of the block. */
void syn_identity_labels(uint64_t seed, uint64_t block, int64_t row0, int64_t n, int64_t M_glob,
                         int64_t n_id, int64_t *out) {
    uint64_t per_epoch = (uint64_t)(n_id / M_glob);
    if (per_epoch == 0) per_epoch = 1;
    uint64_t epoch = block / per_epoch, k = block % per_epoch;
    uint64_t key = mix64(seed ^ 0x5EED1D5ull ^ (epoch * 0x9E3779B97F4A7C15ull));
    for (int64_t i = 0; i < n; ++i)
        out[i] = (int64_t)feistel(k * (uint64_t)M_glob + (uint64_t)(row0 + i), (uint64_t)n_id, key);
}

/* N(0, sigma^2) fp32 vector (G-Net EMA inputs) */
void syn_f32_normal(uint64_t seed, uint64_t stream, int64_t off, int64_t n, double sigma,
                    float *out) {
    const int64_t R = 1024;
#pragma omp parallel for schedule(static)
    for (int64_t b = 0; b < (n + R - 1) / R; ++b) {
        double v[1024];
        gauss_row(row_key(seed, stream, 0, (uint64_t)((off + b * R) / R)), 1024, v);
        int64_t lim = (b + 1) * R < n ? R : n - b * R;
        for (int64_t k = 0; k < lim; ++k) out[b * R + k] = (float)(sigma * v[k]);
    }
}
