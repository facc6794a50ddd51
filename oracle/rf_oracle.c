/*
 * rf_oracle.c -- CPU restatement of the reference attention path (TEST INFRASTRUCTURE ONLY).
 *
 * This file is the parity oracle for the B200 kernels.  It is NOT part of the
 * product: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it.  The product path (paper_2603_12646_b200/)
 * never links or calls anything in oracle/.
 *
 * Parity status: PINNED.  Every function here is checked bit-for-bit against the
 * reference's own sources compiled into oracle/_ref/libref_attn.so (see
 * oracle/Makefile, oracle/ref_shim.cpp and tests/test_oracle_vs_ref.py) and
 * against committed golden vectors generated from that build
 * (tests/golden/make_golden.py).
 *
 * Each function cites the reference file:line whose arithmetic it follows.  The
 * arithmetic ORDER (sequential f64 sums, per-tile online softmax update) is kept
 * identical so that results are bit-exact with the reference; the code structure
 * (flat pointers, one (batch, head) slice per worker thread) is our own.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <pthread.h>

#define RF_MASK_VALUE (-65504.0f)     /* attention.hpp:15 */
#define RF_MASK_THRESHOLD (-30000.0f) /* attention.hpp:16 */

/* ---------------------------------------------------------------------------------------------
 * binary16 emulation (tensor.cpp:47-98): round-to-nearest-even incl. subnormals.
 * ------------------------------------------------------------------------------------------- */
static uint32_t f32_bits(float v) {
    uint32_t b;
    memcpy(&b, &v, 4);
    return b;
}
static float bits_f32(uint32_t b) {
    float v;
    memcpy(&v, &b, 4);
    return v;
}

/* tensor.cpp:47-76 */
uint16_t rf_oracle_float_to_half(float value) {
    const uint32_t bits = f32_bits(value);
    const uint32_t sign = (bits >> 16) & 0x8000u;
    const uint32_t raw_exp = (bits >> 23) & 0xFFu;
    uint32_t frac = bits & 0x7FFFFFu;
    const int32_t e = (int32_t)raw_exp - 127 + 15;

    if (raw_exp == 0xFFu) return (uint16_t)(sign | 0x7C00u | (frac ? 0x200u : 0u));
    if (e >= 0x1F) return (uint16_t)(sign | 0x7C00u);
    if (e <= 0) {
        if (e < -10) return (uint16_t)sign;
        frac |= 0x800000u;
        const int shift = 14 - e;
        uint32_t h = frac >> shift;
        const uint32_t rem = frac & ((1u << shift) - 1u);
        const uint32_t half = 1u << (shift - 1);
        if (rem > half || (rem == half && (h & 1u))) ++h;
        return (uint16_t)(sign | h);
    }
    uint32_t h = sign | ((uint32_t)e << 10) | (frac >> 13);
    const uint32_t rem = frac & 0x1FFFu;
    if (rem > 0x1000u || (rem == 0x1000u && (h & 1u))) ++h; /* carry may bump the exponent */
    return (uint16_t)h;
}

/* tensor.cpp:78-96 */
float rf_oracle_half_to_float(uint16_t bits) {
    const uint32_t sign = ((uint32_t)(bits & 0x8000u)) << 16;
    uint32_t e = (bits >> 10) & 0x1Fu;
    uint32_t frac = bits & 0x3FFu;
    if (e == 0x1Fu) return bits_f32(sign | 0x7F800000u | (frac << 13));
    if (e == 0) {
        if (frac == 0) return bits_f32(sign);
        int shift = 0;
        while ((frac & 0x400u) == 0) {
            frac <<= 1;
            ++shift;
        }
        frac &= 0x3FFu;
        e = (uint32_t)(1 - shift);
    }
    return bits_f32(sign | ((e - 15u + 127u) << 23) | (frac << 13));
}

/* tensor.cpp:98 */
float rf_oracle_quantize_f16(float v) { return rf_oracle_half_to_float(rf_oracle_float_to_half(v)); }

void rf_oracle_quantize_f16_array(const float* in, float* out, int64_t n) {
    for (int64_t i = 0; i < n; ++i) out[i] = rf_oracle_quantize_f16(in[i]);
}

/* pad-bias chain the rewriter installs (rewrite.cpp:303-318, executed by
 * interpreter.cpp:230-257): Cast_f16( (1 - mask) * -65504 ), f32 arithmetic. */
void rf_oracle_pad_bias_from_mask(const float* mask, float* bias, int64_t n) {
    for (int64_t i = 0; i < n; ++i) {
        const float inv = 1.0f - mask[i];
        const float scaled = inv * RF_MASK_VALUE;
        bias[i] = rf_oracle_quantize_f16(scaled);
    }
}

/* ---------------------------------------------------------------------------------------------
 * Tensor::random (tensor.cpp:35-45): mt19937_64, 53-bit draw -> [-1, 1).
 * mt19937_64 itself is the published Matsumoto/Nishimura generator that
 * std::mt19937_64 is specified to be ([rand.predef]); restated here so the
 * fill matches the reference's stream element for element.
 * ------------------------------------------------------------------------------------------- */
typedef struct {
    uint64_t mt[312];
    int idx;
} rf_mt64;

static void mt64_seed(rf_mt64* g, uint64_t seed) {
    g->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    g->idx = 312;
}

static uint64_t mt64_next(rf_mt64* g) {
    if (g->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            const uint64_t x = (g->mt[i] & 0xFFFFFFFF80000000ULL) | (g->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
            uint64_t xa = x >> 1;
            if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
            g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
        }
        g->idx = 0;
    }
    uint64_t y = g->mt[g->idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= (y >> 43);
    return y;
}

/* Opaque generator handle so a caller can draw q, k, v in sequence from one
 * stream exactly as bench_attention.cpp:16-23 does. */
void* rf_oracle_rng_new(uint64_t seed) {
    rf_mt64* g = (rf_mt64*)malloc(sizeof(rf_mt64));
    if (g) mt64_seed(g, seed);
    return g;
}
void rf_oracle_rng_free(void* g) { free(g); }
uint64_t rf_oracle_rng_next(void* g) { return mt64_next((rf_mt64*)g); }

/* tensor.cpp:37-43 */
void rf_oracle_random_fill(void* gen, float* out, int64_t n, int as_f16) {
    rf_mt64* g = (rf_mt64*)gen;
    for (int64_t i = 0; i < n; ++i) {
        const double u = (double)(mt64_next(g) >> 11) * 0x1.0p-53;
        float v = (float)(2.0 * u - 1.0);
        if (as_f16) v = rf_oracle_quantize_f16(v);
        out[i] = v;
    }
}

/* ---------------------------------------------------------------------------------------------
 * flash_attention (attention.cpp:106-213)
 * ------------------------------------------------------------------------------------------- */

/* attention.cpp:34-36 */
double rf_oracle_effective_scale(double scale, int64_t head_dim) {
    return scale != 0.0 ? scale : 1.0 / sqrt((double)head_dim);
}

/* attention.cpp:132-136 */
static inline int window_ok(int64_t i, int64_t j, int64_t wl, int64_t wr) {
    if (wl >= 0 && i - j > wl) return 0;
    if (wr >= 0 && j - i > wr) return 0;
    return 1;
}

/* One (batch, head) slice.  Follows attention.cpp:145-209 line for line in its
 * arithmetic: per key tile, per query: scores (f64 dot, scale, +pad), tile max,
 * correction = exp(old_max - new_max) applied only when != 1, then w = exp(s -
 * new_max) accumulated in key order; final divide by the running sum, 0 for
 * rows with no live key. */
static void flash_slice(const float* qp, const float* kp, const float* vp, float* op,
                        const float* pad, int64_t S, int64_t d, double scale, int64_t wl,
                        int64_t wr, int64_t tile, double* row_max, double* row_sum,
                        double* tile_scores, double* acc) {
    for (int64_t i = 0; i < S; ++i) {
        row_max[i] = -INFINITY;
        row_sum[i] = 0.0;
    }
    memset(acc, 0, sizeof(double) * (size_t)(S * d));

    for (int64_t t0 = 0; t0 < S; t0 += tile) {
        const int64_t t1 = t0 + tile < S ? t0 + tile : S;
        for (int64_t i = 0; i < S; ++i) {
            double tile_max = -INFINITY;
            int any = 0;
            for (int64_t j = t0; j < t1; ++j) {
                double s = -INFINITY;
                if (window_ok(i, j, wl, wr) && (!pad || pad[j] > RF_MASK_THRESHOLD)) {
                    double dot = 0.0;
                    for (int64_t c = 0; c < d; ++c) dot += (double)qp[i * d + c] * (double)kp[j * d + c];
                    s = dot * scale;
                    if (pad) s += (double)pad[j];
                    any = 1;
                }
                tile_scores[j - t0] = s;
                if (s > tile_max) tile_max = s; /* == std::max(tile_max, s) */
            }
            if (!any) continue;

            const double new_max = row_max[i] > tile_max ? row_max[i] : tile_max;
            const double correction = isinf(row_max[i]) ? 0.0 : exp(row_max[i] - new_max);
            if (correction != 1.0) {
                for (int64_t c = 0; c < d; ++c) acc[i * d + c] *= correction;
                row_sum[i] *= correction;
            }
            for (int64_t j = t0; j < t1; ++j) {
                const double s = tile_scores[j - t0];
                if (isinf(s)) continue;
                const double w = exp(s - new_max);
                row_sum[i] += w;
                for (int64_t c = 0; c < d; ++c) acc[i * d + c] += w * (double)vp[j * d + c];
            }
            row_max[i] = new_max;
        }
    }
    for (int64_t i = 0; i < S; ++i) {
        const double denom = row_sum[i];
        for (int64_t c = 0; c < d; ++c)
            op[i * d + c] = denom > 0.0 ? (float)(acc[i * d + c] / denom) : 0.0f;
    }
}

/* Error codes mirror the reference's ShapeMismatch sites (attention.cpp:14-21,110,111-116);
 * the Python wrapper raises ShapeMismatch with the same messages. */
enum { RF_ORACLE_OK = 0, RF_ORACLE_BAD_TILE = 1, RF_ORACLE_BAD_SHAPE = 2, RF_ORACLE_NOMEM = 3 };

/* work descriptor shared by the slice workers */
typedef struct {
    const float *q, *k, *v, *pad_bias;
    float* out;
    int64_t B, H, S, d, wl, wr, tile;
    double scale;
    int64_t next; /* next slice to claim (guarded by mu) */
    int failed;
    pthread_mutex_t mu;
} flash_job;

static void* flash_worker(void* arg) {
    flash_job* job = (flash_job*)arg;
    const int64_t S = job->S, d = job->d;
    double* row_max = (double*)malloc(sizeof(double) * (size_t)(S > 0 ? S : 1));
    double* row_sum = (double*)malloc(sizeof(double) * (size_t)(S > 0 ? S : 1));
    double* tile_scores = (double*)malloc(sizeof(double) * (size_t)job->tile);
    double* acc = (double*)malloc(sizeof(double) * (size_t)(S * d > 0 ? S * d : 1));
    if (!row_max || !row_sum || !tile_scores || !acc) {
        pthread_mutex_lock(&job->mu);
        job->failed = 1;
        pthread_mutex_unlock(&job->mu);
    } else {
        for (;;) {
            pthread_mutex_lock(&job->mu);
            const int64_t s = job->next++;
            pthread_mutex_unlock(&job->mu);
            if (s >= job->B * job->H) break;
            const int64_t b = s / job->H;
            const size_t base = (size_t)(s * S * d);
            const float* pad = job->pad_bias ? job->pad_bias + (size_t)(b * S) : NULL;
            flash_slice(job->q + base, job->k + base, job->v + base, job->out + base, pad, S, d,
                        job->scale, job->wl, job->wr, job->tile, row_max, row_sum, tile_scores, acc);
        }
    }
    free(row_max);
    free(row_sum);
    free(tile_scores);
    free(acc);
    return NULL;
}

/* q,k,v,out: [B,H,S,d] contiguous f32.  pad_bias: [B,S] (the [B,1,1,S] tensor) or NULL.
 * threads <= 1 runs the slices sequentially exactly like the reference's b/h loops
 * (attention.cpp:138-142); slices are independent so any thread count gives identical bits. */
int rf_oracle_flash_attention(const float* q, const float* k, const float* v, float* out,
                              int64_t B, int64_t H, int64_t S, int64_t d, double scale_attr,
                              int64_t wl, int64_t wr, const float* pad_bias, int64_t tile,
                              int threads) {
    if (tile < 1) return RF_ORACLE_BAD_TILE;
    if (B < 0 || H < 0 || S < 0 || d < 0) return RF_ORACLE_BAD_SHAPE;
    flash_job job;
    job.q = q; job.k = k; job.v = v; job.pad_bias = pad_bias; job.out = out;
    job.B = B; job.H = H; job.S = S; job.d = d; job.wl = wl; job.wr = wr; job.tile = tile;
    job.scale = rf_oracle_effective_scale(scale_attr, d);
    job.next = 0;
    job.failed = 0;
    pthread_mutex_init(&job.mu, NULL);
    if (threads > B * H) threads = (int)(B * H);
    if (threads <= 1) {
        flash_worker(&job);
    } else {
        pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
        int started = 0;
        if (th) {
            for (; started < threads; ++started)
                if (pthread_create(&th[started], NULL, flash_worker, &job) != 0) break;
        }
        if (started == 0) flash_worker(&job); /* could not spawn: do it inline */
        for (int t = 0; t < started; ++t) pthread_join(th[t], NULL);
        free(th);
    }
    pthread_mutex_destroy(&job.mu);
    return job.failed ? RF_ORACLE_NOMEM : RF_ORACLE_OK;
}

/* FlashStats (attention.hpp:36-40, filled at attention.cpp:126-130). */
void rf_oracle_flash_stats(int64_t B, int64_t H, int64_t S, int64_t d, int64_t tile,
                           uint64_t* tile_scratch_floats, uint64_t* row_state_floats,
                           uint64_t* output_floats) {
    *tile_scratch_floats = (uint64_t)tile;
    *row_state_floats = (uint64_t)(2 * S);
    *output_floats = (uint64_t)(B * H * S * d);
}

/* ---------------------------------------------------------------------------------------------
 * sdpa (attention.cpp:38-104): naive O(S^2) reference with [mB|1, mH|1, S, S] additive mask.
 * ------------------------------------------------------------------------------------------- */
int rf_oracle_sdpa(const float* q, const float* k, const float* v, float* out, int64_t B,
                   int64_t H, int64_t S, int64_t d, const float* mask2d, int64_t mB, int64_t mH,
                   double scale) {
    if (mask2d && ((mB != 1 && mB != B) || (mH != 1 && mH != H))) return RF_ORACLE_BAD_SHAPE;
    double* scores = (double*)malloc(sizeof(double) * (size_t)(S * S > 0 ? S * S : 1));
    if (!scores) return RF_ORACLE_NOMEM;
    for (int64_t b = 0; b < B; ++b) {
        for (int64_t h = 0; h < H; ++h) {
            const size_t base = (size_t)((b * H + h) * S * d);
            const float* qp = q + base;
            const float* kp = k + base;
            const float* vp = v + base;
            float* op = out + base;
            const float* mp = NULL;
            if (mask2d) {
                const int64_t bb = mB == 1 ? 0 : b;
                const int64_t hh = mH == 1 ? 0 : h;
                mp = mask2d + (size_t)((bb * mH + hh) * S * S);
            }
            for (int64_t i = 0; i < S; ++i)
                for (int64_t j = 0; j < S; ++j) {
                    double dot = 0.0;
                    for (int64_t c = 0; c < d; ++c) dot += (double)qp[i * d + c] * (double)kp[j * d + c];
                    double s = dot * scale;
                    if (mp) s += (double)mp[i * S + j];
                    scores[i * S + j] = s;
                }
            for (int64_t i = 0; i < S; ++i) {
                double* row = scores + i * S;
                double row_max = -INFINITY;
                int any_live = 0;
                for (int64_t j = 0; j < S; ++j) {
                    if (!(mp && mp[i * S + j] <= RF_MASK_THRESHOLD)) any_live = 1;
                    if (row[j] > row_max) row_max = row[j];
                }
                if (!any_live) { /* attention.cpp:84-87 */
                    for (int64_t c = 0; c < d; ++c) op[i * d + c] = 0.0f;
                    continue;
                }
                double denom = 0.0;
                for (int64_t j = 0; j < S; ++j) {
                    row[j] = exp(row[j] - row_max);
                    denom += row[j];
                }
                for (int64_t c = 0; c < d; ++c) {
                    double a = 0.0;
                    for (int64_t j = 0; j < S; ++j) a += row[j] * (double)vp[j * d + c];
                    op[i * d + c] = (float)(a / denom);
                }
            }
        }
    }
    free(scores);
    return RF_ORACLE_OK;
}

/* window_to_mask2d (attention.cpp:215-242): mask[b,0,i,j] = live ? 0 : -65504.  Note that
 * live-but-nonzero bias values are dropped (written as 0), as in the reference (:237). */
int rf_oracle_window_to_mask2d(int64_t S, int64_t wl, int64_t wr, const float* pad_bias, int64_t B,
                               float* mask) {
    if (S < 1) return RF_ORACLE_BAD_SHAPE;
    for (int64_t b = 0; b < B; ++b) {
        const float* pad = pad_bias ? pad_bias + (size_t)(b * S) : NULL;
        float* mp = mask + (size_t)(b * S * S);
        for (int64_t i = 0; i < S; ++i)
            for (int64_t j = 0; j < S; ++j) {
                int live = window_ok(i, j, wl, wr);
                if (pad && pad[j] <= RF_MASK_THRESHOLD) live = 0;
                mp[i * S + j] = live ? 0.0f : RF_MASK_VALUE;
            }
    }
    return RF_ORACLE_OK;
}

/* Memory model (attention.cpp:244-252). */
uint64_t rf_oracle_mask_memory_bytes(uint64_t batch, uint64_t heads, uint64_t seq_len, uint64_t bpe) {
    return batch * heads * seq_len * seq_len * bpe;
}
uint64_t rf_oracle_fa_memory_bytes(uint64_t batch, uint64_t heads, uint64_t seq_len,
                                   uint64_t head_dim, uint64_t tile, uint64_t bpe) {
    return batch * heads * (2 * tile * head_dim + seq_len * head_dim) * bpe;
}

/* ---------------------------------------------------------------------------------------------
 * Independent double-precision SDPA, the reference TEST SUITE's own oracle
 * (tests/support/oracles.cpp:83-121): f64 inputs, no mask, plain softmax.
 * ------------------------------------------------------------------------------------------- */
int rf_oracle_sdpa_double_reference(const double* q, const double* k, const double* v, double* out,
                                    int64_t B, int64_t H, int64_t S, int64_t d, double scale) {
    double* row = (double*)malloc(sizeof(double) * (size_t)(S > 0 ? S : 1));
    if (!row) return RF_ORACLE_NOMEM;
    for (int64_t bh = 0; bh < B * H; ++bh) {
        const size_t base = (size_t)(bh * S * d);
        for (int64_t i = 0; i < S; ++i) {
            for (int64_t j = 0; j < S; ++j) {
                double dot = 0.0;
                for (int64_t c = 0; c < d; ++c) dot += q[base + i * d + c] * k[base + j * d + c];
                row[j] = dot * scale;
            }
            double mx = row[0];
            for (int64_t j = 0; j < S; ++j) mx = row[j] > mx ? row[j] : mx;
            double denom = 0.0;
            for (int64_t j = 0; j < S; ++j) {
                row[j] = exp(row[j] - mx);
                denom += row[j];
            }
            for (int64_t c = 0; c < d; ++c) {
                double a = 0.0;
                for (int64_t j = 0; j < S; ++j) a += row[j] * v[base + j * d + c];
                out[base + i * d + c] = a / denom;
            }
        }
    }
    free(row);
    return RF_ORACLE_OK;
}

/* window predicate used by the reference tests (tests/support/oracles.cpp:123-129). */
int rf_oracle_window_live_reference(int64_t i, int64_t j, int64_t wl, int64_t wr,
                                    const uint8_t* padded, int64_t n_padded) {
    if (wl != -1 && i - j > wl) return 0;
    if (wr != -1 && j - i > wr) return 0;
    if (n_padded > 0 && padded[j]) return 0;
    return 1;
}

/* ---------------------------------------------------------------------------------------------
 * Helpers that are OURS (not in the reference): input rounding shared by both sides of a
 * parity test, and the algorithmic work count of SURVEY.md section 8(d).
 * ------------------------------------------------------------------------------------------- */

/* f32 -> bf16 -> f32, round-to-nearest-even (what cvt.rn.bf16.f32 does). */
void rf_oracle_round_bf16_array(const float* in, float* out, int64_t n) {
    for (int64_t i = 0; i < n; ++i) {
        uint32_t b = f32_bits(in[i]);
        if ((b & 0x7F800000u) != 0x7F800000u) {
            const uint32_t lsb = (b >> 16) & 1u;
            b += 0x7FFFu + lsb;
        }
        b &= 0xFFFF0000u;
        out[i] = bits_f32(b);
    }
}

/* Number of live (query, key) pairs of one batch row: exactly the pairs the reference
 * multiplies (attention.cpp:160-167).  F = 4*d*H*sum_b live_pairs(b). */
uint64_t rf_oracle_live_pairs(int64_t S, int64_t wl, int64_t wr, const float* pad) {
    uint64_t n = 0;
    for (int64_t i = 0; i < S; ++i) {
        int64_t lo = wl >= 0 ? (i - wl > 0 ? i - wl : 0) : 0;
        int64_t hi = wr >= 0 ? (i + wr < S - 1 ? i + wr : S - 1) : S - 1;
        if (!pad) {
            if (hi >= lo) n += (uint64_t)(hi - lo + 1);
        } else {
            for (int64_t j = lo; j <= hi; ++j) n += pad[j] > RF_MASK_THRESHOLD;
        }
    }
    return n;
}
