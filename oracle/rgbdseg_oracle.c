/*
 * rgbdseg_oracle.c -- CPU restatement of the reference per-pixel RGB-D
 * segmentation (GMM + PBAS + counter-based RNG).
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product package
 * (paper_2002_00250_b200/) links, imports or executes this file.  It is used
 * exclusively by tests/ (as the parity checker), by __graft_entry__.smoke()
 * (as the checker of the smoke run) and by bench.py's cpu_baseline leg /
 * `--impl reference` arm (as the timed CPU implementation of the path).
 *
 * It restates, expression for expression, the reference's numba kernels:
 *   - _mix64 / pixel_rng_nb      reference pkg/src/rgbdseg/engine_rng.py:29-44
 *   - _gmm_sub_step / _gmm_band  reference pkg/src/rgbdseg/gmm.py:283-368
 *   - _pbas_band                 reference pkg/src/rgbdseg/pbas.py:344-508
 *   - _apply_intents             reference pkg/src/rgbdseg/pbas.py:511-522
 *   - band split / intent order  reference pkg/src/rgbdseg/engine.py:48-50,114-143
 * State arrays use the reference layout (C order, per-pixel contiguous):
 *   rgb_w (H,W,K) rgb_mu (H,W,K,3) rgb_var (H,W,K) d_w (H,W,Kd) d_mu (H,W,Kd,1)
 *   d_var (H,W,Kd); samples (H,W,n,4) u8, dmin_* (H,W,n) u8, len/pos (H,W) u8,
 *   r_rgb/r_d/t (H,W) f64  (gmm.py:244-249, pbas.py:285-294).
 *
 * Parity pin: the fixtures under tests/golden/ were produced by the reference itself
 * (tests/golden/make_golden.py); tests/test_oracle_golden.py checks this
 * restatement against them bit for bit.
 *
 * Build: oracle/Makefile (gcc -O2 -ffp-contract=off: numba emits no FMA,
 * see SURVEY.md App. B; `exp` is libm's, exactly what numba's llvm.exp.f64
 * lowers to on the same host).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define VAR_FLOOR 1.0 /* gmm.py:34 */

/* ---------------------------------------------------------------- RNG --- */
/* engine_rng.py:15-26 */
#define SALT 0x5851F42D4C957F2DULL
#define K_X 0x9E3779B97F4A7C15ULL
#define K_Y 0xC2B2AE3D27D4EB4FULL
#define K_F 0x165667B19E3779F9ULL
#define K_D 0xD6E8FEB86659FD93ULL
#define M1 0xBF58476D1CE4E5B9ULL
#define M2 0x94D049BB133111EBULL

/* engine_rng.py:29-33 */
static inline uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * M1;
    z = (z ^ (z >> 27)) * M2;
    return z ^ (z >> 31);
}

/* engine_rng.py:36-44 */
double oracle_pixel_rng(uint64_t seed, uint64_t x, uint64_t y, uint64_t f, uint64_t d) {
    uint64_t h = seed ^ SALT;
    h = mix64(h ^ (x * K_X));
    h = mix64(h ^ (y * K_Y));
    h = mix64(h ^ (f * K_F));
    h = mix64(h ^ (d * K_D));
    return (double)(h >> 11) * (1.0 / 9007199254740992.0);
}

/* engine_rng.py:47-52 */
void oracle_rng_stream(uint64_t seed, uint64_t x, uint64_t y, uint64_t f, int64_t count,
                       double* out) {
    for (int64_t i = 0; i < count; ++i) out[i] = oracle_pixel_rng(seed, x, y, f, (uint64_t)i);
}

/* ---------------------------------------------------------------- GMM --- */
typedef struct {
    double alpha, s, tau, lam2, var_init, w_init;
} gmm_consts;

/* gmm.py:283-347 (_gmm_sub_step): seed / fused score+match scan / update /
 * renormalise / floor.  mu is [k][nc]. */
static double gmm_sub_step(const double* xv, int nc, double* w, double* mu, double* var, int nk,
                           const gmm_consts* c) {
    const double PI2 = 2.0 * 3.141592653589793; /* 2.0 * math.pi */
    if (w[0] == 0.0) { /* gmm.py:291-295 */
        w[0] = 1.0;
        for (int ch = 0; ch < nc; ++ch) mu[ch] = xv[ch];
        var[0] = c->var_init;
    }
    double p = 0.0; /* gmm.py:298-315 */
    int m = -1;
    double best_w = -1.0;
    double d2m = 0.0;
    for (int k = 0; k < nk; ++k) {
        double wk = w[k];
        if (wk <= 0.0) continue;
        double d2 = 0.0;
        for (int ch = 0; ch < nc; ++ch) {
            double dd = xv[ch] - mu[k * nc + ch];
            d2 += dd * dd;
        }
        double v = var[k];
        p += wk * ((c->s / (PI2 * v)) * exp(-(d2 / (2.0 * v))));
        if (d2 < c->lam2 * v && wk > best_w) {
            m = k;
            best_w = wk;
            d2m = d2;
        }
    }
    if (m >= 0) { /* gmm.py:317-325 */
        for (int k = 0; k < nk; ++k) {
            double wn = (1.0 - c->alpha) * w[k];
            if (k == m) wn += c->alpha;
            w[k] = wn;
        }
        for (int ch = 0; ch < nc; ++ch)
            mu[m * nc + ch] = (1.0 - c->alpha) * mu[m * nc + ch] + c->alpha * xv[ch];
        var[m] = (1.0 - c->alpha) * var[m] + c->alpha * d2m;
    } else { /* gmm.py:326-337 */
        int r = 0;
        double best = INFINITY;
        for (int k = 0; k < nk; ++k) {
            double f = w[k] / sqrt(var[k]);
            if (f < best) {
                best = f;
                r = k;
            }
        }
        w[r] = c->w_init;
        for (int ch = 0; ch < nc; ++ch) mu[r * nc + ch] = xv[ch];
        var[r] = c->var_init;
    }
    double total = 0.0; /* gmm.py:339-346 */
    for (int k = 0; k < nk; ++k) total += w[k];
    for (int k = 0; k < nk; ++k) w[k] = w[k] / total;
    for (int k = 0; k < nk; ++k)
        if (var[k] < VAR_FLOOR) var[k] = VAR_FLOOR;
    return p;
}

/* gmm.py:350-368 (_gmm_band) over rows [y0, y1). */
void oracle_gmm_band(int64_t width, int64_t height, const uint8_t* frame, int64_t y0, int64_t y1,
                     double* rgb_w, double* rgb_mu, double* rgb_var, double* d_w, double* d_mu,
                     double* d_var, int32_t k_rgb, int32_t k_d, double alpha, double s, double tau,
                     double lam2, double var_init, double w_init, int32_t use_depth,
                     uint8_t* mask) {
    (void)height;
    gmm_consts c = {alpha, s, tau, lam2, var_init, w_init};
    double xrgb[3], xd[1];
    for (int64_t y = y0; y < y1; ++y) {
        for (int64_t x = 0; x < width; ++x) {
            int64_t pix = y * width + x;
            const uint8_t* px = frame + pix * 4;
            xrgb[0] = px[0];
            xrgb[1] = px[1];
            xrgb[2] = px[2];
            double p = gmm_sub_step(xrgb, 3, rgb_w + pix * k_rgb, rgb_mu + pix * k_rgb * 3,
                                    rgb_var + pix * k_rgb, k_rgb, &c);
            if (use_depth && px[3] > 0) {
                xd[0] = px[3];
                double pd = gmm_sub_step(xd, 1, d_w + pix * k_d, d_mu + pix * k_d,
                                         d_var + pix * k_d, k_d, &c);
                p = p * pd;
            }
            mask[pix] = (p >= tau) ? 0 : 255;
        }
    }
}

/* ---------------------------------------------------------------- PBAS -- */
typedef struct {
    int64_t width, height;
    const uint8_t* frame;
    int64_t frame_idx;
    uint8_t *samples, *dmin_rgb, *dmin_d, *len_rgb, *pos_rgb, *len_d, *pos_d;
    double *r_rgb, *r_d, *t;
    uint64_t seed;
    int32_t n, min_matches;
    double r_lower, r_scale, r_inc_dec, t_lower, t_upper, t_inc, t_dec;
    int32_t use_depth;
    uint8_t* mask;
    /* opt-in gradient feature (NOT in the reference, see oracle_pbas_frame_g);
     * gsamples == NULL: off */
    uint8_t* gsamples;   /* (H,W,n) u8 gradient magnitude of every sample */
    const uint8_t* gmap; /* (H,W) u8 this frame's gradient magnitudes */
    int64_t gw;          /* the frame's gradient weight in 1/256 units */
} pbas_args;

static const int NBR_DY[8] = {-1, -1, -1, 0, 0, 1, 1, 1}; /* pbas.py:34,340-341 */
static const int NBR_DX[8] = {-1, 0, 1, -1, 1, -1, 0, 1};

static inline int64_t iabs64(int64_t v) { return v < 0 ? -v : v; }

/* pbas.py:344-508 (_pbas_band) over rows [y0, y1) with GLOBAL coordinates;
 * intents (ny, nx, slot) are appended in row-major emission order. */
static int64_t pbas_band(const pbas_args* a, int64_t y0, int64_t y1, int64_t* intents,
                         int64_t* emitters) {
    const int64_t width = a->width, height = a->height, n = a->n;
    int64_t n_intents = 0;
    for (int64_t y = y0; y < y1; ++y) {
        for (int64_t x = 0; x < width; ++x) {
            int64_t pix = y * width + x;
            const uint8_t* px = a->frame + pix * 4;
            uint8_t r = px[0], g = px[1], b = px[2];
            uint8_t d = a->use_depth ? px[3] : 0; /* pbas.py:367 */
            uint8_t* smp = a->samples + pix * n * 4;

            if (a->frame_idx < n) { /* pbas.py:369-376 */
                uint8_t* s = smp + a->frame_idx * 4;
                s[0] = r;
                s[1] = g;
                s[2] = b;
                s[3] = d;
                if (a->gsamples) a->gsamples[pix * n + a->frame_idx] = a->gmap[pix];
                a->mask[pix] = 0;
                continue;
            }

            int64_t cnt = 0, dminr = 255; /* pbas.py:378-396 */
            double rr = a->r_rgb[pix];
            if (!a->gsamples) {
                for (int64_t i = 0; i < n; ++i) {
                    const uint8_t* s = smp + i * 4;
                    int64_t dr = iabs64((int64_t)r - (int64_t)s[0]);
                    int64_t dg = iabs64((int64_t)g - (int64_t)s[1]);
                    int64_t db = iabs64((int64_t)b - (int64_t)s[2]);
                    int64_t dist = dr;
                    if (dg > dist) dist = dg;
                    if (db > dist) dist = db;
                    if ((double)dist < rr) cnt += 1;
                    if (dist < dminr) dminr = dist;
                }
            } else { /* gradient feature: 256 dist + gw |gm - gm_i| against 256 R */
                const int64_t gm = a->gmap[pix];
                const uint8_t* gs = a->gsamples + pix * n;
                int64_t dmin256 = 255 * 256;
                for (int64_t i = 0; i < n; ++i) {
                    const uint8_t* s = smp + i * 4;
                    int64_t dr = iabs64((int64_t)r - (int64_t)s[0]);
                    int64_t dg = iabs64((int64_t)g - (int64_t)s[1]);
                    int64_t db = iabs64((int64_t)b - (int64_t)s[2]);
                    int64_t dist = dr;
                    if (dg > dist) dist = dg;
                    if (db > dist) dist = db;
                    int64_t dd = 256 * dist + a->gw * iabs64(gm - (int64_t)gs[i]);
                    if ((double)dd < 256.0 * rr) cnt += 1; /* both sides exact */
                    if (dd < dmin256) dmin256 = dd;
                }
                dminr = dmin256 >> 8; /* ring entry: floor(min / 256) <= 255 */
            }
            int bg_rgb = cnt >= a->min_matches;

            int depth_eval = 0, bg_depth = 1; /* pbas.py:398-419 */
            int64_t dmind = 255;
            if (d > 0) {
                int64_t valid = 0, cntd = 0;
                double rd = a->r_d[pix];
                for (int64_t i = 0; i < n; ++i) {
                    uint8_t sd = smp[i * 4 + 3];
                    if (sd == 0) continue;
                    valid += 1;
                    int64_t dist = iabs64((int64_t)d - (int64_t)sd);
                    if ((double)dist < rd) cntd += 1;
                    if (dist < dmind) dmind = dist;
                }
                if (valid >= a->min_matches) {
                    depth_eval = 1;
                    bg_depth = cntd >= a->min_matches;
                }
            }

            int fg = (!bg_rgb) || (depth_eval && !bg_depth); /* pbas.py:421-422 */
            a->mask[pix] = fg ? 255 : 0;

            /* pbas.py:424-438: RGB dmin ring + R_rgb */
            uint8_t* ringr = a->dmin_rgb + pix * n;
            ringr[a->pos_rgb[pix]] = (uint8_t)dminr;
            a->pos_rgb[pix] = (uint8_t)((a->pos_rgb[pix] + 1) % n);
            if (a->len_rgb[pix] < n) a->len_rgb[pix] += 1;
            int64_t total = 0;
            for (int64_t i = 0; i < a->len_rgb[pix]; ++i) total += ringr[i];
            double avg_rgb = (double)total / (double)a->len_rgb[pix];
            if (a->r_rgb[pix] > avg_rgb * a->r_scale)
                a->r_rgb[pix] = a->r_rgb[pix] * (1.0 - a->r_inc_dec);
            else
                a->r_rgb[pix] = a->r_rgb[pix] * (1.0 + a->r_inc_dec);
            if (a->r_rgb[pix] < a->r_lower) a->r_rgb[pix] = a->r_lower;

            if (depth_eval) { /* pbas.py:440-454 */
                uint8_t* ringd = a->dmin_d + pix * n;
                ringd[a->pos_d[pix]] = (uint8_t)dmind;
                a->pos_d[pix] = (uint8_t)((a->pos_d[pix] + 1) % n);
                if (a->len_d[pix] < n) a->len_d[pix] += 1;
                int64_t totd = 0;
                for (int64_t i = 0; i < a->len_d[pix]; ++i) totd += ringd[i];
                double avg_d = (double)totd / (double)a->len_d[pix];
                if (a->r_d[pix] > avg_d * a->r_scale)
                    a->r_d[pix] = a->r_d[pix] * (1.0 - a->r_inc_dec);
                else
                    a->r_d[pix] = a->r_d[pix] * (1.0 + a->r_inc_dec);
                if (a->r_d[pix] < a->r_lower) a->r_d[pix] = a->r_lower;
            }

            double guard = avg_rgb > 1.0 ? avg_rgb : 1.0; /* pbas.py:456-465 */
            if (fg)
                a->t[pix] = a->t[pix] + a->t_inc / guard;
            else
                a->t[pix] = a->t[pix] - a->t_dec / guard;
            if (a->t[pix] < a->t_lower)
                a->t[pix] = a->t_lower;
            else if (a->t[pix] > a->t_upper)
                a->t[pix] = a->t_upper;

            if (!fg) { /* pbas.py:467-507 */
                double prob = 1.0 / a->t[pix];
                double u0 = oracle_pixel_rng(a->seed, (uint64_t)x, (uint64_t)y,
                                             (uint64_t)a->frame_idx, 0);
                if (u0 < prob) {
                    int64_t slot = (int64_t)((u0 / prob) * (double)n);
                    if (slot >= n) slot = n - 1;
                    uint8_t* s = smp + slot * 4;
                    s[0] = r;
                    s[1] = g;
                    s[2] = b;
                    s[3] = d;
                    if (a->gsamples) a->gsamples[pix * n + slot] = a->gmap[pix];
                }
                double u1 = oracle_pixel_rng(a->seed, (uint64_t)x, (uint64_t)y,
                                             (uint64_t)a->frame_idx, 1);
                if (u1 < prob) {
                    int64_t m = 0;
                    for (int j = 0; j < 8; ++j) {
                        int64_t ny = y + NBR_DY[j], nx = x + NBR_DX[j];
                        if (0 <= ny && ny < height && 0 <= nx && nx < width) m += 1;
                    }
                    int64_t pick = (int64_t)((u1 / prob) * (double)m);
                    if (pick >= m) pick = m - 1;
                    double u2 = oracle_pixel_rng(a->seed, (uint64_t)x, (uint64_t)y,
                                                 (uint64_t)a->frame_idx, 2);
                    int64_t slot = (int64_t)(u2 * (double)n);
                    if (slot >= n) slot = n - 1;
                    int64_t seen = 0;
                    for (int j = 0; j < 8; ++j) {
                        int64_t ny = y + NBR_DY[j], nx = x + NBR_DX[j];
                        if (0 <= ny && ny < height && 0 <= nx && nx < width) {
                            if (seen == pick) {
                                intents[n_intents * 3 + 0] = ny;
                                intents[n_intents * 3 + 1] = nx;
                                intents[n_intents * 3 + 2] = slot;
                                if (emitters) { /* test hook: who asked (row-band halo tests) */
                                    emitters[n_intents * 2 + 0] = y;
                                    emitters[n_intents * 2 + 1] = x;
                                }
                                n_intents += 1;
                                break;
                            }
                            seen += 1;
                        }
                    }
                }
            }
        }
    }
    return n_intents;
}

/* pbas.py:511-522 (_apply_intents) */
void oracle_pbas_apply_intents(int64_t width, int32_t n, uint8_t* samples, const uint8_t* frame,
                               const int64_t* intents, int64_t count, int32_t use_depth) {
    for (int64_t i = 0; i < count; ++i) {
        int64_t y = intents[i * 3 + 0], x = intents[i * 3 + 1], slot = intents[i * 3 + 2];
        int64_t pix = y * width + x;
        uint8_t* s = samples + (pix * n + slot) * 4;
        const uint8_t* px = frame + pix * 4;
        s[0] = px[0];
        s[1] = px[1];
        s[2] = px[2];
        s[3] = use_depth ? px[3] : 0;
    }
}

/* _apply_intents plus the gradient feature: the target's own magnitude. */
static void apply_intents_g(int64_t width, int32_t n, uint8_t* samples, const uint8_t* frame,
                            const int64_t* intents, int64_t count, int32_t use_depth,
                            uint8_t* gsamples, const uint8_t* gmap) {
    oracle_pbas_apply_intents(width, n, samples, frame, intents, count, use_depth);
    if (!gsamples) return;
    for (int64_t i = 0; i < count; ++i) {
        int64_t pix = intents[i * 3 + 0] * width + intents[i * 3 + 1];
        gsamples[pix * n + intents[i * 3 + 2]] = gmap[pix];
    }
}

/* Public single-band entry: the reference's PbasState.segment_rows
 * (pbas.py:320-333).  Returns the number of intents written. */
int64_t oracle_pbas_band(int64_t width, int64_t height, const uint8_t* frame, int64_t frame_idx,
                         int64_t y0, int64_t y1, uint8_t* samples, uint8_t* dmin_rgb,
                         uint8_t* dmin_d, uint8_t* len_rgb, uint8_t* pos_rgb, uint8_t* len_d,
                         uint8_t* pos_d, double* r_rgb, double* r_d, double* t, uint64_t seed,
                         int32_t n, int32_t min_matches, double r_lower, double r_scale,
                         double r_inc_dec, double t_lower, double t_upper, double t_inc,
                         double t_dec, int32_t use_depth, uint8_t* mask, int64_t* intents) {
    pbas_args a = {width, height,  frame,   frame_idx, samples, dmin_rgb,  dmin_d,
                   len_rgb, pos_rgb, len_d, pos_d,   r_rgb,   r_d,       t,
                   seed,  n,       min_matches, r_lower, r_scale, r_inc_dec, t_lower,
                   t_upper, t_inc, t_dec,   use_depth, mask, NULL, NULL, 0};
    return pbas_band(&a, y0, y1, intents, NULL);
}

/* Same as oracle_pbas_band, also recording each intent's emitter (y, x):
 * used by the row-band halo tests to rebuild per-emitter intent codes. */
int64_t oracle_pbas_band_emit(int64_t width, int64_t height, const uint8_t* frame,
                              int64_t frame_idx, int64_t y0, int64_t y1, uint8_t* samples,
                              uint8_t* dmin_rgb, uint8_t* dmin_d, uint8_t* len_rgb,
                              uint8_t* pos_rgb, uint8_t* len_d, uint8_t* pos_d, double* r_rgb,
                              double* r_d, double* t, uint64_t seed, int32_t n,
                              int32_t min_matches, double r_lower, double r_scale,
                              double r_inc_dec, double t_lower, double t_upper, double t_inc,
                              double t_dec, int32_t use_depth, uint8_t* mask, int64_t* intents,
                              int64_t* emitters) {
    pbas_args a = {width, height,  frame,   frame_idx, samples, dmin_rgb,  dmin_d,
                   len_rgb, pos_rgb, len_d, pos_d,   r_rgb,   r_d,       t,
                   seed,  n,       min_matches, r_lower, r_scale, r_inc_dec, t_lower,
                   t_upper, t_inc, t_dec,   use_depth, mask, NULL, NULL, 0};
    return pbas_band(&a, y0, y1, intents, emitters);
}

/* ------------------------------------------------- multi-threaded frames - */
/* The reference engine's row-band split (engine.py:48-50):
 * edges = np.linspace(0, H, workers+1).astype(int64). */
static void band_bounds(int64_t height, int workers, int64_t* edges) {
    double step = (double)height / (double)workers; /* numpy linspace: i*step + start */
    for (int i = 0; i <= workers; ++i) {
        double v = (double)i * step;
        if (i == workers) v = (double)height;
        edges[i] = (int64_t)v;
    }
}

typedef struct {
    int kind; /* 0 gmm, 1 pbas */
    int64_t y0, y1;
    /* gmm */
    int64_t width, height;
    const uint8_t* frame;
    double *rgb_w, *rgb_mu, *rgb_var, *d_w, *d_mu, *d_var;
    int32_t k_rgb, k_d;
    double alpha, s, tau, lam2, var_init, w_init;
    int32_t use_depth;
    uint8_t* mask;
    /* pbas */
    const pbas_args* pa;
    int64_t* intents;
    int64_t count;
} band_job;

static void* band_worker(void* p) {
    band_job* j = (band_job*)p;
    if (j->kind == 0)
        oracle_gmm_band(j->width, j->height, j->frame, j->y0, j->y1, j->rgb_w, j->rgb_mu,
                        j->rgb_var, j->d_w, j->d_mu, j->d_var, j->k_rgb, j->k_d, j->alpha, j->s,
                        j->tau, j->lam2, j->var_init, j->w_init, j->use_depth, j->mask);
    else
        j->count = pbas_band(j->pa, j->y0, j->y1, j->intents, NULL);
    return NULL;
}

/* One GMM frame over `workers` row bands on pthreads (engine.py:114-124). */
int oracle_gmm_frame(int64_t width, int64_t height, const uint8_t* frame, double* rgb_w,
                     double* rgb_mu, double* rgb_var, double* d_w, double* d_mu, double* d_var,
                     int32_t k_rgb, int32_t k_d, double alpha, double s, double tau, double lam2,
                     double var_init, double w_init, int32_t use_depth, uint8_t* mask,
                     int32_t workers) {
    if (workers < 1) workers = 1;
    int64_t* edges = (int64_t*)malloc(sizeof(int64_t) * (workers + 1));
    band_job* jobs = (band_job*)calloc(workers, sizeof(band_job));
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * workers);
    if (!edges || !jobs || !th) return -1;
    band_bounds(height, workers, edges);
    for (int i = 0; i < workers; ++i) {
        band_job* j = &jobs[i];
        j->kind = 0;
        j->y0 = edges[i];
        j->y1 = edges[i + 1];
        j->width = width;
        j->height = height;
        j->frame = frame;
        j->rgb_w = rgb_w;
        j->rgb_mu = rgb_mu;
        j->rgb_var = rgb_var;
        j->d_w = d_w;
        j->d_mu = d_mu;
        j->d_var = d_var;
        j->k_rgb = k_rgb;
        j->k_d = k_d;
        j->alpha = alpha;
        j->s = s;
        j->tau = tau;
        j->lam2 = lam2;
        j->var_init = var_init;
        j->w_init = w_init;
        j->use_depth = use_depth;
        j->mask = mask;
    }
    for (int i = 1; i < workers; ++i) pthread_create(&th[i], NULL, band_worker, &jobs[i]);
    band_worker(&jobs[0]);
    for (int i = 1; i < workers; ++i) pthread_join(th[i], NULL);
    free(edges);
    free(jobs);
    free(th);
    return 0;
}

/* One PBAS frame over `workers` row bands, then the sequential intent phase
 * in band order (engine.py:126-143).  Returns total intents applied. */
static int64_t pbas_frame_run(const pbas_args* a, int32_t workers) {
    const int64_t width = a->width, height = a->height;
    const int32_t n = a->n, use_depth = a->use_depth;
    uint8_t* samples = a->samples;
    const uint8_t* frame = a->frame;
    if (workers < 1) workers = 1;
    int64_t* edges = (int64_t*)malloc(sizeof(int64_t) * (workers + 1));
    band_job* jobs = (band_job*)calloc(workers, sizeof(band_job));
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * workers);
    if (!edges || !jobs || !th) return -1;
    band_bounds(height, workers, edges);
    for (int i = 0; i < workers; ++i) {
        band_job* j = &jobs[i];
        j->kind = 1;
        j->y0 = edges[i];
        j->y1 = edges[i + 1];
        j->pa = a;
        int64_t rows = j->y1 - j->y0;
        j->intents = (int64_t*)malloc(sizeof(int64_t) * 3 * (rows * width + 1));
        if (!j->intents) return -1;
    }
    for (int i = 1; i < workers; ++i) pthread_create(&th[i], NULL, band_worker, &jobs[i]);
    band_worker(&jobs[0]);
    for (int i = 1; i < workers; ++i) pthread_join(th[i], NULL);
    int64_t total = 0;
    for (int i = 0; i < workers; ++i) {
        apply_intents_g(width, n, samples, frame, jobs[i].intents, jobs[i].count, use_depth,
                        a->gsamples, a->gmap);
        total += jobs[i].count;
        free(jobs[i].intents);
    }
    free(edges);
    free(jobs);
    free(th);
    return total;
}

int64_t oracle_pbas_frame(int64_t width, int64_t height, const uint8_t* frame, int64_t frame_idx,
                          uint8_t* samples, uint8_t* dmin_rgb, uint8_t* dmin_d, uint8_t* len_rgb,
                          uint8_t* pos_rgb, uint8_t* len_d, uint8_t* pos_d, double* r_rgb,
                          double* r_d, double* t, uint64_t seed, int32_t n, int32_t min_matches,
                          double r_lower, double r_scale, double r_inc_dec, double t_lower,
                          double t_upper, double t_inc, double t_dec, int32_t use_depth,
                          uint8_t* mask, int32_t workers) {
    pbas_args a = {width, height,  frame,   frame_idx, samples, dmin_rgb,  dmin_d,
                   len_rgb, pos_rgb, len_d, pos_d,   r_rgb,   r_d,       t,
                   seed,  n,       min_matches, r_lower, r_scale, r_inc_dec, t_lower,
                   t_upper, t_inc, t_dec,   use_depth, mask, NULL, NULL, 0};
    return pbas_frame_run(&a, workers);
}

/* ------------------------------------------- opt-in gradient feature ----
 * NOT part of the reference (SPEC.md:314 omits the original PBAS gradient
 * term); this package's definition, restated here as the checker of the
 * device path (csrc/pbas.cu K2G) -- parity for it is against this
 * restatement only:
 *   g(x,y) = max over r,g,b of (|Sx| + |Sy|) >> 3, the 3x3 Sobel responses
 *            with coordinates clamped into the frame (replicated border);
 *   sample distance (RGB group), in 1/256 units:
 *            D_i = 256 dist_i + w |g - g_i|, a match when D_i < 256 R
 *            (exact: D_i < 2^24 and 256 R are both exact doubles), with the
 *            frame's integer weight w = min(65535, floor(alpha * 256 / m +
 *            0.5)), m = max(mean, 1), mean = the previous frame's mean g
 *            (prev_sum / (W H), f64) or mean_init before the first frame;
 *   dmin ring entry = floor(min_i D_i / 256), capped at 255;
 *   every sample write also stores the magnitude of the pixel observed.
 * Returns the frame's magnitude sum. */
uint64_t oracle_pbas_gradient_map(int64_t width, int64_t height, const uint8_t* frame,
                                  uint8_t* gmap) {
    uint64_t sum = 0;
    for (int64_t y = 0; y < height; ++y) {
        for (int64_t x = 0; x < width; ++x) {
            int64_t ys[3], xs[3];
            for (int k = 0; k < 3; ++k) {
                int64_t yy = y - 1 + k, xx = x - 1 + k;
                ys[k] = yy < 0 ? 0 : (yy >= height ? height - 1 : yy);
                xs[k] = xx < 0 ? 0 : (xx >= width ? width - 1 : xx);
            }
            int64_t best = 0;
            for (int c = 0; c < 3; ++c) {
#define PX(i, j) ((int64_t)frame[(ys[i] * width + xs[j]) * 4 + c])
                int64_t sx = (PX(0, 2) + 2 * PX(1, 2) + PX(2, 2)) - (PX(0, 0) + 2 * PX(1, 0) + PX(2, 0));
                int64_t sy = (PX(2, 0) + 2 * PX(2, 1) + PX(2, 2)) - (PX(0, 0) + 2 * PX(0, 1) + PX(0, 2));
#undef PX
                int64_t m = iabs64(sx) + iabs64(sy);
                if (m > best) best = m;
            }
            gmap[y * width + x] = (uint8_t)(best >> 3);
            sum += (uint64_t)(best >> 3);
        }
    }
    return sum;
}

/* The frame's weight w from the previous frame's magnitude sum. */
uint32_t oracle_pbas_gradient_weight(uint64_t prev_sum, int64_t npix, double alpha,
                                     double mean_init) {
    const double mean = prev_sum == UINT64_MAX ? mean_init : (double)prev_sum / (double)npix;
    const double q = floor(alpha * 256.0 / (mean > 1.0 ? mean : 1.0) + 0.5);
    return q > 65535.0 ? 65535u : (uint32_t)q;
}

/* One PBAS frame with the gradient feature.  *prev_sum: the previous frame's
 * magnitude sum (UINT64_MAX before the first frame); updated to this
 * frame's.  gmap_out (H*W u8, may be NULL) receives the magnitude map. */
int64_t oracle_pbas_frame_g(int64_t width, int64_t height, const uint8_t* frame, int64_t frame_idx,
                            uint8_t* samples, uint8_t* dmin_rgb, uint8_t* dmin_d, uint8_t* len_rgb,
                            uint8_t* pos_rgb, uint8_t* len_d, uint8_t* pos_d, double* r_rgb,
                            double* r_d, double* t, uint64_t seed, int32_t n, int32_t min_matches,
                            double r_lower, double r_scale, double r_inc_dec, double t_lower,
                            double t_upper, double t_inc, double t_dec, int32_t use_depth,
                            uint8_t* mask, int32_t workers, uint8_t* gsamples, uint64_t* prev_sum,
                            double alpha, double mean_init, uint8_t* gmap_out) {
    uint8_t* gmap = gmap_out ? gmap_out : (uint8_t*)malloc((size_t)(width * height));
    if (!gmap) return -1;
    const uint64_t sum = oracle_pbas_gradient_map(width, height, frame, gmap);
    pbas_args a = {width, height,  frame,   frame_idx, samples, dmin_rgb,  dmin_d,
                   len_rgb, pos_rgb, len_d, pos_d,   r_rgb,   r_d,       t,
                   seed,  n,       min_matches, r_lower, r_scale, r_inc_dec, t_lower,
                   t_upper, t_inc, t_dec,   use_depth, mask, gsamples, gmap,
                   (int64_t)oracle_pbas_gradient_weight(*prev_sum, width * height, alpha,
                                                        mean_init)};
    int64_t rc = pbas_frame_run(&a, workers);
    *prev_sum = sum;
    if (!gmap_out) free(gmap);
    return rc;
}
