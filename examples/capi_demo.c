/*
 * capi_demo.c -- a plain C host driving the B200 path through the C-ABI
 * only (include/rgbdseg_b200.h): no Python, no torch.  What a non-Python
 * caller of the reference's plugin boundary would write.
 *
 * usage: capi_demo {gmm|pbas} W H FRAMES SEED OUT.bin
 * Generates FRAMES deterministic synthetic RGB-D frames (an LCG background
 * with ~5 % depth holes and, from frame 22, a moving bright block), runs them through
 * rgbdseg_*_process_host, and writes the frames (FRAMES x H x W x 4), every
 * mask (FRAMES x H x W) and the final state field R_RGB (PBAS) / RGB_W (GMM)
 * to OUT.bin, so a test can replay the frames through the Python engine.
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "../include/rgbdseg_b200.h"

static uint32_t lcg(uint32_t* s) {
    *s = *s * 1664525u + 1013904223u;
    return *s >> 8;
}

/* frame t of the synthetic sequence, (H, W, 4) u8 r,g,b,d */
static void make_frame(uint8_t* f, int w, int h, int t, uint32_t seed) {
    uint32_t bg = seed * 2654435761u + 1u, nz = seed ^ (uint32_t)(t * 2246822519u);
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            uint8_t* px = f + 4 * ((size_t)y * w + x);
            for (int c = 0; c < 3; ++c) {
                int v = (int)(lcg(&bg) & 0xFF) + (int)(lcg(&nz) % 9) - 4;
                px[c] = (uint8_t)(v < 0 ? 0 : v > 255 ? 255 : v);
            }
            px[3] = (lcg(&nz) % 20 == 0) ? 0 : 155;
            const int bx = (t * 3) % (w > 8 ? w - 8 : 1), by = h / 3;
            if (t >= 22 && x >= bx && x < bx + 8 && y >= by && y < by + 6) {  /* after PBAS warm-up */
                px[0] = px[1] = px[2] = 240;
                px[3] = 75;
            }
        }
}

static int fail(const char* what) {
    fprintf(stderr, "%s: %s\n", what, rgbdseg_last_error());
    return 1;
}

int main(int argc, char** argv) {
    if (argc != 7) {
        fprintf(stderr, "usage: %s {gmm|pbas} W H FRAMES SEED OUT.bin\n", argv[0]);
        return 2;
    }
    const int pbas = strcmp(argv[1], "pbas") == 0;
    const int w = atoi(argv[2]), h = atoi(argv[3]), frames = atoi(argv[4]);
    const uint32_t seed = (uint32_t)strtoul(argv[5], NULL, 10);
    if (rgbdseg_device_count() < 1) {
        fprintf(stderr, "no CUDA device\n");
        return 3;
    }
    uint8_t* allf = malloc((size_t)w * h * 4 * frames);
    uint8_t* masks = malloc((size_t)w * h * frames);
    rgbdseg_gmm* g = NULL;
    rgbdseg_pbas* p = NULL;
    if (pbas) {
        /* PbasParams defaults (pbas.py:45-55) */
        rgbdseg_pbas_params prm = {20, 2, 18.0, 18.0, 5.0, 0.05, 18.0, 2.0, 200.0, 1.0, 0.05};
        if (rgbdseg_pbas_create(w, h, &prm, 1, (uint64_t)seed + 1, 0, &p)) return fail("pbas_create");
    } else {
        /* GmmParams defaults (gmm.py:45-52) */
        rgbdseg_gmm_params prm = {7, 3, 0.001, 10000.0, 1.0, 2.5, 225.0, 0.05};
        if (rgbdseg_gmm_create(w, h, &prm, 1, 0, &g)) return fail("gmm_create");
    }
    for (int t = 0; t < frames; ++t) {
        uint8_t* frame = allf + (size_t)t * w * h * 4;
        make_frame(frame, w, h, t, seed);
        uint8_t* m = masks + (size_t)t * w * h;
        if (pbas ? rgbdseg_pbas_process_host(p, frame, m, 1) : rgbdseg_gmm_process_host(g, frame, m, 1))
            return fail("process_host");
    }
    const int field = pbas ? RGBDSEG_PBAS_R_RGB : RGBDSEG_GMM_RGB_W;
    const int64_t nb = pbas ? rgbdseg_pbas_state_bytes(p, field) : rgbdseg_gmm_state_bytes(g, field);
    uint8_t* st = malloc((size_t)nb);
    if (pbas ? rgbdseg_pbas_read_state(p, field, st, nb) : rgbdseg_gmm_read_state(g, field, st, nb))
        return fail("read_state");
    FILE* out = fopen(argv[6], "wb");
    if (!out) return fail("open output");
    fwrite(allf, 1, (size_t)w * h * 4 * frames, out);
    fwrite(masks, 1, (size_t)w * h * frames, out);
    fwrite(st, 1, (size_t)nb, out);
    fclose(out);
    uint64_t fg = 0;
    for (size_t i = 0; i < (size_t)w * h * frames; ++i) fg += masks[i] != 0;
    printf("%s %dx%d x %d frames: %llu foreground pixels, state %lld bytes\n", argv[1], w, h, frames,
           (unsigned long long)fg, (long long)nb);
    if (pbas)
        rgbdseg_pbas_destroy(p);
    else
        rgbdseg_gmm_destroy(g);
    free(allf);
    free(masks);
    free(st);
    return 0;
}
