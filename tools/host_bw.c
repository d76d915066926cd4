// Host write-bandwidth probe: how fast can the host cores expand 0/1 bit
// planes into float32 observation arrays (the e2e contract's host buffers)?
//   gcc -O3 -march=native -fopenmp tools/host_bw.c -o /tmp/host_bw && /tmp/host_bw [GB]
#include <immintrin.h>
#include <omp.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

static double now(void) {
    struct timespec t;
    clock_gettime(CLOCK_MONOTONIC, &t);
    return t.tv_sec + 1e-9 * t.tv_nsec;
}

int main(int argc, char **argv) {
    double gb = argc > 1 ? atof(argv[1]) : 4.0;
    size_t nf = (size_t)(gb * 1e9 / 4) & ~(size_t)255;
    float *dst = aligned_alloc(64, nf * 4);
    uint32_t *bits = aligned_alloc(64, nf / 8);
    for (size_t i = 0; i < nf / 32; i++) bits[i] = (uint32_t)(i * 2654435761u);
#pragma omp parallel for schedule(static)
    for (size_t i = 0; i < nf; i += 1024) dst[i] = 0.f;  // first touch
    int maxt = omp_get_max_threads();
    for (int th = 1; th <= maxt; th *= 2) {
        for (int mode = 0; mode < 4; mode++) {
            double best = 1e9;
            for (int rep = 0; rep < 3; rep++) {
                double t0 = now();
#pragma omp parallel for num_threads(th) schedule(static)
                for (size_t w = 0; w < nf / 32; w++) {
                    uint32_t x = bits[w];
                    float *o = dst + w * 32;
                    if (mode == 3) {  // AVX-512: one 64-byte NT store per 16 elements
                        for (int k = 0; k < 2; k++) {
                            __mmask16 m = (__mmask16)((x >> (16 * k)) & 0xFFFF);
                            __m512 f = _mm512_maskz_mov_ps(m, _mm512_set1_ps(1.0f));
                            _mm512_stream_ps(o + 16 * k, f);
                        }
                    } else if (mode == 0) {  // plain NT store of zeros (write ceiling)
                        __m256 z = _mm256_setzero_ps();
                        for (int k = 0; k < 4; k++) _mm256_stream_ps(o + 8 * k, z);
                    } else {
                        const __m256i sh = _mm256_setr_epi32(1, 2, 4, 8, 16, 32, 64, 128);
                        for (int k = 0; k < 4; k++) {
                            __m256i v = _mm256_set1_epi32((int)((x >> (8 * k)) & 255));
                            __m256i m = _mm256_cmpeq_epi32(_mm256_and_si256(v, sh), sh);
                            __m256 f = _mm256_and_ps(_mm256_castsi256_ps(m), _mm256_set1_ps(1.0f));
                            if (mode == 1) _mm256_stream_ps(o + 8 * k, f);
                            else _mm256_store_ps(o + 8 * k, f);
                        }
                    }
                }
                _mm_sfence();
                double dt = now() - t0;
                if (dt < best) best = dt;
            }
            printf("threads %2d %-14s %7.1f GB/s\n", th,
                   mode == 0 ? "nt-zero" : mode == 1 ? "expand-nt" : mode == 2 ? "expand-store" : "expand-nt512",
                   nf * 4 / best / 1e9);
        }
    }
    return 0;
}
