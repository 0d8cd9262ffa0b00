/*
 * CPU oracle for the im2win path — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference algorithms, used by tests/, by
 * __graft_entry__.smoke() as the checker, and by bench.py's cpu_baseline /
 * --impl reference arm.  It is never called by the product path.
 *
 * Pinned against the reference's own outputs: tests/golden/ holds vectors
 * and sha256 checksums produced by importing the reference package
 * (/root/reference/pkg/src/winconv) with tests/golden/make_golden.py, and
 * tests/test_oracle.py checks this file against every one of them.
 *
 * Arithmetic contract (reference kernels/reference.py:4-8, :89):
 *   every output element is  acc = +0.0f;  for k = (c, fh, fw) ascending:
 *   acc = acc + (x * f)  in float32 with an UNFUSED multiply and add.
 * Compile with -ffp-contract=off (no FMA contraction) and without
 * -ffast-math (no reassociation).  The loops below are reordered so the
 * compiler can vectorise across output columns, but each output element
 * still sees exactly the ascending-k sequence of rounded adds.
 */
#include <pthread.h>
#include <stdint.h>
#include <string.h>
#include <unistd.h>

/* Minimal static-partition parallel-for over [0, n) on POSIX threads. */
typedef void (*range_fn)(const void* ctx, int64_t begin, int64_t end);
typedef struct { range_fn fn; const void* ctx; int64_t begin, end; } range_job;

static void* run_range(void* p) {
  const range_job* j = (const range_job*)p;
  j->fn(j->ctx, j->begin, j->end);
  return NULL;
}

static void parallel_for(int64_t n, int32_t threads, range_fn fn, const void* ctx) {
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  if (threads > n) threads = (int32_t)(n > 0 ? n : 1);
  pthread_t tid[256];
  range_job jobs[256];
  for (int32_t t = 0; t < threads; ++t) {
    jobs[t].fn = fn;
    jobs[t].ctx = ctx;
    jobs[t].begin = n * t / threads;
    jobs[t].end = n * (t + 1) / threads;
  }
  for (int32_t t = 1; t < threads; ++t) pthread_create(&tid[t], NULL, run_range, &jobs[t]);
  run_range(&jobs[0]);
  for (int32_t t = 1; t < threads; ++t) pthread_join(tid[t], NULL);
}

/* layouts.py:73-83  dst[i,r,m,c*hf+u] = src[i,r,m*s+u,c], c < w_eff, u < hf */
typedef struct {
  const float* src; float* dst; int64_t h, w, h_out, w_eff, row_len; int32_t hf, s;
} fill_ctx;

static void fill_range(const void* p, int64_t begin, int64_t end) {
  const fill_ctx* a = (const fill_ctx*)p;
  for (int64_t pl = begin; pl < end; ++pl) {
    const float* sp = a->src + pl * a->h * a->w;
    float* dp = a->dst + pl * a->h_out * a->row_len;
    for (int64_t m = 0; m < a->h_out; ++m)
      for (int64_t col = 0; col < a->w_eff; ++col)
        for (int32_t u = 0; u < a->hf; ++u)
          dp[m * a->row_len + col * a->hf + u] = sp[(m * a->s + u) * a->w + col];
  }
}

void oracle_im2win_fill(const float* src, float* dst, int64_t n, int64_t c_in, int64_t h,
                        int64_t w, int32_t hf, int32_t wf, int32_t s, int32_t threads) {
  fill_ctx a;
  a.src = src; a.dst = dst; a.h = h; a.w = w; a.hf = hf; a.s = s;
  a.h_out = (h - hf) / s + 1;
  const int64_t w_out = (w - wf) / s + 1;
  a.w_eff = (w_out - 1) * s + wf;
  a.row_len = (int64_t)hf * a.w_eff;
  parallel_for(n * c_in, threads, fill_range, &a);
}

/* reference.py:70-90 (direct conv), unfused ascending-k per output element. */
typedef struct {
  const float* inp; const float* flt; float* out;
  int64_t c_in, h, w, c_out, h_out, w_out, row_len; int32_t hf, wf, s;
} conv_ctx;

static void direct_range(const void* p, int64_t begin, int64_t end) {
  const conv_ctx* a = (const conv_ctx*)p;
  const float* inp = a->inp; const float* flt = a->flt; float* out = a->out;
  const int64_t c_in = a->c_in, h = a->h, w = a->w, c_out = a->c_out;
  const int64_t h_out = a->h_out, w_out = a->w_out, hw = h_out * w_out;
  const int32_t hf = a->hf, wf = a->wf, s = a->s;
  for (int64_t plane = begin; plane < end; ++plane) {
    const int64_t i = plane / c_out;
    const int64_t j = plane % c_out;
    float* o = out + plane * hw;
    for (int64_t q = 0; q < hw; ++q) o[q] = 0.0f;
    for (int64_t r = 0; r < c_in; ++r) {
      const float* ip = inp + (i * c_in + r) * h * w;
      for (int32_t u = 0; u < hf; ++u) {
        for (int32_t v = 0; v < wf; ++v) {
          const float f = flt[((j * c_in + r) * hf + u) * wf + v];
          for (int64_t m = 0; m < h_out; ++m) {
            const float* row = ip + (m * s + u) * w + v;
            float* orow = o + m * w_out;
            if (s == 1) {
              for (int64_t q = 0; q < w_out; ++q) {
                float prod = row[q] * f;
                orow[q] = orow[q] + prod;
              }
            } else {
              for (int64_t q = 0; q < w_out; ++q) {
                float prod = row[q * s] * f;
                orow[q] = orow[q] + prod;
              }
            }
          }
        }
      }
    }
  }
}

/* reference.py:180-206 (Alg. 2, basic window-order kernel): reads through the Ĩ map. */
void oracle_conv_direct(const float* inp, const float* flt, float* out, int64_t n, int64_t c_in,
                        int64_t h, int64_t w, int64_t c_out, int32_t hf, int32_t wf, int32_t s,
                        int32_t threads) {
  conv_ctx a;
  a.inp = inp; a.flt = flt; a.out = out; a.c_in = c_in; a.h = h; a.w = w; a.c_out = c_out;
  a.hf = hf; a.wf = wf; a.s = s; a.h_out = (h - hf) / s + 1; a.w_out = (w - wf) / s + 1;
  a.row_len = 0;
  parallel_for(n * c_out, threads, direct_range, &a);
}

static void windows_range(const void* p, int64_t begin, int64_t end) {
  const conv_ctx* a = (const conv_ctx*)p;
  const float* win = a->inp; const float* flt = a->flt; float* out = a->out;
  const int64_t c_in = a->c_in, c_out = a->c_out, h_out = a->h_out, w_out = a->w_out;
  const int64_t row_len = a->row_len, hw = h_out * w_out;
  const int32_t hf = a->hf, wf = a->wf, s = a->s;
  const int64_t dim_k = c_in * hf * wf;
  for (int64_t plane = begin; plane < end; ++plane) {
    const int64_t i = plane / c_out;
    const int64_t j = plane % c_out;
    float* o = out + plane * hw;
    for (int64_t q = 0; q < hw; ++q) o[q] = 0.0f;
    for (int64_t k = 0; k < dim_k; ++k) {
      const int64_t r = k / (hf * wf);
      const int32_t u = (int32_t)((k % (hf * wf)) / wf);
      const int32_t v = (int32_t)(k % wf);
      const float f = flt[j * dim_k + k];
      const float* wp = win + (i * c_in + r) * h_out * row_len + (int64_t)v * hf + u;
      for (int64_t m = 0; m < h_out; ++m) {
        const float* row = wp + m * row_len;
        float* orow = o + m * w_out;
        for (int64_t q = 0; q < w_out; ++q) {
          float prod = row[q * s * hf] * f;
          orow[q] = orow[q] + prod;
        }
      }
    }
  }
}

void oracle_conv_from_windows(const float* win, const float* flt, float* out, int64_t n,
                              int64_t c_in, int64_t h_out, int64_t w_out, int64_t row_len,
                              int64_t c_out, int32_t hf, int32_t wf, int32_t s, int32_t threads) {
  conv_ctx a;
  a.inp = win; a.flt = flt; a.out = out; a.c_in = c_in; a.h = 0; a.w = 0; a.c_out = c_out;
  a.hf = hf; a.wf = wf; a.s = s; a.h_out = h_out; a.w_out = w_out; a.row_len = row_len;
  parallel_for(n * c_out, threads, windows_range, &a);
}

int32_t oracle_max_threads(void) {
  long n = sysconf(_SC_NPROCESSORS_ONLN);
  return (int32_t)(n > 0 ? n : 1);
}
