/*
 * lcnn_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C, single-threaded restatement of the reference CPU algorithms of
 * the memory-bound CNN layer path (/root/reference/proj/src/*.cpp).  It is
 * the checker for the CUDA product path: only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  The
 * product library (paper_1610_03618_b200/lib/liblcnn_cuda.so) never links or
 * calls anything here.
 *
 * Parity pinning: every function below is checked in tests/test_oracle.py
 * against (a) the golden vectors transcribed from the reference's own tests
 * (tests/golden/reference_kats.json, with file:line of each) and (b) the
 * compiled reference itself (oracle/_ref/liblcnn_ref.so, built from
 * /root/reference sources by oracle/Makefile) on seeded inputs, bit-exact
 * for the integer/data-movement/max paths and for every path that shares the
 * reference's fp32 operation order (avg pooling, softmax with the same libm
 * expf).  The golden fixtures made from the reference (tests/golden/*.npz)
 * travel with the repo so the GPU box can pin without /root/reference.
 *
 * Floating-point rules: compiled with -ffp-contract=off so no a*b+c is fused
 * (the reference's avg pooling / softmax have no fusable pairs either).
 * Status codes are the lcnn_status values of include/lcnn_cuda.h.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum { OK = 0, ESHAPE = 1, ELAYOUT = 3, EPLAN = 4, EDOMAIN = 6, EUNSUPPORTED = 7 };
enum { NCHW = 0, CHWN = 1, NHWC = 2, HWCN = 3 };

/* layout_strides (tensor.cpp:55-85); out = {sn, sc, sh, sw} */
void orc_layout_strides(int layout, uint32_t n, uint32_t c, uint32_t h, uint32_t w,
                        uint64_t out[4]) {
  uint64_t sn = 0, sc = 0, sh = 0, sw = 0;
  switch (layout) {
    case NCHW: sw = 1; sh = w; sc = (uint64_t)h * w; sn = (uint64_t)c * h * w; break;
    case CHWN: sn = 1; sw = n; sh = (uint64_t)w * n; sc = (uint64_t)h * w * n; break;
    case NHWC: sc = 1; sw = c; sh = (uint64_t)w * c; sn = (uint64_t)h * w * c; break;
    default:   sn = 1; sc = n; sw = (uint64_t)c * n; sh = (uint64_t)w * c * n; break;
  }
  out[0] = sn; out[1] = sc; out[2] = sh; out[3] = sw;
}

static int check_volume(uint32_t n, uint32_t c, uint32_t h, uint32_t w) {
  /* checked_volume (tensor.cpp:16-29) */
  if (!n || !c || !h || !w) return ESHAPE;
  if ((uint64_t)n * c * h * w > 0xffffffffull) return ESHAPE;
  return OK;
}

/* transform_naive (layout.cpp:77-97): the oracle of every transform. */
int orc_transform(const float* src, float* dst, uint32_t n, uint32_t c, uint32_t h,
                  uint32_t w, int src_layout, int dst_layout) {
  uint64_t si[4], so[4];
  if (check_volume(n, c, h, w)) return ESHAPE;
  orc_layout_strides(src_layout, n, c, h, w, si);
  orc_layout_strides(dst_layout, n, c, h, w, so);
  for (uint64_t a = 0; a < n; ++a)
    for (uint64_t b = 0; b < c; ++b)
      for (uint64_t y = 0; y < h; ++y) {
        uint64_t oi = a * si[0] + b * si[1] + y * si[2];
        uint64_t oo = a * so[0] + b * so[1] + y * so[2];
        for (uint64_t x = 0; x < w; ++x) {
          dst[oo] = src[oi];
          oi += si[3];
          oo += so[3];
        }
      }
  return OK;
}

/* check_window (pool.cpp:19-26) */
static int check_window(uint32_t h, uint32_t w, uint32_t wh, uint32_t ww, uint32_t s) {
  if (wh < 1 || ww < 1 || s < 1) return ESHAPE;
  if (wh > h || ww > w) return ESHAPE;
  return OK;
}

/* covered_extent (pool.cpp:29-33) */
static uint64_t covered(uint32_t out, uint32_t win, uint32_t s) {
  if (s >= win) return (uint64_t)out * win;
  return (uint64_t)s * (out - 1) + win;
}

/* pool_output_extents (pool.cpp:44-47) */
int orc_pool_extents(uint32_t h, uint32_t w, uint32_t wh, uint32_t ww, uint32_t s,
                     uint32_t* ho, uint32_t* wo) {
  if (check_window(h, w, wh, ww, s)) return ESHAPE;
  *ho = (h - wh) / s + 1;
  *wo = (w - ww) / s + 1;
  return OK;
}

static float ref_max(float a, float b) { return (a < b) ? b : a; } /* std::max */

/* pool_oracle (pool.cpp:49-84): any layout in, NCHW out, fp64 sum, max
 * seeded from the first tap. */
int orc_pool_oracle(const float* src, float* dst, uint32_t n, uint32_t c, uint32_t h,
                    uint32_t w, int layout, uint32_t wh, uint32_t ww, uint32_t s, int avg) {
  uint32_t ho, wo;
  uint64_t si[4], oi = 0;
  if (check_volume(n, c, h, w) || orc_pool_extents(h, w, wh, ww, s, &ho, &wo)) return ESHAPE;
  orc_layout_strides(layout, n, c, h, w, si);
  for (uint32_t a = 0; a < n; ++a)
    for (uint32_t b = 0; b < c; ++b)
      for (uint32_t oh = 0; oh < ho; ++oh)
        for (uint32_t ow = 0; ow < wo; ++ow, ++oi) {
          double sum = 0.0;
          float best = src[a * si[0] + b * si[1] + (uint64_t)oh * s * si[2] +
                           (uint64_t)ow * s * si[3]];
          for (uint32_t y = 0; y < wh; ++y)
            for (uint32_t x = 0; x < ww; ++x) {
              const float v = src[a * si[0] + b * si[1] + ((uint64_t)oh * s + y) * si[2] +
                                  ((uint64_t)ow * s + x) * si[3]];
              sum += v;
              best = ref_max(best, v);
            }
          dst[oi] = avg ? (float)(sum / wh / ww) : best;
        }
  return OK;
}

/* pool_plain (pool.cpp:88-168): the layout kernels' exact fp32 semantics.
 * report = {input_loads, output_stores, distinct_inputs} (may be NULL). */
int orc_pool_plain(const float* src, float* dst, uint32_t n, uint32_t c, uint32_t h,
                   uint32_t w, int layout, uint32_t wh, uint32_t ww, uint32_t s, int avg,
                   uint64_t* report) {
  uint32_t ho, wo;
  uint64_t loads = 0, stores = 0;
  if (check_volume(n, c, h, w) || orc_pool_extents(h, w, wh, ww, s, &ho, &wo)) return ESHAPE;
  if (layout == CHWN) {
    const uint64_t in_row = (uint64_t)w * n, in_chan = (uint64_t)h * in_row;
    const float inv_win = 1.0f / (float)(wh * ww);
    float* lane = (float*)malloc(sizeof(float) * n);
    for (uint32_t ch = 0; ch < c; ++ch)
      for (uint32_t oh = 0; oh < ho; ++oh)
        for (uint32_t ow = 0; ow < wo; ++ow) {
          for (uint32_t b = 0; b < n; ++b) lane[b] = avg ? 0.0f : -INFINITY;
          for (uint32_t y = 0; y < wh; ++y) {
            const float* row = src + ch * in_chan + ((uint64_t)oh * s + y) * in_row +
                               (uint64_t)ow * s * n;
            for (uint32_t x = 0; x < ww; ++x) {
              const float* tap = row + (uint64_t)x * n;
              for (uint32_t b = 0; b < n; ++b)
                lane[b] = avg ? lane[b] + tap[b] : ref_max(lane[b], tap[b]);
            }
          }
          loads += (uint64_t)wh * ww * n;
          float* o = dst + (((uint64_t)ch * ho + oh) * wo + ow) * n;
          for (uint32_t b = 0; b < n; ++b) o[b] = avg ? lane[b] * inv_win : lane[b];
          stores += n;
        }
    free(lane);
  } else if (layout == NCHW) {
    const uint64_t in_hw = (uint64_t)h * w;
    uint64_t oi = 0;
    for (uint32_t a = 0; a < n; ++a)
      for (uint32_t ch = 0; ch < c; ++ch) {
        const float* chan = src + ((uint64_t)a * c + ch) * in_hw;
        for (uint32_t oh = 0; oh < ho; ++oh)
          for (uint32_t ow = 0; ow < wo; ++ow, ++oi) {
            const float* win0 = chan + (uint64_t)oh * s * w + (uint64_t)ow * s;
            float red = avg ? 0.0f : -INFINITY;
            for (uint32_t y = 0; y < wh; ++y)
              for (uint32_t x = 0; x < ww; ++x)
                red = avg ? red + win0[(uint64_t)y * w + x] : ref_max(red, win0[(uint64_t)y * w + x]);
            loads += (uint64_t)wh * ww;
            dst[oi] = avg ? red / (float)(wh * ww) : red;
            ++stores;
          }
      }
  } else {
    return ELAYOUT;
  }
  if (report) {
    report[0] = loads;
    report[1] = stores;
    report[2] = (uint64_t)n * c * covered(ho, wh, s) * covered(wo, ww, s);
  }
  return OK;
}

/* pool_coarsened (pool.cpp:178-270): per (channel, block) the union of the
 * block's windows is staged once, then each output reduces from the stage. */
int orc_pool_coarsened(const float* src, float* dst, uint32_t n, uint32_t c, uint32_t h,
                       uint32_t w, int layout, uint32_t wh, uint32_t ww, uint32_t s, int avg,
                       uint32_t fh, uint32_t fw, uint64_t* report) {
  uint32_t ho, wo;
  uint64_t loads = 0, stores = 0;
  if (check_volume(n, c, h, w) || orc_pool_extents(h, w, wh, ww, s, &ho, &wo)) return ESHAPE;
  if (fh < 1 || fw < 1) return EPLAN;
  if ((uint64_t)fh * fw > 64) return EPLAN;
  if (layout != CHWN) return ELAYOUT;
  const uint64_t in_row = (uint64_t)w * n, in_chan = (uint64_t)h * in_row;
  const uint64_t out_row = (uint64_t)wo * n, out_chan = (uint64_t)ho * out_row;
  const float inv_win = 1.0f / (float)(wh * ww);
  const uint32_t max_uh = s * (fh - 1) + wh, max_uw = s * (fw - 1) + ww;
  float* local = (float*)malloc(sizeof(float) * (uint64_t)max_uh * max_uw * n);
  float* lane = (float*)malloc(sizeof(float) * n);
  for (uint32_t ch = 0; ch < c; ++ch)
    for (uint32_t oh0 = 0; oh0 < ho; oh0 += fh) {
      const uint32_t bh = fh < ho - oh0 ? fh : ho - oh0;
      const uint32_t uh = s * (bh - 1) + wh;
      for (uint32_t ow0 = 0; ow0 < wo; ow0 += fw) {
        const uint32_t bw = fw < wo - ow0 ? fw : wo - ow0;
        const uint32_t uw = s * (bw - 1) + ww;
        const float* base = src + ch * in_chan + (uint64_t)oh0 * s * in_row + (uint64_t)ow0 * s * n;
        for (uint32_t y = 0; y < uh; ++y)
          for (uint32_t x = 0; x < uw; ++x)
            memcpy(local + ((uint64_t)y * uw + x) * n, base + (uint64_t)y * in_row + (uint64_t)x * n,
                   sizeof(float) * n);
        loads += (uint64_t)uh * uw * n;
        for (uint32_t by = 0; by < bh; ++by)
          for (uint32_t bx = 0; bx < bw; ++bx) {
            for (uint32_t b = 0; b < n; ++b) lane[b] = avg ? 0.0f : -INFINITY;
            for (uint32_t y = 0; y < wh; ++y)
              for (uint32_t x = 0; x < ww; ++x) {
                const float* tap = local + (((uint64_t)by * s + y) * uw + (uint64_t)bx * s + x) * n;
                for (uint32_t b = 0; b < n; ++b)
                  lane[b] = avg ? lane[b] + tap[b] : ref_max(lane[b], tap[b]);
              }
            float* o = dst + ch * out_chan + ((uint64_t)oh0 + by) * out_row + ((uint64_t)ow0 + bx) * n;
            for (uint32_t b = 0; b < n; ++b) o[b] = avg ? lane[b] * inv_win : lane[b];
            stores += n;
          }
      }
    }
  free(local);
  free(lane);
  if (report) {
    report[0] = loads;
    report[1] = stores;
    report[2] = (uint64_t)n * c * covered(ho, wh, s) * covered(wo, ww, s);
  }
  return OK;
}

/* blocked_sum (softmax.cpp:23-32): sequential within 256-blocks */
static float blocked_sum(const float* v, uint32_t len) {
  float result = 0.0f;
  for (uint32_t b0 = 0; b0 < len; b0 += 256) {
    const uint32_t bn = 256 < len - b0 ? 256 : len - b0;
    float s = 0.0f;
    for (uint32_t i = 0; i < bn; ++i) s += v[b0 + i];
    result += s;
  }
  return result;
}

/* softmax_reference (softmax.cpp:36-98); report = {materializations, sweeps} */
int orc_softmax_reference(const float* in, float* out, uint32_t rows, uint32_t cols,
                          uint32_t* report) {
  if (rows < 1 || cols < 1) return ESHAPE;
  const uint64_t total = (uint64_t)rows * cols;
  float* maxv = (float*)malloc(sizeof(float) * rows);
  float* sumv = (float*)malloc(sizeof(float) * rows);
  float* mid1 = (float*)malloc(sizeof(float) * total);
  float* mid2 = (float*)malloc(sizeof(float) * total);
  int rc = OK;
  for (uint32_t i = 0; i < rows && rc == OK; ++i) {
    const float* row = in + (uint64_t)i * cols;
    float m = row[0];
    for (uint32_t j = 0; j < cols; ++j) {
      if (!isfinite(row[j])) { rc = EDOMAIN; break; }
      m = ref_max(m, row[j]);
    }
    maxv[i] = m;
  }
  if (rc == OK) {
    for (uint64_t k = 0; k < total; ++k) mid1[k] = in[k] - maxv[k / cols];
    for (uint64_t k = 0; k < total; ++k) mid2[k] = expf(mid1[k]);
    for (uint32_t i = 0; i < rows; ++i) sumv[i] = blocked_sum(mid2 + (uint64_t)i * cols, cols);
    for (uint32_t i = 0; i < rows; ++i) {
      const float inv = 1.0f / sumv[i];
      for (uint32_t j = 0; j < cols; ++j)
        out[(uint64_t)i * cols + j] = mid2[(uint64_t)i * cols + j] * inv;
    }
    if (report) { report[0] = 3; report[1] = 8; }
  }
  free(maxv); free(sumv); free(mid1); free(mid2);
  return rc;
}

/* softmax_fused (softmax.cpp:100-180), both the staged and the streaming
 * schedule (identical arithmetic, as the reference promises). */
int orc_softmax_fused(const float* in, float* out, uint32_t rows, uint32_t cols,
                      uint32_t local_limit, uint32_t* report) {
  if (rows < 1 || cols < 1) return ESHAPE;
  for (uint32_t i = 0; i < rows; ++i) {
    const float* row = in + (uint64_t)i * cols;
    float* orow = out + (uint64_t)i * cols;
    float m = row[0];
    for (uint32_t b0 = 0; b0 < cols; b0 += 256) {
      const uint32_t bn = 256 < cols - b0 ? 256 : cols - b0;
      float bm = row[b0];
      for (uint32_t j = 0; j < bn; ++j) {
        if (!isfinite(row[b0 + j])) return EDOMAIN;
        bm = ref_max(bm, row[b0 + j]);
      }
      m = ref_max(m, bm);
    }
    float sum = 0.0f;
    for (uint32_t b0 = 0; b0 < cols; b0 += 256) {
      const uint32_t bn = 256 < cols - b0 ? 256 : cols - b0;
      float bs = 0.0f;
      for (uint32_t j = 0; j < bn; ++j) {
        const float e = expf(row[b0 + j] - m);
        orow[b0 + j] = e;
        bs += e;
      }
      sum += bs;
    }
    const float inv = 1.0f / sum;
    for (uint32_t j = 0; j < cols; ++j) orow[j] = orow[j] * inv;
  }
  if (report) { report[0] = 0; report[1] = cols <= local_limit ? 2 : 5; }
  return OK;
}

/* conv_output_extents (conv.cpp:22-33) */
int orc_conv_extents(uint32_t h, uint32_t w, uint32_t fh, uint32_t fw, uint32_t stride,
                     uint32_t pad, uint32_t* ho, uint32_t* wo) {
  if (stride < 1) return ESHAPE;
  const int64_t sh = (int64_t)h + 2 * (int64_t)pad - fh, sw = (int64_t)w + 2 * (int64_t)pad - fw;
  if (sh < 0 || sw < 0) return ESHAPE;
  *ho = (uint32_t)(sh / stride + 1);
  *wo = (uint32_t)(sw / stride + 1);
  return OK;
}

/* conv_oracle (conv.cpp:53-93): fp64 quadruple sum, any layout in, NCHW out;
 * padded taps are clipped (tap_range conv.cpp:42-49). */
int orc_conv_oracle(const float* in, const float* filt, float* out, uint32_t n, uint32_t ci,
                    uint32_t h, uint32_t w, int layout, uint32_t co, uint32_t fh, uint32_t fw,
                    uint32_t stride, uint32_t pad) {
  uint32_t ho, wo;
  uint64_t si[4], oi = 0;
  if (orc_conv_extents(h, w, fh, fw, stride, pad, &ho, &wo)) return ESHAPE;
  orc_layout_strides(layout, n, ci, h, w, si);
  for (uint32_t a = 0; a < n; ++a)
    for (uint32_t o = 0; o < co; ++o)
      for (uint32_t oh = 0; oh < ho; ++oh)
        for (uint32_t ow = 0; ow < wo; ++ow, ++oi) {
          double acc = 0.0;
          for (uint32_t k = 0; k < ci; ++k)
            for (uint32_t y = 0; y < fh; ++y) {
              const int64_t ih = (int64_t)oh * stride + y - pad;
              if (ih < 0 || ih >= h) continue;
              for (uint32_t x = 0; x < fw; ++x) {
                const int64_t iw = (int64_t)ow * stride + x - pad;
                if (iw < 0 || iw >= w) continue;
                acc += (double)in[a * si[0] + k * si[1] + ih * si[2] + iw * si[3]] *
                       (double)filt[(((uint64_t)o * ci + k) * fh + y) * fw + x];
              }
            }
          out[oi] = (float)acc;
        }
  return OK;
}

/* fp64 row-major product, the oracle of gemm_blocked / fc_forward
 * (conv.cpp:252-304, softmax.cpp:182-184). */
void orc_gemm_f64(const float* a, const float* b, float* c, uint64_t m, uint64_t n, uint64_t k) {
  for (uint64_t i = 0; i < m; ++i)
    for (uint64_t j = 0; j < n; ++j) {
      double acc = 0.0;
      for (uint64_t q = 0; q < k; ++q) acc += (double)a[i * k + q] * (double)b[q * n + j];
      c[i * n + j] = (float)acc;
    }
}

/* choose_layout (select.cpp:39-52); kind: 0 conv, 1 pool, 2 softmax, 3 fc, 4 input */
int orc_choose_layout(int kind, uint32_t n, uint32_t c, uint32_t c_t, uint32_t n_t) {
  if (kind == 1) return CHWN;
  if (kind == 0) return (c < c_t || n >= n_t) ? CHWN : NCHW;
  return NCHW;
}

/* calibrate (select.cpp:65-97) over the published sweeps (select.hpp:49-51). */
typedef double (*orc_bench_fn)(int layout, uint32_t n, uint32_t c, void* ctx);
int orc_calibrate(orc_bench_fn bench, void* ctx, uint32_t* c_t, uint32_t* n_t) {
  static const uint32_t batches[] = {16, 32, 64, 128};
  static const uint32_t chans[] = {3, 16, 32, 64, 128, 256};
  uint32_t nt = 0, ct = 0;
  for (int i = 0; i < 4; ++i) {
    const double a = bench(CHWN, batches[i], 256, ctx), b = bench(NCHW, batches[i], 256, ctx);
    if (!nt && a < b) nt = batches[i];
  }
  for (int i = 0; i < 6; ++i) {
    const double a = bench(CHWN, 64, chans[i], ctx), b = bench(NCHW, 64, chans[i], ctx);
    if (!ct && b < a) ct = chans[i];
  }
  *n_t = nt ? nt : 129;
  *c_t = ct ? ct : 257;
  return OK;
}

/* autotune_pool hill climb (pool.cpp:296-330) */
typedef double (*orc_cost_fn)(uint32_t fh, uint32_t fw, void* ctx);
void orc_autotune(orc_cost_fn cost, void* ctx, uint32_t* fh_out, uint32_t* fw_out) {
  uint32_t fh = 2, fw = 2;
  double best = cost(fh, fw, ctx);
  int gh = 1, gw = 1;
  while (gh || gw) {
    if (gh) {
      if ((uint64_t)(fh + 1) * fw > 64) gh = 0;
      else {
        const double c = cost(fh + 1, fw, ctx);
        if (c < best) { best = c; fh += 1; } else gh = 0;
      }
    }
    if (gw) {
      if ((uint64_t)fh * (fw + 1) > 64) gw = 0;
      else {
        const double c = cost(fh, fw + 1, ctx);
        if (c < best) { best = c; fw += 1; } else gw = 0;
      }
    }
  }
  *fh_out = fh;
  *fw_out = fw;
}

/* plan_transforms (net.cpp:197-215) over per-layer (kind, layout) arrays;
 * only conv (0) and pool (1) layers carry layouts.  Returns the step count,
 * writing (position, src, dst) triples. */
int orc_plan_transforms(const int* kinds, const int* layouts, int count, int* pos, int* src,
                        int* dst) {
  int steps = 0, have_prev = 0, prev = 0;
  for (int i = 0; i < count; ++i) {
    if (kinds[i] != 0 && kinds[i] != 1) continue;
    if (have_prev && prev != layouts[i]) {
      pos[steps] = i;
      src[steps] = prev;
      dst[steps] = layouts[i];
      ++steps;
    }
    prev = layouts[i];
    have_prev = 1;
  }
  return steps;
}
