// extern "C" entry points of librocket (see include/rocket.h).
#include <stdlib.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>

#include <algorithm>
#include <string>

#include "internal.h"

namespace rk {

static thread_local std::string g_last_error;

rk_status set_error(rk_status st, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return st;
}

rk_status check_cuda(cudaError_t err, const char* what) {
  return set_error(RK_ERR_DEVICE, "%s: %s (%s)", what, cudaGetErrorName(err), cudaGetErrorString(err));
}

rk_status status_begin(rk_app* app, cudaStream_t s, int** d_status) {
  if (!app->d_status) {
    RK_CUDA(cudaMalloc(&app->d_status, sizeof(int)));
    RK_CUDA(cudaHostAlloc(&app->h_status, sizeof(int), cudaHostAllocDefault));
  }
  RK_CUDA(cudaMemsetAsync(app->d_status, 0, sizeof(int), s));
  *d_status = app->d_status;
  return RK_OK;
}

rk_status status_end(rk_app* app, cudaStream_t s, int* h_status) {
  RK_CUDA(cudaMemcpyAsync(app->h_status, app->d_status, sizeof(int), cudaMemcpyDeviceToHost, s));
  RK_CUDA(cudaStreamSynchronize(s));
  *h_status = *app->h_status;
  return RK_OK;
}

size_t stride_pad(const char* env, size_t dflt) {
  const char* v = getenv(env);
  if (!v || !*v) return dflt;
  return (size_t)strtoull(v, nullptr, 10) / 256 * 256;
}

double threshold_or_nan(const rk_app* app) { return app->p.threshold; }

rk_status synth_tile(rk_app* app, int32_t r0, int32_t r1, int32_t c0, int32_t c1, double* d_out, uint8_t* d_flags,
                     cudaStream_t s);
rk_status synth_prnu(int32_t h, int32_t w, int32_t first_key, int32_t n_items, int32_t cameras, uint64_t seed,
                     float* d_out, cudaStream_t s);
rk_status cv_init(rk_app* app);
rk_status cv_preprocess(rk_app* app, const void* d_parsed, size_t parsed_stride, int n_items, void* d_slots,
                        size_t slot_stride, const int32_t* h_slot_idx, cudaStream_t s);
rk_status cv_compare_list(rk_app* app, const void* d_slots, size_t slot_stride, const rk_pair* pairs, int n,
                          double* d_out, uint8_t* d_flags, cudaStream_t s);

static rk_status check_pairs(const rk_app* app, const rk_pair* h_pairs, int n_pairs) {
  for (int k = 0; k < n_pairs; ++k) {
    const rk_pair& q = h_pairs[k];
    if (!(0 <= q.i && q.i < q.j && q.j < app->p.n))
      return set_error(RK_ERR_VALUE, "pairs are evaluated with left < right < n, got (%d, %d) for n=%d", q.i, q.j,
                       app->p.n);
  }
  return RK_OK;
}

int batch_limit(const rk_app* app) {
  // by-value pair lists of up to 1,024 pairs (PairJob) for the heavy apps
  if (app->p.kind == RK_APP_PCE) return pce_batch_limit(app);
  if (app->p.kind == RK_APP_GMM || app->p.kind == RK_APP_CV) return kListPairs;
  return kMaxBatch;
}

rk_status compare_batch(rk_app* app, const void* d_slots, size_t slot_stride, const PairBatch& b, double* d_out,
                        uint8_t* d_flags, cudaStream_t s) {
  switch (app->p.kind) {
    case RK_APP_SYNTHETIC: return synth_compare(app, b, d_out, d_flags, s);
    case RK_APP_NCC: return ncc_compare(app, d_slots, slot_stride, b, d_out, d_flags, s);
    default: return set_error(RK_ERR_UNSUPPORTED, "compare not built for app kind %d", app->p.kind);
  }
}

rk_status compare_pairs(rk_app* app, const void* d_slots, size_t slot_stride, const rk_pair* h_pairs, int n_pairs,
                        double* d_out, uint8_t* d_flags, cudaStream_t s) {
  if (app->p.kind == RK_APP_PCE) return pce_compare_list(app, d_slots, slot_stride, h_pairs, n_pairs, d_out, d_flags, s);
  if (app->p.kind == RK_APP_GMM) return gmm_compare_list(app, d_slots, slot_stride, h_pairs, n_pairs, d_out, d_flags, s);
  if (app->p.kind == RK_APP_CV) return cv_compare_list(app, d_slots, slot_stride, h_pairs, n_pairs, d_out, d_flags, s);
  const int lim = batch_limit(app);
  PairBatch b;
  for (int base = 0; base < n_pairs; base += lim) {
    const int m = std::min(lim, n_pairs - base);
    b.npairs = m;
    for (int k = 0; k < m; ++k) {
      const rk_pair& q = h_pairs[base + k];
      b.slot_a[k] = q.slot_a;
      b.slot_b[k] = q.slot_b;
      b.key_i[k] = q.i;
      b.key_j[k] = q.j;
      b.pid[k] = pair_id(app->p.n, q.i, q.j);
    }
    RK_TRY(compare_batch(app, d_slots, slot_stride, b, d_out, d_flags, s));
  }
  return RK_OK;
}

}  // namespace rk

using namespace rk;

extern "C" {

int rk_abi_version(void) { return RK_ABI_VERSION; }

const char* rk_last_error(void) { return g_last_error.c_str(); }

const char* rk_status_name(int status) {
  switch (status) {
    case RK_OK: return "RK_OK";
    case RK_ERR_VALUE: return "RK_ERR_VALUE";
    case RK_ERR_MALFORMED: return "RK_ERR_MALFORMED";
    case RK_ERR_SLOT_OVERFLOW: return "RK_ERR_SLOT_OVERFLOW";
    case RK_ERR_NO_EVICTABLE: return "RK_ERR_NO_EVICTABLE";
    case RK_ERR_DEVICE: return "RK_ERR_DEVICE";
    case RK_ERR_UNSUPPORTED: return "RK_ERR_UNSUPPORTED";
    case RK_ERR_DUPLICATE: return "RK_ERR_DUPLICATE";
    default: return "RK_ERR_UNKNOWN";
  }
}

int64_t rk_pair_id(int64_t n, int64_t i, int64_t j) {
  if (!(0 <= i && i < j && j < n)) return -1;
  return pair_id(n, i, j);
}

rk_status rk_pair_from_id(int64_t n, int64_t pid, int64_t* i_out, int64_t* j_out) {
  const int64_t total = n * (n - 1) / 2;
  if (pid < 0 || pid >= total) return set_error(RK_ERR_VALUE, "pair id %lld out of range for n=%lld", (long long)pid, (long long)n);
  // row i starts at i*(2n-i-1)/2; invert the quadratic then fix rounding
  const double nn = (double)n;
  int64_t i = (int64_t)floor(((2.0 * nn - 1.0) - sqrt((2.0 * nn - 1.0) * (2.0 * nn - 1.0) - 8.0 * (double)pid)) / 2.0);
  if (i < 0) i = 0;
  while (i > 0 && i * (2 * n - i - 1) / 2 > pid) --i;
  while ((i + 1) * (2 * n - i - 2) / 2 <= pid) ++i;
  *i_out = i;
  *j_out = pid - i * (2 * n - i - 1) / 2 + i + 1;
  return RK_OK;
}

rk_status rk_app_create(const rk_app_params* params, int device, rk_app** out) {
  if (!params || !out) return set_error(RK_ERR_VALUE, "null argument");
  *out = nullptr;
  if (params->n < 1) return set_error(RK_ERR_VALUE, "item count must be >= 1, got %d", params->n);
  RK_CUDA(cudaSetDevice(device));
  rk_app* app = new rk_app();
  app->p = *params;
  app->device = device;
  rk_status st = RK_OK;
  switch (params->kind) {
    case RK_APP_SYNTHETIC:
      app->slot_bytes = 8;
      app->parsed_bytes = 8;
      break;
    case RK_APP_PCE: st = pce_init(app); break;
    case RK_APP_CV: st = cv_init(app); break;
    case RK_APP_NCC: st = ncc_init(app); break;
    case RK_APP_GMM: st = gmm_init(app); break;
    default: st = set_error(RK_ERR_UNSUPPORTED, "app kind %d not built", params->kind);
  }
  if (st != RK_OK) {
    rk_app_destroy(app);
    return st;
  }
  *out = app;
  return RK_OK;
}

void rk_app_destroy(rk_app* app) {
  if (!app) return;
  cudaSetDevice(app->device);
  if (app->p.kind == RK_APP_PCE) pce_free(app);
  if (app->p.kind == RK_APP_NCC) ncc_free(app);
  delete app->job;
  cudaFree(app->gmm_scratch);
  cudaFree(app->d_status);
  if (app->h_status) cudaFreeHost(app->h_status);
  cudaFree(app->cv_scratch);
  cudaFree(app->cv_prep);
  delete app;
}

size_t rk_app_slot_bytes(const rk_app* app) { return app ? app->slot_bytes : 0; }
size_t rk_app_parsed_bytes(const rk_app* app) { return app ? app->parsed_bytes : 0; }
int32_t rk_app_slot_group(const rk_app* app) { return app ? app->slot_group : 1; }

rk_status rk_preprocess(rk_app* app, const void* d_parsed, size_t parsed_stride, int n_items, void* d_slots,
                        size_t slot_stride, const int32_t* h_slot_idx, void* stream) {
  if (!app) return set_error(RK_ERR_VALUE, "null app");
  if (n_items <= 0) return RK_OK;
  if (slot_stride < app->slot_bytes)
    return set_error(RK_ERR_SLOT_OVERFLOW, "preprocessed item of %zu bytes exceeds slot stride %zu", app->slot_bytes,
                     slot_stride);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  switch (app->p.kind) {
    case RK_APP_SYNTHETIC: return RK_OK;  // identity payload (apps.py:196-199)
    case RK_APP_PCE: return pce_preprocess(app, d_parsed, parsed_stride, n_items, d_slots, slot_stride, h_slot_idx, s);
    case RK_APP_CV: return cv_preprocess(app, d_parsed, parsed_stride, n_items, d_slots, slot_stride, h_slot_idx, s);
    case RK_APP_NCC: return ncc_preprocess(app, d_parsed, parsed_stride, n_items, d_slots, slot_stride, h_slot_idx, s);
    case RK_APP_GMM: return gmm_preprocess(app, d_parsed, parsed_stride, n_items, d_slots, slot_stride, h_slot_idx, s);
    default: return set_error(RK_ERR_UNSUPPORTED, "preprocess not built for app kind %d", app->p.kind);
  }
}

rk_status rk_compare_pairs(rk_app* app, const void* d_slots, size_t slot_stride, const rk_pair* h_pairs, int n_pairs,
                           double* d_out, uint8_t* d_flags, void* stream) {
  if (!app) return set_error(RK_ERR_VALUE, "null app");
  if (n_pairs <= 0) return RK_OK;
  RK_TRY(check_pairs(app, h_pairs, n_pairs));
  return compare_pairs(app, d_slots, slot_stride, h_pairs, n_pairs, d_out, d_flags, static_cast<cudaStream_t>(stream));
}

rk_status rk_compare_tile(rk_app* app, const void* d_slots, size_t slot_stride, int32_t r0, int32_t r1, int32_t c0,
                          int32_t c1, const int32_t* h_slot_of_key, double* d_out, uint8_t* d_flags, void* stream) {
  if (!app) return set_error(RK_ERR_VALUE, "null app");
  if (!(0 <= r0 && r0 <= r1 && 0 <= c0 && c0 <= c1 && r1 <= app->p.n && c1 <= app->p.n))
    return set_error(RK_ERR_VALUE, "malformed region [%d,%d)x[%d,%d) for n=%d", r0, r1, c0, c1, app->p.n);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (app->p.kind == RK_APP_SYNTHETIC) return synth_tile(app, r0, r1, c0, c1, d_out, d_flags, s);
  std::vector<rk_pair> pairs;
  for (int32_t i = r0; i < r1; ++i)
    for (int32_t j = std::max(c0, i + 1); j < c1; ++j)
      pairs.push_back(rk_pair{i, j, h_slot_of_key[i], h_slot_of_key[j]});
  if (pairs.empty()) return RK_OK;
  return compare_pairs(app, d_slots, slot_stride, pairs.data(), (int)pairs.size(), d_out, d_flags, s);
}

rk_status rk_ncc_gram(rk_app* app, const void* d_slots, size_t slot_stride, int32_t n_rows, int32_t rank, int32_t world,
                      double* d_out, uint8_t* d_flags, void* stream) {
  if (!app) return set_error(RK_ERR_VALUE, "null app");
  if (app->p.kind != RK_APP_NCC) return set_error(RK_ERR_VALUE, "rk_ncc_gram needs an NCC app");
  return ncc_gram(app, d_slots, slot_stride, n_rows, rank, world, d_out, d_flags, static_cast<cudaStream_t>(stream));
}

rk_status rk_device_alloc(size_t bytes, int device, void** d_ptr) {
  if (!d_ptr) return set_error(RK_ERR_VALUE, "null argument");
  RK_CUDA(cudaSetDevice(device));
  RK_CUDA(cudaMalloc(d_ptr, bytes));
  return RK_OK;
}

rk_status rk_device_free(void* d_ptr) {
  RK_CUDA(cudaFree(d_ptr));
  return RK_OK;
}

rk_status rk_memcpy_d2d(void* dst, const void* src, size_t bytes, void* stream) {
  RK_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, static_cast<cudaStream_t>(stream)));
  return RK_OK;
}

rk_status rk_ncc_gram_block(rk_app* app, const void* d_slots, size_t slot_stride, int32_t n_rows, int32_t a_row0,
                            int32_t a_key0, int32_t a_cnt, int32_t b_row0, int32_t b_key0, int32_t b_cnt,
                            double* d_out, uint8_t* d_flags, void* stream) {
  if (!app || !d_slots || !d_out) return set_error(RK_ERR_VALUE, "null argument");
  if (app->p.kind != RK_APP_NCC) return set_error(RK_ERR_VALUE, "rk_ncc_gram_block needs an NCC app");
  RK_CUDA(cudaSetDevice(app->device));
  return ncc_gram_block(app, d_slots, slot_stride, n_rows, a_row0, a_key0, a_cnt, b_row0, b_key0, b_cnt, d_out,
                        d_flags, static_cast<cudaStream_t>(stream));
}

rk_status rk_synth_prnu(int32_t h, int32_t w, int32_t first_key, int32_t n_items, int32_t cameras, uint64_t seed,
                        float* d_out, void* stream) {
  if (h <= 0 || w <= 0 || n_items < 0 || cameras <= 0) return set_error(RK_ERR_VALUE, "bad synth_prnu arguments");
  if (n_items == 0) return RK_OK;
  return synth_prnu(h, w, first_key, n_items, cameras, seed, d_out, static_cast<cudaStream_t>(stream));
}

}  // extern "C"
