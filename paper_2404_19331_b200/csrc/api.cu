// C ABI of libfcm.so (include/fcm.h): synchronous validation, tile defaults, dispatch.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "common.cuh"

#include "host.h"
#include "tiles.h"

namespace fcm {

std::atomic<uint64_t> g_launches{0};
static thread_local std::string t_err;

int set_error(int status, const std::string& msg) {
  t_err = msg;
  return status;
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(FCM_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return FCM_OK;
}

const DevProps& device_props() {
  static DevProps props[16];
  static std::once_flag once[16];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 16) dev = 0;
  std::call_once(once[dev], [dev]() {
    DevProps& p = props[dev];
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess) p.sms = v;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) == cudaSuccess) p.smem_optin = v;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrL2CacheSize, dev) == cudaSuccess) p.l2_bytes = v;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrComputeCapabilityMajor, dev) == cudaSuccess) p.cc_major = v;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrComputeCapabilityMinor, dev) == cudaSuccess) p.cc_minor = v;
    cudaGetLastError();
  });
  return props[dev];
}

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                     const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                     CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

bool pdl_enabled() {
  static const bool on = [] { const char* e = getenv("FCM_PDL"); return !(e && e[0] == '0'); }();
  return on;
}

bool encode_tmap(CUtensorMap* m, CUtensorMapDataType dt, uint32_t rank, const void* base, const uint64_t* dims,
                 const uint64_t* strides_bytes, const uint32_t* box, CUtensorMapSwizzle swz) {
  static PFN_encodeTiled fn = nullptr;
  static std::once_flag once;
  std::call_once(once, []() {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled>(p);
    cudaGetLastError();
  });
  if (!fn) return false;
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUresult r = fn(m, dt, rank, const_cast<void*>(base), reinterpret_cast<const cuuint64_t*>(dims),
                  reinterpret_cast<const cuuint64_t*>(strides_bytes), reinterpret_cast<const cuuint32_t*>(box), estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

CUtensorMapDataType tmap_dtype(int dt) {
  switch (dt) {
    case FCM_F32: return CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    case FCM_BF16: return CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
    case FCM_F16: return CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
    default: return CU_TENSOR_MAP_DATA_TYPE_UINT8;
  }
}

int elem_size(int dt) { return dt == FCM_F32 ? 4 : (dt == FCM_S8 ? 1 : 2); }

}  // namespace fcm

using namespace fcm;

namespace {

bool valid_dtype(int dt) { return dt == FCM_F32 || dt == FCM_BF16 || dt == FCM_F16 || dt == FCM_S8; }

size_t tensor_bytes(const fcm_tensor* t) {
  return (size_t)t->n * t->h * t->w * t->c * elem_size(t->dtype);
}

int check_tensor(const fcm_tensor* t, const char* name, bool allow_nchw) {
  if (!t) return set_error(FCM_E_INVAL, std::string(name) + " is NULL");
  if (!t->data) return set_error(FCM_E_INVAL, std::string(name) + "->data is NULL");
  if (!valid_dtype(t->dtype)) return set_error(FCM_E_INVAL, std::string(name) + ": bad dtype");
  if (t->layout != FCM_NHWC && !(allow_nchw && t->layout == FCM_NCHW))
    return set_error(t->layout == FCM_NCHW ? FCM_E_UNSUPPORTED : FCM_E_INVAL,
                     std::string(name) + ": layout must be NHWC on this path");
  if (t->n < 1 || t->h < 1 || t->w < 1 || t->c < 1) return set_error(FCM_E_INVAL, std::string(name) + ": empty dims");
  if (reinterpret_cast<uintptr_t>(t->data) % 16) return set_error(FCM_E_ALIGN, std::string(name) + ": not 16-B aligned");
  return FCM_OK;
}

bool pitch_ok(const fcm_tensor* t) { return ((size_t)t->c * elem_size(t->dtype)) % 16 == 0; }

bool overlaps(const fcm_tensor* a, const fcm_tensor* b) {
  const char* a0 = static_cast<const char*>(a->data);
  const char* b0 = static_cast<const char*>(b->data);
  return a0 < b0 + tensor_bytes(b) && b0 < a0 + tensor_bytes(a);
}

int check_geom(const fcm_dw_geom* g) {
  if (!g) return set_error(FCM_E_INVAL, "geom is NULL");
  if (g->k < 1 || g->stride < 1 || g->pad_t < 0 || g->pad_l < 0 || g->pad_b < 0 || g->pad_r < 0)
    return set_error(FCM_E_INVAL, "bad DW geometry");
  return FCM_OK;
}

int check_epi(const fcm_epilogue* e, int dt, const char* name) {
  if (!e) return set_error(FCM_E_INVAL, std::string(name) + " is NULL");
  if (dt == FCM_S8) {
    if (!e->mult_q || !e->shift_q) return set_error(FCM_E_INVAL, std::string(name) + ": int8 needs mult_q/shift_q");
    if (e->qmin > e->qmax || e->qmin < -128 || e->qmax > 127)
      return set_error(FCM_E_INVAL, std::string(name) + ": qmin/qmax must lie in [-128,127]");
    if (e->zp_in != 0) return set_error(FCM_E_UNSUPPORTED, std::string(name) + ": GPU paths need zp_in == 0");
    if (e->residual) return set_error(FCM_E_UNSUPPORTED, std::string(name) + ": int8 residual add");
  } else if (e->act < FCM_ACT_NONE || e->act > FCM_ACT_GELU) {
    return set_error(FCM_E_INVAL, std::string(name) + ": bad activation");
  }
  return FCM_OK;
}

// an epilogue that may not carry a residual (it does not write the call's output through a PW)
int no_residual(const fcm_epilogue* e, const char* name) {
  return e && e->residual ? set_error(FCM_E_UNSUPPORTED, std::string(name) + ": residual add only on a PW output epilogue")
                          : FCM_OK;
}

// residual: 16-byte aligned (vector loads) and not overlapping the output
int check_residual(const fcm_epilogue* e, const fcm_tensor* y, const char* name) {
  if (!e || !e->residual) return FCM_OK;
  if (reinterpret_cast<uintptr_t>(e->residual) % 16)
    return set_error(FCM_E_ALIGN, std::string(name) + ": residual not 16-byte aligned");
  const char* r0 = static_cast<const char*>(e->residual);
  const char* y0 = static_cast<const char*>(y->data);
  const size_t nb = tensor_bytes(y);
  if (r0 < y0 + nb && y0 < r0 + nb) return set_error(FCM_E_INVAL, std::string(name) + ": residual overlaps the output");
  return FCM_OK;
}

Epi to_epi(const fcm_epilogue* e) {
  return Epi{e->act, e->scale, e->bias, e->bias_q, e->mult_q, e->shift_q, e->zp_in, e->zp_out, e->qmin, e->qmax,
             e->residual};
}

// floor((in + p0 + p1 - k) / s) + 1; a window that does not fit the padded input gives 0 (-> the
// caller's shape check rejects it with FCM_E_INVAL) instead of C++'s truncation toward zero
int out_dim(int in, int k, int s, int p0, int p1) {
  const int span = in + p0 + p1 - k;
  return span < 0 ? 0 : span / s + 1;
}

#define FCM_TRY(x)            \
  do {                        \
    int _r = (x);             \
    if (_r != FCM_OK) return _r; \
  } while (0)

}  // namespace

extern "C" {

int fcm_version(void) { return FCM_VERSION; }

uint64_t fcm_launch_count(void) { return g_launches.load(); }

const char* fcm_last_error(void) { return t_err.c_str(); }

const char* fcm_status_str(int s) {
  switch (s) {
    case FCM_OK: return "FCM_OK";
    case FCM_E_INVAL: return "FCM_E_INVAL";
    case FCM_E_ALIGN: return "FCM_E_ALIGN";
    case FCM_E_UNSUPPORTED: return "FCM_E_UNSUPPORTED";
    case FCM_E_INFEASIBLE: return "FCM_E_INFEASIBLE";
    case FCM_E_CUDA: return "FCM_E_CUDA";
    case FCM_E_BUFSZ: return "FCM_E_BUFSZ";
  }
  return "FCM_E_UNKNOWN";
}

size_t fcm_pack_pw_bytes(int32_t dtype, int32_t c_in, int32_t c_out) {
  if (!valid_dtype(dtype) || c_in < 1 || c_out < 1) return 0;
  return (size_t)c_in * c_out * elem_size(dtype);
}

int fcm_pack_pw(int32_t dtype, int32_t c_in, int32_t c_out, const void* w_pw, void* w_packed, void* stream) {
  if (!valid_dtype(dtype) || c_in < 1 || c_out < 1) return set_error(FCM_E_INVAL, "pack_pw: bad dtype/dims");
  if (!w_pw || !w_packed) return set_error(FCM_E_INVAL, "pack_pw: NULL pointer");
  if (reinterpret_cast<uintptr_t>(w_packed) % 16) return set_error(FCM_E_ALIGN, "pack_pw: dst not 16-B aligned");
  return launch_pack_pw(dtype, c_in, c_out, w_pw, w_packed, static_cast<cudaStream_t>(stream));
}

int fcm_dw(const fcm_tensor* x, const void* w_dw, const fcm_dw_geom* geom, const fcm_epilogue* ep, fcm_tensor* y,
           const fcm_tile* tile, void* stream) {
  FCM_TRY(check_tensor(x, "x", true));
  FCM_TRY(check_tensor(y, "y", true));
  FCM_TRY(check_geom(geom));
  if (!w_dw) return set_error(FCM_E_INVAL, "w_dw is NULL");
  if (x->dtype != y->dtype || x->layout != y->layout) return set_error(FCM_E_INVAL, "x/y dtype or layout differ");
  FCM_TRY(check_epi(ep, x->dtype, "ep"));
  FCM_TRY(no_residual(ep, "ep"));
  const int Ho = out_dim(x->h, geom->k, geom->stride, geom->pad_t, geom->pad_b);
  const int Wo = out_dim(x->w, geom->k, geom->stride, geom->pad_l, geom->pad_r);
  if (Ho < 1 || Wo < 1) return set_error(FCM_E_INVAL, "dw: empty output");
  if (y->n != x->n || y->c != x->c || y->h != Ho || y->w != Wo) return set_error(FCM_E_INVAL, "dw: y dims mismatch");
  if (overlaps(x, y)) return set_error(FCM_E_INVAL, "dw: x and y overlap");
  Geo g{x->n, x->h, x->w, x->c, Ho, Wo, x->c, geom->k, geom->stride, geom->pad_t, geom->pad_l, 1, 0, 0};
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (x->layout == FCM_NCHW) return launch_dw_nchw(x->dtype, x->data, w_dw, to_epi(ep), y->data, g, st);
  // channel pitch not a multiple of 4 B: the word-per-lane kernels cannot address it -> CUDA-core
  // kernel (multiples of 4 but not 16: the tiled kernel stages with cp.async instead of TMA)
  if (((size_t)x->c * elem_size(x->dtype)) % 4)
    return launch_dw_simt(x->dtype, x->data, w_dw, to_epi(ep), y->data, g, st);
  default_dw_tile(g, elem_size(x->dtype));
  if (tile) {
    if (tile->tile_h > 0) g.th = tile->tile_h;
    if (tile->tile_w > 0) g.tw = tile->tile_w;
  }
  return launch_dw(x->dtype, x->data, w_dw, to_epi(ep), y->data, g, st);
}

int fcm_pw(const fcm_tensor* x, const void* w_pw_packed, const fcm_epilogue* ep, fcm_tensor* y, const fcm_tile* tile,
           void* stream) {
  FCM_TRY(check_tensor(x, "x", false));
  FCM_TRY(check_tensor(y, "y", false));
  if (!w_pw_packed) return set_error(FCM_E_INVAL, "w_pw is NULL");
  if (x->dtype != y->dtype) return set_error(FCM_E_INVAL, "x/y dtype differ");
  FCM_TRY(check_epi(ep, x->dtype, "ep"));
  FCM_TRY(check_residual(ep, y, "ep"));
  if (y->n != x->n || y->h != x->h || y->w != x->w) return set_error(FCM_E_INVAL, "pw: y spatial dims mismatch");
  if (overlaps(x, y)) return set_error(FCM_E_INVAL, "pw: x and y overlap");
  const int M = x->n * x->h * x->w;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // fp32: 3xTF32 on the tensor cores (FCM_PW_F32_TC=0: the FFMA kernel)
  static const bool f32_tc = [] { const char* e = getenv("FCM_PW_F32_TC"); return !e || atoi(e) != 0; }();
  const bool f32_simt = x->dtype == FCM_F32 && !f32_tc;
  if (f32_simt || !pitch_ok(x) || !pitch_ok(y))
    return launch_pw_simt(x->dtype, x->data, w_pw_packed, to_epi(ep), y->data, M, x->c, y->c, st);
  // tile: only n_split (the number of C_out slices) applies to the tensor-core PW
  return launch_pw_tc(x->dtype, x->data, w_pw_packed, to_epi(ep), y->data, M, x->c, y->c,
                      tile && tile->n_split > 0 ? tile->n_split : 0, st);
}

int fcm_dwpw(const fcm_tensor* x, const void* w_dw, const fcm_dw_geom* geom, const fcm_epilogue* ep_dw,
             const void* w_pw_packed, const fcm_epilogue* ep_pw, fcm_tensor* y, const fcm_tile* tile, void* stream) {
  FCM_TRY(check_tensor(x, "x", false));
  FCM_TRY(check_tensor(y, "y", false));
  FCM_TRY(check_geom(geom));
  if (!w_dw || !w_pw_packed) return set_error(FCM_E_INVAL, "weights NULL");
  if (x->dtype != y->dtype) return set_error(FCM_E_INVAL, "x/y dtype differ");
  FCM_TRY(check_epi(ep_dw, x->dtype, "ep_dw"));
  FCM_TRY(check_epi(ep_pw, x->dtype, "ep_pw"));
  FCM_TRY(no_residual(ep_dw, "ep_dw"));
  FCM_TRY(check_residual(ep_pw, y, "ep_pw"));
  if (x->dtype == FCM_S8 && ep_pw->zp_in != ep_dw->zp_out)
    return set_error(FCM_E_INVAL, "dwpw: ep_pw.zp_in must equal ep_dw.zp_out (T's zero point)");
  const int Ho = out_dim(x->h, geom->k, geom->stride, geom->pad_t, geom->pad_b);
  const int Wo = out_dim(x->w, geom->k, geom->stride, geom->pad_l, geom->pad_r);
  if (Ho < 1 || Wo < 1) return set_error(FCM_E_INVAL, "dwpw: empty output");
  if (y->n != x->n || y->h != Ho || y->w != Wo) return set_error(FCM_E_INVAL, "dwpw: y dims mismatch");
  if (overlaps(x, y)) return set_error(FCM_E_INVAL, "dwpw: x and y overlap");
  Geo g{x->n, x->h, x->w, x->c, Ho, Wo, y->c, geom->k, geom->stride, geom->pad_t, geom->pad_l, 1, 0, 0};
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // fp32: the tensor-core kernel (DW on FFMA, PW 3xTF32) when its resident weight split fits shared
  // memory, else the FFMA kernel (FCM_DWPW_F32_TC=0: always the FFMA kernel)
  static const bool f32_tc = [] { const char* e = getenv("FCM_DWPW_F32_TC"); return !e || atoi(e) != 0; }();
  const bool f32_try_tc = x->dtype == FCM_F32 && f32_tc && (geom->k == 3 || geom->k == 5);
  if ((x->dtype == FCM_F32 && !f32_try_tc) || !pitch_ok(x) || !pitch_ok(y))
    return launch_dwpw_simt(x->dtype, x->data, w_dw, to_epi(ep_dw), w_pw_packed, to_epi(ep_pw), y->data, g, st);
  int nsplit = 0;
  default_dwpw_tile(g, dwpw_mmax(x->dtype, g), dwpw_pair_dt(x->dtype, g));
  if (tile) {
    if (tile->tile_h > 0) g.th = tile->tile_h;
    if (tile->tile_w > 0) g.tw = tile->tile_w;
    if (tile->tile_n > 0) g.nb = tile->tile_n;
    if (tile->n_split > 0) nsplit = tile->n_split;
  }
  const int rc = launch_dwpw_tc(x->dtype, x->data, w_dw, to_epi(ep_dw), w_pw_packed, to_epi(ep_pw), y->data, g, nsplit, st);
  if (rc == FCM_E_INFEASIBLE && x->dtype == FCM_F32) {
    Geo gs{x->n, x->h, x->w, x->c, Ho, Wo, y->c, geom->k, geom->stride, geom->pad_t, geom->pad_l, 1, 0, 0};
    return launch_dwpw_simt(x->dtype, x->data, w_dw, to_epi(ep_dw), w_pw_packed, to_epi(ep_pw), y->data, gs, st);
  }
  return rc;
}

int fcm_pwpw(const fcm_tensor* x, const void* w1_packed, int32_t c_mid, const fcm_epilogue* ep1,
             const void* w2_packed, const fcm_epilogue* ep2, fcm_tensor* y, const fcm_tile* tile, void* stream) {
  (void)tile;
  FCM_TRY(check_tensor(x, "x", false));
  FCM_TRY(check_tensor(y, "y", false));
  if (!w1_packed || !w2_packed) return set_error(FCM_E_INVAL, "weights NULL");
  if (x->dtype != y->dtype) return set_error(FCM_E_INVAL, "x/y dtype differ");
  if (c_mid < 1) return set_error(FCM_E_INVAL, "pwpw: c_mid < 1");
  FCM_TRY(check_epi(ep1, x->dtype, "ep1"));
  FCM_TRY(check_epi(ep2, x->dtype, "ep2"));
  FCM_TRY(no_residual(ep1, "ep1"));
  FCM_TRY(check_residual(ep2, y, "ep2"));
  if (x->dtype == FCM_S8 && ep2->zp_in != ep1->zp_out)
    return set_error(FCM_E_INVAL, "pwpw: ep2.zp_in must equal ep1.zp_out (T's zero point)");
  if (y->n != x->n || y->h != x->h || y->w != x->w) return set_error(FCM_E_INVAL, "pwpw: y spatial dims mismatch");
  if (overlaps(x, y)) return set_error(FCM_E_INVAL, "pwpw: x and y overlap");
  if (x->dtype == FCM_F32 || !pitch_ok(x) || !pitch_ok(y) || ((size_t)c_mid * elem_size(x->dtype)) % 16)
    return set_error(FCM_E_UNSUPPORTED, "pwpw: tensor-core path needs bf16/f16/int8 and 16-byte pitches of x, T, y");
  const int M = x->n * x->h * x->w;
  return launch_pwpw_tc(x->dtype, x->data, w1_packed, to_epi(ep1), w2_packed, to_epi(ep2), y->data, M, x->c, c_mid,
                        y->c, static_cast<cudaStream_t>(stream));
}

int fcm_pwdw_r(const fcm_tensor* x, const void* w_pw_packed, const fcm_epilogue* ep_pw, const void* w_dw,
               const fcm_dw_geom* geom, const fcm_epilogue* ep_dw, fcm_tensor* y, const fcm_tile* tile, void* stream) {
  FCM_TRY(check_tensor(x, "x", false));
  FCM_TRY(check_tensor(y, "y", false));
  FCM_TRY(check_geom(geom));
  if (!w_dw || !w_pw_packed) return set_error(FCM_E_INVAL, "weights NULL");
  if (x->dtype != y->dtype) return set_error(FCM_E_INVAL, "x/y dtype differ");
  FCM_TRY(check_epi(ep_pw, x->dtype, "ep_pw"));
  if (x->dtype == FCM_S8 && ep_dw && ep_dw->zp_in != ep_pw->zp_out)
    return set_error(FCM_E_INVAL, "pwdw_r: ep_dw.zp_in must equal ep_pw.zp_out (T's zero point)");
  FCM_TRY(check_epi(ep_dw, x->dtype, "ep_dw"));
  FCM_TRY(no_residual(ep_pw, "ep_pw"));
  FCM_TRY(no_residual(ep_dw, "ep_dw"));
  const int Ho = out_dim(x->h, geom->k, geom->stride, geom->pad_t, geom->pad_b);
  const int Wo = out_dim(x->w, geom->k, geom->stride, geom->pad_l, geom->pad_r);
  if (Ho < 1 || Wo < 1) return set_error(FCM_E_INVAL, "pwdw_r: empty output");
  if (y->n != x->n || y->h != Ho || y->w != Wo) return set_error(FCM_E_INVAL, "pwdw_r: y dims mismatch");
  if (overlaps(x, y)) return set_error(FCM_E_INVAL, "pwdw_r: x and y overlap");
  Geo g{x->n, x->h, x->w, x->c, Ho, Wo, y->c, geom->k, geom->stride, geom->pad_t, geom->pad_l, 1, 0, 0};
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (x->dtype == FCM_F32 || !pitch_ok(x) || !pitch_ok(y))
    return launch_pwdw_simt(x->dtype, x->data, w_pw_packed, to_epi(ep_pw), w_dw, to_epi(ep_dw), y->data, g, st);
  default_pwdw_tile(g);
  if (tile) {
    if (tile->tile_h > 0) g.th = tile->tile_h;
    if (tile->tile_w > 0) g.tw = tile->tile_w;
    if (tile->tile_n > 0) g.nb = tile->tile_n;
  }
  return launch_pwdw_tc(x->dtype, x->data, w_pw_packed, to_epi(ep_pw), w_dw, to_epi(ep_dw), y->data, g, st);
}

}  // extern "C"
