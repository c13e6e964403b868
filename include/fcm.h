/*
 * fcm.h -- C ABI of libfcm.so: Fused Convolutional Modules (FCMs) for NVIDIA B200 (sm_100a).
 *
 * Implements the data-parallel hot path of "Fusing Depthwise and Pointwise Convolutions for
 * Efficient Inference on GPUs" (arXiv 2404.19331; citations P:<line> are PAPER.md lines):
 *
 *   fcm_dw      layer-by-layer depthwise conv + Norm + Act      ("LBL")
 *   fcm_pw      layer-by-layer pointwise conv + Norm + Act
 *   fcm_dwpw    FCM DWPW: DW -> on-chip commBuffer -> PW          (Listing 1)
 *   fcm_pwdw_r  FCM PWDW_R: PW over the halo tile (recomputed) -> on-chip -> DW
 *               (PWDW without redundancy is the full-map tile of the same call)
 *   fcm_pwpw    FCM PWPW: PW -> on-chip T -> PW
 *   fcm_pack_pw offline PW weight packing ("weight packing is done offline")
 *   fcm_plan    FusePlanner re-parameterised for B200
 *
 * Definitions (identical to oracle/conv.py):
 *   DW  O[n,y,x,c]  = eps_c( sum_{i,j<k} X[n, y*s-pad_t+i, x*s-pad_l+j, c] * Wdw[i][j][c] ),
 *                     out-of-image taps contribute 0; Ho = (H+pad_t+pad_b-k)/s + 1 (floor).
 *   PW  O[p,co]     = eps_co( sum_ci X[p,ci] * Wpw[ci][co] ) for every pixel p.
 *   eps (float)     v = acc*scale[c] + bias[c]; NONE | RELU | RELU6 | SILU | GELU; + residual
 *                     (optional); round-to-nearest-even to the output dtype (scale/bias NULL -> 1 / 0).
 *   eps (int8)      r = ((acc + bias_q[c]) * mult_q[c] + 2^(shift_q[c]-1)) >> shift_q[c]
 *                     (64-bit product, arithmetic shift) + zp_out, clamped to [qmin, qmax].
 *                     acc = sum (q - zp_in) * w, int32. RELU/RELU6 are encoded by qmin/qmax.
 *   DWPW  = PW(DW(X)); PWDW_R = DW(PW(X)); PWPW = PW2(PW1(X)). The intermediate T is rounded/requantised to the
 *   feature-map dtype but never exists in global memory; the DW of PWDW_R
 *   zero-pads T itself (an out-of-image T tap is 0 / the zero point, not eps_pw(PW(0))).
 *
 * Layouts and dtypes
 *   Activations: NHWC (FCM_NHWC) dense; fcm_dw also accepts NCHW.
 *   Wdw: [k][k][C] dense, same dtype as the activations (int8: symmetric, no zero point).
 *   Wpw: canonical [C_in][C_out]; every PW-consuming call takes the PACKED form produced by
 *        fcm_pack_pw (currently K-major [C_out][C_in]; size from fcm_pack_pw_bytes).
 *   Epilogue vectors: float scale/bias [C] for float paths; int32 bias_q/mult_q/shift_q [C]
 *        for int8. mult_q in [2^30, 2^31), shift_q in [1, 62].
 *   dtype FCM_F32 / FCM_BF16 / FCM_F16 / FCM_S8 applies to X, T, Y and the weights alike.
 *
 * Ownership / concurrency
 *   Every pointer is caller-owned device memory (the epilogue vectors too); the library
 *   allocates nothing on the hot path and keeps no pointer after return. Work is enqueued on
 *   `stream` (a cudaStream_t passed as void*; NULL = legacy default stream) and is
 *   asynchronous; there is no implicit synchronisation. Input and output must not overlap.
 *   Re-entrant and thread-safe.
 *   Kernels are launched with programmatic stream serialization (programmatic dependent
 *   launch): a call's kernel may start its prologue (barrier / TMEM setup, weight and epilogue
 *   constant staging) while the previous kernel on the stream drains, and waits for that kernel
 *   to complete (griddepcontrol.wait) before it reads activations or writes its output. So
 *   stream order is preserved for activations; weights and epilogue vectors must not be written
 *   by the kernel immediately preceding the call on the same stream (synchronise or insert any
 *   other stream operation in between). Environment FCM_PDL=0 turns this off (plain
 *   stream-ordered launches).
 *
 * Errors
 *   Every entry point returns FCM_OK (0) or a negative FCM_E_* code; validation is synchronous
 *   and happens before any launch, so on error nothing was enqueued. fcm_last_error() returns a
 *   thread-local human-readable detail of the last failure on the calling thread.
 */
#ifndef FCM_H_
#define FCM_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FCM_VERSION 1

/* status codes */
#define FCM_OK 0
#define FCM_E_INVAL (-1)       /* null pointer, shape/geometry mismatch, bad enum */
#define FCM_E_ALIGN (-2)       /* base pointer or row pitch not 16-byte aligned */
#define FCM_E_UNSUPPORTED (-3) /* valid request not (yet) implemented on the GPU path */
#define FCM_E_INFEASIBLE (-4)  /* tile config violates smem / TMEM / grid limits */
#define FCM_E_CUDA (-5)        /* CUDA launch / driver error (detail in fcm_last_error) */
#define FCM_E_BUFSZ (-6)       /* output string buffer too small; *needed is set */

/* dtypes, layouts, activations */
#define FCM_F32 0
#define FCM_BF16 1
#define FCM_F16 2
#define FCM_S8 3
#define FCM_NHWC 0
#define FCM_NCHW 1
#define FCM_ACT_NONE 0
#define FCM_ACT_RELU 1
#define FCM_ACT_RELU6 2
#define FCM_ACT_SILU 3 /* v * sigmoid(v) (EfficientNet); float paths only */
#define FCM_ACT_GELU 4 /* 0.5 v (1 + erf(v / sqrt 2)) (CeiT / CMT); float paths only */

/* A dense 4-D activation tensor in device memory. n,h,w,c are logical dims (any layout). */
typedef struct {
  void* data;
  int32_t dtype;  /* FCM_F32 | FCM_BF16 | FCM_F16 | FCM_S8 */
  int32_t layout; /* FCM_NHWC | FCM_NCHW */
  int32_t n, h, w, c;
} fcm_tensor;

/* Depthwise geometry: square k x k filter, uniform stride (P:173 single "Strides"),
 * explicit 4-sided zero padding, dilation 1, channel multiplier 1. */
typedef struct {
  int32_t k, stride, pad_t, pad_l, pad_b, pad_r;
} fcm_dw_geom;

/* Conv-Norm-Activation epilogue. Float paths use act/scale/bias; int8 uses the
 * quantised fields (bias_q, mult_q, shift_q, zp_in, zp_out, qmin, qmax). Device pointers.
 * residual (optional, NULL = none, the inverted-residual / MBConv / IRFFN
 * shortcut): a tensor of the OUTPUT's shape and dtype (NHWC, dense) added after the
 * activation, y = round(act(acc*scale + bias) + residual). Float dtypes only, and only on the
 * epilogue that writes a call's output through a pointwise conv: fcm_pw, fcm_dwpw's ep_pw,
 * fcm_pwpw's ep2 (elsewhere FCM_E_UNSUPPORTED). It may not overlap the output. */
typedef struct {
  int32_t act;
  const float* scale;
  const float* bias;
  const int32_t* bias_q;
  const int32_t* mult_q;
  const int32_t* shift_q;
  int32_t zp_in, zp_out, qmin, qmax;
  const void* residual;
} fcm_epilogue;

/* Optional tile override (NULL = the library's default for the shape). Output-space tile
 * tile_h x tile_w pixels of tile_n images; n_split = number of C_out slices (DWPW, and the
 * tensor-core PW: its only tile field) or the intermediate-channel slice width td (PWDW_R, as
 * c_chunk). 0 = default for that field. DWPW tiles hold at most 256 pixels (two M=128 MMA row
 * blocks) on the bf16/f16 3x3 path and 128 otherwise; PWDW_R halo tiles at most 512 pixels for
 * bf16/f16 (four row blocks), 256 for int8. The int8 stride-1 3x3 / 5x5 DW on maps >= 14 x 14
 * runs on the tensor cores with a fixed 16 x 8 output tile (the tile is ignored there). A tile
 * whose staging does not fit shared memory / TMEM returns FCM_E_INFEASIBLE. */
typedef struct {
  int32_t tile_h, tile_w, tile_n, c_chunk, n_split;
} fcm_tile;

/* Layer-by-layer depthwise conv. x [N,H,W,C], w_dw [k][k][C], y [N,Ho,Wo,C].
 * k in {3, 5, 7}, stride in {1, 2} (else FCM_E_UNSUPPORTED). NHWC pixel pitch C * elem:
 * a multiple of 16 B -> TMA-staged tiles; a multiple of 4 B -> the same tiles staged with
 * cp.async; otherwise an element-wise CUDA-core kernel. The fused calls (fcm_dwpw,
 * fcm_pwdw_r) are built for k in {3, 5}. */
int fcm_dw(const fcm_tensor* x, const void* w_dw, const fcm_dw_geom* geom, const fcm_epilogue* ep,
           fcm_tensor* y, const fcm_tile* tile, void* stream);

/* Layer-by-layer pointwise conv. x [N,H,W,C_in], w_pw_packed from fcm_pack_pw, y [N,H,W,C_out].
 * bf16 / f16 / int8 on the tensor cores; fp32 too, as 3xTF32 (x_hi.w_hi + x_hi.w_lo + x_lo.w_hi,
 * ~fp32 accuracy; env FCM_PW_F32_TC=0 selects the FFMA kernel). Pixel pitches that are not a
 * multiple of 16 B run the CUDA-core kernel. */
int fcm_pw(const fcm_tensor* x, const void* w_pw_packed, const fcm_epilogue* ep, fcm_tensor* y,
           const fcm_tile* tile, void* stream);

/* FCM DWPW: y = PW(DW(x)). x [N,H,W,C_in], w_dw [k][k][C_in], w_pw_packed (C_in -> C_out),
 * y [N,Ho,Wo,C_out]. For int8, ep_pw->zp_in must equal ep_dw->zp_out (T's zero point). fp32 runs the
 * tensor-core kernel (3xTF32 PW) when the C_in x C_out weights and their split fit shared memory,
 * else the FFMA kernel. */
int fcm_dwpw(const fcm_tensor* x, const void* w_dw, const fcm_dw_geom* geom, const fcm_epilogue* ep_dw,
             const void* w_pw_packed, const fcm_epilogue* ep_pw, fcm_tensor* y, const fcm_tile* tile,
             void* stream);

/* FCM PWDW_R: y = DW(PW(x)). x [N,H,W,C_in], w_pw_packed (C_in -> C_mid), w_dw [k][k][C_mid],
 * y [N,Ho,Wo,C_mid]. For int8, ep_dw->zp_in must equal ep_pw->zp_out. */
int fcm_pwdw_r(const fcm_tensor* x, const void* w_pw_packed, const fcm_epilogue* ep_pw, const void* w_dw,
               const fcm_dw_geom* geom, const fcm_epilogue* ep_dw, fcm_tensor* y, const fcm_tile* tile,
               void* stream);

/* FCM PWPW: y = PW2(PW1(x)). x [N,H,W,C_in], w1_packed (C_in -> c_mid), w2_packed (c_mid -> C_out),
 * y [N,H,W,C_out]; T = eps1(x . W1) is rounded / requantised to the feature-map dtype and stays in
 * shared memory (one 128-pixel tile at a time). Tensor-core path only: bf16 / f16 / int8, c_mid <=
 * 128, 16-byte pixel pitches for x, T and y (otherwise FCM_E_UNSUPPORTED: run two fcm_pw calls).
 * For int8, ep2->zp_in must equal ep1->zp_out. `tile` is reserved (pass NULL). */
int fcm_pwpw(const fcm_tensor* x, const void* w1_packed, int32_t c_mid, const fcm_epilogue* ep1,
             const void* w2_packed, const fcm_epilogue* ep2, fcm_tensor* y, const fcm_tile* tile, void* stream);

/* Bytes of the packed PW weight buffer for (dtype, C_in, C_out). 0 on invalid input. */
size_t fcm_pack_pw_bytes(int32_t dtype, int32_t c_in, int32_t c_out);

/* Offline PW weight packing: w_pw [C_in][C_out] (device) -> w_packed (device,
 * fcm_pack_pw_bytes bytes, caller-allocated). Asynchronous on `stream`. */
int fcm_pack_pw(int32_t dtype, int32_t c_in, int32_t c_out, const void* w_pw, void* w_packed, void* stream);

/* FusePlanner. model_json: {"dtype", "batch", "layers": [...], ...};
 * gpu_json: B200 spec overrides or NULL (defaults: 148 SMs, 227 KB smem/CTA, 512 TMEM cols,
 * L2 queried from the current device if one is present). Writes a NUL-terminated plan JSON into
 * out[cap]; *needed receives the required size including the NUL. Host-only, no CUDA work. */
int fcm_plan(const char* model_json, const char* gpu_json, char* out, size_t cap, size_t* needed);

/* Number of kernels launched by this library since load (process-wide counter). */
uint64_t fcm_launch_count(void);

const char* fcm_status_str(int status);
const char* fcm_last_error(void);
int fcm_version(void);

#ifdef __cplusplus
}
#endif
#endif /* FCM_H_ */
