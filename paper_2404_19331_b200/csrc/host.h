// Host-side internals of libfcm.so (not part of the public ABI).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <string>
#include <utility>

#include "fcm.h"

namespace fcm {

struct Epi;  // common.cuh

// thread-local error detail + status helper
int set_error(int status, const std::string& msg);
extern std::atomic<uint64_t> g_launches;

struct DevProps {
  int sms = 148;
  int smem_optin = 232448;
  int l2_bytes = 126 * 1024 * 1024;
  int cc_major = 10, cc_minor = 0;
};
const DevProps& device_props();  // cached per process (device of the calling thread at first use)

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda needed).
bool encode_tmap(CUtensorMap* m, CUtensorMapDataType dt, uint32_t rank, const void* base, const uint64_t* dims,
                 const uint64_t* strides_bytes, const uint32_t* box, CUtensorMapSwizzle swz);
CUtensorMapDataType tmap_dtype(int dt);
int elem_size(int dt);

// Tile geometry resolved for a launch.
struct Geo {
  int N, H, W, C, Ho, Wo, Cout;   // Cout: PW output (DWPW) or C_mid (PWDW)
  int k, s, pt, pl;
  int nb, th, tw;                 // images x rows x cols per output tile
};

// launchers (return FCM_OK or an FCM_E_* code; all validation already done by the API layer)
int launch_dw(int dt, const void* x, const void* wdw, const Epi& ep, void* y, const Geo& g, cudaStream_t st);
int launch_pw_tc(int dt, const void* x, const void* wp, const Epi& ep, void* y, int M, int K, int N, int nsplit,
                 cudaStream_t st);  // nsplit <= 0: default C_out split
int launch_pw_simt(int dt, const void* x, const void* wp, const Epi& ep, void* y, int M, int K, int N, cudaStream_t st);
int launch_dw_simt(int dt, const void* x, const void* wdw, const Epi& ep, void* y, const Geo& g, cudaStream_t st);
int launch_dwpw_tc(int dt, const void* x, const void* wdw, const Epi& ed, const void* wp, const Epi& ep, void* y,
                   const Geo& g, int n_split, cudaStream_t st);
int launch_dwpw_simt(int dt, const void* x, const void* wdw, const Epi& ed, const void* wp, const Epi& ep, void* y,
                     const Geo& g, cudaStream_t st);
int launch_pwdw_tc(int dt, const void* x, const void* wp, const Epi& ep, const void* wdw, const Epi& ed, void* y,
                   const Geo& g, cudaStream_t st);
int launch_pwdw_simt(int dt, const void* x, const void* wp, const Epi& ep, const void* wdw, const Epi& ed, void* y,
                     const Geo& g, cudaStream_t st);
int launch_pwpw_tc(int dt, const void* x, const void* w1, const Epi& ep1, const void* w2, const Epi& ep2, void* y,
                   int M, int K1, int Cmid, int N, cudaStream_t st);
int launch_pack_pw(int dt, int cin, int cout, const void* w, void* packed, cudaStream_t st);
int launch_dw_tc_i8(const void* x, const void* wdw, const Epi& ep, void* y, const Geo& g, cudaStream_t st);
int launch_dw_nchw(int dt, const void* x, const void* wdw, const Epi& ep, void* y, const Geo& g, cudaStream_t st);

int check_launch(const char* what);

// Programmatic dependent launch (FCM_PDL=0 disables): consecutive kernels on a stream overlap the
// successor's prologue with the predecessor's tail; kernels call pdl_wait() before touching
// activations, so results are unchanged.
bool pdl_enabled();
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                            Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

}  // namespace fcm
