// common.cuh — shared device/host helpers for the STR library (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <cstdlib>
#include <stdint.h>

#include <mutex>
#include <utility>

#ifndef __CUDA_ARCH__
#include <string>
#endif

#define STR_MAXR 16          // max TR rank per mode supported by the register-resident kernels
#define STR_MAXW 128         // max R_n R_{n+1}

namespace strb200 {

// One factor of a chained slice product: slices G(i) of shape Ra x Rb stored in the
// G(2) layout used on the device, element (a, b) of slice i at G[i*Ra*Rb + a + Ra*b]
// (classical mode-2 unfolding, column r_n + R_n r_{n+1}).  The factor's index is
// i = (e / stride) % I for a flat multi-index e.
struct Factor {
  const double *G;
  int32_t I;
  int32_t Ra, Rb;
  int64_t stride;
};

constexpr int kMaxFactors = 8;

struct FactorList {
  Factor f[kMaxFactors];
  int32_t n;
};

// Absorb descriptor: contract one index of a matrix-valued tensor Y with core slices.
//   Y has multi-index dims d[0..nd-1] (first fastest) and entries P x Q row-major.
//   left : Y'(rest)[p', q] = sum_i A(i)[p', p] Y(rest, i)[p, q]    (A: P' x P)
//   right: Y'(rest)[p, q'] = sum_i Y(rest, i)[p, q] A(i)[q, q']    (A: Q x Q')
struct AbsorbDesc {
  int32_t nd;
  int64_t d[8];
  int32_t pos;     // which index of Y is contracted
  int32_t P, Q;    // entry shape of Y
  int32_t left;    // 1 = left, 0 = right
  const double *A; // slices in G(2) layout
  int32_t Ra, Rb;  // A slice shape
};

// Chained-slice table over work units (t', l-block of 32): entries e = l + Lk t', l < Lk, t' < tk.
// Npad > 0 additionally emits the pre-tiled 3xTF32 operand blocks (2 Npad rows x 32 k).
struct TableDesc {
  FactorList fl;
  int64_t Lk, tk;
  int32_t Npad;
  float4 *zero = nullptr;   // optional: zeroed by the table kernel (the next contraction's output)
  int64_t zero_n4 = 0;      // float4s to zero
  float *out32 = nullptr;   // optional: the rows also in fp32 (same layout as out64)
};

// Epilogue of k_chain_gemm: mode 0 = store C; 1 = Q = H_<2>; 2 = Q += H_<2> (Rn = R_n, Rn1 = R_{n+1}).
struct QEpi {
  double *Q;
  int32_t Rn, Rn1;
  int32_t mode;
  // mode 4 (fit epilogue of str_fit): C[row][col] = X^hat at (l, r, t) with row = l + L t, col = r;
  // per-CTA partial sums (sum (x - x^hat)^2, sum x^2) of the tile go to part[CTA]
  const void *X = nullptr;
  int64_t L = 0, Rr = 0;
  int32_t xf64 = 0;
  double2 *part = nullptr;
};

__host__ __device__ inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Function attributes (dynamic shared-memory opt-ins, carve-out preferences) are per device and
// handles on different devices may be created concurrently: run the setup once per device ordinal.
constexpr int kMaxDevices = 64;
struct PerDeviceOnce {
  std::once_flag f[kMaxDevices];
};
template <class F>
inline void once_per_device(PerDeviceOnce &o, F &&fn) {
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess || d < 0 || d >= kMaxDevices) d = 0;
  std::call_once(o.f[d], std::forward<F>(fn));
}

// Launch with the programmatic-stream-serialization attribute (programmatic dependent launch): the
// kernel may start while its predecessor in the stream finishes; kernels launched this way begin
// with griddepcontrol.launch_dependents + griddepcontrol.wait (PDL_PROLOGUE) before touching
// memory.  STR_PDL=<mask> selects the kernel classes (0: none).
#define PDL_PROLOGUE()                                              \
  do {                                                              \
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); \
    asm volatile("griddepcontrol.wait;" ::: "memory");              \
  } while (0)
// Kernel classes for the PDL mask (STR_PDL = bitmask; default kPdlDefault)
constexpr int kPdlDmma = 1, kPdlAbsorb = 2, kPdlInv = 4, kPdlRstr = 8;
constexpr int kPdlDefault = kPdlDmma | kPdlInv | kPdlRstr;   // measured: PDL on the absorbs slows C5 (their early CTAs crowd the passes)
static int pdl_mask() {
  static const int m = [] {
    const char *e = getenv("STR_PDL");
    return e ? atoi(e) : kPdlDefault;
  }();
  return m;
}
template <typename... KArgs, typename... Args>
static void pdl_launch(int cls, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args... args) {
  const bool on = (pdl_mask() & cls) != 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = on ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kern, ((KArgs)args)...);
}

}  // namespace strb200
