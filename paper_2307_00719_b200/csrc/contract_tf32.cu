// contract_tf32.cu — the dominant kernel: contraction of X_new with a chained-slice table on
// the 5th-generation tensor cores (tcgen05, kind::tf32, fp32 accumulators in TMEM), with
// 3xTF32 splitting for fp32-level accuracy.
//
// Math: the two passes of the exact two-pass schedule evaluate
//   pass 1: Y_L[(l,t)][w] = sum_r X[l + L r + L Rr t] T_R[r][w]         A = X_t^T (M = l; loaded MN-major, transposed to K-major by the converters)
//   pass 2: Y_R[r][w]     = sum_{l,t} X[l + L r + L Rr t] T_L[(l,t)][w]  A = X      (M = r, K-major)
// i.e. the products X^new_[n] G^{≠n}_[2] of Alg. 4 l.9 / l.14, grouped.
// 3xTF32: A = A_hi + A_lo (A_hi = A with the low 13 mantissa bits cleared, A_lo = A - A_hi exact
// in fp32), B = B_hi + B_lo (rounded from the fp64 table), and
//   A B ~= A_hi [B_hi | B_lo] + A_lo B_hi      (two UMMAs per k-step, N = 2 Npad and Npad).
//
// Structure (one CTA per SM, persistent "stream-K" over units (M-tile, K-tile)):
//   warp 0      TMA producer: X tile via cp.async.bulk.tensor (128B swizzle, OOB zero-fill) and
//               the pre-tiled table block via cp.async.bulk, both on the stage's mbarrier
//   warp 1      UMMA issuer (one thread): 4 k-steps x 2 tcgen05.mma per stage, commit -> empty
//   warp 2      TMEM allocator (512 columns: two accumulator buffers)
//   warps 4-7   split converters: A_hi / A_lo (K-major) in shared memory, fence.proxy.async, arrive
//   warps 8-11  epilogue: tcgen05.ld the accumulator, hi+lo sum, fp32 red.add into Y
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>

#include "common.cuh"
#include "kernels.h"
#include "str_internal.h"
#include "tc_ptx.cuh"

namespace strb200 {

constexpr int kTcThreads = 384;
constexpr int kBM = 128;       // UMMA M
constexpr int kBK = 32;        // K per stage (one 128-byte swizzle row of fp32)
constexpr int kABytes = kBM * kBK * 4;   // 16 KB

struct TcParams {
  int64_t L, Rr, tn;
  int W, Npad, stages;
  int mb_per_t;    // pass 1: ceil(L/128) M-tiles per t
  int nlb;         // pass 2: ceil(L/32) K-tiles per t
  int64_t KT, U, upc;
  const float *Btiles;   // [KT][2 Npad rows][32 k] fp32, 128B-swizzled K-major blocks
  float *Y;              // fp32 output rows (zeroed), row stride W
};

template <int PASS>
__global__ void __launch_bounds__(kTcThreads, 1)
    k_contract_tf32(const __grid_constant__ CUtensorMap tmap, const TcParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int BBYTES = 2 * p.Npad * 128;
  const int STAGE = 2 * kABytes + BBYTES;
  const int S = p.stages;
  uint64_t *full = (uint64_t *)(smem + (size_t)S * STAGE);
  uint64_t *conv = full + S;
  uint64_t *empty = conv + S;
  uint64_t *accf = empty + S;
  uint64_t *acce = accf + 2;
  uint32_t *tslot = (uint32_t *)(acce + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t u0 = (int64_t)blockIdx.x * p.upc;
  const int64_t u1 = (u0 + p.upc < p.U) ? (u0 + p.upc) : p.U;
  if (u0 >= u1) return;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < S; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&conv[s], 128);
      tc::mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&accf[b], 1);
      tc::mbar_init(&acce[b], 128);
    }
    tc::fence_barrier_init();
    tc::prefetch_tmap(&tmap);
  }
  if (warp == 2) tc::tmem_alloc(tslot, 512);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tbase = *tslot;

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------------ TMA producer
      int s = 0;
      uint32_t ph = 0;
      for (int64_t u = u0; u < u1; ++u) {
        tc::mbar_wait(&empty[s], ph ^ 1);
        const int64_t tile = u / p.KT, kt = u % p.KT;
        uint8_t *A = smem + (size_t)s * STAGE;
        uint8_t *B = A + 2 * kABytes;
        tc::mbar_arrive_expect_tx(&full[s], kABytes + BBYTES);
        if (PASS == 1) {
          const int t = (int)(tile / p.mb_per_t), mb = (int)(tile % p.mb_per_t);
#pragma unroll
          for (int j = 0; j < 4; ++j) tc::tma_load_3d(A + j * 4096, &tmap, &full[s], mb * kBM + 32 * j, (int)kt * kBK, t);
        } else {
          const int t = (int)(kt / p.nlb), lb = (int)(kt % p.nlb);
          tc::tma_load_3d(A, &tmap, &full[s], lb * kBK, (int)tile * kBM, t);
        }
        tc::bulk_load(B, p.Btiles + kt * (int64_t)(BBYTES / 4), BBYTES, &full[s]);
        if (++s == S) { s = 0; ph ^= 1; }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ------------------------------------------------------------ UMMA issuer
      const uint32_t idesc2 = tc::idesc_tf32(kBM, 2 * p.Npad, 0, 0);
      const uint32_t idesc1 = tc::idesc_tf32(kBM, p.Npad, 0, 0);
      int s = 0;
      uint32_t ph = 0;
      int seg = 0;
      uint32_t use0 = 0, use1 = 0;
      for (int64_t u = u0; u < u1; ++u) {
        const bool first = (u == u0) || (u % p.KT == 0);
        const bool last = (u == u1 - 1) || ((u + 1) % p.KT == 0);
        const int buf = seg & 1;
        if (first) {
          tc::mbar_wait(&acce[buf], ((buf ? use1 : use0) & 1) ^ 1);
          tc::tc_fence_after();
        }
        tc::mbar_wait(&conv[s], ph);
        tc::tc_fence_after();
        const uint32_t a_hi = tc::smem_u32(smem + (size_t)s * STAGE);
        const uint32_t a_lo = a_hi + kABytes;
        const uint32_t b0 = a_hi + 2 * kABytes;
        const uint32_t d = tbase + (uint32_t)(buf * 256);
#pragma unroll
        for (int ks = 0; ks < kBK / 8; ++ks) {
          // K-major (both passes): advance 32 B (8 fp32) inside the 128-byte swizzle row
          const uint64_t ah = tc::smem_desc_sw128(a_hi + ks * 32, 16, 1024);
          const uint64_t al = tc::smem_desc_sw128(a_lo + ks * 32, 16, 1024);
          const uint64_t bd = tc::smem_desc_sw128(b0 + ks * 32, 16, 1024);
          tc::mma_tf32(d, ah, bd, idesc2, (first && ks == 0) ? 0u : 1u);
          tc::mma_tf32(d, al, bd, idesc1, 1u);
        }
        tc::mma_commit(&empty[s]);
        if (last) {
          tc::mma_commit(&accf[buf]);
          if (buf) use1++; else use0++;
          seg++;
        }
        if (++s == S) { s = 0; ph ^= 1; }
      }
    }
  } else if (warp >= 4 && warp < 8) {
    // -------------------------------------------------------------- 3xTF32 split converters
    // Pass 2: the TMA tile is already K-major; split in place (hi) and into the lo buffer.
    // Pass 1: the TMA tile is MN-major (4 boxes of [32 k][32 m]); each thread loads two 4x4
    // blocks, the 128 converter threads sync on a named barrier, then hi / lo are written
    // transposed into the K-major 128B-swizzled layout [128 m][32 k] (same as pass 2), so both
    // passes feed the tensor core through K-major descriptors.
    const int ct = threadIdx.x - 128;
    int s = 0;
    uint32_t ph = 0;
    for (int64_t u = u0; u < u1; ++u) {
      tc::mbar_wait(&full[s], ph);
      uint8_t *abase = smem + (size_t)s * STAGE;
      if (PASS == 2) {
        float4 *a = (float4 *)abase;
        float4 *alo = (float4 *)(abase + kABytes);
#pragma unroll
        for (int i = ct; i < kABytes / 16; i += 128) {
          float4 x = a[i], h, l;
          h.x = __uint_as_float(__float_as_uint(x.x) & 0xFFFFE000u);
          h.y = __uint_as_float(__float_as_uint(x.y) & 0xFFFFE000u);
          h.z = __uint_as_float(__float_as_uint(x.z) & 0xFFFFE000u);
          h.w = __uint_as_float(__float_as_uint(x.w) & 0xFFFFE000u);
          l.x = x.x - h.x;
          l.y = x.y - h.y;
          l.z = x.z - h.z;
          l.w = x.w - h.w;
          a[i] = h;
          alo[i] = l;
        }
      } else {
        float v[2][4][4];   // [block][d = k offset][e = m offset]
#pragma unroll
        for (int bI = 0; bI < 2; ++bI) {
          const int b = ct + 128 * bI;
          const int kq = b % 8, mq = b / 8;             // 4x4 block: k = 4kq.., m = 4mq..
          const int box = mq / 8, mc = mq % 8;          // m chunk inside the 32-wide box
#pragma unroll
          for (int d = 0; d < 4; ++d) {
            const int k = 4 * kq + d;
            const float4 x = *(const float4 *)(abase + box * 4096 + k * 128 + ((mc ^ (k % 8)) * 16));
            v[bI][d][0] = x.x;
            v[bI][d][1] = x.y;
            v[bI][d][2] = x.z;
            v[bI][d][3] = x.w;
          }
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
#pragma unroll
        for (int bI = 0; bI < 2; ++bI) {
          const int b = ct + 128 * bI;
          const int kq = b % 8, mq = b / 8;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int m = 4 * mq + e;
            float4 h, l;
            float *hp = &h.x, *lp = &l.x;
#pragma unroll
            for (int d = 0; d < 4; ++d) {
              const float x = v[bI][d][e];
              hp[d] = __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
              lp[d] = x - hp[d];
            }
            const int off = m * 128 + ((kq ^ (m % 8)) * 16);
            *(float4 *)(abase + off) = h;
            *(float4 *)(abase + kABytes + off) = l;
          }
        }
      }
      tc::fence_proxy_async_smem();
      tc::mbar_arrive(&conv[s]);
      if (++s == S) { s = 0; ph ^= 1; }
    }
  } else if (warp >= 8) {
    // -------------------------------------------------------------- epilogue
    const int q = warp % 4;
    const int row = q * 32 + lane;
    int seg = 0;
    int64_t u = u0;
    while (u < u1) {
      const int64_t tile = u / p.KT;
      const int64_t uend = ((tile + 1) * p.KT < u1) ? (tile + 1) * p.KT : u1;
      const int buf = seg & 1;
      tc::mbar_wait(&accf[buf], (uint32_t)((seg >> 1) & 1));
      tc::tc_fence_after();
      int64_t yrow;
      bool valid;
      if (PASS == 1) {
        const int64_t t = tile / p.mb_per_t, mb = tile % p.mb_per_t;
        const int64_t l = mb * kBM + row;
        valid = l < p.L;
        yrow = l + p.L * t;
      } else {
        const int64_t r = tile * kBM + row;
        valid = r < p.Rr;
        yrow = r;
      }
      const uint32_t taddr = tbase + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * 256);
      float *yr = p.Y + yrow * p.W;
      for (int c0 = 0; c0 < p.Npad; c0 += 16) {
        float hi[16], lo[16];
        tc::tmem_ld16(taddr + c0, hi);
        tc::tmem_ld16(taddr + p.Npad + c0, lo);
        if (valid) {
          if ((p.W & 3) == 0 && c0 + 16 <= p.W) {
#pragma unroll
            for (int i = 0; i < 16; i += 4)
              atomicAdd((float4 *)(yr + c0 + i),
                        make_float4(hi[i] + lo[i], hi[i + 1] + lo[i + 1], hi[i + 2] + lo[i + 2], hi[i + 3] + lo[i + 3]));
          } else {
#pragma unroll
            for (int i = 0; i < 16; ++i)
              if (c0 + i < p.W) atomicAdd(yr + c0 + i, hi[i] + lo[i]);
          }
        }
      }
      tc::tc_fence_before();
      tc::mbar_arrive(&acce[buf]);
      seg++;
      u = uend;
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (warp == 2) tc::tmem_dealloc(tbase, 512);
}

}  // namespace strb200

// =============================================================================================
// Host side.
using namespace strb200;

static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

static str_status tf_fail(str_state *h, const std::string &m) {
  h->err = m;
  return STR_E_CUDA;
}

str_status tf32_prepare(str_state *h) {
  if (h->dtype != STR_F32) {
    h->err = "3xTF32 contraction requires fp32 data (use STR_CONTRACT_F64 for fp64 X)";
    return STR_E_ARG;
  }
  if (h->L % 4 != 0) {
    h->err = "3xTF32 contraction needs the local product of the left-group dims (I_1/p * ... * I_k) to be a "
             "multiple of 4 (16-byte TMA row stride); use STR_CONTRACT_F64 or another split_k";
    return STR_E_ARG;
  }
  if (!g_encode) {
    cudaDriverEntryPointQueryResult q;
    void *fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return tf_fail(h, "cuTensorMapEncodeTiled unavailable");
    g_encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  }
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_contract_tf32<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(k_contract_tf32<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    attr = true;
  }
  h->tf32_ready = true;
  return STR_OK;
}

static int npad_of(int W) { return (W + 15) / 16 * 16; }

str_status tf32_ensure_workspace(str_state *h, int64_t tn) {
  const int N = h->N, k = h->k;
  const int W = h->R[k] * h->R[N - 1];   // R_{k+1} R_N
  const int Np = npad_of(W);
  const int64_t kt1 = cdiv(h->Rr, 32);
  const int64_t kt2 = tn * cdiv(h->L, 32);
  size_t tiles = (size_t)std::max(kt1, kt2) * 2 * Np * 32 * sizeof(float);
  size_t yf = (size_t)std::max<int64_t>(h->L * tn, h->Rr) * W * sizeof(float);
  auto grow = [&](DevBuf &b, size_t bytes) -> bool {
    if (b.bytes >= bytes) return true;
    if (b.p) cudaFree(b.p);
    b.p = nullptr;
    b.bytes = 0;
    if (cudaMalloc(&b.p, bytes) != cudaSuccess) return false;
    b.bytes = bytes;
    return true;
  };
  if (!grow(h->tab_split, tiles) || !grow(h->tf_part, yf) || !grow(h->tf_part2, yf)) {
    h->err = "cudaMalloc failed (3xTF32 workspace)";
    return STR_E_OOM;
  }
  return STR_OK;
}

int tf32_npad(int W) { return npad_of(W); }

static bool encode_x_map(str_state *h, CUtensorMap *tmap, const void *X, int pass, int64_t tn) {
  const int64_t L = h->L, Rr = h->Rr;
  cuuint64_t dims[3] = {(cuuint64_t)L, (cuuint64_t)Rr, (cuuint64_t)tn};
  cuuint64_t strides[2] = {(cuuint64_t)L * 4, (cuuint64_t)L * Rr * 4};
  cuuint32_t box[3] = {32, (cuuint32_t)(pass == 1 ? 32 : 128), 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = g_encode(tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void *>(X), dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    h->err = "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")";
    return false;
  }
  return true;
}

str_status tf32_graph_update(str_state *h, cudaGraphExec_t exec, int pass, const void *X, int64_t tn) {
  CUtensorMap tmap;
  if (!encode_x_map(h, &tmap, X, pass, tn)) return STR_E_CUDA;
  TcParams p;
  memcpy(&p, h->tf_params[pass - 1], sizeof(TcParams));
  void *args[2] = {&tmap, &p};
  cudaKernelNodeParams kp = {};
  kp.func = pass == 1 ? (void *)k_contract_tf32<1> : (void *)k_contract_tf32<2>;
  kp.gridDim = dim3(h->tf_grid[pass - 1]);
  kp.blockDim = dim3(kTcThreads);
  kp.sharedMemBytes = (unsigned)h->tf_smem[pass - 1];
  kp.kernelParams = args;
  kp.extra = nullptr;
  cudaError_t e = cudaGraphExecKernelNodeSetParams(exec, h->tf_node[pass - 1], &kp);
  if (e != cudaSuccess) {
    h->err = std::string("cudaGraphExecKernelNodeSetParams: ") + cudaGetErrorString(e);
    return STR_E_CUDA;
  }
  return STR_OK;
}

int launch_contract_tf32(str_state *h, const void *X, int pass, int W, int64_t tn, float *Y) {
  cudaStream_t st = h->st;
  const int Np = npad_of(W);
  const int64_t L = h->L, Rr = h->Rr;
  // tensor map over X: dims (l, r, t), 128B swizzle, box {32, 32|128, 1}
  CUtensorMap tmap;
  if (!encode_x_map(h, &tmap, X, pass, tn)) return -1;
  // 3. the persistent stream-K contraction
  TcParams p;
  p.L = L;
  p.Rr = Rr;
  p.tn = tn;
  p.W = W;
  p.Npad = Np;
  const int stage_bytes = 2 * kABytes + 2 * Np * 128;
  p.stages = std::min(6, (int)((220 * 1024 - 1024 - 256) / stage_bytes));
  p.mb_per_t = (int)cdiv(L, kBM);
  p.nlb = (int)cdiv(L, 32);
  const int64_t tiles = pass == 1 ? (int64_t)p.mb_per_t * tn : cdiv(Rr, kBM);
  p.KT = pass == 1 ? cdiv(Rr, kBK) : tn * p.nlb;
  p.U = tiles * p.KT;
  int grid = (int)std::min<int64_t>(148, p.U);
  p.upc = cdiv(p.U, grid);
  grid = (int)cdiv(p.U, p.upc);
  p.Btiles = (const float *)h->tab_split.p;
  p.Y = Y;
  const int64_t M = pass == 1 ? L * tn : Rr;
  cudaMemsetAsync(p.Y, 0, (size_t)M * W * sizeof(float), st);
  tl_mark(h, "memset", 0);
  const size_t smem = (size_t)p.stages * stage_bytes + 1024 + 256;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (h->profiling) {
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, st);
  }
  if (pass == 1)
    k_contract_tf32<1><<<grid, kTcThreads, smem, st>>>(tmap, p);
  else
    k_contract_tf32<2><<<grid, kTcThreads, smem, st>>>(tmap, p);
  if (h->capturing) {
    // remember the node so that graph replays can re-point it at new X (tf32_graph_update)
    cudaStreamCaptureStatus cs;
    const cudaGraphNode_t *deps = nullptr;
    size_t nd = 0;
    if (cudaStreamGetCaptureInfo(st, &cs, nullptr, nullptr, &deps, &nd) != cudaSuccess || nd != 1) {
      h->err = "cannot locate the captured contraction node";
      return -1;
    }
    h->tf_node[pass - 1] = deps[0];
    static_assert(sizeof(TcParams) <= sizeof(h->tf_params[0]), "TcParams too large");
    memcpy(h->tf_params[pass - 1], &p, sizeof(TcParams));
    h->tf_grid[pass - 1] = grid;
    h->tf_smem[pass - 1] = smem;
  }
  tl_mark(h, pass == 1 ? "contract_tf32_p1" : "contract_tf32_p2");
  if (h->profiling) {
    cudaEventRecord(e1, st);
    h->prof_events.push_back({pass, e0, e1});
  }
  return 0;
}
