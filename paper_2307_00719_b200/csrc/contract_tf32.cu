// contract_tf32.cu — the dominant kernel: contraction of X_new with a chained-slice table on
// the 5th-generation tensor cores (tcgen05, kind::tf32, fp32 accumulators in TMEM), with
// 3xTF32 splitting for fp32-level accuracy.
//
// Math: the two passes of the exact two-pass schedule evaluate
//   pass 1: Y_L[(l,t)][w] = sum_r X[l + L r + L Rr t] T_R[r][w]         A = X_t^T (M = l; MN-major tile)
//   pass 2: Y_R[r][w]     = sum_{l,t} X[l + L r + L Rr t] T_L[(l,t)][w]  A = X      (M = r, K-major tile)
// i.e. the products X^new_[n] G^{≠n}_[2] of Alg. 4 l.9 / l.14, grouped.
// 3xTF32: A = A_hi + A_lo (A_hi = A with the low 13 mantissa bits cleared, A_lo = A - A_hi exact
// in fp32), B = B_hi + B_lo (rounded from the fp64 table), and
//   A B ~= A_hi B_hi + A_hi B_lo + A_lo B_hi      (three UMMAs per k-step into one accumulator).
//
// Structure (one CTA per SM, persistent "stream-K" over units (M-block of 256 rows, K-tile of 32)):
//   warp 0       TMA producer: the two 128-row X tiles (cp.async.bulk.tensor, 128B swizzle, OOB
//                zero-fill) into the X ring
//   warp 3       table producer: the pre-tiled hi/lo table block (cp.async.bulk) into the table ring
//   warp 1       UMMA issuer (one thread): per M-tile and k-step 3 x tcgen05.mma.kind::tf32 with A
//                from TMEM (A_hi | A_lo) and B from shared memory (B_hi | B_lo); one B stage feeds
//                both M-tiles, halving the table traffic per FLOP
//   warp 2       TMEM allocator (512 columns: 2 accumulators of Npad, 2 slots of A_hi|A_lo per M-tile)
//   warps 4-11   split converters: each thread reads its X row from the stage, splits hi / lo and
//                writes them to TMEM (tcgen05.st), so neither the split operands nor the MMA's A
//                reads touch shared memory
//   warps 12-15  epilogue: tcgen05.ld the accumulators, fp32 red.add into Y (stream-K partials)
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

constexpr int kTcThreads = 512;
constexpr int kTcThreadsGen = 576;   // + warps 16, 17: table generators with warps 2, 3 (fused pass 2)
constexpr int kBM = 128;       // UMMA M
constexpr int kMT = 2;         // M-tiles per CTA (share every B stage)
constexpr int kBK = 32;        // K per stage (one 128-byte swizzle row of fp32)
constexpr int kABytes = kBM * kBK * 4;   // 16 KB per X tile
constexpr uint32_t kASlot0 = 256;        // A slots at [256, 512): slot a, M-tile mt at 256 + (2a + mt) * 64
// epilogue staging: per lane quarter one [32 rows][Wb] fp32 box (W <= 128) -> one M-tile.  Each
// lane writes its row; the row stride Wb >= W is padded to Wb = 4 (mod 32) floats so that the lanes'
// 16-byte stores spread over all banks (W = 64 would put every lane on the same four banks).  The
// TMA box is Wb wide; its columns >= W lie outside the tensor and are clipped by the reduce-add.
__host__ __device__ constexpr int ybox_w(int W) { return W + ((4 - W) % 32 + 32) % 32; }
__host__ __device__ constexpr int ystage_box_bytes(int W) { return (32 * ybox_w(W) * 4 + 1023) / 1024 * 1024; }
__host__ __device__ constexpr int ystage_bytes(int W) { return 4 * ystage_box_bytes(W); }

struct TcParams {
  int64_t L, Rr, tn;
  int W, Npad, stages, bstages;   // X ring / table ring depths
  int mt_per_t;    // 128-row M-tiles per t (pass 1: ceil(L/128)) or in all (pass 2: ceil(Rr/128))
  int mtiles;      // M-tiles in all (pass 1: mt_per_t tn); an M-block pairs tiles 2b, 2b+1
  int nlb;         // pass 2: ceil(L/32) K-tiles per t
  int yred;        // 1: epilogue by TMA reduce-add through a one-tile staging area (W % 4 == 0); 0: red.add
  int64_t KT, U, upc;
  const float *Btiles;   // [KT][2 Npad rows][32 k] fp32, 128B-swizzled K-major blocks
  float *Y;              // fp32 output rows (zeroed), row stride W (pass 1: row l + L t)
  long long *dbg;        // optional pipeline trace of CTA 0 (diagnostic; nullptr in production)
  int dbg_flags;         // diagnostic: bit0 skip table loads, bit1 skip X loads, bit2 skip TMEM stores, bit3 one commit per unit, bit4 spin waits, bit5 converters skip smem reads (wrong results)
  // fused table generation (pass 2, GR > 0): T_L[(l, t)] = F[(l mod P) + P t] G_k(l / P)
  const float *GA;       // fp32 prefix rows F, each R x R row-major ([a][b]), row f + P t
  const double *GB;      // G_k core slices, R x R column-major (b + R c), slice i at i R^2
  int P;                 // prefix period Lf = (I_1/p) I_2 ... I_{k-1} (>= 32)
};

__device__ __forceinline__ void cp_async16(void *smem, const void *g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(tc::smem_u32(smem)), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void gen_bar_sync() { asm volatile("bar.sync 1, 128;" ::: "memory"); }   // the 4 generator warps

__device__ __forceinline__ float tf32_rna_f(float x) {   // round to the nearest tf32 (ties away)
  return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
}

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),
      "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
      "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// D[tmem] (+)= A[tmem] * B[smem], kind::tf32 (fp32 accumulate), one CTA.  Executed by a whole
// warp with warp-uniform operands (kept in uniform registers); one elected lane issues.
__device__ __forceinline__ void mma_tf32_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_commit_elect(uint64_t *bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(tc::smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

template <int PASS, int GR>
__global__ void __launch_bounds__(GR ? kTcThreadsGen : kTcThreads, 1)
    k_contract_tf32(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ CUtensorMap ymap,
                    const TcParams p) {
  if (p.dbg && threadIdx.x == 0) p.dbg[1024 + blockIdx.x * 4 + 0] = gtimer();
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  // X ring (HBM stream; slots freed by the converters as soon as the tile is in TMEM) and a
  // shallower table ring (L2-resident; slots freed by the MMA commit).
  const int BBYTES = 2 * p.Npad * 128;
  const int XSTAGE = kMT * kABytes;
  const int SX = p.stages, SB = p.bstages;
  uint8_t *xbuf = smem;
  uint8_t *bbuf = smem + (size_t)SX * XSTAGE;
  uint8_t *ystage = bbuf + (size_t)SB * BBYTES;   // one-tile epilogue staging ([q] dense [32][W] fp32 boxes)
  // fused generation: two stages of the K-tile's 32 prefix rows F (fp32, R x R each)
  float *astage = (float *)(ystage + (p.yred ? ystage_bytes(p.W) : 0));
  uint64_t *xfull = (uint64_t *)((uint8_t *)astage + (GR ? 2 * 32 * GR * GR * 4 : 0));
  uint64_t *xempty = xfull + SX;
  uint64_t *bfull = xempty + SX;
  uint64_t *bempty = bfull + SB;
  uint64_t *conv = bempty + SB;    // [2] A slot filled (converters -> MMA)
  uint64_t *aempty = conv + 2;     // [2] A slot free   (MMA -> converters)
  uint64_t *accf = aempty + 2;     // accumulators complete (MMA -> epilogue)
  uint64_t *acce = accf + 1;       // [2] accumulator of M-tile mt drained (epilogue -> MMA)
  uint64_t *bfree = bempty;
  uint32_t *tslot = (uint32_t *)(acce + 2);

  // warp index broadcast from lane 0: provably warp-uniform, so role branches are uniform and the
  // MMA warp keeps its descriptors / TMEM addresses in uniform registers (no per-MMA R2UR)
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x / 32), 0), lane = threadIdx.x % 32;
  const int64_t u0 = (int64_t)blockIdx.x * p.upc;
  const int64_t u1 = (u0 + p.upc < p.U) ? (u0 + p.upc) : p.U;
  if (u0 >= u1) return;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < SX; ++s) {
      tc::mbar_init(&xfull[s], 1);
      tc::mbar_init(&xempty[s], 8);    // one arrival per converter warp
    }
    for (int s = 0; s < SB; ++s) {
      tc::mbar_init(&bfull[s], GR ? 4 : 1);   // (fused: one arrival per generator warp)
      tc::mbar_init(&bempty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      tc::mbar_init(&conv[a], 8);
      tc::mbar_init(&aempty[a], 1);
    }
    tc::mbar_init(accf, 1);
    tc::mbar_init(&acce[0], 4);      // one arrival per epilogue warp
    tc::mbar_init(&acce[1], 4);
    tc::fence_barrier_init();
    tc::prefetch_tmap(&tmap);
    if (p.yred) tc::prefetch_tmap(&ymap);
  }
  if (warp == 2) tc::tmem_alloc(tslot, 512);
  if (p.W < p.Npad) {   // table padding rows are never loaded: zero them once (read by the MMA)
    const int prow = p.Npad - p.W;                       // padding rows per half, 128 B each
    const int per = 2 * prow * 8;                        // float4 per slot
    for (int i = threadIdx.x; i < SB * per; i += blockDim.x) {
      const int slot = i / per, r = i % per, half = r / (prow * 8), w = r % (prow * 8);
      ((float4 *)(bbuf + (size_t)slot * BBYTES + (size_t)half * p.Npad * 128 + (size_t)p.W * 128))[w] =
          make_float4(0, 0, 0, 0);
    }
    tc::fence_proxy_async_smem();
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tbase = __shfl_sync(0xffffffffu, *tslot, 0);
  if (p.dbg && threadIdx.x == 0) p.dbg[1024 + blockIdx.x * 4 + 1] = gtimer();

  if ((p.dbg_flags & 256) && warp != 1 && !(p.dbg_flags & 512)) {
    // diagnostic mode: every other role idles (with bit 9 they run their loops)
  } else if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------------ TMA producer
      int sx = 0;
      uint32_t phx = 0;
      const uint64_t pol = tc::policy_evict_first();   // X is read exactly once
      int mblk = (int)(u0 / p.KT), kt = (int)(u0 % p.KT);   // 32-bit, advanced incrementally
      for (int64_t u = u0; u < u1; ++u, (++kt == (int)p.KT) ? (kt = 0, ++mblk) : 0) {
        const int nmt = (2 * mblk + 1 < p.mtiles) ? 2 : 1;   // the last M-block may hold one tile
        tc::mbar_wait(&xempty[sx], phx ^ 1);
        if (p.dbg && blockIdx.x == gridDim.x / 2 && u - u0 < 64) p.dbg[(u - u0) * 16 + 0] = clock64();
        uint8_t *A = xbuf + (size_t)sx * XSTAGE;
        if (p.dbg_flags & 2) {
          tc::mbar_arrive(&xfull[sx]);
        } else {
        tc::mbar_arrive_expect_tx(&xfull[sx], nmt * kABytes);
        if (PASS == 1) {
          // M-tile g = 2 mblk + mt covers rows l in [128 (g mod mt_per_t), +128) of slice t = g / mt_per_t
          for (int mt = 0; mt < nmt; ++mt) {
            const int g = 2 * mblk + mt, t = g / p.mt_per_t, lt = g - t * p.mt_per_t;
            tc::tma_load_3d_hint(A + mt * kABytes, &tmap, &xfull[sx], lt * kBM, (int)kt * kBK, t, pol);
          }
        } else {
          const int t = kt / p.nlb, lb = kt - t * p.nlb;
          for (int mt = 0; mt < nmt; ++mt)
            tc::tma_load_3d_hint(A + mt * kABytes, &tmap, &xfull[sx], lb * kBK, (2 * mblk + mt) * kBM, t, pol);
        }
        }
        if (++sx == SX) { sx = 0; phx ^= 1; }
      }
    }
  } else if (GR && (warp == 2 || warp == 3 || warp == 16 || warp == 17)) {
    // -------------------------------------------------------------- table generators (fused
    // subchain generation, Def. 3): lane j forms row l = 32 lb + j of the K-tile,
    // T_L(l, t) = F(l mod P, t) G_k(l / P) (R x R), for its warp's quarter (rows a, columns c) of
    // the product, splits each entry into tf32 hi / lo and writes both into the table ring in the
    // 128B-swizzled K-major layout the MMA reads (row n = a R + c, k-column j): the table never
    // exists in HBM.  The K-tile's prefix rows F are staged by the four warps themselves with
    // cp.async (two stages, the next unit's rows in flight while this unit is formed).
    if constexpr (GR > 0) {
      constexpr int R = GR, H = GR / 2, RR2 = GR * GR, CH = RR2 / 4;   // CH: 16-byte chunks per row
      const int gi = warp == 2 ? 0 : warp == 3 ? 1 : warp == 16 ? 2 : 3;
      const int a0 = (gi & 1) * H, c0 = (gi >> 1) * H;
      const int gt = gi * 32 + lane;
      const int Lr = (int)p.L;
      auto stage_rows = [&](int64_t uu, int st) {
        const int ktu = (int)(uu % p.KT);
        const int t = ktu / p.nlb, lb = ktu - t * p.nlb;
        const int j = gt >> 2, l = lb * 32 + j;   // four threads per row
        if (l < Lr) {
          float *dst = astage + st * 32 * RR2 + j * RR2;
          const float *src = p.GA + ((int64_t)(l % p.P) + (int64_t)p.P * t) * RR2;
          for (int w = gt & 3; w < CH; w += 4) cp_async16(dst + 4 * w, src + 4 * w);
        }
        cp_async_commit();
      };
      stage_rows(u0, 0);
      int sb = 0;
      uint32_t phb = 0;
      int kt = (int)(u0 % p.KT);
      const int kk = lane, chunk = kk >> 2, within = kk & 3;
      for (int64_t u = u0; u < u1; ++u, (++kt == (int)p.KT) ? (kt = 0) : 0) {
        const int sa = (int)((u - u0) & 1);
        const int lb = kt - (kt / p.nlb) * p.nlb;
        const int l = lb * 32 + lane;
        const bool valid = l < Lr;
        // this lane's G_k slice, columns [c0, c0 + H), as fp32 (at most two distinct slices per
        // tile: L1 broadcasts)
        float bv[R][H];
        {
          const double *gb = p.GB + (int64_t)(valid ? l / p.P : 0) * RR2;
#pragma unroll
          for (int c = 0; c < H; ++c)
#pragma unroll
            for (int b = 0; b < R; ++b) bv[b][c] = (float)__ldg(gb + b + R * (c0 + c));
        }
        gen_bar_sync();                                  // every generator is done with stage sa ^ 1
        if (u + 1 < u1) stage_rows(u + 1, sa ^ 1); else cp_async_commit();
        cp_async_wait_1();                               // this thread's rows of unit u have landed
        gen_bar_sync();                                  // ... and everyone's
        const float *arow = astage + sa * 32 * RR2 + lane * RR2;
        float acc[H][H];
#pragma unroll
        for (int a = 0; a < H; ++a) {
          float av[R];
#pragma unroll
          for (int b = 0; b < R; b += 2) {
            const float2 v2 = *(const float2 *)(arow + (a0 + a) * R + b);
            av[b] = v2.x;
            av[b + 1] = v2.y;
          }
#pragma unroll
          for (int c = 0; c < H; ++c) {
            float x = 0.0f;
#pragma unroll
            for (int b = 0; b < R; ++b) x = fmaf(av[b], bv[b][c], x);
            acc[a][c] = valid ? x : 0.0f;
          }
        }
        tc::mbar_wait(&bfree[sb], phb ^ 1);               // the MMAs two units back have read the slot
        float *B = (float *)(bbuf + (size_t)sb * BBYTES);
#pragma unroll
        for (int a = 0; a < H; ++a)
#pragma unroll
          for (int c = 0; c < H; ++c) {
            const float hi = tf32_rna_f(acc[a][c]);
            const float lo = tf32_rna_f(acc[a][c] - hi);
            const int n = (a0 + a) * R + c0 + c, n2 = p.Npad + n;
            B[n * 32 + ((chunk ^ (n & 7)) << 2) + within] = hi;
            B[n2 * 32 + ((chunk ^ (n2 & 7)) << 2) + within] = lo;
          }
        tc::fence_proxy_async_smem();   // generic-proxy stores -> the MMA's async-proxy reads
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&bfull[sb]);
        if (++sb == SB) { sb = 0; phb ^= 1; }
      }
      cp_async_wait_0();
    }
  } else if (warp == 3) {
    if (lane == 0) {
      // ------------------------------------------------------------ table-block producer (own
      // thread, so the table ring runs ahead independently of the X ring)
      int sb = 0;
      uint32_t phb = 0;
      int kt = (int)(u0 % p.KT);
      const uint64_t pol = tc::policy_evict_last();    // each table block is read by several CTAs
      for (int64_t u = u0; u < u1; ++u, (++kt == (int)p.KT) ? (kt = 0) : 0) {
        tc::mbar_wait(&bfree[sb], phb ^ 1);
        if (p.dbg && blockIdx.x == gridDim.x / 2 && u - u0 < 64) p.dbg[(u - u0) * 16 + 8] = clock64();
        uint8_t *B = bbuf + (size_t)sb * BBYTES;
        {   // only the W real rows of B_hi and B_lo travel; the padding rows stay zero in smem
          const int rb = p.W * 128;
          const uint8_t *src = (const uint8_t *)(p.Btiles + kt * (int64_t)(BBYTES / 4));
          if (p.dbg_flags & 1) {
            tc::mbar_arrive(&bfull[sb]);
          } else {
            tc::mbar_arrive_expect_tx(&bfull[sb], 2 * rb);
            tc::bulk_load_hint(B, src, rb, &bfull[sb], pol);
            tc::bulk_load_hint(B + p.Npad * 128, src + p.Npad * 128, rb, &bfull[sb], pol);
          }
        }
        if (++sb == SB) { sb = 0; phb ^= 1; }
      }
    }
  } else if (warp == 1) {
    {   // the whole warp walks the loop (warp-uniform operands); mma / commit elect one lane
      // ------------------------------------------------------------ UMMA issuer
      const uint32_t idesc = tc::idesc_tf32(kBM, p.Npad, 0, 0);
      if (p.dbg_flags & 256) {   // diagnostic: the bare MMA sequence, no waits (probe inside the kernel)
        const uint32_t b0 = tc::smem_u32(bbuf);
        long long t0 = clock64();
        for (int64_t u = u0; u < u1; ++u) {
          const int a = (int)(u & 1);
#pragma unroll
          for (int mt = 0; mt < kMT; ++mt) {
            const uint32_t d = tbase + (uint32_t)(mt * 128);
            const uint32_t ahi = tbase + kASlot0 + (uint32_t)((2 * a + mt) * 64);
#pragma unroll
            for (int ks = 0; ks < kBK / 8; ++ks) {
              const uint64_t bhi = tc::smem_desc_sw128(b0 + ks * 32, 16, 1024);
              const uint64_t blo = tc::smem_desc_sw128(b0 + p.Npad * 128 + ks * 32, 16, 1024);
              mma_tf32_ts(d, ahi + ks * 8, bhi, idesc, 1u);
              mma_tf32_ts(d, ahi + ks * 8, blo, idesc, 1u);
              mma_tf32_ts(d, ahi + 32 + ks * 8, bhi, idesc, 1u);
            }
          }
          mma_commit_elect(&bempty[(int)((u - u0) % SB)]);
          mma_commit_elect(&aempty[(int)((u - u0) & 1)]);
        }
        mma_commit_elect(accf);
        tc::mbar_wait(accf, 0);
        if (p.dbg && lane == 0 && blockIdx.x == gridDim.x / 2) p.dbg[63 * 16 + 0] = clock64() - t0;
      } else {
      // Every value that reaches an MMA operand is re-broadcast from lane 0 each unit (shfl), so the
      // compiler keeps the operands in uniform registers (no per-MMA R2UR after the barrier waits).
      // The A-slot and table-slot commits of unit u follow its MMAs at once; the accumulator commit
      // of a segment's last unit is deferred past the next unit's waits.
      int s = 0, a = 0;
      uint32_t pha = 0, phe = 0;
      int kt = (int)(u0 % p.KT), mblk = (int)(u0 / p.KT);
      bool pend_accf = false;
      const bool dbgcta = p.dbg != nullptr && blockIdx.x == gridDim.x / 2;
      const uint64_t bdesc0 = tc::smem_desc_sw128(tc::smem_u32(bbuf), 16, 1024);
      const uint32_t bstep = (uint32_t)(BBYTES >> 4), lostep = (uint32_t)((p.Npad * 128) >> 4);
      for (int64_t u = u0; u < u1; ++u, (++kt == (int)p.KT) ? (kt = 0, ++mblk) : 0) {   // s: table slot, a: TMEM A slot
        const int nmt = (2 * mblk + 1 < p.mtiles) ? 2 : 1;
        const bool first = (u == u0) || (kt == 0);
        const bool last = (u == u1 - 1) || (kt == (int)p.KT - 1);
        if (first && pend_accf) { mma_commit_elect(accf); pend_accf = false; }   // previous segment's accf first
        // (the table block of this unit has landed: the converters arrive on conv only after bfull)
        if (dbgcta && u - u0 < 64) p.dbg[(u - u0) * 16 + 4] = clock64();
        if (!(p.dbg_flags & 128)) tc::mbar_wait(&conv[a], pha);
        __syncwarp();
        if (dbgcta && u - u0 < 64) p.dbg[(u - u0) * 16 + 5] = clock64();
        if (pend_accf) { mma_commit_elect(accf); pend_accf = false; }
        tc::tc_fence_after();
        const int su = __shfl_sync(0xffffffffu, s, 0), au = __shfl_sync(0xffffffffu, a, 0);
        const int nmu = __shfl_sync(0xffffffffu, nmt, 0);
        const uint32_t acc0 = __shfl_sync(0xffffffffu, first ? 0u : 1u, 0);
        const uint64_t bd = bdesc0 + (uint64_t)(su * bstep);
        const bool firstu = __shfl_sync(0xffffffffu, first ? 1 : 0, 0) != 0;
#pragma unroll
        for (int mt = 0; mt < kMT; ++mt) {
          if (mt >= nmu) break;
          if (firstu) {   // the previous segment's accumulator of this tile has been drained
            tc::mbar_wait(&acce[mt], phe ^ 1);
            __syncwarp();
            tc::tc_fence_after();
          }
          const uint32_t d = tbase + (uint32_t)(mt * 128);
          const uint32_t ahi = tbase + kASlot0 + (uint32_t)((2 * au + mt) * 64);
#pragma unroll
          for (int ks = 0; ks < kBK / 8; ++ks) {
            const uint64_t bhi = bd + (uint64_t)(ks * 2), blo = bd + (uint64_t)(lostep + ks * 2);
            mma_tf32_ts(d, ahi + ks * 8, bhi, idesc, ks == 0 ? acc0 : 1u);
            mma_tf32_ts(d, ahi + ks * 8, blo, idesc, 1u);
            mma_tf32_ts(d, ahi + 32 + ks * 8, bhi, idesc, 1u);
          }
        }
        if (dbgcta && u - u0 < 64) p.dbg[(u - u0) * 16 + 6] = clock64();
        if (firstu) phe ^= 1;
        mma_commit_elect(&aempty[au]);    // the converters may refill this A slot as soon as possible
        mma_commit_elect(&bempty[su]);    // ... and the table producer this table slot
        pend_accf = last;
        if (dbgcta && u - u0 < 64) p.dbg[(u - u0) * 16 + 7] = clock64();
        if (++s == SB) s = 0;
        if (++a == 2) { a = 0; pha ^= 1; }
      }
      if (pend_accf) mma_commit_elect(accf);
      if (p.dbg && lane == 0) p.dbg[1024 + blockIdx.x * 4 + 2] = gtimer();
      }
    }
  } else if (warp >= 4 && warp < 12) {
    // -------------------------------------------------------------- 3xTF32 split converters
    // thread = row m of M-tile mt; reads its 32 k-values from the stage, writes hi / lo to TMEM.
    const int mt = (warp - 4) / 4, q = warp % 4;
    const int m = q * 32 + lane;
    int s = 0, a = 0, sb = 0;
    uint32_t ph = 0, pha = 0, phb = 0;
    int ckt = (int)(u0 % p.KT), cmb = (int)(u0 / p.KT);
    for (int64_t u = u0; u < u1; ++u, (++ckt == (int)p.KT) ? (ckt = 0, ++cmb) : 0) {   // s: X ring slot, a: TMEM A slot, sb: table ring slot
      const bool present = 2 * cmb + mt < p.mtiles;   // (an absent tile's MMAs are skipped)
      if (p.dbg_flags & 2048) tc::mbar_wait_sleep(&xfull[s], ph); else tc::mbar_wait(&xfull[s], ph);
      if (p.dbg && blockIdx.x == gridDim.x / 2 && u - u0 < 64 && threadIdx.x == 128) p.dbg[(u - u0) * 16 + 1] = clock64();
      if (p.dbg_flags & 2048) tc::mbar_wait_sleep(&aempty[a], pha ^ 1); else tc::mbar_wait(&aempty[a], pha ^ 1);
      if (p.dbg && blockIdx.x == gridDim.x / 2 && u - u0 < 64 && threadIdx.x == 128) p.dbg[(u - u0) * 16 + 2] = clock64();
      const uint8_t *xt = xbuf + (size_t)s * XSTAGE + mt * kABytes;
      uint32_t hi[32], lo[32];
      if ((p.dbg_flags & 32) || !present) {
#pragma unroll
        for (int k = 0; k < 32; ++k) { hi[k] = 0; lo[k] = 0; }
      } else if (PASS == 2) {
        // K-major [128 m][32 k]: row m at m*128, 16-byte chunk c at (c ^ (m % 8))
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const float4 x = *(const float4 *)(xt + m * 128 + ((c ^ (m & 7)) << 4));
          const float xv[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const uint32_t h = __float_as_uint(xv[e]) & 0xFFFFE000u;
            hi[4 * c + e] = h;
            lo[4 * c + e] = __float_as_uint(xv[e] - __uint_as_float(h));
          }
        }
      } else {
        // MN-major [32 k][128 m], unswizzled: (k, m) at (k * 128 + m) * 4
        const float *bx = (const float *)xt + m;
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          const float xv = bx[k * 128];
          const uint32_t h = __float_as_uint(xv) & 0xFFFFE000u;
          hi[k] = h;
          lo[k] = __float_as_uint(xv - __uint_as_float(h));
        }
      }
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&xempty[s]);   // the X slot is free once the tile sits in registers
      const uint32_t ta = tbase + ((uint32_t)(q * 32) << 16) + kASlot0 + (uint32_t)((2 * a + mt) * 64);
      if (!(p.dbg_flags & 4) && present) {
        tmem_st32(ta, hi);
        tmem_st32(ta + 32, lo);
        tmem_st_wait();
      }
      tc::tc_fence_before();
      if (p.dbg && blockIdx.x == gridDim.x / 2 && u - u0 < 64 && threadIdx.x == 128) p.dbg[(u - u0) * 16 + 3] = clock64();
      // conv[a] also certifies that this unit's table block has landed (the MMA waits only conv)
      if (lane == 0) tc::mbar_wait(&bfull[sb], phb);
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&conv[a]);
      if (++s == SX) { s = 0; ph ^= 1; }
      if (++a == 2) { a = 0; pha ^= 1; }
      if (++sb == SB) { sb = 0; phb ^= 1; }
    }
  } else if (warp >= 12 && warp < 16) {
    // -------------------------------------------------------------- epilogue
    // Lane quarter q of both accumulators.  yred: tile by tile, TMEM -> a dense [32][W] box in the
    // one-tile staging area -> release that tile's accumulator -> one TMA reduce-add (coalesced,
    // clipped at the tensor edges); the next tile reuses the area once the reduce has read it.  In
    // the CTA's last segment the second tile stages in the drained X ring instead (no wait).
    // Otherwise (W % 4 != 0) per-lane red.add from registers.
    const int q = warp % 4;
    const int row = q * 32 + lane;
    const int ybox = ystage_box_bytes(p.W);
    bool pending = false;   // a reduce may still be reading the staging area
    uint32_t phf = 0;
    int64_t u = u0;
    while (u < u1) {
      const int64_t mblk = u / p.KT;
      const int64_t uend = ((mblk + 1) * p.KT < u1) ? (mblk + 1) * p.KT : u1;
      const bool lastseg = uend == u1;
      if (p.dbg_flags & 1024) tc::mbar_wait_sleep(accf, phf); else tc::mbar_wait(accf, phf);
      phf ^= 1;
      tc::tc_fence_after();
#pragma unroll
      for (int mt = 0; mt < kMT; ++mt) {
        const int g = 2 * (int)mblk + mt;
        if (g >= p.mtiles) {
          if (lane == 0) tc::mbar_arrive(&acce[mt]);   // absent tile: keep the phases in step
          continue;
        }
        int t = 0, r0 = g * kBM;   // tile rows [r0, r0 + 128) of slice t
        if (PASS == 1) {
          t = g / p.mt_per_t;
          r0 = (g - t * p.mt_per_t) * kBM;
        }
        const uint32_t taddr = tbase + ((uint32_t)(q * 32) << 16) + (uint32_t)(mt * 128);
        if (p.yred) {
          uint8_t *box = (lastseg && mt == 1 ? xbuf : ystage) + q * ybox;
          if (pending && box != xbuf + q * ybox) {
            if (lane == 0) tc::bulk_wait_read<0>();
            __syncwarp();
          }
          float *dst = (float *)box + lane * ybox_w(p.W);
          for (int c0 = 0; c0 < p.W; c0 += 32) {
            float v[32];
            tmem_ld32(taddr + c0, v);   // columns >= Npad are never written by the MMA: not stored
#pragma unroll
            for (int i = 0; i < 32; i += 4)
              if (c0 + i < p.W) *(float4 *)(dst + c0 + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
          }
          tc::tc_fence_before();
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(&acce[mt]);   // the MMA may restart this tile now
          tc::fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tc::tma_reduce_add_3d(&ymap, box, 0, r0 + q * 32, t);
            tc::bulk_commit();
          }
          pending = true;
          continue;
        }
        const int64_t rr = r0 + row;
        const bool valid = rr < (PASS == 1 ? p.L : p.Rr);
        float *yr = p.Y + (rr + (PASS == 1 ? p.L * t : 0)) * p.W;
        for (int c0 = 0; c0 < p.Npad; c0 += 32) {
          float v[32];
          if (c0 + 32 <= p.Npad) {
            tmem_ld32(taddr + c0, v);
          } else {
            float w16[16];
            tc::tmem_ld16(taddr + c0, w16);
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] = w16[i];
#pragma unroll
            for (int i = 16; i < 32; ++i) v[i] = 0.0f;
          }
          if (c0 + 32 >= p.Npad) {   // last TMEM load of this tile: release the accumulator
            tc::tc_fence_before();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&acce[mt]);
          }
          if (valid) {
            if ((p.W & 3) == 0) {
#pragma unroll
              for (int i = 0; i < 32; i += 4)
                if (c0 + i < p.W) atomicAdd((float4 *)(yr + c0 + i), make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]));
            } else {
#pragma unroll
              for (int i = 0; i < 32; ++i)
                if (c0 + i < p.W) atomicAdd(yr + c0 + i, v[i]);
            }
          }
        }
      }
      u = uend;
    }
    // the CTA may leave once its reduce-adds have READ their staging (the async-proxy writes are
    // performed before the grid completes, which every consumer of Y waits for)
    if (p.yred && lane == 0) tc::bulk_wait_read<0>();
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (warp == 2) tc::tmem_dealloc(tbase, 512);
  if (p.dbg && threadIdx.x == 0) p.dbg[1024 + blockIdx.x * 4 + 3] = gtimer();
}

// Y = 0 before the stream-K reductions (a library kernel with the max-shared carve-out, so the SMs
// keep their configuration between the table kernel, this and the contraction).
__global__ void __launch_bounds__(256) k_zero_f32(float4 *__restrict__ y, int64_t n4) {
  for (int64_t i = blockIdx.x * 256 + threadIdx.x; i < n4; i += (int64_t)gridDim.x * 256)
    y[i] = make_float4(0.f, 0.f, 0.f, 0.f);
}

}  // namespace strb200

// =============================================================================================
// Host side.
using namespace strb200;

static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

// The instantiations: pass 1, pass 2 from the pre-tiled table, pass 2 with the table generated in
// the kernel (uniform rank 4 / 8 / 10).
static void *tf_kernel(int pass, int gr) {
  if (pass == 1) return (void *)k_contract_tf32<1, 0>;
  switch (gr) {
    case 4: return (void *)k_contract_tf32<2, 4>;
    case 8: return (void *)k_contract_tf32<2, 8>;
    case 10: return (void *)k_contract_tf32<2, 10>;
    default: return (void *)k_contract_tf32<2, 0>;
  }
}

static int64_t gen_period(const str_state *h) {   // Lf = (I_1/p) I_2 ... I_{k-1}
  int64_t P = 1;
  for (int i = 0; i < h->k - 1; ++i) P *= h->md[i].I;
  return P;
}

int tf32_gen_rank(const str_state *h) {
  if (!h->tf_gen_opt || h->contract != STR_CONTRACT_3XTF32 || h->k < 2) return 0;
  const int R = h->R[h->N - 1];
  if (!(R == 4 || R == 8 || R == 10) || h->R[h->k - 1] != R || h->R[h->k] != R) return 0;
  return gen_period(h) >= 32 ? R : 0;
}

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
  static std::once_flag enc_once;
  std::call_once(enc_once, [] {
    cudaDriverEntryPointQueryResult q;
    void *fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess && fn)
      g_encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  });
  if (!g_encode) return tf_fail(h, "cuTensorMapEncodeTiled unavailable");
  {   // opt-in (measured slower than the pre-tiled table): STR_TF_GEN=1 at str_init
    const char *e = getenv("STR_TF_GEN");
    h->tf_gen_opt = e && atoi(e) == 1;
  }
  static PerDeviceOnce attr_once;
  once_per_device(attr_once, [&] {
    for (int v = 0; v < 5; ++v) {
      const void *f = tf_kernel(v == 0 ? 1 : 2, v <= 1 ? 0 : (v == 2 ? 4 : v == 3 ? 8 : 10));
      cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
      cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    }
    prefer_max_smem(k_zero_f32);
    // (Npad <= 128 keeps 2 Npad x 128 B of table per stage; 3 stages fit)
  });
  h->tf32_ready = true;
  return STR_OK;
}

static int npad_of(int W) { return (W + 7) / 8 * 8; }   // UMMA N granularity 8 (cta_group::1, M = 128)

str_status tf32_ensure_workspace(str_state *h, int64_t tn) {
  const int N = h->N, k = h->k;
  const int W = h->R[k] * h->R[N - 1];   // R_{k+1} R_N
  const int Np = npad_of(W);
  const int64_t kt1 = cdiv(h->Rr, 32);
  const int64_t kt2 = tn * cdiv(h->L, 32);
  const size_t tiles1 = (size_t)kt1 * 2 * Np * 32 * sizeof(float), tiles2 = (size_t)kt2 * 2 * Np * 32 * sizeof(float);
  size_t yf = ((size_t)std::max<int64_t>(h->L * tn, h->Rr) * W * sizeof(float) + 15) / 16 * 16;
  auto grow = [&](DevBuf &b, size_t bytes) -> bool {
    if (b.bytes >= bytes) return true;
    if (b.p) {   // captured graphs may hold the old pointer
      h->reset_graphs();
      cudaFree(b.p);
    }
    b.p = nullptr;
    b.bytes = 0;
    if (cudaMalloc(&b.p, bytes) != cudaSuccess) return false;
    b.bytes = bytes;
    return true;
  };
  const int gr = tf32_gen_rank(h);
  const size_t f32 = gr ? (size_t)tn * gen_period(h) * gr * gr * sizeof(float) : 16;
  if (!grow(h->tab_split, tiles1) || !grow(h->tab_split2, gr ? 16 : tiles2) || !grow(h->tf_part, yf) ||
      !grow(h->tf_part2, yf) || !grow(h->F32, f32)) {
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
  // pass 1: one [32 k][128 m] box per M-tile, unswizzled (only the converters read it: lanes take
  // consecutive m, conflict-free); pass 2: one [128 m][32 k] box, 128B-swizzled (lanes take rows)
  cuuint32_t box[3] = {(cuuint32_t)(pass == 1 ? 128 : 32), (cuuint32_t)(pass == 1 ? 32 : 128), 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = g_encode(tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void *>(X), dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, pass == 1 ? CU_TENSOR_MAP_SWIZZLE_NONE : CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    h->err = "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")";
    return false;
  }
  return true;
}

// Output map for the TMA reduce-add epilogue: Y as [t][rows][W] fp32 (pass 1: rows l < L, t < tn;
// pass 2: rows r < Rr, one t), box [1][32][W], unswizzled (matches the dense staging boxes).
static bool encode_y_map(str_state *h, CUtensorMap *ymap, float *Y, int pass, int W, int64_t tn) {
  const int64_t rows = pass == 1 ? h->L : h->Rr, tt = pass == 1 ? tn : 1;
  cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)rows, (cuuint64_t)tt};
  cuuint64_t strides[2] = {(cuuint64_t)W * 4, (cuuint64_t)(rows * W * 4)};
  cuuint32_t box[3] = {(cuuint32_t)ybox_w(W), 32, 1};   // (columns >= W: out of bounds, clipped)
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = g_encode(ymap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, Y, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    h->err = "cuTensorMapEncodeTiled (Y) failed (" + std::to_string((int)r) + ")";
    return false;
  }
  return true;
}

str_status tf32_graph_update(str_state *h, int slot, int pass, const void *X, int64_t tn) {
  CUtensorMap tmap, ymap;
  if (!encode_x_map(h, &tmap, X, pass, tn)) return STR_E_CUDA;
  const str_state::GraphSlot &g = h->gs[slot];
  memcpy(&ymap, g.tf_ymap[pass - 1], sizeof(CUtensorMap));
  TcParams p;
  memcpy(&p, g.tf_params[pass - 1], sizeof(TcParams));
  void *args[3] = {&tmap, &ymap, &p};
  cudaKernelNodeParams kp = {};
  kp.func = tf_kernel(pass, g.tf_gen[pass - 1]);
  kp.gridDim = dim3(g.tf_grid[pass - 1]);
  kp.blockDim = dim3(g.tf_gen[pass - 1] ? kTcThreadsGen : kTcThreads);
  kp.sharedMemBytes = (unsigned)g.tf_smem[pass - 1];
  kp.kernelParams = args;
  kp.extra = nullptr;
  cudaError_t e = cudaGraphExecKernelNodeSetParams(h->gs[slot].exec, h->gs[slot].tf[pass - 1], &kp);
  if (e != cudaSuccess) {
    h->err = std::string("cudaGraphExecKernelNodeSetParams: ") + cudaGetErrorString(e);
    return STR_E_CUDA;
  }
  return STR_OK;
}

int launch_contract_tf32(str_state *h, const void *X, int pass, int W, int64_t tn, float *Y, bool y_zeroed) {
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
  const int bbytes = 2 * Np * 128;
  p.yred = (W % 4 == 0 && W <= 128) ? 1 : 0;   // TMA needs 16-byte row strides; box width <= 256
  const int ybytes = p.yred ? ystage_bytes(W) : 0;
  const int gr = pass == 2 ? tf32_gen_rank(h) : 0;
  const int gbytes = gr ? 2 * 32 * gr * gr * 4 : 0;   // the two prefix-row stages (fused generation)
  p.bstages = 2;
  if (const char *ev = getenv("STR_TF_BSTAGES")) p.bstages = std::max(2, atoi(ev));   // tuning knob
  p.stages = std::min(6, (int)((227 * 1024 - 1024 - 256 - ybytes - gbytes - p.bstages * bbytes) / (kMT * kABytes)));

  if (p.stages < 2) {
    h->err = "3xTF32 contraction: shared memory too small for the ring depths";
    return -1;
  }
  if (p.yred && p.stages * kMT * kABytes < ystage_bytes(W)) p.yred = 0;   // (last-segment tile 1 uses the X ring)
  p.mt_per_t = (int)cdiv(pass == 1 ? L : Rr, kBM);
  p.mtiles = pass == 1 ? p.mt_per_t * (int)tn : p.mt_per_t;
  p.nlb = (int)cdiv(L, 32);
  const int64_t blocks = cdiv(p.mtiles, kMT);   // M-blocks (tile pairs; pass 1 pairs across t)
  p.KT = pass == 1 ? cdiv(Rr, kBK) : tn * p.nlb;
  p.U = blocks * p.KT;
  // persistent grid: every SM but those the chain stream's kernels occupy while the pass runs (a pass
  // CTA waiting for such an SM would hold the whole pass back): beside pass 1 only the factor of Hq
  // runs (one CTA, or a two-CTA cluster for S_N > 64) (the step's other chain products are formed at the previous step's end); beside pass 2
  // the next mode's Gram-chain product and factor (kSideSMs)
  const int nsm = h->nsm;
  int maxg = std::max(1, nsm - (pass == 1 ? (h->SN > 64 ? 2 : 1) : kSideSMs));   // (S > 64: two-CTA factor)
  if (const char *ev = getenv("STR_TF_GRID")) maxg = std::max(1, std::min(nsm, atoi(ev)));   // tuning knob
  int grid = (int)std::min<int64_t>(maxg, p.U);
  p.upc = cdiv(p.U, grid);
  grid = (int)cdiv(p.U, p.upc);
  p.Btiles = (const float *)(pass == 1 ? h->tab_split.p : h->tab_split2.p);
  p.GA = gr ? (const float *)h->F32.p : nullptr;
  p.GB = gr ? (const double *)h->md[h->k - 1].G.p : nullptr;
  p.P = gr ? (int)gen_period(h) : 1;
  p.Y = Y;
  p.dbg = h->tf_dbg ? h->tf_dbg + (pass - 1) * str_state::kTfDbgWords : nullptr;
  p.dbg_flags = 0;
  if (g_dbg_skip & 4) p.U = 0;   // what-if diagnostic: every CTA exits at once
#ifdef STR_DIAG
  if (h->tf_dbg) {   // pipeline what-if flags (wrong results; tools/gpu_flags2.sh, diagnostic builds only)
    const char *ev = getenv("STR_TF_DBGFLAGS");
    if (ev) p.dbg_flags = atoi(ev);
  }
#endif
  CUtensorMap ymap;
  memset(&ymap, 0, sizeof(ymap));
  if (p.yred && !encode_y_map(h, &ymap, Y, pass, W, tn)) return -1;
  const int64_t M = pass == 1 ? L * tn : Rr;
  if (!y_zeroed) {
    const int64_t n = M * W;   // floats; the buffer is allocated in whole float4s
    const int64_t n4 = (n + 3) / 4;
    k_zero_f32<<<(unsigned)std::min<int64_t>(296, (n4 + 255) / 256), 256, 0, st>>>((float4 *)p.Y, n4);
    tl_mark(h, "zero_y");
  }
  const size_t smem = (size_t)p.stages * kMT * kABytes + (size_t)p.bstages * bbytes + ybytes + gbytes + 1024 + 256;
  prof_mark(h, 2 * (pass - 1));
  {
    void *args[3] = {&tmap, &ymap, &p};
    if (cudaLaunchKernel(tf_kernel(pass, gr), dim3(grid), dim3(gr ? kTcThreadsGen : kTcThreads), args, smem, st) !=
        cudaSuccess) {
      h->err = "contraction launch failed";
      return -1;
    }
  }
  if (h->capturing) {
    // remember the node so that graph replays can re-point it at new X (tf32_graph_update)
    cudaStreamCaptureStatus cs;
    const cudaGraphNode_t *deps = nullptr;
    size_t nd = 0;
    if (cudaStreamGetCaptureInfo(st, &cs, nullptr, nullptr, &deps, &nd) != cudaSuccess || nd != 1) {
      h->err = "cannot locate the captured contraction node";
      return -1;
    }
    str_state::GraphSlot &g = h->gs[h->cur_slot];
    g.tf[pass - 1] = deps[0];
    static_assert(sizeof(TcParams) <= sizeof(g.tf_params[0]), "TcParams too large");
    memcpy(g.tf_params[pass - 1], &p, sizeof(TcParams));
    memcpy(g.tf_ymap[pass - 1], &ymap, sizeof(CUtensorMap));
    g.tf_grid[pass - 1] = grid;
    g.tf_smem[pass - 1] = smem;
    g.tf_gen[pass - 1] = gr;
  }
  tl_mark(h, pass == 1 ? "contract_tf32_p1" : "contract_tf32_p2");
  prof_mark(h, 2 * (pass - 1) + 1);
  return 0;
}
