// str_internal.h — the opaque str_state and cross-file internal entry points.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "str.h"

// Collective backend of the mode-1-sharded step (comm.cu): NCCL across processes or an in-process
// loopback group.  Every call enqueues on stream s; the return value is "" or an error message.
struct Comm {
  int p = 1, rank = 0;
  virtual ~Comm() = default;
  virtual std::string allreduce(void *buf, size_t n, bool f32, cudaStream_t s) = 0;          // sum, in place
  virtual std::string allgather(const double *send, double *recv, size_t n, cudaStream_t s) = 0;  // rank-major
  virtual bool loopback() const { return false; }
};
struct str_state;
namespace strb200 {
Comm *comm_nccl(int p, int rank, const void *nccl_id, std::string &why);
Comm *comm_loopback(void *group, int p, int rank, str_state *h, std::string &why);
str_state *loopback_member(void *group, int rank);
struct LoopbackGroup;
LoopbackGroup *loopback_group_of(Comm *c);
cudaGraphExec_t &loopback_exec(LoopbackGroup *g, int64_t **tn, std::vector<const void *> **xs);
}  // namespace strb200

struct DevBuf {
  void *p = nullptr;
  size_t bytes = 0;
};

struct ModeBuf {
  int64_t I = 0;        // local rows (mode 1 is sharded across ranks)
  int64_t I_glob = 0;
  int Ra = 0, Rb = 0;   // R_n, R_{n+1}
  DevBuf G;             // I x Ra*Rb, G_n(2) rows (column r_n + R_n r_{n+1})
  DevBuf P;             // I x Ra*Rb (Eq. partial)
  DevBuf Q;             // (Ra*Rb)^2 (Eq. partial)
  DevBuf Zm;            // Gram tensor Z_n as chain matrix: Rb^2 x Ra^2
  DevBuf Qi;            // V^T of Q_n (Q_n^{-1} = VT VT^T; launch_spd_factor)
  // rSTR
  DevBuf samp;          // sampled slices (G_n)_S: m x Ra*Rb (G(2) layout rows)
  std::vector<int32_t> idx_host;
};

struct str_state {
  // configuration
  int N = 0;
  std::vector<int64_t> dims_g;
  std::vector<int> R;               // R_1..R_N
  str_dtype dtype = STR_F32;
  str_contract contract = STR_CONTRACT_F64;
  str_variant variant = STR_DET;
  int64_t m = 0;
  uint64_t seed = 0;
  int k = 1;                        // two-pass split
  int p = 1, rank = 0, device = 0;
  int nsm = 148;                    // SMs of the device
  int xbytes = 4;
  int64_t i1_off = 0;
  cudaStream_t st = nullptr;
  bool own_stream = false;
  cudaStream_t st2 = nullptr, st_main = nullptr;   // side stream for the independent branches
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaStream_t st3 = nullptr;                      // third branch: the contraction passes' tables
  cudaEvent_t ev_fork3 = nullptr, ev_join3 = nullptr;
  cudaEvent_t ev_z = nullptr;       // STR step: the chain stream's Z_j (and G_j) handed to the data stream
  cudaEvent_t ev_hq = nullptr;      // STR step: the next step's Hq formed (chain stream, step end)
  bool side_ready = false;                         // Sf_n and Hq hold the chains of the current Z's
  bool tr_ready = false;                           // pass-1 table built for the current cores, output cleared
  Comm *comm = nullptr;             // collectives when p > 1 (comm.cu)
  void *loop_group = nullptr;       // loopback group (in-process ranks), if any

  // geometry (local)
  int64_t L = 1, Rr = 1;            // prod of left dims (modes 1..k), right dims (k+1..N-1)
  int SN = 0;                       // R_N R_1

  // state
  std::vector<ModeBuf> md;          // modes 1..N-1
  DevBuf GN;                        // temporal rows: Tcap x SN (G_N(2) rows)
  int64_t T = 0, Tcap = 0;
  DevBuf ZmN;                       // Z_N^new (update) / Z_N (init): R_1^2 x R_N^2
  std::vector<DevBuf> Sf;           // suffix chains Sf_n (index n)
  std::vector<DevBuf> Rc;           // R_n = Z_{N-2} ... Z_{n+1} (index n <= N-4; R_{N-3} is Z_{N-2})
  DevBuf Lp[2], T1, H, Hq, Hi;       // Hq = H^{≠N}_<2> (temporal normal matrix), Hi = its factor V^T

  // workspaces
  int64_t ws_t = 0;
  DevBuf TR, TL, YL, YR, Wt, tmpA, tmpB, Mt, ws, Xstage;
  DevBuf info_buf;
  int *d_info = nullptr;

  // 3xTF32 path
  bool tf32_ready = false;
  DevBuf tab_split, tab_split2;     // hi/lo fp32 tables of the tensor-core passes 1 and 2
  DevBuf tf_part, tf_part2;         // pass-1 / pass-2 fp32 outputs (stream-K red.add targets)
  // pass 2 with in-kernel table generation (tf32_gen_rank > 0): the fp32 prefix rows
  // F[(f, t)] = G_N(t) G_1(i_1) ... G_{k-1}(i_{k-1}); the contraction forms T_L = F G_k per K-tile
  DevBuf F32;
  bool tf_gen_opt = false;          // STR_TF_GEN=1 at str_init: pass 2 generates its table in the kernel

  // CUDA-graph replay of the STR step: the step is captured once per t_new and
  // replayed; X enters through the device slot dX (f64 path) or by re-pointing the two tensor-core
  // contraction nodes (3xTF32 path).  New temporal rows go to the fixed scratch GNnew and are
  // appended at the device-side row counter dT.
  DevBuf GNnew, dT, dX;
  bool use_graph = true;
  bool use_graph_forced_off = false;   // loopback ranks: the group owns the step graph
  struct GraphSlot {
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    int64_t tn = 0, launches = 0;
    cudaGraphNode_t setx = nullptr, tf[2] = {nullptr, nullptr};
    // launch parameters of the captured contraction nodes (per pass), re-used when a replay is
    // re-pointed at new X (tf32_graph_update)
    alignas(16) unsigned char tf_params[2][256];
    alignas(64) unsigned char tf_ymap[2][128];   // CUtensorMap of the pass outputs (TMA reduce epilogue)
    int tf_grid[2] = {0, 0};
    size_t tf_smem[2] = {0, 0};
    int tf_gen[2] = {0, 0};   // rank of the in-kernel table generation (0: pre-tiled table)
    void reset() {
      if (exec) cudaGraphExecDestroy(exec);
      if (graph) cudaGraphDestroy(graph);
      exec = nullptr;
      graph = nullptr;
      tn = 0;
    }
  };
  GraphSlot gs[2];                  // [0] production replay, [1] profiling replay (events around the passes)
  int cur_slot = 0;                 // slot being captured / replayed
  bool chain_prio = false;          // STR_CHAIN_PRIO=1: chain stream at the highest priority (A/B knob)
  cudaEvent_t pev[4] = {};          // profiling: pass-1 begin/end, pass-2 begin/end
  double prof_ms[2] = {0.0, 0.0};
  int64_t prof_n[2] = {0, 0};
  bool capturing = false;
  // every captured graph holds raw device pointers: any (re)allocation of a buffer invalidates both
  void reset_graphs() {
    gs[0].reset();
    gs[1].reset();
  }
  long long *tf_dbg = nullptr;      // device buffer for the contraction pipeline trace (diagnostic)
  static constexpr int kTfDbgWords = 1024 + 4 * 160;   // per pass

  // rSTR
  DevBuf sidx, sX, sG, sGram, sTmp, sIdxDev, sSk, sSk2;   // sSk2: split-K workspace of the side branch
  int32_t *idx_pinned = nullptr;    // pinned index staging, one m-slot per mode
  cudaEvent_t idx_ev[17] = {};       // last upload from each slot
  std::vector<int32_t> forced_idx[16];
  std::vector<int32_t> last_idx[16];
  int64_t tau = 0;
  DevBuf dTau;                      // device copy of tau (advanced by the step itself)
  bool rstr_dev = true;             // draws on the device (STR_RSTR_HOST_DRAWS=1: host sampler)
  bool idx_dev[17] = {};            // index table k was drawn on the device (copy back on request)
  // rSTR-K (KSRFT): mixed batch X^ (complex, fp32 pairs or fp64 pairs per `contract`), the step's
  // sign flips D_1..D_N (mode j at ks_off[j-1]; D_N has t_new entries)
  DevBuf ksXh, ksSign, ksCore;
  int64_t ks_off[17] = {};
  bool ksrft() const { return variant == STR_SAMPLE_KSRFT; }

  // bookkeeping
  int64_t launches = 0;
  int64_t collectives = 0;
  bool profiling = false;
  // launch timeline (diagnostic): an event after every launch, named by kernel
  bool timeline = false;
  std::vector<std::pair<const char *, cudaEvent_t>> tl;
  std::string err;
  bool poisoned = false;

  void free_all() {
    auto fr = [](DevBuf &b) {
      if (b.p) cudaFree(b.p);
      b.p = nullptr;
      b.bytes = 0;
    };
    for (auto &m : md) {
      fr(m.G); fr(m.P); fr(m.Q); fr(m.Zm); fr(m.Qi); fr(m.samp);
    }
    fr(GN); fr(ZmN);
    for (auto &b : Sf) fr(b);
    fr(Lp[0]); fr(Lp[1]); fr(T1); fr(H); fr(Hq); fr(Hi);
    fr(TR); fr(TL); fr(YL); fr(YR); fr(Wt); fr(tmpA); fr(tmpB); fr(Mt); fr(ws); fr(Xstage); fr(info_buf);
    fr(tab_split); fr(tab_split2); fr(tf_part); fr(tf_part2); fr(F32);
    fr(GNnew); fr(dT); fr(dX);
    gs[0].reset();
    gs[1].reset();
    for (auto &e : pev)
      if (e) { cudaEventDestroy(e); e = nullptr; }
    fr(sidx); fr(sX); fr(sG); fr(sGram); fr(sTmp); fr(sIdxDev); fr(sSk); fr(sSk2); fr(dTau); fr(ksXh); fr(ksSign); fr(ksCore);
    if (idx_pinned) cudaFreeHost(idx_pinned);
    idx_pinned = nullptr;
    for (auto &e : idx_ev)
      if (e) { cudaEventDestroy(e); e = nullptr; }
  }
};

// Profiling event i (pass-1 begin/end, pass-2 begin/end) on the library stream; inside a stream
// capture it must be an external record node (a plain record there is only a capture dependency).
inline void prof_mark(str_state *h, int i) {
  if (!h->profiling) return;
  cudaEventRecordWithFlags(h->pev[i], h->st, h->capturing ? cudaEventRecordExternal : cudaEventRecordDefault);
}

// Count a launch (n kernels) and, when the timeline is on, record a named event after it on the
// handle's stream: consecutive events bracket each launch's in-stream time (incl. its gap).
inline void tl_mark(str_state *h, const char *name, int n = 1) {
  h->launches += n;
  if (h->timeline) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, h->st);
    h->tl.push_back({name, e});
  }
}

// str_api.cu
str_status ensure_temporal_capacity(str_state *h, int64_t need);

// rstr.cu
str_status rstr_init(str_state *h, const void *X, int64_t tn);
str_status rstr_update(str_state *h, const void *X, int64_t tn);

// contract_tf32.cu
str_status tf32_prepare(str_state *h);
str_status tf32_ensure_workspace(str_state *h, int64_t tn);
// Tensor-core pass over X with the pre-tiled table operand already in h->tab_split; fp32 output Y
// (zeroed here unless y_zeroed, then accumulated).  Returns 0, or -1 with h->err set.
int launch_contract_tf32(str_state *h, const void *X, int pass, int W, int64_t tn, float *Y, bool y_zeroed);
int tf32_npad(int W);
// Pass 2 forms its table in the contraction kernel (the fused subchain generation) when this returns
// the uniform rank R (> 0): R_N = R_k = R_{k+1} = R in {4, 8, 10}, k >= 2, and the prefix period
// Lf = (I_1/p) I_2 ... I_{k-1} >= 32 (a K-tile of 32 rows then spans at most two G_k slices);
// 0 otherwise (the pre-tiled table path).  Opt-in per handle (STR_TF_GEN=1 at str_init): measured
// slower than the pre-tiled table at C5.
int tf32_gen_rank(const str_state *h);
// Re-point captured contraction node `pass` of exec at new data X (3xTF32 path).
str_status tf32_graph_update(str_state *h, int slot, int pass, const void *X, int64_t tn);
