// comm.cu — the collectives of the mode-1-sharded STR step (sites C1, C2, C2' and the
// init / get_cores / fit reductions): NCCL between processes (one per GPU, the production path), or
// an in-process loopback group (the p ranks are p handles in one process on one GPU, driven by p host
// threads; used to test the library's sharded path on a single GPU).
//
// Loopback collective at a site: every rank records an event on its stream and registers its buffer;
// the last rank to arrive makes its stream wait for all the events, runs ONE plain kernel that reads
// every rank's buffer and writes the sum (fixed rank order) back into each, and records a done event
// that every rank's stream waits for.  Ranks meet on the host (mutex + condition variable); no kernel
// ever waits for another kernel (no spinning on the device).  Under a graph capture that spans the p
// ranks' streams (strdbg_loopback_step) the same calls become graph edges and one sum node.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <condition_variable>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include <nccl.h>

#include "common.cuh"
#include "str_internal.h"

namespace strb200 {

// ------------------------------------------------------------------------------------ NCCL (dlopen)
struct NcclApi {
  void *lib = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*allReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*allGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  const char *(*getErrorString)(ncclResult_t) = nullptr;
};
static NcclApi g_nccl;
static std::once_flag g_nccl_once;

static bool load_nccl(std::string &why) {
  std::call_once(g_nccl_once, [] {
    const char *names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char *nm : names) {
      g_nccl.lib = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
      if (g_nccl.lib) break;
    }
    if (!g_nccl.lib) return;
    g_nccl.commInitRank = (decltype(g_nccl.commInitRank))dlsym(g_nccl.lib, "ncclCommInitRank");
    g_nccl.allReduce = (decltype(g_nccl.allReduce))dlsym(g_nccl.lib, "ncclAllReduce");
    g_nccl.allGather = (decltype(g_nccl.allGather))dlsym(g_nccl.lib, "ncclAllGather");
    g_nccl.commDestroy = (decltype(g_nccl.commDestroy))dlsym(g_nccl.lib, "ncclCommDestroy");
    g_nccl.getErrorString = (decltype(g_nccl.getErrorString))dlsym(g_nccl.lib, "ncclGetErrorString");
  });
  if (!g_nccl.lib) {
    why = "cannot dlopen libnccl.so.2";
    return false;
  }
  if (!g_nccl.commInitRank || !g_nccl.allReduce || !g_nccl.allGather || !g_nccl.commDestroy) {
    why = "libnccl is missing symbols";
    return false;
  }
  return true;
}

struct NcclComm : Comm {
  ncclComm_t c = nullptr;
  std::string err(ncclResult_t r, const char *what) {
    return std::string(what) + ": " + (g_nccl.getErrorString ? g_nccl.getErrorString(r) : "error");
  }
  std::string allreduce(void *buf, size_t n, bool f32, cudaStream_t s) override {
    ncclResult_t r = g_nccl.allReduce(buf, buf, n, f32 ? ncclFloat32 : ncclFloat64, ncclSum, c, s);
    return r == ncclSuccess ? std::string() : err(r, "ncclAllReduce");
  }
  std::string allgather(const double *send, double *recv, size_t n, cudaStream_t s) override {
    ncclResult_t r = g_nccl.allGather(send, recv, n, ncclFloat64, c, s);
    return r == ncclSuccess ? std::string() : err(r, "ncclAllGather");
  }
  ~NcclComm() override {
    if (c && g_nccl.commDestroy) g_nccl.commDestroy(c);
  }
};

Comm *comm_nccl(int p, int rank, const void *nccl_id, std::string &why) {
  if (!nccl_id) {
    why = "nccl_id required";
    return nullptr;
  }
  if (!load_nccl(why)) return nullptr;
  ncclUniqueId id;
  memcpy(&id, nccl_id, sizeof(id));
  NcclComm *nc = new NcclComm();
  nc->p = p;
  nc->rank = rank;
  ncclResult_t r = g_nccl.commInitRank(&nc->c, p, id, rank);
  if (r != ncclSuccess) {
    why = nc->err(r, "ncclCommInitRank");
    nc->c = nullptr;
    delete nc;
    return nullptr;
  }
  return nc;
}

// ------------------------------------------------------------------------------------ loopback
constexpr int kLoopMax = 16;
struct LoopPtrs {
  void *b[kLoopMax];
};

// buf_q[i] = sum_{r < p} buf_r[i] for every q (fixed summation order: deterministic, equal on all ranks)
template <typename T>
__global__ void k_loop_sum(LoopPtrs ptrs, int p, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    T s = ((const T *)ptrs.b[0])[i];
    for (int r = 1; r < p; ++r) s += ((const T *)ptrs.b[r])[i];
    for (int r = 0; r < p; ++r) ((T *)ptrs.b[r])[i] = s;
  }
}

struct LoopbackGroup {
  int p = 1;
  std::mutex mu;
  std::condition_variable cv;
  std::vector<int64_t> seq;                 // per rank: index of its next collective site
  struct Site {
    int kind = 0, count = 0, left = 0;      // kind 1: sum-allreduce, 2: allgather (fp64)
    size_t n = 0;
    bool f32 = false, ready = false;
    void *a[kLoopMax] = {}, *b[kLoopMax] = {};
    cudaEvent_t ev[kLoopMax] = {};
    cudaEvent_t done = nullptr;
  };
  std::map<int64_t, Site> sites;
  std::vector<str_state *> members;         // handle of each rank (str_get_cores of the sharded core)
  // the graph of one step of all ranks (strdbg_loopback_step)
  cudaGraphExec_t exec = nullptr;
  int64_t exec_tn = 0;
  std::vector<const void *> exec_x;

  std::string site(int r, int kind, void *a, void *b, size_t n, bool f32, cudaStream_t s) {
    std::unique_lock<std::mutex> lk(mu);
    const int64_t id = seq[r]++;
    Site &st = sites[id];
    if (st.count == 0) {
      st.kind = kind;
      st.n = n;
      st.f32 = f32;
    } else if (st.kind != kind || st.n != n || st.f32 != f32) {
      return "loopback: ranks disagree at a collective site";
    }
    if (cudaEventCreateWithFlags(&st.ev[r], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventRecord(st.ev[r], s) != cudaSuccess)
      return "loopback: event record failed";
    st.a[r] = a;
    st.b[r] = b;
    const bool last = ++st.count == p;
    if (last) {
      for (int q = 0; q < p; ++q)
        if (q != r) cudaStreamWaitEvent(s, st.ev[q], 0);
      if (kind == 1) {
        LoopPtrs ptrs;
        for (int q = 0; q < p; ++q) ptrs.b[q] = st.a[q];
        const unsigned grid = (unsigned)std::min<int64_t>(592, std::max<int64_t>(1, cdiv((int64_t)n, 256)));
        if (f32) k_loop_sum<float><<<grid, 256, 0, s>>>(ptrs, p, (int64_t)n);
        else k_loop_sum<double><<<grid, 256, 0, s>>>(ptrs, p, (int64_t)n);
      } else {
        for (int d = 0; d < p; ++d)
          for (int q = 0; q < p; ++q)
            cudaMemcpyAsync((double *)st.b[d] + (size_t)q * n, st.a[q], n * sizeof(double), cudaMemcpyDeviceToDevice, s);
      }
      cudaEventCreateWithFlags(&st.done, cudaEventDisableTiming);
      if (cudaEventRecord(st.done, s) != cudaSuccess || cudaGetLastError() != cudaSuccess)
        return "loopback: collective enqueue failed";
      st.ready = true;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return st.ready; });
      cudaStreamWaitEvent(s, st.done, 0);
    }
    if (++st.left == p) {
      for (int q = 0; q < p; ++q) cudaEventDestroy(st.ev[q]);
      cudaEventDestroy(st.done);
      sites.erase(id);
    }
    return std::string();
  }
};

struct LoopbackComm : Comm {
  LoopbackGroup *g = nullptr;
  std::string allreduce(void *buf, size_t n, bool f32, cudaStream_t s) override {
    return g->site(rank, 1, buf, nullptr, n, f32, s);
  }
  std::string allgather(const double *send, double *recv, size_t n, cudaStream_t s) override {
    return g->site(rank, 2, const_cast<double *>(send), recv, n, false, s);
  }
  bool loopback() const override { return true; }
  ~LoopbackComm() override {
    std::lock_guard<std::mutex> lk(g->mu);
    if (rank < (int)g->members.size()) g->members[rank] = nullptr;
  }
};

Comm *comm_loopback(void *group, int p, int rank, str_state *h, std::string &why) {
  LoopbackGroup *g = (LoopbackGroup *)group;
  if (!g || g->p != p || rank < 0 || rank >= p) {
    why = "loopback group missing or of another size";
    return nullptr;
  }
  LoopbackComm *c = new LoopbackComm();
  c->g = g;
  c->p = p;
  c->rank = rank;
  std::lock_guard<std::mutex> lk(g->mu);
  g->members[rank] = h;
  return c;
}

str_state *loopback_member(void *group, int rank) {
  LoopbackGroup *g = (LoopbackGroup *)group;
  std::lock_guard<std::mutex> lk(g->mu);
  return rank < (int)g->members.size() ? g->members[rank] : nullptr;
}

LoopbackGroup *loopback_group_of(Comm *c) {
  return (c && c->loopback()) ? static_cast<LoopbackComm *>(c)->g : nullptr;
}

cudaGraphExec_t &loopback_exec(LoopbackGroup *g, int64_t **tn, std::vector<const void *> **xs) {
  *tn = &g->exec_tn;
  *xs = &g->exec_x;
  return g->exec;
}

}  // namespace strb200

using namespace strb200;

extern "C" STR_API str_status str_loopback_create(int32_t world_size, void **group) {
  if (!group || world_size < 1 || world_size > kLoopMax) return STR_E_ARG;
  LoopbackGroup *g = new LoopbackGroup();
  g->p = world_size;
  g->seq.assign(world_size, 0);
  g->members.assign(world_size, nullptr);
  *group = g;
  return STR_OK;
}

extern "C" STR_API void str_loopback_destroy(void *group) {
  LoopbackGroup *g = (LoopbackGroup *)group;
  if (!g) return;
  if (g->exec) cudaGraphExecDestroy(g->exec);
  delete g;
}
