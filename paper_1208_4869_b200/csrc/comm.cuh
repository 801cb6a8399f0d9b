// comm.cuh — the collectives of the row-sharded multi-GPU path.
//
//   allgather_inplace  C1: gather the row slices of a GEMV input vector
//   allgather          C3: gather every rank's K partial sums (scalar phase)
//   reduce_scatter     C2: sum the per-rank full-length Aᴴ·x partials
//   halo               C4: exchange the z-slab halo planes of a CSR operator
//
// Two implementations behind one interface:
//   NcclComm      — NCCL 2.28 over NVLink/NVSwitch (one process per GPU),
//                   dlopen'ed on demand so single-GPU use needs no NCCL.
//   LoopbackComm  — `world` handles in ONE process on ONE device, each driven
//                   by its own host thread; every collective is a host-side
//                   barrier + device-to-device copies.  No kernel ever waits
//                   on another rank's kernel (all waiting is on the host), so
//                   the whole sharded code path can be validated on a single
//                   GPU (tests/test_gpu_multirank.py).
#pragma once
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <stdint.h>
#include <stdlib.h>

#include <condition_variable>
#include <mutex>
#include <string>
#include <vector>

#include "nccl.h"

namespace ccg {

struct NcclApi {
  bool loaded = false;
  std::string err;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*ReduceScatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                                cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  // symmetric memory (NCCL ≥ 2.27; optional: only the P2P mirror mode needs them)
  ncclResult_t (*MemAlloc)(void**, size_t) = nullptr;
  ncclResult_t (*MemFree)(void*) = nullptr;
  ncclResult_t (*WindowRegister)(ncclComm_t, void*, size_t, ncclWindow_t*, int) = nullptr;
  ncclResult_t (*WindowDeregister)(ncclComm_t, ncclWindow_t) = nullptr;
};
inline NcclApi g_nccl;

inline bool nccl_load() {
  if (g_nccl.loaded) return true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    const char* p = getenv("CCG_NCCL_LIB");
    if (p) h = dlopen(p, RTLD_NOW | RTLD_GLOBAL);
  }
  if (!h) { g_nccl.err = "cannot dlopen libnccl.so.2 (set CCG_NCCL_LIB)"; return false; }
#define CCG_LOADSYM(field, name)                                          \
  g_nccl.field = reinterpret_cast<decltype(g_nccl.field)>(dlsym(h, name)); \
  if (!g_nccl.field) { g_nccl.err = std::string("missing NCCL symbol ") + name; return false; }
  CCG_LOADSYM(GetUniqueId, "ncclGetUniqueId");
  CCG_LOADSYM(CommInitRank, "ncclCommInitRank");
  CCG_LOADSYM(CommDestroy, "ncclCommDestroy");
  CCG_LOADSYM(AllGather, "ncclAllGather");
  CCG_LOADSYM(ReduceScatter, "ncclReduceScatter");
  CCG_LOADSYM(Send, "ncclSend");
  CCG_LOADSYM(Recv, "ncclRecv");
  CCG_LOADSYM(GroupStart, "ncclGroupStart");
  CCG_LOADSYM(GroupEnd, "ncclGroupEnd");
  CCG_LOADSYM(GetErrorString, "ncclGetErrorString");
#undef CCG_LOADSYM
  g_nccl.MemAlloc = reinterpret_cast<decltype(g_nccl.MemAlloc)>(dlsym(h, "ncclMemAlloc"));
  g_nccl.MemFree = reinterpret_cast<decltype(g_nccl.MemFree)>(dlsym(h, "ncclMemFree"));
  g_nccl.WindowRegister = reinterpret_cast<decltype(g_nccl.WindowRegister)>(dlsym(h, "ncclCommWindowRegister"));
  g_nccl.WindowDeregister =
      reinterpret_cast<decltype(g_nccl.WindowDeregister)>(dlsym(h, "ncclCommWindowDeregister"));
  g_nccl.loaded = true;
  return true;
}

// element type of a collective buffer
enum CommType { CT_F32 = 0, CT_F64 = 1, CT_I64 = 2 };
inline size_t ct_size(CommType t) { return t == CT_F32 ? 4 : 8; }

struct Comm {
  int world = 1, rank = 0;
  std::string err;
  bool graph_safe = true;  // may be captured in a CUDA graph
  int kind = 0;            // 1 = NCCL, 2 = loopback (ccg_get_stat CCG_STAT_COMM_KIND)
  int64_t calls = 0;       // collective calls issued (host side; a captured call counts once)
  virtual ~Comm() {}
  // buf holds world chunks of `count` elements; chunk `rank` is filled
  virtual int allgather_inplace(void* buf, size_t count, CommType t, cudaStream_t s) = 0;
  virtual int allgather(const void* send, void* recv, size_t count, CommType t, cudaStream_t s) = 0;
  // recv[count] = Σ_ranks send[rank·count : (rank+1)·count]
  virtual int reduce_scatter(const void* send, void* recv, size_t count, CommType t, cudaStream_t s) = 0;
  // full-length buffer in global indexing; rank owns [row0, row0+nloc): send the
  // first / last h elements to rank-1 / rank+1, which store them at the SAME
  // global positions (their halo), and receive theirs.
  virtual int halo(void* buf, int64_t row0, int64_t nloc, int64_t h, size_t esz, CommType t,
                   cudaStream_t s) = 0;
  // P2P mirror exchange (p2p.cuh): a point where every rank's preceding work
  // is complete.  NCCL: nothing (the device flags order it); loopback: a host
  // barrier, so that no kernel ever waits on another rank's kernel.
  virtual int sync_point(cudaStream_t) { return 0; }
};

// ---------------------------------------------------------------------------
struct NcclComm : Comm {
  ncclComm_t comm = nullptr;
  static ncclDataType_t nt(CommType t) { return t == CT_F32 ? ncclFloat32 : t == CT_F64 ? ncclFloat64 : ncclInt64; }
  int fail(ncclResult_t r, const char* what) {
    err = std::string(what) + ": " + g_nccl.GetErrorString(r);
    return -6;
  }
  int init(int w, int r, const uint8_t* id) {
    world = w; rank = r;
    kind = 1;
    if (!nccl_load()) { err = g_nccl.err; return -6; }
    ncclUniqueId u;
    memcpy(u.internal, id, 128);
    ncclResult_t e = g_nccl.CommInitRank(&comm, w, u, r);
    return e == ncclSuccess ? 0 : fail(e, "ncclCommInitRank");
  }
  ~NcclComm() override {
    if (comm && g_nccl.loaded) g_nccl.CommDestroy(comm);
  }
  // symmetric-memory window of `bytes` (collective over the ranks)
  int window_alloc(size_t bytes, void** ptr, ncclWindow_t* win) {
    if (!g_nccl.MemAlloc || !g_nccl.WindowRegister) { err = "NCCL has no symmetric-memory windows"; return -3; }
    ncclResult_t e = g_nccl.MemAlloc(ptr, bytes);
    if (e != ncclSuccess) return fail(e, "ncclMemAlloc");
    e = g_nccl.WindowRegister(comm, *ptr, bytes, win, NCCL_WIN_COLL_SYMMETRIC);
    if (e != ncclSuccess) { g_nccl.MemFree(*ptr); *ptr = nullptr; return fail(e, "ncclCommWindowRegister"); }
    return 0;
  }
  void window_free(void* ptr, ncclWindow_t win) {
    if (win && g_nccl.WindowDeregister) g_nccl.WindowDeregister(comm, win);
    if (ptr && g_nccl.MemFree) g_nccl.MemFree(ptr);
  }
  int allgather_inplace(void* buf, size_t count, CommType t, cudaStream_t s) override {
    ++calls;
    char* b = static_cast<char*>(buf);
    ncclResult_t e = g_nccl.AllGather(b + rank * count * ct_size(t), b, count, nt(t), comm, s);
    return e == ncclSuccess ? 0 : fail(e, "ncclAllGather");
  }
  int allgather(const void* send, void* recv, size_t count, CommType t, cudaStream_t s) override {
    ++calls;
    ncclResult_t e = g_nccl.AllGather(send, recv, count, nt(t), comm, s);
    return e == ncclSuccess ? 0 : fail(e, "ncclAllGather");
  }
  int reduce_scatter(const void* send, void* recv, size_t count, CommType t, cudaStream_t s) override {
    ++calls;
    ncclResult_t e = g_nccl.ReduceScatter(send, recv, count, nt(t), ncclSum, comm, s);
    return e == ncclSuccess ? 0 : fail(e, "ncclReduceScatter");
  }
  int halo(void* buf, int64_t row0, int64_t nloc, int64_t h, size_t esz, CommType t, cudaStream_t s) override {
    ++calls;
    if (h == 0) return 0;
    char* b = static_cast<char*>(buf);
    const size_t cnt = (size_t)h * esz / ct_size(t);
    ncclResult_t e = g_nccl.GroupStart();
    if (e != ncclSuccess) return fail(e, "ncclGroupStart");
    if (rank > 0) {
      if ((e = g_nccl.Send(b + row0 * esz, cnt, nt(t), rank - 1, comm, s)) != ncclSuccess) return fail(e, "ncclSend");
      if ((e = g_nccl.Recv(b + (row0 - h) * esz, cnt, nt(t), rank - 1, comm, s)) != ncclSuccess)
        return fail(e, "ncclRecv");
    }
    if (rank < world - 1) {
      if ((e = g_nccl.Send(b + (row0 + nloc - h) * esz, cnt, nt(t), rank + 1, comm, s)) != ncclSuccess)
        return fail(e, "ncclSend");
      if ((e = g_nccl.Recv(b + (row0 + nloc) * esz, cnt, nt(t), rank + 1, comm, s)) != ncclSuccess)
        return fail(e, "ncclRecv");
    }
    e = g_nccl.GroupEnd();
    return e == ncclSuccess ? 0 : fail(e, "ncclGroupEnd");
  }
};

// ---------------------------------------------------------------------------
// in-process loopback (validation of the sharded path on one GPU)
// ---------------------------------------------------------------------------
template <typename V>
__global__ void loopback_rs_sum(const V* const* src, int world, size_t off, size_t count, V* out) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
    V s = 0;
    for (int p = 0; p < world; ++p) s += src[p][off + i];  // rank order
    out[i] = s;
  }
}

struct LoopbackGroup {
  int world;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  long gen = 0;
  std::vector<const void*> ptr;
  const void** dptr = nullptr;  // device copy of ptr (per rank slot)
  int refs = 0;
  explicit LoopbackGroup(int w) : world(w), ptr(w, nullptr) {}
  void barrier() {
    std::unique_lock<std::mutex> lk(m);
    long g = gen;
    if (++arrived == world) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

struct LoopbackComm : Comm {
  LoopbackGroup* g = nullptr;
  const void** dptrs = nullptr;  // this rank's device array of peer pointers
  LoopbackComm(LoopbackGroup* grp, int r) : g(grp) {
    world = grp->world;
    rank = r;
    graph_safe = false;
    kind = 2;
  }
  ~LoopbackComm() override {
    if (dptrs) cudaFree(dptrs);
    bool last = false;
    {
      std::lock_guard<std::mutex> lk(g->m);
      last = (--g->refs == 0);
    }
    if (last) delete g;
  }
  int cu(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return 0;
    err = std::string(what) + ": " + cudaGetErrorString(e);
    return -5;
  }
  int publish(const void* p, cudaStream_t s) {
    int rc = cu(cudaStreamSynchronize(s), "loopback sync");
    g->ptr[rank] = p;
    g->barrier();
    return rc;
  }
  int done(cudaStream_t s) {
    int rc = cu(cudaStreamSynchronize(s), "loopback sync");
    g->barrier();
    return rc;
  }
  int allgather_inplace(void* buf, size_t count, CommType t, cudaStream_t s) override {
    ++calls;
    const size_t bytes = count * ct_size(t);
    int rc = publish(buf, s);
    for (int p = 0; p < world && !rc; ++p)
      if (p != rank)
        rc = cu(cudaMemcpyAsync(static_cast<char*>(buf) + p * bytes, static_cast<const char*>(g->ptr[p]) + p * bytes,
                                bytes, cudaMemcpyDeviceToDevice, s), "loopback copy");
    int rc2 = done(s);
    return rc ? rc : rc2;
  }
  int allgather(const void* send, void* recv, size_t count, CommType t, cudaStream_t s) override {
    ++calls;
    const size_t bytes = count * ct_size(t);
    int rc = publish(send, s);
    for (int p = 0; p < world && !rc; ++p)
      rc = cu(cudaMemcpyAsync(static_cast<char*>(recv) + p * bytes, g->ptr[p], bytes, cudaMemcpyDeviceToDevice, s),
              "loopback copy");
    int rc2 = done(s);
    return rc ? rc : rc2;
  }
  int reduce_scatter(const void* send, void* recv, size_t count, CommType t, cudaStream_t s) override {
    ++calls;
    int rc = publish(send, s);
    if (!rc && !dptrs) rc = cu(cudaMalloc(&dptrs, sizeof(void*) * world), "loopback alloc");
    if (!rc) rc = cu(cudaMemcpyAsync(dptrs, g->ptr.data(), sizeof(void*) * world, cudaMemcpyHostToDevice, s),
                     "loopback ptrs");
    if (!rc) {
      const int grid = (int)std::min<size_t>(1024, (count + 255) / 256);
      if (t == CT_F32)
        loopback_rs_sum<float><<<grid, 256, 0, s>>>(reinterpret_cast<const float* const*>(dptrs), world,
                                                     rank * count, count, static_cast<float*>(recv));
      else
        loopback_rs_sum<double><<<grid, 256, 0, s>>>(reinterpret_cast<const double* const*>(dptrs), world,
                                                      rank * count, count, static_cast<double*>(recv));
      rc = cu(cudaGetLastError(), "loopback reduce");
    }
    int rc2 = done(s);
    return rc ? rc : rc2;
  }
  int sync_point(cudaStream_t s) override { return done(s); }
  int halo(void* buf, int64_t row0, int64_t nloc, int64_t h, size_t esz, CommType, cudaStream_t s) override {
    ++calls;
    int rc = publish(buf, s);
    char* b = static_cast<char*>(buf);
    if (!rc && h > 0 && rank > 0)
      rc = cu(cudaMemcpyAsync(b + (row0 - h) * esz, static_cast<const char*>(g->ptr[rank - 1]) + (row0 - h) * esz,
                              h * esz, cudaMemcpyDeviceToDevice, s), "loopback halo");
    if (!rc && h > 0 && rank < world - 1)
      rc = cu(cudaMemcpyAsync(b + (row0 + nloc) * esz, static_cast<const char*>(g->ptr[rank + 1]) + (row0 + nloc) * esz,
                              h * esz, cudaMemcpyDeviceToDevice, s), "loopback halo");
    int rc2 = done(s);
    return rc ? rc : rc2;
  }
};

}  // namespace ccg
