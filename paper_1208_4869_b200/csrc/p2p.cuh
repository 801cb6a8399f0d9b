// p2p.cuh — SURVEY §8(f) NEXT-2 (i): collective fusion over NVLink for the
// replicated-vector mode (CCG_OPT_P2P).
//
// In replicated mode every product ends with a gather: A·x's rows (and the
// CSR / stencil Aᴴ rows) of every rank into the whole vector, the dense
// Aᴴ·x full-length partial of every rank into a world × n array.  Instead of
// an NCCL allgather after the product kernel, the product's epilogue STORES
// its outputs straight into the mirror buffer of every rank (peer pointers
// of an NCCL symmetric-memory window, ncclCommWindowRegister /
// ncclGetPeerPointer; on the one-GPU loopback, the other handles' buffers),
// then one thread per rank publishes a release flag on every peer and the
// consumer waits for all ranks' flags of this exchange (acquire) — the
// transfer rides on the product's own stores, tile by tile, and the
// collective launch disappears.
//
// Buffers are double-buffered by the parity of a device-side exchange epoch:
// a rank that runs ahead (replicated mode has no other synchronisation) can
// only write buffer e%2 after every peer has signalled exchange e−1, i.e.
// after every peer has consumed exchange e−2 from that buffer.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace ccg {

constexpr int P2P_MAX = 8;   // ranks on one NVLink/NVSwitch domain (one node)

struct P2pCtl {
  uint64_t* flags[P2P_MAX];   // flags[p]: rank p's flag array (P2P_MAX slots, one per source rank)
  uint64_t* ctr;              // this rank: ctr[0] = send epoch, ctr[1] = receive epoch
  int world, rank;
};

__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// after the product kernel (stream order + PDL wait: its stores are done):
// publish this rank's epoch on every peer
static __global__ void p2p_signal(P2pCtl c, const int* gate) {
  if (pdl_gate(gate)) return;
  const uint64_t e = c.ctr[0] + 1;
  c.ctr[0] = e;
  __threadfence_system();
  for (int p = 0; p < c.world; ++p) st_release_sys(c.flags[p] + c.rank, e);
}

// before the consumer: every rank's epoch of this exchange has arrived
static __global__ void p2p_wait(P2pCtl c, const int* gate) {
  if (pdl_gate(gate)) return;
  const uint64_t e = c.ctr[1] + 1;
  c.ctr[1] = e;
  const uint64_t* mine = c.flags[c.rank];
  for (int p = 0; p < c.world; ++p)
    while (ld_acquire_sys(mine + p) < e) __nanosleep(64);
  __threadfence_system();
}

// product epilogue: out[i] -> every rank's mirror buffer of this exchange's
// parity, at element offset `off` (this rank's rows / partial slot)
template <typename T>
struct MirrorStore {
  static constexpr int K = 0;
  using C = typename CT<T>::c;
  C* dst[2][P2P_MAX];          // [parity][rank]
  const uint64_t* ctr;          // send epoch: this product is exchange ctr[0] + 1
  int world;
  int par;
  __device__ void load(const State*) { par = (int)((ctr[0] + 1) & 1); }
  __device__ void operator()(int64_t i, C v, double2*) {
#pragma unroll 1
    for (int p = 0; p < world; ++p) dst[par][p][i] = v;
  }
  static __device__ void finish(State*, const double2*) {}
};

// the consumer's view of this rank's mirror buffer (receive-epoch parity)
template <typename T>
struct MirrorView {
  using C = typename CT<T>::c;
  const C* buf[2];
  const uint64_t* ctr;
  __device__ const C* get() const { return buf[ctr[1] & 1]; }
};

// the method epilogue over the gathered vector (as EpiPass, buffer by parity)
template <typename T, class Epi>
struct EpiPassMirror {
  static constexpr int K = Epi::K;
  using C = typename CT<T>::c;
  Epi epi;
  MirrorView<T> v;
  const C* w;
  __device__ void load(const State* st) { epi.load(st); w = v.get(); }
  __device__ void operator()(int64_t i, double2* acc) { epi(i, w[i], acc); }
  static __device__ void finish(State* st, const double2* s) { Epi::finish(st, s); }
};

// ... and over Σ_ranks parts[r][i] in rank order (dense Aᴴ, as EpiPassSum)
template <typename T, class Epi>
struct EpiPassMirrorSum {
  static constexpr int K = Epi::K;
  using C = typename CT<T>::c;
  Epi epi;
  MirrorView<T> v;
  int world;
  int64_t n;
  const C* w;
  __device__ void load(const State* st) { epi.load(st); w = v.get(); }
  __device__ void operator()(int64_t i, double2* acc) {
    double2 s = make_double2(0.0, 0.0);
    for (int r = 0; r < world; ++r) {
      const C a = w[(int64_t)r * n + i];
      s.x += (double)a.x;
      s.y += (double)a.y;
    }
    epi(i, fromd2<C>(s), acc);
  }
  static __device__ void finish(State* st, const double2* s) { Epi::finish(st, s); }
};

}  // namespace ccg
