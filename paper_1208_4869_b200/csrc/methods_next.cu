// methods_next.cu — Engine<CCG_T> member definitions: SURVEY §8(f) NEXT-3: BiCG, CGS, CGNR, COCR (§3.4), TFQMR.
// Compiled once per dtype (-DCCG_T=float / double) by build.py.
#include "engine.cuh"

#ifndef CCG_T
#error "compile with -DCCG_T=float or -DCCG_T=double"
#endif

template <typename T>
int Engine<T>::bicg_setup(ccg_ctx* c, bool x0) { return init_residual(c, x0, L(c, 2), L(c, 3), nullptr, nullptr); }

template <typename T>
int Engine<T>::bicg_iter(ccg_ctx* c) {
  const int* g = &c->st->done;
  TRY(pass(c, BgP<T>{L(c, 2), L(c, 3), Fs(c, 0), L(c, 4)}, g));
  TRY(allgather(c, 0));
  TRY(matvec_pair(c, 0, L(c, 4), BgQ<T>{L(c, 5), L(c, 4)}, Store<T>{L(c, 6)}, g));
  return pass(c, BgX<T>{L(c, X), L(c, 2), L(c, 3), Fs(c, 0), L(c, 5), L(c, 6)}, g);
}

template <typename T>
int Engine<T>::cgs_setup(ccg_ctx* c, bool x0) { return init_residual(c, x0, L(c, 2), L(c, 3), nullptr, nullptr); }

template <typename T>
int Engine<T>::cgs_iter(ccg_ctx* c) {
  const int* g = &c->st->done;
  TRY(pass(c, CsP<T>{L(c, 2), L(c, 5), Fs(c, 0), L(c, 4)}, g));
  TRY(allgather(c, 0));
  TRY(matvec_a(c, F(c, 0), CsV<T>{L(c, 6), L(c, 3)}, g));
  TRY(pass(c, CsQ<T>{L(c, 4), L(c, 6), L(c, 5), Fs(c, 1), L(c, X)}, g));
  TRY(allgather(c, 1));
  return matvec_a(c, F(c, 1), CsR<T>{L(c, 2), L(c, 3)}, g);
}

template <typename T>
int Engine<T>::cocr_setup(ccg_ctx* c, bool x0) {
  TRY(init_residual(c, x0, Fs(c, 0), nullptr, nullptr, nullptr));
  TRY(allgather(c, 0));
  return matvec_a(c, F(c, 0), CrAr0<T>{L(c, 2), Fs(c, 0)}, &c->st->done);
}

template <typename T>
int Engine<T>::cocr_iter(ccg_ctx* c) {
  const int* g = &c->st->done;
  TRY(pass(c, CrP<T>{Fs(c, 0), L(c, 2), L(c, 3), L(c, 4)}, g));
  TRY(pass(c, CrX<T>{L(c, X), Fs(c, 0), L(c, 3), L(c, 4)}, g));
  TRY(allgather(c, 0));
  return matvec_a(c, F(c, 0), CrAr<T>{L(c, 2), Fs(c, 0)}, g);
}

template <typename T>
int Engine<T>::cgnr_setup(ccg_ctx* c, bool x0) {
  TRY(init_residual(c, x0, L(c, 2), nullptr, nullptr, nullptr));
  return matvec_h(c, L(c, 2), true, CnZ0<T>{Fs(c, 0)}, &c->st->done);
}

template <typename T>
int Engine<T>::cgnr_iter(ccg_ctx* c) {
  const int* g = &c->st->done;
  TRY(allgather(c, 0));
  TRY(matvec_a(c, F(c, 0), CnW<T>{L(c, 3)}, g));
  TRY(pass(c, CnX<T>{L(c, X), L(c, 2), Fs(c, 0), L(c, 3)}, g));
  TRY(matvec_h(c, L(c, 2), true, CnZ<T>{L(c, 4)}, g));
  return pass(c, CnP<T>{L(c, 4), Fs(c, 0)}, g);
}

template <typename T>
int Engine<T>::tfqmr_setup(ccg_ctx* c, bool x0) {
  TRY(init_residual(c, x0, L(c, 2), L(c, 3), Fs(c, 0), nullptr));
  TRY(allgather(c, 0));
  return matvec_a(c, F(c, 0), TfV0<T>{L(c, 4), L(c, 6), L(c, 2)}, &c->st->done);
}

template <typename T>
int Engine<T>::tfqmr_iter(ccg_ctx* c) {
  const int* g = &c->st->done;
  const int* g2 = &c->st->gate2;
  TRY(pass(c, TfE<T>{Fs(c, 0), L(c, 4), L(c, 6), Fs(c, 1), L(c, 3), L(c, 5)}, g));
  TRY(allgather(c, 1));
  TRY(matvec_a(c, F(c, 1), TfO<T>{L(c, 7), L(c, X), L(c, 3), L(c, 5), Fs(c, 1), L(c, 2)}, g2));
  TRY(pass(c, TfU<T>{L(c, X), L(c, 5), L(c, 3), Fs(c, 1), Fs(c, 0)}, g));
  TRY(allgather(c, 0));
  return matvec_a(c, F(c, 0), TfV<T>{L(c, 6), L(c, 7), L(c, 4), L(c, 2)}, g);
}

// instantiations
template int Engine<CCG_T>::bicg_setup(ccg_ctx* c, bool x0);
template int Engine<CCG_T>::bicg_iter(ccg_ctx* c);
template int Engine<CCG_T>::cgs_setup(ccg_ctx* c, bool x0);
template int Engine<CCG_T>::cgs_iter(ccg_ctx* c);
template int Engine<CCG_T>::cocr_setup(ccg_ctx* c, bool x0);
template int Engine<CCG_T>::cocr_iter(ccg_ctx* c);
template int Engine<CCG_T>::cgnr_setup(ccg_ctx* c, bool x0);
template int Engine<CCG_T>::cgnr_iter(ccg_ctx* c);
template int Engine<CCG_T>::tfqmr_setup(ccg_ctx* c, bool x0);
template int Engine<CCG_T>::tfqmr_iter(ccg_ctx* c);
