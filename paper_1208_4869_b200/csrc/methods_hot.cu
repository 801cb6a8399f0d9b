// methods_hot.cu — Engine<CCG_T> member definitions: the five hot-path methods of SURVEY §8(a): BiCGSTAB, CGNE, QMR (PIM90 set, §2.1; QMR per P:101 §6), BiCOR and CORS (§2.4) — recurrences O1-O5 of SURVEY §8(c).
// Compiled once per dtype (-DCCG_T=float / double) by build.py.
#include "engine.cuh"

#ifndef CCG_T
#error "compile with -DCCG_T=float or -DCCG_T=double"
#endif

template <typename T>
int Engine<T>::bicgstab_setup(ccg_ctx* c, bool x0) {
  TRY(init_residual(c, x0, L(c, 2), L(c, 3), nullptr, nullptr));
  if (bs_merge_ok(c)) return pass(c, BsP<T>{L(c, 2), Fs(c, 0), L(c, 4)}, &c->st->done);   // p = r; later p's come from BsXP
  return CCG_OK;
}

template <typename T>
int Engine<T>::bicgstab_iter(ccg_ctx* c) {
  const int* g = &c->st->done;
  const int* g2 = &c->st->gate2;
  if (bs_merge_ok(c)) {   // X and P passes merged, ρ' from the t = A s reduction (methods.cuh BsTm / BsXP)
    TRY(matvec_a(c, F(c, 0), BsV<T>{L(c, 4), L(c, 3)}, g));
    TRY(pass(c, BsS<T>{L(c, 2), L(c, 4), Fs(c, 1)}, g));
    TRY(matvec_a(c, F(c, 1), BsTm<T>{L(c, 5), Fs(c, 1), L(c, 3)}, g2));
    return pass(c, BsXP<T>{L(c, X), L(c, 2), Fs(c, 0), Fs(c, 1), L(c, 5), L(c, 4)}, g);
  }
  if (in_fuse_ok(c)) {   // P and S formed inside the products (methods.cuh BsPIn / BsSIn)
    TRY(matvec_a_in(c, BsPIn<T>{L(c, 2), Fs(c, 0), L(c, 4)}, BsV2<T>{L(c, 4), L(c, 3), L(c, 2), Fs(c, 0)}, g));
    TRY(matvec_a_in(c, BsSIn<T>{L(c, 2), L(c, 4)}, BsT2<T>{L(c, 5), Fs(c, 1), L(c, 2), L(c, 4)}, g));
    return pass(c, BsX<T>{L(c, X), L(c, 2), Fs(c, 0), Fs(c, 1), L(c, 5), L(c, 3)}, g);
  }
  TRY(pass(c, BsP<T>{L(c, 2), Fs(c, 0), L(c, 4)}, g));
  TRY(allgather(c, 0));
  TRY(matvec_a(c, F(c, 0), BsV<T>{L(c, 4), L(c, 3)}, g));
  if (in_fuse_ro_ok(c)) {   // stencil / SELL: s = r − αv formed inside t = A s (BsSIn / BsT2)
    TRY(matvec_a_in(c, BsSIn<T>{L(c, 2), L(c, 4)}, BsT2<T>{L(c, 5), Fs(c, 1), L(c, 2), L(c, 4)}, g));
    return pass(c, BsX<T>{L(c, X), L(c, 2), Fs(c, 0), Fs(c, 1), L(c, 5), L(c, 3)}, g);
  }
  TRY(pass(c, BsS<T>{L(c, 2), L(c, 4), Fs(c, 1)}, g));
  TRY(allgather(c, 1));
  TRY(matvec_a(c, F(c, 1), BsT<T>{L(c, 5), Fs(c, 1)}, g2));
  return pass(c, BsX<T>{L(c, X), L(c, 2), Fs(c, 0), Fs(c, 1), L(c, 5), L(c, 3)}, g);
}

template <typename T>
int Engine<T>::cgne_setup(ccg_ctx* c, bool x0) {
  TRY(init_residual(c, x0, L(c, 2), nullptr, nullptr, nullptr));
  return matvec_h(c, L(c, 2), true, CgP0<T>{Fs(c, 0)}, &c->st->done);
}

template <typename T>
int Engine<T>::cgne_iter(ccg_ctx* c) {
  const int* g = &c->st->done;
  TRY(allgather(c, 0));
  TRY(matvec_a(c, F(c, 0), CgQ<T>{L(c, 2), L(c, X), Fs(c, 0)}, g));
  return matvec_h(c, L(c, 2), true, CgP<T>{Fs(c, 0)}, g);
}

template <typename T>
int Engine<T>::qmr_setup(ccg_ctx* c, bool x0) {
  TRY(init_residual(c, x0, L(c, 2), L(c, 3), L(c, 4), nullptr));
  return pass(c, QmV<T>{L(c, 3), L(c, 4), L(c, 5), L(c, 6)}, &c->st->done);
}

template <typename T>
int Engine<T>::qmr_iter(ccg_ctx* c) {
  const int* g = &c->st->done;
  TRY(pass(c, QmP<T>{L(c, 5), L(c, 6), Fs(c, 0), L(c, 7)}, g));
  TRY(allgather(c, 0));
  if (c->opk == OPK_DENSE && c->cols_ok && c->qmr_dual && !c->rep && !c->jac_active) {
    TRY(matvec_dual(c, F(c, 0), L(c, 7), QmPt<T>{L(c, 8), L(c, 7)},
                    QmVW<T>{L(c, 3), L(c, 4), L(c, 8), L(c, 5), L(c, 6)}, g));
  } else {
    TRY(matvec_a(c, F(c, 0), QmPt<T>{L(c, 8), L(c, 7)}, g));
    TRY(matvec_h(c, L(c, 7), true, QmVW<T>{L(c, 3), L(c, 4), L(c, 8), L(c, 5), L(c, 6)}, g));
  }
  return pass(c, QmDV<T>{L(c, 9), L(c, 10), L(c, X), L(c, 2), Fs(c, 0), L(c, 8), L(c, 3), L(c, 4), L(c, 5),
                         L(c, 6)},
              g);
}

template <typename T>
int Engine<T>::bicor_setup(ccg_ctx* c, bool x0) { return init_residual(c, x0, Fs(c, 0), L(c, 2), nullptr, nullptr); }

template <typename T>
int Engine<T>::bicor_iter(ccg_ctx* c) {
  const int* g = &c->st->done;
  TRY(allgather(c, 0));
  TRY(matvec_a(c, F(c, 0), RhoEpi<T>{L(c, 3), L(c, 2)}, g));
  TRY(pass(c, BcP<T>{Fs(c, 0), L(c, 2), L(c, 3), L(c, 4), L(c, 5), L(c, 6)}, g));
  TRY(matvec_h(c, L(c, 5), true, BcQs<T>{L(c, 7), L(c, 6)}, g));
  return pass(c, BcX<T>{L(c, X), Fs(c, 0), L(c, 2), L(c, 4), L(c, 6), L(c, 7)}, g);
}

template <typename T>
int Engine<T>::cors_setup(ccg_ctx* c, bool x0) { return init_residual(c, x0, Fs(c, 0), L(c, 2), nullptr, nullptr); }

template <typename T>
int Engine<T>::cors_iter(ccg_ctx* c) {
  const int* g = &c->st->done;
  TRY(allgather(c, 0));
  TRY(matvec_a(c, F(c, 0), RhoEpi<T>{L(c, 3), L(c, 2)}, g));
  TRY(pass(c, CoP<T>{Fs(c, 0), L(c, 3), L(c, 6), L(c, 7), L(c, 4), L(c, 5), Fs(c, 1)}, g));
  TRY(allgather(c, 1));
  TRY(matvec_a(c, F(c, 1), CoQ<T>{L(c, 8), L(c, 2)}, g));
  return pass(c, CoH<T>{L(c, 4), L(c, 5), Fs(c, 1), L(c, 8), L(c, 6), L(c, 7), L(c, X), Fs(c, 0)}, g);
}

// instantiations
template int Engine<CCG_T>::bicgstab_setup(ccg_ctx* c, bool x0);
template int Engine<CCG_T>::bicgstab_iter(ccg_ctx* c);
template int Engine<CCG_T>::cgne_setup(ccg_ctx* c, bool x0);
template int Engine<CCG_T>::cgne_iter(ccg_ctx* c);
template int Engine<CCG_T>::qmr_setup(ccg_ctx* c, bool x0);
template int Engine<CCG_T>::qmr_iter(ccg_ctx* c);
template int Engine<CCG_T>::bicor_setup(ccg_ctx* c, bool x0);
template int Engine<CCG_T>::bicor_iter(ccg_ctx* c);
template int Engine<CCG_T>::cors_setup(ccg_ctx* c, bool x0);
template int Engine<CCG_T>::cors_iter(ccg_ctx* c);
