// methods_core.cu — Engine<CCG_T> member definitions: per-method dispatch, the true residual, Jacobi scaling and ccg_apply.
// Compiled once per dtype (-DCCG_T=float / double) by build.py.
#include "engine.cuh"

#ifndef CCG_T
#error "compile with -DCCG_T=float or -DCCG_T=double"
#endif

template <typename T>
int Engine<T>::setup(ccg_ctx* c, int m, bool x0) {
  switch (m) {
    case M_BICGSTAB: return bicgstab_setup(c, x0);
    case M_CGNE: return cgne_setup(c, x0);
    case M_QMR: return qmr_setup(c, x0);
    case M_BICOR: return bicor_setup(c, x0);
    case M_CORS: return cors_setup(c, x0);
    case M_BICG: return bicg_setup(c, x0);
    case M_CGS: return cgs_setup(c, x0);
    case M_COCR: return cocr_setup(c, x0);
    case M_TFQMR: return tfqmr_setup(c, x0);
    case M_GMRES: return gmres_setup(c, x0);
    case M_BICGSTABL: return bicgstabl_setup(c, x0);
    case M_PBICGSTAB: return pbicgstab_setup(c, x0);
    default: return cgnr_setup(c, x0);
  }
}

template <typename T>
int Engine<T>::iter(ccg_ctx* c, int m) {
  switch (m) {
    case M_BICGSTAB: return bicgstab_iter(c);
    case M_CGNE: return cgne_iter(c);
    case M_QMR: return qmr_iter(c);
    case M_BICOR: return bicor_iter(c);
    case M_CORS: return cors_iter(c);
    case M_BICG: return bicg_iter(c);
    case M_CGS: return cgs_iter(c);
    case M_COCR: return cocr_iter(c);
    case M_TFQMR: return tfqmr_iter(c);
    case M_GMRES: return gmres_iter(c);
    case M_BICGSTABL: return bicgstabl_iter(c);
    case M_PBICGSTAB: return pbicgstab_iter(c);
    default: return cgnr_iter(c);
  }
}

template <typename T>
int Engine<T>::true_residual(ccg_ctx* c) {
  const int* g = c->zero_gate;
  TRY(pass(c, Copy<T>{L(c, X), Fs(c, 2)}, g));
  TRY(allgather(c, 2));
  return matvec_a(c, F(c, 2), TrueRes<T>{L(c, 1)}, g);
}

template <typename T>
int Engine<T>::jac_in(ccg_ctx* c) {
  return pass_count(c, JacScale<T>{L(c, X), reinterpret_cast<const C*>(c->jac_d) + c->row0, L(c, X)}, c->nloc,
                    c->zero_gate);
}

template <typename T>
int Engine<T>::jac_out(ccg_ctx* c) {
  return pass_count(c, JacScale<T>{L(c, X), reinterpret_cast<const C*>(c->jac_dinv) + c->row0, L(c, X)}, c->nloc,
                    c->zero_gate);
}

template <typename T>
int Engine<T>::apply(ccg_ctx* c, int op, const C* xin, C* yout) {
  const int* g = c->zero_gate;
  if (op == CCG_OP_A || (op == CCG_OP_AT && (c->opk == OPK_CSR || c->opk == OPK_STENCIL))) {
    CK(c, cudaMemcpyAsync(Fs(c, 2), xin, c->nloc * sizeof(C), cudaMemcpyDeviceToDevice, c->stream));
    TRY(allgather(c, 2));
    return matvec_a(c, F(c, 2), Store<T>{yout}, g);
  }
  CK(c, cudaMemcpyAsync(L(c, 2), xin, c->nloc * sizeof(C), cudaMemcpyDeviceToDevice, c->stream));
  return matvec_h(c, L(c, 2), op == CCG_OP_AH, Store<T>{yout}, g);
}

// instantiations
template int Engine<CCG_T>::setup(ccg_ctx* c, int m, bool x0);
template int Engine<CCG_T>::iter(ccg_ctx* c, int m);
template int Engine<CCG_T>::true_residual(ccg_ctx* c);
template int Engine<CCG_T>::jac_in(ccg_ctx* c);
template int Engine<CCG_T>::jac_out(ccg_ctx* c);
template int Engine<CCG_T>::apply(ccg_ctx* c, int op, const C* xin, C* yout);
