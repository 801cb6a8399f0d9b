// methods_krylov.cu — Engine<CCG_T> member definitions: GMRES(m) ("rgmres"), BiCGstab(ℓ) (§3.1) and the pipelined BiCGSTAB of SURVEY §8(f) NEXT-2 (iii).
// Compiled once per dtype (-DCCG_T=float / double) by build.py.
#include "engine.cuh"

#ifndef CCG_T
#error "compile with -DCCG_T=float or -DCCG_T=double"
#endif

template <typename T>
int Engine<T>::gmres_setup(ccg_ctx* c, bool x0) {
  TRY(init_residual(c, x0, Vb(c), nullptr, nullptr, nullptr));
  launch_k(c, gm_normalize<T>, c->gm_vgrid, NT, 0, c->stream, Vb(c), c->nloc, Vb(c), Fs(c, 0), c->nloc, c->gm_dev, 1,
                                                       &c->st->done);
  c->launches++;
  CK(c, cudaGetLastError());
  return CCG_OK;
}

template <typename T>
int Engine<T>::gmres_iter(ccg_ctx* c) {
  const int* g = &c->st->done;
  GmDev* gm = c->gm_dev;
  C* w = L(c, 2);
  TRY(allgather(c, 0));
  TRY(matvec_a(c, F(c, 0), Store<T>{w}, g));
  TRY(gm_pass_launch<0>(c, w, nullptr, gm->hcol, g));
  TRY(gm_pass_launch<1>(c, w, gm->hcol, gm->h2, g));
  TRY(gm_pass_launch<2>(c, w, gm->h2, &gm->ww2, g));
  launch_k(c, gm_step, 1, 1, 0, c->stream, c->st, gm, g);
  launch_k(c, gm_normalize<T>, c->gm_vgrid, NT, 0, c->stream, Vb(c), c->nloc, w, Fs(c, 0), c->nloc, gm, 0, &gm->endflag);
  launch_k(c, gm_trisolve, 1, 1, 0, c->stream, c->st, gm, &gm->noend);
  launch_k(c, gm_xupdate<T>, c->gm_vgrid, NT, 0, c->stream, L(c, X), Vb(c), c->nloc, c->nloc, gm, &gm->noxupd);
  c->launches += 4;
  CK(c, cudaGetLastError());
  TRY(pass(c, Copy<T>{L(c, X), Fs(c, 2)}, &gm->norestart));
  TRY(allgather(c, 2));
  TRY(matvec_a(c, F(c, 2), GmR<T>{L(c, 1), Vb(c)}, &gm->norestart));
  launch_k(c, gm_normalize<T>, c->gm_vgrid, NT, 0, c->stream, Vb(c), c->nloc, Vb(c), Fs(c, 0), c->nloc, gm, 1,
                                                       &gm->norestart);
  launch_k(c, gm_reset, 1, 1, 0, c->stream, gm);
  c->launches += 2;
  CK(c, cudaGetLastError());
  return CCG_OK;
}

template <typename T>
int Engine<T>::bicgstabl_setup(ccg_ctx* c, bool x0) {
  TRY(init_residual(c, x0, BRs(c, 0), L(c, 3), nullptr, nullptr));
  CK(c, cudaMemsetAsync(BUs(c, 0), 0, (size_t)c->nloc * sizeof(C), c->stream));
  return CCG_OK;
}

template <typename T>
int Engine<T>::bicgstabl_iter(ccg_ctx* c) {
  const int* g = &c->st->done;
  const int ell = c->bl_l;
  for (int j = 0; j < ell; ++j) {
    BlP<T> P{};
    for (int a = 0; a <= j; ++a) { P.u[a] = BUs(c, a); P.r[a] = BRs(c, a); }
    P.J = j;
    TRY(pass(c, P, g));
    TRY(allgather_buf(c, BLU(c, j)));
    TRY(matvec_a(c, BLU(c, j), BlU<T>{BUs(c, j + 1), L(c, 3)}, g));
    BlX<T> Xp{};
    for (int a = 0; a <= j; ++a) Xp.r[a] = BRs(c, a);
    for (int a = 0; a <= j + 1; ++a) Xp.u[a] = BUs(c, a);
    Xp.x = L(c, X);
    Xp.J = j;
    TRY(pass(c, Xp, g));
    TRY(allgather_buf(c, BLR(c, j)));
    if (j < ell - 1)
      TRY(matvec_a(c, BLR(c, j), BlR<T>{BRs(c, j + 1), L(c, 3)}, g));
    else
      TRY(matvec_a(c, BLR(c, j), BlRL<T>{BRs(c, j + 1)}, g));
  }
  switch (ell) {
    case 1: return bicgstabl_mr<1>(c, g);
    case 2: return bicgstabl_mr<2>(c, g);
    case 3: return bicgstabl_mr<3>(c, g);
    default: return bicgstabl_mr<4>(c, g);
  }
}

template <typename T>
int Engine<T>::pbicgstab_setup(ccg_ctx* c, bool x0) {
  const int* g = &c->st->done;
  TRY(init_residual(c, x0, L(c, 2), L(c, 3), Fs(c, 0), nullptr));
  TRY(allgather(c, 0));
  TRY(matvec_a(c, F(c, 0), PbW0<T>{Fs(c, 1), L(c, 3)}, g));
  TRY(allgather(c, 1));
  return matvec_a(c, F(c, 1), PbStore<T>{L(c, 9)}, g);
}

template <typename T>
int Engine<T>::pbicgstab_iter(ccg_ctx* c) {
  const int* g = &c->st->done;
  const int* g2 = &c->st->gate2;
  TRY(pass(c, PbP1<T>{L(c, 2), Fs(c, 1), L(c, 9), L(c, 8), L(c, 4), L(c, 5), Fs(c, 0), L(c, 6), L(c, 7)}, g));
  TRY(allgather(c, 0));
  TRY(matvec_a(c, F(c, 0), PbStore<T>{L(c, 8)}, g2));
  TRY(pass(c, PbP2<T>{L(c, X), L(c, 2), Fs(c, 1), L(c, 4), L(c, 6), L(c, 7), L(c, 9), L(c, 8), L(c, 5), Fs(c, 0),
                      L(c, 3)},
           g));
  TRY(allgather(c, 1));
  return matvec_a(c, F(c, 1), PbT<T>{L(c, 9)}, g);
}

// instantiations
template int Engine<CCG_T>::gmres_setup(ccg_ctx* c, bool x0);
template int Engine<CCG_T>::gmres_iter(ccg_ctx* c);
template int Engine<CCG_T>::bicgstabl_setup(ccg_ctx* c, bool x0);
template int Engine<CCG_T>::bicgstabl_iter(ccg_ctx* c);
template int Engine<CCG_T>::pbicgstab_setup(ccg_ctx* c, bool x0);
template int Engine<CCG_T>::pbicgstab_iter(ccg_ctx* c);
