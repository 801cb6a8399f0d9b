// methods_cluster.cu — Engine<CCG_T> member definitions: the whole-solve single-cluster launch for small dense systems (cluster.cuh).
// Compiled once per dtype (-DCCG_T=float / double) by build.py.
#include "engine.cuh"

#ifndef CCG_T
#error "compile with -DCCG_T=float or -DCCG_T=double"
#endif

template <typename T>
int Engine<T>::cluster_run(ccg_ctx* c, int m) {
  switch (m) {
    case M_BICGSTAB:
      if (c->cl_redundant)
        return launch_cluster(c, ClBicgstabR<T>{BsP<T>{L(c, 2), Fs(c, 0), L(c, 4)}, BsV<T>{L(c, 4), L(c, 3)},
                                                BsS<T>{L(c, 2), L(c, 4), Fs(c, 1)}, BsT<T>{L(c, 5), Fs(c, 1)},
                                                BsX<T>{L(c, X), L(c, 2), Fs(c, 0), Fs(c, 1), L(c, 5), L(c, 3)},
                                                F(c, 0), F(c, 1), F(c, 2)});
      return launch_cluster(c, ClBicgstab<T>{BsP<T>{L(c, 2), Fs(c, 0), L(c, 4)}, BsV<T>{L(c, 4), L(c, 3)},
                                             BsS<T>{L(c, 2), L(c, 4), Fs(c, 1)}, BsT<T>{L(c, 5), Fs(c, 1)},
                                             BsX<T>{L(c, X), L(c, 2), Fs(c, 0), Fs(c, 1), L(c, 5), L(c, 3)},
                                             F(c, 0), F(c, 1)});
    case M_CGNE:
      return launch_cluster(c, ClCgne<T>{CgQ<T>{L(c, 2), L(c, X), Fs(c, 0)}, CgP<T>{Fs(c, 0)}, CgP0<T>{Fs(c, 0)},
                                         F(c, 0), L(c, 2)});
    case M_QMR:
      return launch_cluster(
          c, ClQmr<T>{QmP<T>{L(c, 5), L(c, 6), Fs(c, 0), L(c, 7)}, QmPt<T>{L(c, 8), L(c, 7)},
                      QmVW<T>{L(c, 3), L(c, 4), L(c, 8), L(c, 5), L(c, 6)},
                      QmDV<T>{L(c, 9), L(c, 10), L(c, X), L(c, 2), Fs(c, 0), L(c, 8), L(c, 3), L(c, 4), L(c, 5),
                              L(c, 6)},
                      QmV<T>{L(c, 3), L(c, 4), L(c, 5), L(c, 6)}, F(c, 0), L(c, 7)});
    case M_BICOR:
      return launch_cluster(c, ClBicor<T>{RhoEpi<T>{L(c, 3), L(c, 2)},
                                          BcP<T>{Fs(c, 0), L(c, 2), L(c, 3), L(c, 4), L(c, 5), L(c, 6)},
                                          BcQs<T>{L(c, 7), L(c, 6)},
                                          BcX<T>{L(c, X), Fs(c, 0), L(c, 2), L(c, 4), L(c, 6), L(c, 7)}, F(c, 0),
                                          L(c, 5)});
    case M_CORS:
      return launch_cluster(
          c, ClCors<T>{RhoEpi<T>{L(c, 3), L(c, 2)}, CoP<T>{Fs(c, 0), L(c, 3), L(c, 6), L(c, 7), L(c, 4), L(c, 5), Fs(c, 1)},
                       CoQ<T>{L(c, 8), L(c, 2)},
                       CoH<T>{L(c, 4), L(c, 5), Fs(c, 1), L(c, 8), L(c, 6), L(c, 7), L(c, X), Fs(c, 0)}, F(c, 0),
                       F(c, 1)});
    case M_BICG:
      return launch_cluster(c, ClBicg<T>{BgP<T>{L(c, 2), L(c, 3), Fs(c, 0), L(c, 4)}, BgQ<T>{L(c, 5), L(c, 4)},
                                         Store<T>{L(c, 6)},
                                         BgX<T>{L(c, X), L(c, 2), L(c, 3), Fs(c, 0), L(c, 5), L(c, 6)}, F(c, 0),
                                         L(c, 4)});
    case M_CGS:
      return launch_cluster(c, ClCgs<T>{CsP<T>{L(c, 2), L(c, 5), Fs(c, 0), L(c, 4)}, CsV<T>{L(c, 6), L(c, 3)},
                                        CsQ<T>{L(c, 4), L(c, 6), L(c, 5), Fs(c, 1), L(c, X)},
                                        CsR<T>{L(c, 2), L(c, 3)}, F(c, 0), F(c, 1)});
    case M_COCR:
      return launch_cluster(c, ClCocr<T>{CrP<T>{Fs(c, 0), L(c, 2), L(c, 3), L(c, 4)},
                                         CrX<T>{L(c, X), Fs(c, 0), L(c, 3), L(c, 4)}, CrAr<T>{L(c, 2), Fs(c, 0)},
                                         CrAr0<T>{L(c, 2), Fs(c, 0)}, F(c, 0)});
    case M_TFQMR:
      return launch_cluster(c, ClTfqmr<T>{TfE<T>{Fs(c, 0), L(c, 4), L(c, 6), Fs(c, 1), L(c, 3), L(c, 5)},
                                          TfO<T>{L(c, 7), L(c, X), L(c, 3), L(c, 5), Fs(c, 1), L(c, 2)},
                                          TfU<T>{L(c, X), L(c, 5), L(c, 3), Fs(c, 1), Fs(c, 0)},
                                          TfV<T>{L(c, 6), L(c, 7), L(c, 4), L(c, 2)},
                                          TfV0<T>{L(c, 4), L(c, 6), L(c, 2)}, F(c, 0), F(c, 1)});
    case M_PBICGSTAB:
      return launch_cluster(
          c, ClPbicgstab<T>{PbW0<T>{Fs(c, 1), L(c, 3)}, PbStore<T>{L(c, 9)},
                            PbP1<T>{L(c, 2), Fs(c, 1), L(c, 9), L(c, 8), L(c, 4), L(c, 5), Fs(c, 0), L(c, 6), L(c, 7)},
                            PbStore<T>{L(c, 8)},
                            PbP2<T>{L(c, X), L(c, 2), Fs(c, 1), L(c, 4), L(c, 6), L(c, 7), L(c, 9), L(c, 8), L(c, 5),
                                    Fs(c, 0), L(c, 3)},
                            PbT<T>{L(c, 9)}, F(c, 0), F(c, 1)});
    default:
      return launch_cluster(c, ClCgnr<T>{CnW<T>{L(c, 3)}, CnX<T>{L(c, X), L(c, 2), Fs(c, 0), L(c, 3)},
                                         CnZ<T>{L(c, 4)}, CnP<T>{L(c, 4), Fs(c, 0)}, CnZ0<T>{Fs(c, 0)}, F(c, 0),
                                         L(c, 2)});
  }
}

// instantiations
template int Engine<CCG_T>::cluster_run(ccg_ctx* c, int m);
