// tfg_vote_inst.cu — the vote kernel instantiations of one quantiser
// (TFG_QUANT = tfg::Quant), compiled once per quantiser as tfg_vote_q<N>.o so
// the four sets build in parallel. tfg_engine.cu dispatches through
// tfg_pick_vote_q<N>(strat, ksel) (glcm_vote_kernel), tfg_pick_jobs_q<N>(strat)
// (glcm_vote_jobs_kernel, L <= 64) and tfg_pick_jobs1_q<N>(strat, ksel)
// (glcm_vote_jobs1/2_kernel, L > 64).
#define TFG_VOTE_ONLY
#include "tfg_kernels.cuh"

#ifndef TFG_QUANT
#error "define TFG_QUANT (0..3)"
#endif

using VoteKernel = void (*)(const tfg::VoteParams);

namespace {
template <int Q, int S>
VoteKernel pick_k(int ksel) {
  switch (ksel) {
    case 0: return tfg::glcm_vote_kernel<Q, S, 0>;
    case 1: return tfg::glcm_vote_kernel<Q, S, 1>;
    case 2: return tfg::glcm_vote_kernel<Q, S, 2>;
    case 3: return tfg::glcm_vote_kernel<Q, S, 3>;
    case 5: return tfg::glcm_vote_kernel<Q, S, 5>;
    case 6: return tfg::glcm_vote_kernel<Q, S, 6>;
    case 7: return tfg::glcm_vote_kernel<Q, S, 7>;
    case 8: return tfg::glcm_vote_kernel<Q, S, 8>;
    default: return tfg::glcm_vote_kernel<Q, S, 4>;
  }
}
}  // namespace

#define TFG_CAT2(a, b) a##b
#define TFG_CAT(a, b) TFG_CAT2(a, b)
VoteKernel TFG_CAT(tfg_pick_vote_q, TFG_QUANT)(int strat, int ksel) {
  constexpr int Q = TFG_QUANT;
  switch (strat) {
    case tfg::S_COPIES32: return pick_k<Q, tfg::S_COPIES32>(ksel);
    case tfg::S_COPIES8: return pick_k<Q, tfg::S_COPIES8>(ksel);
    case tfg::S_COPY1: return pick_k<Q, tfg::S_COPY1>(ksel);
    case tfg::S_P16X16: return pick_k<Q, tfg::S_P16X16>(ksel);
    default: return pick_k<Q, tfg::S_PACKED16>(ksel);
  }
}

using JobsKernel = void (*)(const tfg::VoteJobs);
// the multi-job kernel of a layout without per-CTA partials (L <= 64)
JobsKernel TFG_CAT(tfg_pick_jobs_q, TFG_QUANT)(int strat) {
  constexpr int Q = TFG_QUANT;
  switch (strat) {
    case tfg::S_COPIES32: return tfg::glcm_vote_jobs_kernel<Q, tfg::S_COPIES32>;
    case tfg::S_COPIES8: return tfg::glcm_vote_jobs_kernel<Q, tfg::S_COPIES8>;
    case tfg::S_P16X16: return tfg::glcm_vote_jobs_kernel<Q, tfg::S_P16X16>;
    default: return nullptr;  // COPY1, PACKED16: tfg_pick_jobs1_q<N>
  }
}

namespace {
template <int Q, int S>
JobsKernel pick_j1(int ksel) {
  switch (ksel) {
    case 0: return tfg::glcm_vote_jobs1_kernel<Q, S, 0>;
    case 1: return tfg::glcm_vote_jobs1_kernel<Q, S, 1>;
    case 2: return tfg::glcm_vote_jobs1_kernel<Q, S, 2>;
    case 3: return tfg::glcm_vote_jobs1_kernel<Q, S, 3>;
    case 5: return tfg::glcm_vote_jobs1_kernel<Q, S, 5>;
    case 6: return tfg::glcm_vote_jobs1_kernel<Q, S, 6>;
    case 7: return tfg::glcm_vote_jobs1_kernel<Q, S, 7>;
    case 8: return tfg::glcm_vote_jobs1_kernel<Q, S, 8>;
    default: return tfg::glcm_vote_jobs1_kernel<Q, S, 4>;
  }
}
}  // namespace

// the multi-job kernel of a layout with per-CTA partials (cooperative
// launches) for a KSEL group (tfg_engine.cu ksel_group): COPY1 one KSEL,
// PACKED16 a KSEL pair or KSEL 4
JobsKernel TFG_CAT(tfg_pick_jobs1_q, TFG_QUANT)(int strat, int ksel) {
  constexpr int Q = TFG_QUANT;
  constexpr int P = tfg::S_PACKED16;
  switch (strat) {
    case tfg::S_COPY1: return pick_j1<Q, tfg::S_COPY1>(ksel);
    case tfg::S_PACKED16:
      switch (ksel) {
        case 0: case 1: return tfg::glcm_vote_jobs2_kernel<Q, P, 0, 1>;
        case 2: case 3: return tfg::glcm_vote_jobs2_kernel<Q, P, 2, 3>;
        case 5: case 6: return tfg::glcm_vote_jobs2_kernel<Q, P, 5, 6>;
        case 7: case 8: return tfg::glcm_vote_jobs2_kernel<Q, P, 7, 8>;
        default: return tfg::glcm_vote_jobs1_kernel<Q, P, 4>;
      }
    default: return nullptr;
  }
}
