// aca_dim.cu -- the ACA size-class kernels instantiated for ONE point dimension
// (compiled once per HM_ACA_DIM in {0 (generic d > 4), 1, 2, 3, 4}, see Makefile), so the
// heavy template instantiations build in parallel.  Launch order per chunk: the general
// CTA kernel (epsilon criterion / k > 32), the cluster kernels, the big-block kernel,
// then the window kernels from the largest class down (largest-first within a class).
#include "aca_impl.cuh"

#include <type_traits>

#ifndef HM_ACA_DIM
#error "compile with -DHM_ACA_DIM=<0..4>"
#endif
#define HM_CAT2(a, b) a##b
#define HM_CAT(a, b) HM_CAT2(a, b)

namespace hmb {
namespace aca_detail {

template <int DIM, int KIND>
static void classes_kind(const AcaClassLaunch& L, cudaStream_t s0) {
  KernelEntry<DIM, KIND> E{L.coords, L.n, L.d, L.kp};
  PhaseTrace& tr = *L.tr;
  const int kmax = L.J[0].kmax;
  const int sms = L.sms;
  // the size classes are independent: the cluster and big-block kernels go to a second
  // stream so their tails overlap the window kernels (and vice versa)
  cudaStream_t s = L.s2 ? L.s2 : s0;
  if (kmax <= 16) {
    bool done = false;
    if constexpr (DIM > 0) {
      if (L.smooth) {
        // smooth-path cluster kernels, then the general cluster kernels on their fallbacks
        auto two_pass = [&](auto clc, int q) {
          constexpr int CLq = decltype(clc)::value;
          AcaJob Js = L.J[q];
          Js.fb_list = L.fb_list + L.first[q];
          Js.fb_count = L.fb_count + q;
          launch_smooth_cluster<DIM, KIND, CLq>(Js, E, sms, s);
          AcaJob Jw = L.J[q];
          Jw.order = Js.fb_list;
          Jw.njobs_dev = Js.fb_count;
          Jw.counter = L.fb_counter + q;
          launch_cluster<DIM, KIND, 16, CLq>(Jw, E, sms, s);
        };
        two_pass(std::integral_constant<int, 4>{}, kAcaCl4);
        two_pass(std::integral_constant<int, 8>{}, kAcaCl8);
        done = true;
      }
    }
    if (!done) {
      launch_cluster<DIM, KIND, 16, 4>(L.J[kAcaCl4], E, sms, s);
      launch_cluster<DIM, KIND, 16, 8>(L.J[kAcaCl8], E, sms, s);
    }
  } else {
    launch_cluster<DIM, KIND, 32, 4>(L.J[kAcaCl4], E, sms, s);
    launch_cluster<DIM, KIND, 32, 8>(L.J[kAcaCl8], E, sms, s);
  }
  tr.mark("clusters (<=4096)", s);
  if (L.J[kAcaBig].njobs > 0) {
    const bool big_one = L.big_one;
    if (kmax <= 16) launch_big<DIM, KIND, 16>(L.J[kAcaBig], E, L.max_rows_big, sms, *L.big_scratch, s, big_one);
    else launch_big<DIM, KIND, 32>(L.J[kAcaBig], E, L.max_rows_big, sms, *L.big_scratch, s, big_one);
    tr.mark("big (>4096)", s);
  }
  s = s0;
  if (kmax <= 16) {
    bool mid_done = false;
    if constexpr (DIM > 0) {
      if (L.smooth && L.smooth_mid) {
        // <= 512 and <= 1024: the smooth cluster kernel on 1 and 2 CTAs (512 rows each),
        // the window kernels on the blocks it hands back
        auto two_pass = [&](auto clc, int q) {
          constexpr int CLq = decltype(clc)::value;
          AcaJob Js = L.J[q];
          Js.fb_list = L.fb_list + L.first[q];
          Js.fb_count = L.fb_count + q;
          launch_smooth_cluster<DIM, KIND, CLq>(Js, E, sms, s);
          AcaJob Jw = L.J[q];
          Jw.order = Js.fb_list;
          Jw.njobs_dev = Js.fb_count;
          Jw.counter = L.fb_counter + q;
          if constexpr (CLq == 2) launch_win<DIM, KIND, 16, 16, 8, true>(Jw, E, sms, s);
          else launch_win<DIM, KIND, 8, 16, 8, true, 2>(Jw, E, sms, s);
        };
        two_pass(std::integral_constant<int, 2>{}, 4);
        tr.mark("smooth CL=2 (<=1024)", s);
        two_pass(std::integral_constant<int, 1>{}, 3);
        tr.mark("smooth CL=1 (<=512)", s);
        mid_done = true;
      }
    }
    if (!mid_done) {
      launch_win<DIM, KIND, 16, 16, 8, true>(L.J[4], E, sms, s);
      tr.mark("win NW=16 (<=1024)", s);
      launch_win<DIM, KIND, 8, 16, 8, true, 2>(L.J[3], E, sms, s);
      tr.mark("NW=8 (<=512)", s);
    }
    if constexpr (DIM > 0) {
      if (L.smooth) {
        // smooth-path kernels, then the general window kernel over the blocks they handed back
        auto smooth_then_window = [&](auto nwc, int q) {
          constexpr int NWq = decltype(nwc)::value;
          AcaJob Js = L.J[q];
          Js.fb_list = L.fb_list + L.first[q];
          Js.fb_count = L.fb_count + q;
          if (L.smooth_pre) launch_smooth<DIM, KIND, NWq, true>(Js, E, sms, s);
          else launch_smooth<DIM, KIND, NWq, false>(Js, E, sms, s);
          AcaJob Jw = L.J[q];
          Jw.order = Js.fb_list;
          Jw.njobs_dev = Js.fb_count;
          Jw.counter = L.fb_counter + q;
          if constexpr (NWq == 4) launch_win<DIM, KIND, 4, 16, 16, true, 3>(Jw, E, sms, s);
          else if constexpr (NWq == 2) launch_win<DIM, KIND, 2, 16, 16, true, 3>(Jw, E, sms, s);
          else launch_win<DIM, KIND, 1, 16, 8, true, 3>(Jw, E, sms, s);
        };
        smooth_then_window(std::integral_constant<int, 4>{}, 2);
        tr.mark("smooth NW=4 (<=256)", s);
        smooth_then_window(std::integral_constant<int, 2>{}, 1);
        tr.mark("smooth NW=2 (<=128)", s);
        smooth_then_window(std::integral_constant<int, 1>{}, 0);
        tr.mark("smooth NW=1 (<=64)", s);
        return;
      }
    }
    launch_win<DIM, KIND, 4, 16, 16, true, 3>(L.J[2], E, sms, s);
    tr.mark("NW=4 (<=256)", s);
    // the small blocks are latency-bound: registers capped for 12 warps per SM (ncu: at
    // 208 registers / 8 warps the <= 64 class issues at IPC ~1.5, at 128 it spends 20% of
    // its instructions rematerialising addresses; 3 CTAs per SM is the measured optimum)
    launch_win<DIM, KIND, 2, 16, 16, true, 3>(L.J[1], E, sms, s);
    tr.mark("NW=2 (<=128)", s);
    launch_win<DIM, KIND, 1, 16, 8, true, 3>(L.J[0], E, sms, s);
    tr.mark("NW=1 (<=64)", s);
  } else {
    launch_win<DIM, KIND, 16, 32, 16, false>(L.J[4], E, sms, s);
    launch_win<DIM, KIND, 8, 32, 32, false>(L.J[3], E, sms, s);
    launch_win<DIM, KIND, 4, 32, 32, false>(L.J[2], E, sms, s);
    launch_win<DIM, KIND, 2, 32, 16, true>(L.J[1], E, sms, s);
    launch_win<DIM, KIND, 1, 32, 16, true>(L.J[0], E, sms, s);
  }
}

void HM_CAT(aca_classes_d, HM_ACA_DIM)(const AcaClassLaunch& L, cudaStream_t s) {
  constexpr int DIM = HM_ACA_DIM;
  if (L.J[kAcaCta].njobs > 0) {
    // the CTA kernel runs first on the same stream: sharing SMs with the window kernels
    // starves their 1-CTA/SM launches
    KernelEntry<DIM> E{L.coords, L.n, L.d, L.kp};
    launch_kernel_aca<DIM>(L.J[kAcaCta], E, L.sms, s);
    L.tr->mark("cta kernel", s);
  }
  if (L.kind == kGaussian) classes_kind<DIM, 0>(L, s);
  else classes_kind<DIM, 1>(L, s);
}

}  // namespace aca_detail
}  // namespace hmb
