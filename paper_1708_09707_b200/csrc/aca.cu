// aca.cu -- K7 host side: factorisation schedule (plan_aca_chunk), the per-chunk launch
// sequence (compute_aca) and the explicit-matrix seam.  Kernels: aca_impl.cuh,
// instantiated per point dimension by aca_dim.cu.
#include "aca_impl.cuh"

#include <mutex>

namespace hmb {
using namespace aca_detail;

namespace {

__global__ void class_key_kernel(const int* __restrict__ m, const int* __restrict__ nn, long long begin, long long cnt,
                                 int kmax, int has_eps, int clusters, unsigned long long* __restrict__ keys,
                                 unsigned* __restrict__ vals) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < cnt;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long b = begin + i;
    const int cls = aca_class(m[b], nn[b], kmax, has_eps != 0, clusters != 0);
    keys[i] = (static_cast<unsigned long long>(cls) << 32) | static_cast<unsigned long long>(0x7fffffff - nn[b]);
    vals[i] = static_cast<unsigned>(b);
  }
}

__global__ void size_key_kernel(const int* __restrict__ m, const int* __restrict__ nn, const int* __restrict__ cl,
                                long long begin, long long cnt, unsigned long long* __restrict__ keys,
                                unsigned* __restrict__ vals) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < cnt;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long b = begin + i;
    // long leaves (n >= 4096, whose folds are the critical path) first, largest first;
    // the rest in leaf order, i.e. V in address order (a sequential HBM stream)
    const unsigned long long big = nn[b] >= 4096 ? static_cast<unsigned long long>(nn[b]) : 0ull;
    keys[i] = ((~big & 0xffffffffull) << 32) | static_cast<unsigned long long>(b - begin);
    vals[i] = static_cast<unsigned>(b);
  }
}

// All chunks' schedules at once: per own leaf b (chunk c = upper_bound(starts, b) - 1) the
// fold-order key (chunk | long-leaves-first | position) and the class key (chunk | class |
// largest n first), plus the per-chunk class histogram and largest big-class m.
__global__ void chunk_keys_kernel(const int* __restrict__ m, const int* __restrict__ nn, long long lo, long long cnt,
                                  const long long* __restrict__ starts, int nchunks, int kmax, int has_eps,
                                  int clusters, unsigned long long* __restrict__ okeys, unsigned* __restrict__ ovals,
                                  unsigned long long* __restrict__ ckeys, unsigned* __restrict__ cvals,
                                  unsigned long long* __restrict__ hist, int* __restrict__ maxrows) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < cnt;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long b = lo + i;
    int a = 0, z = nchunks;  // starts[a] <= b < starts[z]
    while (z - a > 1) {
      const int mid = (a + z) >> 1;
      if (starts[mid] <= b) a = mid;
      else z = mid;
    }
    const unsigned long long c = static_cast<unsigned long long>(a);
    const int mb = m[b], nb = nn[b];
    const unsigned long long big = nb >= 4096 ? static_cast<unsigned long long>(nb) : 0ull;
    okeys[i] = (c << 54) | (((0x7ffffffull - big) & 0x7ffffffull) << 27) | static_cast<unsigned long long>(b - starts[a]);
    ovals[i] = static_cast<unsigned>(b);
    const int cls = aca_class(mb, nb, kmax, has_eps != 0, clusters != 0);
    ckeys[i] = (c << 31) | (static_cast<unsigned long long>(cls) << 27) | static_cast<unsigned long long>(0x7ffffff - nb);
    cvals[i] = static_cast<unsigned>(b);
    atomicAdd(hist + c * kAcaClasses + cls, 1ull);
    if (cls == kAcaBig) atomicMax(maxrows + c, mb);
  }
}

}  // namespace

// epsilon criterion (aca.cpp:497-538) is live only for eta <= 1: the bound is
// eps (1 - eta) / (1 + eps) * ||A_r||_F, negative for eta > 1, while ||u_r|| ||v_r|| >= 0
// (u_r[p] = 1), so the stop test can never fire -- such blocks run on the
// fast size-class kernels with identical results.
static bool eps_live(const HMatrix& h) {
  if (!h.cfg.has_epsilon) return false;
  const double f = h.cfg.epsilon * (1.0 - h.cfg.eta) / (1.0 + h.cfg.epsilon);
  return !(f < 0.0);
}

// One pass for every chunk (setup time): two radix sorts over all own leaves instead of two
// per chunk.  Same orders as plan_aca_chunk (stable sorts: ties keep leaf order).
bool plan_aca_chunks_all(HMatrix& h, long long lo, long long hi, cudaStream_t s) {
  const long long cnt = hi - lo;
  const int nch = static_cast<int>(h.chunks.size());
  if (cnt <= 0 || nch == 0 || nch > 1000 || cnt >= (1ll << 27) || h.n >= (1ll << 27)) return false;
  if (h.cfg.k > kKmax) raise(kEinval, "k > 64 is not supported by the device ACA");
  const bool eps = eps_live(h);
  const bool clus = std::getenv("HM_NO_CLUSTER") == nullptr;
  std::vector<long long> starts(nch + 1);
  for (int c = 0; c < nch; ++c) starts[c] = h.chunks[c].c0;
  starts[nch] = h.chunks.back().c1;
  DevBuf<long long> dstarts;
  DevBuf<unsigned long long> okeys, ckeys, hist;
  DevBuf<int> maxrows;
  dstarts.alloc(nch + 1, s);
  okeys.alloc(cnt, s);
  ckeys.alloc(cnt, s);
  hist.alloc(static_cast<size_t>(nch) * kAcaClasses, s);
  maxrows.alloc(nch, s);
  hist.zero(s);
  maxrows.zero(s);
  HM_CUDA(cudaMemcpyAsync(dstarts.get(), starts.data(), sizeof(long long) * (nch + 1), cudaMemcpyHostToDevice, s));
  unsigned* order = reinterpret_cast<unsigned*>(h.sched_order.get());
  unsigned* jobs = reinterpret_cast<unsigned*>(h.sched_jobs.get());
  chunk_keys_kernel<<<grid_for(cnt, 256, 1 << 16), 256, 0, s>>>(h.aca.m.get(), h.aca.n.get(), lo, cnt, dstarts.get(),
                                                                 nch, static_cast<int>(h.cfg.k), eps ? 1 : 0,
                                                                 clus ? 1 : 0, okeys.get(), order, ckeys.get(), jobs,
                                                                 hist.get(), maxrows.get());
  HM_LAUNCH_CHECK();
  radix_sort_pairs(okeys.get(), order, cnt, s);
  radix_sort_pairs(ckeys.get(), jobs, cnt, s);
  std::vector<unsigned long long> hh(static_cast<size_t>(nch) * kAcaClasses);
  std::vector<int> hm(nch);
  HM_CUDA(cudaMemcpyAsync(hh.data(), hist.get(), sizeof(unsigned long long) * hh.size(), cudaMemcpyDeviceToHost, s));
  HM_CUDA(cudaMemcpyAsync(hm.data(), maxrows.get(), sizeof(int) * nch, cudaMemcpyDeviceToHost, s));
  HM_CUDA(cudaStreamSynchronize(s));
  for (int c = 0; c < nch; ++c) {
    AcaChunk& ch = h.chunks[c];
    for (int q = 0; q < kAcaClasses; ++q) ch.ccount[q] = static_cast<long long>(hh[static_cast<size_t>(c) * kAcaClasses + q]);
    ch.max_rows_big = hm[c];
  }
  return true;
}

void reset_aca_rejections(HMatrix& h, cudaStream_t s) {
  if (h.aca_rej.size() < 2) h.aca_rej.alloc(2, s);
  h.aca_rej.zero(s);
}

// Schedule of aca leaves [c.c0, c.c1): the long-leaves-first order of the V^T x fold and
// the per-class job lists (largest n first within a class), both sorted once here.
void plan_aca_chunk(HMatrix& h, AcaChunk& c, cudaStream_t s) {
  const long long cnt = c.c1 - c.c0;
  for (int q = 0; q < kAcaClasses; ++q) c.ccount[q] = 0;
  c.max_rows_big = 0;
  if (cnt <= 0) return;
  if (h.cfg.k > kKmax) raise(kEinval, "k > 64 is not supported by the device ACA");
  if (h.sched_jobs.size() < static_cast<size_t>(c.sched_off + cnt))
    raise(kElogic, "plan_aca_chunk: schedule buffer too small");
  const bool eps = eps_live(h);
  const bool clus = std::getenv("HM_NO_CLUSTER") == nullptr;
  {
    std::mutex mu;
    parallel_blocks(c.c1 - c.c0, [&](long long b0, long long b1) {
      long long cc[kAcaClasses] = {};
      int mr = 0;
      for (long long b = c.c0 + b0; b < c.c0 + b1; ++b) {
        const int q = aca_class(h.aca.h_m[b], h.aca.h_n[b], h.cfg.k, eps, clus);
        ++cc[q];
        if (q == kAcaBig) mr = std::max(mr, h.aca.h_m[b]);
      }
      std::lock_guard<std::mutex> lk(mu);
      for (int q = 0; q < kAcaClasses; ++q) c.ccount[q] += cc[q];
      c.max_rows_big = std::max(c.max_rows_big, mr);
    });
  }
  DevBuf<unsigned long long> keys;
  keys.alloc(cnt, s);
  unsigned* order = reinterpret_cast<unsigned*>(h.sched_order.get() + c.sched_off);
  unsigned* jobs = reinterpret_cast<unsigned*>(h.sched_jobs.get() + c.sched_off);
  size_key_kernel<<<grid_for(cnt, 256, 1 << 16), 256, 0, s>>>(h.aca.m.get(), h.aca.n.get(), h.aca.cl.get(), c.c0, cnt,
                                                               keys.get(), order);
  HM_LAUNCH_CHECK();
  radix_sort_pairs(keys.get(), order, cnt, s);
  class_key_kernel<<<grid_for(cnt, 256, 1 << 16), 256, 0, s>>>(h.aca.m.get(), h.aca.n.get(), c.c0, cnt,
                                                                static_cast<int>(h.cfg.k), eps ? 1 : 0, clus ? 1 : 0,
                                                                keys.get(), jobs);
  HM_LAUNCH_CHECK();
  radix_sort_pairs(keys.get(), jobs, cnt, s);
}

// Factorises the planned chunk c into h.U / h.V at offsets h.u_off[b] - c.ub (so a chunk
// workspace can be reused).  Stream-ordered only: no host synchronisation.
void compute_aca(HMatrix& h, const AcaChunk& c, cudaStream_t s) {
  const long long cnt = c.c1 - c.c0;
  if (cnt <= 0) return;
  PhaseTrace tr;
  tr.mark("start", s);
  // [0, K) job counters, [K, 2K) fallback counts, [2K, 3K) fallback job counters
  if (h.aca_counters.size() < static_cast<size_t>(3 * kAcaClasses)) h.aca_counters.alloc(3 * kAcaClasses, s);
  h.aca_counters.zero(s);
  if (h.aca_fallback.size() < static_cast<size_t>(cnt)) h.aca_fallback.alloc(cnt, s);
  if (h.aca_rej.size() < 2) reset_aca_rejections(h, s);
  AcaJob J{};
  J.rl = h.aca.rl.get();
  J.m = h.aca.m.get();
  J.cl = h.aca.cl.get();
  J.nn = h.aca.n.get();
  J.order = nullptr;
  J.njobs = cnt;
  J.u_off = h.u_off.get();
  J.v_off = h.v_off.get();
  J.u_base = c.ub;
  J.v_base = c.vb;
  J.U = h.U.get();
  J.V = h.V.get();
  J.k_eff = h.k_eff.get();
  J.row_piv = h.row_piv.get();
  J.col_piv = h.col_piv.get();
  J.kmax = static_cast<int>(h.cfg.k);
  J.has_eps = eps_live(h) ? 1 : 0;
  J.eps_factor = h.cfg.epsilon * (1.0 - h.cfg.eta) / (1.0 + h.cfg.epsilon);
  J.rejections = h.aca_rej.get();
  J.evals = nullptr;
  J.tile_shift = h.u_tile_shift;
  {
    // window kernels: one fresh column per rank until a rejection, d >= 3 (HM_WIN_ONE=0/1)
    const char* ew = std::getenv("HM_WIN_ONE");
    J.win_one = (ew ? std::atoi(ew) != 0 : h.d >= 3) ? 1 : 0;
  }
  const int* jobs = h.sched_jobs.get() + c.sched_off;
  const long long* ccount = c.ccount;
  int sms = 0;
  HM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h.device));
  long long first[kAcaClasses + 1];
  first[0] = 0;
  for (int q = 0; q < kAcaClasses; ++q) first[q + 1] = first[q] + ccount[q];
  DevBuf<unsigned long long> evals;
  if (tr.on) {
    evals.alloc(3 * kAcaClasses, s);
    evals.zero(s);
  }
  auto sub = [&](int q) {
    AcaJob Jc = J;
    Jc.evals = tr.on ? evals.get() + 3 * q : nullptr;
    Jc.order = jobs + first[q];
    Jc.njobs = ccount[q];
    Jc.counter = h.aca_counters.get() + q;
    return Jc;
  };
  AcaClassLaunch L;
  for (int q = 0; q < kAcaClasses; ++q) L.J[q] = sub(q);
  L.sms = sms;
  L.max_rows_big = c.max_rows_big;
  L.kind = h.kp.kind;
  L.kp = h.kp;
  L.coords = h.coords.get();
  L.n = h.n;
  L.d = h.d;
  L.device = h.device;
  L.big_scratch = &h.aca_big_scratch;
  L.tr = &tr;
  // smooth-path kernels: by default for d >= 3 (no noise floor);
  // HM_SMOOTH=0/1 forces them off/on (results are bitwise identical either way)
  {
    const char* e = std::getenv("HM_SMOOTH");
    L.smooth = (e ? std::atoi(e) != 0 : h.d >= 3) && h.cfg.k == 16 && h.d <= 4;
    const char* ep = std::getenv("HM_SMOOTH_PRE");
    L.smooth_pre = ep ? std::atoi(ep) != 0 : false;
    const char* em = std::getenv("HM_SMOOTH_MID");
    L.smooth_mid = em ? std::atoi(em) != 0 : false;
    const char* eb = std::getenv("HM_BIG_ONE");
    L.big_one = eb ? std::atoi(eb) != 0 : h.d >= 3;
  }
  L.fb_list = h.aca_fallback.get();
  L.fb_count = h.aca_counters.get() + kAcaClasses;
  L.fb_counter = h.aca_counters.get() + 2 * kAcaClasses;
  for (int q = 0; q <= kAcaClasses; ++q) L.first[q] = first[q];
  // HM_ACA_2STREAM=1: cluster / big-block kernels on the auxiliary stream beside the window
  // kernels (tails overlap).  Measured at config 3: 5.80 s vs 5.70 s per product on one
  // stream (the co-resident kernels compete for the same SMs), so one stream by default.
  const bool two = std::getenv("HM_ACA_2STREAM") != nullptr && !tr.on && h.aux != nullptr;
  if (two) {
    HM_CUDA(cudaEventRecord(h.ev_fork, s));
    HM_CUDA(cudaStreamWaitEvent(h.aux, h.ev_fork, 0));
    L.s2 = h.aux;
  }
  switch (h.d) {
    case 1: aca_classes_d1(L, s); break;
    case 2: aca_classes_d2(L, s); break;
    case 3: aca_classes_d3(L, s); break;
    case 4: aca_classes_d4(L, s); break;
    default: aca_classes_d0(L, s); break;
  }
  if (two) {
    HM_CUDA(cudaEventRecord(h.ev_join, h.aux));
    HM_CUDA(cudaStreamWaitEvent(s, h.ev_join, 0));
  }
  if (tr.on) {
    std::fprintf(stderr, "[hm_trace] aca classes: %lld %lld %lld %lld %lld | cl4 %lld cl8 %lld big %lld cta %lld\n",
                 ccount[0], ccount[1], ccount[2], ccount[3], ccount[4], ccount[5], ccount[6], ccount[7], ccount[8]);
    tr.dump();
    unsigned long long ev[3 * kAcaClasses];
    HM_CUDA(cudaMemcpyAsync(ev, evals.get(), sizeof(ev), cudaMemcpyDeviceToHost, s));
    HM_CUDA(cudaStreamSynchronize(s));
    for (int q = 0; q < kAcaClasses; ++q)
      std::fprintf(stderr, "[hm_trace] class %d: blocks %llu col-entries %.4g row-entries %.4g\n", q, ev[3 * q + 2],
                   static_cast<double>(ev[3 * q]), static_cast<double>(ev[3 * q + 1]));
  }
}

// Explicit-matrix seam (aca.cpp:567-578): host blocks in, host factors out in the
// oracle's layout (u: kmax x m rank-major, v: kmax x n rank-major, zero padded).
void aca_dense_blocks(long long nb, const long long* shapes, const double* entries_host, long long kmax, bool has_eps,
                      double eps, double eta, long long* k_eff_out, long long* row_piv_out, long long* col_piv_out,
                      double* u_host, double* v_host, cudaStream_t s) {
  if (kmax < 1) raise(kEinval, "aca: max_rank must be >= 1");
  if (kmax > kKmax) raise(kEinval, "k > 64 is not supported by the device ACA");
  std::vector<int> hm(nb), hn(nb), hz(nb, 0), hord(nb);
  std::vector<long long> uoff(nb), voff(nb), doff(nb);
  long long su = 0, sv = 0, sd = 0;
  for (long long b = 0; b < nb; ++b) {
    hm[b] = static_cast<int>(shapes[2 * b]);
    hn[b] = static_cast<int>(shapes[2 * b + 1]);
    if (hm[b] < 1 || hn[b] < 1) raise(kEinval, "aca: empty block");
    uoff[b] = su;
    voff[b] = sv;
    doff[b] = sd;
    su += kmax * hm[b];
    sv += kmax * hn[b];
    sd += static_cast<long long>(hm[b]) * hn[b];
    hord[b] = static_cast<int>(b);
  }
  DevBuf<int> dm, dn, dz, dord, dk, drp, dcp, cnt;
  DevBuf<long long> duo, dvo, ddo;
  DevBuf<double> dA, dU, dV;
  auto up = [&](auto& buf, const auto& vec) {
    buf.alloc(vec.size(), s);
    HM_CUDA(cudaMemcpyAsync(buf.get(), vec.data(), vec.size() * sizeof(vec[0]), cudaMemcpyHostToDevice, s));
  };
  up(dm, hm);
  up(dn, hn);
  up(dz, hz);
  up(dord, hord);
  up(duo, uoff);
  up(dvo, voff);
  up(ddo, doff);
  dA.alloc(sd, s);
  HM_CUDA(cudaMemcpyAsync(dA.get(), entries_host, sizeof(double) * sd, cudaMemcpyHostToDevice, s));
  dU.alloc(su, s);
  dV.alloc(sv, s);
  dU.zero(s);
  dV.zero(s);
  dk.alloc(nb, s);
  drp.alloc(nb * kmax, s);
  dcp.alloc(nb * kmax, s);
  cnt.alloc(1, s);
  cnt.zero(s);
  AcaJob J{};
  J.rl = dz.get();
  J.m = dm.get();
  J.cl = dz.get();
  J.nn = dn.get();
  J.order = dord.get();
  J.njobs = nb;
  J.u_off = duo.get();
  J.v_off = dvo.get();
  J.U = dU.get();
  J.V = dV.get();
  J.k_eff = dk.get();
  J.row_piv = drp.get();
  J.col_piv = dcp.get();
  J.kmax = static_cast<int>(kmax);
  J.has_eps = has_eps ? 1 : 0;
  J.eps_factor = eps * (1.0 - eta) / (1.0 + eps);
  J.counter = cnt.get();
  J.tile_shift = -1;
  J.dense = dA.get();
  J.dense_off = ddo.get();
  KernelEntry<1> E{nullptr, 0, 1, KernelParams{0, 1, 0.0}};
  aca_kernel<1, true><<<static_cast<unsigned>(std::min<long long>(nb, 1024)), kAcaThreads, 0, s>>>(J, E);
  HM_LAUNCH_CHECK();
  std::vector<int> hk(nb), hrp(nb * kmax), hcp(nb * kmax);
  std::vector<double> hu(su), hv(sv);
  HM_CUDA(cudaMemcpyAsync(hk.data(), dk.get(), sizeof(int) * nb, cudaMemcpyDeviceToHost, s));
  HM_CUDA(cudaMemcpyAsync(hrp.data(), drp.get(), sizeof(int) * nb * kmax, cudaMemcpyDeviceToHost, s));
  HM_CUDA(cudaMemcpyAsync(hcp.data(), dcp.get(), sizeof(int) * nb * kmax, cudaMemcpyDeviceToHost, s));
  HM_CUDA(cudaMemcpyAsync(hu.data(), dU.get(), sizeof(double) * su, cudaMemcpyDeviceToHost, s));
  HM_CUDA(cudaMemcpyAsync(hv.data(), dV.get(), sizeof(double) * sv, cudaMemcpyDeviceToHost, s));
  HM_CUDA(cudaStreamSynchronize(s));
  for (long long b = 0; b < nb; ++b) {
    const long long m = hm[b], n = hn[b];
    k_eff_out[b] = hk[b];
    for (long long l = 0; l < kmax; ++l) {
      row_piv_out[b * kmax + l] = hrp[b * kmax + l];
      col_piv_out[b * kmax + l] = hcp[b * kmax + l];
      const bool live = l < hk[b];
      for (long long i = 0; i < m; ++i) u_host[uoff[b] + l * m + i] = live ? hu[uoff[b] + l * m + i] : 0.0;
      for (long long j = 0; j < n; ++j) v_host[voff[b] + l * n + j] = live ? hv[voff[b] + j * kmax + l] : 0.0;
    }
  }
}

}  // namespace hmb
