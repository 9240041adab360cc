// fm_api.cu -- the extern "C" boundary declared in include/fastmnmf.h.
#include <cstdarg>
#include <mutex>

#include "fm_impl.cuh"

extern template struct fm::Impl<float>;
extern template struct fm::Impl<double>;

namespace fm {

static thread_local char g_err[512] = "";


void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int validate_dims(const fm_dims* d) {
  if (!d) { set_error("null dims"); return FM_EINVAL; }
  if (d->dtype != FM_F32 && d->dtype != FM_F64) { set_error("dtype %d", d->dtype); return FM_EINVAL; }
  if (d->B < 1 || d->F < 1 || d->T < 1) { set_error("empty problem B=%lld F=%lld T=%lld", (long long)d->B, (long long)d->F, (long long)d->T); return FM_EINVAL; }
  if (d->M < 1 || d->M > 16) { set_error("M=%lld outside 1..16", (long long)d->M); return FM_EINVAL; }
  if (d->N < 1 || d->N > NMAX) { set_error("N=%lld outside 1..%d", (long long)d->N, NMAX); return FM_EINVAL; }
  if (d->K < 1 || d->K > 64) { set_error("K=%lld outside 1..64", (long long)d->K); return FM_EINVAL; }
  if (d->ip_sweeps < 1) { set_error("ip_sweeps must be >= 1"); return FM_EINVAL; }
  if (d->F > 65535 || d->B > 65535) { set_error("F and B must be <= 65535"); return FM_EINVAL; }
  return FM_OK;
}

static int check_m(int64_t M) {
  if (M < 1 || M > 16) { set_error("M=%lld outside 1..16", (long long)M); return FM_EINVAL; }
  return FM_OK;
}

// Cached CUDA graphs of one full iteration (launch-bound configs), keyed by
// the device, the kernel selection (variant_key: V kernel, segment knob) and
// the exact (dims, state[, dp]) they were captured for. One capture stream
// per device. A small LRU keeps a few problems alive at once.
struct GraphEntry {
  int dev = -1;
  unsigned long long variant = 0;
  int unroll = 1;  // iterations captured in the graph
  bool dp = false;
  fm_dims d;
  fm_state s;
  fm_dp p;
  cudaGraphExec_t exec = nullptr;
  unsigned long long used = 0;
};
constexpr int GRAPH_SLOTS = 12, MAX_DEV = 64;
static GraphEntry g_graphs[GRAPH_SLOTS];
static cudaStream_t g_cap[MAX_DEV];
static unsigned long long g_tick = 0;
static std::mutex g_graph_mu;

}  // namespace fm

using namespace fm;

#define FM_BY_DTYPE(dt, CALL)                                      \
  ((dt) == FM_F64 ? Impl<double>::CALL : ((dt) == FM_F32 ? Impl<float>::CALL \
   : (set_error("dtype %d", (int)(dt)), FM_EINVAL)))

extern "C" {

int64_t fm_stft_frames(int64_t n_samples, int64_t window_length, int64_t hop) {
  if (window_length < 2 || hop < 1 || n_samples < window_length) return 0;
  return stft_frames(n_samples, window_length, hop);
}

int fm_stft(int dtype, int64_t n_samples, int64_t M, int64_t window_length, int64_t hop,
            const void* wave, void* spec, void* stream) {
  return FM_BY_DTYPE(dtype, stft(n_samples, M, window_length, hop, wave, spec, (cudaStream_t)stream));
}

size_t fm_istft_workspace_bytes(int dtype, int64_t n_frames, int64_t M, int64_t window_length) {
  const size_t rs = dtype == FM_F64 ? 8 : 4;
  return (size_t)std::max<int64_t>(n_frames, 1) * (size_t)std::max<int64_t>(M, 1) *
         (size_t)std::max<int64_t>(window_length, 1) * rs;
}

int fm_istft(int dtype, int64_t n_frames, int64_t M, int64_t window_length, int64_t hop,
             int64_t length, const void* spec, void* work, void* out, void* stream) {
  return FM_BY_DTYPE(dtype, istft(n_frames, M, window_length, hop, length, spec, work, out,
                                  (cudaStream_t)stream));
}

size_t fm_fullrank_workspace_bytes(int dtype, int64_t F, int64_t T, int64_t M) {
  return fr_workspace(dtype == FM_F64 ? 8 : 4, F, T, M);
}

int fm_fullrank_stats(int dtype, int64_t F, int64_t T, int64_t M, int64_t N, const void* X,
                      const void* G, const void* lam, double ridge, int want_ab, int want_phi,
                      void* phi, void* A, void* B, void* work, double* loglik, void* stream) {
  return FM_BY_DTYPE(dtype, fr_stats(F, T, M, N, X, G, lam, ridge, want_ab, want_phi, phi, A, B, work,
                                     loglik, (cudaStream_t)stream));
}

int fm_update_scm(int dtype, int64_t N, int64_t F, int64_t M, void* G, const void* A, const void* B,
                  int normalize, void* c, uint64_t* status, void* stream) {
  return FM_BY_DTYPE(dtype, fr_scm(N, F, M, G, A, B, normalize, c, status, (cudaStream_t)stream));
}

int fm_wiener_fullrank(int dtype, int64_t N, int64_t F, int64_t T, int64_t M, const void* lam,
                       const void* G, const void* X, double ridge, void* images, uint64_t* status,
                       void* stream) {
  return FM_BY_DTYPE(dtype, fr_wiener(N, F, T, M, lam, G, X, ridge, images, status,
                                      (cudaStream_t)stream));
}

int fm_nmf_mu(int dtype, int64_t N, int64_t F, int64_t T, int64_t K, const void* phi, void* W, void* H,
              int step, void* stream) {
  return FM_BY_DTYPE(dtype, fr_nmf_mu(N, F, T, K, phi, W, H, step, (cudaStream_t)stream));
}

int fm_nmf_absorb(int dtype, int64_t N, int64_t F, int64_t K, void* W, const void* c, void* stream) {
  return FM_BY_DTYPE(dtype, fr_absorb(N, F, K, W, c, (cudaStream_t)stream));
}

int fm_reconstruct_scm(int dtype, int64_t N, int64_t F, int64_t M, const void* Q, const void* g,
                       void* G, uint64_t* status, void* stream) {
  return FM_BY_DTYPE(dtype, fr_reconstruct(N, F, M, Q, g, G, status, (cudaStream_t)stream));
}

const char* fm_last_error(void) { return g_err; }
int fm_version(void) { return 1; }


int fm_fast_stats(int dtype, int64_t F, int64_t T, int64_t M, int64_t N, const void* xt,
                  const void* g, const void* lam, double floor, int want_gain, int want_phi,
                  void* phi1, void* phi2, void* gnum, void* gden, double* loglik_host,
                  void* stream) {
  if (int rc = check_m(M)) return rc;
  return FM_BY_DTYPE(dtype, fast_stats(F, T, M, N, xt, g, lam, floor, want_gain, want_phi, phi1,
                                       phi2, gnum, gden, loglik_host, (cudaStream_t)stream));
}

int fm_mix_power(int dtype, int64_t N, int64_t F, int64_t T, int64_t M, const void* lam,
                 const void* g, double floor, void* y, void* stream) {
  return FM_BY_DTYPE(dtype, mix_power(N, F, T, M, lam, g, floor, y, (cudaStream_t)stream));
}

int fm_ip_weights(int dtype, int64_t F, int64_t T, int64_t M, const void* X, const void* y,
                  void* V, void* stream) {
  if (int rc = check_m(M)) return rc;
  return FM_BY_DTYPE(dtype, ip_weights(F, T, M, X, y, V, (cudaStream_t)stream));
}

int fm_project_power(int dtype, int64_t F, int64_t T, int64_t M, const void* Q, const void* X,
                     void* xt, void* stream) {
  if (int rc = check_m(M)) return rc;
  return FM_BY_DTYPE(dtype, project(F, T, M, Q, X, xt, (cudaStream_t)stream));
}

int fm_update_diagonalizer(int dtype, int64_t F, int64_t T, int64_t M, void* Q, const void* X,
                           const void* y, int sweeps, uint64_t* status, void* stream) {
  if (int rc = check_m(M)) return rc;
  return FM_BY_DTYPE(dtype, update_diagonalizer(F, T, M, Q, X, y, sweeps, status,
                                                (cudaStream_t)stream));
}

int fm_logdet(int dtype, int64_t F, int64_t M, const void* Q, double* logdet, void* stream) {
  if (int rc = check_m(M)) return rc;
  return FM_BY_DTYPE(dtype, logdet(F, M, Q, logdet, (cudaStream_t)stream));
}

int fm_wiener_fast(int dtype, int64_t N, int64_t F, int64_t T, int64_t M, const void* lam,
                   const void* Q, const void* g, const void* X, void* images, uint64_t* status,
                   void* stream) {
  if (int rc = check_m(M)) return rc;
  return FM_BY_DTYPE(dtype, wiener(N, F, T, M, lam, Q, g, X, images, status, (cudaStream_t)stream));
}

int fm_data_term(const fm_dims* d, const fm_state* s, double* out_host, void* stream) {
  if (int rc = validate_dims(d)) return rc;
  if (!s || !out_host) { set_error("null state or output"); return FM_EINVAL; }
  const Plan p = make_plan(d);
  // data-term partials per mixture: (F, ntile) from k_back (deep prior),
  // (nfb, bseg) from k_bpass
  const size_t per = (d->dp || !use_fused(d)) ? (size_t)d->F * p.ntile : (size_t)p.nfb * p.bseg;
  const size_t n = (size_t)d->B * per;
  std::vector<double> h(n);
  FM_CUDA(cudaMemcpyAsync(h.data(), reinterpret_cast<unsigned char*>(s->work) + p.off_llp,
                          n * sizeof(double), cudaMemcpyDeviceToHost, (cudaStream_t)stream));
  FM_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  for (int64_t b = 0; b < d->B; ++b) {  // fixed order: bins, then tiles
    double acc = 0.0;
    for (size_t e = 0; e < per; ++e) acc += h[(size_t)b * per + e];
    out_host[b] = acc;
  }
  return FM_OK;
}

size_t fm_workspace_bytes(const fm_dims* d) {
  if (validate_dims(d)) return 0;
  return make_plan(d).total;
}

int fm_nmf_lambda(const fm_dims* d, const void* W, const void* H, void* lam, void* stream) {
  if (int rc = validate_dims(d)) return rc;
  if (d->dtype == FM_F64)
    return Impl<double>::lambda(d, (const double*)W, (const double*)H, (double*)lam,
                                (cudaStream_t)stream);
  return Impl<float>::lambda(d, (const float*)W, (const float*)H, (float*)lam, (cudaStream_t)stream);
}

int fm_prologue(const fm_dims* d, const fm_state* s, void* stream) {
  if (int rc = validate_dims(d)) return rc;
  if (d->dp) { set_error("dims.dp set: use fm_prologue_dp"); return FM_EINVAL; }
  return FM_BY_DTYPE(d->dtype, prologue(d, s, (cudaStream_t)stream));
}

int fm_refresh(const fm_dims* d, const fm_state* s, void* stream) {
  if (int rc = validate_dims(d)) return rc;
  if (d->dp) { set_error("dims.dp set: use fm_prologue_dp"); return FM_EINVAL; }
  return FM_BY_DTYPE(d->dtype, prologue(d, s, (cudaStream_t)stream, false));
}

int fm_schedule(const fm_dims* d) {
  if (validate_dims(d)) return -1;
  return d->dp ? FM_SCHED_SPLIT : schedule_of(d);
}

int fm_iterate(const fm_dims* d, const fm_state* s, void* stream) {
  if (int rc = validate_dims(d)) return rc;
  if (d->dp) { set_error("dims.dp set: use fm_iterate_dp"); return FM_EINVAL; }
  return FM_BY_DTYPE(d->dtype, iterate_phase(d, s, 2, nullptr, (cudaStream_t)stream));
}

int fm_iterate_phase(const fm_dims* d, const fm_state* s, int phase, void* hstat, void* stream) {
  if (int rc = validate_dims(d)) return rc;
  if (phase != 0 && phase != 1) { set_error("phase must be 0 or 1"); return FM_EINVAL; }
  return FM_BY_DTYPE(d->dtype, iterate_phase(d, s, phase, hstat, (cudaStream_t)stream));
}

int fm_iterate_profiled(const fm_dims* d, const fm_state* s, float* ms_host, int* n_intervals,
                        void* stream) {
  // One iteration captured into a CUDA graph with external event-record
  // nodes between its launches, replayed once: the device ms of each launch
  // as it runs inside a graph replay (the production path), not as
  // separately synchronised eager launches (fastmnmf.h lists the order).
  if (int rc = validate_dims(d)) return rc;
  if (d->dp) { set_error("fm_iterate_profiled: plain FastMNMF only"); return FM_EINVAL; }
  cudaStream_t st = (cudaStream_t)stream;
  constexpr int NEV = 11;
  const int nint = use_bin(d) ? 3 : use_fused(d) ? 6 : 10;
  cudaEvent_t ev[NEV];
  for (int i = 0; i < NEV; ++i) FM_CUDA(cudaEventCreate(&ev[i]));
  cudaStream_t cap = nullptr;
  FM_CUDA(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  int rc = FM_OK;
  FM_CUDA(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
  rc = d->dtype == FM_F64 ? Impl<double>::iterate_phase(d, s, 2, nullptr, cap, ev)
                          : Impl<float>::iterate_phase(d, s, 2, nullptr, cap, ev);
  cudaError_t ce = cudaStreamEndCapture(cap, &graph);
  if (rc == FM_OK && ce != cudaSuccess) {
    set_error("profiled capture: %s", cudaGetErrorString(ce));
    rc = FM_ECUDA;
  }
  if (rc == FM_OK && cudaGraphInstantiate(&exec, graph, 0) != cudaSuccess) {
    set_error("profiled instantiate failed");
    rc = FM_ECUDA;
  }
  if (rc == FM_OK) {
    FM_CUDA(cudaGraphLaunch(exec, st));
    FM_CUDA(cudaStreamSynchronize(st));
    for (int i = 0; i < nint; ++i) FM_CUDA(cudaEventElapsedTime(&ms_host[i], ev[i], ev[i + 1]));
    if (n_intervals) *n_intervals = nint;
  }
  if (exec) cudaGraphExecDestroy(exec);
  if (graph) cudaGraphDestroy(graph);
  cudaStreamDestroy(cap);
  for (int i = 0; i < NEV; ++i) cudaEventDestroy(ev[i]);
  return rc;
}

static int validate_dp(const fm_dims* d, const fm_dp* p) {
  if (!p) { set_error("null fm_dp"); return FM_EINVAL; }
  if (!d->dp) { set_error("fm_dims.dp must be 1 for the deep-prior entry points"); return FM_EINVAL; }
  if (d->N < 2) { set_error("deep-prior methods need n_sources >= 2"); return FM_EINVAL; }
  if (p->D < 1 || p->Hd < 1 || p->D > DEC_DMAX || p->Hd > DEC_HMAX) {
    set_error("decoder sizes D=%lld Hd=%lld outside 1..%d / 1..%d", (long long)p->D, (long long)p->Hd,
              DEC_DMAX, DEC_HMAX);
    return FM_EINVAL;
  }
  if (p->decoder_kind != FM_DEC_EXP_MLP && p->decoder_kind != FM_DEC_TOY) {
    set_error("unknown decoder_kind %d", (int)p->decoder_kind);
    return FM_EINVAL;
  }
  if (p->decoder_kind == FM_DEC_TOY && p->adam_steps > 0 && p->mh_steps <= 0) {
    set_error("the Adam latent update needs the exp-MLP decoder (decoder_kind 0)");
    return FM_EINVAL;
  }
  if (p->mh_steps < 0 || (p->mh_steps > 0 && !(p->mh_std > 0.0))) {
    set_error("Metropolis needs mh_steps >= 0 and a positive proposal std");
    return FM_EINVAL;
  }
  if ((p->mh_noise == nullptr) != (p->mh_unif == nullptr)) {
    set_error("mh_noise and mh_unif must both be set (caller draws) or both NULL (Philox)");
    return FM_EINVAL;
  }
  if (p->decoder_kind == FM_DEC_EXP_MLP && (p->D % 4 || p->Hd % 4)) {
    set_error("decoder sizes D=%lld Hd=%lld must be multiples of 4", (long long)p->D, (long long)p->Hd);
    return FM_EINVAL;
  }
  const void* wp[] = {p->W1, p->W2, p->W3};
  for (const void* q : wp)
    if (reinterpret_cast<uintptr_t>(q) % 16) {
      set_error("decoder weights must be 16-byte aligned");
      return FM_EINVAL;
    }
  return FM_OK;
}

size_t fm_dp_workspace_bytes(const fm_dims* d, const fm_dp* p) {
  if (validate_dims(d) || !p) return 0;
  // the output-layer weights transposed (Hd, F) for coalesced streaming in the
  // Metropolis kernel (written by fm_prologue_dp); the Adam kernel keeps its
  // state on chip
  const size_t rs = d->dtype == FM_F64 ? 8 : 4;
  return 256 + (((size_t)p->Hd * (size_t)d->F * rs + 255) & ~(size_t)255);
}

int fm_prologue_dp(const fm_dims* d, const fm_state* s, const fm_dp* p, void* stream) {
  if (int rc = validate_dims(d)) return rc;
  if (int rc = validate_dp(d, p)) return rc;
  return FM_BY_DTYPE(d->dtype, prologue_dp(d, s, p, (cudaStream_t)stream));
}

int fm_iterate_dp(const fm_dims* d, const fm_state* s, const fm_dp* p, void* stream) {
  if (int rc = validate_dims(d)) return rc;
  if (int rc = validate_dp(d, p)) return rc;
  return FM_BY_DTYPE(d->dtype, iterate_dp(d, s, p, (cudaStream_t)stream));
}

static int dp_profiled(const fm_dims* d, const fm_state* s, const fm_dp* p, float* ms_host,
                       int* n_out, cudaStream_t st) {
  constexpr int NEV = 24;
  cudaEvent_t ev[NEV];
  for (int i = 0; i < NEV; ++i) FM_CUDA(cudaEventCreate(&ev[i]));
  cudaStream_t cap = nullptr;
  FM_CUDA(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  FM_CUDA(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
  int rc = d->dtype == FM_F64 ? Impl<double>::iterate_dp(d, s, p, cap, ev)
                              : Impl<float>::iterate_dp(d, s, p, cap, ev);
  cudaError_t ce = cudaStreamEndCapture(cap, &graph);
  if (rc == FM_OK && ce != cudaSuccess) {
    set_error("profiled capture: %s", cudaGetErrorString(ce));
    rc = FM_ECUDA;
  }
  if (rc == FM_OK && cudaGraphInstantiate(&exec, graph, 0) != cudaSuccess) {
    set_error("profiled instantiate failed");
    rc = FM_ECUDA;
  }
  int nint = 0;
  if (rc == FM_OK) {
    FM_CUDA(cudaGraphLaunch(exec, st));
    FM_CUDA(cudaStreamSynchronize(st));
    const int nlaunch = 19 + ((p->mh_steps > 0 || p->adam_steps > 0) ? 2 : 0);
    for (int i = 0; i < nlaunch; ++i) FM_CUDA(cudaEventElapsedTime(&ms_host[i], ev[i], ev[i + 1]));
    nint = nlaunch;
  }
  if (exec) cudaGraphExecDestroy(exec);
  if (graph) cudaGraphDestroy(graph);
  cudaStreamDestroy(cap);
  for (int i = 0; i < NEV; ++i) cudaEventDestroy(ev[i]);
  *n_out = nint;
  return rc;
}

int fm_iterate_dp_profiled(const fm_dims* d, const fm_state* s, const fm_dp* p, float* ms_host,
                           int* n_intervals, void* stream) {
  if (int rc = validate_dims(d)) return rc;
  if (int rc = validate_dp(d, p)) return rc;
  if (!ms_host || !n_intervals) { set_error("null output"); return FM_EINVAL; }
  return dp_profiled(d, s, p, ms_host, n_intervals, (cudaStream_t)stream);
}

// Iterations captured per graph: 1 unless FM_UNROLL says otherwise (read at
// every run). Measured at config 1 (B200): unrolling 2 / 5 / 10 / 25
// iterations into one graph gives 7178 / 7116 / 7091 / 7080 iterations/s
// against 7295 for single-iteration graphs -- the graph boundary costs
// nothing, and the programmatic edge from an iteration's k_trace into the next
// k_wstats only delays that kernel's CTAs.
static int graph_unroll(const fm_dims* d, int n_iterations) {
  int u = 1;
  (void)d;
  if (const char* e = getenv("FM_UNROLL")) {
    const int v = atoi(e);
    if (v >= 1 && v <= 64) u = v;
  }
  return std::max(1, std::min(u, n_iterations));
}

// The cached graph of `unroll` consecutive iterations (captured on a miss).
static int graph_for(const fm_dims* d, const fm_state* s, const fm_dp* p, int unroll, int dev,
                     unsigned long long variant, cudaGraphExec_t* out) {
  auto one = [&](void* strm) { return p ? fm_iterate_dp(d, s, p, strm) : fm_iterate(d, s, strm); };
  GraphEntry* hit = nullptr;
  for (auto& e : g_graphs) {
    if (e.exec && e.dev == dev && e.variant == variant && e.unroll == unroll && e.dp == (p != nullptr) &&
        std::memcmp(&e.d, d, sizeof(fm_dims)) == 0 && std::memcmp(&e.s, s, sizeof(fm_state)) == 0 &&
        (!p || std::memcmp(&e.p, p, sizeof(fm_dp)) == 0)) {
      hit = &e;
      break;
    }
  }
  if (!hit) {
    hit = &g_graphs[0];  // empty slot, else the least recently used
    for (auto& e : g_graphs) {
      if (!e.exec) { hit = &e; break; }
      if (e.used < hit->used) hit = &e;
    }
    if (hit->exec) { cudaGraphExecDestroy(hit->exec); hit->exec = nullptr; }
    if (!g_cap[dev]) FM_CUDA(cudaStreamCreateWithFlags(&g_cap[dev], cudaStreamNonBlocking));
    cudaGraph_t graph = nullptr;
    FM_CUDA(cudaStreamBeginCapture(g_cap[dev], cudaStreamCaptureModeThreadLocal));
    int rc = FM_OK;
    for (int u = 0; u < unroll && rc == FM_OK; ++u) rc = one((void*)g_cap[dev]);
    cudaError_t ce = cudaStreamEndCapture(g_cap[dev], &graph);
    if (rc) { if (graph) cudaGraphDestroy(graph); return rc; }
    if (ce != cudaSuccess) { set_error("graph capture: %s", cudaGetErrorString(ce)); return FM_ECUDA; }
    ce = cudaGraphInstantiate(&hit->exec, graph, 0);
    cudaGraphDestroy(graph);
    if (ce != cudaSuccess) {
      hit->exec = nullptr;
      set_error("graph instantiate: %s", cudaGetErrorString(ce));
      return FM_ECUDA;
    }
    hit->dev = dev;
    hit->variant = variant;
    hit->unroll = unroll;
    hit->dp = p != nullptr;
    hit->d = *d;
    hit->s = *s;
    if (p) hit->p = *p;
  }
  hit->used = ++g_tick;
  *out = hit->exec;
  return FM_OK;
}

// n iterations, optionally replayed from captured CUDA graphs (graph_unroll
// iterations each, single-iteration graphs for the remainder).
static int run_common(const fm_dims* d, const fm_state* s, const fm_dp* p, int n_iterations,
                      int use_graph, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (!use_graph) {
    for (int i = 0; i < n_iterations; ++i)
      if (int rc = p ? fm_iterate_dp(d, s, p, stream) : fm_iterate(d, s, stream)) return rc;
    return FM_OK;
  }
  if (n_iterations <= 0) return FM_OK;
  int dev = 0;
  FM_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= MAX_DEV) { set_error("device %d", dev); return FM_EINVAL; }
  const unsigned long long variant = variant_key(d);
  const int U = graph_unroll(d, n_iterations);
  std::lock_guard<std::mutex> lk(g_graph_mu);
  cudaGraphExec_t ex = nullptr;
  int left = n_iterations;
  if (U > 1) {
    if (int rc = graph_for(d, s, p, U, dev, variant, &ex)) return rc;
    for (; left >= U; left -= U) FM_CUDA(cudaGraphLaunch(ex, st));
  }
  if (left > 0) {
    if (int rc = graph_for(d, s, p, 1, dev, variant, &ex)) return rc;
    for (; left > 0; --left) FM_CUDA(cudaGraphLaunch(ex, st));
  }
  return FM_OK;
}

int fm_run(const fm_dims* d, const fm_state* s, int n_iterations, int use_graph, void* stream) {
  if (int rc = validate_dims(d)) return rc;
  return run_common(d, s, nullptr, n_iterations, use_graph, stream);
}

int fm_run_dp(const fm_dims* d, const fm_state* s, const fm_dp* p, int n_iterations, int use_graph,
              void* stream) {
  if (int rc = validate_dims(d)) return rc;
  if (int rc = validate_dp(d, p)) return rc;
  return run_common(d, s, p, n_iterations, use_graph, stream);
}

int fm_observation_stats(const fm_dims* d, const void* X, double* sumsq_host, double* maxsq_host,
                         void* stream) {
  if (int rc = validate_dims(d)) return rc;
  return FM_BY_DTYPE(d->dtype, obs_stats(d, X, sumsq_host, maxsq_host, (cudaStream_t)stream));
}

int fm_scale_observation(const fm_dims* d, void* X, const double* scale_host, void* stream) {
  if (int rc = validate_dims(d)) return rc;
  return FM_BY_DTYPE(d->dtype, scale(d, X, scale_host, (cudaStream_t)stream));
}

int fm_spatial_init(const fm_dims* d, const void* X, void* Q, double* w, void* stream) {
  if (!d) { set_error("null dims"); return FM_EINVAL; }
  if (d->dtype != FM_F32 && d->dtype != FM_F64) { set_error("dtype %d", d->dtype); return FM_EINVAL; }
  if (d->B < 1 || d->F < 1 || d->T < 1) { set_error("empty problem"); return FM_EINVAL; }
  if (d->F > 65535 || d->B > 65535) { set_error("F and B must be <= 65535"); return FM_EINVAL; }
  if (int rc = check_m(d->M)) return rc;
  if (!X || !Q) { set_error("null X or Q"); return FM_EINVAL; }
  return FM_BY_DTYPE(d->dtype, spatial_init(d, X, Q, w, (cudaStream_t)stream));
}

}  // extern "C"
