/*
 * fastmnmf.h -- C ABI of the B200-native FastMNMF update (libfastmnmf.so).
 *
 * Plain pointers and sizes only; every device pointer is a CUDA global-memory
 * address, every `stream` a cudaStream_t passed as void*. Arrays are dense,
 * row-major ("C order"), with the axis order of the reference's suffixed
 * names: X_FTM (F,T,M) complex, xt_FTM (F,T,M) real,
 * g_NFM (N,F,M), lam_NFT (N,F,T), W_NFK (N,F,K), H_NKT (N,K,T), Q_FMM (F,M,M)
 * complex with ROW m OF Q_f = q_fm^H, V_FMMM (F,M,M,M) complex. Complex
 * numbers are interleaved (re, im). The fused entry points carry a leading
 * batch axis B (independent mixtures; BASELINE config 2).
 *
 * dtype: FM_F32 = complex64/float32 storage and arithmetic (fp64 for the
 * log-likelihood accumulation and the M x M solves), FM_F64 =
 * complex128/float64 throughout (the reference's only precision).
 *
 * Reference seam replaced (paths relative to /root/reference/pkg/src/fastsep):
 * the reference has no C ABI; its operator seam is the Python module
 * _kernels.py (backend picked at import, _kernels.py:16-31). Each fm_* per-op
 * function below replaces one function of that seam (or of spatial.py /
 * separate.py that wraps it), cited on its declaration. The fused
 * fm_iterate* entry points replace one _DiagLoop.iterate call
 * (separate.py:201-234).
 *
 * Return value: 0 on success, otherwise an FM_E* code; fm_last_error() gives
 * a message. Numerical failures inside a kernel (the reference's
 * SingularMatrixError, spatial.py:189-198 / separate.py:121-124) are not
 * return codes: they are written to a device status word (see FM_STATUS_*)
 * that the host reads when it synchronises.
 */
#ifndef FASTMNMF_H
#define FASTMNMF_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FM_F32 0
#define FM_F64 1

#define FM_OK 0
#define FM_EINVAL 1     /* bad sizes / dtype / unsupported M (1..16 supported) */
#define FM_ECUDA 2      /* a CUDA launch or API call failed */

/* Device status word (uint64, initialise to FM_STATUS_CLEAR). Kernels
 * atomicMin an encoded key, so the first failure in (iteration, row m,
 * frequency f) order wins -- the one the reference would raise first. */
#define FM_STATUS_CLEAR 0xFFFFFFFFFFFFFFFFull
#define FM_STATUS_NONPOS_NORM 1 /* spatial.py:194-198 "non-positive normalization" */
#define FM_STATUS_SINGULAR_QV 2 /* spatial.py:189-192 zgesv LinAlgError */
#define FM_STATUS_SINGULAR_Q 3  /* separate.py:121-124 inv(Q) LinAlgError */
/* key = iteration<<44 | m<<24 | f<<2 | code  (f is the GLOBAL bin index). */

/* ---- per-op entry points (the _kernels.py seam) -------------------------- */

/* _kernels.fast_stats (_kernels.py:254-267; numba :208-251). Outputs that are
 * not wanted may be NULL. phi1/phi2 (N,F,T); gnum/gden (N,F,M); *loglik_host
 * receives the data term sum(-x~/y - log y) (synchronises the stream). */
int fm_fast_stats(int dtype, int64_t F, int64_t T, int64_t M, int64_t N,
                  const void* xt, const void* g, const void* lam, double floor,
                  int want_gain, int want_phi, void* phi1, void* phi2, void* gnum,
                  void* gden, double* loglik_host, void* stream);

/* _kernels.mix_power (_kernels.py:325-331): y = max(sum_n lam g, floor). */
int fm_mix_power(int dtype, int64_t N, int64_t F, int64_t T, int64_t M, const void* lam,
                 const void* g, double floor, void* y, void* stream);

/* _kernels.ip_weights (_kernels.py:296-302): V[f,m] = (1/T) sum_t x x^H / y. */
int fm_ip_weights(int dtype, int64_t F, int64_t T, int64_t M, const void* X, const void* y,
                  void* V, void* stream);

/* _kernels.project_power (_kernels.py:353-359): xt = |Q x|^2. */
int fm_project_power(int dtype, int64_t F, int64_t T, int64_t M, const void* Q,
                     const void* X, void* xt, void* stream);

/* spatial.update_diagonalizer (spatial.py:172-200), in place on Q.
 * status: device uint64 (see FM_STATUS_*; iteration field 0). */
int fm_update_diagonalizer(int dtype, int64_t F, int64_t T, int64_t M, void* Q,
                           const void* X, const void* y, int sweeps, uint64_t* status,
                           void* stream);

/* np.linalg.slogdet(Q)[1] per bin (spatial.py:241, separate.py:238): (F) fp64. */
int fm_logdet(int dtype, int64_t F, int64_t M, const void* Q, double* logdet, void* stream);

/* separate.wiener_fast (separate.py:110-125): images (N,F,T,M) complex. */
int fm_wiener_fast(int dtype, int64_t N, int64_t F, int64_t T, int64_t M, const void* lam,
                   const void* Q, const void* g, const void* X, void* images,
                   uint64_t* status, void* stream);

/* ---- fused FastMNMF iteration (_DiagLoop, separate.py:175-243) ----------- */

typedef struct fm_dims {
  int64_t B;        /* independent mixtures (batch) */
  int64_t F;        /* frequency bins held by this process */
  int64_t T, M, N, K;
  int64_t f_offset; /* global index of local bin 0 (frequency sharding) */
  int32_t dtype;    /* FM_F32 | FM_F64 */
  int32_t normalize;/* SeparatorConfig.normalize (separate.py:52) */
  int32_t ip_sweeps;/* SeparatorConfig.ip_sweeps (separate.py:53) */
  int32_t dp;       /* 1: FastMNMF-DP -- source 0 is the deep prior, W/H hold the
                       N-1 NMF noise sources (DeepPriorPlusNmfSource, sources.py:223-271) */
} fm_dims;

typedef struct fm_state {
  void* X;        /* (B,F,T,M) complex: scaled observation Xs (separate.py:293) */
  void* xt;       /* (B,F,T,M) real: projected power (separate.py:183, :230) */
  void* Q;        /* (B,F,M,M) complex */
  void* g;        /* (B,N,F,M) real */
  void* W;        /* (B,N,F,K) real */
  void* H;        /* (B,N,K,T) real (replicated across frequency shards) */
  void* floor;    /* (B) real: 1e-12 max|Xs|^2 (spatial.py:64-66) */
  double* trace;  /* (n_iterations, B): loglik of the state after iteration i */
  uint64_t* status; /* device status word */
  void* work;     /* fm_workspace_bytes() bytes, 256-B aligned */
} fm_state;

/* Workspace: lambda (B,N,F,T) (written once per iteration for the V pass),
 * the W of the coming H step (B,N,F,K), segment partials of the gain, V, W
 * and H statistics and of the log-likelihood, counters; the deep-prior path
 * also phi (B,2,N,F,T). */
size_t fm_workspace_bytes(const fm_dims* d);

/* ---- FastMNMF-DP (BASELINE config 4) ------------------------------------ */

/* Deep-prior source 0: lambda_0[f,t] = u_f v_t r[t,f], r = exp(dec(z)) with the
 * config-4 decoder dec: D -> Hd tanh -> Hd tanh -> F linear (weights as
 * PyTorch Linear: W1 (Hd,D), W2 (Hd,Hd), W3 (F,Hd), biases b1, b2, b3), and
 * `adam_steps` Adam steps on z per outer iteration at the reference's latent
 * hook (separate.py:205-213) against the NLL sum(x~/y + log y) with the rest
 * of the model frozen. All arrays device, real type of the dims' dtype. */
typedef struct fm_dp {
  int64_t D, Hd;
  const void *W1, *b1, *W2, *b2, *W3, *b3;
  void* u;        /* (B,F) */
  void* v;        /* (B,T) */
  void* z;        /* (B,T,D) */
  void* r;        /* (B,T,F) decoder output */
  void* adam_m;   /* (B,T,D) */
  void* adam_v;   /* (B,T,D) */
  uint32_t* adam_step; /* unused (reserved); the Adam step index is
                          iteration * adam_steps + s + 1 from the device counter */
  void* work;     /* fm_dp_workspace_bytes() */
  int32_t adam_steps;
  float lr, beta1, beta2, eps;
  /* ---- the reference's own latent update and decoder ----
   * decoder_kind FM_DEC_TOY: ToyDecoder (sources.py:52-80), r = max(softplus(
   * W3 tanh(W1 z + b1) + b3), 1e-8) with hidden width Hd; W2/b2 unused.
   * mh_steps > 0 replaces the Adam steps by the Metropolis random walk of
   * update_latents_fast (sources.py:307-339): per step z' = z + mh_std *
   * noise, accept per frame iff log(unif) <= log gamma_t
   * (metropolis_log_gamma_fast, sources.py:292-304). noise (mh_steps,B,T,D)
   * and unif (mh_steps,B,T) are caller-filled each iteration (the
   * reference's numpy stream), or both NULL: counter-based Philox-4x32-10
   * draws keyed by mh_seed and the device iteration counter. */
  int32_t decoder_kind;  /* FM_DEC_EXP_MLP (0) | FM_DEC_TOY (1) */
  int32_t mh_steps;
  double mh_std;         /* sqrt(MetropolisConfig.proposal_var) */
  const void* mh_noise;
  const void* mh_unif;
  uint64_t mh_seed;
} fm_dp;

#define FM_DEC_EXP_MLP 0
#define FM_DEC_TOY 1

size_t fm_dp_workspace_bytes(const fm_dims* d, const fm_dp* p);
/* decoder forward r = exp(dec(z)), lambda, projection and the first
 * statistics pass (the DP analogue of fm_prologue) */
int fm_prologue_dp(const fm_dims* d, const fm_state* s, const fm_dp* p, void* stream);
/* one FastMNMF-DP iteration: latents (Adam), U, V, W, H steps with refreshes,
 * gains, IP, normalisations (u absorbs c[0]), projection, statistics */
int fm_iterate_dp(const fm_dims* d, const fm_state* s, const fm_dp* p, void* stream);
/* n fm_iterate_dp calls, optionally from one captured CUDA graph */
int fm_run_dp(const fm_dims* d, const fm_state* s, const fm_dp* p, int n_iterations, int use_graph,
              void* stream);

/* NmfSource.lam (sources.py:184-187): lam (B,N,F,T) = W (B,N,F,K) H (B,N,K,T). */
int fm_nmf_lambda(const fm_dims* d, const void* W, const void* H, void* lam, void* stream);

/* Data term sum(-x~/y - log y) of the current state per mixture (B values,
 * host), i.e. what the first statistics pass of the next iteration returns
 * (_DiagLoop._refresh, separate.py:186-193; _kernels.py:233). Valid after
 * fm_prologue / any full iteration. Synchronises `stream`. */
int fm_data_term(const fm_dims* d, const fm_state* s, double* out_host, void* stream);

/* Zero counters; the projected power xt = |Q X|^2, the data term of the
 * initial state and iteration 0's W step (separate.py:183, :186-193, :214-216)
 * -- one k_bpass launch. */
int fm_prologue(const fm_dims* d, const fm_state* s, void* stream);

/* fm_prologue without the counter reset: re-derives xt, the transposed H and
 * the coming W step from the current state after the caller changed Q, g, W
 * or H between iterations (the reference loop's attributes are plain
 * assignable arrays, separate.py:178-184); the trace index continues. */
int fm_refresh(const fm_dims* d, const fm_state* s, void* stream);

/* Iteration schedules (fm_schedule). Default: the per-bin
 * schedule where it is eligible and the batch holds >= 4096 (bin, mixture)
 * pairs (BASELINE config 2), the split schedule otherwise. The environment
 * variable FM_SCHEDULE=split|fused|bin forces one (bin only where eligible).
 * Kernel variants inside a schedule are picked by shape: complex64
 * with even M in 10..16 accumulates V_fm on the tensor cores (k_vacc_tc; X
 * must then be 16-byte aligned) and complex64 with M > 8 projects on the
 * tensor cores (k_back_tc; FM_BACK=simt forces the SIMT kernel).
 * FM_VACC=blk|simt|tc|p forces a V kernel (p: the persistent k_vacc_p,
 * complex64 M = 5..8, opt-in). FM_UNROLL=n captures n iterations per CUDA
 * graph in fm_run (default 1; measured slower at config 1, DESIGN 8a). */
#define FM_SCHED_SPLIT 0
#define FM_SCHED_FUSED 1
#define FM_SCHED_BIN 2

/* The schedule fm_iterate / fm_run use for these dims: FM_SCHED_*, or -1
 * for invalid dims. The per-bin schedule (FM_SCHED_BIN) is three launches
 * per iteration (k_hstats, k_binw, k_trace) for complex64 with M <= 4,
 * 2 <= N <= 4, K <= 8 and H of a mixture (N x 8 x T floats) within shared
 * memory. */
int fm_schedule(const fm_dims* d);

/* One full iteration (separate.py:201-234) on one process. Split schedule:
 * ten launches (k_wstats, k_lambda, k_phi, k_hstats, k_lambda,
 * k_gain, k_vacc, k_ip, k_back, k_trace). Fused schedule (FM_SCHEDULE=fused):
 * six (k_hpass, k_gpass, k_vacc, k_ip, k_bpass, k_trace), lambda formed on
 * chip and the W step of the NEXT iteration inside k_bpass (the state W after
 * a call is still the reference's post-absorb W). B > 1 adds the counter
 * advance. Appends
 * trace[i] (i = number of previous fm_iterate calls since fm_prologue) =
 * data term + 2T sum_f log|det Q_f| of the state after this iteration. */
int fm_iterate(const fm_dims* d, const fm_state* s, void* stream);

/* Frequency-sharded iteration, split around the one exchange step: phase 0
 * runs the H statistics of this shard (its W step ran in the previous k_bpass) and leaves the packed
 * [num_H | den_H] (B,2,N,K,T) sums in *hstat (device, caller-sized); the
 * caller all-reduces it (sum) across shards; phase 1 applies the H update
 * from *hstat and runs the per-frequency rest of the iteration. */
int fm_iterate_phase(const fm_dims* d, const fm_state* s, int phase, void* hstat,
                     void* stream);

/* One fm_iterate captured into a CUDA graph with event-record nodes between
 * its launches and replayed once on `stream` (synchronises): ms_host (>= 10
 * floats) receives the device ms of each launch as it runs inside a graph
 * replay, *n_intervals their count -- split schedule (default, 10): k_wstats,
 * k_lambda, k_phi, k_hstats, k_lambda, k_gain, k_vacc, k_ip, k_back, k_trace;
 * fused schedule (FM_SCHEDULE=fused, 6): k_hpass, k_gpass, k_vacc, k_ip,
 * k_bpass, k_trace; per-bin schedule (3): k_hstats, k_binw, k_trace. Used by
 * bench.py for the per-kernel roofline. */
int fm_iterate_profiled(const fm_dims* d, const fm_state* s, float* ms_host, int* n_intervals,
                        void* stream);

/* The same for one fm_iterate_dp: ms_host (>= 21 floats) receives the device
 * ms of each launch in order (k_lambda, k_dp_lambda, [latent hook, k_dp_lambda,]
 * k_phi, k_dp_umu, k_dp_lambda, k_phi, k_dp_vmu, k_dp_lambda, k_phi, k_wstats,
 * k_lambda, k_phi, k_hstats, k_lambda, k_gain, k_vacc, k_ip, k_back,
 * k_trace); *n_intervals their count (21 with a latent hook, else 19). */
int fm_iterate_dp_profiled(const fm_dims* d, const fm_state* s, const fm_dp* p, float* ms_host,
                           int* n_intervals, void* stream);

/* n fm_iterate calls, optionally captured once into a CUDA graph that is
 * replayed (launch-bound configs). */
int fm_run(const fm_dims* d, const fm_state* s, int n_iterations, int use_graph,
           void* stream);

/* The observation prologue of run() (separate.py:284-293, spatial.py:64-66),
 * split so a frequency-sharded caller can all-reduce in between:
 * fm_observation_stats -> per mixture sum|X|^2 and max|X|^2 (fp64, host
 * arrays of B); fm_scale_observation -> X /= scale[b] in place (device,
 * scale given on the host, fp64). floor = 1e-12 max|Xs|^2 is then the
 * max of a second fm_observation_stats call, exactly as power_floor does. */
int fm_observation_stats(const fm_dims* d, const void* X, double* sumsq_host,
                         double* maxsq_host, void* stream);
int fm_scale_observation(const fm_dims* d, void* X, const double* scale_host, void* stream);

/* The reference's default spatial initialisation, per mixture and bin
 * (spatial.py:109-121 circular_init -> init_spatial(..., "diagonalizable")
 * spatial.py:93-105, clamp_psd linalg.py:85-94, hermitian_eig
 * linalg.py:23-33): G1 = clamp_psd(sum_t x x^H / T), w, U = eig descending,
 * Q = U^H. X is the SCALED observation (B, F, T, M) on the device; Q
 * (B, F, M, M) complex of d->dtype; w (B, F, M) fp64 clamped eigenvalues,
 * descending (may be NULL). Only d->B, F, T, M, dtype are read. fp64
 * throughout; eigenvector phases are arbitrary (as in LAPACK). */
int fm_spatial_init(const fm_dims* d, const void* X, void* Q, double* w, void* stream);

/* ---- STFT front / back end (stft.py:27-91) ---------------
 * Periodic Hann window of length L (power of two), reflect padding by L/2,
 * frames every hop samples (0 < hop <= L), zero tail to a whole frame.
 * fm_stft_frames: the frame count T = 1 + ceil((n + 2 (L/2) - L) / hop).
 * fm_stft: wave (n, M) real of dtype -> spec (L/2+1, T, M) complex, device.
 * fm_istft: spec (L/2+1, T, M) -> out (length, M), length <= (T-1) hop
 * (the de-padded signal, trimmed); windowed overlap-add divided by the
 * summed squared window (max with TINY); work: fm_istft_workspace_bytes.
 * Validation (power of two, hop range, n >= L) is the caller's, as in the
 * reference's Python; invalid sizes return FM_EINVAL. */
int64_t fm_stft_frames(int64_t n_samples, int64_t window_length, int64_t hop);
int fm_stft(int dtype, int64_t n_samples, int64_t M, int64_t window_length, int64_t hop,
            const void* wave, void* spec, void* stream);
size_t fm_istft_workspace_bytes(int dtype, int64_t n_frames, int64_t M, int64_t window_length);
int fm_istft(int dtype, int64_t n_frames, int64_t M, int64_t window_length, int64_t hop,
             int64_t length, const void* spec, void* work, void* out, void* stream);

/* ---- full-rank MNMF comparator (method "mnmf") ------------
 * X (F,T,M) complex, G (N,F,M,M) complex Hermitian SCMs, lam (N,F,T) real,
 * M <= 8; fp64 per-bin linear algebra, storage in the dtype.
 * fm_fullrank_stats: _kernels.fullrank_stats (_kernels.py:62-180): phi
 *   (2,N,F,T) = [phi1 | phi2] when want_phi, A/B (N,F,M,M) when want_ab,
 *   *loglik (device fp64, may be NULL) = sum_ft (-x^H Y^-1 x - log|Y|);
 *   work: fm_fullrank_workspace_bytes.
 * fm_update_scm: spatial.update_scm (spatial.py:145-169) on G in place, then
 *   normalize_trace (spatial.py:252-257) when normalize (c (N,F) = tr/M);
 *   status code 1 at (n, f) = negative spectrum (NumericalBreakdownError).
 * fm_wiener_fullrank: separate.wiener_fullrank (separate.py:83-107) ->
 *   images (N,F,T,M); status code 2 at (f, t) = singular mixture covariance.
 * fm_nmf_mu: NmfSource.apply_mu (sources.py:191-198) from phi, step 0 = W,
 *   1 = H; fm_nmf_absorb: W (N,F,K) *= c (N,F) (sources.py:202-204).
 * fm_reconstruct_scm: spatial.reconstruct_scm (spatial.py:211-223), status
 *   code 3 at f = singular Q. */
size_t fm_fullrank_workspace_bytes(int dtype, int64_t F, int64_t T, int64_t M);
int fm_fullrank_stats(int dtype, int64_t F, int64_t T, int64_t M, int64_t N, const void* X,
                      const void* G, const void* lam, double ridge, int want_ab, int want_phi,
                      void* phi, void* A, void* B, void* work, double* loglik, void* stream);
int fm_update_scm(int dtype, int64_t N, int64_t F, int64_t M, void* G, const void* A, const void* B,
                  int normalize, void* c, uint64_t* status, void* stream);
int fm_wiener_fullrank(int dtype, int64_t N, int64_t F, int64_t T, int64_t M, const void* lam,
                       const void* G, const void* X, double ridge, void* images, uint64_t* status,
                       void* stream);
int fm_nmf_mu(int dtype, int64_t N, int64_t F, int64_t T, int64_t K, const void* phi, void* W, void* H,
              int step, void* stream);
int fm_nmf_absorb(int dtype, int64_t N, int64_t F, int64_t K, void* W, const void* c, void* stream);
int fm_reconstruct_scm(int dtype, int64_t N, int64_t F, int64_t M, const void* Q, const void* g,
                       void* G, uint64_t* status, void* stream);

const char* fm_last_error(void);
int fm_version(void);

#ifdef __cplusplus
}
#endif
#endif /* FASTMNMF_H */
