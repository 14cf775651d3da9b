/*
 * str.h — C ABI of the B200-native streaming tensor-ring (STR / rSTR) per-batch update.
 *
 * Method: Yu & Li, "Tracking Tensor Ring Decompositions of Streaming Tensors",
 * arXiv 2307.00719 (cited as P:<line> of /root/reference/PAPER.md at build time; the
 * file is not needed at run time).
 *
 * Problem statement: given the TR decomposition of X^old (temporal mode N)
 * and the intermediate information kept by the method, update the decomposition with the
 * new temporal block X^new only.  The library keeps, on one GPU (or sharded over several),
 * the state of Alg. 4: the cores G_1..G_{N-1}, the temporal core G_N (one row
 * per processed time step), the complementary matrices P_n (I_n x R_nR_{n+1}) and
 * Q_n (R_nR_{n+1} x R_nR_{n+1}) of Eq. (partial), and the Gram tensors Z_n of
 * Alg. 4 l.2.  rSTR (Alg. 6; Alg. 7; Alg. 8)
 * keeps the same P_n/Q_n built from sampled rows and the sampled core slices; rSTR-K (Alg. 9
 * P:1194-1258) builds them from rows of the KSRFT-mixed problem (real parts, R17-R22).
 *
 * Conventions
 *   - Modes are numbered 1..N as in the paper; mode N is time.  All indices are 0-based.
 *   - Tensor data X (init, batches, fit input) use the paper's linearization P:119:
 *     element (i_1, ..., i_{N-1}, t) at offset i_1 + I_1*(i_2 + I_2*(... + I_{N-1}*t)).
 *   - Cores at this boundary use the paper layout G_n in R^{R_n x I_n x R_{n+1}}, first index
 *     fastest: element (a, i, b) at offset a + R_n*(i + I_n*b), R_{N+1} = R_1.
 *   - State is always fp64.  The data type of X (STR_F32 / STR_F64) and the precision of the
 *     dense contraction (STR_CONTRACT_3XTF32 / STR_CONTRACT_F64) are chosen separately.
 *
 * Execution model
 *   - Device work is enqueued on the stream given in the config (or an internal stream when
 *     NULL) and the call returns without waiting; call str_sync() to wait.  Host-side argument
 *     errors are reported immediately.  Device-side numerical failures (a non-positive
 *     pivot in the SPD inversion of Q_n or of a temporal Gram) are reported by the next str_sync(),
 *     str_get_cores(), str_get_temporal_rows() or str_fit() as STR_E_NUMERIC, after which
 *     the handle is poisoned (every later call returns STR_E_POISONED).
 *   - A handle is used by one host thread at a time.  Distinct handles may run
 *     concurrently on distinct streams.
 *   - No C++ exception crosses this boundary.
 */
#ifndef STR_B200_H
#define STR_B200_H

#include <stdint.h>

#if defined(__GNUC__)
#define STR_API __attribute__((visibility("default")))
#else
#define STR_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct str_state str_state; /* opaque; owns all device state */

typedef enum {
  STR_OK = 0,
  STR_E_ARG = 1,       /* invalid argument (NULL pointer, bad mode, capacity too small) */
  STR_E_SHAPE = 2,     /* shape mismatch */
  STR_E_PRECOND = 3,   /* rSTR with m < max_n R_nR_{n+1}, I_1 % world_size != 0 */
  STR_E_NUMERIC = 4,   /* SPD inversion of Q_n (or of a temporal Gram) met a non-positive pivot */
  STR_E_CUDA = 5,      /* CUDA runtime error */
  STR_E_NCCL = 6,      /* NCCL error (multi-GPU) */
  STR_E_OOM = 7,       /* device allocation failed */
  STR_E_POISONED = 8   /* an earlier failure poisoned the handle */
} str_status;

typedef enum { STR_F32 = 0, STR_F64 = 1 } str_dtype;
typedef enum { STR_CONTRACT_3XTF32 = 0, STR_CONTRACT_F64 = 1 } str_contract;
/* STR (Alg. 4); rSTR-U (Alg. 7), rSTR-L (Alg. 8); rSTR-K: KSRFT mixing + uniform rows (Def. 10
   P:614-627, Alg. 9; readings R17-R22) */
typedef enum { STR_DET = 0, STR_SAMPLE_UNIFORM = 1, STR_SAMPLE_LEVERAGE = 2, STR_SAMPLE_KSRFT = 3 } str_variant;
/* Collectives of the sharded step (world_size > 1): NCCL between processes (one per GPU), or an
   in-process loopback group (the ranks are handles of one process sharing one GPU; tests) */
typedef enum { STR_COMM_NCCL = 0, STR_COMM_LOOPBACK = 1 } str_comm;

typedef struct {
  int32_t order;          /* N >= 3 */
  const int64_t *dims;    /* I_1 .. I_{N-1}: GLOBAL sizes of the non-temporal modes */
  const int32_t *ranks;   /* R_1 .. R_N, each in [1, 16]; R_n R_{n+1} <= 128; STR also needs
                             R_{k+1} R_N <= 128 for the two-pass split k (STR_E_ARG otherwise) */
  str_dtype dtype;        /* element type of every X passed in */
  str_contract contract;  /* precision of the X contractions (state is always fp64) */
  str_variant variant;    /* STR (Alg. 4) or rSTR-U / rSTR-L / rSTR-K (Alg. 7 / 8 / 9) */
  int64_t sketch_rows;    /* rSTR m; must be >= max_n R_n R_{n+1} */
  uint64_t seed;          /* rSTR sampler seed (reading R11) */
  int64_t t_capacity;     /* initial capacity of temporal rows kept on the device (0 = 4096);
                             grows automatically */
  int32_t split_k;        /* two-pass split point k in [1, N-2] (0 = automatic) */
  int32_t world_size;     /* >= 1: X is sharded along mode 1 across world_size processes */
  int32_t rank;           /* this process' shard: rows [rank*I_1/p, (rank+1)*I_1/p) of mode 1 */
  const void *nccl_id;    /* STR_COMM_NCCL: 128-byte ncclUniqueId shared by all ranks; STR_COMM_LOOPBACK:
                             the group from str_loopback_create (ignored if world_size == 1) */
  int32_t device;         /* CUDA device ordinal */
  void *stream;           /* cudaStream_t to enqueue on, or NULL for an internal stream (created
                             blocking with respect to the legacy default stream) */
  int32_t comm;           /* str_comm (0 = NCCL) */
} str_config;

/* Alg. 4 l.1-5, Alg. 7 l.1-16, Alg. 8 l.1-17.
 * X_init: DEVICE pointer to this rank's shard (I_1/p x I_2 x ... x I_{N-1} x t_init), read
 *         during the call only (caller keeps ownership).
 * init_cores: HOST array of N pointers to GLOBAL cores in paper layout; core N holds t_init
 *         temporal rows (R_N x t_init x R_1).  Remark P:386-392: any feasible initialization.
 * out: receives the handle.  Errors: STR_E_ARG/SHAPE/PRECOND/CUDA/NCCL/OOM. */
STR_API str_status str_init(const str_config *cfg, const void *X_init, int64_t t_init,
                    const double *const *init_cores, str_state **out);

/* One time step (Alg. 4 l.7-19; Alg. 7 l.17-41; Alg. 8 l.18-43).
 * X_new: DEVICE pointer to this rank's shard (I_1/p x ... x I_{N-1} x t_new), t_new >= 1.
 * Lifetime: the call returns before the step has run; the caller must keep X_new valid and
 * unchanged until the enqueued work has completed (str_sync, any call documented as waiting, or an
 * event recorded on the library's stream after this call).  X_new must be produced before the call
 * in the stream order of the library's stream (or of the legacy default stream when the library's
 * internal stream is used).  The library never retains X_new after the step: the method never
 * revisits old data.  Collective when world_size > 1 (every rank calls with the same
 * t_new). */
STR_API str_status str_update_batch(str_state *h, const void *X_new, int64_t t_new);

/* Same step with X_new in HOST memory (pinned for full speed): the library copies it to the
 * device on its stream (the copy is part of the enqueued work). */
STR_API str_status str_update_batch_host(str_state *h, const void *X_new_host, int64_t t_new);

/* Copies GLOBAL core n (1..N) into host_out in paper layout; n = N gives R_N x T x R_1 where
 * T = str_processed().  capacity is in doubles.  Waits for the stream.  Collective for n = 1
 * when world_size > 1 (G_1 is row-sharded). */
STR_API str_status str_get_cores(str_state *h, int32_t n, double *host_out, int64_t capacity);

/* Copies temporal rows [t0, t0+t) of G_N(2) (t x R_N R_1, column r_N + R_N r_1) to host. */
STR_API str_status str_get_temporal_rows(str_state *h, int64_t t0, int64_t t, double *host_out);

/* ||X - TR(G)||_F / ||X||_F over temporal rows [t0, t0+t), always in fp64 with
 * direct differences.  X: DEVICE pointer to this rank's shard of those t slices.  Collective
 * when world_size > 1.  ||X|| = 0 gives STR_E_ARG. Waits for the stream. */
STR_API str_status str_fit(str_state *h, const void *X, int64_t t0, int64_t t, double *rel_err);

/* Batch TR-ALS on the GPU (Alg. 1; initialization protocol P:734; SURVEY
 * §8(f) NEXT-1).  Re-fits every core to X (t temporal slices, DEVICE pointer to this rank's shard,
 * element type cfg.dtype, paper linearization, caller-owned, read during the call) by `sweeps`
 * ALS sweeps starting from the cores the handle holds, then rebuilds the streaming state of Alg. 4
 * l.1-5 (Z_n, P_n, Q_n) from X and the fitted cores, as if X had been X_init: the stream
 * continues from there.  A sweep updates the modes in the cyclic order N, 1, ..., N-1 (Alg. 1's
 * order 1..N started one mode earlier), each mode by the exact LS solution of Eq. (tr_als)
 * P:160-164 formed through Prop. 1 (normal equations, Q = H^{≠n}_<2>), so one sweep is one
 * empty-history STR step over X.  The processed count becomes t.  rel_err (optional, host) gets
 * ||X - TR(G)||_F / ||X||_F after the last sweep (str_fit over X).  STR variant only
 * (STR_E_ARG for rSTR handles); collective when world_size > 1.  Waits for the stream. */
STR_API str_status str_tr_als(str_state *h, const void *X, int64_t t, int32_t sweeps, double *rel_err);

/* Waits for all enqueued work; reports deferred numerical failures. */
STR_API str_status str_sync(str_state *h);

STR_API int64_t str_processed(const str_state *h);          /* T = temporal rows so far */
STR_API const char *str_error_string(const str_state *h);   /* last error text ("" if none) */
STR_API void str_destroy(str_state *h);                     /* idempotent on NULL */

/* Number of CUDA kernels this library has launched on the handle's stream so far. */
STR_API int64_t str_kernel_launches(const str_state *h);

/* Profiling: when enabled, CUDA events bracket the dominant kernels on the handle's stream;
 * str_profile returns accumulated milliseconds and step counts since the last reset (waits for
 * the stream): STR — the pass-1 and pass-2 contractions; rSTR-K — the span of the N KSRFT mixing
 * passes in the pass-1 slot (pass-2 slot unused); rSTR-U/L — nothing is bracketed. */
STR_API str_status str_set_profiling(str_state *h, int32_t enable);
STR_API str_status str_profile(str_state *h, double *pass1_ms, int64_t *pass1_launches, double *pass2_ms,
                       int64_t *pass2_launches);

/* In-process loopback group of world_size ranks (STR_COMM_LOOPBACK): the ranks' handles are created
 * by str_init with cfg.comm = STR_COMM_LOOPBACK and cfg.nccl_id = group, from concurrent host
 * threads (str_init is collective); destroy the group after its handles. */
STR_API str_status str_loopback_create(int32_t world_size, void **group);
STR_API void str_loopback_destroy(void *group);

/* rSTR test hooks: the index table drawn for mode k (1..N) at the most
 * recent draw (m entries), or force the table used at the next draw of mode k. */
STR_API str_status str_get_index_table(str_state *h, int32_t mode, int32_t *idx, int64_t m);
STR_API str_status str_set_index_table(str_state *h, int32_t mode, const int32_t *idx, int64_t m);

#ifdef __cplusplus
}
#endif
#endif /* STR_B200_H */
