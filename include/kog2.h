/*
 * kog2.h — C-ABI of the B200-native batched enhanced 2x2 Kogbetliantz SVD.
 *
 * Every routine declared in the reference's proj/include/kogsvd2 keeps its
 * per-matrix meaning and gains a batched structure-of-arrays entry point here.
 * Each declaration cites the reference interface it replaces (paths relative to
 * /root/reference/proj/include/kogsvd2/).
 *
 * Conventions:
 *   - plain pointers and sizes only; no torch or C++ types cross this ABI;
 *   - `*_batch_*` entry points take DEVICE pointers and a cudaStream_t passed as
 *     `void* stream` (NULL = legacy default stream); they are stream-ordered and
 *     do not synchronize; the caller owns every buffer;
 *   - reentrant: any number of calls may be in flight at once on different
 *     streams or host threads.  Internal scratch (deferred-lane lists, study
 *     chunk buffers) is allocated per call on the caller's stream from a
 *     per-device stream-ordered memory pool and freed on it after last use;
 *     no call shares device scratch with another;
 *   - return value: KOG_OK (0) on success, a negative KOG_ERR_* code for an
 *     argument or CUDA error (message via kog_last_error()), or — for the
 *     routines whose reference throws std::domain_error — a positive count is
 *     never returned asynchronously: the per-element status/flags word carries
 *     the domain-error bit instead (no exceptions cross the ABI);
 *   - `kog_run_batch` and `kog_svd2_host_*` are synchronous host-level calls.
 *   - Working precisions: `_f64` = binary64, `_f32` = binary32 (WorkingFloat,
 *     fpcore.hpp:17-18).
 */
#ifndef KOG2_H
#define KOG2_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------------ status */
#define KOG_OK 0
#define KOG_ERR_ARG (-1)
#define KOG_ERR_CUDA (-2)
#define KOG_ERR_NODEV (-3)
#define KOG_ERR_ABORT (-4) /* kog_run_batch: BatchAbort (harness.hpp:108-110) */

const char* kog_last_error(void);
const char* kog_version(void);
/* Select the CUDA device for this host thread's subsequent calls (the library
 * carries its own CUDA runtime; callers without one select devices here). */
int kog_set_device(int device);

/* ---------------------------------------------------------------- options */
/* Options (svd2.hpp:122-132).  wide_channel: 0 = wider_type, 1 = kahan_det. */
typedef struct kog_options {
  uint8_t hypot_is_cr;  /* default 1 */
  uint8_t ominus_for_d; /* default 0 */
  uint8_t wide_channel; /* default 0 (KOG_WIDE_WIDER_TYPE) */
  uint8_t reserved;
} kog_options;
#define KOG_WIDE_WIDER_TYPE 0
#define KOG_WIDE_KAHAN_DET 1

/* ------------------------------------------------- compact result layout */
/*
 * Svd2Result<T> (svd2.hpp:134-140) in compact SoA form:
 * u = [[u11, u12], [u21, u22]] with |u21| == |u12| and |u22| == |u11| bit-exactly,
 * so only u11, u12 and the sign bits of u21, u22 are stored (same for V).
 * sigma_i = 2^sig_e * sig_f (EPair, epair.hpp:16-46), s = prescale exponent.
 * The 32-bit flags word packs the sign bits and the BranchTrace (svd2.hpp:108-120).
 */
#define KOG_F_SIGN_U21 (1u << 0)
#define KOG_F_SIGN_U22 (1u << 1)
#define KOG_F_SIGN_V21 (1u << 2)
#define KOG_F_SIGN_V22 (1u << 3)
#define KOG_F_PATH_SHIFT 4 /* 3 bits: SvdPath (svd2.hpp:98-106) */
#define KOG_F_T2P_SHIFT 7  /* 3 bits: Tan2PhiBranch (svd2.hpp:88-96) */
#define KOG_F_TANPSI_INF (1u << 10)
#define KOG_F_DIAG_SWAP (1u << 11)
#define KOG_F_SIGMA_SWAP (1u << 12)
#define KOG_F_COMPOSE_MINUS (1u << 13)
#define KOG_F_PRESCALE_INEXACT (1u << 14)
#define KOG_F_URV_COL_SWAP (1u << 15)
#define KOG_F_URV_ROW_SWAP (1u << 16)
#define KOG_F_TYPE_INIT_SHIFT 17   /* 4 bits: trace.type_initial */
#define KOG_F_TYPE_SCALED_SHIFT 21 /* 4 bits: trace.type_scaled */
#define KOG_F_DOMAIN_ERROR (1u << 31) /* the reference would have thrown */

/* SvdPath values (svd2.hpp:98-106) */
#define KOG_PATH_SIMPLE 0
#define KOG_PATH_MONO_COL 1
#define KOG_PATH_MONO_ROW 2
#define KOG_PATH_TRI13 3
#define KOG_PATH_URV15 4
#define KOG_PATH_URV15_TO_DIAG 5
#define KOG_PATH_URV15_TO_ROW 6
/* Tan2PhiBranch values (svd2.hpp:88-96) */
#define KOG_T2P_NONE 0
#define KOG_T2P_DIAG_EQUAL 1
#define KOG_T2P_OFFDIAG_EQUAL 2
#define KOG_T2P_SMALL_RATIO 3
#define KOG_T2P_FALLBACK 4
#define KOG_T2P_GENERAL 5
#define KOG_T2P_GENERAL_INF 6

/* Matrix2<T> batch (classify.hpp:14-19), one array per element. */
typedef struct kog_mat_f64 { double *g11, *g12, *g21, *g22; } kog_mat_f64;
typedef struct kog_mat_f32 { float *g11, *g12, *g21, *g22; } kog_mat_f32;

typedef struct kog_svd_out_f64 {
  double *sig1_f, *sig2_f;
  int32_t *sig1_e, *sig2_e;
  double *u11, *u12, *v11, *v12;
  int32_t* s;
  uint32_t* flags;
} kog_svd_out_f64;
typedef struct kog_svd_out_f32 {
  float *sig1_f, *sig2_f;
  int32_t *sig1_e, *sig2_e;
  float *u11, *u12, *v11, *v12;
  int32_t* s;
  uint32_t* flags;
} kog_svd_out_f32;

/* ------------------------------------------------------------ headline op */
/* svd2(const Matrix2<T>&, const Options&) -> Svd2Result<T>  (svd2.hpp:603-687) */
int kog_svd2_batch_f64(const kog_mat_f64* in, const kog_svd_out_f64* out, uint64_t n,
                       const kog_options* opt, void* stream);
int kog_svd2_batch_f32(const kog_mat_f32* in, const kog_svd_out_f32* out, uint64_t n,
                       const kog_options* opt, void* stream);

/* Same operation on HOST buffers (any host memory; pinned is fastest): chunked
 * H2D -> svd2 -> D2H pipeline over CUDA streams on the current device.  This is
 * the drop-in for a CPU caller of svd2 over an array of matrices.  Synchronous. */
int kog_svd2_host_f64(const kog_mat_f64* in, const kog_svd_out_f64* out, uint64_t n,
                      const kog_options* opt);
int kog_svd2_host_f32(const kog_mat_f32* in, const kog_svd_out_f32* out, uint64_t n,
                      const kog_options* opt);

/* Host-buffer forms of the per-matrix routines the C++ shim
 * (include/kog2/kogsvd2_gpu.hpp) needs: each stages its arrays through device
 * memory on a private stream and is synchronous.  hypot_cr (fpcore.hpp:140-188),
 * svd2_ext (oracle.hpp:102-238), run_one's svd2 + svd2_ext + metrics
 * (harness.hpp:190-222, oracle.hpp:269-301), generate (harness.hpp:139-186). */
int kog_hypot_host_f64(const double* a, const double* b, double* out, uint64_t n);
int kog_hypot_host_f32(const float* a, const float* b, float* out, uint64_t n);
/* (kog_svd2_ext_host_*, kog_metrics_host_*, kog_generate_host_*: declared
 * below, after their record types) */

/* ------------------------------------------------ fpcore.hpp unit routines */
/* hypot_cr<T> (fpcore.hpp:140-188) */
int kog_hypot_batch_f64(const double* a, const double* b, double* out, uint64_t n, void* stream);
int kog_hypot_batch_f32(const float* a, const float* b, float* out, uint64_t n, void* stream);
/* split (fpcore.hpp:41-47) */
int kog_split_batch_f64(const double* x, int64_t* e, double* f, uint64_t n, void* stream);
int kog_split_batch_f32(const float* x, int64_t* e, float* f, uint64_t n, void* stream);
/* assemble (fpcore.hpp:51-55) */
int kog_assemble_batch_f64(const int64_t* e, const double* f, double* out, uint64_t n, void* stream);
int kog_assemble_batch_f32(const int64_t* e, const float* f, float* out, uint64_t n, void* stream);
/* tan_from_double_angle (fpcore.hpp:192-196) */
int kog_tan_from_double_angle_batch_f64(const double* t2, double* out, uint64_t n, void* stream);
int kog_tan_from_double_angle_batch_f32(const float* t2, float* out, uint64_t n, void* stream);
/* sec_from_tan (fpcore.hpp:198-201) */
int kog_sec_from_tan_batch_f64(const double* t, double* out, uint64_t n, void* stream);
int kog_sec_from_tan_batch_f32(const float* t, float* out, uint64_t n, void* stream);

/* ------------------------------------------------- epair.hpp unit routines */
/* EPair op selector for kog_epair_batch_*:
 *   OPLUS/OMINUS: (x,y) plain values in xf, yf (epair.hpp:57-77);
 *   MUL/DIV: EPair operands (xe,xf), (ye,yf) (epair.hpp:79-88);
 *   LESS: out_f = 1 or 0 (epair.hpp:119-127); RECIP: (xe,xf) only (112-116);
 *   MAKE: EPair(xe, xf) normalising constructor (epair.hpp:23-36).
 * Domain errors (the reference throws) set status[i] = 1 (else 0). */
#define KOG_EPAIR_OPLUS 0
#define KOG_EPAIR_OMINUS 1
#define KOG_EPAIR_MUL 2
#define KOG_EPAIR_DIV 3
#define KOG_EPAIR_LESS 4
#define KOG_EPAIR_RECIP 5
#define KOG_EPAIR_MAKE 6
int kog_epair_batch_f64(int op, const int64_t* xe, const double* xf, const int64_t* ye,
                        const double* yf, int64_t* out_e, double* out_f, uint8_t* status,
                        uint64_t n, void* stream);
int kog_epair_batch_f32(int op, const int64_t* xe, const float* xf, const int64_t* ye,
                        const float* yf, int64_t* out_e, float* out_f, uint8_t* status,
                        uint64_t n, void* stream);

/* ---------------------------------------------- classify.hpp unit routines */
/* classify (classify.hpp:44-58) + prescale (classify.hpp:67-78) fused: info
 * fields and the prescaled matrix.  status[i] = 1 on non-finite input. */
typedef struct kog_classify_out {
  uint8_t* t;
  int32_t* s_type;
  int64_t* s;
  int64_t* e_G; /* INT64_MIN for the zero matrix (kExpSentinel, classify.hpp:27) */
  uint8_t* inexact_underflow;
  uint8_t* status;
} kog_classify_out;
int kog_classify_prescale_batch_f64(const kog_mat_f64* in, const kog_classify_out* out,
                                    const kog_mat_f64* gp, uint64_t n, void* stream);
int kog_classify_prescale_batch_f32(const kog_mat_f32* in, const kog_classify_out* out,
                                    const kog_mat_f32* gp, uint64_t n, void* stream);

/* ------------------------------------------------- svd2.hpp phase routines */
/* urv15 (svd2.hpp:325-384), AoS record per matrix. */
typedef struct kog_urv15_f64 {
  double gppp[4]; /* g11, g12, g21, g22 of the pivoted input */
  double tan_theta, sec_theta, r11, r12_raw, r22_raw;
  double r[4]; /* positive upper triangle when next == triangular */
  int32_t sr0, sr1, s12, s22;
  uint8_t col_swap, row_swap, ext_is_r22, next; /* next: 0 tri, 1 diag, 2 row */
} kog_urv15_f64;
typedef struct kog_urv15_f32 {
  float gppp[4];
  float tan_theta, sec_theta, r11, r12_raw, r22_raw;
  float r[4];
  int32_t sr0, sr1, s12, s22;
  uint8_t col_swap, row_swap, ext_is_r22, next;
} kog_urv15_f32;
int kog_urv15_batch_f64(const kog_mat_f64* gp, kog_urv15_f64* out, uint64_t n,
                        const kog_options* opt, void* stream);
int kog_urv15_batch_f32(const kog_mat_f32* gp, kog_urv15_f32* out, uint64_t n,
                        const kog_options* opt, void* stream);

/* tan2phi (svd2.hpp:389-426) and tri_svd (svd2.hpp:428-474) on rt =
 * [[r11, r12], [0, r22]]; t13 selects the triangular-input shortcut. */
typedef struct kog_trisvd_f64 {
  double tan_phi, sec_phi, cos_phi, sin_phi, tan_psi, sec_psi, cos_psi, sin_psi;
  double sig1_f, sig2_f, t2f;
  int64_t sig1_e, sig2_e;
  uint8_t sigma_swapped, tanpsi_inf, t2p, status;
} kog_trisvd_f64;
typedef struct kog_trisvd_f32 {
  float tan_phi, sec_phi, cos_phi, sin_phi, tan_psi, sec_psi, cos_psi, sin_psi;
  float sig1_f, sig2_f, t2f;
  int64_t sig1_e, sig2_e;
  uint8_t sigma_swapped, tanpsi_inf, t2p, status;
} kog_trisvd_f32;
int kog_tri_svd_batch_f64(const double* r11, const double* r12, const double* r22,
                          const uint8_t* t13, kog_trisvd_f64* out, uint64_t n,
                          const kog_options* opt, void* stream);
int kog_tri_svd_batch_f32(const float* r11, const float* r12, const float* r22,
                          const uint8_t* t13, kog_trisvd_f32* out, uint64_t n,
                          const kog_options* opt, void* stream);

/* compose_left (svd2.hpp:485-515) */
int kog_compose_left_batch_f64(const double* tan_phi_bold, const double* tan_theta,
                               const uint8_t* minus_form, double* c, double* s, uint64_t n,
                               void* stream);
int kog_compose_left_batch_f32(const float* tan_phi_bold, const float* tan_theta,
                               const uint8_t* minus_form, float* c, float* s, uint64_t n,
                               void* stream);

/* triangularize13 (svd2.hpp:257-271): R and the two signed permutations
 * (row-major int8 2x2 each, 4 bytes per matrix). */
int kog_triangularize13_batch_f64(const kog_mat_f64* gp, const uint8_t* t, const kog_mat_f64* r,
                                  int8_t* uplus, int8_t* vplus, uint64_t n, void* stream);
int kog_triangularize13_batch_f32(const kog_mat_f32* gp, const uint8_t* t, const kog_mat_f32* r,
                                  int8_t* uplus, int8_t* vplus, uint64_t n, void* stream);

/* --------------------------------------------- extfloat.hpp / oracle.hpp */
/* ExtFloat (extfloat.hpp:19-25): value = 2^e * (hi + lo). */
typedef struct kog_extfloat {
  int64_t e;
  double hi, lo;
} kog_extfloat;

/* svd2_ext (oracle.hpp:102-238): reference SVD in ExtFloat. */
typedef struct kog_extsvd {
  kog_extfloat sigma1, sigma2;
  kog_extfloat u[4], v[4]; /* row-major a11, a12, a21, a22 */
} kog_extsvd;
int kog_svd2_ext_batch_f64(const kog_mat_f64* g, kog_extsvd* out, uint64_t n, void* stream);
int kog_svd2_ext_batch_f32(const kog_mat_f32* g, kog_extsvd* out, uint64_t n, void* stream);

/* ErrorMetrics (oracle.hpp:243-247) of svd2(g) against svd2_ext(g), i.e. the
 * per-matrix body of run_one (harness.hpp:190-222) without generation. */
typedef struct kog_metrics {
  double reG, reS1, reS2, reU, reV;
  kog_extfloat kappa2;
  uint32_t kappa_inf;
  uint32_t flags; /* svd2 flags word incl. KOG_F_DOMAIN_ERROR; bit 30 = NaN metric,
                     bit 29 = non-finite factor */
} kog_metrics;
#define KOG_M_NAN_METRIC (1u << 30)
#define KOG_M_NONFINITE_FACTOR (1u << 29)
int kog_metrics_batch_f64(const kog_mat_f64* g, kog_metrics* out, uint64_t n,
                          const kog_options* opt, void* stream);
int kog_metrics_batch_f32(const kog_mat_f32* g, kog_metrics* out, uint64_t n,
                          const kog_options* opt, void* stream);

/* ------------------------------------------------------------- harness */
/* Shape / Regime / Routine (harness.hpp:23-25).  KOG_REGIME_RANGED is the kog2
 * extension for the BASELINE configs 2-5: each element is
 * ranged(elo, ehi), or ranged(tail_lo, tail_hi) when tail_mod != 0 and a
 * leading draw t satisfies t % tail_mod == 0; zero_mask_rule = 1 adds one draw
 * z after the four elements and, if (z & 7) == 0, zeroes the entries selected
 * by (z >> 3) & 15 in classify's bit order. */
#define KOG_SHAPE_TRI 0
#define KOG_SHAPE_GEN 1
#define KOG_REGIME_CIRC 0
#define KOG_REGIME_BULLET 1
#define KOG_REGIME_SIGMA 2
#define KOG_REGIME_RANGED 3
#define KOG_ROUTINE_KOG 0
#define KOG_ROUTINE_LASV2 1

/* RunConfig (harness.hpp:27-37) plus the generator extension. */
typedef struct kog_run_config {
  uint8_t single_precision;
  uint8_t shape;
  uint8_t regime;
  uint8_t routine;
  int32_t varsigma;
  uint64_t count;
  uint64_t seed;
  int32_t threads; /* accepted for signature parity; the GPU ignores it */
  kog_options options;
  /* kog2 generator extension (regime KOG_REGIME_RANGED) */
  int32_t elo, ehi;
  int32_t tail_lo, tail_hi;
  uint32_t tail_mod;
  uint32_t zero_mask_rule;
} kog_run_config;

/* generate<T>(cfg, index) (harness.hpp:139-186) for indices [index0, index0+n). */
int kog_generate_batch_f64(const kog_run_config* cfg, uint64_t index0, const kog_mat_f64* out,
                           uint64_t n, void* stream);
int kog_generate_batch_f32(const kog_run_config* cfg, uint64_t index0, const kog_mat_f32* out,
                           uint64_t n, void* stream);
/* host-buffer forms (synchronous; see kog_hypot_host_f64 above) */
int kog_generate_host_f64(const kog_run_config* cfg, uint64_t index0, const kog_mat_f64* out, uint64_t n);
int kog_generate_host_f32(const kog_run_config* cfg, uint64_t index0, const kog_mat_f32* out, uint64_t n);
int kog_svd2_ext_host_f64(const kog_mat_f64* g, kog_extsvd* out, uint64_t n);
int kog_svd2_ext_host_f32(const kog_mat_f32* g, kog_extsvd* out, uint64_t n);
int kog_metrics_host_f64(const kog_mat_f64* g, kog_metrics* out, uint64_t n, const kog_options* opt);
int kog_metrics_host_f32(const kog_mat_f32* g, kog_metrics* out, uint64_t n, const kog_options* opt);

/* ErrorStats + BranchCounts (harness.hpp:50-106), plus the index at which the
 * max kappa was first attained (tie-break = reference merge order) and the
 * first failure key (index*4 + reason, reason 1 = non-finite factor,
 * 2 = NaN metric; UINT64_MAX if none). */
typedef struct kog_stats {
  double reG, reS1, reS2, reU, reV;
  kog_extfloat max_kappa2;
  uint64_t max_kappa2_index;
  uint64_t kappa_inf;
  uint64_t t2p[7];
  uint64_t path[7];
  uint64_t tanpsi_inf, diag_swap, compose_minus, sigma_swap, prescale_inexact;
  uint64_t fail_key;
} kog_stats;
#define KOG_FAIL_NONFINITE 1
#define KOG_FAIL_NAN_METRIC 2

void kog_stats_init(kog_stats* st);
/* ErrorStats::merge (harness.hpp:96-105); `o` covers later indices than `st`. */
void kog_stats_merge(kog_stats* st, const kog_stats* o);

/* Fused study over indices [index0, index0+n) of cfg on the current device:
 * generate -> svd2_ext -> svd2 (or lasv2) -> finiteness -> metrics -> absorb,
 * reduced on device into *stats_dev (a device kog_stats, initialised with
 * kog_stats_init and copied to the device by the caller, or by
 * kog_study_batch_init).  Stream-ordered. */
int kog_study_stats_alloc(kog_stats** stats_dev);
int kog_study_stats_free(kog_stats* stats_dev);
int kog_study_stats_reset(kog_stats* stats_dev, void* stream);
int kog_study_batch(const kog_run_config* cfg, uint64_t index0, uint64_t n, kog_stats* stats_dev,
                    void* stream);

/* validate<T> (harness.hpp:39-48): KOG_OK or KOG_ERR_ARG with the message. */
int kog_validate(const kog_run_config* cfg);
/* run_batch_any (harness.hpp:226-271, 319-321), GPU-backed, synchronous.
 * Returns KOG_ERR_ABORT with the reference's BatchAbort message in
 * kog_last_error() when a matrix fails. */
int kog_run_batch(const kog_run_config* cfg, kog_stats* out);
/* BatchAbort text for a failure key (harness.hpp:194-198). */
int kog_abort_message(const kog_run_config* cfg, uint64_t fail_key, char* buf, size_t cap);

/* --------------------------------------------------------- multi-GPU study */
/* contiguous index shards [k*N/G, (k+1)*N/G) (the last takes
 * the remainder), one study per device, and ONE ncclAllReduce(MAX) of a small
 * packed int64 vector; the per-rank blocks are merged on the host in rank
 * order (ErrorStats::merge, harness.hpp:96-105), so any device count gives the
 * stats (and CSV row) of kog_run_batch.  NCCL is dlopen'ed on first use
 * (libnccl.so.2); KOG_ERR_NODEV if it is absent. */
void kog_study_shard(uint64_t count, int rank, int world, uint64_t* lo, uint64_t* hi);
size_t kog_stats_slot_count(int world);
/* slots[kog_stats_slot_count(world)]: 0-4 metric bit patterns, 5 kappa_inf,
 * 6 = 2^62 - fail_key (or -1), then 23 fields per rank as 32-bit halves */
int kog_stats_pack(const kog_stats* st, int rank, int world, int64_t* slots);
int kog_stats_unpack(const int64_t* slots, int world, kog_stats* out);
/* One process per device (torchrun / MPI): rank 0 makes the id, the caller
 * distributes its 128 bytes, every rank makes its communicator on its current
 * device, and kog_study_allreduce combines that rank's host stats in place. */
int kog_nccl_available(void);
int kog_nccl_unique_id(uint8_t* id, size_t cap);
int kog_nccl_comm_init(const uint8_t* id, int world, int rank, void** comm);
int kog_nccl_comm_destroy(void* comm);
int kog_study_allreduce(void* comm, int rank, int world, kog_stats* stats, void* stream);
/* One process, one host thread per device (the reference's run_batch worker
 * pool, harness.hpp:226-271, with devices as workers): the whole study of cfg
 * over devices[0..ndev) (NULL = 0..ndev-1), synchronous.  *device_seconds
 * (optional) = max over devices of the device time of study + all-reduce.
 * Returns KOG_ERR_ABORT with the BatchAbort text like kog_run_batch. */
int kog_study_multi(const kog_run_config* cfg, const int* devices, int ndev, kog_stats* out,
                    double* device_seconds);

/* csv_header / csv_row (harness.hpp:286-317); returns the length written. */
int kog_csv_header(char* buf, size_t cap);
int kog_csv_row(const kog_run_config* cfg, const kog_stats* st, char* buf, size_t cap);

/* -------------------------------------------------------------- lasv2 */
/* lasv2_ref(f, g, h) (lasv2.hpp:22-127): ssmin, ssmax, snr, csr, snl, csl. */
int kog_lasv2_batch_f64(const double* f, const double* g, const double* h, double* out6,
                        uint64_t n, void* stream);
int kog_lasv2_batch_f32(const float* f, const float* g, const float* h, float* out6,
                        uint64_t n, void* stream);

/* ---------------------------------------------------------- diagnostics */
/* FP64 pipe probe: a DFMA chain, `iters` per thread over the whole device;
 * writes one value per thread to sink[] so the work cannot be elided. */
int kog_fp64_probe(double* sink, uint64_t threads, uint32_t iters, void* stream);
/* Correctly rounded x / y as used on the svd2 path (significand division with
 * the general IEEE division out of line), exposed for verification. */
int kog_div_batch_f64(const double* x, const double* y, double* out, uint64_t n, void* stream);
int kog_div_batch_f32(const float* x, const float* y, float* out, uint64_t n, void* stream);
/* Matrices that left the specialised path and were recomputed by the general
 * kernel, summed over every kog_svd2_batch_* call (default Options) on the
 * current device since the library was loaded (synchronous; -1 on error).
 * Diagnostics only: take differences around the calls of interest. */
int64_t kog_svd2_deferred_count(void);
/* kog_svd2_batch_f64 launches (default Options, batches of 2^23 matrices and more) whose
 * input sample kept them on the two-speed kernel (k_svd2_lean) instead of
 * handing the batch back to k_svd2_fast, on the current device since load
 * (synchronous; -1 on error).  Diagnostics only. */
int64_t kog_svd2_lean_count(void);
/* Tuning knob: the smallest kog_svd2_batch_f64 batch (default Options) that is
 * offered to the two-speed kernel (default 2^23; at least 2^16).  Returns the
 * previous value.  Results do not depend on it. */
uint64_t kog_svd2_set_lean_min(uint64_t n);
/* Tuning knob: log2 of the matrices per chunk of kog_study_batch's pipeline
 * (default 24; clamped to [16, 26]; the chunk buffers take 192 B per matrix,
 * twice).  Returns the previous value.  Results do not depend on it. */
int kog_study_set_chunk_log2(int log2_matrices);
/* number of kernel launches issued by this library since load */
uint64_t kog_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* KOG2_H */
