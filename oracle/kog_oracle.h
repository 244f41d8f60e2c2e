/*
 * TEST INFRASTRUCTURE ONLY — the plain-C restatement of the reference's hot
 * path (oracle/kog_oracle.c).  Never linked into the product; only tests/,
 * __graft_entry__.smoke() and bench.py's CPU legs load it.
 *
 * Surface: the same host-array functions as oracle/_ref (prefix kogora_
 * instead of kogref_), struct layouts from include/kog2.h.
 *
 * Parity pin: checked bit-for-bit against the reference compiled in place
 * (oracle/_ref/libkogref.so) and against the committed golden fixtures in
 * tests/golden/ (tests/test_oracle.py).
 */
#ifndef KOG_ORACLE_H
#define KOG_ORACLE_H
#include <stddef.h>
#include <stdint.h>

#include "kog2.h"

#ifdef __cplusplus
extern "C" {
#endif

const char* kogora_last_error(void);
unsigned kogora_hardware_threads(void);
int kogora_hypot_f64(const double* a, const double* b, double* o, uint64_t n);
int kogora_hypot_f32(const float* a, const float* b, float* o, uint64_t n);
int kogora_split_f64(const double* x, int64_t* e, double* f, uint64_t n);
int kogora_split_f32(const float* x, int64_t* e, float* f, uint64_t n);
int kogora_assemble_f64(const int64_t* e, const double* f, double* o, uint64_t n);
int kogora_assemble_f32(const int64_t* e, const float* f, float* o, uint64_t n);
int kogora_tan2_f64(const double* t, double* o, uint64_t n);
int kogora_tan2_f32(const float* t, float* o, uint64_t n);
int kogora_sec_f64(const double* t, double* o, uint64_t n);
int kogora_sec_f32(const float* t, float* o, uint64_t n);
int kogora_epair_f64(int op, const int64_t* xe, const double* xf, const int64_t* ye, const double* yf,
                     int64_t* oe, double* of, uint8_t* st, uint64_t n);
int kogora_epair_f32(int op, const int64_t* xe, const float* xf, const int64_t* ye, const float* yf,
                     int64_t* oe, float* of, uint8_t* st, uint64_t n);
int kogora_classify_prescale_f64(const kog_mat_f64* in, const kog_classify_out* o, const kog_mat_f64* gp,
                                 uint64_t n);
int kogora_classify_prescale_f32(const kog_mat_f32* in, const kog_classify_out* o, const kog_mat_f32* gp,
                                 uint64_t n);
int kogora_urv15_f64(const kog_mat_f64* g, kog_urv15_f64* o, uint64_t n, const kog_options* opt);
int kogora_urv15_f32(const kog_mat_f32* g, kog_urv15_f32* o, uint64_t n, const kog_options* opt);
int kogora_tri_svd_f64(const double* a, const double* b, const double* c, const uint8_t* t13,
                       kog_trisvd_f64* o, uint64_t n, const kog_options* opt);
int kogora_tri_svd_f32(const float* a, const float* b, const float* c, const uint8_t* t13,
                       kog_trisvd_f32* o, uint64_t n, const kog_options* opt);
int kogora_compose_left_f64(const double* tp, const double* tt, const uint8_t* m, double* c, double* s,
                            uint64_t n);
int kogora_compose_left_f32(const float* tp, const float* tt, const uint8_t* m, float* c, float* s,
                            uint64_t n);
int kogora_triangularize13_f64(const kog_mat_f64* g, const uint8_t* t, const kog_mat_f64* r, int8_t* up,
                               int8_t* vp, uint64_t n);
int kogora_triangularize13_f32(const kog_mat_f32* g, const uint8_t* t, const kog_mat_f32* r, int8_t* up,
                               int8_t* vp, uint64_t n);
int kogora_svd2_f64(const kog_mat_f64* in, const kog_svd_out_f64* out, uint64_t n, const kog_options* opt,
                    int threads);
int kogora_svd2_f32(const kog_mat_f32* in, const kog_svd_out_f32* out, uint64_t n, const kog_options* opt,
                    int threads);
int kogora_svd2_ext_f64(const kog_mat_f64* g, kog_extsvd* o, uint64_t n);
int kogora_svd2_ext_f32(const kog_mat_f32* g, kog_extsvd* o, uint64_t n);
int kogora_metrics_f64(const kog_mat_f64* g, kog_metrics* o, uint64_t n, const kog_options* opt, int threads);
int kogora_metrics_f32(const kog_mat_f32* g, kog_metrics* o, uint64_t n, const kog_options* opt, int threads);
int kogora_generate_f64(const kog_run_config* c, uint64_t index0, const kog_mat_f64* o, uint64_t n,
                        int threads);
int kogora_generate_f32(const kog_run_config* c, uint64_t index0, const kog_mat_f32* o, uint64_t n,
                        int threads);
int kogora_run_batch(const kog_run_config* c, kog_stats* out);
int kogora_csv_row(const kog_run_config* c, const kog_stats* st, char* buf, size_t cap);
int kogora_lasv2_f64(const double* f, const double* g, const double* h, double* o6, uint64_t n);
int kogora_lasv2_f32(const float* f, const float* g, const float* h, float* o6, uint64_t n);

#ifdef __cplusplus
}
#endif
#endif
