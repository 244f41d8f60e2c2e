// kog2_k_svd2.cu — the hot kernel: batched svd2 (svd2.hpp:603-687) over
// structure-of-arrays device buffers, one thread per matrix, compact result
// layout of include/kog2.h.  The default Options are a compile-time constant
// (branches on them fold away); any other Options run the same code with the
// values read from the kernel argument.
#include <cstdlib>

#include "kog2_common.cuh"

using namespace kog2;

namespace {

template <class T>
struct OutP {
  T *sig1_f, *sig2_f;
  int32_t *sig1_e, *sig2_e;
  T *u11, *u12, *v11, *v12;
  int32_t* s;
  uint32_t* flags;
};

template <class T>
__device__ __forceinline__ uint32_t sign_flags(const Result<T>& r) {
  uint32_t f = 0;
  if (sign_bit(r.u.g21)) f |= KOG_F_SIGN_U21;
  if (sign_bit(r.u.g22)) f |= KOG_F_SIGN_U22;
  if (sign_bit(r.v.g21)) f |= KOG_F_SIGN_V21;
  if (sign_bit(r.v.g22)) f |= KOG_F_SIGN_V22;
  return f;
}

template <class T, bool DEF, int MINB>
__global__ void __launch_bounds__(kThreads, MINB) k_svd2(InP<T> in, OutP<T> out, uint64_t n, Opt ropt) {
  const Opt o = DEF ? opt_default() : ropt;
  for (uint64_t i = gtid(); i < n; i += gstride()) {
    const Mat<T> g{ld_cs(in.g11 + i), ld_cs(in.g12 + i), ld_cs(in.g21 + i), ld_cs(in.g22 + i)};
    Result<T> r;
    svd2<T>(g, o, r);
    st_cs(out.sig1_f + i, r.sigma1.f);
    st_cs(out.sig2_f + i, r.sigma2.f);
    st_cs(out.sig1_e + i, static_cast<int32_t>(r.sigma1.e));
    st_cs(out.sig2_e + i, static_cast<int32_t>(r.sigma2.e));
    st_cs(out.u11 + i, r.u.g11);
    st_cs(out.u12 + i, r.u.g12);
    st_cs(out.v11 + i, r.v.g11);
    st_cs(out.v12 + i, r.v.g12);
    st_cs(out.s + i, static_cast<int32_t>(r.s));
    st_cs(out.flags + i, r.flags | sign_flags(r));
  }
}

template <class T, class MatC, class OutC>
int launch_svd2(const MatC* in, const OutC* out, uint64_t n, const kog_options* opt, cudaStream_t st) {
  if (n == 0) return KOG_OK;  // empty batch: nothing is dereferenced
  if (!in || !out) return kog2_arg_error("kog_svd2_batch: null argument");
  const OutP<T> op{out->sig1_f, out->sig2_f, out->sig1_e, out->sig2_e, out->u11,
                   out->u12,    out->v11,    out->v12,    out->s,      out->flags};
  if (!mat_ok<T>(in) || !op.sig1_f || !op.sig2_f || !op.sig1_e || !op.sig2_e || !op.u11 || !op.u12 ||
      !op.v11 || !op.v12 || !op.s || !op.flags)
    return kog2_arg_error("kog_svd2_batch: null array pointer");
  const Opt o = opt_of(opt);
  const int grid = grid_for(n);
  static const int minb = [] {  // occupancy variant (tuning knob, default 2)
    const char* e = std::getenv("KOG2_SVD2_MINB");
    return e ? std::atoi(e) : 3;
  }();
  if (!opt_is_default(o))
    k_svd2<T, false, 2><<<grid, kThreads, 0, st>>>(in_of<T>(in), op, n, o);
  else if (minb >= 4)
    k_svd2<T, true, 4><<<grid, kThreads, 0, st>>>(in_of<T>(in), op, n, o);
  else if (minb == 3)
    k_svd2<T, true, 3><<<grid, kThreads, 0, st>>>(in_of<T>(in), op, n, o);
  else
    k_svd2<T, true, 2><<<grid, kThreads, 0, st>>>(in_of<T>(in), op, n, o);
  return launched("k_svd2");
}

}  // namespace

extern "C" {

int kog_svd2_batch_f64(const kog_mat_f64* in, const kog_svd_out_f64* out, uint64_t n,
                       const kog_options* opt, void* stream) {
  return launch_svd2<double>(in, out, n, opt, KOG2_ST(stream));
}
int kog_svd2_batch_f32(const kog_mat_f32* in, const kog_svd_out_f32* out, uint64_t n,
                       const kog_options* opt, void* stream) {
  return launch_svd2<float>(in, out, n, opt, KOG2_ST(stream));
}

}  // extern "C"
