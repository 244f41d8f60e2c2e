// kog2_svd2batch — GPU-backed drop-in for the reference's `svd2batch` CLI
// (proj/tools/svd2batch.cpp:31-102): same flags, defaults, CSV and exit codes
// (0 ok, 1 batch aborted, 2 usage/configuration error); run_batch runs on the
// current CUDA device through the C-ABI (kog_run_batch, kog_csv_row).
//
// Extensions: --regime ranged with --elo/--ehi, --tail LO..HI:MOD and
// --zero-mask (the BASELINE config generator rules, include/kog2.h),
// --device N, and --gpus N (the study sharded over devices 0..N-1 with one
// NCCL all-reduce of the stats, kog_study_multi; the CSV is the same).
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <string>

#include "kog2.h"

namespace {

int usage(const char* msg) {
  std::cerr << msg << "\n"
            << "usage: kog2_svd2batch [--precision single|double] [--shape tri|gen] [--regime circ|bullet|sigma|ranged]\n"
               "                      [--varsigma N] [--count N] [--seed HEX] [--routine kog|lasv2] [--threads N]\n"
               "                      [--out PATH] [--sweep varsigma=A..B:step] [--emulate-noncr-hypot]\n"
               "                      [--elo E --ehi E] [--tail LO..HI:MOD] [--zero-mask] [--device N] [--gpus N]\n";
  return 2;
}

bool parse_int(const char* s, long long& v) {
  char* end = nullptr;
  v = std::strtoll(s, &end, 10);
  return end && *end == '\0' && end != s;
}

}  // namespace

int main(int argc, char** argv) {
  std::string precision = "double", shape = "tri", regime = "circ", routine = "kog";
  std::string seed_hex = "0", out_path, sweep_spec, tail_spec;
  kog_run_config cfg;
  std::memset(&cfg, 0, sizeof cfg);
  cfg.count = 1ull << 20;
  cfg.threads = 1;
  cfg.options.hypot_is_cr = 1;
  int device = -1, gpus = 0;
  for (int i = 1; i < argc; ++i) {
    const std::string a = argv[i];
    auto need = [&](const char* what) -> const char* {
      if (i + 1 >= argc) return nullptr;
      (void)what;
      return argv[++i];
    };
    const char* v = nullptr;
    long long n = 0;
    if (a == "--emulate-noncr-hypot") {
      cfg.options.hypot_is_cr = 0;
    } else if (a == "--zero-mask") {
      cfg.zero_mask_rule = 1;
    } else if (a == "--precision" || a == "--shape" || a == "--regime" || a == "--routine" || a == "--seed" ||
               a == "--out" || a == "--sweep" || a == "--tail") {
      if (!(v = need(a.c_str()))) return usage(("missing value for " + a).c_str());
      std::string s = v;
      if (a == "--precision") precision = s;
      if (a == "--shape") shape = s;
      if (a == "--regime") regime = s;
      if (a == "--routine") routine = s;
      if (a == "--seed") seed_hex = s;
      if (a == "--out") out_path = s;
      if (a == "--sweep") sweep_spec = s;
      if (a == "--tail") tail_spec = s;
    } else if (a == "--varsigma" || a == "--count" || a == "--threads" || a == "--elo" || a == "--ehi" ||
               a == "--device" || a == "--gpus") {
      if (!(v = need(a.c_str())) || !parse_int(v, n)) return usage(("bad value for " + a).c_str());
      if (a == "--varsigma") cfg.varsigma = static_cast<int32_t>(n);
      if (a == "--count") {
        if (n < 0) return usage("--count must be >= 0");
        cfg.count = static_cast<uint64_t>(n);
      }
      if (a == "--threads") cfg.threads = static_cast<int32_t>(n);
      if (a == "--elo") cfg.elo = static_cast<int32_t>(n);
      if (a == "--ehi") cfg.ehi = static_cast<int32_t>(n);
      if (a == "--device") device = static_cast<int>(n);
      if (a == "--gpus") {
        if (n < 1) return usage("--gpus must be >= 1");
        gpus = static_cast<int>(n);
      }
    } else {
      return usage(("unknown argument " + a).c_str());
    }
  }
  if (precision != "single" && precision != "double") return usage("--precision: single|double");
  if (shape != "tri" && shape != "gen") return usage("--shape: tri|gen");
  if (regime != "circ" && regime != "bullet" && regime != "sigma" && regime != "ranged")
    return usage("--regime: circ|bullet|sigma|ranged");
  if (routine != "kog" && routine != "lasv2") return usage("--routine: kog|lasv2");
  cfg.single_precision = precision == "single";
  cfg.shape = shape == "tri" ? KOG_SHAPE_TRI : KOG_SHAPE_GEN;
  cfg.regime = regime == "circ" ? KOG_REGIME_CIRC
               : regime == "bullet" ? KOG_REGIME_BULLET
               : regime == "sigma"  ? KOG_REGIME_SIGMA
                                    : KOG_REGIME_RANGED;
  cfg.routine = routine == "kog" ? KOG_ROUTINE_KOG : KOG_ROUTINE_LASV2;
  if (!tail_spec.empty()) {
    int lo, hi;
    unsigned mod;
    if (std::sscanf(tail_spec.c_str(), "%d..%d:%u", &lo, &hi, &mod) != 3 || mod == 0)
      return usage("--tail expects LO..HI:MOD");
    cfg.tail_lo = lo;
    cfg.tail_hi = hi;
    cfg.tail_mod = mod;
  }
  try {
    size_t pos = 0;
    cfg.seed = std::stoull(seed_hex, &pos, 16);
    if (pos != seed_hex.size()) throw std::invalid_argument("seed");
  } catch (const std::exception&) {
    std::cerr << "bad --seed, expected hexadecimal\n";
    return 2;
  }
  if (device >= 0 && gpus > 0) return usage("--device and --gpus are exclusive");
  // NCCL's own log lines (NCCL_DEBUG) go to stdout unless redirected: keep the CSV clean
  if (gpus > 0 && !std::getenv("NCCL_DEBUG_FILE")) setenv("NCCL_DEBUG_FILE", "/dev/stderr", 1);
  if (device >= 0 && kog_set_device(device) != KOG_OK) {
    std::cerr << "cannot select CUDA device " << device << "\n";
    return 2;
  }

  std::ofstream file;
  std::ostream* out = &std::cout;
  if (!out_path.empty()) {
    file.open(out_path, std::ios::binary | std::ios::trunc);
    if (!file) {
      std::cerr << "cannot open " << out_path << "\n";
      return 2;
    }
    out = &file;
  }

  char buf[1024];
  kog_csv_header(buf, sizeof buf);
  *out << buf << "\n";
  auto run = [&]() -> int {
    kog_stats st;
    const int rc = gpus > 0 ? kog_study_multi(&cfg, nullptr, gpus, &st, nullptr) : kog_run_batch(&cfg, &st);
    if (rc == KOG_ERR_ABORT) {
      std::cerr << "batch aborted: " << kog_last_error() << "\n";
      return 1;
    }
    if (rc != KOG_OK) {
      std::cerr << kog_last_error() << "\n";
      return 2;
    }
    kog_csv_row(&cfg, &st, buf, sizeof buf);
    *out << buf << "\n";
    return 0;
  };
  if (!sweep_spec.empty()) {  // varsigma=A..B:step, one row per varsigma (svd2batch.cpp:21-27, 84-89)
    int lo = 0, hi = 0, step = 1;
    if (std::sscanf(sweep_spec.c_str(), "varsigma=%d..%d:%d", &lo, &hi, &step) < 2 || step < 1 || hi < lo)
      return usage("--sweep expects varsigma=A..B:step");
    cfg.regime = KOG_REGIME_SIGMA;
    for (int vs = lo; vs <= hi; vs += step) {
      cfg.varsigma = vs;
      const int rc = run();
      if (rc) return rc;
    }
    return 0;
  }
  return run();
}
