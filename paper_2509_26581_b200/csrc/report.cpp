// Report wire format: the reference's to_json / to_csv (include/gopt/report.hpp:11-73)
// for a gb_solve_report + its IterationRecords, as byte strings.
//
// JSON: the reference builds an nlohmann::json object and callers dump() it
// (src/experiment.cpp:84). nlohmann's default object type is an ordered
// std::map, so dump() writes keys in ascending byte order, compactly, with
// doubles in nlohmann's to_chars form: Grisu2 round-trip digits, plain
// notation for decimal exponents in (-4, 15], scientific otherwise
// ("1e-05", "1.5e+20"), a trailing ".0" on integral values, null for
// non-finite values. This writer reproduces that byte for byte without the
// nlohmann dependency (tests/test_report_cpu.py compares it with the
// reference's own report.hpp compiled against nlohmann 3.11.3).
//
// CSV: report.hpp:51-71 (std::to_string for the '#' header values, %.17g /
// %.6f for the rows).

#include <cstdint>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>

#include "gb_bal.h"

namespace {

const char* term_name(int t) {
  switch (t) {
    case GB_TERM_MAX_ITERATIONS: return "max_iterations";
    case GB_TERM_TOLERANCE_REACHED: return "tolerance_reached";
    case GB_TERM_GRADIENT_SMALL: return "gradient_small";
    case GB_TERM_DAMPING_OVERFLOW: return "damping_overflow";
    case GB_TERM_NON_FINITE_LINEARIZATION: return "non_finite_linearization";
    case GB_TERM_NO_FREE_PARAMETERS: return "no_free_parameters";
  }
  return "?";  // levenberg_marquardt.hpp:46
}

// ---- shortest-digit generation: Grisu2 (Loitsch, "Printing floating-point
// numbers quickly and accurately with integers", PLDI 2010), the variant
// nlohmann/json's to_chars uses: boundaries m-/m+ of the double, one cached
// power of ten that brings the exponent into [-60, -32], digit generation
// between the (conservatively narrowed) boundaries, then the round-towards-v
// correction. Grisu2 is not always the shortest representation (it is always
// a correct round trip), so the digits differ from Ryu / std::to_chars on
// ~1% of values; reproducing nlohmann's bytes needs this exact algorithm.
struct DiyFp {
  uint64_t f;
  int e;
};
DiyFp dsub(DiyFp x, DiyFp y) { return {x.f - y.f, x.e}; }
DiyFp dmul(DiyFp x, DiyFp y) {  // upper 64 bits of the 128-bit product, rounded half up
  const unsigned __int128 p = static_cast<unsigned __int128>(x.f) * y.f;
  const uint64_t h = static_cast<uint64_t>(p >> 64), l = static_cast<uint64_t>(p);
  return {h + (l >> 63), x.e + y.e + 64};
}
DiyFp dnorm(DiyFp x) {
  while ((x.f >> 63) == 0) {
    x.f <<= 1;
    --x.e;
  }
  return x;
}
DiyFp dnorm_to(DiyFp x, int e) { return {x.f << (x.e - e), e}; }

struct CachedPow {
  uint64_t f;
  int e, k;
};
constexpr CachedPow kPow10[] = {
#include "pow10_table.inc"
};

// digits of v into buf (no sign), *len digits, value = digits * 10^*dexp
void grisu2(double v, char* buf, int* len, int* dexp) {
  uint64_t bits;
  std::memcpy(&bits, &v, 8);
  const uint64_t E = bits >> 52, F = bits & ((uint64_t(1) << 52) - 1);
  const DiyFp w = E == 0 ? DiyFp{F, 1 - 1075} : DiyFp{F + (uint64_t(1) << 52), static_cast<int>(E) - 1075};
  const bool lower_closer = F == 0 && E > 1;
  const DiyFp mp{2 * w.f + 1, w.e - 1};
  const DiyFp mm = lower_closer ? DiyFp{4 * w.f - 1, w.e - 2} : DiyFp{2 * w.f - 1, w.e - 1};
  const DiyFp wp = dnorm(mp);
  const DiyFp wm = dnorm_to(mm, wp.e);
  const DiyFp vn = dnorm(w);
  // cached power c = 10^-k with alpha <= e(c * w+) + 64 <= gamma
  const int f = -60 - wp.e - 1;
  const int k = (f * 78913) / (1 << 18) + (f > 0);
  const CachedPow c = kPow10[(300 + k + 7) / 8];
  const DiyFp cm{c.f, c.e};
  const DiyFp W = dmul(vn, cm), Wm = dmul(wm, cm), Wp = dmul(wp, cm);
  const DiyFp Mm{Wm.f + 1, Wm.e}, Mp{Wp.f - 1, Wp.e};
  *dexp = -c.k;
  // digit generation
  uint64_t delta = dsub(Mp, Mm).f, dist = dsub(Mp, W).f;
  const DiyFp one{uint64_t(1) << -Mp.e, Mp.e};
  uint32_t p1 = static_cast<uint32_t>(Mp.f >> -one.e);
  uint64_t p2 = Mp.f & (one.f - 1);
  auto round = [&](uint64_t rest, uint64_t ten_k) {
    while (rest < dist && delta - rest >= ten_k && (rest + ten_k < dist || dist - rest > rest + ten_k - dist)) {
      --buf[*len - 1];
      rest += ten_k;
    }
  };
  uint32_t pow10;
  int n;
  if (p1 >= 1000000000) pow10 = 1000000000, n = 10;
  else if (p1 >= 100000000) pow10 = 100000000, n = 9;
  else if (p1 >= 10000000) pow10 = 10000000, n = 8;
  else if (p1 >= 1000000) pow10 = 1000000, n = 7;
  else if (p1 >= 100000) pow10 = 100000, n = 6;
  else if (p1 >= 10000) pow10 = 10000, n = 5;
  else if (p1 >= 1000) pow10 = 1000, n = 4;
  else if (p1 >= 100) pow10 = 100, n = 3;
  else if (p1 >= 10) pow10 = 10, n = 2;
  else pow10 = 1, n = 1;
  *len = 0;
  while (n > 0) {
    const uint32_t d = p1 / pow10, r = p1 % pow10;
    buf[(*len)++] = static_cast<char>('0' + d);
    p1 = r;
    --n;
    const uint64_t rest = (static_cast<uint64_t>(p1) << -one.e) + p2;
    if (rest <= delta) {
      *dexp += n;
      round(rest, static_cast<uint64_t>(pow10) << -one.e);
      return;
    }
    pow10 /= 10;
  }
  int m = 0;
  for (;;) {
    p2 *= 10;
    const uint64_t d = p2 >> -one.e, r = p2 & (one.f - 1);
    buf[(*len)++] = static_cast<char>('0' + d);
    p2 = r;
    ++m;
    delta *= 10;
    dist *= 10;
    if (p2 <= delta) break;
  }
  *dexp -= m;
  round(p2, one.f);
}

// nlohmann::detail::to_chars of a double: sign, "0.0", Grisu2 digits, then
// plain notation for decimal-point positions in (-4, 15], else scientific
void put_double(std::string& out, double v) {
  if (!std::isfinite(v)) {
    out += "null";
    return;
  }
  if (std::signbit(v)) {
    out += '-';
    v = -v;
  }
  if (v == 0) {
    out += "0.0";
    return;
  }
  char dig[32];
  int k = 0, dexp = 0;
  grisu2(v, dig, &k, &dexp);
  const std::string digits(dig, dig + k);
  const int n = k + dexp;  // position of the decimal point relative to the digits
  constexpr int kMinExp = -4, kMaxExp = 15;
  if (k <= n && n <= kMaxExp) {  // integral: digits, zeros, ".0"
    out += digits;
    out.append(static_cast<size_t>(n - k), '0');
    out += ".0";
  } else if (0 < n && n <= kMaxExp) {  // dddd.ddd
    out += digits.substr(0, static_cast<size_t>(n));
    out += '.';
    out += digits.substr(static_cast<size_t>(n));
  } else if (kMinExp < n && n <= 0) {  // 0.000ddd
    out += "0.";
    out.append(static_cast<size_t>(-n), '0');
    out += digits;
  } else {  // d[.ddd]e+-XX (at least two exponent digits)
    out += digits[0];
    if (k > 1) {
      out += '.';
      out += digits.substr(1);
    }
    const int e = n - 1;
    char eb[16];
    std::snprintf(eb, sizeof(eb), "e%c%02d", e < 0 ? '-' : '+', e < 0 ? -e : e);
    out += eb;
  }
}

struct Writer {
  std::string out;
  void key(const char* k) {
    out += '"';
    out += k;
    out += "\":";
  }
  void num(double v) { put_double(out, v); }
  void integer(long long v) { out += std::to_string(v); }
  void uinteger(unsigned long long v) { out += std::to_string(v); }
  void boolean(bool b) { out += b ? "true" : "false"; }
  void str(const char* s) {
    out += '"';
    out += s;
    out += '"';
  }
};

// keys below are written in ascending byte order (nlohmann's std::map)
void record_json(Writer& w, const gb_iteration_record& r) {
  w.out += '{';
  w.key("accepted"), w.boolean(r.accepted != 0), w.out += ',';
  w.key("chi2_after"), w.num(r.chi2_after), w.out += ',';
  w.key("chi2_before"), w.num(r.chi2_before), w.out += ',';
  w.key("iteration"), w.integer(r.iteration), w.out += ',';
  w.key("lambda"), w.num(r.lambda), w.out += ',';
  w.key("low_quality_step"), w.boolean(r.low_quality_step != 0), w.out += ',';
  w.key("pcg_converged"), w.boolean(r.pcg_converged != 0), w.out += ',';
  w.key("pcg_iterations"), w.integer(r.pcg_iterations), w.out += ',';
  w.key("pcg_relative_residual"), w.num(r.pcg_relative_residual), w.out += ',';
  w.key("precond_fallback_blocks"), w.integer(r.precond_fallback_blocks), w.out += ',';
  w.key("wall_seconds"), w.num(r.wall_seconds);
  w.out += '}';
}

std::string report_json(const gb_solve_report& rep, const gb_iteration_record* recs, int n) {
  Writer w;
  w.out += '{';
  w.key("iterations");
  w.out += '[';
  for (int i = 0; i < n; ++i) {
    if (i) w.out += ',';
    record_json(w, recs[i]);
  }
  w.out += "],";
  w.key("memory_account");
  w.out += '{';
  w.key("graph_bytes"), w.uinteger(rep.memory.graph_bytes), w.out += ',';
  w.key("jacobian_bytes"), w.uinteger(rep.memory.jacobian_bytes), w.out += ',';
  w.key("preconditioner_bytes"), w.uinteger(rep.memory.preconditioner_bytes), w.out += ',';
  w.key("workspace_bytes"), w.uinteger(rep.memory.workspace_bytes);
  w.out += "},";
  w.key("summary");
  w.out += '{';
  w.key("accepted_steps"), w.integer(rep.accepted_steps), w.out += ',';
  w.key("active_factors"), w.uinteger(rep.active_factors), w.out += ',';
  w.key("final_chi2"), w.num(rep.final_chi2), w.out += ',';
  w.key("free_dims"), w.integer(rep.free_dims), w.out += ',';
  w.key("initial_chi2"), w.num(rep.initial_chi2), w.out += ',';
  w.key("iterations_run"), w.uinteger(static_cast<unsigned long long>(n)), w.out += ',';
  w.key("residual_dims"), w.integer(rep.residual_dims), w.out += ',';
  w.key("termination"), w.str(term_name(rep.termination)), w.out += ',';
  w.key("total_seconds"), w.num(rep.total_seconds);
  w.out += "}}";
  return w.out;
}

std::string report_csv(const gb_solve_report& rep, const gb_iteration_record* recs, int n) {
  std::string out;
  auto line = [&out](const std::string& s) { out += s + "\n"; };
  line("# initial_chi2=" + std::to_string(rep.initial_chi2) + " final_chi2=" + std::to_string(rep.final_chi2) +
       " accepted_steps=" + std::to_string(rep.accepted_steps) + " termination=" + term_name(rep.termination));
  line("# jacobian_bytes=" + std::to_string(rep.memory.jacobian_bytes) +
       " preconditioner_bytes=" + std::to_string(rep.memory.preconditioner_bytes) +
       " workspace_bytes=" + std::to_string(rep.memory.workspace_bytes) +
       " graph_bytes=" + std::to_string(rep.memory.graph_bytes));
  line("iteration,chi2_before,chi2_after,lambda,pcg_iterations,pcg_converged,"
       "pcg_relative_residual,low_quality_step,precond_fallback_blocks,accepted,wall_seconds");
  char buf[512];
  for (int i = 0; i < n; ++i) {
    const gb_iteration_record& r = recs[i];
    std::snprintf(buf, sizeof(buf), "%d,%.17g,%.17g,%.17g,%d,%d,%.17g,%d,%d,%d,%.6f", r.iteration, r.chi2_before,
                  r.chi2_after, r.lambda, r.pcg_iterations, r.pcg_converged ? 1 : 0, r.pcg_relative_residual,
                  r.low_quality_step ? 1 : 0, r.precond_fallback_blocks, r.accepted ? 1 : 0, r.wall_seconds);
    line(buf);
  }
  return out;
}

int emit(const std::string& s, char* buf, uint64_t cap, uint64_t* needed) {
  if (needed) *needed = s.size() + 1;
  if (buf && cap) {
    const size_t n = std::min<uint64_t>(cap - 1, s.size());
    std::memcpy(buf, s.data(), n);
    buf[n] = '\0';
  }
  return GB_OK;
}

}  // namespace

extern "C" int gb_report_json(const gb_solve_report* rep, const gb_iteration_record* recs, int32_t n, char* buf,
                              uint64_t cap, uint64_t* needed) {
  if (!rep || (n > 0 && !recs) || n < 0) return GB_ERR_INVALID_ARGUMENT;
  return emit(report_json(*rep, recs, n), buf, cap, needed);
}

extern "C" int gb_report_csv(const gb_solve_report* rep, const gb_iteration_record* recs, int32_t n, char* buf,
                             uint64_t cap, uint64_t* needed) {
  if (!rep || (n > 0 && !recs) || n < 0) return GB_ERR_INVALID_ARGUMENT;
  return emit(report_csv(*rep, recs, n), buf, cap, needed);
}
