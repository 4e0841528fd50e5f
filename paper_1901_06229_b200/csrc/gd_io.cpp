// Ligand ingest: parse_ligand_library (io.cpp:96-140) for the whole library at once, multi-threaded,
// into the flat SoA of the C-ABI (gd_library). Paths are relative to /root/reference/proj.
//
// The .lgd format is a stream of whitespace-separated tokens (the reference's TokenReader splits
// lines on '\n' and tokens on isspace, io.cpp:24-45); record r is
//   ligand NAME atoms n {x y z r}*n bonds m {i j}*m rotamers k {i j}*k end
// The parse is three passes: (1) every thread tokenises a line-aligned slice of the text (token
// start offsets); (2) one sequential walk over the record headers (keywords and counts only, a
// handful of tokens per record) fixes every record's token range and array offsets; (3) threads
// convert the numbers and validate each record (validate_ligand, molecule.cpp:176-238). The error
// reported is the reference's: the first failing token in stream order, where a record's
// validation (run after its "end", io.cpp:136-137) follows its own tokens and precedes the next
// record. Messages and 1-based line numbers match ParseError (errors.hpp:15-27).
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cerrno>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <charconv>
#include <cfloat>
#include <cstring>
#include <memory>
#include <utility>
#include <string>
#include <thread>
#include <vector>

#include "gd_ligand.h"
#include "geodock_b200.h"

struct gd_pocketbuf {
  uint32_t dims[3] = {0, 0, 0};
  double origin[3] = {0, 0, 0};
  double spacing = 0;
  std::vector<double> field;
};

// Allocator whose resize leaves trivially-constructible elements uninitialised: the parser writes
// every element of the big arrays in its parallel pass (a failed parse discards the buffer), so a
// zero fill on one thread first would only cost time (~170 MB per 100k C2 ligands).
template <class T>
struct UninitAlloc : std::allocator<T> {
  template <class U>
  struct rebind {
    using other = UninitAlloc<U>;
  };
  UninitAlloc() = default;
  template <class U>
  UninitAlloc(const UninitAlloc<U>&) noexcept {}
  template <class U>
  void construct(U* p) noexcept {
    ::new (static_cast<void*>(p)) U;
  }
  template <class U, class... A>
  void construct(U* p, A&&... a) {
    ::new (static_cast<void*>(p)) U(std::forward<A>(a)...);
  }
};

struct gd_libbuf {
  std::vector<uint32_t> atom_off, bond_off, rot_off, name_off;
  std::vector<uint32_t, UninitAlloc<uint32_t>> bonds, rots;
  std::vector<double, UninitAlloc<double>> xyz, radius;
  std::vector<double> dihedrals;
  std::string names;
};

namespace {

inline bool is_space(char c) { return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r'; }

template <class F>
void parallel_chunks(size_t n, F&& f) {  // f(chunk, begin, end) over ~hardware_concurrency chunks
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const size_t nt = std::max<size_t>(1, std::min<size_t>(hw, n / 4096 + 1));
  std::vector<std::thread> th;
  for (size_t t = 0; t < nt; ++t) th.emplace_back([&, t] { f(t, n * t / nt, n * (t + 1) / nt); });
  for (auto& x : th) x.join();
}

// Token offsets: written once by the tokeniser's threads, so not zero-filled first (a vector's
// resize would memset ~8 bytes per token on one thread before the parallel pass).
struct Offsets {
  std::unique_ptr<uint64_t[]> p;
  size_t n = 0;
  void resize_uninit(size_t m) {
    p.reset(new uint64_t[m ? m : 1]);
    n = m;
  }
  size_t size() const { return n; }
  uint64_t* data() { return p.get(); }
  uint64_t operator[](size_t i) const { return p[i]; }
};

struct Tok {
  const char* text;
  Offsets start;  // token start offsets, stream order
  size_t len;
  uint64_t end_of(size_t i) const {
    uint64_t e = start[i];
    while (e < len && !is_space(text[e])) ++e;
    return e;
  }
  std::string str(size_t i) const { return std::string(text + start[i], text + end_of(i)); }
  size_t line_of(uint64_t off) const {  // 1-based line of byte offset off
    return size_t(std::count(text, text + off, '\n')) + 1;
  }
  size_t lines() const {  // lines std::getline reads from the whole text
    if (len == 0) return 0;
    return size_t(std::count(text, text + len, '\n')) + (text[len - 1] == '\n' ? 0 : 1);
  }
};

// A token as a NUL-terminated string (stack buffer for the usual short tokens), so strtod never
// reads past it.
struct TokStr {
  char buf[64];
  std::string big;
  const char* p;
  size_t n;
  TokStr(const Tok& tk, size_t i) {
    const uint64_t b = tk.start[i], e = tk.end_of(i);
    n = size_t(e - b);
    if (n < sizeof buf) {
      std::memcpy(buf, tk.text + b, n);
      buf[n] = 0;
      p = buf;
    } else {
      big.assign(tk.text + b, n);
      p = big.c_str();
    }
  }
};

// std::stod / std::stoll with the reference's acceptance rule (whole token, no ERANGE,
// io.cpp:56-82).
// A plain decimal [-]d+[.d*][(e|E)[+-]d+] (or [-].d+...): std::from_chars rounds it correctly, as
// strtod does, so the value is strtod's; anything else (a '+', hex, inf/nan, ...) and any result
// strtod would flag (overflow, underflow, subnormal) takes strtod itself.
bool plain_decimal(const char* p, size_t n, bool& zero_digits) {
  size_t k = 0, digits = 0;
  zero_digits = true;
  if (k < n && p[k] == '-') ++k;
  for (; k < n && p[k] >= '0' && p[k] <= '9'; ++k, ++digits) zero_digits &= p[k] == '0';
  if (k < n && p[k] == '.') {
    ++k;
    for (; k < n && p[k] >= '0' && p[k] <= '9'; ++k, ++digits) zero_digits &= p[k] == '0';
  }
  if (digits == 0) return false;
  if (k < n && (p[k] == 'e' || p[k] == 'E')) {
    ++k;
    if (k < n && (p[k] == '+' || p[k] == '-')) ++k;
    const size_t e0 = k;
    for (; k < n && p[k] >= '0' && p[k] <= '9'; ++k) {
    }
    if (k == e0) return false;
  }
  return k == n;
}

bool to_double(const Tok& tk, size_t i, double& v) {
  {
    const uint64_t b = tk.start[i], e = tk.end_of(i);
    const char* p = tk.text + b;
    bool zero_digits = false;
    if (plain_decimal(p, size_t(e - b), zero_digits)) {
      const auto r = std::from_chars(p, tk.text + e, v);
      if (r.ec == std::errc() && r.ptr == tk.text + e && std::isfinite(v) &&
          (std::fabs(v) >= DBL_MIN || (v == 0.0 && zero_digits)))
        return true;
    }
  }
  const TokStr s(tk, i);
  errno = 0;
  char* end = nullptr;
  v = std::strtod(s.p, &end);
  return end == s.p + s.n && end != s.p && errno != ERANGE;
}

bool to_index(const Tok& tk, size_t i, uint64_t& v) {
  {  // plain digits (at most 18: no overflow) are strtoll's value
    const uint64_t b = tk.start[i], e = tk.end_of(i);
    if (e > b && e - b <= 18) {
      uint64_t x = 0;
      uint64_t k = b;
      for (; k < e && tk.text[k] >= '0' && tk.text[k] <= '9'; ++k) x = 10 * x + uint64_t(tk.text[k] - '0');
      if (k == e) {
        v = x;
        return true;
      }
    }
  }
  const TokStr s(tk, i);
  errno = 0;
  char* end = nullptr;
  const long long x = std::strtoll(s.p, &end, 10);
  if (end != s.p + s.n || end == s.p || errno == ERANGE || x < 0) return false;
  v = uint64_t(x);
  return true;
}

bool tok_is(const Tok& tk, size_t i, const char* kw) {
  const size_t n = std::strlen(kw);
  return tk.end_of(i) - tk.start[i] == n && std::memcmp(tk.text + tk.start[i], kw, n) == 0;
}

// ParseError's message suffix (errors.hpp:18-20): none when the line is unknown (0)
std::string line_suffix(size_t line) { return line > 0 ? " (line " + std::to_string(line) + ")" : std::string(); }

struct Err {  // a ParseError / ValidationError candidate at a stream position
  uint64_t pos = ~0ull;  // token index (validation: the record's "end" token + 0.5 -> 2*idx+1)
  int code = GD_OK;
  std::string msg;
  void set(uint64_t p, int c, std::string m) {
    if (p < pos) {
      pos = p;
      code = c;
      msg = std::move(m);
    }
  }
};

struct Rec {
  uint64_t tok = 0;                               // token index of "ligand"
  uint64_t n = 0, m = 0, k = 0;                   // atoms, bonds, rotamers
  uint64_t atom0 = 0, bond0 = 0, rot0 = 0, name0 = 0;
  static Rec of(uint64_t tok, uint64_t n, uint64_t m, uint64_t k) {
    Rec r;
    r.tok = tok;
    r.n = n;
    r.m = m;
    r.k = k;
    return r;
  }
};

}  // namespace

extern "C" {

int gd_parse_library(const char* text, size_t len, gd_libbuf** out, char* err, uint32_t cap) {
  if (!out || (!text && len)) return GD_ERR_ARGUMENT;
  *out = nullptr;
  auto fail = [&](int code, const std::string& msg) {
    if (err && cap) std::snprintf(err, cap, "%s", msg.c_str());
    return code;
  };
  const bool trace = std::getenv("GD_TRACE_PARSE") != nullptr;
  auto now = [] { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count(); };
  const double t_start = now();
  // (1) tokens, one line-aligned slice per thread
  Tok tk{text, {}, len};
  {
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const size_t nt = std::max<size_t>(1, std::min<size_t>(hw, len / (1 << 16) + 1));
    std::vector<size_t> cut(nt + 1, len);
    cut[0] = 0;
    for (size_t t = 1; t < nt; ++t) {
      size_t c = len * t / nt;
      while (c < len && text[c] != '\n') ++c;
      cut[t] = std::max(cut[t - 1], std::min(len, c + (c < len ? 1 : 0)));
    }
    // two passes over each slice: count its tokens, then write their offsets in place
    std::vector<size_t> ntok(nt + 1, 0);
    auto scan = [&](size_t t, uint64_t* dst) {
      bool in = false;
      size_t k = 0;
      for (size_t i = cut[t]; i < cut[t + 1]; ++i) {
        const bool sp = is_space(text[i]);
        if (!sp && !in) {
          if (dst) dst[k] = i;
          ++k;
        }
        in = !sp;
      }
      return k;
    };
    {
      std::vector<std::thread> th;
      for (size_t t = 0; t < nt; ++t) th.emplace_back([&, t] { ntok[t + 1] = scan(t, nullptr); });
      for (auto& x : th) x.join();
    }
    for (size_t t = 0; t < nt; ++t) ntok[t + 1] += ntok[t];
    tk.start.resize_uninit(ntok[nt]);
    {
      std::vector<std::thread> th;
      for (size_t t = 0; t < nt; ++t) th.emplace_back([&, t] { scan(t, tk.start.data() + ntok[t]); });
      for (auto& x : th) x.join();
    }
  }
  const uint64_t T = tk.start.size();
  const double t_tok = now();
  auto at_eof = [&](const char* what) {
    return Err{T, GD_ERR_PARSE, std::string("unexpected end of input, expected ") + what + line_suffix(tk.lines())};
  };
  auto tok_err = [&](uint64_t i, const std::string& m) {
    return m + line_suffix(tk.line_of(tk.start[i]));
  };
  // (2) record headers: the reference's walk (with its errors) — sequential, resumable at any
  // record start, bounded by `limit`; `stop` once it has reported an error
  std::vector<Rec> recs;
  Err e;
  uint64_t i = 0, na = 0, nb = 0, nr = 0, nn = 0;
  auto keyword = [&](uint64_t at, const char* kw) -> bool {
    if (at >= T) {
      const Err x = at_eof(kw);
      e.set(x.pos, x.code, x.msg);
      return false;
    }
    if (!tok_is(tk, at, kw)) {
      e.set(at, GD_ERR_PARSE, tok_err(at, std::string("expected '") + kw + "', got '" + tk.str(at) + "'"));
      return false;
    }
    return true;
  };
  auto count = [&](uint64_t at, const char* what, uint64_t& v) -> bool {
    if (at >= T) {
      const Err x = at_eof(what);
      e.set(x.pos, x.code, x.msg);
      return false;
    }
    if (!to_index(tk, at, v)) {
      e.set(at, GD_ERR_PARSE,
            tok_err(at, std::string("expected a non-negative integer for ") + what + ", got '" + tk.str(at) + "'"));
      return false;
    }
    return true;
  };
  bool stop = false;
  auto seq_walk = [&](uint64_t limit) {
  while (i < T && i < limit) {
    if (!tok_is(tk, i, "ligand")) {
      e.set(i, GD_ERR_PARSE, tok_err(i, "expected 'ligand', got '" + tk.str(i) + "'"));
      stop = true;
      break;
    }
    Rec r;
    r.tok = i;
    if (i + 1 >= T) {
      const Err x = at_eof("ligand name");
      e.set(x.pos, x.code, x.msg);
      stop = true;
      break;
    }
    if (!keyword(i + 2, "atoms") || !count(i + 3, "atom count", r.n)) {
      stop = true;
      break;
    }
    // body sizes; a count the text cannot hold ends at the end of input inside the record
    uint64_t p = i + 4 + 4 * std::min<uint64_t>(r.n, T);
    if (p > T) {  // numbers run out: the reference fails on the first missing one
      const uint64_t have = T - (i + 4);
      static const char* what[4] = {"atom x", "atom y", "atom z", "atom radius"};
      const Err x = at_eof(what[have % 4]);
      e.set(x.pos, x.code, x.msg);
      r.n = have / 4;  // the complete atoms still get their numbers checked below
      r.m = r.k = 0;
      recs.push_back(r);
      stop = true;
      break;
    }
    if (!keyword(p, "bonds") || !count(p + 1, "bond count", r.m)) {
      recs.push_back(Rec::of(r.tok, r.n, 0, 0));
      stop = true;
      break;
    }
    p += 2;
    if (p + 2 * std::min<uint64_t>(r.m, T) > T) {
      const uint64_t have = T - p;
      const Err x = at_eof(have % 2 ? "bond atom j" : "bond atom i");
      e.set(x.pos, x.code, x.msg);
      recs.push_back(Rec::of(r.tok, r.n, have / 2, 0));
      stop = true;
      break;
    }
    p += 2 * r.m;
    if (!keyword(p, "rotamers") || !count(p + 1, "rotamer count", r.k)) {
      recs.push_back(Rec::of(r.tok, r.n, r.m, 0));
      stop = true;
      break;
    }
    p += 2;
    if (p + 2 * std::min<uint64_t>(r.k, T) > T) {
      const uint64_t have = T - p;
      const Err x = at_eof(have % 2 ? "rotamer atom j" : "rotamer atom i");
      e.set(x.pos, x.code, x.msg);
      recs.push_back(Rec::of(r.tok, r.n, r.m, have / 2));
      stop = true;
      break;
    }
    p += 2 * r.k;
    if (!keyword(p, "end")) {
      recs.push_back(r);
      stop = true;
      break;
    }
    recs.push_back(r);
    i = p + 1;
  }
  };
  // The walk in parallel: every thread follows the record chain from the first plausible record
  // start ("ligand" NAME "atoms") of its token slice, structure only (no error text). A slice's
  // chain is adopted when the reference walk arrives at one of its record starts — a walk from a
  // true record start is deterministic, so the records are the ones it would find — and the
  // reference walk crosses the rest itself (a slice whose chain began at a false start, or stopped
  // at a malformed record, which it then reports exactly as before).
  {
    constexpr uint64_t NONE = ~0ull;
    auto walk_one = [&](uint64_t at, Rec& r) -> uint64_t {
      uint64_t n = 0, m = 0, k = 0;
      if (at + 3 >= T || !tok_is(tk, at, "ligand") || !tok_is(tk, at + 2, "atoms") || !to_index(tk, at + 3, n) ||
          n > T)
        return NONE;
      uint64_t p = at + 4 + 4 * n;
      if (p + 1 >= T || !tok_is(tk, p, "bonds") || !to_index(tk, p + 1, m) || m > T) return NONE;
      p += 2 + 2 * m;
      if (p + 1 >= T || !tok_is(tk, p, "rotamers") || !to_index(tk, p + 1, k) || k > T) return NONE;
      p += 2 + 2 * k;
      if (p >= T || !tok_is(tk, p, "end")) return NONE;
      r = Rec::of(at, n, m, k);
      return p + 1;
    };
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const size_t nt = std::max<size_t>(1, std::min<size_t>(hw, size_t(T / 65536) + 1));
    std::vector<uint64_t> cut(nt + 1);
    for (size_t t = 0; t <= nt; ++t) cut[t] = T * t / nt;
    std::vector<std::vector<Rec>> srec(nt);
    std::vector<uint64_t> snext(nt, NONE);
    {
      std::vector<std::thread> th;
      for (size_t t = 1; t < nt; ++t)
        th.emplace_back([&, t] {
          uint64_t j = cut[t];
          while (j + 3 < T && j < cut[t + 1] && !(tok_is(tk, j, "ligand") && tok_is(tk, j + 2, "atoms"))) ++j;
          while (j < cut[t + 1]) {
            Rec r;
            const uint64_t nx = walk_one(j, r);
            if (nx == NONE) break;
            srec[t].push_back(r);
            j = nx;
          }
          snext[t] = j;
        });
      for (auto& x : th) x.join();
    }
    for (size_t t = 0; t < nt && !stop && i < T; ++t) {
      if (i >= cut[t + 1]) continue;
      if (t > 0 && !srec[t].empty()) {
        const auto it = std::lower_bound(srec[t].begin(), srec[t].end(), i,
                                         [](const Rec& r, uint64_t v) { return r.tok < v; });
        if (it != srec[t].end() && it->tok == i) {
          recs.insert(recs.end(), it, srec[t].end());
          i = snext[t];
        }
      }
      seq_walk(cut[t + 1]);
    }
    if (!stop) seq_walk(T);
  }
  // offsets (also for the partial record an early error left behind)
  for (Rec& r : recs) {
    r.atom0 = na;
    r.bond0 = nb;
    r.rot0 = nr;
    r.name0 = nn;
    na += r.n;
    nb += r.m;
    nr += r.k;
    nn += (r.tok + 1 < T) ? tk.end_of(r.tok + 1) - tk.start[r.tok + 1] : 0;
  }
  const bool complete = e.code == GD_OK;
  if (na > 0xffffffffull || nb > 0xffffffffull || nr > 0xffffffffull || recs.size() > 0xffffffffull)
    return fail(GD_ERR_UNSUPPORTED, "library too large for 32-bit offsets");
  auto* b = new gd_libbuf();
  const size_t L = recs.size();
  b->atom_off.resize(L + 1);
  b->bond_off.resize(L + 1);
  b->rot_off.resize(L + 1);
  b->name_off.resize(L + 1);
  for (size_t l = 0; l < L; ++l) {
    b->atom_off[l] = uint32_t(recs[l].atom0);
    b->bond_off[l] = uint32_t(recs[l].bond0);
    b->rot_off[l] = uint32_t(recs[l].rot0);
    b->name_off[l] = uint32_t(recs[l].name0);
  }
  b->atom_off[L] = uint32_t(na);
  b->bond_off[L] = uint32_t(nb);
  b->rot_off[L] = uint32_t(nr);
  b->name_off[L] = uint32_t(nn);
  b->xyz.resize(3 * na);
  b->radius.resize(na);
  b->bonds.resize(2 * nb);
  b->rots.resize(2 * nr);
  b->dihedrals.assign(nr, 0.0);  // io.cpp:134
  b->names.resize(nn);
  const double t_walk = now();
  // (3) numbers + validation, per record in parallel; each record keeps its first error
  std::vector<Err> rerr(L);
  std::atomic<uint64_t> first_bad{L};
  parallel_chunks(L, [&](size_t, size_t lo, size_t hi) {
    for (size_t l = lo; l < hi; ++l) {
      if (l > first_bad.load(std::memory_order_relaxed)) break;
      const Rec& r = recs[l];
      Err& re = rerr[l];
      if (r.tok + 1 < T) {
        const std::string nm = tk.str(r.tok + 1);
        std::memcpy(&b->names[r.name0], nm.data(), nm.size());
      }
      static const char* awhat[4] = {"atom x", "atom y", "atom z", "atom radius"};
      uint64_t t = r.tok + 4;
      for (uint64_t a = 0; a < r.n && re.code == GD_OK; ++a)
        for (int c = 0; c < 4; ++c, ++t) {
          double v;
          if (!to_double(tk, t, v)) {
            re.set(t, GD_ERR_PARSE,
                   tok_err(t, std::string("expected a number for ") + awhat[c] + ", got '" + tk.str(t) + "'"));
            break;
          }
          if (c < 3) b->xyz[3 * (r.atom0 + a) + c] = v;
          else b->radius[r.atom0 + a] = v;
        }
      // indices: values above 32 bits are out of range for any real ligand (stored clamped); a bond
      // with such an index switches to the 64-bit restatement of validate_ligand below
      bool big_bond = false;
      auto idx = [&](uint64_t at, const char* what, uint32_t& dst, bool bond) -> bool {
        uint64_t v;
        if (!to_index(tk, at, v)) {
          re.set(at, GD_ERR_PARSE,
                 tok_err(at, std::string("expected a non-negative integer for ") + what + ", got '" + tk.str(at) + "'"));
          return false;
        }
        dst = v > 0xffffffffull ? 0xffffffffu : uint32_t(v);
        big_bond |= bond && v > 0xffffffffull;
        return true;
      };
      const uint64_t tb = r.tok + 4 + 4 * r.n + 2, trt = tb + 2 * r.m + 2;
      for (uint64_t q = 0; q < r.m && re.code == GD_OK; ++q)
        if (!idx(tb + 2 * q, "bond atom i", b->bonds[2 * (r.bond0 + q)], true) ||
            !idx(tb + 2 * q + 1, "bond atom j", b->bonds[2 * (r.bond0 + q) + 1], true))
          break;
      for (uint64_t q = 0; q < r.k && re.code == GD_OK; ++q)
        if (!idx(trt + 2 * q, "rotamer atom i", b->rots[2 * (r.rot0 + q)], false) ||
            !idx(trt + 2 * q + 1, "rotamer atom j", b->rots[2 * (r.rot0 + q) + 1], false))
          break;
      // validate_ligand after "end" (io.cpp:136-137), only for a record that parsed completely
      const bool whole = complete || l + 1 < L;
      if (re.code == GD_OK && whole) {
        std::vector<std::string> v;
        if (!big_bond) {
          gd_library one{};
          const uint32_t ao[2] = {0, uint32_t(r.n)}, bo[2] = {0, uint32_t(r.m)}, ro[2] = {0, uint32_t(r.k)},
                         no[2] = {0, uint32_t(b->name_off[l + 1] - b->name_off[l])};
          one.n_ligands = 1;
          one.atom_off = ao;
          one.xyz = b->xyz.data() + 3 * r.atom0;
          one.radius = b->radius.data() + r.atom0;
          one.bond_off = bo;
          one.bonds = b->bonds.data() + 2 * r.bond0;
          one.rot_off = ro;
          one.rots = b->rots.data() + 2 * r.rot0;
          one.name_off = no;
          one.names = b->names.data() + r.name0;
          v = gdl::validate(gdl::view_of(&one, 0));
        } else {
          // a bond index >= 2^32 >= n: validate_ligand stops after the per-atom, bond-range,
          // self-bond and rotamer-count checks (molecule.cpp:176-203); self-bonds print the
          // parsed (size_t) value
          if (r.n == 0) v.push_back("ligand has no atoms");
          for (uint64_t a = 0; a < r.n; ++a) {
            const double* x = &b->xyz[3 * (r.atom0 + a)];
            if (!(b->radius[r.atom0 + a] > 0.0)) v.push_back("atom " + std::to_string(a) + " has non-positive radius");
            if (!std::isfinite(x[0]) || !std::isfinite(x[1]) || !std::isfinite(x[2]))
              v.push_back("atom " + std::to_string(a) + " has non-finite coordinates");
          }
          if (r.n > 0) {
            v.push_back("bond index out of range");
            for (uint64_t q = 0; q < r.m; ++q) {
              uint64_t x = 0, y = 0;
              to_index(tk, tb + 2 * q, x);
              to_index(tk, tb + 2 * q + 1, y);
              if (x == y) v.push_back("self-bond on atom " + std::to_string(x));
            }
            if (r.k > GD_MAX_ROTAMERS)
              v.push_back("rotamer count exceeds the supported limit of " + std::to_string(GD_MAX_ROTAMERS));
          }
        }
        if (!v.empty()) re.set(trt + 2 * r.k, GD_ERR_INVALID_LIGAND, gdl::validation_message(tk.str(r.tok + 1), v));
      }
      if (re.code != GD_OK) {
        uint64_t cur = first_bad.load();
        while (l < cur && !first_bad.compare_exchange_weak(cur, l)) {
        }
      }
    }
  });
  if (trace)
    std::fprintf(stderr, "parse: tokens %.1f ms, headers %.1f ms, numbers+validation %.1f ms (%zu records)\n",
                 t_tok - t_start, t_walk - t_tok, now() - t_walk, L);
  Err best = e;
  for (size_t l = 0; l < L; ++l)
    if (rerr[l].code != GD_OK) {
      // validation errors sit at the record's "end" token; a parse error in the same record
      // precedes it (lower token index) and later records' errors come after it
      best.set(rerr[l].pos, rerr[l].code, rerr[l].msg);
      break;
    }
  if (best.code != GD_OK) {
    delete b;
    return fail(best.code, best.msg);
  }
  *out = b;
  return GD_OK;
}

int gd_libbuf_view(const gd_libbuf* b, gd_library* v) {
  if (!b || !v) return GD_ERR_ARGUMENT;
  v->n_ligands = uint32_t(b->atom_off.size() - 1);
  v->atom_off = b->atom_off.data();
  v->xyz = b->xyz.data();
  v->radius = b->radius.data();
  v->bond_off = b->bond_off.data();
  v->bonds = b->bonds.data();
  v->rot_off = b->rot_off.data();
  v->rots = b->rots.data();
  v->dihedrals = b->dihedrals.data();
  v->name_off = b->name_off.data();
  v->names = b->names.data();
  return GD_OK;
}

void gd_libbuf_free(gd_libbuf* b) { delete b; }

// parse_pocket (io.cpp:162-206): header, then dims[0]*dims[1]*dims[2] field values in [0, 1]
// (x-fastest), nothing after them. Sequential (a pocket is at most a few hundred thousand values);
// messages as ParseError / RangeError (errors.hpp:15-33).
int gd_parse_pocket(const char* text, size_t len, gd_pocketbuf** out, char* err, uint32_t cap) {
  if (!out || (!text && len)) return GD_ERR_ARGUMENT;
  *out = nullptr;
  auto fail = [&](const std::string& msg) {
    if (err && cap) std::snprintf(err, cap, "%s", msg.c_str());
    return GD_ERR_PARSE;
  };
  Tok tk{text, {}, len};
  {
    std::vector<uint64_t> st;
    bool in = false;
    for (size_t i = 0; i < len; ++i) {
      const bool sp = is_space(text[i]);
      if (!sp && !in) st.push_back(i);
      in = !sp;
    }
    tk.start.resize_uninit(st.size());
    std::copy(st.begin(), st.end(), tk.start.data());
  }
  const uint64_t T = tk.start.size();
  uint64_t i = 0;
  // line of the reader after consuming token i (its own line) / at the end of input
  auto at_line = [&](uint64_t t) { return line_suffix(tk.line_of(tk.start[t])); };
  auto eof_line = [&]() { return line_suffix(tk.lines()); };
  std::string msg;
  auto keyword = [&](const char* kw) -> bool {
    if (i >= T) {
      msg = std::string("unexpected end of input, expected ") + kw + eof_line();
      return false;
    }
    if (!tok_is(tk, i, kw)) {
      msg = std::string("expected '") + kw + "', got '" + tk.str(i) + "'" + at_line(i);
      return false;
    }
    ++i;
    return true;
  };
  auto number = [&](const char* what, double& v) -> bool {
    if (i >= T) {
      msg = std::string("unexpected end of input, expected ") + what + eof_line();
      return false;
    }
    if (!to_double(tk, i, v)) {
      msg = std::string("expected a number for ") + what + ", got '" + tk.str(i) + "'" + at_line(i);
      return false;
    }
    ++i;
    return true;
  };
  auto index = [&](const char* what, uint64_t& v) -> bool {
    if (i >= T) {
      msg = std::string("unexpected end of input, expected ") + what + eof_line();
      return false;
    }
    if (!to_index(tk, i, v)) {
      msg = std::string("expected a non-negative integer for ") + what + ", got '" + tk.str(i) + "'" + at_line(i);
      return false;
    }
    ++i;
    return true;
  };
  auto* p = new gd_pocketbuf();
  uint64_t d[3] = {0, 0, 0};
  const bool ok = keyword("origin") && number("origin x", p->origin[0]) && number("origin y", p->origin[1]) &&
                  number("origin z", p->origin[2]) && keyword("spacing") && number("spacing", p->spacing) &&
                  ([&] {
                    if (!(p->spacing > 0.0)) {
                      msg = "spacing must be positive" + at_line(i - 1);
                      return false;
                    }
                    return true;
                  }()) &&
                  keyword("dims") && index("nx", d[0]) && index("ny", d[1]) && index("nz", d[2]) && ([&] {
                    if (d[0] < 2 || d[1] < 2 || d[2] < 2) {
                      msg = "dims must each be >= 2" + at_line(i - 1);
                      return false;
                    }
                    if (d[0] > 0xffffffffull || d[1] > 0xffffffffull || d[2] > 0xffffffffull) {
                      msg = "dims too large for this build";
                      return false;
                    }
                    return true;
                  }());
  if (!ok) {
    delete p;
    return fail(msg);
  }
  const uint64_t expected = d[0] * d[1] * d[2];
  while (p->field.size() < expected && i < T) {
    double v;
    if (!to_double(tk, i, v)) {
      delete p;
      return fail("expected a field value, got '" + tk.str(i) + "'" + at_line(i));
    }
    if (v < 0.0 || v > 1.0) {
      char num[40];
      std::snprintf(num, sizeof num, "%.9g", v);  // format_double, io.cpp:14-18
      const std::string m = std::string("field value ") + num + " outside [0,1]" + at_line(i);
      delete p;
      return fail(m);
    }
    p->field.push_back(v);
    ++i;
  }
  if (p->field.size() != expected) {
    const std::string m = "expected " + std::to_string(expected) + " values, got " + std::to_string(p->field.size()) +
                          eof_line();
    delete p;
    return fail(m);
  }
  if (i < T) {
    const std::string m = "trailing content after field values: '" + tk.str(i) + "'" + at_line(i);
    delete p;
    return fail(m);
  }
  for (int a = 0; a < 3; ++a) p->dims[a] = uint32_t(d[a]);
  *out = p;
  return GD_OK;
}

int gd_pocketbuf_view(const gd_pocketbuf* p, uint32_t dims[3], double origin[3], double* spacing, const double** field) {
  if (!p || !dims || !origin || !spacing || !field) return GD_ERR_ARGUMENT;
  for (int a = 0; a < 3; ++a) {
    dims[a] = p->dims[a];
    origin[a] = p->origin[a];
  }
  *spacing = p->spacing;
  *field = p->field.data();
  return GD_OK;
}

void gd_pocketbuf_free(gd_pocketbuf* p) { delete p; }

}  // extern "C"
