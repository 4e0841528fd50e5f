// Ligand graph helpers shared by the C-ABI host code (gd_capi.cpp) and the library parser
// (gd_io.cpp): the flat per-ligand view, adjacency lists, reachability and validate_ligand
// (molecule.cpp:176-238) with the reference's exact messages. Host-only, internal.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <string>
#include <string_view>
#include <vector>

#include "geodock_b200.h"

namespace gdl {

// ------------------------------------------------------------------ ligand graph checks
// validate_ligand (molecule.cpp:176-238) restated over the flat layout. Messages match the
// reference's so ValidationError text is identical.
struct LigView {
  uint32_t n, nb, nr;
  const double* xyz;
  const double* radius;
  const uint32_t* bonds;
  const uint32_t* rots;
  std::string_view name;
};

inline LigView view_of(const gd_library* lib, uint32_t l) {
  LigView v;
  v.n = lib->atom_off[l + 1] - lib->atom_off[l];
  v.nb = lib->bond_off[l + 1] - lib->bond_off[l];
  v.nr = lib->rot_off[l + 1] - lib->rot_off[l];
  v.xyz = lib->xyz + 3 * size_t(lib->atom_off[l]);
  v.radius = lib->radius + lib->atom_off[l];
  v.bonds = lib->bonds + 2 * size_t(lib->bond_off[l]);
  v.rots = lib->rots + 2 * size_t(lib->rot_off[l]);
  v.name = std::string_view(lib->names + lib->name_off[l], lib->name_off[l + 1] - lib->name_off[l]);
  return v;
}

struct Adj {
  std::vector<uint32_t> start, nbr;  // CSR
};

inline Adj adjacency(const LigView& v) {  // adjacency_lists (molecule.cpp:12-20)
  Adj a;
  a.start.assign(v.n + 1, 0);
  for (uint32_t b = 0; b < v.nb; ++b) {
    a.start[v.bonds[2 * b] + 1]++;
    a.start[v.bonds[2 * b + 1] + 1]++;
  }
  for (uint32_t i = 0; i < v.n; ++i) a.start[i + 1] += a.start[i];
  a.nbr.resize(a.start[v.n]);
  std::vector<uint32_t> fill(a.start.begin(), a.start.end() - 1);
  for (uint32_t b = 0; b < v.nb; ++b) {
    const uint32_t x = v.bonds[2 * b], y = v.bonds[2 * b + 1];
    a.nbr[fill[x]++] = y;
    a.nbr[fill[y]++] = x;
  }
  return a;
}

// reachable (molecule.cpp:22-41) with one edge optionally deleted.
inline void reachable(const Adj& a, uint32_t n, uint32_t start, uint32_t skip_a, uint32_t skip_b,
               std::vector<char>& seen, std::vector<uint32_t>& stack) {
  seen.assign(n, 0);
  stack.clear();
  stack.push_back(start);
  seen[start] = 1;
  while (!stack.empty()) {
    const uint32_t u = stack.back();
    stack.pop_back();
    for (uint32_t e = a.start[u]; e < a.start[u + 1]; ++e) {
      const uint32_t w = a.nbr[e];
      if ((u == skip_a && w == skip_b) || (u == skip_b && w == skip_a)) continue;
      if (!seen[w]) {
        seen[w] = 1;
        stack.push_back(w);
      }
    }
  }
}

inline std::vector<std::string> validate(const LigView& v) {
  std::vector<std::string> out;
  const uint32_t n = v.n;
  if (n == 0) {
    out.push_back("ligand has no atoms");
    return out;
  }
  for (uint32_t a = 0; a < n; ++a) {
    if (!(v.radius[a] > 0.0)) out.push_back("atom " + std::to_string(a) + " has non-positive radius");
    if (!std::isfinite(v.xyz[3 * a]) || !std::isfinite(v.xyz[3 * a + 1]) || !std::isfinite(v.xyz[3 * a + 2])) {
      out.push_back("atom " + std::to_string(a) + " has non-finite coordinates");
    }
  }
  bool indices_ok = true;
  for (uint32_t b = 0; b < v.nb; ++b) {
    if (v.bonds[2 * b] >= n || v.bonds[2 * b + 1] >= n) indices_ok = false;
  }
  if (!indices_ok) out.push_back("bond index out of range");
  for (uint32_t b = 0; b < v.nb; ++b) {
    if (v.bonds[2 * b] == v.bonds[2 * b + 1]) out.push_back("self-bond on atom " + std::to_string(v.bonds[2 * b]));
  }
  if (v.nr > GD_MAX_ROTAMERS) {
    out.push_back("rotamer count exceeds the supported limit of " + std::to_string(GD_MAX_ROTAMERS));
  }
  if (!indices_ok) return out;
  const Adj adj = adjacency(v);
  std::vector<char> seen;
  std::vector<uint32_t> stack;
  reachable(adj, n, 0, ~0u, ~0u, seen, stack);
  if (std::find(seen.begin(), seen.end(), 0) != seen.end()) {
    out.push_back("bond graph is not connected");
    return out;
  }
  for (uint32_t r = 0; r < v.nr; ++r) {
    const uint32_t i = v.rots[2 * r], j = v.rots[2 * r + 1];
    if (i >= n || j >= n) {
      out.push_back("rotamer " + std::to_string(r) + " atom index out of range");
      continue;
    }
    bool bonded = false;
    for (uint32_t e = adj.start[i]; e < adj.start[i + 1]; ++e) bonded |= adj.nbr[e] == j;
    if (!bonded) {
      out.push_back("rotamer bond (" + std::to_string(i) + "," + std::to_string(j) + ") is not a bond");
      continue;
    }
    reachable(adj, n, j, i, j, seen, stack);
    if (seen[i]) {
      out.push_back("rotamer bond (" + std::to_string(i) + "," + std::to_string(j) +
                    ") does not disconnect graph");
    }
  }
  return out;
}

inline std::string validation_message(std::string_view name, const std::vector<std::string>& v) {
  std::string msg = "ligand '" + std::string(name) + "' is invalid:";  // errors.hpp:37-41
  for (const auto& s : v) msg += " [" + s + "]";
  return msg;
}


}  // namespace gdl
