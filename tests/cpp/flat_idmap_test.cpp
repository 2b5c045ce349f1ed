// FlatIdMap (paper_2604_00499_b200/csrc/flat_idmap.hpp, the scheduler's id -> slot map) against
// std::unordered_map under a random operation mix: inserts of absent ids, erases, lookups,
// iteration, growth and tombstone rehashes, the two largest uint64 ids.  Host-only (g++).
#include <cstdio>
#include <random>
#include <unordered_map>
#include <vector>

#include "flat_idmap.hpp"

int main() {
  int fail = 0;
  for (int seed = 1; seed <= 3; ++seed) {
    tie::host::FlatIdMap f;
    std::unordered_map<uint64_t, uint32_t> u;
    if (seed == 2) f.reserve(5000);
    std::mt19937_64 r(seed);
    std::vector<uint64_t> pool;
    const uint64_t specials[] = {~0ull, ~0ull - 1, 0ull, 1ull};
    for (int op = 0; op < 400000; ++op) {
      const int kind = (int)(r() % 10);
      uint64_t id;
      if (op < 4) id = specials[op];
      else if (kind < 4) id = seed == 3 ? (uint64_t)op : r();  // sequential ids for seed 3
      else id = pool.empty() ? r() : pool[r() % pool.size()];
      if ((op < 4 || kind < 5) && !u.count(id)) {  // insert (absent)
        const uint32_t v = (uint32_t)r();
        f.emplace(id, v);
        u.emplace(id, v);
        pool.push_back(id);
      } else if (kind < 8) {  // erase (present or not)
        if (f.erase(id) != u.erase(id)) ++fail;
      } else {  // lookup
        auto it = f.find(id);
        auto jt = u.find(id);
        if ((it == f.end()) != (jt == u.end()) || (jt != u.end() && it->second != jt->second))
          ++fail;
        if (f.count(id) != u.count(id)) ++fail;
      }
      if (f.size() != u.size()) ++fail;
      if (op % 50000 == 0) {  // iteration: every live pair exactly once; values writable
        size_t n = 0;
        for (auto& kv : f) {
          auto jt = u.find(kv.first);
          if (jt == u.end() || jt->second != kv.second) ++fail;
          kv.second ^= 1u;
          jt->second ^= 1u;
          ++n;
        }
        if (n != u.size()) ++fail;
      }
    }
  }
  std::printf("flat_idmap_test: %s (%d mismatches)\n", fail ? "FAIL" : "ok", fail);
  return fail ? 1 : 0;
}
