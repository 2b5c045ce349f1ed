// Request id -> queue slot index of the scheduler's host mirror (the reference heap's pos_
// map, sched.hpp:67): an open-addressing table with linear probing, replacing a node-based
// std::unordered_map.  A scheduler step touches ~100 random ids (arrival checks + inserts,
// prediction lookups, pop erases); with millions of waiting requests each is a cache miss, and
// a node map pays two (bucket + node) plus an allocation per insert.  Here an entry is one
// 16-byte cell (one miss per lookup) and inserts do not allocate.
//
// Interface: the subset of std::unordered_map<uint64_t, uint32_t> the queue uses (count, find
// / end, emplace of an absent key, erase, reserve, size, iteration over {first, second}).
// Any uint64_t is a valid id (the cell state is a separate field, no sentinel keys).
#pragma once

#include <cstddef>
#include <cstdint>
#include <vector>

namespace tie::host {

class FlatIdMap {
 public:
  struct Cell {
    uint64_t first;   // id
    uint32_t second;  // slot
    uint32_t state;   // kEmpty / kFull / kGone (tombstone)
  };
  static constexpr uint32_t kEmpty = 0, kFull = 1, kGone = 2;

  class iterator {
   public:
    iterator(Cell* c, Cell* e) : c_(c), e_(e) { skip(); }
    Cell& operator*() const { return *c_; }
    Cell* operator->() const { return c_; }
    iterator& operator++() {
      ++c_;
      skip();
      return *this;
    }
    bool operator==(const iterator& o) const { return c_ == o.c_; }
    bool operator!=(const iterator& o) const { return c_ != o.c_; }

   private:
    void skip() {
      while (c_ != e_ && c_->state != kFull) ++c_;
    }
    Cell* c_;
    Cell* e_;
  };

  FlatIdMap() { rehash(16); }

  size_t size() const { return n_; }
  iterator begin() { return iterator(cells_.data(), cells_.data() + cells_.size()); }
  iterator end() { return iterator(cells_.data() + cells_.size(), cells_.data() + cells_.size()); }

  void reserve(size_t n) {
    size_t cap = 16;
    while (cap < 2 * n) cap <<= 1;
    if (cap > cells_.size()) rehash(cap);
  }

  iterator find(uint64_t id) {
    const size_t i = locate(id);
    return i == kNone ? end() : iterator(cells_.data() + i, cells_.data() + cells_.size());
  }
  // read-only views (the iterator type is shared; const callers do not write through it)
  iterator begin() const { return const_cast<FlatIdMap*>(this)->begin(); }
  iterator end() const { return const_cast<FlatIdMap*>(this)->end(); }
  iterator find(uint64_t id) const { return const_cast<FlatIdMap*>(this)->find(id); }
  size_t count(uint64_t id) const { return locate(id) == kNone ? 0 : 1; }

  // insert an id that is not present (the callers have checked); returns true
  bool emplace(uint64_t id, uint32_t slot) {
    if (2 * (n_ + gone_ + 1) > cells_.size())  // load (live + tombstones) <= 1/2
      rehash(4 * (n_ + 1) > cells_.size() ? 2 * cells_.size() : cells_.size());
    size_t i = home(id);
    while (cells_[i].state == kFull) i = (i + 1) & mask_;
    if (cells_[i].state == kGone) --gone_;
    cells_[i] = Cell{id, slot, kFull};
    ++n_;
    return true;
  }

  size_t erase(uint64_t id) {
    const size_t i = locate(id);
    if (i == kNone) return 0;
    cells_[i].state = kGone;
    --n_;
    ++gone_;
    return 1;
  }

 private:
  static constexpr size_t kNone = ~size_t(0);
  size_t home(uint64_t id) const {  // Fibonacci hashing: the top bits of id * 2^64/phi
    return (size_t)((id * 0x9E3779B97F4A7C15ull) >> shift_);
  }
  size_t locate(uint64_t id) const {
    for (size_t i = home(id);; i = (i + 1) & mask_) {
      const Cell& c = cells_[i];
      if (c.state == kEmpty) return kNone;
      if (c.state == kFull && c.first == id) return i;
    }
  }
  void rehash(size_t cap) {  // cap: a power of two; drops the tombstones
    std::vector<Cell> old;
    old.swap(cells_);
    cells_.assign(cap, Cell{0, 0, kEmpty});
    mask_ = cap - 1;
    shift_ = 64;
    for (size_t c = cap; c > 1; c >>= 1) --shift_;
    n_ = gone_ = 0;
    for (const Cell& c : old)
      if (c.state == kFull) {
        size_t i = home(c.first);
        while (cells_[i].state == kFull) i = (i + 1) & mask_;
        cells_[i] = c;
        ++n_;
      }
  }

  std::vector<Cell> cells_;
  size_t mask_ = 0, n_ = 0, gone_ = 0;
  int shift_ = 64;
};

}  // namespace tie::host
