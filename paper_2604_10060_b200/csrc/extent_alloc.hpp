// extent_alloc.hpp -- first-fit allocator of contiguous page runs with coalescing frees.
//
// Used for the host tier (one contiguous extent of pinned pages per Host-resident cluster, so a
// fetch / offload is ONE copy per cluster -- the reference moves a cluster as one batched
// transfer, store.cpp:95-130) and for the HBM staging runs of in-flight migrations.
#pragma once

#include <cstdint>
#include <iterator>
#include <map>

namespace kvc {

class ExtentAlloc {
 public:
  void reset(std::int64_t capacity) {
    free_.clear();
    cap_ = capacity;
    used_ = 0;
    if (capacity > 0) free_[0] = capacity;
  }
  // start of a run of n units, or -1
  std::int64_t alloc(std::int64_t n) {
    if (n <= 0) return -1;
    for (auto it = free_.begin(); it != free_.end(); ++it) {
      if (it->second < n) continue;
      const std::int64_t s = it->first, len = it->second;
      free_.erase(it);
      if (len > n) free_[s + n] = len - n;
      used_ += n;
      return s;
    }
    return -1;
  }
  void release(std::int64_t s, std::int64_t n) {
    if (s < 0 || n <= 0) return;
    used_ -= n;
    auto it = free_.emplace(s, n).first;
    if (it != free_.begin()) {  // merge with the run before
      auto p = std::prev(it);
      if (p->first + p->second == it->first) {
        p->second += it->second;
        free_.erase(it);
        it = p;
      }
    }
    auto nx = std::next(it);
    if (nx != free_.end() && it->first + it->second == nx->first) {
      it->second += nx->second;
      free_.erase(nx);
    }
  }
  std::int64_t used() const { return used_; }
  std::int64_t capacity() const { return cap_; }

 private:
  std::map<std::int64_t, std::int64_t> free_;  // start -> length
  std::int64_t cap_ = 0, used_ = 0;
};

}  // namespace kvc
