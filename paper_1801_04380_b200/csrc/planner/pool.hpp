// Mechanism primitives of the unified tensor pool (memsched L4):
//   BlockPool  -- 1 KiB-block two-ended first-fit arena (poolalloc.py:35-163);
//                 offsets are the device-arena offsets the executor uses.
//   LruCache   -- recency-ordered registry of reusable device tensors
//                 (offload.py:82-132).
//   OrderedKeys-- insertion-ordered key set (CPython dict order semantics).
//   PySet      -- CPython 3.12 set-of-int table layout, so that iterating the
//                 "transient" set visits tensors in exactly the reference's
//                 order (simulator.py:618-621); see SURVEY Appendix A.1.
#pragma once
#include <algorithm>
#include <cstdint>
#include <list>
#include <string>
#include <unordered_map>
#include <vector>

#include "core.hpp"

namespace snp {

constexpr int64_t kBlockBytes = 1024;

enum KeyKind { K_ACT = 0, K_GRAD = 1, K_WS = 2 };
inline int64_t key_code(int kind, int64_t id) { return (static_cast<int64_t>(kind) << 40) | (id & ((1ll << 40) - 1)); }
inline int key_kind(int64_t code) { return static_cast<int>(code >> 40); }
inline int64_t key_id(int64_t code) { return code & ((1ll << 40) - 1); }
std::string key_repr(int64_t code);  // "('act', 3)"

inline int64_t blocks_for(int64_t nbytes) {
  if (nbytes < 0) fail(SN_EK_POOL, "negative allocation size " + std::to_string(nbytes));
  const int64_t b = (nbytes + kBlockBytes - 1) / kBlockBytes;
  return b < 1 ? 1 : b;
}

class BlockPool {
 public:
  explicit BlockPool(int64_t capacity_bytes);
  int64_t alloc(int64_t key, int64_t nbytes, bool high);  // returns block offset
  void free(int64_t key);
  bool contains(int64_t key) const { return alloc_.count(key) != 0; }
  std::pair<int64_t, int64_t> span(int64_t key) const { return alloc_.at(key); }
  int64_t used_bytes() const { return used_ * kBlockBytes; }
  int64_t free_bytes() const { return (cap_ - used_) * kBlockBytes; }
  int64_t high_water_bytes() const { return high_ * kBlockBytes; }
  int64_t capacity_blocks() const { return cap_; }
  size_t n_keys() const { return alloc_.size(); }
  const std::vector<std::pair<int64_t, int64_t>>& free_spans() const { return free_; }
  const std::unordered_map<int64_t, std::pair<int64_t, int64_t>>& allocated() const { return alloc_; }
  void check() const;

 private:
  int64_t cap_, used_ = 0, high_ = 0;
  std::vector<std::pair<int64_t, int64_t>> free_;  // sorted by offset
  std::unordered_map<int64_t, std::pair<int64_t, int64_t>> alloc_;
};

// Insertion-ordered set of int64 keys with O(1) insert/erase/contains.
class OrderedKeys {
 public:
  bool contains(int64_t k) const { return pos_.count(k) != 0; }
  bool insert(int64_t k) {  // appends; false if present
    if (contains(k)) return false;
    order_.push_back(k);
    pos_[k] = std::prev(order_.end());
    return true;
  }
  bool erase(int64_t k) {
    auto it = pos_.find(k);
    if (it == pos_.end()) return false;
    order_.erase(it->second);
    pos_.erase(it);
    return true;
  }
  void move_to_end(int64_t k) {
    auto it = pos_.find(k);
    order_.splice(order_.end(), order_, it->second);
  }
  size_t size() const { return pos_.size(); }
  bool empty() const { return pos_.empty(); }
  int64_t front() const { return order_.front(); }
  std::vector<int64_t> snapshot() const { return std::vector<int64_t>(order_.begin(), order_.end()); }

 private:
  std::list<int64_t> order_;
  std::unordered_map<int64_t, std::list<int64_t>::iterator> pos_;
};

// The simulator never locks entries (simulator.py:348-350), so eviction takes
// the least recently inserted/touched key.
class LruCache {
 public:
  bool contains(int lid) const { return keys_.contains(lid); }
  // Returns true when the key was new ("insert"), false on a touch.
  bool insert(int lid) {
    if (keys_.contains(lid)) {
      keys_.move_to_end(lid);
      return false;
    }
    keys_.insert(lid);
    return true;
  }
  bool discard(int lid) { return keys_.erase(lid); }
  int evict_lru() {
    if (keys_.empty()) fail(SN_EK_ALLLOCKED, "no unlocked cached tensor is available for eviction");
    const int lid = static_cast<int>(keys_.front());
    keys_.erase(lid);
    return lid;
  }
  size_t size() const { return keys_.size(); }

 private:
  OrderedKeys keys_;
};

// CPython 3.12 setobject.c open-addressing table for non-negative small ints
// (hash(i) == i): LINEAR_PROBES = 9, PERTURB_SHIFT = 5, PySet_MINSIZE = 8,
// grow when fill*5 >= mask*3 to the smallest power of two > used*4
// (used*2 above 50000).  No deletions are ever made, so there are no dummies.
class PySet {
 public:
  PySet() : table_(8, kEmpty), mask_(7) {}
  void add(int64_t key);
  void update(const PySet& other);  // set_merge
  bool contains(int64_t key) const;
  std::vector<int64_t> items() const;  // iteration order
  size_t size() const { return used_; }

 private:
  static constexpr int64_t kEmpty = -1;
  static constexpr size_t kProbes = 9;
  void resize(size_t minused);
  static void insert_clean(std::vector<int64_t>& table, size_t mask, int64_t key);
  std::vector<int64_t> table_;
  size_t mask_;
  size_t fill_ = 0, used_ = 0;
};

}  // namespace snp
