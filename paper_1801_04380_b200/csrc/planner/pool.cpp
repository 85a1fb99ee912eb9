// BlockPool / PySet implementations; see pool.hpp.
#include "pool.hpp"

namespace snp {

std::string key_repr(int64_t code) {
  static const char* names[] = {"act", "grad", "ws"};
  return std::string("('") + names[key_kind(code)] + "', " + std::to_string(key_id(code)) + ")";
}

BlockPool::BlockPool(int64_t capacity_bytes) {
  if (capacity_bytes < kBlockBytes)
    fail(SN_EK_POOL, "pool capacity must be at least " + std::to_string(kBlockBytes) + " bytes");
  cap_ = capacity_bytes / kBlockBytes;
  free_.push_back({0, cap_});
}

int64_t BlockPool::alloc(int64_t key, int64_t nbytes, bool high) {
  if (alloc_.count(key)) fail(SN_EK_POOL, "key " + key_repr(key) + " is already allocated");
  const int64_t need = blocks_for(nbytes);
  const int64_t n = static_cast<int64_t>(free_.size());
  for (int64_t step = 0; step < n; ++step) {
    const int64_t i = high ? n - 1 - step : step;
    int64_t offset = free_[i].first;
    const int64_t length = free_[i].second;
    if (length < need) continue;
    if (length == need) {
      free_.erase(free_.begin() + i);
    } else if (high) {
      offset = offset + length - need;
      free_[i].second = length - need;
    } else {
      free_[i] = {offset + need, length - need};
    }
    alloc_[key] = {offset, need};
    used_ += need;
    if (used_ > high_) high_ = used_;
    return offset;
  }
  fail(SN_EK_POOLEXH, "no contiguous " + std::to_string(need) + " blocks available (" +
                          std::to_string(free_bytes()) + " bytes free, fragmented)");
}

void BlockPool::free(int64_t key) {
  auto it = alloc_.find(key);
  if (it == alloc_.end()) fail(SN_EK_POOL, "key " + key_repr(key) + " is not allocated");
  const int64_t offset = it->second.first;
  int64_t length = it->second.second;
  alloc_.erase(it);
  used_ -= length;
  // bisect_left(free, (offset, 0))
  size_t idx = static_cast<size_t>(
      std::lower_bound(free_.begin(), free_.end(), std::make_pair(offset, int64_t(0))) - free_.begin());
  if (idx < free_.size() && free_[idx].first == offset + length) {
    length += free_[idx].second;
    free_.erase(free_.begin() + idx);
  }
  if (idx > 0) {
    const int64_t p_off = free_[idx - 1].first, p_len = free_[idx - 1].second;
    if (p_off + p_len == offset) {
      free_[idx - 1].second = p_len + length;
      return;
    }
    if (p_off + p_len > offset) fail(SN_EK_POOL, "free list corrupted: overlapping spans");
  }
  const auto span = std::make_pair(offset, length);
  free_.insert(std::upper_bound(free_.begin(), free_.end(), span), span);
}

void BlockPool::check() const {
  struct S { int64_t off, len; int tag; };  // tag 0 free, 1 used (sorts "free" < "used")
  std::vector<S> spans;
  for (auto& f : free_) spans.push_back({f.first, f.second, 0});
  int64_t used_sum = 0;
  for (auto& kv : alloc_) {
    spans.push_back({kv.second.first, kv.second.second, 1});
    used_sum += kv.second.second;
  }
  std::sort(spans.begin(), spans.end(), [](const S& a, const S& b) {
    if (a.off != b.off) return a.off < b.off;
    if (a.len != b.len) return a.len < b.len;
    return a.tag < b.tag;
  });
  int64_t cursor = 0;
  int prev = -1;
  for (const S& s : spans) {
    if (s.off != cursor)
      fail(SN_EK_POOL, "arena gap or overlap at block " + std::to_string(cursor) + ": next span starts at " +
                           std::to_string(s.off));
    if (s.tag == 0 && prev == 0) fail(SN_EK_POOL, "adjacent free spans not coalesced at block " + std::to_string(s.off));
    cursor = s.off + s.len;
    prev = s.tag;
  }
  if (cursor != cap_)
    fail(SN_EK_POOL, "arena ends at block " + std::to_string(cursor) + ", capacity is " + std::to_string(cap_));
  if (used_ != used_sum) fail(SN_EK_POOL, "used-block counter out of sync");
}

// ---------------------------------------------------------------------------

bool PySet::contains(int64_t key) const {
  for (int64_t v : table_)
    if (v == key) return true;
  return false;
}

void PySet::add(int64_t key) {
  size_t perturb = static_cast<size_t>(key);
  size_t i = static_cast<size_t>(key) & mask_;
  while (true) {
    size_t probes = (i + kProbes <= mask_) ? kProbes : 0;
    size_t j = i;
    while (true) {
      if (table_[j] == kEmpty) {
        table_[j] = key;
        ++fill_;
        ++used_;
        if (fill_ * 5 < mask_ * 3) return;
        resize(used_ > 50000 ? used_ * 2 : used_ * 4);
        return;
      }
      if (table_[j] == key) return;
      if (probes == 0) break;
      --probes;
      ++j;
    }
    perturb >>= 5;
    i = (i * 5 + 1 + perturb) & mask_;
  }
}

void PySet::insert_clean(std::vector<int64_t>& table, size_t mask, int64_t key) {
  size_t perturb = static_cast<size_t>(key);
  size_t i = static_cast<size_t>(key) & mask;
  while (true) {
    if (table[i] == kEmpty) {
      table[i] = key;
      return;
    }
    if (i + kProbes <= mask) {
      for (size_t j = 1; j <= kProbes; ++j)
        if (table[i + j] == kEmpty) {
          table[i + j] = key;
          return;
        }
    }
    perturb >>= 5;
    i = (i * 5 + 1 + perturb) & mask;
  }
}

void PySet::resize(size_t minused) {
  size_t newsize = 8;
  while (newsize <= minused) newsize <<= 1;
  std::vector<int64_t> old;
  old.swap(table_);
  table_.assign(newsize, kEmpty);
  mask_ = newsize - 1;
  for (int64_t k : old)
    if (k != kEmpty) insert_clean(table_, mask_, k);
  fill_ = used_;
}

void PySet::update(const PySet& other) {
  if (&other == this || other.used_ == 0) return;
  if ((fill_ + other.used_) * 5 >= mask_ * 3) resize((used_ + other.used_) * 2);
  if (fill_ == 0 && mask_ == other.mask_) {
    table_ = other.table_;
    fill_ = other.fill_;
    used_ = other.used_;
    return;
  }
  if (fill_ == 0) {
    fill_ = other.used_;
    used_ = other.used_;
    for (int64_t k : other.table_)
      if (k != kEmpty) insert_clean(table_, mask_, k);
    return;
  }
  for (int64_t k : other.table_)
    if (k != kEmpty) add(k);
}

std::vector<int64_t> PySet::items() const {
  std::vector<int64_t> out;
  for (int64_t k : table_)
    if (k != kEmpty) out.push_back(k);
  return out;
}

}  // namespace snp
