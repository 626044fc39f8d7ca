// Paged KV block manager (new: the reference keeps a byte ledger only,
// simulator.cpp:96-98,223-244,443-492).
//
// Admission still follows the reference byte rule (kept in the engine), so
// this class only turns "request r now holds n tokens of KV" into pages.
// Deterministic spec (mirrored by oracle/kvpages_model.py):
//   - a request's page list grows on demand, before the launch that writes
//     positions beyond its current pages;
//   - each new page is the lowest free page id;
//   - all pages of a request are released (in list order) when it finishes.
#pragma once

#include <cstdint>
#include <map>
#include <set>
#include <string>
#include <vector>

namespace nxb {

class PagePool {
 public:
  void configure(int32_t page_tokens, int32_t num_pages) {
    page_tokens_ = page_tokens;
    num_pages_ = num_pages;
    free_.clear();
    for (int32_t p = 0; p < num_pages; ++p) free_.insert(p);
    owned_.clear();
    log_.clear();
  }
  int32_t page_tokens() const { return page_tokens_; }
  int32_t num_pages() const { return num_pages_; }
  bool configured() const { return page_tokens_ > 0; }

  // Grow request `id` to cover `tokens` positions; returns false if the pool
  // ran dry (pages allocated before the failure stay allocated). `fresh`
  // receives the (index, page) pairs added, for the device mirror.
  bool ensure(uint64_t id, int64_t tokens, std::vector<std::pair<int32_t, int32_t>>* fresh) {
    std::vector<int32_t>& pages = owned_[id];
    while (static_cast<int64_t>(pages.size()) * page_tokens_ < tokens) {
      if (free_.empty()) return false;
      const int32_t p = *free_.begin();
      free_.erase(free_.begin());
      if (fresh) fresh->push_back({static_cast<int32_t>(pages.size()), p});
      pages.push_back(p);
      if (logging_) log_ += "alloc " + std::to_string(id) + " " + std::to_string(p) + "\n";
    }
    return true;
  }

  void release(uint64_t id) {
    auto it = owned_.find(id);
    if (it == owned_.end()) return;
    for (int32_t p : it->second) {
      free_.insert(p);
      if (logging_) log_ += "free " + std::to_string(id) + " " + std::to_string(p) + "\n";
    }
    owned_.erase(it);
  }

  const std::vector<int32_t>* table(uint64_t id) const {
    auto it = owned_.find(id);
    return it == owned_.end() ? nullptr : &it->second;
  }
  size_t free_pages() const { return free_.size(); }
  const std::string& log() const { return log_; }
  void set_logging(bool on) { logging_ = on; }

 private:
  int32_t page_tokens_ = 0, num_pages_ = 0;
  std::set<int32_t> free_;
  std::map<uint64_t, std::vector<int32_t>> owned_;
  std::string log_;
  bool logging_ = true;
};

}  // namespace nxb
