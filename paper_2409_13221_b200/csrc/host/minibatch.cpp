// fuseplan-b200 — length-balanced mini-batch assignment (host).
//
// Restates balance_minibatch of the reference (workflow.cpp:160-182): an LPT
// greedy. O(n log n + n dp); dp is the data-parallel degree (<= a few
// hundred), so the linear scan for the least-loaded group is cheaper than a
// heap and keeps the tie rule (lowest group index) explicit.
#include "fuseplan/minibatch.hpp"

#include <algorithm>
#include <numeric>
#include <stdexcept>

namespace fuseplan {

std::vector<std::vector<int>> balance_minibatch(const std::vector<int>& lengths, int dp) {
  if (dp < 1) throw std::invalid_argument("balance_minibatch: dp must be >= 1");
  const int n = static_cast<int>(lengths.size());
  if (n < dp) throw std::invalid_argument("balance_minibatch: need at least dp samples");
  std::vector<int> by_len(n);
  std::iota(by_len.begin(), by_len.end(), 0);
  // longest first; equal lengths keep index order
  std::stable_sort(by_len.begin(), by_len.end(), [&](int a, int b) { return lengths[a] > lengths[b]; });
  std::vector<std::vector<int>> out(dp);
  std::vector<long long> used(dp, 0);
  for (const int s : by_len) {
    const int g = static_cast<int>(std::min_element(used.begin(), used.end()) - used.begin());  // first minimum
    out[g].push_back(s);
    used[g] += lengths[s];
  }
  return out;
}

}  // namespace fuseplan
