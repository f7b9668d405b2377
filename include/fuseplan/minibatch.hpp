// fuseplan-b200 — experience hand-off: length-balanced data-parallel mini-batches.
//
// Source-compatible with the reference declaration of balance_minibatch
// (proj/include/fuseplan/workflow.hpp:63-66; semantics workflow.cpp:160-182):
// the reference header also drags in the training-schedule search
// (annealer.hpp / fusion.hpp), which is out of this repo's scope, so the one
// hot-path function lives in its own header here.
#pragma once

#include <vector>

namespace fuseplan {

// Longest-processing-time packing of sample lengths into `dp` groups: samples
// in decreasing length (ties: lower index first) each go to the currently
// least-loaded group (ties: lower group). Returns the sample indices of each
// group in insertion order. The max group load never exceeds sum/dp + max.
// Throws std::invalid_argument for dp < 1 or fewer samples than groups.
std::vector<std::vector<int>> balance_minibatch(const std::vector<int>& lengths, int dp);

}  // namespace fuseplan
