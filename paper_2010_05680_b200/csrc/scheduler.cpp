// scheduler.cpp -- NEXT-4: the DP batch scheduler of PAPER.md §5 (Algorithm 2,
// Eq. 2), host C++.  Contract: include/tt_sched.h.
#include <math.h>

#include <algorithm>
#include <numeric>
#include <vector>

#include "../../include/tt_sched.h"

namespace {

inline double cost_at(const double* cost, int64_t max_batch, int64_t len, int64_t count) {
    return cost[len * (max_batch + 1) + count];
}

bool valid_entry(double c) { return !std::isnan(c) && c >= 0.0; }

tt_status check_lengths(const int32_t* lengths, int64_t n, int64_t max_len) {
    for (int64_t i = 0; i < n; ++i)
        if (lengths[i] < 1 || lengths[i] > max_len) return TT_ERROR_INVALID_VALUE;
    return TT_SUCCESS;
}

}  // namespace

extern "C" {

tt_status tt_dp_schedule(const int32_t* lengths, int64_t n, const double* cost, int64_t max_len,
                         int64_t max_batch, int32_t* order, int32_t* batch_start,
                         int64_t* n_batches, double* total_cost) {
    if (n < 0 || max_len < 1 || max_batch < 1 || !n_batches || !total_cost)
        return TT_ERROR_INVALID_VALUE;
    if (n > 0 && (!lengths || !cost || !order || !batch_start)) return TT_ERROR_INVALID_VALUE;
    if (n > 0x7ffffffeLL) return TT_ERROR_INVALID_VALUE;
    *n_batches = 0;
    *total_cost = 0.0;
    if (n == 0) {
        if (batch_start) batch_start[0] = 0;
        return TT_SUCCESS;
    }
    if (check_lengths(lengths, n, max_len) != TT_SUCCESS) return TT_ERROR_INVALID_VALUE;

    // Alg. 2 line 1: sort in increasing length (stable: equal lengths keep
    // queue order, i.e. FIFO within a length class)
    std::vector<int32_t> idx(n);
    std::iota(idx.begin(), idx.end(), 0);
    std::stable_sort(idx.begin(), idx.end(),
                     [&](int32_t a, int32_t b) { return lengths[a] < lengths[b]; });

    // states[i]: minimum cost of the first i sorted requests; start[i]: 1-based
    // index of the first request of the last batch of that optimum
    std::vector<double> states(n + 1, 0.0);
    std::vector<int64_t> start(n + 1, 0);
    for (int64_t i = 1; i <= n; ++i) {
        const int64_t len = lengths[idx[i - 1]];  // longest of any batch ending at i
        double best = INFINITY;
        int64_t arg = -1;
        const int64_t jlo = std::max<int64_t>(1, i - max_batch + 1);
        for (int64_t j = i; j >= jlo; --j) {  // batch = sorted requests j..i (1-based)
            const int64_t count = i - j + 1;
            const double c = cost_at(cost, max_batch, len, count);
            if (!valid_entry(c)) return TT_ERROR_INVALID_VALUE;
            const double tmp = states[j - 1] + c * (double)count;
            if (tmp < best) {  // strict: ties keep the larger start (smaller batch)
                best = tmp;
                arg = j;
            }
        }
        states[i] = best;
        start[i] = arg;
    }
    // backtrack (Alg. 2 lines 16-20)
    std::vector<int64_t> cuts;
    for (int64_t i = n; i > 0; i = start[i] - 1) cuts.push_back(start[i] - 1);
    std::reverse(cuts.begin(), cuts.end());
    for (int64_t i = 0; i < n; ++i) order[i] = idx[i];
    for (size_t b = 0; b < cuts.size(); ++b) batch_start[b] = (int32_t)cuts[b];
    batch_start[cuts.size()] = (int32_t)n;
    *n_batches = (int64_t)cuts.size();
    *total_cost = states[n];
    return TT_SUCCESS;
}

tt_status tt_schedule_cost(const int32_t* lengths, int64_t n, const double* cost, int64_t max_len,
                           int64_t max_batch, const int32_t* idx, const int32_t* batch_start,
                           int64_t n_batches, double* total_cost) {
    if (n < 0 || n_batches < 0 || max_len < 1 || max_batch < 1 || !total_cost)
        return TT_ERROR_INVALID_VALUE;
    if (n > 0 && (!lengths || !cost || !idx || !batch_start)) return TT_ERROR_INVALID_VALUE;
    if (check_lengths(lengths, n, max_len) != TT_SUCCESS) return TT_ERROR_INVALID_VALUE;
    if (n_batches == 0) {
        *total_cost = 0.0;
        return n == 0 ? TT_SUCCESS : TT_ERROR_INVALID_VALUE;
    }
    if (batch_start[0] != 0 || batch_start[n_batches] != n) return TT_ERROR_INVALID_VALUE;
    std::vector<char> seen(n, 0);
    double total = 0.0;
    for (int64_t b = 0; b < n_batches; ++b) {
        const int64_t lo = batch_start[b], hi = batch_start[b + 1];
        const int64_t count = hi - lo;
        if (count < 1 || count > max_batch) return TT_ERROR_INVALID_VALUE;
        int64_t len = 0;
        for (int64_t k = lo; k < hi; ++k) {
            const int32_t r = idx[k];
            if (r < 0 || r >= n || seen[r]) return TT_ERROR_INVALID_VALUE;
            seen[r] = 1;
            len = std::max<int64_t>(len, lengths[r]);
        }
        const double c = cost_at(cost, max_batch, len, count);
        if (!valid_entry(c)) return TT_ERROR_INVALID_VALUE;
        total += c * (double)count;
    }
    *total_cost = total;
    return TT_SUCCESS;
}

}  // extern "C"
