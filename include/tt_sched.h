/*
 * tt_sched.h -- NEXT-4: the sequence-length-aware DP batch
 * scheduler of TurboTransformers (§5, Algorithm 2 "Batch Scheduler
 * With DP", l.619-648; Bellman equation Eq. 2, l.609-615), as host C++ in
 * libtt.so.  It decides how a queue of variable-length requests is cut into
 * padded batches for the kernels of tt.h.
 *
 * Cost model (Alg. 2): cached_cost[len][count] is the per-request cost of a
 * batch of `count` requests padded to `len` tokens; a batch costs
 * cached_cost[len][count] * count.  The caller supplies the table (built by
 * timing the kernels over the (len, count) grid -- tools/cost_table.py) as a
 * dense row-major double array [max_len + 1][max_batch + 1]; entries with
 * count = 0 or len = 0 are ignored; NaN marks a missing entry.
 *
 * Algorithm (as Alg. 2 executes): stable-sort the requests by length (ties
 * keep queue order), states[0] = 0,
 *   states[i] = min_{i - max_batch < j <= i} states[j-1]
 *               + cached_cost[len(i)][i-j+1] * (i-j+1)      (1-based, sorted)
 * where len(i) is the longest request of the batch, i.e. request i; backtrack
 * the argmins into contiguous batches of the sorted order.  O(n * max_batch).
 */
#ifndef TT_SCHED_H_
#define TT_SCHED_H_

#include "tt.h"

#ifdef __cplusplus
extern "C" {
#endif

/* lengths       HOST int32[n], request lengths in queue (arrival) order, each in
 *               [1, max_len].
 * cost          HOST double[(max_len + 1) * (max_batch + 1)].
 * order         HOST int32[n] out: request indices in the sorted order.
 * batch_start   HOST int32[n + 1] out: batch b is order[batch_start[b] ..
 *               batch_start[b+1]-1]; batches in increasing padded length.
 * n_batches     HOST out.   total_cost  HOST out: states[n].
 * Errors: TT_ERROR_INVALID_VALUE for null pointers, n < 0, max_len < 1,
 * max_batch < 1, a length outside [1, max_len], or a NaN / negative cost
 * entry that the recursion reads (the plan is then undefined).  n = 0 gives
 * zero batches.  Pure host code: no CUDA call. */
TT_API tt_status tt_dp_schedule(const int32_t* lengths, int64_t n, const double* cost,
                                int64_t max_len, int64_t max_batch, int32_t* order,
                                int32_t* batch_start, int64_t* n_batches, double* total_cost);

/* Cost of a given plan under the same model (for comparing schedules, e.g.
 * the naive "everything in one batch" or fixed-size arrival-order batches):
 * batch b = requests idx[batch_start[b] .. batch_start[b+1]-1] (any order),
 * padded to its longest member.  Errors as above, plus batches larger than
 * max_batch. */
TT_API tt_status tt_schedule_cost(const int32_t* lengths, int64_t n, const double* cost,
                                  int64_t max_len, int64_t max_batch, const int32_t* idx,
                                  const int32_t* batch_start, int64_t n_batches,
                                  double* total_cost);

#ifdef __cplusplus
}
#endif
#endif /* TT_SCHED_H_ */
