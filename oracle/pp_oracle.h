/*
 * pp_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C, FP64, single-threaded restatement of the reference hot path
 * (/root/reference/proj/src/{dpps,intercept,ball_model,pass_eval,offball,
 * motion}.cpp), compiled with -ffp-contract=off like the reference.  It is
 * the checker the tests and bench.py's CPU leg use; the product never links
 * it.  Entry points mirror the product C-ABI (include/passplan_b200.h) with an
 * `or_` prefix and fill the same result-block layouts.
 *
 * Parity: pinned against golden vectors produced by the reference itself
 * (tests/golden/make_golden.py via oracle/_ref); see tests/test_oracle.py.
 */
#ifndef PP_ORACLE_H_
#define PP_ORACLE_H_

#include <stddef.h>
#include <stdint.h>

#include "passplan_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Work counters of the reference's pruned scan (kernel.hpp:33-44,
 * dpps.cpp:140-207): per-sample quick rejects, full arrival tests, rest-rule
 * evaluations, and per-robot scan calls (== sbip_calls). */
typedef struct or_counts {
  uint64_t quick_rejects, full_tests, rest_evals, scans, bounds;
} or_counts;

void or_params_default(pp_params* p);
void or_direction_table(int32_t n, double* xy);
int32_t or_nearest_teammate(const pp_world* w);

int or_dpps(const pp_world* w, const pp_params* p, const pp_search_grid* grid, int32_t kicker_id,
            void* block, char* msg, size_t msg_len);
int or_dpps_counted(const pp_world* w, const pp_params* p, const pp_search_grid* grid,
                    int32_t kicker_id, void* block, or_counts* counts, char* msg, size_t msg_len);
int or_score_cells(const pp_world* w, const pp_params* p, int64_t n, const double* rx,
                   const double* ry, const double* our_time, const double* opp_time,
                   const uint8_t* feasible, double* score_out, pp_pass_features* feat_out,
                   char* msg, size_t msg_len);
int or_goal_views(const pp_world* w, double radius, int64_t n, const double* px, const double* py,
                  double* angle, double* lo, double* hi, double* ty);
int64_t or_runmap_count(const pp_world* w, const pp_params* p, uint32_t zone_mask);
int or_runmap(const pp_world* w, const pp_params* p, const pp_runmap_request* req, void* block,
              int64_t block_vertices, char* msg, size_t msg_len);

/* intercept_all, possession, decide_shot, plan_free_kick */
int or_intercept_all(const pp_world* w, const pp_params* p, const pp_kick* k, double dt,
                     pp_intercept* out, char* msg, size_t msg_len);
int or_possession(const pp_world* w, const pp_params* p, pp_possession_report* out, char* msg,
                  size_t msg_len);
int or_decide_shot(const pp_world* w, const pp_params* p, int32_t shooter_id,
                   pp_shot_decision* out, char* msg, size_t msg_len);
int or_plan_free_kick(const pp_world* w, const pp_params* p, int32_t kicker_id,
                      const pp_candidate* c, pp_free_kick_plan* out, char* msg, size_t msg_len);

#ifdef __cplusplus
}
#endif

#endif /* PP_ORACLE_H_ */
