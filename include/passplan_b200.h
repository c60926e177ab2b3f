/*
 * passplan_b200.h -- C-ABI of the B200-native SBIP-DPPS pass planner.
 *
 * This is the drop-in boundary for the reference's hot path
 * (arXiv 1909.07717, reference tree `proj/`).  Plain C: POD structs, plain
 * pointers and sizes, status codes instead of exceptions, no C++ or torch
 * types.  Every entry point names the reference interface it replaces.
 *
 *   reference (C++, proj/include/passplan/...)          this ABI
 *   ------------------------------------------------    ----------------------
 *   run_dpps / run_dpps_serial   dpps.hpp:90-96          pp_dpps
 *   best_pass (all/flat/chip)    pass_eval.hpp:55-60     pp_dpps (fused summary)
 *   score_pass                   pass_eval.hpp:43-44     pp_score_cells
 *   goal_view / shoot_angle      pass_eval.hpp:34-37     pp_goal_views
 *   score_running_point          offball.hpp:62-63       pp_runmap (per vertex)
 *   best_running_points          offball.hpp:96-99       pp_runmap (per zone)
 *   kernels::KernelBackend       kernels/kernel.hpp:48-53  (name only: "sm100a")
 *   ErrorCategory                errors.hpp:11-17        pp_status
 *
 * Threading: one pp_ctx is used by one host thread at a time (the C++
 * drop-in keeps one context per thread and device).  Results are
 * bit-identical for any batch composition (SPEC determinism rule).
 */
#ifndef PASSPLAN_B200_H_
#define PASSPLAN_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PP_ABI_VERSION 1
#define PP_MAX_TEAM 16 /* world.hpp:62 "at most 16 robots per team" */

/* ErrorCategory (errors.hpp:11-17) + a CUDA failure class. */
typedef enum pp_status {
  PP_OK = 0,
  PP_SCHEMA = 1,
  PP_VALIDATION = 2,
  PP_CONFIG = 3,
  PP_DOMAIN = 4,
  PP_INTERNAL = 5,
  PP_CUDA = 6
} pp_status;

/* ---- world state (world.hpp:12-80) ------------------------------------ */
typedef struct pp_field { /* FieldGeometry, world.hpp:12-17 */
  double length, width, goal_width, defense_depth, defense_width;
} pp_field;

typedef struct pp_robot { /* RobotState, world.hpp:46-51 */
  int32_t id;
  int32_t reserved;
  double px, py, vx, vy, theta;
} pp_robot;

typedef struct pp_world { /* WorldState, world.hpp:65-80 (teams in caller order) */
  pp_field field;
  double ball_px, ball_py, ball_vx, ball_vy;
  int32_t n_ours, n_theirs;
  pp_robot ours[PP_MAX_TEAM];
  pp_robot theirs[PP_MAX_TEAM];
} pp_world;

/* ---- planner configuration (config.hpp:29-71, weights.hpp) ------------ */
typedef struct pp_ball_model { /* BallModelParams, ball_model.hpp:14-23 */
  double slide_decel, roll_decel, transition_ratio, power_min, power_max,
      chip_flight_fraction;
} pp_ball_model;

typedef struct pp_motion_limits { /* MotionLimits, motion.hpp:9-15 */
  double max_speed, max_accel, max_decel;
} pp_motion_limits;

typedef struct pp_search_grid { /* SearchGrid, dpps.hpp:20-31 */
  int32_t n_directions, n_powers;
  double power_min, power_max;
  int32_t flat, chip;
} pp_search_grid;

typedef struct pp_pass_weights { /* PassWeights, weights.hpp:10-16 */
  double teammate_time, shoot_angle, dist_goal, refraction, margin;
} pp_pass_weights;

typedef struct pp_run_weights { /* RunWeights, weights.hpp:20-26 */
  double dist_goal, dist_ball, angle, guard_time, exposure;
} pp_run_weights;

typedef struct pp_norm_bounds { /* NormBounds, weights.hpp:30-33 */
  double length_upper, angle_upper;
} pp_norm_bounds;

typedef struct pp_angle_band { /* AngleBand, weights.hpp:38-43 */
  double full_lo, peak_lo, peak_hi, full_hi;
} pp_angle_band;

typedef struct pp_thresholds { /* PlannerThresholds, config.hpp:29-45 */
  double sbip_dt, robot_radius, safety_margin, buffer_time, possession_radius,
      angle_threshold, shot_power, margin_cap, possession_dt, contest_epsilon,
      grid_step, min_zone_width, guard_time_cap, drag_v_min, marking_radius;
} pp_thresholds;

typedef struct pp_params { /* PlannerConfig minus SvgStyle, config.hpp:47-71 */
  pp_ball_model ball;
  pp_motion_limits motion_ours, motion_theirs;
  pp_search_grid grid;
  pp_pass_weights pass_weights;
  pp_run_weights run_weights;
  pp_norm_bounds norm;
  pp_angle_band angle_band;
  pp_thresholds thresholds;
} pp_params;

/* Fills the reference defaults (config.hpp, weights.hpp, dpps.hpp). */
void pp_params_default(pp_params* out);

/* PlannerConfig::validate (config.cpp:172-200, SvgStyle excluded) and
 * SearchGrid::validate (dpps.cpp:22-28).  PP_CONFIG on the first bad value. */
pp_status pp_params_validate(const pp_params* params, char* msg, size_t msg_len);

/* ---- per-cell result block -------------------------------------------- *
 * One contiguous block per frame so the device->host copy is one DMA.
 * Cells are ordered [kick_type slot][dir_index][power_index] exactly like
 * CandidateGrid::cells (dpps.hpp:74-79).  Robots are reported as SLOTS into
 * the id-sorted team tables carried in the summary (slot -1 = none), times
 * are FP64 bit-identical to PassCandidate::our_time / opp_time (kNever =
 * +inf), receive points are meaningful iff our_time is finite.
 */
typedef struct pp_pass_features { /* PassFeatures, pass_eval.hpp:13-19 */
  double teammate_intercept_time, shoot_angle_at_receive, dist_receive_to_goal,
      refraction_angle, intercept_margin;
} pp_pass_features;

typedef struct pp_dpps_summary {
  int64_t n_cells;
  int32_t n_kick_types;
  int32_t kick_types[2]; /* 0 = flat, 1 = chip (SearchGrid::kick_types order) */
  int32_t n_directions, n_powers;
  int32_t kicker_id, kicker_slot, kicker_in_possession;
  int32_t n_ours, n_theirs;
  int32_t ours_ids[PP_MAX_TEAM];   /* slot -> robot id, id-sorted */
  int32_t theirs_ids[PP_MAX_TEAM]; /* slot -> robot id, id-sorted */
  uint64_t sbip_calls;             /* DppsTelemetry::sbip_calls */
  int64_t n_feasible[3];           /* all / flat / chip */
  int64_t best_cell[3];            /* best_pass all / flat / chip; -1 = nullopt */
  double best_score[3];
  pp_pass_features best_features[3];
  double device_ms;                /* kernel span of this frame on the device, ms
                                      (first scan CTA start -> final fold) */
} pp_dpps_summary;

typedef struct pp_grid_view { /* typed pointers into a result block */
  pp_dpps_summary* summary;
  double* our_time;
  double* opp_time;
  double* rx;
  double* ry;
  float* score;      /* score_pass, FP32 map; -inf for infeasible cells */
  int8_t* our_slot;  /* -1 = our_id -1 */
  int8_t* opp_slot;  /* -1 = opp_id -1 */
  uint8_t* feasible; /* PassCandidate::feasible */
} pp_grid_view;

/* What pp_dpps copies back to the host. */
#define PP_COPY_SUMMARY 0u /* summary only (best pass, counts, telemetry) */
#define PP_COPY_ALL 1u     /* summary + every per-cell array */

/* Bytes of a result block for n_cells cells (16-byte aligned arrays). */
size_t pp_grid_bytes(int64_t n_cells);
/* Typed view of a block of pp_grid_bytes(n_cells) bytes starting at `block`. */
void pp_grid_view_of(void* block, int64_t n_cells, pp_grid_view* out);

/* ---- running-point map ------------------------------------------------ */
typedef struct pp_run_features { /* RunningPointFeatures, offball.hpp:49-55 */
  double dist_to_goal, dist_to_ball, angle_to_goal, guard_time, defense_exposure;
} pp_run_features;

typedef struct pp_running_point { /* RunningPoint, offball.hpp:77-82 */
  int32_t zone; /* 0..3 = I..IV */
  int32_t valid;
  double px, py, score;
  pp_run_features features;
} pp_running_point;

typedef struct pp_runmap_summary {
  double cut_x, cut_y;
  int32_t zone_nx[4], zone_ny[4];  /* lattice shape per zone (0 if not requested) */
  int64_t zone_offset[4];          /* first vertex of each zone in the map */
  int64_t n_vertices;              /* total lattice vertices of requested zones */
  int64_t n_scorable;              /* vertices score_running_point accepts */
  pp_running_point best[4];        /* best_running_points, indexed by zone */
  int32_t n_best;
  int32_t best_order[4];           /* zones of the result vector, I..IV order */
} pp_runmap_summary;

typedef struct pp_runmap_request {
  uint32_t zone_mask;       /* bit z = rasterise zone z for the map (heatmap --zone) */
  uint32_t occupied_mask;   /* best_running_points `occupied` */
  int32_t n_runners;        /* best_running_points n_runners */
  int32_t has_best_pass_point;
  double best_pass_px, best_pass_py;
  int32_t want_map;         /* copy the per-vertex map back */
} pp_runmap_request;

/* Per-vertex map, x-major per zone, zones in I..IV order (the CLI
 * `heatmap --mode run` iteration order, passplan_main.cpp:186-196). */
typedef struct pp_runmap_view {
  pp_runmap_summary* summary;
  double* px;
  double* py;
  double* score;          /* NaN where score_running_point throws */
  pp_run_features* features;
  uint8_t* scorable;
} pp_runmap_view;

size_t pp_runmap_bytes(int64_t n_vertices);
void pp_runmap_view_of(void* block, int64_t n_vertices, pp_runmap_view* out);
/* Vertices that pp_runmap will produce for this world/params/zone mask. */
pp_status pp_runmap_count(const pp_world* world, const pp_params* params, uint32_t zone_mask,
                          int64_t* n_vertices);

/* ---- context ------------------------------------------------------------ */
typedef struct pp_ctx pp_ctx;

pp_status pp_ctx_create(int device, pp_ctx** out);
void pp_ctx_destroy(pp_ctx* ctx);
/* Context options.  PP_OPT_EXACT_ONLY (value 1 = on): verification switch
 * that turns off every FP32 shortcut of the kernels -- the reach / arrival
 * lower-bound rejects, skip-ahead, upper-bound accepts and window prunes of
 * the scan and interception kernels, and the FP32 gate / geometric band of
 * goal_view -- so every in-window sample and every bisection step takes the
 * reference's exact FP64 test (kernel.hpp:33-44, pass_eval.cpp:15-51).
 * Results must be byte-identical either way; only speed differs.  The
 * environment variable PP_EXACT_ONLY=1 sets it at pp_ctx_create. */
#define PP_OPT_EXACT_ONLY 1
pp_status pp_ctx_set_option(pp_ctx* ctx, int32_t option, int32_t value);
/* Message of the last failing call on this context (valid until the next call). */
const char* pp_last_error(const pp_ctx* ctx);
/* KernelBackend::name equivalent (kernel.hpp:50-53): "sm100a". */
const char* pp_kernel_name(void);
int pp_abi_version(void);
/* Host bytes one pp_dpps call sends to the device: the packed frame and its
 * robots' filter constants, as kernel parameters (no copy node). */
size_t pp_dpps_upload_bytes(void);

/* Pinned host memory for result blocks / frame arrays (fast DMA). */
void* pp_host_alloc(size_t bytes);
void pp_host_free(void* p);

/* ---- single frame: DPPS search + value function + argmax --------------- *
 * run_dpps (dpps.cpp:217-309) for `grid` (NULL = params->grid), then
 * score_pass over the feasible cells and best_pass for all / flat / chip.
 * Errors: PP_CONFIG (grid/params), PP_VALIDATION (kicker not on ours).
 * `block` is a caller-owned host buffer of pp_grid_bytes(n_cells) bytes
 * (pinned via pp_host_alloc for full DMA speed).  Synchronous. */
pp_status pp_dpps(pp_ctx* ctx, const pp_world* world, const pp_params* params,
                  const pp_search_grid* grid, int32_t kicker_id, uint32_t copy_flags,
                  void* block);

/* Re-launch the last pp_dpps search on its staged frame, asynchronously on
 * the context's stream, without host copies (device-resident timing). */
pp_status pp_dpps_relaunch(pp_ctx* ctx);
/* The context's cudaStream_t, for callers that time or order work on it. */
void* pp_ctx_stream(pp_ctx* ctx);
/* Measurement helper: re-run the last pp_dpps search `reps` times with CUDA
 * events around each of its two kernels (scan, value); average ms of each. */
pp_status pp_dpps_kernel_times(pp_ctx* ctx, int32_t reps, float* scan_ms, float* value_ms);

/* Cell count of a grid: kick_type_count * n_directions * n_powers. */
int64_t pp_grid_cells(const pp_search_grid* grid);

/* ---- score_pass on explicit candidates (pass_eval.cpp:148-173) ---------
 * Candidates are given as receive points + times; `feasible` must be set
 * for every entry (PP_DOMAIN otherwise, like score_pass). */
pp_status pp_score_cells(pp_ctx* ctx, const pp_world* world, const pp_params* params,
                         int64_t n, const double* rx, const double* ry, const double* our_time,
                         const double* opp_time, const uint8_t* feasible, double* score_out,
                         pp_pass_features* features_out);

/* goal_view at n points (pass_eval.cpp:55-126): angle, window, target. */
pp_status pp_goal_views(pp_ctx* ctx, const pp_world* world, double robot_radius, int64_t n,
                        const double* px, const double* py, double* angle, double* window_lo,
                        double* window_hi, double* target_y);

/* ---- running-point map + best_running_points (offball.cpp:176-258) ---- */
pp_status pp_runmap(pp_ctx* ctx, const pp_world* world, const pp_params* params,
                    const pp_runmap_request* req, void* block, int64_t block_vertices);

/* score_running_point at n explicit points (offball.cpp:176-201).  ok[i] = 0
 * where the reference throws domain_error (outside the front field or
 * strictly inside their defense area); score/features are then undefined. */
pp_status pp_score_running_points(pp_ctx* ctx, const pp_world* world, const pp_params* params,
                                  int64_t n, const double* px, const double* py,
                                  double* score_out, pp_run_features* features_out,
                                  uint8_t* ok_out);

/* guard_points (offball.hpp:75, offball.cpp:125-135) and guard_time
 * (offball.hpp:72, offball.cpp:137-174) at n points of the plane.  The
 * guards are the world's opponents ranked by distance to their defense area
 * (ties by id); `limits` are the guards' motion limits.  cap must be positive
 * and finite (PP_DOMAIN otherwise, as guard_time throws).  guard_pq: n x 4
 * doubles (P.x, P.y, Q.x, Q.y) or NULL; guard_time: n or NULL; ok[i] = 0
 * where the reference throws domain_error (strictly inside the area). */
pp_status pp_guard_points(pp_ctx* ctx, const pp_world* world, const pp_motion_limits* limits,
                          double cap, int64_t n, const double* px, const double* py,
                          double* guard_pq, double* guard_time, uint8_t* ok_out);

/* ---- the reference's per-pair plug-in point -----------------------------
 * kernels::KernelBackend::scan_first (kernels/kernel.hpp:46-53): for one ray
 * of trajectory samples and one robot, the first k in [k_begin, k_end) whose
 * sample passes sample_feasible (kernel.hpp:33-44), else -1.  The search
 * (pp_dpps) does not go through this interface -- one call is a single
 * (trajectory, robot) pair -- it is here so the reference's backend registry
 * has a B200 entry ("sm100a").  n independent pairs per call, one warp each;
 * ts / ss are the caller's host arrays (read for [k_begin, k_end) only). */
typedef struct pp_robot_kin { /* kernels::RobotKin, kernel.hpp:10-16 */
  double px, py, vx, vy, accel, decel, vmax, radius, vbound;
} pp_robot_kin;

typedef struct pp_scan_batch { /* kernels::ScanBatch, kernel.hpp:20-27 */
  const double* ts;
  const double* ss;
  int32_t k_begin, k_end; /* k_end exclusive */
  double ox, oy, ux, uy;
} pp_scan_batch;

pp_status pp_scan_first(pp_ctx* ctx, int64_t n, const pp_scan_batch* batches,
                        const pp_robot_kin* kins, int32_t* first_k);

/* ---- batched frames (log replay / what-if states) ----------------------
 * Independent frames share params and grid; each gets the pp_dpps summary.
 * kicker_ids may be NULL: then the kicker is the teammate nearest the ball
 * (ties to the earlier entry).  Frames shard across contexts/devices by the
 * caller (one context per GPU, contiguous ranges). */
pp_status pp_dpps_batch(pp_ctx* ctx, const pp_world* frames, int64_t n_frames,
                        const pp_params* params, const pp_search_grid* grid,
                        const int32_t* kicker_ids, pp_dpps_summary* summaries);

/* Compact per-frame result of a batch (48 B): what log replay / what-if
 * callers keep of each frame -- best_pass for all / flat / chip and the
 * feasible counts (pass_eval.cpp:175-192, dpps.cpp:64-70). */
typedef struct pp_frame_summary {
  double best_score[3];   /* 0 when best_cell is -1 */
  int32_t best_cell[3];   /* cell index (CandidateGrid order), -1 = nullopt */
  int32_t n_feasible[3];  /* all / flat / chip */
} pp_frame_summary;

/* Batched frames end to end (the C5 log-replay path): the raw world states
 * are copied to the device (one DMA; pinned memory from pp_host_alloc for
 * full speed) and staged there -- teams id-sorted (dpps.cpp:79-92), the
 * kicker chosen (kicker_ids[i], or the teammate nearest the ball when
 * kicker_ids is NULL, ties to the earlier entry) -- then searched, scored
 * and reduced on the device; one pp_frame_summary per frame comes back.
 * PP_VALIDATION names the first frame whose kicker is not on team ours or
 * whose team size is outside [0, 16] (the reference's run_dpps check,
 * dpps.cpp:221-223).  Frames shard across devices by the caller. */
pp_status pp_dpps_frames(pp_ctx* ctx, const pp_world* frames, int64_t n_frames,
                         const pp_params* params, const pp_search_grid* grid,
                         const int32_t* kicker_ids, pp_frame_summary* out);

/* pp_dpps_frames over several devices from one process (SURVEY.md 8(b)3's
 * pp_dpps_batch(per_gpu, n_gpu, ...) shape): frames split into n_ctx
 * contiguous ranges, range i on ctxs[i] (one context per GPU; distinct
 * contexts), all devices searching concurrently; out[i] is frame i's result
 * as pp_dpps_frames gives it.  Errors: the first failing context's status;
 * pp_last_error(ctxs[0]) names the context and the frame (index into
 * `frames`).  Replaces the reference's frame loop over run_dpps + best_pass
 * (passplan_main.cpp:87,102-104; dpps.cpp:217-321). */
pp_status pp_dpps_frames_multi(pp_ctx* const* ctxs, int32_t n_ctx, const pp_world* frames,
                               int64_t n_frames, const pp_params* params,
                               const pp_search_grid* grid, const int32_t* kicker_ids,
                               pp_frame_summary* out);

/* Device-resident pieces of pp_dpps_frames, for benchmarking and pipelined
 * callers: pp_batch_upload copies the raw frames to HBM (asynchronously on
 * the context's stream); pp_batch_run stages them and runs the search on the
 * device, enqueued on the context's stream and NOT synchronised (device_ms,
 * if non-NULL, synchronises and returns the device time of the run);
 * pp_batch_download waits and copies the per-frame results back. */
pp_status pp_batch_upload(pp_ctx* ctx, const pp_world* frames, int64_t n_frames,
                          const int32_t* kicker_ids);
pp_status pp_batch_run(pp_ctx* ctx, const pp_params* params, const pp_search_grid* grid,
                       float* device_ms);
pp_status pp_batch_download(pp_ctx* ctx, pp_frame_summary* out);
/* Kernels of the last pp_batch_run: number of pipeline launches and
 * the summed device time of its scan and value kernels, measured on a
 * re-run with events between the two (no overlap), `reps` times averaged. */
pp_status pp_batch_kernel_times(pp_ctx* ctx, const pp_params* params, const pp_search_grid* grid,
                                int32_t reps, float* stage_ms, float* scan_ms, float* value_ms,
                                int32_t* n_scan_launches);

/* ---- interception, possession, shot decision, free kick ----------------
 * (SURVEY §8(f) rows 2-4.)  One trajectory against robots, one warp per
 * robot scanning 32 samples per step on the device. */

typedef struct pp_kick { /* BallTrajectory::{flat_kick,chip_kick,free_roll}, ball_model.hpp:43-52 */
  double origin_x, origin_y;
  double dir_x, dir_y; /* kick direction; for a free roll the ball velocity */
  double speed;        /* kick speed; ignored for a free roll (|velocity|) */
  int32_t kind;        /* 0 flat kick, 1 chip kick, 2 free roll */
  int32_t pad;
} pp_kick;

typedef struct pp_trajectory { /* BallTrajectory, ball_model.hpp:27-66 */
  double origin_x, origin_y;
  double dir_x, dir_y; /* unit direction */
  double kick_speed, v1, slide_decel, roll_decel;
  double slide_end_time, slide_end_distance, stop_time, stop_distance, interceptable_from;
  int32_t kick_type; /* 0 flat, 1 chip */
  int32_t pad;
} pp_trajectory;

/* BallTrajectory::{flat_kick,chip_kick,free_roll} (ball_model.cpp:12-75):
 * PP_CONFIG for an invalid ball model, PP_DOMAIN for a negative / non-finite
 * speed or a zero direction with speed > 0.  Host only; msg may be NULL. */
pp_status pp_kick_trajectory(const pp_kick* kick, const pp_ball_model* ball, pp_trajectory* out,
                             char* msg, size_t msg_len);

typedef struct pp_intercept { /* InterceptResult, intercept.hpp:13-20 */
  int32_t team;     /* 0 ours, 1 theirs */
  int32_t robot_id;
  int32_t finite;   /* 0 = Never (intercept_time nullopt) */
  int32_t pad;
  double time, point_x, point_y;
} pp_intercept;

/* intercept_all (intercept.hpp:50-53, intercept.cpp:167-196): out[] gets
 * n_ours + n_theirs results, ours then theirs, each team in id order; the
 * teams' motion limits and robot_radius come from params.  dt <= 0 ->
 * PP_DOMAIN. */
pp_status pp_intercept_all(pp_ctx* ctx, const pp_world* world, const pp_params* params,
                           const pp_trajectory* traj, double dt, pp_intercept* out);

typedef struct pp_possession_report { /* PossessionReport, pass_eval.hpp:93-99 */
  int32_t side; /* 0 ours, 1 theirs, 2 contested */
  int32_t has_our, has_their, pad;
  double our_time, their_time;
} pp_possession_report;

/* possession (pass_eval.cpp:271-298): the ball's free roll sampled at
 * thresholds.possession_dt against both teams. */
pp_status pp_possession(pp_ctx* ctx, const pp_world* world, const pp_params* params,
                        pp_possession_report* out);

typedef struct pp_shot_decision { /* ShotDecision, pass_eval.hpp:62-70 */
  int32_t shoot, blocked;
  int32_t reason; /* 0 angle_too_small, 1 interceptable, 2 clear */
  int32_t pad;
  double shot_angle, target_x, target_y;
} pp_shot_decision;

/* decide_shot (pass_eval.cpp:194-233) for our robot shooter_id (not on team
 * ours -> PP_VALIDATION, as the CLI's lookup). */
pp_status pp_decide_shot(pp_ctx* ctx, const pp_world* world, const pp_params* params,
                         int32_t shooter_id, pp_shot_decision* out);

typedef struct pp_candidate { /* PassCandidate, dpps.hpp:47-57 */
  int32_t kick_type; /* 0 flat, 1 chip */
  int32_t dir_index, power_index, our_id, opp_id, feasible;
  double our_time, opp_time, receive_x, receive_y;
} pp_candidate;

typedef struct pp_free_kick_plan { /* FreeKickPlan, pass_eval.hpp:79-86 */
  double t_ball, t_robot;
  int32_t order; /* 0 robot_first, 1 kick_first */
  int32_t pad;
  double kick_delay;
} pp_free_kick_plan;

/* plan_free_kick (pass_eval.cpp:235-269), host scalar arithmetic. */
pp_status pp_plan_free_kick(pp_ctx* ctx, const pp_world* world, const pp_params* params,
                            int32_t kicker_id, const pp_candidate* target,
                            pp_free_kick_plan* out);

#ifdef __cplusplus
}
#endif

#endif /* PASSPLAN_B200_H_ */
