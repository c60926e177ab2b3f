/*
 * passplan_b200_layout.h -- byte layout of the result blocks declared in
 * passplan_b200.h.  Header-only so the product library, the CPU oracle and
 * the reference shim agree on one layout without linking each other.
 *
 * Grid block:    [summary][our_time f64][opp_time f64][rx f64][ry f64]
 *                [score f32][our_slot i8][opp_slot i8][feasible u8]
 * Runmap block:  [summary][px f64][py f64][score f64][features 5xf64][scorable u8]
 * Every array starts on a 16-byte boundary.  The order puts the summary
 * first so PP_COPY_SUMMARY is a prefix copy.
 */
#ifndef PASSPLAN_B200_LAYOUT_H_
#define PASSPLAN_B200_LAYOUT_H_

#include "passplan_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

static inline size_t pp_align16_(size_t x) { return (x + 15u) & ~(size_t)15u; }

typedef struct pp_grid_offsets_ {
  size_t summary, our_time, opp_time, rx, ry, score, our_slot, opp_slot, feasible, total;
} pp_grid_offsets_;

static inline pp_grid_offsets_ pp_grid_offsets_for_(int64_t n_cells) {
  pp_grid_offsets_ o;
  const size_t n = (size_t)(n_cells > 0 ? n_cells : 0);
  size_t at = 0;
  o.summary = at;  at = pp_align16_(at + sizeof(pp_dpps_summary));
  o.our_time = at; at = pp_align16_(at + 8 * n);
  o.opp_time = at; at = pp_align16_(at + 8 * n);
  o.rx = at;       at = pp_align16_(at + 8 * n);
  o.ry = at;       at = pp_align16_(at + 8 * n);
  o.score = at;    at = pp_align16_(at + 4 * n);
  o.our_slot = at; at = pp_align16_(at + n);
  o.opp_slot = at; at = pp_align16_(at + n);
  o.feasible = at; at = pp_align16_(at + n);
  o.total = at;
  return o;
}

static inline void pp_grid_view_of_(void* block, int64_t n_cells, pp_grid_view* v) {
  const pp_grid_offsets_ o = pp_grid_offsets_for_(n_cells);
  char* b = (char*)block;
  v->summary = (pp_dpps_summary*)(b + o.summary);
  v->our_time = (double*)(b + o.our_time);
  v->opp_time = (double*)(b + o.opp_time);
  v->rx = (double*)(b + o.rx);
  v->ry = (double*)(b + o.ry);
  v->score = (float*)(b + o.score);
  v->our_slot = (int8_t*)(b + o.our_slot);
  v->opp_slot = (int8_t*)(b + o.opp_slot);
  v->feasible = (uint8_t*)(b + o.feasible);
}

typedef struct pp_runmap_offsets_ {
  size_t summary, px, py, score, features, scorable, total;
} pp_runmap_offsets_;

static inline pp_runmap_offsets_ pp_runmap_offsets_for_(int64_t n_vertices) {
  pp_runmap_offsets_ o;
  const size_t n = (size_t)(n_vertices > 0 ? n_vertices : 0);
  size_t at = 0;
  o.summary = at;  at = pp_align16_(at + sizeof(pp_runmap_summary));
  o.px = at;       at = pp_align16_(at + 8 * n);
  o.py = at;       at = pp_align16_(at + 8 * n);
  o.score = at;    at = pp_align16_(at + 8 * n);
  o.features = at; at = pp_align16_(at + sizeof(pp_run_features) * n);
  o.scorable = at; at = pp_align16_(at + n);
  o.total = at;
  return o;
}

static inline void pp_runmap_view_of_(void* block, int64_t n_vertices, pp_runmap_view* v) {
  const pp_runmap_offsets_ o = pp_runmap_offsets_for_(n_vertices);
  char* b = (char*)block;
  v->summary = (pp_runmap_summary*)(b + o.summary);
  v->px = (double*)(b + o.px);
  v->py = (double*)(b + o.py);
  v->score = (double*)(b + o.score);
  v->features = (pp_run_features*)(b + o.features);
  v->scorable = (uint8_t*)(b + o.scorable);
}

#ifdef __cplusplus
}
#endif

#endif /* PASSPLAN_B200_LAYOUT_H_ */
