// dev_ik.cuh — parameters of the damped-least-squares contact IK (reference
// ik.cpp:31-139) and realize_grasp (pipeline.cpp:185-253).  The solver itself
// is warp-cooperative, see dev_ikw.cuh.
#pragma once

#include "dev_geom.cuh"

namespace lgd {

struct IkCfg {
  double beta, step_clamp, residual_tol, damping_scale, damping_min;
  int iterations, max_backtracks;
};

}  // namespace lgd
