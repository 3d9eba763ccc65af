// bode_program.cuh -- everything a run-time-compiled solver specialisation
// instantiates (bode_program.cu compiles it with NVRTC for sm_100a): the
// init pass and persistent kernel, the step_once kernel and the unit ops,
// for the method / dynamics the generated source defines
// (bode::Tab<BODE_METHOD_CUSTOM> for a user tableau, bode::UserDyn<O> for
// user dynamics or an alias of a registered functor).
#pragma once
#include "bode_joint_dev.cuh"
#include "bode_solver.cuh"
#include "bode_stepper.cuh"
#include "bode_units_dev.cuh"
