// Opaque C handle behind sn_plan* (shared by libsnplan and libsnexec).
#pragma once
#include "sim.hpp"

struct sn_plan {
  snp::Plan plan;
};
