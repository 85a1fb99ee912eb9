// One training iteration of the memory-scheduled step, as a deterministic
// event loop (memsched L5, simulator.py:191-731).  Produces the SimReport
// fields, the step rows, the conv-algorithm selections and -- for the B200
// executor -- the physical event tape (arena offsets, copies, replays).
#pragma once
#include <vector>

#include "analysis.hpp"
#include "pool.hpp"

namespace snp {

struct Features {
  bool liveness = false, offload = false, cache = false, convselect = false;
  int recompute = SN_RC_NONE;
};

struct Row {
  double index;
  int layer, phase;  // phase 0 fwd, 1 bwd, 2 replay
  int64_t resident, live, pool_used;
  double compute_s, stall_s;
  int64_t transfer;
};

struct Sel {
  double step;
  int layer, phase, algo;
  int64_t ws, free;
};

struct Event {
  char op;
  int a = 0, b = 0, e = 0;
  int64_t c = 0, d = 0;
};

struct Plan {
  Net net;
  Schedule sched;
  std::vector<Cost> costs;
  CostCfg cost_cfg;
  Features feats;
  int64_t pool_bytes = 0;
  // results
  std::vector<int64_t> demands;
  int64_t min_pool = 0;
  sn_report report{};
  std::vector<Row> rows;
  std::vector<Sel> sels;
  std::vector<int> modes;
  std::vector<Event> tape;
  std::vector<sn_event> tape_c;  // C-ABI view
  int64_t pool_capacity_blocks = 0;
};

// Full planning + simulation (run_simulation).  Throws PlanError.
void run_plan(Plan& p);
// Costs, order and demands only (analysis API); no pool-size check.
void analyze_plan(Plan& p);
// Cost table only (costmodel.build_costs semantics: no schedule validation).
void costs_only(Plan& p);

}  // namespace snp
