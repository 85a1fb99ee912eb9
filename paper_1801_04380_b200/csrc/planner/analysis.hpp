// Static analyses over the schedule (memsched L3): tensor use steps and
// lifetimes, gradient-buffer windows, the offload plan, recompute segments and
// policy, and the per-step demand floor max_i(l_i).  Each table is computed once
// (the reference rebuilds use tables per segment, O(N*S); here it is O(N)).
#pragma once
#include <vector>

#include "core.hpp"

namespace snp {

struct GradBuf {
  int owner;
  int64_t nbytes;
  int create_step, free_step;
};

struct Liveness {
  std::vector<std::vector<int>> fwd_uses, bwd_uses;  // sorted steps per producer
  std::vector<int> last_use, last_fwd_use;
};
Liveness build_liveness(const Net& net, const Schedule& s);

// liveness.grad_buffers (liveness.py:75-111): sorted by owner id.
std::vector<GradBuf> grad_buffers(const Net& net, const std::vector<Cost>& costs, const Schedule& s,
                                  bool materialize_seed);

struct Segment {
  int index;
  std::vector<int> members, anchors;
};
std::vector<Segment> build_segments(const Net& net, const Schedule& s);

struct OffloadPlan {
  std::vector<int> cp_ids;
  std::vector<int> drop_after;                 // -1 when absent
  std::vector<int> prefetch_issue;             // -1 when absent
  std::vector<int> first_bwd_use, last_bwd_use;  // -1 when absent
};
OffloadPlan build_offload_plan(const Net& net, const Schedule& s, const Liveness& lv);

struct RecomputePlan {
  int policy = SN_RC_NONE;
  std::vector<Segment> segments;
  std::vector<int> modes;  // SN_RC_SPEED or SN_RC_MEMORY per segment
  std::vector<char> spill;  // by layer id
  int64_t extra_forward_steps = 0;
  std::vector<int64_t> predictions;
};
RecomputePlan plan_recompute(const Net& net, const std::vector<Cost>& costs, const Schedule& s,
                             const Liveness& lv, int policy, const std::vector<char>& offloaded,
                             int64_t floor);

// recompute.step_demands (recompute.py:173-205).
std::vector<int64_t> step_demands(const Net& net, const std::vector<Cost>& costs, const Schedule& s);

// liveness.working_set_bytes (liveness.py:192-223).
int64_t working_set_bytes(const Net& net, const std::vector<Cost>& costs, const Schedule& s,
                          const std::vector<GradBuf>& buffers, int step);

// liveness.resident_curve(mode="liveness") peak (liveness.py:154-189).
int64_t liveness_peak(const Net& net, const std::vector<Cost>& costs, const Schedule& s, const Liveness& lv);

}  // namespace snp
