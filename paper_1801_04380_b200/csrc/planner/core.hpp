// Planner core types: the validated layer graph, its 2N-step schedule and the
// per-layer cost table.  Restates memsched's L1/L2 (netgraph.py, costmodel.py)
// in C++ with exact integer byte accounting and IEEE-double time arithmetic in
// the reference's operation order (compiled with -ffp-contract=off).
#pragma once
#include <array>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "superneurons.h"

namespace snp {

// Exception carrying the reference exception kind (sn_error_kind).
struct PlanError : std::runtime_error {
  int kind;
  PlanError(int k, const std::string& msg) : std::runtime_error(msg), kind(k) {}
};

[[noreturn]] inline void fail(int kind, const std::string& msg) { throw PlanError(kind, msg); }

enum Kind { DATA = 0, CONV, POOL, ACT, LRN, BN, FC, DROPOUT, SOFTMAX, JOIN, NKIND };

inline bool is_inplace(int k) { return k == ACT || k == DROPOUT; }         // GRAD_INPLACE_KINDS
inline bool is_checkpoint(int k) { return k == CONV || k == FC; }          // CHECKPOINT_KINDS
inline bool is_offload_kind(int k) { return k == CONV; }                   // OFFLOAD_KINDS
inline bool is_heavy(int k) { return k == CONV || k == FC; }               // HEAVY_KINDS
inline bool needs_x(int k) { return k == CONV || k == FC || k == POOL || k == ACT || k == LRN || k == BN; }
inline bool needs_y(int k) { return k == POOL || k == ACT || k == LRN || k == BN || k == DROPOUT || k == SOFTMAX; }
inline bool has_backward_needs(int k) { return needs_x(k) || needs_y(k); }

struct Net {
  std::string name;
  int n = 0;
  std::vector<int> kind;
  std::vector<std::string> names, reprs;
  std::vector<std::vector<int>> prev, next;
  std::vector<std::array<int8_t, SN_NPARAM>> pstate;
  std::vector<std::array<int64_t, SN_NPARAM>> pint;
  std::vector<std::array<std::string, SN_NPARAM>> prepr;

  static Net from_desc(const sn_net_desc* d);
  int terminal_id() const;  // first layer with no successors
  // Producer ids whose forward tensors layer `lid`'s backward reads (with
  // duplicates, BACKWARD_NEEDS order: "x" = every prev, then "y" = itself).
  void backward_reads(int lid, std::vector<int>& out) const;
  // Same, de-duplicated preserving first occurrence (dict.fromkeys).
  std::vector<int> backward_reads_unique(int lid) const;
  int grad_owner(int lid) const;  // -1 == None
};

struct Schedule {
  std::vector<int> forward_ids;
  std::vector<int> fwd_step_of, bwd_step_of;  // by layer id
  int n = 0;
  int num_steps() const { return 2 * n; }
  int layer_at(int step) const {
    return step < n ? forward_ids[step] : forward_ids[2 * n - 1 - step];
  }
  bool is_forward(int step) const { return step < n; }
};

// Iterative DFS with join gating (Alg. 1).  Returns fewer ids than layers
// when some layer is unreachable or on a cycle.
std::vector<int> forward_order_raw(const Net& net);
Schedule build_schedule(const Net& net);

struct Cost {
  std::vector<int64_t> shape;
  int64_t out_elems = 0, out_bytes = 0, device_bytes = 0, grad_bytes = 0, param_bytes = 0;
  double fwd_time = 0.0, bwd_time = 0.0;
};

struct CostCfg {
  int64_t batch = 200, dtype_bytes = 4;
  double time_per_elem = 2e-9, heavy_time_per_elem = 2e-8, backward_time_factor = 2.0;
  double bandwidth = 8e9;
};

std::vector<Cost> build_costs(const Net& net, const CostCfg& cfg);

// Overflow-checked int64 helpers (Python ints are unbounded; we refuse instead).
int64_t mul_checked(int64_t a, int64_t b);
int64_t add_checked(int64_t a, int64_t b);
int64_t py_floordiv(int64_t a, int64_t b);  // raises ZeroDivisionError kind on b == 0

std::string py_tuple_repr(const std::vector<int64_t>& v);
std::string py_list_repr_names(const Net& net, const std::vector<int>& ids);

}  // namespace snp
