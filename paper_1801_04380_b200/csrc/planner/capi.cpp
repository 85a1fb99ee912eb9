// C ABI of the planner (declared in include/superneurons.h).
#include <algorithm>
#include <array>
#include <cstring>
#include <exception>
#include <new>
#include <string>

#include "handle.hpp"

namespace {
thread_local std::string g_err;
thread_local int g_err_kind = SN_EK_NONE;

int set_err(int kind, const std::string& msg) {
  g_err = msg;
  g_err_kind = kind;
  switch (kind) {
    case SN_EK_SCHED:
    case SN_EK_POOLEXH:
    case SN_EK_ALLLOCKED:
      return SN_ERR_SCHED;
    case SN_EK_CONFIG:
    case SN_EK_COST:
    case SN_EK_NETVALID:
    case SN_EK_POOL:
      return SN_ERR_CONFIG;
    case SN_EK_CUDA:
      return SN_ERR_CUDA;
    default:
      return SN_ERR_OTHER;
  }
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    g_err_kind = SN_EK_NONE;
    return SN_OK;
  } catch (const snp::PlanError& e) {
    return set_err(e.kind, e.what());
  } catch (const std::bad_alloc&) {
    return set_err(SN_EK_INTERNAL, "out of host memory");
  } catch (const std::exception& e) {
    return set_err(SN_EK_INTERNAL, e.what());
  }
}

snp::Plan make_plan(const sn_net_desc* net, const sn_sim_config* cfg) {
  snp::Plan p;
  p.net = snp::Net::from_desc(net);
  p.pool_bytes = cfg->pool_bytes;
  p.feats.liveness = cfg->liveness != 0;
  p.feats.offload = cfg->offload != 0;
  p.feats.cache = cfg->cache != 0;
  p.feats.recompute = cfg->recompute;
  p.feats.convselect = cfg->convselect != 0;
  p.cost_cfg.batch = cfg->batch;
  p.cost_cfg.dtype_bytes = cfg->dtype_bytes;
  p.cost_cfg.time_per_elem = cfg->time_per_elem;
  p.cost_cfg.heavy_time_per_elem = cfg->heavy_time_per_elem;
  p.cost_cfg.backward_time_factor = cfg->backward_time_factor;
  p.cost_cfg.bandwidth = cfg->bandwidth_bytes_per_s;
  return p;
}

template <class T, class Src, class Conv>
int copy_out_array(const Src& src, T* dst, size_t cap, size_t* n, Conv conv) {
  if (n) *n = src.size();
  if (!dst) return SN_OK;
  if (cap < src.size()) return set_err(SN_EK_INTERNAL, "output buffer too small");
  for (size_t i = 0; i < src.size(); ++i) dst[i] = conv(src[i]);
  return SN_OK;
}
}  // namespace

extern "C" {

const char* sn_last_error(void) { return g_err.c_str(); }
int sn_last_error_kind(void) { return g_err_kind; }

int sn_plan_create(const sn_net_desc* net, const sn_sim_config* cfg, sn_plan** out) {
  if (!net || !cfg || !out) return set_err(SN_EK_INTERNAL, "null argument");
  *out = nullptr;
  sn_plan* h = new (std::nothrow) sn_plan;
  if (!h) return set_err(SN_EK_INTERNAL, "out of host memory");
  const int rc = guarded([&] {
    h->plan = make_plan(net, cfg);
    snp::run_plan(h->plan);
  });
  if (rc != SN_OK) {
    delete h;
    return rc;
  }
  *out = h;
  return SN_OK;
}

int sn_analyze(const sn_net_desc* net, const sn_sim_config* cfg, sn_plan** out) {
  if (!net || !cfg || !out) return set_err(SN_EK_INTERNAL, "null argument");
  *out = nullptr;
  sn_plan* h = new (std::nothrow) sn_plan;
  if (!h) return set_err(SN_EK_INTERNAL, "out of host memory");
  const int rc = guarded([&] {
    h->plan = make_plan(net, cfg);
    snp::analyze_plan(h->plan);
  });
  if (rc != SN_OK) {
    delete h;
    return rc;
  }
  *out = h;
  return SN_OK;
}

int sn_build_costs(const sn_net_desc* net, const sn_sim_config* cfg, sn_plan** out) {
  if (!net || !cfg || !out) return set_err(SN_EK_INTERNAL, "null argument");
  *out = nullptr;
  sn_plan* h = new (std::nothrow) sn_plan;
  if (!h) return set_err(SN_EK_INTERNAL, "out of host memory");
  const int rc = guarded([&] {
    h->plan = make_plan(net, cfg);
    snp::costs_only(h->plan);
  });
  if (rc != SN_OK) {
    delete h;
    return rc;
  }
  *out = h;
  return SN_OK;
}

void sn_plan_destroy(sn_plan* plan) { delete plan; }

int sn_plan_report(const sn_plan* plan, sn_report* out) {
  if (!plan || !out) return set_err(SN_EK_INTERNAL, "null argument");
  *out = plan->plan.report;
  return SN_OK;
}

int sn_plan_rows(const sn_plan* plan, sn_step_row* rows, size_t cap, size_t* n) {
  if (!plan) return set_err(SN_EK_INTERNAL, "null argument");
  return copy_out_array(plan->plan.rows, rows, cap, n, [](const snp::Row& r) {
    sn_step_row o{};
    o.index = r.index;
    o.layer = r.layer;
    o.phase = r.phase;
    o.resident_bytes = r.resident;
    o.live_count = r.live;
    o.pool_used_bytes = r.pool_used;
    o.compute_s = r.compute_s;
    o.stall_s = r.stall_s;
    o.transfer_bytes = r.transfer;
    return o;
  });
}

int sn_plan_selections(const sn_plan* plan, sn_selection* sel, size_t cap, size_t* n) {
  if (!plan) return set_err(SN_EK_INTERNAL, "null argument");
  return copy_out_array(plan->plan.sels, sel, cap, n, [](const snp::Sel& s) {
    sn_selection o{};
    o.step = s.step;
    o.layer = s.layer;
    o.phase = s.phase;
    o.algo = s.algo;
    o.workspace_bytes = s.ws;
    o.free_bytes = s.free;
    return o;
  });
}

int sn_plan_modes(const sn_plan* plan, int32_t* modes, size_t cap, size_t* n) {
  if (!plan) return set_err(SN_EK_INTERNAL, "null argument");
  return copy_out_array(plan->plan.modes, modes, cap, n, [](int m) { return static_cast<int32_t>(m); });
}

int sn_plan_tape(const sn_plan* plan, const sn_event** events, size_t* n) {
  if (!plan || !events || !n) return set_err(SN_EK_INTERNAL, "null argument");
  *events = plan->plan.tape_c.data();
  *n = plan->plan.tape_c.size();
  return SN_OK;
}

int sn_plan_costs(const sn_plan* plan, sn_layer_cost* costs, size_t cap, size_t* n) {
  if (!plan) return set_err(SN_EK_INTERNAL, "null argument");
  return copy_out_array(plan->plan.costs, costs, cap, n, [](const snp::Cost& c) {
    sn_layer_cost o{};
    o.ndim = static_cast<int32_t>(c.shape.size());
    for (size_t i = 0; i < c.shape.size() && i < 3; ++i) o.shape[i] = c.shape[i];
    o.out_elems = c.out_elems;
    o.out_bytes = c.out_bytes;
    o.device_bytes = c.device_bytes;
    o.grad_bytes = c.grad_bytes;
    o.param_bytes = c.param_bytes;
    o.fwd_time = c.fwd_time;
    o.bwd_time = c.bwd_time;
    return o;
  });
}

int sn_plan_order(const sn_plan* plan, int32_t* ids, size_t cap, size_t* n) {
  if (!plan) return set_err(SN_EK_INTERNAL, "null argument");
  return copy_out_array(plan->plan.sched.forward_ids, ids, cap, n, [](int v) { return static_cast<int32_t>(v); });
}

int sn_plan_demands(const sn_plan* plan, int64_t* demands, size_t cap, size_t* n) {
  if (!plan) return set_err(SN_EK_INTERNAL, "null argument");
  return copy_out_array(plan->plan.demands, demands, cap, n, [](int64_t v) { return v; });
}

struct sn_pool {
  snp::BlockPool pool;
  explicit sn_pool(int64_t cap) : pool(cap) {}
};

int sn_pool_create(int64_t capacity_bytes, sn_pool** out) {
  if (!out) return set_err(SN_EK_INTERNAL, "null argument");
  *out = nullptr;
  return guarded([&] { *out = new sn_pool(capacity_bytes); });
}

void sn_pool_destroy(sn_pool* pool) { delete pool; }

int sn_pool_alloc(sn_pool* pool, int64_t key, int64_t nbytes, int32_t high, int64_t* block_offset) {
  if (!pool) return set_err(SN_EK_INTERNAL, "null argument");
  return guarded([&] {
    const int64_t off = pool->pool.alloc(key, nbytes, high != 0);
    if (block_offset) *block_offset = off;
  });
}

int sn_pool_free(sn_pool* pool, int64_t key) {
  if (!pool) return set_err(SN_EK_INTERNAL, "null argument");
  return guarded([&] { pool->pool.free(key); });
}

int sn_pool_check(const sn_pool* pool) {
  if (!pool) return set_err(SN_EK_INTERNAL, "null argument");
  return guarded([&] { pool->pool.check(); });
}

int sn_pool_stats(const sn_pool* pool, int64_t* used, int64_t* free_bytes, int64_t* high_water,
                  int64_t* capacity_blocks, int64_t* n_keys) {
  if (!pool) return set_err(SN_EK_INTERNAL, "null argument");
  if (used) *used = pool->pool.used_bytes();
  if (free_bytes) *free_bytes = pool->pool.free_bytes();
  if (high_water) *high_water = pool->pool.high_water_bytes();
  if (capacity_blocks) *capacity_blocks = pool->pool.capacity_blocks();
  if (n_keys) *n_keys = static_cast<int64_t>(pool->pool.n_keys());
  return SN_OK;
}

int sn_pool_spans(const sn_pool* pool, int32_t is_free, int64_t* offsets, int64_t* lengths, int64_t* keys,
                  size_t cap, size_t* n) {
  if (!pool || !n) return set_err(SN_EK_INTERNAL, "null argument");
  std::vector<std::array<int64_t, 3>> spans;
  if (is_free) {
    for (const auto& f : pool->pool.free_spans()) spans.push_back({f.first, f.second, -1});
  } else {
    for (const auto& kv : pool->pool.allocated()) spans.push_back({kv.second.first, kv.second.second, kv.first});
    std::sort(spans.begin(), spans.end());
  }
  *n = spans.size();
  if (!offsets) return SN_OK;
  if (cap < spans.size()) return set_err(SN_EK_INTERNAL, "output buffer too small");
  for (size_t i = 0; i < spans.size(); ++i) {
    offsets[i] = spans[i][0];
    if (lengths) lengths[i] = spans[i][1];
    if (keys) keys[i] = spans[i][2];
  }
  return SN_OK;
}

int sn_debug_pyset(const int64_t* a, size_t na, const int64_t* b, size_t nb, const int64_t* a2, size_t na2,
                   int64_t* out, size_t cap, size_t* n) {
  snp::PySet A, B;
  for (size_t i = 0; i < na; ++i) A.add(a[i]);
  for (size_t i = 0; i < nb; ++i) B.add(b[i]);
  A.update(B);
  for (size_t i = 0; i < na2; ++i) A.add(a2[i]);
  const std::vector<int64_t> items = A.items();
  return copy_out_array(items, out, cap, n, [](int64_t v) { return v; });
}

}  // extern "C"
