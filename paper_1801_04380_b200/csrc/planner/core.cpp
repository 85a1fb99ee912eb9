// Graph, schedule and cost table.  Follows memsched netgraph.py:241-321 and
// costmodel.py:93-221; every error path raises the reference's exception kind
// with the reference's message text.
#include "core.hpp"

#include <limits>

namespace snp {

static const char* kParamKeys[SN_NPARAM] = {"c", "h", "w", "out", "k", "s", "p"};

Net Net::from_desc(const sn_net_desc* d) {
  Net net;
  net.name = d->name ? d->name : "net";
  net.n = d->n_layers;
  net.kind.assign(d->kinds, d->kinds + net.n);
  net.names.resize(net.n);
  net.reprs.resize(net.n);
  net.prev.resize(net.n);
  net.next.resize(net.n);
  net.pstate.resize(net.n);
  net.pint.resize(net.n);
  net.prepr.resize(net.n);
  for (int i = 0; i < net.n; ++i) {
    if (net.kind[i] < 0 || net.kind[i] >= NKIND) fail(SN_EK_INTERNAL, "bad layer kind");
    net.names[i] = d->names[i];
    net.reprs[i] = d->name_reprs ? d->name_reprs[i] : ("'" + net.names[i] + "'");
    for (int j = d->prev_off[i]; j < d->prev_off[i + 1]; ++j) net.prev[i].push_back(d->prev_idx[j]);
    for (int j = d->next_off[i]; j < d->next_off[i + 1]; ++j) net.next[i].push_back(d->next_idx[j]);
    for (int p = 0; p < SN_NPARAM; ++p) {
      const size_t at = static_cast<size_t>(i) * SN_NPARAM + p;
      net.pstate[i][p] = d->param_state ? d->param_state[at] : 0;
      net.pint[i][p] = d->param_int ? d->param_int[at] : 0;
      if (net.pstate[i][p] == 2 && d->param_repr && d->param_repr[at]) net.prepr[i][p] = d->param_repr[at];
    }
  }
  for (int i = 0; i < net.n; ++i) {
    for (int v : net.prev[i])
      if (v < 0 || v >= net.n) fail(SN_EK_INTERNAL, "prev id out of range");
    for (int v : net.next[i])
      if (v < 0 || v >= net.n) fail(SN_EK_INTERNAL, "next id out of range");
  }
  return net;
}

int Net::terminal_id() const {
  for (int i = 0; i < n; ++i)
    if (next[i].empty()) return i;
  fail(SN_EK_NETVALID, "network has no terminal layer");
}

void Net::backward_reads(int lid, std::vector<int>& out) const {
  out.clear();
  const int k = kind[lid];
  if (needs_x(k)) out.insert(out.end(), prev[lid].begin(), prev[lid].end());
  if (needs_y(k)) out.push_back(lid);
}

std::vector<int> Net::backward_reads_unique(int lid) const {
  std::vector<int> raw, out;
  backward_reads(lid, raw);
  for (int r : raw) {
    bool seen = false;
    for (int o : out) seen |= (o == r);
    if (!seen) out.push_back(r);
  }
  return out;
}

int Net::grad_owner(int lid) const {
  while (true) {
    const int k = kind[lid];
    if (k == DATA) return -1;
    if (is_inplace(k)) {
      lid = prev[lid][0];
      continue;
    }
    return lid;
  }
}

std::vector<int> forward_order_raw(const Net& net) {
  int entry = -1;
  for (int i = 0; i < net.n; ++i)
    if (net.kind[i] == DATA && net.prev[i].empty()) {
      entry = i;
      break;
    }
  std::vector<int> order;
  if (entry < 0) return order;
  std::vector<int> arrived(net.n, 0);
  order.push_back(entry);
  std::vector<std::pair<int, size_t>> stack{{entry, 0}};
  while (!stack.empty()) {
    auto& top = stack.back();
    const std::vector<int>& succ = net.next[top.first];
    if (top.second == succ.size()) {
      stack.pop_back();
      continue;
    }
    const int nid = succ[top.second++];
    if (++arrived[nid] == static_cast<int>(net.prev[nid].size())) {
      order.push_back(nid);
      stack.emplace_back(nid, 0);
    }
  }
  return order;
}

Schedule build_schedule(const Net& net) {
  Schedule s;
  s.forward_ids = forward_order_raw(net);
  if (static_cast<int>(s.forward_ids.size()) != net.n)
    fail(SN_EK_NETVALID, "network has unreachable or cyclic layers");
  s.n = net.n;
  s.fwd_step_of.assign(net.n, -1);
  s.bwd_step_of.assign(net.n, -1);
  for (int i = 0; i < net.n; ++i) {
    s.fwd_step_of[s.forward_ids[i]] = i;
    s.bwd_step_of[s.forward_ids[i]] = 2 * net.n - 1 - i;
  }
  return s;
}

// ---------------------------------------------------------------------------

int64_t mul_checked(int64_t a, int64_t b) {
  int64_t r;
  if (__builtin_mul_overflow(a, b, &r)) fail(SN_EK_INTERNAL, "integer overflow in byte accounting");
  return r;
}
int64_t add_checked(int64_t a, int64_t b) {
  int64_t r;
  if (__builtin_add_overflow(a, b, &r)) fail(SN_EK_INTERNAL, "integer overflow in byte accounting");
  return r;
}
int64_t py_floordiv(int64_t a, int64_t b) {
  if (b == 0) fail(SN_EK_ZERODIV, "integer division or modulo by zero");
  int64_t q = a / b;
  if ((a % b != 0) && ((a < 0) != (b < 0))) --q;
  return q;
}

std::string py_tuple_repr(const std::vector<int64_t>& v) {
  std::string s = "(";
  for (size_t i = 0; i < v.size(); ++i) {
    if (i) s += ", ";
    s += std::to_string(v[i]);
  }
  if (v.size() == 1) s += ",";
  return s + ")";
}

std::string py_list_repr_names(const Net& net, const std::vector<int>& ids) {
  std::string s = "[";
  for (size_t i = 0; i < ids.size(); ++i) {
    if (i) s += ", ";
    s += net.reprs[ids[i]];
  }
  return s + "]";
}

namespace {

// costmodel._int_param (costmodel.py:70-80).  has_default == false means
// "no default" (the reference passes None).
int64_t int_param(const Net& net, int lid, int key, bool has_default, int64_t def) {
  const int8_t st = net.pstate[lid][key];
  if (st == 0) {
    if (has_default) return def;
    fail(SN_EK_COST, "layer " + net.reprs[lid] + " is missing parameter '" + kParamKeys[key] + "'");
  }
  if (st != 1)
    fail(SN_EK_COST, "layer " + net.reprs[lid] + " parameter '" + kParamKeys[key] +
                         "' must be an integer, got " + net.prepr[lid][key]);
  return net.pint[lid][key];
}

// costmodel._window (costmodel.py:83-90).
int64_t window(const Net& net, int lid, int64_t size, int64_t kernel, int64_t stride, int64_t pad) {
  const int64_t num = add_checked(add_checked(size, mul_checked(2, pad)), -kernel);
  const int64_t out = py_floordiv(num, stride) + 1;
  if (out < 1)
    fail(SN_EK_COST, "layer " + net.reprs[lid] + ": kernel " + std::to_string(kernel) + " stride " +
                         std::to_string(stride) + " pad " + std::to_string(pad) +
                         " does not fit input extent " + std::to_string(size));
  return out;
}

std::vector<int64_t> layer_shape(const Net& net, int lid, const std::vector<std::vector<int64_t>>& shapes) {
  const int k = net.kind[lid];
  if (k == DATA) {
    const int64_t c = int_param(net, lid, SN_P_C, false, 0);
    const int64_t h = int_param(net, lid, SN_P_H, false, 0);
    const int64_t w = int_param(net, lid, SN_P_W, false, 0);
    return {c, h, w};
  }
  const auto& prev = net.prev[lid];
  if (k == JOIN) {
    const auto& first = shapes[prev[0]];
    for (int pid : prev)
      if (shapes[pid] != first)
        fail(SN_EK_COST, "JOIN layer " + net.reprs[lid] + " merges mismatched shapes " +
                             py_tuple_repr(first) + " and " + py_tuple_repr(shapes[pid]) +
                             " (from " + net.reprs[pid] + ")");
    return first;
  }
  const auto& src = shapes[prev[0]];
  if (k == CONV) {
    if (src.size() != 3)
      fail(SN_EK_COST, "CONV layer " + net.reprs[lid] + " needs a (c, h, w) input, got " + py_tuple_repr(src));
    const int64_t out_c = int_param(net, lid, SN_P_OUT, false, 0);
    const int64_t kk = int_param(net, lid, SN_P_K, false, 0);
    const int64_t s = int_param(net, lid, SN_P_S, true, 1);
    const int64_t p = int_param(net, lid, SN_P_P, true, 0);
    const int64_t h = window(net, lid, src[1], kk, s, p);
    const int64_t w = window(net, lid, src[2], kk, s, p);
    return {out_c, h, w};
  }
  if (k == POOL) {
    if (src.size() != 3)
      fail(SN_EK_COST, "POOL layer " + net.reprs[lid] + " needs a (c, h, w) input, got " + py_tuple_repr(src));
    const int64_t kk = int_param(net, lid, SN_P_K, false, 0);
    const int64_t s = int_param(net, lid, SN_P_S, true, kk);
    const int64_t p = int_param(net, lid, SN_P_P, true, 0);
    const int64_t h = window(net, lid, src[1], kk, s, p);
    const int64_t w = window(net, lid, src[2], kk, s, p);
    return {src[0], h, w};
  }
  if (k == FC) return {int_param(net, lid, SN_P_OUT, false, 0)};
  return src;  // ACT, LRN, BN, DROPOUT, SOFTMAX
}

int64_t prod(const std::vector<int64_t>& v) {
  int64_t p = 1;
  for (int64_t x : v) p = mul_checked(p, x);
  return p;
}

}  // namespace

std::vector<Cost> build_costs(const Net& net, const CostCfg& cfg) {
  // propagate_shapes (costmodel.py:93-110): rounds over the still-pending layers
  // in id order; a layer resolves as soon as all its inputs have shapes.
  std::vector<std::vector<int64_t>> shapes(net.n);
  std::vector<char> have(net.n, 0);
  std::vector<int> pending(net.n);
  for (int i = 0; i < net.n; ++i) pending[i] = i;
  while (!pending.empty()) {
    bool progressed = false;
    std::vector<int> remaining;
    for (int lid : pending) {
      bool ready = true;
      for (int p : net.prev[lid]) ready &= have[p] != 0;
      if (ready) {
        shapes[lid] = layer_shape(net, lid, shapes);
        have[lid] = 1;
        progressed = true;
      } else {
        remaining.push_back(lid);
      }
    }
    if (!progressed) fail(SN_EK_COST, "cannot resolve shapes for layers " + py_list_repr_names(net, remaining));
    pending.swap(remaining);
  }

  std::vector<Cost> table(net.n);
  for (int lid = 0; lid < net.n; ++lid) {
    Cost& c = table[lid];
    const int k = net.kind[lid];
    c.shape = shapes[lid];
    c.out_elems = mul_checked(cfg.batch, prod(c.shape));
    c.out_bytes = mul_checked(c.out_elems, cfg.dtype_bytes);
    if (k == DATA) {
      c.device_bytes = 0;
      c.fwd_time = 0.0;
    } else {
      c.device_bytes = c.out_bytes;
      const double per_elem = is_heavy(k) ? cfg.heavy_time_per_elem : cfg.time_per_elem;
      c.fwd_time = per_elem * static_cast<double>(c.out_elems);
    }
    c.grad_bytes = (is_inplace(k) || k == DATA) ? 0 : c.device_bytes;
    const std::vector<int64_t>& in_shape = net.prev[lid].empty() ? c.shape : shapes[net.prev[lid][0]];
    int64_t pe = 0;
    if (k == CONV) {
      const int64_t kk = int_param(net, lid, SN_P_K, false, 0);
      pe = add_checked(mul_checked(mul_checked(mul_checked(kk, kk), in_shape[0]), c.shape[0]), c.shape[0]);
    } else if (k == FC) {
      pe = add_checked(mul_checked(prod(in_shape), c.shape[0]), c.shape[0]);
    } else if (k == BN) {
      pe = mul_checked(4, c.shape[0]);
    }
    c.param_bytes = mul_checked(pe, cfg.dtype_bytes);
    c.bwd_time = cfg.backward_time_factor * c.fwd_time;
  }
  return table;
}

}  // namespace snp
