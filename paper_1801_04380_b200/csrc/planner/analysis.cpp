// Static analyses; see analysis.hpp.  Reference: memsched liveness.py:26-228,
// offload.py:25-73, recompute.py:61-253, netgraph.py:324-360.
#include "analysis.hpp"

#include <algorithm>
#include <unordered_map>

namespace snp {

Liveness build_liveness(const Net& net, const Schedule& s) {
  Liveness lv;
  lv.fwd_uses.assign(net.n, {});
  lv.bwd_uses.assign(net.n, {});
  std::vector<int> reads;
  for (int lid = 0; lid < net.n; ++lid) {
    for (int pid : net.prev[lid]) lv.fwd_uses[pid].push_back(s.fwd_step_of[lid]);
    const int step = s.bwd_step_of[lid];
    net.backward_reads(lid, reads);
    for (int t : reads) lv.bwd_uses[t].push_back(step);
  }
  lv.last_use.assign(net.n, 0);
  lv.last_fwd_use.assign(net.n, 0);
  for (int lid = 0; lid < net.n; ++lid) {
    std::sort(lv.fwd_uses[lid].begin(), lv.fwd_uses[lid].end());
    std::sort(lv.bwd_uses[lid].begin(), lv.bwd_uses[lid].end());
    int lf = s.fwd_step_of[lid];
    for (int u : lv.fwd_uses[lid]) lf = std::max(lf, u);
    int la = lf;
    for (int u : lv.bwd_uses[lid]) la = std::max(la, u);
    lv.last_fwd_use[lid] = lf;
    lv.last_use[lid] = la;
  }
  return lv;
}

std::vector<GradBuf> grad_buffers(const Net& net, const std::vector<Cost>& costs, const Schedule& s,
                                  bool materialize_seed) {
  std::vector<int> create(net.n, -1);
  auto note = [&](int owner, int step) {
    if (create[owner] < 0 || step < create[owner]) create[owner] = step;
  };
  for (int lid = 0; lid < net.n; ++lid) {
    if (net.kind[lid] == DATA) continue;
    const int step = s.bwd_step_of[lid];
    for (int pid : net.prev[lid]) {
      const int owner = net.grad_owner(pid);
      if (owner >= 0) note(owner, step);
    }
  }
  if (materialize_seed) {
    const int term = net.terminal_id();
    const int owner = net.grad_owner(term);
    if (owner >= 0) note(owner, s.bwd_step_of[term]);
  }
  std::vector<GradBuf> out;
  for (int owner = 0; owner < net.n; ++owner)
    if (create[owner] >= 0) out.push_back({owner, costs[owner].grad_bytes, create[owner], s.bwd_step_of[owner]});
  return out;
}

std::vector<Segment> build_segments(const Net& net, const Schedule& s) {
  std::vector<Segment> segs;
  std::vector<int> cur;
  auto flush = [&]() {
    if (cur.empty()) return;
    Segment seg;
    seg.index = static_cast<int>(segs.size());
    seg.members = cur;
    // netgraph.external_inputs: producers outside the run, first-use order.
    std::vector<char> inside(net.n, 0), seen(net.n, 0);
    for (int m : cur) inside[m] = 1;
    for (int m : cur)
      for (int p : net.prev[m])
        if (!inside[p] && !seen[p]) {
          seen[p] = 1;
          seg.anchors.push_back(p);
        }
    segs.push_back(std::move(seg));
    cur.clear();
  };
  for (int lid : s.forward_ids) {
    const int k = net.kind[lid];
    if (k == DATA || is_checkpoint(k))
      flush();
    else
      cur.push_back(lid);
  }
  flush();
  return segs;
}

OffloadPlan build_offload_plan(const Net& net, const Schedule& s, const Liveness& lv) {
  OffloadPlan p;
  for (int lid : s.forward_ids)
    if (is_offload_kind(net.kind[lid])) p.cp_ids.push_back(lid);
  p.drop_after.assign(net.n, -1);
  p.prefetch_issue.assign(net.n, -1);
  p.first_bwd_use.assign(net.n, -1);
  p.last_bwd_use.assign(net.n, -1);
  for (size_t pos = 0; pos < p.cp_ids.size(); ++pos) {
    const int cp = p.cp_ids[pos];
    p.drop_after[cp] = lv.last_fwd_use[cp];
    const auto& uses = lv.bwd_uses[cp];
    if (uses.empty()) continue;
    p.first_bwd_use[cp] = uses.front();
    p.last_bwd_use[cp] = uses.back();
    const int cand = pos + 1 < p.cp_ids.size() ? s.bwd_step_of[p.cp_ids[pos + 1]] : uses.front();
    p.prefetch_issue[cp] = std::min(cand, uses.front());
  }
  return p;
}

namespace {

int first_backward_use(const Liveness& lv, const Segment& seg) {
  int best = -1;
  for (int m : seg.members)
    for (int u : lv.bwd_uses[m])
      if (best < 0 || u < best) best = u;
  return best;
}

int64_t speed_prediction(const Net& net, const std::vector<Cost>& costs, const Schedule& s,
                         const Liveness& lv, const Segment& seg, int terminal) {
  const int step = first_backward_use(lv, seg);
  if (step < 0) return 0;
  int64_t total = 0;
  for (int a : seg.anchors) total = add_checked(total, costs[a].device_bytes);
  for (int m : seg.members) total = add_checked(total, costs[m].device_bytes);
  const int user = s.layer_at(step);
  const int dy_owner = net.grad_owner(user);
  if (dy_owner >= 0 && user != terminal) total = add_checked(total, costs[dy_owner].grad_bytes);
  for (int pid : net.prev[user]) {
    const int owner = net.grad_owner(pid);
    if (owner >= 0 && owner != dy_owner) total = add_checked(total, costs[owner].grad_bytes);
  }
  return total;
}

}  // namespace

RecomputePlan plan_recompute(const Net& net, const std::vector<Cost>& costs, const Schedule& s,
                             const Liveness& lv, int policy, const std::vector<char>& offloaded,
                             int64_t floor) {
  RecomputePlan rp;
  rp.policy = policy;
  rp.segments = build_segments(net, s);
  const int terminal = net.terminal_id();
  for (const Segment& seg : rp.segments) rp.predictions.push_back(speed_prediction(net, costs, s, lv, seg, terminal));
  for (const Segment& seg : rp.segments) {
    int mode;
    if (policy == SN_RC_SPEED) mode = SN_RC_SPEED;
    else if (policy == SN_RC_MEMORY) mode = SN_RC_MEMORY;
    else mode = rp.predictions[seg.index] <= floor ? SN_RC_SPEED : SN_RC_MEMORY;
    rp.modes.push_back(mode);
  }
  for (const Segment& seg : rp.segments) {
    if (rp.modes[seg.index] == SN_RC_SPEED) {
      if (first_backward_use(lv, seg) >= 0) rp.extra_forward_steps += static_cast<int64_t>(seg.members.size());
    } else {
      for (size_t i = 0; i < seg.members.size(); ++i)
        if (has_backward_needs(net.kind[seg.members[i]])) rp.extra_forward_steps += static_cast<int64_t>(i + 1);
    }
  }
  rp.spill.assign(net.n, 0);
  std::vector<char> member(net.n, 0);
  for (const Segment& seg : rp.segments)
    for (int m : seg.members) member[m] = 1;
  std::vector<int> reads;
  for (int lid = 0; lid < net.n; ++lid) {
    if (net.kind[lid] == DATA) continue;
    net.backward_reads(lid, reads);
    for (int r : reads)
      if (!member[r] && !offloaded[r] && costs[r].device_bytes > 0) rp.spill[r] = 1;
  }
  for (const Segment& seg : rp.segments) {
    for (int a : seg.anchors)
      if (!offloaded[a] && costs[a].device_bytes > 0) rp.spill[a] = 1;
    if (rp.modes[seg.index] == SN_RC_MEMORY) {
      std::vector<char> inside(net.n, 0);
      for (int m : seg.members) inside[m] = 1;
      for (int m : seg.members)
        for (int nx : net.next[m])
          if (!inside[nx]) {
            rp.spill[m] = 1;
            break;
          }
    }
  }
  return rp;
}

namespace {

// recompute._replay_phase_max (recompute.py:208-239).
int64_t replay_phase_max(const Net& net, const std::vector<Cost>& costs, int lid, const std::vector<int>& reads,
                         const std::vector<Segment>& segs, const std::vector<int>& seg_of) {
  const int own = seg_of[lid];
  std::vector<int> replayed, fetched;
  for (int r : reads) {
    if (own >= 0 && seg_of[r] == own) replayed.push_back(r);
    else fetched.push_back(r);
  }
  std::unordered_map<int, int64_t> alive;
  int64_t total = 0;
  for (int r : fetched) {
    if (!alive.count(r)) alive[r] = costs[r].device_bytes;
    // dict comprehension keeps one entry per key; reads are unique anyway
  }
  for (const auto& kv : alive) total = add_checked(total, kv.second);
  int64_t peak = total;
  if (replayed.empty()) return peak;
  const auto& members = segs[own].members;
  size_t depth = 0;
  for (int r : replayed) {
    const size_t idx = static_cast<size_t>(std::find(members.begin(), members.end(), r) - members.begin());
    depth = std::max(depth, idx);
  }
  std::unordered_map<int, int> last_need;
  for (size_t slot = 0; slot <= depth; ++slot)
    for (int pid : net.prev[members[slot]]) last_need[pid] = static_cast<int>(slot);
  std::vector<char> keep(net.n, 0);
  for (int r : reads) keep[r] = 1;
  for (size_t slot = 0; slot <= depth; ++slot) {
    const int mid = members[slot];
    for (int pid : net.prev[mid])
      if (!alive.count(pid)) {
        alive[pid] = costs[pid].device_bytes;
        total = add_checked(total, costs[pid].device_bytes);
      }
    alive[mid] = costs[mid].device_bytes;
    total = add_checked(total, costs[mid].device_bytes);
    peak = std::max(peak, total);
    for (auto it = alive.begin(); it != alive.end();) {
      const int tid = it->first;
      auto ln = last_need.find(tid);
      if (!keep[tid] && ln != last_need.end() && ln->second == static_cast<int>(slot)) {
        total -= it->second;
        it = alive.erase(it);
      } else {
        ++it;
      }
    }
  }
  return peak;
}

}  // namespace

std::vector<int64_t> step_demands(const Net& net, const std::vector<Cost>& costs, const Schedule& s) {
  const std::vector<Segment> segs = build_segments(net, s);
  std::vector<int> seg_of(net.n, -1);
  for (const Segment& seg : segs)
    for (int m : seg.members) seg_of[m] = seg.index;
  const std::vector<GradBuf> bufs = grad_buffers(net, costs, s, false);
  std::vector<int64_t> demands(s.num_steps(), 0);
  for (int lid : s.forward_ids) {
    int64_t total = costs[lid].device_bytes;
    for (int pid : net.prev[lid]) total = add_checked(total, costs[pid].device_bytes);
    demands[s.fwd_step_of[lid]] = total;
  }
  // Gradient bytes alive at each step via difference arrays.
  const int T = s.num_steps();
  std::vector<int64_t> d_all(T + 2, 0), d_pre(T + 2, 0);
  for (const GradBuf& b : bufs) {
    if (b.create_step > b.free_step) continue;  // never alive
    d_all[b.create_step] += b.nbytes;
    d_all[b.free_step + 1] -= b.nbytes;
    // create < step <= free
    d_pre[b.create_step + 1] += b.nbytes;
    d_pre[b.free_step + 1] -= b.nbytes;
  }
  std::vector<int64_t> bg_all(T, 0), bg_pre(T, 0);
  int64_t a = 0, p = 0;
  for (int t = 0; t < T; ++t) {
    a += d_all[t];
    p += d_pre[t];
    bg_all[t] = a;
    bg_pre[t] = p;
  }
  for (int lid : s.forward_ids) {
    const int step = s.bwd_step_of[lid];
    const std::vector<int> reads = net.backward_reads_unique(lid);
    int64_t compute_total = bg_all[step];
    for (int r : reads) compute_total = add_checked(compute_total, costs[r].device_bytes);
    const int64_t phase = replay_phase_max(net, costs, lid, reads, segs, seg_of);
    demands[step] = std::max(compute_total, add_checked(phase, bg_pre[step]));
  }
  return demands;
}

int64_t working_set_bytes(const Net& net, const std::vector<Cost>& costs, const Schedule& s,
                          const std::vector<GradBuf>& buffers, int step) {
  const int lid = s.layer_at(step);
  if (step < s.n) {
    int64_t total = costs[lid].device_bytes;
    for (int pid : net.prev[lid]) total += costs[pid].device_bytes;
    return total;
  }
  int64_t total = 0;
  for (int t : net.backward_reads_unique(lid)) total += costs[t].device_bytes;
  std::vector<int> buf_of(net.n, -1);
  for (size_t i = 0; i < buffers.size(); ++i) buf_of[buffers[i].owner] = static_cast<int>(i);
  std::vector<char> counted(net.n, 0);
  const int dy_owner = net.grad_owner(lid);
  if (dy_owner >= 0 && buf_of[dy_owner] >= 0) {
    const GradBuf& b = buffers[buf_of[dy_owner]];
    if (b.create_step <= step && step <= b.free_step) {
      total += b.nbytes;
      counted[dy_owner] = 1;
    }
  }
  for (int pid : net.prev[lid]) {
    const int owner = net.grad_owner(pid);
    if (owner < 0 || counted[owner] || buf_of[owner] < 0) continue;
    counted[owner] = 1;
    total += buffers[buf_of[owner]].nbytes;
  }
  return total;
}

int64_t liveness_peak(const Net& net, const std::vector<Cost>& costs, const Schedule& s, const Liveness& lv) {
  const int T = s.num_steps();
  std::vector<int64_t> d(T + 1, 0);
  for (int lid : s.forward_ids) {
    const int64_t nb = costs[lid].device_bytes;
    if (!nb) continue;
    d[s.fwd_step_of[lid]] += nb;
    d[lv.last_use[lid] + 1] -= nb;
  }
  for (const GradBuf& b : grad_buffers(net, costs, s, false)) {
    if (!b.nbytes || b.create_step > b.free_step) continue;
    d[b.create_step] += b.nbytes;
    d[b.free_step + 1] -= b.nbytes;
  }
  int64_t cur = 0, peak = 0;
  bool first = true;
  for (int t = 0; t < T; ++t) {
    cur += d[t];
    if (first || cur > peak) peak = cur;
    first = false;
  }
  return peak;
}

}  // namespace snp
