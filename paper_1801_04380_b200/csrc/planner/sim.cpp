// The iteration event loop.  Decision-for-decision restatement of memsched's
// _Simulation (simulator.py:191-731): scheduled-residency ledger, physical
// block pool with LRU eviction, FIFO transfer engine (float time model in the
// reference's operation order), recompute replays, conv workspace selection.
// Every physical action is also appended to the event tape replayed by the
// executor on the device arena.
#include "sim.hpp"

#include <algorithm>
#include <cstdio>
#include <unordered_map>

namespace snp {
namespace {

constexpr double kAlgoTime[3] = {1.0, 0.8, 0.6};  // implicit-gemm, gemm-workspace, fft
constexpr int64_t kAlgoWs[3] = {0, 1, 3};          // workspace factor x out_bytes
// sorted(ALGORITHMS, key=(time_factor, workspace_factor, name)): fft, gemm-workspace, implicit-gemm
constexpr int kAlgoSorted[3] = {2, 1, 0};

enum DropKind { DROP_DEAD = 0, DROP_BACKED = 1 };

struct TransferEngine {
  double bandwidth = 8e9, busy_until = 0.0, total_duration = 0.0;
  int64_t total_bytes = 0, count = 0;
  double submit(int64_t nbytes, double now) {
    const double duration = static_cast<double>(nbytes) / bandwidth;
    const double start = now > busy_until ? now : busy_until;  // max(busy_until, now)
    busy_until = start + duration;
    total_bytes += nbytes;
    total_duration += duration;
    count += 1;
    return busy_until;
  }
};

struct ReplayRow {
  int mid;
  double t;
  int64_t res;
  int64_t live;
};

class Sim {
 public:
  explicit Sim(Plan& p);
  void run();

 private:
  Plan& P;
  const Net& net;
  const Schedule& sched;
  const std::vector<Cost>& costs;
  const Features& F;
  int terminal;
  BlockPool pool;
  LruCache cache;
  TransferEngine engine;
  Liveness lv;
  std::vector<GradBuf> grad_windows;
  std::vector<int> grad_free_at;  // step -> index into grad_windows or -1
  bool have_off = false, have_plan = false;
  OffloadPlan off;
  RecomputePlan rp;
  std::vector<char> backed;
  std::vector<int> seg_of;
  std::vector<char> seg_replayed;

  OrderedKeys resident;
  std::unordered_map<int64_t, int64_t> res_bytes;
  int64_t res_total = 0, live_peak = 0, peak_count = 0, step_max = 0, step_count = 0;
  int peak_step = 0, current_step = 0;
  double clock = 0.0;
  std::vector<double> backup_done, arrival_done;
  double stall_prefetch = 0.0, stall_demand = 0.0, stall_backup = 0.0;
  int64_t scheduled_bytes = 0, scheduled_count = 0, demand_bytes = 0, demand_count = 0;
  int64_t cache_hits = 0, evictions = 0, extra_steps = 0, step_transfer = 0;
  double compute_total = 0.0;
  std::vector<std::vector<std::pair<int, int>>> drop_events;
  std::vector<int> pending_backed;
  std::vector<std::vector<int>> prefetch_at;

  void emit(char op, int a = 0, int b = 0, int64_t c = 0, int64_t d = 0, int e = 0) {
    Event ev;
    ev.op = op;
    ev.a = a;
    ev.b = b;
    ev.c = c;
    ev.d = d;
    ev.e = e;
    P.tape.push_back(ev);
  }
  bool is_res(int kind, int id) const { return resident.contains(key_code(kind, id)); }

  void build_static_events();
  void add_drop(int step, int kind, int lid) { drop_events[step].push_back({kind, lid}); }
  void bump();
  void track_add(int64_t key, int64_t nbytes);
  void track_remove(int64_t key);
  void pool_alloc(int64_t key, int64_t nbytes, bool high);
  void pool_free(int64_t key) {
    pool.free(key);
    emit('F', key_kind(key), static_cast<int>(key_id(key)));
  }
  bool materialize(int lid, int64_t nbytes);
  void drop_act(int lid, bool cacheable);
  void copy_out(int lid);
  void fetch_scheduled(int lid);
  void fetch_demand(int lid);
  void ensure_read(int lid, PySet& transient);
  void replay_member(int mid, std::vector<ReplayRow>& rows);
  void replay_prefix(const Segment& seg, size_t depth, const std::vector<char>& keep, PySet& transient,
                     std::vector<ReplayRow>& rows);
  void speed_replay(int seg_index, PySet& transient, std::vector<ReplayRow>& rows);
  void run_replay(int lid, const std::vector<int>& reads, PySet& transient, std::vector<ReplayRow>& rows);
  double forward_step(int s, int lid);
  double backward_step(int s, int lid, std::vector<ReplayRow>& rows);
  std::pair<double, int> select_workspace(int s, int lid, int phase, int* algo_out);
  void end_of_step(int s);
  void build_report();
  std::string where() const {
    return "step " + std::to_string(current_step) + " (" + net.names[sched.layer_at(current_step)] + ")";
  }
};

int64_t ceil_kib(int64_t n) { return ((n + 1023) / 1024) * 1024; }

std::string fmt_mib(int64_t nbytes) {
  char buf[64];
  std::snprintf(buf, sizeof buf, "%.3f", static_cast<double>(nbytes) / static_cast<double>(1 << 20));
  return buf;
}

Sim::Sim(Plan& p)
    : P(p), net(p.net), sched(p.sched), costs(p.costs), F(p.feats), terminal(-1),
      pool((p.pool_bytes >= 1 ? ceil_kib(p.pool_bytes) : p.pool_bytes)) {
  terminal = net.terminal_id();
  engine.bandwidth = p.cost_cfg.bandwidth;
  lv = build_liveness(net, sched);
  grad_windows = grad_buffers(net, costs, sched, !F.liveness);
  grad_free_at.assign(sched.num_steps() + 1, -1);
  for (size_t i = 0; i < grad_windows.size(); ++i) {
    const int fs = grad_windows[i].free_step;
    if (fs >= 0 && fs < sched.num_steps() && grad_free_at[fs] < 0) grad_free_at[fs] = static_cast<int>(i);
  }
  std::vector<char> offloaded(net.n, 0);
  if (F.offload) {
    off = build_offload_plan(net, sched, lv);
    have_off = true;
    for (int cp : off.cp_ids) offloaded[cp] = 1;
  }
  if (F.recompute != SN_RC_NONE) {
    rp = plan_recompute(net, costs, sched, lv, F.recompute, offloaded, P.min_pool);
    have_plan = true;
    P.modes = rp.modes;
  }
  backed = offloaded;
  seg_of.assign(net.n, -1);
  if (have_plan) {
    for (int i = 0; i < net.n; ++i)
      if (rp.spill[i]) backed[i] = 1;
    for (const Segment& seg : rp.segments)
      for (int m : seg.members) seg_of[m] = seg.index;
    seg_replayed.assign(rp.segments.size(), 0);
  }
  backup_done.assign(net.n, 0.0);
  arrival_done.assign(net.n, 0.0);
  drop_events.assign(sched.num_steps(), {});
  prefetch_at.assign(sched.num_steps(), {});
  P.pool_capacity_blocks = pool.capacity_blocks();
  build_static_events();
}

void Sim::build_static_events() {
  if (!F.liveness) return;
  for (int lid : sched.forward_ids) {
    if (costs[lid].device_bytes == 0) continue;
    if (F.recompute != SN_RC_NONE) {
      add_drop(lv.last_fwd_use[lid], backed[lid] ? DROP_BACKED : DROP_DEAD, lid);
    } else if (F.offload && have_off && off.drop_after[lid] >= 0) {
      add_drop(off.drop_after[lid], DROP_BACKED, lid);
      if (off.last_bwd_use[lid] >= 0) add_drop(off.last_bwd_use[lid], DROP_DEAD, lid);
    } else {
      add_drop(lv.last_use[lid], DROP_DEAD, lid);
    }
  }
  if (F.offload && F.recompute == SN_RC_NONE && !F.cache && have_off)
    for (int cp : off.cp_ids)
      if (off.prefetch_issue[cp] >= 0) prefetch_at[off.prefetch_issue[cp]].push_back(cp);
}

void Sim::bump() {
  if (res_total > step_max) {
    step_max = res_total;
    step_count = static_cast<int64_t>(resident.size());
  }
  if (res_total > live_peak) {
    live_peak = res_total;
    peak_step = current_step;
    peak_count = static_cast<int64_t>(resident.size());
  }
}

void Sim::track_add(int64_t key, int64_t nbytes) {
  if (!resident.insert(key)) fail(SN_EK_SCHED, "internal: " + key_repr(key) + " already resident");
  res_bytes[key] = nbytes;
  res_total += nbytes;
  bump();
}

void Sim::track_remove(int64_t key) {
  resident.erase(key);
  auto it = res_bytes.find(key);
  res_total -= it->second;
  res_bytes.erase(it);
}

void Sim::pool_alloc(int64_t key, int64_t nbytes, bool high) {
  while (true) {
    try {
      const int64_t off_blocks = pool.alloc(key, nbytes, high);
      emit('A', key_kind(key), static_cast<int>(key_id(key)), off_blocks, pool.span(key).second, high ? 1 : 0);
      return;
    } catch (const PlanError& exc) {
      if (exc.kind != SN_EK_POOLEXH) throw;
      if (!F.cache) fail(SN_EK_SCHED, "out of pool memory at " + where() + ": " + exc.what());
      int elid;
      try {
        elid = cache.evict_lru();
      } catch (const PlanError& e2) {
        if (e2.kind != SN_EK_ALLLOCKED) throw;
        fail(SN_EK_SCHED, "out of pool memory at " + where() + " with no cached tensor left to evict: " + exc.what());
      }
      emit('E', 0, elid);
      const double done = backup_done[elid];
      if (done > clock) {
        stall_backup += done - clock;
        clock = done;
      }
      pool_free(key_code(K_ACT, elid));
      evictions += 1;
    }
  }
}

bool Sim::materialize(int lid, int64_t nbytes) {
  const int64_t key = key_code(K_ACT, lid);
  if (cache.contains(lid)) {
    cache.discard(lid);
    emit('X', 0, lid);
    track_add(key, nbytes);
    cache_hits += 1;
    emit('H', 0, lid);
    return false;
  }
  if (pool.contains(key)) {
    auto it = std::find(pending_backed.begin(), pending_backed.end(), lid);
    if (it == pending_backed.end()) fail(SN_EK_INTERNAL, "list.remove(x): x not in list");
    pending_backed.erase(it);
    track_add(key, nbytes);
    emit('V', 0, lid);
    return false;
  }
  pool_alloc(key, nbytes, false);
  track_add(key, nbytes);
  return true;
}

void Sim::drop_act(int lid, bool cacheable) {
  const int64_t key = key_code(K_ACT, lid);
  if (resident.contains(key)) track_remove(key);
  if (!pool.contains(key)) return;
  if (cacheable && F.cache && backed[lid]) {
    emit(cache.contains(lid) ? 'T' : 'I', 0, lid);
    cache.insert(lid);
  } else {
    if (cache.discard(lid)) emit('X', 0, lid);
    pool_free(key);
  }
}

void Sim::copy_out(int lid) {
  emit('O', 0, lid);
  const int64_t nb = costs[lid].device_bytes;
  backup_done[lid] = engine.submit(nb, clock);
  scheduled_bytes += nb;
  scheduled_count += 1;
  step_transfer += nb;
}

void Sim::fetch_scheduled(int lid) {
  emit('P', 0, lid);
  const int64_t nb = costs[lid].device_bytes;
  arrival_done[lid] = engine.submit(nb, clock);
  scheduled_bytes += nb;
  scheduled_count += 1;
  step_transfer += nb;
}

void Sim::fetch_demand(int lid) {
  emit('D', 0, lid);
  const int64_t nb = costs[lid].device_bytes;
  const double done = engine.submit(nb, clock);
  stall_demand += done - clock;
  clock = done;
  demand_bytes += nb;
  demand_count += 1;
  step_transfer += nb;
}

void Sim::ensure_read(int lid, PySet& transient) {
  const int64_t nb = costs[lid].device_bytes;
  if (nb == 0 || is_res(K_ACT, lid)) return;
  if (!backed[lid])
    fail(SN_EK_SCHED, "tensor of layer " + net.reprs[lid] + " is needed at step " + std::to_string(current_step) +
                          " but is neither resident nor recoverable from a host backup");
  if (materialize(lid, nb)) fetch_demand(lid);
  if (F.recompute != SN_RC_NONE) transient.add(lid);
}

void Sim::replay_member(int mid, std::vector<ReplayRow>& rows) {
  if (materialize(mid, costs[mid].device_bytes)) {
    compute_total += costs[mid].fwd_time;
    clock += costs[mid].fwd_time;
    extra_steps += 1;
    rows.push_back({mid, costs[mid].fwd_time, res_total, static_cast<int64_t>(resident.size())});
    emit('R', 0, mid);
  }
}

void Sim::replay_prefix(const Segment& seg, size_t depth, const std::vector<char>& keep, PySet& transient,
                        std::vector<ReplayRow>& rows) {
  std::unordered_map<int, int> last_need;
  for (size_t slot = 0; slot <= depth; ++slot)
    for (int pid : net.prev[seg.members[slot]]) last_need[pid] = static_cast<int>(slot);
  for (size_t slot = 0; slot <= depth; ++slot) {
    const int mid = seg.members[slot];
    for (int pid : net.prev[mid])
      if (!is_res(K_ACT, pid)) ensure_read(pid, transient);
    if (!is_res(K_ACT, mid)) {
      replay_member(mid, rows);
      transient.add(mid);
    }
    for (int64_t tid : resident.snapshot()) {
      if (key_kind(tid) != K_ACT) continue;
      const int lid = static_cast<int>(key_id(tid));
      if (keep[lid]) continue;
      auto ln = last_need.find(lid);
      if (ln != last_need.end() && ln->second == static_cast<int>(slot) && transient.contains(lid))
        drop_act(lid, true);
    }
  }
}

void Sim::speed_replay(int seg_index, PySet& transient, std::vector<ReplayRow>& rows) {
  if (seg_replayed[seg_index]) return;
  seg_replayed[seg_index] = 1;
  PySet anchors_fetched;
  for (int mid : rp.segments[seg_index].members) {
    for (int pid : net.prev[mid])
      if (!is_res(K_ACT, pid)) ensure_read(pid, anchors_fetched);
    if (!is_res(K_ACT, mid)) replay_member(mid, rows);
    int use = lv.last_fwd_use[mid];
    for (int u : lv.bwd_uses[mid]) use = std::max(use, u);
    add_drop(std::max(use, current_step), DROP_DEAD, mid);
  }
  transient.update(anchors_fetched);
}

void Sim::run_replay(int lid, const std::vector<int>& reads, PySet& transient, std::vector<ReplayRow>& rows) {
  const int own = seg_of[lid];
  std::vector<int> same;
  for (int r : reads) {
    const int rseg = seg_of[r];
    if (rseg >= 0 && rseg == own)
      same.push_back(r);
    else if (rseg >= 0 && rp.modes[rseg] == SN_RC_SPEED)
      speed_replay(rseg, transient, rows);
    else
      ensure_read(r, transient);
  }
  if (same.empty()) return;
  if (rp.modes[own] == SN_RC_SPEED) {
    speed_replay(own, transient, rows);
    return;
  }
  const Segment& seg = rp.segments[own];
  size_t depth = 0;
  for (int r : same) {
    const size_t idx = static_cast<size_t>(std::find(seg.members.begin(), seg.members.end(), r) - seg.members.begin());
    depth = std::max(depth, idx);
  }
  std::vector<char> keep(net.n, 0);
  for (int r : reads) keep[r] = 1;
  replay_prefix(seg, depth, keep, transient, rows);
  for (int64_t tid : resident.snapshot()) {
    if (key_kind(tid) != K_ACT) continue;
    const int t = static_cast<int>(key_id(tid));
    if (transient.contains(t) && !keep[t]) drop_act(t, true);
  }
}

std::pair<double, int> Sim::select_workspace(int s, int lid, int phase, int* algo_out) {
  *algo_out = -1;
  if (!(F.convselect && net.kind[lid] == CONV)) return {1.0, -1};
  const int64_t out_bytes = costs[lid].out_bytes;
  const int64_t free_b = P.pool_bytes - res_total;
  const int64_t budget = free_b > 0 ? free_b : 0;
  // convselect.select_algorithm: fastest eligible; ties by (ws bytes, name).
  int first = -1;
  for (int a : {0, 1, 2}) {
    const int64_t ws = mul_checked(kAlgoWs[a], out_bytes);
    if (ws > budget) continue;
    if (first < 0) {
      first = a;
      continue;
    }
    const int64_t fws = mul_checked(kAlgoWs[first], out_bytes);
    static const char* names[3] = {"implicit-gemm", "gemm-workspace", "fft"};
    const bool better = kAlgoTime[a] < kAlgoTime[first] ||
                        (kAlgoTime[a] == kAlgoTime[first] &&
                         (ws < fws || (ws == fws && std::string(names[a]) < std::string(names[first]))));
    if (better) first = a;
  }
  if (first < 0) fail(SN_EK_INTERNAL, "min() arg is an empty sequence");
  int cands[3];
  int nc = 0;
  cands[nc++] = first;
  for (int a : kAlgoSorted)
    if (a != first) cands[nc++] = a;
  int algo = cands[nc - 1];
  int64_t ws = 0;
  int ws_key = -1;
  for (int i = 0; i < nc; ++i) {
    const int cand = cands[i];
    const int64_t nb = mul_checked(kAlgoWs[cand], out_bytes);
    if (nb == 0) {
      algo = cand;
      ws = 0;
      break;
    }
    try {
      pool_alloc(key_code(K_WS, s), nb, false);
    } catch (const PlanError& e) {
      if (e.kind == SN_EK_SCHED || e.kind == SN_EK_POOLEXH || e.kind == SN_EK_ALLLOCKED) continue;
      throw;
    }
    algo = cand;
    ws = nb;
    ws_key = s;
    break;
  }
  P.sels.push_back({static_cast<double>(s), lid, phase, algo, ws, free_b});
  *algo_out = algo;
  return {kAlgoTime[algo], ws_key};
}

double Sim::forward_step(int s, int lid) {
  if (net.kind[lid] == DATA) return 0.0;
  for (int pid : net.prev[lid])
    if (costs[pid].device_bytes && !is_res(K_ACT, pid))
      fail(SN_EK_SCHED, "forward input " + net.reprs[pid] + " missing at step " + std::to_string(s));
  const int64_t nb = costs[lid].device_bytes;
  if (nb) {
    pool_alloc(key_code(K_ACT, lid), nb, false);
    track_add(key_code(K_ACT, lid), nb);
  }
  int algo;
  const auto mw = select_workspace(s, lid, 0, &algo);
  emit('C', 0, lid, 0, mw.second, algo);
  const double elapsed = costs[lid].fwd_time * mw.first;
  compute_total += elapsed;
  clock += elapsed;
  if (mw.second >= 0) pool_free(key_code(K_WS, mw.second));
  if (backed[lid]) copy_out(lid);
  return elapsed;
}

double Sim::backward_step(int s, int lid, std::vector<ReplayRow>& rows) {
  if (net.kind[lid] == DATA) return 0.0;
  for (int cp : prefetch_at[s])
    if (!is_res(K_ACT, cp))
      if (materialize(cp, costs[cp].device_bytes)) fetch_scheduled(cp);
  const std::vector<int> reads = net.backward_reads_unique(lid);
  PySet transient;
  if (F.recompute != SN_RC_NONE)
    run_replay(lid, reads, transient, rows);
  else
    for (int r : reads) ensure_read(r, transient);
  for (int r : reads) {
    const double done = arrival_done[r];
    if (done > clock) {
      stall_prefetch += done - clock;
      clock = done;
    }
  }
  const int dy_owner = net.grad_owner(lid);
  if (lid == terminal) {
    if (!F.liveness && dy_owner >= 0 && !is_res(K_GRAD, dy_owner)) {
      pool_alloc(key_code(K_GRAD, dy_owner), costs[dy_owner].grad_bytes, true);
      track_add(key_code(K_GRAD, dy_owner), costs[dy_owner].grad_bytes);
    }
  } else if (dy_owner >= 0 && !is_res(K_GRAD, dy_owner)) {
    fail(SN_EK_SCHED, "gradient buffer of " + net.reprs[dy_owner] + " missing at step " + std::to_string(s));
  }
  for (int pid : net.prev[lid]) {
    const int owner = net.grad_owner(pid);
    if (owner < 0) continue;
    if (!is_res(K_GRAD, owner)) {
      pool_alloc(key_code(K_GRAD, owner), costs[owner].grad_bytes, true);
      track_add(key_code(K_GRAD, owner), costs[owner].grad_bytes);
    }
  }
  int algo;
  const auto mw = select_workspace(s, lid, 1, &algo);
  emit('B', 0, lid, 0, mw.second, algo);
  const double elapsed = costs[lid].bwd_time * mw.first;
  compute_total += elapsed;
  clock += elapsed;
  if (mw.second >= 0) pool_free(key_code(K_WS, mw.second));
  if (F.recompute != SN_RC_NONE)
    for (int64_t t : transient.items())
      if (is_res(K_ACT, static_cast<int>(t))) drop_act(static_cast<int>(t), true);
  return elapsed;
}

void Sim::end_of_step(int s) {
  if (F.liveness) {
    const int gi = grad_free_at[s];
    if (gi >= 0) {
      const int64_t key = key_code(K_GRAD, grad_windows[gi].owner);
      if (resident.contains(key)) {
        track_remove(key);
        pool_free(key);
      }
    }
  }
  std::vector<int> still;
  const std::vector<int> pend = pending_backed;
  for (int lid : pend) {
    if (backup_done[lid] <= clock)
      drop_act(lid, true);
    else
      still.push_back(lid);
  }
  pending_backed = still;
  for (size_t i = 0; i < drop_events[s].size(); ++i) {
    const int kind = drop_events[s][i].first, lid = drop_events[s][i].second;
    if (kind == DROP_DEAD) {
      drop_act(lid, false);
    } else if (backup_done[lid] <= clock) {
      drop_act(lid, true);
    } else {
      if (is_res(K_ACT, lid)) track_remove(key_code(K_ACT, lid));
      pending_backed.push_back(lid);
    }
  }
  emit('S', 0, s);
}

void Sim::run() {
  std::vector<ReplayRow> replay_rows;
  for (int step = 0; step < sched.num_steps(); ++step) {
    current_step = step;
    step_max = res_total;
    step_count = static_cast<int64_t>(resident.size());
    step_transfer = 0;
    double step_compute = 0.0;
    const double stall_before = stall_prefetch + stall_demand + stall_backup;
    const int lid = sched.layer_at(step);
    const bool fwd = sched.is_forward(step);
    replay_rows.clear();
    if (fwd)
      step_compute += forward_step(step, lid);
    else
      step_compute += backward_step(step, lid, replay_rows);
    end_of_step(step);
    const double stall_here = (stall_prefetch + stall_demand + stall_backup) - stall_before;
    const size_t k = replay_rows.size();
    for (size_t j = 0; j < k; ++j) {
      const ReplayRow& r = replay_rows[j];
      const double index = static_cast<double>(step - 1) + static_cast<double>(j + 1) / static_cast<double>(k + 1);
      P.rows.push_back({index, r.mid, 2, r.res, r.live, pool.used_bytes(), r.t, 0.0, 0});
    }
    P.rows.push_back({static_cast<double>(step), lid, fwd ? 0 : 1, step_max, step_count, pool.used_bytes(),
                      step_compute, stall_here, step_transfer});
  }
  pool.check();
  std::stable_sort(P.rows.begin(), P.rows.end(), [](const Row& a, const Row& b) { return a.index < b.index; });
  build_report();
}

void Sim::build_report() {
  sn_report& r = P.report;
  const std::vector<GradBuf> bufs = grad_buffers(net, costs, sched, !F.liveness);
  int64_t working = working_set_bytes(net, costs, sched, bufs, peak_step);
  working = std::min(working, live_peak);
  const double total = clock >= engine.busy_until ? clock : engine.busy_until;  // max(clock, busy_until)
  const double stall = stall_prefetch + stall_demand + stall_backup;
  int64_t base = 0;
  for (const Cost& c : costs) base = add_checked(base, c.device_bytes);
  for (const Cost& c : costs) base = add_checked(base, c.grad_bytes);
  r.num_layers = net.n;
  r.num_steps = sched.num_steps();
  r.peak_bytes = live_peak;
  r.peak_step = peak_step;
  r.peak_layer = sched.layer_at(peak_step);
  r.peak_live_count = peak_count;
  r.peak_working_bytes = working;
  r.peak_stash_bytes = live_peak - working;
  r.min_pool_bytes = P.min_pool;
  r.baseline_peak_bytes = base;
  r.liveness_peak_bytes = liveness_peak(net, costs, sched, lv);
  r.compute_s = compute_total;
  r.stall_s = stall;
  r.stall_prefetch_s = stall_prefetch;
  r.stall_demand_s = stall_demand;
  r.stall_backup_s = stall_backup;
  r.transfer_busy_s = engine.total_duration;
  r.total_s = total;
  r.scheduled_transfer_bytes = scheduled_bytes;
  r.scheduled_transfer_count = scheduled_count;
  r.demand_transfer_bytes = demand_bytes;
  r.demand_transfer_count = demand_count;
  r.cache_hits = cache_hits;
  r.evictions = evictions;
  r.extra_forward_steps = extra_steps;
  r.planned_extra_forward_steps = have_plan ? rp.extra_forward_steps : 0;
  r.pool_high_water_bytes = pool.high_water_bytes();
  r.n_rows = static_cast<int32_t>(P.rows.size());
  r.n_selections = static_cast<int32_t>(P.sels.size());
  r.n_modes = static_cast<int32_t>(P.modes.size());
}

}  // namespace

void analyze_plan(Plan& p) {
  p.sched = build_schedule(p.net);
  p.costs = build_costs(p.net, p.cost_cfg);
  p.demands = step_demands(p.net, p.costs, p.sched);
  p.min_pool = p.demands.empty() ? 0 : *std::max_element(p.demands.begin(), p.demands.end());
}

void costs_only(Plan& p) { p.costs = build_costs(p.net, p.cost_cfg); }

void run_plan(Plan& p) {
  analyze_plan(p);
  if (p.pool_bytes < p.min_pool)
    fail(SN_EK_CONFIG, "pool of " + std::to_string(p.pool_bytes) + " bytes is below the minimum schedulable demand of " +
                           std::to_string(p.min_pool) + " bytes (" + fmt_mib(p.min_pool) + " MiB)");
  Sim sim(p);
  sim.run();
  p.tape_c.resize(p.tape.size());
  for (size_t i = 0; i < p.tape.size(); ++i) {
    sn_event& e = p.tape_c[i];
    e = sn_event{};
    e.op = p.tape[i].op;
    e.a = p.tape[i].a;
    e.b = p.tape[i].b;
    e.c = p.tape[i].c;
    e.d = p.tape[i].d;
    e.e = p.tape[i].e;
  }
}

}  // namespace snp
