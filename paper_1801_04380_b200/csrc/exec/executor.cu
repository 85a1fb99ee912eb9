// The B200 executor: replays a plan's event tape on one device.
//
//  * One cudaMalloc'd arena of the planner's pool capacity; a tensor lives at
//    base + block_offset * 1024 exactly where the planner's BlockPool put it.
//    The executor itself never allocates during a step.
//  * Three streams: compute (S0), copy-out D2H (S1), fetch H2D (S2).  Copies
//    are ordered against compute with events derived statically from the tape:
//      - a copy-out waits for its producer; a freed region whose copy-out may
//        still be reading it is not rewritten before that copy completes;
//      - a fetch waits for every earlier compute on the stream (previous
//        occupants' readers) and for the tensor's own copy-out; the first
//        kernel that reads a fetched tensor waits for the fetch.
//  * The whole iteration (all three streams) is captured once into a CUDA
//    graph, legal because the tape is iteration-invariant.
//  * Gradient buffers follow the planner's windows; the first write into a
//    freshly allocated buffer overwrites, later writes accumulate.
//  * Optional plan-driven backup elision: a copy-out whose tensor the tape
//    never fetches back is not issued (residency/offsets are unchanged).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <string>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "../kernels/kernels.hpp"
#include "../planner/handle.hpp"
#include "nccl_dl.hpp"
#include "superneurons.h"

namespace {

using snp::Net;
thread_local std::string g_xerr;
thread_local int g_xerr_kind = SN_EK_NONE;

struct ExecError {
  int kind;
  std::string msg;
};
[[noreturn]] void xfail(int kind, const std::string& msg) { throw ExecError{kind, msg}; }
void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) xfail(SN_EK_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

int xset(int kind, const std::string& msg) {
  g_xerr = msg;
  g_xerr_kind = kind;
  return kind == SN_EK_CUDA ? SN_ERR_CUDA : SN_ERR_OTHER;
}

constexpr int64_t kAlignFloats = 64;  // 256 B parameter slice alignment
int64_t align_up(int64_t v, int64_t a) { return (v + a - 1) / a * a; }

struct LayerRt {
  int kind = 0;
  int C = 1, H = 1, W = 1;   // output per sample (stored channels for DATA)
  int C_raw = 1;             // channels before the DATA padding
  int64_t per_sample = 0;    // output elements per sample (stored)
  int64_t w_off = -1, w_n = 0, b_off = -1, b_n = 0;
  int64_t state_off = -1;    // BN: stats[2C] then running[2C]
  sn_layer_numerics num{};
  sn::ConvShape conv{};
  sn::PoolShape pool{};
  int fc_in = 0, fc_splits = 1, wgrad_splits = 1;
  // CONV kernel variants (forward, dgrad, wgrad): the process defaults, or the
  // fastest measured one when the executor benchmarks them (opt.autotune)
  sn::ConvKnobs kf{}, kd{}, kw{};
  int stats_tiles = 0, stats_rows = 0;  // CONV: BN statistics tiles its forward can emit
  uint8_t* argmax = nullptr;            // max POOL: per-output window argmax saved by the forward
  float* wt_pre = nullptr;              // CONV: its dgrad weights, transformed once per step (prep_dgrad_weights)
};

struct Action {
  std::function<void()> fn;
  int kernels = 0;
  int layer = -1;
  int type = 3;  // 0 forward, 1 replay, 2 backward, 3 copy / sync / other
};

}  // namespace

struct sn_exec {
  const sn_plan* plan = nullptr;
  const Net* net = nullptr;
  int B = 0;
  int device = 0;
  sn_exec_options opt{};
  std::vector<LayerRt> L;
  int terminal = -1;
  // device memory
  char* arena = nullptr;
  int64_t arena_bytes = 0;
  float* params = nullptr;
  float* grads = nullptr;
  int64_t n_params = 0;
  float* state = nullptr;
  int64_t n_state = 0;
  float* images = nullptr;    // user-facing input batch, NHWC with the net's own channel count
  int64_t image_floats = 0;
  float* data_buf = nullptr;  // the DATA activation as the consumers read it (== images unless padded)
  int data_id = -1;
  int stem_layer = -1;        // CONV reading a spatially padded C=4 copy of the images (TMA stem path)
  std::vector<char> elided;   // per layer: output fused away (never written)
  std::vector<int> eff_owner;  // per layer: the buffer holding its output gradient (see setup_layers)
  std::vector<char> side_root;
  std::unordered_map<int, float*> side;  // side root -> its output-gradient buffer (outside the pool)
  int32_t* labels = nullptr;
  float* loss_rows = nullptr;
  float* loss = nullptr;
  uint32_t* iteration = nullptr;
  float* wt_scratch = nullptr;
  sn::DgradPrepJob* prep_jobs = nullptr;  // the batched dgrad weight transforms (device table)
  float* partial = nullptr;
  int64_t partial_cap = 0;
  float* red = nullptr;
  float* tstats = nullptr;  // per-tile BN statistics from a CONV forward to the BN right after it
  void* pool_scratch = nullptr;
  const float** ptr_table = nullptr;
  std::vector<const float*> ptr_host;
  // host stash
  std::unordered_map<int, char*> stash;
  // streams / events
  cudaStream_t s0 = nullptr, s1 = nullptr, s2 = nullptr;
  // s3: weight gradients (off the backward critical path) run on a side
  // stream, overlapping the next layers' backward; their own scratch buffers
  cudaStream_t s3 = nullptr;
  int wgrad_ws_in_pool = 0, wgrad_ws_outside = 0;  // CONV weight gradients: partials in the granted workspace or not
  float* partial_w = nullptr;
  float* red_w = nullptr;
  float* wt_w = nullptr;
  std::vector<cudaEvent_t> events;
  cudaEvent_t t_begin = nullptr, t_end = nullptr;
  // pipelined host input (sn_exec_step_host_pipelined, sn_exec_train_host):
  // the next batch's images are copied host -> device on s4 straight into
  // `images` once the running iteration has consumed them (inputs_free_ev,
  // recorded inside the iteration right after the DATA layer laid them out,
  // or at its end when consumers read `images` in place); its labels (read by
  // the loss) go to a staging buffer copied on s0 right before the iteration
  cudaStream_t s4 = nullptr;
  int32_t* labels_stage = nullptr;
  cudaEvent_t staged_ev = nullptr, consumed_ev = nullptr, inputs_free_ev = nullptr;
  const void* staged_src = nullptr;
  float* loss_pinned = nullptr;  // [2] loss slots of consecutive steps (sn_exec_train_host)
  cudaEvent_t loss_ev[2] = {nullptr, nullptr};
  // compiled program
  std::vector<Action> prog;
  int64_t kernels_per_step = 0;
  int64_t d2h_bytes = 0, h2d_bytes = 0;
  std::unordered_map<int64_t, std::pair<int64_t, int64_t>> final_keys;  // key -> (off, blocks) at tape end
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t gexec = nullptr;
  bool graph_ready = false;
  // profiling (sn_exec_profile / sn_exec_census): run the side-stream weight
  // gradients on the compute stream, so per-action events on s0 bracket all of
  // an action's kernels and nothing overlaps
  bool serial = false;
  int32_t* marker = nullptr;  // census: per-action memset marker target
  // measured CONV kernel-variant catalog (opt.autotune): every variant timed per
  // layer shape and op, the fastest applied
  struct CatEntry {
    int layer, op;  // representative layer of the shape; 0 fwd, 1 dgrad, 2 wgrad
    sn::ConvKnobs k;
    float us;
    int chosen;
  };
  std::vector<CatEntry> catalog;
  // data-parallel replica: buckets of the weight-gradient all-reduce, issued on
  // s5 after the backward steps of their layers
  struct Bucket {
    int64_t lo = 0, hi = 0;  // floats of the flat gradient block
    int after_layer = -1;    // issued right after this layer's backward action
    std::vector<int> layers;
  };
  std::vector<Bucket> buckets;
  cudaStream_t s5 = nullptr;
  int32_t* update_flag = nullptr;
  bool dp() const { return opt.dp_comm != nullptr; }
  // device / pinned bytes by category (sn_exec_memory)
  enum { M_ARENA, M_PARAMS, M_STATE, M_INPUT, M_WGRAD, M_OTHER, M_STASH, M_HOST, M_PEER, M_N };
  std::vector<std::pair<char*, int>> peer_stash;  // device stash allocations (pointer, device)
  int64_t mem[M_N] = {};
  int64_t wgrad_partial_outside = 0;  // floats of split-K scratch the plan's workspaces could not hold
  template <class T>
  void dmalloc(T** p, int64_t bytes, int cat, const char* what) {
    ck(cudaMalloc(reinterpret_cast<void**>(p), static_cast<size_t>(bytes)), what);
    mem[cat] += bytes;
  }

  cudaEvent_t new_event() {
    cudaEvent_t e;
    ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
    events.push_back(e);
    return e;
  }
  // Transfer evidence (sn_exec_transfer_stats): timing events around every
  // issued copy on its copy stream, and around every compute-stream wait for
  // a fetch (the exposed, non-overlapped part of a transfer).
  struct Timer {
    cudaEvent_t a, b;
    int64_t bytes;
    int kind;  // 0 D2H copy-out, 1 H2D fetch, 2 compute stream blocked on a fetch
  };
  std::vector<Timer> timers;
  Timer& new_timer(int kind, int64_t bytes) {
    Timer t{nullptr, nullptr, bytes, kind};
    ck(cudaEventCreate(&t.a), "cudaEventCreate");
    ck(cudaEventCreate(&t.b), "cudaEventCreate");
    events.push_back(t.a);
    events.push_back(t.b);
    timers.push_back(t);
    return timers.back();
  }
};

namespace {

int64_t key_code(int kind, int64_t id) { return snp::key_code(kind, id); }

// A timing event readable after the step: inside a graph capture the record
// must be an external node (an internal one only orders the graph)
cudaError_t record_timer(cudaEvent_t e, cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaError_t err = cudaStreamIsCapturing(st, &cs);
  if (err != cudaSuccess) return err;
  return cs == cudaStreamCaptureStatusActive ? cudaEventRecordWithFlags(e, st, cudaEventRecordExternal)
                                             : cudaEventRecord(e, st);
}

void setup_layers(sn_exec* ex, const sn_layer_numerics* numerics) {
  const snp::Plan& P = ex->plan->plan;
  const Net& net = P.net;
  const int n = net.n;
  ex->L.assign(n, LayerRt{});
  ex->terminal = net.terminal_id();
  if (net.kind[ex->terminal] != snp::SOFTMAX)
    xfail(SN_EK_UNSUPPORTED, "numeric execution needs a SOFTMAX terminal (cross-entropy loss)");
  // DATA is stored with channels padded to 4 when only CONVs read it, so the
  // stem convolution keeps 16-byte aligned cp.async gathers.
  int64_t poff = 0, soff = 0;
  for (int i = 0; i < n; ++i) {
    LayerRt& l = ex->L[i];
    l.kind = net.kind[i];
    if (numerics) l.num = numerics[i];
    const auto& shp = P.costs[i].shape;
    if (shp.size() == 3) {
      l.C = static_cast<int>(shp[0]);
      l.H = static_cast<int>(shp[1]);
      l.W = static_cast<int>(shp[2]);
    } else {
      l.C = static_cast<int>(shp[0]);
      l.H = l.W = 1;
    }
    l.C_raw = l.C;
    if (l.kind == snp::DATA) ex->data_id = i;
    if (l.kind == snp::DATA && l.C % 4 != 0) {
      bool only_conv = true;
      for (int nx : net.next[i]) only_conv &= net.kind[nx] == snp::CONV;
      if (only_conv) l.C = (l.C + 3) / 4 * 4;
    }
    l.per_sample = static_cast<int64_t>(l.C) * l.H * l.W;
    if (static_cast<int64_t>(ex->B) * l.per_sample >= (1ll << 31))
      xfail(SN_EK_UNSUPPORTED, "tensor of layer '" + net.names[i] + "' exceeds 2^31 elements");
  }
  // Gradient buffers.  The reference aliases an ACT / DROPOUT gradient with
  // its producer's (GRAD_INPLACE_KINDS, costmodel.py:207-221).  When that
  // producer forks, its other consumers' gradients would mix with the in-place
  // layer's own incoming gradient in the one buffer; the first in-place layer
  // after such a fork (a "side root") gets its own output-gradient buffer
  // outside the pool, and its backward adds its masked gradient into the
  // producer's.  eff_owner[i]: the buffer holding d(output of i) -- a pool
  // gradient key, a side root's id, or -1 (no gradient).
  ex->eff_owner.assign(n, -2);
  ex->side_root.assign(n, 0);
  std::function<int(int)> eo = [&](int i) -> int {
    if (ex->eff_owner[i] != -2) return ex->eff_owner[i];
    int r;
    if (snp::is_inplace(net.kind[i])) {
      const int p = net.prev[i][0];
      if (net.next[p].size() != 1 && net.grad_owner(p) >= 0) {
        ex->side_root[i] = 1;
        r = i;
      } else {
        r = eo(p);
      }
    } else {
      r = net.grad_owner(i);
    }
    return ex->eff_owner[i] = r;
  };
  for (int i = 0; i < n; ++i) eo(i);
  for (int i = 0; i < n; ++i) {
    LayerRt& l = ex->L[i];
    const int k = l.kind;
    if (k == snp::SOFTMAX && i != ex->terminal)
      xfail(SN_EK_UNSUPPORTED, "SOFTMAX is only supported as the terminal layer");
    if (k == snp::CONV || k == snp::POOL) {
      const LayerRt& in = ex->L[net.prev[i][0]];
      const int K = static_cast<int>(net.pint[i][SN_P_K]);
      const int s = net.pstate[i][SN_P_S] == 1 ? static_cast<int>(net.pint[i][SN_P_S]) : (k == snp::CONV ? 1 : K);
      const int pd = net.pstate[i][SN_P_P] == 1 ? static_cast<int>(net.pint[i][SN_P_P]) : 0;
      if (s < 1 || pd < 0) xfail(SN_EK_UNSUPPORTED, "non-positive stride / negative pad in '" + net.names[i] + "'");
      if (k == snp::CONV) {
        l.conv = sn::ConvShape{ex->B, in.H, in.W, in.C, l.C, K, K, l.H, l.W, s, pd};
        l.w_off = poff;
        l.w_n = static_cast<int64_t>(l.C) * K * K * in.C;
        poff = align_up(poff + l.w_n, kAlignFloats);
        l.b_off = poff;
        l.b_n = l.C;
        poff = align_up(poff + l.b_n, kAlignFloats);
      } else {
        l.pool = sn::PoolShape{ex->B, in.H, in.W, in.C, l.H, l.W, K, s, pd, l.num.pool_mode};
      }
    } else if (k == snp::FC) {
      const LayerRt& in = ex->L[net.prev[i][0]];
      l.fc_in = static_cast<int>(in.per_sample);
      l.w_off = poff;
      l.w_n = static_cast<int64_t>(l.C) * l.fc_in;
      poff = align_up(poff + l.w_n, kAlignFloats);
      l.b_off = poff;
      l.b_n = l.C;
      poff = align_up(poff + l.b_n, kAlignFloats);
    } else if (k == snp::BN) {
      l.w_off = poff;  // gamma
      l.w_n = l.C;
      poff = align_up(poff + l.w_n, kAlignFloats);
      l.b_off = poff;  // beta
      l.b_n = l.C;
      poff = align_up(poff + l.b_n, kAlignFloats);
      l.state_off = soff;
      soff = align_up(soff + 4 * static_cast<int64_t>(l.C), kAlignFloats);
    }
  }
  ex->n_params = std::max<int64_t>(poff, kAlignFloats);
  ex->n_state = std::max<int64_t>(soff, kAlignFloats);
  const sn::ConvKnobs defaults = sn::conv_knobs();
  for (LayerRt& l : ex->L) l.kf = l.kd = l.kw = defaults;
  // A lone CONV on a 4-channel DATA layer reads a spatially padded copy of the
  // images through the sliding-window TMA stem kernels (conv_tma.cu).
  if (ex->data_id >= 0 && net.next[ex->data_id].size() == 1) {
    const int c = net.next[ex->data_id][0];
    if (ex->L[c].kind == snp::CONV && ex->L[ex->data_id].C == 4 && sn::use_tma() && sn::conv_stem_ok(ex->L[c].conv))
      ex->stem_layer = c;
  }
}

// Measured kernel-variant catalog (the reference's convselect benchmarks the
// memory-feasible algorithms; here the algorithms are this
// executor's kernel variants): for every distinct CONV shape and op, time each
// variant of the dispatch knobs on scratch buffers (1 warm-up + median of 3,
// CUDA events) and give the layers of that shape the fastest.  Weight-gradient
// variants whose split-K partials exceed the 64 Mi-float scratch cap are not
// memory-feasible and are skipped.  Summation orders differ between
// variants, so this is a non-parity mode (off by default).
void autotune(sn_exec* ex) {
  const Net& net = ex->plan->plan.net;
  std::map<std::vector<int>, std::vector<int>> shapes;  // shape key -> CONV layers
  for (int i = 0; i < net.n; ++i) {
    const LayerRt& l = ex->L[i];
    if (l.kind != snp::CONV || i == ex->stem_layer) continue;
    const sn::ConvShape& c = l.conv;
    const bool dgrad = net.kind[net.prev[i][0]] != snp::DATA;
    shapes[{c.N, c.H, c.W, c.C, c.K, c.R, c.S, c.P, c.Q, c.stride, c.pad, dgrad ? 1 : 0}].push_back(i);
  }
  if (shapes.empty()) return;
  int64_t nx = 64, nw = 64, ny = 64, nwt = 64, nred = 64;
  const int64_t cap = 64ll << 20;
  for (const auto& kv : shapes) {
    const sn::ConvShape& c = ex->L[kv.second[0]].conv;
    nx = std::max<int64_t>(nx, static_cast<int64_t>(c.N) * c.H * c.W * c.C);
    ny = std::max<int64_t>(ny, static_cast<int64_t>(c.N) * c.P * c.Q * c.K);
    nw = std::max<int64_t>(nw, static_cast<int64_t>(c.K) * c.R * c.S * c.C);
    nwt = std::max<int64_t>(nwt, std::max<int64_t>(nw, sn::conv_dgrad_scratch_floats(c)));
    nred = std::max<int64_t>(nred, sn::red_scratch_floats(std::max(c.C, c.K)));
  }
  std::vector<void*> bufs;
  auto dal = [&](int64_t floats) {
    void* p = nullptr;
    ck(cudaMalloc(&p, static_cast<size_t>(floats) * 4), "cudaMalloc(autotune)");
    ck(cudaMemset(p, 0, static_cast<size_t>(floats) * 4), "memset(autotune)");
    bufs.push_back(p);
    return static_cast<float*>(p);
  };
  struct Free {
    std::vector<void*>* b;
    ~Free() {
      for (void* p : *b) cudaFree(p);
    }
  } free_bufs{&bufs};
  float *x = dal(nx), *y = dal(ny), *dy = dal(ny), *dx = dal(nx), *w = dal(nw), *bias = dal(4096), *dw = dal(nw);
  float *wt = dal(nwt), *red = dal(nred), *part = dal(cap);
  cudaEvent_t e0, e1;
  ck(cudaEventCreate(&e0), "event");
  ck(cudaEventCreate(&e1), "event");
  cudaStream_t st = ex->s0;
  auto time_us = [&](const std::function<cudaError_t()>& f) -> float {
    ck(f(), "autotune warm-up");
    float t[3];
    for (int r = 0; r < 3; ++r) {
      ck(cudaEventRecord(e0, st), "record");
      ck(f(), "autotune launch");
      ck(cudaEventRecord(e1, st), "record");
      ck(cudaEventSynchronize(e1), "sync");
      ck(cudaEventElapsedTime(&t[r], e0, e1), "elapsed");
    }
    std::sort(t, t + 3);
    return t[1] * 1000.f;
  };
  const sn::ConvKnobs base = sn::conv_knobs();
  auto with = [&](int halo, int pairs, int bn, int subpix) {
    sn::ConvKnobs k = base;
    if (halo >= 0) k.halo = halo;
    if (pairs >= 0) k.pairs = pairs;
    if (bn >= 0) k.bn = bn;
    if (subpix >= 0) k.subpix = subpix;
    return k;
  };
  const std::vector<sn::ConvKnobs> fwd_v = {base, with(0, -1, -1, -1), with(-1, 0, -1, -1), with(0, 0, -1, -1),
                                           with(0, -1, 128, -1), with(0, -1, 64, -1)};
  const std::vector<sn::ConvKnobs> dgrad_v = {base, with(0, -1, -1, -1), with(-1, 0, -1, -1), with(-1, -1, -1, 0),
                                             with(0, 0, -1, -1)};
  const std::vector<sn::ConvKnobs> wgrad_v = {base, with(0, -1, -1, -1), with(-1, 0, -1, -1), with(0, 0, -1, -1)};
  for (const auto& kv : shapes) {
    const int rep = kv.second[0];
    const sn::ConvShape cs = ex->L[rep].conv;
    const bool has_dgrad = kv.first.back() != 0;
    for (int op = 0; op < 3; ++op) {
      if (op == 1 && !has_dgrad) continue;
      const auto& vs = op == 0 ? fwd_v : (op == 1 ? dgrad_v : wgrad_v);
      float best = 0.f;
      sn::ConvKnobs pick = base;
      const size_t first = ex->catalog.size();
      std::vector<sn::ConvKnobs> seen;
      for (const sn::ConvKnobs& k : vs) {
        if (std::find(seen.begin(), seen.end(), k) != seen.end()) continue;
        seen.push_back(k);
        sn::KnobScope ks(k);
        float us = 0.f;
        if (op == 0) {
          us = time_us([&] { return sn::conv_fwd(cs, x, w, bias, y, st, nullptr); });
        } else if (op == 1) {
          if (sn::conv_dgrad_scratch_floats(cs) > nwt) continue;
          us = time_us([&] { return sn::conv_dgrad(cs, dy, w, wt, dx, 0, st); });
        } else {
          const int sp = sn::conv_wgrad_splits(cs, cap);
          if (static_cast<int64_t>(sp) * cs.R * cs.S * cs.C * cs.K > cap) continue;  // not memory-feasible
          us = time_us([&] { return sn::conv_wgrad(cs, x, dy, dw, nullptr, part, sp, red, st); });
        }
        ex->catalog.push_back({rep, op, k, us, 0});
        if (ex->catalog.size() == first + 1 || us < best) {
          best = us;
          pick = k;
        }
      }
      for (size_t j = first; j < ex->catalog.size(); ++j) ex->catalog[j].chosen = ex->catalog[j].k == pick;
      for (int lid : kv.second) (op == 0 ? ex->L[lid].kf : (op == 1 ? ex->L[lid].kd : ex->L[lid].kw)) = pick;
    }
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  ck(cudaDeviceSynchronize(), "autotune");
}

// Buckets in backward (issue) order: a bucket is a contiguous float range of
// the parameter block holding whole layers; it grows with each parameter
// layer whose backward step completes, as long as the range it would span
// holds no layer still waiting for its backward step or already in a closed
// bucket, and up to `cap_bytes`.
void plan_buckets(sn_exec* ex, int64_t cap_bytes) {
  const snp::Plan& P = ex->plan->plan;
  const Net& net = P.net;
  struct Iv {
    int64_t lo, hi;
    int lid;
  };
  std::vector<Iv> ivs;
  for (int i = 0; i < net.n; ++i) {
    const LayerRt& l = ex->L[i];
    if (l.w_off < 0) continue;
    ivs.push_back({std::min(l.w_off, l.b_off), std::max(l.w_off + l.w_n, l.b_off + l.b_n), i});
  }
  std::sort(ivs.begin(), ivs.end(), [](const Iv& a, const Iv& b) { return a.lo < b.lo; });
  std::vector<int> state(net.n, 0);  // 0 pending, 1 in the open bucket, 2 in a closed bucket
  ex->buckets.clear();
  sn_exec::Bucket cur;
  auto close = [&] {
    if (cur.layers.empty()) return;
    for (int l : cur.layers) state[l] = 2;
    ex->buckets.push_back(cur);
    cur = sn_exec::Bucket{};
  };
  auto fits = [&](int64_t lo, int64_t hi) {
    for (const Iv& v : ivs)
      if (v.lo < hi && lo < v.hi && state[v.lid] != 1) return false;
    return true;
  };
  std::vector<char> seen(net.n, 0);
  for (const auto& ev : P.tape) {
    if (ev.op != 'B' || ex->L[ev.b].w_off < 0 || seen[ev.b]) continue;
    seen[ev.b] = 1;
    const LayerRt& l = ex->L[ev.b];
    const int64_t lo = std::min(l.w_off, l.b_off), hi = std::max(l.w_off + l.w_n, l.b_off + l.b_n);
    state[ev.b] = 1;
    if (!cur.layers.empty()) {
      const int64_t nlo = std::min(cur.lo, lo), nhi = std::max(cur.hi, hi);
      if ((nhi - nlo) * 4 > cap_bytes || !fits(nlo, nhi)) {
        state[ev.b] = 0;
        close();
        state[ev.b] = 1;
      }
    }
    if (cur.layers.empty()) {
      cur.lo = lo;
      cur.hi = hi;
    } else {
      cur.lo = std::min(cur.lo, lo);
      cur.hi = std::max(cur.hi, hi);
    }
    cur.layers.push_back(ev.b);
    cur.after_layer = ev.b;
  }
  close();
}

void alloc_device(sn_exec* ex) {
  const snp::Plan& P = ex->plan->plan;
  const Net& net = P.net;
  ex->arena_bytes = P.pool_capacity_blocks * snp::kBlockBytes;
  ex->dmalloc(&ex->arena, ex->arena_bytes, sn_exec::M_ARENA, "cudaMalloc(arena)");
  ex->dmalloc(&ex->params, ex->n_params * 4, sn_exec::M_PARAMS, "cudaMalloc(params)");
  ex->dmalloc(&ex->grads, ex->n_params * 4, sn_exec::M_PARAMS, "cudaMalloc(grads)");
  ck(cudaMemset(ex->grads, 0, ex->n_params * sizeof(float)), "memset");
  ex->dmalloc(&ex->state, ex->n_state * 4, sn_exec::M_STATE, "cudaMalloc(state)");
  // BN state: stats {mean 0, invstd 1}, running {mean 0, var 1}
  std::vector<float> st(ex->n_state, 0.f);
  int64_t wt = 0, red = sn::red_scratch_floats(4), partial = 0;
  for (int i = 0; i < net.n; ++i) {
    LayerRt& l = ex->L[i];
    if (l.kind == snp::BN) {
      for (int c = 0; c < l.C; ++c) {
        st[l.state_off + l.C + c] = 1.f;
        st[l.state_off + 3 * l.C + c] = 1.f;
      }
    }
    if (l.kind == snp::BN || l.kind == snp::CONV || l.kind == snp::FC)
      red = std::max(red, sn::red_scratch_floats(l.C));
    if (l.kind == snp::CONV) {
      sn::KnobScope ks(l.kd);
      wt = std::max(wt, std::max<int64_t>(l.w_n, sn::conv_dgrad_scratch_floats(l.conv)));
    }
    if (l.kind == snp::FC) wt = std::max(wt, l.w_n);  // fc_dgrad's transposed weights
  }
  ck(cudaMemcpy(ex->state, st.data(), st.size() * sizeof(float), cudaMemcpyHostToDevice), "memcpy(state)");
  // split-K partials: a CONV weight gradient writes them into the conv
  // workspace its step was granted (Compiler::backward) and only otherwise
  // into wgrad scratch outside the pool, sized by those layers alone
  // (Compiler::size_wgrad_scratch); the split counts (capped at 64 Mi
  // floats of partials) are fixed per layer, so the summation order -- and
  // the gradients -- do not depend on the schedule.  `partial` here is the
  // FC layers' own split-K scratch.
  const int64_t cap = 64ll << 20;
  for (int i = 0; i < net.n; ++i) {
    LayerRt& l = ex->L[i];
    if (l.kind == snp::CONV) {
      sn::KnobScope ks(l.kw);
      l.wgrad_splits = sn::conv_wgrad_splits(l.conv, cap);
    } else if (l.kind == snp::FC) {
      l.fc_splits = sn::fc_splits(ex->B, l.fc_in, l.C, cap);
      partial = std::max(partial, static_cast<int64_t>(l.fc_splits) * ex->B * std::max(l.fc_in, l.C));
      l.wgrad_splits = sn::fc_wgrad_splits(ex->B, l.fc_in, l.C, cap);
      partial = std::max(partial, static_cast<int64_t>(l.wgrad_splits) * l.fc_in * l.C);
    }
  }
  if (ex->stem_layer >= 0) wt = std::max(wt, sn::stem_weight_floats(ex->L[ex->stem_layer].conv));
  int64_t tstats = 64;
  for (int i = 0; i < net.n; ++i) {
    LayerRt& l = ex->L[i];
    if (l.kind != snp::CONV) continue;
    sn::KnobScope ks(l.kf);
    l.stats_tiles = sn::conv_fwd_stats_tiles(l.conv, i == ex->stem_layer, &l.stats_rows);
    tstats = std::max(tstats, static_cast<int64_t>(l.stats_tiles) * 4 * l.C);
  }
  ex->dmalloc(&ex->tstats, tstats * 4, sn_exec::M_OTHER, "cudaMalloc(tile stats)");
  ex->partial_cap = std::max<int64_t>(partial, 64);
  ex->dmalloc(&ex->partial, ex->partial_cap * 4, sn_exec::M_OTHER, "cudaMalloc(partial)");
  ex->dmalloc(&ex->wt_scratch, std::max<int64_t>(wt, 64) * 4, sn_exec::M_OTHER, "cudaMalloc(wt)");
  ex->dmalloc(&ex->red, red * 4, sn_exec::M_OTHER, "cudaMalloc(red)");
  ex->dmalloc(&ex->wt_w, std::max<int64_t>(wt, 64) * 4, sn_exec::M_WGRAD, "cudaMalloc(wt_w)");
  ex->dmalloc(&ex->red_w, red * 4, sn_exec::M_WGRAD, "cudaMalloc(red_w)");
  int64_t pool_bytes = 256;
  for (int i = 0; i < net.n; ++i)
    if (ex->L[i].kind == snp::POOL) pool_bytes = std::max(pool_bytes, sn::pool_scratch_bytes(ex->L[i].pool));
  ex->dmalloc(&ex->pool_scratch, pool_bytes, sn_exec::M_OTHER, "cudaMalloc(pool scratch)");
  // saved max-pool argmaxes: layer state outside the pool accounting, like the
  // BN saved statistics (one byte per output element)
  for (int i = 0; i < net.n; ++i) {
    LayerRt& l = ex->L[i];
    if (l.kind == snp::POOL && sn::pool_saves_argmax(l.pool))
      ex->dmalloc(&l.argmax, static_cast<int64_t>(l.pool.N) * l.pool.P * l.pool.Q * l.pool.C, sn_exec::M_STATE,
                  "cudaMalloc(argmax)");
  }
  if (ex->data_id < 0) xfail(SN_EK_UNSUPPORTED, "numeric execution needs a DATA layer");
  const LayerRt& data = ex->L[ex->data_id];
  ex->image_floats = static_cast<int64_t>(ex->B) * data.H * data.W * data.C_raw;
  ex->dmalloc(&ex->images, ex->image_floats * 4, sn_exec::M_INPUT, "cudaMalloc(images)");
  ck(cudaMemset(ex->images, 0, ex->image_floats * sizeof(float)), "memset(images)");
  if (ex->stem_layer >= 0 || data.C != data.C_raw) {
    const int64_t n = ex->stem_layer >= 0 ? sn::stem_padded_floats(ex->L[ex->stem_layer].conv)
                                          : static_cast<int64_t>(ex->B) * data.per_sample;
    ex->dmalloc(&ex->data_buf, n * 4, sn_exec::M_INPUT, "cudaMalloc(data)");
    ck(cudaMemset(ex->data_buf, 0, n * sizeof(float)), "memset(data)");
  } else {
    ex->data_buf = ex->images;
  }
  ex->dmalloc(&ex->labels, ex->B * 4, sn_exec::M_INPUT, "cudaMalloc(labels)");
  ck(cudaMemset(ex->labels, 0, ex->B * sizeof(int32_t)), "memset(labels)");
  ex->dmalloc(&ex->loss_rows, ex->B * 4, sn_exec::M_OTHER, "cudaMalloc(loss_rows)");
  ex->dmalloc(&ex->loss, 16, sn_exec::M_OTHER, "cudaMalloc(loss)");
  ex->dmalloc(&ex->iteration, 16, sn_exec::M_OTHER, "cudaMalloc(iteration)");
  for (int i = 0; i < net.n; ++i)
    if (ex->side_root[i]) {
      float* p = nullptr;
      ex->dmalloc(&p, static_cast<int64_t>(ex->B) * ex->L[i].per_sample * 4, sn_exec::M_OTHER, "cudaMalloc(fork grad)");
      ex->side[i] = p;
    }
  ck(cudaMemset(ex->iteration, 0, sizeof(uint32_t) * 4), "memset(iteration)");
}

// ---------------------------------------------------------------------------
// Tape compilation.

struct Compiler {
  sn_exec* ex;
  const snp::Plan& P;
  const Net& net;
  std::unordered_map<int64_t, std::pair<int64_t, int64_t>> where;  // key -> (block off, blocks)
  std::unordered_map<int, bool> fresh;                             // grad owner -> not yet written
  std::unordered_map<int, cudaEvent_t> d2h_live;                   // act lid -> copy-out event
  std::vector<std::pair<std::pair<int64_t, int64_t>, cudaEvent_t>> freed_reading;  // region being read by D2H
  // buffers allocated over such regions: the events their first use must wait for
  std::unordered_map<int64_t, std::vector<cudaEvent_t>> pending_wait;
  std::unordered_set<cudaEvent_t> waited;
  std::unordered_map<int, cudaEvent_t> h2d_live;                   // act lid -> fetch event (not yet waited)
  std::vector<char> fetched;                                       // lids fetched anywhere in the tape
  bool used_s1 = false, used_s2 = false, used_s3 = false;
  // activation / gradient keys a side-stream weight gradient still reads: when
  // the tape frees one, later allocations over its blocks wait for that event
  std::unordered_map<int64_t, cudaEvent_t> side_reads;
  std::unordered_map<int, cudaEvent_t> wgrad_done;  // CONV layer -> its s3 weight-gradient completion
  bool used_s5 = false;
  cudaEvent_t wt_ready = nullptr;  // every CONV's dgrad weights prepared (s3); s0 waits before the first dgrad
  bool wt_waited = false;
  size_t next_bucket = 0;
  int data_id = -1;

  Compiler(sn_exec* e) : ex(e), P(e->plan->plan), net(e->plan->plan.net) {
    fetched.assign(net.n, 0);
    for (const auto& ev : P.tape)
      if (ev.op == 'P' || ev.op == 'D') fetched[ev.b] = 1;
    for (int i = 0; i < net.n; ++i)
      if (net.kind[i] == snp::DATA) data_id = i;
  }

  int cur_layer = -1, cur_type = 3;
  void push(std::function<void()> fn, int kernels) {
    ex->prog.push_back(Action{std::move(fn), kernels, kernels ? cur_layer : -1, kernels ? cur_type : 3});
  }

  float* ptr(int kind, int id) {
    if (kind == snp::K_ACT && id == data_id) return ex->data_buf;
    const int64_t key = key_code(kind, id);
    auto it = where.find(key);
    if (it == where.end())
      xfail(SN_EK_INTERNAL, std::string("tape references non-resident ") + (kind == 0 ? "act " : kind == 1 ? "grad " : "ws ") +
                                std::to_string(id));
    // first use of a buffer allocated over blocks another stream may still be
    // reading: the compute stream waits here, not at the allocation
    if (!pending_wait.empty()) {
      auto pw = pending_wait.find(key);
      if (pw != pending_wait.end()) {
        const std::vector<cudaEvent_t> evs = std::move(pw->second);
        pending_wait.erase(pw);
        for (cudaEvent_t ev : evs) flush_hazard(ev);
      }
    }
    return reinterpret_cast<float*>(ex->arena + it->second.first * snp::kBlockBytes);
  }

  // s0 waits for a reader event once; every hazard it covers is then retired
  void flush_hazard(cudaEvent_t ev) {
    if (waited.count(ev)) return;
    waited.insert(ev);
    s0_wait(ev);
    for (size_t i = 0; i < freed_reading.size();) {
      if (freed_reading[i].second == ev)
        freed_reading.erase(freed_reading.begin() + i);
      else
        ++i;
    }
  }

  void s0_wait(cudaEvent_t e) {
    cudaStream_t s0 = ex->s0;
    push([s0, e] { ck(cudaStreamWaitEvent(s0, e, 0), "wait"); }, 0);
  }

  void wait_fetch(int lid) {
    auto it = h2d_live.find(lid);
    if (it != h2d_live.end()) {
      // exposed transfer time: from when the compute stream reaches the wait
      // to when the fetch has landed
      const sn_exec::Timer tm = ex->new_timer(2, P.costs[lid].device_bytes);
      cudaStream_t s0 = ex->s0;
      push([=] { ck(record_timer(tm.a, s0), "record"); }, 0);
      s0_wait(it->second);
      push([=] { ck(record_timer(tm.b, s0), "record"); }, 0);
      h2d_live.erase(it);
    }
  }

  static bool overlap(int64_t a0, int64_t an, int64_t b0, int64_t bn) { return a0 < b0 + bn && b0 < a0 + an; }

  void on_alloc(const snp::Event& e) {
    const int64_t key = key_code(e.a, e.b);
    where[key] = {e.c, e.d};
    if (e.a == snp::K_GRAD) fresh[e.b] = true;
    // regions another stream may still be reading: waited at this buffer's
    // first use (ptr), not here
    for (const auto& h : freed_reading)
      if (overlap(e.c, e.d, h.first.first, h.first.second)) pending_wait[key].push_back(h.second);
  }

  void on_free(const snp::Event& e) {
    const int64_t key = key_code(e.a, e.b);
    auto it = where.find(key);
    if (it == where.end()) xfail(SN_EK_INTERNAL, "tape frees an unknown key");
    pending_wait.erase(key);  // never used: its hazards stay registered for the next occupant
    auto sr = side_reads.find(key);
    if (sr != side_reads.end()) {
      freed_reading.push_back({it->second, sr->second});
      side_reads.erase(sr);
    }
    if (e.a == snp::K_ACT) {
      auto d = d2h_live.find(e.b);
      if (d != d2h_live.end()) {
        freed_reading.push_back({it->second, d->second});
        // the stash keeps its copy; further fetches wait on the same event
      }
      wait_fetch(e.b);
    }
    where.erase(it);
  }

  void on_copy_out(int lid) {
    if (ex->opt.elide_backups && !fetched[lid]) return;
    const int64_t nbytes = P.costs[lid].device_bytes;
    char* host = ex->stash[lid];
    if (!host) host = ex->stash[lid] = stash_alloc(nbytes);
    const float* src = ptr(snp::K_ACT, lid);
    cudaEvent_t prod = ex->new_event(), done = ex->new_event();
    cudaStream_t s0 = ex->s0, s1 = ex->s1;
    const sn_exec::Timer tm = ex->new_timer(0, nbytes);
    const cudaMemcpyKind kind = ex->opt.stash ? cudaMemcpyDefault : cudaMemcpyDeviceToHost;
    push([=] {
      ck(cudaEventRecord(prod, s0), "record");
      ck(cudaStreamWaitEvent(s1, prod, 0), "wait");
      ck(record_timer(tm.a, s1), "record");
      ck(cudaMemcpyAsync(host, src, static_cast<size_t>(nbytes), kind, s1), "copy-out");
      ck(record_timer(tm.b, s1), "record");
      ck(cudaEventRecord(done, s1), "record");
    }, 0);
    d2h_live[lid] = done;
    ex->d2h_bytes += nbytes;
    used_s1 = true;
  }

  // Where a copied-out tensor lives (reference UTP: host
  // DRAM or "DRAM of other GPUs"): pinned host memory over PCIe, or HBM of
  // opt.stash_device -- an NVLink peer's spare memory, or this device itself
  // (loopback) -- addressed through UVA with peer access enabled.
  char* stash_alloc(int64_t nbytes) {
    char* p = nullptr;
    if (!ex->opt.stash) {
      ck(cudaHostAlloc(&p, static_cast<size_t>(nbytes), cudaHostAllocPortable), "cudaHostAlloc(stash)");
      ex->mem[sn_exec::M_HOST] += nbytes;
      return p;
    }
    const int dev = ex->opt.stash_device;
    if (dev != ex->device) {
      int can = 0;
      ck(cudaDeviceCanAccessPeer(&can, ex->device, dev), "cudaDeviceCanAccessPeer");
      if (!can)
        xfail(SN_EK_CONFIG, "stash device " + std::to_string(dev) + " is not a peer of device " +
                                std::to_string(ex->device));
      const cudaError_t e = cudaDeviceEnablePeerAccess(dev, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) ck(e, "cudaDeviceEnablePeerAccess");
      cudaGetLastError();
      ck(cudaSetDevice(dev), "cudaSetDevice(stash)");
    }
    const cudaError_t e = cudaMalloc(&p, static_cast<size_t>(nbytes));
    if (dev != ex->device) ck(cudaSetDevice(ex->device), "cudaSetDevice");
    ck(e, "cudaMalloc(device stash)");
    ex->mem[dev == ex->device ? sn_exec::M_STASH : sn_exec::M_PEER] += nbytes;
    ex->peer_stash.push_back({p, dev});
    return p;
  }

  void on_fetch(int lid) {
    const int64_t nbytes = P.costs[lid].device_bytes;
    auto d = d2h_live.find(lid);
    if (d == d2h_live.end()) xfail(SN_EK_INTERNAL, "fetch of a tensor that was never copied out");
    char* host = ex->stash[lid];
    float* dst = ptr(snp::K_ACT, lid);
    cudaEvent_t before = ex->new_event(), done = ex->new_event(), out = d->second;
    cudaStream_t s0 = ex->s0, s2 = ex->s2;
    const sn_exec::Timer tm = ex->new_timer(1, nbytes);
    const cudaMemcpyKind kind = ex->opt.stash ? cudaMemcpyDefault : cudaMemcpyHostToDevice;
    push([=] {
      ck(cudaEventRecord(before, s0), "record");
      ck(cudaStreamWaitEvent(s2, before, 0), "wait");
      ck(cudaStreamWaitEvent(s2, out, 0), "wait");
      ck(record_timer(tm.a, s2), "record");
      ck(cudaMemcpyAsync(dst, host, static_cast<size_t>(nbytes), kind, s2), "fetch");
      ck(record_timer(tm.b, s2), "record");
      ck(cudaEventRecord(done, s2), "record");
    }, 0);
    h2d_live[lid] = done;
    ex->h2d_bytes += nbytes;
    used_s2 = true;
  }

  // ---- layer kernels ----
  void forward(int lid, bool replay) {
    if (replay && dead_at[cur_ti] && net.kind[lid] != snp::ACT) return;  // output never read (plan_fusions)
    const LayerRt& l = ex->L[lid];
    for (int p : net.prev[lid]) wait_fetch(p);
    float* y = ptr(snp::K_ACT, lid);
    const float* x = net.prev[lid].empty() ? nullptr : ptr(snp::K_ACT, net.prev[lid][0]);
    const int64_t n = static_cast<int64_t>(ex->B) * l.per_sample;
    cudaStream_t st = ex->s0;
    sn_exec* e = ex;
    switch (l.kind) {
      case snp::CONV: {
        const float* w = ex->params + l.w_off;
        const float* b = ex->params + l.b_off;
        const sn::ConvShape cs = l.conv;
        float* ts = conv_stats_now ? ex->tstats : nullptr;
        if (lid == ex->stem_layer) {
          float* wp = ex->wt_scratch;
          push([=] { ck(sn::conv_stem_fwd(cs, x, w, wp, b, y, ts, st), "conv_stem_fwd"); }, 2);
          break;
        }
        const sn::ConvKnobs kf = l.kf;
        push([=] {
          sn::KnobScope ks(kf);
          ck(sn::conv_fwd(cs, x, w, b, y, st, ts), "conv_fwd");
        }, 1);
        break;
      }
      case snp::FC: {
        const float* w = ex->params + l.w_off;
        const float* b = ex->params + l.b_off;
        const int B = ex->B, I = l.fc_in, O = l.C, sp = l.fc_splits;
        float* part = ex->partial;
        push([=] { ck(sn::fc_fwd(B, I, O, x, w, b, y, part, sp, st), "fc_fwd"); }, sn::fc_fwd_launches(B, I, O));
        break;
      }
      case snp::BN: {
        const float* g = ex->params + l.w_off;
        const float* b = ex->params + l.b_off;
        float* stats = ex->state + l.state_off;
        float* running = replay ? nullptr : ex->state + l.state_off + 2 * l.C;
        const int64_t rows = static_cast<int64_t>(ex->B) * l.H * l.W;
        const int C = l.C;
        const float eps = l.num.bn_eps, mom = l.num.bn_momentum;
        const int compute = replay ? 0 : 1;
        float* red = ex->red;
        if (fuse_next) bn_in_ptr[lid] = x;  // the deferred apply reads it (see bn_input)
        if (bn_tiles_now && !replay) {
          // statistics from the producing CONV's epilogue tiles
          const float* ts = ex->tstats;
          const int nt = ex->L[net.prev[lid][0]].stats_tiles, tr = ex->L[net.prev[lid][0]].stats_rows;
          push([=] {
            ck(sn::bn_stats_from_tiles(ts, nt, tr, x, rows, C, stats, running, eps, mom, red, st), "bn_tile_stats");
          }, 2);
          if (!fuse_next)
            push([=] { ck(sn::bn_fwd(x, rows, C, g, b, y, stats, nullptr, eps, mom, 0, red, st), "bn_apply"); }, 1);
          break;
        }
        if (fuse_next) {
          // apply deferred to the consuming ReLU (bn_apply_relu); statistics now
          if (!replay)
            push([=] { ck(sn::bn_fwd(x, rows, C, g, b, nullptr, stats, running, eps, mom, 1, red, st), "bn_stats"); },
                 3);
          break;
        }
        push([=] { ck(sn::bn_fwd(x, rows, C, g, b, y, stats, running, eps, mom, compute, red, st), "bn_fwd"); },
             replay ? 1 : 4);
        break;
      }
      case snp::ACT:
        if (fused_bn >= 0 && join_fuse_at[cur_ti] >= 0) break;  // launched at the JOIN (bn_apply_relu_join)
        if (fused_bn >= 0 && pool_fuse_at[cur_ti] >= 0) break;  // launched at the POOL (pool_fwd_bn_relu)
        if (dead_at[cur_ti]) break;                                // output never read (plan_fusions)
        if (fused_bn >= 0) {
          const LayerRt& bl = ex->L[fused_bn];
          const float* bx = bn_input(fused_bn);
          // the BN output this ReLU reads; not written when nothing else reads it
          float* by = elide_out[fused_bn] ? nullptr : const_cast<float*>(x);
          const float* g = ex->params + bl.w_off;
          const float* b = ex->params + bl.b_off;
          const float* stats = ex->state + bl.state_off;
          const int64_t rows = static_cast<int64_t>(ex->B) * bl.H * bl.W;
          const int C = bl.C;
          push([=] { ck(sn::bn_apply_relu(bx, rows, C, g, b, stats, by, y, st), "bn_apply_relu"); }, 1);
          break;
        }
        push([=] { ck(sn::relu_fwd(x, y, n, st), "relu_fwd"); }, 1);
        break;
      case snp::POOL: {
        const sn::PoolShape ps = l.pool;
        uint8_t* am = l.argmax;
        if (pool_from[cur_ti] >= 0) {
          // BN apply + ReLU + max pool in one pass (peephole, see plan_fusions)
          const int ra = P.tape[pool_from[cur_ti]].b;
          const int bn = net.prev[ra][0];
          const LayerRt& bl = ex->L[bn];
          const float* bx = bn_input(bn);
          float* ry = elide_out[ra] ? nullptr : ptr(snp::K_ACT, ra);
          const float* g = ex->params + bl.w_off;
          const float* b = ex->params + bl.b_off;
          const float* stats = ex->state + bl.state_off;
          push([=] { ck(sn::pool_fwd_bn_relu(ps, bx, g, b, stats, ry, y, am, st), "pool_fwd_bn_relu"); }, 1);
          break;
        }
        push([=] { ck(sn::pool_fwd(ps, x, y, st, am), "pool_fwd"); }, 1);
        break;
      }
      case snp::LRN: {
        const int64_t pix = static_cast<int64_t>(ex->B) * l.H * l.W;
        const sn_layer_numerics nm = l.num;
        const int C = l.C;
        push([=] { ck(sn::lrn_fwd(x, y, pix, C, nm.lrn_size, nm.lrn_alpha, nm.lrn_beta, nm.lrn_k, st), "lrn_fwd"); }, 1);
        break;
      }
      case snp::DROPOUT: {
        const float rate = l.num.dropout_rate;
        const uint64_t seed = ex->opt.seed;
        push([=] { ck(sn::dropout_fwd(x, y, n, rate, seed, lid, e->iteration, st), "dropout_fwd"); }, 1);
        break;
      }
      case snp::SOFTMAX: {
        const int B = ex->B, F = static_cast<int>(l.per_sample);
        float* rows = replay ? nullptr : ex->loss_rows;
        const int32_t* lab = ex->labels;
        float* loss = ex->loss;
        push([=] {
          ck(sn::softmax_fwd(x, y, B, F, lab, rows, st), "softmax_fwd");
          if (rows) ck(sn::loss_reduce(rows, B, loss, st), "loss_reduce");
        }, replay ? 1 : 2);
        break;
      }
      case snp::JOIN: {
        if (join_from[cur_ti] >= 0) {
          // BN apply + ReLU + JOIN in one pass (peephole, see plan_fusions)
          const int ra = P.tape[join_from[cur_ti]].b;
          const int bn = net.prev[ra][0];
          const LayerRt& bl = ex->L[bn];
          const float* bx = bn_input(bn);
          float* by = elide_out[bn] ? nullptr : ptr(snp::K_ACT, bn);
          float* ry = elide_out[ra] ? nullptr : ptr(snp::K_ACT, ra);
          const int other = net.prev[lid][0] == ra ? net.prev[lid][1] : net.prev[lid][0];
          const float* oth = ptr(snp::K_ACT, other);
          const float* g = ex->params + bl.w_off;
          const float* b = ex->params + bl.b_off;
          const float* stats = ex->state + bl.state_off;
          const int64_t rows = static_cast<int64_t>(ex->B) * bl.H * bl.W;
          const int C = bl.C;
          push([=] { ck(sn::bn_apply_relu(bx, rows, C, g, b, stats, by, ry, st, oth, y), "bn_apply_relu_join"); }, 1);
          break;
        }
        const size_t at = ex->ptr_host.size();
        for (int p : net.prev[lid]) ex->ptr_host.push_back(ptr(snp::K_ACT, p));
        const int nin = static_cast<int>(net.prev[lid].size());
        push([=] { ck(sn::join_fwd(e->ptr_table + at, nin, y, n, st), "join_fwd"); }, 1);
        break;
      }
      default:
        xfail(SN_EK_UNSUPPORTED, "forward of unsupported layer kind");
    }
  }

  // Destination for d(input pid) and whether it is the first write.
  // the buffer of gradient owner `owner` (eff_owner numbering)
  float* grad_ptr(int owner) { return ex->side_root[owner] ? ex->side.at(owner) : ptr(snp::K_GRAD, owner); }

  float* dx_target(int pid, int* accumulate) {
    const int owner = ex->eff_owner[pid];
    if (owner < 0) return nullptr;
    float* p = grad_ptr(owner);
    auto it = fresh.find(owner);
    *accumulate = (it != fresh.end() && it->second) ? 0 : 1;
    fresh[owner] = false;
    return p;
  }

  void backward(int lid) {
    const LayerRt& l = ex->L[lid];
    for (int r : net.backward_reads_unique(lid)) wait_fetch(r);
    cudaStream_t st = ex->s0;
    sn_exec* e = ex;
    const int64_t n = static_cast<int64_t>(ex->B) * l.per_sample;
    const int owner = ex->eff_owner[lid];
    float* dy = (owner >= 0 && lid != ex->terminal) ? grad_ptr(owner) : nullptr;
    const int pid = net.prev[lid].empty() ? -1 : net.prev[lid][0];
    switch (l.kind) {
      case snp::CONV: {
        const float* x = ptr(snp::K_ACT, pid);
        const sn::ConvShape cs = l.conv;
        int acc = 0;
        float* dx = dx_target(pid, &acc);
        const float* w = ex->params + l.w_off;
        float* dw = ex->grads + l.w_off;
        float* db = ex->grads + l.b_off;
        const int pre = l.wt_pre && dx ? 1 : 0;
        float* wt = pre ? l.wt_pre : ex->wt_scratch;
        if (pre && !wt_waited) {
          s0_wait(wt_ready);
          wt_waited = true;
        }
        float* part = ex->partial;
        float* red = ex->red;
        if (conv_bias_done[lid]) db = nullptr;  // summed by the BN backward's dx pass
        const int nbias = db ? 2 : 0;
        // weight gradient on the side stream s3 (after everything s0 has issued so
        // far: x and dy are ready), dgrad on s0 right away
        cudaStream_t s3 = ex->s3;
        float* part_w = ex->partial_w;
        float* red_w = ex->red_w;
        float* wt_w = ex->wt_w;
        cudaEvent_t ready = ex->new_event(), wdone = ex->new_event();
        used_s3 = true;
        wgrad_done[lid] = wdone;
        side_reads[snp::key_code(snp::K_ACT, pid)] = wdone;
        if (owner >= 0 && !ex->side_root[owner]) side_reads[snp::key_code(snp::K_GRAD, owner)] = wdone;
        // The split-K partials go to the conv workspace the planner granted this
        // step (the selected algorithm's factor x output bytes, sized from the
        // free pool) when they fit; else to the executor's scratch outside the
        // pool.  The split count itself stays fixed per layer: it sets the
        // summation order, and the gradients must be bit-identical under every
        // feature set / schedule.
        const int sp = l.wgrad_splits;
        {
          const snp::Event& bev = P.tape[cur_ti];
          float* ws = nullptr;
          int64_t ws_floats = 0;
          const int64_t wkey = snp::key_code(snp::K_WS, bev.d);
          if (bev.d >= 0 && where.count(wkey)) {
            ws = ptr(snp::K_WS, static_cast<int>(bev.d));
            ws_floats = where[wkey].second * snp::kBlockBytes / static_cast<int64_t>(sizeof(float));
          }
          const int64_t need = wgrad_partial_floats(lid);
          if (ws && ws_floats >= need) {
            part_w = ws;
            side_reads[wkey] = wdone;  // written on s3 after the tape frees it
            ++ex->wgrad_ws_in_pool;
          } else {
            ++ex->wgrad_ws_outside;
          }
        }
        if (lid == ex->stem_layer) {  // DATA has no gradient
          const bool fused = stem_fuse_pending;
          const sn::StemBnFuse fz = stem_fuse;
          if (fused) {  // the BN input and dy (or the pool gradient) are read on s3 after the tape frees them
            side_reads[stem_fuse_keys[0]] = wdone;
            if (stem_fuse_keys[1] >= 0) side_reads[stem_fuse_keys[1]] = wdone;
            stem_fuse_pending = false;
          }
          const bool rows = sn::conv_stem_wgrad_rows_ok(cs);
          const int nk = rows ? 2 + sn::splitk_reduce_launches(148, cs.R * 32, cs.K) + (db ? 1 : 0) : 3 + nbias;
          push([=] {
            const cudaStream_t sw = e->serial ? st : s3;
            ck(cudaEventRecord(ready, st), "record");
            ck(cudaStreamWaitEvent(sw, ready, 0), "wait");
            ck(sn::conv_stem_wgrad(cs, x, dy, part_w, wt_w, dw, db, red_w, sw, fused ? &fz : nullptr),
               "conv_stem_wgrad");
            ck(cudaEventRecord(wdone, sw), "record");
          }, nk);
          break;
        }
        const sn::ConvKnobs kd = l.kd, kw = l.kw;
        int ndgrad = 0, nwgrad = 0;
        {
          sn::KnobScope ks(kd);
          ndgrad = !dx ? 0 : sn::conv_dgrad_launches(cs, pre);
        }
        {
          sn::KnobScope ks(kw);
          nwgrad = sn::conv_wgrad_launches(cs, sp, db != nullptr);
        }
        push([=] {
          const cudaStream_t sw = e->serial ? st : s3;
          ck(cudaEventRecord(ready, st), "record");
          ck(cudaStreamWaitEvent(sw, ready, 0), "wait");
          {
            sn::KnobScope ks(kw);
            ck(sn::conv_wgrad(cs, x, dy, dw, db, part_w, sp, red_w, sw), "conv_wgrad");
          }
          ck(cudaEventRecord(wdone, sw), "record");
          if (dx) {
            sn::KnobScope ks(kd);
            ck(sn::conv_dgrad(cs, dy, w, wt, dx, acc, st, pre), "conv_dgrad");
          }
        }, nwgrad + ndgrad);
        (void)nbias;
        (void)part;
        (void)red;
        break;
      }
      case snp::FC: {
        const float* x = ptr(snp::K_ACT, pid);
        int acc = 0;
        float* dx = dx_target(pid, &acc);
        const int B = ex->B, I = l.fc_in, O = l.C, sp = l.fc_splits;
        const float* w = ex->params + l.w_off;
        float* dw = ex->grads + l.w_off;
        float* db = ex->grads + l.b_off;
        float* part = ex->partial;
        float* red = ex->red;
        float* wt = ex->wt_scratch;
        const int wsp = l.wgrad_splits;
        push([=] {
          ck(sn::fc_wgrad(B, I, O, x, dy, dw, db, red, st, part, wsp), "fc_wgrad");
          if (dx) ck(sn::fc_dgrad(B, I, O, dy, w, dx, acc, part, sp, st, wt), "fc_dgrad");
        }, sn::fc_bwd_launches(B, I, O, wsp, dx != nullptr));
        break;
      }
      case snp::BN: {
        const float* x = ptr(snp::K_ACT, pid);
        int acc = 0;
        float* dx = dx_target(pid, &acc);
        const float* g = ex->params + l.w_off;
        float* dg = ex->grads + l.w_off;
        float* dbt = ex->grads + l.b_off;
        const float* beta = ex->params + l.b_off;
        const float* stats = ex->state + l.state_off;
        const int64_t rows = static_cast<int64_t>(ex->B) * l.H * l.W;
        const int C = l.C;
        float* red = ex->red;
        const int relu = bwd_relu ? 1 : 0;
        float* cpy = nullptr;
        int cpy_acc = 0;
        float* own = nullptr;
        if (bn_from_join[cur_ti] >= 0) {
          auto pj = pending_join.find(static_cast<int>(cur_ti));
          if (pj == pending_join.end()) xfail(SN_EK_INTERNAL, "fused JOIN backward not recorded");
          dy = const_cast<float*>(pj->second.dy);
          cpy = pj->second.other;
          cpy_acc = pj->second.other_acc;
          own = pj->second.own;
          pending_join.erase(pj);
        }
        float* dcb = nullptr;
        if (bn_bias_now && dx) {
          dcb = ex->grads + ex->L[pid].b_off;
          conv_bias_done[pid] = 1;
        }
        const int pool = bn_pool_at[cur_ti];
        if (pool >= 0) {  // statistics in the following max pool's block order
          const sn::PoolShape ps = ex->L[pool].pool;
          const uint8_t* am = ex->L[pool].argmax;
          auto pg = pending_gather.find(static_cast<int>(cur_ti));
          const bool gather = pool_gather_at[cur_ti] && pg != pending_gather.end() && dx && !acc;
          if (pool_gather_at[cur_ti] && !gather) xfail(SN_EK_INTERNAL, "pool gather planned but not possible");
          if (gather) {
            const float* dyp = pg->second.dy_pool;
            stem_fuse = sn::StemBnFuse{x, nullptr, stats, g, beta, sn::bn_coef_ptr(red, C), rows, relu,
                                       dyp, am, ps.P, ps.Q};
            stem_fuse_pending = true;
            stem_fuse_keys[0] = snp::key_code(snp::K_ACT, pid);
            stem_fuse_keys[1] = pg->second.key;
            pending_gather.erase(pg);
            push([=] {
              ck(sn::bn_bwd_pool_stats(ps, am, dyp, nullptr, x, C, g, beta, stats, relu, dg, dbt, red, st),
                 "bn_bwd_pool_stats");
            }, 2);
            break;
          }
          const float* dym = dy;
          push([=] {
            ck(sn::bn_bwd_pool_stats(ps, am, nullptr, dym, x, C, g, beta, stats, relu, dg, dbt, red, st),
               "bn_bwd_pool_stats");
          }, 2);
          if (stem_bn_fuse_at[cur_ti] && dx && !acc) {
            stem_fuse = sn::StemBnFuse{x, dy, stats, g, beta, sn::bn_coef_ptr(red, C), rows, relu};
            stem_fuse_pending = true;
            stem_fuse_keys[0] = snp::key_code(snp::K_ACT, pid);
            stem_fuse_keys[1] = snp::key_code(snp::K_GRAD, lid);
            break;
          }
          if (dx)
            push([=] { ck(sn::bn_bwd_dx(x, dy, rows, C, g, beta, stats, relu, dx, acc, red, st, dcb), "bn_bwd_dx"); },
                 dcb ? 2 : 1);
          break;
        }
        if (stem_bn_fuse_at[cur_ti] && dx && !acc) {  // dx formed inside the stem weight gradient
          stem_fuse = sn::StemBnFuse{x, dy, stats, g, beta, sn::bn_coef_ptr(red, C), rows, relu};
          stem_fuse_pending = true;
          stem_fuse_keys[0] = snp::key_code(snp::K_ACT, pid);
          stem_fuse_keys[1] = snp::key_code(snp::K_GRAD, lid);
          push([=] {
            ck(sn::bn_bwd(x, dy, rows, C, g, beta, stats, relu, nullptr, 0, dg, dbt, red, st), "bn_bwd_stats");
          }, 2);
          break;
        }
        push([=] {
          ck(sn::bn_bwd(x, dy, rows, C, g, beta, stats, relu, dx, acc, dg, dbt, red, st, dcb, cpy, cpy_acc, own),
             "bn_bwd");
        },
             dx ? (dcb ? 4 : 3) : 2);
        break;
      }
      case snp::ACT: {
        if (ex->side_root[lid]) {  // own gradient buffer: add the masked gradient into the producer's
          const bool written = !(fresh.count(lid) && fresh[lid]);
          int acc = 0;
          float* g = dx_target(pid, &acc);
          const float* y = ptr(snp::K_ACT, lid);
          if (g && written) push([=] { ck(sn::relu_bwd_to(y, dy, g, n, acc, st), "relu_bwd_to"); }, 1);
          break;
        }
        int acc = 0;
        float* g = dx_target(pid, &acc);
        if (g && dy && g != dy) xfail(SN_EK_INTERNAL, "in-place gradient buffer mismatch");
        if (bwd_skip) break;  // folded into the next action, the BN backward
        const float* y = ptr(snp::K_ACT, lid);
        if (g) push([=] { ck(sn::relu_bwd_inplace(y, g, n, st), "relu_bwd"); }, 1);
        break;
      }
      case snp::DROPOUT: {
        const float rate = l.num.dropout_rate;
        const uint64_t seed = ex->opt.seed;
        if (ex->side_root[lid]) {
          const bool written = !(fresh.count(lid) && fresh[lid]);
          int acc = 0;
          float* g = dx_target(pid, &acc);
          if (g && written)
            push([=] { ck(sn::dropout_bwd_to(dy, g, n, rate, seed, lid, e->iteration, acc, st), "dropout_bwd_to"); },
                 1);
          break;
        }
        int acc = 0;
        float* g = dx_target(pid, &acc);
        if (g) push([=] { ck(sn::dropout_bwd_inplace(g, n, rate, seed, lid, e->iteration, st), "dropout_bwd"); }, 1);
        break;
      }
      case snp::POOL: {
        const float* x = ptr(snp::K_ACT, pid);
        const float* y = ptr(snp::K_ACT, lid);
        int acc = 0;
        float* dx = dx_target(pid, &acc);
        const sn::PoolShape ps = l.pool;
        void* scratch = ex->pool_scratch;
        const int nk = sn::pool_bwd_kernels(ps);
        const uint8_t* am = l.argmax;
        const int bi = pool_skip_at[cur_ti];
        if (bi >= 0) {
          if (dx && !acc) {  // gathered by the BN backward and the stem weight gradient
            const int po = ex->eff_owner[lid];
            pending_gather[bi] =
                PendingGather{dy, ex->side_root[po] ? int64_t(-1) : snp::key_code(snp::K_GRAD, po)};
            break;
          }
          pool_gather_at[bi] = 0;
        }
        if (dx) push([=] { ck(sn::pool_bwd(ps, x, y, dy, dx, acc, scratch, st, am), "pool_bwd"); }, nk);
        break;
      }
      case snp::LRN: {
        const float* x = ptr(snp::K_ACT, pid);
        const float* y = ptr(snp::K_ACT, lid);
        int acc = 0;
        float* dx = dx_target(pid, &acc);
        const int64_t pix = static_cast<int64_t>(ex->B) * l.H * l.W;
        const sn_layer_numerics nm = l.num;
        const int C = l.C;
        if (dx)
          push([=] {
            ck(sn::lrn_bwd(x, y, dy, dx, pix, C, nm.lrn_size, nm.lrn_alpha, nm.lrn_beta, nm.lrn_k, acc, st), "lrn_bwd");
          }, 1);
        break;
      }
      case snp::SOFTMAX: {
        const float* y = ptr(snp::K_ACT, lid);
        int acc = 0;
        float* dx = dx_target(pid, &acc);
        const int B = ex->B, F = static_cast<int>(l.per_sample);
        const int32_t* lab = ex->labels;
        if (dx) push([=] { ck(sn::softmax_ce_bwd(y, lab, dx, B, F, acc, st), "softmax_bwd"); }, 1);
        break;
      }
      case snp::JOIN: {
        const auto& pv = net.prev[lid];
        auto ds = dense_at.find(cur_ti);
        if (ds != dense_at.end() && !dense_off[ds->second.chain]) {
          const DenseStep& d = ds->second;
          if (d.k == 0)  // the chain's sums start from dy(J_1): every input's buffer must be fresh
            for (int p : pv) {
              auto it = fresh.find(ex->eff_owner[p]);
              if (it == fresh.end() || !it->second) dense_off[d.chain] = 1;
            }
          if (!dense_off[d.chain]) {
            if (d.k == 0)
              for (int p : pv) fresh[ex->eff_owner[p]] = false;  // written from here on (deferred)
            float* r = grad_ptr(ex->eff_owner[d.p0]);
            const int acc_r = d.k == 0 ? 0 : 1;
            std::vector<float*> dsts;
            std::vector<int> accs;
            for (int q : d.finals) {
              dsts.push_back(grad_ptr(ex->eff_owner[q]));
              accs.push_back(0);
            }
            const int k = static_cast<int>(dsts.size());
            push([=] { ck(sn::grad_prefix(dy, r, acc_r, dsts.data(), accs.data(), k, n, st), "join_bwd_dense"); },
                 sn::grad_prefix_launches(k));
            break;
          }
        }
        if (join_to_bn[cur_ti] >= 0) {
          // deferred into the BN backward (see plan_fusions): record the pointers now
          const int ra = join_relu[cur_ti];
          const int other = pv[0] == ra ? pv[1] : pv[0];
          int a_r = 0, a_o = 0;
          float* own = dx_target(ra, &a_r);  // the BN's own gradient buffer: written only with copy_own
          if (join_copy_own[cur_ti] && a_r) xfail(SN_EK_INTERNAL, "JOIN fold: the BN's dy buffer is not fresh");
          float* d_o = dx_target(other, &a_o);
          pending_join[join_to_bn[cur_ti]] = PendingJoin{dy, d_o, a_o, join_copy_own[cur_ti] ? own : nullptr};
          break;
        }
        if (pv.size() == 2 && n % 4 == 0) {
          const int o0 = ex->eff_owner[pv[0]], o1 = ex->eff_owner[pv[1]];
          if (o0 >= 0 && o1 >= 0 && o0 != o1) {  // one read of dy, two destinations
            int a0 = 0, a1 = 0;
            float* d0 = dx_target(pv[0], &a0);
            float* d1 = dx_target(pv[1], &a1);
            push([=] { ck(sn::grad_copy2(dy, d0, a0, d1, a1, n, st), "join_bwd2"); }, 1);
            break;
          }
        }
        if (pv.size() > 2 && n % 4 == 0) {
          std::vector<int> owners;
          for (int p : pv) owners.push_back(ex->eff_owner[p]);
          std::vector<int> sorted = owners;
          std::sort(sorted.begin(), sorted.end());
          if (std::adjacent_find(sorted.begin(), sorted.end()) == sorted.end()) {  // distinct buffers
            std::vector<float*> dsts;
            std::vector<int> accs;
            for (int p : pv) {
              int acc = 0;
              float* dx = dx_target(p, &acc);
              if (!dx) continue;
              dsts.push_back(dx);
              accs.push_back(acc);
            }
            const int k = static_cast<int>(dsts.size());
            if (k) push([=] { ck(sn::grad_copy_multi(dy, dsts.data(), accs.data(), k, n, st), "join_bwd_k"); },
                        sn::grad_copy_multi_launches(k));
            break;
          }
        }
        for (int p : pv) {
          int acc = 0;
          float* dx = dx_target(p, &acc);
          if (dx) push([=] { ck(sn::grad_copy(dy, dx, n, acc, st), "join_bwd"); }, 1);
        }
        break;
      }
      default:
        xfail(SN_EK_UNSUPPORTED, "backward of unsupported layer kind");
    }
  }

  // Peephole fusion on the tape: a BN forward (or replay) whose very next
  // device action is the forward (replay) of the ReLU reading it, with neither
  // the BN input nor its output freed in between, is split into "statistics
  // now" + "apply fused into the ReLU" (one pass writes both outputs).
  //
  // Backward: a ReLU backward whose next compute action is the backward of the
  // BN it reads (its only consumer) is folded into that BN backward, which
  // recomputes the mask from the BN input.  When every forward / replay of the
  // pair is fused as well, nothing reads the BN output, so it is not written.
  bool fuse_next = false;
  int fused_bn = -1;
  // BN input of a deferred (fused) apply, recorded at the BN: the tape may free
  // it before the consuming ReLU / POOL / JOIN runs (plan_fusions checks that
  // nothing is allocated over it meanwhile)
  std::unordered_map<int, const float*> bn_in_ptr;
  const float* bn_input(int bn) {
    const int p = net.prev[bn][0];
    if (where.count(snp::key_code(snp::K_ACT, p))) return ptr(snp::K_ACT, p);
    auto it = bn_in_ptr.find(bn);
    if (it == bn_in_ptr.end()) xfail(SN_EK_INTERNAL, "fused BN apply: input neither resident nor recorded");
    return it->second;
  }
  size_t cur_ti = 0;
  // BN+ReLU (fused) forward / replay whose next compute action is the same op
  // of a 2-input JOIN reading the ReLU: the whole chain runs at the JOIN.
  std::vector<int> join_fuse_at, join_from;
  std::vector<int> pool_fuse_at, pool_from;  // BN+ReLU -> max POOL: ACT tape index <-> POOL tape index
  std::vector<char> dead_at;  // forward / replay whose outputs are never read: not launched
  // JOIN backward folded into the BN backward of the ReLU it feeds: join_to_bn[i]
  // = tape index of that BN backward; the JOIN's gradient is read there
  // directly and copied into the other input's buffer by the reduction pass.
  std::vector<int> join_to_bn, bn_from_join, join_relu;
  struct PendingJoin {
    const float* dy = nullptr;
    float* other = nullptr;
    int other_acc = 0;
    float* own = nullptr;  // join_copy_own: the BN's own dy buffer, written by the first pass
  };
  std::vector<char> join_copy_own;
  std::unordered_map<int, PendingJoin> pending_join;  // keyed by BN-backward tape index
  // Dense JOIN chains (DenseNet-style blocks, JOIN = sum): JOIN backwards
  // J_1 .. J_m in tape order whose input sets are nested, I(J_{k+1}) = I(J_k)
  // minus one input q_k.  The gradient of q_k is complete after J_k: it is
  // the running sum dy(J_1) + ... + dy(J_k), kept in the buffer of an input
  // p0 common to the whole chain (whose gradient is the chain's full sum).
  // Each J_k adds its dy into the running sum and writes the buffers of the
  // inputs it finishes -- 2 + 2 tensor passes per JOIN instead of 1 + 2 |I(J)|
  // -- bit-identical to the per-input backward (every buffer receives the same
  // additions in the same order).
  struct DenseStep {
    int chain = -1, k = 0, p0 = -1;
    std::vector<int> finals;  // inputs whose gradient is finished at this step
  };
  std::unordered_map<size_t, DenseStep> dense_at;  // JOIN backward tape index -> its step
  std::vector<char> dense_off;                      // per chain: disabled (an input's buffer was not fresh)
  // stem BN backward -> stem CONV backward: the BN's dx pass runs inside the
  // stem weight gradient (sn::StemBnFuse), dx is never written
  std::vector<char> stem_bn_fuse_at;
  bool stem_fuse_pending = false;
  sn::StemBnFuse stem_fuse{};
  int64_t stem_fuse_keys[2] = {0, 0};
  // BN -> ReLU -> 3x3/s2 max pool (saved argmax): the BN backward statistics
  // run in the pool's 2 x 2 block order (bn_bwd_pool_stats; a reassociating
  // fusion, same bits whether dy is gathered or read).  bn_pool_at: BN
  // backward index -> the pool layer.  pool_gather_at: BN backward index whose
  // statistics and (stem weight gradient) dx gather dy from the pool's
  // gradient and argmax; pool_skip_at: that pool's backward index -> the BN
  // backward index (its dx is never written).
  std::vector<int> bn_pool_at, pool_skip_at;
  std::vector<char> pool_gather_at;
  struct PendingGather {
    const float* dy_pool = nullptr;
    int64_t key = -1;  // the pool gradient's arena key (-1: outside the arena)
  };
  std::unordered_map<int, PendingGather> pending_gather;  // keyed by BN-backward tape index
  // CONV forward -> BN forward (next compute action, reading that output): the
  // CONV epilogue emits per-tile statistics, the BN only combines them.
  bool conv_stats_now = false, bn_tiles_now = false;
  std::vector<char> conv_stats_at, bn_tiles_at;
  // BN backward whose input is a CONV output consumed only by this BN: the dx
  // pass also sums the CONV's bias gradient (the CONV's gradient buffer gets
  // nothing else; replays in between do not touch it).
  bool bn_bias_now = false;
  std::vector<char> bn_bias_at;
  std::vector<char> conv_bias_done;
  bool bwd_skip = false, bwd_relu = false;
  std::vector<char> fuse_at, act_bwd_skip, bn_bwd_relu;
  std::vector<int> fused_into;
  std::vector<char> fused_x_freed;  // that BN+ReLU fusion reads a BN input the tape freed before the ReLU
  std::vector<char> elide_out;  // per layer: output never materialised
  static bool is_compute(char op) { return op == 'C' || op == 'R' || op == 'B'; }
  bool bn_relu_pair(int act) const {
    if (net.kind[act] != snp::ACT || net.prev[act].size() != 1) return false;
    const int bn = net.prev[act][0];
    return net.kind[bn] == snp::BN && net.next[bn].size() == 1 && ex->L[bn].C % 4 == 0 && !net.prev[bn].empty();
  }
  void plan_fusions() {
    const size_t T = P.tape.size();
    fuse_at.assign(T, 0);
    fused_into.assign(T, -1);
    fused_x_freed.assign(T, 0);
    act_bwd_skip.assign(T, 0);
    bn_bwd_relu.assign(T, 0);
    elide_out.assign(net.n, 0);
    conv_stats_at.assign(T, 0);
    bn_tiles_at.assign(T, 0);
    join_fuse_at.assign(T, -1);
    join_from.assign(T, -1);
    pool_fuse_at.assign(T, -1);
    pool_from.assign(T, -1);
    dead_at.assign(T, 0);
    join_to_bn.assign(T, -1);
    bn_from_join.assign(T, -1);
    join_relu.assign(T, -1);
    join_copy_own.assign(T, 0);
    stem_bn_fuse_at.assign(T, 0);
    bn_pool_at.assign(T, -1);
    pool_skip_at.assign(T, -1);
    pool_gather_at.assign(T, 0);
    bn_bias_at.assign(T, 0);
    conv_bias_done.assign(net.n, 0);
    const char* env = std::getenv("SN_FUSE");  // SN_FUSE=0: one kernel per layer (A/B and bitwise tests)
    if (env && env[0] == '0') {
      ex->elided = elide_out;
      return;
    }
    // SN_FUSE_REASSOC=0: keep the fusions that reorder floating-point sums off
    // (CONV-epilogue BN statistics, BN-backward CONV bias gradient), so the
    // remaining fusions can be checked bit-exactly against SN_FUSE=0
    const char* env_ra = std::getenv("SN_FUSE_REASSOC");
    const bool reassoc = !(env_ra && env_ra[0] == '0');
    if (reassoc) {
      for (size_t i = 0; i < T; ++i) {
        const snp::Event& e = P.tape[i];
        if (e.op != 'C' || net.kind[e.b] != snp::CONV || ex->L[e.b].stats_tiles <= 0) continue;
        for (size_t j = i + 1; j < T; ++j) {
          const snp::Event& f = P.tape[j];
          if (!is_compute(f.op)) continue;
          if (f.op == 'C' && net.kind[f.b] == snp::BN && net.prev[f.b].size() == 1 && net.prev[f.b][0] == e.b) {
            conv_stats_at[i] = 1;
            bn_tiles_at[j] = 1;
          }
          break;
        }
      }
    }
    for (size_t i = 0; i < T && reassoc; ++i) {
      const snp::Event& e = P.tape[i];
      if (e.op != 'B' || net.kind[e.b] != snp::BN || net.prev[e.b].size() != 1) continue;
      const int cv = net.prev[e.b][0];
      if (net.kind[cv] != snp::CONV || net.next[cv].size() != 1 || !sn::bn_bwd_bias_ok(ex->L[e.b].C)) continue;
      // the stem's weight-gradient kernel sums its bias gradient itself (fused or not, same order)
      if (cv == ex->stem_layer && sn::conv_stem_wgrad_rows_ok(ex->L[cv].conv)) continue;
      bn_bias_at[i] = 1;
    }
    for (size_t i = 0; i < T; ++i) {
      const snp::Event& e = P.tape[i];
      if ((e.op != 'C' && e.op != 'R') || net.kind[e.b] != snp::BN) continue;
      const int bn = e.b;
      if (ex->L[bn].C % 4 != 0 || net.prev[bn].empty()) continue;
      // The BN input may be freed before the ReLU runs (DenseNet-style: the JOIN
      // output feeding the BN is dropped right after the BN, for recompute): the
      // fused apply at the ReLU still reads it, so that is allowed only while no
      // allocation lands on its blocks, except the ReLU's own output at exactly
      // those blocks (elementwise in place: each element read, then written).
      const int bx = net.prev[bn][0];
      int64_t xoff = -1, xblk = 0;
      bool x_freed = false;
      for (size_t j = i; j-- > 0;) {
        const snp::Event& f = P.tape[j];
        if (f.op == 'A' && f.a == snp::K_ACT && f.b == bx) {
          xoff = f.c;
          xblk = f.d;
          break;
        }
      }
      for (size_t j = i + 1; j < T; ++j) {
        const snp::Event& f = P.tape[j];
        if (f.op == 'F' && f.a == snp::K_ACT && f.b == bn) break;
        if (f.op == 'F' && f.a == snp::K_ACT && f.b == bx) {
          if (xoff < 0 || net.kind[bx] == snp::DATA) break;
          x_freed = true;
          continue;
        }
        if (x_freed && f.op == 'A' && overlap(f.c, f.d, xoff, xblk)) {
          const bool own_out = f.a == snp::K_ACT && net.kind[f.b] == snp::ACT && net.prev[f.b].size() == 1 &&
                               net.prev[f.b][0] == bn && f.c == xoff && f.d == xblk;
          if (!own_out) break;
          continue;
        }
        if (f.op == 'C' || f.op == 'R' || f.op == 'B' || f.op == 'O' || f.op == 'P' || f.op == 'D') {
          if (f.op == e.op && net.kind[f.b] == snp::ACT && net.prev[f.b].size() == 1 && net.prev[f.b][0] == bn) {
            fuse_at[i] = 1;
            fused_into[j] = bn;
            fused_x_freed[j] = x_freed ? 1 : 0;
          }
          break;
        }
      }
    }
    std::vector<int> act_fwd(net.n, 0), act_fwd_fused(net.n, 0), bn_fwd(net.n, 0), bn_fwd_fused(net.n, 0);
    std::vector<char> act_bwd_fused(net.n, 0);
    // BN replays the reference schedules between the ReLU backward and the BN
    // backward (for BACKWARD_NEEDS the fused backward does not have): dead
    std::vector<char> pre_bwd_replay(T, 0);
    for (size_t i = 0; i < T; ++i) {
      const snp::Event& e = P.tape[i];
      if (e.op == 'C' || e.op == 'R') {
        if (net.kind[e.b] == snp::ACT) {
          ++act_fwd[e.b];
          act_fwd_fused[e.b] += fused_into[i] >= 0;
        } else if (net.kind[e.b] == snp::BN && !pre_bwd_replay[i]) {
          ++bn_fwd[e.b];
          bn_fwd_fused[e.b] += fuse_at[i];
        }
      }
      if (e.op != 'B' || !bn_relu_pair(e.b)) continue;
      const int bn = net.prev[e.b][0];
      std::vector<size_t> bn_replays;
      for (size_t j = i + 1; j < T; ++j) {
        const snp::Event& f = P.tape[j];
        if (!is_compute(f.op)) continue;
        if (f.op == 'R' && f.b == bn && !fuse_at[j]) {  // recomputes the BN output nobody reads now
          bn_replays.push_back(j);
          continue;
        }
        if (f.op == 'B' && f.b == bn) {
          act_bwd_skip[i] = 1;
          bn_bwd_relu[j] = 1;
          act_bwd_fused[e.b] = 1;
          for (size_t k : bn_replays) {
            pre_bwd_replay[k] = 1;
            dead_at[k] = 1;
          }
        }
        break;
      }
    }
    for (int a = 0; a < net.n; ++a) {
      if (!bn_relu_pair(a) || !act_bwd_fused[a]) continue;
      const int bn = net.prev[a][0];
      if (act_fwd[a] == act_fwd_fused[a] && bn_fwd[bn] == bn_fwd_fused[bn]) elide_out[bn] = 1;
    }
    // ReLU -> JOIN: every event between the two may allocate (the JOIN output)
    // or touch unrelated tensors, but must not free / copy the BN input, the
    // BN output (unless it is never materialised) or the ReLU output (they are
    // read or written at the JOIN).
    std::vector<int> act_join_fused(net.n, 0);
    for (size_t i = 0; i < T; ++i) {
      if (fused_into[i] < 0 || fused_x_freed[i]) continue;  // launched at the ReLU only
      const snp::Event& e = P.tape[i];
      const int ra = e.b, bn = fused_into[i], bin = net.prev[bn][0];
      for (size_t j = i + 1; j < T; ++j) {
        const snp::Event& f = P.tape[j];
        if ((f.op == 'F' && f.a == snp::K_ACT) || f.op == 'O' || f.op == 'P' || f.op == 'D') {
          // the BN output, when never materialised, may be dropped in between
          if (f.op == 'F' && f.b == bn && elide_out[bn]) continue;
          if (f.b == ra || f.b == bn || f.b == bin) break;
          continue;
        }
        if (!is_compute(f.op)) continue;
        const auto& pv = net.prev[f.b];
        if (f.op == e.op && net.kind[f.b] == snp::JOIN && pv.size() == 2 && (pv[0] == ra) != (pv[1] == ra) &&
            ex->L[f.b].C % 4 == 0) {
          join_fuse_at[i] = static_cast<int>(j);
          join_from[j] = static_cast<int>(i);
          ++act_join_fused[ra];
        }
        break;
      }
    }
    // ReLU -> max POOL (saved argmax, so the pool backward reads neither
    // activation): the same window rules as ReLU -> JOIN
    std::vector<int> act_pool_fused(net.n, 0), pool_fwd_n(net.n, 0), pool_fwd_fused(net.n, 0);
    for (size_t i = 0; i < T; ++i) {
      const snp::Event& e = P.tape[i];
      if ((e.op == 'C' || e.op == 'R') && net.kind[e.b] == snp::POOL) ++pool_fwd_n[e.b];
      if (fused_into[i] < 0 || fused_x_freed[i] || join_fuse_at[i] >= 0) continue;
      const int ra = e.b, bn = fused_into[i], bin = net.prev[bn][0];
      for (size_t j = i + 1; j < T; ++j) {
        const snp::Event& f = P.tape[j];
        if ((f.op == 'F' && f.a == snp::K_ACT) || f.op == 'O' || f.op == 'P' || f.op == 'D') {
          if (f.op == 'F' && f.b == bn && elide_out[bn]) continue;
          if (f.b == ra || f.b == bn || f.b == bin) break;
          continue;
        }
        if (!is_compute(f.op)) continue;
        const auto& pv = net.prev[f.b];
        if (f.op == e.op && net.kind[f.b] == snp::POOL && pv.size() == 1 && pv[0] == ra && ex->L[f.b].argmax &&
            sn::pool_fwd_bn_relu_ok(ex->L[f.b].pool)) {
          pool_fuse_at[i] = static_cast<int>(j);
          pool_from[j] = static_cast<int>(i);
          ++act_pool_fused[ra];
          ++pool_fwd_fused[f.b];
        }
        break;
      }
    }
    for (int a = 0; a < net.n; ++a) {
      if (!bn_relu_pair(a) || !act_bwd_fused[a] || net.next[a].size() != 1) continue;
      // (ReLU output elision: after the dead-write analysis below)
    }
    // Dead writes: a fused BN+ReLU forward / replay (BN output not
    // materialised) whose ReLU output nobody reads before it is freed or
    // rewritten -- typically a replay the reference schedules because the
    // ReLU backward reads y, which here is folded into the BN backward.
    for (size_t i = 0; i < T; ++i) {
      if (fused_into[i] < 0 || join_fuse_at[i] >= 0 || pool_fuse_at[i] >= 0 || !elide_out[fused_into[i]]) continue;
      const int ra = P.tape[i].b;
      bool read = false;
      for (size_t j = i + 1; j < T && !read; ++j) {
        const snp::Event& f = P.tape[j];
        if (f.op == 'F' && f.a == snp::K_ACT && f.b == ra) break;
        if ((f.op == 'C' || f.op == 'R') && f.b == ra) break;  // rewritten
        if (f.op == 'O' && f.b == ra) read = true;
        if ((f.op == 'C' || f.op == 'R') && join_from[j] < 0 && pool_from[j] < 0)
          for (int p : net.prev[f.b]) read |= p == ra;
        if (f.op == 'B') {
          if (f.b == ra) read |= !act_bwd_skip[j];
          const int k = net.kind[f.b];
          const bool pool_am = k == snp::POOL && ex->L[f.b].argmax && sn::pool_bwd_argmax_only(ex->L[f.b].pool);
          if (k == snp::CONV || k == snp::BN || (k == snp::POOL && !pool_am) || k == snp::LRN || k == snp::FC)
            for (int p : net.prev[f.b]) read |= p == ra;
        }
      }
      if (!read) dead_at[i] = 1;
    }
    // ReLU -> JOIN / POOL chains: the ReLU output is never materialised when
    // every live (not dead) forward of the ReLU is fused into its single
    // consumer and every forward of that consumer is such a fused chain (the
    // reference replays ReLU outputs for the ReLU backward, which is folded
    // into the BN backward here: those replays are dead)
    std::vector<int> join_fwd_n(net.n, 0), join_fwd_fused(net.n, 0);
    for (size_t i = 0; i < T; ++i) {
      const snp::Event& e = P.tape[i];
      if ((e.op != 'C' && e.op != 'R') || net.kind[e.b] != snp::JOIN) continue;
      ++join_fwd_n[e.b];
      join_fwd_fused[e.b] += join_from[i] >= 0;
    }
    for (int a = 0; a < net.n; ++a) {
      if (!bn_relu_pair(a) || !act_bwd_fused[a] || net.next[a].size() != 1) continue;
      const int nx = net.next[a][0];
      int live = 0;
      for (size_t i = 0; i < T; ++i)
        live += (P.tape[i].op == 'C' || P.tape[i].op == 'R') && P.tape[i].b == a && !dead_at[i];
      if (act_join_fused[a] > 0 && live == act_join_fused[a] && join_fwd_n[nx] == join_fwd_fused[nx])
        elide_out[a] = 1;
      if (act_pool_fused[a] > 0 && live == act_pool_fused[a] && pool_fwd_n[nx] == pool_fwd_fused[nx])
        elide_out[a] = 1;
    }
    // Dead replays (general): a replay of an unfused layer whose output no later
    // action reads before it is freed or rewritten -- under the kernels' actual
    // reads, which are narrower than the reference's BACKWARD_NEEDS (the ReLU
    // backward folded into the BN backward reads the BN input, not the BN
    // output; average-pool backward reads neither x nor y).
    auto reads_act = [&](size_t j, int L) -> bool {
      const snp::Event& f = P.tape[j];
      const int M = f.b;
      if (f.op == 'O') return M == L;
      if (f.op == 'C' || f.op == 'R') {
        if (dead_at[j] || join_fuse_at[j] >= 0 || pool_fuse_at[j] >= 0) return false;  // not launched here
        if (pool_from[j] >= 0) return L == net.prev[net.prev[P.tape[pool_from[j]].b][0]][0];  // reads the BN input
        if (fused_into[j] >= 0) return net.prev[fused_into[j]][0] == L;  // BN+ReLU: reads the BN input
        if (join_from[j] >= 0) {
          const int ra = P.tape[join_from[j]].b, bnj = net.prev[ra][0];
          const int oth = net.prev[M][0] == ra ? net.prev[M][1] : net.prev[M][0];
          return L == net.prev[bnj][0] || L == oth;
        }
        if (net.kind[M] == snp::BN && fuse_at[j] && f.op == 'R') return false;  // stats only on replay: none
        for (int p : net.prev[M])
          if (p == L) return true;
        return false;
      }
      if (f.op == 'B') {
        const int k = net.kind[M];
        const bool x = !net.prev[M].empty() && net.prev[M][0] == L;
        switch (k) {
          case snp::CONV: case snp::FC: case snp::BN: return x;
          case snp::POOL:
            if (ex->L[M].argmax && sn::pool_bwd_argmax_only(ex->L[M].pool)) return false;
            return ex->L[M].pool.mode == 0 && (x || M == L);
          case snp::LRN: return x || M == L;
          case snp::SOFTMAX: return M == L;
          case snp::ACT: return M == L && !act_bwd_skip[j];
          default: return false;  // JOIN, DROPOUT read no activations
        }
      }
      return false;
    };
    for (size_t i = 0; i < T; ++i) {
      const snp::Event& e = P.tape[i];
      if (e.op != 'R' || dead_at[i] || fused_into[i] >= 0 || join_from[i] >= 0 || join_fuse_at[i] >= 0 ||
          pool_from[i] >= 0)
        continue;
      const int L = e.b;
      if (net.kind[L] == snp::BN && fuse_at[i]) continue;  // launches nothing anyway
      if (net.kind[L] == snp::SOFTMAX) continue;          // keeps its loss-row side effect simple
      bool read = false;
      for (size_t j = i + 1; j < T && !read; ++j) {
        const snp::Event& f = P.tape[j];
        if (f.op == 'F' && f.a == snp::K_ACT && f.b == L) {
          // freed, but a deferred BN apply fused into the next compute event
          // (a ReLU) may still read it as the BN input (see the fusion above)
          for (size_t k = j + 1; k < T; ++k) {
            if (!is_compute(P.tape[k].op)) continue;
            read = fused_into[k] >= 0 && net.prev[fused_into[k]][0] == L && !dead_at[k] &&
                   join_fuse_at[k] < 0 && pool_fuse_at[k] < 0;
            break;
          }
          break;
        }
        if ((f.op == 'C' || f.op == 'R') && f.b == L) break;
        read = reads_act(j, L);
      }
      if (!read) dead_at[i] = 1;
    }
    // JOIN backward -> BN backward: safe when the JOIN's gradient buffer is not
    // re-allocated (over its block range) before the BN backward reads it
    for (size_t i = 0; i < T; ++i) {
      const snp::Event& e = P.tape[i];
      if (e.op != 'B' || net.kind[e.b] != snp::JOIN || net.prev[e.b].size() != 2) continue;
      const int jn = e.b;
      int ra = -1;
      for (int p : net.prev[jn])
        if (bn_relu_pair(p) && net.next[p].size() == 1) ra = p;
      if (ra < 0) continue;
      const int other = net.prev[jn][0] == ra ? net.prev[jn][1] : net.prev[jn][0];
      if (other == ra || net.grad_owner(other) < 0 || ex->L[jn].C % 4 != 0) continue;
      const int bn = net.prev[ra][0];
      if (net.grad_owner(ra) != bn) continue;
      int64_t joff = -1, jblk = 0;  // the JOIN gradient buffer's blocks
      for (size_t j = i; j-- > 0;) {
        const snp::Event& f = P.tape[j];
        if (f.op == 'A' && f.a == snp::K_GRAD && f.b == jn) {
          joff = f.c;
          jblk = f.d;
          break;
        }
      }
      if (joff < 0) continue;
      const int bn_dx_owner = net.grad_owner(net.prev[bn][0]);
      // the BN's own dy buffer (the ReLU's gradient, in place), allocated before
      int64_t ooff = -1, oblk = 0, xoff = -1, xblk = 0;
      for (size_t j = i; j-- > 0;) {
        const snp::Event& f = P.tape[j];
        if (f.op == 'A' && f.a == snp::K_GRAD && f.b == bn) {
          ooff = f.c;
          oblk = f.d;
          break;
        }
      }
      bool copy_own = false;
      for (size_t j = i + 1; j < T; ++j) {
        const snp::Event& f = P.tape[j];
        // a new buffer over the JOIN gradient's blocks breaks the fusion, except
        // the BN's own dx target: placed exactly there, dx = f(dy, x) is
        // elementwise, so reading dy and writing dx at the same address is safe;
        // placed partly over it, the first (statistics) pass also copies dy into
        // the BN's own dy buffer and the dx pass reads that copy (copy_own)
        if (f.op == 'A' && overlap(f.c, f.d, joff, jblk)) {
          if (!(f.a == snp::K_GRAD && f.b == bn_dx_owner)) break;
          if (!(f.c == joff && f.d == jblk)) {
            copy_own = true;
            xoff = f.c;
            xblk = f.d;
          }
        }
        if (f.op == 'B' && f.b == bn) {
          const bool own_ok = !copy_own || (ooff >= 0 && !overlap(ooff, oblk, joff, jblk) &&
                                            !overlap(ooff, oblk, xoff, xblk));
          if (bn_bwd_relu[j] && own_ok) {
            join_to_bn[i] = static_cast<int>(j);
            bn_from_join[j] = static_cast<int>(i);
            join_relu[i] = ra;
            join_copy_own[i] = copy_own ? 1 : 0;
          }
          break;
        }
        if (f.op == 'B' && f.b != ra) break;  // another backward in between: keep it simple
      }
    }
    // stem BN backward -> stem CONV backward (next compute action): the stem
    // weight gradient reads the BN input and the BN's dy and forms dx itself,
    // provided nothing is allocated over those two tensors' blocks before it
    // has read them (they are freed at the end of the BN's backward step)
    const int stem = ex->stem_layer;
    const char* env_sb = std::getenv("SN_FUSE_STEM_BN");  // =0: materialise the stem BN's dx (A/B test)
    for (size_t i = 0; i < T && stem >= 0 && !(env_sb && env_sb[0] == '0'); ++i) {
      const snp::Event& e = P.tape[i];
      if (e.op != 'B' || net.kind[e.b] != snp::BN || net.prev[e.b].size() != 1 || net.prev[e.b][0] != stem) continue;
      const int bn = e.b;
      if (net.next[stem].size() != 1 || bn_from_join[i] >= 0 || !sn::conv_stem_wgrad_rows_ok(ex->L[stem].conv) ||
          ex->eff_owner[bn] != bn)
        continue;
      int64_t xo = -1, xb = 0, go = -1, gb = 0;
      for (size_t j = i; j-- > 0 && (xo < 0 || go < 0);) {
        const snp::Event& f = P.tape[j];
        if (f.op != 'A') continue;
        if (xo < 0 && f.a == snp::K_ACT && f.b == stem) xo = f.c, xb = f.d;
        if (go < 0 && f.a == snp::K_GRAD && f.b == bn) go = f.c, gb = f.d;
      }
      if (xo < 0 || go < 0) continue;
      for (size_t j = i + 1; j < T; ++j) {
        const snp::Event& f = P.tape[j];
        if (f.op == 'A' && (overlap(f.c, f.d, xo, xb) || overlap(f.c, f.d, go, gb))) break;
        if (f.op == 'B' && f.b == stem) {
          stem_bn_fuse_at[i] = 1;
          break;
        }
        if (is_compute(f.op)) break;
      }
    }
    plan_pool_stats(reassoc);
    plan_dense_chains();
    ex->elided = elide_out;
  }

  // Dense JOIN chains (see DenseStep).  A chain is kept only when, between its
  // first JOIN backward and the step that finishes an input, nothing else
  // reads, writes or frees that input's gradient buffer, and every input owns
  // its buffer (no in-place aliasing, no side roots).
  void plan_dense_chains() {
    const char* env = std::getenv("SN_FUSE_DENSE");  // =0: the per-input JOIN backward (A/B)
    if (env && env[0] == '0') return;
    const size_t T = P.tape.size();
    std::vector<size_t> jb;
    for (size_t i = 0; i < T; ++i) {
      const snp::Event& e = P.tape[i];
      if (e.op == 'B' && net.kind[e.b] == snp::JOIN && net.prev[e.b].size() >= 2 && join_to_bn[i] < 0) jb.push_back(i);
    }
    auto inputs = [&](size_t ti) {
      std::vector<int> v = net.prev[P.tape[ti].b];
      std::sort(v.begin(), v.end());
      return v;
    };
    std::vector<char> used(jb.size(), 0);
    for (size_t a = 0; a < jb.size(); ++a) {
      if (used[a]) continue;
      std::vector<size_t> chain{jb[a]}, members{a};
      std::vector<int> qs;
      std::vector<int> cur = inputs(jb[a]);
      const std::vector<int> all = cur;
      for (size_t b = a + 1; b < jb.size(); ++b) {
        if (used[b]) continue;
        const std::vector<int> nx = inputs(jb[b]);
        bool shares = false;
        for (int x : nx) shares |= std::binary_search(cur.begin(), cur.end(), x);
        if (!shares) continue;
        if (nx.size() + 1 != cur.size() || !std::includes(cur.begin(), cur.end(), nx.begin(), nx.end())) break;
        int q = -1;
        for (int x : cur)
          if (!std::binary_search(nx.begin(), nx.end(), x)) q = x;
        qs.push_back(q);
        chain.push_back(jb[b]);
        members.push_back(b);
        cur = nx;
      }
      if (chain.size() < 2) continue;
      // every input owns its gradient buffer; the JOIN's size suits the float4 kernel
      bool ok = std::adjacent_find(all.begin(), all.end()) == all.end();
      const LayerRt& jl = ex->L[P.tape[chain[0]].b];
      ok &= (static_cast<int64_t>(ex->B) * jl.per_sample) % 4 == 0;
      for (int p : all) ok &= ex->eff_owner[p] == p && !ex->side_root[p];
      if (!ok) continue;
      std::vector<char> in_chain(net.n, 0);
      for (size_t ti : chain) in_chain[P.tape[ti].b] = 1;
      // nothing touches input p's gradient between the chain's start and fin (exclusive)
      auto quiet = [&](int p, size_t fin) {
        bool allocated = false;  // the buffer exists when the chain starts (the reference allocates it for J_1)
        for (size_t j = chain[0]; j-- > 0;) {
          const snp::Event& f = P.tape[j];
          if (f.a != snp::K_GRAD || f.b != p || (f.op != 'A' && f.op != 'F')) continue;
          allocated = f.op == 'A';
          break;
        }
        if (!allocated) return false;
        for (size_t j = chain[0] + 1; j < fin; ++j) {
          const snp::Event& f = P.tape[j];
          if ((f.op == 'F' || f.op == 'A') && f.a == snp::K_GRAD && f.b == p) return false;
          if (f.op != 'B' || in_chain[f.b]) continue;
          if (f.b == p) return false;  // p's own backward reads its gradient
          for (int x : net.prev[f.b])
            if (x == p) return false;  // another consumer writes it
        }
        return true;
      };
      for (size_t k = 0; k < qs.size() && ok; ++k) ok &= quiet(qs[k], chain[k]);
      if (!ok) continue;
      int p0 = -1;
      for (int c : cur)
        if (quiet(c, chain.back())) {
          p0 = c;
          break;
        }
      if (p0 < 0) continue;
      for (int c : cur) ok &= quiet(c, chain.back());
      if (!ok) continue;
      const int id = static_cast<int>(dense_off.size());
      dense_off.push_back(0);
      for (size_t k = 0; k < chain.size(); ++k) {
        DenseStep d;
        d.chain = id;
        d.k = static_cast<int>(k);
        d.p0 = p0;
        if (k < qs.size()) {
          d.finals = {qs[k]};
        } else {
          for (int c : cur)
            if (c != p0) d.finals.push_back(c);
        }
        dense_at[chain[k]] = d;
      }
      for (size_t m : members) used[m] = 1;
    }
  }

  // BN -> ReLU -> max POOL (k3 s2 p1, saved argmax, H = 2P): pool-order BN
  // backward statistics always (with the reassociating fusions); when the BN's
  // dx goes into the stem weight gradient (stem_bn_fuse_at), the ReLU backward
  // is folded into the BN and the pool backward is the compute action right
  // before them, the pool backward is dropped and both consumers gather dy --
  // provided nothing is allocated over the pool gradient's blocks until the
  // stem weight gradient has read them.
  void plan_pool_stats(bool reassoc) {
    const size_t T = P.tape.size();
    const char* env_pg = std::getenv("SN_FUSE_POOL_GATHER");  // =0: run the pool backward (A/B test)
    const bool gather_ok = !(env_pg && env_pg[0] == '0');
    for (size_t i = 0; i < T && reassoc; ++i) {
      const snp::Event& e = P.tape[i];
      if (e.op != 'B' || net.kind[e.b] != snp::BN || bn_from_join[i] >= 0 || net.next[e.b].size() != 1) continue;
      const int bn = e.b, act = net.next[bn][0];
      if (!bn_relu_pair(act) || net.next[act].size() != 1) continue;
      const int pool = net.next[act][0];
      if (net.kind[pool] != snp::POOL || !ex->L[pool].argmax || !sn::pool_bn_stats_ok(ex->L[pool].pool, ex->L[bn].C))
        continue;
      if (ex->eff_owner[bn] != bn && ex->eff_owner[bn] != act) continue;
      bn_pool_at[i] = pool;
      if (!gather_ok || !stem_bn_fuse_at[i] || !bn_bwd_relu[i]) continue;
      const sn::ConvShape& cs = ex->L[ex->stem_layer].conv;
      if (!sn::stem_pool_gather_ok(cs, ex->L[pool].pool.P, ex->L[pool].pool.Q)) continue;
      // the compute actions right before: [ReLU backward (folded)], pool backward
      size_t ip = SIZE_MAX;
      for (size_t j = i; j-- > 0;) {
        const snp::Event& f = P.tape[j];
        if (!is_compute(f.op)) continue;
        if (f.op == 'B' && f.b == act && act_bwd_skip[j]) continue;
        if (f.op == 'B' && f.b == pool) ip = j;
        break;
      }
      if (ip == SIZE_MAX) continue;
      const int po = ex->eff_owner[pool];
      if (po < 0) continue;
      size_t is = SIZE_MAX;  // the stem backward
      for (size_t j = i + 1; j < T; ++j)
        if (P.tape[j].op == 'B') {
          if (P.tape[j].b == ex->stem_layer) is = j;
          break;
        }
      if (is == SIZE_MAX) continue;
      bool ok = true;
      if (!ex->side_root[po]) {
        int64_t go = -1, gb = 0;
        for (size_t j = ip; j-- > 0;) {
          const snp::Event& f = P.tape[j];
          if (f.op == 'A' && f.a == snp::K_GRAD && f.b == po) {
            go = f.c, gb = f.d;
            break;
          }
        }
        if (go < 0) continue;
        for (size_t j = ip + 1; j < is && ok; ++j) {
          const snp::Event& f = P.tape[j];
          if (f.op == 'A' && overlap(f.c, f.d, go, gb)) ok = false;
        }
      }
      if (!ok) continue;
      pool_gather_at[i] = 1;
      pool_skip_at[ip] = static_cast<int>(i);
    }
  }

  // Data-parallel bucket all-reduce + update on s5, right after the backward
  // step that completes the bucket: s5 waits for everything s0 issued (BN /
  // FC / bias gradients) and for the side-stream weight gradients of the
  // bucket's CONV layers.  Each layer's parameters are not read again in
  // this iteration after its backward step (its replays precede it), so the
  // bucket's update can run while the backward continues.
  void dp_after_backward(int lid) {
    while (next_bucket < ex->buckets.size() && ex->buckets[next_bucket].after_layer == lid) {
      const sn_exec::Bucket& b = ex->buckets[next_bucket++];
      std::vector<cudaEvent_t> waits;
      for (int l : b.layers) {
        auto it = wgrad_done.find(l);
        if (it != wgrad_done.end()) waits.push_back(it->second);
      }
      cudaEvent_t e0 = ex->new_event();
      sn_exec* e = ex;
      const int64_t lo = b.lo, n = b.hi - b.lo;
      const float lr = ex->opt.lr, scale = ex->opt.grad_scale;
      push([=] {
        std::string err;
        const sndp::Nccl* nc = sndp::nccl(&err);
        if (!nc) xfail(SN_EK_CUDA, err);
        ck(cudaEventRecord(e0, e->s0), "record");
        ck(cudaStreamWaitEvent(e->s5, e0, 0), "wait");
        for (cudaEvent_t w : waits) ck(cudaStreamWaitEvent(e->s5, w, 0), "wait");
        const ncclResult_t r = nc->AllReduce(e->grads + lo, e->grads + lo, static_cast<size_t>(n), ncclFloat32,
                                             ncclSum, static_cast<ncclComm_t>(e->opt.dp_comm), e->s5);
        if (r != ncclSuccess) xfail(SN_EK_CUDA, std::string("ncclAllReduce: ") + nc->GetErrorString(r));
        ck(sn::sgd_update_flagged(e->params + lo, e->grads + lo, n, lr, scale, e->update_flag, e->s5), "sgd");
      }, 2);
      used_s5 = true;
    }
  }

  // split-K partial floats of a CONV weight gradient
  int64_t wgrad_partial_floats(int lid) const {
    const LayerRt& l = ex->L[lid];
    if (lid == ex->stem_layer) return sn::stem_wgrad_partial_floats(l.conv);
    return static_cast<int64_t>(l.wgrad_splits) * l.conv.R * l.conv.S * l.conv.C * l.conv.K;
  }

  // The wgrad scratch outside the pool holds only the partials of the CONV
  // backward steps whose granted workspace (the planner's selection,
  // reference simulator.py:624-654) is too small for them.
  void size_wgrad_scratch() {
    std::unordered_map<int64_t, int64_t> ws_blocks;  // ws key id -> blocks of its latest allocation
    int64_t outside = 0;
    for (const auto& ev : P.tape) {
      if (ev.op == 'A' && ev.a == snp::K_WS) ws_blocks[ev.b] = ev.d;
      if (ev.op != 'B' || net.kind[ev.b] != snp::CONV) continue;
      int64_t have = 0;
      if (ev.d >= 0) {
        auto it = ws_blocks.find(ev.d);
        if (it != ws_blocks.end()) have = it->second * snp::kBlockBytes / static_cast<int64_t>(sizeof(float));
      }
      const int64_t need = wgrad_partial_floats(ev.b);
      if (have < need) outside = std::max(outside, need);
    }
    ex->wgrad_partial_outside = outside;
    ex->dmalloc(&ex->partial_w, std::max<int64_t>(outside, 64) * 4, sn_exec::M_WGRAD, "cudaMalloc(partial_w)");
  }

  // The iteration no longer reads `images` after this point: the host input
  // pipeline may copy the next batch in (an external record inside a graph).
  void inputs_consumed() {
    cur_layer = -1, cur_type = 3;
    cudaEvent_t ev = ex->inputs_free_ev;
    cudaStream_t st = ex->s0;
    push([=] { ck(record_timer(ev, st), "record inputs free"); }, 0);
  }

  // DATA layer: lay the user's images out the way the consumers read them.
  void prepare_inputs() {
    const LayerRt& d = ex->L[data_id];
    if (ex->data_buf == ex->images) return;
    cur_layer = data_id, cur_type = 0;
    const float* raw = ex->images;
    float* out = ex->data_buf;
    cudaStream_t st = ex->s0;
    if (ex->stem_layer >= 0) {
      const sn::ConvShape cs = ex->L[ex->stem_layer].conv;
      const int H = d.H, W = d.W, Cr = d.C_raw;
      push([=] { ck(sn::stem_pad_input(cs, H, W, Cr, cs.pad, raw, out, st), "stem_pad_input"); }, 1);
    } else {
      const int Cr = d.C_raw, Cs = d.C;
      const int64_t pix = static_cast<int64_t>(ex->B) * d.H * d.W;
      push([=] { ck(sn::pad_channels(raw, Cr, out, Cs, pix, st), "pad_channels"); }, 1);
    }
  }

  // The weights do not change within a step: every CONV's dgrad weight
  // transform (flipped / transposed filter, sub-pixel blocks) runs at the start
  // of the iteration as ONE batched launch on the side stream s3, overlapping
  // the forward, into per-layer buffers outside the pool (sn_exec_memory:
  // "dgrad weights") -- instead of one short launch per layer on the backward's
  // dgrad chain (ResNet-2534g b16: 842 launches, ~2.4 us each in the graph).
  static constexpr int kPrepMinJobs = 64;
  void prep_dgrad_weights() {
    const char* env = std::getenv("SN_DGRAD_PREP");  // A/B: 0 = never, 1 = always (tests)
    if (env && env[0] == '0') return;
    std::vector<sn::DgradPrepJob> jobs;
    for (int i = 0; i < net.n; ++i) {
      LayerRt& l = ex->L[i];
      if (l.kind != snp::CONV || i == ex->stem_layer || net.prev[i].empty()) continue;
      if (ex->eff_owner[net.prev[i][0]] < 0) continue;  // no input gradient: no dgrad
      sn::KnobScope ks(l.kd);
      sn::DgradPrepJob job{};
      if (!sn::conv_dgrad_prep_job(l.conv, ex->params + l.w_off, nullptr, &job)) continue;
      ex->dmalloc(&l.wt_pre, sn::conv_dgrad_scratch_floats(l.conv) * 4, sn_exec::M_PARAMS, "cudaMalloc(dgrad weights)");
      job.wt = l.wt_pre;
      jobs.push_back(job);
    }
    // Only deep nets gain: the batched launch at the step start contends with
    // the first forward kernels (ResNet-50g b256, 13 jobs: 9.03 -> 9.11 ms),
    // while ResNet-2534g b16 (842 jobs) saves 82.3 -> 80.5 ms.
    if (static_cast<int>(jobs.size()) < kPrepMinJobs && !(env && env[0] == '1')) {
      for (int i = 0; i < net.n; ++i)
        if (ex->L[i].wt_pre) {
          cudaFree(ex->L[i].wt_pre);
          ex->mem[sn_exec::M_PARAMS] -= sn::conv_dgrad_scratch_floats(ex->L[i].conv) * 4;
          ex->L[i].wt_pre = nullptr;
        }
      return;
    }
    ex->dmalloc(&ex->prep_jobs, static_cast<int64_t>(jobs.size() * sizeof(sn::DgradPrepJob)), sn_exec::M_OTHER,
                "cudaMalloc(dgrad weight jobs)");
    sn::DgradPrepJob* d_jobs = ex->prep_jobs;
    ck(cudaMemcpy(d_jobs, jobs.data(), jobs.size() * sizeof(sn::DgradPrepJob), cudaMemcpyHostToDevice),
       "memcpy(dgrad weight jobs)");
    cur_layer = -1, cur_type = 3;
    wt_ready = ex->new_event();
    cudaEvent_t go = ex->new_event(), ready = wt_ready;  // locals: the action outlives this Compiler
    used_s3 = true;
    sn_exec* e = ex;
    cudaStream_t s0 = ex->s0, s3 = ex->s3;
    const int nj = static_cast<int>(jobs.size());
    push([=] {
      const cudaStream_t sw = e->serial ? s0 : s3;
      ck(cudaEventRecord(go, s0), "record");
      ck(cudaStreamWaitEvent(sw, go, 0), "wait");
      ck(sn::conv_dgrad_prep_batch(d_jobs, nj, sw), "conv_dgrad_prep_batch");
      ck(cudaEventRecord(ready, sw), "record");
    }, 1);
  }

  void compile() {
    for (int i = 0; i < net.n; ++i)
      if (ex->side_root[i]) fresh[i] = true;  // side gradient buffers: the first write overwrites
    plan_fusions();
    size_wgrad_scratch();
    prep_dgrad_weights();
    prepare_inputs();
    const bool images_in_place = ex->data_buf == ex->images;
    if (!images_in_place) inputs_consumed();
    for (size_t ti = 0; ti < P.tape.size(); ++ti) {
      const snp::Event& ev = P.tape[ti];
      cur_ti = ti;
      fuse_next = fuse_at[ti] != 0;
      fused_bn = fused_into[ti];
      conv_stats_now = conv_stats_at[ti] != 0;
      bn_tiles_now = bn_tiles_at[ti] != 0;
      bn_bias_now = bn_bias_at[ti] != 0;
      bwd_skip = act_bwd_skip[ti] != 0;
      bwd_relu = bn_bwd_relu[ti] != 0;
      switch (ev.op) {
        case 'A': on_alloc(ev); break;
        case 'F': on_free(ev); break;
        case 'C':
          cur_layer = ev.b, cur_type = 0;
          forward(ev.b, false);
          break;
        case 'R':
          cur_layer = ev.b, cur_type = 1;
          forward(ev.b, true);
          break;
        case 'B':
          cur_layer = ev.b, cur_type = 2;
          backward(ev.b);
          if (ex->dp()) {
            cur_layer = -1, cur_type = 3;
            dp_after_backward(ev.b);
          }
          break;
        case 'O': on_copy_out(ev.b); break;
        case 'P':
        case 'D': on_fetch(ev.b); break;
        default: break;  // cache bookkeeping and step markers need no device work
      }
    }
    // Join the copy streams back into the compute stream (no layer: the
    // trailing actions must not inherit the last tape event's layer / type).
    cur_layer = -1, cur_type = 3;
    cudaStream_t s0 = ex->s0;
    if (used_s1) {
      cudaEvent_t j = ex->new_event();
      cudaStream_t s1 = ex->s1;
      push([=] {
        ck(cudaEventRecord(j, s1), "record");
        ck(cudaStreamWaitEvent(s0, j, 0), "wait");
      }, 0);
    }
    if (used_s2) {
      cudaEvent_t j = ex->new_event();
      cudaStream_t s2 = ex->s2;
      push([=] {
        ck(cudaEventRecord(j, s2), "record");
        ck(cudaStreamWaitEvent(s0, j, 0), "wait");
      }, 0);
    }
    if (used_s3) {
      cudaEvent_t j = ex->new_event();
      cudaStream_t s3 = ex->s3;
      sn_exec* e = ex;
      push([=] {
        if (e->serial) return;  // profiling: the weight gradients ran on s0
        ck(cudaEventRecord(j, s3), "record");
        ck(cudaStreamWaitEvent(s0, j, 0), "wait");
      }, 0);
    }
    if (used_s5) {
      cudaEvent_t j = ex->new_event();
      cudaStream_t s5 = ex->s5;
      push([=] {
        ck(cudaEventRecord(j, s5), "record");
        ck(cudaStreamWaitEvent(s0, j, 0), "wait");
      }, 0);
    }
    if (ex->dp() && next_bucket != ex->buckets.size()) xfail(SN_EK_INTERNAL, "data-parallel buckets not all issued");
    if (images_in_place) inputs_consumed();
    uint32_t* it = ex->iteration;
    push([=] { ck(sn::bump_iteration(it, s0), "bump"); }, 1);
    ex->final_keys = where;
    for (const Action& a : ex->prog) ex->kernels_per_step += a.kernels;
  }
};

// The kernels' numeric mode is process-wide (sn::set_precision); every entry
// point that launches or captures this executor's work sets its own.
struct PrecisionScope {
  int saved;
  explicit PrecisionScope(const sn_exec* ex) : saved(sn::precision()) { sn::set_precision(ex->opt.precision); }
  ~PrecisionScope() { sn::set_precision(saved); }
};

void run_program(sn_exec* ex) {
  for (const Action& a : ex->prog) a.fn();
}

void ensure_graph(sn_exec* ex) {
  if (ex->graph_ready) return;
  ck(cudaStreamBeginCapture(ex->s0, cudaStreamCaptureModeThreadLocal), "BeginCapture");
  try {
    run_program(ex);
  } catch (...) {
    cudaGraph_t g;
    cudaStreamEndCapture(ex->s0, &g);
    if (g) cudaGraphDestroy(g);
    throw;
  }
  ck(cudaStreamEndCapture(ex->s0, &ex->graph), "EndCapture");
  ck(cudaGraphInstantiate(&ex->gexec, ex->graph, 0), "GraphInstantiate");
  // exact launch count of one iteration: the kernel nodes of the graph
  size_t nn = 0;
  ck(cudaGraphGetNodes(ex->graph, nullptr, &nn), "GraphGetNodes");
  std::vector<cudaGraphNode_t> nodes(nn);
  ck(cudaGraphGetNodes(ex->graph, nodes.data(), &nn), "GraphGetNodes");
  int64_t kern = 0;
  for (cudaGraphNode_t nd : nodes) {
    cudaGraphNodeType t;
    ck(cudaGraphNodeGetType(nd, &t), "GraphNodeGetType");
    kern += t == cudaGraphNodeTypeKernel;
  }
  ex->kernels_per_step = kern;
  ex->graph_ready = true;
}

template <class F>
int xguard(F&& f) {
  try {
    f();
    g_xerr_kind = SN_EK_NONE;
    return SN_OK;
  } catch (const ExecError& e) {
    return xset(e.kind, e.msg);
  } catch (const snp::PlanError& e) {
    return xset(e.kind, e.what());
  } catch (const std::exception& e) {
    return xset(SN_EK_INTERNAL, e.what());
  }
}

void destroy(sn_exec* ex) {
  if (!ex) return;
  if (ex->gexec) cudaGraphExecDestroy(ex->gexec);
  if (ex->graph) cudaGraphDestroy(ex->graph);
  for (cudaEvent_t e : ex->events) cudaEventDestroy(e);
  if (ex->t_begin) cudaEventDestroy(ex->t_begin);
  if (ex->t_end) cudaEventDestroy(ex->t_end);
  if (ex->staged_ev) cudaEventDestroy(ex->staged_ev);
  if (ex->consumed_ev) cudaEventDestroy(ex->consumed_ev);
  if (ex->inputs_free_ev) cudaEventDestroy(ex->inputs_free_ev);
  for (cudaEvent_t e : ex->loss_ev)
    if (e) cudaEventDestroy(e);
  if (ex->loss_pinned) cudaFreeHost(ex->loss_pinned);
  if (ex->s4) cudaStreamDestroy(ex->s4);
  if (!ex->opt.stash)
    for (auto& kv : ex->stash)
      if (kv.second) cudaFreeHost(kv.second);
  for (auto& pd : ex->peer_stash) {
    cudaSetDevice(pd.second);
    cudaFree(pd.first);
  }
  if (!ex->peer_stash.empty()) cudaSetDevice(ex->device);
  if (ex->data_buf && ex->data_buf != ex->images) cudaFree(ex->data_buf);
  void* bufs[] = {ex->arena, ex->params, ex->grads, ex->state, ex->images, ex->labels, ex->loss_rows, ex->loss,
                  ex->iteration, ex->wt_scratch, ex->partial, ex->red, ex->tstats, ex->pool_scratch,
                  ex->partial_w, ex->red_w, ex->wt_w, ex->labels_stage,
                  const_cast<float**>(ex->ptr_table), ex->marker, ex->update_flag};
  for (void* b : bufs)
    if (b) cudaFree(b);
  for (auto& l : ex->L) {
    if (l.argmax) cudaFree(l.argmax);
    if (l.wt_pre) cudaFree(l.wt_pre);
  }
  if (ex->prep_jobs) cudaFree(ex->prep_jobs);
  for (auto& kv : ex->side) cudaFree(kv.second);
  if (ex->s0) cudaStreamDestroy(ex->s0);
  if (ex->s1) cudaStreamDestroy(ex->s1);
  if (ex->s2) cudaStreamDestroy(ex->s2);
  if (ex->s3) cudaStreamDestroy(ex->s3);
  if (ex->s5) cudaStreamDestroy(ex->s5);
  delete ex;
}

}  // namespace

extern "C" {

const char* sn_exec_last_error(void) { return g_xerr.c_str(); }
int sn_exec_last_error_kind(void) { return g_xerr_kind; }

int sn_exec_create(const sn_plan* plan, const sn_net_desc* /*net*/, const sn_layer_numerics* numerics,
                   const sn_exec_options* opts, sn_exec** out) {
  if (!plan || !opts || !out) return xset(SN_EK_INTERNAL, "null argument");
  *out = nullptr;
  sn_exec* ex = new sn_exec;
  const int rc = xguard([&] {
    ex->plan = plan;
    ex->net = &plan->plan.net;
    ex->opt = *opts;
    if (ex->opt.precision != 0 && ex->opt.precision != 1) xfail(SN_EK_CONFIG, "precision must be 0 (tf32) or 1 (fp32)");
    if (ex->opt.stash != 0 && ex->opt.stash != 1) xfail(SN_EK_CONFIG, "stash must be 0 (pinned host) or 1 (device)");
    PrecisionScope prec(ex);
    ex->device = opts->device;
    ex->B = static_cast<int>(plan->plan.cost_cfg.batch);
    if (plan->plan.cost_cfg.dtype_bytes != 4)
      xfail(SN_EK_UNSUPPORTED, "the executor computes in fp32: CostConfig.dtype_bytes must be 4");
    ck(cudaSetDevice(ex->device), "cudaSetDevice");
    ck(cudaStreamCreateWithFlags(&ex->s0, cudaStreamNonBlocking), "stream");
    ck(cudaStreamCreateWithFlags(&ex->s1, cudaStreamNonBlocking), "stream");
    ck(cudaStreamCreateWithFlags(&ex->s2, cudaStreamNonBlocking), "stream");
    ck(cudaStreamCreateWithFlags(&ex->s3, cudaStreamNonBlocking), "stream");
    ck(cudaEventCreate(&ex->t_begin), "event");
    ck(cudaEventCreate(&ex->t_end), "event");
    ck(cudaEventCreateWithFlags(&ex->inputs_free_ev, cudaEventDisableTiming), "event");
    ck(cudaEventRecord(ex->inputs_free_ev, ex->s0), "record");
    setup_layers(ex, numerics);
    if (ex->opt.autotune) autotune(ex);
    alloc_device(ex);
    if (ex->dp()) {
      if (ex->opt.dp_world < 1 || ex->opt.dp_rank < 0 || ex->opt.dp_rank >= ex->opt.dp_world)
        xfail(SN_EK_CONFIG, "bad data-parallel world / rank");
      plan_buckets(ex, ex->opt.dp_bucket_bytes > 0 ? ex->opt.dp_bucket_bytes : (8ll << 20));
      ck(cudaStreamCreateWithFlags(&ex->s5, cudaStreamNonBlocking), "stream");
      ex->dmalloc(&ex->update_flag, 4, sn_exec::M_OTHER, "cudaMalloc(update flag)");
      ck(cudaMemset(ex->update_flag, 0, 4), "memset(flag)");
      // one eager all-reduce of every bucket (the gradients are still zero) so
      // NCCL sets up its connections outside the CUDA-graph capture
      std::string nerr;
      const sndp::Nccl* nc = sndp::nccl(&nerr);
      if (!nc) xfail(SN_EK_CUDA, nerr);
      for (const auto& b : ex->buckets) {
        const ncclResult_t r = nc->AllReduce(ex->grads + b.lo, ex->grads + b.lo, static_cast<size_t>(b.hi - b.lo),
                                             ncclFloat32, ncclSum, static_cast<ncclComm_t>(ex->opt.dp_comm), ex->s5);
        if (r != ncclSuccess) xfail(SN_EK_CUDA, std::string("ncclAllReduce (warm-up): ") + nc->GetErrorString(r));
      }
      ck(cudaStreamSynchronize(ex->s5), "sync(warm-up)");
    }
    Compiler comp(ex);
    comp.compile();
    const size_t nptr = std::max<size_t>(1, ex->ptr_host.size());
    ex->dmalloc(&ex->ptr_table, static_cast<int64_t>(nptr * sizeof(float*)), sn_exec::M_OTHER, "cudaMalloc(ptr_table)");
    if (!ex->ptr_host.empty())
      ck(cudaMemcpy(ex->ptr_table, ex->ptr_host.data(), ex->ptr_host.size() * sizeof(float*), cudaMemcpyHostToDevice),
         "memcpy(ptr_table)");
    ck(cudaDeviceSynchronize(), "sync");
  });
  if (rc != SN_OK) {
    destroy(ex);
    return rc;
  }
  *out = ex;
  return SN_OK;
}

void sn_exec_destroy(sn_exec* ex) { destroy(ex); }

int sn_exec_params(sn_exec* ex, float** params, float** grads, int64_t* n_floats) {
  if (!ex) return xset(SN_EK_INTERNAL, "null argument");
  if (params) *params = ex->params;
  if (grads) *grads = ex->grads;
  if (n_floats) *n_floats = ex->n_params;
  return SN_OK;
}

int sn_exec_param_slice(sn_exec* ex, int32_t layer, int64_t* w_off, int64_t* w_n, int64_t* b_off, int64_t* b_n) {
  if (!ex || layer < 0 || layer >= static_cast<int>(ex->L.size())) return xset(SN_EK_INTERNAL, "bad layer");
  const LayerRt& l = ex->L[layer];
  if (w_off) *w_off = l.w_off;
  if (w_n) *w_n = l.w_n;
  if (b_off) *b_off = l.b_off;
  if (b_n) *b_n = l.b_n;
  return SN_OK;
}

// Entry points outside the host input pipeline drop a batch it staged for
// the next pipelined call (its image copy into `images` finishes first).
void drop_stage(sn_exec* ex) {
  if (!ex->staged_src) return;
  ck(cudaStreamSynchronize(ex->s4), "sync staged input");
  ex->staged_src = nullptr;
}

int sn_exec_inputs(sn_exec* ex, float** images, int32_t** labels, int64_t* image_floats) {
  if (!ex) return xset(SN_EK_INTERNAL, "null argument");
  if (const int rc = xguard([&] { drop_stage(ex); })) return rc;
  if (images) *images = ex->images;
  if (labels) *labels = ex->labels;
  if (image_floats) *image_floats = ex->image_floats;
  return SN_OK;
}

void* sn_exec_stream(sn_exec* ex) { return ex ? ex->s0 : nullptr; }

int sn_exec_step(sn_exec* ex, int32_t update, float* loss_host, sn_step_timing* timing) {
  if (!ex) return xset(SN_EK_INTERNAL, "null argument");
  return xguard([&] {
    ck(cudaSetDevice(ex->device), "cudaSetDevice");
    drop_stage(ex);
    PrecisionScope prec(ex);
    if (ex->opt.use_graph) ensure_graph(ex);
    ck(cudaEventRecord(ex->t_begin, ex->s0), "record");
    if (ex->dp()) ck(cudaMemsetAsync(ex->update_flag, update ? 1 : 0, 4, ex->s0), "update flag");
    if (ex->opt.use_graph)
      ck(cudaGraphLaunch(ex->gexec, ex->s0), "GraphLaunch");
    else
      run_program(ex);
    if (update && !ex->dp())
      ck(sn::sgd_update(ex->params, ex->grads, ex->n_params, ex->opt.lr, ex->opt.grad_scale, ex->s0), "sgd");
    ck(cudaEventRecord(ex->t_end, ex->s0), "record");
    if (loss_host) ck(cudaMemcpyAsync(loss_host, ex->loss, sizeof(float), cudaMemcpyDeviceToHost, ex->s0), "loss D2H");
    ck(cudaStreamSynchronize(ex->s0), "sync");
    if (timing) {
      float ms = 0.f;
      ck(cudaEventElapsedTime(&ms, ex->t_begin, ex->t_end), "elapsed");
      timing->step_ms = ms;
      timing->h2d_ms = timing->d2h_ms = 0.f;
      timing->kernels = ex->kernels_per_step + (update ? 1 : 0);
      timing->d2h_bytes = ex->d2h_bytes;
      timing->h2d_bytes = ex->h2d_bytes;
      timing->arena_high_water = ex->plan->plan.report.pool_high_water_bytes;
    }
  });
}

int sn_exec_step_host(sn_exec* ex, const float* images_host, const int32_t* labels_host, int32_t update,
                      float* loss_host, sn_step_timing* timing) {
  if (!ex) return xset(SN_EK_INTERNAL, "null argument");
  const int rc = xguard([&] {
    ck(cudaSetDevice(ex->device), "cudaSetDevice");
    PrecisionScope prec(ex);
    drop_stage(ex);
    if (ex->opt.use_graph) ensure_graph(ex);
    ck(cudaEventRecord(ex->t_begin, ex->s0), "record");
    ck(cudaMemcpyAsync(ex->images, images_host, ex->image_floats * sizeof(float), cudaMemcpyHostToDevice, ex->s0),
       "images H2D");
    ck(cudaMemcpyAsync(ex->labels, labels_host, ex->B * sizeof(int32_t), cudaMemcpyHostToDevice, ex->s0),
       "labels H2D");
    if (ex->dp()) ck(cudaMemsetAsync(ex->update_flag, update ? 1 : 0, 4, ex->s0), "update flag");
    if (ex->opt.use_graph)
      ck(cudaGraphLaunch(ex->gexec, ex->s0), "GraphLaunch");
    else
      run_program(ex);
    if (update && !ex->dp())
      ck(sn::sgd_update(ex->params, ex->grads, ex->n_params, ex->opt.lr, ex->opt.grad_scale, ex->s0), "sgd");
    ck(cudaMemcpyAsync(loss_host, ex->loss, sizeof(float), cudaMemcpyDeviceToHost, ex->s0), "loss D2H");
    ck(cudaEventRecord(ex->t_end, ex->s0), "record");
    ck(cudaStreamSynchronize(ex->s0), "sync");
    if (timing) {
      float ms = 0.f;
      ck(cudaEventElapsedTime(&ms, ex->t_begin, ex->t_end), "elapsed");
      timing->step_ms = ms;
      timing->kernels = ex->kernels_per_step + (update ? 1 : 0);
      timing->d2h_bytes = ex->d2h_bytes;
      timing->h2d_bytes = ex->h2d_bytes;
      timing->arena_high_water = ex->plan->plan.report.pool_high_water_bytes;
    }
  });
  return rc;
}

namespace {

void ensure_input_pipeline(sn_exec* ex) {
  if (ex->s4) return;
  ck(cudaStreamCreateWithFlags(&ex->s4, cudaStreamNonBlocking), "stream");
  ex->dmalloc(&ex->labels_stage, static_cast<int64_t>(ex->B * sizeof(int32_t)), sn_exec::M_INPUT,
              "cudaMalloc(labels_stage)");
  ck(cudaEventCreateWithFlags(&ex->staged_ev, cudaEventDisableTiming), "event");
  ck(cudaEventCreateWithFlags(&ex->consumed_ev, cudaEventDisableTiming), "event");
  ck(cudaEventRecord(ex->consumed_ev, ex->s0), "record");
  ck(cudaHostAlloc(reinterpret_cast<void**>(&ex->loss_pinned), 2 * sizeof(float), cudaHostAllocDefault),
     "cudaHostAlloc(loss)");
  for (auto& e : ex->loss_ev) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
}

// Copy a host batch in on s4: images straight into `images` after the last
// launched iteration consumed its own, labels into the staging buffer after
// the last iteration's copy of it.
void stage_batch(sn_exec* ex, const float* img, const int32_t* lab) {
  ck(cudaStreamWaitEvent(ex->s4, ex->inputs_free_ev, 0), "wait");
  ck(cudaMemcpyAsync(ex->images, img, ex->image_floats * sizeof(float), cudaMemcpyHostToDevice, ex->s4),
     "images H2D");
  ck(cudaStreamWaitEvent(ex->s4, ex->consumed_ev, 0), "wait");
  ck(cudaMemcpyAsync(ex->labels_stage, lab, ex->B * sizeof(int32_t), cudaMemcpyHostToDevice, ex->s4), "labels H2D");
  ck(cudaEventRecord(ex->staged_ev, ex->s4), "record");
  ex->staged_src = img;
}

// One iteration on the staged batch (s0), plus the SGD update.
void launch_staged(sn_exec* ex, int32_t update) {
  ck(cudaStreamWaitEvent(ex->s0, ex->staged_ev, 0), "wait");
  ck(cudaMemcpyAsync(ex->labels, ex->labels_stage, ex->B * sizeof(int32_t), cudaMemcpyDeviceToDevice, ex->s0),
     "labels D2D");
  ck(cudaEventRecord(ex->consumed_ev, ex->s0), "record");
  ex->staged_src = nullptr;
  if (ex->dp()) ck(cudaMemsetAsync(ex->update_flag, update ? 1 : 0, 4, ex->s0), "update flag");
  if (ex->opt.use_graph)
    ck(cudaGraphLaunch(ex->gexec, ex->s0), "GraphLaunch");
  else
    run_program(ex);
  if (update && !ex->dp())
    ck(sn::sgd_update(ex->params, ex->grads, ex->n_params, ex->opt.lr, ex->opt.grad_scale, ex->s0), "sgd");
}

void fill_timing(sn_exec* ex, int32_t update, float ms, sn_step_timing* timing) {
  if (!timing) return;
  timing->step_ms = ms;
  timing->kernels = ex->kernels_per_step + (update ? 1 : 0);
  timing->d2h_bytes = ex->d2h_bytes;
  timing->h2d_bytes = ex->h2d_bytes;
  timing->arena_high_water = ex->plan->plan.report.pool_high_water_bytes;
}

}  // namespace

int sn_exec_step_host_pipelined(sn_exec* ex, const float* images_host, const int32_t* labels_host,
                                const float* next_images_host, const int32_t* next_labels_host, int32_t update,
                                float* loss_host, sn_step_timing* timing) {
  if (!ex || !images_host || !labels_host) return xset(SN_EK_INTERNAL, "null argument");
  const int rc = xguard([&] {
    ck(cudaSetDevice(ex->device), "cudaSetDevice");
    PrecisionScope prec(ex);
    if (ex->opt.use_graph) ensure_graph(ex);
    ensure_input_pipeline(ex);
    ck(cudaEventRecord(ex->t_begin, ex->s0), "record");
    if (ex->staged_src != images_host) stage_batch(ex, images_host, labels_host);  // first call of a run
    launch_staged(ex, update);
    // stage the next batch now (it waits for this iteration's DATA layer)
    if (next_images_host && next_labels_host) stage_batch(ex, next_images_host, next_labels_host);
    ck(cudaMemcpyAsync(loss_host, ex->loss, sizeof(float), cudaMemcpyDeviceToHost, ex->s0), "loss D2H");
    ck(cudaEventRecord(ex->t_end, ex->s0), "record");
    ck(cudaStreamSynchronize(ex->s0), "sync");
    float ms = 0.f;
    if (timing) ck(cudaEventElapsedTime(&ms, ex->t_begin, ex->t_end), "elapsed");
    fill_timing(ex, update, ms, timing);
  });
  return rc;
}

int sn_exec_train_host(sn_exec* ex, int32_t n, const float* const* images_host, const int32_t* const* labels_host,
                       int32_t update, float* losses, sn_step_timing* timing) {
  if (!ex || n < 0 || (n > 0 && (!images_host || !labels_host || !losses))) return xset(SN_EK_INTERNAL, "null argument");
  if (n == 0) return SN_OK;
  const int rc = xguard([&] {
    ck(cudaSetDevice(ex->device), "cudaSetDevice");
    PrecisionScope prec(ex);
    if (ex->opt.use_graph) ensure_graph(ex);
    ensure_input_pipeline(ex);
    for (int i = 0; i < n; ++i)
      if (!images_host[i] || !labels_host[i]) xfail(SN_EK_INTERNAL, "null batch pointer");
    ck(cudaEventRecord(ex->t_begin, ex->s0), "record");
    if (ex->staged_src != images_host[0]) stage_batch(ex, images_host[0], labels_host[0]);
    for (int k = 0; k < n; ++k) {
      launch_staged(ex, update);
      if (k + 1 < n) stage_batch(ex, images_host[k + 1], labels_host[k + 1]);
      // step k's loss lands in a pinned slot; the host reads step k-1's while
      // step k runs, so the device never waits for the host between steps
      ck(cudaMemcpyAsync(ex->loss_pinned + (k & 1), ex->loss, sizeof(float), cudaMemcpyDeviceToHost, ex->s0),
         "loss D2H");
      ck(cudaEventRecord(ex->loss_ev[k & 1], ex->s0), "record");
      if (k >= 1) {
        ck(cudaEventSynchronize(ex->loss_ev[(k - 1) & 1]), "sync loss");
        losses[k - 1] = ex->loss_pinned[(k - 1) & 1];
      }
    }
    ck(cudaEventRecord(ex->t_end, ex->s0), "record");
    ck(cudaEventSynchronize(ex->loss_ev[(n - 1) & 1]), "sync loss");
    losses[n - 1] = ex->loss_pinned[(n - 1) & 1];
    ck(cudaStreamSynchronize(ex->s0), "sync");
    float ms = 0.f;
    if (timing) ck(cudaEventElapsedTime(&ms, ex->t_begin, ex->t_end), "elapsed");
    fill_timing(ex, update, ms / n, timing);
  });
  return rc;
}

int sn_exec_profile(sn_exec* ex, float* action_ms, int32_t* action_layer, int32_t* action_type, size_t cap,
                    size_t* n) {
  if (!ex || !n) return xset(SN_EK_INTERNAL, "null argument");
  *n = ex->prog.size();
  if (!action_ms) return SN_OK;
  if (cap < ex->prog.size()) return xset(SN_EK_INTERNAL, "output buffer too small");
  return xguard([&] {
    ck(cudaSetDevice(ex->device), "cudaSetDevice");
    PrecisionScope prec(ex);
    std::vector<cudaEvent_t> ev(ex->prog.size() + 1);
    for (auto& e : ev) ck(cudaEventCreate(&e), "event");
    ex->serial = true;
    struct Restore {
      sn_exec* e;
      ~Restore() { e->serial = false; }
    } restore{ex};
    if (ex->dp()) ck(cudaMemsetAsync(ex->update_flag, 0, 4, ex->s0), "update flag");
    ck(cudaEventRecord(ev[0], ex->s0), "record");
    for (size_t i = 0; i < ex->prog.size(); ++i) {
      ex->prog[i].fn();
      ck(cudaEventRecord(ev[i + 1], ex->s0), "record");
    }
    ck(cudaStreamSynchronize(ex->s0), "sync");
    ck(cudaDeviceSynchronize(), "sync");
    for (size_t i = 0; i < ex->prog.size(); ++i) {
      float ms = 0.f;
      ck(cudaEventElapsedTime(&ms, ev[i], ev[i + 1]), "elapsed");
      action_ms[i] = ms;
      if (action_layer) action_layer[i] = ex->prog[i].layer;
      if (action_type) action_type[i] = ex->prog[i].type;
    }
    for (auto& e : ev) cudaEventDestroy(e);
  });
}

namespace {
// Holds the stream for `ns` nanoseconds of GPU time: queued behind it, the
// replayed launches and their events run back to back instead of at the pace
// the host issues them.
__global__ void hold_stream_kernel(uint64_t ns) {
  uint64_t t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  } while (t - t0 < ns);
}

// One serial iteration captured with a memset marker (value = action index)
// before every action: the graph's nodes in issue order, each tagged with the
// action that issued it (markers and external timer events excluded).
struct Census {
  cudaGraph_t graph = nullptr;
  std::vector<std::pair<cudaGraphNode_t, int>> nodes;  // (node, action)
  ~Census() {
    if (graph) cudaGraphDestroy(graph);
  }
};

void capture_census(sn_exec* ex, Census& c) {
  if (!ex->marker) ex->dmalloc(&ex->marker, 4, sn_exec::M_OTHER, "cudaMalloc(marker)");
  ex->serial = true;
  struct Restore {
    sn_exec* e;
    ~Restore() { e->serial = false; }
  } restore{ex};
  ck(cudaStreamBeginCapture(ex->s0, cudaStreamCaptureModeThreadLocal), "BeginCapture");
  try {
    for (size_t i = 0; i < ex->prog.size(); ++i) {
      ck(cudaMemsetAsync(ex->marker, static_cast<int>(i & 0xff), sizeof(int32_t), ex->s0), "marker");
      ex->prog[i].fn();
    }
  } catch (...) {
    cudaGraph_t g = nullptr;
    cudaStreamEndCapture(ex->s0, &g);
    if (g) cudaGraphDestroy(g);
    throw;
  }
  ck(cudaStreamEndCapture(ex->s0, &c.graph), "EndCapture");
  size_t nn = 0;
  ck(cudaGraphGetNodes(c.graph, nullptr, &nn), "GraphGetNodes");
  std::vector<cudaGraphNode_t> nodes(nn);
  ck(cudaGraphGetNodes(c.graph, nodes.data(), &nn), "GraphGetNodes");
  long cur = -1;
  for (cudaGraphNode_t nd : nodes) {
    cudaGraphNodeType t;
    ck(cudaGraphNodeGetType(nd, &t), "GraphNodeGetType");
    if (t == cudaGraphNodeTypeMemset) {
      cudaMemsetParams mp;
      ck(cudaGraphMemsetNodeGetParams(nd, &mp), "MemsetNodeGetParams");
      if (mp.dst == ex->marker) {
        ++cur;
        if (cur >= static_cast<long>(ex->prog.size()) || static_cast<int>(mp.value) != static_cast<int>(cur & 0xff))
          xfail(SN_EK_INTERNAL, "census markers out of order");
        continue;
      }
    }
    if (cur < 0 || (t != cudaGraphNodeTypeKernel && t != cudaGraphNodeTypeMemcpy && t != cudaGraphNodeTypeMemset))
      continue;
    c.nodes.push_back({nd, static_cast<int>(cur)});
  }
}
}  // namespace

int sn_exec_census(sn_exec* ex, int32_t* action_kernels, size_t cap, char* names, size_t names_cap, size_t* n) {
  if (!ex || !n) return xset(SN_EK_INTERNAL, "null argument");
  *n = ex->prog.size();
  if (!action_kernels) return SN_OK;
  if (cap < ex->prog.size()) return xset(SN_EK_INTERNAL, "output buffer too small");
  return xguard([&] {
    ck(cudaSetDevice(ex->device), "cudaSetDevice");
    PrecisionScope prec(ex);
    ck(cudaDeviceSynchronize(), "sync");
    Census c;
    capture_census(ex, c);
    std::vector<std::string> nm(ex->prog.size());
    std::fill(action_kernels, action_kernels + ex->prog.size(), 0);
    for (const auto& na : c.nodes) {
      cudaGraphNodeType t;
      ck(cudaGraphNodeGetType(na.first, &t), "GraphNodeGetType");
      if (t != cudaGraphNodeTypeKernel) continue;
      cudaKernelNodeParams kp;
      ck(cudaGraphKernelNodeGetParams(na.first, &kp), "KernelNodeGetParams");
      const char* fname = nullptr;
      if (cudaFuncGetName(&fname, kp.func) != cudaSuccess || !fname) fname = "?";
      ++action_kernels[na.second];
      nm[na.second] += fname;
      nm[na.second] += '\n';
    }
    if (names && names_cap) {
      std::string all;
      for (size_t i = 0; i < nm.size(); ++i) all += nm[i] + "\x1e";  // record separator per action
      const size_t k = std::min(all.size(), names_cap - 1);
      std::memcpy(names, all.data(), k);
      names[k] = 0;
    }
  });
}

int sn_exec_kernel_times(sn_exec* ex, int32_t reps, float* us, int32_t* action, size_t cap, size_t* n) {
  if (!ex || !n) return xset(SN_EK_INTERNAL, "null argument");
  return xguard([&] {
    ck(cudaSetDevice(ex->device), "cudaSetDevice");
    PrecisionScope prec(ex);
    ck(cudaDeviceSynchronize(), "sync");
    Census c;
    capture_census(ex, c);
    size_t nk = 0;
    for (const auto& na : c.nodes) {
      cudaGraphNodeType t;
      ck(cudaGraphNodeGetType(na.first, &t), "GraphNodeGetType");
      nk += t == cudaGraphNodeTypeKernel;
    }
    *n = nk;
    if (!us) return;
    if (cap < nk) xfail(SN_EK_INTERNAL, "output buffer too small");
    // replay the iteration node by node on s0 (copies and memsets too, so the
    // data each kernel sees is the real one), an event pair around every kernel
    std::vector<cudaEvent_t> ev(2 * nk);
    for (auto& e : ev) ck(cudaEventCreate(&e), "event");
    std::vector<std::vector<float>> t(nk);
    cudaStream_t st = ex->s0;
    for (int r = 0; r < std::max(1, static_cast<int>(reps)); ++r) {
      size_t k = 0;
      hold_stream_kernel<<<1, 1, 0, st>>>(static_cast<uint64_t>(nk) * 40000ull);  // ~40 us of host time per kernel
      for (const auto& na : c.nodes) {
        cudaGraphNodeType ty;
        ck(cudaGraphNodeGetType(na.first, &ty), "GraphNodeGetType");
        if (ty == cudaGraphNodeTypeMemcpy) {
          cudaMemcpy3DParms mp;
          ck(cudaGraphMemcpyNodeGetParams(na.first, &mp), "MemcpyNodeGetParams");
          ck(cudaMemcpy3DAsync(&mp, st), "replay copy");
          continue;
        }
        if (ty == cudaGraphNodeTypeMemset) {
          cudaMemsetParams mp;
          ck(cudaGraphMemsetNodeGetParams(na.first, &mp), "MemsetNodeGetParams");
          if (mp.height <= 1)
            ck(cudaMemsetAsync(mp.dst, static_cast<int>(mp.value), mp.width * mp.elementSize, st), "replay memset");
          else
            ck(cudaMemset2DAsync(mp.dst, mp.pitch, static_cast<int>(mp.value), mp.width * mp.elementSize, mp.height,
                                 st),
               "replay memset");
          continue;
        }
        cudaKernelNodeParams kp;
        ck(cudaGraphKernelNodeGetParams(na.first, &kp), "KernelNodeGetParams");
        cudaLaunchAttributeValue cl{};
        const bool has_cl =
            cudaGraphKernelNodeGetAttribute(na.first, cudaLaunchAttributeClusterDimension, &cl) == cudaSuccess &&
            cl.clusterDim.x * cl.clusterDim.y * cl.clusterDim.z > 1;
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = kp.gridDim;
        cfg.blockDim = kp.blockDim;
        cfg.dynamicSmemBytes = kp.sharedMemBytes;
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        if (has_cl) {
          at[0].id = cudaLaunchAttributeClusterDimension;
          at[0].val = cl;
          cfg.attrs = at;
          cfg.numAttrs = 1;
        }
        ck(cudaEventRecord(ev[2 * k], st), "record");
        ck(cudaLaunchKernelExC(&cfg, kp.func, kp.kernelParams), "replay launch");
        ck(cudaEventRecord(ev[2 * k + 1], st), "record");
        if (r == 0) action[k] = na.second;
        ++k;
      }
      ck(cudaStreamSynchronize(st), "sync");
      for (size_t i = 0; i < nk; ++i) {
        float ms = 0.f;
        ck(cudaEventElapsedTime(&ms, ev[2 * i], ev[2 * i + 1]), "elapsed");
        t[i].push_back(ms * 1000.f);
      }
    }
    for (size_t i = 0; i < nk; ++i) {
      std::sort(t[i].begin(), t[i].end());
      us[i] = t[i][t[i].size() / 2];
    }
    for (auto& e : ev) cudaEventDestroy(e);
  });
}

int sn_exec_transfer_stats(sn_exec* ex, int64_t* d2h_bytes, double* d2h_ms, int64_t* h2d_bytes, double* h2d_ms,
                           double* exposed_ms) {
  if (!ex) return xset(SN_EK_INTERNAL, "null argument");
  return xguard([&] {
    ck(cudaSetDevice(ex->device), "cudaSetDevice");
    ck(cudaStreamSynchronize(ex->s0), "sync");
    int64_t bytes[3] = {0, 0, 0};
    double ms[3] = {0, 0, 0};
    for (const auto& t : ex->timers) {
      float m = 0.f;
      ck(cudaEventElapsedTime(&m, t.a, t.b), "elapsed");
      bytes[t.kind] += t.bytes;
      ms[t.kind] += m;
    }
    if (d2h_bytes) *d2h_bytes = bytes[0];
    if (d2h_ms) *d2h_ms = ms[0];
    if (h2d_bytes) *h2d_bytes = bytes[1];
    if (h2d_ms) *h2d_ms = ms[1];
    if (exposed_ms) *exposed_ms = ms[2];
  });
}

namespace {
constexpr uint32_t kArenaSentinel = 0xFFFFFFFFu;  // a NaN no kernel writes
__global__ void arena_scan_kernel(const uint32_t* __restrict__ a, int64_t blocks, unsigned long long* hi,
                                  unsigned long long* touched) {
  // one warp per 1 KiB block (256 words, 8 per lane)
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t b = w0; b < blocks; b += nw) {
    const uint4* p = reinterpret_cast<const uint4*>(a + b * 256) + lane * 2;
    const uint4 x = p[0], y = p[1];
    const bool used = (x.x & x.y & x.z & x.w & y.x & y.y & y.z & y.w) != kArenaSentinel;
    if (__any_sync(0xffffffffu, used) && lane == 0) {
      atomicMax(hi, static_cast<unsigned long long>(b + 1));
      atomicAdd(touched, 1ull);
    }
  }
}
}  // namespace

int sn_exec_memory(const sn_exec* ex, sn_exec_mem* out) {
  if (!ex || !out) return xset(SN_EK_INTERNAL, "null argument");
  out->arena_bytes = ex->mem[sn_exec::M_ARENA];
  out->params_grads_bytes = ex->mem[sn_exec::M_PARAMS];
  out->layer_state_bytes = ex->mem[sn_exec::M_STATE];
  out->input_bytes = ex->mem[sn_exec::M_INPUT];
  out->wgrad_scratch_bytes = ex->mem[sn_exec::M_WGRAD];
  out->other_scratch_bytes = ex->mem[sn_exec::M_OTHER];
  out->host_stash_bytes = ex->mem[sn_exec::M_HOST];
  out->device_stash_bytes = ex->mem[sn_exec::M_STASH];
  out->peer_stash_bytes = ex->mem[sn_exec::M_PEER];
  out->device_total_bytes = 0;
  for (int c = 0; c <= sn_exec::M_STASH; ++c) out->device_total_bytes += ex->mem[c];
  out->wgrad_partials_outside_pool_bytes = ex->wgrad_partial_outside * 4;
  out->planned_arena_high_water = ex->plan->plan.report.pool_high_water_bytes;
  return SN_OK;
}

int sn_exec_arena_fill(sn_exec* ex) {
  if (!ex) return xset(SN_EK_INTERNAL, "null argument");
  return xguard([&] {
    ck(cudaSetDevice(ex->device), "cudaSetDevice");
    ck(cudaMemsetAsync(ex->arena, 0xFF, static_cast<size_t>(ex->arena_bytes), ex->s0), "memset(arena)");
    ck(cudaStreamSynchronize(ex->s0), "sync");
  });
}

int sn_exec_arena_scan(sn_exec* ex, int64_t* high_water_bytes, int64_t* touched_bytes) {
  if (!ex) return xset(SN_EK_INTERNAL, "null argument");
  return xguard([&] {
    ck(cudaSetDevice(ex->device), "cudaSetDevice");
    ck(cudaDeviceSynchronize(), "sync");
    unsigned long long* d = nullptr;
    ck(cudaMalloc(&d, 2 * sizeof(unsigned long long)), "cudaMalloc(scan)");
    cudaMemsetAsync(d, 0, 2 * sizeof(unsigned long long), ex->s0);
    const int64_t blocks = ex->arena_bytes / snp::kBlockBytes;
    arena_scan_kernel<<<148 * 8, 256, 0, ex->s0>>>(reinterpret_cast<const uint32_t*>(ex->arena), blocks, d, d + 1);
    unsigned long long h[2] = {0, 0};
    const cudaError_t e1 = cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, ex->s0);
    const cudaError_t e2 = cudaStreamSynchronize(ex->s0);
    cudaFree(d);
    ck(e1, "scan D2H");
    ck(e2, "scan");
    if (high_water_bytes) *high_water_bytes = static_cast<int64_t>(h[0]) * snp::kBlockBytes;
    if (touched_bytes) *touched_bytes = static_cast<int64_t>(h[1]) * snp::kBlockBytes;
  });
}

int sn_dp_buckets(const sn_plan* plan, int64_t bucket_bytes, int64_t* lo, int64_t* hi, int32_t* after_layer,
                  size_t cap, size_t* n) {
  if (!plan || !n) return xset(SN_EK_INTERNAL, "null argument");
  sn_exec tmp;  // host-side layout only: no device resources are created
  tmp.plan = plan;
  tmp.net = &plan->plan.net;
  tmp.B = static_cast<int>(plan->plan.cost_cfg.batch);
  return xguard([&] {
    setup_layers(&tmp, nullptr);
    plan_buckets(&tmp, bucket_bytes > 0 ? bucket_bytes : (8ll << 20));
    *n = tmp.buckets.size();
    if (!lo) return;
    if (cap < tmp.buckets.size()) xfail(SN_EK_INTERNAL, "output buffer too small");
    for (size_t i = 0; i < tmp.buckets.size(); ++i) {
      lo[i] = tmp.buckets[i].lo;
      hi[i] = tmp.buckets[i].hi;
      if (after_layer) after_layer[i] = tmp.buckets[i].after_layer;
    }
  });
}

int sn_exec_catalog(const sn_exec* ex, sn_catalog_entry* out, size_t cap, size_t* n) {
  if (!ex || !n) return xset(SN_EK_INTERNAL, "null argument");
  *n = ex->catalog.size();
  if (!out) return SN_OK;
  if (cap < ex->catalog.size()) return xset(SN_EK_INTERNAL, "output buffer too small");
  for (size_t i = 0; i < ex->catalog.size(); ++i) {
    const auto& c = ex->catalog[i];
    out[i] = sn_catalog_entry{c.layer, c.op, c.k.halo, c.k.pairs, c.k.bn, c.k.subpix, c.us, c.chosen};
  }
  return SN_OK;
}

int sn_exec_workspace_use(const sn_exec* ex, int32_t* wgrad_in_pool, int32_t* wgrad_outside) {
  if (!ex) return xset(SN_EK_INTERNAL, "null argument");
  if (wgrad_in_pool) *wgrad_in_pool = ex->wgrad_ws_in_pool;
  if (wgrad_outside) *wgrad_outside = ex->wgrad_ws_outside;
  return SN_OK;
}

int sn_exec_apply_update(sn_exec* ex, float lr, float grad_scale) {
  if (!ex) return xset(SN_EK_INTERNAL, "null argument");
  return xguard([&] {
    ck(sn::sgd_update(ex->params, ex->grads, ex->n_params, lr, grad_scale, ex->s0), "sgd");
    ck(cudaStreamSynchronize(ex->s0), "sync");
  });
}

int sn_exec_read_tensor(sn_exec* ex, int32_t kind, int32_t layer, float* dst, int64_t n_floats) {
  if (!ex) return xset(SN_EK_INTERNAL, "null argument");
  return xguard([&] {
    if (kind == snp::K_ACT && layer >= 0 && layer < static_cast<int>(ex->elided.size()) && ex->elided[layer])
      xfail(SN_EK_UNSUPPORTED, "output of '" + ex->net->names[layer] +
                                   "' is fused into its ReLU and never materialised (SN_FUSE=0 keeps it)");
    auto it = ex->final_keys.find(snp::key_code(kind, layer));
    if (it == ex->final_keys.end()) xfail(SN_EK_INTERNAL, "tensor is not resident at the end of the iteration");
    const float* src = reinterpret_cast<const float*>(ex->arena + it->second.first * snp::kBlockBytes);
    ck(cudaMemcpy(dst, src, static_cast<size_t>(n_floats) * sizeof(float), cudaMemcpyDeviceToDevice), "read");
  });
}

}  // extern "C"
