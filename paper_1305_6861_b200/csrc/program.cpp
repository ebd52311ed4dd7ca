// Host compiler: flattened OperatorTables -> device op stream.
//
// Input is exactly the reference's EsTable content (engine.py:51-70) flattened
// into SoA arrays by the caller.  Output: DevOp stream + GEv / matrix side
// tables + the compact-sample -> output-position map.  See program.h for the
// op set.  The walk order is the reference's (engine.py:276-308): per ES the
// pulse, then its events in order; every compiled op covers a contiguous run
// of that walk, so the device replays the same operator sequence.
#include "program_host.h"
#include "resident.h"

#include <algorithm>
#include <array>
#include <functional>
#include <map>
#include <set>
#include <cmath>
#include <cstdlib>
#include <stdexcept>
#include <string>

namespace bloch {

namespace {

inline bool moving(double dt, const double* dm) {
  // engine.py:288 — `dt != 0.0 or dmom.any()`
  return dt != 0.0 || dm[0] != 0.0 || dm[1] != 0.0 || dm[2] != 0.0;
}

inline double inf_norm(const double* a) {
  return std::max(std::fabs(a[0]), std::max(std::fabs(a[1]), std::fabs(a[2])));
}

// Relative tolerance separating rounding noise of t_i - t_{i-1} and
// partial[i] - partial[i-1] (engine.py:130-131; ~1e-13 relative) from any
// physical difference (>= 1e-3 relative for the waveforms of sequence.py).
constexpr double kRtol = 1e-9;

// Two intervals are "the same": equal up to rounding, exact zeros stay zeros
// so relaxation-free / gradient-free intervals keep their class.
inline bool same_interval(double dt_a, const double* a, double dt_b, const double* b) {
  if ((dt_a == 0.0) != (dt_b == 0.0)) return false;
  if (std::fabs(dt_a - dt_b) > kRtol * std::fabs(dt_b)) return false;
  const double mag = inf_norm(b);
  for (int k = 0; k < 3; ++k) {
    if ((a[k] == 0.0) != (b[k] == 0.0)) return false;
    if (std::fabs(a[k] - b[k]) > kRtol * mag) return false;
  }
  return true;
}

}  // namespace

void fuse_intervals(Program& prog, const std::function<int32_t(double)>& relax_class);
void find_progressions(Program& prog);
void find_chirp_classes(Program& prog);
void fuse_pulses(Program& prog);
void find_train_classes(Program& prog);
void assign_planes(Program& prog);
void defer_windows(Program& prog, int short_runs);

void compile_program(const TablesView& t, Program& prog) {
  prog = Program();
  prog.n_acq = t.n_acq;
  prog.max_samples = t.max_samples;
  prog.n_snap = t.n_snap;
  if (t.n_es < 0 || t.n_acq < 0 || t.max_samples < 0 || t.n_snap < 0)
    throw std::invalid_argument("negative table dimension");
  if (t.n_acq > 0 && t.max_samples <= 0) throw std::invalid_argument("n_acq > 0 requires max_samples > 0");
  if (t.n_es && t.es_ev_offset[0] != 0) throw std::invalid_argument("es_ev_offset[0] must be 0");
  const int64_t E = t.n_es ? t.es_ev_offset[t.n_es] : 0;
  for (int32_t es = 0; es < t.n_es; ++es) {
    if (t.es_ev_offset[es + 1] < t.es_ev_offset[es] || t.es_ev_offset[es + 1] > E)
      throw std::invalid_argument("es_ev_offset not monotone");
    if (t.es_acq[es] >= t.n_acq) throw std::invalid_argument("es_acq out of range");
  }
  for (int64_t i = 0; i < E; ++i) {
    if (t.ev_snap[i] >= t.n_snap) throw std::invalid_argument("ev_snap out of range");
    // The reference's own tables can hold a -1e-18 s interval: a snapshot at the sequence end that the
    // running clock places a rounding step inside the last elementary sequence leaves a negative
    // remainder, which compute_block applies as is.  Rejected: non-finite values and intervals more
    // negative than such a rounding residue.
    if (!std::isfinite(t.ev_dt[i]) || t.ev_dt[i] < -1e-12)
      throw std::invalid_argument("negative (beyond rounding) or non-finite event interval");
    for (int a = 0; a < 3; ++a)
      if (!std::isfinite(t.ev_dmom[3 * i + a])) throw std::invalid_argument("non-finite event moment");
  }

  auto dm = [&](int64_t i) { return t.ev_dmom + 3 * i; };
  std::map<double, int32_t> classes;  // exact interval length -> relax class (engine.py:293)
  auto relax_class = [&](double T) -> int32_t {
    if (T == 0.0) return -1;
    auto it = classes.find(T);
    if (it != classes.end()) return it->second;
    const int32_t c = static_cast<int32_t>(prog.relax_t.size());
    classes.emplace(T, c);
    prog.relax_t.push_back(T);
    return c;
  };
  auto n_ev = [&](int32_t es) { return t.es_ev_offset[es + 1] - t.es_ev_offset[es]; };

  // an ES that can join an RF train: exactly one event, no ADC, no snapshot
  auto train_es = [&](int32_t es) {
    if (n_ev(es) != 1) return false;
    const int64_t e = t.es_ev_offset[es];
    return !t.ev_sample[e] && t.ev_snap[e] < 0;
  };

  int32_t es = 0;
  while (es < t.n_es) {
    // ---- RF train: consecutive (pulse?, identical interval) elementary sequences
    if (train_es(es)) {
      const int64_t e0 = t.es_ev_offset[es];
      int32_t k = es + 1;
      while (k < t.n_es && train_es(k) &&
             same_interval(t.ev_dt[t.es_ev_offset[k]], dm(t.es_ev_offset[k]), t.ev_dt[e0], dm(e0)))
        ++k;
      if (k - es >= kMinTrain) {
        DevOp op{};
        op.kind = OP_RFTRAIN;
        op.count = k - es;
        op.aux = static_cast<int32_t>(prog.mats.size() / 9);
        double sdt = 0.0, sm[3] = {0.0, 0.0, 0.0};
        for (int32_t j = es; j < k; ++j) {
          const int64_t e = t.es_ev_offset[j];
          sdt += t.ev_dt[e];
          for (int a = 0; a < 3; ++a) sm[a] += dm(e)[a];
          if (t.es_has_pulse[j]) {
            for (int q = 0; q < 9; ++q) prog.mats.push_back(t.es_pulse_mat[9 * j + q]);
            prog.n_rot++;
          } else {
            const double id[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
            prog.mats.insert(prog.mats.end(), id, id + 9);
          }
        }
        const double n = static_cast<double>(k - es);
        op.p[0] = t.ev_dt[e0] == 0.0 ? 0.0 : sdt / n;
        for (int a = 0; a < 3; ++a) op.p[1 + a] = dm(e0)[a] == 0.0 ? 0.0 : sm[a] / n;
        op.flags = (moving(op.p[0], op.p + 1) ? EV_MOVE : 0) | (op.p[0] != 0.0 ? EV_RELAX : 0);
        op.cls = relax_class(op.p[0]);
        op.rot = -1;
        // a real envelope (phase 0 or pi, sequence.py:650-674) rotates about x only: the kernel then
        // needs 4 of the 9 entries.  sin(pi) leaves ~1e-16 off-axis terms, below the 1e-15 cut.
        op.tmode = 1;
        for (int32_t j = 0; j < op.count && op.tmode; ++j) {
          const double* m = prog.mats.data() + 9 * (static_cast<size_t>(op.aux) + j);
          if (std::fabs(m[0] - 1.0) > 1e-15 || std::fabs(m[1]) > 1e-15 || std::fabs(m[2]) > 1e-15 ||
              std::fabs(m[3]) > 1e-15 || std::fabs(m[6]) > 1e-15)
            op.tmode = 0;
        }
        prog.ops.push_back(op);
        prog.n_events += k - es;
        prog.n_train_ops++;
        prog.n_train_pairs += k - es;
        es = k;
        continue;
      }
    }

    const int64_t e0 = t.es_ev_offset[es], e1 = t.es_ev_offset[es + 1];
    const int32_t acq = t.es_acq[es];
    if (t.es_has_pulse[es]) {  // engine.py:277-283
      DevOp op{};
      op.kind = OP_ROT;
      for (int k = 0; k < 9; ++k) op.p[k] = t.es_pulse_mat[9 * es + k];
      prog.ops.push_back(op);
      prog.n_rot++;
    }
    prog.n_events += e1 - e0;

    int32_t sample_idx = 0;  // engine.py:284 — running sample index within the ES
    auto record_sample = [&]() -> int32_t {
      if (acq < 0) throw std::invalid_argument("sample event in an ES without acquisition");
      if (sample_idx >= t.max_samples) throw std::invalid_argument("more samples than max_samples");
      const int32_t s = static_cast<int32_t>(prog.sample_g.size());
      prog.sample_g.push_back(static_cast<int64_t>(acq) * t.max_samples + sample_idx);
      ++sample_idx;
      return s;
    };
    // length of a uniform sampled run starting at event j (0 if none)
    auto run_len = [&](int64_t j) -> int64_t {
      if (j >= e1 || !t.ev_sample[j] || !moving(t.ev_dt[j], dm(j))) return 0;
      int64_t k = j + 1;
      while (k < e1 && t.ev_sample[k] && same_interval(t.ev_dt[k], dm(k), t.ev_dt[j], dm(j))) ++k;
      return k - j;
    };
    // (lead, rotations) of a window starting at event i, or 0
    auto window_at = [&](int64_t i, int& lead) -> int64_t {
      lead = 0;
      if (i >= e1 || !t.ev_sample[i]) return 0;
      if (!moving(t.ev_dt[i], dm(i))) {
        const int64_t r = run_len(i + 1);
        if (r >= kMinWindow) {
          lead = 1;
          return r;
        }
        return 0;
      }
      const int64_t r = run_len(i);
      return r >= kMinWindow ? r : 0;
    };
    // length of a linear-increment sampled run starting at j (0 if < kMinChirp)
    auto chirp_at = [&](int64_t j) -> int64_t {
      if (j + 2 >= e1) return 0;
      for (int64_t q = j; q < j + 2; ++q)
        if (!t.ev_sample[q] || t.ev_snap[q] >= 0) return 0;
      const double dt = t.ev_dt[j];
      if ((t.ev_dt[j + 1] == 0.0) != (dt == 0.0) || std::fabs(t.ev_dt[j + 1] - dt) > kRtol * std::fabs(dt))
        return 0;
      double dd[3];
      for (int a = 0; a < 3; ++a) dd[a] = dm(j + 1)[a] - dm(j)[a];
      if (inf_norm(dd) == 0.0) return 0;  // a uniform run, not a chirp
      int64_t k = j + 2;
      while (k < e1 && t.ev_sample[k] && t.ev_snap[k] < 0) {
        if ((t.ev_dt[k] == 0.0) != (dt == 0.0) || std::fabs(t.ev_dt[k] - dt) > kRtol * std::fabs(dt)) break;
        const double mag = std::max(inf_norm(dm(k)), inf_norm(dm(j)));
        bool ok = true;
        for (int a = 0; a < 3 && ok; ++a) {
          const double pred = dm(j)[a] + static_cast<double>(k - j) * dd[a];
          ok = std::fabs(dm(k)[a] - pred) <= kRtol * mag;
        }
        if (!ok) break;
        ++k;
      }
      return k - j >= kMinChirp ? k - j : 0;
    };

    int64_t i = e0;
    while (i < e1) {
      const double dt = t.ev_dt[i];
      if (!t.ev_sample[i]) {  // interval (+ snapshot)
        DevOp op{};
        op.kind = OP_EVENT;
        op.count = (moving(dt, dm(i)) ? EV_MOVE : 0) | (dt != 0.0 ? EV_RELAX : 0);
        op.aux = t.ev_snap[i];
        op.p[0] = dt;
        for (int k = 0; k < 3; ++k) op.p[1 + k] = dm(i)[k];
        op.cls = -1;  // classes are assigned by fuse_intervals()
        op.rot = -1;
        prog.ops.push_back(op);
        prog.n_interval++;
        ++i;
        continue;
      }
      int lead = 0;
      const int64_t rot = window_at(i, lead);
      if (rot > 0) {  // uniform window: mean interval of the run
        const int64_t j0 = i + lead;
        double sdt = 0.0, sm[3] = {0.0, 0.0, 0.0};
        for (int64_t k = j0; k < j0 + rot; ++k) {
          sdt += t.ev_dt[k];
          for (int a = 0; a < 3; ++a) sm[a] += dm(k)[a];
        }
        DevOp op{};
        op.kind = OP_WINDOW;
        op.count = static_cast<int32_t>(rot + lead);
        op.aux = lead;
        op.p[0] = t.ev_dt[j0] == 0.0 ? 0.0 : sdt / static_cast<double>(rot);
        for (int a = 0; a < 3; ++a) op.p[1 + a] = dm(j0)[a] == 0.0 ? 0.0 : sm[a] / static_cast<double>(rot);
        op.cls = -1;
        op.rot = -1;  // assigned by fuse_intervals()
        op.s0 = record_sample();
        for (int64_t k = 1; k < rot + lead; ++k) record_sample();
        prog.ops.push_back(op);
        prog.n_window_ops++;
        prog.n_window_samples += rot + lead;
        i += rot + lead;
        continue;
      }
      const int64_t ch = chirp_at(i);
      if (ch > 0) {  // linear-increment run: least-squares-free, exact endpoints
        DevOp op{};
        op.kind = OP_CHIRP;
        op.count = static_cast<int32_t>(ch);
        op.p[0] = dt;
        const double m = static_cast<double>(ch - 1);
        for (int a = 0; a < 3; ++a) {
          op.p[1 + a] = dm(i)[a];
          // slope from the run's end points keeps the accumulated moment exact
          op.p[4 + a] = (dm(i + ch - 1)[a] - dm(i)[a]) / m;
        }
        op.cls = relax_class(dt);
        op.rot = -1;
        op.s0 = record_sample();
        for (int64_t k = 1; k < ch; ++k) record_sample();
        prog.ops.push_back(op);
        prog.n_chirp_ops++;
        prog.n_chirp_samples += ch;
        i += ch;
        continue;
      }
      // generic sampled intervals, up to kChunkSlots per op
      DevOp op{};
      op.kind = OP_GSAMP;
      op.aux = static_cast<int32_t>(prog.gev.size());
      op.count = 0;
      while (i < e1 && op.count < kChunkSlots && t.ev_sample[i]) {
        int l2 = 0;
        if (op.count > 0 && (window_at(i, l2) > 0 || chirp_at(i) > 0)) break;
        GEv g{};
        g.dt = t.ev_dt[i];
        g.dmx = dm(i)[0];
        g.dmy = dm(i)[1];
        g.dmz = dm(i)[2];
        g.flags = (moving(g.dt, dm(i)) ? EV_MOVE : 0) | (g.dt != 0.0 ? EV_RELAX : 0);
        g.cls = relax_class(g.dt);
        prog.gev.push_back(g);
        const int32_t s = record_sample();
        if (op.count == 0) op.s0 = s;
        op.count++;
        ++i;
      }
      prog.ops.push_back(op);
      prog.n_gsamp_events += op.count;
    }
    ++es;
  }
  prog.n_events += prog.n_rot;
  prog.n_samples = static_cast<int64_t>(prog.sample_g.size());
  fuse_intervals(prog, relax_class);
}

// Interval fusion and class assignment.
//
// Consecutive intervals with no pulse, ADC sample or snapshot between them
// compose exactly into one interval: the transverse factors multiply
// (e2_a e^{-i th_a}) (e2_b e^{-i th_b}) = e^{-(dt_a+dt_b)/T2} e^{-i (th_a+th_b)}
// with th linear in (dmom, dt), and the longitudinal affine maps compose to
// mz -> e1_a e1_b mz + m0 (1 - e1_a e1_b) — so (dt, dmom) simply add
// (engine.py:288-302 applied back to back).
//
// Rotation classes (tabulated per-spin propagators, program.h) pay off only
// when reused: a window absorbs the merged interval right before it (pre) and
// right after it (post) when the resulting (pre, window, post) class occurs at
// least kMinReuse times; other intervals get a class when they occur at least
// kMinReuse times.  At most kMaxRotClasses classes are made (table memory is
// classes x spins x 64 B); everything else is evaluated on the fly.
void fuse_intervals(Program& prog, const std::function<int32_t(double)>& relax_class) {
  constexpr int64_t kMinReuse = 4;
  constexpr size_t kMaxRotClasses = 64;
  struct Item {
    DevOp op;
    bool interval;  // merged EVENT
  };
  std::vector<Item> items;
  for (const DevOp& op : prog.ops) {
    if (op.kind == OP_EVENT) {
      if (!items.empty() && items.back().interval && items.back().op.aux < 0) {
        DevOp& m = items.back().op;  // extend the open interval
        m.p[0] += op.p[0];
        for (int a = 0; a < 3; ++a) m.p[1 + a] += op.p[1 + a];
        m.aux = op.aux;  // a snapshot closes the merged interval
      } else {
        items.push_back({op, true});
      }
      continue;
    }
    items.push_back({op, false});
  }
  const size_t n_items = items.size();
  using Key = std::array<double, 4>;
  auto key_of = [](const DevOp& op) { return Key{op.p[0], op.p[1], op.p[2], op.p[3]}; };
  const double none[4] = {0.0, 0.0, 0.0, 0.0};
  using RotKey = std::array<double, 13>;
  auto rot_key = [](const double* pre, const double* main, double mult, const double* post) {
    RotKey key;
    for (int a = 0; a < 4; ++a) {
      key[a] = pre[a];
      key[4 + a] = main[a];
      key[9 + a] = post[a];
    }
    key[8] = mult;
    return key;
  };
  auto free_interval = [&](size_t k) { return k < n_items && items[k].interval && items[k].op.aux < 0; };

  // 1. windows: candidate absorption, kept when the absorbed class is reused
  std::vector<int> pre_of(n_items, 0), post_of(n_items, 0);  // 1 = absorbs neighbour
  std::map<RotKey, int64_t> win_uses;
  auto win_key = [&](size_t k, int pre, int post) {
    const DevOp& w = items[k].op;
    return rot_key(pre ? items[k - 1].op.p : none, w.p, static_cast<double>(w.count - w.aux),
                   post ? items[k + 1].op.p : none);
  };
  for (size_t k = 0; k < n_items; ++k)
    if (items[k].op.kind == OP_WINDOW && !items[k].interval) {
      pre_of[k] = k > 0 && free_interval(k - 1);
      post_of[k] = free_interval(k + 1);
    }
  for (size_t k = 0; k + 1 < n_items; ++k)  // an interval between two windows goes to the earlier one
    if (items[k].op.kind == OP_WINDOW && post_of[k] && k + 2 < n_items && pre_of[k + 2]) pre_of[k + 2] = 0;
  for (size_t k = 0; k < n_items; ++k)
    if (items[k].op.kind == OP_WINDOW && !items[k].interval) win_uses[win_key(k, pre_of[k], post_of[k])]++;
  // absorbing keys reused often enough, most reused first, within the class cap: a window may only absorb
  // its neighbours if its whole (pre, window, post) run gets a tabulated class
  std::vector<std::pair<int64_t, RotKey>> absorbing;
  for (const auto& kv : win_uses) {
    const RotKey& key = kv.first;
    const bool absorbs = std::any_of(key.begin(), key.begin() + 4, [](double v) { return v != 0.0; }) ||
                         std::any_of(key.begin() + 9, key.end(), [](double v) { return v != 0.0; });
    if (absorbs && kv.second >= kMinReuse) absorbing.push_back({-kv.second, key});
  }
  std::sort(absorbing.begin(), absorbing.end());
  if (absorbing.size() > kMaxRotClasses) absorbing.resize(kMaxRotClasses);
  std::set<RotKey> classed_absorbing;
  for (const auto& a : absorbing) classed_absorbing.insert(a.second);
  for (size_t k = 0; k < n_items; ++k)
    if (items[k].op.kind == OP_WINDOW && !items[k].interval && (pre_of[k] || post_of[k]) &&
        !classed_absorbing.count(win_key(k, pre_of[k], post_of[k])))
      pre_of[k] = post_of[k] = 0;
  std::vector<bool> absorbed(n_items, false);
  for (size_t k = 0; k < n_items; ++k) {
    if (pre_of[k]) absorbed[k - 1] = true;
    if (post_of[k]) absorbed[k + 1] = true;
  }
  // 2. reuse counts of the intervals that stay separate
  std::map<Key, int64_t> iv_uses;
  std::map<RotKey, int64_t> plain_win_uses;
  for (size_t k = 0; k < n_items; ++k) {
    if (items[k].interval && !absorbed[k]) iv_uses[key_of(items[k].op)]++;
    if (items[k].op.kind == OP_WINDOW && !items[k].interval) plain_win_uses[win_key(k, pre_of[k], post_of[k])]++;
  }

  std::map<RotKey, int32_t> rot_ids;
  auto rot_class = [&](const RotKey& key) -> int32_t {
    auto f = rot_ids.find(key);
    if (f != rot_ids.end()) return f->second;
    if (prog.rot_classes.size() >= kMaxRotClasses) return -1;
    const int32_t c = static_cast<int32_t>(prog.rot_classes.size());
    rot_ids.emplace(key, c);
    RotClass rc{};
    for (int a = 0; a < 4; ++a) {
      rc.pre[a] = key[a];
      rc.main[a] = key[4 + a];
      rc.post[a] = key[9 + a];
    }
    rc.mult = key[8];
    prog.rot_classes.push_back(rc);
    return c;
  };

  // 3. emit; the absorbing windows claim their classes first, then the remaining windows and the
  // reused intervals in order of reuse (most reused first)
  for (const auto& a : absorbing) rot_class(a.second);
  std::vector<std::pair<int64_t, RotKey>> order;
  for (const auto& kv : plain_win_uses) order.push_back({-kv.second, kv.first});
  for (const auto& kv : iv_uses)
    if (kv.second >= kMinReuse && moving(kv.first[0], kv.first.data() + 1))
      order.push_back({-kv.second, rot_key(none, kv.first.data(), 1.0, none)});
  std::sort(order.begin(), order.end());
  for (const auto& o : order) rot_class(o.second);

  std::vector<DevOp> out;
  for (size_t k = 0; k < n_items; ++k) {
    if (absorbed[k]) continue;
    DevOp op = items[k].op;
    op.prg = -1;
    if (op.kind == OP_WINDOW && !items[k].interval) {
      const RotKey key = win_key(k, pre_of[k], post_of[k]);
      auto f = rot_ids.find(key);
      op.rot = f != rot_ids.end() ? f->second : -1;
      if (op.rot < 0) {  // on-the-fly window: no absorbed neighbours (kept separate above only if classed)
        if (pre_of[k] || post_of[k]) throw std::logic_error("absorbing window without a class");
        op.cls = relax_class(op.p[0]);
        op.flags = relax_class(op.p[0] * static_cast<double>(op.count - op.aux));  // whole-window class
      }
      prog.n_fused_windows += pre_of[k] + post_of[k];
      out.push_back(op);
      continue;
    }
    if (items[k].interval) {
      const bool mv = moving(op.p[0], op.p + 1);
      op.count = (mv ? EV_MOVE : 0) | (op.p[0] != 0.0 ? EV_RELAX : 0);
      op.rot = -1;
      op.cls = -1;
      if (mv) {
        auto f = rot_ids.find(rot_key(none, op.p, 1.0, none));
        if (f != rot_ids.end()) op.rot = f->second;
        else op.cls = relax_class(op.p[0]);
      }
      if (!mv && op.aux < 0) continue;  // a no-op interval (dt = 0, dmom = 0) without snapshot
      prog.n_fused_intervals++;
    }
    out.push_back(op);
  }
  prog.ops.swap(out);
  find_progressions(prog);
  find_chirp_classes(prog);
  find_train_classes(prog);
  fuse_pulses(prog);
  assign_planes(prog);
  // Short runs (tabulated chirps, single-sample events) join the contraction when that makes the program
  // fully deferred and covered by the resident-table integrator (resident.h): config 3 4.64 vs 5.82 ms
  // (profiles/r3e_shards.txt).  Otherwise they cost more in the contraction than in the integrator (each
  // group is a 64-sample M-tile pass over every spin whatever its length: 7.22 vs 5.70 ms on config 3 with
  // integrate_kernel, profiles/r2gg_short_runs.txt).  BLOCH_DEFER_SHORT=1 / 0 forces either.
  static const int short_env = [] {
    const char* e = getenv("BLOCH_DEFER_SHORT");
    return e ? (atoi(e) != 0 ? 1 : 0) : -1;
  }();
  if (short_env == 1) {
    defer_windows(prog, 1);
    return;
  }
  if (short_env != 0) {
    for (int mode = 1; mode <= 2; ++mode) {  // a few stragglers (a ramp cut by a snapshot) as groups of their own
      Program alt = prog;
      defer_windows(alt, mode);
      ResidentPlan plan;
      resident_compile(alt, plan);
      size_t small = 0;
      for (const WinGroup& g : alt.groups)
        small += !(g.chirp == 0 && g.count >= kMinDeferWindow) && g.n_windows < kMinDeferGroup;
      if (plan.ok && small <= 4) {
        prog = std::move(alt);
        return;
      }
    }
  }
  defer_windows(prog, 0);
}

// The deferred-window view (program.h OP_UWIN, contract.h): every tabulated window of at least
// kMinDeferWindow samples is grouped by (z plane, sample count); its samples are then formed by one
// tensor-core product per group instead of per-warp sums in the integrator.  U rows are numbered group
// by group, in op order inside a group.  The remaining sampled ops keep their samples under new
// compact ids (dsample_g), so the integrator's partial rows only hold those.
// short_runs: 0 = long windows only; 1 = also tabulated chirps and single-sample events in groups of at
// least kMinDeferGroup; 2 = also their smaller groups (one contraction launch each)
void defer_windows(Program& prog, int short_runs) {
  prog.dops.clear();
  prog.dsample_g.clear();
  prog.groups.clear();
  prog.urow_out0.clear();
  prog.n_deferred_samples = 0;
  // plane dedup over the existing planes (assign_planes' keys), for the planes of single-sample events
  using PKey = std::array<double, 6>;
  std::map<PKey, int32_t> pids;
  auto pkey = [](const PlaneDesc& pd) {
    return PKey{static_cast<double>(pd.kind * 16 + pd.flags), pd.T, pd.d[0], pd.d[1], pd.d[2], pd.tw};
  };
  for (size_t k = 0; k < prog.planes.size(); ++k)
    if (!(prog.planes[k].flags & PL_MUTABLE)) pids.emplace(pkey(prog.planes[k]), static_cast<int32_t>(k));
  auto plane = [&](int32_t kind, int32_t flags, double T, const double* d, double tw) -> int32_t {
    PlaneDesc pd{};
    pd.kind = kind;
    pd.flags = flags;
    pd.T = T;
    for (int a = 0; a < 3; ++a) pd.d[a] = kind == PL_PHASE ? d[a] : 0.0;
    pd.tw = kind == PL_PHASE ? tw : 0.0;
    auto f = pids.find(pkey(pd));
    if (f != pids.end()) return f->second;
    const int32_t id = static_cast<int32_t>(prog.planes.size());
    prog.planes.push_back(pd);
    pids.emplace(pkey(pd), id);
    return id;
  };
  // a single-sample generic event as a one-sample window: u = w m z, exit C = z (fp64), (A, B) of its dt
  const double zero3[3] = {0.0, 0.0, 0.0};
  auto single = [&](const DevOp& op, DevOp& w) {
    const GEv& g = prog.gev[op.aux];
    const double dt = g.dt, dm[3] = {g.dmx, g.dmy, g.dmz};
    const bool mv = (g.flags & EV_MOVE) != 0, rx = (g.flags & EV_RELAX) != 0;
    const double T = rx ? dt : 0.0;
    w = op;
    w.kind = OP_WINDOW;
    w.count = 1;
    w.aux = 0;  // no leading no-op sample: the sample follows the interval
    w.pre = -1;
    w.pl[0] = plane(PL_PHASE, PL_WEIGHT | PL_SAMPLE, 0.0, zero3, 0.0);
    w.pl[1] = plane(PL_PHASE, PL_SAMPLE, T, mv ? dm : zero3, mv ? dt : 0.0);
    w.pl[2] = plane(PL_PHASE, 0, T, mv ? dm : zero3, mv ? dt : 0.0);
    w.pl[3] = plane(PL_AB, 0, T, zero3, 0.0);
  };
  // candidates: tabulated windows, tabulated chirps, single-sample generic events (grouped below)
  struct Cand {
    size_t k;
    DevOp op;  // as deferred (single samples rewritten as one-sample windows)
  };
  using GKey = std::array<int32_t, 5>;  // (chirp, z / r0 plane, q plane, conj, count)
  std::map<GKey, std::vector<Cand>> by_key;
  std::vector<GKey> key_order;
  for (size_t k = 0; k < prog.ops.size(); ++k) {
    const DevOp& op = prog.ops[k];
    GKey key;
    DevOp d = op;
    if (op.kind == OP_WINDOW && op.rot >= 0 && op.count >= kMinDeferWindow && op.count <= kMaxDeferWindow) {
      key = {0, op.pl[1], -1, 0, op.count};
    } else if (short_runs && op.kind == OP_CHIRP && op.rot >= 0 && op.count <= kMaxDeferChirp) {
      key = {1, op.pl[0], op.pl[1], op.tmode & 1, op.count};
    } else if (short_runs && op.kind == OP_GSAMP && op.count == 1) {
      single(op, d);
      key = {0, d.pl[1], -1, 0, 1};
    } else {
      continue;
    }
    auto f = by_key.find(key);
    if (f == by_key.end()) {
      key_order.push_back(key);
      f = by_key.emplace(key, std::vector<Cand>()).first;
    }
    f->second.push_back(Cand{k, d});
  }
  std::vector<int32_t> row_of(prog.ops.size(), -1);
  std::vector<DevOp> as_deferred(prog.ops.size());
  int32_t row = 0;
  for (const GKey& key : key_order) {
    const std::vector<Cand>& mem = by_key[key];
    const bool long_window = key[0] == 0 && key[4] >= kMinDeferWindow;
    if (!long_window && short_runs < 2 && static_cast<int32_t>(mem.size()) < kMinDeferGroup) continue;
    WinGroup g{key[1], key[4], row, static_cast<int32_t>(mem.size()), key[0], key[2], key[3]};
    prog.groups.push_back(g);
    for (const Cand& c : mem) {
      const DevOp& op = prog.ops[c.k];
      const int64_t first = prog.sample_g[op.s0];
      for (int32_t q = 1; q < op.count; ++q)
        if (prog.sample_g[op.s0 + q] != first + q) throw std::logic_error("window samples not contiguous");
      prog.urow_out0.push_back(first);
      prog.n_deferred_samples += op.count;
      as_deferred[c.k] = c.op;
      row_of[c.k] = row++;
    }
  }
  for (size_t k = 0; k < prog.ops.size(); ++k) {
    DevOp op = prog.ops[k];
    if (row_of[k] >= 0) {
      op = as_deferred[k];
      op.kind = op.kind == OP_CHIRP ? OP_UCHIRP : OP_UWIN;
      op.s0 = row_of[k];
    } else if (op.kind == OP_WINDOW || op.kind == OP_CHIRP || op.kind == OP_GSAMP) {
      const int32_t s0 = static_cast<int32_t>(prog.dsample_g.size());
      for (int32_t q = 0; q < op.count; ++q) prog.dsample_g.push_back(prog.sample_g[op.s0 + q]);
      op.s0 = s0;
    }
    prog.dops.push_back(op);
  }
}

// A hard pulse followed by an interval or a window is applied by that op
// (DevOp.pre): one op dispatch less per pulse.  The matrix moves to the shared
// matrix table; the arithmetic is unchanged (R m first, then the op), so results
// are bit-identical.  Only programs of pulses, intervals and windows are fused:
// their kernel variant (kFull = false) is the one that handles DevOp.pre.
void fuse_pulses(Program& prog) {
  std::vector<DevOp> out;
  out.reserve(prog.ops.size());
  bool basic = true;  // only pulses, intervals and windows: the kernel variant that handles DevOp.pre
  for (auto& op : prog.ops) {
    op.pre = -1;
    if (op.kind == OP_RFTRAIN || op.kind == OP_CHIRP || op.kind == OP_GSAMP) basic = false;
  }
  if (!basic) return;
  for (size_t k = 0; k < prog.ops.size(); ++k) {
    const DevOp& op = prog.ops[k];
    if (op.kind == OP_ROT && k + 1 < prog.ops.size() &&
        (prog.ops[k + 1].kind == OP_EVENT || prog.ops[k + 1].kind == OP_WINDOW)) {
      DevOp next = prog.ops[k + 1];
      next.pre = static_cast<int32_t>(prog.mats.size() / 9);
      prog.mats.insert(prog.mats.end(), op.p, op.p + 9);
      // hard pulses about x (phi = 0) or y (phi = pi/2; cos(pi/2) leaves ~6e-17 terms): 4-entry rotation
      const double* m = op.p;
      auto tiny = [](double v) { return std::fabs(v) <= 1e-15; };
      if (tiny(m[0] - 1.0) && tiny(m[1]) && tiny(m[2]) && tiny(m[3]) && tiny(m[6]))
        next.tmode = 1;
      else if (tiny(m[4] - 1.0) && tiny(m[1]) && tiny(m[3]) && tiny(m[5]) && tiny(m[7]))
        next.tmode = 2;
      else
        next.tmode = 0;
      out.push_back(next);
      prog.n_fused_pulses++;
      ++k;
      continue;
    }
    out.push_back(op);
  }
  prog.ops.swap(out);
}

// Chirp classes (program.h ChirpClass): a ramp that recurs (every EPI line) is
// tabulated once per spin; OP_CHIRP.rot then indexes the chirp table.
void find_chirp_classes(Program& prog) {
  constexpr size_t kMaxChirp = 16;
  using Key = std::array<double, 7>;
  std::map<Key, int64_t> uses;
  auto key_of = [](const DevOp& op) { return Key{op.p[0], op.p[1], op.p[2], op.p[3], op.p[4], op.p[5], op.p[6]}; };
  for (const DevOp& op : prog.ops)
    if (op.kind == OP_CHIRP) uses[key_of(op)]++;
  std::map<Key, int32_t> ids;
  for (DevOp& op : prog.ops) {
    if (op.kind != OP_CHIRP) continue;
    const Key k = key_of(op);
    op.rot = -1;
    // a ramp that occurs once (e.g. cut short by a snapshot) is a class too: tabulating it costs what its
    // on-the-fly evaluation would, and a program whose chirps are all classes can be fully deferred
    auto f = ids.find(k);
    if (f == ids.end()) {
      if (prog.chirp_classes.size() >= kMaxChirp) continue;
      ChirpClass cc{};
      cc.dt = k[0];
      for (int a = 0; a < 3; ++a) {
        cc.d0[a] = k[1 + a];
        cc.dd[a] = k[4 + a];
      }
      f = ids.emplace(k, static_cast<int32_t>(prog.chirp_classes.size())).first;
      prog.chirp_classes.push_back(cc);
    }
    op.rot = f->second;
  }
}

// Planes (program.h PlaneDesc): every class quantity an op reads becomes a plane
// id in DevOp.pl; identical planes are stored once.  Pure gradient phases
// (T = 0, tw = 0) are kept with a canonical sign, so a ramp and its mirror share
// one q plane (the op conjugates).  Progression running factors are rewritten in
// place and are never shared.
void assign_planes(Program& prog) {
  using Key = std::array<double, 7>;
  std::map<Key, int32_t> ids;
  auto plane = [&](int32_t kind, int32_t flags, double T, const double* d, double tw) -> int32_t {
    PlaneDesc pd{};
    pd.kind = kind;
    pd.flags = flags;
    pd.T = T;
    for (int a = 0; a < 3; ++a) pd.d[a] = kind == PL_PHASE ? d[a] : 0.0;
    pd.tw = kind == PL_PHASE ? tw : 0.0;
    const Key key{static_cast<double>(kind * 16 + flags), pd.T, pd.d[0], pd.d[1], pd.d[2], pd.tw, 0.0};
    if (!(flags & PL_MUTABLE)) {
      auto f = ids.find(key);
      if (f != ids.end()) return f->second;
    }
    const int32_t id = static_cast<int32_t>(prog.planes.size());
    prog.planes.push_back(pd);
    if (!(flags & PL_MUTABLE)) ids.emplace(key, id);
    return id;
  };
  const double zero[3] = {0.0, 0.0, 0.0};
  // pure gradient phase with a canonical sign: returns the plane, sets conj when d was negated
  auto gphase = [&](const double* d, bool& conj) {
    double c[3] = {d[0], d[1], d[2]};
    conj = false;
    for (int a = 0; a < 3; ++a)
      if (c[a] != 0.0) {
        conj = c[a] < 0.0;
        break;
      }
    if (conj)
      for (int a = 0; a < 3; ++a) c[a] = -c[a];
    return plane(PL_PHASE, PL_SAMPLE, 0.0, c, 0.0);
  };
  std::vector<std::array<int32_t, 4>> prog_pl(prog.prog_classes.size(), {-1, -1, -1, -1});
  for (size_t k = 0; k < prog.prog_classes.size(); ++k) {
    const ProgClass& pc = prog.prog_classes[k];
    const double two[3] = {2.0 * pc.step[0], 2.0 * pc.step[1], 2.0 * pc.step[2]};
    prog_pl[k] = {plane(PL_PHASE, PL_MUTABLE, pc.dt, pc.d0, pc.dt), plane(PL_PHASE, 0, 0.0, pc.step, 0.0),
                  plane(PL_PHASE, 0, 0.0, two, 0.0), plane(PL_AB, 0, pc.dt, zero, 0.0)};
  }
  for (DevOp& op : prog.ops) {
    op.pl[0] = op.pl[1] = op.pl[2] = op.pl[3] = -1;
    if ((op.kind == OP_EVENT || op.kind == OP_WINDOW) && op.rot >= 0) {
      const RotClass& rc = prog.rot_classes[op.rot];
      const double T = rc.pre[0] + rc.main[0] * rc.mult + rc.post[0];
      double d[3];
      for (int a = 0; a < 3; ++a) d[a] = rc.pre[1 + a] + rc.main[1 + a] * rc.mult + rc.post[1 + a];
      const int32_t C = plane(PL_PHASE, 0, T, d, T), AB = plane(PL_AB, 0, T, zero, 0.0);
      if (op.kind == OP_EVENT) {
        op.pl[0] = C;
        op.pl[1] = AB;
      } else {
        op.pl[0] = plane(PL_PHASE, PL_WEIGHT | PL_SAMPLE, rc.pre[0], rc.pre + 1, rc.pre[0]);
        op.pl[1] = plane(PL_PHASE, PL_SAMPLE, rc.main[0], rc.main + 1, rc.main[0]);
        op.pl[2] = C;
        op.pl[3] = AB;
      }
    } else if (op.kind == OP_EVENT && op.prg >= 0) {
      for (int q = 0; q < 4; ++q) op.pl[q] = prog_pl[op.prg][q];
    } else if (op.kind == OP_CHIRP && op.rot >= 0) {
      // sample k applies (dt, d0 + k dd): r_k = r0 q^k; the whole run is (K dt, K d0 + K(K-1)/2 dd)
      const ChirpClass& cc = prog.chirp_classes[op.rot];
      const double K = static_cast<double>(op.count), tri = 0.5 * K * (K - 1.0);
      double d[3];
      for (int a = 0; a < 3; ++a) d[a] = K * cc.d0[a] + tri * cc.dd[a];
      bool conj = false;
      op.pl[0] = plane(PL_PHASE, PL_SAMPLE, cc.dt, cc.d0, cc.dt);
      op.pl[1] = gphase(cc.dd, conj);
      op.pl[2] = plane(PL_PHASE, 0, K * cc.dt, d, K * cc.dt);
      op.pl[3] = plane(PL_AB, 0, K * cc.dt, zero, 0.0);
      op.tmode = conj ? 1 : 0;
    }
  }
}

// Train classes (program.h TrainClass): an RF train that recurs with bit-identical
// sub-pulse matrices and interval (the same shaped pulse under the same gradient,
// sequence.py:650-674, repeated every line) is composed once per spin into its
// affine propagator; OP_RFTRAIN.rot then indexes the train table.  A run that
// occurs once stays on the fly (composing costs ~4 passes of the train).
void find_train_classes(Program& prog) {
  constexpr size_t kMaxTrain = 8;
  using Key = std::vector<double>;
  auto key_of = [&](const DevOp& op) {
    Key k(op.p, op.p + 4);
    k.push_back(static_cast<double>(op.count));
    k.push_back(static_cast<double>(op.flags));
    const double* m = prog.mats.data() + 9 * static_cast<size_t>(op.aux);
    k.insert(k.end(), m, m + 9 * static_cast<size_t>(op.count));
    return k;
  };
  std::map<Key, int64_t> uses;
  for (const DevOp& op : prog.ops)
    if (op.kind == OP_RFTRAIN) uses[key_of(op)]++;
  std::map<Key, int32_t> ids;
  for (DevOp& op : prog.ops) {
    if (op.kind != OP_RFTRAIN) continue;
    const Key k = key_of(op);
    op.rot = -1;
    if (uses[k] < 2) continue;
    auto f = ids.find(k);
    if (f == ids.end()) {
      if (prog.train_classes.size() >= kMaxTrain) continue;
      TrainClass tc{};
      tc.aux = op.aux;
      tc.count = op.count;
      tc.flags = op.flags;
      for (int a = 0; a < 4; ++a) tc.p[a] = op.p[a];
      f = ids.emplace(k, static_cast<int32_t>(prog.train_classes.size())).first;
      prog.train_classes.push_back(tc);
    }
    op.rot = f->second;
    prog.n_train_class_ops++;
  }
}

// Progression classes for the intervals left on the fly (program.h ProgClass).
// Within each group of equal dt (op order), members are partitioned greedily
// into arithmetic series d_j = d_prev + m*step, m in {1, 2}; a 1-member series
// takes a second member only if the series it would start continues later in
// the group (lookahead), so interleaved series (TSE blip-in / blip-out) split
// correctly.  Series of >= 3 members become classes (at most kMaxProg).
void find_progressions(Program& prog) {
  constexpr size_t kMaxProg = 32;
  constexpr int kLook = 6;
  std::map<double, std::vector<size_t>> groups;
  for (size_t k = 0; k < prog.ops.size(); ++k) {
    const DevOp& op = prog.ops[k];
    if (op.kind == OP_EVENT && op.rot < 0 && (op.count & EV_MOVE)) groups[op.p[0]].push_back(k);
  }
  auto close = [](const double* a, const double* b) {
    const double mag = std::max(inf_norm(a), inf_norm(b));
    for (int c = 0; c < 3; ++c)
      if (std::fabs(a[c] - b[c]) > 1e-9 * mag) return false;
    return true;
  };
  for (auto& g : groups) {
    const std::vector<size_t>& mem = g.second;
    if (mem.size() < 3) continue;
    struct Series {
      std::vector<size_t> idx;
      std::vector<int> mult;  // multiple of step from the previous member
      double step[3];
      bool has_step = false;
    };
    std::vector<Series> ser;
    auto dm = [&](size_t k) { return prog.ops[k].p + 1; };
    for (size_t a = 0; a < mem.size(); ++a) {
      const double* x = dm(mem[a]);
      bool placed = false;
      for (Series& s : ser) {  // continue a series with a known step
        if (!s.has_step) continue;
        const double* last = dm(s.idx.back());
        for (int m = 1; m <= 2 && !placed; ++m) {
          double pred[3];
          for (int c = 0; c < 3; ++c) pred[c] = last[c] + m * s.step[c];
          if (close(x, pred)) {
            s.idx.push_back(mem[a]);
            s.mult.push_back(m);
            placed = true;
          }
        }
        if (placed) break;
      }
      for (size_t si = 0; si < ser.size() && !placed; ++si) {  // second member of a 1-member series?
        Series& s = ser[si];
        if (s.has_step) continue;
        const double* last = dm(s.idx.back());
        double step[3], pred[3];
        for (int c = 0; c < 3; ++c) {
          step[c] = x[c] - last[c];
          pred[c] = x[c] + step[c];
        }
        if (inf_norm(step) == 0.0) continue;
        bool continues = false;
        for (size_t b = a + 1; b < mem.size() && b <= a + kLook && !continues; ++b) continues = close(dm(mem[b]), pred);
        if (continues) {
          s.idx.push_back(mem[a]);
          s.mult.push_back(1);
          for (int c = 0; c < 3; ++c) s.step[c] = step[c];
          s.has_step = true;
          placed = true;
        }
      }
      if (!placed) {
        Series s;
        s.idx.push_back(mem[a]);
        s.mult.push_back(0);
        ser.push_back(s);
      }
    }
    for (const Series& s : ser) {
      if (s.idx.size() < 3 || prog.prog_classes.size() >= kMaxProg) continue;
      ProgClass pc{};
      pc.dt = g.first;
      for (int c = 0; c < 3; ++c) {
        pc.d0[c] = dm(s.idx[0])[c];
        pc.step[c] = s.step[c];
      }
      const int32_t id = static_cast<int32_t>(prog.prog_classes.size());
      prog.prog_classes.push_back(pc);
      for (size_t j = 0; j < s.idx.size(); ++j) {
        DevOp& op = prog.ops[s.idx[j]];
        op.prg = id;
        op.flags = j + 1 < s.idx.size() ? s.mult[j + 1] : 0;  // advance to the next member: C *= q^m
      }
      prog.n_prog_intervals += static_cast<int64_t>(s.idx.size());
    }
  }
}

}  // namespace bloch
