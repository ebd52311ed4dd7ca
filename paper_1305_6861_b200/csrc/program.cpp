// Host compiler: flattened OperatorTables -> device op stream.
//
// Input is exactly the reference's EsTable content (engine.py:51-70) flattened
// into SoA arrays by the caller.  Output: DevOp stream + GEv / matrix side
// tables + the compact-sample -> output-position map.  See program.h for the
// op set.  The walk order is the reference's (engine.py:276-308): per ES the
// pulse, then its events in order; every compiled op covers a contiguous run
// of that walk, so the device replays the same operator sequence.
#include "program_host.h"

#include <algorithm>
#include <cmath>
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
    if (!(t.ev_dt[i] >= 0.0)) throw std::invalid_argument("negative or NaN event interval");
  }

  auto dm = [&](int64_t i) { return t.ev_dmom + 3 * i; };
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
}

}  // namespace bloch
