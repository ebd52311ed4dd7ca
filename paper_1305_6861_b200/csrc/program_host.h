// Host-side view of the flattened tables and the compiled program.
#pragma once
#include <stdint.h>

#include <vector>

#include "program.h"

namespace bloch {

struct TablesView {  // borrowed pointers, see bloch_set_tables() in include/bloch_b200.h
  int32_t n_es;
  const int64_t* es_ev_offset;
  const uint8_t* es_has_pulse;
  const double* es_pulse_mat;
  const int32_t* es_acq;
  const double* ev_dt;
  const double* ev_dmom;
  const uint8_t* ev_sample;
  const int32_t* ev_snap;
  int32_t n_acq, max_samples, n_snap;
};

struct Program {
  std::vector<DevOp> ops;
  std::vector<GEv> gev;
  std::vector<double> mats;       // OP_RFTRAIN side table, 9 doubles (row-major) per pair
  std::vector<int64_t> sample_g;  // compact sample -> acq * max_samples + index
  std::vector<double> relax_t;    // interval length of every relax class
  std::vector<RotClass> rot_classes;
  std::vector<ProgClass> prog_classes;
  std::vector<ChirpClass> chirp_classes;
  std::vector<TrainClass> train_classes;
  std::vector<PlaneDesc> planes;  // per-spin class quantities (assign_planes)
  int32_t n_acq = 0, max_samples = 0, n_snap = 0;
  int64_t n_events = 0;  // reference table size incl. pulses
  int64_t n_samples = 0;
  int64_t n_rot = 0, n_interval = 0, n_window_ops = 0, n_window_samples = 0, n_gsamp_events = 0;
  int64_t n_chirp_ops = 0, n_chirp_samples = 0, n_train_ops = 0, n_train_pairs = 0;
  int64_t n_fused_windows = 0, n_fused_intervals = 0, n_prog_intervals = 0, n_fused_pulses = 0;
  int64_t n_train_class_ops = 0;  // RF trains applied from the train table
  // deferred-window view of the same program (defer_windows): tabulated windows of >= kMinDeferWindow
  // samples become OP_UWIN; every other sampled op keeps its samples, renumbered compactly (dsample_g)
  std::vector<DevOp> dops;
  std::vector<int64_t> dsample_g;
  std::vector<WinGroup> groups;
  std::vector<int64_t> urow_out0;  // per U row: output index (acq * max_samples + first sample)
  int64_t n_deferred_samples = 0;
};

// Throws std::invalid_argument on malformed tables.
void compile_program(const TablesView& t, Program& prog);

}  // namespace bloch
