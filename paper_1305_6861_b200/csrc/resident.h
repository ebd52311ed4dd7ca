// The resident-table integrator: the deferred-window program (program.h, Program::dops) run with every
// per-spin class table of a CTA's spins held in shared memory for the whole launch.
//
// The reference evaluates each event's rotation and relaxation per spin (engine.py:288-302); the op
// program replaces them by per-spin class tables ("planes", plane_kernel).  integrate_kernel re-reads
// those planes from L2 at every op: on config 2 that is 1569 ops x ~40 B per spin, 47 GB per launch
// through an L2 that delivers ~12 TB/s — the kernel's actual bound.  A program only has a few dozen
// planes (config 2: 17, 248 B per spin), so one CTA can keep the planes of ~900 spins in its 227 KB of
// shared memory: each plane value crosses L2 once per launch, every op reads 16-byte words at
// shared-memory latency, and the progression running factors are updated in place.  One spin per
// thread, the fp64 state in registers, the op stream decoded from compact 48-byte records.
//
// Eligible programs: fp32 mode, every window deferred (OP_UWIN / OP_UCHIRP), RF trains tabulated
// (train classes).  Programs with on-the-fly chirps, generic sampled events or in-kernel windows keep
// integrate_kernel.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "program.h"
#include "program_host.h"

namespace bloch {

enum ROpKind : int32_t {
  R_NOP = 0,     // only the fused pulse (a standalone OP_ROT)
  R_TAB = 1,     // OP_EVENT of a rotation class: m+ *= C, mz = A mz + B            off: C, AB
  R_PROG = 2,    // OP_EVENT of a progression: the running factor, then *= q^adv     off: run, q, q^2, AB
  R_FLY = 3,     // OP_EVENT evaluated per spin (engine.py:288-302)                  src: the DevOp
  R_UWIN = 4,    // OP_UWIN: store u = Cpre m (z), apply the exit propagator         off: Cpre, z, C, AB
  R_UCHIRP = 5,  // OP_UCHIRP: store u = w m, apply the run's closed form            off: -, -, C, AB
  R_TRAIN = 6    // OP_RFTRAIN of a train class: m = A m + b                          off[0]: 6 x 16 B
};

struct alignas(16) ROp {
  int32_t kind;
  int32_t pre;     // fused hard pulse applied first: index into the plan's matrices, -1 = none
  int32_t tmode;   // axis of `pre`: 1 x, 2 y, 0 general
  int32_t aux;     // events: snapshot index or -1; R_UWIN: lead flag
  int32_t off[4];  // per-thread byte offsets of the op's tables in the CTA's resident area (x blockDim)
  int32_t s0;      // R_UWIN / R_UCHIRP: U row
  int32_t flags;   // R_FLY: EV_* flags; R_PROG: advance (0, 1, 2)
  int32_t cls;     // R_FLY: relax class or -1
  int32_t src;     // index of the DevOp (R_FLY: dt and moments)
};
static_assert(sizeof(ROp) == 48, "ROp must be 48 bytes");

// one table copied into the resident area at kernel start
struct RLoad {
  int32_t kind;  // 0: double2 plane, 1: float2 plane (PL_SAMPLE), 2: one 16-byte word of a train-class row
  int32_t id;    // plane id, or train class
  int32_t word;  // kind 2: word 0..5 of the 96-byte row
  int32_t off;   // per-thread byte offset
};

struct ResidentPlan {
  bool ok = false;
  std::vector<ROp> rops;
  std::vector<RLoad> loads;
  std::vector<double> mats;   // distinct general fused pulse matrices, 9 doubles each
  std::vector<double> mats4;  // distinct rotations about x / y: (r4, r5, r7, r8) / (r0, r2, r6, r8)
  int32_t bytes_per_spin = 0;
};

constexpr int kResidentMaxMats = 128;
constexpr int kResidentMaxMats4 = 1024;
constexpr int kResidentMaxThreads = 1024;
constexpr int kResidentMinThreads = 128;   // below this many spins per CTA the resident tables do not pay
constexpr int kResidentTwoSpinMin = 768;   // CTAs of at least this many spins run two spins per thread
constexpr int kResidentSmemBytes = 227 * 1024;

// Compile the deferred program into resident form; plan.ok = false when an op is not covered.
void resident_compile(const Program& P, ResidentPlan& plan);

struct RParams {
  const ROp* rops;
  int32_t n_rops;
  const RLoad* loads;
  int32_t n_loads;
  const double* mats;
  int32_t n_mats;
  const double* mats4;
  int32_t n_mats4;
  const DevOp* ops;              // the deferred program (R_FLY reads dt and the moments)
  int64_t n;
  const double *mx0, *my0, *mz0;
  const double2* planes;
  const float2* planes32;
  const double* train;
  const void* sc;                // SpinConst records
  const double* relax;
  const double2* w1;             // single-coil receive weight (R_UCHIRP), or nullptr
  double* snaps;
  uint32_t *uhi, *ulo;
  int64_t urows;
  int32_t n_big, bd_big, bd_small;  // CTAs [0, n_big) run bd_big threads, the rest bd_small (ResidentShape)
};

// the launch of n spins: `grid` CTAs of `block` threads, of which the first n_big use bd_big threads and the rest
// bd_small (a CTA's spins: spins_per_thread x its threads, consecutive)
struct ResidentShape {
  int grid, block, n_big, bd_big, bd_small;
};
void resident_grid(int64_t n, int n_sm, int threads, int spins_per_thread, ResidentShape* out);

// threads per CTA and spins per thread (1 or 2) for n spins on n_sm SMs (0: the tables of
// kResidentMinThreads spins do not fit)
int resident_threads(const ResidentPlan& plan, int64_t n, int n_sm, int* spins_per_thread);
cudaError_t launch_resident(const RParams& rp, const ResidentPlan& plan, int spins_per_thread, int grid, int threads,
                            cudaStream_t stream);

}  // namespace bloch
