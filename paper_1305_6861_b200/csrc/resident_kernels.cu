// resident_integrate_kernel — see resident.h.  One spin per thread; the spin's class tables sit in the
// CTA's shared memory as [table][thread] words (consecutive threads, consecutive 16 or 8 bytes: every
// access is a conflict-free LDS.128 / LDS.64), the fp64 state in registers.  Restates the same walk as
// integrate_kernel's deferred-window variant (engine.py:276-308 per op kind, see program.h).
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <array>

#include "contract.h"
#include "kernels.h"
#include "resident.h"

namespace bloch {

// ---------------------------------------------------------------------------
// host: the resident plan of a deferred program
// ---------------------------------------------------------------------------

void resident_compile(const Program& P, ResidentPlan& plan) {
  plan = ResidentPlan{};
  const std::vector<DevOp>& ops = P.dops;
  if (ops.empty() || P.groups.empty()) return;
  const int n_planes = static_cast<int>(P.planes.size());
  std::vector<int32_t> plane_off(n_planes, -1);
  std::vector<int32_t> train_off(P.train_classes.size(), -1);
  std::vector<uint8_t> want(n_planes, 0), want_train(P.train_classes.size(), 0);
  // fused pulses, deduplicated: general ones as 9 entries, rotations about x or y as the 4 entries the
  // kernel uses (a TSE train with per-echo flip angles has hundreds of distinct ones)
  std::map<std::array<uint64_t, 9>, int32_t> mat_ids;
  std::map<std::array<uint64_t, 4>, int32_t> mat4_ids;
  auto mat_id = [&](const double* m, int mode) -> int32_t {
    if (mode == 1 || mode == 2) {
      const double v[4] = {mode == 1 ? m[4] : m[0], mode == 1 ? m[5] : m[2], mode == 1 ? m[7] : m[6], m[8]};
      std::array<uint64_t, 4> key;
      std::memcpy(key.data(), v, 32);
      auto it = mat4_ids.find(key);
      if (it != mat4_ids.end()) return it->second;
      const int32_t id = static_cast<int32_t>(plan.mats4.size() / 4);
      plan.mats4.insert(plan.mats4.end(), v, v + 4);
      mat4_ids.emplace(key, id);
      return id;
    }
    std::array<uint64_t, 9> key;
    std::memcpy(key.data(), m, 72);
    auto it = mat_ids.find(key);
    if (it != mat_ids.end()) return it->second;
    const int32_t id = static_cast<int32_t>(plan.mats.size() / 9);
    plan.mats.insert(plan.mats.end(), m, m + 9);
    mat_ids.emplace(key, id);
    return id;
  };
  auto need = [&](int32_t pl) -> bool {
    if (pl < 0 || pl >= n_planes) return false;
    want[pl] = 1;
    return true;
  };
  // pass 1: coverage and the set of tables
  for (const DevOp& op : ops) {
    bool ok = true;
    switch (op.kind) {
      case OP_ROT: break;
      case OP_EVENT:
        if (op.rot >= 0) ok = need(op.pl[0]) && need(op.pl[1]);
        else if (op.prg >= 0) {
          ok = need(op.pl[0]) && need(op.pl[3]);
          if (op.flags == 1) ok = ok && need(op.pl[1]);
          if (op.flags == 2) ok = ok && need(op.pl[2]);
          ok = ok && op.flags >= 0 && op.flags <= 2 && (P.planes[op.pl[0]].flags & PL_SAMPLE) == 0;
        }
        break;
      case OP_UWIN: ok = need(op.pl[0]) && need(op.pl[1]) && need(op.pl[2]) && need(op.pl[3]); break;
      case OP_UCHIRP: ok = need(op.pl[2]) && need(op.pl[3]); break;
      case OP_RFTRAIN:
        ok = op.rot >= 0 && op.rot < static_cast<int32_t>(want_train.size());
        if (ok) want_train[op.rot] = 1;
        break;
      default: ok = false;
    }
    if (!ok) {
      if (getenv("BLOCH_RESIDENT_DEBUG")) fprintf(stderr, "resident: op kind %d rot %d prg %d flags %d pl %d %d %d %d not covered\n", op.kind, op.rot, op.prg, op.flags, op.pl[0], op.pl[1], op.pl[2], op.pl[3]);
      return;
    }
  }
  // resident layout: 16-byte tables first (double2 planes, train rows), then the float2 planes
  int32_t off = 0;
  for (int p = 0; p < n_planes; ++p)
    if (want[p] && !(P.planes[p].flags & PL_SAMPLE)) {
      plane_off[p] = off;
      plan.loads.push_back(RLoad{0, p, 0, off});
      off += 16;
    }
  for (size_t t = 0; t < want_train.size(); ++t)
    if (want_train[t]) {
      train_off[t] = off;
      for (int k = 0; k < 6; ++k) plan.loads.push_back(RLoad{2, static_cast<int32_t>(t), k, off + 16 * k});
      off += 96;
    }
  for (int p = 0; p < n_planes; ++p)
    if (want[p] && (P.planes[p].flags & PL_SAMPLE)) {
      plane_off[p] = off;
      plan.loads.push_back(RLoad{1, p, 0, off});
      off += 8;
    }
  plan.bytes_per_spin = off;
  // pass 2: the records
  plan.rops.reserve(ops.size());
  for (size_t o = 0; o < ops.size(); ++o) {
    const DevOp& op = ops[o];
    ROp r{};
    r.pre = -1;
    r.aux = -1;
    r.cls = -1;
    r.src = static_cast<int32_t>(o);
    for (int k = 0; k < 4; ++k) r.off[k] = 0;
    auto fused = [&] {
      if (op.pre >= 0) {
        r.tmode = (op.tmode == 1 || op.tmode == 2) ? op.tmode : 0;
        r.pre = mat_id(P.mats.data() + 9 * static_cast<size_t>(op.pre), r.tmode);
      }
    };
    switch (op.kind) {
      case OP_ROT:
        r.kind = R_NOP;
        r.pre = mat_id(op.p, 0);
        r.tmode = 0;
        break;
      case OP_EVENT:
        fused();
        r.aux = op.aux;
        if (op.rot >= 0) {
          r.kind = R_TAB;
          r.off[0] = plane_off[op.pl[0]];
          r.off[1] = plane_off[op.pl[1]];
        } else if (op.prg >= 0) {
          r.kind = R_PROG;
          r.flags = op.flags;
          r.off[0] = plane_off[op.pl[0]];
          r.off[1] = op.flags == 2 ? plane_off[op.pl[2]] : op.flags == 1 ? plane_off[op.pl[1]] : 0;
          r.off[3] = plane_off[op.pl[3]];
        } else {
          r.kind = R_FLY;
          r.flags = op.count;
          r.cls = op.cls;
        }
        break;
      case OP_UWIN:
        fused();
        r.kind = R_UWIN;
        r.aux = op.aux;
        r.s0 = op.s0;
        for (int k = 0; k < 4; ++k) r.off[k] = plane_off[op.pl[k]];
        // Cpre and z feed fp32 samples only: they must be the float2 tables, C and AB the double2 ones
        if (!(P.planes[op.pl[0]].flags & PL_SAMPLE) || !(P.planes[op.pl[1]].flags & PL_SAMPLE) ||
            (P.planes[op.pl[2]].flags & PL_SAMPLE) || (P.planes[op.pl[3]].flags & PL_SAMPLE)) {
          if (getenv("BLOCH_RESIDENT_DEBUG")) fprintf(stderr, "resident: UWIN plane kinds %d %d %d %d\n", P.planes[op.pl[0]].flags, P.planes[op.pl[1]].flags, P.planes[op.pl[2]].flags, P.planes[op.pl[3]].flags);
          return;
        }
        break;
      case OP_UCHIRP:
        fused();
        r.kind = R_UCHIRP;
        r.s0 = op.s0;
        r.off[2] = plane_off[op.pl[2]];
        r.off[3] = plane_off[op.pl[3]];
        if ((P.planes[op.pl[2]].flags & PL_SAMPLE) || (P.planes[op.pl[3]].flags & PL_SAMPLE)) return;
        break;
      case OP_RFTRAIN:
        r.kind = R_TRAIN;
        r.off[0] = train_off[op.rot];
        break;
      default: return;
    }
    if ((op.kind == OP_EVENT && op.rot >= 0) &&
        ((P.planes[op.pl[0]].flags & PL_SAMPLE) || (P.planes[op.pl[1]].flags & PL_SAMPLE)))
      return;
    plan.rops.push_back(r);
  }
  if (getenv("BLOCH_RESIDENT_DEBUG"))
    fprintf(stderr, "resident: %zu + %zu matrices, %d bytes per spin\n", plan.mats.size() / 9, plan.mats4.size() / 4,
            plan.bytes_per_spin);
  if (plan.mats.size() / 9 > static_cast<size_t>(kResidentMaxMats) ||
      plan.mats4.size() / 4 > static_cast<size_t>(kResidentMaxMats4))
    return;
  plan.ok = true;
}

constexpr int kResidentFixedBytes = 2 * 64 * 32;  // the two staged record chunks (kRecChunk x 32 B)

// shared memory ahead of the tables: the axis pulses (32 B each), then the general ones (80 B each: 9
// entries padded so that every matrix starts on a 16-byte boundary)
static size_t resident_mats_bytes(const ResidentPlan& plan) { return plan.mats4.size() * 8 + plan.mats.size() / 9 * 80; }

// BLOCH_RESIDENT_UNEVEN=1: equal CTAs of whole warps with a ragged last wave (the earlier launch, kept as the
// A/B reference); =0 / unset: two-spin launches deal the spins in units over full waves (resident_grid)
static int resident_uneven_mode() {
  static const int mode = [] {
    const char* e = getenv("BLOCH_RESIDENT_UNEVEN");
    return e ? (atoi(e) ? 1 : 0) : -1;
  }();
  return mode;
}

constexpr int kDealThreads = 4;  // dealing unit of a two-spin launch: 4 threads = 8 spins (one 32-byte U sector)

int resident_threads(const ResidentPlan& plan, int64_t n, int n_sm, int* spins_per_thread) {
  if (!plan.ok || n <= 0) return 0;
  const int64_t room = kResidentSmemBytes - kResidentFixedBytes - static_cast<int64_t>(resident_mats_bytes(plan));
  const int64_t fit = plan.bytes_per_spin > 0 ? room / plan.bytes_per_spin : kResidentMaxThreads;  // spins per CTA
  static const int force_s = [] {  // experiment hook: BLOCH_RESIDENT_SPINS=1|2
    const char* e = getenv("BLOCH_RESIDENT_SPINS");
    return e ? atoi(e) : 0;
  }();
  // two spins per thread, CTA sizes in units of 8 spins: the tables decide how many spins a CTA holds, not the
  // warp rounding (config 2: 1016 of the 1019 that fit, so 5 waves instead of 6 at 896)
  if (resident_uneven_mode() != 1 && force_s != 1) {
    const int64_t u = 2 * kDealThreads;
    const int64_t cap = std::min<int64_t>(kResidentMaxThreads, (fit / u) * u);
    if (cap >= kResidentTwoSpinMin) {
      const int64_t per_wave = static_cast<int64_t>(n_sm) * cap;
      const int64_t waves = (n + per_wave - 1) / per_wave;
      int64_t spins = (n + n_sm * waves - 1) / (n_sm * waves);  // per CTA
      if (spins >= kResidentTwoSpinMin || force_s == 2) {
        spins = std::max<int64_t>(u, std::min<int64_t>(cap, ((spins + u - 1) / u) * u));
        if (spins_per_thread) *spins_per_thread = 2;
        return static_cast<int>(spins / 2);
      }
    }
  }
  // whole warps, with 1 KB of the budget left free (as measured so far)
  int64_t cap = plan.bytes_per_spin > 0 ? (room - 1024) / plan.bytes_per_spin : kResidentMaxThreads;
  cap = std::min<int64_t>(kResidentMaxThreads, (cap / 64) * 64);
  if (cap < kResidentMinThreads) return 0;
  // equal waves of one CTA per SM
  const int64_t per_wave = static_cast<int64_t>(n_sm) * cap;
  const int64_t waves = (n + per_wave - 1) / per_wave;
  int64_t spins = (n + n_sm * waves - 1) / (n_sm * waves);  // per CTA
  // two spins per thread amortise the record decode, the pulse loads and the branches; one spin per thread
  // keeps enough warps when a CTA has few spins (shards)
  int S = spins >= kResidentTwoSpinMin ? 2 : 1;
  if (force_s == 1 || force_s == 2) S = force_s;
  const int64_t q = 32 * S;
  spins = ((spins + q - 1) / q) * q;
  spins = std::max<int64_t>(q, std::min<int64_t>(cap, spins));
  if (spins_per_thread) *spins_per_thread = S;
  return static_cast<int>(spins / S);
}

void resident_grid(int64_t n, int n_sm, int threads, int spins_per_thread, ResidentShape* out) {
  ResidentShape r{};
  r.bd_big = r.bd_small = threads;
  r.block = ((threads + 31) / 32) * 32;
  const int64_t spc = static_cast<int64_t>(threads) * spins_per_thread;
  r.grid = r.n_big = static_cast<int>((n + spc - 1) / spc);
  // Two-spin launches: the spins are dealt in units of kDealThreads threads over n_sm x waves CTAs, so CTA sizes
  // differ by one unit and the last wave is as full as the others.  One-spin launches keep equal CTAs: there a
  // CTA's time hardly depends on its size (profiles/r4b_even_waves_ab.txt: config 4 -1.6%, config 3 +1.1%).
  if (spins_per_thread == 2 && resident_uneven_mode() != 1 && threads % kDealThreads == 0) {
    const int64_t us = static_cast<int64_t>(kDealThreads) * spins_per_thread;  // spins per unit
    const int64_t units = (n + us - 1) / us, ub = threads / kDealThreads;
    const int64_t waves = ((units + ub - 1) / ub + n_sm - 1) / n_sm;
    const int64_t ctas = waves * n_sm;
    const int64_t per = (units + ctas - 1) / ctas;       // units of a big CTA
    const int64_t extra = units - ctas * (per - 1);      // how many CTAs are big
    if (per >= 2 && extra >= 1 && extra <= ctas && per <= ub) {
      r.grid = static_cast<int>(ctas);
      r.n_big = static_cast<int>(extra);
      r.bd_big = static_cast<int>(per * kDealThreads);
      r.bd_small = static_cast<int>((per - 1) * kDealThreads);
      r.block = ((r.bd_big + 31) / 32) * 32;
    }
  }
  *out = r;
}

// ---------------------------------------------------------------------------
// device
// ---------------------------------------------------------------------------

namespace {

__device__ __forceinline__ double r_reduce_2pi(double th) {
  const double kInv2Pi = 0.15915494309189535;
  const double kHi = 6.283185307179586;
  const double kLo = 2.4492935982947064e-16;
  const double k = rint(th * kInv2Pi);
  return fma(-k, kLo, fma(-k, kHi, th));
}

// shared memory through 32-bit shared-window addresses (no generic-address arithmetic per access).  All
// volatile: the progression running factors are rewritten in place, so loads and stores keep program order.
__device__ __forceinline__ double2 lds_d2(uint32_t a) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ float2 lds_f2(uint32_t a) {
  float2 v;
  asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ int4 lds_i4(uint32_t a) {
  int4 v;
  asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts_d2(uint32_t a, double2 v) {
  asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(v.x), "d"(v.y) : "memory");
}
__device__ __forceinline__ void sts_f2(uint32_t a, float2 v) {
  asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(a), "f"(v.x), "f"(v.y) : "memory");
}
__device__ __forceinline__ void sts_i4(uint32_t a, int4 v) {
  asm volatile("st.shared.v4.s32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

// U word pair of an fp32 complex value (contract.h contract_split_f, same round-to-nearest-even words) with
// the packed bf16 conversion: hi = bf16x2 (Re, Im), lo = bf16x2 of the exact residuals
__device__ __forceinline__ void split_bf16x2(float re, float im, uint32_t& hi, uint32_t& lo) {
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(hi) : "f"(im), "f"(re));
  const float fr = __uint_as_float(hi << 16), fm = __uint_as_float(hi & 0xffff0000u);
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(lo) : "f"(im - fm), "f"(re - fr));
}

constexpr int kRecChunk = 64;  // staged records per chunk (two chunks of 32-byte records: 4 KB)

// staged op kinds: bit 2 = the common exit (m+ *= C, mz = A mz + B)
enum : int { SK_NOP = 0, SK_FLY = 1, SK_TRAIN = 2, SK_TAB = 4, SK_PROG = 5, SK_UWIN = 6, SK_UCHIRP = 7 };
constexpr int kSnapBit = 16;  // w0.z: the event takes a snapshot (index in w0.w)

// one interval evaluated per spin: precession (+ relaxation), engine.py:288-302 (rare: out of line)
// (state by value: a reference would pin the caller's state registers to local memory)
__device__ __noinline__ double3 fly_interval(const ROp* rop, const DevOp* ops, const void* sc, const double* relax,
                                             int64_t n, int64_t i, double x, double y, double z) {
  const int flags = __ldg(&rop->flags), cls = __ldg(&rop->cls);
  if (!(flags & EV_MOVE)) return make_double3(x, y, z);
  const DevOp* op = ops + __ldg(&rop->src);
  const double dt = __ldg(&op->p[0]), dmx = __ldg(&op->p[1]), dmy = __ldg(&op->p[2]), dmz = __ldg(&op->p[3]);
  const double2* s = reinterpret_cast<const double2*>(static_cast<const SpinConst*>(sc) + i);
  const double2 s0 = __ldg(s), s1 = __ldg(s + 1), s2 = __ldg(s + 2);  // (x, y), (z, dw), (m0, r1)
  const double2 e = cls >= 0 ? __ldg(reinterpret_cast<const double2*>(relax) + (static_cast<int64_t>(cls) * n + i))
                             : make_double2(1.0, 1.0);
  const double th = fma(s1.x, dmz, fma(s0.y, dmy, s0.x * dmx)) + s1.y * dt;  // engine.py:289
  double sn, cs;
  sincos(r_reduce_2pi(th), &sn, &cs);
  const double ms = -sn;
  const double nx = e.y * (cs * x - ms * y);  // clockwise: (c - i s)(x + i y), bloch.py:10-17
  y = e.y * (cs * y + ms * x);
  x = nx;
  if (cls >= 0) z = fma(z, e.x, s2.x * (1.0 - e.x));
  return make_double3(x, y, z);
}

}  // namespace

// Staged record (shared memory, 32 bytes), decoded once per chunk per CTA from the 48-byte ROp:
//   w0 = (staged kind, shared address of the fused pulse or 0, tmode | arg << 2 | snapshot bit,
//         U byte offset (windows) / snapshot index (events))
//   w1 = shared addresses (slot 0's word) of C, (A, B), and two more: PROG q; UWIN Cpre, z; TRAIN the row
// arg: UWIN lead flag, PROG advance.  A thread's word of slot s: + (s blockDim + tid) * 16 (or * 8).
template <int S>
__global__ void __launch_bounds__(kResidentMaxThreads / S, 1) resident_integrate_kernel(const RParams rp) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // CTAs [0, n_big) run bd_big threads, the rest bd_small (resident_grid); the launch's other threads leave
  // before the first barrier
  const int tid = threadIdx.x, cta = blockIdx.x;
  const int bd = cta < rp.n_big ? rp.bd_big : rp.bd_small;
  if (tid >= bd) return;
  const int64_t cta0 = cta < rp.n_big ? static_cast<int64_t>(cta) * (S * rp.bd_big)
                                      : static_cast<int64_t>(rp.n_big) * (S * rp.bd_big) +
                                            static_cast<int64_t>(cta - rp.n_big) * (S * rp.bd_small);
  const int64_t base = cta0 + tid;  // spin of slot 0; slot s: + s bd
  const uint32_t s_base = static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw));
  const uint32_t s_rec = s_base;                                    // [2][kRecChunk] staged records
  const uint32_t s_m4 = s_rec + 2 * kRecChunk * 32;                 // axis pulses, 32 B each
  const uint32_t s_m9 = s_m4 + 32u * rp.n_mats4;                    // general pulses, 80 B each
  const uint32_t s_area = s_m9 + 80u * rp.n_mats;                   // the tables, [table][slot][thread]
  {
    double* m4 = reinterpret_cast<double*>(smem_raw + 2 * kRecChunk * 32);
    double* m9 = m4 + 4 * rp.n_mats4;
    for (int k = tid; k < 4 * rp.n_mats4; k += bd) m4[k] = __ldg(rp.mats4 + k);
    for (int k = tid; k < 9 * rp.n_mats; k += bd) m9[(k / 9) * 10 + k % 9] = __ldg(rp.mats + k);
  }
  bool act[S];
  uint32_t t16[S], t8[S];
#pragma unroll
  for (int s = 0; s < S; ++s) {
    act[s] = base + s * bd < rp.n;
    t16[s] = (s * bd + tid) * 16;
    t8[s] = (s * bd + tid) * 8;
  }
  // the CTA's tables: each value crosses L2 once per launch
  for (int j = 0; j < rp.n_loads; ++j) {
    const RLoad* L = rp.loads + j;
    const int kind = __ldg(&L->kind), id = __ldg(&L->id);
    const uint32_t off = s_area + static_cast<uint32_t>(__ldg(&L->off)) * (S * bd);
    const int word = __ldg(&L->word);
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const int64_t i = base + s * bd;
      if (kind == 1) {
        sts_f2(off + t8[s], act[s] ? __ldg(rp.planes32 + (static_cast<int64_t>(id) * rp.n + i)) : make_float2(1.f, 0.f));
      } else if (kind == 0) {
        sts_d2(off + t16[s], act[s] ? __ldg(rp.planes + (static_cast<int64_t>(id) * rp.n + i)) : make_double2(1.0, 0.0));
      } else {
        sts_d2(off + t16[s], act[s] ? __ldg(reinterpret_cast<const double2*>(rp.train) +
                                           ((static_cast<int64_t>(id) * rp.n + i) * 6 + word))
                                    : make_double2(0.0, 0.0));
      }
    }
  }
  // stage chunk `ch` of the op records into buffer ch & 1
  auto stage = [&](int ch) {
    for (int r = tid; r < kRecChunk; r += bd) {
      const int o = ch * kRecChunk + r;
      if (o >= rp.n_rops) break;
      const int4* g = reinterpret_cast<const int4*>(rp.rops + o);
      const int4 a = __ldg(g), b = __ldg(g + 1), c = __ldg(g + 2);
      const int kind = a.x, pre = a.y, tmode = a.z;
      const uint32_t sb = S * bd;
      auto at = [&](int off) { return static_cast<int>(s_area + static_cast<uint32_t>(off) * sb); };
      int4 w0, w1 = make_int4(0, 0, 0, 0);
      int sk = SK_NOP, arg = 0;
      w0.w = a.w;  // events: snapshot index
      switch (kind) {
        case R_TAB: sk = SK_TAB; w1.x = at(b.x); w1.y = at(b.y); break;
        case R_PROG: sk = SK_PROG; arg = c.y; w1.x = at(b.x); w1.y = at(b.w); w1.z = at(b.y); break;
        case R_UWIN: sk = SK_UWIN; arg = a.w != 0; w0.w = c.x * 64; w1.x = at(b.z); w1.y = at(b.w); w1.z = at(b.x);
                     w1.w = at(b.y); break;
        case R_UCHIRP: sk = SK_UCHIRP; w0.w = c.x * 64; w1.x = at(b.z); w1.y = at(b.w); break;
        case R_TRAIN: sk = SK_TRAIN; w1.z = at(b.x); break;
        case R_FLY: sk = SK_FLY; break;
        default: break;
      }
      const bool snap = (kind == R_TAB || kind == R_PROG || kind == R_FLY) && a.w >= 0 && rp.snaps != nullptr;
      w0.x = sk;
      w0.y = pre < 0 ? 0 : static_cast<int>((tmode == 1 || tmode == 2) ? s_m4 + 32u * pre : s_m9 + 80u * pre);
      w0.z = tmode | (arg << 2) | (snap ? kSnapBit : 0);
      const uint32_t dst = s_rec + ((ch & 1) * kRecChunk + r) * 32;
      sts_i4(dst, w0);
      sts_i4(dst + 16, w1);
    }
  };
  stage(0);
  __syncthreads();  // the matrices and chunk 0 (the tables are read only by the thread that wrote them)

  double x[S], y[S], z[S];
  const char *uhi0[S], *ulo0[S];
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const int64_t i = base + s * bd;
    x[s] = act[s] ? rp.mx0[i] : 0.0;
    y[s] = act[s] ? rp.my0[i] : 0.0;
    z[s] = act[s] ? rp.mz0[i] : 0.0;
    // contract_u_index(rows, r, i) = ((i >> 4) rows + r) 16 + (i & 15): this spin's word of row 0
    const int64_t ub = act[s] ? (i >> 4) * rp.urows * 16 + (i & 15) : 0;
    uhi0[s] = reinterpret_cast<const char*>(rp.uhi + ub);
    ulo0[s] = reinterpret_cast<const char*>(rp.ulo + ub);
  }

  const int n_chunks = (rp.n_rops + kRecChunk - 1) / kRecChunk;
  for (int ch = 0; ch < n_chunks; ++ch) {
    if (ch + 1 < n_chunks) stage(ch + 1);  // lands during this chunk; the barrier below publishes it
    const int cnt = min(kRecChunk, rp.n_rops - ch * kRecChunk);
    uint32_t ra = s_rec + (ch & 1) * kRecChunk * 32;
    for (int r = 0; r < cnt; ++r, ra += 32) {
      const int4 w0 = lds_i4(ra), w1 = lds_i4(ra + 16);
      const int kind = w0.x;
      if (w0.y) {  // a fused hard pulse first (bloch.py:124-139)
        const uint32_t ma = static_cast<uint32_t>(w0.y);
        const int tmode = w0.z & 3;
        if (tmode == 1) {  // about x: (x, r4 y + r5 z, r7 y + r8 z)
          const double2 m0 = lds_d2(ma), m1 = lds_d2(ma + 16);
#pragma unroll
          for (int s = 0; s < S; ++s) {
            const double ny = m0.x * y[s] + m0.y * z[s];
            z[s] = m1.x * y[s] + m1.y * z[s];
            y[s] = ny;
          }
        } else if (tmode == 2) {  // about y: (r0 x + r2 z, y, r6 x + r8 z)
          const double2 m0 = lds_d2(ma), m1 = lds_d2(ma + 16);
#pragma unroll
          for (int s = 0; s < S; ++s) {
            const double nx = m0.x * x[s] + m0.y * z[s];
            z[s] = m1.x * x[s] + m1.y * z[s];
            x[s] = nx;
          }
        } else {
          const double2 m0 = lds_d2(ma), m1 = lds_d2(ma + 16), m2 = lds_d2(ma + 32), m3 = lds_d2(ma + 48);
          double m8;
          asm volatile("ld.shared.f64 %0, [%1];" : "=d"(m8) : "r"(ma + 64));
#pragma unroll
          for (int s = 0; s < S; ++s) {
            const double nx = m0.x * x[s] + m0.y * y[s] + m1.x * z[s];
            const double ny = m1.y * x[s] + m2.x * y[s] + m2.y * z[s];
            z[s] = m3.x * x[s] + m3.y * y[s] + m8 * z[s];
            x[s] = nx;
            y[s] = ny;
          }
        }
      }
      if (kind & 4) {  // m+ *= C, mz = A mz + B, after the kind's own work on the entry state
        double2 cc[S], ab[S];
#pragma unroll
        for (int s = 0; s < S; ++s) {
          cc[s] = lds_d2(static_cast<uint32_t>(w1.x) + t16[s]);
          ab[s] = lds_d2(static_cast<uint32_t>(w1.y) + t16[s]);
        }
        if (kind == SK_PROG) {
          if (w0.z & 12) {  // advance the running factor by q or q^2
#pragma unroll
            for (int s = 0; s < S; ++s) {
              const double2 q = lds_d2(static_cast<uint32_t>(w1.z) + t16[s]);
              sts_d2(static_cast<uint32_t>(w1.x) + t16[s],
                     make_double2(cc[s].x * q.x - cc[s].y * q.y, cc[s].x * q.y + cc[s].y * q.x));
            }
          }
        } else if (kind == SK_UWIN) {
          float2 cp[S], zz[S];
          const bool lead = (w0.z & 4) != 0;
#pragma unroll
          for (int s = 0; s < S; ++s) {
            cp[s] = lds_f2(static_cast<uint32_t>(w1.z) + t8[s]);
            if (!lead) zz[s] = lds_f2(static_cast<uint32_t>(w1.w) + t8[s]);
          }
#pragma unroll
          for (int s = 0; s < S; ++s) {
            // u = Cpre m in fp32 (two conversions of the state): equal to ~2^-24, inside the bf16 hi + lo split
            const float fx = static_cast<float>(x[s]), fy = static_cast<float>(y[s]);
            float ur = cp[s].x * fx - cp[s].y * fy, ui = cp[s].x * fy + cp[s].y * fx;
            if (!lead) {  // no leading no-op sample: the first sample follows one interval
              const float t = ur * zz[s].x - ui * zz[s].y;
              ui = ur * zz[s].y + ui * zz[s].x;
              ur = t;
            }
            if (act[s]) {
              uint32_t hi, lo;
              split_bf16x2(ur, ui, hi, lo);
              __stcs(reinterpret_cast<uint32_t*>(const_cast<char*>(uhi0[s] + w0.w)), hi);  // streamed: read by the
              __stcs(reinterpret_cast<uint32_t*>(const_cast<char*>(ulo0[s] + w0.w)), lo);  // contraction
            }
          }
        } else if (kind == SK_UCHIRP) {
#pragma unroll
          for (int s = 0; s < S; ++s) {
            if (!act[s]) continue;
            const double2 w = rp.w1 != nullptr ? __ldg(rp.w1 + (base + s * bd)) : make_double2(1.0, 0.0);
            const float wx = static_cast<float>(w.x), wy = static_cast<float>(w.y);
            const float fx = static_cast<float>(x[s]), fy = static_cast<float>(y[s]);
            uint32_t hi, lo;
            split_bf16x2(wx * fx - wy * fy, wx * fy + wy * fx, hi, lo);
            __stcs(reinterpret_cast<uint32_t*>(const_cast<char*>(uhi0[s] + w0.w)), hi);
            __stcs(reinterpret_cast<uint32_t*>(const_cast<char*>(ulo0[s] + w0.w)), lo);
          }
        }
#pragma unroll
        for (int s = 0; s < S; ++s) {
          const double nx = cc[s].x * x[s] - cc[s].y * y[s];
          y[s] = cc[s].x * y[s] + cc[s].y * x[s];
          x[s] = nx;
          z[s] = fma(z[s], ab[s].x, ab[s].y);
        }
      } else if (kind == SK_TRAIN) {
        const uint32_t st = 16u * S * bd;
#pragma unroll
        for (int s = 0; s < S; ++s) {
          const uint32_t ta = static_cast<uint32_t>(w1.z) + t16[s];
          const double2 t0 = lds_d2(ta), t1 = lds_d2(ta + st), t2 = lds_d2(ta + 2 * st), t3 = lds_d2(ta + 3 * st),
                        t4 = lds_d2(ta + 4 * st), t5 = lds_d2(ta + 5 * st);
          const double nx = fma(t0.x, x[s], fma(t0.y, y[s], fma(t1.x, z[s], t4.y)));
          const double ny = fma(t1.y, x[s], fma(t2.x, y[s], fma(t2.y, z[s], t5.x)));
          z[s] = fma(t3.x, x[s], fma(t3.y, y[s], fma(t4.x, z[s], t5.y)));
          x[s] = nx;
          y[s] = ny;
        }
      } else if (kind == SK_FLY) {
#pragma unroll
        for (int s = 0; s < S; ++s)
          if (act[s]) {
            const double3 m = fly_interval(rp.rops + (ch * kRecChunk + r), rp.ops, rp.sc, rp.relax, rp.n, base + s * bd,
                                           x[s], y[s], z[s]);
            x[s] = m.x;
            y[s] = m.y;
            z[s] = m.z;
          }
      }
      if (w0.z & kSnapBit) {  // events: the optional snapshot (engine.py:306-308)
#pragma unroll
        for (int s = 0; s < S; ++s) {
          if (!act[s]) continue;
          double* q = rp.snaps + (static_cast<int64_t>(w0.w) * rp.n + (base + s * bd)) * 3;
          q[0] = x[s];
          q[1] = y[s];
          q[2] = z[s];
        }
      }
    }
    __syncthreads();  // chunk ch + 1 staged; every warp is done with chunk ch's buffer before it is restaged
  }
}

static std::mutex g_res_mu;

template <int S>
static cudaError_t launch_resident_s(const RParams& rp, size_t smem, int grid, int threads, cudaStream_t stream) {
  static size_t smem_set[kMaxDevices] = {};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  {
    std::lock_guard<std::mutex> lk(g_res_mu);
    if (dev >= 0 && dev < kMaxDevices && smem > 48 * 1024 && smem > smem_set[dev]) {
      e = cudaFuncSetAttribute(resident_integrate_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               kResidentSmemBytes);
      if (e != cudaSuccess) return e;
      smem_set[dev] = kResidentSmemBytes;
    }
  }
  resident_integrate_kernel<S><<<grid, threads, smem, stream>>>(rp);
  return cudaGetLastError();
}

cudaError_t launch_resident(const RParams& rp, const ResidentPlan& plan, int spins_per_thread, int grid, int threads,
                            cudaStream_t stream) {
  // the tables are laid out for the big CTAs' bd_big threads; `threads` is bd_big rounded up to whole warps
  const size_t smem = kResidentFixedBytes + resident_mats_bytes(plan) +
                      static_cast<size_t>(plan.bytes_per_spin) * rp.bd_big * spins_per_thread;
  if (smem > static_cast<size_t>(kResidentSmemBytes) || rp.bd_big > threads) return cudaErrorInvalidValue;
  if (spins_per_thread == 2) return launch_resident_s<2>(rp, smem, grid, threads, stream);
  return launch_resident_s<1>(rp, smem, grid, threads, stream);
}

}  // namespace bloch
