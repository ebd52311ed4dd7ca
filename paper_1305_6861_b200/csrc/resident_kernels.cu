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

// shared memory ahead of the tables: the axis pulses (32 B each), then the general ones (72 B each)
static size_t resident_mats_bytes(const ResidentPlan& plan) {
  return plan.mats4.size() * 8 + ((plan.mats.size() * 8 + 15) & ~size_t(15));
}

int resident_threads(const ResidentPlan& plan, int64_t n, int n_sm) {
  if (!plan.ok || n <= 0) return 0;
  const int64_t room = kResidentSmemBytes - 1024 - kResidentFixedBytes - static_cast<int64_t>(resident_mats_bytes(plan));
  int64_t cap = plan.bytes_per_spin > 0 ? room / plan.bytes_per_spin : kResidentMaxThreads;
  cap = std::min<int64_t>(kResidentMaxThreads, (cap / 32) * 32);
  if (cap < kResidentMinThreads) return 0;
  // equal waves of one CTA per SM
  const int64_t per_wave = static_cast<int64_t>(n_sm) * cap;
  const int64_t waves = (n + per_wave - 1) / per_wave;
  int64_t t = (n + n_sm * waves - 1) / (n_sm * waves);
  t = ((t + 31) / 32) * 32;
  return static_cast<int>(std::max<int64_t>(32, std::min<int64_t>(cap, t)));
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

}  // namespace

// Staged record (shared memory, 32 bytes), decoded once per chunk per CTA from the 48-byte ROp:
//   w0 = (kind, shared address of the fused pulse or 0, tmode | arg << 2, U byte offset / snapshot index)
//   w1 = shared addresses of the op's four tables (thread 0's word; a thread adds tid * 16 or tid * 8)
// arg: R_UWIN lead flag, R_PROG advance.
__global__ void __launch_bounds__(kResidentMaxThreads, 1) resident_integrate_kernel(const RParams rp) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tid = threadIdx.x, bd = blockDim.x;
  const int64_t i = static_cast<int64_t>(blockIdx.x) * bd + tid;
  const bool act = i < rp.n;
  const uint32_t s_base = static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw));
  const uint32_t s_rec = s_base;                                    // [2][kRecChunk] staged records
  const uint32_t s_m4 = s_rec + 2 * kRecChunk * 32;                 // axis pulses, 32 B each
  const uint32_t s_m9 = s_m4 + 32u * rp.n_mats4;                    // general pulses, 72 B each
  const uint32_t s_area = s_m9 + ((72u * rp.n_mats + 15u) & ~15u);  // the tables, [table][thread]
  {
    double* m4 = reinterpret_cast<double*>(smem_raw + 2 * kRecChunk * 32);
    double* m9 = m4 + 4 * rp.n_mats4;
    for (int k = tid; k < 4 * rp.n_mats4; k += bd) m4[k] = __ldg(rp.mats4 + k);
    for (int k = tid; k < 9 * rp.n_mats; k += bd) m9[k] = __ldg(rp.mats + k);
  }
  const uint32_t t16 = s_area + tid * 16, t8 = s_area + tid * 8;
  // the CTA's tables: each value crosses L2 once per launch
  for (int j = 0; j < rp.n_loads; ++j) {
    const RLoad* L = rp.loads + j;
    const int kind = __ldg(&L->kind), id = __ldg(&L->id);
    const uint32_t off = static_cast<uint32_t>(__ldg(&L->off)) * bd;
    if (kind == 1) {
      sts_f2(t8 + off, act ? __ldg(rp.planes32 + (static_cast<int64_t>(id) * rp.n + i)) : make_float2(1.f, 0.f));
    } else if (kind == 0) {
      sts_d2(t16 + off, act ? __ldg(rp.planes + (static_cast<int64_t>(id) * rp.n + i)) : make_double2(1.0, 0.0));
    } else {
      const int word = __ldg(&L->word);
      sts_d2(t16 + off, act ? __ldg(reinterpret_cast<const double2*>(rp.train) +
                                    ((static_cast<int64_t>(id) * rp.n + i) * 6 + word))
                            : make_double2(0.0, 0.0));
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
      int4 w0, w1;
      w0.x = kind;
      w0.y = pre < 0 ? 0 : static_cast<int>((tmode == 1 || tmode == 2) ? s_m4 + 32u * pre : s_m9 + 72u * pre);
      const int arg = kind == R_UWIN ? (a.w != 0) : kind == R_PROG ? c.y : 0;
      w0.z = tmode | (arg << 2);
      w0.w = (kind == R_UWIN || kind == R_UCHIRP) ? c.x * 64 : a.w;
      w1.x = static_cast<int>(s_area + static_cast<uint32_t>(b.x) * bd);
      w1.y = static_cast<int>(s_area + static_cast<uint32_t>(b.y) * bd);
      w1.z = static_cast<int>(s_area + static_cast<uint32_t>(b.z) * bd);
      w1.w = static_cast<int>(s_area + static_cast<uint32_t>(b.w) * bd);
      const uint32_t dst = s_rec + ((ch & 1) * kRecChunk + r) * 32;
      sts_i4(dst, w0);
      sts_i4(dst + 16, w1);
    }
  };
  stage(0);
  __syncthreads();  // the matrices and chunk 0 (the tables are read only by the thread that wrote them)

  double x = act ? rp.mx0[i] : 0.0, y = act ? rp.my0[i] : 0.0, z = act ? rp.mz0[i] : 0.0;
  // contract_u_index(rows, r, i) = ((i >> 4) rows + r) 16 + (i & 15): this spin's word of row 0
  const int64_t ubase = act ? (i >> 4) * rp.urows * 16 + (i & 15) : 0;
  const char* uhi0 = reinterpret_cast<const char*>(rp.uhi + ubase);
  const char* ulo0 = reinterpret_cast<const char*>(rp.ulo + ubase);
  const uint32_t tid16 = tid * 16, tid8 = tid * 8;

  const int n_chunks = (rp.n_rops + kRecChunk - 1) / kRecChunk;
  for (int ch = 0; ch < n_chunks; ++ch) {
    if (ch + 1 < n_chunks) stage(ch + 1);  // lands during this chunk; the barrier below publishes it
    const int cnt = min(kRecChunk, rp.n_rops - ch * kRecChunk);
    uint32_t ra = s_rec + (ch & 1) * kRecChunk * 32;
    int4 n0 = lds_i4(ra), n1 = lds_i4(ra + 16);
    for (int r = 0; r < cnt; ++r) {
      const int4 w0 = n0, w1 = n1;
      ra += 32;  // the next record while this one runs (the slot after the buffer's last is never used)
      if (r + 1 < cnt) {
        n0 = lds_i4(ra);
        n1 = lds_i4(ra + 16);
      }
      const int kind = w0.x;
      if (w0.y) {  // a fused hard pulse first (bloch.py:124-139)
        const uint32_t ma = static_cast<uint32_t>(w0.y);
        const int tmode = w0.z & 3;
        if (tmode == 1) {  // about x: (x, r4 y + r5 z, r7 y + r8 z)
          const double2 m0 = lds_d2(ma), m1 = lds_d2(ma + 16);
          const double ny = m0.x * y + m0.y * z;
          z = m1.x * y + m1.y * z;
          y = ny;
        } else if (tmode == 2) {  // about y: (r0 x + r2 z, y, r6 x + r8 z)
          const double2 m0 = lds_d2(ma), m1 = lds_d2(ma + 16);
          const double nx = m0.x * x + m0.y * z;
          z = m1.x * x + m1.y * z;
          x = nx;
        } else {
          const double2 m0 = lds_d2(ma), m1 = lds_d2(ma + 16), m2 = lds_d2(ma + 32), m3 = lds_d2(ma + 48);
          double m8;
          asm volatile("ld.shared.f64 %0, [%1];" : "=d"(m8) : "r"(ma + 64));
          const double nx = m0.x * x + m0.y * y + m1.x * z;
          const double ny = m1.y * x + m2.x * y + m2.y * z;
          z = m3.x * x + m3.y * y + m8 * z;
          x = nx;
          y = ny;
        }
      }
      if (kind == R_PROG) {
        const uint32_t pa = static_cast<uint32_t>(w1.x) + tid16;
        const double2 cc = lds_d2(pa);
        const double2 ab = lds_d2(static_cast<uint32_t>(w1.w) + tid16);
        if (w0.z >> 2) {  // advance the running factor by q or q^2
          const double2 q = lds_d2(static_cast<uint32_t>(w1.y) + tid16);
          sts_d2(pa, make_double2(cc.x * q.x - cc.y * q.y, cc.x * q.y + cc.y * q.x));
        }
        const double nx = cc.x * x - cc.y * y;
        y = cc.x * y + cc.y * x;
        x = nx;
        z = fma(z, ab.x, ab.y);
      } else if (kind == R_UWIN) {
        const float2 cp = lds_f2(static_cast<uint32_t>(w1.x) + tid8);
        const double2 cc = lds_d2(static_cast<uint32_t>(w1.z) + tid16);
        const double2 ab = lds_d2(static_cast<uint32_t>(w1.w) + tid16);
        // u = Cpre m in fp32 (two conversions of the state): equal to ~2^-24, inside the bf16 hi + lo split
        const float fx = static_cast<float>(x), fy = static_cast<float>(y);
        float ur = cp.x * fx - cp.y * fy, ui = cp.x * fy + cp.y * fx;
        if (!(w0.z >> 2)) {  // no leading no-op sample: the first sample follows one interval
          const float2 zz = lds_f2(static_cast<uint32_t>(w1.y) + tid8);
          const float t = ur * zz.x - ui * zz.y;
          ui = ur * zz.y + ui * zz.x;
          ur = t;
        }
        if (act) {
          uint32_t hi, lo;
          split_bf16x2(ur, ui, hi, lo);
          __stcs(reinterpret_cast<uint32_t*>(const_cast<char*>(uhi0 + w0.w)), hi);  // streamed: read by the contraction
          __stcs(reinterpret_cast<uint32_t*>(const_cast<char*>(ulo0 + w0.w)), lo);
        }
        const double nx = cc.x * x - cc.y * y;
        y = cc.x * y + cc.y * x;
        x = nx;
        z = fma(z, ab.x, ab.y);
        continue;
      } else if (kind == R_TAB) {
        const double2 cc = lds_d2(static_cast<uint32_t>(w1.x) + tid16);
        const double2 ab = lds_d2(static_cast<uint32_t>(w1.y) + tid16);
        const double nx = cc.x * x - cc.y * y;
        y = cc.x * y + cc.y * x;
        x = nx;
        z = fma(z, ab.x, ab.y);
      } else if (kind == R_TRAIN) {
        const uint32_t ta = static_cast<uint32_t>(w1.x) + tid16, st = 16u * bd;
        const double2 t0 = lds_d2(ta), t1 = lds_d2(ta + st), t2 = lds_d2(ta + 2 * st), t3 = lds_d2(ta + 3 * st),
                      t4 = lds_d2(ta + 4 * st), t5 = lds_d2(ta + 5 * st);
        const double nx = fma(t0.x, x, fma(t0.y, y, fma(t1.x, z, t4.y)));
        const double ny = fma(t1.y, x, fma(t2.x, y, fma(t2.y, z, t5.x)));
        z = fma(t3.x, x, fma(t3.y, y, fma(t4.x, z, t5.y)));
        x = nx;
        y = ny;
        continue;
      } else if (kind == R_UCHIRP) {
        const double2 cc = lds_d2(static_cast<uint32_t>(w1.z) + tid16);
        const double2 ab = lds_d2(static_cast<uint32_t>(w1.w) + tid16);
        if (act) {
          const double2 w = rp.w1 != nullptr ? __ldg(rp.w1 + i) : make_double2(1.0, 0.0);
          const float wx = static_cast<float>(w.x), wy = static_cast<float>(w.y);
          const float fx = static_cast<float>(x), fy = static_cast<float>(y);
          uint32_t hi, lo;
          split_bf16x2(wx * fx - wy * fy, wx * fy + wy * fx, hi, lo);
          __stcs(reinterpret_cast<uint32_t*>(const_cast<char*>(uhi0 + w0.w)), hi);
          __stcs(reinterpret_cast<uint32_t*>(const_cast<char*>(ulo0 + w0.w)), lo);
        }
        const double nx = cc.x * x - cc.y * y;
        y = cc.x * y + cc.y * x;
        x = nx;
        z = fma(z, ab.x, ab.y);
        continue;
      } else if (kind == R_FLY) {  // one interval per spin: precession (+ relaxation), engine.py:288-302
        const ROp* rop = rp.rops + (ch * kRecChunk + r);
        const int flags = __ldg(&rop->flags), cls = __ldg(&rop->cls);
        if ((flags & EV_MOVE) && act) {
          const DevOp* op = rp.ops + __ldg(&rop->src);
          const double dt = __ldg(&op->p[0]), dmx = __ldg(&op->p[1]), dmy = __ldg(&op->p[2]), dmz = __ldg(&op->p[3]);
          const double2* s = reinterpret_cast<const double2*>(static_cast<const SpinConst*>(rp.sc) + i);
          const double2 s0 = __ldg(s), s1 = __ldg(s + 1), s2 = __ldg(s + 2);  // (x, y), (z, dw), (m0, r1)
          const double2 e = cls >= 0 ? __ldg(reinterpret_cast<const double2*>(rp.relax) +
                                             (static_cast<int64_t>(cls) * rp.n + i))
                                     : make_double2(1.0, 1.0);
          const double th = fma(s1.x, dmz, fma(s0.y, dmy, s0.x * dmx)) + s1.y * dt;  // engine.py:289
          double sn, cs;
          sincos(r_reduce_2pi(th), &sn, &cs);
          const double ms = -sn;
          const double nx = e.y * (cs * x - ms * y);  // clockwise: (c - i s)(x + i y), bloch.py:10-17
          y = e.y * (cs * y + ms * x);
          x = nx;
          if (cls >= 0) z = fma(z, e.x, s2.x * (1.0 - e.x));
        }
      }
      // events: the optional snapshot (engine.py:306-308)
      if (kind != R_NOP && w0.w >= 0 && rp.snaps != nullptr && act) {
        double* q = rp.snaps + (static_cast<int64_t>(w0.w) * rp.n + i) * 3;
        q[0] = x;
        q[1] = y;
        q[2] = z;
      }
    }
    __syncthreads();  // chunk ch + 1 staged; every warp is done with chunk ch's buffer before it is restaged
  }
}

static std::mutex g_res_mu;

cudaError_t launch_resident(const RParams& rp, const ResidentPlan& plan, int grid, int threads, cudaStream_t stream) {
  const size_t smem = kResidentFixedBytes + resident_mats_bytes(plan) + static_cast<size_t>(plan.bytes_per_spin) * threads;
  static size_t smem_set[kMaxDevices] = {};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  {
    std::lock_guard<std::mutex> lk(g_res_mu);
    if (dev >= 0 && dev < kMaxDevices && smem > 48 * 1024 && smem > smem_set[dev]) {
      e = cudaFuncSetAttribute(resident_integrate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               kResidentSmemBytes);
      if (e != cudaSuccess) return e;
      smem_set[dev] = kResidentSmemBytes;
    }
  }
  resident_integrate_kernel<<<grid, threads, smem, stream>>>(rp);
  return cudaGetLastError();
}

}  // namespace bloch
