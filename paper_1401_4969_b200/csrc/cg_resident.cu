// SM-resident batched Jacobi-PCG: the reference's cg_solve (sparse.cpp:199-258)
// for every system of a CgBatch, with each system's iterates held ON CHIP for
// the whole solve instead of being streamed from HBM/L2 every iteration.
//
// Layout.  One cooperative launch, one 256-thread CTA per SM.  The CTAs are
// grouped into `lanes` of C CTAs; a lane solves its list of systems one after
// another.  A system (lattice window w x h, row pitch w + 1 with a zero pad
// column) is cut into C horizontal slabs of R = ceil(h / C) rows; CTA i of the
// lane owns slab rows [iR, min((i+1)R, h)).  Point j of a slab (row-major over
// the pitched rows) belongs to thread j mod 256, register slot j / 256:
//   registers   r, q = A p                 (48 points per thread: 192 registers)
//   shared mem  p with one ghost row above and below the slab, and x.
//
// One iteration (the one-reduction rearrangement of cg.cu, same scalars via
// update_ctl): phase 1, pointwise, applies the pending update and forms the new
// direction  r -= a q; x += a p; z = D^-1 r; p = z + b p  for the slab rows AND
// for the two ghost rows, whose r and p the CTA keeps itself (shared memory)
// and advances with the neighbour's published q row -- bitwise the values the
// neighbour computes for those rows, same operations in the same order, so
// only ONE row per side (q) crosses L2 per iteration; phase 2 computes q = A p
// from shared memory and the five dot products r.r, r.z, p.q, q.z, q.D^-1q,
// then publishes q of the slab's first and last rows.  (At the start and after
// a true-residual restart the published row is r, which re-seeds the ghosts.)
//
// Lane synchronisation = the reduction itself: the CTA's five sums and its
// boundary rows are released by one fence + arrival on the lane's monotonic
// counter; after the C arrivals every CTA reads the C x 5 partials and sums
// them in CTA order, and runs update_ctl: the scalars are identical in every
// CTA and run-to-run deterministic.  (Measured alternatives, all slower on
// B200, where a word written by one SM reaches another in about a
// microsecond: partial sums as self-validating tagged words polled by five
// warps, per-CTA mailboxes, tagged boundary rows -- strong .gpu loads and
// stores cost far more than weak ones plus one fence -- one warp running the
// whole chain, and two 256-thread CTAs per SM.)  The true residual check
// (sparse.cpp:232-246) exchanges the boundary rows of x behind a plain lane
// barrier and evaluates b - A x from shared memory.
//
// Traffic per point and iteration: shared memory 72 B (phase 1 loads/stores p
// and x, phase 2 loads five p values), no HBM; L2 carries only the boundary
// rows (1 double per slab column and side) and the partial sums.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <type_traits>
#include <vector>

#include "cg.cuh"
#include "cg_ctl.cuh"

namespace mlg {
namespace {

// CTA shape: kResT threads x kResPT points.  The SM's register file holds r and
// q of 12,288 points (3/4 of it) whatever the shape; with 256 threads x 48
// points a thread keeps 63 registers for everything else (384 x 32: ~40,
// 512 x 24: 32), which lets the point loops overlap the loads and FP64 chains
// that register reuse serialised: config 5 local 1.625 s (512 x 24) -> 1.54 s
// (384 x 32) -> 1.49 s (256 x 48); 448 x 28 is capped at 128 registers: 1.86 s.
#ifndef MLG_RES_PT
#define MLG_RES_PT 48
#endif
#ifndef MLG_RES_T
#define MLG_RES_T 256
#endif
constexpr int kResT = MLG_RES_T;     // threads per CTA
#ifndef MLG_RES_PERSM
#define MLG_RES_PERSM 1
#endif
constexpr int kResPerSM = MLG_RES_PERSM;  // co-resident CTAs per SM (2 x 256 threads measured +80 %)
constexpr int kResPT = MLG_RES_PT;  // points per thread (registers r, q)
#ifndef MLG_RES_CHUNK
#define MLG_RES_CHUNK 0  // 0: one chunk (A/B hook)
#endif
// The pointwise phases can run their points in chunks of MLG_RES_CHUNK with a
// scheduling fence between chunks: the loads of one chunk are hoisted and
// overlapped, but not across chunks (one chunk measured best at 256 x 48).
constexpr int kResCap = kResT * kResPT;  // points per CTA of the largest instantiation
static_assert(MLG_RES_PT <= 64, "one in-system flag per register slot");
// Instantiated slab capacities (points per thread).  A slab of R rows x pitch
// points runs the smallest variant that holds it: the unrolled point loops
// cost their full trip count whatever the slab holds (config 2's strip, 7 rows
// x 1024 = 28 x 256 points, paid for 48 slots before).
constexpr int kResVariants[] = {MLG_RES_PT, 36, 28, 20, 12};
// MLG_RES_GHOSTR = 1: the CTA keeps r of its two ghost rows in shared memory
// and the neighbours publish one row per side (q); 0: they publish r and q and
// no ghost r is kept (2 x pitch doubles less shared memory: the 2-CTAs/SM shape)
#ifndef MLG_RES_GHOSTR
#define MLG_RES_GHOSTR 1
#endif
constexpr bool kGhostR = MLG_RES_GHOSTR != 0;
// MLG_RES_FUSEPUB = 1: normal iterations store q of the slab's first and last
// rows from inside phase 2 (two predicated stores per slot) instead of a
// separate pass of CTA-uniform branches over the slots afterwards
#ifndef MLG_RES_FUSEPUB
#define MLG_RES_FUSEPUB 1
#endif
constexpr bool kFusePub = MLG_RES_FUSEPUB != 0 && MLG_RES_GHOSTR != 0;
constexpr int kFirstSlots = 8;  // slots that can hold a point of the slab's first row
constexpr int kTailSlots = 12;  // ... of its last row, when the slab is (nearly) full
#ifndef MLG_RES_GHOSTPRE
#define MLG_RES_GHOSTPRE 6
#endif
constexpr int kGhostPre = MLG_RES_GHOSTPRE;  // ghost points per thread requested ahead
constexpr int kHaloFields = kGhostR ? 1 : 2;
constexpr unsigned kFullMask = 0xffffffffu;
__host__ __device__ constexpr int part_cpad(int C) { return (C + 15) & ~15; }  // 128-byte rows

struct ResArgs {
  const CgSys* sys;
  const int* lanes;  // [nlanes][per_lane] system ids, -1 terminated
  int per_lane, C, nlanes;
  const double* bsrc;
  int bstride, nxp1;
  double* X;
  CgCtl* ctl;
  double* part;   // partial sums [nlanes][2 parity][kCgDots][part_cpad(C)]
  double* halo;   // boundary rows [nlanes][2 parity][C][2 sides][kHaloFields][hpitch]
  unsigned* bar;  // [nlanes * 32] arrival counters (one 128-byte line per lane)
  int hpitch;
  double* bslab;  // [2][gridDim.x][kResCap]: slab right-hand sides, true-residual scratch
  StripGeom sg;
  int masked;     // strip systems: points of the closed G_j are outside
  double tol;
  Stencil ust;
  double udinv;
  unsigned long long* trace;  // MLG_RES_TRACE: per-CTA cycle sums of the iteration phases
};

__device__ __forceinline__ bool point_in_system(const ResArgs& A, const CgSys& S, int gx,
                                                int gy) {
  if (A.masked) {  // strip membership (cg.cu in_strip): outside every closed G_j and the hole
    const StripGeom& g = A.sg;
    const int bx = min(gx / (g.bw * g.scale), g.side - 1);
    const int by = min(gy / (g.bh * g.scale), g.side - 1);
    const int x0 = (bx == 0 ? 0 : bx * g.bw + g.dc) * g.scale;
    const int x1 = (bx == g.side - 1 ? g.nx0 : (bx + 1) * g.bw - g.dc) * g.scale;
    const int y0 = (by == 0 ? 0 : by * g.bh + g.dc) * g.scale;
    const int y1 = (by == g.side - 1 ? g.ny0 : (by + 1) * g.bh - g.dc) * g.scale;
    return !(gx >= x0 && gx <= x1 && gy >= y0 && gy <= y1) && !g.in_hole(gx, gy);
  }
  return !A.sg.in_hole(gx, gy);
}

// Predicated shared-memory store (a predicate, not a branch: keeps the unrolled
// point loops straight-line so their loads can overlap).
__device__ __forceinline__ void sts_if(double* p, double v, bool pred) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q st.shared.f64 [%0], %1;\n\t}" ::"r"(
          static_cast<unsigned>(__cvta_generic_to_shared(p))),
      "d"(v), "r"(static_cast<int>(pred)));  // no memory clobber: other points' loads may
}                                              // move across (they never read this point)

// Row product of the constant-coefficient stencil from the pitched shared
// buffer (the paired form of cg.cu product_lat: same rounding as k_cg_iter).
template <bool LAP>
__device__ __forceinline__ double res_product(const double* P, int i, int pitch,
                                              const Stencil& u) {
  const double pc = P[i], pw = P[i - 1], pe = P[i + 1], ps = P[i - pitch], pn = P[i + pitch];
  if constexpr (LAP) {
    return fma(-1.0, pw + pe, fma(-1.0, ps + pn, 4.0 * pc));
  } else {
    const double psw = P[i - pitch - 1], pne = P[i + pitch + 1];
    return fma(u.e, pw + pe, fma(u.n, ps + pn, fma(u.ne, psw + pne, u.c * pc)));
  }
}

// Release / acquire fence at gpu scope (lighter than __threadfence(), which is
// the sequentially consistent fence.sc.gpu).
__device__ __forceinline__ void fence_acq_rel() {
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
}

// One thread's arrival on the lane's monotonic counter (release: with the
// preceding bar.sync it covers every earlier global write of the CTA) and its
// wait for arrival number `target` (acquire).  Polling with acquire loads
// measured 0.6 k cycles per iteration cheaper than relaxed loads followed by a
// fence (config 5 local 1.68 -> 1.62 s); a release reduction instead of
// fence + atomic made no difference.
__device__ __forceinline__ void arrive_and_wait(unsigned* bar, unsigned target) {
  fence_acq_rel();
  atomicAdd(bar, 1u);
  unsigned seen;
  do {
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(bar) : "memory");
  } while (seen < target);
}

// Plain lane barrier (true-residual checks only).
__device__ __forceinline__ void lane_barrier(unsigned* bar, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) arrive_and_wait(bar, target);
  __syncthreads();
}

// The lane's reduction and its only synchronisation.  Warp trees (the five
// quantities interleaved), one bar.sync, warp k sums quantity k over the warps
// and stores it; then ONE thread releases the five sums -- and, cumulatively,
// every earlier global write of the CTA (its boundary rows) -- with one fence
// + arrival on the lane's monotonic counter, waits for the C arrivals of this
// reduction and acquires; warp k then reads the C partials of quantity k (both
// loads of a lane in flight together) and sums them in CTA order (fixed xor
// tree: identical in every CTA, run-to-run deterministic).
// `after_barrier` runs in every thread as soon as the arrivals are complete:
// the kernel requests the neighbours' boundary rows there, so that their L2
// latency overlaps the reading of the partial sums and update_ctl.
//   part: the lane's partial sums [2 parity][kCgDots][C rounded up to 16] (dense per
//   quantity; 64-byte slots per CTA measured 2 % slower)
template <typename MARK, typename AFTER>
__device__ __forceinline__ void res_reduce(double (&acc)[kCgDots], double* red, double* ssum,
                                           double* part, unsigned* bar, unsigned target, int par,
                                           int ci, int C, double (&a)[kCgDots], MARK&& mark,
                                           AFTER&& after_barrier) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int nw = kResT / 32;
  const int cpad = part_cpad(C);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
    for (int k = 0; k < kCgDots; ++k) acc[k] += __shfl_xor_sync(kFullMask, acc[k], o);
  }
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < kCgDots; ++k) red[k * nw + warp] = acc[k];
  }
  __syncthreads();
  mark(6);
  double* slots = part + (static_cast<long long>(par) * kCgDots + warp) * cpad;
  if (warp < kCgDots) {
    double v = lane < nw ? red[warp * nw + lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFullMask, v, o);  // lanes >= nw add 0
    if (lane == 0) __stcg(slots + ci, v);
  }
  __syncthreads();
  if (threadIdx.x == 0) arrive_and_wait(bar, target);
  __syncthreads();
  after_barrier();  // (all threads: loads that only need the barrier, not the sums)
  mark(7);
  if (warp < kCgDots) {
    // every load of the lane in flight together (C <= 160 CTAs: five per lane);
    // a serial tail cost one L2 round trip per 32 CTAs beyond 64 (config 2's
    // strip, 114 CTAs: lane sums 5.1 k cycles against 3.4 k at C <= 64)
    double sv[5];
#pragma unroll
    for (int k = 0; k < 5; ++k) sv[k] = lane + 32 * k < C ? __ldcg(slots + lane + 32 * k) : 0.0;
    double s = sv[0] + sv[1];
#pragma unroll
    for (int k = 2; k < 5; ++k) s += sv[k];
    for (int c = lane + 160; c < C; c += 32) s += __ldcg(slots + c);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(kFullMask, s, o);
    if (lane == 0) ssum[warp] = s;
  }
  __syncthreads();
  mark(8);
#pragma unroll
  for (int k = 0; k < kCgDots; ++k) a[k] = ssum[k];
}

template <bool LAP, int PT>
__global__ void __launch_bounds__(kResT, kResPerSM) k_cg_resident(ResArgs A) {
  // PT points per thread (register slots of r and q); the point loops run PT
  // slots whatever the slab holds, so small slabs use a smaller instantiation
  constexpr int kCap = kResT * PT;
  constexpr int kCh = MLG_RES_CHUNK > 0 && PT % MLG_RES_CHUNK == 0 ? MLG_RES_CHUNK : PT;
  using Act = std::conditional_t<(PT > 32), unsigned long long, unsigned>;
  // ghost points per thread requested ahead: the smaller instantiations have the
  // registers for 8 (two rows of pitch <= 1024: config 2's strip)
  constexpr int kGP = PT >= MLG_RES_PT ? kGhostPre : (kGhostPre > 8 ? kGhostPre : 8);
  auto sched_fence = [] {
    if constexpr (kCh < PT) asm volatile("" ::: "memory");
  };
  extern __shared__ double smem[];
  __shared__ double s_red[(kResT / 32) * kCgDots];
  __shared__ CgCtl s_ctl;
  __shared__ double s_sum[8];
  __shared__ unsigned long long s_tr[16];
  if (threadIdx.x < 16) s_tr[threadIdx.x] = 0;
  const int lane_id = blockIdx.x / A.C;
  const int ci = blockIdx.x % A.C;
  if (lane_id >= A.nlanes) return;
  const int t = threadIdx.x;
  const int C = A.C;
  unsigned* bar = A.bar + lane_id * 32;
  unsigned epoch = 0;  // lane barriers so far: buffer parity; arrivals so far = C * epoch
  long long tmark = clock64();
  // (diagnostics) cycles since the previous mark, summed per CTA into slot s
#ifdef MLG_RES_SKEW
  // (diagnostics) GPU-wide timer stamps of 16 iterations of the lane's first
  // system: iteration start, tagged store, reduction complete
  auto stamp = [&](int li, int it, int what) {
    if (A.trace != nullptr && t == 0 && li == 0 && it >= 500 && it < 516) {
      unsigned long long g;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
      A.trace[gridDim.x * 16 + (blockIdx.x * 16 + (it - 500)) * 4 + what] = g;
    }
  };
#endif
  auto mark = [&](int s) {
    if (A.trace != nullptr && t == 0) {
      const long long now = clock64();
      s_tr[s] += static_cast<unsigned long long>(now - tmark);
      tmark = now;
    }
  };
  const Stencil u = A.ust;
  const double dv = LAP ? 0.25 : A.udinv;
  for (int li = 0; li < A.per_lane; ++li) {
    const int sid = A.lanes[lane_id * A.per_lane + li];
    if (sid < 0) break;
    const CgSys& S = A.sys[sid];  // fields re-read from global where used (registers)
    const int pitch = S.pitch;
    const int maxit = S.maxit;
    const int R = (S.h + C - 1) / C;
    const int ya = ci * R;
    const int nr = max(min(ya + R, S.h) - ya, 0);
    const int npts = nr * pitch;
    const bool has_lo = nr > 0 && ci > 0;                  // neighbour slab below
    const bool has_hi = nr > 0 && (ci + 1) * R < S.h;       // neighbour slab above
    double* P = smem;                           // (R + 2) * pitch + 2, point (row, col) at
    const int off = pitch + 1;                  //   off + row * pitch + col
    // Every slot j < kCap of the unrolled point loops may READ P[off + j +-
    // pitch +- 1] and Xs[j] (slots past the slab are masked, never stored), so
    // the buffers cover the full capacity: straight-line loops, affine addresses.
    const int plen = kCap + 2 * pitch + 4;
    double* Xs = smem + plen;                   // kCap
    double* Rg = Xs + kCap;                  // (kGhostR) r of the ghost rows: [2 sides][pitch]
    for (int i = t; i < plen; i += kResT) P[i] = 0.0;
    for (int i = t; i < kCap; i += kResT) Xs[i] = 0.0;
    if constexpr (kGhostR)
      for (int i = t; i < 2 * pitch; i += kResT) Rg[i] = 0.0;
    // in-system flags of the thread's points and the slab's right-hand side
    // (0 outside the system), gathered once into the CTA's bslab row: the
    // register arrays below are then filled and refilled without divisions
    double* bs = A.bslab + static_cast<long long>(blockIdx.x) * kCap;
    Act act = 0;  // bit k: slot k is a point of the system
#pragma unroll 1
    for (int k = 0; k < PT; ++k) {
      const int j = t + k * kResT;
      double b = 0.0;
      if (j < npts) {
        const int row = j / pitch, col = j - row * pitch;
        if (col < S.w) {
          const int gx = S.x0 + col, gy = S.y0 + ya + row;
          if (point_in_system(A, S, gx, gy)) {
            act |= static_cast<Act>(1) << k;
            b = A.bsrc[(static_cast<long long>(gy) * A.nxp1 + gx) * A.bstride + S.rhs];
          }
        }
        bs[j] = b;
      }
    }
    double r[PT], q[PT];
#pragma unroll
    for (int k = 0; k < PT; ++k) {
      const int j = t + k * kResT;
      r[k] = (act >> k & 1u) ? bs[j] : 0.0;
      q[k] = 0.0;
    }
    double* part_lane = A.part + static_cast<long long>(lane_id) * 2 * kCgDots * part_cpad(C);
    double* halo_base =
        A.halo + static_cast<long long>(lane_id) * 2 * C * 2 * kHaloFields * A.hpitch;
    auto halo_row = [&](int par, int cta, int side, int field) {
      return halo_base +
             (((static_cast<long long>(par) * C + cta) * 2 + side) * kHaloFields + field) *
                 A.hpitch;
    };
    // publish one field of the slab's first (side 0) and last (side 1) rows.
    // The slot tests are CTA-uniform (no divergence); only the slots that can
    // hold a point of those rows reach the per-thread test.
    const int first_end = min(pitch, npts), last_begin = npts - pitch;
    // (fused publish: nobody reads the last row of the lane's top slab)
    const int lb_pub = has_hi ? last_begin : 0x3fffffff;
    const bool last_in_tail = PT > kTailSlots && lb_pub >= (PT - kTailSlots) * kResT;
    auto publish = [&](const double (&v)[PT], int par, int field) {
      double* row0 = halo_row(par, ci, 0, field);
      double* row1 = halo_row(par, ci, 1, field) - last_begin;
#pragma unroll
      for (int k = 0; k < PT; ++k) {
        const int j = t + k * kResT;
        if (k * kResT < first_end) {
          if (j < first_end) __stcg(row0 + j, v[k]);
        }
        if ((k + 1) * kResT > last_begin && k * kResT < npts) {
          if (j >= last_begin && j < npts) __stcg(row1 + j, v[k]);
        }
      }
    };
    // The neighbours' published rows were written by other SMs: their L2 reads
    // take microseconds.  The first kGhostPre ghost points of the thread are
    // requested right after the lane barrier that makes them visible (inside
    // res_reduce) and consumed in phase 1 of the next iteration.
    double gpre[kGP > 0 ? kGP : 1];
    auto prefetch_ghost = [&](int par) {
      if constexpr (kGhostR) {
#pragma unroll
        for (int g = 0; g < kGP; ++g) {
          const int i = t + g * kResT;
          const int side = i >= pitch;
          gpre[g] = 0.0;
          if (i < 2 * pitch && (side ? has_hi : has_lo))
            gpre[g] = __ldcg(halo_row(par, side ? ci + 1 : ci - 1, side ? 0 : 1, 0) +
                             (i - side * pitch));
        }
      }
    };
    double acc[kCgDots];
#pragma unroll
    for (int k = 0; k < kCgDots; ++k) acc[k] = 0.0;
#pragma unroll
    for (int k = 0; k < PT; ++k) acc[0] += r[k] * r[k];
    __syncthreads();  // P, Xs, Rg zeroed
    publish(r, epoch & 1, 0);  // r rows: the first iteration is a (re)start
    if constexpr (!kGhostR) publish(q, epoch & 1, 1);  // (zeros)
    {
      double a[kCgDots];
      res_reduce(acc, s_red, s_sum, part_lane, bar, C * (epoch + 1), epoch & 1, ci, C, a,
                 [](int) {}, [&] { prefetch_ghost(epoch & 1); });
      if (t == 0) {
        CgCtl c{};
        update_ctl<kPhaseInit>(c, a, A.tol, S.maxit);
        s_ctl = c;
      }
    }
    ++epoch;
    __syncthreads();
    while (true) {
      // only the scalars this iteration needs (the full CgCtl would hold ~16
      // registers through the unrolled loops)
      if (s_ctl.status != kRunning) break;
#ifdef MLG_RES_SKEW
      const int it_now = s_ctl.iters;
      stamp(li, it_now, 0);
#endif
#pragma unroll
      for (int k = 0; k < kCgDots; ++k) acc[k] = 0.0;
      const int par_prev = (epoch + 1) & 1;  // buffers of the previous barrier
      if (s_ctl.mode == kModeNormal) {
        const bool rst = s_ctl.restart != 0;
        const double al = rst ? 0.0 : s_ctl.alpha;
        const double be = rst ? 0.0 : s_ctl.beta;
        // phase 1: own points
#pragma unroll
        for (int k0 = 0; k0 < PT; k0 += kCh) {
#pragma unroll
          for (int k = k0; k < k0 + kCh; ++k) {
            // branch-free (loads of consecutive points overlap): points of the
            // slab outside the system hold r = q = p = 0 and stay so; slots past
            // the slab read a valid dummy point and do not store
            const int j = t + k * kResT;
            const bool in = j < npts;
            const double po = P[off + j];
            const double xo = Xs[j];
            const double rn = fma(-al, q[k], r[k]);
            const double tz = __dmul_rn(dv, rn);
            sts_if(P + off + j, fma(be, po, tz), in);
            sts_if(Xs + j, fma(al, po, xo), in);
            r[k] = rn;
          }
          sched_fence();
        }
        mark(0);
        // phase 1: ghost rows (same operations as their owner): r and p of
        // the ghosts are kept here, the neighbour's q row (r row at a
        // (re)start) comes from its published boundary row
        if (has_lo || has_hi) {
          auto ghost_point = [&](int i, bool pre, double pv) {
            const int side = i >= pitch;  // 0: row -1 (from ci-1's last row), 1: row nr
            const int col = i - side * pitch;
            if (side ? !has_hi : !has_lo) return;
            const int src = side ? ci + 1 : ci - 1;
            double rn;
            if constexpr (kGhostR) {
              const double hv = pre ? pv : __ldcg(halo_row(par_prev, src, side ? 0 : 1, 0) + col);
              rn = rst ? hv : fma(-al, hv, Rg[i]);
              Rg[i] = rn;
            } else {
              const double rg = __ldcg(halo_row(par_prev, src, side ? 0 : 1, 0) + col);
              const double qg = __ldcg(halo_row(par_prev, src, side ? 0 : 1, 1) + col);
              rn = fma(-al, qg, rg);
            }
            const double tz = __dmul_rn(dv, rn);
            double* pg = P + (side ? off + nr * pitch + col : off - pitch + col);
            *pg = fma(be, *pg, tz);
          };
          if constexpr (kGhostR) {
#pragma unroll
            for (int g = 0; g < kGP; ++g)
              if (t + g * kResT < 2 * pitch) ghost_point(t + g * kResT, true, gpre[g]);
            for (int i = t + kGP * kResT; i < 2 * pitch; i += kResT)
              ghost_point(i, false, 0.0);
          } else {
            for (int i = t; i < 2 * pitch; i += kResT) ghost_point(i, false, 0.0);
          }
        }
        __syncthreads();
        mark(1);
        // phase 2: q = A p, dot products
        // (per-thread bases: the slot offsets k * kResT are immediates)
        double* const pub0 = halo_row(epoch & 1, ci, 0, 0) + t;
        double* const pub1 = halo_row(epoch & 1, ci, 1, 0) - last_begin + t;
        // Two copies of the loop: when the slab's last row lies in the last
        // kTailSlots slots (full slabs: every CTA of configs 2 and 5) only those
        // slots carry the last-row test.
        auto phase2 = [&](auto tailc) {
          constexpr bool TAIL = decltype(tailc)::value;
  #pragma unroll
          for (int k0 = 0; k0 < PT; k0 += kCh) {
  #pragma unroll
            for (int k = k0; k < k0 + kCh; ++k) {
              // branch-free: q of points outside the system is forced to 0, so
              // every dot term of such a point is an exact zero (r = p = 0 there)
              const int j = t + k * kResT;
              const double qa = res_product<LAP>(P, off + j, pitch, u);
              const double qq = (act >> k & 1u) ? qa : 0.0;
              const double pv = P[off + j];  // finite; its term is 0 where qq is masked
              q[k] = qq;
              if constexpr (kFusePub) {  // boundary rows for the neighbours' ghosts
                // first row: slots below kFirstSlots only (pitch <= kFirstSlots * kResT,
                // host plan).  (A per-thread slot mask for the last row instead of the
                // two compares spilled the 48-point kernel: local 1.45 -> 1.62 s.)
                if (k < kFirstSlots) {  // (folded: the loop is fully unrolled)
                  if (j < first_end) __stcg(pub0 + k * kResT, qq);
                }
                if (!TAIL || k >= PT - kTailSlots) {  // (folded)
                  if (j >= lb_pub && j < npts) __stcg(pub1 + k * kResT, qq);
                }
              }
              acc[0] += r[k] * r[k];
              acc[2] += pv * qq;
              if constexpr (LAP) {  // D^-1 = 1/4: the z terms are exact quarters (below)
                acc[1] += qq * r[k];
                acc[4] += qq * qq;
              } else {
                const double tz = __dmul_rn(dv, r[k]);
                acc[1] += r[k] * tz;
                acc[3] += qq * tz;
                acc[4] += qq * __dmul_rn(dv, qq);
              }
            }
            sched_fence();
          }
        };
        if (last_in_tail)
          phase2(std::true_type{});
        else
          phase2(std::false_type{});
        if constexpr (LAP) {
          // z = r / 4 exactly, so r.z = (r.r)/4, q.z = (q.r)/4, q.D^-1q = (q.q)/4
          // term by term (power-of-two scaling commutes with every rounding of
          // the sums): bitwise the sums of the general formula
          acc[3] = 0.25 * acc[1];
          acc[1] = 0.25 * acc[0];
          acc[4] = 0.25 * acc[4];
        }
        mark(2);
      } else {  // kModeCheck: r = b - A x (sparse.cpp:232-246)
        const int par = epoch & 1;
        // exchange the boundary rows of x
        for (int j = t; j < first_end; j += kResT) __stcg(halo_row(par, ci, 0, 0) + j, Xs[j]);
        for (int j = max(last_begin, 0) + t; j < npts; j += kResT)
          __stcg(halo_row(par, ci, 1, 0) + (j - last_begin), Xs[j]);
        lane_barrier(bar, C * (epoch + 1));
        ++epoch;
        for (int i = t; i < 2 * pitch; i += kResT) {
          const int side = i >= pitch;
          const int col = i - side * pitch;
          if (side ? !has_hi : !has_lo) continue;
          const int src = side ? ci + 1 : ci - 1;
          const double xg = __ldcg(halo_row(par, src, side ? 0 : 1, 0) + col);
          P[side ? off + nr * pitch + col : off - pitch + col] = xg;
        }
        for (int j = t; j < npts; j += kResT) P[off + j] = Xs[j];
        __syncthreads();
        // (rolled loop through the CTA's scratch row: no register arrays live
        // in this rarely taken branch)
        double* rt = bs + static_cast<long long>(gridDim.x) * kCap;  // 2nd half of bslab
#pragma unroll 1
        for (int k = 0; k < PT; ++k) {
          const int j = t + k * kResT;
          if (act >> k & 1u) {
            const double ax = res_product<LAP>(P, off + j, pitch, u);
            const double v = __dsub_rn(bs[j], ax);
            rt[j] = v;
            acc[0] += v * v;
          }
        }
#pragma unroll
        for (int k = 0; k < PT; ++k) {
          const int j = t + k * kResT;
          r[k] = (act >> k & 1u) ? rt[j] : 0.0;
          q[k] = 0.0;
        }
        __syncthreads();  // P (holding x) is read by phase 1 of a restart only as 0 * p
      }
      // normal iterations publish q; a true-residual check publishes the new
      // r, which re-seeds the neighbours' ghost rows at the restart
      if constexpr (kGhostR) {
        if (s_ctl.mode == kModeNormal) {
          if constexpr (!kFusePub) publish(q, epoch & 1, 0);
        } else {
          publish(r, epoch & 1, 0);
        }
      } else {
        publish(r, epoch & 1, 0);
        publish(q, epoch & 1, 1);
      }
      mark(3);
#ifdef MLG_RES_SKEW
      stamp(li, it_now, 1);
#endif
      double a[kCgDots];
      res_reduce(acc, s_red, s_sum, part_lane, bar, C * (epoch + 1), epoch & 1, ci, C, a, mark,
                 [&] { prefetch_ghost(epoch & 1); });
      mark(4);
#ifdef MLG_RES_SKEW
      stamp(li, it_now, 2);
#endif
      ++epoch;
      if (t == 0) {
        CgCtl cc = s_ctl;
        update_ctl<kPhaseIter>(cc, a, A.tol, maxit);
        s_ctl = cc;
      }
      __syncthreads();
      mark(5);
      if (A.trace != nullptr && t == 0) s_tr[15] += 1;
    }
    // x of the slab -> pooled output (cg_index layout)
    for (int j = t; j < npts; j += kResT) {
      const int row = j / pitch, col = j - row * pitch;
      if (col < S.w) A.X[cg_index(S, ya + row, col)] = Xs[j];
    }
    if (ci == 0 && t == 0) A.ctl[sid] = s_ctl;
    __syncthreads();  // shared memory is reused by the next system
  }
  if (A.trace != nullptr && t < 16) A.trace[blockIdx.x * 16 + t] = s_tr[t];
}

constexpr int kResNVar = static_cast<int>(sizeof(kResVariants) / sizeof(kResVariants[0]));
template <int V>
const void* res_kernel_v(bool lap) {
  return lap ? reinterpret_cast<const void*>(&k_cg_resident<true, kResVariants[V]>)
             : reinterpret_cast<const void*>(&k_cg_resident<false, kResVariants[V]>);
}
const void* res_kernel(int v, bool lap) {
  static_assert(kResNVar == 5, "one case per instantiated capacity");
  switch (v) {
    case 0: return res_kernel_v<0>(lap);
    case 1: return res_kernel_v<1>(lap);
    case 2: return res_kernel_v<2>(lap);
    case 3: return res_kernel_v<3>(lap);
    default: return res_kernel_v<4>(lap);
  }
}

}  // namespace

// Host plan: CTAs per lane C, the kernel instantiation (points per thread) and
// the system -> lane assignment.  Every system must fit: ceil(h / C) rows x
// pitch points per CTA within the instantiation's capacity, plus the shared
// buffers (p with ghost rows, x); each C runs the smallest instantiation that
// fits.  Among the feasible plans the smallest estimated makespan wins: a
// lane's time is the sum over its systems of iterations (~ proportional to the
// window's larger side) x per-iteration cost (the lane exchange + the point
// loops' slots).
bool CgBatch::solve_resident(Ctx& c, double tol, CgResult& res) {
  static const int env = [] {
    const char* e = std::getenv("MLG_CG_RESIDENT");  // A/B hook: 0 disables
    return e ? std::atoi(e) : 1;
  }();
  if (!env || L->uniform == 0 || sys_h.empty()) return false;
  for (const CgSys& s : sys_h)  // (fused publish: the first row lies in the first slots)
    if (s.pitch > kFirstSlots * kResT) return false;
  int dev = 0, nsm = 0, smem_optin = 0;
  MLG_CUDA(cudaGetDevice(&dev));
  MLG_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  MLG_CUDA(cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  int smem_sm = 0;
  MLG_CUDA(cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev));
  // kResPerSM CTAs share an SM's shared memory (1 KB per CTA reserved by the driver)
  const int smem_cta = std::min(smem_optin, smem_sm / kResPerSM - 1024);
  const int slots = nsm * kResPerSM;  // co-resident CTAs of the cooperative launch
  // static shared memory of the kernel (s_red, s_sum, s_ctl, trace slots)
  const int static_smem = [] {
    std::size_t m = 0;
    for (int v = 0; v < kResNVar; ++v)
      for (int lap = 0; lap < 2; ++lap) {
        cudaFuncAttributes fa{};
        cudaFuncGetAttributes(&fa, res_kernel(v, lap != 0));
        m = std::max(m, fa.sharedSizeBytes);
      }
    return static_cast<int>(m) + 64;
  }();
  const int nsys = static_cast<int>(sys_h.size());
  int max_pitch = 1, max_h = 1;
  for (const CgSys& s : sys_h) {
    max_pitch = std::max(max_pitch, s.pitch);
    max_h = std::max(max_h, s.h);
  }
  auto smem_for = [&](int cap) {  // p with ghost rows, x, ghost r (kernel layout)
    return (2LL * cap + (kGhostR ? 4 : 2) * max_pitch + 4) * 8;
  };
  // smallest instantiated capacity that holds every system's slab with C CTAs per lane
  auto variant_for = [&](int C) {
    long long need = 0;
    for (const CgSys& s : sys_h) need = std::max(need, static_cast<long long>((s.h + C - 1) / C) * s.pitch);
    int best_v = -1;
    for (int v = 0; v < kResNVar; ++v) {
      const long long cap = static_cast<long long>(kResT) * kResVariants[v];
      if (cap < need || smem_for(static_cast<int>(cap)) + static_smem > smem_cta) continue;
      if (best_v < 0 || kResVariants[v] < kResVariants[best_v]) best_v = v;
    }
    return best_v;
  };
  // per-iteration cost model (microseconds), from the cycle traces of configs 2
  // and 5 (profiles/r2E_resident_trace_c2.txt, r2E_resident_trace_c5.txt): the
  // lane exchange (L2 round trips + the fixed per-iteration work, growing slowly
  // with the lane width) plus ~200 cycles per register slot of the point loops
  auto iter_cost = [&](int C, int pt) { return 2.95 + 0.006 * C + 0.100 * pt; };
  double best = 1e300;
  int bestC = 0, bestV = -1;
  std::vector<std::vector<int>> best_lanes;
  std::vector<int> order(static_cast<std::size_t>(nsys));
  std::iota(order.begin(), order.end(), 0);
  for (int C = 1; C <= slots; ++C) {
    const int var = variant_for(C);
    if (var < 0) continue;
    const int nl = slots / C;
    if (nl < 1) break;
    // LPT: systems by decreasing cost to the least-loaded lane
    std::vector<double> cost(static_cast<std::size_t>(nsys));
    for (int s = 0; s < nsys; ++s) {
      const CgSys& S = sys_h[static_cast<std::size_t>(s)];
      cost[static_cast<std::size_t>(s)] = std::max(S.w, S.h) * iter_cost(C, kResVariants[var]);
    }
    std::vector<int> ord = order;
    std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) {
      return cost[static_cast<std::size_t>(a)] > cost[static_cast<std::size_t>(b)];
    });
    std::vector<double> load(static_cast<std::size_t>(nl), 0.0);
    std::vector<std::vector<int>> lanes(static_cast<std::size_t>(nl));
    for (int s : ord) {
      const auto it = std::min_element(load.begin(), load.end());
      const std::size_t l = static_cast<std::size_t>(it - load.begin());
      lanes[l].push_back(s);
      load[l] += cost[static_cast<std::size_t>(s)];
    }
    const double span = *std::max_element(load.begin(), load.end());
    if (span < best * 0.999) {
      best = span;
      bestC = C;
      bestV = var;
      best_lanes = lanes;
    }
  }
  if (bestC == 0) return false;
  const int C = bestC;
  while (!best_lanes.empty() && best_lanes.back().empty()) best_lanes.pop_back();
  const int nl = static_cast<int>(best_lanes.size());
  std::size_t per = 1;
  for (const auto& l : best_lanes) per = std::max(per, l.size() + 1);
  std::vector<int> lanes_h(static_cast<std::size_t>(nl) * per, -1);
  for (int l = 0; l < nl; ++l)
    for (std::size_t k = 0; k < best_lanes[static_cast<std::size_t>(l)].size(); ++k)
      lanes_h[static_cast<std::size_t>(l) * per + k] = best_lanes[static_cast<std::size_t>(l)][k];
  cudaStream_t st = c.stream;
  res_lanes.ensure(lanes_h.size());
  res_lanes.upload(lanes_h.data(), lanes_h.size(), st);
  res_bar.ensure(static_cast<std::size_t>(nl) * 32);
  res_bar.zero(st);
  res_part.ensure(static_cast<std::size_t>(nl) * 2 * kCgDots * part_cpad(C));
  res_halo.ensure(static_cast<std::size_t>(nl) * 2 * C * 2 * kHaloFields * max_pitch);
  const int cap = kResT * kResVariants[bestV];
  res_bslab.ensure(static_cast<std::size_t>(2) * nl * C * cap);
  ctl_d.zero(st);

  ResArgs A{};
  A.sys = sys_d.get();
  A.lanes = res_lanes.get();
  A.per_lane = static_cast<int>(per);
  A.C = C;
  A.nlanes = nl;
  A.bsrc = bsrc;
  A.bstride = bstride;
  A.nxp1 = L->nx + 1;
  A.X = X.get();
  A.ctl = ctl_d.get();
  A.part = res_part.get();
  A.halo = res_halo.get();
  A.hpitch = max_pitch;
  A.bslab = res_bslab.get();
  A.bar = res_bar.get();
  A.sg = L->strip_geom;
  A.masked = mask != nullptr;
  A.tol = tol;
  A.ust = L->ust;
  A.udinv = L->udinv;
  static const bool trace_on = std::getenv("MLG_RES_TRACE") != nullptr;
  DevBuf<unsigned long long> trace_buf;
  if (trace_on) {
    trace_buf.alloc(static_cast<std::size_t>(nl) * C * 16 * 5);
    trace_buf.zero(st);
    A.trace = trace_buf.get();
  }
  const bool lap = L->ust.c == 4.0 && L->ust.e == -1.0 && L->ust.n == -1.0 &&
                   L->ust.ne == 0.0 && L->udinv == 0.25 &&
                   std::getenv("MLG_CG_NOLAP") == nullptr;  // (test hook: generic stencil)
  const void* fn = res_kernel(bestV, lap);
  const int dyn = static_cast<int>(smem_for(cap));
  MLG_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn));
  int per_sm = 0;
  MLG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kResT, dyn));
  if (per_sm * nsm < nl * C) return false;  // cooperative launch needs co-residency
  const bool prof = c.profile;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (prof) {
    e0 = c.event(0);
    e1 = c.event(1);
    MLG_CUDA(cudaEventRecord(e0, st));
  }
  void* args[] = {(void*)&A};
  MLG_CUDA(cudaLaunchCooperativeKernel(fn, dim3(nl * C), dim3(kResT), args, dyn, st));
  ++launch_counter();
  if (prof) MLG_CUDA(cudaEventRecord(e1, st));
  std::vector<CgCtl> ctl(static_cast<std::size_t>(nsys));
  ctl_d.download(ctl.data(), ctl.size(), st);
  c.sync();
  if (trace_on) {
    std::vector<unsigned long long> tr(static_cast<std::size_t>(nl) * C * 16 * 5);
    trace_buf.download(tr.data(), tr.size(), st);
    c.sync();
    double sum[16] = {0}, mx[16] = {0};
    for (int b = 0; b < nl * C; ++b)
      for (int k = 0; k < 16; ++k) {
        sum[k] += static_cast<double>(tr[static_cast<std::size_t>(b) * 16 + k]);
        mx[k] = std::max(mx[k], static_cast<double>(tr[static_cast<std::size_t>(b) * 16 + k]));
      }
    const double it = std::max(1.0, sum[15] / (nl * C));
    // marks in program order (thread 0): cycles since the previous mark
    static const int order[] = {0, 1, 2, 3, 6, 7, 8, 4, 5, 9};
    static const char* names[] = {"phase1", "ghost+sync", "phase2", "publish", "warp trees+sync",
                                  "block sums+arrive+wait", "lane sums+sync", "(-)", "ctl",
                                  "(unused)"};
    fprintf(stderr, "resident trace: %d lanes x %d CTAs x %d points/thread, %d systems, %s, %.0f iterations/CTA; "
            "cycles per iteration (thread 0), mean over CTAs (max over CTAs of the per-CTA mean):",
            nl, C, kResVariants[bestV], nsys, mask ? "strip" : "local", it);
    double tot = 0.0;
    for (int k = 0; k < 10; ++k) {
      fprintf(stderr, " %s %.0f (%.0f),", names[k], sum[order[k]] / (nl * C) / it,
              mx[order[k]] / it);
      tot += sum[order[k]] / (nl * C) / it;
    }
    fprintf(stderr, " total %.0f\n", tot);
#ifdef MLG_RES_SKEW
    {  // lane 0: per stamped iteration, spread over the lane's CTAs of each stamp (ns)
      const std::size_t base = static_cast<std::size_t>(nl) * C * 16;
      for (int i = 0; i < 16; ++i) {
        unsigned long long lo[3] = {~0ull, ~0ull, ~0ull}, hi[3] = {0, 0, 0};
        for (int b = 0; b < C; ++b)
          for (int w = 0; w < 3; ++w) {
            const unsigned long long v = tr[base + (static_cast<std::size_t>(b) * 16 + i) * 4 + w];
            lo[w] = std::min(lo[w], v);
            hi[w] = std::max(hi[w], v);
          }
        fprintf(stderr, "skew it %d: start spread %llu ns, store spread %llu ns (first store "
                "%llu ns after first start), done spread %llu ns (first done %llu ns after last "
                "store)\n", 500 + i, hi[0] - lo[0], hi[1] - lo[1], lo[1] - lo[0], hi[2] - lo[2],
                lo[2] - hi[1]);
      }
      // per-CTA store time relative to the lane's first store, iteration 508
      fprintf(stderr, "skew it 508 store offsets (ns) by CTA:");
      unsigned long long first = ~0ull;
      for (int b = 0; b < C; ++b) first = std::min(first, tr[base + (static_cast<std::size_t>(b) * 16 + 8) * 4 + 1]);
      for (int b = 0; b < C; ++b)
        fprintf(stderr, " %llu", tr[base + (static_cast<std::size_t>(b) * 16 + 8) * 4 + 1] - first);
      fprintf(stderr, "\n");
    }
#endif
  }
  for (const CgCtl& q : ctl)
    if (q.status == kIndefinite)
      throw SolverError("cg_solve: matrix is not positive definite (p'Mp <= 0)");
  res.reports.assign(ctl.size(), SolveReport{});
  res.iters_max = 0;
  double row_iters = 0.0;
  for (std::size_t k = 0; k < ctl.size(); ++k) {
    res.reports[k].iterations = ctl[k].iters;
    res.reports[k].final_residual = ctl[k].final_res;
    res.reports[k].converged = ctl[k].status == kConverged ? 1 : 0;
    res.iters_max = std::max(res.iters_max, ctl[k].iters);
    row_iters += static_cast<double>(sys_h[k].nrows) * ctl[k].iters;
  }
  if (prof) {
    float ms = 0.f;
    MLG_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    if (mask) {
      c.times.ks_ms += ms;
      c.times.ks_launches += 1;
      c.times.ks_row_iters += row_iters;
      c.times.ks_bytes_per_row = 72;
    } else {
      c.times.ka_ms_sum += ms;
      c.times.ka_launches += 1;
      c.times.ka_launches_all += 1;
      c.times.ka_rows += row_iters;
      c.times.ka_uniform = 3;
    }
  }
  (mask ? c.times.ks_kernel : c.times.ka_kernel) = 2;
  return true;
}

}  // namespace mlg
