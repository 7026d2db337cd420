// fused.cu — whole-interval propagation of small systems in ONE kernel.
//
// For N <= 256 nodes a launched-kernel RK2 step is six launches of a few microseconds of
// work each (BASELINE configs[0]: one 100-node flagellum), i.e. launch bound.  This kernel
// runs `steps` Euler / midpoint-RK2 steps (propagators.cpp:126-162) on a thread-block
// cluster with the state resident in shared memory:
//   * every CTA redundantly holds the full state and redundantly does the O(N) phases
//     (segment loads with sqrt_rotation, nodal loads, LJ, source staging, advance);
//   * the O(N^2) MRS is split across the CTAs of the cluster by target: each CTA computes
//     its targets' (target, source chunk) items, reduces the chunk partials in fixed order
//     in its own shared memory, and pushes each target's 6 velocities to every CTA through
//     distributed shared memory; one cluster barrier per rhs (velocities double-buffered).
// All per-element arithmetic is the kernels.cuh routines of the launched path, and the MRS
// decomposition (origin, chunk boundaries, chunk order) is the one mrs_plan picks for the
// same N, so a fused propagate is bitwise identical to the multi-kernel one.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>

#include "kernels.cuh"
#include "tma.cuh"

namespace cg = cooperative_groups;

namespace pswim {
namespace {

// Threads per CTA: 12 warps for KP = 256 (>= the 9 front warps at N = 256; 168 registers),
// 8 warps for KP = 128 (N <= 128: <= 5 front warps).  Every phase loops over the CTA's
// threads, so the count only sets the warps in flight; fewer idle warps make the per-rhs CTA
// barriers cheaper (flagellum, 16 CTAs: 169.7k -> 172.9k RK2 steps/s at 256 threads).
template <int KP>
constexpr int fused_threads() {
    return KP == 128 ? 256 : 384;
}
constexpr int kFrontNodes = 30;  // nodes owned per warp in the warp-tiled front pass
// KP (template): plane stride of the shared-memory state, velocity, position and source-record
// planes, 128 or 256 (>= n): a compile-time constant, so every strided access in the per-node
// chains folds into an immediate offset instead of integer address arithmetic.

struct FusedArgs {
    RodArgs rod;
    LjArgs lj;
    MrsConsts mc;
    int n;        // total nodes
    int rods, m;  // layout
    int chunks;   // MRS source chunks (== mrs_plan(n, n).chunks)
    int chunk_fixed;  // mrs_plan(n, n).fixed: sources per chunk (0: c N / C bounds)
    unsigned m_magic;  // __umulhi(g, m_magic) == g / m for g, m < 2^16 (no division on the chains)
    int lj_on;
    double max_disp;
    // shared-memory offsets (doubles)
    int off_x, off_xm, off_pos, off_f, off_n, off_seg, off_lj, off_rec, off_part, off_vel;
    int off_x2, off_tile;  // second step-start state buffer; per-warp front tiles (32 x 12)
    int off_bar;           // two mbarriers (velocity buffers)
    int off_om;            // preferred strain per segment index (m - 1), two tables: rhs r reads r & 1
    int off_cb;            // MRS chunk bounds (chunks + 1 ints)
    unsigned long long* prof;  // kFusedPhases clock64 counters (CTA 0, thread 0), nullptr = off
};

// In-kernel phase timer: clock64 deltas between the CTA barriers that end each phase, as seen
// by thread 0 of cluster rank 0 (the stage timers of propagators.hpp:55-65 for a path that is
// one kernel).  Phases: 0 segment loads (+LJ), 1 nodal loads, 2 MRS source staging, 3 MRS
// pairs, 4 chunk reduction + DSMEM velocity push, 5 cluster barrier, 6 advance.
template <bool kOn>
struct PhaseClock {
    // cycles accumulate in registers (the phase index is a constant at every inlined call
    // site) and reach global memory once, at the end of the launch: a global read-modify-write
    // per mark would put its load latency into the next phase's count
    unsigned long long* prof;
    long long t;
    unsigned long long acc[kFusedPhases];
    __device__ __forceinline__ PhaseClock(unsigned long long* p, long long t0) : prof(p), t(t0) {
#pragma unroll
        for (int i = 0; i < kFusedPhases; ++i) acc[i] = 0ull;
    }
    __device__ __forceinline__ void mark(int phase) {
        if constexpr (kOn) {
            const long long c = clock64();
            acc[phase] += (unsigned long long)(c - t);
            t = c;
        }
    }
    __device__ __forceinline__ void flush() {
        if constexpr (kOn) {
            if (prof)
#pragma unroll
                for (int i = 0; i < kFusedPhases; ++i) prof[i] += acc[i];
        }
    }
};

template <int CS>
__device__ __forceinline__ void cluster_barrier() {
    if constexpr (CS > 1) {
        cg::this_cluster().sync();
    } else {
        __syncthreads();
    }
}

// The preferred strain of every segment index at time t (rod.cpp:29-32) into table `om`:
// `sin` leaves the segment chains of the front pass (the same explicit-rounding rod_strain as
// every kernel).  Filled from the top thread down.
__device__ __forceinline__ void strain_table(const FusedArgs& a, double* om, double t) {
    for (int k = (int)blockDim.x - 1 - (int)threadIdx.x; k >= 0; k -= (int)blockDim.x)
        if (k < a.m - 1) om[k] = rod_strain(a.rod, k, t);
}

// Front half of an rhs (propagators.cpp:38-91): produce the rhs state -- `src` itself
// (vadv == nullptr) or dst = advance_state(src, vadv, h) node by node (propagators.cpp:93-124)
// -- and, on that state, the segment and nodal loads and the MRS source records (rec) and
// target positions (pos).
//
// Systems without LJ take a warp-tiled pass with no CTA barrier inside: warp w covers nodes
// 30 w - 1 + lane (lanes 1..30 own a node, lanes 0 and 31 recompute a neighbour's advance),
// advances them into a per-warp tile, computes segment (g, g+1) per lane and gets segment
// g - 1 by one shuffle -- the layout of rod_loads_wtma_kernel.  LJ needs every advanced
// position first, so LJ systems take the phased version.
template <int CS, int KP, bool kLj, bool kProf>
__device__ __forceinline__ void fused_front(const FusedArgs& a, double* sm, const double* src, const double* vadv, double h,
                                            double* dst, const double* om, double* om_next, double t_next, unsigned& fl,
                                            PhaseClock<kProf>& pc) {
    const int tid = threadIdx.x, bs = blockDim.x, N = a.n, m = a.m, nseg = a.rods * (m - 1);
    double* pos = sm + a.off_pos;
    double2* rec = reinterpret_cast<double2*>(sm + a.off_rec);
    if constexpr (!kLj) {
        const int warp = tid >> 5, lane = tid & 31, nw = (N + kFrontNodes - 1) / kFrontNodes;
        if (warp >= nw) {
            // the warps without front nodes tabulate the next rhs's preferred strain meanwhile
            // (its sin chains leave the MRS phase)
            for (int k = tid - 32 * nw; k < a.m - 1; k += bs - 32 * nw) om_next[k] = rod_strain(a.rod, k, t_next);
        } else {
            const int base = kFrontNodes * warp - 1, g = base + lane;
            const bool valid = g >= 0 && g < N;
            double* tile = sm + a.off_tile + warp * 32 * 12;  // planes [12][32]: slot l = node base + l
            // origin of the MRS coordinates: node 0 of the rhs state (advance_node's position
            // update, same operations)
            const d3 o = vadv ? ld3s(src, KP) + ld3s(vadv, KP) * h : ld3s(src, KP);
            // the rhs state's node into the warp tile: advanced from src (owner lanes 1..30 also
            // write it into the state buffer dst), or src's node itself for the first rhs
            if (valid && vadv)
                fl |= advance_node(src + g, vadv + g, vadv + 3 * KP + g, h, a.max_disp, tile + lane, KP, KP, 32,
                                   lane >= 1 && lane <= kFrontNodes ? dst + g : nullptr, KP);
            else if (valid)
#pragma unroll
                for (int q = 0; q < 12; ++q) tile[q * 32 + lane] = src[q * KP + g];
            __syncwarp();
            pc.mark(1);
            const int rod = valid ? (int)__umulhi((unsigned)g, a.m_magic) : 0, k = valid ? g - rod * m : 0;
            // the rod's node 0 and the plane stride (tile or state)
            const double* xs = tile + (rod * m - base);
            constexpr int xc = 32;
            double seg[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
            if (valid && lane < 31 && k + 1 < m)
                if (!rod_segment_om(a.rod, xs, k, om[k], seg, xc)) fl |= kFlagDegenerate;
            double prev[6];
#pragma unroll
            for (int q = 0; q < 6; ++q) prev[q] = __shfl_up_sync(0xffffffffu, seg[q], 1);
            pc.mark(2);
            if (valid && lane >= 1 && lane <= kFrontNodes) {
                const d3 xk = ld3s(xs + k, xc);
                const d3 xnext = k + 1 < m ? ld3s(xs + k + 1, xc) : xk;
                const d3 xprev = k > 0 ? ld3s(xs + k - 1, xc) : xk;
                d3 f, tq;
                node_loads(a.rod, k, seg, prev, xprev, xk, xnext, f, tq);
                st3s(pos + g, KP, xk);
                double2 r[9];
                if (!mrs_stage(&xk.x, 3, &f.x, &tq.x, 0, o.x, o.y, o.z, a.mc.scale, r)) fl |= kFlagNonFinite;
#pragma unroll
                for (int q = 0; q < 9; ++q) rec[q * KP + g] = r[q];
            }
        }
        __syncthreads();
        pc.mark(0);
    } else {
        // phased (LJ) version
        if (vadv) {
            for (int i = tid; i < N; i += bs)
                fl |= advance_node(src + i, vadv + i, vadv + 3 * KP + i, h, a.max_disp, dst + i, KP, KP, KP);
            __syncthreads();
        }
        const double* xs = vadv ? dst : src;
        double* fo = sm + a.off_f;
        double* no = sm + a.off_n;
        double* seg = sm + a.off_seg;
        double* ljf = sm + a.off_lj;
        for (int s = tid; s < nseg; s += bs) {
            const int r = s / (m - 1), k = s % (m - 1);
            if (!rod_segment_om(a.rod, xs + m * r, k, om[k], seg + 6 * s, KP)) fl |= kFlagDegenerate;
        }
        for (int i = tid; i < N; i += bs) {
            double fx = 0, fy = 0, fz = 0;
            const double xi = xs[i], yi = xs[KP + i], zi = xs[2 * KP + i];
            const int ri = i / m, ki = i - ri * m;
            for (int rj = 0, j = 0; rj < a.lj.rods; ++rj)
                for (int kj = 0; kj < m; ++kj, ++j)
                    lj_pair(a.lj, ri, ki, rj, kj, xi - xs[j], yi - xs[KP + j], zi - xs[2 * KP + j], fx, fy, fz);
            ljf[3 * i] = fx;
            ljf[3 * i + 1] = fy;
            ljf[3 * i + 2] = fz;
        }
        __syncthreads();
        for (int g = tid; g < N; g += bs) {
            const int r = g / m, k = g % m;
            d3 f, tq;
            rod_node(a.rod, xs + m * r, seg + 6 * (m - 1) * r, k, f, tq, KP);
            f = f + ld3(ljf + 3 * g) * a.rod.inv_ds;
            st3s(pos + g, KP, ld3s(xs + g, KP));
            st3(fo + 3 * g, f);
            st3(no + 3 * g, tq);
        }
        __syncthreads();
        strain_table(a, om_next, t_next);  // (this rhs's segment pass is done: barrier above)
        // stage every source relative to node 0 (the single target block's origin in mrs.cu)
        const double ox = pos[0], oy = pos[KP], oz = pos[2 * KP];
        for (int j = tid; j < N; j += bs) {
            double2 r[9];
            const d3 pj = ld3s(pos + j, KP);
            if (!mrs_stage(&pj.x, 0, fo, no, j, ox, oy, oz, a.mc.scale, r)) fl |= kFlagNonFinite;
#pragma unroll
            for (int q = 0; q < 9; ++q) rec[q * KP + j] = r[q];
        }
        __syncthreads();
        pc.mark(0);
    }
}

// Back half of an rhs: the O(N^2) MRS of the staged sources into vel[6 n] = (u, w) per node.
__device__ __forceinline__ uint32_t cluster_addr(uint32_t local, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
    return r;
}

// Asynchronous remote store of one double into CTA `rank`'s shared memory whose completion
// is counted (8 bytes of transaction) on that CTA's mbarrier.
__device__ __forceinline__ void st_async_f64(uint32_t raddr, double v, uint32_t rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(raddr), "d"(v),
                 "r"(rbar)
                 : "memory");
}

// Wait until this CTA's velocity buffer of the given mbarrier holds all N x 6 values of the
// rhs (every CTA's st.async pushes counted as transaction bytes): thread 0 posts the
// expected bytes and the one arrival, every thread waits on the phase parity.
// `phases` holds one phase-parity bit per velocity buffer (a register, not a local array).
template <int CS>
__device__ __forceinline__ void vel_wait(uint64_t* vbar, uint32_t& phases, int buf, int n) {
    if constexpr (CS > 1) {
        if (threadIdx.x == 0) mbar_expect_tx(vbar, (uint32_t)(6 * n * sizeof(double)));
        mbar_wait(vbar, (phases >> buf) & 1u);
        phases ^= 1u << buf;
    } else {
        __syncthreads();
    }
}

// This CTA's MRS targets [i0, i0 + nloc) of the cluster split (tpc per CTA), fixed for the
// launch: computed once, not per rhs (the divisions sat on every rhs's MRS path).
struct MrsSplit {
    int i0, nloc, tpc;
    unsigned nloc_magic;  // __umulhi(w, nloc_magic) == w / nloc for w < 2^16
    const int* cb;        // chunk bounds j0(c) = c N / C, c = 0..C (shared memory)
};

template <int CS, int KP, bool kProf>
__device__ __forceinline__ void fused_mrs(const FusedArgs& a, double* sm, double* vel, uint64_t* vbar,
                                          PhaseClock<kProf>& pc, const MrsSplit& sp) {
    const int tid = threadIdx.x, bs = blockDim.x, N = a.n;
    const double* pos = sm + a.off_pos;
    const double2* rec = reinterpret_cast<const double2*>(sm + a.off_rec);
    const double ox = pos[0], oy = pos[KP], oz = pos[2 * KP];
    // MRS: this CTA owns targets [i0, i1); items (target, source chunk) computed here, the
    // chunk partials reduced locally in fixed order (mrs.cu's last-CTA reduction), and each
    // target's 6 velocities pushed to every CTA of the cluster through DSMEM.
    const int tpc = sp.tpc, i0 = sp.i0, nloc = sp.nloc;
    double* lpart = sm + a.off_part;  // [chunks][6][tpc]
    const unsigned nloc_magic = sp.nloc_magic;
    for (int w = tid; w < nloc * a.chunks; w += bs) {
        const int c = (int)__umulhi((unsigned)w, nloc_magic), il = w - c * nloc, i = i0 + il;
        const int j0 = sp.cb[c], j1 = sp.cb[c + 1];
        const double tx = pos[i] - ox, ty = pos[KP + i] - oy, tz = pos[2 * KP + i] - oz;
        MrsAcc acc;
        acc.zero();
#pragma unroll 2
        for (int j = j0; j < j1; ++j)
            mrs_pair(acc, tx, ty, tz, rec[j], rec[KP + j], rec[2 * KP + j], rec[3 * KP + j], rec[4 * KP + j],
                     rec[5 * KP + j], rec[6 * KP + j], rec[7 * KP + j], rec[8 * KP + j], a.mc.e2, a.mc.c15e2, a.mc.cm75e4,
                     a.mc.c25e2);
        double out[6];
        mrs_finish(acc, tx, ty, tz, out);
#pragma unroll
        for (int q = 0; q < 6; ++q) lpart[(c * 6 + q) * tpc + il] = out[q];  // [chunk][component][target]
    }
    __syncthreads();
    pc.mark(3);
    // one thread per (target, component): the chunk partials summed in chunk order 0..C-1
    // (mrs.cu's last-CTA reduction, bitwise), then pushed to every CTA of the cluster
    for (int w = tid; w < nloc * 6; w += bs) {
        const int q = (int)__umulhi((unsigned)w, nloc_magic), il = w - q * nloc;  // lane-consecutive targets
        double sum = lpart[q * tpc + il];
#pragma unroll 8
        for (int c = 1; c < a.chunks; ++c) sum += lpart[(c * 6 + q) * tpc + il];
        const int i = i0 + il;
        if constexpr (CS > 1) {
            // st.async into every CTA (itself included), completion counted on its mbarrier:
            // no cluster barrier and no GPU-scope fence per rhs
            const uint32_t laddr = smem_u32(vel + q * KP + i), lbar = smem_u32(vbar);
#pragma unroll
            for (int rr = 0; rr < CS; ++rr) st_async_f64(cluster_addr(laddr, rr), sum, cluster_addr(lbar, rr));
        } else {
            vel[q * KP + i] = sum;
        }
    }
    if constexpr (kProf) __syncthreads();  // phase timer only: end of the push as one CTA-wide instant
    pc.mark(4);
}

template <int CS, int KP, bool kLj, bool kProf>
__global__ void __launch_bounds__(fused_threads<KP>(), 1)
fused_kernel(FusedArgs a, double* __restrict__ state, int64_t steps, double t0, double dt, int scheme,
             unsigned* __restrict__ flags) {
    extern __shared__ __align__(16) double sm[];
    const int tid = threadIdx.x, bs = blockDim.x, N = a.n;
    // shared-memory state: component planes [12][KP] (lane-consecutive nodes, no bank conflicts)
    for (int k = tid; k < 12 * N; k += bs) sm[a.off_x + (k % 12) * KP + k / 12] = state[k];
    uint64_t* vbar = reinterpret_cast<uint64_t*>(sm + a.off_bar);  // one mbarrier per velocity buffer
    if (tid == 0) {
        mbar_init(&vbar[0], 1);
        mbar_init(&vbar[1], 1);
        fence_mbar_init();
    }
    strain_table(a, sm + a.off_om, t0);  // table 0: rhs 0
    MrsSplit sp;
    {
        const int rank = CS > 1 ? (int)cg::this_cluster().block_rank() : 0;
        sp.tpc = (N + CS - 1) / CS;
        sp.i0 = rank * sp.tpc;
        sp.nloc = max(0, min(N, sp.i0 + sp.tpc) - sp.i0);
        sp.nloc_magic = sp.nloc > 0 ? 0xFFFFFFFFu / (unsigned)sp.nloc + 1u : 0u;
        int* cb = reinterpret_cast<int*>(sm + a.off_cb);
        // the plan's chunk bounds (mrs_chunk_bound): c N / C, or `fixed` sources per chunk
        for (int c = tid; c <= a.chunks; c += bs)
            cb[c] = a.chunk_fixed > 0 ? min(c * a.chunk_fixed, N) : c * N / a.chunks;  // (N <= 256: no overflow)
        sp.cb = cb;
    }
    cluster_barrier<CS>();  // barriers initialised before any CTA pushes into them
    unsigned fl = 0;
    const int crank = CS > 1 ? (int)cg::this_cluster().block_rank() : 0;
    PhaseClock<kProf> pc((kProf && tid == 0 && crank == 0) ? a.prof : nullptr, kProf ? clock64() : 0);
    // One loop iteration per rhs (one call site of each phase: half the code of a per-step
    // body, which matters for the instruction cache).  Buffers are picked by shared-memory
    // offsets (no runtime-indexed local arrays, so every state access stays an LDS):
    //   * step s starts from state buffer S(s) = x (s even) / x2 (s odd); the advance that
    //     produces an rhs state runs inside that rhs's front pass, never in place (overlap
    //     lanes read neighbours' old states); xm holds the RK2 midpoint;
    //   * rhs r writes velocity buffer r & 1 (double-buffered: a CTA that runs ahead pushes
    //     the next rhs into the other buffer while slower CTAs still read this one).
    // step_rk2 (propagators.cpp:130-133): mid = advance(S(s), v1, dt/2), S(s+1) = advance(S(s), v2, dt).
    const bool rk2 = scheme != PSWIM_EULER;
    const int64_t nrhs = rk2 ? 2 * steps : steps;
    uint32_t vph = 0u;  // phase-parity bit per velocity buffer
    double t = t0;
    for (int64_t r = 0; r < nrhs; ++r) {
        const int p = (int)(r & 1);
        const bool mid = rk2 && p;  // the RK2 midpoint rhs
        const int64_t s = rk2 ? (r >> 1) : r;
        const int o_start = (s & 1) ? a.off_x2 : a.off_x, o_prev = (s & 1) ? a.off_x : a.off_x2;
        const double* vadv = r > 0 ? sm + a.off_vel + (p ^ 1) * 6 * KP : nullptr;
        if (r > 0) vel_wait<CS>(&vbar[p ^ 1], vph, p ^ 1, N);
        pc.mark(5);
        const double* src = sm + (mid ? o_start : (r > 0 ? o_prev : o_start));
        double* dst = sm + (mid ? a.off_xm : o_start);
        // strain tables: this rhs reads table p; the next rhs's (at t + dt/2 for the RK2
        // midpoint, else the next step's t; t += dt below) goes to table p ^ 1 meanwhile
        fused_front<CS, KP, kLj, kProf>(a, sm, src, vadv, mid ? 0.5 * dt : dt, dst, sm + a.off_om + p * a.m,
                                   sm + a.off_om + (p ^ 1) * a.m, rk2 && !mid ? t + 0.5 * dt : t + dt, fl, pc);
        fused_mrs<CS, KP, kProf>(a, sm, sm + a.off_vel + p * 6 * KP, &vbar[p], pc, sp);
        if (!rk2 || mid) t += dt;  // propagators.cpp:159
    }
    // the last step's closing advance (no rhs follows): S(steps) = advance(S(steps - 1), v, dt)
    double* out = sm + ((steps & 1) ? a.off_x2 : a.off_x);
    if (nrhs > 0) {
        const int pl = (int)((nrhs - 1) & 1);
        const double* vadv = sm + a.off_vel + pl * 6 * KP;
        const double* src = sm + ((steps & 1) ? a.off_x : a.off_x2);
        vel_wait<CS>(&vbar[pl], vph, pl, N);
        pc.mark(5);
        for (int i = tid; i < N; i += bs)
            fl |= advance_node(src + i, vadv + i, vadv + 3 * KP + i, dt, a.max_disp, out + i, KP, KP, KP);
        __syncthreads();
        pc.mark(6);
    }
    if (crank == 0)
        for (int k = tid; k < 12 * N; k += bs) state[k] = out[(k % 12) * KP + k / 12];
    if (fl) atomicOr(flags, fl);
    pc.flush();
    cluster_barrier<CS>();  // no CTA may exit while others still push partials into it
}

// Function attributes are set once per process, at context creation (fused_preload), never on
// a launch path: a driver call that takes the context lock while a peer's device-side wait is
// pending could otherwise stall another thread's launch (Parareal peer hand-offs).
template <int CS, int KP, bool kLj, bool kProf>
cudaError_t configure_one() {
    cudaError_t e = cudaFuncSetAttribute(fused_kernel<CS, KP, kLj, kProf>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e == cudaSuccess && CS > 8)
        e = cudaFuncSetAttribute(fused_kernel<CS, KP, kLj, kProf>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    return e;
}

template <int CS, int KP>
void load_cs() {
    cudaFuncAttributes fa;  // loads the module on the current device (lazy loading)
    cudaFuncGetAttributes(&fa, fused_kernel<CS, KP, false, false>);
    cudaFuncGetAttributes(&fa, fused_kernel<CS, KP, false, true>);
    cudaFuncGetAttributes(&fa, fused_kernel<CS, KP, true, false>);
    cudaFuncGetAttributes(&fa, fused_kernel<CS, KP, true, true>);
}

template <int CS, int KP>
void configure_cs() {
    configure_one<CS, KP, false, false>();
    configure_one<CS, KP, false, true>();
    configure_one<CS, KP, true, false>();
    configure_one<CS, KP, true, true>();
}

template <int CS, int KP, bool kLj, bool kProf>
cudaError_t launch_one(const FusedArgs& a, size_t smem, double* state, int64_t steps, double t0, double dt, int scheme,
                      unsigned* flags, cudaStream_t st) {
    // (function attributes: configure_cs, run by fused_preload at context creation)
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(CS);
    cfg.blockDim = dim3(fused_threads<KP>());
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, fused_kernel<CS, KP, kLj, kProf>, a, state, steps, t0, dt, scheme, flags);
}

// the phase-timer instantiation only for pswim_fused_profile: the production kernel has no
// timer code at all
template <int CS, int KP>
cudaError_t launch_cs(const FusedArgs& a, size_t smem, double* state, int64_t steps, double t0, double dt, int scheme,
                      unsigned* flags, cudaStream_t st) {
    // LJ systems take the phased front, the others the warp-tiled one: separate kernels, so
    // neither carries the other's code (the flagellum kernel is 3.4k instead of 5.1k SASS
    // instructions: +2.2 % from instruction-cache misses alone)
    if (a.lj_on)
        return a.prof ? launch_one<CS, KP, true, true>(a, smem, state, steps, t0, dt, scheme, flags, st)
                      : launch_one<CS, KP, true, false>(a, smem, state, steps, t0, dt, scheme, flags, st);
    return a.prof ? launch_one<CS, KP, false, true>(a, smem, state, steps, t0, dt, scheme, flags, st)
                  : launch_one<CS, KP, false, false>(a, smem, state, steps, t0, dt, scheme, flags, st);
}

// Shared-memory layout of a fused launch (offsets in doubles, 16-B aligned) into a; returns the
// doubles used.  Planes of stride KP: x, xm, x2 (12 each), pos (3), rec (18 = 9 double2),
// velocities (2 x 6); the warp-tiled front's tiles (fast path) share one region with the
// phased path's f / n / lj / segment buffers (LJ systems), which never coexist.
int64_t fused_layout(const RodParams& p, const MrsPlan& plan, int cs, FusedArgs& a) {
    const int64_t n = p.rods * p.m, kp = n <= 128 ? 128 : 256, tpc = (n + cs - 1) / cs;
    int64_t off = 0;
    auto take = [&](int64_t count) {
        const int64_t o = off;
        off += (count + 1) & ~int64_t(1);  // keep 16-B alignment
        return (int)o;
    };
    a.off_x = take(12 * kp);
    a.off_xm = take(12 * kp);
    a.off_x2 = take(12 * kp);
    a.off_pos = take(3 * kp);
    a.off_rec = take(18 * kp);
    a.off_vel = take(12 * kp);
    a.off_part = take(plan.chunks * tpc * 6);
    const int64_t shared = off;  // union: front tiles | f, n, lj, seg
    a.off_tile = take(((n + kFrontNodes - 1) / kFrontNodes) * 32 * 12);
    const int64_t after_tiles = off;
    off = shared;
    a.off_f = take(3 * n);
    a.off_n = take(3 * n);
    a.off_lj = take(3 * n);
    a.off_seg = take(6 * p.rods * (p.m - 1));
    off = std::max(off, after_tiles);
    a.off_bar = take(2);
    a.off_om = take(2 * p.m);
    a.off_cb = take((plan.chunks + 2) / 2);
    return off;
}

}  // namespace

// Returns the cluster size the fused path would use for this scenario (0 = not eligible).
int fused_cluster_size(const RodParams& p, int max_hint) {
    const int64_t n = p.rods * p.m;
    if (n > 256 || n < 2) return 0;
    const MrsPlan plan = mrs_plan(n, n);
    static const int max_cs_env = [] {
        const char* e = std::getenv("PSWIM_FUSED_MAX_CLUSTER");
        const int v = e ? std::atoi(e) : 8;
        return (v == 1 || v == 2 || v == 4 || v == 8 || v == 16) ? v : 8;
    }();
    static const int min_tpc_env = [] {
        const char* e = std::getenv("PSWIM_FUSED_MIN_TARGETS");
        return e ? std::max(1, std::atoi(e)) : 12;
    }();
    // a per-context hint (pswim_set_fused 2..16) overrides the default: a lone small system
    // runs fastest on 16 CTAs (>= 6 targets each); concurrent Parareal lanes keep <= 8
    const int max_cs = max_hint >= 2 ? max_hint : max_cs_env;
    const int min_tpc = max_hint >= 16 ? 6 : min_tpc_env;
    int cs = 1;
    while (cs < max_cs && (n + 2 * cs - 1) / (2 * cs) >= min_tpc) cs *= 2;  // >= min_tpc targets per CTA
    FusedArgs a;
    const int64_t doubles = fused_layout(p, plan, cs, a);
    if (doubles * 8 > 220 * 1024) return 0;
    return cs;
}

void fused_preload() {
    // attributes set once per process, modules loaded on every device that creates a context
    // (every launch path stays free of attribute calls and lazy-loading synchronisation)
    static const bool once = [] {
        configure_cs<1, 128>();
        configure_cs<2, 128>();
        configure_cs<4, 128>();
        configure_cs<8, 128>();
        configure_cs<16, 128>();
        configure_cs<1, 256>();
        configure_cs<2, 256>();
        configure_cs<4, 256>();
        configure_cs<8, 256>();
        configure_cs<16, 256>();
        return true;
    }();
    (void)once;
    load_cs<1, 128>();
    load_cs<2, 128>();
    load_cs<4, 128>();
    load_cs<8, 128>();
    load_cs<16, 128>();
    load_cs<1, 256>();
    load_cs<2, 256>();
    load_cs<4, 256>();
    load_cs<8, 256>();
    load_cs<16, 256>();
}

cudaError_t fused_propagate_launch(const RodParams& p, double* state, int64_t steps, double t0, double dt, int scheme,
                                   unsigned* flags, cudaStream_t st, unsigned long long* prof, int max_hint) {
    const int cs = fused_cluster_size(p, max_hint);
    if (cs == 0) return cudaErrorInvalidValue;
    const int64_t n = p.rods * p.m;
    const MrsPlan plan = mrs_plan(n, n);
    FusedArgs a;
    a.rod = rod_args(p);
    a.lj = lj_args(p);
    a.mc = mrs_consts(p.epsilon, p.mu);
    a.n = (int)n;
    a.rods = (int)p.rods;
    a.m = (int)p.m;
    a.chunks = plan.chunks;
    a.chunk_fixed = plan.fixed;
    a.m_magic = 0xFFFFFFFFu / (unsigned)p.m + 1u;
    a.lj_on = (p.rods >= 2 && p.lj_well > 0.0) ? 1 : 0;  // propagators.cpp:70
    a.max_disp = 10.0 * p.ds;
    a.prof = prof;
    const int64_t doubles = fused_layout(p, plan, cs, a);
    const size_t smem = (size_t)doubles * sizeof(double);
    if (n <= 128) {
        switch (cs) {
            case 1: return launch_cs<1, 128>(a, smem, state, steps, t0, dt, scheme, flags, st);
            case 2: return launch_cs<2, 128>(a, smem, state, steps, t0, dt, scheme, flags, st);
            case 4: return launch_cs<4, 128>(a, smem, state, steps, t0, dt, scheme, flags, st);
            case 8: return launch_cs<8, 128>(a, smem, state, steps, t0, dt, scheme, flags, st);
            default: return launch_cs<16, 128>(a, smem, state, steps, t0, dt, scheme, flags, st);
        }
    }
    switch (cs) {
        case 1: return launch_cs<1, 256>(a, smem, state, steps, t0, dt, scheme, flags, st);
        case 2: return launch_cs<2, 256>(a, smem, state, steps, t0, dt, scheme, flags, st);
        case 4: return launch_cs<4, 256>(a, smem, state, steps, t0, dt, scheme, flags, st);
        case 8: return launch_cs<8, 256>(a, smem, state, steps, t0, dt, scheme, flags, st);
        default: return launch_cs<16, 256>(a, smem, state, steps, t0, dt, scheme, flags, st);
    }
}

}  // namespace pswim
