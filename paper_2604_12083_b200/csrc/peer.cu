// peer.cu — fused sharded MRS + all-gather over peer memory.
//
// Every rank owns one exchange block in its HBM: [arrival counter | u0 | w0 | u1 | w1]
// (velocities double-buffered by rhs parity).  Ranks map each other's blocks -- CUDA IPC
// handles across processes (NVLink P2P on an NVSwitch box), raw pointers for in-process
// ranks -- and the sharded MRS kernel (mrs.cu, kPeer epilogue) stores each finished target's
// (u, w) into EVERY rank's block and bumps every rank's counter with a system-scope atomic.
// No separate collective runs: the all-gather is the producing kernel's epilogue.  A
// one-thread acquire spin (peer_wait_kernel) orders the consumer (advance) after all ranks'
// arrivals for this rhs.  Results are bitwise identical to the single-GPU propagate.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "ctx.h"
#include "internal.h"

struct pswim_peer_group {
    pswim_ctx* ctx = nullptr;
    int rank = 0, world = 1;
    int64_t n = 0;            // nodes
    size_t block_bytes = 0;
    void* block = nullptr;    // local exchange block
    std::vector<void*> peers;  // every rank's block as seen from this device
    std::vector<bool> opened;  // IPC-opened (to close on destroy)
    pswim::PeerOut* d_out[2] = {nullptr, nullptr};  // device-resident epilogue tables, per parity
    unsigned long long gen = 0;  // rhs evaluations completed
    int parity = 0;
    std::string err;

    unsigned long long* flag_of(void* base) const { return static_cast<unsigned long long*>(base); }
    double* u_of(void* base, int par) const {
        return reinterpret_cast<double*>(static_cast<char*>(base) + 256) + par * 6 * n;
    }
    double* w_of(void* base, int par) const { return u_of(base, par) + 3 * n; }
};

namespace {

int build_tables(pswim_peer_group* g) {
    for (int par = 0; par < 2; ++par) {
        pswim::PeerOut h;
        h.world = g->world;
        for (int r = 0; r < g->world; ++r) {
            h.u[r] = g->u_of(g->peers[r], par);
            h.w[r] = g->w_of(g->peers[r], par);
            h.flag[r] = g->flag_of(g->peers[r]);
        }
        if (!g->d_out[par] && cudaMalloc(&g->d_out[par], sizeof(pswim::PeerOut)) != cudaSuccess) return PSWIM_ECUDA;
        if (cudaMemcpy(g->d_out[par], &h, sizeof h, cudaMemcpyHostToDevice) != cudaSuccess) return PSWIM_ECUDA;
    }
    return PSWIM_OK;
}

}  // namespace

// ---- sharded rhs / step through the peer group ------------------------------------------
namespace pswim {

int peer_rhs(pswim_ctx* ctx, pswim_peer_group* g, const double* state, double t, double** u, double** w) {
    const RodParams& rp = ctx->rp;
    const bool lj = rp.rods >= 2 && rp.lj_well > 0.0;  // propagators.cpp:70
    if (lj) {
        const int rc = ctx->lj(state, ctx->d_lj);
        if (rc) return rc;
    }
    cudaError_t e = rod_loads_launch(rp, state, t, nullptr, ctx->d_f, ctx->d_n, nullptr, nullptr,
                                     lj ? ctx->d_lj : nullptr, nullptr, nullptr, ctx->d_flags, ctx->stream);
    if (e != cudaSuccess) return ctx->fail(PSWIM_ECUDA, std::string("rod_loads_launch: ") + cudaGetErrorString(e));
    const int64_t total = rp.rods * rp.m;
    const MrsPlan plan = mrs_plan(total, total);
    int rc = ctx->ensure_mrs(plan);
    if (rc) return rc;
    const int bpr = (plan.target_blocks + g->world - 1) / g->world;
    const int tb0 = std::min(plan.target_blocks, g->rank * bpr), tb1 = std::min(plan.target_blocks, tb0 + bpr);
    if (tb1 > tb0)
        e = mrs_launch_blocks(plan, tb0, tb1, state, state, 12, ctx->d_f, ctx->d_n, ctx->rs.epsilon, ctx->rs.mu,
                              nullptr, nullptr, ctx->d_scratch, ctx->d_counters, ctx->d_flags, ctx->stream,
                              g->d_out[g->parity]);
    else
        e = peer_token_launch(g->d_out[g->parity], ctx->stream);
    if (e != cudaSuccess) return ctx->fail(PSWIM_ECUDA, std::string("mrs peer launch: ") + cudaGetErrorString(e));
    // every rank's blocks have arrived (each of the plan's target blocks signals once per rhs,
    // each rank with an empty range once)
    int idle = 0;
    for (int r = 0; r < g->world; ++r)
        if (std::min(plan.target_blocks, r * bpr) >= plan.target_blocks) ++idle;
    ++g->gen;
    e = peer_wait_launch(g->flag_of(g->block), g->gen * (unsigned long long)(plan.target_blocks + idle), ctx->stream);
    if (e != cudaSuccess) return ctx->fail(PSWIM_ECUDA, "peer_wait");
    *u = g->u_of(g->block, g->parity);
    *w = g->w_of(g->block, g->parity);
    g->parity ^= 1;
    return PSWIM_OK;
}

int peer_step(pswim_ctx* ctx, pswim_peer_group* g, int scheme, const double* state, double t, double dt,
              double* out) {
    double *u = nullptr, *w = nullptr;
    int rc = peer_rhs(ctx, g, state, t, &u, &w);
    if (rc) return rc;
    if (scheme == PSWIM_EULER) return ctx->advance(state, u, w, dt, out);
    rc = ctx->advance(state, u, w, 0.5 * dt, ctx->d_mid);
    if (rc) return rc;
    rc = peer_rhs(ctx, g, ctx->d_mid, t + 0.5 * dt, &u, &w);
    if (rc) return rc;
    return ctx->advance(state, u, w, dt, out);
}

}  // namespace pswim

extern "C" {

pswim_peer_group* pswim_peer_group_create(pswim_ctx* ctx, int32_t rank, int32_t world) {
    if (!ctx || !ctx->has_scenario || world < 1 || world > pswim::kMaxPeers || rank < 0 || rank >= world)
        return nullptr;
    auto* g = new pswim_peer_group();
    g->ctx = ctx;
    g->rank = rank;
    g->world = world;
    g->n = ctx->rp.rods * ctx->rp.m;
    g->block_bytes = 256 + 2 * 6 * (size_t)g->n * sizeof(double);
    ctx->use();
    pswim::peer_preload();
    if (cudaMalloc(&g->block, g->block_bytes) != cudaSuccess || cudaMemset(g->block, 0, 256) != cudaSuccess ||
        cudaDeviceSynchronize() != cudaSuccess) {
        if (g->block) cudaFree(g->block);
        delete g;
        return nullptr;
    }
    g->peers.assign(world, nullptr);
    g->opened.assign(world, false);
    g->peers[rank] = g->block;
    return g;
}

int pswim_peer_group_handle(pswim_peer_group* g, uint8_t* handle64) {
    if (!g || !handle64) return PSWIM_EINVAL;
    cudaIpcMemHandle_t h;
    if (cudaIpcGetMemHandle(&h, g->block) != cudaSuccess) return PSWIM_ECUDA;
    static_assert(sizeof(h) == 64, "IPC handle size");
    std::memcpy(handle64, &h, sizeof h);
    return PSWIM_OK;
}

void* pswim_peer_group_local_base(pswim_peer_group* g) { return g ? g->block : nullptr; }

int pswim_peer_group_connect(pswim_peer_group* g, const uint8_t* handles, void* const* local_bases) {
    if (!g || (!handles && !local_bases)) return PSWIM_EINVAL;
    g->ctx->use();
    for (int r = 0; r < g->world; ++r) {
        if (r == g->rank) continue;
        if (local_bases) {
            g->peers[r] = local_bases[r];  // in-process rank (same process, any device)
        } else {
            cudaIpcMemHandle_t h;
            std::memcpy(&h, handles + 64 * r, sizeof h);
            void* p = nullptr;
            if (cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) return PSWIM_ECOMM;
            g->peers[r] = p;
            g->opened[r] = true;
        }
    }
    return build_tables(g) ? PSWIM_ECUDA : PSWIM_OK;
}

void pswim_peer_group_destroy(pswim_peer_group* g) {
    if (!g) return;
    g->ctx->use();
    cudaDeviceSynchronize();
    for (int r = 0; r < g->world; ++r)
        if (g->opened[r]) cudaIpcCloseMemHandle(g->peers[r]);
    for (auto* p : g->d_out)
        if (p) cudaFree(p);
    cudaFree(g->block);
    delete g;
}

int pswim_propagate_sharded_peer(pswim_ctx* ctx, pswim_peer_group* g, const double* d_in, double t0, double t1,
                                 int scheme, int64_t spi, double dtc, double* d_out) {
    if (!ctx || !g || g->ctx != ctx || !g->d_out[0]) return PSWIM_EINVAL;
    int rc = ctx->use();
    if (rc) return rc;
    if (t1 < t0) return ctx->fail(PSWIM_EINVAL, "propagate: t1 < t0");
    if (!ctx->has_scenario) return ctx->fail(PSWIM_EINVAL, "propagate: context has no scenario");
    if (ctx->sc.wall_mode == 1) return ctx->fail(PSWIM_EUNSUPPORTED_WALL, kWallMsg);
    const size_t bytes = sizeof(double) * 12 * static_cast<size_t>(g->n);
    if (d_in != d_out && cudaMemcpyAsync(d_out, d_in, bytes, cudaMemcpyDeviceToDevice, ctx->stream) != cudaSuccess)
        return ctx->fail(PSWIM_ECUDA, "propagate: copy");
    if (t1 > t0) {
        int64_t steps = 0;
        double dt = 0.0;
        if ((rc = ctx->resolve_steps(t0, t1, spi, dtc, &steps, &dt))) return rc;
        double t = t0;
        for (int64_t i = 0; i < steps; ++i) {
            if ((rc = pswim::peer_step(ctx, g, scheme, d_out, t, dt, d_out))) return rc;
            t += dt;  // propagators.cpp:159
        }
    }
    return ctx->sync();
}

}  // extern "C"
