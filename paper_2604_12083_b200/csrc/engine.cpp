// engine.cpp — parareal::run on one device as a stream/event DAG (pswim_parareal_run_gpu), and
// the same scheduler over host propagator callbacks (pswim_parareal_run_host).
//
// What it computes is the reference's recurrence (src/parareal.cpp:58-89, the serial blocks
// coarse_sweep_initial / fine_parallel / correct):
//   X[0][n] = G(X[0][n-1])                                     iteration 0, the coarse sweep
//   X[k][k] = F(X[k-1][k-1]),  X[k][n] = X[k-1][n] for n < k   (converged prefix, frozen)
//   X[k][n] = (F(X[k-1][n-1]) + G(X[k][n-1])) - G(X[k-1][n-1])   k < n <= N
// with eta_tilde_k = max_n metric(X[k][n], X[k-1][n]), eta_k = max_n metric(ref[n], X[k][n]),
// the stop rule eta_tilde_k < tol or k == N (converged), k == min(l_max, N) (not), and reports
// in iteration order (parareal.hpp:47-58, parareal.cpp:366-393).
//
// How it runs is GPU-first rather than a worker-thread dispatcher.  The whole task set of an
// iteration is known once its predecessor is enqueued, so the host walks the (k, n) grid
// iteration by iteration and ENQUEUES every task at once onto CUDA streams, each task waiting
// on the events of exactly the states it reads:
//   * fine lanes (low priority): F[k][n] on lane 1 + (n-1) % (m-1), the reference's fine-task
//     placement (parareal.cpp:262-273), so m-1 fine solves run side by side on the GPU;
//   * wavefront lanes (highest priority): the coarse sweep and each iteration's corrector
//     chain G + correct, one stream per in-flight iteration, so iteration k+1's chain can run
//     while iteration k's is still finishing -- the overlap the pipelined schedule exists for;
//   * the iteration metrics are one batched kernel on the wavefront lane whose row is copied
//     to pinned memory behind an event.
// There is no host synchronisation per task.  The host blocks only on an iteration's metric
// row, once per iteration, and only after it has already enqueued `lookahead` further
// iterations (pipelined mode): fine(k+1, n) is speculative exactly as in the reference, which
// dispatches it when X[k][n-1] appears, before eta_tilde_k is known.  Regular mode enqueues
// iteration k+1 after the iteration-k decision (the barrier) and orders each iteration's
// correctors after all of its fine solves.
//
// States are one slab of HBM, (count x 12N doubles), with every (k, n) state a fixed slot;
// frozen states and X[k][k] are aliases, never copies.  Results are bitwise independent of
// the mode, the worker count and the lookahead (every value is computed by the same kernels
// from the same inputs), which tests/test_gpu_parareal.py checks.
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <utility>
#include <vector>

#include "ctx.h"
#include "parareal_common.h"

namespace pswim {

int parareal_lookahead(const pswim_plan& plan) {
    if (plan.mode != 1) return 0;
    int w = 1;
    if (const char* e = std::getenv("PSWIM_PARAREAL_LOOKAHEAD")) w = std::max(1, std::atoi(e));
    return w;
}

namespace {

// Lane contexts are pooled across runs (one process runs Parareal many times: the bench's
// l sweeps, an application's repeated solves): creating a context allocates HBM workspaces
// and synchronises, which would otherwise dominate short runs.  Keyed by device, stream
// priority and scenario; a returned context is drained and its error flags cleared.
class LanePool {
  public:
    pswim_ctx* get(int device, const pswim_scenario& sc, int prio) {
        {
            std::lock_guard<std::mutex> lk(mu_);
            for (size_t i = 0; i < free_.size(); ++i)
                if (free_[i].device == device && free_[i].prio == prio &&
                    std::memcmp(&free_[i].sc, &sc, sizeof sc) == 0) {
                    pswim_ctx* c = free_[i].ctx;
                    free_.erase(free_.begin() + static_cast<long>(i));
                    return c;
                }
        }
        return pswim_create(device, &sc, prio);
    }
    void put(pswim_ctx* c, int prio) {
        if (!c) return;
        c->sync();  // drains the stream, clears any raised device flag
        std::lock_guard<std::mutex> lk(mu_);
        free_.push_back(Entry{c->device, prio, c->sc, c});
        while (free_.size() > kMaxPooled) {  // oldest first
            pswim_destroy(free_.front().ctx);
            free_.erase(free_.begin());
        }
    }

  private:
    static constexpr size_t kMaxPooled = 48;
    struct Entry {
        int device, prio;
        pswim_scenario sc;
        pswim_ctx* ctx;
    };
    std::mutex mu_;
    std::vector<Entry> free_;
};

}  // namespace

LanePool& lane_pool() {
    static LanePool* pool = new LanePool();  // never destroyed: contexts outlive static teardown order
    return *pool;
}

pswim_ctx* pooled_ctx(int device, const pswim_scenario& sc, int prio) { return lane_pool().get(device, sc, prio); }
void release_ctx(pswim_ctx* c, int prio) { lane_pool().put(c, prio); }

namespace {


// ---------------------------------------------------------------------------------------
// Executors: where a task runs.  A mark is the "ready" token of a task's output.
// ---------------------------------------------------------------------------------------
using Pairs = std::vector<std::pair<int, int>>;  // (first, second) buffers of a metric

class Executor {
  public:
    virtual ~Executor() = default;
    virtual void reserve(int buffers) = 0;
    virtual void upload(int buf, const double* h) = 0;
    // out = G or F of `in` over [t0, t1]; kind kCoarse (sweep) or kFine; (k, n) for the trace
    virtual int propagate(int lane, int worker, TaskKind kind, int k, int n, double t0, double t1, int in, int out,
                          const std::vector<int>& deps) = 0;
    // gn = G(in) over [t0, t1]; xn = (fp + gn) - go   (one corrector task, kind kCorrect)
    virtual int correct(int lane, int k, int n, double t0, double t1, int in, int fp, int go, int gn, int xn,
                        const std::vector<int>& deps) = 0;
    // iteration k's metric row: eta_tilde over `et`, eta over `e`
    virtual void metrics(int lane, int k, const Pairs& et, const Pairs& e, const std::vector<int>& deps) = 0;
    virtual void read_metrics(int k, double* eta_tilde, double* eta) = 0;  // blocks for row k
    virtual void finish() = 0;                                             // drain; throws on failure
    virtual void download(int buf, double* h) = 0;
    virtual double trace(std::vector<pswim_trace_event>* out) = 0;         // returns W
};

class HostExec final : public Executor {
  public:
    HostExec(int64_t len, pswim_propagator_fn c, void* cu, pswim_propagator_fn f, void* fu, int dim, int stride)
        : len_(len), c_(c), cu_(cu), f_(f), fu_(fu), dim_(dim), stride_(stride), origin_(Clock::now()) {}
    void reserve(int buffers) override { bufs_.assign(buffers, std::vector<double>(len_)); }
    void upload(int buf, const double* h) override { std::memcpy(bufs_[buf].data(), h, len_ * sizeof(double)); }
    int propagate(int, int worker, TaskKind kind, int k, int n, double t0, double t1, int in, int out,
                  const std::vector<int>&) override {
        const double a = now();
        call(kind == kFine ? f_ : c_, kind == kFine ? fu_ : cu_, t0, t1, in, out);
        events_.push_back(pswim_trace_event{worker, kind, a, now(), k, n});
        return -1;
    }
    int correct(int, int k, int n, double t0, double t1, int in, int fp, int go, int gn, int xn,
                const std::vector<int>&) override {
        const double a = now();
        call(c_, cu_, t0, t1, in, gn);
        const double *p = bufs_[fp].data(), *g = bufs_[gn].data(), *o = bufs_[go].data();
        double* x = bufs_[xn].data();
        for (int64_t i = 0; i < len_; ++i) x[i] = (p[i] + g[i]) - o[i];  // parareal.cpp:52
        events_.push_back(pswim_trace_event{0, kCorrect, a, now(), k, n});
        return -1;
    }
    void metrics(int, int k, const Pairs& et, const Pairs& e, const std::vector<int>&) override {
        double a = 0.0, b = 0.0;
        for (auto [x, y] : et) a = std::max(a, host_metric(bufs_[x].data(), bufs_[y].data(), len_, dim_, stride_));
        for (auto [x, y] : e) b = std::max(b, host_metric(bufs_[x].data(), bufs_[y].data(), len_, dim_, stride_));
        if ((int)rows_.size() <= k) rows_.resize(k + 1);
        rows_[k] = {a, b};
    }
    void read_metrics(int k, double* eta_tilde, double* eta) override {
        *eta_tilde = rows_[k].first;
        *eta = rows_[k].second;
    }
    void finish() override {}
    void download(int buf, double* h) override { std::memcpy(h, bufs_[buf].data(), len_ * sizeof(double)); }
    double trace(std::vector<pswim_trace_event>* out) override {
        *out = events_;
        return finalize_idle(out);
    }

  private:
    double now() const { return std::chrono::duration<double>(Clock::now() - origin_).count(); }
    void call(pswim_propagator_fn fn, void* user, double t0, double t1, int in, int out) {
        const int rc = fn(user, t0, t1, bufs_[in].data(), bufs_[out].data(), len_, nullptr);
        if (rc) throw CodeError(rc, "parareal: propagator failed");
    }
    int64_t len_;
    pswim_propagator_fn c_;
    void* cu_;
    pswim_propagator_fn f_;
    void* fu_;
    int dim_, stride_;
    Clock::time_point origin_;
    std::vector<std::vector<double>> bufs_;
    std::vector<std::pair<double, double>> rows_;
    std::vector<pswim_trace_event> events_;
};

// One device: lane contexts (own stream + rhs workspaces each), a slab of state slots, and a
// timed event pair per task (the schedule trace is read from the device clock afterwards).
class GpuExec final : public Executor {
  public:
    GpuExec(const pswim_scenario& sc, int device, int wave_lanes, int fine_lanes, int64_t fine_steps,
            int64_t coarse_steps)
        : device_(device), len_(12 * sc.rod_count * sc.nodes_per_rod), fine_steps_(fine_steps),
          coarse_steps_(coarse_steps) {
        int lo = 0, hi = 0;
        cudaSetDevice(device);
        cudaDeviceGetStreamPriorityRange(&lo, &hi);
        for (int i = 0; i < wave_lanes + fine_lanes; ++i) {
            const int prio = i < wave_lanes ? hi : lo;
            pswim_ctx* c = pooled_ctx(device, sc, prio);
            if (!c) throw CodeError(PSWIM_ECUDA, "parareal: cannot create lane context");
            // Small systems (fused cluster kernel): the wavefront lanes (coarse sweep,
            // correctors: the sequential critical path) take 16-CTA clusters while at most 8
            // fine lanes run 8-CTA ones beside them (flagellum, n = 8: l = 1 823k -> 851k
            // simulated steps/s; fine lanes on 16 CTAs no longer fit side by side: 631k).
            // The cluster size only splits targets: results are bitwise unchanged.
            if (i < wave_lanes && fine_lanes <= 8) pswim_set_fused(c, 16);
            lanes_.push_back(c);
            prios_.push_back(prio);
        }
    }
    ~GpuExec() override {
        drain();
        cudaSetDevice(device_);
        for (auto& t : tasks_) {
            cudaEventDestroy(t.a);
            cudaEventDestroy(t.b);
        }
        if (origin_) cudaEventDestroy(origin_);
        for (auto& r : rows_)
            if (r.ready) cudaEventDestroy(r.ready);
        if (slab_) cudaFree(slab_);
        if (d_rows_) cudaFree(d_rows_);
        if (h_rows_) cudaFreeHost(h_rows_);
        for (size_t i = 0; i < lanes_.size(); ++i) {
            pswim_set_fused(lanes_[i], 1);  // the pool's default cluster cap
            release_ctx(lanes_[i], prios_[i]);
        }
    }
    void reserve(int buffers) override {
        cudaSetDevice(device_);
        const size_t bytes = static_cast<size_t>(buffers) * len_ * sizeof(double);
        if (cudaMalloc(&slab_, bytes) != cudaSuccess) {
            cudaGetLastError();
            throw CodeError(PSWIM_ECUDA, "parareal: the state slab (" + std::to_string(bytes >> 20) +
                                             " MiB) does not fit in HBM");
        }
        nbuf_ = buffers;
    }
    void upload(int buf, const double* h) override {
        lanes_[0]->use();
        if (cudaMemcpyAsync(ptr(buf), h, len_ * sizeof(double), cudaMemcpyHostToDevice, lanes_[0]->stream) !=
            cudaSuccess)
            throw CodeError(PSWIM_ECUDA, "parareal: upload");
    }
    // allocations of the run (metric rows; the state slab is reserve())
    void prepare(int iterations, int row_len) {
        lanes_[0]->use();
        row_len_ = row_len;
        const size_t n = static_cast<size_t>(iterations + 1) * row_len;
        if (cudaMalloc(&d_rows_, n * sizeof(double)) != cudaSuccess ||
            cudaMallocHost(&h_rows_, n * sizeof(double)) != cudaSuccess)
            throw CodeError(PSWIM_ECUDA, "parareal: metric rows");
        rows_.assign(iterations + 1, Row{});
        cudaEventCreate(&origin_);
    }
    // the schedule's time origin: after the uploads
    void start() {
        cudaStreamSynchronize(lanes_[0]->stream);  // uploads done; pageable sources released
        cudaEventRecord(origin_, lanes_[0]->stream);
    }
    int propagate(int lane, int worker, TaskKind kind, int k, int n, double t0, double t1, int in, int out,
                  const std::vector<int>& deps) override {
        pswim_ctx* c = begin(lane, deps, worker, kind, k, n);
        const bool fine = kind == kFine;
        const int rc = c->propagate_async(ptr(in), t0, t1, fine ? PSWIM_RK2 : PSWIM_EULER,
                                          fine ? fine_steps_ : coarse_steps_, 0.0, ptr(out));
        if (rc) throw CodeError(rc, c->err);
        return end(c);
    }
    int correct(int lane, int k, int n, double t0, double t1, int in, int fp, int go, int gn, int xn,
                const std::vector<int>& deps) override {
        pswim_ctx* c = begin(lane, deps, 0, kCorrect, k, n);
        const int rc = c->propagate_async(ptr(in), t0, t1, PSWIM_EULER, coarse_steps_, 0.0, ptr(gn));
        if (rc) throw CodeError(rc, c->err);
        if (correct_launch(ptr(fp), ptr(gn), ptr(go), len_, ptr(xn), c->stream) != cudaSuccess)
            throw CodeError(PSWIM_ECUDA, "parareal: correct");
        return end(c);
    }
    void metrics(int lane, int k, const Pairs& et, const Pairs& e, const std::vector<int>& deps) override {
        pswim_ctx* c = lanes_[lane];
        c->use();
        wait(c, deps);
        double* row = d_rows_ + static_cast<size_t>(k) * row_len_;
        Pairs all = et;
        all.insert(all.end(), e.begin(), e.end());
        for (size_t base = 0; base < all.size(); base += kMetricPairs) {
            MetricPairs mp;
            mp.count = static_cast<int>(std::min<size_t>(kMetricPairs, all.size() - base));
            for (int i = 0; i < mp.count; ++i) {
                mp.x[i] = ptr(all[base + i].first);
                mp.y[i] = ptr(all[base + i].second);
            }
            if (metric_pairs_launch(mp, len_, row + base, c->stream) != cudaSuccess)
                throw CodeError(PSWIM_ECUDA, "parareal: metric");
        }
        Row& r = rows_[k];
        r.et = static_cast<int>(et.size());
        r.e = static_cast<int>(e.size());
        if (cudaMemcpyAsync(h_rows_ + static_cast<size_t>(k) * row_len_, row, all.size() * sizeof(double),
                            cudaMemcpyDeviceToHost, c->stream) != cudaSuccess ||
            cudaEventCreateWithFlags(&r.ready, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventRecord(r.ready, c->stream) != cudaSuccess)
            throw CodeError(PSWIM_ECUDA, "parareal: metric row");
    }
    void read_metrics(int k, double* eta_tilde, double* eta) override {
        const Row& r = rows_[k];
        if (cudaEventSynchronize(r.ready) != cudaSuccess) throw CodeError(PSWIM_ECUDA, "parareal: metric wait");
        const double* h = h_rows_ + static_cast<size_t>(k) * row_len_;
        double a = 0.0, b = 0.0;
        for (int i = 0; i < r.et; ++i) a = std::max(a, h[i]);
        for (int i = 0; i < r.e; ++i) b = std::max(b, h[r.et + i]);
        *eta_tilde = a;
        *eta = b;
    }
    void finish() override {
        for (auto* c : lanes_) {
            const int rc = c->sync();  // stream drained + device error flags (stiffness, ...)
            if (rc) throw CodeError(rc, c->err);
        }
    }
    void download(int buf, double* h) override {
        cudaSetDevice(device_);
        if (cudaMemcpy(h, ptr(buf), len_ * sizeof(double), cudaMemcpyDeviceToHost) != cudaSuccess)
            throw CodeError(PSWIM_ECUDA, "parareal: download");
    }
    double trace(std::vector<pswim_trace_event>* out) override {
        out->clear();
        for (const auto& t : tasks_) {
            float a = 0.f, b = 0.f;
            cudaEventElapsedTime(&a, origin_, t.a);
            cudaEventElapsedTime(&b, origin_, t.b);
            out->push_back(pswim_trace_event{t.worker, t.kind, 1e-3 * a, 1e-3 * b, t.k, t.n});
        }
        return finalize_idle(out);
    }

  private:
    struct Task {
        cudaEvent_t a = nullptr, b = nullptr;
        int32_t worker = 0, kind = 0, k = 0, n = 0;
    };
    struct Row {
        cudaEvent_t ready = nullptr;
        int et = 0, e = 0;
    };
    double* ptr(int buf) const { return slab_ + static_cast<size_t>(buf) * len_; }
    void wait(pswim_ctx* c, const std::vector<int>& deps) {
        for (int d : deps)
            if (d >= 0 && cudaStreamWaitEvent(c->stream, tasks_[d].b, 0) != cudaSuccess)
                throw CodeError(PSWIM_ECUDA, "parareal: event wait");
    }
    pswim_ctx* begin(int lane, const std::vector<int>& deps, int worker, TaskKind kind, int k, int n) {
        pswim_ctx* c = lanes_[lane];
        c->use();
        wait(c, deps);
        Task t;
        t.worker = worker;
        t.kind = kind;
        t.k = k;
        t.n = n;
        if (cudaEventCreate(&t.a) != cudaSuccess || cudaEventCreate(&t.b) != cudaSuccess ||
            cudaEventRecord(t.a, c->stream) != cudaSuccess)
            throw CodeError(PSWIM_ECUDA, "parareal: task event");
        tasks_.push_back(t);
        return c;
    }
    int end(pswim_ctx* c) {
        if (cudaEventRecord(tasks_.back().b, c->stream) != cudaSuccess)
            throw CodeError(PSWIM_ECUDA, "parareal: task event");
        return static_cast<int>(tasks_.size()) - 1;
    }
    void drain() {
        for (auto* c : lanes_) {
            cudaSetDevice(device_);
            cudaStreamSynchronize(c->stream);
        }
    }

    int device_;
    int64_t len_, fine_steps_, coarse_steps_;
    std::vector<pswim_ctx*> lanes_;
    std::vector<int> prios_;
    double* slab_ = nullptr;
    int nbuf_ = 0;
    std::vector<Task> tasks_;
    cudaEvent_t origin_ = nullptr;
    double* d_rows_ = nullptr;
    double* h_rows_ = nullptr;
    int row_len_ = 0;
    std::vector<Row> rows_;
};

// ---------------------------------------------------------------------------------------
// The scheduler: walks the (k, n) grid and enqueues each iteration as a unit.
// ---------------------------------------------------------------------------------------
class Wavefront {
  public:
    // lanes: [0, wave) wavefront lanes, [wave, wave + fine) fine lanes (fine == 0: all on 0)
    Wavefront(const pswim_plan& plan, Executor& ex, int wave, int fine)
        : p_(plan), ex_(ex), N_(plan.intervals), L_(std::min(plan.max_iterations, plan.intervals)),
          M_(plan.workers), wave_(wave), fine_(fine), W_(parareal_lookahead(plan)) {
        const auto grid = [&](std::vector<std::vector<Cell>>& g) { g.assign(L_ + 1, std::vector<Cell>(N_ + 1)); };
        grid(X_);
        grid(G_);
        grid(F_);
    }

    // Slots the run needs: x0, the sweep's G, per iteration k its F (N-k+1), G and X (N-k
    // each), and the N+1 reference states.
    static int slots(int N, int L, bool ref) {
        int s = 1 + N;
        for (int k = 1; k <= L; ++k) s += (N - k + 1) + 2 * (N - k);
        return s + (ref ? N + 1 : 0);
    }

    void run(const double* x0, const double* ref, int64_t len, double* states_out, pswim_report* rep,
             std::vector<pswim_trace_event>* trace, GpuExec* gpu) {
        // setup (allocations) is not part of the run's wall time; uploads and downloads are
        ex_.reserve(slots(N_, L_, ref != nullptr));
        if (gpu) gpu->prepare(L_, 2 * N_);
        const auto t_run = Clock::now();
        X_[0][0] = Cell{take(), -1};
        ex_.upload(X_[0][0].buf, x0);
        if (ref) {
            ref_.resize(N_ + 1);
            for (int n = 0; n <= N_; ++n) {
                ref_[n] = take();
                ex_.upload(ref_[n], ref + len * n);
            }
        }
        if (gpu) gpu->start();
        sweep();
        int queued = 0, final_k = 0;
        bool converged = false;
        std::vector<double> et, ea;
        for (int k = 1; k <= L_; ++k) {
            while (queued < std::min(L_, k + W_)) iteration(++queued);
            double a = 0.0, b = 0.0;
            ex_.read_metrics(k, &a, &b);
            et.push_back(a);
            ea.push_back(b);
            final_k = k;
            if (a < p_.tolerance || k == N_) {  // at k = N every interval is exact (parareal.cpp:383-386)
                converged = true;
                break;
            }
        }
        ex_.finish();  // speculative iterations past the stop drain here
        for (int n = 0; n <= N_; ++n) ex_.download(X_[final_k][n].buf, states_out + len * n);
        rep->wall_seconds = std::chrono::duration<double>(Clock::now() - t_run).count();
        rep->iterations_used = final_k;
        rep->converged = converged ? 1 : 0;
        rep->eta_count = static_cast<int32_t>(et.size());
        for (size_t k = 0; k < et.size(); ++k) {
            if (rep->eta_tilde) rep->eta_tilde[k] = et[k];
            if (rep->eta && ref) rep->eta[k] = ea[k];
        }
        if (trace) rep->schedule_idle = ex_.trace(trace);
    }

  private:
    struct Cell {
        int buf = -1;
        int mark = -1;  // -1: ready before the schedule starts
    };
    int take() { return next_++; }
    int wave_lane(int k) const { return wave_ > 1 ? k % wave_ : 0; }
    int fine_lane(int n) const { return fine_ > 0 ? wave_ + (n - 1) % fine_ : 0; }
    int fine_worker(int n) const { return M_ >= 2 ? 1 + (n - 1) % (M_ - 1) : 0; }
    double t(int n) const { return boundary_time(p_, n); }

    void sweep() {  // iteration 0: X[0][n] = G(X[0][n-1])
        for (int n = 1; n <= N_; ++n) {
            const int out = take();
            const int mark = ex_.propagate(wave_lane(0), 0, kCoarse, 0, n, t(n - 1), t(n), X_[0][n - 1].buf, out,
                                           {X_[0][n - 1].mark});
            G_[0][n] = X_[0][n] = Cell{out, mark};
        }
    }

    void iteration(int k) {
        for (int n = 0; n < k; ++n) X_[k][n] = X_[k - 1][n];  // frozen prefix (parareal.cpp:332)
        std::vector<int> all_fine;
        for (int n = k; n <= N_; ++n) {  // fine_parallel: F(X[k-1][n-1])
            const int out = take();
            const int mark = ex_.propagate(fine_lane(n), fine_worker(n), kFine, k, n, t(n - 1), t(n), X_[k - 1][n - 1].buf,
                                           out, {X_[k - 1][n - 1].mark});
            F_[k][n] = Cell{out, mark};
            all_fine.push_back(mark);
        }
        X_[k][k] = F_[k][k];
        const int wl = wave_lane(k);
        for (int n = k + 1; n <= N_; ++n) {  // correct: the wavefront
            // regular: correctors after every fine solve of the iteration
            std::vector<int> deps = p_.mode == 0 ? all_fine : std::vector<int>{F_[k][n].mark};
            deps.push_back(X_[k][n - 1].mark);
            deps.push_back(G_[k - 1][n].mark);
            const int gn = take(), xn = take();
            const int mark = ex_.correct(wl, k, n, t(n - 1), t(n), X_[k][n - 1].buf, F_[k][n].buf, G_[k - 1][n].buf, gn,
                                         xn, deps);
            G_[k][n] = Cell{gn, mark};
            X_[k][n] = Cell{xn, mark};
        }
        Pairs et, e;
        std::vector<int> deps;
        for (int n = 1; n <= N_; ++n) {
            if (n >= k) et.emplace_back(X_[k][n].buf, X_[k - 1][n].buf);  // frozen: same slot, 0
            deps.push_back(X_[k][n].mark);
            deps.push_back(X_[k - 1][n].mark);
            if (!ref_.empty()) e.emplace_back(ref_[n], X_[k][n].buf);
        }
        ex_.metrics(wl, k, et, e, deps);
    }

    const pswim_plan p_;
    Executor& ex_;
    const int N_, L_, M_, wave_, fine_, W_;
    int next_ = 0;
    std::vector<std::vector<Cell>> X_, G_, F_;
    std::vector<int> ref_;
};

int run_schedule(const pswim_plan& plan, Executor& ex, GpuExec* gpu, int wave, int fine, const double* x0,
                 const double* ref, int64_t len, double* states_out, pswim_report* rep, pswim_trace_event* trace_out,
                 int64_t trace_cap, int64_t* trace_len) {
    try {
        Wavefront wf(plan, ex, wave, fine);
        std::vector<pswim_trace_event> trace;
        wf.run(x0, ref, len, states_out, rep, &trace, gpu);
        if (trace_len) *trace_len = static_cast<int64_t>(trace.size());
        if (trace_out) {
            const int64_t n = std::min<int64_t>(trace_cap, static_cast<int64_t>(trace.size()));
            std::copy(trace.begin(), trace.begin() + n, trace_out);
        }
    } catch (const CodeError& e) {
        return e.code;
    } catch (const std::exception&) {
        return PSWIM_ESTATE;
    }
    return PSWIM_OK;
}

}  // namespace
}  // namespace pswim

extern "C" {

int pswim_parareal_run_host(const pswim_plan* plan, pswim_propagator_fn coarse, void* cu, pswim_propagator_fn fine,
                            void* fu, const double* x0, int64_t len, int32_t dim, int32_t stride,
                            const double* reference, double* states_out, pswim_report* rep,
                            pswim_trace_event* trace_out, int64_t trace_cap, int64_t* trace_len) {
    using namespace pswim;
    if (plan_check(plan) || !coarse || !fine || !x0 || !states_out || !rep || len <= 0) return PSWIM_EINVAL;
    if (dim < 1 || stride < dim || len % stride != 0) return PSWIM_EINVAL;
    HostExec ex(len, coarse, cu, fine, fu, dim, stride);
    return run_schedule(*plan, ex, nullptr, 1, 0, x0, reference, len, states_out, rep, trace_out, trace_cap,
                        trace_len);
}

int pswim_parareal_run_gpu(const pswim_plan* plan, const pswim_scenario* sc, int device, int64_t fine_steps,
                           int64_t coarse_steps, const double* x0, const double* reference, double* states_out,
                           pswim_report* rep, pswim_trace_event* trace_out, int64_t trace_cap, int64_t* trace_len) {
    using namespace pswim;
    if (plan_check(plan) || !sc || !x0 || !states_out || !rep || fine_steps < 1 || coarse_steps < 1)
        return PSWIM_EINVAL;
    // m = 1: one stream runs everything in enqueue order (a topological order).  m >= 2: m-1
    // fine lanes plus one wavefront lane per iteration in flight.
    const int m = plan->workers;
    const int wave = m >= 2 ? parareal_lookahead(*plan) + 1 : 1;
    const int fine = m >= 2 ? m - 1 : 0;
    try {
        GpuExec ex(*sc, device, wave, fine, fine_steps, coarse_steps);
        return run_schedule(*plan, ex, &ex, wave, fine, x0, reference, 12 * sc->rod_count * sc->nodes_per_rod,
                            states_out, rep, trace_out, trace_cap, trace_len);
    } catch (const CodeError& e) {
        return e.code;
    }
}

}  // extern "C"
