// parareal.cpp — time-parallel drivers.
//
// (1) Engine: the physics-agnostic task-graph driver of parareal::run (reference
//     include/pintswim/parareal.hpp:85-86, src/parareal.cpp:118-438): regular and pipelined
//     schedules, worker lanes (serial lane 0 with priority, fine task n on lane
//     1 + (n-1) % (m-1)), stop rule, iteration-ordered reports, schedule trace.  Backends:
//       HostBackend  host states + C propagator callbacks  (pswim_parareal_run_host)
//       GpuBackend   HBM states, one device context (stream) per worker lane, coarse =
//                    Euler / fine = RK2 as harness::prepare (harness.cpp:5-33)
//                                                           (pswim_parareal_run_gpu)
// (2) RankDriver: one time slice per rank (rank p owns interval p+1, intervals == world),
//     the same recurrence (parareal.cpp:58-89) with one state hand-off per iteration to
//     rank p+1 and one allreduce(max) of [eta_tilde, eta] per iteration; coarse/corrector on
//     a high-priority stream, fine on a low-priority stream; pipelined mode launches the
//     next fine solve the moment its input arrives.  Transports: NCCL (one process per GPU,
//     nccl_transport.cpp), in-process threads + peer copies (pswim_parareal_run_threads),
//     host callbacks (CPU tests over gloo).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstring>
#include <deque>
#include <exception>
#include <functional>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "ctx.h"
#include "internal.h"

namespace pswim {
namespace {

using Clock = std::chrono::steady_clock;

struct CodeError : std::runtime_error {
    int code;
    CodeError(int c, const std::string& w) : std::runtime_error(w), code(c) {}
};

int plan_check(const pswim_plan* p) {
    // validate, parareal.cpp:38-45
    if (!p || p->intervals < 1 || p->workers < 1) return PSWIM_EINVAL;
    if (p->max_iterations < 1) return PSWIM_EINVAL;
    if (!(p->tolerance > 0.0)) return PSWIM_EINVAL;
    if (p->horizon <= 0.0) return PSWIM_EINVAL;
    return PSWIM_OK;
}

// ParallelPlan::boundary_time, parareal.hpp:44 — every caller uses this expression so all
// propagator calls see bitwise-identical interval ends.
inline double boundary_time(const pswim_plan& p, int n) { return p.t0 + (p.horizon / p.intervals) * n; }

// pointwise metric over groups: |x_i - y_i| / |x_i| on `dim` entries every `stride`
// (parareal.cpp:15-34 with stride == dim; io.cpp:49-68 with dim 3, stride 12).
double host_metric(const double* x, const double* y, int64_t len, int dim, int stride) {
    double worst = 0.0;
    for (int64_t i = 0; i < len; i += stride) {
        double num = 0.0, den = 0.0;
        for (int c = 0; c < dim; ++c) {
            const double d = x[i + c] - y[i + c];
            num += d * d;
            den += x[i + c] * x[i + c];
        }
        num = std::sqrt(num);
        den = std::sqrt(den);
        worst = std::max(worst, den < 1e-14 ? num : num / den);
    }
    return worst;
}

// ---------------------------------------------------------------------------------------
// Engine backends
// ---------------------------------------------------------------------------------------
struct State {
    std::vector<double> host;
    double* dev = nullptr;
    std::function<void(double*)> release;
    ~State() {
        if (dev && release) release(dev);
    }
};
using StatePtr = std::shared_ptr<const State>;

class EngineBackend {
  public:
    virtual ~EngineBackend() = default;
    virtual StatePtr initial(const double* x0) = 0;
    // Runs on worker `w`'s thread; returns when the result is complete.
    virtual StatePtr propagate(int w, bool coarse, double t0, double t1, const State& in) = 0;
    // Driver thread.
    virtual StatePtr corrected(const State& xp, const State& gn, const State& go) = 0;
    virtual double metric(const State& x, const State& y) = 0;
    virtual double metric_ref(const double* ref_host, const State& x) = 0;
    virtual void download(const State& s, double* out) = 0;
};

class HostBackend final : public EngineBackend {
  public:
    HostBackend(int64_t len, pswim_propagator_fn c, void* cu, pswim_propagator_fn f, void* fu, int dim, int stride)
        : len_(len), coarse_(c), cuser_(cu), fine_(f), fuser_(fu), dim_(dim), stride_(stride) {}
    StatePtr initial(const double* x0) override {
        auto s = std::make_shared<State>();
        s->host.assign(x0, x0 + len_);
        return s;
    }
    StatePtr propagate(int, bool coarse, double t0, double t1, const State& in) override {
        auto s = std::make_shared<State>();
        s->host.resize(len_);
        const int rc = coarse ? coarse_(cuser_, t0, t1, in.host.data(), s->host.data(), len_, nullptr)
                              : fine_(fuser_, t0, t1, in.host.data(), s->host.data(), len_, nullptr);
        if (rc) throw CodeError(rc, "propagator failed");
        return s;
    }
    StatePtr corrected(const State& xp, const State& gn, const State& go) override {
        auto s = std::make_shared<State>();
        s->host.resize(len_);
        for (int64_t i = 0; i < len_; ++i) s->host[i] = xp.host[i] + gn.host[i] - go.host[i];  // parareal.cpp:52
        return s;
    }
    double metric(const State& x, const State& y) override {
        return host_metric(x.host.data(), y.host.data(), len_, dim_, stride_);
    }
    double metric_ref(const double* ref, const State& x) override {
        return host_metric(ref, x.host.data(), len_, dim_, stride_);
    }
    void download(const State& s, double* out) override { std::memcpy(out, s.host.data(), len_ * sizeof(double)); }

  private:
    int64_t len_;
    pswim_propagator_fn coarse_;
    void* cuser_;
    pswim_propagator_fn fine_;
    void* fuser_;
    int dim_, stride_;
};

// Fixed-size device buffer pool shared by every lane (all states have one size).
class DevicePool {
  public:
    DevicePool(int device, int64_t len) : device_(device), bytes_(len * sizeof(double)) {}
    ~DevicePool() {
        cudaSetDevice(device_);
        for (double* p : free_) cudaFree(p);
    }
    double* get() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            if (!free_.empty()) {
                double* p = free_.back();
                free_.pop_back();
                return p;
            }
        }
        cudaSetDevice(device_);
        double* p = nullptr;
        if (cudaMalloc(&p, bytes_) != cudaSuccess) throw CodeError(PSWIM_ECUDA, "parareal: out of device memory");
        return p;
    }
    void put(double* p) {
        std::lock_guard<std::mutex> lk(mu_);
        free_.push_back(p);
    }
    size_t bytes() const { return bytes_; }
    // Allocate up front (cudaMalloc inside a run would serialise against running kernels).
    void reserve(int count) {
        cudaSetDevice(device_);
        std::lock_guard<std::mutex> lk(mu_);
        for (int i = 0; i < count; ++i) {
            double* p = nullptr;
            if (cudaMalloc(&p, bytes_) != cudaSuccess) break;
            free_.push_back(p);
        }
    }

  private:
    int device_;
    size_t bytes_;
    std::mutex mu_;
    std::vector<double*> free_;
};

class GpuBackend final : public EngineBackend {
  public:
    GpuBackend(const pswim_scenario& sc, int device, int workers, int64_t fine_steps, int64_t coarse_steps,
               int reserve_states)
        : len_(12 * sc.rod_count * sc.nodes_per_rod), fine_steps_(fine_steps), coarse_steps_(coarse_steps) {
        pool_ = std::make_shared<DevicePool>(device, len_);
        pool_->reserve(reserve_states);
        int lo = 0, hi = 0;
        cudaDeviceGetStreamPriorityRange(&lo, &hi);
        // lane 0 = serial wavefront (coarse + correctors): highest priority
        for (int w = 0; w < workers; ++w) {
            pswim_ctx* c = pswim_create(device, &sc, w == 0 ? hi : lo);
            if (!c) throw CodeError(PSWIM_ECUDA, "parareal: cannot create worker context");
            lanes_.push_back(c);
        }
        driver_ = pswim_create(device, nullptr, hi);
        if (!driver_) throw CodeError(PSWIM_ECUDA, "parareal: cannot create driver context");
    }
    ~GpuBackend() override {
        for (auto* c : lanes_) pswim_destroy(c);
        pswim_destroy(driver_);
    }
    StatePtr make() {
        auto s = std::make_shared<State>();
        auto pool = pool_;
        s->dev = pool->get();
        s->release = [pool](double* p) { pool->put(p); };
        return s;
    }
    StatePtr initial(const double* x0) override {
        auto s = make();
        driver_->use();
        if (cudaMemcpy(s->dev, x0, pool_->bytes(), cudaMemcpyHostToDevice) != cudaSuccess)
            throw CodeError(PSWIM_ECUDA, "parareal: upload");
        return s;
    }
    StatePtr propagate(int w, bool coarse, double t0, double t1, const State& in) override {
        auto s = make();
        pswim_ctx* c = lanes_[w];
        c->use();
        int rc = c->propagate_async(in.dev, t0, t1, coarse ? PSWIM_EULER : PSWIM_RK2,
                                    coarse ? coarse_steps_ : fine_steps_, 0.0, s->dev);
        if (!rc) rc = c->sync();
        if (rc) throw CodeError(rc, c->err);
        return s;
    }
    StatePtr corrected(const State& xp, const State& gn, const State& go) override {
        auto s = make();
        driver_->use();
        if (correct_launch(xp.dev, gn.dev, go.dev, len_, s->dev, driver_->stream) != cudaSuccess)
            throw CodeError(PSWIM_ECUDA, "parareal: correct");
        const int rc = driver_->sync();
        if (rc) throw CodeError(rc, driver_->err);
        return s;
    }
    double metric(const State& x, const State& y) override {
        double v = 0.0;
        const int rc = pswim_position_metric(driver_, x.dev, y.dev, len_, &v);
        if (rc) throw CodeError(rc, driver_->err);
        return v;
    }
    double metric_ref(const double* ref, const State& x) override {
        return host_metric_vs(ref, x);
    }
    void download(const State& s, double* out) override {
        driver_->use();
        if (cudaMemcpy(out, s.dev, pool_->bytes(), cudaMemcpyDeviceToHost) != cudaSuccess)
            throw CodeError(PSWIM_ECUDA, "parareal: download");
    }

  private:
    double host_metric_vs(const double* ref, const State& x) {
        std::vector<double> h(len_);
        download(x, h.data());
        return host_metric(ref, h.data(), len_, 3, 12);
    }
    int64_t len_, fine_steps_, coarse_steps_;
    std::shared_ptr<DevicePool> pool_;
    std::vector<pswim_ctx*> lanes_;
    pswim_ctx* driver_ = nullptr;
};

// ---------------------------------------------------------------------------------------
// Engine: task graph over slots (k, n), k = 0..L, n = 0..N.
// ---------------------------------------------------------------------------------------
enum Kind { kCoarse = 0, kFine = 1, kCorrect = 2, kIdle = 3 };

struct Task {
    Kind kind = kFine;
    int k = 0, n = 0;
    double t0 = 0, t1 = 0;
    StatePtr input;
};

struct Done {
    Task task;
    StatePtr result;
    std::exception_ptr error;
};

class Engine {
  public:
    Engine(const pswim_plan& plan, EngineBackend& be, const double* reference, int64_t len)
        : plan_(plan), be_(be), ref_(reference), len_(len), N_(plan.intervals),
          L_(std::min(plan.max_iterations, plan.intervals)), M_(plan.workers), lanes_(plan.workers),
          lane_events_(plan.workers) {
        const auto grid = [&](auto& v) { v.assign(L_ + 1, std::vector<typename std::decay_t<decltype(v)>::value_type::value_type>(N_ + 1)); };
        grid(X_);
        grid(G_);
        grid(F_);
        fine_sent_.assign(L_ + 1, std::vector<char>(N_ + 1, 0));
        corr_sent_.assign(L_ + 1, std::vector<char>(N_ + 1, 0));
        fines_left_.assign(L_ + 1, 0);
        for (int k = 1; k <= L_; ++k) fines_left_[k] = N_ - k + 1;
        slots_left_.assign(L_ + 1, N_);
        iter_ready_.assign(L_ + 1, 0);
    }

    void run(const double* x0, double* states_out, pswim_report* rep, std::vector<pswim_trace_event>* trace) {
        origin_ = Clock::now();
        put_state(0, 0, be_.initial(x0));
        // The sweep head is queued before any lane starts so lane 0's serial tier
        // outranks a fine task seeded at t = 0 (parareal.cpp:147-151).
        submit(Task{kCoarse, 0, 1, boundary_time(plan_, 0), boundary_time(plan_, 1), X_[0][0]});
        notify_pending();
        std::vector<std::thread> threads;
        for (int w = 0; w < M_; ++w) threads.emplace_back([this, w] { lane_loop(w); });
        while (outstanding_ > 0) {
            Done d = next_done();
            --outstanding_;
            if (d.error && !failure_) {
                failure_ = d.error;
                halt_ = true;  // drain: a propagator failure aborts the run
            }
            if (!halt_ && d.result) {
                try {
                    on_done(d);
                } catch (...) {
                    if (!failure_) failure_ = std::current_exception();
                    halt_ = true;
                }
            }
            notify_pending();
        }
        for (auto& l : lanes_) {
            std::lock_guard<std::mutex> lk(l.mu);
            l.closed = true;
            l.cv.notify_one();
        }
        for (auto& t : threads) t.join();
        if (failure_) std::rethrow_exception(failure_);

        const int kf = final_k_;
        for (int n = 0; n <= N_; ++n) {
            if (!X_[kf][n]) throw CodeError(PSWIM_ESTATE, "parareal: missing boundary state at termination");
            be_.download(*X_[kf][n], states_out + len_ * n);
        }
        rep->iterations_used = report_iters_;
        rep->converged = converged_ ? 1 : 0;
        rep->eta_count = static_cast<int32_t>(eta_tilde_.size());
        for (size_t k = 0; k < eta_tilde_.size(); ++k) {
            rep->eta_tilde[k] = eta_tilde_[k];
            if (rep->eta && ref_) rep->eta[k] = eta_[k];
        }
        if (trace) collect_trace(trace, rep);
    }

  private:
    struct Lane {
        std::mutex mu;
        std::condition_variable cv;
        std::deque<Task> serial, fine;
        bool closed = false;
    };

    // ---- lanes ---------------------------------------------------------------------------
    void lane_loop(int w) {
        Lane& lane = lanes_[w];
        for (;;) {
            Task t;
            {
                std::unique_lock<std::mutex> lk(lane.mu);
                lane.cv.wait(lk, [&] { return lane.closed || !lane.serial.empty() || !lane.fine.empty(); });
                if (lane.serial.empty() && lane.fine.empty()) return;
                std::deque<Task>& q = lane.serial.empty() ? lane.fine : lane.serial;
                t = std::move(q.front());
                q.pop_front();
            }
            Done d;
            if (!halt_) {
                try {
                    const double a = since(Clock::now());
                    d.result = be_.propagate(w, t.kind != kFine, t.t0, t.t1, *t.input);
                    const double b = since(Clock::now());
                    lane_events_[w].push_back(pswim_trace_event{w, static_cast<int32_t>(t.kind), a, b});
                } catch (...) {
                    d.error = std::current_exception();
                }
            }
            d.task = std::move(t);
            {
                std::lock_guard<std::mutex> lk(done_mu_);
                done_.push_back(std::move(d));
            }
            done_cv_.notify_one();
        }
    }

    Done next_done() {
        std::unique_lock<std::mutex> lk(done_mu_);
        done_cv_.wait(lk, [&] { return !done_.empty(); });
        Done d = std::move(done_.front());
        done_.pop_front();
        return d;
    }

    double since(Clock::time_point t) const { return std::chrono::duration<double>(t - origin_).count(); }

    int lane_of(const Task& t) const {
        if (t.kind != kFine) return 0;
        return M_ >= 2 ? 1 + (t.n - 1) % (M_ - 1) : 0;
    }

    void submit(Task t) {
        const int w = lane_of(t);
        ++outstanding_;
        {
            std::lock_guard<std::mutex> lk(lanes_[w].mu);
            (t.kind == kFine ? lanes_[w].fine : lanes_[w].serial).push_back(std::move(t));
        }
        wake_.push_back(w);
    }

    // Tasks created while handling one completion are queued together and the lanes woken
    // afterwards, so a waking lane sees this round's serial task before its fine task.
    void notify_pending() {
        for (int w : wake_) lanes_[w].cv.notify_one();
        wake_.clear();
    }

    // ---- driver --------------------------------------------------------------------------
    void on_done(const Done& d) {
        const Task& t = d.task;
        if (t.kind == kCoarse) {
            G_[0][t.n] = d.result;
            put_state(0, t.n, d.result);
            try_correct(1, t.n);
            if (t.n < N_ && !halt_)
                submit(Task{kCoarse, 0, t.n + 1, boundary_time(plan_, t.n), boundary_time(plan_, t.n + 1), X_[0][t.n]});
        } else if (t.kind == kFine) {
            F_[t.k][t.n] = d.result;
            --fines_left_[t.k];
            if (t.n == t.k)
                put_state(t.k, t.k, d.result);  // X_k^k = fine result
            else
                try_correct(t.k, t.n);
            if (plan_.mode == 0 && fines_left_[t.k] == 0) try_correct(t.k, t.k + 1);
        } else {
            G_[t.k][t.n] = d.result;
            put_state(t.k, t.n, be_.corrected(*F_[t.k][t.n], *d.result, *G_[t.k - 1][t.n]));
            try_correct(t.k + 1, t.n);
        }
    }

    void put_state(int k, int n, const StatePtr& v) {
        if (X_[k][n]) return;
        X_[k][n] = v;
        if (n >= 1 && --slots_left_[k] == 0) {
            iter_ready_[k] = 1;
            // reports come out in iteration order even when speculative pipelined work
            // finishes a later iteration first
            while (next_report_ <= L_ && iter_ready_[next_report_] && !halt_) finish_iteration(next_report_++);
            if (halt_) return;
        }
        if (n + 1 <= N_) try_correct(k, n + 1);
        if (k + 1 <= L_) {
            if (n <= k) put_state(k + 1, n, v);          // converged prefix is frozen
            if (plan_.mode == 1 && n >= k + 1) try_fine(k + 1, n);  // streaming hand-off
        }
    }

    void try_fine(int k, int n) {
        if (halt_ || k > L_ || n < k || n > N_ || fine_sent_[k][n] || !X_[k - 1][n - 1]) return;
        fine_sent_[k][n] = 1;
        submit(Task{kFine, k, n, boundary_time(plan_, n - 1), boundary_time(plan_, n), X_[k - 1][n - 1]});
    }

    void try_correct(int k, int n) {
        if (halt_ || k < 1 || k > L_ || n < k + 1 || n > N_ || corr_sent_[k][n]) return;
        if (!F_[k][n] || !X_[k][n - 1] || !G_[k - 1][n]) return;
        if (plan_.mode == 0 && fines_left_[k] > 0) return;
        corr_sent_[k][n] = 1;
        submit(Task{kCorrect, k, n, boundary_time(plan_, n - 1), boundary_time(plan_, n), X_[k][n - 1]});
    }

    void finish_iteration(int k) {
        if (k == 0) {
            if (plan_.mode == 0)
                for (int n = 1; n <= N_; ++n) try_fine(1, n);
            return;
        }
        double et = 0.0, e = 0.0;
        for (int n = 1; n <= N_; ++n) {
            et = std::max(et, be_.metric(*X_[k][n], *X_[k - 1][n]));
            if (ref_) e = std::max(e, be_.metric_ref(ref_ + len_ * n, *X_[k][n]));
        }
        eta_tilde_.push_back(et);
        if (ref_) eta_.push_back(e);
        report_iters_ = k;
        if (et < plan_.tolerance || k == N_) {
            converged_ = true;  // at k = n every interval is exact (parareal.cpp:383-386)
            halt_at(k);
        } else if (k == L_) {
            halt_at(k);
        } else if (plan_.mode == 0) {
            for (int n = k + 1; n <= N_; ++n) try_fine(k + 1, n);
        }
    }

    void halt_at(int k) {
        final_k_ = k;
        halt_ = true;
    }

    void collect_trace(std::vector<pswim_trace_event>* out, pswim_report* rep) {
        // ScheduleTrace::finalize_idle (schedule_trace.cpp:17-41): idle gaps on every lane but
        // the serial one, from t = 0 to each task start.
        std::vector<pswim_trace_event> ev;
        for (auto& l : lane_events_) ev.insert(ev.end(), l.begin(), l.end());
        auto order = [](const pswim_trace_event& a, const pswim_trace_event& b) {
            return a.worker != b.worker ? a.worker < b.worker : a.t_start < b.t_start;
        };
        std::stable_sort(ev.begin(), ev.end(), order);
        std::vector<pswim_trace_event> gaps;
        double cursor = 0.0, idle = 0.0;
        int cur = -1;
        for (const auto& e : ev) {
            if (e.worker != cur) {
                cur = e.worker;
                cursor = 0.0;
            }
            if (e.worker != 0 && e.t_start > cursor) {
                gaps.push_back(pswim_trace_event{e.worker, kIdle, cursor, e.t_start});
                idle += e.t_start - cursor;
            }
            cursor = std::max(cursor, e.t_end);
        }
        ev.insert(ev.end(), gaps.begin(), gaps.end());
        std::stable_sort(ev.begin(), ev.end(), order);
        *out = std::move(ev);
        rep->schedule_idle = idle;
    }

    const pswim_plan plan_;
    EngineBackend& be_;
    const double* ref_;
    const int64_t len_;
    const int N_, L_, M_;
    std::vector<std::vector<StatePtr>> X_, G_, F_;
    std::vector<std::vector<char>> fine_sent_, corr_sent_;
    std::vector<int> fines_left_, slots_left_;
    std::vector<char> iter_ready_;
    int next_report_ = 0;
    std::vector<Lane> lanes_;
    std::vector<std::vector<pswim_trace_event>> lane_events_;
    std::mutex done_mu_;
    std::condition_variable done_cv_;
    std::deque<Done> done_;
    std::vector<int> wake_;
    std::atomic<bool> halt_{false};
    std::exception_ptr failure_;
    int outstanding_ = 0;
    int final_k_ = 0;
    Clock::time_point origin_;
    std::vector<double> eta_tilde_, eta_;
    int report_iters_ = 0;
    bool converged_ = false;
};

int run_engine(const pswim_plan* plan, EngineBackend& be, const double* x0, int64_t len, const double* ref,
               double* states_out, pswim_report* rep, pswim_trace_event* trace_out, int64_t trace_cap,
               int64_t* trace_len) {
    const auto t0 = Clock::now();
    try {
        Engine eng(*plan, be, ref, len);
        std::vector<pswim_trace_event> trace;
        eng.run(x0, states_out, rep, &trace);
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
    rep->wall_seconds = std::chrono::duration<double>(Clock::now() - t0).count();
    return PSWIM_OK;
}

}  // namespace
}  // namespace pswim

// =========================================================================================
// Rank driver (one slice per rank)
// =========================================================================================
namespace pswim {
namespace {

// Asynchronous slice backend: three ordered queues (coarse/corrector, fine, comm) with
// events between them.  The host form executes everything synchronously.
class SliceBackend {
  public:
    virtual ~SliceBackend() = default;
    virtual int alloc(int count) = 0;  // buffers 0..count-1
    bool allocated() const { return allocated_; }

  protected:
    bool allocated_ = false;

  public:
    virtual double* buf(int i) = 0;
    virtual int upload(int i, const double* h) = 0;
    virtual int download(double* h, int i) = 0;
    virtual int coarse(int in, double t0, double t1, int out) = 0;  // coarse queue
    virtual int fine(int in, double t0, double t1, int out) = 0;    // fine queue
    virtual int correct(int xp, int gn, int go, int out) = 0;       // coarse queue
    virtual int copy(int src, int dst) = 0;                         // coarse queue
    virtual int metric(int x, int y, int slot) = 0;                 // coarse queue -> metric slot
    virtual int metric_ref(const double* h_ref, int x, int slot) = 0;
    virtual double* metric_slot(int slot) = 0;                      // pointer for the transport
    virtual int read_metric(int slot, double* out2) = 0;            // waits for comm queue
    virtual int set_metric(int slot, double a, double b) = 0;
    // cross-queue ordering: 0 coarse, 1 fine, 2 comm
    virtual int mark(int queue, int tag) = 0;
    virtual int wait(int queue, int tag) = 0;
    virtual void* stream(int queue) = 0;
    virtual int finish() = 0;
    virtual std::string error() = 0;
};

class HostSlice final : public SliceBackend {
  public:
    HostSlice(int64_t len, pswim_propagator_fn c, void* cu, pswim_propagator_fn f, void* fu, int dim, int stride)
        : len_(len), c_(c), cu_(cu), f_(f), fu_(fu), dim_(dim), stride_(stride) {}
    int alloc(int count) override {
        bufs_.assign(count, std::vector<double>(len_, 0.0));
        metric_.assign(2 * count, 0.0);
        allocated_ = true;
        return PSWIM_OK;
    }
    double* buf(int i) override { return bufs_[i].data(); }
    int upload(int i, const double* h) override {
        std::memcpy(bufs_[i].data(), h, len_ * sizeof(double));
        return PSWIM_OK;
    }
    int download(double* h, int i) override {
        std::memcpy(h, bufs_[i].data(), len_ * sizeof(double));
        return PSWIM_OK;
    }
    int coarse(int in, double t0, double t1, int out) override {
        return c_(cu_, t0, t1, bufs_[in].data(), bufs_[out].data(), len_, nullptr);
    }
    int fine(int in, double t0, double t1, int out) override {
        return f_(fu_, t0, t1, bufs_[in].data(), bufs_[out].data(), len_, nullptr);
    }
    int correct(int xp, int gn, int go, int out) override {
        for (int64_t i = 0; i < len_; ++i) bufs_[out][i] = bufs_[xp][i] + bufs_[gn][i] - bufs_[go][i];
        return PSWIM_OK;
    }
    int copy(int src, int dst) override {
        bufs_[dst] = bufs_[src];
        return PSWIM_OK;
    }
    int metric(int x, int y, int slot) override {
        metric_[2 * slot] = host_metric(bufs_[x].data(), bufs_[y].data(), len_, dim_, stride_);
        return PSWIM_OK;
    }
    int metric_ref(const double* h_ref, int x, int slot) override {
        metric_[2 * slot + 1] = host_metric(h_ref, bufs_[x].data(), len_, dim_, stride_);
        return PSWIM_OK;
    }
    double* metric_slot(int slot) override { return &metric_[2 * slot]; }
    int read_metric(int slot, double* out2) override {
        out2[0] = metric_[2 * slot];
        out2[1] = metric_[2 * slot + 1];
        return PSWIM_OK;
    }
    int set_metric(int slot, double a, double b) override {
        metric_[2 * slot] = a;
        metric_[2 * slot + 1] = b;
        return PSWIM_OK;
    }
    int mark(int, int) override { return PSWIM_OK; }
    int wait(int, int) override { return PSWIM_OK; }
    void* stream(int) override { return nullptr; }
    int finish() override { return PSWIM_OK; }
    std::string error() override { return "host propagator failed"; }

  private:
    int64_t len_;
    pswim_propagator_fn c_;
    void* cu_;
    pswim_propagator_fn f_;
    void* fu_;
    int dim_, stride_;
    std::vector<std::vector<double>> bufs_;
    std::vector<double> metric_;
};

class GpuSlice final : public SliceBackend {
  public:
    // space_coarse / space_fine: optional space-group transports (hybrid space x time): the
    // slice's coarse and fine propagations then shard their MRS over the group, one transport
    // per context so the two streams' all-gathers never interleave
    GpuSlice(const pswim_scenario& sc, int device, int64_t fine_steps, int64_t coarse_steps,
             const pswim_transport* space_coarse = nullptr, const pswim_transport* space_fine = nullptr)
        : device_(device), len_(12 * sc.rod_count * sc.nodes_per_rod), fine_steps_(fine_steps),
          coarse_steps_(coarse_steps), sp_c_(space_coarse), sp_f_(space_fine) {
        int lo = 0, hi = 0;
        cudaSetDevice(device);
        cudaDeviceGetStreamPriorityRange(&lo, &hi);
        cctx_ = pswim_create(device, &sc, hi);  // coarse + corrector: the critical wavefront
        fctx_ = pswim_create(device, &sc, lo);  // fine solves
        if (!cctx_ || !fctx_) throw CodeError(PSWIM_ECUDA, "rank: cannot create contexts");
        cudaStreamCreateWithPriority(&comm_, cudaStreamNonBlocking, hi);
    }
    ~GpuSlice() override {
        cudaSetDevice(device_);
        if (comm_) cudaStreamSynchronize(comm_);
        for (double* p : bufs_) cudaFree(p);
        if (d_metric_) cudaFree(d_metric_);
        if (h_metric_) cudaFreeHost(h_metric_);
        for (auto& e : events_) cudaEventDestroy(e);
        if (comm_) cudaStreamDestroy(comm_);
        pswim_destroy(cctx_);
        pswim_destroy(fctx_);
    }
    int alloc(int count) override {
        cudaSetDevice(device_);
        bufs_.assign(count, nullptr);
        events_needed_ = 8 * (count + 2);
        for (auto& p : bufs_)
            if (cudaMalloc(&p, len_ * sizeof(double)) != cudaSuccess) return fail("rank: cudaMalloc");
        if (cudaMalloc(&d_metric_, 2 * count * sizeof(double)) != cudaSuccess) return fail("rank: cudaMalloc metric");
        if (cudaMallocHost(&h_metric_, 2 * count * sizeof(double)) != cudaSuccess) return fail("rank: pinned");
        cudaMemset(d_metric_, 0, 2 * count * sizeof(double));
        events_.resize(events_needed_);
        for (auto& e : events_) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
        cudaDeviceSynchronize();
        allocated_ = true;
        return PSWIM_OK;
    }
    double* buf(int i) override { return bufs_[i]; }
    int upload(int i, const double* h) override {
        cudaSetDevice(device_);
        return cudaMemcpy(bufs_[i], h, len_ * sizeof(double), cudaMemcpyHostToDevice) == cudaSuccess ? PSWIM_OK
                                                                                                    : fail("upload");
    }
    int download(double* h, int i) override {
        cudaSetDevice(device_);
        return cudaMemcpy(h, bufs_[i], len_ * sizeof(double), cudaMemcpyDeviceToHost) == cudaSuccess ? PSWIM_OK
                                                                                                    : fail("download");
    }
    int coarse(int in, double t0, double t1, int out) override {
        const int rc = cctx_->propagate_async(bufs_[in], t0, t1, PSWIM_EULER, coarse_steps_, 0.0, bufs_[out], sp_c_);
        return rc ? fail(cctx_->err, rc) : PSWIM_OK;
    }
    int fine(int in, double t0, double t1, int out) override {
        const int rc = fctx_->propagate_async(bufs_[in], t0, t1, PSWIM_RK2, fine_steps_, 0.0, bufs_[out], sp_f_);
        return rc ? fail(fctx_->err, rc) : PSWIM_OK;
    }
    int correct(int xp, int gn, int go, int out) override {
        return correct_launch(bufs_[xp], bufs_[gn], bufs_[go], len_, bufs_[out], cctx_->stream) == cudaSuccess
                   ? PSWIM_OK
                   : fail("correct");
    }
    int copy(int src, int dst) override {
        return cudaMemcpyAsync(bufs_[dst], bufs_[src], len_ * sizeof(double), cudaMemcpyDeviceToDevice,
                               cctx_->stream) == cudaSuccess
                   ? PSWIM_OK
                   : fail("copy");
    }
    int metric(int x, int y, int slot) override {
        return metric_launch(bufs_[x], bufs_[y], len_, nullptr, nullptr, d_metric_ + 2 * slot, cctx_->stream) ==
                       cudaSuccess
                   ? PSWIM_OK
                   : fail("metric");
    }
    int metric_ref(const double* h_ref, int x, int slot) override {
        // true-error column: host reference slice, computed once per iteration
        std::vector<double> h(len_);
        cudaStreamSynchronize(cctx_->stream);
        if (download(h.data(), x)) return PSWIM_ECUDA;
        const double v = host_metric(h_ref, h.data(), len_, 3, 12);
        return cudaMemcpyAsync(d_metric_ + 2 * slot + 1, &v, sizeof(double), cudaMemcpyHostToDevice, cctx_->stream) ==
                       cudaSuccess && cudaStreamSynchronize(cctx_->stream) == cudaSuccess
                   ? PSWIM_OK
                   : fail("metric_ref");
    }
    double* metric_slot(int slot) override { return d_metric_ + 2 * slot; }
    int read_metric(int slot, double* out2) override {
        if (cudaMemcpyAsync(h_metric_ + 2 * slot, d_metric_ + 2 * slot, 2 * sizeof(double), cudaMemcpyDeviceToHost,
                            comm_) != cudaSuccess ||
            cudaStreamSynchronize(comm_) != cudaSuccess)
            return fail("read_metric");
        out2[0] = h_metric_[2 * slot];
        out2[1] = h_metric_[2 * slot + 1];
        return PSWIM_OK;
    }
    int set_metric(int slot, double a, double b) override {
        h_metric_[2 * slot] = a;
        h_metric_[2 * slot + 1] = b;
        return cudaMemcpyAsync(d_metric_ + 2 * slot, h_metric_ + 2 * slot, 2 * sizeof(double), cudaMemcpyHostToDevice,
                               cctx_->stream) == cudaSuccess
                   ? PSWIM_OK
                   : fail("set_metric");
    }
    cudaStream_t q(int queue) { return queue == 0 ? cctx_->stream : (queue == 1 ? fctx_->stream : comm_); }
    int mark(int queue, int tag) override {
        return cudaEventRecord(events_[tag], q(queue)) == cudaSuccess ? PSWIM_OK : fail("event record");
    }
    int wait(int queue, int tag) override {
        return cudaStreamWaitEvent(q(queue), events_[tag], 0) == cudaSuccess ? PSWIM_OK : fail("event wait");
    }
    void* stream(int queue) override { return q(queue); }
    int finish() override {
        cudaStreamSynchronize(comm_);
        int rc = cctx_->sync();
        if (rc) return fail(cctx_->err, rc);
        rc = fctx_->sync();
        if (rc) return fail(fctx_->err, rc);
        return PSWIM_OK;
    }
    std::string error() override { return err_; }

  private:
    int fail(const std::string& w, int code = PSWIM_ECUDA) {
        err_ = w;
        return code;
    }
    int device_;
    int64_t len_, fine_steps_, coarse_steps_;
    const pswim_transport* sp_c_ = nullptr;
    const pswim_transport* sp_f_ = nullptr;
    pswim_ctx* cctx_ = nullptr;
    pswim_ctx* fctx_ = nullptr;
    cudaStream_t comm_ = nullptr;
    std::vector<double*> bufs_;
    double* d_metric_ = nullptr;
    double* h_metric_ = nullptr;
    std::vector<cudaEvent_t> events_;
    int events_needed_ = 0;
    std::string err_;
};

// Buffers a slice rank needs (see rank_run).
inline int slice_buffer_count(const pswim_plan& plan, int rank) {
    const int K = std::min(plan.max_iterations, plan.intervals);
    const int Kn = std::min(rank + 1, K);
    return 4 * (Kn + 1);
}

// Event tags: per iteration k, tag = 8 k + kind.
enum { kTagIn = 0, kTagX = 1, kTagFine = 2, kTagMetric = 3 };
inline int tag(int k, int what) { return 8 * k + what; }

// The slice recurrence for rank p (interval n = p + 1), parareal.cpp:58-89:
//   X[0][n] = G(X[0][n-1]);  X[k][k] = F(X[k-1][k-1]);
//   X[k][n] = F(X[k-1][n-1]) + G(X[k][n-1]) - G(X[k-1][n-1])   (1 <= k < n)
//   X[k][n] = X[n][n]                                           (k > n, frozen)
// Rank p receives X[k][n-1] from p-1 for k = 0..min(n-1, K) and sends X[k][n] to p+1 for
// k = 0..min(n, K); every rank joins one allreduce(max) of [eta_tilde_k, eta_k] per
// iteration, and the stop rule of parareal.cpp:366-393 is evaluated identically on every
// rank from that reduced value.  Communication for iteration k+1 is only issued once the
// iteration-k decision is known, so no rank ever waits on a message that will not come.
int rank_run(const pswim_plan& plan, SliceBackend& be, const pswim_transport& tr, int64_t len, const double* x0,
             const double* ref_slice, double* out, pswim_report* rep) {
    const auto t_begin = Clock::now();
    const int p = tr.rank, m = tr.world;
    if (plan.intervals != m || p < 0 || p >= m) return PSWIM_EINVAL;
    const int n = p + 1;
    const int K = std::min(plan.max_iterations, plan.intervals);  // l = min(l_max, n)
    const int Kn = std::min(n, K);                               // last iteration with work here
    const bool pipelined = plan.mode == 1;
    const bool has_prev = p > 0, has_next = p + 1 < m;
    if (K + 1 > 500) return PSWIM_EINVAL;  // event tag space
    // buffers: IN+k = X[k][n-1]; XB+k = corrected X[k][n]; FB+k = F(X[k-1][n-1]); GB+k = G(X[k][n-1])
    const int IN = 0, XB = IN + (Kn + 1), FB = XB + (Kn + 1), GB = FB + (Kn + 1);
    if (!be.allocated()) {
        const int rc = be.alloc(GB + Kn + 1);
        if (rc) return rc;
    }
    void* cs = be.stream(2);
    const double t_lo = boundary_time(plan, n - 1), t_hi = boundary_time(plan, n);
    std::vector<int> xidx(Kn + 1, -1);

#define RK(call)                  \
    do {                          \
        const int rc_ = (call);   \
        if (rc_) return rc_;      \
    } while (0)
#define RT(call)                                        \
    do {                                                \
        if ((call) != 0) return PSWIM_ECOMM;            \
    } while (0)

    auto launch_fine = [&](int k) -> int {
        // F(X[k][n-1]) for iteration k+1, on the fine queue, after the input arrived and after
        // this rank's own coarse / corrector on the same input produced X[k][n]: the coarse
        // chain through the ranks is the sequential critical path, and sharing the GPU with
        // its own fine solve slows each link (measured 4.65 -> 6.10 ms per coarse interval at
        // 64 x 256, tools/probe_contention.py), while F only starts T_G later.
        if (k + 1 > Kn) return PSWIM_OK;
        if (has_prev) RK(be.wait(1, tag(k, kTagIn)));
        RK(be.wait(1, tag(k, kTagX)));
        RK(be.fine(IN + k, t_lo, t_hi, FB + k + 1));
        return be.mark(1, tag(k + 1, kTagFine));
    };

    // ---- iteration 0: coarse sweep ----
    if (has_prev) {
        RT(tr.recv(tr.user, be.buf(IN), len, p - 1, cs));
        RK(be.mark(2, tag(0, kTagIn)));
        RK(be.wait(0, tag(0, kTagIn)));
    } else {
        RK(be.upload(IN, x0));
    }
    RK(be.coarse(IN, t_lo, t_hi, GB));
    xidx[0] = GB;  // X[0][n] = G(X[0][n-1])
    RK(be.mark(0, tag(0, kTagX)));
    if (has_next) {
        RK(be.wait(2, tag(0, kTagX)));
        RT(tr.send(tr.user, be.buf(xidx[0]), len, p + 1, cs));
    }
    if (pipelined) {
        RK(launch_fine(0));
    } else {
        // regular: iteration-0 barrier before the first fine phase (parareal.cpp:367-371)
        RK(be.set_metric(0, 0.0, 0.0));
        RK(be.mark(0, tag(0, kTagMetric)));
        RK(be.wait(2, tag(0, kTagMetric)));
        RT(tr.allreduce_max(tr.user, be.metric_slot(0), 2, cs));
        double v[2];
        RK(be.read_metric(0, v));
        RK(launch_fine(0));
    }

    int k_final = 0;
    bool converged = false;
    std::vector<double> eta_tilde, eta;
    for (int k = 1; k <= K; ++k) {
        if (k <= Kn) {
            if (k < n) {
                RT(tr.recv(tr.user, be.buf(IN + k), len, p - 1, cs));
                RK(be.mark(2, tag(k, kTagIn)));
                RK(be.wait(0, tag(k, kTagIn)));
                RK(be.coarse(IN + k, t_lo, t_hi, GB + k));
                RK(be.wait(0, tag(k, kTagFine)));
                RK(be.correct(FB + k, GB + k, GB + k - 1, XB + k));
                xidx[k] = XB + k;
            } else {  // k == n: the interval is exact from here on
                RK(be.wait(0, tag(k, kTagFine)));
                xidx[k] = FB + k;
            }
            RK(be.mark(0, tag(k, kTagX)));
            if (has_next) {
                RK(be.wait(2, tag(k, kTagX)));
                RT(tr.send(tr.user, be.buf(xidx[k]), len, p + 1, cs));
            }
            if (pipelined && k < n) RK(launch_fine(k));
            RK(be.metric(xidx[k], xidx[k - 1], k));
            if (ref_slice) RK(be.metric_ref(ref_slice, xidx[k], k));
        } else {
            // frozen: contributes 0 to eta_tilde and its unchanged true error
            RK(be.set_metric(k, 0.0, 0.0));
            if (ref_slice) RK(be.metric_ref(ref_slice, xidx[Kn], k));
        }
        RK(be.mark(0, tag(k, kTagMetric)));
        RK(be.wait(2, tag(k, kTagMetric)));
        RT(tr.allreduce_max(tr.user, be.metric_slot(k), 2, cs));
        double v[2];
        RK(be.read_metric(k, v));
        eta_tilde.push_back(v[0]);
        eta.push_back(v[1]);
        k_final = k;
        if (v[0] < plan.tolerance || k == plan.intervals) {
            converged = true;
            break;
        }
        if (k == K) break;
        if (!pipelined && k < n) RK(launch_fine(k));
    }
    RK(be.finish());
    RK(be.download(out, xidx[std::min(k_final, Kn)]));
#undef RK
#undef RT
    rep->iterations_used = k_final;
    rep->converged = converged ? 1 : 0;
    rep->eta_count = static_cast<int32_t>(eta_tilde.size());
    for (size_t k = 0; k < eta_tilde.size(); ++k) {
        if (rep->eta_tilde) rep->eta_tilde[k] = eta_tilde[k];
        if (rep->eta && ref_slice) rep->eta[k] = eta[k];
    }
    rep->wall_seconds = std::chrono::duration<double>(Clock::now() - t_begin).count();
    rep->schedule_idle = 0.0;
    return PSWIM_OK;
}

// ---------------------------------------------------------------------------------------
// In-process transport: slice ranks as threads, one context pair per rank (any devices).
// send = peer copy into a per-message staging buffer on the receiver's device + event;
// recv = stream wait on that event + local copy; allreduce = host barrier on 2 doubles.
// ---------------------------------------------------------------------------------------
class ThreadHub {
  public:
    ThreadHub(int world, const int* devices, int64_t len, int slots)
        : world_(world), len_(len), devices_(devices, devices + world), links_(world) {
        for (int p = 0; p + 1 < world; ++p) {
            cudaSetDevice(devices_[p + 1]);
            links_[p].staging.resize(slots, nullptr);
            for (auto& b : links_[p].staging) cudaMalloc(&b, len * sizeof(double));
            links_[p].events.resize(slots);
            for (auto& e : links_[p].events) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
        }
        for (int a = 0; a < world; ++a)
            for (int b = 0; b < world; ++b)
                if (a != b && devices_[a] != devices_[b]) {
                    int ok = 0;
                    cudaDeviceCanAccessPeer(&ok, devices_[a], devices_[b]);
                    if (ok) {
                        cudaSetDevice(devices_[a]);
                        cudaDeviceEnablePeerAccess(devices_[b], 0);
                        cudaGetLastError();
                    }
                }
    }
    ~ThreadHub() {
        for (int p = 0; p + 1 < world_; ++p) {
            cudaSetDevice(devices_[p + 1]);
            for (auto b : links_[p].staging) cudaFree(b);
            for (auto e : links_[p].events) cudaEventDestroy(e);
        }
    }
    struct Link {
        std::vector<double*> staging;
        std::vector<cudaEvent_t> events;
        std::deque<int> ready;  // slot indices posted by the sender
        int next_send = 0;
    };
    int send(int from, const double* buf, int64_t len, int to, cudaStream_t st) {
        if (to != from + 1) return PSWIM_ECOMM;
        Link& l = links_[from];
        int slot;
        {
            std::lock_guard<std::mutex> lk(mu_);
            slot = l.next_send++;
        }
        if (slot >= (int)l.staging.size()) return PSWIM_ECOMM;
        cudaSetDevice(devices_[from]);
        if (cudaMemcpyPeerAsync(l.staging[slot], devices_[to], buf, devices_[from], len * sizeof(double), st) !=
                cudaSuccess ||
            cudaEventRecord(l.events[slot], st) != cudaSuccess)
            return PSWIM_ECOMM;
        {
            std::lock_guard<std::mutex> lk(mu_);
            l.ready.push_back(slot);
        }
        cv_.notify_all();
        return PSWIM_OK;
    }
    int recv(int at, double* buf, int64_t len, int from, cudaStream_t st) {
        if (from != at - 1) return PSWIM_ECOMM;
        Link& l = links_[from];
        int slot;
        {
            std::unique_lock<std::mutex> lk(mu_);
            cv_.wait(lk, [&] { return !l.ready.empty() || aborted_; });
            if (aborted_) return PSWIM_ECOMM;
            slot = l.ready.front();
            l.ready.pop_front();
        }
        cudaSetDevice(devices_[at]);
        if (cudaStreamWaitEvent(st, l.events[slot], 0) != cudaSuccess ||
            cudaMemcpyAsync(buf, l.staging[slot], len * sizeof(double), cudaMemcpyDeviceToDevice, st) != cudaSuccess)
            return PSWIM_ECOMM;
        return PSWIM_OK;
    }
    int allreduce_max(int rank, double* dbuf, int64_t len, cudaStream_t st) {
        std::vector<double> h(len);
        cudaSetDevice(devices_[rank]);
        if (cudaMemcpyAsync(h.data(), dbuf, len * sizeof(double), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
            cudaStreamSynchronize(st) != cudaSuccess)
            return PSWIM_ECOMM;
        {
            std::unique_lock<std::mutex> lk(mu_);
            const long gen = gen_;
            if (arrived_ == 0) acc_.assign(len, -INFINITY);
            for (int64_t i = 0; i < len; ++i) acc_[i] = std::max(acc_[i], h[i]);
            if (++arrived_ == world_) {
                result_ = acc_;
                arrived_ = 0;
                ++gen_;
                cv_.notify_all();
            } else {
                cv_.wait(lk, [&] { return gen_ != gen || aborted_; });
                if (aborted_) return PSWIM_ECOMM;
            }
            h = result_;
        }
        if (cudaMemcpyAsync(dbuf, h.data(), len * sizeof(double), cudaMemcpyHostToDevice, st) != cudaSuccess ||
            cudaStreamSynchronize(st) != cudaSuccess)
            return PSWIM_ECOMM;
        return PSWIM_OK;
    }
    // Host barrier over the world (generation counted).
    bool barrier() {
        std::unique_lock<std::mutex> lk(mu_);
        const long gen = bgen_;
        if (++barrived_ == world_) {
            barrived_ = 0;
            ++bgen_;
            cv_.notify_all();
            return !aborted_;
        }
        cv_.wait(lk, [&] { return bgen_ != gen || aborted_; });
        return !aborted_;
    }
    // recv[r * count ..] = send of rank r: stream-ordered peer copies; a second exchange of
    // "copied" events keeps every rank's send buffer alive until all peers have read it.
    int allgather(int rank, const double* send, double* recv, int64_t count, cudaStream_t st) {
        cudaSetDevice(devices_[rank]);
        {
            std::lock_guard<std::mutex> lk(mu_);
            if (ag_send_.empty()) {
                ag_send_.assign(world_, nullptr);
                ag_ready_.assign(world_, nullptr);
                ag_done_.assign(world_, nullptr);
            }
            if (!ag_ready_[rank]) {
                cudaEventCreateWithFlags(&ag_ready_[rank], cudaEventDisableTiming);
                cudaEventCreateWithFlags(&ag_done_[rank], cudaEventDisableTiming);
            }
            ag_send_[rank] = send;
        }
        if (cudaEventRecord(ag_ready_[rank], st) != cudaSuccess) return PSWIM_ECOMM;
        if (!barrier()) return PSWIM_ECOMM;
        const size_t bytes = (size_t)count * sizeof(double);
        for (int r = 0; r < world_; ++r) {
            cudaError_t e;
            if (r == rank) {
                e = cudaMemcpyAsync(recv + r * count, send, bytes, cudaMemcpyDeviceToDevice, st);
            } else {
                e = cudaStreamWaitEvent(st, ag_ready_[r], 0);
                if (e == cudaSuccess)
                    e = cudaMemcpyPeerAsync(recv + r * count, devices_[rank], ag_send_[r], devices_[r], bytes, st);
            }
            if (e != cudaSuccess) return PSWIM_ECOMM;
        }
        if (cudaEventRecord(ag_done_[rank], st) != cudaSuccess) return PSWIM_ECOMM;
        if (!barrier()) return PSWIM_ECOMM;
        for (int r = 0; r < world_; ++r)
            if (r != rank && cudaStreamWaitEvent(st, ag_done_[r], 0) != cudaSuccess) return PSWIM_ECOMM;
        if (!barrier()) return PSWIM_ECOMM;  // events may be re-recorded only after all waits are queued
        return PSWIM_OK;
    }
    void abort() {
        std::lock_guard<std::mutex> lk(mu_);
        aborted_ = true;
        cv_.notify_all();
    }

  private:
    int world_;
    int64_t len_;
    std::vector<int> devices_;
    std::vector<Link> links_;
    std::mutex mu_;
    std::condition_variable cv_;
    int arrived_ = 0;
    long gen_ = 0;
    std::vector<double> acc_, result_;
    bool aborted_ = false;
    int barrived_ = 0;
    long bgen_ = 0;
    std::vector<const double*> ag_send_;
    std::vector<cudaEvent_t> ag_ready_, ag_done_;
};

struct HubUser {
    ThreadHub* hub;
    int rank;
};
int hub_send(void* u, const double* b, int64_t len, int32_t peer, void* st) {
    auto* h = static_cast<HubUser*>(u);
    return h->hub->send(h->rank, b, len, peer, static_cast<cudaStream_t>(st));
}
int hub_recv(void* u, double* b, int64_t len, int32_t peer, void* st) {
    auto* h = static_cast<HubUser*>(u);
    return h->hub->recv(h->rank, b, len, peer, static_cast<cudaStream_t>(st));
}
int hub_allreduce(void* u, double* b, int64_t len, void* st) {
    auto* h = static_cast<HubUser*>(u);
    return h->hub->allreduce_max(h->rank, b, len, static_cast<cudaStream_t>(st));
}
int hub_allgather(void* u, const double* s, double* r, int64_t count, void* st) {
    auto* h = static_cast<HubUser*>(u);
    return h->hub->allgather(h->rank, s, r, count, static_cast<cudaStream_t>(st));
}

// Standalone in-process transports (pswim_threads_transports_create).
struct HubBundle {
    ThreadHub hub;
    std::vector<HubUser> users;
    std::vector<pswim_transport> trs;
    HubBundle(int world, const int* devices, int64_t len, int slots) : hub(world, devices, len, slots) {}
};

}  // namespace
}  // namespace pswim

// =========================================================================================
// C ABI
// =========================================================================================
extern "C" {

int pswim_parareal_run_host(const pswim_plan* plan, pswim_propagator_fn coarse, void* cu, pswim_propagator_fn fine,
                            void* fu, const double* x0, int64_t len, int32_t dim, int32_t stride,
                            const double* reference, double* states_out, pswim_report* rep,
                            pswim_trace_event* trace_out, int64_t trace_cap, int64_t* trace_len) {
    using namespace pswim;
    if (plan_check(plan) || !coarse || !fine || !x0 || !states_out || !rep || len <= 0) return PSWIM_EINVAL;
    if (dim < 1 || stride < dim || len % stride != 0) return PSWIM_EINVAL;
    HostBackend be(len, coarse, cu, fine, fu, dim, stride);
    return run_engine(plan, be, x0, len, reference, states_out, rep, trace_out, trace_cap, trace_len);
}

int pswim_parareal_run_gpu(const pswim_plan* plan, const pswim_scenario* sc, int device, int64_t fine_steps,
                           int64_t coarse_steps, const double* x0, const double* reference, double* states_out,
                           pswim_report* rep, pswim_trace_event* trace_out, int64_t trace_cap, int64_t* trace_len) {
    using namespace pswim;
    if (plan_check(plan) || !sc || !x0 || !states_out || !rep || fine_steps < 1 || coarse_steps < 1)
        return PSWIM_EINVAL;
    try {
        const int L = std::min(plan->max_iterations, plan->intervals);
        // X, G, F slots of the task graph (+1 input); bounded so huge states do not exhaust HBM
        const int64_t want = 3LL * (L + 1) * (plan->intervals + 1) + 1;
        const int64_t cap = (int64_t)((8ULL << 30) / (sizeof(double) * 12ULL * sc->rod_count * sc->nodes_per_rod));
        GpuBackend be(*sc, device, plan->workers, fine_steps, coarse_steps, (int)std::min<int64_t>(want, cap));
        return run_engine(plan, be, x0, 12 * sc->rod_count * sc->nodes_per_rod, reference, states_out, rep, trace_out,
                          trace_cap, trace_len);
    } catch (const CodeError& e) {
        return e.code;
    }
}

int pswim_parareal_rank_gpu(const pswim_plan* plan, const pswim_scenario* sc, int device, const pswim_transport* tr,
                            int64_t fine_steps, int64_t coarse_steps, const double* x0, const double* ref_slice,
                            double* state_out, pswim_report* rep) {
    using namespace pswim;
    if (plan_check(plan) || !sc || !tr || !x0 || !state_out || !rep || fine_steps < 1 || coarse_steps < 1)
        return PSWIM_EINVAL;
    try {
        GpuSlice be(*sc, device, fine_steps, coarse_steps);
        return rank_run(*plan, be, *tr, 12 * sc->rod_count * sc->nodes_per_rod, x0, ref_slice, state_out, rep);
    } catch (const CodeError& e) {
        return e.code;
    }
}

int pswim_parareal_rank_gpu_hybrid(const pswim_plan* plan, const pswim_scenario* sc, int device,
                                   const pswim_transport* time_tr, const pswim_transport* space_coarse,
                                   const pswim_transport* space_fine, int64_t fine_steps, int64_t coarse_steps,
                                   const double* x0, const double* ref_slice, double* state_out, pswim_report* rep) {
    using namespace pswim;
    if (plan_check(plan) || !sc || !time_tr || !space_coarse || !space_fine || !x0 || !state_out || !rep ||
        fine_steps < 1 || coarse_steps < 1)
        return PSWIM_EINVAL;
    if (space_coarse->world != space_fine->world || space_coarse->rank != space_fine->rank || !space_coarse->allgather ||
        !space_fine->allgather)
        return PSWIM_EINVAL;
    try {
        GpuSlice be(*sc, device, fine_steps, coarse_steps, space_coarse, space_fine);
        return rank_run(*plan, be, *time_tr, 12 * sc->rod_count * sc->nodes_per_rod, x0, ref_slice, state_out, rep);
    } catch (const CodeError& e) {
        return e.code;
    }
}

int pswim_parareal_rank_host(const pswim_plan* plan, pswim_propagator_fn coarse, void* cu, pswim_propagator_fn fine,
                             void* fu, const pswim_transport* tr, const double* x0, int64_t len, int32_t dim,
                             int32_t stride, const double* ref_slice, double* state_out, pswim_report* rep) {
    using namespace pswim;
    if (plan_check(plan) || !coarse || !fine || !tr || !x0 || !state_out || !rep || len <= 0) return PSWIM_EINVAL;
    if (dim < 1 || stride < dim || len % stride != 0) return PSWIM_EINVAL;
    HostSlice be(len, coarse, cu, fine, fu, dim, stride);
    return rank_run(*plan, be, *tr, len, x0, ref_slice, state_out, rep);
}

pswim_transport* pswim_threads_transports_create(int32_t world, const int* devices, int64_t len, int32_t slots) {
    using namespace pswim;
    if (world < 1 || !devices) return nullptr;
    try {
        auto* b = new HubBundle(world, devices, len > 0 ? len : 1, slots > 0 ? slots : 1);
        b->users.resize(world);
        b->trs.resize(world + 1);
        for (int p = 0; p < world; ++p) {
            b->users[p] = HubUser{&b->hub, p};
            b->trs[p] = pswim_transport{&b->users[p], p, world, hub_send, hub_recv, hub_allreduce, hub_allgather};
        }
        // trailing sentinel remembers the bundle for destroy
        b->trs[world] = pswim_transport{b, -1, world, nullptr, nullptr, nullptr, nullptr};
        return b->trs.data();
    } catch (...) {
        return nullptr;
    }
}

void pswim_threads_transports_destroy(pswim_transport* trs) {
    if (!trs) return;
    const int world = trs[0].world;
    delete static_cast<pswim::HubBundle*>(trs[world].user);
}

int pswim_parareal_run_threads(const pswim_plan* plan, const pswim_scenario* sc, const int* devices,
                               int64_t fine_steps, int64_t coarse_steps, const double* x0, const double* reference,
                               double* states_out, pswim_report* rep) {
    using namespace pswim;
    if (plan_check(plan) || !sc || !devices || !x0 || !states_out || !rep || fine_steps < 1 || coarse_steps < 1)
        return PSWIM_EINVAL;
    const int world = plan->intervals;
    const int64_t len = 12 * sc->rod_count * sc->nodes_per_rod;
    const int K = std::min(plan->max_iterations, plan->intervals);
    const auto t0 = Clock::now();
    try {
        ThreadHub hub(world, devices, len, K + 2);
        std::vector<HubUser> users(world);
        std::vector<pswim_transport> trs(world);
        std::vector<std::vector<double>> et(world, std::vector<double>(K + 1)), ea(world, std::vector<double>(K + 1));
        std::vector<pswim_report> reps(world);
        std::vector<int> rcs(world, PSWIM_OK);
        std::vector<std::thread> threads;
        std::mutex start_mu;
        std::condition_variable start_cv;
        int ready = 0;
        Clock::time_point t_start = Clock::now();
        for (int p = 0; p < world; ++p) {
            users[p] = HubUser{&hub, p};
            trs[p] = pswim_transport{&users[p], p, world, hub_send, hub_recv, hub_allreduce, hub_allgather};
            reps[p] = *rep;
            reps[p].eta_tilde = et[p].data();
            reps[p].eta = ea[p].data();
            threads.emplace_back([&, p] {
                try {
                    GpuSlice be(*sc, devices[p], fine_steps, coarse_steps);
                    rcs[p] = be.alloc(slice_buffer_count(*plan, p));
                    // every rank set up (contexts, HBM buffers) before the clock starts
                    {
                        std::unique_lock<std::mutex> lk(start_mu);
                        if (++ready == world) {
                            t_start = Clock::now();
                            start_cv.notify_all();
                        } else {
                            start_cv.wait(lk, [&] { return ready == world; });
                        }
                    }
                    if (!rcs[p])
                        rcs[p] = rank_run(*plan, be, trs[p], len, x0, reference ? reference + len * (p + 1) : nullptr,
                                          states_out + len * (p + 1), &reps[p]);
                } catch (const CodeError& e) {
                    rcs[p] = e.code;
                } catch (...) {
                    rcs[p] = PSWIM_ESTATE;
                }
                if (rcs[p]) hub.abort();
            });
        }
        for (auto& t : threads) t.join();
        for (int p = 0; p < world; ++p)
            if (rcs[p]) return rcs[p];
        std::memcpy(states_out, x0, len * sizeof(double));
        rep->iterations_used = reps[0].iterations_used;
        rep->converged = reps[0].converged;
        rep->eta_count = reps[0].eta_count;
        for (int k = 0; k < reps[0].eta_count; ++k) {
            if (rep->eta_tilde) rep->eta_tilde[k] = et[0][k];
            if (rep->eta && reference) rep->eta[k] = ea[0][k];
        }
        rep->wall_seconds = std::chrono::duration<double>(Clock::now() - t_start).count();
    } catch (const CodeError& e) {
        return e.code;
    }
    (void)t0;
    rep->schedule_idle = 0.0;
    return PSWIM_OK;
}

}  // extern "C"
