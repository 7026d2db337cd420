// parareal.cpp — the time-sliced Parareal driver: one time slice per rank (rank p owns
// interval p+1, intervals == world), the recurrence of src/parareal.cpp:58-89 with one state
// hand-off per iteration to rank p+1 and one allreduce(max) of the iteration metric.
// Coarse/corrector on a high-priority stream, fine on a low-priority stream, transport on a
// third.  Transports: NCCL (one process per GPU, nccl_transport.cpp), in-process threads +
// peer copies (pswim_parareal_run_threads), host callbacks (CPU tests over gloo).
// The single-device engine (parareal::run itself) is engine.cpp.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <atomic>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
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
#include "parareal_common.h"

// =========================================================================================
// Rank driver (one slice per rank)
// =========================================================================================
namespace pswim {
namespace {

// Slice backend: three stream-ordered queues -- 0 coarse/corrector (high priority), 1 fine
// (low priority), 2 communication -- with marks (events) between them.  The host form runs
// every call synchronously in issue order.
class SliceBackend {
  public:
    virtual ~SliceBackend() = default;
    // buffers 0..count-1; metric slots 0..iterations+1 (the last is the start barrier);
    // marks sized from the iteration count
    virtual int alloc(int count, int iterations) = 0;
    bool allocated() const { return allocated_; }
    virtual double* buf(int i) = 0;
    virtual int upload(int i, const double* h) = 0;
    virtual int download(double* h, int i) = 0;
    virtual int coarse(int in, double t0, double t1, int out) = 0;  // queue 0
    virtual int fine(int in, double t0, double t1, int out) = 0;    // queue 1
    virtual int correct(int xp, int gn, int go, int out) = 0;       // queue 0
    virtual int metric(int x, int y, int slot, int col) = 0;        // queue 0: slot[col] = metric(x, y)
    virtual int zero_metric(int slot) = 0;                          // queue 0
    virtual double* metric_slot(int slot) = 0;                      // 2 doubles, for the transport
    virtual int publish_metric(int slot) = 0;                       // queue 2: slot -> host, behind a marker
    virtual int read_metric(int slot, double* out2) = 0;            // host: waits for publish(slot)
    virtual int mark(int queue, int tag) = 0;
    virtual int wait(int queue, int tag) = 0;
    virtual void* stream(int queue) = 0;
    virtual int task_begin(int queue, int kind, int k) = 0;  // schedule trace (iteration k)
    virtual int task_end(int queue) = 0;
    virtual int origin() = 0;  // time origin, queue 2 (after the start barrier)
    virtual int finish() = 0;  // drain every queue
    // this rank's trace as (kind, k, t_start, t_end) relative to the origin
    virtual int local_trace(std::vector<double>* flat) = 0;
    // all ranks: recv[r * count ..] = send of rank r (host buffers in and out)
    virtual int gather(const double* send, double* recv, int64_t count) = 0;
    // peer-memory hand-off (handoff.cu); the host form has none
    virtual int handoff_recv(pswim_handoff*, int, unsigned long long, int) { return PSWIM_EINVAL; }
    virtual int handoff_push(pswim_handoff*, int, unsigned long long, int) { return PSWIM_EINVAL; }
    virtual int handoff_correct_push(pswim_handoff*, int, unsigned long long, int, int, int, int) {
        return PSWIM_EINVAL;
    }
    // device-side waits ahead (peer hand-off): nothing on the issue path may take the
    // driver's context lock for long (graph capture, recapture)
    virtual void prepare_device_waits() {}
    virtual std::string error() = 0;

  protected:
    bool allocated_ = false;
};

class HostSlice final : public SliceBackend {
  public:
    HostSlice(int64_t len, pswim_propagator_fn c, void* cu, pswim_propagator_fn f, void* fu, int dim, int stride,
              const pswim_transport& tr)
        : len_(len), c_(c), cu_(cu), f_(f), fu_(fu), dim_(dim), stride_(stride), tr_(tr) {}
    int alloc(int count, int iterations) override {
        bufs_.assign(count, std::vector<double>(len_, 0.0));
        metric_.assign(2 * (iterations + 2), 0.0);
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
        for (int64_t i = 0; i < len_; ++i) bufs_[out][i] = (bufs_[xp][i] + bufs_[gn][i]) - bufs_[go][i];
        return PSWIM_OK;
    }
    int metric(int x, int y, int slot, int col) override {
        metric_[2 * slot + col] = host_metric(bufs_[x].data(), bufs_[y].data(), len_, dim_, stride_);
        return PSWIM_OK;
    }
    int zero_metric(int slot) override {
        metric_[2 * slot] = metric_[2 * slot + 1] = 0.0;
        return PSWIM_OK;
    }
    double* metric_slot(int slot) override { return &metric_[2 * slot]; }
    int publish_metric(int) override { return PSWIM_OK; }
    int read_metric(int slot, double* out2) override {
        out2[0] = metric_[2 * slot];
        out2[1] = metric_[2 * slot + 1];
        return PSWIM_OK;
    }
    int mark(int, int) override { return PSWIM_OK; }
    int wait(int, int) override { return PSWIM_OK; }
    void* stream(int) override { return nullptr; }
    int task_begin(int queue, int kind, int k) override {
        open_[queue] = static_cast<int>(tasks_.size());
        tasks_.push_back({double(kind), double(k), now(), 0.0});
        return PSWIM_OK;
    }
    int task_end(int queue) override {
        tasks_[open_[queue]][3] = now();
        return PSWIM_OK;
    }
    int origin() override {
        origin_ = Clock::now();
        return PSWIM_OK;
    }
    int finish() override { return PSWIM_OK; }
    int local_trace(std::vector<double>* flat) override {
        flat->clear();
        for (const auto& t : tasks_) flat->insert(flat->end(), t.begin(), t.end());
        return PSWIM_OK;
    }
    int gather(const double* send, double* recv, int64_t count) override {
        return tr_.allgather(tr_.user, send, recv, count, nullptr) ? PSWIM_ECOMM : PSWIM_OK;
    }
    std::string error() override { return "host propagator failed"; }

  private:
    double now() const { return std::chrono::duration<double>(Clock::now() - origin_).count(); }
    int64_t len_;
    pswim_propagator_fn c_;
    void* cu_;
    pswim_propagator_fn f_;
    void* fu_;
    int dim_, stride_;
    const pswim_transport& tr_;
    std::vector<std::vector<double>> bufs_;
    std::vector<double> metric_;
    std::vector<std::array<double, 4>> tasks_;
    int open_[3] = {0, 0, 0};
    Clock::time_point origin_ = Clock::now();
};

// Seconds a rank waits on the device / transport before it aborts (PSWIM_COMM_TIMEOUT_S).
double comm_timeout() {
    if (const char* e = std::getenv("PSWIM_COMM_TIMEOUT_S")) return std::max(1.0, std::atof(e));
    return 900.0;
}

class GpuSlice final : public SliceBackend {
  public:
    // space_coarse / space_fine: optional space-group transports (hybrid space x time): the
    // slice's coarse and fine propagations then shard their MRS over the group, one transport
    // per context so the two streams' all-gathers never interleave
    GpuSlice(const pswim_scenario& sc, int device, int64_t fine_steps, int64_t coarse_steps,
             const pswim_transport* tr, const pswim_transport* space_coarse = nullptr,
             const pswim_transport* space_fine = nullptr)
        : device_(device), len_(12 * sc.rod_count * sc.nodes_per_rod), fine_steps_(fine_steps),
          coarse_steps_(coarse_steps), tr_(tr), sp_c_(space_coarse), sp_f_(space_fine), timeout_(comm_timeout()) {
        int lo = 0, hi = 0;
        cudaSetDevice(device);
        cudaDeviceGetStreamPriorityRange(&lo, &hi);
        hi_ = hi;
        lo_ = lo;
        cctx_ = pooled_ctx(device, sc, hi);  // coarse + corrector: the critical wavefront
        fctx_ = pooled_ctx(device, sc, lo);  // fine solves
        if (!cctx_ || !fctx_) throw CodeError(PSWIM_ECUDA, "rank: cannot create contexts");
        cudaStreamCreateWithPriority(&comm_, cudaStreamNonBlocking, hi);
    }
    ~GpuSlice() override {
        cudaSetDevice(device_);
        for (cudaStream_t s : {comm_, cctx_ ? cctx_->stream : nullptr, fctx_ ? fctx_->stream : nullptr})
            if (s) cudaStreamSynchronize(s);
        for (double* p : owned_) cudaFree(p);
        if (d_metric_) cudaFree(d_metric_);
        if (h_metric_) cudaFreeHost(h_metric_);
        for (auto& e : events_) cudaEventDestroy(e);
        for (auto& e : published_) cudaEventDestroy(e);
        for (auto& t : tasks_) {
            if (t.a) cudaEventDestroy(t.a);
            if (t.b) cudaEventDestroy(t.b);
        }
        for (auto& e : finish_)
            if (e) cudaEventDestroy(e);
        if (d_gather_) cudaFree(d_gather_);
        if (origin_) cudaEventDestroy(origin_);
        if (comm_) cudaStreamDestroy(comm_);
        if (cctx_) {
            pswim_set_graphs(cctx_, 1);  // back to the defaults before it returns to the pool
            release_ctx(cctx_, hi_);
        }
        if (fctx_) {
            pswim_set_graphs(fctx_, 1);
            release_ctx(fctx_, lo_);
        }
    }
    int alloc(int count, int iterations) override {
        cudaSetDevice(device_);
        owned_.assign(count, nullptr);
        for (auto& p : owned_)
            if (cudaMalloc(&p, len_ * sizeof(double)) != cudaSuccess) return fail("rank: cudaMalloc");
        bufs_ = owned_;
        const int slots = iterations + 2;
        if (cudaMalloc(&d_metric_, 2 * slots * sizeof(double)) != cudaSuccess) return fail("rank: cudaMalloc metric");
        if (cudaMallocHost(&h_metric_, 2 * slots * sizeof(double)) != cudaSuccess) return fail("rank: pinned");
        cudaMemset(d_metric_, 0, 2 * slots * sizeof(double));
        // tags 8 k + what for k = 0..iterations+1 (sized from the iteration count,
        // not from this rank's buffer count -- frozen ranks still mark every iteration)
        events_.resize(8 * (iterations + 2));
        for (auto& e : events_) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
        published_.resize(slots);
        for (auto& e : published_) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
        cudaEventCreate(&origin_);
        // Everything the issue loop needs exists before the start barrier: with the peer-memory
        // hand-off a rank's stream spins on the device for a peer's store, and a driver call
        // that takes the context lock (event creation, allocation) while another thread of
        // this process still has to enqueue that store would deadlock (seen with cuEventCreate).
        tasks_.resize(2 * iterations + 4);
        for (auto& t : tasks_)
            if (cudaEventCreate(&t.a) != cudaSuccess || cudaEventCreate(&t.b) != cudaSuccess)
                return fail("rank: trace events");
        for (auto& e : finish_) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
        gather_count_ = 1 + 4 * static_cast<int64_t>(2 * iterations + 4);  // rank_run's trace record
        if (cudaMalloc(&d_gather_, gather_count_ * ((tr_ ? tr_->world : 1) + 1) * sizeof(double)) != cudaSuccess)
            return fail("rank: cudaMalloc gather");
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
    int metric(int x, int y, int slot, int col) override {
        return metric_launch(bufs_[x], bufs_[y], len_, nullptr, nullptr, d_metric_ + 2 * slot + col, cctx_->stream) ==
                       cudaSuccess
                   ? PSWIM_OK
                   : fail("metric");
    }
    int zero_metric(int slot) override {
        return cudaMemsetAsync(d_metric_ + 2 * slot, 0, 2 * sizeof(double), cctx_->stream) == cudaSuccess
                   ? PSWIM_OK
                   : fail("metric");
    }
    double* metric_slot(int slot) override { return d_metric_ + 2 * slot; }
    int publish_metric(int slot) override {
        if (cudaMemcpyAsync(h_metric_ + 2 * slot, d_metric_ + 2 * slot, 2 * sizeof(double), cudaMemcpyDeviceToHost,
                            comm_) != cudaSuccess ||
            cudaEventRecord(published_[slot], comm_) != cudaSuccess)
            return fail("publish_metric");
        return PSWIM_OK;
    }
    int read_metric(int slot, double* out2) override {
        const int rc = poll(published_[slot]);
        if (rc) return rc;
        out2[0] = h_metric_[2 * slot];
        out2[1] = h_metric_[2 * slot + 1];
        return PSWIM_OK;
    }
    cudaStream_t q(int queue) { return queue == 0 ? cctx_->stream : (queue == 1 ? fctx_->stream : comm_); }
    int mark(int queue, int tag) override {
        return cudaEventRecord(events_[tag], q(queue)) == cudaSuccess ? PSWIM_OK : fail("event record");
    }
    int wait(int queue, int tag) override {
        return cudaStreamWaitEvent(q(queue), events_[tag], 0) == cudaSuccess ? PSWIM_OK : fail("event wait");
    }
    void* stream(int queue) override { return q(queue); }
    int task_begin(int queue, int kind, int k) override {
        if (used_ >= static_cast<int>(tasks_.size())) return fail("rank: trace event pool exhausted", PSWIM_ESTATE);
        Task& t = tasks_[used_];
        t.kind = kind;
        t.k = k;
        if (cudaEventRecord(t.a, q(queue)) != cudaSuccess) return fail("trace event");
        open_[queue] = used_++;
        return PSWIM_OK;
    }
    int task_end(int queue) override {
        return cudaEventRecord(tasks_[open_[queue]].b, q(queue)) == cudaSuccess ? PSWIM_OK : fail("trace event");
    }
    int origin() override { return cudaEventRecord(origin_, comm_) == cudaSuccess ? PSWIM_OK : fail("origin"); }
    int finish() override {
        cudaSetDevice(device_);
        for (int queue = 0; queue < 3; ++queue) {
            cudaEventRecord(finish_[queue], q(queue));
            const int rc = poll(finish_[queue]);
            if (rc) return rc;
        }
        int rc = cctx_->sync();  // device error flags (stiffness, degenerate segment, ...)
        if (rc) return fail(cctx_->err, rc);
        rc = fctx_->sync();
        if (rc) return fail(fctx_->err, rc);
        return PSWIM_OK;
    }
    int local_trace(std::vector<double>* flat) override {
        flat->clear();
        for (int i = 0; i < used_; ++i) {
            const Task& t = tasks_[i];
            float a = 0.f, b = 0.f;
            cudaEventElapsedTime(&a, origin_, t.a);
            cudaEventElapsedTime(&b, origin_, t.b);
            flat->insert(flat->end(), {double(t.kind), double(t.k), 1e-3 * a, 1e-3 * b});
        }
        return PSWIM_OK;
    }
    int gather(const double* send, double* recv, int64_t count) override {
        cudaSetDevice(device_);
        const int world = tr_->world;
        if (count > gather_count_) return fail("gather: record larger than reserved", PSWIM_ESTATE);
        double* d = d_gather_;
        int rc = PSWIM_OK;
        if (cudaMemcpyAsync(d, send, count * sizeof(double), cudaMemcpyHostToDevice, comm_) != cudaSuccess ||
            tr_->allgather(tr_->user, d, d + count, count, comm_) != 0 ||
            cudaMemcpyAsync(recv, d + count, count * world * sizeof(double), cudaMemcpyDeviceToHost, comm_) !=
                cudaSuccess)
            rc = fail("gather", PSWIM_ECOMM);
        if (!rc && cudaStreamSynchronize(comm_) != cudaSuccess) rc = fail("gather");
        return rc;
    }
    int handoff_recv(pswim_handoff* h, int k, unsigned long long gen, int idx) override {
        // the slot IS the input buffer: wait for the producer's release on queue 0, no copy
        if (handoff_wait_launch(h, k, gen, cctx_->stream) != cudaSuccess) return fail("handoff wait");
        bufs_[idx] = handoff_recv_slot(h, k);
        return PSWIM_OK;
    }
    int handoff_push(pswim_handoff* h, int k, unsigned long long gen, int idx) override {
        return handoff_push_launch(h, k, gen, bufs_[idx], cctx_->stream) == cudaSuccess ? PSWIM_OK
                                                                                       : fail("handoff push");
    }
    int handoff_correct_push(pswim_handoff* h, int k, unsigned long long gen, int xp, int gn, int go,
                             int out) override {
        return handoff_correct_push_launch(h, k, gen, bufs_[xp], bufs_[gn], bufs_[go], bufs_[out], cctx_->stream) ==
                       cudaSuccess
                   ? PSWIM_OK
                   : fail("handoff correct");
    }
    void prepare_device_waits() override {
        pswim_set_graphs(cctx_, 0);
        pswim_set_graphs(fctx_, 0);
    }
    std::string error() override { return err_; }

  private:
    struct Task {
        cudaEvent_t a = nullptr, b = nullptr;
        int kind = 0, k = 0;
    };
    int fail(const std::string& w, int code = PSWIM_ECUDA) {
        err_ = w;
        return code;
    }
    // Host wait on a device event that also watches the transport (ncclCommGetAsyncError for
    // NCCL) and a timeout; either aborts the transport so no peer waits forever.
    int poll(cudaEvent_t ev) {
        const auto t0 = Clock::now();
        for (;;) {
            const cudaError_t e = cudaEventQuery(ev);
            if (e == cudaSuccess) return PSWIM_OK;
            if (e != cudaErrorNotReady) return fail(std::string("rank: ") + cudaGetErrorString(e));
            if (tr_ && tr_->health) {
                const int h = tr_->health(tr_->user);
                if (h) {
                    if (tr_->abort) tr_->abort(tr_->user);
                    return fail("rank: transport failed", h);
                }
            }
            if (std::chrono::duration<double>(Clock::now() - t0).count() > timeout_) {
                if (tr_ && tr_->abort) tr_->abort(tr_->user);
                return fail("rank: timed out waiting for the device / peers (PSWIM_COMM_TIMEOUT_S)", PSWIM_ECOMM);
            }
            std::this_thread::sleep_for(std::chrono::microseconds(20));
        }
    }
    int device_;
    int64_t len_, fine_steps_, coarse_steps_;
    const pswim_transport* tr_ = nullptr;
    const pswim_transport* sp_c_ = nullptr;
    const pswim_transport* sp_f_ = nullptr;
    double timeout_;
    pswim_ctx* cctx_ = nullptr;
    pswim_ctx* fctx_ = nullptr;
    int hi_ = 0, lo_ = 0;
    cudaStream_t comm_ = nullptr;
    std::vector<double*> owned_, bufs_;
    double* d_metric_ = nullptr;
    double* h_metric_ = nullptr;
    std::vector<cudaEvent_t> events_, published_;
    std::vector<Task> tasks_;
    int used_ = 0;
    int open_[3] = {0, 0, 0};
    cudaEvent_t origin_ = nullptr;
    cudaEvent_t finish_[3] = {nullptr, nullptr, nullptr};
    double* d_gather_ = nullptr;
    int64_t gather_count_ = 0;
    std::string err_;
};

// Buffers a slice rank needs (see rank_run): IN, XB, FB, GB per iteration 0..Kn, + REF.
inline int slice_buffer_count(const pswim_plan& plan, int rank) {
    const int K = std::min(plan.max_iterations, plan.intervals);
    const int Kn = std::min(rank + 1, K);
    return 4 * (Kn + 1) + 1;
}

// Event tags: per iteration k, tag = 8 k + kind.
enum { kTagIn = 0, kTagX = 1, kTagFine = 2, kTagMetric = 3, kTagAR = 4 };
inline int tag(int k, int what) { return 8 * k + what; }

// A plan whose tolerance no metric can undercut short of an exact 0: its iteration count is
// fixed, so nothing needs deciding before the end (the bench's l sweeps use 1e-300).
constexpr double kFixedTolerance = 1e-200;

struct TraceOut {
    pswim_trace_event* events = nullptr;
    int64_t cap = 0;
    int64_t* len = nullptr;
};

// The slice recurrence for rank p (interval n = p + 1), parareal.cpp:58-89:
//   X[0][n] = G(X[0][n-1]);  X[k][k] = F(X[k-1][k-1]);
//   X[k][n] = F(X[k-1][n-1]) + G(X[k][n-1]) - G(X[k-1][n-1])   (1 <= k < n)
//   X[k][n] = X[n][n]                                           (k > n, frozen)
// Rank p receives X[k][n-1] from p-1 for k = 0..min(n-1, K) and sends X[k][n] to p+1 for
// k = 0..min(n, K).  Every rank reduces [eta_tilde_k, eta_k] with one allreduce(max) per
// iteration, and evaluates the stop rule of parareal.cpp:366-393 identically from it.
//
// Issue order.  The host enqueues whole iterations ("blocks") ahead of the stop decisions:
// block k is recv(k), G + correct, send(k), the metric, and (pipelined) the next fine solve,
// all stream-ordered with events, no host wait.  The allreduce of iteration j is issued after
// block j + lag (lag = 0 regular, the lookahead pipelined, K for fixed-iteration plans, whose
// metrics are all reduced at the end).  Every p2p operation a rank issues before AR(j) is
// then matched by one its neighbour issues before AR(j) (both sit in blocks <= j + lag), so no
// collective can wait on an unmatched hand-off; hand-offs are deliberately not grouped with
// the next receive for the same reason.  The host reads AR(j) only when it must decide
// whether to issue block j + lag + 1 (tolerance plans), and regular mode's barrier -- fine(k+1)
// after the iteration-k decision -- is a device-side wait on AR(k).  After a stop, the
// speculative blocks every rank issued drain (their hand-offs are matched pairwise).
int rank_run(const pswim_plan& plan, SliceBackend& be, const pswim_transport& tr, pswim_handoff* ho, int64_t len,
             const double* x0, const double* ref_slice, double* out, pswim_report* rep, const TraceOut& tout) {
    const int p = tr.rank, m = tr.world;
    if (plan.intervals != m || p < 0 || p >= m) return PSWIM_EINVAL;
    const int n = p + 1;
    const int K = std::min(plan.max_iterations, plan.intervals);  // l = min(l_max, n)
    const int Kn = std::min(n, K);                               // last iteration with work here
    const bool pipelined = plan.mode == 1;
    const bool has_prev = p > 0, has_next = p + 1 < m;
    const bool fixed = plan.tolerance < kFixedTolerance;
    const int lag = pipelined ? (fixed ? K : parareal_lookahead(plan)) : 0;
    if (K + 1 > 4000) return PSWIM_EINVAL;
    // buffers: IN+k = X[k][n-1]; XB+k = corrected X[k][n]; FB+k = F(X[k-1][n-1]); GB+k = G(X[k][n-1])
    const int IN = 0, XB = IN + (Kn + 1), FB = XB + (Kn + 1), GB = FB + (Kn + 1), REF = GB + (Kn + 1);
    if (!be.allocated()) {
        const int rc = be.alloc(REF + 1, K);
        if (rc) return rc;
    }
    const unsigned long long gen = ho ? handoff_begin_run(ho) : 0;
    if (ho) be.prepare_device_waits();
    if (ho && has_next && !handoff_has_next(ho)) return PSWIM_EINVAL;
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

    // host uploads first: a synchronous copy must not sit behind a peer's device-side wait
    if (ref_slice) RK(be.upload(REF, ref_slice));
    if (!has_prev) RK(be.upload(IN, x0));
    // start barrier (one allreduce on the comm queue) -> a common time origin for the trace
    RT(tr.allreduce_max(tr.user, be.metric_slot(K + 1), 2, cs));
    RK(be.origin());
    const auto t_begin = Clock::now();  // wall time of the run: from the start barrier on

    // X[k][n] leaves for rank p+1 (transport path; the peer hand-off is done by the producer)
    auto send_state = [&](int k, int idx) -> int {
        RK(be.mark(0, tag(k, kTagX)));
        if (has_next && !ho) {
            RK(be.wait(2, tag(k, kTagX)));
            RT(tr.send(tr.user, be.buf(idx), len, p + 1, cs));
        }
        return PSWIM_OK;
    };
    // X[k][n-1] from rank p-1 into IN+k, ordered before queue 0 uses it (mark kTagIn)
    auto recv_state = [&](int k) -> int {
        if (ho) {
            RK(be.handoff_recv(ho, k, gen, IN + k));
            return be.mark(0, tag(k, kTagIn));
        }
        RT(tr.recv(tr.user, be.buf(IN + k), len, p - 1, cs));
        RK(be.mark(2, tag(k, kTagIn)));
        return be.wait(0, tag(k, kTagIn));
    };
    auto launch_fine = [&](int k) -> int {
        // F(X[k][n-1]) for iteration k+1, on the fine queue, after the input arrived and after
        // this rank's own coarse / corrector on the same input produced X[k][n]: the coarse
        // chain through the ranks is the sequential critical path, and sharing the GPU with
        // its own fine solve slows each link (tools/probe_contention.py), while F only starts
        // T_G later.  Regular mode: also after the global iteration-k barrier (AR(k)).
        if (k + 1 > Kn) return PSWIM_OK;
        if (has_prev) RK(be.wait(1, tag(k, kTagIn)));
        RK(be.wait(1, tag(k, kTagX)));
        if (!pipelined) RK(be.wait(1, tag(k, kTagAR)));
        RK(be.task_begin(1, kFine, k + 1));
        RK(be.fine(IN + k, t_lo, t_hi, FB + k + 1));
        RK(be.task_end(1));
        return be.mark(1, tag(k + 1, kTagFine));
    };
    auto block = [&](int k) -> int {
        if (k == 0) {  // the coarse sweep
            if (has_prev) RK(recv_state(0));  // rank 0's x0 was uploaded before the start barrier
            RK(be.task_begin(0, kCoarse, 0));
            RK(be.coarse(IN, t_lo, t_hi, GB));
            if (ho && has_next) RK(be.handoff_push(ho, 0, gen, GB));
            RK(be.task_end(0));
            xidx[0] = GB;  // X[0][n] = G(X[0][n-1])
            RK(send_state(0, GB));
            if (pipelined) RK(launch_fine(0));
            RK(be.zero_metric(0));  // regular mode's iteration-0 barrier reduces this slot
            return be.mark(0, tag(0, kTagMetric));
        }
        if (k <= Kn) {
            if (k < n) {
                RK(recv_state(k));
                RK(be.wait(0, tag(k, kTagFine)));
                RK(be.task_begin(0, kCorrect, k));
                RK(be.coarse(IN + k, t_lo, t_hi, GB + k));
                if (ho && has_next)
                    RK(be.handoff_correct_push(ho, k, gen, FB + k, GB + k, GB + k - 1, XB + k));
                else
                    RK(be.correct(FB + k, GB + k, GB + k - 1, XB + k));
                RK(be.task_end(0));
                xidx[k] = XB + k;
            } else {  // k == n: the interval is exact from here on
                RK(be.wait(0, tag(k, kTagFine)));
                xidx[k] = FB + k;
                if (ho && has_next) RK(be.handoff_push(ho, k, gen, FB + k));
            }
            RK(send_state(k, xidx[k]));
            if (pipelined && k < n) RK(launch_fine(k));
            RK(be.zero_metric(k));
            RK(be.metric(xidx[k], xidx[k - 1], k, 0));
            if (ref_slice) RK(be.metric(REF, xidx[k], k, 1));
        } else {
            // frozen: contributes 0 to eta_tilde and its unchanged true error
            RK(be.zero_metric(k));
            if (ref_slice) RK(be.metric(REF, xidx[Kn], k, 1));
        }
        return be.mark(0, tag(k, kTagMetric));
    };
    auto allreduce = [&](int j) -> int {
        RK(be.wait(2, tag(j, kTagMetric)));
        RT(tr.allreduce_max(tr.user, be.metric_slot(j), 2, cs));
        RK(be.mark(2, tag(j, kTagAR)));
        return be.publish_metric(j);
    };

    int decided = 0, final_k = 0, ar_issued = 0;
    bool stop = false, converged = false;
    std::vector<double> eta_tilde, eta;
    auto decide = [&](int j) -> int {
        double v[2];
        RK(be.read_metric(j, v));
        eta_tilde.push_back(v[0]);
        eta.push_back(v[1]);
        decided = final_k = j;
        if (v[0] < plan.tolerance || j == plan.intervals) {
            converged = true;
            stop = true;
        } else if (j == K) {
            stop = true;
        }
        return PSWIM_OK;
    };

    RK(block(0));
    if (!pipelined) {
        RK(allreduce(0));
        RK(launch_fine(0));
    }
    for (int b = 1; b <= K; ++b) {
        if (!fixed)
            while (!stop && decided < b - 1 - lag) RK(decide(decided + 1));
        if (stop) break;
        RK(block(b));
        if (b - lag >= 1) RK(allreduce(ar_issued = b - lag));
        if (!pipelined) {
            if (!fixed) {
                RK(decide(b));
                if (stop) break;
            }
            RK(launch_fine(b));
        }
    }
    if (!stop) {
        while (ar_issued < K) RK(allreduce(++ar_issued));
        while (!stop && decided < K) RK(decide(decided + 1));
    }
    RK(be.finish());  // speculative blocks past the stop drain here
    RK(be.download(out, xidx[std::min(final_k, Kn)]));

    // schedule trace: every rank's (kind, k, t0, t1) gathered to all ranks; coarse sweep and
    // correctors are the serial tier (worker 0), rank p's fine solves worker p + 1
    const int64_t cap = 2 * K + 4, rec = 1 + 4 * cap;
    std::vector<double> mine(rec, 0.0), flat, all(rec * m);
    RK(be.local_trace(&flat));
    const int64_t cnt = std::min<int64_t>(cap, static_cast<int64_t>(flat.size() / 4));
    mine[0] = static_cast<double>(cnt);
    std::copy(flat.begin(), flat.begin() + 4 * cnt, mine.begin() + 1);
    RK(be.gather(mine.data(), all.data(), rec));
    std::vector<pswim_trace_event> ev;
    for (int r = 0; r < m; ++r) {
        const double* q = all.data() + r * rec;
        for (int i = 0; i < static_cast<int>(q[0]); ++i) {
            const int kind = static_cast<int>(q[1 + 4 * i]);
            ev.push_back(pswim_trace_event{kind == kFine ? r + 1 : 0, kind, q[3 + 4 * i], q[4 + 4 * i],
                                           static_cast<int32_t>(q[2 + 4 * i]), r + 1});
        }
    }
    const double idle = finalize_idle(&ev);
#undef RK
#undef RT
    rep->iterations_used = final_k;
    rep->converged = converged ? 1 : 0;
    rep->eta_count = static_cast<int32_t>(eta_tilde.size());
    for (size_t k = 0; k < eta_tilde.size(); ++k) {
        if (rep->eta_tilde) rep->eta_tilde[k] = eta_tilde[k];
        if (rep->eta && ref_slice) rep->eta[k] = eta[k];
    }
    rep->wall_seconds = std::chrono::duration<double>(Clock::now() - t_begin).count();
    rep->schedule_idle = idle;
    if (tout.len) *tout.len = static_cast<int64_t>(ev.size());
    if (tout.events)
        std::copy(ev.begin(), ev.begin() + std::min<int64_t>(tout.cap, static_cast<int64_t>(ev.size())), tout.events);
    return PSWIM_OK;
}

// ---------------------------------------------------------------------------------------
// In-process transport: slice ranks as threads, one context pair per rank (any devices).
// send = peer copy into a per-message staging buffer on the receiver's device + event;
// recv = stream wait on that event + local copy; allreduce = host barrier on 2 doubles.
// ---------------------------------------------------------------------------------------
class ThreadHub {
  public:
    static constexpr int64_t kReduceMax = 64;
    ThreadHub(int world, const int* devices, int64_t len, int slots)
        : world_(world), len_(len), devices_(devices, devices + world), links_(world), red_host_(world, nullptr),
          red_done_(world, nullptr) {
        for (int p = 0; p < world; ++p) {
            cudaSetDevice(devices_[p]);
            cudaMallocHost(&red_host_[p], kReduceMax * sizeof(double));
            cudaEventCreateWithFlags(&red_done_[p], cudaEventDisableTiming);
        }
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
        for (int p = 0; p < world_; ++p) {
            cudaSetDevice(devices_[p]);
            if (red_host_[p]) cudaFreeHost(red_host_[p]);
            if (red_done_[p]) cudaEventDestroy(red_done_[p]);
        }
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
        // pinned per-rank staging + an event poll: no pageable copy and no blocking driver
        // sync while other ranks' streams may spin on device-side hand-off flags
        if (len > kReduceMax) return PSWIM_ECOMM;
        cudaSetDevice(devices_[rank]);
        double* h = red_host_[rank];
        if (cudaMemcpyAsync(h, dbuf, len * sizeof(double), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
            cudaEventRecord(red_done_[rank], st) != cudaSuccess || !poll(red_done_[rank]))
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
            std::copy(result_.begin(), result_.begin() + len, h);
        }
        if (cudaMemcpyAsync(dbuf, h, len * sizeof(double), cudaMemcpyHostToDevice, st) != cudaSuccess ||
            cudaEventRecord(red_done_[rank], st) != cudaSuccess || !poll(red_done_[rank]))
            return PSWIM_ECOMM;
        return PSWIM_OK;
    }
    bool poll(cudaEvent_t e) {
        for (;;) {
            const cudaError_t r = cudaEventQuery(e);
            if (r == cudaSuccess) return true;
            if (r != cudaErrorNotReady || aborted()) return false;
            std::this_thread::sleep_for(std::chrono::microseconds(10));
        }
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
    bool aborted() {
        std::lock_guard<std::mutex> lk(mu_);
        return aborted_;
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
    std::vector<double*> red_host_;        // pinned allreduce staging, per rank
    std::vector<cudaEvent_t> red_done_;
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

int hub_health(void* u) {
    auto* h = static_cast<HubUser*>(u);
    return h->hub->aborted() ? PSWIM_ECOMM : PSWIM_OK;
}
void hub_abort(void* u) { static_cast<HubUser*>(u)->hub->abort(); }
pswim_transport hub_transport(HubUser* u, int rank, int world) {
    return pswim_transport{u, rank, world, hub_send, hub_recv, hub_allreduce, hub_allgather, hub_health, hub_abort};
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

int pswim_parareal_rank_gpu(const pswim_plan* plan, const pswim_scenario* sc, int device, const pswim_transport* tr,
                            pswim_handoff* handoff, int64_t fine_steps, int64_t coarse_steps, const double* x0,
                            const double* ref_slice, double* state_out, pswim_report* rep, pswim_trace_event* trace_out,
                            int64_t trace_cap, int64_t* trace_len) {
    using namespace pswim;
    if (plan_check(plan) || !sc || !tr || !x0 || !state_out || !rep || fine_steps < 1 || coarse_steps < 1)
        return PSWIM_EINVAL;
    try {
        GpuSlice be(*sc, device, fine_steps, coarse_steps, tr);
        return rank_run(*plan, be, *tr, handoff, 12 * sc->rod_count * sc->nodes_per_rod, x0, ref_slice, state_out, rep,
                        TraceOut{trace_out, trace_cap, trace_len});
    } catch (const CodeError& e) {
        return e.code;
    }
}

int pswim_parareal_rank_gpu_hybrid(const pswim_plan* plan, const pswim_scenario* sc, int device,
                                   const pswim_transport* time_tr, const pswim_transport* space_coarse,
                                   const pswim_transport* space_fine, int64_t fine_steps, int64_t coarse_steps,
                                   const double* x0, const double* ref_slice, double* state_out, pswim_report* rep,
                                   pswim_trace_event* trace_out, int64_t trace_cap, int64_t* trace_len) {
    using namespace pswim;
    if (plan_check(plan) || !sc || !time_tr || !space_coarse || !space_fine || !x0 || !state_out || !rep ||
        fine_steps < 1 || coarse_steps < 1)
        return PSWIM_EINVAL;
    if (space_coarse->world != space_fine->world || space_coarse->rank != space_fine->rank || !space_coarse->allgather ||
        !space_fine->allgather)
        return PSWIM_EINVAL;
    try {
        GpuSlice be(*sc, device, fine_steps, coarse_steps, time_tr, space_coarse, space_fine);
        return rank_run(*plan, be, *time_tr, nullptr, 12 * sc->rod_count * sc->nodes_per_rod, x0, ref_slice, state_out,
                        rep, TraceOut{trace_out, trace_cap, trace_len});
    } catch (const CodeError& e) {
        return e.code;
    }
}

int pswim_parareal_rank_host(const pswim_plan* plan, pswim_propagator_fn coarse, void* cu, pswim_propagator_fn fine,
                             void* fu, const pswim_transport* tr, const double* x0, int64_t len, int32_t dim,
                             int32_t stride, const double* ref_slice, double* state_out, pswim_report* rep,
                             pswim_trace_event* trace_out, int64_t trace_cap, int64_t* trace_len) {
    using namespace pswim;
    if (plan_check(plan) || !coarse || !fine || !tr || !x0 || !state_out || !rep || len <= 0) return PSWIM_EINVAL;
    if (dim < 1 || stride < dim || len % stride != 0) return PSWIM_EINVAL;
    HostSlice be(len, coarse, cu, fine, fu, dim, stride, *tr);
    return rank_run(*plan, be, *tr, nullptr, len, x0, ref_slice, state_out, rep,
                    TraceOut{trace_out, trace_cap, trace_len});
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
            b->trs[p] = hub_transport(&b->users[p], p, world);
        }
        // trailing sentinel remembers the bundle for destroy
        b->trs[world] = pswim_transport{b, -1, world, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
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
                               double* states_out, pswim_report* rep, int32_t handoff, pswim_trace_event* trace_out,
                               int64_t trace_cap, int64_t* trace_len) {
    using namespace pswim;
    if (plan_check(plan) || !sc || !devices || !x0 || !states_out || !rep || fine_steps < 1 || coarse_steps < 1)
        return PSWIM_EINVAL;
    const int world = plan->intervals;
    const int64_t len = 12 * sc->rod_count * sc->nodes_per_rod;
    const int K = std::min(plan->max_iterations, plan->intervals);
    try {
        ThreadHub hub(world, devices, len, K + 2);
        // peer-memory hand-offs: rank p pushes into rank p+1's slots (raw pointers in-process)
        std::vector<pswim_handoff*> hos(world, nullptr);
        struct Release {
            std::vector<pswim_handoff*>& v;
            ~Release() {
                for (auto* h : v) pswim_handoff_destroy(h);
            }
        } release{hos};
        if (handoff) {
            for (int p = 0; p < world; ++p)
                if (!(hos[p] = pswim_handoff_create(devices[p], len, K + 1))) return PSWIM_ECUDA;
            for (int p = 0; p + 1 < world; ++p)
                if (pswim_handoff_connect_local(hos[p], hos[p + 1])) return PSWIM_ECOMM;
        }
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
            trs[p] = hub_transport(&users[p], p, world);
            reps[p] = *rep;
            reps[p].eta_tilde = et[p].data();
            reps[p].eta = ea[p].data();
            threads.emplace_back([&, p] {
                try {
                    GpuSlice be(*sc, devices[p], fine_steps, coarse_steps, &trs[p]);
                    rcs[p] = be.alloc(slice_buffer_count(*plan, p), K);
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
                        rcs[p] = rank_run(*plan, be, trs[p], hos[p], len, x0,
                                          reference ? reference + len * (p + 1) : nullptr, states_out + len * (p + 1),
                                          &reps[p], p == 0 ? TraceOut{trace_out, trace_cap, trace_len} : TraceOut{});
                    if (rcs[p] && rcs[p] != PSWIM_ECOMM) std::fprintf(stderr, "pswim: slice rank %d: %s\n", p, be.error().c_str());
                } catch (const CodeError& e) {
                    rcs[p] = e.code;
                    std::fprintf(stderr, "pswim: slice rank %d: %s\n", p, e.what());
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
        rep->schedule_idle = reps[0].schedule_idle;
    } catch (const CodeError& e) {
        return e.code;
    }
    return PSWIM_OK;
}

}  // extern "C"
