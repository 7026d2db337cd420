// parareal.cpp — the time-sliced Parareal driver: one time slice per rank (rank p owns
// interval p+1, intervals == world), the recurrence of src/parareal.cpp:58-89 with one state
// hand-off per iteration to rank p+1 and one allreduce(max) of the iteration metric.
// Coarse/corrector on a high-priority stream, fine on a low-priority stream, transport on a
// third.  Transports: NCCL (one process per GPU, nccl_transport.cpp), in-process threads +
// peer copies (pswim_parareal_run_threads), host callbacks (CPU tests over gloo).
// The single-device engine (parareal::run itself) is engine.cpp.
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
#include "parareal_common.h"

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
