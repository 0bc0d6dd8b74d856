// ctk_driver.cu -- native run_gmres: the whole (hybrid) AB-/BA-GMRES loop of
// ctkrylov/gmres.py:135-241 in C++, no Python per iteration.
//
// Two streams: A runs the Arnoldi process ahead (LOOKAHEAD steps in flight,
// independent of lambda); B runs the iterate updates x_k = x0 + (B) W y_k and
// true residuals.  The host thread waits only for each step's Hessenberg
// column, hands the fp64 projected problem (SVD, lambda grid, L-curve/GCV,
// Tikhonov; ctk_host.cpp) to native worker threads, and consumes results in
// iteration order (the degenerate-curve fallback needs the previous lambda,
// gmres.py:196-200).  Stopping rules dp / rns need each iterate's residual
// before the next record; they sync on it (the Arnoldi look-ahead keeps
// running).  ncp, x_true metrics and snapshots stay in the Python driver.
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <chrono>
#include <condition_variable>
#include <deque>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include "ctk_common.cuh"

namespace {

constexpr int IB_BATCH = 8;         // iterates per ctk_iterate_batch launch

struct Job {
    int k = 0;
    std::vector<double> H;      // (k+1) x k row-major
    double beta = 0.0;
    int strategy = 0;
    double value = 0.0;
    double out[4] = {0, 0, 0, 0};
    std::vector<double> y;
    int rc = 0;
    bool done = false;
};

class Pool {
  public:
    explicit Pool(int n) {
        for (int i = 0; i < n; ++i) th_.emplace_back([this] { loop(); });
    }
    ~Pool() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : th_) t.join();
    }
    void submit(std::shared_ptr<Job> j) {
        {
            std::lock_guard<std::mutex> lk(mu_);
            q_.push_back(std::move(j));
        }
        cv_.notify_one();
    }
    void wait(const std::shared_ptr<Job>& j) {
        std::unique_lock<std::mutex> lk(mu_);
        done_cv_.wait(lk, [&] { return j->done; });
    }
    // The last column's problem runs on the calling thread (it would only
    // wait for it): two thread hand-offs off the solve's critical tail.
    void run_inline(const std::shared_ptr<Job>& j) {
        solve(*j);
        std::lock_guard<std::mutex> lk(mu_);
        j->done = true;
    }
    bool ready(const std::shared_ptr<Job>& j) {
        std::lock_guard<std::mutex> lk(mu_);
        return j->done;
    }

  private:
    static void solve(Job& j) {
        j.y.assign(j.k, 0.0);
        j.rc = ctk_projected_solve(j.H.data(), j.k, j.beta, j.strategy, j.value, 200, NAN, j.out,
                                   j.y.data());
    }
    void loop() {
        for (;;) {
            std::shared_ptr<Job> j;
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return stop_ || !q_.empty(); });
                if (stop_ && q_.empty()) return;
                j = std::move(q_.front());
                q_.pop_front();
            }
            solve(*j);
            {
                std::lock_guard<std::mutex> lk(mu_);
                j->done = true;
            }
            done_cv_.notify_all();
        }
    }
    std::vector<std::thread> th_;
    std::deque<std::shared_ptr<Job>> q_;
    std::mutex mu_;
    std::condition_variable cv_, done_cv_;
    bool stop_ = false;
};

Pool& pool() {
    static Pool p([] {
        unsigned n = std::thread::hardware_concurrency();
        int w = n > 2 ? (int)n - 1 : 2;
        w = w > 8 ? 8 : w;
        const char* e = getenv("CTK_POOL_THREADS");        // tuning override
        if (e && atoi(e) > 0) w = atoi(e);
        return w;
    }());
    return p;
}

// scal[2] = 1 / sqrt(scal[0]) (0 when the residual is exactly zero): the
// cycle start normalises w0 on the device, so the Arnoldi pipeline starts
// without a host round trip for beta.
// Sharded solve: the x-norm entries of norms[slot][2] are replicated (every
// rank holds the whole image); ranks other than 0 zero theirs before the
// norms are summed over ranks, so the sum is rank 0's value on every rank.
__global__ void k_zero_odd(double* v, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) v[2 * i + 1] = 0.0;
}

__global__ void k_set_inv(double* scal) {
    const double s = scal[0];
    scal[2] = s > 0.0 ? 1.0 / sqrt(s) : 0.0;
}

// Events are recycled across solves (a solve creates ~2K+ of them; create +
// destroy costs ~1-2 us each on the host).  Every event handed out has
// completed when its solve returns (the solve ends with stream syncs).
struct EventPool {
    std::mutex mu;
    std::vector<cudaEvent_t> free_ev[2];      // [timing]
    int device = -1;
};

EventPool& event_pool() {
    static EventPool* p = new EventPool();    // never destroyed (CUDA may be gone at exit)
    return *p;
}

struct Events {
    std::vector<cudaEvent_t> ev[2];
    ~Events() {
        EventPool& p = event_pool();
        std::lock_guard<std::mutex> lk(p.mu);
        for (int t = 0; t < 2; ++t)
            p.free_ev[t].insert(p.free_ev[t].end(), ev[t].begin(), ev[t].end());
    }
    cudaEvent_t make(bool timing) {
        const int t = timing ? 1 : 0;
        cudaEvent_t e = nullptr;
        {
            EventPool& p = event_pool();
            std::lock_guard<std::mutex> lk(p.mu);
            int dev = 0;
            cudaGetDevice(&dev);
            if (p.device != dev) {                // pool is per device: drop on switch
                for (int q = 0; q < 2; ++q) p.free_ev[q].clear();
                p.device = dev;
            }
            if (!p.free_ev[t].empty()) {
                e = p.free_ev[t].back();
                p.free_ev[t].pop_back();
            }
        }
        if (!e) cudaEventCreateWithFlags(&e, timing ? cudaEventDefault : cudaEventDisableTiming);
        ev[t].push_back(e);
        return e;
    }
};

}  // namespace

extern "C" int ctk_solve(const ctk_geom_t* g, const ctk_solve_cfg* cfg, ctk_solve_bufs* bf,
                         ctk_solve_out* out) {
    if (!g || !cfg || !bf || !out) return ctk_fail(CTK_ERR_ARG, "null argument");
    const bool ab = cfg->ab != 0;
    const int K = cfg->max_iter;
    const int p = cfg->restart_period > 0 ? cfg->restart_period : K;
    const int rows = (p < K ? p : K) + 1;
    if (bf->rows < rows || bf->hcols < rows + 5) return ctk_fail(CTK_ERR_ARG, "buffers too small");
    const int na = g->n_angles;
    const int64_t n = (int64_t)g->nx * g->ny, m = (int64_t)na * g->det_count;
    const int64_t L = ab ? m : n;
    cudaStream_t sa = ctk_stream(bf->stream_a), sb = ctk_stream(bf->stream_b);
    const int hc = bf->hcols;
    const int look = cfg->lookahead > 0 ? cfg->lookahead : 6;
    const ctk_comm* comm = bf->comm;       // angle-sharded solve (ctk_comm.cu), or NULL
    if (comm && !(bf->aux1 && bf->d0 && (!ab || bf->aux2)))
        return ctk_fail(CTK_ERR_ARG, "the sharded solve needs the linear iterate rows (aux, d0)");
    CTK_CUDA(cudaSetDevice(g->device));
    Events evs;
    cudaEvent_t ev_start = evs.make(true);
    const char* tr_env = getenv("CTK_TRACE");
    const bool trace = tr_env && tr_env[0] == '1';
    std::vector<cudaEvent_t> ev_h(rows), ev_it(K + 1);
    for (int i = 0; i < rows; ++i) ev_h[i] = evs.make(trace);
    for (int i = 0; i <= K; ++i) ev_it[i] = evs.make(true);
    cudaEvent_t ev_sync = evs.make(false);
    CTK_CUDA(cudaEventRecord(ev_start, sa));
    CTK_CUDA(cudaStreamWaitEvent(sb, ev_start, 0));

    // CTK_TRACE=1: per-step GPU timeline of stream A (debug; stderr)
    std::vector<cudaEvent_t> tr_beg(trace ? rows : 0);
    std::vector<double> tr_host(trace ? rows : 0, 0.0);
    double tr_wait = 0.0, tr_consumed_at = 0.0;
    for (auto& e : tr_beg) e = evs.make(true);
    int nrec = 0, cycles = 0, stop = CTK_STOP_NONE;
    double prev_lam = 0.0;
    std::vector<double> history;
    std::vector<int> rec_slot;                        // record -> norms slot (-1: host-known)
    auto t0 = std::chrono::steady_clock::now();
    const char* ib_env = getenv("CTK_ITER_BATCH");          // 0: one iterate per launch
    const bool can_batch = !(ib_env && ib_env[0] == '0') && bf->aux1 && bf->d0 &&
                           (!ab || bf->aux2) && !bf->x_true && bf->snapshot_stride <= 0 &&
                           cfg->stopping == CTK_STOP_NONE;
    bool first = true;
    int rc;
    while (stop == CTK_STOP_NONE && nrec < K) {
        if (!first) {   // restart from the current iterate (gmres.py:172-175)
            CTK_CUDA(cudaEventRecord(ev_sync, sb));
            CTK_CUDA(cudaStreamWaitEvent(sa, ev_sync, 0));
            CTK_CUDA(cudaMemcpyAsync(bf->x_cur, bf->xk, sizeof(float) * n,
                                     cudaMemcpyDeviceToDevice, sa));
        }
        first = false;
        float* w0 = bf->W;
        if (ab) {
            if ((rc = ctk_forward(g, bf->x_cur, w0, 0, na, bf->b, bf->stage_a, bf->stream_a))) return rc;
            if ((rc = ctk_norm2(w0, L, bf->scal, bf->scratch_a, bf->stream_a))) return rc;
            if (comm && (rc = ctk_comm_sum_f64(comm, bf->scal, 1, sa))) return rc;
        } else {
            if ((rc = ctk_forward(g, bf->x_cur, bf->tmp, 0, na, bf->b, bf->stage_a, bf->stream_a)))
                return rc;
            if ((rc = ctk_norm2(bf->tmp, m, bf->scal + 1, bf->scratch_a, bf->stream_a))) return rc;
            if (comm) {
                if ((rc = ctk_comm_sum_f64(comm, bf->scal + 1, 1, sa))) return rc;
                if ((rc = ctk_comm_back_sum(comm, g, bf->tmp, w0, bf->back_a, sa))) return rc;
            } else if ((rc = ctk_back(g, bf->tmp, w0, 0, na, nullptr, bf->back_a, bf->stream_a))) {
                return rc;
            }
            if ((rc = ctk_norm2(w0, L, bf->scal, bf->scratch_a, bf->stream_a))) return rc;
        }
        if (bf->aux1 && bf->d0)     // d0 = b - A x0 for the linear iterate path
            CTK_CUDA(cudaMemcpyAsync(bf->d0, ab ? w0 : bf->tmp, sizeof(float) * m,
                                     cudaMemcpyDeviceToDevice, sa));
        CTK_CUDA(cudaMemcpyAsync(bf->scal_host, bf->scal, 2 * sizeof(double), cudaMemcpyDeviceToHost, sa));
        CTK_CUDA(cudaEventRecord(ev_sync, sa));
        k_set_inv<<<1, 1, 0, sa>>>(bf->scal);
        ctk_count_launch();
        if ((rc = ctk_scale(w0, w0, L, bf->scal + 2, bf->stream_a))) return rc;
        CTK_CUDA(cudaStreamWaitEvent(sb, ev_sync, 0));
        const int steps = (p < K - nrec) ? p : K - nrec;
        // the first Arnoldi steps go out before beta is known on the host
        int queued = 0;
        std::vector<std::shared_ptr<Job>> jobs(steps + 1);
        auto enqueue_to = [&](int upto) -> int {
            while (queued < (upto < steps ? upto : steps)) {
                if (trace) CTK_CUDA(cudaEventRecord(tr_beg[queued], sa));
                int r2 = ctk_arnoldi_step_ex(g, ab, cfg->reorthogonalize ? 2 : 1, bf->W, bf->ld,
                                             queued, bf->q, bf->tmp, bf->aux1,
                                             bf->ld1, bf->aux2, bf->ld2, bf->stage_a,
                                             bf->back_a, bf->hs + (size_t)queued * hc, hc,
                                             bf->h_host + (size_t)queued * hc, bf->scratch_a,
                                             bf->stream_a, comm);
                if (r2) return r2;
                CTK_CUDA(cudaEventRecord(ev_h[queued], sa));
                if (trace) {
                    tr_host[queued] = std::chrono::duration<double>(
                        std::chrono::steady_clock::now() - t0).count();
                }
                ++queued;
            }
            return CTK_OK;
        };
        if ((rc = enqueue_to(look))) return rc;
        CTK_CUDA(cudaEventSynchronize(ev_sync));
        const double beta = sqrt(bf->scal_host[0]);
        const double d0n = ab ? beta : sqrt(bf->scal_host[1]);
        if (beta == 0.0) {           // exact solution in hand (gmres.py:176-182)
            CTK_CUDA(cudaStreamSynchronize(sa));   // let the (discarded) steps drain
            stop = CTK_STOP_BREAKDOWN;
            if (nrec == 0) {
                if ((rc = ctk_norm2(bf->x_cur, n, bf->scal + 2, bf->scratch_a, bf->stream_a))) return rc;
                CTK_CUDA(cudaMemcpyAsync(bf->scal_host + 2, bf->scal + 2, sizeof(double),
                                         cudaMemcpyDeviceToHost, sa));
                CTK_CUDA(cudaStreamSynchronize(sa));
                out->k[0] = 0;
                out->lambda[0] = 0.0;
                out->residual[0] = 0.0;
                out->data_residual[0] = d0n;
                out->proj_residual[0] = 0.0;
                out->solution_norm[0] = sqrt(bf->scal_host[2]);
                out->elapsed[0] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
                out->warn[0] = 0;
                rec_slot.push_back(-1);
                nrec = 1;
                out->x_is_x0 = 1;
            }
            break;
        }
        ++cycles;
        std::vector<double> Hfull((size_t)(steps + 1) * steps, 0.0);
        int done_k = 0, last_k = steps, broke_at = -1;
        // Batched iterate norms (no per-iterate consumer: no x_true metrics,
        // snapshots or per-iteration stopping rule): up to IB_BATCH iterates
        // share one pass over the basis (ctk_iterate_batch); xk / r hold the
        // batch's last iterate, so the cycle ends with x_k of its last step.
        int pend_n = 0, pend_slot0 = 0;
        auto flush = [&](int k_last) -> int {
            const int nb = pend_n, k0 = k_last - nb + 1;
            pend_n = 0;
            CTK_CUDA(cudaStreamWaitEvent(sb, ev_h[k_last - 1], 0));
            CTK_CUDA(cudaMemcpyAsync(bf->y_dev + (size_t)pend_slot0 * bf->rows,
                                     bf->y_host + (size_t)pend_slot0 * bf->rows,
                                     sizeof(double) * (size_t)bf->rows * nb, cudaMemcpyHostToDevice,
                                     sb));
            int r2 = ctk_iterate_batch(ab ? bf->aux1 : bf->W, ab ? bf->ld1 : bf->ld, bf->x_cur,
                                       bf->xk, n, ab ? bf->aux2 : bf->aux1, ab ? bf->ld2 : bf->ld1,
                                       bf->d0, bf->r, m, k0, nb,
                                       bf->y_dev + (size_t)pend_slot0 * bf->rows, bf->rows,
                                       bf->norms + 2 * (size_t)pend_slot0, bf->scratch_b,
                                       bf->rows + 2, bf->stream_b);
            if (r2) return r2;
            for (int q = 0; q < nb; ++q) CTK_CUDA(cudaEventRecord(ev_it[pend_slot0 + q], sb));
            return CTK_OK;
        };
        auto consume = [&](int k) -> int {
            auto& job = jobs[k];
            const auto tw0 = std::chrono::steady_clock::now();
            pool().wait(job);
            if (trace) {
                tr_wait += std::chrono::duration<double>(std::chrono::steady_clock::now() - tw0).count();
                tr_consumed_at = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            }
            if (job->rc) return job->rc;
            double lam = 0.0;
            int warn = 0;
            const double* y = job->y.data();
            double proj = job->out[1];
            std::vector<double> y2;
            if (cfg->hybrid) {
                if (job->out[2] != 0.0) {     // DegenerateCurveError -> previous lambda
                    lam = prev_lam;
                    warn = 1;
                    double o2[4];
                    y2.assign(k, 0.0);
                    int r2 = ctk_projected_solve(job->H.data(), k, beta, 1, lam, 200, NAN, o2,
                                                 y2.data());
                    if (r2) return r2;
                    y = y2.data();
                    proj = o2[1];
                } else {
                    lam = job->out[0];
                }
            }
            prev_lam = lam;
            const int slot = nrec;
            double* yh = bf->y_host + (size_t)slot * bf->rows;
            memcpy(yh, y, sizeof(double) * k);
            const bool batched = can_batch && ctk_iterate_batch_ok(k - pend_n, pend_n + 1,
                                                                   bf->rows + 2, n, m);
            if (!batched && pend_n > 0 && (rc = flush(k - 1))) return rc;
            if (batched) {
                if (pend_n == 0) pend_slot0 = slot;
                ++pend_n;
                if (pend_n == IB_BATCH || k == steps || k == broke_at) {
                    if ((rc = flush(k))) return rc;
                }
            } else {
                CTK_CUDA(cudaStreamWaitEvent(sb, ev_h[k - 1], 0));
                int r2 = ctk_iterate(g, ab, bf->W, bf->ld, k, yh, bf->y_dev + (size_t)slot * bf->rows,
                                     bf->x_cur, bf->xk, bf->z, bf->b, bf->r, bf->norms + 2 * slot,
                                     bf->aux1, bf->ld1, bf->aux2, bf->ld2, bf->d0,
                                     bf->stage_b, bf->back_b, bf->scratch_b, bf->stream_b);
                if (r2) return r2;
                if (bf->x_true) {       // device-side RRE / SSIM of x_k (row f1)
                    int r3 = ctk_metrics(bf->xk, bf->x_true, bf->img_nx, bf->img_ny, bf->dyn_range,
                                         bf->metrics + 2 * slot, bf->scratch_m, bf->stream_b);
                    if (r3) return r3;
                }
                if (bf->snapshot_stride > 0 && (slot + 1) % bf->snapshot_stride == 0) {
                    const int si = (slot + 1) / bf->snapshot_stride - 1;
                    if (si < bf->n_snaps)
                        CTK_CUDA(cudaMemcpyAsync(bf->snaps[si], bf->xk, sizeof(float) * n,
                                                 cudaMemcpyDeviceToHost, sb));
                }
                CTK_CUDA(cudaEventRecord(ev_it[slot], sb));
            }
            out->k[slot] = slot + 1;
            out->lambda[slot] = lam;
            out->proj_residual[slot] = proj;
            out->warn[slot] = warn;
            rec_slot.push_back(slot);
            nrec = slot + 1;
            if (cfg->stopping == CTK_STOP_DP || cfg->stopping == CTK_STOP_RNS) {
                if (comm) {
                    // sharded: this iterate's residual norm summed over ranks,
                    // on the Arnoldi stream -- every collective of the solve
                    // goes through one stream, in the same order on all ranks
                    CTK_CUDA(cudaStreamWaitEvent(sa, ev_it[slot], 0));
                    if ((rc = ctk_comm_sum_f64(comm, bf->norms + 2 * slot, 1, sa))) return rc;
                    CTK_CUDA(cudaMemcpyAsync(bf->norms_host + 2 * slot, bf->norms + 2 * slot,
                                             2 * sizeof(double), cudaMemcpyDeviceToHost, sa));
                    CTK_CUDA(cudaStreamSynchronize(sa));
                } else {
                    CTK_CUDA(cudaMemcpyAsync(bf->norms_host + 2 * slot, bf->norms + 2 * slot,
                                             2 * sizeof(double), cudaMemcpyDeviceToHost, sb));
                    CTK_CUDA(cudaStreamSynchronize(sb));
                }
                const double dn = sqrt(bf->norms_host[2 * slot]);
                history.push_back(dn);
                if (cfg->stopping == CTK_STOP_DP) {
                    if (dn <= cfg->dp_tau * cfg->noise_norm) stop = CTK_STOP_DP;
                } else if (history.size() >= 2) {
                    const double pv = history[history.size() - 2], cv = history.back();
                    if (pv == 0.0 || fabs(pv - cv) / pv < cfg->rns_epsilon) stop = CTK_STOP_RNS;
                }
            }
            if (broke_at == k && stop == CTK_STOP_NONE) stop = CTK_STOP_BREAKDOWN;
            return CTK_OK;
        };
        for (int j = 0; j < steps; ++j) {
            CTK_CUDA(cudaEventSynchronize(ev_h[j]));
            const double* hr = bf->h_host + (size_t)j * hc;
            const int k = j + 1;
            for (int i = 0; i <= k; ++i) Hfull[(size_t)i * steps + j] = hr[i];
            const bool broke = hr[hc - 3] != 0.0;
            auto job = std::make_shared<Job>();
            job->k = k;
            job->H.resize((size_t)(k + 1) * k);
            for (int i = 0; i <= k; ++i)
                memcpy(&job->H[(size_t)i * k], &Hfull[(size_t)i * steps], sizeof(double) * k);
            job->beta = beta;
            job->strategy = cfg->hybrid ? cfg->strategy : 0;
            job->value = cfg->lambda_value;
            jobs[k] = job;
            if (broke || k == steps) pool().run_inline(job);
            else pool().submit(job);
            if (broke) {
                broke_at = last_k = k;
            } else if ((rc = enqueue_to(k + look))) {
                return rc;
            }
            const bool sync_mode = cfg->stopping != CTK_STOP_NONE;
            while (stop == CTK_STOP_NONE && done_k + 1 <= k &&
                   (sync_mode || pool().ready(jobs[done_k + 1]))) {
                if ((rc = consume(++done_k))) return rc;
            }
            if (stop != CTK_STOP_NONE || broke) break;
        }
        while (stop == CTK_STOP_NONE && done_k < last_k && jobs[done_k + 1]) {
            if ((rc = consume(++done_k))) return rc;
        }
        if (stop == CTK_STOP_NONE && broke_at > 0) stop = CTK_STOP_BREAKDOWN;
    }
    if (comm && cfg->stopping == CTK_STOP_NONE) {
        // every rank's residual norms are partial sums over its rows; the
        // image norms are replicated (kept from rank 0 only).  On the Arnoldi
        // stream, after the iterate stream: one stream for all collectives.
        CTK_CUDA(cudaEventRecord(ev_sync, sb));
        CTK_CUDA(cudaStreamWaitEvent(sa, ev_sync, 0));
        if (ctk_comm_rank_of(comm) != 0) {
            k_zero_odd<<<(K + 1 + 127) / 128, 128, 0, sa>>>(bf->norms, K + 1);
            ctk_count_launch();
        }
        if ((rc = ctk_comm_sum_f64(comm, bf->norms, 2 * (int64_t)(K + 1), sa))) return rc;
    }
    CTK_CUDA(cudaStreamSynchronize(sa));
    CTK_CUDA(cudaStreamSynchronize(sb));
    if (comm && (rc = ctk_comm_check(comm))) return rc;
    CTK_CUDA(cudaMemcpy(bf->norms_host, bf->norms, sizeof(double) * 2 * (K + 1),
                        cudaMemcpyDeviceToHost));
    if (bf->x_true)
        CTK_CUDA(cudaMemcpy(bf->metrics_host, bf->metrics, sizeof(double) * 2 * (K + 1),
                            cudaMemcpyDeviceToHost));
    for (int i = 0; i < nrec; ++i) {
        if (out->rre) {
            out->rre[i] = bf->x_true && rec_slot[i] >= 0 ? bf->metrics_host[2 * i] : NAN;
            out->ssim[i] = bf->x_true && rec_slot[i] >= 0 ? bf->metrics_host[2 * i + 1] : NAN;
        }
        if (rec_slot[i] < 0) continue;
        const double dn = sqrt(bf->norms_host[2 * i]);
        out->data_residual[i] = dn;
        out->solution_norm[i] = sqrt(bf->norms_host[2 * i + 1]);
        out->residual[i] = ab ? dn : out->proj_residual[i];
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ev_start, ev_it[i]);
        out->elapsed[i] = ms / 1000.0;
    }
    if (trace && cycles == 1) {
        // per step: GPU busy (begin -> h event) and idle gap before the next step
        double busy = 0.0, gap = 0.0;
        const int nst = nrec < rows - 1 ? nrec : rows - 1;
        for (int j = 0; j < nst; ++j) {
            float b_ms = 0.f, g_ms = 0.f;
            cudaEventElapsedTime(&b_ms, tr_beg[j], ev_h[j]);
            busy += b_ms;
            if (j + 1 < nst) {
                cudaEventElapsedTime(&g_ms, ev_h[j], tr_beg[j + 1]);
                gap += g_ms;
            }
        }
        cudaGetLastError();
        fprintf(stderr, "[ctk trace] %d steps: stream-A busy %.3f ms, idle %.3f ms; host enqueue of last step at %.3f ms; "
                "host waited %.3f ms on projected solves, last consumed at %.3f ms\n",
                nst, busy, gap, nst > 0 ? 1e3 * tr_host[nst - 1] : 0.0, 1e3 * tr_wait, 1e3 * tr_consumed_at);
    }
    out->n_records = nrec;
    out->cycles = cycles > 0 ? cycles : 1;
    out->stop_reason = stop == CTK_STOP_NONE ? CTK_STOP_MAXITER : stop;
    return CTK_OK;
}
