// solver.cu — host driver of the lpsg dense revised simplex and its C ABI.
//
// The iteration loop of lps::SimplexSolver (solver.cpp:278-293) runs on the
// device as a fused four-kernel chain per pivot:
//
//     k_ratio  -> k_pivot -> k_price(W_{t+1}) -> k_update(T_t -> T_{t+1}, Y_{t+1})
//
// Every decision (entering column, leaving row, optimality, unboundedness, the
// iteration budget) is taken on the device and recorded in the control block,
// so the host enqueues batches of pivots and only synchronises once per batch
// to drain the pivot log (note_iteration's tabu bookkeeping and the observer).
// Ratio-test ties under the tabu rule (select_leaving, solver.cpp:215-238) stop
// the device chain; the host applies the tabu filter and scores the survivors
// with the batched device lookahead, then resumes.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <thread>
#include <type_traits>
#include <unordered_set>
#include <vector>

#include "comm.h"
#include "device.cuh"
#include "lpsg.h"

namespace lpsg {

namespace {
thread_local std::string g_err;

struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& w) : std::runtime_error(w), code(c) {}
};

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        const int code = e == cudaErrorMemoryAllocation ? LPSG_OUT_OF_MEMORY : LPSG_CUDA_ERROR;
        cudaGetLastError();
        throw Error(code, std::string(what) + ": " + cudaGetErrorString(e));
    }
}
#define CK(x) ck((x), #x)
#define CK_SET_DEVICE(dev) ::lpsg::ck(cudaSetDevice(dev), "cudaSetDevice")

template <class T>
T* dalloc(size_t n) {
    void* p = nullptr;
    CK(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)));
    return static_cast<T*>(p);
}

// Stream-ordered temporaries: cudaMalloc/cudaFree may synchronise the whole
// device, which would deadlock against another shard's spin-waiting exchange
// kernel when shards share a GPU.
template <class T>
T* talloc(size_t n, cudaStream_t st, cudaMemPool_t pool) {
    void* p = nullptr;
    CK(cudaMallocFromPoolAsync(&p, std::max<size_t>(n, 1) * sizeof(T), pool, st));
    return static_cast<T*>(p);
}

double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

long long round_up(long long v, long long a) { return (v + a - 1) / a * a; }

// select_leaving tries the bounded selection (k_la_probe*) from this many
// survivors up; smaller ties are cheap to score in full.
constexpr int kLaBoundMin = 16;

// The lookahead GEMMs encode their TMA descriptors per batch (the operand
// buffers are stream-ordered temporaries).
void la_ok(bool ok) {
    if (!ok) throw Error(LPSG_CUDA_ERROR, "lookahead: cuTensorMapEncodeTiled failed");
}

// Two timing events, destroyed on every exit (the throwing ones included).
struct EventPair {
    cudaEvent_t a = nullptr, b = nullptr;
    EventPair() {
        CK(cudaEventCreate(&a));
        CK(cudaEventCreate(&b));
    }
    ~EventPair() {
        if (a) cudaEventDestroy(a);
        if (b) cudaEventDestroy(b);
    }
    EventPair(const EventPair&) = delete;
    EventPair& operator=(const EventPair&) = delete;
};

// Owns one device allocation until released (staging buffers freed on throw).
struct DevBuf {
    void* p = nullptr;
    ~DevBuf() {
        if (p) cudaFree(p);
    }
};

// The LP's row-major A (host) -> column-major A_cm (n columns of pitch ld) on
// the current device, in row blocks of <= 128 MB through one staging buffer,
// so the upload never holds a second full-size copy of A in HBM (9.2 GB at
// C5). Throws LPSG_INVALID_ARGUMENT when A holds an inf/NaN (SURVEY.md
// Appendix A.8), after the upload has been drained.
void upload_A_cm(const lpsg_problem& lp, double* A_cm, long long ld, cudaStream_t st) {
    const int m = lp.m, n = lp.n_total;
    const long long chunk_el = 16LL << 20;  // 128 MB of doubles
    const int rows = (int)std::max<long long>(32, std::min<long long>(m, chunk_el / std::max(1, n) / 32 * 32));
    DevBuf stage, flag;
    CK(cudaMalloc(&stage.p, sizeof(double) * (size_t)rows * n));
    CK(cudaMalloc(&flag.p, sizeof(int)));
    int* nonfinite = static_cast<int*>(flag.p);
    CK(cudaMemsetAsync(nonfinite, 0, sizeof(int), st));
    CK(cudaMemsetAsync(A_cm, 0, sizeof(double) * ((size_t)n * ld + 64), st));
    for (int i0 = 0; i0 < m; i0 += rows) {
        const int nr = std::min(rows, m - i0);
        CK(cudaMemcpyAsync(stage.p, lp.A + (size_t)i0 * n, sizeof(double) * (size_t)nr * n,
                           cudaMemcpyHostToDevice, st));
        launch_transpose(static_cast<const double*>(stage.p), A_cm + i0, nr, n, ld, nonfinite, st);
        CK(cudaGetLastError());
    }
    int bad = 0;
    CK(cudaMemcpyAsync(&bad, nonfinite, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (bad)
        throw Error(LPSG_INVALID_ARGUMENT,
                    "A holds an inf/NaN coefficient: reduced costs would not be finite, and the "
                    "reference's first-scanned-column pricing rule is not reproduced for them");
}
}  // namespace

class Solver {
public:
    // comm == nullptr: single GPU. Otherwise this object is shard comm->rank of
    // comm->size; every rank must make the same calls.
    // shared_A_cm: a column-major A (upload_A_cm, pitch round_up(m, 4)) owned by
    // the caller and shared by the in-process shards of one device (read-only)
    Solver(const lpsg_problem& lp, const lpsg_config& cfg, Comm* comm = nullptr,
           double* shared_A_cm = nullptr);
    ~Solver();

    void solve(lpsg_report* rep);
    void get_x(double* x, int n);

    // step API (solver.hpp:79-168)
    void step_price(int* optimal, int* entering, double* red);
    void step_compute_direction(int entering, double red);
    void step_ratio(int* unbounded, double* theta, std::vector<int>& cand);
    int select_leaving(const std::vector<int>& cand, int entering);
    // first_proven != nullptr: select_leaving's bounded path may settle the
    // choice (then *first_proven = true and `scores` is not filled)
    void lookahead(const std::vector<int>& rows, int entering, std::vector<double>& scores,
                   bool* first_proven = nullptr);
    long long la_bounded_ = 0, la_full_ = 0;  // select_leaving lookaheads: settled by the probe / fully scored
    long long la_price_bounded_ = 0, la_price_exact_ = 0;  // lookahead pricings: DMMA screen held / exact GEMM rerun
    long long la_probe_rounds_ = 0;  // bounded selections that needed the exact probe rounds
    int la_bound_min_ = 16;                   // survivors from which the probe / bounded pricing are used
    double* anorm_ = nullptr;                 // ||a_j||_2 of A's columns (bounded pricing), made on first use
    unsigned char* la_arena_ = nullptr;       // lookahead buffers, kept across ties (pool memory)
    size_t la_arena_bytes_ = 0;
    void step_pivot(int r, int q);
    void read_row(int i, double* out);

    int m() const { return m_; }
    int n_total() const { return n_total_; }
    int n_work() const { return n_work_; }
    int phase() const { return phase_; }
    const Dev& dev() const { return d_; }
    const std::vector<int>& basic() const { return basic_; }

    lpsg_observer observer = nullptr;
    void* observer_user = nullptr;
    // SolverConfig::observer with the whole IterationView (solver.hpp:21-32)
    lpsg_view_observer view_observer = nullptr;
    void* view_user = nullptr;
    bool view_rows = false;      // the callback may read tableau rows: unfused, one pivot per round trip
    lpsg_solver* handle = nullptr;  // the C handle, for lpsg_read_row from inside the callback
    lpsg_memory memory() const;
    bool keep_trace = false;
    std::vector<lpsg_trace> trace;

private:
    void init(const lpsg_problem& lp);
    void release();
    int run_phase();
    int run_phase_stepwise();
    int handle_stop(int st, bool* resumed);
    void enter_phase2();
    void drive_out_artificials();
    void rebuild_top_row();
    void pull(bool with_log);
    void push();
    void drain_log();
    void snapshot();
    void note_pivot(const LogEntry& e);
    void enqueue_pivots(int n);
    long long room_ = 0;  // pivots the device budget still allows (run_phase)
    void seq_pivot();
    void seq_price();
    void seq_update();
    std::vector<int> gather_overflow_candidates();
    void single_gpu_only(const char* what) const;
    int owner_of_row(int i) const;
    void temp_alloc_fence();
    double objective_value();

    lpsg_config cfg_;
    int m_, n_total_, n_art_ = 0, n_work_ = 0;
    long long max_iter_ = 0;
    int phase_ = 1;
    long long total_iter_ = 0, phase_iter_[2] = {0, 0};
    std::vector<int> basic_;
    std::vector<char> frozen_;
    std::unordered_map<int, std::unordered_set<int>> banned_;  // TabuState (solver.hpp:66-69)
    double last_objective_ = 0.0;
    int final_status_ = LPSG_ITERATION_LIMIT;
    bool solved_ = false;
    bool done_ = false;        // terminal status reached (not resumable)
    long long n_scan_host_ = 0;

    cudaStream_t st_ = nullptr;
    Dev d_{};
    Ctl* hctl_ = nullptr;       // pinned mirror of the control block
    LogEntry* hlog_ = nullptr;  // pinned mirror of the pivot log (a ring of log_cap entries)
    long long log_seen_ = 0;    // log entries already drained
    cudaEvent_t ev_snap_ = nullptr;
    cudaMemPool_t pool_ = nullptr;  // stream-ordered temporaries
    int* hone_ = nullptr;       // pinned constant 1 (stream-ordered flag writes)
    double* scratch_ = nullptr;
    double* cost_buf_ = nullptr;
    CUtensorMap* tmaps_ = nullptr;
    int n_tmaps_ = 0;
    int batch_ = 16;
    bool unfused_ratio_ = false;  // debug knob (cfg.reserved[0] & 1): standalone ratio kernel
    Comm* comm_ = nullptr;
    double* shared_A_cm_ = nullptr;  // not owned (lpsg_solve_sharded)
    bool sharded_ = false;        // comm_ attached: the exchange path runs even for one rank
    bool dbg_trace_ = getenv("LPSG_TRACE_COMM") != nullptr;
    int world_ = 1, rank_ = 0;
    double* chain_ = nullptr;     // world > 1: rebuild_top_row partial sums (m+1)
    // opt-in reinversion (lpsg_config.reinvert_every, csrc/reinvert.cu)
    long long reinv_every_ = 0;
    long long reinv_at_ = -1;       // total_iter_ of the last rebuild (-1: none yet)
    double* b0_ = nullptr;          // the LP's b (device), for b_bar = B^-1 b
    int* art_row_ = nullptr;        // artificial n_total + k is the unit column of row art_row_[k]
    std::vector<int> art_row_host_;
    int run_phase_any();
    void reinvert();

    // ---- Case 2: out-of-core tiling (tiled_engine.cpp:29-54, 165-184, 246-263)
    struct Part {
        int row0, rows;    // rows [row0, row0 + rows) of [B^-1 | b_bar]
        double* host;      // page-locked, column-major, pitch `rows`
    };
    bool tiled_ = false;
    std::vector<Part> parts_;
    int resident_ = -1;          // the partition in the device slab d_.T (-1: none)
    RatioMsg* part_msgs_ = nullptr;
    int* part_row0_ = nullptr;
    double* xbuf_own_ = nullptr;  // Case 2: the pivot-row buffer (sharded runs use the comm heap)
    double* host_T_ = nullptr;    // Case 2: page-locked rows of [B^-1 | b_bar], partition p at row0 * (m+1)
    void plan_tiles(int m, int n);
    Dev part_dev(int p) const;
    int part_of_row(int i) const;
    void ensure_resident(int p);
    void tiled_pass();
    void tiled_pivot();
    int run_phase_tiled();
    void gather_row_any(int i, double* out);
    int rows_local() const { return tiled_ ? m_ : d_.mloc; }

public:
    long reinv_count = 0, reinv_steps = 0;
    double reinv_res_before = 0.0, reinv_res_after = 0.0, reinv_seconds = 0.0;

private:

public:
    // ---- counters and optional per-kernel CUDA-event profile
    // K_LA_*: the batched tie-break lookahead; their "bytes" are fp64 flops
    // (2 per multiply-add of the batched dots)
    enum Kind { K_RATIO = 0, K_PIVOT, K_PRICE, K_UPDATE, K_OTHER, K_COMM, K_LA_PRICE, K_LA_THETA, K_NUM };
    struct KStat {
        long launches = 0;
        double ms = 0.0;
        double bytes = 0.0;
    };
    KStat kstat[K_NUM];
    long launches_total = 0;
    double last_device_ms = 0.0;   // CUDA-event span of the last solve() on the solver stream
    long long h2d_bytes = 0, d2h_bytes = 0;
    double dev_read_bytes = 0.0, dev_write_bytes = 0.0;  // algorithmic, per pivot done (lpsg_memory)
    void set_profile(bool on);
    void set_max_iter(long long v);

private:
    bool prof_ = false;
    unsigned long long work_seen_[4] = {0, 0, 0, 0};
    std::vector<cudaEvent_t> ev_pool_;
    struct EvRec {
        int kind;
        cudaEvent_t a, b;
        double bytes;
    };
    std::vector<EvRec> ev_used_;
    cudaEvent_t ev_chain_ = nullptr;  // last boundary event, reusable as the next start
    template <class F>
    void L(int kind, double bytes, F&& f);
    void flush_profile();
    double bytes_of(int kind) const;
};

template <class F>
void Solver::L(int kind, double bytes, F&& f) {
    ++launches_total;
    if (!prof_) {
        f();
        return;
    }
    if (ev_pool_.size() < 2) {
        for (int k = 0; k < 64; ++k) {
            cudaEvent_t e;
            CK(cudaEventCreate(&e));
            ev_pool_.push_back(e);
        }
    }
    // One event per kernel boundary: the previous kernel's end event is this
    // kernel's start event unless another stream operation came in between.
    cudaEvent_t a;
    if (ev_chain_) {
        a = ev_chain_;
    } else {
        a = ev_pool_.back();
        ev_pool_.pop_back();
        CK(cudaEventRecord(a, st_));
    }
    f();
    cudaEvent_t b = ev_pool_.back();
    ev_pool_.pop_back();
    CK(cudaEventRecord(b, st_));
    ev_used_.push_back(EvRec{kind, a, b, bytes});
    ev_chain_ = b;
}

// Algorithmic bytes are credited per launch that did its work (ctl.work
// counters), not per launch: the kernels enqueued behind a stop (budget,
// optimality, a tie) exit at once and move nothing.
void Solver::flush_profile() {
    std::vector<cudaEvent_t> seen;
    const int widx[K_NUM] = {-1, 2, 0, 1, -1, -1, -1, -1};
    for (int k = 0; k < K_NUM; ++k) {
        if (widx[k] < 0) continue;
        const unsigned long long w = hctl_->work[widx[k]];
        kstat[k].bytes += (double)(w - work_seen_[widx[k]]) * bytes_of(k);
        work_seen_[widx[k]] = w;
    }
    for (auto& r : ev_used_) {
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, r.a, r.b));
        kstat[r.kind].launches += 1;
        kstat[r.kind].ms += ms;
        if (r.kind != K_PRICE && r.kind != K_UPDATE && r.kind != K_PIVOT) kstat[r.kind].bytes += r.bytes;
        seen.push_back(r.a);
        seen.push_back(r.b);
    }
    std::sort(seen.begin(), seen.end());
    seen.erase(std::unique(seen.begin(), seen.end()), seen.end());
    for (cudaEvent_t e : seen) ev_pool_.push_back(e);
    ev_used_.clear();
    ev_chain_ = nullptr;
}

// Algorithmic HBM bytes per launch: what the reference's step
// must touch, not what the kernel happens to move.
double Solver::bytes_of(int kind) const {
    const double m = m_;
    switch (kind) {
        case K_PRICE: return 8.0 * m * (double)n_scan_host_ + 8.0 * m;       // A_nb slots + W
        case K_UPDATE: return 16.0 * d_.mloc * (m + 1.0) + 16.0 * d_.mloc;   // T read+write, y, a_q
        case K_RATIO: return 16.0 * d_.mloc;                                 // y, b_bar
        case K_PIVOT: return 8.0 * (m + 1.0) * 3.0 + 16.0 * m;               // row r, x, W; slot copy
        default: return 0.0;
    }
}

void Solver::set_profile(bool on) {
    prof_ = on;
    for (auto& k : kstat) k = KStat{};
    for (int k = 0; k < 4; ++k) work_seen_[k] = hctl_->work[k];
}

void Solver::set_max_iter(long long v) {
    max_iter_ = v > 0 ? v : 50LL * (m_ + n_work_);
    hctl_->budget = max_iter_;
    push();
    CK(cudaStreamSynchronize(st_));
}

// A constructor that throws never runs ~Solver, so everything init() acquired
// is released here before the exception leaves (lpsg_create then reports it).
Solver::Solver(const lpsg_problem& lp, const lpsg_config& cfg, Comm* comm, double* shared_A_cm)
    : cfg_(cfg), m_(lp.m), n_total_(lp.n_total), comm_(comm), shared_A_cm_(shared_A_cm) {
    try {
        init(lp);
    } catch (...) {
        release();
        throw;
    }
}

void Solver::init(const lpsg_problem& lp) {
    const lpsg_config& cfg = cfg_;
    if (comm_) {
        sharded_ = true;
        world_ = comm_->size;
        rank_ = comm_->rank;
    }
    if (lp.m <= 0 || lp.n_total <= 0)
        throw Error(LPSG_EMPTY_PROBLEM, "lpsg_create: problem has no rows or no columns");
    if (!lp.A || !lp.b || !lp.c || !lp.col_kind)
        throw Error(LPSG_INVALID_ARGUMENT, "lpsg_create: null problem array");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= 0) {
        cudaGetLastError();
        throw Error(LPSG_CUDA_ERROR, "lpsg_create: no CUDA device available (the solver has no CPU fallback)");
    }
    if (cfg.device < 0 || cfg.device >= ndev) throw Error(LPSG_INVALID_ARGUMENT, "lpsg_create: bad device ordinal");
    if (world_ > lp.m || world_ > 32)
        throw Error(LPSG_INVALID_ARGUMENT, "lpsg_create: more shards than rows (or than 32)");
    CK(cudaSetDevice(cfg.device));
    CK(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking));
    {
        // Stream-ordered temporaries (lookahead batches, overflow gathers) come
        // from this solver's own pool, which keeps freed blocks cached. Its own
        // pool, not the device default: shards of one process must not reuse each
        // other's freed blocks, which would order one shard's stream behind
        // another's (a deadlock against spin-waiting exchange kernels).
        cudaMemPoolProps props = {};
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = cfg.device;
        CK(cudaMemPoolCreate(&pool_, &props));
        uint64_t keep = UINT64_MAX;
        CK(cudaMemPoolSetAttribute(pool_, cudaMemPoolAttrReleaseThreshold, &keep));
    }
    const int m = m_, n = n_total_;

    // ---- start basis (solver.cpp:27-39): first row i (ascending) with A[i][j] == 1.0
    // for each slack column j (ascending), skipping rows already taken.
    basic_.assign(m, -1);
    {
        std::vector<int> slack_cols;
        for (int j = 0; j < n; ++j)
            if (lp.col_kind[j] == LPSG_COL_SLACK) slack_cols.push_back(j);
        if (!slack_cols.empty()) {
            std::vector<std::vector<int>> ones(slack_cols.size());
            for (int i = 0; i < m; ++i) {
                const double* row = lp.A + (size_t)i * n;
                for (size_t k = 0; k < slack_cols.size(); ++k)
                    if (row[slack_cols[k]] == 1.0) ones[k].push_back(i);
            }
            for (size_t k = 0; k < slack_cols.size(); ++k)
                for (int i : ones[k])
                    if (basic_[i] < 0) {
                        basic_[i] = slack_cols[k];
                        break;
                    }
        }
    }
    for (int i = 0; i < m; ++i)
        if (basic_[i] < 0) ++n_art_;
    n_work_ = n + n_art_;
    std::vector<double> cost(2 * (size_t)n_work_, 0.0);  // [c_phase1 | c_true]
    for (int j = 0; j < n; ++j) {
        if (!std::isfinite(lp.c[j]))  // see the A check below
            throw Error(LPSG_INVALID_ARGUMENT, "c holds an inf/NaN cost: reduced costs would not be finite");
        cost[n_work_ + j] = lp.c[j];
    }
    {
        int next = n;
        for (int i = 0; i < m; ++i) {
            if (basic_[i] >= 0) continue;
            cost[next] = 1.0;  // c_phase1 of the artificial (solver.cpp:56)
            art_row_host_.push_back(i);
            basic_[i] = next++;
        }
    }
    frozen_.assign(m, 0);
    max_iter_ = cfg_.max_iter > 0 ? cfg_.max_iter : 50LL * (m + n_work_);
    phase_ = n_art_ > 0 ? 1 : 2;

    // ---- device layout
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, cfg.device));
    d_.m = m;
    d_.n_total = n;
    d_.n_work = n_work_;
    // shard geometry: contiguous row blocks of T, contiguous
    // original-column blocks for pricing
    d_.world = world_;
    d_.rank = rank_;
    d_.sharded = sharded_ ? 1 : 0;
    {
        int r1 = 0;
        lpsg_shard_range(m, world_, rank_, &d_.row0, &r1);
        d_.mloc = r1 - d_.row0;
        lpsg_shard_range(n, world_, rank_, &d_.col0, &d_.col1);
    }
    d_.ld_nb = round_up(std::max(1, d_.col1 - d_.col0), 32) + 32;
    d_.ld_cm = round_up(m, 4);
    d_.num_sms = prop.multiProcessorCount;
    d_.opt_tol = cfg_.opt_tol;
    d_.pivot_tol = cfg_.pivot_tol;
    d_.feas_tol = cfg_.feas_tol;
    d_.ratio_tie_tol = cfg_.ratio_tie_tol;
    d_.anticycle = cfg_.anticycle;
    if (cfg_.kernel != 0 && cfg_.kernel != 1) throw Error(LPSG_INVALID_ARGUMENT, "lpsg_create: kernel must be 0 (cached) or 1 (naive)");
    if (cfg_.reinvert_every < 0) throw Error(LPSG_INVALID_ARGUMENT, "lpsg_create: reinvert_every must be >= 0");
    if (cfg_.reinvert_every > 0 && sharded_)
        throw Error(LPSG_INVALID_ARGUMENT, "lpsg_create: reinversion is single-GPU only");
    reinv_every_ = cfg_.reinvert_every;
    d_.naive = cfg_.kernel == 1 ? 1 : 0;
    d_.dbg = cfg_.reserved[2] & ~(kLookaheadExactBit | kLookaheadBoundAllBit | kLookaheadBoundOffBit);
    d_.la_exact = (cfg_.reserved[2] & kLookaheadExactBit) != 0;  // (dbg: -DLPSG_EXPERIMENTS only)
    la_bound_min_ = (cfg_.reserved[2] & kLookaheadBoundOffBit) ? INT_MAX
                    : (cfg_.reserved[2] & kLookaheadBoundAllBit) ? 2 : kLaBoundMin;
    // PDL hides kernel-boundary latency; it pays up to m ~ 10^4 (C1 +21 %, C3
    // +1.4 %) and was measured to cost ~17 % at m = 24000, where the boundaries
    // are noise against 3 ms pivots
    plan_tiles(m, n);
    d_.pdl = (!comm_ && !tiled_ && m <= 12000 && xp_env("LPSG_NO_PDL") == nullptr) ? 1 : 0;
    d_.upd_tma_store = xp_env("LPSG_UPD_STG") == nullptr ? 1 : 0;
    d_.price_pf = xp_env("LPSG_PRICE_PF") ? atoi(xp_env("LPSG_PRICE_PF")) : 8;
    d_.l2_hint = xp_env("LPSG_NO_L2_HINT") == nullptr ? 1 : 0;
    configure_kernels(d_);
    CK(cudaGetLastError());
    d_.ldT = round_up(std::max<long long>(d_.mloc + 1, (long long)d_.update_grid * d_.upd_h), 32);
    unfused_ratio_ = !sharded_ && (cfg_.reserved[0] & 1) != 0;  // standalone k_ratio (result-identical)
    batch_ = cfg_.batch > 0 ? cfg_.batch : (m <= 1024 ? 64 : m <= 4096 ? 16 : 4);
    d_.log_cap = 2 * batch_ + 8;  // ring: the drained batch + the one in flight

    d_.T = dalloc<double>((size_t)(m + 1) * d_.ldT + 64);
    d_.top = dalloc<double>(m + 520);  // + padding: TMA-side W segments may run past m+2
    d_.Y = dalloc<double>(rows_local());
    d_.xrow = dalloc<double>(m + 4);
    if (tiled_) {
        xbuf_own_ = dalloc<double>(m + 4);
        d_.xbuf = xbuf_own_;
        part_msgs_ = dalloc<RatioMsg>(parts_.size());
        part_row0_ = dalloc<int>(parts_.size());
        chain_ = dalloc<double>(m + 1);
        std::vector<int> r0;
        for (const Part& q : parts_) r0.push_back(q.row0);
        CK(cudaMemcpy(part_row0_, r0.data(), sizeof(int) * r0.size(), cudaMemcpyHostToDevice));
        // one page-locked block for every partition (a tiny budget can mean
        // thousands of partitions; one allocation each would be slow)
        CK(cudaMallocHost(&host_T_, sizeof(double) * (size_t)m * (m + 1)));
        for (Part& q : parts_) q.host = host_T_ + (size_t)q.row0 * (m + 1);
    }
    if (sharded_) {
        d_.xbuf = static_cast<double*>(comm_->sym_alloc(sizeof(double) * (m + 4)));
        d_.xbuf_zero = std::strcmp(comm_->transport(), "p2p") != 0;
        d_.pmsg = dalloc<PriceMsg>(world_ + 1);
        d_.rmsg = dalloc<RatioMsg>(world_ + 1);
        chain_ = dalloc<double>(m + 1);
    }
    double* A_cm = shared_A_cm_ ? shared_A_cm_ : dalloc<double>((size_t)n * d_.ld_cm + 64);
    d_.A_cm = A_cm;
    d_.A_nb = dalloc<double>((size_t)m * d_.ld_nb + 64);
    d_.slot2col = dalloc<int>(d_.ld_nb);
    d_.col2slot = dalloc<int>(n);
    d_.basic = dalloc<int>(m);
    d_.frozen = dalloc<unsigned char>(m);
    cost_buf_ = dalloc<double>(2 * (size_t)n_work_);
    d_.cost_p1 = cost_buf_;
    d_.cost_true = cost_buf_ + n_work_;
    d_.ctl = dalloc<Ctl>(1);
    d_.cand = dalloc<int>(m);
    d_.cand_ratio = dalloc<double>(m);
    d_.pz = dalloc<double>(d_.price_grid);
    d_.pj = dalloc<int>(d_.price_grid);
    d_.log = dalloc<LogEntry>(d_.log_cap);
    d_.rc_theta = dalloc<double>(d_.update_grid);
    d_.rc_cnt = dalloc<int>(d_.update_grid);
    d_.rc_row = dalloc<int>((size_t)d_.update_grid * d_.upd_h);
    d_.rc_ratio = dalloc<double>((size_t)d_.update_grid * d_.upd_h);
    scratch_ = dalloc<double>(m + 4);
    if (!create_tensor_maps(d_, &tmaps_, &n_tmaps_))
        throw Error(LPSG_CUDA_ERROR, "lpsg_create: cuTensorMapEncodeTiled failed");
    CK(cudaMallocHost(&hctl_, sizeof(Ctl)));
    CK(cudaMallocHost(&hlog_, sizeof(LogEntry) * d_.log_cap));
    CK(cudaMallocHost(&hone_, sizeof(int)));
    CK(cudaEventCreateWithFlags(&ev_snap_, cudaEventDisableTiming));
    *hone_ = 1;

    // ---- upload A once (row-major), derive the column-major copy and the
    // nonbasic pricing matrix, then drop the staging copy.
    std::vector<char> in_basis(n_work_, 0);
    for (int i = 0; i < m; ++i) in_basis[basic_[i]] = 1;
    std::vector<int> slot2col, col2slot(n, -1);
    for (int j = d_.col0; j < d_.col1; ++j)
        if (!in_basis[j]) {
            col2slot[j] = (int)slot2col.size();
            slot2col.push_back(j);
        }
    const int n_scan = (int)slot2col.size();
    n_scan_host_ = n_scan;
    CK(cudaMemsetAsync(d_.slot2col, 0xff, sizeof(int) * d_.ld_nb, st_));
    if (n_scan)
        CK(cudaMemcpyAsync(d_.slot2col, slot2col.data(), sizeof(int) * n_scan, cudaMemcpyHostToDevice, st_));
    CK(cudaMemcpyAsync(d_.col2slot, col2slot.data(), sizeof(int) * n, cudaMemcpyHostToDevice, st_));
    if (!shared_A_cm_) upload_A_cm(lp, A_cm, d_.ld_cm, st_);
    CK(cudaMemsetAsync(d_.A_nb, 0, sizeof(double) * ((size_t)m * d_.ld_nb + 64), st_));
    launch_build_nb_from_cm(d_, n_scan, st_);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(d_.basic, basic_.data(), sizeof(int) * m, cudaMemcpyHostToDevice, st_));
    CK(cudaMemsetAsync(d_.frozen, 0, m, st_));
    CK(cudaMemcpyAsync(cost_buf_, cost.data(), sizeof(double) * cost.size(), cudaMemcpyHostToDevice, st_));
    CK(cudaMemsetAsync(d_.Y, 0, sizeof(double) * rows_local(), st_));
    CK(cudaMemsetAsync(d_.top, 0, sizeof(double) * (m + 520), st_));

    // ---- initial Figure-1 tableau B = I, b_bar = b (solver.cpp:66-72)
    CK(cudaMemsetAsync(d_.T, 0, sizeof(double) * (size_t)(m + 1) * d_.ldT, st_));
    if (sharded_) {
        // the sharded pivot row travels in xbuf; k_update reads it as xrow
        CK(cudaFree(d_.xrow));
        d_.xrow = d_.xbuf;
        CK(cudaMemsetAsync(d_.xbuf, 0, sizeof(double) * (m + 4), st_));
        CK(cudaMemsetAsync(d_.rmsg, 0, sizeof(RatioMsg) * (world_ + 1), st_));
    }
    CK(cudaMemcpyAsync(scratch_, lp.b, sizeof(double) * m, cudaMemcpyHostToDevice, st_));
    if (tiled_) {
        // Case 2: the tableau rows start host-side (begin_solve leaves them
        // there, tiled_engine.cpp:142-149): B^-1 = I, b_bar = b per partition
        CK(cudaFree(d_.xrow));
        d_.xrow = d_.xbuf;
        CK(cudaMemsetAsync(d_.xbuf, 0, sizeof(double) * (m + 4), st_));
        CK(cudaMemsetAsync(part_msgs_, 0, sizeof(RatioMsg) * parts_.size(), st_));
        for (Part& q : parts_) {
            std::memset(q.host, 0, sizeof(double) * (size_t)q.rows * (m + 1));
            for (int li = 0; li < q.rows; ++li) {
                q.host[(size_t)(q.row0 + li) * q.rows + li] = 1.0;
                q.host[(size_t)m * q.rows + li] = lp.b[q.row0 + li];
            }
        }
        resident_ = -1;
    } else {
        launch_init_tableau(d_, scratch_, st_);
    }
    if (reinv_every_ > 0) {
        b0_ = dalloc<double>(m);
        CK(cudaMemcpyAsync(b0_, lp.b, sizeof(double) * m, cudaMemcpyHostToDevice, st_));
        art_row_ = dalloc<int>(std::max<size_t>(1, art_row_host_.size()));
        if (!art_row_host_.empty())
            CK(cudaMemcpyAsync(art_row_, art_row_host_.data(), sizeof(int) * art_row_host_.size(),
                               cudaMemcpyHostToDevice, st_));
        CK(cudaStreamSynchronize(st_));  // art_row_host_ is host-pageable
    }

    h2d_bytes += 8LL * m * n + 8LL * m + 8LL * (long long)cost.size() + 4LL * (n_scan + n + m);
    std::memset(hctl_, 0, sizeof(Ctl));
    hctl_->status = ST_HOLD;
    hctl_->q = -1;
    hctl_->r = -1;
    hctl_->n_scan = n_scan;
    hctl_->budget = max_iter_;
    hctl_->phase = phase_;
    hctl_->upd_r = -1;
    hctl_->found = INT_MAX;
    push();
    // shards sharing a process finish their (device-synchronising) setup before
    // any of them starts spinning in an exchange
    if (comm_) {
        CK(cudaStreamSynchronize(st_));
        comm_->host_barrier();
    }
    rebuild_top_row();
    last_objective_ = objective_value();
}

Solver::~Solver() { release(); }

void Solver::release() {
    if (la_arena_ && st_) cudaFreeAsync(la_arena_, st_);
    if (st_) cudaStreamSynchronize(st_);
    if (sharded_ && d_.xbuf) {
        comm_->sym_free(d_.xbuf);
        if (d_.xrow == d_.xbuf) d_.xrow = nullptr;
    }
    if (xbuf_own_ && d_.xrow == xbuf_own_) d_.xrow = nullptr;
    void* bufs[] = {d_.T, d_.top, d_.Y, d_.xrow, shared_A_cm_ ? nullptr : (void*)d_.A_cm, d_.A_nb, d_.slot2col, d_.col2slot,
                    d_.basic, d_.frozen, cost_buf_, d_.ctl, d_.cand, d_.pz, d_.pj, d_.log, scratch_, tmaps_,
                    d_.rc_theta, d_.rc_cnt, d_.rc_row, d_.rc_ratio, d_.cand_ratio, d_.pmsg, d_.rmsg,
                    chain_, b0_, art_row_, part_msgs_, part_row0_, xbuf_own_, anorm_};
    for (void* p : bufs)
        if (p) cudaFree(p);
    if (host_T_) cudaFreeHost(host_T_);
    host_T_ = nullptr;
    parts_.clear();
    part_msgs_ = nullptr;
    part_row0_ = nullptr;
    xbuf_own_ = nullptr;
    anorm_ = nullptr;
    la_arena_ = nullptr;
    la_arena_bytes_ = 0;
    if (hctl_) cudaFreeHost(hctl_);
    if (hlog_) cudaFreeHost(hlog_);
    if (hone_) cudaFreeHost(hone_);
    if (ev_snap_) cudaEventDestroy(ev_snap_);
    for (cudaEvent_t e : ev_pool_) cudaEventDestroy(e);
    for (auto& r : ev_used_) {
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
    if (pool_) cudaMemPoolDestroy(pool_);
    if (st_) cudaStreamDestroy(st_);
    d_ = Dev{};
    cost_buf_ = scratch_ = chain_ = b0_ = nullptr;
    art_row_ = nullptr;
    tmaps_ = nullptr;
    hctl_ = nullptr;
    hlog_ = nullptr;
    hone_ = nullptr;
    ev_snap_ = nullptr;
    ev_pool_.clear();
    ev_used_.clear();
    pool_ = nullptr;
    st_ = nullptr;
    cudaGetLastError();
}

void Solver::push() {
    ev_chain_ = nullptr;
    CK(cudaMemcpyAsync(d_.ctl, hctl_, sizeof(Ctl), cudaMemcpyHostToDevice, st_));
    h2d_bytes += sizeof(Ctl);
}

void Solver::pull(bool with_log) {
    ev_chain_ = nullptr;
    CK(cudaMemcpyAsync(hctl_, d_.ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st_));
    d2h_bytes += sizeof(Ctl);
    if (with_log) {
        CK(cudaMemcpyAsync(hlog_, d_.log, sizeof(LogEntry) * d_.log_cap, cudaMemcpyDeviceToHost, st_));
        d2h_bytes += sizeof(LogEntry) * d_.log_cap;
    }
    CK(cudaStreamSynchronize(st_));
    CK(cudaGetLastError());
    if (comm_) comm_->check(st_);
}

double Solver::objective_value() {
    double v = 0.0;
    CK(cudaMemcpyAsync(&v, d_.top + m_, sizeof(double), cudaMemcpyDeviceToHost, st_));
    CK(cudaStreamSynchronize(st_));
    return v;
}

// rebuild_top_row (solver.cpp:318-329). Sharded: an ordered chain, shard g
// continuing shard g-1's partial sums (an allreduce would reorder the sum).
void Solver::rebuild_top_row() {
    if (tiled_) {
        // the ordered chain over the partitions, ascending rows (solver.cpp:318-329)
        for (size_t p = 0; p < parts_.size(); ++p) {
            ensure_resident((int)p);
            launch_rebuild_top(part_dev((int)p), p == 0 ? nullptr : chain_, chain_, st_);
            CK(cudaGetLastError());
        }
        CK(cudaMemcpyAsync(d_.top, chain_, sizeof(double) * (m_ + 1), cudaMemcpyDeviceToDevice, st_));
        CK(cudaMemsetAsync(d_.top + m_ + 1, 0, sizeof(double), st_));
        return;
    }
    if (!sharded_) {
        launch_rebuild_top(d_, nullptr, d_.top, st_);
        CK(cudaGetLastError());
        return;
    }
    for (int g = 0; g < world_; ++g) {
        if (g == rank_) launch_rebuild_top(d_, g == 0 ? nullptr : chain_, chain_, st_);
        CK(cudaGetLastError());
        comm_->bcast(chain_, sizeof(double) * (m_ + 1), g, st_);
    }
    CK(cudaMemcpyAsync(d_.top, chain_, sizeof(double) * (m_ + 1), cudaMemcpyDeviceToDevice, st_));
    CK(cudaMemsetAsync(d_.top + m_ + 1, 0, sizeof(double), st_));
}

// Shards sharing a GPU: growing a memory pool may wait for the whole device,
// including another shard's spin-waiting exchange kernel, which in turn waits
// for this shard. Before stream-ordered allocations on a sharded path, every
// shard drains its stream and meets the others (a no-op across processes).
void Solver::temp_alloc_fence() {
    if (!comm_) return;
    CK(cudaStreamSynchronize(st_));
    comm_->host_barrier();
}

int Solver::owner_of_row(int i) const {
    // inverse of row0(g) = floor(m g / G)
    int g = (int)(((long long)i * world_ + world_ - 1) / std::max(1, m_));
    g = std::min(std::max(g, 0), world_ - 1);
    while (g > 0 && (long long)m_ * g / world_ > i) --g;
    while (g + 1 < world_ && (long long)m_ * (g + 1) / world_ <= i) ++g;
    return g;
}

void Solver::single_gpu_only(const char* what) const {
    if (sharded_) throw Error(LPSG_INVALID_ARGUMENT, std::string(what) + ": step API is single-GPU only");
    if (tiled_) throw Error(LPSG_INVALID_ARGUMENT, std::string(what) + ": step API needs the in-core tableau");
}

// note_iteration (solver.cpp:256-276) for one logged pivot.
void Solver::note_pivot(const LogEntry& e) {
    ++total_iter_;
    ++phase_iter_[phase_ - 1];
    basic_[e.row] = e.entering;
    const bool q_local = e.entering >= d_.col0 && e.entering < d_.col1;
    const bool p_local = e.leaving < n_total_ && e.leaving >= d_.col0 && e.leaving < d_.col1;
    n_scan_host_ += (p_local ? 1 : 0) - (q_local ? 1 : 0);
    if (last_objective_ - e.objective > cfg_.opt_tol) banned_.clear();
    last_objective_ = e.objective;
    {
        // algorithmic HBM traffic of this pivot: pricing reads
        // the scanned A columns and W; the update reads + writes this shard's
        // [B^-1 | b_bar] rows; the pivot row is read, divided, written; W updated
        const double m = m_;
        const double rows = rows_local();
        dev_read_bytes += 8.0 * m * (double)n_scan_host_ + 8.0 * m + 8.0 * rows * (m + 1.0) +
                          8.0 * (m + 1.0) * 2.0 + 8.0 * m;
        dev_write_bytes += 8.0 * rows * (m + 1.0) + 8.0 * (m + 1.0) * 2.0;
    }
    lpsg_trace t{(long)e.iteration, e.phase, e.row, e.leaving, e.entering, e.objective};
    if (keep_trace) trace.push_back(t);
    if (observer) observer(&t, observer_user);
    if (view_observer) {
        const lpsg_memory mem = memory();
        lpsg_iteration_view v{e.phase, (long)e.iteration, e.objective, basic_.data(), m_, m_ + 2,
                              e.row, e.leaving, e.entering, &mem, handle};
        view_observer(&v, view_user);
    }
}

lpsg_memory Solver::memory() const {
    lpsg_memory mm{};
    mm.device_read_bytes = (uint64_t)dev_read_bytes;
    mm.device_write_bytes = (uint64_t)dev_write_bytes;
    mm.h2d_bytes = (uint64_t)h2d_bytes;
    mm.d2h_bytes = (uint64_t)d2h_bytes;
    mm.kernel_launches = (uint64_t)launches_total;
    return mm;
}

// The device appends to a ring (log_len is monotonic); entries
// [log_seen_, log_len) are new since the last drain.
void Solver::drain_log() {
    const long long n = (long long)hctl_->log_len - log_seen_;
    if (n > d_.log_cap) throw Error(LPSG_CUDA_ERROR, "pivot log overflow");
    for (long long k = 0; k < n; ++k) note_pivot(hlog_[(log_seen_ + k) % d_.log_cap]);
    log_seen_ = hctl_->log_len;
}

// Asynchronous snapshot of the control block and the log ring, ordered after
// everything enqueued so far; ev_snap_ completes when it has landed.
void Solver::snapshot() {
    ev_chain_ = nullptr;
    CK(cudaMemcpyAsync(hctl_, d_.ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st_));
    CK(cudaMemcpyAsync(hlog_, d_.log, sizeof(LogEntry) * d_.log_cap, cudaMemcpyDeviceToHost, st_));
    d2h_bytes += sizeof(Ctl) + sizeof(LogEntry) * d_.log_cap;
    CK(cudaEventRecord(ev_snap_, st_));
}

// One pivot's device work in the fused schedule; world > 1 adds the three
// per-pivot exchanges: the pivot row from its owner, the
// pricing (z, j) and the ratio-test messages.
void Solver::seq_pivot() {
    if (tiled_) {
        tiled_pivot();
        return;
    }
    if (!sharded_) {
        L(K_PIVOT, bytes_of(K_PIVOT), [&] { launch_pivot(d_, st_); });
        return;
    }
    d_.fused_x = 0;
    if (comm_->fused_slot(&d_.px_x)) {
        // P2P: the owner's k_pivot_row stores x into the peers' xbuf itself
        d_.fused_x = 1;
        d_.xbuf_off = comm_->sym_offset(d_.xbuf);
        L(K_PIVOT, bytes_of(K_PIVOT), [&] { launch_pivot_row(d_, st_); });
        L(K_COMM, 0.0, [&] { comm_->wait_slot(d_.px_x, st_); });
        d_.fused_x = 0;
    } else {
        L(K_PIVOT, bytes_of(K_PIVOT), [&] { launch_pivot_row(d_, st_); });
        L(K_COMM, 0.0, [&] { comm_->owner_bcast(d_.xbuf, sizeof(double) * ((size_t)m_ + 3), &d_.ctl->x_owner, st_); });
    }
    L(K_PIVOT, 0.0, [&] { launch_pivot(d_, st_); });
}

// With a device-initiated transport the (z, j) and ratio messages are stored
// into the peers' mailboxes by the producing kernel's last CTA (no collective
// launch); the *_final kernels wait on the flags.
void Solver::seq_price() {
    d_.fused = 0;
    if (sharded_ && comm_->fused_slot(&d_.px_price)) d_.fused = 1;
    L(K_PRICE, bytes_of(K_PRICE), [&] { launch_price(d_, st_); });
    if (sharded_) {
        if (!d_.fused) L(K_COMM, 0.0, [&] { comm_->allgather(d_.pmsg, d_.pmsg + 1, sizeof(PriceMsg), st_); });
        L(K_OTHER, 0.0, [&] { launch_price_final(d_, st_); });
    }
    d_.fused = 0;
}

void Solver::seq_update() {
    if (tiled_) {
        tiled_pass();
        return;
    }
    d_.fused = 0;
    if (sharded_ && comm_->fused_slot(&d_.px_ratio)) d_.fused = 1;
    L(K_UPDATE, bytes_of(K_UPDATE), [&] { launch_update(d_, st_); });
    if (sharded_) {
        if (!d_.fused) L(K_COMM, 0.0, [&] { comm_->allgather(d_.rmsg, d_.rmsg + 1, sizeof(RatioMsg), st_); });
        L(K_OTHER, 0.0, [&] { launch_ratio_final(d_, st_); });
    }
    d_.fused = 0;
}

// One pivot per iteration. With the fused pivot (d_.fuse_pivot) the previous
// k_update's last CTA already ran pivot_update, so a pivot is k_price +
// k_update; otherwise k_pivot (or the sharded pivot-row exchange) leads.
void Solver::enqueue_pivots(int n) {
    // never enqueue pivots past the budget: they would only run as no-op
    // launches behind the stop (room_ is set by run_phase)
    n = (int)std::min<long long>(n, room_);
    room_ -= n;
    for (int k = 0; k < n; ++k) {
        if (unfused_ratio_) L(K_RATIO, bytes_of(K_RATIO), [&] { launch_ratio(d_, st_); });
        if (!d_.fuse_pivot) seq_pivot();
        seq_price();
        seq_update();
    }
    CK(cudaGetLastError());
}

// ST_OVERFLOW (world > 1): a shard had more local candidates than a RatioMsg
// holds. Gather every shard's full local list and apply the global window on
// the host with the device's formula (solver.cpp:154-160).
std::vector<int> Solver::gather_overflow_candidates() {
    const int G = world_;
    std::vector<RatioMsg> msgs(G);
    CK(cudaMemcpyAsync(msgs.data(), d_.rmsg + 1, sizeof(RatioMsg) * G, cudaMemcpyDeviceToHost, st_));
    CK(cudaStreamSynchronize(st_));
    int maxn = 1;
    for (auto& mm : msgs) maxn = std::max(maxn, mm.any ? mm.n : 0);
    temp_alloc_fence();
    int* rows_d = talloc<int>((size_t)G * maxn, st_, pool_);
    double* rat_d = talloc<double>((size_t)G * maxn, st_, pool_);
    comm_->allgather(d_.cand, rows_d, sizeof(int) * maxn, st_);
    comm_->allgather(d_.cand_ratio, rat_d, sizeof(double) * maxn, st_);
    std::vector<int> rows((size_t)G * maxn);
    std::vector<double> rat((size_t)G * maxn);
    CK(cudaMemcpyAsync(rows.data(), rows_d, sizeof(int) * rows.size(), cudaMemcpyDeviceToHost, st_));
    CK(cudaMemcpyAsync(rat.data(), rat_d, sizeof(double) * rat.size(), cudaMemcpyDeviceToHost, st_));
    CK(cudaStreamSynchronize(st_));
    CK(cudaFreeAsync(rows_d, st_));
    CK(cudaFreeAsync(rat_d, st_));
    const double th = hctl_->theta;
    const double window = th + cfg_.ratio_tie_tol * std::max(1.0, std::fabs(th));
    std::vector<int> cand;
    for (int g = 0; g < G; ++g) {
        if (!msgs[g].any) continue;
        for (int e = 0; e < msgs[g].n; ++e)
            if (rat[(size_t)g * maxn + e] <= window) cand.push_back(rows[(size_t)g * maxn + e]);
    }
    return cand;
}

// run_phase (solver.cpp:278-293) in the fused schedule.
int Solver::run_phase() {
    // the fused pivot needs the whole pivot row in one CTA's registers
    // (kernels.cu pivot_cta: 4 elements per thread). It pays where the pivot
    // is launch-bound (C1 m = 256: 38-40k -> 42.5k it/s); at C2 (m = 2000) the
    // single-CTA tail cost more than the k_pivot launch it saved (17.1k ->
    // 16.2k it/s with 16 elements per thread), so larger m keep k_pivot
    d_.fuse_pivot = (!sharded_ && !unfused_ratio_ && !tiled_ && (long long)m_ + 1 <= 4LL * d_.upd_threads &&
                     xp_env("LPSG_NO_FUSED_PIVOT") == nullptr) ? 1 : 0;
    struct Unfuse {
        Dev& d;
        ~Unfuse() { d.fuse_pivot = 0; }  // every other schedule pivots with k_pivot
    } unfuse{d_};
    hctl_->status = ST_RUNNING;
    hctl_->pending = 0;
    hctl_->no_ftran = 0;
    hctl_->no_ratio = unfused_ratio_ ? 1 : 0;
    hctl_->phase = phase_;
    room_ = std::max<long long>(0, hctl_->budget - hctl_->total_iter);
    push();
    seq_price();   // price(W_t), first pivot of the phase
    seq_update();  // standalone FTRAN (pending == 0) + ratio test
    CK(cudaGetLastError());
    // Pipelined batches: batch k+1 is enqueued before the host waits for batch
    // k's snapshot, so the GPU never idles on the host round trip. Kernels of
    // an in-flight batch no-op once the device status leaves RUNNING, so a
    // stop (optimal, tie, budget) seen in snapshot k leaves the state exactly as
    // batch k ended. Profiling windows stay synchronous (their events must be
    // complete when read).
    const bool pipelined = !prof_ && xp_env("LPSG_NO_PIPELINE") == nullptr && (!comm_ || comm_->allows_pipelining());
    bool enqueued = false;
    // Adaptive batch: a tie stops the device chain, and the rest of the batch (and
    // the one in flight) then runs as no-op launches. Degenerate LPs tie on most
    // pivots, so shrink the batch after a tie and grow it back after clean ones.
    int cur = batch_;
    for (;;) {
        if (!enqueued) enqueue_pivots(cur);
        enqueued = false;
        if (pipelined) {
            snapshot();
            enqueue_pivots(cur);
            enqueued = true;
            CK(cudaEventSynchronize(ev_snap_));
            CK(cudaGetLastError());
            if (comm_) comm_->check(st_);
        } else {
            pull(true);
        }
        if (prof_) flush_profile();
        if (dbg_trace_)
            fprintf(stderr, "[solver r%d] status %d log %d q %d r %d ncand %d iter %lld\n", rank_, hctl_->status,
                    hctl_->log_len, hctl_->q, hctl_->r, hctl_->ncand, (long long)hctl_->total_iter);
        drain_log();
        const int st = hctl_->status;
        if (st == ST_RUNNING) {
            cur = std::min(batch_, cur * 2);
            if (!pipelined) push();
            continue;
        }
        if (st == ST_TIE || st == ST_OVERFLOW) cur = std::max(1, cur / 4);
        enqueued = false;  // an in-flight batch (if any) no-ops: the device stopped
        bool resumed = false;
        const int out = handle_stop(st, &resumed);
        if (resumed) {
            seq_pivot();
            seq_price();
            seq_update();
            // the device stopped at hctl_->total_iter; the resumed pivot is the next one
            room_ = std::max<long long>(0, hctl_->budget - hctl_->total_iter - 1);
            continue;
        }
        return out;
    }
}

// A stopped device chain: a ratio-test tie (select_leaving on the host, then
// *resumed with hctl_->r set and pushed: the caller enqueues the pivot) or a
// final status of the phase (returned).
int Solver::handle_stop(int st, bool* resumed) {
    *resumed = false;
    if (st == ST_TIE || st == ST_OVERFLOW) {
        std::vector<int> cand;
        if (st == ST_TIE) {
            cand.resize(hctl_->ncand);
            CK(cudaMemcpyAsync(cand.data(), d_.cand, sizeof(int) * cand.size(), cudaMemcpyDeviceToHost, st_));
            CK(cudaStreamSynchronize(st_));
        } else {
            cand = gather_overflow_candidates();
            if (cand.empty()) throw Error(LPSG_CUDA_ERROR, "sharded ratio test lost its candidates");
        }
        const int r = cand.size() == 1 || cfg_.anticycle == 1 ? cand.front() : select_leaving(cand, hctl_->q);
        hctl_->r = r;
        hctl_->status = ST_RUNNING;
        push();
        *resumed = true;
        return 0;
    }
    if (st == ST_PIVOT_ERR) throw Error(LPSG_PIVOT_TOO_SMALL, "pivot element below pivot_tol");
    if (st == ST_OPTIMAL) return LPSG_OPTIMAL;
    if (st == ST_UNBOUNDED) return LPSG_UNBOUNDED;
    if (st == ST_ITER_LIMIT) return LPSG_ITERATION_LIMIT;
    throw Error(LPSG_CUDA_ERROR, "unexpected control status " + std::to_string(st));
}

// run_phase (solver.cpp:278-293) one pivot per host round trip, unfused: price,
// FTRAN + ratio test, [select_leaving], pivot, update without the next FTRAN.
// After every pivot the device holds exactly the reference's tableau at its
// observer call (column m+1 included: tiled_engine.cpp:240-242,265), so a
// view observer with rows can read any row (lpsg_read_row).
int Solver::run_phase_stepwise() {
    hctl_->status = ST_RUNNING;
    hctl_->pending = 0;
    hctl_->no_ftran = 0;
    hctl_->no_ratio = unfused_ratio_ ? 1 : 0;
    hctl_->phase = phase_;
    push();
    for (;;) {
        seq_price();
        if (unfused_ratio_) {
            seq_update();  // FTRAN only
            L(K_RATIO, bytes_of(K_RATIO), [&] { launch_ratio(d_, st_); });
        } else {
            seq_update();  // FTRAN + fused ratio test
        }
        CK(cudaGetLastError());
        pull(false);
        if (prof_) flush_profile();
        const int st = hctl_->status;
        if (st != ST_RUNNING) {
            bool resumed = false;
            const int out = handle_stop(st, &resumed);
            if (!resumed) return out;
        }
        seq_pivot();
        CK(cudaMemcpyAsync(&d_.ctl->no_ftran, hone_, sizeof(int), cudaMemcpyHostToDevice, st_));
        seq_update();  // the rank-1 update only
        CK(cudaGetLastError());
        pull(true);
        if (prof_) flush_profile();
        if (hctl_->status == ST_PIVOT_ERR) throw Error(LPSG_PIVOT_TOO_SMALL, "pivot element below pivot_tol");
        drain_log();
        hctl_->no_ftran = 0;
        push();
    }
}

// select_leaving (solver.cpp:215-238)
int Solver::select_leaving(const std::vector<int>& cand, int entering) {
    if (cand.size() == 1) return cand.front();
    if (cfg_.anticycle == 1) return cand.front();
    auto& banned = banned_[entering];
    std::vector<int> survivors;
    for (int r : cand)
        if (!banned.count(basic_[r])) survivors.push_back(r);
    if (survivors.empty()) survivors = cand;  // aspiration override
    int chosen = survivors.front();
    if (survivors.size() > 1) {
        std::vector<double> scores;
        bool first = false;
        lookahead(survivors, entering, scores, &first);
        if (first) {  // proven: every later score <= the first one's (+-0)
            banned.insert(basic_[chosen]);
            return chosen;
        }
        double best = -1.0;
        for (size_t k = 0; k < survivors.size(); ++k)
            if (scores[k] > best) {
                best = scores[k];
                chosen = survivors[k];
            }
    }
    banned.insert(basic_[chosen]);
    return chosen;
}

// lookahead_score (solver.cpp:164-213) for every row in `rows`, batched on the
// device. Sharded: pivot rows from their owners, pricing and theta' per shard,
// exact max / min merges (every rank computes the same scores).
void Solver::lookahead(const std::vector<int>& rows, int entering, std::vector<double>& scores,
                       bool* first_proven) {
    const int K = (int)rows.size();
    scores.assign(K, 0.0);
    if (K == 0) return;
    if (first_proven) *first_proven = false;
    const int m = m_;
    const int G = world_;
    const int ldx = (int)round_up(m + 1, 32);
    const size_t per = (size_t)2 * ldx * sizeof(double);
    const int kmax = (int)std::max<size_t>(1, std::min<size_t>(4096, ((size_t)2 << 30) / per));
    const int kb = std::min(K, kmax);
    LookaheadDev la{};
    la.ldx = ldx;
    la.q = entering;
    la.nblk = (hctl_->n_scan + 127) / 128 + 1;  // 128-slot tiles + the leaving column
    la.nblk_t = std::max(1, (d_.mloc + 63) / 64);  // 64-row theta tiles
    const int P = tiled_ ? (int)parts_.size() : 1;
    la.x_owned_only = tiled_ ? 1 : 0;
    std::vector<int> porder;  // Case 2: the resident partition first, then the others
    if (tiled_) {
        if (resident_ >= 0) porder.push_back(resident_);
        for (int p = 0; p < P; ++p)
            if (p != resident_) porder.push_back(p);
    }
    // bounded pricing (kernels.cu k_la_screen, k_la_cands, k_la_exact): from
    // la_bound_min_ candidates up, the exact argmax without the exact GEMM
    const bool bounded = kb >= la_bound_min_;
    // bounded selection (kernels.cu, k_la_probe*): one GPU, in-core, one batch
    const bool probe = first_proven && !sharded_ && !tiled_ && kb == K && K >= la_bound_min_;
    if (bounded && !anorm_) {
        anorm_ = dalloc<double>(n_total_);
        launch_colnorm(d_, anorm_, st_);
    }
    la.anorm = anorm_;
    // Every buffer of this lookahead is carved from one arena that persists
    // across lookaheads (grown when a larger tie needs it): a tie costs no
    // allocator calls (30-odd stream-ordered allocations and frees before).
    const size_t nt = (size_t)kb * std::max(1, la.nblk - 1);
    int* rows_d = nullptr;
    auto carve = [&](unsigned char* base) -> size_t {
        size_t off = 0;
        auto take = [&](auto*& ptr, size_t n) {
            using T = std::remove_pointer_t<std::remove_reference_t<decltype(ptr)>>;
            ptr = base ? reinterpret_cast<T*>(base + off) : nullptr;
            off += (std::max<size_t>(n, 1) * sizeof(T) + 255) & ~size_t(255);
        };
        take(rows_d, kb);
        take(la.X, (size_t)kb * ldx);
        take(la.Wp, (size_t)kb * ldx);
        take(la.bz, kb);
        take(la.bj, kb);
        take(la.theta, kb);
        take(la.score, kb);
        take(la.part_z, (size_t)kb * la.nblk);
        take(la.part_j, (size_t)kb * la.nblk);
        take(la.part_t, (size_t)kb * la.nblk_t);
        take(la.pm, kb);
        if (sharded_) take(la.pm_all, (size_t)kb * G);
        take(la.tl, kb);
        take(la.own_t, kb);
        if (sharded_) take(la.tl_all, (size_t)kb * G);
        else if (tiled_) take(la.tl_all, (size_t)kb * P);
        take(la.nonfinite, 1);
        if (bounded) {
            take(la.wnorm, kb);
            take(la.tl_s, nt * kLaTile);
            take(la.tl_z, nt * kLaTile);
            take(la.tl_n, nt);
            take(la.part_L, (size_t)kb * la.nblk);
            take(la.cj, (size_t)kb * kLaCand);
            take(la.cz, (size_t)kb * kLaCand);
            take(la.cn, kb);
            take(la.pairs, kLaPairs);
            take(la.npairs, 1);
            take(la.fail, 1);
        }
        if (probe) {
            take(la.prow, kLaProbe);
            take(la.nprow, 1);
            take(la.Tg, (size_t)m * kLaProbe);
            take(la.ok, K);
            take(la.clist, K);
            take(la.yacc, (size_t)K * 128);
            take(la.pxb, K);
            take(la.pxn, K);
            take(la.pbn, K);
            take(la.ptn, 128);
            take(la.ncl, 1);
            take(la.first, 1);
        }
        return off;
    };
    const size_t need = carve(nullptr);
    if (need > la_arena_bytes_) {
        if (la_arena_) CK(cudaFreeAsync(la_arena_, st_));
        la_arena_bytes_ = need + need / 4;
        la_arena_ = talloc<unsigned char>(la_arena_bytes_, st_, pool_);
    }
    carve(la_arena_);
    la.rows = rows_d;
    CK(cudaMemsetAsync(la.X, 0, sizeof(double) * (size_t)kb * ldx, st_));
    if (dbg_trace_) fprintf(stderr, "[solver r%d] lookahead K=%d\n", rank_, K);
    temp_alloc_fence();
    for (int k0 = 0; k0 < K; k0 += kb) {
        la.K = std::min(kb, K - k0);
        CK(cudaMemcpyAsync(rows_d, rows.data() + k0, sizeof(int) * la.K, cudaMemcpyHostToDevice, st_));
        CK(cudaMemsetAsync(la.nonfinite, 0, sizeof(int), st_));
        ev_chain_ = nullptr;  // the copy is not a kernel of the profile
        // fp64 flops of the batched work: pricing K x m x n_scan(shard) dot terms
        // (DMUL + DADD); theta K x mloc x m terms of (T_ij - y_i X_kj) a_j
        // (two more for the updated element)
        const double kf = 2.0 * la.K * (double)m;
        if (tiled_) {
            // Case 2: each partition writes its candidates' pivot rows
            for (int k = 0; k < P; ++k) {
                const int p = porder[k];
                ensure_resident(p);
                const Dev dp = part_dev(p);
                L(K_OTHER, 0.0, [&] { launch_la_x(dp, la, st_); });
            }
        } else {
            L(K_OTHER, 0.0, [&] { launch_la_x(d_, la, st_); });
        }
        if (sharded_) L(K_COMM, 0.0, [&] { comm_->sum_i64(reinterpret_cast<long long*>(la.X), (size_t)la.K * ldx, st_); });
        L(K_LA_PRICE, kf * (double)hctl_->n_scan, [&] { la_ok(launch_la_price(d_, la, bounded, st_)); });
        if (sharded_) L(K_COMM, 0.0, [&] { comm_->allgather(la.pm, la.pm_all, sizeof(PriceMsg) * la.K, st_); });
        L(K_OTHER, 0.0, [&] { launch_la_decide(d_, la, sharded_ ? la.pm_all : la.pm, G, st_); });
        // bounded selection (kernels.cu, k_la_probe*): one GPU, in-core, one batch
        if (probe) {
            L(K_LA_THETA, 2.0 * kf * kLaProbeRound, [&] { la_ok(launch_la_probe(d_, la, st_)); });
            CK(cudaGetLastError());
            int first = 0, ncl = 0;
            CK(cudaMemcpyAsync(&first, la.first, sizeof(int), cudaMemcpyDeviceToHost, st_));
            CK(cudaMemcpyAsync(&ncl, la.ncl, sizeof(int), cudaMemcpyDeviceToHost, st_));
            int pfail = 0;
            if (bounded) CK(cudaMemcpyAsync(&pfail, la.fail, sizeof(int), cudaMemcpyDeviceToHost, st_));
            CK(cudaStreamSynchronize(st_));
            if (first != 1 && ncl > 0) {  // the screen left candidates unproven: exact rounds
                ++la_probe_rounds_;
                L(K_LA_THETA, 0.0, [&] { launch_la_probe_rounds(d_, la, st_); });
                CK(cudaGetLastError());
                CK(cudaMemcpyAsync(&first, la.first, sizeof(int), cudaMemcpyDeviceToHost, st_));
                CK(cudaStreamSynchronize(st_));
            }
            if (bounded) ++(pfail ? la_price_exact_ : la_price_bounded_);
            if (dbg_trace_) {
                std::vector<int> bjh(K), okh(K);
                int np = 0;
                CK(cudaMemcpy(bjh.data(), la.bj, sizeof(int) * K, cudaMemcpyDeviceToHost));
                CK(cudaMemcpy(okh.data(), la.ok, sizeof(int) * K, cudaMemcpyDeviceToHost));
                int unc_hi = 0, unc_lo = 0;
                for (int k = 0; k < K; ++k)
                    if (bjh[k] >= 0 && !okh[k]) (bjh[k] >= n_total_ - m ? unc_hi : unc_lo)++;
                fprintf(stderr, "[solver r%d]   uncertified: %d with best_j in the last m columns, %d below\n", rank_,
                        unc_hi, unc_lo);
                CK(cudaMemcpy(&np, la.nprow, sizeof(int), cudaMemcpyDeviceToHost));
                std::sort(bjh.begin(), bjh.end());
                const long distinct = std::unique(bjh.begin(), bjh.end()) - bjh.begin();
                std::vector<double> bb(m);
                CK(cudaMemcpy(bb.data(), d_.T + (size_t)m * d_.ldT, sizeof(double) * m, cudaMemcpyDeviceToHost));
                np = (int)std::count_if(bb.begin(), bb.end(), [](double v) { return v <= 0.0; });
                fprintf(stderr, "[solver r%d] bounded selection K=%d: %d uncertified, first %s, %ld distinct best_j, %d rows with b_bar <= 0\n",
                        rank_, K, first == 1 ? 0 : (-first - 1) / 2,
                        first != 1 && ((-first - 1) & 1) ? "not provably 0" : "ok", distinct, np);
            }
            if (first == 1) {
                ++la_bounded_;
                *first_proven = true;
                return;
            }
            ++la_full_;
        } else if (first_proven) {
            ++la_full_;
        }
        if (tiled_) {
            // Case 2: theta' per partition (resident first), merged by the exact min of la_score
            for (int k = 0; k < P; ++k) {
                const int p = porder[k];
                ensure_resident(p);
                const Dev dp = part_dev(p);
                L(K_LA_THETA, 2.0 * kf * (double)dp.mloc, [&] { la_ok(launch_la_theta(dp, la, st_)); });
                CK(cudaMemcpyAsync(la.tl_all + (size_t)p * la.K, la.tl, sizeof(double) * la.K,
                                   cudaMemcpyDeviceToDevice, st_));
                ev_chain_ = nullptr;
            }
            L(K_OTHER, 0.0, [&] { launch_la_score(d_, la, la.tl_all, P, st_); });
        } else {
            L(K_LA_THETA, 2.0 * kf * (double)d_.mloc, [&] { la_ok(launch_la_theta(d_, la, st_)); });
            if (sharded_) L(K_COMM, 0.0, [&] { comm_->allgather(la.tl, la.tl_all, sizeof(double) * la.K, st_); });
            L(K_OTHER, 0.0, [&] { launch_la_score(d_, la, sharded_ ? la.tl_all : la.tl, G, st_); });
        }
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(scores.data() + k0, la.score, sizeof(double) * la.K, cudaMemcpyDeviceToHost, st_));
        int pfail = 0;
        if (bounded) CK(cudaMemcpyAsync(&pfail, la.fail, sizeof(int), cudaMemcpyDeviceToHost, st_));
        CK(cudaStreamSynchronize(st_));
        if (bounded) ++(pfail ? la_price_exact_ : la_price_bounded_);
    }
}

// One phase, through the reinversion mode when it is on: the device budget
// stops the pivot chain every reinv_every_ pivots for a rebuild, and an optimal
// or unbounded outcome is only accepted on a freshly rebuilt inverse (the
// drift that makes the reference call SCSD1 unbounded, or end C3 with a
// phase-1 objective above feas_tol, is gone after the rebuild).
int Solver::run_phase_any() {
    if (tiled_) return view_rows ? run_phase_stepwise() : run_phase_tiled();
    if (reinv_every_ <= 0) return view_rows ? run_phase_stepwise() : run_phase();
    for (;;) {
        const long long since = reinv_at_ >= 0 ? reinv_at_ : 0;
        const long long stop = std::min<long long>(max_iter_, std::max<long long>(total_iter_ + 1, since + reinv_every_));
        hctl_->budget = stop;
        const int st = view_rows ? run_phase_stepwise() : run_phase();
        hctl_->budget = max_iter_;
        push();
        const bool fresh = reinv_at_ == total_iter_;
        if (st == LPSG_ITERATION_LIMIT && total_iter_ < max_iter_) {
            reinvert();
            continue;
        }
        if ((st == LPSG_OPTIMAL || st == LPSG_UNBOUNDED) && !fresh) {
            reinvert();
            continue;
        }
        return st;
    }
}

// B^-1 rebuilt from the basis columns of the original A (csrc/reinvert.cu):
// Newton-Schulz X <- X + X (I - B X), repeated while the starting residual
// max|I - B X| is not small (>= 1e-6; one step from a residual eps leaves
// ~eps^2), then a probe |B X 1 - 1| of the result, b_bar = X b, and row 0 by
// rebuild_top_row (W = c_B^T X, obj = c_B . b_bar).
void Solver::reinvert() {
    const int m = m_;
    const long long ld = round_up(m, 4);
    const EventPair ev;
    cudaEvent_t e0 = ev.a, e1 = ev.b;
    CK(cudaEventRecord(e0, st_));
    double* Bm = talloc<double>((size_t)ld * m, st_, pool_);
    double* R = talloc<double>((size_t)ld * m, st_, pool_);
    double* Xn = talloc<double>((size_t)ld * m, st_, pool_);
    double* vec = talloc<double>(2 * (size_t)ld, st_, pool_);
    unsigned long long* amax = talloc<unsigned long long>(2, st_, pool_);
    auto read_max = [&](int k) {
        unsigned long long bits = 0;
        CK(cudaMemcpyAsync(&bits, amax + k, sizeof(bits), cudaMemcpyDeviceToHost, st_));
        CK(cudaStreamSynchronize(st_));
        double v;
        std::memcpy(&v, &bits, sizeof(v));
        return v;
    };
    launch_form_basis(d_, art_row_, Bm, ld, st_);
    int steps = 0;
    double before = 0.0;
    for (;;) {
        // R = I - B X, its max, X' = X + X R (into Xn, then back into T)
        launch_dgemm_nn(m, m, m, Bm, ld, d_.T, d_.ldT, R, ld, -1.0, nullptr, 0, st_);
        CK(cudaMemsetAsync(amax, 0, sizeof(unsigned long long), st_));
        launch_absmax(R, m, ld, amax, st_);
        const double res = read_max(0);
        if (steps == 0) before = res;
        if (!(res < 0.5)) throw Error(LPSG_CUDA_ERROR, "reinversion: the inverse drifted too far to refine");
        if (steps > 0 && res < 1e-14) break;  // converged: X is already the rebuilt inverse
        launch_dgemm_nn(m, m, m, d_.T, d_.ldT, R, ld, Xn, ld, 1.0, d_.T, d_.ldT, st_);
        CK(cudaMemcpy2DAsync(d_.T, sizeof(double) * d_.ldT, Xn, sizeof(double) * ld, sizeof(double) * m, m,
                             cudaMemcpyDeviceToDevice, st_));
        ++steps;
        if (res < 1e-6 || steps >= 4) break;  // quadratic convergence: one more step is below rounding
    }
    CK(cudaMemsetAsync(amax + 1, 0, sizeof(unsigned long long), st_));
    launch_probe_residual(m, Bm, ld, d_.T, d_.ldT, vec, vec + ld, amax + 1, st_);
    const double after = read_max(1);
    launch_gemv_bbar(d_, b0_, st_);
    CK(cudaGetLastError());
    rebuild_top_row();
    void* tmp[] = {Bm, R, Xn, vec, amax};
    for (void* p : tmp) CK(cudaFreeAsync(p, st_));
    CK(cudaEventRecord(e1, st_));
    CK(cudaStreamSynchronize(st_));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    ++reinv_count;
    reinv_steps += steps;
    reinv_res_before = before;
    reinv_res_after = after;
    reinv_seconds += ms / 1e3;
    reinv_at_ = total_iter_;
    last_objective_ = objective_value();
}

// ---- Case 2: out-of-core tiling ---------------------------------------------
// plan() (tiled_engine.cpp:29-54) on the reference's (m+1) x (m+2) tableau:
// in-core when it fits the budget; else partitions of capacity_rows - 1 whole
// tableau rows (one row slot stays reserved for the pivot row). Tableau row 0
// (W | obj | d) always stays on the device here, so partition p of tableau
// rows [b, e) holds rows [max(b, 1) - 1, e - 1) of [B^-1 | b_bar]; an empty
// one (the first, when it held row 0 only) is dropped. memory_budget 0 means
// unlimited, except that a tableau that does not fit the free HBM beside A
// is tiled with the HBM that is left.
void Solver::plan_tiles(int m, int n) {
    unsigned long long budget = cfg_.memory_budget;
    const unsigned long long row_bytes = 8ULL * (unsigned long long)(m + 2);
    const unsigned long long total = row_bytes * (unsigned long long)(m + 1);
    if (budget == 0 && !sharded_) {
        size_t free_b = 0, tot_b = 0;
        CK(cudaMemGetInfo(&free_b, &tot_b));
        const unsigned long long other = 8ULL * (unsigned long long)n * round_up(m, 4) +
                                         8ULL * (unsigned long long)m * (unsigned long long)d_.ld_nb +
                                         (512ULL << 20);
        if (total + other > free_b) {
            if (free_b <= other + 2 * row_bytes)
                throw Error(LPSG_OUT_OF_MEMORY, "lpsg_create: A alone does not fit the device");
            budget = free_b - other;
        }
    }
    if (budget == 0 || total <= budget) return;  // Case 1, in-core
    if (sharded_) throw Error(LPSG_INVALID_ARGUMENT, "lpsg_create: the out-of-core (tiled) case is single-GPU only");
    if (reinv_every_ > 0) throw Error(LPSG_INVALID_ARGUMENT, "lpsg_create: reinversion needs the in-core tableau");
    const unsigned long long cap_rows = budget / row_bytes;
    if (cap_rows < 2)
        throw Error(LPSG_BUDGET_TOO_SMALL, "device budget of " + std::to_string(budget) +
                                               " bytes cannot hold one data row plus the pivot row (row is " +
                                               std::to_string(row_bytes) + " bytes)");
    const int rpp = (int)std::min<unsigned long long>(cap_rows - 1, (unsigned long long)m + 1);
    for (int b = 0; b < m + 1; b += rpp) {
        const int e = std::min(b + rpp, m + 1);
        const int r0 = std::max(b, 1) - 1, r1 = e - 1;
        if (r1 > r0) parts_.push_back(Part{r0, r1 - r0, nullptr});
    }
    tiled_ = true;
    int mx = 0;
    for (const Part& q : parts_) mx = std::max(mx, q.rows);
    d_.mloc = mx;  // the device slab holds the largest partition
}

// The kernels see partition p as a shard of rows [row0, row0 + rows) living
// in the slab: Y, the candidate lists and the ratio message are this
// partition's slices of the global buffers.
Dev Solver::part_dev(int p) const {
    Dev dp = d_;
    const Part& q = parts_[p];
    dp.row0 = q.row0;
    dp.mloc = q.rows;
    dp.Y = d_.Y + q.row0;
    dp.cand = d_.cand + q.row0;
    dp.cand_ratio = d_.cand_ratio + q.row0;
    dp.rmsg = part_msgs_ + p;
    dp.sharded = 1;  // k_update leaves a RatioMsg, k_pivot reads the divided row from xbuf
    dp.fused = 0;
    dp.update_grid = (q.rows + d_.upd_h - 1) / d_.upd_h;
    dp.keep_pending = 0;
    return dp;
}

int Solver::part_of_row(int i) const {
    for (size_t p = 0; p < parts_.size(); ++p)
        if (i >= parts_[p].row0 && i < parts_[p].row0 + parts_[p].rows) return (int)p;
    throw Error(LPSG_CUDA_ERROR, "row outside every partition");
}

// upload_partition / download_resident (tiled_engine.cpp:165-184): the slab's
// partition goes back to the host before another one comes up.
void Solver::ensure_resident(int p) {
    if (resident_ == p) return;
    ev_chain_ = nullptr;
    const size_t w = sizeof(double);
    if (resident_ >= 0) {
        const Part& q = parts_[resident_];
        CK(cudaMemcpy2DAsync(q.host, w * q.rows, d_.T, w * d_.ldT, w * q.rows, m_ + 1, cudaMemcpyDeviceToHost, st_));
        d2h_bytes += (long long)(w * q.rows * (m_ + 1));
    }
    const Part& q = parts_[p];
    CK(cudaMemcpy2DAsync(d_.T, w * d_.ldT, q.host, w * q.rows, w * q.rows, m_ + 1, cudaMemcpyHostToDevice, st_));
    h2d_bytes += (long long)(w * q.rows * (m_ + 1));
    resident_ = p;
}

// One partitioned update (tiled_engine.cpp:246-263): the resident partition
// first, then the others in order; the last one stays resident. Each launch
// is the fused k_update of the in-core path on that partition (update(t),
// FTRAN(t+1), the ratio test's partition message); the messages are merged
// after the last one.
void Solver::tiled_pass() {
    const int P = (int)parts_.size();
    std::vector<int> order;
    if (resident_ >= 0) order.push_back(resident_);
    for (int p = 0; p < P; ++p)
        if (p != resident_) order.push_back(p);
    for (int k = 0; k < P; ++k) {
        const int p = order[k];
        ensure_resident(p);
        Dev dp = part_dev(p);
        dp.keep_pending = k + 1 < P ? 1 : 0;
        L(K_UPDATE, bytes_of(K_UPDATE), [&] { launch_update(dp, st_); });
    }
    L(K_OTHER, 0.0, [&] { launch_ratio_merge_parts(d_, part_msgs_, part_row0_, P, st_); });
    CK(cudaGetLastError());
}

// pivot_update's division (solver.cpp:246-247) of row r, then k_pivot. The
// resident partition divides in place in the slab; any other partition's row
// is gathered from its host copy into the pivot-row buffer, divided there and
// written back (the reference divides host-side and uploads the pivot row,
// tiled_engine.cpp:232-235).
void Solver::tiled_pivot() {
    const int r = hctl_->r;
    const int p = part_of_row(r);
    if (p == resident_) {
        const Dev dr = part_dev(p);
        L(K_PIVOT, 0.0, [&] { launch_pivot_row(dr, st_); });
    } else {
        const Part& q = parts_[p];
        const int li = r - q.row0;
        const size_t w = sizeof(double);
        ev_chain_ = nullptr;
        CK(cudaMemcpy2DAsync(d_.xbuf, w, q.host + li, w * q.rows, w, m_ + 1, cudaMemcpyHostToDevice, st_));
        Dev dx = d_;
        dx.T = d_.xbuf;  // the row as a one-row slab
        dx.ldT = 1;
        dx.row0 = r;
        dx.mloc = 1;
        dx.Y = d_.Y + r;
        dx.sharded = 1;
        L(K_PIVOT, 0.0, [&] { launch_pivot_row(dx, st_); });
        ev_chain_ = nullptr;
        CK(cudaMemcpy2DAsync(q.host + li, w * q.rows, d_.xbuf, w, w, m_ + 1, cudaMemcpyDeviceToHost, st_));
        h2d_bytes += (long long)(w * (m_ + 1));
        d2h_bytes += (long long)(w * (m_ + 1));
    }
    Dev dk = d_;
    dk.sharded = 1;
    L(K_PIVOT, bytes_of(K_PIVOT), [&] { launch_pivot(dk, st_); });
    CK(cudaGetLastError());
}

// run_phase (solver.cpp:278-293) for Case 2: the fused schedule of run_phase
// (pivot(t), price(t+1), one pass over the partitions for update(t) +
// FTRAN(t+1) + ratio), one pivot per host round trip: the host needs r to
// place the pivot-row division.
int Solver::run_phase_tiled() {
    hctl_->status = ST_RUNNING;
    hctl_->pending = 0;
    hctl_->no_ftran = 0;
    hctl_->no_ratio = 0;
    hctl_->phase = phase_;
    push();
    seq_price();
    tiled_pass();
    pull(true);
    if (prof_) flush_profile();
    for (;;) {
        const int st = hctl_->status;
        if (st != ST_RUNNING) {
            bool resumed = false;
            const int out = handle_stop(st, &resumed);
            if (!resumed) return out;
        }
        tiled_pivot();
        seq_price();
        tiled_pass();
        pull(true);
        if (prof_) flush_profile();
        if (hctl_->status == ST_PIVOT_ERR) throw Error(LPSG_PIVOT_TOO_SMALL, "pivot element below pivot_tol");
        drain_log();
    }
}

// Row i of [B^-1 | b_bar] (m+1 doubles) into device memory `out`, wherever it lives.
void Solver::gather_row_any(int i, double* out) {
    if (!tiled_) {
        launch_gather_row(d_, i - d_.row0, out, st_);
        return;
    }
    const int p = part_of_row(i);
    const Part& q = parts_[p];
    if (p == resident_) {
        launch_gather_row(part_dev(p), i - q.row0, out, st_);
    } else {
        const size_t w = sizeof(double);
        CK(cudaMemcpy2DAsync(out, w, q.host + (i - q.row0), w * q.rows, w, m_ + 1, cudaMemcpyHostToDevice, st_));
        h2d_bytes += (long long)(w * (m_ + 1));
    }
}

// drive_out_artificials (solver.cpp:295-316)
void Solver::drive_out_artificials() {
    for (int i = 0; i < m_; ++i) {
        if (basic_[i] < n_total_) continue;
        hctl_->found = INT_MAX;
        hctl_->status = ST_HOLD;
        push();
        const int owner = owner_of_row(i);
        if (owner == rank_) gather_row_any(i, scratch_);
        if (sharded_) comm_->bcast(scratch_, sizeof(double) * (m_ + 1), owner, st_);
        launch_drive_scan(d_, scratch_, st_);
        if (sharded_) comm_->min_i32(&d_.ctl->found, 1, st_);
        launch_drive_red(d_, st_);
        CK(cudaGetLastError());
        pull(false);
        const int found = hctl_->found;
        if (found < 0) {
            frozen_[i] = 1;
            const unsigned char one = 1;
            CK(cudaMemcpyAsync(d_.frozen + i, &one, 1, cudaMemcpyHostToDevice, st_));
            CK(cudaStreamSynchronize(st_));
            continue;
        }
        // compute_direction(found, red) then pivot_update(i, found), unfused
        hctl_->q = found;
        hctl_->d = hctl_->found_red;
        hctl_->r = i;
        hctl_->status = ST_RUNNING;
        hctl_->pending = 0;
        hctl_->no_ftran = 0;
        hctl_->no_ratio = 1;
        push();
        seq_update();  // FTRAN only
        seq_pivot();
        CK(cudaMemcpyAsync(&d_.ctl->no_ftran, hone_, sizeof(int), cudaMemcpyHostToDevice, st_));
        seq_update();  // update only
        CK(cudaGetLastError());
        pull(true);
        if (hctl_->status == ST_PIVOT_ERR) throw Error(LPSG_PIVOT_TOO_SMALL, "pivot element below pivot_tol");
        drain_log();
        hctl_->no_ftran = 0;
        hctl_->no_ratio = unfused_ratio_ ? 1 : 0;
        hctl_->status = ST_HOLD;
        push();
    }
}

void Solver::enter_phase2() {
    phase_ = 2;
    hctl_->phase = 2;
    hctl_->status = ST_HOLD;
    push();
    rebuild_top_row();
    banned_.clear();
    last_objective_ = objective_value();
}

// SimplexSolver::solve (solver.cpp:331-392). Resumable: a solve stopped by the
// iteration budget continues from the same state after set_max_iter (the
// benchmark uses this to time K pivots after W warm-up pivots); any other
// outcome is final.
void Solver::solve(lpsg_report* rep) {
    const EventPair ev;
    cudaEvent_t e0 = ev.a, e1 = ev.b;
    CK(cudaEventRecord(e0, st_));
    const double t0 = now_s();
    int status = final_status_;
    if (!done_) {
        status = LPSG_OPTIMAL;
        bool finished = false;
        if (phase_ == 1) {
            const int st = run_phase_any();
            if (st == LPSG_ITERATION_LIMIT) {
                status = LPSG_ITERATION_LIMIT;
                finished = true;
            } else if (st == LPSG_UNBOUNDED || objective_value() > cfg_.feas_tol) {
                status = LPSG_INFEASIBLE;
                finished = true;
            } else {
                drive_out_artificials();
                enter_phase2();
            }
        }
        if (!finished) status = run_phase_any();
        done_ = status != LPSG_ITERATION_LIMIT;
    }
    hctl_->status = ST_HOLD;
    push();
    CK(cudaEventRecord(e1, st_));
    CK(cudaStreamSynchronize(st_));
    const double t1 = now_s();
    {
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        last_device_ms = ms;
    }
    final_status_ = status;
    solved_ = true;

    rep->status = status;
    switch (status) {
        case LPSG_OPTIMAL:
        case LPSG_ITERATION_LIMIT: rep->objective = objective_value(); break;
        case LPSG_UNBOUNDED: rep->objective = -std::numeric_limits<double>::infinity(); break;
        default: rep->objective = std::numeric_limits<double>::quiet_NaN();
    }
    rep->iterations_phase1 = phase_iter_[0];
    rep->iterations_phase2 = phase_iter_[1];
    rep->total_seconds = t1 - t0;
    rep->tpi_seconds = rep->total_seconds / (double)std::max<long long>(1, total_iter_);
    rep->case_used = tiled_ ? 1 : 0;
}

// report.x (solver.cpp:378-383)
void Solver::get_x(double* x, int n) {
    if (n != n_total_) throw Error(LPSG_INVALID_ARGUMENT, "lpsg_get_x: n must equal n_total");
    std::fill(x, x + n, 0.0);
    if (solved_ && !(final_status_ == LPSG_OPTIMAL || final_status_ == LPSG_ITERATION_LIMIT)) return;
    std::vector<double> bbar(m_);
    const double* bcol = d_.T + (size_t)m_ * d_.ldT;
    if (tiled_) {
        CK(cudaStreamSynchronize(st_));
        for (size_t p = 0; p < parts_.size(); ++p) {
            const Part& q = parts_[p];
            if ((int)p == resident_)
                CK(cudaMemcpyAsync(bbar.data() + q.row0, bcol, sizeof(double) * q.rows, cudaMemcpyDeviceToHost, st_));
            else
                std::memcpy(bbar.data() + q.row0, q.host + (size_t)m_ * q.rows, sizeof(double) * q.rows);
        }
    } else if (!sharded_) {
        CK(cudaMemcpyAsync(bbar.data(), bcol, sizeof(double) * m_, cudaMemcpyDeviceToHost, st_));
    } else {
        // every shard's b_bar rows, padded to the largest shard, in rank order
        const int pad = m_ / world_ + 1;
        temp_alloc_fence();
        double* tmp = talloc<double>((size_t)pad * (world_ + 1), st_, pool_);
        CK(cudaMemcpyAsync(tmp, bcol, sizeof(double) * d_.mloc, cudaMemcpyDeviceToDevice, st_));
        comm_->allgather(tmp, tmp + pad, sizeof(double) * pad, st_);
        std::vector<double> all((size_t)pad * world_);
        CK(cudaMemcpyAsync(all.data(), tmp + pad, sizeof(double) * all.size(), cudaMemcpyDeviceToHost, st_));
        CK(cudaStreamSynchronize(st_));
        CK(cudaFreeAsync(tmp, st_));
        for (int g = 0; g < world_; ++g) {
            int r0 = 0, r1 = 0;
            lpsg_shard_range(m_, world_, g, &r0, &r1);
            for (int i = r0; i < r1; ++i) bbar[i] = all[(size_t)g * pad + (i - r0)];
        }
    }
    d2h_bytes += 8LL * m_;
    CK(cudaStreamSynchronize(st_));
    for (int i = 0; i < m_; ++i)
        if (basic_[i] < n_total_) x[basic_[i]] = bbar[i];
}

// ---- step API ---------------------------------------------------------------
void Solver::step_price(int* optimal, int* entering, double* red) {
    single_gpu_only("price");
    hctl_->status = ST_RUNNING;
    hctl_->budget = LLONG_MAX;
    push();
    launch_price(d_, st_);
    CK(cudaGetLastError());
    pull(false);
    *optimal = hctl_->status == ST_OPTIMAL;
    *entering = hctl_->q;
    *red = hctl_->d;
    hctl_->status = ST_HOLD;
    hctl_->budget = max_iter_;
    push();
}

void Solver::step_compute_direction(int entering, double red) {
    single_gpu_only("compute_direction");
    if (entering < 0 || entering >= n_total_) throw Error(LPSG_INVALID_ARGUMENT, "compute_direction: bad column");
    hctl_->q = entering;
    hctl_->d = red;
    hctl_->status = ST_RUNNING;
    hctl_->pending = 0;
    hctl_->no_ftran = 0;
    hctl_->no_ratio = 1;
    push();
    launch_update(d_, st_);
    CK(cudaGetLastError());
    pull(false);
    hctl_->status = ST_HOLD;
    push();
}

void Solver::step_ratio(int* unbounded, double* theta, std::vector<int>& cand) {
    single_gpu_only("ratio_test");
    hctl_->status = ST_RUNNING;
    hctl_->pending = 0;
    push();
    launch_ratio(d_, st_);
    CK(cudaGetLastError());
    pull(false);
    *unbounded = hctl_->status == ST_UNBOUNDED;
    cand.clear();
    *theta = 0.0;
    if (!*unbounded) {
        *theta = hctl_->theta;
        cand.resize(hctl_->ncand);
        CK(cudaMemcpyAsync(cand.data(), d_.cand, sizeof(int) * cand.size(), cudaMemcpyDeviceToHost, st_));
        CK(cudaStreamSynchronize(st_));
    }
    hctl_->status = ST_HOLD;
    push();
}

void Solver::step_pivot(int r, int q) {
    single_gpu_only("pivot_update");
    if (r < 0 || r >= m_ || q < 0 || q >= n_work_) throw Error(LPSG_INVALID_ARGUMENT, "pivot_update: bad index");
    hctl_->r = r;
    hctl_->q = q;
    hctl_->status = ST_RUNNING;
    hctl_->pending = 0;
    hctl_->no_ftran = 1;
    push();
    launch_pivot(d_, st_);
    launch_update(d_, st_);
    CK(cudaGetLastError());
    pull(true);
    if (hctl_->status == ST_PIVOT_ERR) {
        hctl_->status = ST_HOLD;
        hctl_->no_ftran = 0;
        push();
        throw Error(LPSG_PIVOT_TOO_SMALL, "pivot element in row " + std::to_string(r) + " below pivot_tol");
    }
    // pivot_update itself does not count an iteration (run_phase does)
    if (hctl_->log_len > log_seen_) {
        const LogEntry& e = hlog_[(hctl_->log_len - 1) % d_.log_cap];
        basic_[e.row] = e.entering;
    }
    log_seen_ = hctl_->log_len;
    hctl_->total_iter -= 1;
    hctl_->status = ST_HOLD;
    hctl_->no_ftran = 0;
    push();
}

void Solver::read_row(int i, double* out) {
    if (i < 0 || i > m_) throw Error(LPSG_INVALID_ARGUMENT, "read_row: bad row");
    if (i == 0) {
        CK(cudaMemcpyAsync(out, d_.top, sizeof(double) * (m_ + 2), cudaMemcpyDeviceToHost, st_));
    } else {
        const int owner = owner_of_row(i - 1);
        if (owner == rank_) {
            const int li = i - 1 - d_.row0;
            gather_row_any(i - 1, scratch_);
            CK(cudaMemcpyAsync(scratch_ + m_ + 1, d_.Y + li, sizeof(double), cudaMemcpyDeviceToDevice, st_));
        }
        if (sharded_) comm_->bcast(scratch_, sizeof(double) * (m_ + 2), owner, st_);
        CK(cudaMemcpyAsync(out, scratch_, sizeof(double) * (m_ + 2), cudaMemcpyDeviceToHost, st_));
    }
    CK(cudaStreamSynchronize(st_));
}

}  // namespace lpsg

// ============================================================== C ABI ===
struct lpsg_solver {
    lpsg::Solver* s;
    std::unique_ptr<lpsg::Comm> comm;
};

struct lpsg_peer {
    std::unique_ptr<lpsg::PeerHeap> heap;
};

namespace {
template <class F>
int guard(F&& f) {
    try {
        f();
        return LPSG_OK;
    } catch (const lpsg::Error& e) {
        lpsg::g_err = e.what();
        return e.code;
    } catch (const lpsg::CommError& e) {
        lpsg::g_err = e.what();
        return LPSG_NCCL_ERROR;
    } catch (const std::bad_alloc&) {
        lpsg::g_err = "host out of memory";
        return LPSG_OUT_OF_MEMORY;
    } catch (const std::exception& e) {
        lpsg::g_err = e.what();
        return LPSG_CUDA_ERROR;
    }
}
int bad(const char* what) {
    lpsg::g_err = what;
    return LPSG_INVALID_ARGUMENT;
}
}  // namespace

extern "C" {

const char* lpsg_last_error(void) { return lpsg::g_err.c_str(); }
const char* lpsg_version(void) { return "lpsg 0.1 (sm_100a, fp64)"; }

int lpsg_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

void lpsg_config_default(lpsg_config* cfg) {
    std::memset(cfg, 0, sizeof(*cfg));
    cfg->opt_tol = 1e-7;
    cfg->pivot_tol = 1e-9;
    cfg->feas_tol = 1e-7;
    cfg->ratio_tie_tol = 1e-9;
}

int lpsg_create(const lpsg_problem* lp, const lpsg_config* cfg, lpsg_solver** out) {
    if (!lp || !out) return bad("lpsg_create: null argument");
    lpsg_config c;
    if (cfg) c = *cfg;
    else lpsg_config_default(&c);
    if (c.world_size > 1 && (c.rank < 0 || c.rank >= c.world_size)) return bad("lpsg_create: bad rank");
    return guard([&] {
        auto* h = new lpsg_solver{nullptr, nullptr};
        try {
            if (c.peer) {
                if (!c.peer->heap) throw lpsg::CommError("lpsg_create: peer heap not created");
                if (c.peer->heap->device != c.device)
                    throw lpsg::CommError("lpsg_create: peer heap lives on another device");
                h->comm = lpsg::make_peer_comm(c.peer->heap.get());
            } else if (c.world_size > 1 || (c.reserved[1] & 1)) {
                h->comm = lpsg::make_nccl_comm(c.nccl_id, c.rank, std::max(1, c.world_size), c.device);
                if (!h->comm) throw lpsg::CommError("NCCL communicator");
            }
            h->s = new lpsg::Solver(*lp, c, h->comm.get());
        } catch (...) {
            delete h->s;
            delete h;
            throw;
        }
        *out = h;
    });
}

int lpsg_solve(lpsg_solver* s, lpsg_report* rep) {
    if (!s || !rep) return bad("lpsg_solve: null argument");
    return guard([&] { s->s->solve(rep); });
}

int lpsg_get_x(lpsg_solver* s, double* x, int n) {
    if (!s || !x) return bad("lpsg_get_x: null argument");
    return guard([&] { s->s->get_x(x, n); });
}

void lpsg_destroy(lpsg_solver* s) {
    if (!s) return;
    delete s->s;
    s->comm.reset();
    delete s;
}

int lpsg_nccl_unique_id(unsigned char out[128]) {
    if (!out) return bad("lpsg_nccl_unique_id: null argument");
    std::string err;
    if (!lpsg::nccl_unique_id(out, &err)) {
        lpsg::g_err = "lpsg_nccl_unique_id: " + err;
        return LPSG_NCCL_ERROR;
    }
    return LPSG_OK;
}

int lpsg_peer_create(int rank, int world, int device, size_t heap_bytes, lpsg_peer** out, unsigned char handle[64]) {
    if (!out || world < 1 || world > 32 || rank < 0 || rank >= world) return bad("lpsg_peer_create: bad argument");
    return guard([&] {
        auto* p = new lpsg_peer;
        try {
            p->heap = lpsg::peer_heap_create(rank, world, device, heap_bytes, handle);
        } catch (...) {
            delete p;
            throw;
        }
        *out = p;
    });
}

int lpsg_peer_connect(lpsg_peer* p, const unsigned char* handles) {
    if (!p || !handles) return bad("lpsg_peer_connect: null argument");
    return guard([&] { lpsg::peer_heap_connect(p->heap.get(), handles); });
}

void lpsg_peer_destroy(lpsg_peer* p) { delete p; }

const char* lpsg_transport(lpsg_solver* s) {
    if (!s) return "";
    return s->comm ? s->comm->transport() : "single";
}

int lpsg_solve_sharded(const lpsg_problem* lp, const lpsg_config* cfg, int shards, int flags, lpsg_report* rep,
                       double* x, lpsg_trace* trace, long cap, long* len) {
    const bool spread = (flags & LPSG_SHARD_SPREAD) != 0;
    const bool p2p = (flags & LPSG_SHARD_P2P) != 0;
    if (!lp || !rep || shards < 1 || shards > 32) return bad("lpsg_solve_sharded: bad argument");
    lpsg_config c;
    if (cfg) c = *cfg;
    else lpsg_config_default(&c);
    const int ndev = lpsg_device_count();
    if (ndev <= 0) {
        lpsg::g_err = "lpsg_solve_sharded: no CUDA device available (the solver has no CPU fallback)";
        return LPSG_CUDA_ERROR;
    }
    if (p2p && !spread && shards > 1) {
        // P2P shards sharing one GPU spin-wait on each other's flags, so every
        // shard's stream needs its own hardware work queue; the CUDA runtime sizes
        // them from CUDA_DEVICE_MAX_CONNECTIONS when the context is created
        // (default 8). The library never sets it itself (it would change every
        // other CUDA user of the process); the caller exports it before the
        // first CUDA call (tests/conftest.py does).
        const char* e = getenv("CUDA_DEVICE_MAX_CONNECTIONS");
        if (!e || atoi(e) < 2 * shards)
            return bad("lpsg_solve_sharded: P2P shards sharing one GPU need CUDA_DEVICE_MAX_CONNECTIONS >= "
                       "2 * shards in the environment before the CUDA context is created");
    }
    // One column-major A per device, shared read-only by the shards placed on
    // it (C5: 9.2 GB once instead of once per shard).
    std::vector<double*> shared_A(ndev, nullptr);
    struct SharedAFree {
        std::vector<double*>& v;
        ~SharedAFree() {
            for (size_t dv = 0; dv < v.size(); ++dv)
                if (v[dv]) {
                    cudaSetDevice((int)dv);
                    cudaFree(v[dv]);
                }
        }
    } shared_A_free{shared_A};
    {
        const int rc = guard([&] {
            for (int g = 0; g < shards; ++g) {
                const int dv = spread ? (c.device + g) % ndev : c.device;
                if (dv < 0 || dv >= ndev) throw lpsg::Error(LPSG_INVALID_ARGUMENT, "lpsg_solve_sharded: bad device");
                if (shared_A[dv] || lp->m <= 0 || lp->n_total <= 0 || !lp->A) continue;
                CK_SET_DEVICE(dv);
                const long long ld = (lp->m + 3) / 4 * 4;  // Solver's ld_cm
                void* p = nullptr;
                lpsg::ck(cudaMalloc(&p, sizeof(double) * ((size_t)lp->n_total * ld + 64)), "cudaMalloc(A_cm)");
                shared_A[dv] = static_cast<double*>(p);
                cudaStream_t st = nullptr;
                lpsg::ck(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "cudaStreamCreate");
                try {
                    lpsg::upload_A_cm(*lp, shared_A[dv], ld, st);
                } catch (...) {
                    cudaStreamDestroy(st);
                    throw;
                }
                cudaStreamDestroy(st);
            }
        });
        if (rc != LPSG_OK) return rc;
    }
    lpsg::LocalHub hub(shards);
    std::vector<char*> bases(shards, nullptr);
    std::vector<int> rc(shards, LPSG_OK);
    std::vector<std::string> msg(shards);
    std::vector<std::thread> th;
    for (int g = 0; g < shards; ++g) {
        th.emplace_back([&, g] {
            lpsg_config cg = c;
            cg.world_size = 1;  // the in-process comm below, not NCCL
            cg.peer = nullptr;
            cg.device = spread ? (c.device + g) % ndev : c.device;
            std::unique_ptr<lpsg::PeerHeap> heap;
            bool heap_ok = true;
            if (p2p) {
                // every shard allocates its heap, then all adopt each other's pointers
                try {
                    heap = lpsg::peer_heap_create(g, shards, cg.device, 0, nullptr);
                    bases[g] = heap->base;
                } catch (...) {
                    heap_ok = false;
                }
                hub.barrier();
                for (char* b : bases) heap_ok = heap_ok && b != nullptr;
            }
            rc[g] = guard([&] {
                CK_SET_DEVICE(cg.device);
                if (!heap_ok) throw lpsg::CommError("peer heap allocation failed on some shard");
                std::unique_ptr<lpsg::Comm> comm;
                if (p2p) {
                    heap->hub = &hub;
                    lpsg::peer_heap_connect_local(heap.get(), bases);
                    comm = lpsg::make_peer_comm(heap.get());
                } else {
                    comm = lpsg::make_local_comm(&hub, g);
                }
                lpsg::Solver s(*lp, cg, comm.get(), shared_A[cg.device]);
                s.keep_trace = g == 0 && trace != nullptr;
                lpsg_report r{};
                s.solve(&r);
                std::vector<double> xv(lp->n_total);
                s.get_x(xv.data(), lp->n_total);
                if (g == 0) {
                    *rep = r;
                    if (x) std::copy(xv.begin(), xv.end(), x);
                    if (len) *len = (long)s.trace.size();
                    if (trace)
                        for (long k = 0; k < std::min<long>(cap, (long)s.trace.size()); ++k) trace[k] = s.trace[k];
                }
            });
            msg[g] = lpsg::g_err;
            // the other shards may be blocked in an exchange with this one: say so now
            if (rc[g] != LPSG_OK) fprintf(stderr, "lpsg: shard %d failed: %s\n", g, msg[g].c_str());
        });
    }
    for (auto& t : th) t.join();
    for (int g = 0; g < shards; ++g)
        if (rc[g] != LPSG_OK) {
            lpsg::g_err = "shard " + std::to_string(g) + ": " + msg[g];
            return rc[g];
        }
    return LPSG_OK;
}

int lpsg_shard_range(int n, int world, int rank, int* lo, int* hi) {
    if (n < 0 || world < 1 || rank < 0 || rank >= world || !lo || !hi) return bad("lpsg_shard_range: bad argument");
    *lo = (int)((long long)n * rank / world);
    *hi = (int)((long long)n * (rank + 1) / world);
    return LPSG_OK;
}

int lpsg_comm_stats(lpsg_solver* s, long long* calls, double* bytes) {
    if (!s) return bad("lpsg_comm_stats: null solver");
    if (calls) *calls = s->comm ? s->comm->calls : 0;
    if (bytes) *bytes = s->comm ? s->comm->bytes : 0.0;
    return LPSG_OK;
}

int lpsg_shard_info(lpsg_solver* s, int* world, int* rank, int* row0, int* rows, int* col0, int* col1) {
    if (!s) return bad("lpsg_shard_info: null solver");
    const lpsg::Dev& d = s->s->dev();
    if (world) *world = d.world;
    if (rank) *rank = d.rank;
    if (row0) *row0 = d.row0;
    if (rows) *rows = d.mloc;
    if (col0) *col0 = d.col0;
    if (col1) *col1 = d.col1;
    return LPSG_OK;
}

int lpsg_two_phase_solve(const lpsg_problem* lp, const lpsg_config* cfg, lpsg_report* rep, double* x) {
    lpsg_solver* h = nullptr;
    int rc = lpsg_create(lp, cfg, &h);
    if (rc) return rc;
    rc = lpsg_solve(h, rep);
    if (!rc && x) rc = lpsg_get_x(h, x, lp->n_total);
    lpsg_destroy(h);
    return rc;
}

int lpsg_set_observer(lpsg_solver* s, lpsg_observer cb, void* user) {
    if (!s) return bad("lpsg_set_observer: null solver");
    s->s->observer = cb;
    s->s->observer_user = user;
    return LPSG_OK;
}

int lpsg_set_view_observer(lpsg_solver* s, lpsg_view_observer cb, void* user, int with_rows) {
    if (!s) return bad("lpsg_set_view_observer: null solver");
    s->s->view_observer = cb;
    s->s->view_user = user;
    s->s->view_rows = cb != nullptr && with_rows != 0;
    s->s->handle = s;
    return LPSG_OK;
}

int lpsg_get_memory(lpsg_solver* s, lpsg_memory* out) {
    if (!s || !out) return bad("lpsg_get_memory: null argument");
    *out = s->s->memory();
    return LPSG_OK;
}

int lpsg_reinvert_stats(lpsg_solver* s, long* rebuilds, long* steps, double* residual_before,
                        double* residual_after, double* seconds) {
    if (!s) return bad("lpsg_reinvert_stats: null solver");
    if (rebuilds) *rebuilds = s->s->reinv_count;
    if (steps) *steps = s->s->reinv_steps;
    if (residual_before) *residual_before = s->s->reinv_res_before;
    if (residual_after) *residual_after = s->s->reinv_res_after;
    if (seconds) *seconds = s->s->reinv_seconds;
    return LPSG_OK;
}

int lpsg_lookahead_stats(lpsg_solver* s, long long* bounded, long long* full, long long* price_bounded,
                         long long* price_exact, long long* probe_rounds) {
    if (!s) return bad("lpsg_lookahead_stats: null solver");
    if (probe_rounds) *probe_rounds = s->s->la_probe_rounds_;
    if (bounded) *bounded = s->s->la_bounded_;
    if (full) *full = s->s->la_full_;
    if (price_bounded) *price_bounded = s->s->la_price_bounded_;
    if (price_exact) *price_exact = s->s->la_price_exact_;
    return LPSG_OK;
}

int lpsg_keep_trace(lpsg_solver* s, int keep) {
    if (!s) return bad("lpsg_keep_trace: null solver");
    s->s->keep_trace = keep != 0;
    return LPSG_OK;
}

int lpsg_get_trace(lpsg_solver* s, lpsg_trace* out, long cap, long* len) {
    if (!s || !len) return bad("lpsg_get_trace: null argument");
    const auto& t = s->s->trace;
    *len = (long)t.size();
    if (out)
        for (long k = 0; k < std::min<long>(cap, *len); ++k) out[k] = t[k];
    return LPSG_OK;
}

int lpsg_price(lpsg_solver* s, int* optimal, int* entering, double* red) {
    if (!s || !optimal || !entering || !red) return bad("lpsg_price: null argument");
    return guard([&] { s->s->step_price(optimal, entering, red); });
}

int lpsg_compute_direction(lpsg_solver* s, int entering, double red) {
    if (!s) return bad("lpsg_compute_direction: null solver");
    return guard([&] { s->s->step_compute_direction(entering, red); });
}

int lpsg_ratio_test(lpsg_solver* s, int* unbounded, double* theta, int* cand, int cap, int* ncand) {
    if (!s || !unbounded || !theta || !ncand) return bad("lpsg_ratio_test: null argument");
    return guard([&] {
        std::vector<int> c;
        s->s->step_ratio(unbounded, theta, c);
        *ncand = (int)c.size();
        if (cand)
            for (int k = 0; k < std::min(cap, *ncand); ++k) cand[k] = c[k];
    });
}

int lpsg_select_leaving(lpsg_solver* s, const int* cand, int ncand, int entering, int* row) {
    if (!s || !cand || ncand <= 0 || !row) return bad("lpsg_select_leaving: bad argument");
    return guard([&] { *row = s->s->select_leaving(std::vector<int>(cand, cand + ncand), entering); });
}

int lpsg_lookahead_scores(lpsg_solver* s, const int* rows, int k, int entering, double* scores) {
    if (!s || !rows || k < 0 || !scores) return bad("lpsg_lookahead_scores: bad argument");
    return guard([&] {
        std::vector<double> sc;
        s->s->lookahead(std::vector<int>(rows, rows + k), entering, sc);
        std::copy(sc.begin(), sc.end(), scores);
    });
}

int lpsg_pivot_update(lpsg_solver* s, int r, int q) {
    if (!s) return bad("lpsg_pivot_update: null solver");
    return guard([&] { s->s->step_pivot(r, q); });
}

int lpsg_dims(lpsg_solver* s, int* m, int* n_total, int* n_work) {
    if (!s) return bad("lpsg_dims: null solver");
    if (m) *m = s->s->m();
    if (n_total) *n_total = s->s->n_total();
    if (n_work) *n_work = s->s->n_work();
    return LPSG_OK;
}

int lpsg_read_row(lpsg_solver* s, int i, double* out) {
    if (!s || !out) return bad("lpsg_read_row: null argument");
    return guard([&] { s->s->read_row(i, out); });
}

int lpsg_basis(lpsg_solver* s, int* basic, int m) {
    if (!s || !basic || m != s->s->m()) return bad("lpsg_basis: bad argument");
    std::copy(s->s->basic().begin(), s->s->basic().end(), basic);
    return LPSG_OK;
}

int lpsg_phase(lpsg_solver* s) { return s ? s->s->phase() : -1; }

int lpsg_set_max_iter(lpsg_solver* s, long max_iter) {
    if (!s) return bad("lpsg_set_max_iter: null solver");
    return guard([&] { s->s->set_max_iter(max_iter); });
}

int lpsg_profile(lpsg_solver* s, int enable) {
    if (!s) return bad("lpsg_profile: null solver");
    return guard([&] { s->s->set_profile(enable != 0); });
}

int lpsg_profile_get(lpsg_solver* s, lpsg_kernel_stat* out, int cap, int* n) {
    if (!s || !n) return bad("lpsg_profile_get: null argument");
    static const char* names[] = {"ratio", "pivot", "price", "update_ftran", "other", "exchange",
                                  "lookahead_price", "lookahead_theta"};
    static_assert(sizeof(names) / sizeof(names[0]) == lpsg::Solver::K_NUM, "kernel kind names");
    *n = lpsg::Solver::K_NUM;
    for (int k = 0; out && k < std::min(cap, (int)lpsg::Solver::K_NUM); ++k) {
        out[k].name = names[k];
        out[k].launches = s->s->kstat[k].launches;
        out[k].milliseconds = s->s->kstat[k].ms;
        out[k].algorithmic_bytes = s->s->kstat[k].bytes;
    }
    return LPSG_OK;
}

int lpsg_fp64_peak(int device, double* tflops) {
    if (!tflops) return bad("lpsg_fp64_peak: null argument");
    return guard([&] {
        CK_SET_DEVICE(device);
        *tflops = lpsg::fp64_probe_tflops(0);
        if (*tflops <= 0.0) throw lpsg::Error(LPSG_CUDA_ERROR, "lpsg_fp64_peak: probe failed");
    });
}

int lpsg_host_alloc(size_t bytes, void** out) {
    if (!out) return bad("lpsg_host_alloc: null argument");
    return guard([&] {
        const cudaError_t e = cudaHostAlloc(out, std::max<size_t>(bytes, 16), cudaHostAllocPortable);
        if (e != cudaSuccess) {
            cudaGetLastError();
            throw lpsg::Error(LPSG_CUDA_ERROR, std::string("cudaHostAlloc: ") + cudaGetErrorString(e));
        }
    });
}

void lpsg_host_free(void* p) {
    if (p) cudaFreeHost(p);
}

int lpsg_last_solve_device_ms(lpsg_solver* s, double* ms) {
    if (!s || !ms) return bad("lpsg_last_solve_device_ms: null argument");
    *ms = s->s->last_device_ms;
    return LPSG_OK;
}

int lpsg_counters(lpsg_solver* s, long* launches, long long* h2d, long long* d2h) {
    if (!s) return bad("lpsg_counters: null solver");
    if (launches) *launches = s->s->launches_total;
    if (h2d) *h2d = s->s->h2d_bytes;
    if (d2h) *d2h = s->s->d2h_bytes;
    return LPSG_OK;
}

}  // extern "C"
