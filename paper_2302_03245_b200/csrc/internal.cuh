// internal.cuh -- shared definitions of libpushrank_cuda (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/pushrank_cuda.h"

namespace pr {

// Gauss-Seidel sections of a dense sweep (rounds.cu): at most this many
#define PR_MAX_SECTIONS 8
// Gauss-Seidel sections of a dense sweep from the round's working set ws
// (bytes) against L2 (rounds.cu "Gauss-Seidel sections"): none while the
// round is short (C2, C4), 2 past 1.5x L2 (C3: 3 / 4 sections 10.6 / 11.0 ms
// against 9.9), 6 past 16x (C5 IFP2 4 / 5 / 6 / 7 / 8 sections: 461 / 475 /
// 441 / 462 / 448 ms; IFP1 4 / 6 / 7: 491 / 451 / 489 ms)
static inline int gs_sections_default(double ws, double l2) { return ws > 16.0 * l2 ? 6 : ws > 1.5 * l2 ? 2 : 1; }

// ---------------------------------------------------------------- errors
void set_error(const std::string &msg);
int fail(int code, const std::string &msg);

#define PR_CUDA(call)                                                                      \
    do {                                                                                   \
        cudaError_t _e = (call);                                                           \
        if (_e != cudaSuccess)                                                             \
            return ::pr::fail(PR_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(_e) + \
                                               " (" + __FILE__ + ":" + std::to_string(__LINE__) + ")"); \
    } while (0)

#define PR_TRY(call)                   \
    do {                               \
        int _rc = (call);              \
        if (_rc != PR_OK) return _rc;  \
    } while (0)

// ---------------------------------------------------------------- device buffers
// Buffers come from the device's stream-ordered memory pool (cudaMallocAsync
// on the context stream, release threshold kept at "never"), so building a
// graph, its schedules and workspaces costs no cudaMalloc/cudaFree syncs.
// alloc_stream() is the stream of the context the current C-ABI call runs on.
cudaStream_t &alloc_stream();

struct DevBuf {
    void *ptr = nullptr;
    size_t bytes = 0;
    DevBuf() = default;
    DevBuf(const DevBuf &) = delete;
    DevBuf &operator=(const DevBuf &) = delete;
    ~DevBuf() { release(); }
    void release() {
        if (ptr) cudaFreeAsync(ptr, alloc_stream());
        ptr = nullptr;
        bytes = 0;
    }
    template <class T> T *as() const { return reinterpret_cast<T *>(ptr); }
};
// grows (never shrinks) a buffer; contents are not preserved
int ensure(DevBuf &b, size_t bytes);

struct Uploader;  // hostio.cu

struct Ctx {
    int device = 0;
    int sm_count = 148;
    size_t l2_bytes = 0;
    cudaStream_t stream = nullptr;
    DevBuf scratch;          // CUB temporaries
    DevBuf flush;            // L2 flush buffer (bench)
    // Instantiated round-loop graphs, keyed by the bytes of their launch plan
    // (every pointer, size and parameter the kernels receive).  The stream-
    // ordered pool hands a re-uploaded graph of the same shape the same
    // addresses, so a new pr_graph usually hits here and skips instantiation.
    struct ExecSlot {
        std::vector<unsigned char> key;
        cudaGraph_t graph = nullptr;
        cudaGraphExec_t exec = nullptr;
        uint64_t used = 0;
    } execs[8];
    uint64_t exec_tick = 0;
    // page-locked host side of the observed-run ring (sync_simulate's
    // on_iteration): grown on demand, freed with the context
    void *obs_host = nullptr;
    size_t obs_host_bytes = 0;
    // host threads, page-locked staging and copy streams of the pipelined
    // index upload (hostio.cu), created on the first large upload
    Uploader *up = nullptr;
};
void uploader_destroy(Ctx &ctx);
// int64 host indices -> int32 device array (hostio.cu); *h2d += PCIe bytes.
// extra: plain host -> device copies queued on the same copy lanes first.
struct RawCopy {
    void *dst;
    const void *src;
    size_t bytes;
};
int upload_narrow(Ctx &ctx, const int64_t *h, int64_t count, int32_t *d, int64_t *h2d,
                  const RawCopy *extra = nullptr, int n_extra = 0);
void release_execs(Ctx &ctx);

// Per-block partial statistics of one round (reduced in fixed order).
struct Partial {
    double l1, above, nd_above;
    int64_t conv_all, conv_scan, nact, work, push_ops, push_dang;
    uint64_t digest;
};

// Device-side control block of a round loop (one per run workspace).
struct RunCtl {
    int64_t round;            // index t of the state being drained next
    int64_t rows;             // rows produced
    int64_t push_ops, push_ops_dangling;
    int64_t pull_rounds, push_rounds;
    int64_t fsize[2];         // frontier sizes (ping-pong by round parity)
    int32_t mode;             // 0 pull, 1 push (for the next round)
    int32_t done;             // 1 = converged, 2 = max_rounds exhausted
    uint32_t blocks_done;     // last-block arrival counter
    int32_t append;           // record push items during the next epilogue
    uint64_t t0_ns;           // globaltimer at prologue
    double bytes;             // algorithmic bytes accumulated
    // constant contributions of vertices outside the round set (rows >= 1)
    double c_l1, c_above, c_nd_above;
    int64_t c_conv_all, c_conv_scan;
    double mass_total;
    int64_t settled;
    unsigned long long unit_ctr;  // pull-unit dispatch counter (bins.cuh), reset every round
    unsigned long long launches;  // kernels launched in this solve (each counts itself once)
    // per-kernel device timing (globaltimer): the first block of a round's
    // first kernel stamps t_k0, the finalising block closes the round
    uint32_t k_started;
    int32_t next_mode;        // mode of the round being timed (set when it was chosen)
    uint64_t t_k0;
    double next_bytes;        // algorithmic bytes of that round
    double pull_ns, pull_bytes, sparse_ns;
    // Gauss-Seidel sections (rounds.cu): statistics of the sections of the
    // current sweep, and the kind of the next round
    Partial sec_acc;
    int32_t gs;               // next pull round is a Gauss-Seidel sweep
    int32_t push_filter;      // next push round follows a GS sweep
    // observed exact runs (sync_simulate on_iteration): states snapshotted
    // into the ring since the batch began, and the round index of the first
    int64_t obs_count, obs_t0;
};


struct Graph {
    Ctx *ctx = nullptr;
    int64_t n = 0, m = 0, raw = 0;
    int64_t h2d_bytes = 0;   // bytes copied host -> device by pr_graph_upload / attach_out_targets
    DevBuf orig_ids;  // int64 [n] first-appearance id table (ingest.cu); empty = identity
    // run layout only: vertices [live_end, n) are the dangling ones (classes
    // out=0&in>0, isolated), so their in-edges are the CSC tail
    int64_t live_end = -1;
    int64_t class0_end = -1;   // run layout: [0, class0_end) have in>0 & out>0
    DevBuf out_off;   // int64 [n+1]
    DevBuf out_tgt;   // int32 [m] (absent until attached when uploaded CSC-only)
    bool has_csr = true;
    DevBuf out_deg;   // int32 [n]
    DevBuf in_off;    // int64 [n+1]
    DevBuf in_src;    // int32 [m]
    // classification (pr_classify)
    bool classified = false;
    pr_class_counts counts{};
    DevBuf cls_flags;  // uint8 [n]: bit0 dangling, bit1 unreferenced, bit2 weak d, bit3 weak u
    // dangling target counts (IFP1 push_ops_dangling), int32 [n]
    bool has_dtc = false;
    DevBuf dtc;
    // IFP2 split (pr_preprocess_ifp2)
    bool has_ifp2 = false;       // split arrays built
    bool ifp2_counted = false;   // counts known (pr_preprocess_ifp2 ran)
    pr_ifp2_counts ifp2{};
    DevBuf live_off, live_tgt, live_deg;     // int64 [n+1], int32 [live_m], int32 [n]
    DevBuf dang_ids, src_off, src_ids;       // int32 [n_d], int64 [n_d+1], int32 [m_d]
    // Pull schedules, built lazily: [0] ifp1/fp-full destinations (in-degree
    // > 0), [1] ifp2 (non-dangling, in-degree > 0), [2] power (in-degree > 0;
    // the zero-in-degree vertices are listed separately).  Rows are ordered by
    // descending in-degree and cut into block units of near-equal cost --
    // hub-row chunks (rows > HUB_DEG), warp-row ranges (> THREAD_DEG),
    // thread-row ranges -- dealt round-robin to a persistent grid (bins.cuh).
    struct Sched {
        bool built = false;
        int64_t count = 0;        // |D|
        int64_t edges = 0;        // edges of the D rows
        int64_t n_hub = 0, n_warp = 0;    // rows [0,n_hub) hubs, [n_hub, n_hub+n_warp) warp rows
        int64_t n_chunks = 0;     // CHUNK-edge units of the hub rows
        DevBuf ids;               // int32 [|D|] vertex id of each row (descending in-degree)
        DevBuf doff;              // int64 [|D|+1] compacted CSC offsets
        DevBuf csc;               // int32 compacted sources: hub and warp rows CSR (doff), thread
                                  // rows SELL-32 (sell_off), then CSC_PAD
        int64_t n_slices = 0;     // 32-row slices of the thread-row bin
        DevBuf sell_off;          // int64 [n_slices+1] csc offset of each slice (column-major, 32 wide)
        DevBuf chunk_base;        // int64 [n_hub+1] first chunk of each hub row
        DevBuf row_cum;           // int64 [|D|+1] exclusive prefix of row costs (edges + ROW_COST)
        int64_t unit_blocks = 0;  // grid size the units below were cut for
        int nsec = 0;             // Gauss-Seidel sections the units were cut for
        int64_t sec_row[PR_MAX_SECTIONS + 1] = {};   // section row bounds (equal edges)
        int64_t sec_unit[PR_MAX_SECTIONS + 1] = {};  // section unit bounds
        int64_t sec_id[PR_MAX_SECTIONS + 1] = {};    // IFP1: id bound of earlier sections' sources
        DevBuf sec_of;            // IFP1: uint8 [n] section of each vertex's row (255: not a row)
        int64_t n_units = 0;
        DevBuf units;             // int2 [n_units]: (row_begin, row_end) or hub chunk (row, -(chunk+1))
        DevBuf row_cnt;           // int32 [n_hub] chunk arrival counters
        DevBuf chunk_part;        // double [n_chunks] chunk partial sums
        int64_t n_zero = 0;       // power: in-degree-0 vertices
        DevBuf zero_ids;
        int64_t n_seed = 0;       // vertices outside D active at round 0 (scatter seeds)
        DevBuf seed_ids;          // int32
    } sched[3];
    // run workspace
    DevBuf h, reserved, s2, act, in_d, frontier2, partials, ctl, rows;
    DevBuf obs_ring;          // observed exact runs: K (reserved, pending) snapshots
    int64_t rows_cap = 0;
    int64_t max_blocks = 0;     // partial slots per region (partials holds 3 regions)
    int64_t n_dangling = -1;    // #(out_degree == 0), computed lazily
    int64_t settle_big = -1;    // leading dangling vertices with > 32 sources (run layout)
    DevBuf pw;                // power-method workspace
    // Run layout of the fast engines (graph.cu): the same graph with
    // vertices renumbered by class (in>0&out>0 | out>0&in=0 | out=0&in>0 |
    // isolated) and, inside the receiving classes, by descending in-degree:
    // pull rows of similar degree are adjacent (uniform warps), hot sources
    // (in/out degrees correlate on power-law graphs) are dense in L1/L2, and
    // the IFP2 destination set is a contiguous id range.  Exact mode keeps
    // the original layout (bit-exact summation order).
    Graph *run = nullptr;
    Graph *orig = nullptr;    // run layout: the graph it was built from (non-owning)
    // run layout: its CSC rows' sources are sorted ascending (HBM-bound
    // graphs, graph.cu) before the second fast solve -- a graph solved once
    // (the e2e path) does not pay the segmented sort (~100 ms at C5) for a
    // ~4% faster solve
    bool sort_deferred = false;
    int64_t fast_solves = 0;
    DevBuf perm;              // int32 [n]: run id -> original id
    DevBuf rank;              // int32 [n]: original id -> run id
    ~Graph();
};

int ensure_dtc(Graph &g);
int need_csr(const Graph &g, const char *what);
int attach_out_targets(Graph &g, const int64_t *out_tgt);
int count_dangling(Graph &g);
int ensure_run_layout(Graph &g);
int ensure_run_csr(Graph &r);
int ensure_sched(Graph &g, int which);
// sort the sources of every CSC row ascending (in place; segmented radix sort)
int sort_csc_rows(Ctx &ctx, const DevBuf &in_off, DevBuf &in_src, int64_t n, int64_t m);
int ensure_units(Graph &g, int which, int64_t blocks, int nsec = 1);
int load_edge_list_device(Ctx &ctx, const char *text, int64_t len, Graph **out);
int rank_order(Ctx &ctx, const double *h_values, const int64_t *h_ids, int64_t n, int64_t k, int64_t *h_order);
int write_ranking_csv(Ctx &ctx, const double *values, const int64_t *ids, int64_t n, const char *path);
int format_score(double x, char *out);
int graph_from_raw_ids(Ctx &ctx, const int64_t *src, const int64_t *dst, int64_t m, Graph **out);
int build_from_device_edges(Ctx &ctx, int64_t n, const int64_t *d_src, const int64_t *d_dst,
                            int64_t m_raw, Graph **out);
int classify_device(Graph &g);
int preprocess_ifp2_device(Graph &g);
int ifp2_counts_device(Graph &g);
int run_rounds(Graph &g, const pr_run_params &p, double *d_values, double *d_reserved, double *d_pending,
               pr_round_stats *rows,
               int64_t row_cap, pr_run_result *res);
int power_device(Graph &g, double damping, int64_t iterations, double tolerance, double threshold,
                 const double *h_personalization, double *h_pi, double *h_deltas, int64_t *h_converged,
                 int (*on_iterate)(void *, int64_t, const double *), void *user, pr_run_result *res,
                 const double *d_ref = nullptr, double target_err = 0.0, int64_t *hit = nullptr);
int error_report(Ctx &ctx, const double *d_est, const double *d_ref, int64_t n, double *max_rel, double *l1,
                 int64_t *worst, int64_t *nonpositive);

constexpr int TILE = 256;   // edges per warp tile (long rows are cut into TILE chunks)
constexpr int CSC_PAD = 1024;  // int32 padding past the compacted CSC for vector loads
// Measured against 32 (bench.py, B200): C2 -1%, C3 -10%, C5 -6%, C4 0;
// 16 and 256 are worse (C2 +23% / +30%), 96 and 128 within 1% of 64.
#ifndef PR_THREAD_DEG
#define PR_THREAD_DEG 64
#endif
constexpr int64_t THREAD_DEG = PR_THREAD_DEG;   // rows up to this in-degree: one thread each
#ifndef PR_HUB_CHUNK
#define PR_HUB_CHUNK 16384
#endif
// thread-row bin stored SELL-32 (sched.cu sell_layout); 0 = row-major CSR (A/B builds)
#ifndef PR_SELL
#define PR_SELL 1
#endif
#ifndef PR_DYNAMIC_UNITS
#define PR_DYNAMIC_UNITS 1
#endif
#ifndef PR_UNITS_PB
#define PR_UNITS_PB 8
#endif
#ifndef PR_HUB_DEG
#define PR_HUB_DEG 4096
#endif
constexpr int64_t HUB_DEG = PR_HUB_DEG;        // rows above: cut into HUB_CHUNK-edge block units
constexpr int64_t HUB_CHUNK = PR_HUB_CHUNK;    // edges per hub unit, summed HUB_STEP at a time
constexpr int64_t HUB_STEP = 4096;             // 256 threads x 16 gathers in flight
static_assert(PR_HUB_CHUNK % 4096 == 0, "hub chunks are whole steps");
constexpr int64_t ROW_COST = 8;                // per-row drain cost in edge units (unit sizing)
constexpr int64_t UNITS_PER_BLOCK = PR_UNITS_PB;  // target work units per block of the persistent grid
constexpr int64_t LONG_UNIT = 100000;           // edge-units: past this, UNITS_PER_BLOCK per section
#ifndef PR_MIN_UNIT
#define PR_MIN_UNIT 10000
#endif

// PUSHRANK_TIMING=1: host-side phase timings (synchronising) on stderr
void phase_mark(cudaStream_t st, const char *what);

// small helpers
inline unsigned grid_for(int64_t items, int per_block) {
    int64_t b = (items + per_block - 1) / per_block;
    return (unsigned)(b < 1 ? 1 : b);
}

}  // namespace pr
