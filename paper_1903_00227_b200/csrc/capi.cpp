// paper_1903_00227_b200/csrc/capi.cpp -- the C ABI of include/wrs.h and
// include/wrs_b200.h on top of the sm_100a kernels.
//
// Mirrors the reference's ABI conventions (capi.cpp:53-75 in the reference):
// every call returns a wrs_status, exceptions never cross the boundary, the
// failure text is kept per thread for wrs_last_error().  CUDA failures map to
// WRS_ENOMEM (allocation) or WRS_EINTERNAL.  There is no CPU compute path:
// a missing or unusable GPU makes every compute call fail loudly.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>  // types only: libnccl.so.2 is dlopen'ed by the multi-GPU calls

#include <algorithm>
#include <atomic>
#include <thread>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <memory>
#include <mutex>
#include <new>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "engine.h"
#include "wrs.h"
#include "wrs_b200.h"

namespace {

using wrsb::Bucket;

// ---- error plumbing ----------------------------------------------------------
struct io_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct format_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct cuda_error : std::runtime_error {
    cudaError_t code;
    cuda_error(cudaError_t c, const std::string& what)
        : std::runtime_error(what + ": " + cudaGetErrorString(c)), code(c) {}
};

thread_local std::string t_last_error = "no error";

wrs_status fail(wrs_status code, std::string msg) {
    t_last_error = std::move(msg);
    return code;
}

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        cudaGetLastError();  // clear sticky-free errors
        throw cuda_error(e, what);
    }
}

template <typename F>
wrs_status guarded(F&& f) {
    try {
        return f();
    } catch (const std::bad_alloc&) {
        return fail(WRS_ENOMEM, "out of memory");
    } catch (const cuda_error& e) {
        return fail(e.code == cudaErrorMemoryAllocation ? WRS_ENOMEM : WRS_EINTERNAL, e.what());
    } catch (const format_error& e) {
        return fail(WRS_EFORMAT, e.what());
    } catch (const io_error& e) {
        return fail(WRS_EIO, e.what());
    } catch (const std::invalid_argument& e) {
        return fail(WRS_EINVAL, e.what());
    } catch (const std::exception& e) {
        return fail(WRS_EINTERNAL, e.what());
    }
}

std::atomic<int> g_timing{0};

// ---- device buffers ------------------------------------------------------------
struct DevBuf {
    void* p = nullptr;
    DevBuf() = default;
    explicit DevBuf(size_t bytes) { ck(wrsb::dev_malloc(&p, bytes ? bytes : 16), "cudaMalloc"); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() {
        if (p) wrsb::dev_free(p);
    }
};

struct Stream {
    cudaStream_t s = nullptr;
    Stream() { ck(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "cudaStreamCreate"); }
    // prio > 0: the device's greatest priority, prio < 0: its least
    explicit Stream(int prio) {
        int least = 0, greatest = 0;
        ck(cudaDeviceGetStreamPriorityRange(&least, &greatest), "priority range");
        ck(cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, prio > 0 ? greatest : least),
           "cudaStreamCreate");
    }
    ~Stream() {
        if (s) cudaStreamDestroy(s);
    }
};

int current_device() {
    int d = 0;
    ck(cudaGetDevice(&d), "cudaGetDevice");
    return d;
}

// Validated weights resident in HBM (weights.hpp:30-64 semantics).
struct WeightsData {
    int device = 0;
    uint64_t n = 0;
    double* d_w = nullptr;
    bool owned = true;
    double total = 0.0;
    std::unique_ptr<DevBuf> storage;
    // set when the values were written or read by work this library did not
    // synchronise itself (device-to-device copies, caller-stream rebuilds):
    // freeing them then waits for the whole device
    std::atomic<bool> ext{false};
    ~WeightsData() {
        wrsb::SyncedFrees synced;
        if (!ext.load()) synced.arm();
        storage.reset();
    }
    mutable std::mutex host_mu;
    mutable std::vector<double> host;  // lazily materialised values()
    mutable bool host_ready = false;

    const double* host_values() const {
        std::lock_guard<std::mutex> g(host_mu);
        if (!host_ready) {
            host.resize(n);
            ck(cudaSetDevice(device), "cudaSetDevice");
            ck(cudaMemcpy(host.data(), d_w, n * sizeof(double), cudaMemcpyDeviceToHost),
               "weights D2H");
            host_ready = true;
        }
        return host.data();
    }
};

// K0 on the device: validation + pairwise total; throws the reference's
// exception for a bad weight (weights.hpp:38-41 / weight_file.hpp:94-96).
void finalize_weights(WeightsData& wd, const std::string& file_for_format_error) {
    if (wd.n == 0) throw std::invalid_argument("weights: need at least one item");
    wrsb::Workspace ws;
    ck(wrsb::workspace_alloc_total(ws, wd.n), "workspace");
    wrsb::SyncedFrees synced;  // destroyed after guard: covers its frees
    struct Guard {
        wrsb::Workspace& w;
        ~Guard() { wrsb::workspace_free(w); }
    } guard{ws};
    Stream st;
    ck(wrsb::launch_total(wd.d_w, wd.n, ws, st.s), "K0 launch");
    wrsb::DevScalars sc{};
    ck(cudaMemcpyAsync(&sc, ws.sc, sizeof sc, cudaMemcpyDeviceToHost, st.s), "scalars D2H");
    ck(cudaStreamSynchronize(st.s), "K0");
    synced.arm();
    if (sc.bad_index != ~0ull) {
        if (!file_for_format_error.empty())
            throw format_error("weight " + std::to_string(sc.bad_index) +
                               " not finite/positive: " + file_for_format_error);
        throw std::invalid_argument("weights: item " + std::to_string(sc.bad_index) +
                                    " is not finite and positive");
    }
    wd.total = sc.total;
}

std::shared_ptr<WeightsData> weights_from_host(const double* w, uint64_t n,
                                               const std::string& file = "") {
    auto wd = std::make_shared<WeightsData>();
    wd->device = current_device();
    wd->n = n;
    if (n == 0) throw std::invalid_argument("weights: need at least one item");
    wd->storage = std::make_unique<DevBuf>(n * sizeof(double));
    wd->d_w = static_cast<double*>(wd->storage->p);
    {
        // on a non-blocking stream, not the legacy one: a synchronous legacy
        // copy was measured waiting behind another host thread's draw
        // downloads, while PCIe carries both directions at once
        Stream st;
        ck(cudaMemcpyAsync(wd->d_w, w, n * sizeof(double), cudaMemcpyHostToDevice, st.s),
           "weights H2D");
        ck(cudaStreamSynchronize(st.s), "weights H2D");
    }
    finalize_weights(*wd, file);
    return wd;
}

// Power-law weights (weight_file.hpp:42-54): (i+1)^-s in order, then the
// reference's Fisher-Yates with RngStream(seed, 'genp').bounded(i).  The
// shuffle is inherently sequential, so it runs once on the host as input
// preparation; the result is uploaded and never recomputed.
std::vector<double> powerlaw_host(uint64_t n, double s, uint64_t seed) {
    if (!(s >= 0.0) || !std::isfinite(s))
        throw std::invalid_argument("power law exponent must be finite and >= 0");
    std::vector<double> w(n);
    for (uint64_t i = 0; i < n; ++i) w[i] = std::pow(static_cast<double>(i + 1), -s);
    const uint64_t key = wrsb::rng_key(seed, 0x67656e70u);
    uint64_t ctr = 0;
    for (uint64_t i = n; i > 1; --i) {
        ctr += wrsb::kGolden;
        const uint64_t r = wrsb::mix64(key + ctr);
        const uint64_t j = static_cast<uint64_t>((static_cast<unsigned __int128>(r) * i) >> 64);
        std::swap(w[i - 1], w[j]);
    }
    return w;
}

// Power-law weights with the shuffle on the device (generate_kernels.cu):
// the powers (i+1)^-s with the host's libm pow in parallel threads (bit-equal
// to the reference's std::pow), then the deal resolved on the GPU.
std::shared_ptr<WeightsData> powerlaw_device(uint64_t n, double s, uint64_t seed) {
    if (!(s >= 0.0) || !std::isfinite(s))
        throw std::invalid_argument("power law exponent must be finite and >= 0");
    if (n == 0) throw std::invalid_argument("weights: need at least one item");
    if (n > static_cast<uint64_t>(std::numeric_limits<int>::max())) {
        const auto w = powerlaw_host(n, s, seed);
        return weights_from_host(w.data(), n);
    }
    std::vector<double> pw(n);
    const unsigned T = std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
    std::vector<std::thread> th;
    for (unsigned t = 0; t < T; ++t)
        th.emplace_back([&, t] {
            const uint64_t lo = n * t / T, hi = n * (t + 1) / T;
            for (uint64_t i = lo; i < hi; ++i) pw[i] = std::pow(static_cast<double>(i + 1), -s);
        });
    for (auto& x : th) x.join();
    auto wd = std::make_shared<WeightsData>();
    wd->device = current_device();
    wd->n = n;
    wd->storage = std::make_unique<DevBuf>(n * sizeof(double));
    wd->d_w = static_cast<double*>(wd->storage->p);
    {
        DevBuf tmp(n * sizeof(double));
        ck(cudaMemcpy(tmp.p, pw.data(), n * sizeof(double), cudaMemcpyHostToDevice), "H2D");
        Stream st;
        ck(wrsb::fisher_yates_device(static_cast<const double*>(tmp.p), wd->d_w, n,
                                     wrsb::rng_key(seed, 0x67656e70u), st.s),
           "power-law deal");
    }
    finalize_weights(*wd, "");
    return wd;
}

// WRS_B200_PSA_EXACT=1 makes "psa" honour `workers` as the job count, so an
// unmodified reference client gets the reference's table (and draw stream)
// byte for byte without switching to "psa-exact".
bool psa_exact_env() {
    const char* e = std::getenv("WRS_B200_PSA_EXACT");
    return e && e[0] == '1';
}

// configs[3]'s lognormal(0, sigma) weights, items [offset, offset + n) of the
// global vector (counter-based: only the slice is generated).
std::shared_ptr<WeightsData> lognormal_device(uint64_t n, uint64_t offset, double sigma,
                                              uint64_t seed) {
    if (!(sigma >= 0.0) || !std::isfinite(sigma) || sigma > 30.0)
        throw std::invalid_argument("lognormal sigma must be in [0, 30]");
    if (n == 0) throw std::invalid_argument("weights: need at least one item");
    auto wd = std::make_shared<WeightsData>();
    wd->device = current_device();
    wd->n = n;
    wd->storage = std::make_unique<DevBuf>(n * sizeof(double));
    wd->d_w = static_cast<double*>(wd->storage->p);
    Stream st;
    ck(wrsb::launch_generate_lognormal(wd->d_w, n, offset, seed, sigma, st.s), "generate");
    ck(cudaStreamSynchronize(st.s), "generate");
    finalize_weights(*wd, "");
    return wd;
}

}  // namespace

struct wrs_weights {
    std::shared_ptr<WeightsData> data;
};

struct wrs_sampler {
    std::shared_ptr<WeightsData> weights;  // retained for verification (capi.cpp:42)
    std::string algo;
    int device = 0;
    uint64_t n = 0, P = 1;
    double total = 0.0, wn = 0.0;
    std::unique_ptr<DevBuf> buckets;
    std::unique_ptr<Stream> stream;
    wrsb::Workspace ws;
    bool keep_ws = false;
    cudaEvent_t ev[8] = {};
    bool timed = false;
    // set once any call ran this sampler's work on a caller's stream: the
    // destructor then cannot know when that work ends and frees with a
    // device-wide wait (otherwise it synchronises its own streams only)
    mutable std::atomic<bool> ext_stream{false};
    std::mutex mu;  // rebuild / stage access
    // draw scratch (region plan), reused across draws; sws_ev orders users
    mutable wrsb::SampleWorkspace sws;
    mutable wrsb::CountWorkspace cws;  // aggregated draws (guarded by sws_mu)
    mutable std::mutex sws_mu;
    mutable cudaEvent_t sws_ev = nullptr;
    // side stream for the table-independent first stage of a draw (the
    // region scatter), so it overlaps a rebuild queued before the draw
    mutable std::unique_ptr<Stream> side;
    mutable cudaEvent_t side_ev = nullptr;
    // rebuilds run on a high-priority stream (event handoff from / to the
    // caller's stream) so their CTAs win the SMs over a concurrent scatter
    std::unique_ptr<Stream> hi;
    cudaEvent_t hi_ev[2] = {};

    ~wrs_sampler() {
        if (device >= 0) cudaSetDevice(device);
        wrsb::SyncedFrees synced;
        if (!ext_stream.load()) {
            bool ok = true;
            for (Stream* st : {stream.get(), side.get(), hi.get()})
                if (st) ok = ok && cudaStreamSynchronize(st->s) == cudaSuccess;
            if (ok) synced.arm();
        } else if (weights) {
            weights->ext = true;
        }
        wrsb::workspace_free(ws);
        if (sws_ev) cudaEventSynchronize(sws_ev), cudaEventDestroy(sws_ev);
        if (side_ev) cudaEventSynchronize(side_ev), cudaEventDestroy(side_ev);
        side.reset();
        for (cudaEvent_t& e : hi_ev)
            if (e) cudaEventSynchronize(e), cudaEventDestroy(e);
        hi.reset();
        sws.release();
        cws.release();
        for (cudaEvent_t& e : ev)
            if (e) cudaEventDestroy(e);
        for (int b = 0; b < 2; ++b) {
            if (built_ev[b]) cudaEventSynchronize(built_ev[b]), cudaEventDestroy(built_ev[b]);
            if (read_ev[b]) cudaEventSynchronize(read_ev[b]), cudaEventDestroy(read_ev[b]);
        }
        buckets.reset();  // inside the SyncedFrees scope
        buckets2.reset();
        weights.reset();
    }
    // Double-buffered tables (wrs_b200_sampler_double_buffer): rebuilds write
    // the back table while draws already issued still read the front one;
    // built_ev[b] marks table b written, read_ev[b] the end of the last draw
    // that read it.  `front` flips when a rebuild is issued.
    std::unique_ptr<DevBuf> buckets2;
    std::atomic<int> front{0};
    bool dbuf = false;
    mutable cudaEvent_t built_ev[2] = {};
    mutable cudaEvent_t read_ev[2] = {};
    Bucket* table(int b) const { return static_cast<Bucket*>((b ? buckets2 : buckets)->p); }
    Bucket* d_b() const { return table(front.load()); }
    // host-side accesses of the front table wait for the rebuild that wrote it
    void sync_table() const {
        if (dbuf) ck(cudaEventSynchronize(built_ev[front.load()]), "table ready");
    }
};

namespace {

// The stream a call runs on: the caller's (marking the sampler, see
// ext_stream) or the sampler's own.
cudaStream_t use_stream(const wrs_sampler& s, void* stream) {
    if (!stream) return s.stream->s;
    s.ext_stream = true;
    return static_cast<cudaStream_t>(stream);
}

void read_scalars(wrs_sampler& s) {
    wrsb::DevScalars sc{};
    ck(cudaMemcpyAsync(&sc, s.ws.sc, sizeof sc, cudaMemcpyDeviceToHost, s.stream->s),
       "scalars D2H");
    ck(cudaStreamSynchronize(s.stream->s), "PSA build");
    if (sc.plan_error) throw std::logic_error("alias split boundaries must be nondecreasing");
    s.total = sc.total;
    s.wn = sc.wn;
}

std::unique_ptr<wrs_sampler> build_psa(const std::shared_ptr<WeightsData>& wd, uint64_t P,
                                       unsigned flags, const char* algo) {
    if (wd->n > std::numeric_limits<uint32_t>::max())
        throw std::invalid_argument("alias table limited to 2^32-1 items");
    ck(cudaSetDevice(wd->device), "cudaSetDevice");
    auto s = std::make_unique<wrs_sampler>();
    s->weights = wd;
    s->algo = algo;
    s->device = wd->device;
    s->n = wd->n;
    s->P = P ? P : 1;
    s->keep_ws = flags & WRS_B200_KEEP_WORKSPACE;
    s->buckets = std::make_unique<DevBuf>(wd->n * sizeof(Bucket));
    s->stream = std::make_unique<Stream>();
    ck(wrsb::workspace_alloc(s->ws, s->n, s->P, s->keep_ws), "workspace");
    ck(wrsb::launch_psa_build(wd->d_w, s->n, wd->total, s->P, s->d_b(), s->ws, s->stream->s,
                              nullptr),
       "PSA launch");
    read_scalars(*s);
    if (!s->keep_ws) {
        wrsb::SyncedFrees synced;  // read_scalars synchronised the build stream
        synced.arm();
        wrsb::workspace_free(s->ws);
    }
    return s;
}

// One draw launch on stream st; the sampler's draw scratch is handed from
// one draw to the next through sws_ev, so draws on different streams never
// share it concurrently.
void sample_on(const wrs_sampler& s, uint64_t seed, uint64_t q0, uint64_t q1, uint64_t k,
               uint32_t workers, uint32_t base, uint32_t* out, cudaStream_t st,
               uint64_t stream_id = wrsb::kSampleStream) {
    std::lock_guard<std::mutex> g(s.sws_mu);
    if (!s.sws_ev) {
        ck(cudaEventCreateWithFlags(&s.sws_ev, cudaEventDisableTiming), "event");
        ck(cudaEventCreateWithFlags(&s.side_ev, cudaEventDisableTiming), "event");
        s.side = std::make_unique<Stream>();
    }
    ck(cudaStreamWaitEvent(st, s.sws_ev, 0), "wait");
    ck(cudaStreamWaitEvent(s.side->s, s.sws_ev, 0), "wait");
    const int tb = s.front.load();
    if (s.dbuf) ck(cudaStreamWaitEvent(st, s.built_ev[tb], 0), "wait");
    // The first scatter of a draw does not read the table, so it may run on
    // the side stream under a preceding rebuild (WRS_B200_SIDE_SCATTER=1).
    // Off by default: with both bandwidth-bound, the bench step measured
    // 10.71 ms with the overlap vs 10.68 ms without.
    const char* side_env = std::getenv("WRS_B200_SIDE_SCATTER");
    const bool side_off = !(side_env && side_env[0] == '1');
    ck(wrsb::launch_sample(s.table(tb), s.n, s.wn, seed, stream_id, q0, q1, k, workers,
                           base, out, st, &s.sws, side_off ? nullptr : s.side->s,
                           side_off ? nullptr : s.side_ev),
       "K5 launch");
    ck(cudaEventRecord(s.sws_ev, st), "event");
    if (s.dbuf) ck(cudaEventRecord(s.read_ev[tb], st), "event");
}

// Aggregated draws on stream st, ordered with the other users of the draw
// scratch like sample_on (the counting plan has no table-independent prefix
// worth a side stream: its scatter is a third of the work).
void count_on(const wrs_sampler& s, uint64_t seed, uint64_t k, uint32_t workers, uint32_t* d_items,
              uint64_t* d_counts, uint64_t* d_n_unique, cudaStream_t st) {
    std::lock_guard<std::mutex> g(s.sws_mu);
    if (!s.sws_ev) {
        ck(cudaEventCreateWithFlags(&s.sws_ev, cudaEventDisableTiming), "event");
        ck(cudaEventCreateWithFlags(&s.side_ev, cudaEventDisableTiming), "event");
        s.side = std::make_unique<Stream>(-1);
    }
    ck(cudaStreamWaitEvent(st, s.sws_ev, 0), "wait");
    const int tb = s.front.load();
    if (s.dbuf) ck(cudaStreamWaitEvent(st, s.built_ev[tb], 0), "wait");
    ck(wrsb::launch_count(s.table(tb), s.n, s.wn, seed, wrsb::kSampleStream, k, workers, st,
                          &s.sws, &s.cws, d_items, d_counts,
                          reinterpret_cast<unsigned long long*>(d_n_unique)),
       "count launch");
    ck(cudaEventRecord(s.sws_ev, st), "event");
    if (s.dbuf) ck(cudaEventRecord(s.read_ev[tb], st), "event");
}

// Synchronous aggregated draws into host or device buffers of min(k, n).
void draw_counts(const wrs_sampler& s, uint64_t seed, uint64_t k, unsigned workers,
                 uint32_t* items, uint64_t* counts, uint64_t* n_unique);

bool is_device_pointer(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// Draw positions [0, count) to a host buffer: chunks are drawn into two device
// buffers and copied back on a second stream so the D2H of chunk c overlaps
// the draw of chunk c+1.
void draw_to_host(const wrs_sampler& s, uint64_t seed, uint64_t count, unsigned workers,
                  uint32_t* out) {
    // chunks of 2^26 draws: the copy-out (the bound, ~55 GB/s over PCIe)
    // starts after one small chunk's draw instead of a 2^28-draw one; the
    // extra table sweeps stay hidden under the copies
    const uint64_t chunk = std::min<uint64_t>(count, 1ull << 26);
    wrsb::SyncedFrees synced;  // armed once both streams are drained
    DevBuf b0(chunk * 4), b1(chunk * 4);
    uint32_t* bufs[2] = {static_cast<uint32_t*>(b0.p), static_cast<uint32_t*>(b1.p)};
    Stream copy;
    cudaEvent_t drawn[2], copied[2];
    for (int i = 0; i < 2; ++i) {
        ck(cudaEventCreateWithFlags(&drawn[i], cudaEventDisableTiming), "event");
        ck(cudaEventCreateWithFlags(&copied[i], cudaEventDisableTiming), "event");
        ck(cudaEventRecord(copied[i], copy.s), "event");
    }
    struct EvGuard {
        cudaEvent_t* a;
        cudaEvent_t* b;
        ~EvGuard() {
            for (int i = 0; i < 2; ++i) {
                cudaEventDestroy(a[i]);
                cudaEventDestroy(b[i]);
            }
        }
    } eg{drawn, copied};
    int c = 0;
    for (uint64_t q = 0; q < count; q += chunk, c ^= 1) {
        const uint64_t e = std::min(count, q + chunk);
        ck(cudaStreamWaitEvent(s.stream->s, copied[c], 0), "wait");
        sample_on(s, seed, q, e, count, workers, 0, bufs[c], s.stream->s);
        ck(cudaEventRecord(drawn[c], s.stream->s), "event");
        ck(cudaStreamWaitEvent(copy.s, drawn[c], 0), "wait");
        ck(cudaMemcpyAsync(out + q, bufs[c], (e - q) * 4, cudaMemcpyDeviceToHost, copy.s), "D2H");
        ck(cudaEventRecord(copied[c], copy.s), "event");
    }
    ck(cudaStreamSynchronize(copy.s), "draw");
    ck(cudaStreamSynchronize(s.stream->s), "draw");
    synced.arm();
}

void draw_counts(const wrs_sampler& s, uint64_t seed, uint64_t k, unsigned workers,
                 uint32_t* items, uint64_t* counts, uint64_t* n_unique) {
    const uint64_t cap = std::min(k, s.n);
    const bool dev = is_device_pointer(items) && is_device_pointer(counts);
    std::unique_ptr<DevBuf> bi, bc;
    uint32_t* d_items = items;
    uint64_t* d_counts = counts;
    if (!dev) {
        bi = std::make_unique<DevBuf>(std::max<uint64_t>(cap, 1) * sizeof(uint32_t));
        bc = std::make_unique<DevBuf>(std::max<uint64_t>(cap, 1) * sizeof(uint64_t));
        d_items = static_cast<uint32_t*>(bi->p);
        d_counts = static_cast<uint64_t*>(bc->p);
    }
    DevBuf nu(sizeof(uint64_t));
    count_on(s, seed, k, workers ? workers : 1, d_items, d_counts, static_cast<uint64_t*>(nu.p),
             s.stream->s);
    uint64_t m = 0;
    ck(cudaMemcpyAsync(&m, nu.p, sizeof m, cudaMemcpyDeviceToHost, s.stream->s), "D2H");
    ck(cudaStreamSynchronize(s.stream->s), "draw counts");
    if (!dev && m) {
        ck(cudaMemcpy(items, d_items, m * sizeof(uint32_t), cudaMemcpyDeviceToHost), "D2H");
        ck(cudaMemcpy(counts, d_counts, m * sizeof(uint64_t), cudaMemcpyDeviceToHost), "D2H");
    }
    *n_unique = m;
}

// implied_masses (verify.hpp:43-54) and max_relative_mass_error (:92-98) on
// the device, bit for bit (verify_kernels.cu); d_m may be null.
double implied_masses(const wrs_sampler& s, double* d_m) {
    s.sync_table();
    ck(cudaStreamSynchronize(s.stream->s), "sync");
    double worst = 0.0;
    ck(wrsb::implied_masses_device(s.d_b(), s.n, s.wn, s.weights->d_w, d_m, &worst,
                                   s.stream->s),
       "implied masses");
    return worst;
}

// Tables of 2^31 buckets or more (beyond the device sort's item count): the
// same Kahan sums on the host over a D2H copy of the table.
double max_rel_mass_error_host(const wrs_sampler& s) {
    std::vector<Bucket> b(s.n);
    s.sync_table();
    ck(cudaMemcpy(b.data(), s.d_b(), s.n * sizeof(Bucket), cudaMemcpyDeviceToHost), "table D2H");
    std::vector<double> sum(s.n, 0.0), comp(s.n, 0.0);
    auto kadd = [&](uint32_t i, double x) {  // kahan_sum::add, verify.hpp:28-33
        const double y = x - comp[i];
        const double t = sum[i] + y;
        comp[i] = (t - sum[i]) - y;
        sum[i] = t;
    };
    for (uint64_t i = 0; i < s.n; ++i) {
        kadd(b[i].item, b[i].share);
        kadd(b[i].alias, s.wn - b[i].share);
    }
    const double* w = s.weights->host_values();
    double worst = 0.0;
    for (uint64_t i = 0; i < s.n; ++i) worst = std::max(worst, std::abs(sum[i] - w[i]) / w[i]);
    return worst;
}

double max_rel_mass_error(const wrs_sampler& s) {
    if (s.n > static_cast<uint64_t>(std::numeric_limits<int>::max())) return max_rel_mass_error_host(s);
    return implied_masses(s, nullptr);
}

}  // namespace

// =============================================================================
extern "C" {

const char* wrs_last_error(void) { return t_last_error.c_str(); }

const char* wrs_status_name(wrs_status status) {
    switch (status) {
        case WRS_OK: return "WRS_OK";
        case WRS_EINVAL: return "WRS_EINVAL";
        case WRS_EIO: return "WRS_EIO";
        case WRS_EFORMAT: return "WRS_EFORMAT";
        case WRS_EVERIFY: return "WRS_EVERIFY";
        case WRS_ENOMEM: return "WRS_ENOMEM";
        case WRS_EINTERNAL: return "WRS_EINTERNAL";
    }
    return "WRS_UNKNOWN";
}

// ---- weights ---------------------------------------------------------------------
wrs_status wrs_weights_from_array(const double* w, uint64_t n, wrs_weights** out) {
    if (!w || !out) return fail(WRS_EINVAL, "null argument");
    return guarded([&] {
        *out = new wrs_weights{weights_from_host(w, n)};
        return WRS_OK;
    });
}

wrs_status wrs_weights_generate(const char* dist, double param, uint64_t n, uint64_t seed,
                                wrs_weights** out) {
    if (!dist || !out) return fail(WRS_EINVAL, "null argument");
    return guarded([&]() -> wrs_status {
        const std::string d = dist;
        if (d == "uniform") {
            auto wd = std::make_shared<WeightsData>();
            wd->device = current_device();
            wd->n = n;
            if (n == 0) throw std::invalid_argument("weights: need at least one item");
            wd->storage = std::make_unique<DevBuf>(n * sizeof(double));
            wd->d_w = static_cast<double*>(wd->storage->p);
            Stream st;
            ck(wrsb::launch_generate_uniform(wd->d_w, n, 0, seed, st.s), "generate");
            ck(cudaStreamSynchronize(st.s), "generate");
            finalize_weights(*wd, "");
            *out = new wrs_weights{wd};
            return WRS_OK;
        }
        if (d == "powerlaw") {
            *out = new wrs_weights{powerlaw_device(n, param, seed)};
            return WRS_OK;
        }
        if (d == "lognormal") {
            *out = new wrs_weights{lognormal_device(n, 0, param, seed)};
            return WRS_OK;
        }
        return fail(WRS_EINVAL, "unknown distribution: " + d);
    });
}

// WRS1 file: "WRS1", u64 count, f64[count] (weight_file.hpp:57-101).
wrs_status wrs_weights_read(const char* path, wrs_weights** out) {
    if (!path || !out) return fail(WRS_EINVAL, "null argument");
    return guarded([&]() -> wrs_status {
        const std::string p = path;
        std::unique_ptr<std::FILE, int (*)(std::FILE*)> f(std::fopen(path, "rb"), &std::fclose);
        if (!f) throw io_error("cannot open for reading: " + p);
        char magic[4];
        uint64_t count = 0;
        if (std::fread(magic, 1, 4, f.get()) != 4) throw format_error("truncated header: " + p);
        if (std::memcmp(magic, "WRS1", 4) != 0)
            throw format_error("bad magic, not a weight file: " + p);
        if (std::fread(&count, sizeof count, 1, f.get()) != 1)
            throw format_error("truncated count: " + p);
        if (count > (uint64_t{1} << 40)) throw format_error("implausible item count: " + p);
        std::vector<double> w(count);
        if (count > 0 && std::fread(w.data(), sizeof(double), count, f.get()) != count)
            throw format_error("truncated payload: " + p);
        *out = new wrs_weights{weights_from_host(w.data(), count, p)};
        return WRS_OK;
    });
}

wrs_status wrs_weights_write(const wrs_weights* w, const char* path) {
    if (!w || !path) return fail(WRS_EINVAL, "null argument");
    return guarded([&]() -> wrs_status {
        const std::string p = path;
        const double* v = w->data->host_values();
        const uint64_t count = w->data->n;
        std::unique_ptr<std::FILE, int (*)(std::FILE*)> f(std::fopen(path, "wb"), &std::fclose);
        if (!f) throw io_error("cannot open for writing: " + p);
        if (std::fwrite("WRS1", 1, 4, f.get()) != 4 ||
            std::fwrite(&count, sizeof count, 1, f.get()) != 1 ||
            (count > 0 && std::fwrite(v, sizeof(double), count, f.get()) != count))
            throw io_error("short write: " + p);
        if (std::fflush(f.get()) != 0) throw io_error("flush failed: " + p);
        return WRS_OK;
    });
}

uint64_t wrs_weights_count(const wrs_weights* w) { return w ? w->data->n : 0; }

const double* wrs_weights_values(const wrs_weights* w) {
    if (!w) return nullptr;
    try {
        return w->data->host_values();
    } catch (const std::exception& e) {
        fail(WRS_EINTERNAL, e.what());
        return nullptr;
    }
}

void wrs_weights_free(wrs_weights* w) { delete w; }

// ---- sampler ---------------------------------------------------------------------
wrs_status wrs_sampler_build(const wrs_weights* w, const char* algo, unsigned workers,
                             uint64_t groups, wrs_sampler** out) {
    (void)groups;
    if (!w || !algo || !out) return fail(WRS_EINVAL, "null argument");
    return guarded([&]() -> wrs_status {
        const std::string name = algo;
        uint64_t P;
        if (name == "psa" && psa_exact_env())
            P = std::max(1u, workers);  // WRS_B200_PSA_EXACT=1: the reference's own job count
        else if (name == "psa")
            P = wrsb::default_jobs(w->data->n);
        else if (name == "psa-exact")
            P = std::max(1u, workers);
        else if (name == "vose" || name == "sweep" || name == "2lvl-classic" ||
                 name == "2lvl-sweep" || name == "compressed")
            return fail(WRS_EINVAL, "sampler algorithm " + name +
                                        " is not part of the B200 PSA path (use \"psa\")");
        else
            return fail(WRS_EINVAL, "unknown sampler algorithm: " + name);
        *out = build_psa(w->data, P, 0, name.c_str()).release();
        return WRS_OK;
    });
}

wrs_status wrs_sampler_verify_masses(const wrs_sampler* s, double rel_tol) {
    if (!s) return fail(WRS_EINVAL, "null argument");
    return guarded([&]() -> wrs_status {
        ck(cudaSetDevice(s->device), "cudaSetDevice");
        const double worst = max_rel_mass_error(*s);
        if (worst > rel_tol)
            return fail(WRS_EVERIFY, "mass deviation " + std::to_string(worst) +
                                         " exceeds tolerance in " + s->algo);
        return WRS_OK;
    });
}

wrs_status wrs_sampler_draw(const wrs_sampler* s, uint64_t seed, uint64_t count,
                            unsigned workers, uint32_t* out) {
    if (!s || !out) return fail(WRS_EINVAL, "null argument");
    return guarded([&]() -> wrs_status {
        ck(cudaSetDevice(s->device), "cudaSetDevice");
        workers = workers ? workers : 1;
        if (count == 0) return WRS_OK;
        if (is_device_pointer(out)) {
            sample_on(*s, seed, 0, count, count, workers, 0, out, s->stream->s);
            ck(cudaStreamSynchronize(s->stream->s), "draw");
        } else {
            draw_to_host(*s, seed, count, workers, out);
        }
        return WRS_OK;
    });
}

void wrs_sampler_free(wrs_sampler* s) { delete s; }

// capi.cpp:222-239 -- bulk with-replacement sample as (item, count) pairs.
wrs_status wrs_sample_with_replacement(const wrs_weights* w, uint64_t k, uint64_t seed,
                                       unsigned workers, uint32_t* items, uint64_t* counts,
                                       uint64_t* n_unique) {
    if (!w || !items || !counts || !n_unique) return fail(WRS_EINVAL, "null argument");
    (void)workers;  // parallelism only: the result must not depend on it (test_capi.cpp:104-111)
    return guarded([&]() -> wrs_status {
        auto s = build_psa(w->data, wrsb::default_jobs(w->data->n), 0, "psa");
        draw_counts(*s, seed, k, 1, items, counts, n_unique);
        return WRS_OK;
    });
}

// ---- outside the hot path --------------------------------------------------------
static wrs_status not_in_path(const char* what) {
    return fail(WRS_EINVAL, std::string(what) + " is not part of the B200 PSA path");
}

wrs_status wrs_sample_without_replacement(const wrs_weights*, uint64_t, uint64_t, unsigned,
                                          uint32_t*) {
    return not_in_path("wrs_sample_without_replacement");
}
wrs_status wrs_permutation(const wrs_weights*, uint64_t, unsigned, uint32_t*) {
    return not_in_path("wrs_permutation");
}
wrs_status wrs_subset_sample(const wrs_weights*, uint64_t, unsigned, uint32_t*, uint64_t*) {
    return not_in_path("wrs_subset_sample");
}
wrs_status wrs_reservoir_create(uint64_t, unsigned, uint64_t, wrs_reservoir** out) {
    if (out) *out = nullptr;
    return not_in_path("wrs_reservoir_create");
}
wrs_status wrs_reservoir_push(wrs_reservoir*, const uint32_t*, const double*, uint64_t) {
    return not_in_path("wrs_reservoir_push");
}
wrs_status wrs_reservoir_items(const wrs_reservoir*, uint32_t*, double*, uint64_t*) {
    return not_in_path("wrs_reservoir_items");
}
double wrs_reservoir_threshold(const wrs_reservoir*) {
    return std::numeric_limits<double>::quiet_NaN();
}
void wrs_reservoir_free(wrs_reservoir*) {}
wrs_status wrs_verify(const char*, uint64_t, int) { return not_in_path("wrs_verify"); }

// ---- B200 extensions -------------------------------------------------------------
uint64_t wrs_b200_default_jobs(uint64_t n) { return wrsb::default_jobs(n); }

uint64_t wrs_b200_release_cache(void) { return wrsb::release_cache(); }

int64_t wrs_b200_check_failures(unsigned* first_line) {
#ifdef WRS_B200_CHECKED
    if (first_line) *first_line = 0;
    return static_cast<int64_t>(
        wrsb::check_failures_psa(first_line) + wrsb::check_failures_sample(first_line) +
        wrsb::check_failures_verify(first_line) + wrsb::check_failures_generate(first_line));
#else
    if (first_line) *first_line = 0;
    return -1;
#endif
}

wrs_status wrs_b200_weights_from_device(const double* d_w, uint64_t n, int copy,
                                        wrs_weights** out) {
    if (!d_w || !out) return fail(WRS_EINVAL, "null argument");
    return guarded([&] {
        auto wd = std::make_shared<WeightsData>();
        wd->device = current_device();
        wd->n = n;
        if (n == 0) throw std::invalid_argument("weights: need at least one item");
        if (copy) {
            wd->storage = std::make_unique<DevBuf>(n * sizeof(double));
            wd->d_w = static_cast<double*>(wd->storage->p);
            ck(cudaMemcpy(wd->d_w, d_w, n * sizeof(double), cudaMemcpyDeviceToDevice), "D2D");
            wd->ext = true;  // legacy-stream copy, not synchronised here
        } else {
            wd->d_w = const_cast<double*>(d_w);
            wd->owned = false;
        }
        finalize_weights(*wd, "");
        *out = new wrs_weights{wd};
        return WRS_OK;
    });
}

wrs_status wrs_b200_weights_generate_range(const char* dist, double param, uint64_t n_total,
                                           uint64_t lo, uint64_t hi, uint64_t seed,
                                           wrs_weights** out) {
    if (!dist || !out) return fail(WRS_EINVAL, "null argument");
    return guarded([&]() -> wrs_status {
        const std::string d = dist;
        if (d != "uniform" && d != "powerlaw" && d != "lognormal")
            return fail(WRS_EINVAL, "unknown distribution: " + d);
        if (lo >= hi || hi > n_total) return fail(WRS_EINVAL, "bad range");
        if (d == "lognormal") {
            *out = new wrs_weights{lognormal_device(hi - lo, lo, param, seed)};
            return WRS_OK;
        }
        if (d == "powerlaw") {
            // the deal is global: generate all n_total, keep [lo, hi)
            auto full = powerlaw_device(n_total, param, seed);
            auto wd = std::make_shared<WeightsData>();
            wd->device = current_device();
            wd->n = hi - lo;
            wd->storage = std::make_unique<DevBuf>(wd->n * sizeof(double));
            wd->d_w = static_cast<double*>(wd->storage->p);
            ck(cudaMemcpy(wd->d_w, full->d_w + lo, wd->n * sizeof(double),
                          cudaMemcpyDeviceToDevice),
               "slice");
            wd->ext = true;  // legacy-stream copy, not synchronised here
            full->ext = true;
            finalize_weights(*wd, "");
            *out = new wrs_weights{wd};
            return WRS_OK;
        }
        auto wd = std::make_shared<WeightsData>();
        wd->device = current_device();
        wd->n = hi - lo;
        wd->storage = std::make_unique<DevBuf>(wd->n * sizeof(double));
        wd->d_w = static_cast<double*>(wd->storage->p);
        Stream st;
        ck(wrsb::launch_generate_uniform(wd->d_w, wd->n, lo, seed, st.s), "generate");
        ck(cudaStreamSynchronize(st.s), "generate");
        finalize_weights(*wd, "");
        *out = new wrs_weights{wd};
        return WRS_OK;
    });
}

double wrs_b200_weights_total(const wrs_weights* w) {
    return w ? w->data->total : std::numeric_limits<double>::quiet_NaN();
}
const double* wrs_b200_weights_device(const wrs_weights* w) { return w ? w->data->d_w : nullptr; }

wrs_status wrs_b200_sampler_build_psa(const wrs_weights* w, uint64_t jobs, unsigned flags,
                                      wrs_sampler** out) {
    if (!w || !out) return fail(WRS_EINVAL, "null argument");
    return guarded([&] {
        const uint64_t P = jobs ? jobs : wrsb::default_jobs(w->data->n);
        if (P > std::numeric_limits<unsigned>::max())
            throw std::invalid_argument("job count limited to 2^32-1");
        *out = build_psa(w->data, P, flags, jobs ? "psa-exact" : "psa").release();
        return WRS_OK;
    });
}

uint64_t wrs_b200_sampler_jobs(const wrs_sampler* s) { return s ? s->P : 0; }
uint64_t wrs_b200_sampler_size(const wrs_sampler* s) { return s ? s->n : 0; }
double wrs_b200_sampler_bucket_mean(const wrs_sampler* s) {
    return s ? s->wn : std::numeric_limits<double>::quiet_NaN();
}
double wrs_b200_sampler_total(const wrs_sampler* s) {
    return s ? s->total : std::numeric_limits<double>::quiet_NaN();
}
const void* wrs_b200_sampler_device_buckets(const wrs_sampler* s) {
    return s ? static_cast<const void*>(s->d_b()) : nullptr;
}

wrs_status wrs_b200_sampler_copy_buckets(const wrs_sampler* s, void* host_out) {
    if (!s || !host_out) return fail(WRS_EINVAL, "null argument");
    return guarded([&] {
        ck(cudaSetDevice(s->device), "cudaSetDevice");
        ck(cudaStreamSynchronize(s->stream->s), "sync");
        s->sync_table();
        ck(cudaMemcpy(host_out, s->d_b(), s->n * sizeof(Bucket), cudaMemcpyDeviceToHost), "D2H");
        return WRS_OK;
    });
}

int wrs_b200_set_timing(int on) { return g_timing.exchange(on ? 1 : 0); }

wrs_status wrs_b200_sampler_rebuild_async(wrs_sampler* s, void* stream) {
    if (!s) return fail(WRS_EINVAL, "null argument");
    return guarded([&] {
        std::lock_guard<std::mutex> g(s->mu);
        ck(cudaSetDevice(s->device), "cudaSetDevice");
        if (!s->ws.sc) ck(wrsb::workspace_alloc(s->ws, s->n, s->P, false), "workspace");
        cudaStream_t st = use_stream(*s, stream);
        s->timed = g_timing.load() != 0;
        if (s->timed && !s->ev[0])
            for (cudaEvent_t& e : s->ev) ck(cudaEventCreate(&e), "event");
        if (!s->hi) {
            s->hi = std::make_unique<Stream>(1);
            for (cudaEvent_t& e : s->hi_ev)
                ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
        }
        ck(cudaEventRecord(s->hi_ev[0], st), "event");
        ck(cudaStreamWaitEvent(s->hi->s, s->hi_ev[0], 0), "wait");
        if (s->dbuf) {
            // into the back table, once the draws reading it are done; draws
            // issued from now on read it (they wait for built_ev themselves)
            std::lock_guard<std::mutex> g2(s->sws_mu);
            const int X = 1 - s->front.load();
            ck(cudaStreamWaitEvent(s->hi->s, s->read_ev[X], 0), "wait");
            ck(wrsb::launch_psa_build(s->weights->d_w, s->n, s->weights->total, s->P,
                                      s->table(X), s->ws, s->hi->s, s->timed ? s->ev : nullptr),
               "PSA launch");
            ck(cudaEventRecord(s->built_ev[X], s->hi->s), "event");
            s->front.store(X);
            return WRS_OK;
        }
        ck(wrsb::launch_psa_build(s->weights->d_w, s->n, s->weights->total, s->P, s->d_b(),
                                  s->ws, s->hi->s, s->timed ? s->ev : nullptr),
           "PSA launch");
        ck(cudaEventRecord(s->hi_ev[1], s->hi->s), "event");
        ck(cudaStreamWaitEvent(st, s->hi_ev[1], 0), "wait");
        return WRS_OK;
    });
}

wrs_status wrs_b200_sampler_implied_masses(const wrs_sampler* s, double* out, double* worst) {
    if (!s || !out) return fail(WRS_EINVAL, "null argument");
    return guarded([&] {
        ck(cudaSetDevice(s->device), "cudaSetDevice");
        const bool dev = is_device_pointer(out);
        std::unique_ptr<DevBuf> tmp;
        double* d_m = out;
        if (!dev) {
            tmp = std::make_unique<DevBuf>(s->n * sizeof(double));
            d_m = static_cast<double*>(tmp->p);
        }
        const double wv = implied_masses(*s, d_m);
        if (!dev) ck(cudaMemcpy(out, d_m, s->n * sizeof(double), cudaMemcpyDeviceToHost), "D2H");
        if (worst) *worst = wv;
        return WRS_OK;
    });
}

wrs_status wrs_b200_sampler_double_buffer(wrs_sampler* s) {
    if (!s) return fail(WRS_EINVAL, "null argument");
    return guarded([&] {
        std::lock_guard<std::mutex> g(s->mu);
        std::lock_guard<std::mutex> g2(s->sws_mu);
        if (s->dbuf) return WRS_OK;
        ck(cudaSetDevice(s->device), "cudaSetDevice");
        ck(cudaDeviceSynchronize(), "sync");
        s->buckets2 = std::make_unique<DevBuf>(s->n * sizeof(Bucket));
        for (int b = 0; b < 2; ++b) {
            ck(cudaEventCreateWithFlags(&s->built_ev[b], cudaEventDisableTiming), "event");
            ck(cudaEventCreateWithFlags(&s->read_ev[b], cudaEventDisableTiming), "event");
            ck(cudaEventRecord(s->built_ev[b], s->stream->s), "event");
            ck(cudaEventRecord(s->read_ev[b], s->stream->s), "event");
        }
        s->dbuf = true;
        return WRS_OK;
    });
}

wrs_status wrs_b200_sampler_check(const wrs_sampler* s) {
    if (!s) return fail(WRS_EINVAL, "null argument");
    return guarded([&] {
        ck(cudaSetDevice(s->device), "cudaSetDevice");
        ck(cudaDeviceSynchronize(), "sync");
        if (s->ws.sc) read_scalars(const_cast<wrs_sampler&>(*s));
        return WRS_OK;
    });
}

int wrs_b200_sampler_stage_times(const wrs_sampler* s, float* ms, int max) {
    if (!s || !ms || !s->timed || !s->ev[0]) return 0;
    int w = 0;
    for (int i = 0; i < 7 && w < max; ++i) {
        if (cudaEventElapsedTime(&ms[w], s->ev[i], s->ev[i + 1]) != cudaSuccess) {
            cudaGetLastError();
            return w;
        }
        ++w;
    }
    return w;
}

wrs_status wrs_b200_sampler_draw_device(const wrs_sampler* s, uint64_t seed, uint64_t count,
                                        unsigned workers, uint32_t* d_out, void* stream) {
    if (!s || (!d_out && count)) return fail(WRS_EINVAL, "null argument");
    return guarded([&] {
        ck(cudaSetDevice(s->device), "cudaSetDevice");
        cudaStream_t st = use_stream(*s, stream);
        sample_on(*s, seed, 0, count, count, workers ? workers : 1, 0, d_out, st);
        return WRS_OK;
    });
}

wrs_status wrs_b200_sampler_draw_philox_device(const wrs_sampler* s, uint64_t seed,
                                               uint64_t count, uint32_t* d_out, void* stream) {
    if (!s || (!d_out && count)) return fail(WRS_EINVAL, "null argument");
    return guarded([&] {
        ck(cudaSetDevice(s->device), "cudaSetDevice");
        cudaStream_t st = use_stream(*s, stream);
        sample_on(*s, seed, 0, count, count, 1, 0, d_out, st, wrsb::kPhiloxStream);
        return WRS_OK;
    });
}

wrs_status wrs_b200_sampler_draw_counts(const wrs_sampler* s, uint64_t seed, uint64_t k,
                                        unsigned workers, uint32_t* items, uint64_t* counts,
                                        uint64_t* n_unique) {
    if (!s || !items || !counts || !n_unique) return fail(WRS_EINVAL, "null argument");
    return guarded([&] {
        ck(cudaSetDevice(s->device), "cudaSetDevice");
        draw_counts(*s, seed, k, workers, items, counts, n_unique);
        return WRS_OK;
    });
}

wrs_status wrs_b200_sampler_draw_counts_device(const wrs_sampler* s, uint64_t seed, uint64_t k,
                                               unsigned workers, uint32_t* d_items,
                                               uint64_t* d_counts, uint64_t* d_n_unique,
                                               void* stream) {
    if (!s || !d_items || !d_counts || !d_n_unique) return fail(WRS_EINVAL, "null argument");
    return guarded([&] {
        ck(cudaSetDevice(s->device), "cudaSetDevice");
        cudaStream_t st = use_stream(*s, stream);
        count_on(*s, seed, k, workers ? workers : 1, d_items, d_counts, d_n_unique, st);
        return WRS_OK;
    });
}

wrs_status wrs_b200_two_level_draw_device(const void* const* d_tables, const uint64_t* sizes,
                                          const double* bucket_means, const uint64_t* bases,
                                          uint64_t groups, const void* d_top, double top_mean,
                                          uint64_t seed, uint64_t q_begin, uint64_t q_end,
                                          uint64_t k, unsigned workers, uint32_t* d_out,
                                          void* stream) {
    if (!d_tables || !sizes || !bucket_means || !bases || !d_top || (!d_out && q_end > q_begin))
        return fail(WRS_EINVAL, "null argument");
    if (groups == 0 || groups > static_cast<uint64_t>(wrsb::kTwoLevelMaxGroups))
        return fail(WRS_EINVAL, "groups must be in [1, 256]");
    if (q_begin > q_end || q_end > k) return fail(WRS_EINVAL, "bad output range");
    return guarded([&] {
        wrsb::TwoLevelDev tl{};
        for (uint64_t g = 0; g < groups; ++g) {
            if (!d_tables[g] || sizes[g] == 0 || sizes[g] > 0xffffffffull)
                throw std::invalid_argument("group tables must be non-empty, < 2^32 buckets");
            tl.tables[g] = static_cast<const Bucket*>(d_tables[g]);
            tl.sizes[g] = sizes[g];
            tl.means[g] = bucket_means[g];
            tl.bases[g] = bases[g];
        }
        tl.top = static_cast<const Bucket*>(d_top);
        tl.groups = groups;
        tl.top_mean = top_mean;
        int dev = 0;
        ck(cudaGetDevice(&dev), "cudaGetDevice");
        ck(wrsb::launch_two_level(tl, seed, q_begin, q_end, k, workers ? workers : 1, d_out,
                                  static_cast<cudaStream_t>(stream)),
           "two-level launch");
        return WRS_OK;
    });
}

wrs_status wrs_b200_sampler_ipc_handle(const wrs_sampler* s, void* handle) {
    if (!s || !handle) return fail(WRS_EINVAL, "null argument");
    return guarded([&] {
        ck(cudaSetDevice(s->device), "cudaSetDevice");
        cudaIpcMemHandle_t h;
        ck(cudaIpcGetMemHandle(&h, s->d_b()), "cudaIpcGetMemHandle");
        static_assert(sizeof h == 64, "IPC handle is 64 bytes");
        std::memcpy(handle, &h, sizeof h);
        return WRS_OK;
    });
}

wrs_status wrs_b200_ipc_open(const void* handle, void** d_ptr) {
    if (!handle || !d_ptr) return fail(WRS_EINVAL, "null argument");
    return guarded([&] {
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handle, sizeof h);
        ck(cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
        return WRS_OK;
    });
}

wrs_status wrs_b200_ipc_close(void* d_ptr) {
    if (!d_ptr) return fail(WRS_EINVAL, "null argument");
    return guarded([&] {
        ck(cudaIpcCloseMemHandle(d_ptr), "cudaIpcCloseMemHandle");
        return WRS_OK;
    });
}

// Shard g draws AliasTable(shard_g).sample_many(seed_g, count, 1) with
// seed_g = RngStream(seed, 'sdrw').derive(g).key, then adds the shard base.
uint64_t wrs_b200_shard_seed(uint64_t seed, uint64_t shard) {
    return wrsb::rng_derive(wrsb::rng_key(seed, 0x73647277u), shard);
}

wrs_status wrs_b200_sampler_draw_shard_device(const wrs_sampler* s, uint64_t seed, uint64_t shard,
                                              uint64_t count, uint64_t base, uint32_t* d_out,
                                              void* stream) {
    if (!s || (!d_out && count)) return fail(WRS_EINVAL, "null argument");
    if (base + s->n > (uint64_t{1} << 32)) return fail(WRS_EINVAL, "global ids exceed 2^32");
    return guarded([&] {
        ck(cudaSetDevice(s->device), "cudaSetDevice");
        cudaStream_t st = use_stream(*s, stream);
        sample_on(*s, wrs_b200_shard_seed(seed, shard), 0, count, count, 1,
                  static_cast<uint32_t>(base), d_out, st);
        return WRS_OK;
    });
}

wrs_status wrs_b200_sampler_stage(const wrs_sampler* s, const char* name, void* host_out,
                                  uint64_t capacity, uint64_t* bytes) {
    if (!s || !name || !bytes) return fail(WRS_EINVAL, "null argument");
    return guarded([&]() -> wrs_status {
        if (!s->ws.sc) return fail(WRS_EINVAL, "build without WRS_B200_KEEP_WORKSPACE");
        ck(cudaSetDevice(s->device), "cudaSetDevice");
        ck(cudaDeviceSynchronize(), "sync");
        wrsb::DevScalars sc{};
        ck(cudaMemcpy(&sc, s->ws.sc, sizeof sc, cudaMemcpyDeviceToHost), "D2H");
        const uint64_t nl = sc.nl, nh = sc.nh;
        const uint64_t nbl = (nl + 2047) / 2048, nbh = (nh + 2047) / 2048;
        const std::string nm = name;
        const void* src = nullptr;
        uint64_t by = 0;
        uint64_t counts[2] = {nl, nh};
        if (nm == "counts") {
            src = counts;
            by = sizeof counts;
        } else if (nm == "light_rank") {
            src = s->ws.lrank;
            by = nl * 4;
        } else if (nm == "heavy_share") {
            src = s->ws.hshare;
            by = nh * 8;
        } else if (nm == "heavy") {
            src = s->ws.hidx;
            by = nh * 4;
        } else if (nm == "light_w") {
            src = s->ws.lw;
            by = nl * 8;
        } else if (nm == "heavy_w") {
            src = s->ws.hw;
            by = nh * 8;
        } else if (nm == "light_prefix" || nm == "heavy_prefix") {
            if (s->ws.ckpt)
                return fail(WRS_EINVAL, "this build kept checkpointed prefixes (light_ckpt / heavy_ckpt)");
            src = nm[0] == 'l' ? s->ws.lpre : s->ws.hpre;
            by = ((nm[0] == 'l' ? nl : nh) + 1) * 8;
        } else if (nm == "light_ckpt" || nm == "heavy_ckpt") {
            if (!s->ws.ckpt) return fail(WRS_EINVAL, "this build kept full prefix arrays");
            src = nm[0] == 'l' ? s->ws.lck : s->ws.hck;
            by = ((nm[0] == 'l' ? nl : nh) + 15) / 16 * 16;  // one (hi, lo) pair per 16 items
        } else if (nm == "block_totals") {
            src = s->ws.totals;
            by = (nbl + nbh) * 8;
        } else if (nm == "carries") {
            src = s->ws.carries;
            by = (nbl + nbh) * 8;
        } else if (nm == "split_light") {
            src = s->ws.split_l;
            by = (s->P + 1) * 4;
        } else if (nm == "split_heavy") {
            src = s->ws.split_h;
            by = (s->P + 1) * 4;
        } else if (nm == "split_spill") {
            src = s->ws.split_s;
            by = (s->P + 1) * 8;
        } else {
            return fail(WRS_EINVAL, "unknown stage: " + nm);
        }
        *bytes = by;
        if (!host_out) return WRS_OK;
        if (capacity < by) return fail(WRS_EINVAL, "stage buffer too small");
        if (nm == "counts")
            std::memcpy(host_out, counts, by);
        else if (by)
            ck(cudaMemcpy(host_out, src, by, cudaMemcpyDeviceToHost), "D2H");
        return WRS_OK;
    });
}


// ---- multi-GPU sampler (NCCL) ------------------------------------------------------
}  // extern "C"

namespace {

// NCCL, loaded on first use (libnccl.so.2: the copy already in the process,
// e.g. PyTorch's, else the system one).
struct Nccl {
    bool ok = false;
    int version = 0;
    std::string err;
    decltype(&ncclGetUniqueId) getUniqueId = nullptr;
    decltype(&ncclCommInitRank) commInitRank = nullptr;
    decltype(&ncclCommInitAll) commInitAll = nullptr;
    decltype(&ncclAllGather) allGather = nullptr;
    decltype(&ncclCommDestroy) commDestroy = nullptr;
    decltype(&ncclGetErrorString) errorString = nullptr;
    decltype(&ncclGroupStart) groupStart = nullptr;
    decltype(&ncclGroupEnd) groupEnd = nullptr;
    decltype(&ncclGetVersion) getVersion = nullptr;
};

Nccl& nccl() {
    static Nccl n = [] {
        Nccl x;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            x.err = std::string("cannot load libnccl.so.2: ") + dlerror();
            return x;
        }
        auto sym = [&](auto& f, const char* name) {
            f = reinterpret_cast<std::remove_reference_t<decltype(f)>>(dlsym(h, name));
            return f != nullptr;
        };
        x.ok = sym(x.getUniqueId, "ncclGetUniqueId") && sym(x.commInitRank, "ncclCommInitRank") &&
               sym(x.commInitAll, "ncclCommInitAll") && sym(x.allGather, "ncclAllGather") &&
               sym(x.commDestroy, "ncclCommDestroy") && sym(x.errorString, "ncclGetErrorString") &&
               sym(x.groupStart, "ncclGroupStart") && sym(x.groupEnd, "ncclGroupEnd") &&
               sym(x.getVersion, "ncclGetVersion");
        if (!x.ok)
            x.err = "libnccl.so.2 lacks a needed symbol";
        else
            x.getVersion(&x.version);
        return x;
    }();
    return n;
}

Nccl& need_nccl() {
    Nccl& n = nccl();
    if (!n.ok) throw std::runtime_error(n.err);
    return n;
}

void nck(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) throw std::runtime_error(std::string(what) + ": " + nccl().errorString(r));
}

}  // namespace

struct wrs_b200_multi {
    std::unique_ptr<wrs_sampler> shard;
    uint32_t rank = 0, ranks = 1;
    uint64_t n_total = 0, lo = 0, hi = 0;
    int device = 0;
    ncclComm_t comm = nullptr;
    std::unique_ptr<DevBuf> d_total, d_totals;  // this shard's total, the gathered totals
    std::vector<double> totals;
    std::shared_ptr<WeightsData> top_w;
    std::unique_ptr<wrs_sampler> top;
    ~wrs_b200_multi() {
        if (device >= 0) cudaSetDevice(device);
        top.reset();
        if (comm && nccl().ok) nccl().commDestroy(comm);
    }
};

namespace {

std::unique_ptr<wrs_b200_multi> multi_new(const wrs_weights* shard, uint64_t n_total, uint32_t rank,
                                          uint32_t ranks) {
    if (ranks == 0 || rank >= ranks) throw std::invalid_argument("rank must be < ranks");
    auto m = std::make_unique<wrs_b200_multi>();
    m->rank = rank;
    m->ranks = ranks;
    m->n_total = n_total;
    wrs_b200_shard_range(n_total, ranks, rank, &m->lo, &m->hi);
    if (shard->data->n != m->hi - m->lo)
        throw std::invalid_argument("shard holds " + std::to_string(shard->data->n) +
                                    " items, rank " + std::to_string(rank) + " owns " +
                                    std::to_string(m->hi - m->lo));
    m->device = shard->data->device;
    ck(cudaSetDevice(m->device), "cudaSetDevice");
    m->shard = build_psa(shard->data, wrsb::default_jobs(shard->data->n), 0, "psa");
    m->d_total = std::make_unique<DevBuf>(sizeof(double));
    m->d_totals = std::make_unique<DevBuf>(ranks * sizeof(double));
    ck(cudaMemcpy(m->d_total->p, &shard->data->total, sizeof(double), cudaMemcpyHostToDevice),
       "total H2D");
    return m;
}

// the top table over the gathered totals (two_level.hpp:56-57)
void multi_set_totals(wrs_b200_multi& m, const double* totals) {
    ck(cudaSetDevice(m.device), "cudaSetDevice");
    const bool same = m.totals.size() == m.ranks &&
                      std::memcmp(m.totals.data(), totals, m.ranks * sizeof(double)) == 0;
    if (same && m.top) return;
    m.totals.assign(totals, totals + m.ranks);
    m.top.reset();
    m.top_w = weights_from_host(m.totals.data(), m.ranks);
    m.top = build_psa(m.top_w, wrsb::default_jobs(m.ranks), 0, "psa");
}

void multi_read_totals(wrs_b200_multi& m, cudaStream_t st) {
    std::vector<double> t(m.ranks);
    ck(cudaMemcpyAsync(t.data(), m.d_totals->p, m.ranks * sizeof(double), cudaMemcpyDeviceToHost, st),
       "totals D2H");
    ck(cudaStreamSynchronize(st), "totals");
    multi_set_totals(m, t.data());
}

}  // namespace

extern "C" {

int wrs_b200_nccl_available(int* version) {
    Nccl& n = nccl();
    if (version) *version = n.ok ? n.version : 0;
    return n.ok ? 1 : 0;
}

wrs_status wrs_b200_nccl_unique_id(void* id128) {
    if (!id128) return fail(WRS_EINVAL, "null argument");
    return guarded([&] {
        ncclUniqueId id;
        nck(need_nccl().getUniqueId(&id), "ncclGetUniqueId");
        static_assert(sizeof id == 128, "NCCL unique id is 128 bytes");
        std::memcpy(id128, &id, sizeof id);
        return WRS_OK;
    });
}

wrs_status wrs_b200_multi_create(const wrs_weights* shard, uint64_t n_total, uint32_t rank,
                                 uint32_t ranks, const void* nccl_id, wrs_b200_multi** out) {
    if (!shard || !out) return fail(WRS_EINVAL, "null argument");
    return guarded([&] {
        auto m = multi_new(shard, n_total, rank, ranks);
        if (nccl_id) {
            Nccl& n = need_nccl();
            ncclUniqueId id;
            std::memcpy(&id, nccl_id, sizeof id);
            nck(n.commInitRank(&m->comm, static_cast<int>(ranks), id, static_cast<int>(rank)),
                "ncclCommInitRank");
            nck(n.allGather(m->d_total->p, m->d_totals->p, 1, ncclFloat64, m->comm,
                            m->shard->stream->s),
                "ncclAllGather");
            multi_read_totals(*m, m->shard->stream->s);
        }
        *out = m.release();
        return WRS_OK;
    });
}

wrs_status wrs_b200_multi_create_local(const wrs_weights* const* shards, uint32_t ranks,
                                       uint64_t n_total, wrs_b200_multi** out) {
    if (!shards || !out || ranks == 0) return fail(WRS_EINVAL, "null argument");
    return guarded([&] {
        Nccl& n = need_nccl();
        std::vector<std::unique_ptr<wrs_b200_multi>> ms;
        std::vector<int> devs;
        for (uint32_t g = 0; g < ranks; ++g) {
            if (!shards[g]) throw std::invalid_argument("null shard");
            ms.push_back(multi_new(shards[g], n_total, g, ranks));
            devs.push_back(ms.back()->device);
        }
        std::vector<ncclComm_t> comms(ranks);
        nck(n.commInitAll(comms.data(), static_cast<int>(ranks), devs.data()), "ncclCommInitAll");
        for (uint32_t g = 0; g < ranks; ++g) ms[g]->comm = comms[g];
        nck(n.groupStart(), "ncclGroupStart");
        for (uint32_t g = 0; g < ranks; ++g) {
            ck(cudaSetDevice(ms[g]->device), "cudaSetDevice");
            nck(n.allGather(ms[g]->d_total->p, ms[g]->d_totals->p, 1, ncclFloat64, ms[g]->comm,
                            ms[g]->shard->stream->s),
                "ncclAllGather");
        }
        nck(n.groupEnd(), "ncclGroupEnd");
        for (uint32_t g = 0; g < ranks; ++g) multi_read_totals(*ms[g], ms[g]->shard->stream->s);
        for (uint32_t g = 0; g < ranks; ++g) out[g] = ms[g].release();
        return WRS_OK;
    });
}

wrs_status wrs_b200_multi_set_totals(wrs_b200_multi* m, const double* totals) {
    if (!m || !totals) return fail(WRS_EINVAL, "null argument");
    return guarded([&] {
        multi_set_totals(*m, totals);
        return WRS_OK;
    });
}

wrs_status wrs_b200_multi_exchange(wrs_b200_multi* m, void* stream) {
    if (!m) return fail(WRS_EINVAL, "null argument");
    return guarded([&] {
        if (!m->comm) throw std::invalid_argument("handle has no NCCL communicator");
        ck(cudaSetDevice(m->device), "cudaSetDevice");
        cudaStream_t st = use_stream(*m->shard, stream);
        nck(need_nccl().allGather(m->d_total->p, m->d_totals->p, 1, ncclFloat64, m->comm, st),
            "ncclAllGather");
        multi_read_totals(*m, st);
        return WRS_OK;
    });
}

wrs_status wrs_b200_multi_rebuild_async(wrs_b200_multi* m, void* stream) {
    if (!m) return fail(WRS_EINVAL, "null argument");
    return wrs_b200_sampler_rebuild_async(m->shard.get(), stream);
}

wrs_status wrs_b200_multi_totals(const wrs_b200_multi* m, double* totals) {
    if (!m || !totals) return fail(WRS_EINVAL, "null argument");
    if (m->totals.size() != m->ranks) return fail(WRS_EINVAL, "totals not exchanged yet");
    std::memcpy(totals, m->totals.data(), m->ranks * sizeof(double));
    return WRS_OK;
}

wrs_status wrs_b200_multi_counts(const wrs_b200_multi* m, uint64_t seed, uint64_t k,
                                 uint64_t* counts) {
    if (!m || !counts) return fail(WRS_EINVAL, "null argument");
    if (m->totals.size() != m->ranks) return fail(WRS_EINVAL, "totals not exchanged yet");
    return wrs_b200_shard_counts(m->totals.data(), m->ranks, seed, k, counts);
}

wrs_status wrs_b200_multi_draw_device(const wrs_b200_multi* m, uint64_t seed, uint64_t k,
                                      uint32_t* d_out, void* stream, uint64_t* count) {
    if (!m || !count) return fail(WRS_EINVAL, "null argument");
    if (m->totals.size() != m->ranks) return fail(WRS_EINVAL, "totals not exchanged yet");
    return guarded([&]() -> wrs_status {
        std::vector<uint64_t> c(m->ranks);
        const wrs_status r = wrs_b200_shard_counts(m->totals.data(), m->ranks, seed, k, c.data());
        if (r != WRS_OK) return r;
        *count = c[m->rank];
        if (!d_out && *count) return fail(WRS_EINVAL, "null output");
        return wrs_b200_sampler_draw_shard_device(m->shard.get(), seed, m->rank, *count, m->lo,
                                                  d_out, stream);
    });
}

wrs_status wrs_b200_multi_top_buckets(const wrs_b200_multi* m, void* host_out, double* bucket_mean) {
    if (!m || !host_out) return fail(WRS_EINVAL, "null argument");
    if (!m->top) return fail(WRS_EINVAL, "totals not exchanged yet");
    if (bucket_mean) *bucket_mean = m->top->wn;
    return wrs_b200_sampler_copy_buckets(m->top.get(), host_out);
}

const wrs_sampler* wrs_b200_multi_shard(const wrs_b200_multi* m) { return m ? m->shard.get() : nullptr; }

void wrs_b200_multi_free(wrs_b200_multi* m) { delete m; }

}  // extern "C"
