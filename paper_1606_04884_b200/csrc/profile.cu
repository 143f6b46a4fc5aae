// profile.cu — CUDA-event timing of the library's hot kernels on their own
// launching stream (bench.py reads it for the roofline's per-launch duration).
#include <atomic>
#include <cstdlib>
#include <map>
#include <mutex>
#include <set>
#include <tuple>
#include <functional>
#include <string>
#include <vector>

#include "common.cuh"

namespace ptb {

namespace {
struct Pending {
    std::string cls, key;
    cudaEvent_t e0, e1;
    double flops, bytes;
};
struct Totals {
    double ms = 0, flops = 0, bytes = 0;
    int64_t launches = 0;
};
std::atomic<bool> g_on{false};
std::mutex g_mu;
std::vector<Pending> g_pending;
std::map<std::string, Totals> g_totals;
thread_local std::string g_tag;        // caller label (bench: the layer name)
thread_local const char* g_pass = "";  // set by the ABI entry point (fwd / dgrad / wgrad)

void drain_locked() {
    for (auto& p : g_pending) {
        float ms = 0.f;
        cudaEventSynchronize(p.e1);
        cudaEventElapsedTime(&ms, p.e0, p.e1);
        for (const std::string* k : {&p.cls, &p.key}) {
            if (k->empty()) continue;
            Totals& t = g_totals[*k];
            t.ms += ms;
            t.flops += p.flops;
            t.bytes += p.bytes;
            t.launches += 1;
        }
        cudaEventDestroy(p.e0);
        cudaEventDestroy(p.e1);
    }
    g_pending.clear();
}
}  // namespace

bool prof_enabled() { return g_on.load(std::memory_order_relaxed); }

PassScope::PassScope(const char* pass) : prev(g_pass) { g_pass = pass; }
PassScope::~PassScope() { g_pass = prev; }

ProfScope::ProfScope(const char* c, cudaStream_t s, double f, double b)
    : cls(c), st(s), flops(f), bytes(b) {
    if (!prof_enabled()) return;
    cudaEventCreate(&e0);
    cudaEventRecord(e0, st);
}

ProfScope::~ProfScope() {
    if (!e0) return;
    cudaEvent_t e1;
    cudaEventCreate(&e1);
    cudaEventRecord(e1, st);
    std::lock_guard<std::mutex> lk(g_mu);
    // per-launch key "class@tag.pass" (e.g. umma_conv@L2.dgrad) beside the class total
    std::string key = g_tag.empty() && !*g_pass ? std::string() : std::string(cls) + "@" + g_tag + "." + g_pass;
    g_pending.push_back({cls, std::move(key), e0, e1, flops, bytes});
}

namespace {
std::atomic<int> g_conc{-1};  // -1: PT_B200_BWD_STREAMS (default on)
}  // namespace

bool concurrency_on() {
    static const bool env_on = [] {
        const char* e = std::getenv("PT_B200_BWD_STREAMS");
        return e ? std::atoi(e) != 0 : true;  // PT_B200_BWD_STREAMS=0: serial
    }();
    const int v = g_conc.load(std::memory_order_relaxed);
    return v < 0 ? env_on : v != 0;
}
void set_concurrency(int on) { g_conc.store(on ? 1 : 0, std::memory_order_relaxed); }

// One internal stream per (device, caller stream, slot): calls on different caller streams
// (other threads, other CUDA-graph captures) never share an aux stream, so a fork/join on
// one caller stream neither waits on nor joins another caller's work.
cudaStream_t aux_stream(cudaStream_t caller, int slot) {
    static std::mutex mu;
    static std::map<std::tuple<int, cudaStream_t, int>, cudaStream_t> streams;
    int dev = 0;
    PTB_CUDA(cudaGetDevice(&dev));
    if (slot < 0 || slot > 1) return nullptr;
    std::lock_guard<std::mutex> lock(mu);
    cudaStream_t& s = streams[{dev, caller, slot}];
    if (!s) PTB_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    return s;
}

void once_per_device(const void* key, const std::function<void()>& set) {
    static std::mutex mu;
    static std::set<std::pair<int, const void*>> done;
    int dev = 0;
    PTB_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(mu);  // held across set(): no launch before it is done
    if (done.count({dev, key})) return;
    set();
    done.insert({dev, key});
}

Fork::Fork(cudaStream_t s, int slot) : st(s), side(s) {
    if (!concurrency_on()) return;
    cudaStream_t a = aux_stream(st, slot);
    if (!a) return;
    cudaEvent_t e;
    PTB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    PTB_CUDA(cudaEventRecord(e, st));
    PTB_CUDA(cudaStreamWaitEvent(a, e, 0));
    PTB_CUDA(cudaEventDestroy(e));
    side = a;
}
Fork::~Fork() {
    if (side == st) return;
    cudaEvent_t e;
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return;
    if (cudaEventRecord(e, side) == cudaSuccess) cudaStreamWaitEvent(st, e, 0);
    cudaEventDestroy(e);
}
void Fork::join() {
    if (side == st) return;
    cudaEvent_t e;
    PTB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    PTB_CUDA(cudaEventRecord(e, side));
    PTB_CUDA(cudaStreamWaitEvent(st, e, 0));
    PTB_CUDA(cudaEventDestroy(e));
    side = st;
}

}  // namespace ptb

extern "C" {
int pt_b200_profile_enable(int on) {
    ptb::g_on.store(on != 0);
    return PT_OK;
}
int pt_b200_profile_tag(const char* tag) {
    ptb::g_tag = tag ? tag : "";
    return PT_OK;
}
int pt_b200_profile_reset(void) {
    std::lock_guard<std::mutex> lk(ptb::g_mu);
    ptb::drain_locked();
    ptb::g_totals.clear();
    return PT_OK;
}
int pt_b200_profile_read(const char* cls, double* total_ms, int64_t* launches, double* flops,
                         double* bytes) {
    std::lock_guard<std::mutex> lk(ptb::g_mu);
    ptb::drain_locked();
    auto it = ptb::g_totals.find(cls ? cls : "");
    ptb::Totals t = it == ptb::g_totals.end() ? ptb::Totals{} : it->second;
    if (total_ms) *total_ms = t.ms;
    if (launches) *launches = t.launches;
    if (flops) *flops = t.flops;
    if (bytes) *bytes = t.bytes;
    return PT_OK;
}
}
