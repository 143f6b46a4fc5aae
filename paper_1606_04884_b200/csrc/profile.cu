// profile.cu — CUDA-event timing of the library's hot kernels on their own
// launching stream (bench.py reads it for the roofline's per-launch duration).
#include <map>
#include <mutex>
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
