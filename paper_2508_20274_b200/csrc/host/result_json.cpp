#include "result_json.hpp"

#include <cmath>
#include <cstdio>

namespace mgb {

namespace {

std::string num(double v) {
    if (std::isnan(v)) return "NaN";
    if (std::isinf(v)) return v > 0 ? "Infinity" : "-Infinity";
    char b[40];
    std::snprintf(b, sizeof(b), "%.17g", v);
    return b;
}
std::string num(uint64_t v) { return std::to_string(v); }
std::string num(int v) { return std::to_string(v); }
std::string str(const std::string& s) { return "\"" + json_escape(s) + "\""; }

}  // namespace

std::string json_escape(const std::string& s) {
    std::string o;
    for (char c : s) {
        if (c == '"' || c == '\\') {
            o += '\\';
            o += c;
        } else if (static_cast<unsigned char>(c) < 0x20) {
            char b[8];
            std::snprintf(b, sizeof(b), "\\u%04x", c);
            o += b;
        } else {
            o += c;
        }
    }
    return o;
}

std::string result_to_json(const RunResult& r) {
    std::string o = "{";
    o += "\"scenario\":" + str(r.scenario_name) + ",\"variant\":" + str(r.variant) + ",\"seed\":" + num(r.seed) +
         ",\"duration_s\":" + num(r.duration_s) + ",\"measure_start_s\":" + num(r.measure_start_s) +
         ",\"n_events\":" + num(r.n_events);
    o += ",\"tenants\":{";
    bool first = true;
    for (const auto& [id, s] : r.tenants) {
        if (!first) o += ",";
        first = false;
        o += str(id) + ":{\"completed_total\":" + num(s.completed_total) + ",\"completed_window\":" +
             num(s.completed_window) + ",\"mean_ms\":" + num(s.mean_ms) + ",\"p50_ms\":" + num(s.p50_ms) +
             ",\"p95_ms\":" + num(s.p95_ms) + ",\"p99_ms\":" + num(s.p99_ms) + ",\"p999_ms\":" + num(s.p999_ms) +
             ",\"miss_rate\":" + num(s.miss_rate) + ",\"throughput_hz\":" + num(s.throughput_hz) +
             ",\"slo_tail_ms\":" + num(s.slo_tail_ms) + "}";
    }
    o += "},\"end_states\":{";
    first = true;
    for (const auto& [id, e] : r.end_states) {
        if (!first) o += ",";
        first = false;
        o += str(id) + ":{\"host\":" + num(e.placement.host) + ",\"gpu\":" + num(e.placement.gpu) +
             ",\"first_slice\":" + num(e.placement.slices.first) +
             ",\"slice_count\":" + num(e.placement.slices.count) + ",\"profile\":" + str(e.profile) +
             ",\"claim_Bps\":" + num(e.claim_Bps) + ",\"status\":\"admitted\",\"cpu_pinned\":" +
             (e.cpu_pinned ? "true" : "false") + "}";
    }
    o += "},\"actions\":[";
    first = true;
    for (const auto& a : r.actions) {
        if (!first) o += ",";
        first = false;
        o += "{\"seq\":" + num(a.seq) + ",\"t_s\":" + num(a.t_s) + ",\"tenant\":" + str(a.tenant) +
             ",\"target\":" + str(a.target) + ",\"kind\":" + str(a.kind) + ",\"diagnosis\":" + str(a.diagnosis) +
             ",\"p99_pre_ms\":" + num(a.p99_pre_ms) + ",\"ema_p99_ms\":" + num(a.ema_p99_ms) +
             ",\"breach_windows\":" + num(a.breach_windows) + ",\"obs_since_prev\":" + num(a.obs_since_prev) +
             ",\"throttle_Bps\":" + num(a.throttle_Bps) + ",\"quota_pct\":" + num(a.quota_pct) +
             ",\"pause_s\":" + num(a.pause_s) + ",\"rolled_back_seq\":" + num(a.rolled_back_seq) +
             ",\"detail\":" + str(a.detail) + "}";
    }
    o += "],\"pauses\":[";
    first = true;
    for (const auto& p : r.pauses) {
        if (!first) o += ",";
        first = false;
        o += "{\"t_s\":" + num(p.t_s) + ",\"tenant\":" + str(p.tenant) + ",\"kind\":" + str(p.kind) +
             ",\"duration_s\":" + num(p.duration_s) + "}";
    }
    o += "],\"stability\":{\"analytic_oversubscribed\":";
    o += r.stability.analytic_oversubscribed ? "true" : "false";
    o += ",\"unbounded_growth\":";
    o += r.stability.unbounded_growth ? "true" : "false";
    o += ",\"notes\":[";
    first = true;
    for (const auto& n : r.stability.notes) {
        if (!first) o += ",";
        first = false;
        o += str(n);
    }
    o += "]}}";
    return o;
}

}  // namespace mgb
