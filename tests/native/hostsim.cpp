// TEST HARNESS ONLY -- not product code and never linked into the product library.
//
// Compiles the engine's device-side logic (csrc/common/*.h, which is __host__ __device__) for the
// CPU so the CPU test suite can differential-test the exact restatement of the reference engine
// against the compiled reference (oracle/_ref) without a GPU.  The product C-ABI
// (libmigsim_b200.so) has no CPU execution path; this library exists only under tests/.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../paper_2508_20274_b200/csrc/common/des_core.h"
#include "../../paper_2508_20274_b200/csrc/host/artifacts.hpp"
#include "../../paper_2508_20274_b200/csrc/host/packer.hpp"
#include "../../paper_2508_20274_b200/csrc/host/result_json.hpp"

using namespace mgb;

namespace {

thread_local std::string g_err;

char* dup(const std::string& s) {
    char* p = static_cast<char*>(std::malloc(s.size() + 1));
    std::memcpy(p, s.c_str(), s.size() + 1);
    return p;
}

struct Arrivals {
    std::vector<double> t, bytes, mult, noise, irq;
    std::vector<int32_t> count;
};

Arrivals generate(const Packed& P, uint64_t seed) {
    const int T = P.scen.n_tenants;
    Arrivals A;
    A.t.assign(static_cast<size_t>(P.cap_sum), 0.0);
    A.bytes = A.mult = A.noise = A.irq = A.t;
    A.count.assign(static_cast<size_t>(T), 0);
    std::vector<uint64_t> mt(mg::kMtN);
    std::vector<double> t_all;
    for (int i = 0; i < T; ++i) {
        const mg::PTenant& p = P.scen.tenants[i];
        const int64_t off = P.off[static_cast<size_t>(i)];
        const int64_t cap = P.cap[static_cast<size_t>(i)];
        t_all.assign(static_cast<size_t>(cap), 0.0);
        mg::Mt64Ref g{mt.data(), 0};
        g.seed(mg::substream_seed(seed, p.name_hash, mg::kArrivals));
        int32_t n_all = 0, n_kept = 0;
        if (!mg::gen_times(g, p, P.scen.duration_s, t_all.data(), A.t.data() + off, cap, &n_all, &n_kept))
            throw std::runtime_error("arrival capacity overflow");
        A.count[static_cast<size_t>(i)] = n_kept;
        const uint64_t purposes[3] = {mg::kTransferSize, mg::kService, mg::kNoise};
        double* outs[3] = {A.bytes.data() + off, A.mult.data() + off, A.noise.data() + off};
        for (int k = 0; k < 3; ++k) {
            mg::Mt64Ref h{mt.data(), 0};
            h.seed(mg::substream_seed(seed, p.name_hash, purposes[k]));
            mg::gen_marks(h, k, p, t_all.data(), n_all, outs[k]);
        }
        if (P.any_irq_noise) {
            mg::Mt64Ref h{mt.data(), 0};
            h.seed(mg::substream_seed(seed, p.name_hash, mg::kIrq));
            mg::gen_irq(h, n_kept, A.irq.data() + off);
        }
    }
    return A;
}

double nearest_rank(std::vector<double>& v, double q) {
    const size_t n = v.size();
    size_t r = static_cast<size_t>(std::ceil(q * static_cast<double>(n)));
    if (r < 1) r = 1;
    if (r > n) r = n;
    return v[r - 1];
}

}  // namespace

extern "C" {

const char* hostsim_last_error() { return g_err.c_str(); }
void hostsim_free(void* p) { std::free(p); }

// Run one replica on the CPU through the engine's own kernel logic.  Flags: -1 keeps the
// scenario's controller setting.  `comp` (optional) receives 6 arrays of per-completion data
// in canonical tenant order (tenant, seq, done, total, compute, transfer) -- see keep_completions.
static char* run_impl(const char* yaml_path, uint64_t seed, int enabled, int mig, int placement, int guard,
                      int keep_completions, double** comp_out, long* n_comp, const char* out_dir) {
    try {
        const bool traces = out_dir != nullptr;
        if (traces) keep_completions = 1;
        const ScenarioSpec spec = load_scenario(yaml_path);
        Variant v;
        v.enabled = enabled;
        v.enable_mig = mig;
        v.enable_placement = placement;
        v.enable_guardrails = guard;
        const Packed P = pack(spec, {v});
        const mg::PController& C = P.ctrl[0];
        const int T = P.scen.n_tenants, R = P.scen.n_roots;
        Arrivals A = generate(P, seed);
        std::vector<double> req(static_cast<size_t>(P.cap_sum), 0.0), win(static_cast<size_t>(P.cap_sum), 0.0);
        std::vector<double> cd, ct, cc, ctr, cn;
        std::vector<int64_t> corder;
        if (keep_completions) {
            cd.assign(static_cast<size_t>(P.cap_sum), 0.0);
            ct = cc = ctr = cn = cd;
            corder.assign(static_cast<size_t>(P.cap_sum), 0);
        }
        const int n_ticks = P.scen.n_ticks;
        std::vector<mg::CounterRow> trc;
        std::vector<mg::FabricRow> trf;
        std::vector<mg::TailWin> trw;
        std::vector<double> trr;
        if (traces) {
            trc.resize(static_cast<size_t>(n_ticks) * T);
            trf.resize(static_cast<size_t>(n_ticks) * R);
            trw.resize(static_cast<size_t>(T));
            trr.resize(static_cast<size_t>(T) * 256);
            for (int i = 0; i < T; ++i) {
                std::memset(&trw[i], 0, sizeof(mg::TailWin));
                trw[i].ring = trr.data() + 256 * i;
                trw[i].cap = 256;
            }
        }
        std::vector<uint64_t> mt(static_cast<size_t>(T) * mg::kMtN);
        std::vector<mg::ActionRec> acts(65536);
        std::vector<mg::PauseRec> pauses(65536);
        std::vector<mg::TenantOut> tout(static_cast<size_t>(T));
        mg::ReplicaOut rout{};
        std::vector<double> backlog(static_cast<size_t>(2 * R), 0.0);
        const mg::SimLayout L = mg::sim_layout(T, R, C.dwell_obs, C.validation_obs, true);
        std::vector<uint8_t> mem(static_cast<size_t>(L.total) + 64);
        uint8_t* base = mem.data();
        mg::SimState& st = *reinterpret_cast<mg::SimState*>(base);
        st.td = reinterpret_cast<mg::TenantDyn*>(base + L.td);
        st.ctl = reinterpret_cast<mg::TenantCtl*>(base + L.ctl);
        st.rd = reinterpret_cast<mg::RootDyn*>(base + L.rd);
        mg::Slot* slots = reinterpret_cast<mg::Slot*>(base + L.slots);
        mg::ReplicaIO io{};
        io.arr_t = A.t.data();
        io.arr_bytes = A.bytes.data();
        io.arr_mult = A.mult.data();
        io.arr_noise = A.noise.data();
        io.irq_e = A.irq.data();
        io.off = P.off.data();
        io.count = A.count.data();
        io.seed = seed;
        io.req_transfer_ms = req.data();
        io.mt_pause = mt.data();
        io.win_lat = win.data();
        io.actions = acts.data();
        io.action_cap = static_cast<int32_t>(acts.size());
        io.pauses = pauses.data();
        io.pause_cap = static_cast<int32_t>(pauses.size());
        io.tout = tout.data();
        io.rout = &rout;
        io.backlog = backlog.data();
        if (keep_completions) {
            io.c_done = cd.data();
            io.c_total = ct.data();
            io.c_compute = cc.data();
            io.c_transfer = ctr.data();
            io.c_noise = cn.data();
            io.c_order = corder.data();
        }
        if (traces) {
            io.tr_cnt = trc.data();
            io.tr_fab = trf.data();
            io.tr_win = trw.data();
        }
        mg::Sim<mg::HostLanes> sim(P.scen, C, io, st, mg::HostLanes{slots}, st.td, st.ctl, st.rd);
        sim.init(P.file_order.data(), reinterpret_cast<double*>(base + L.win), reinterpret_cast<double*>(base + L.vwin));
        sim.run();
        sim.finish();
        if (rout.error) throw std::runtime_error("device-side capacity overflow code " + std::to_string(rout.error));
        std::vector<double> quant(static_cast<size_t>(4 * T), 0.0);
        for (int i = 0; i < T; ++i) {
            const int64_t off = P.off[static_cast<size_t>(i)];
            std::vector<double> lat(win.begin() + off, win.begin() + off + static_cast<int64_t>(tout[i].completed_window));
            if (lat.empty()) continue;
            std::sort(lat.begin(), lat.end());
            quant[4 * i + 0] = nearest_rank(lat, 0.50);
            quant[4 * i + 1] = nearest_rank(lat, 0.95);
            quant[4 * i + 2] = nearest_rank(lat, 0.99);
            quant[4 * i + 3] = nearest_rank(lat, 0.999);
        }
        RunResult r = assemble(spec, P, "as-is", seed, tout.data(), quant.data(), acts.data(), rout.n_actions,
                               pauses.data(), rout.n_pauses, backlog.data(), rout.n_events);
        if (traces) {
            TraceRows tr;
            tr.off = P.off;
            for (int i = 0; i < T; ++i) tr.n_done.push_back(tout[i].completed_total);
            tr.done = cd;
            tr.total = ct;
            tr.compute = cc;
            tr.transfer = ctr;
            tr.noise = cn;
            tr.arrived = A.t;
            tr.bytes = A.bytes;
            tr.order = corder;
            tr.n_ticks = n_ticks;
            tr.counters = trc;
            tr.fabric = trf;
            write_run_artifacts(out_dir, spec, P, r, &tr);
        }
        if (keep_completions && comp_out) {
            long n = 0;
            for (int i = 0; i < T; ++i) n += static_cast<long>(tout[i].completed_total);
            double* out = static_cast<double*>(std::malloc(sizeof(double) * 7 * static_cast<size_t>(n) + 8));
            long k = 0;
            for (int i = 0; i < T; ++i) {
                const int64_t off = P.off[static_cast<size_t>(i)];
                for (uint64_t c = 0; c < tout[i].completed_total; ++c, ++k) {
                    const int64_t o = off + static_cast<int64_t>(c);
                    out[7 * k + 0] = i;
                    out[7 * k + 1] = static_cast<double>(c);
                    out[7 * k + 2] = cd[o];
                    out[7 * k + 3] = ct[o];
                    out[7 * k + 4] = cc[o];
                    out[7 * k + 5] = ctr[o];
                    out[7 * k + 6] = cn[o];
                }
            }
            *comp_out = out;
            *n_comp = n;
        }
        return dup(result_to_json(r));
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

char* hostsim_run(const char* yaml_path, uint64_t seed, int enabled, int mig, int placement, int guard,
                  int keep_completions, double** comp_out, long* n_comp) {
    return run_impl(yaml_path, seed, enabled, mig, placement, guard, keep_completions, comp_out, n_comp, nullptr);
}

// run_scenario with files (RunOptions{seed, out_dir, write_traces=true}) through the engine logic
char* hostsim_run_artifacts(const char* yaml_path, uint64_t seed, const char* out_dir) {
    return run_impl(yaml_path, seed, -1, -1, -1, -1, 1, nullptr, nullptr, out_dir);
}

// Arrival records of one tenant (canonical index) as generated by the engine's generator code.
long hostsim_arrivals(const char* yaml_path, uint64_t seed, int tenant, double* out, long cap) {
    try {
        const ScenarioSpec spec = load_scenario(yaml_path);
        const Packed P = pack(spec, {});
        Arrivals A = generate(P, seed);
        const int64_t off = P.off[static_cast<size_t>(tenant)];
        const long n = A.count[static_cast<size_t>(tenant)];
        for (long k = 0; k < n && k < cap; ++k) {
            out[4 * k + 0] = A.t[off + k];
            out[4 * k + 1] = A.bytes[off + k];
            out[4 * k + 2] = A.mult[off + k];
            out[4 * k + 3] = A.noise[off + k];
        }
        return n;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// latency bins shared by the DES and the select kernel (lat_hist.h): bin and the bin's key floor
void hostsim_lat_bin(const double* x, uint32_t* bin, uint64_t* key, uint64_t* lo, long n) {
    for (long i = 0; i < n; ++i) {
        bin[i] = mg::lat_bin(x[i]);
        key[i] = mg::lat_key(x[i]);
        lo[i] = mg::lat_bin_lo(bin[i]);
    }
}

// glibc-exact math restatement, for the CPU bit-compare test.
void hostsim_math(int fn, const double* x, const double* y, double* out, long n) {
    for (long i = 0; i < n; ++i)
        out[i] = fn == 0 ? mg::gl_log(x[i]) : fn == 1 ? mg::gl_exp(x[i]) : fn == 2 ? mg::gl_pow(x[i], y[i])
                                                                 : mg::fmod_fast(x[i], y[i]);
}

// the engine's sliding window (des_core.h TailWin: cached top-K + linear selection beyond it):
// out[i] = quantile(q) after push i, same contract as the oracle's ref_tailwindow_run
void hostsim_tailwin_run(long capacity, const double* xs, long n, double q, double* out) {
    std::vector<double> ring(static_cast<size_t>(capacity));
    mg::TailWin w{};
    w.ring = ring.data();
    w.cap = static_cast<int32_t>(capacity);
    mg::tw_reset(w, 1e300);
    for (long i = 0; i < n; ++i) {
        mg::tw_push(w, xs[i]);
        out[i] = mg::tw_quantile(w, q);
    }
}

double hostsim_select_jth(const double* v, long n, long j) {
    return mg::select_jth_largest(v, static_cast<int>(n), static_cast<int>(j));
}

}  // extern "C"
