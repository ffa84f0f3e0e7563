// Run artifacts of one replica, byte-identical to the reference's writers:
//   summary.json, actions.jsonl        trace.cpp:98-203 (nlohmann::ordered_json, dump(2) / dump())
//   requests.csv, counters.csv, fabric.csv   trace.cpp:24-96 ("%.9g"), emitted by engine.cpp:279-288,
//                                            :503 (per completion) and :744-775 (per tick)
// The engine (GPU) returns the raw rows; this file only formats them.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "../common/des_types.h"
#include "packer.hpp"

namespace mgb {

// Raw trace data of one replica as the device returns it.
struct TraceRows {
    // completions, canonical tenant t owns [off[t], off[t] + n_done[t]) of each array
    std::vector<int64_t> off;
    std::vector<uint64_t> n_done;
    std::vector<double> done, total, compute, transfer, noise, arrived, bytes;
    std::vector<int64_t> order;  // global completion order of each record
    // per tick: counters [n_ticks][T], fabric [n_ticks][R]
    int n_ticks = 0;
    std::vector<mg::CounterRow> counters;
    std::vector<mg::FabricRow> fabric;
};

std::string fmt_double(double v);  // trace.cpp:24-28
std::string summary_json_text(const RunResult& r);               // summary.json body (dump(2) + "\n")
std::string actions_jsonl_text(const std::vector<ActionRecord>& a);  // actions.jsonl
std::string requests_csv_text(const Packed& p, const TraceRows& t);
std::string counters_csv_text(const Packed& p, const TraceRows& t);
std::string fabric_csv_text(const ScenarioSpec& spec, const Packed& p, const TraceRows& t);

// harness::ExperimentResult aggregates (harness.hpp:54-73) of one plan
struct PlanVariantOut {
    std::string name;
    std::vector<uint64_t> seeds;
    std::vector<double> p99_ms, miss_rate, throughput_hz;  // per seed
    double mean[3] = {0, 0, 0}, half[3] = {0, 0, 0};        // p99, miss, throughput CIs
};
// experiment.json body (harness.cpp:235-269, dump(2)), summary.csv (harness.cpp:271-283),
// render_report of an experiment.json text (harness.cpp:285-313)
std::string experiment_json_text(const std::string& plan, const std::string& scenario, const std::string& focus,
                                 double wall_s, const std::vector<PlanVariantOut>& v);
std::string experiment_csv_text(const std::vector<PlanVariantOut>& v);
std::string render_report_text(const std::string& experiment_json);
void put_text_file(const std::string& path, const std::string& text);

// engine::run_scenario's file side (engine.cpp:279-288, 889-892): creates out_dir, writes the three
// trace streams when `traces` is non-null, then actions.jsonl and summary.json.
void write_run_artifacts(const std::string& out_dir, const ScenarioSpec& spec, const Packed& p, const RunResult& r,
                         const TraceRows* traces);

}  // namespace mgb
