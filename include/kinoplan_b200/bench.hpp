// kinoplan_b200/bench.hpp — scenario files, trial runner and report emitters
// (the reference's `bench` module; src/scenario.cpp,
// src/runner.cpp, src/report.cpp are absent from the reference and restated
// here above the GPU planner).
#pragma once

#include <cstdint>
#include <optional>
#include <string>
#include <vector>

#include "kinoplan_b200/kinoplan.hpp"

namespace kinoplan {

/// Scenario: problem + config + trial controls.
struct Scenario {
    std::string name;
    PlanningProblem problem;
    PlannerConfig config;
    int n_trials = 1;
    uint64_t base_seed = 0;
    int workers = 1;
};

/// CLI-style overrides (flags override scenario values).
struct ScenarioOverrides {
    std::optional<uint64_t> seed;
    std::optional<int> workers;
    std::optional<double> time_limit_ms;
    std::optional<uint64_t> max_iterations;
    std::optional<int> trials;
};

/// Parses the scenario document (SPEC.md:518 keys).  Throws SchemaError with
/// the offending field path ("scenario.problem.goal.radius: ...").
Scenario parse_scenario(const std::string& json_text, const ScenarioOverrides& ov = {});
Scenario load_scenario(const std::string& path, const ScenarioOverrides& ov = {});

/// TrialRecord.
struct TrialRecord {
    uint64_t seed = 0;
    bool success = false;
    std::optional<std::pair<double, double>> first_solution;  // (ms, cost)
    std::optional<std::pair<double, double>> final_solution;  // (ms, cost)
    std::vector<std::pair<double, double>> cost_timeline;    // (ms, cost)
    uint64_t iterations = 0, propagations = 0, first_iteration = 0;
};

/// SummaryRow: medians over successful trials only (odd n:
/// middle order statistic, even n: lower-middle); NaN when none.
struct SummaryRow {
    std::string scenario;
    double first_ms = 0, first_cost = 0, final_ms = 0, final_cost = 0;
    double success_rate = 0;  // percent over all trials
    std::optional<double> normalization;
};

/// Lower-middle median; NaN for an empty sample.
double lower_median(std::vector<double> v);

/// run_trials: n independent runs, trial k uses seed =
/// base_seed + k, on one reusable GPU planner instance.
std::vector<TrialRecord> run_trials(const Scenario& s);
SummaryRow summarize(const std::string& name, const std::vector<TrialRecord>& records,
                     std::optional<double> normalization = std::nullopt);

/// emit_csv: `path` gets a header line + one line per trial
/// (seed, success, first_ms, first_cost, final_ms, final_cost, first_iteration,
/// iterations), `path.summary.csv` the SummaryRow; %.17g round-trip precision.
void emit_csv(const std::vector<TrialRecord>& records, const SummaryRow& summary, const std::string& path);

/// emit_cost_curve: self-contained SVG, log-scaled time axis,
/// per-trial step curves, median curve; an annotated empty plot if no trial
/// has a timeline.
void emit_cost_curve(const std::vector<TrialRecord>& records, const std::string& path);

/// Full trial records (timelines included) as JSON, and the reader, so the
/// emitters can be re-run on stored results (`kinoplan report`).
void emit_records(const std::vector<TrialRecord>& records, const std::string& scenario, const std::string& path);
std::vector<TrialRecord> load_records(const std::string& path, std::string* scenario = nullptr);

/// Writes the solution trajectory (samples, controls, durations) as CSV.
void emit_trajectory(const Trajectory& t, const std::string& path);

}  // namespace kinoplan
