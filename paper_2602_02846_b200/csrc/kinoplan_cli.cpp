// kinoplan_cli.cpp — the `kinoplan` command line (the reference's
// apps/ CLI sources are absent).
//
//   kinoplan plan     --scenario F [--seed S] [--workers W] [--time-limit-ms T]
//                     [--max-iterations N] [--out DIR] [--deterministic]
//   kinoplan bench    --scenario F --out DIR [--trials N] [--workers W] [--seed S]
//                     [--time-limit-ms T] [--max-iterations N] [--deterministic]
//   kinoplan validate --scenario F            (parse + print, no GPU)
//   kinoplan report   --records F --out DIR   (re-emit CSV + SVG from stored records, no GPU)
//
// Exit status: 0 on success, also when planning finds no solution
// (infeasibility is data); 2 for usage errors, 3 for scenario errors, 1 for
// anything else (device, I/O).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <map>
#include <string>

#include "kinoplan_b200/bench.hpp"

namespace fs = std::filesystem;
using namespace kinoplan;

namespace {

struct Args {
    std::string cmd;
    std::map<std::string, std::string> kv;
    bool deterministic = false;
};

[[noreturn]] void usage(const char* msg) {
    std::fprintf(stderr,
                 "%s\nusage: kinoplan plan --scenario F [--seed S] [--workers W] [--time-limit-ms T] "
                 "[--max-iterations N] [--out DIR] [--deterministic]\n"
                 "       kinoplan bench --scenario F --out DIR [--trials N] [--workers W] [--seed S] "
                 "[--time-limit-ms T] [--max-iterations N] [--deterministic]\n"
                 "       kinoplan validate --scenario F\n"
                 "       kinoplan report --records F --out DIR\n",
                 msg);
    std::exit(2);
}

Args parse_args(int argc, char** argv) {
    if (argc < 2) usage("missing command");
    Args a;
    a.cmd = argv[1];
    static const char* known[] = {"--scenario", "--seed", "--workers", "--time-limit-ms", "--max-iterations",
                                  "--out", "--trials", "--records"};
    for (int i = 2; i < argc; ++i) {
        std::string f = argv[i];
        if (f == "--deterministic") { a.deterministic = true; continue; }
        bool ok = false;
        for (const char* k : known) ok |= f == k;
        if (!ok) usage(("unknown flag " + f).c_str());
        if (i + 1 >= argc) usage((f + " needs a value").c_str());
        a.kv[f.substr(2)] = argv[++i];
    }
    return a;
}

ScenarioOverrides overrides(const Args& a) {
    ScenarioOverrides ov;
    try {
        if (a.kv.count("seed")) ov.seed = std::stoull(a.kv.at("seed"));
        if (a.kv.count("workers")) ov.workers = std::stoi(a.kv.at("workers"));
        if (a.kv.count("time-limit-ms")) ov.time_limit_ms = std::stod(a.kv.at("time-limit-ms"));
        if (a.kv.count("max-iterations")) ov.max_iterations = std::stoull(a.kv.at("max-iterations"));
        if (a.kv.count("trials")) ov.trials = std::stoi(a.kv.at("trials"));
    } catch (const std::exception&) {
        usage("malformed numeric flag value");
    }
    if (a.deterministic) ov.workers = 1;
    return ov;
}

std::string num(double v) {
    char b[40];
    std::snprintf(b, sizeof b, "%.17g", v);
    return std::isfinite(v) ? std::string(b) : (std::isnan(v) ? "NaN" : (v > 0 ? "Infinity" : "-Infinity"));
}

void ensure_dir(const std::string& d) {
    std::error_code ec;
    fs::create_directories(d, ec);
    if (ec) throw std::runtime_error(d + ": " + ec.message());
}

int cmd_validate(const Args& a) {
    if (!a.kv.count("scenario")) usage("--scenario is required");
    Scenario s = load_scenario(a.kv.at("scenario"), overrides(a));
    const PlannerConfig& c = s.config;
    std::printf("{\"name\": \"%s\", \"model\": \"%s\", \"state_dim\": %d, \"control_dim\": %d, \"obstacles\": %zu, "
                "\"decomposition_dims\": %zu, \"lambda\": %d, \"i_max\": %d, \"t_prop\": %s, \"t_max_ms\": %s, "
                "\"max_iterations\": %llu, \"capacity\": %llu, \"trials\": %d, \"base_seed\": %llu, \"workers\": %d}\n",
                s.name.c_str(), s.problem.model->id().c_str(), s.problem.model->state_dim(),
                s.problem.model->control_dim(), s.problem.environment.obstacles.size(), c.decomposition.dims.size(),
                c.lambda, c.i_max, num(c.t_prop).c_str(), num(c.t_max * 1e3).c_str(),
                static_cast<unsigned long long>(c.max_iterations), static_cast<unsigned long long>(c.capacity),
                s.n_trials, static_cast<unsigned long long>(s.base_seed), s.workers);
    return 0;
}

int cmd_plan(const Args& a) {
    if (!a.kv.count("scenario")) usage("--scenario is required");
    Scenario s = load_scenario(a.kv.at("scenario"), overrides(a));
    PlanResult r = plan(s.problem, s.config);
    const PlannerStats& st = r.stats;
    std::string stats =
        "{\"scenario\": \"" + s.name + "\", \"seed\": " + std::to_string(s.base_seed) +
        ", \"success\": " + (std::isfinite(r.best.cost) ? "true" : "false") + ", \"best_cost\": " + num(r.best.cost) +
        ", \"best_found_ms\": " + num(r.best.found_at * 1e3) +
        ", \"first_solution_ms\": " + num(st.first_solution ? st.first_solution->first * 1e3 : NAN) +
        ", \"first_solution_cost\": " + num(st.first_solution ? st.first_solution->second : NAN) +
        ", \"first_solution_iteration\": " + std::to_string(st.first_solution_iteration) +
        ", \"iterations\": " + std::to_string(st.iterations) + ", \"elapsed_ms\": " + num(st.elapsed * 1e3) +
        ", \"propagations_attempted\": " + std::to_string(st.propagations_attempted) +
        ", \"propagations_valid\": " + std::to_string(st.propagations_valid) +
        ", \"nodes_committed\": " + std::to_string(st.nodes_committed) +
        ", \"node_count\": " + std::to_string(st.node_count) +
        ", \"capacity_exhausted\": " + (st.capacity_exhausted ? "true" : "false") + "}";
    std::printf("%s\n", stats.c_str());
    if (a.kv.count("out")) {
        const std::string d = a.kv.at("out");
        ensure_dir(d);
        {
            FILE* f = std::fopen((d + "/stats.json").c_str(), "wb");
            if (!f) throw std::runtime_error(d + "/stats.json: " + std::strerror(errno));
            std::fprintf(f, "%s\n", stats.c_str());
            std::fclose(f);
        }
        if (r.trajectory) emit_trajectory(*r.trajectory, d + "/trajectory.csv");
        TrialRecord t;
        t.seed = s.base_seed;
        t.success = std::isfinite(r.best.cost);
        if (st.first_solution) t.first_solution = std::make_pair(st.first_solution->first * 1e3, st.first_solution->second);
        if (t.success) t.final_solution = std::make_pair(r.best.found_at * 1e3, r.best.cost);
        for (const auto& [sec, c] : st.cost_timeline) t.cost_timeline.emplace_back(sec * 1e3, c);
        t.iterations = st.iterations;
        t.propagations = st.propagations_attempted;
        t.first_iteration = st.first_solution_iteration;
        emit_records({t}, s.name, d + "/records.json");
    }
    return 0;
}

void emit_all(const std::vector<TrialRecord>& rec, const std::string& name, const std::string& d) {
    ensure_dir(d);
    emit_records(rec, name, d + "/" + name + ".records.json");
    emit_csv(rec, summarize(name, rec), d + "/" + name + ".csv");
    emit_cost_curve(rec, d + "/" + name + ".svg");
}

int cmd_bench(const Args& a) {
    if (!a.kv.count("scenario")) usage("--scenario is required");
    if (!a.kv.count("out")) usage("--out is required");
    Scenario s = load_scenario(a.kv.at("scenario"), overrides(a));
    std::vector<TrialRecord> rec = run_trials(s);
    emit_all(rec, s.name, a.kv.at("out"));
    SummaryRow sr = summarize(s.name, rec);
    std::printf("{\"scenario\": \"%s\", \"trials\": %zu, \"success_rate\": %s, \"first_ms\": %s, \"first_cost\": %s, "
                "\"final_ms\": %s, \"final_cost\": %s}\n",
                s.name.c_str(), rec.size(), num(sr.success_rate).c_str(), num(sr.first_ms).c_str(),
                num(sr.first_cost).c_str(), num(sr.final_ms).c_str(), num(sr.final_cost).c_str());
    return 0;
}

int cmd_report(const Args& a) {
    if (!a.kv.count("records")) usage("--records is required");
    if (!a.kv.count("out")) usage("--out is required");
    std::string name;
    std::vector<TrialRecord> rec = load_records(a.kv.at("records"), &name);
    if (name.empty()) name = fs::path(a.kv.at("records")).stem().string();
    emit_csv(rec, summarize(name, rec), a.kv.at("out") + "/" + name + ".csv");
    emit_cost_curve(rec, a.kv.at("out") + "/" + name + ".svg");
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    Args a = parse_args(argc, argv);
    try {
        if (a.cmd == "plan") return cmd_plan(a);
        if (a.cmd == "bench") return cmd_bench(a);
        if (a.cmd == "validate") return cmd_validate(a);
        if (a.cmd == "report") {
            ensure_dir(a.kv.count("out") ? a.kv.at("out") : ".");
            return cmd_report(a);
        }
        usage(("unknown command " + a.cmd).c_str());
    } catch (const SchemaError& e) {
        std::fprintf(stderr, "kinoplan: schema error: %s\n", e.what());
        return 3;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "kinoplan: error: %s\n", e.what());
        return 1;
    }
}
