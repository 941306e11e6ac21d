// bench.cpp — scenario files, trial runner and report emitters.
//
// The reference's bench sources (src/scenario.cpp, src/runner.cpp,
// src/report.cpp) are absent; this restates the SPEC module on
// top of the GPU planner (kinoplan::Planner).  Host code only: every plan
// runs through the C-ABI on the device.
#include "kinoplan_b200/bench.hpp"

#include <algorithm>
#include <atomic>
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <limits>
#include <map>
#include <sstream>
#include <thread>
#include <variant>

namespace kinoplan {
namespace {

// ---------------------------------------------------------------------------
// Minimal JSON reader: objects, arrays, numbers (raw text kept so integer
// seeds above 2^53 survive), strings, true/false/null.
// ---------------------------------------------------------------------------
struct Json {
    enum class T { Null, Bool, Num, Str, Arr, Obj } t = T::Null;
    bool b = false;
    std::string s;  // string value, or raw number text
    std::vector<Json> a;
    std::vector<std::pair<std::string, Json>> o;

    const Json* get(const std::string& k) const {
        for (const auto& [kk, v] : o)
            if (kk == k) return &v;
        return nullptr;
    }
};

class Reader {
public:
    explicit Reader(const std::string& src) : p_(src.data()), b_(src.data()), e_(src.data() + src.size()) {}

    Json parse() {
        Json v = value();
        ws();
        if (p_ != e_) fail("trailing characters");
        return v;
    }

private:
    const char *p_, *b_, *e_;

    [[noreturn]] void fail(const std::string& what) const {
        int line = 1, col = 1;
        for (const char* q = b_; q < p_; ++q) {
            if (*q == '\n') { ++line; col = 1; } else { ++col; }
        }
        throw SchemaError("scenario: JSON syntax error at line " + std::to_string(line) + " column " +
                          std::to_string(col) + ": " + what);
    }
    void ws() {
        while (p_ < e_ && (*p_ == ' ' || *p_ == '\t' || *p_ == '\n' || *p_ == '\r')) ++p_;
    }
    bool lit(const char* w) {
        size_t n = std::strlen(w);
        if (static_cast<size_t>(e_ - p_) >= n && std::memcmp(p_, w, n) == 0) { p_ += n; return true; }
        return false;
    }
    Json value() {
        ws();
        if (p_ == e_) fail("unexpected end of input");
        Json v;
        char c = *p_;
        if (c == '{') {
            v.t = Json::T::Obj;
            ++p_;
            ws();
            if (p_ < e_ && *p_ == '}') { ++p_; return v; }
            for (;;) {
                ws();
                if (p_ == e_ || *p_ != '"') fail("expected a key string");
                std::string k = str();
                ws();
                if (p_ == e_ || *p_ != ':') fail("expected ':'");
                ++p_;
                v.o.emplace_back(std::move(k), value());
                ws();
                if (p_ < e_ && *p_ == ',') { ++p_; continue; }
                if (p_ < e_ && *p_ == '}') { ++p_; return v; }
                fail("expected ',' or '}'");
            }
        }
        if (c == '[') {
            v.t = Json::T::Arr;
            ++p_;
            ws();
            if (p_ < e_ && *p_ == ']') { ++p_; return v; }
            for (;;) {
                v.a.push_back(value());
                ws();
                if (p_ < e_ && *p_ == ',') { ++p_; continue; }
                if (p_ < e_ && *p_ == ']') { ++p_; return v; }
                fail("expected ',' or ']'");
            }
        }
        if (c == '"') { v.t = Json::T::Str; v.s = str(); return v; }
        if (lit("true")) { v.t = Json::T::Bool; v.b = true; return v; }
        if (lit("false")) { v.t = Json::T::Bool; return v; }
        if (lit("null")) return v;
        if (lit("NaN")) { v.t = Json::T::Num; v.s = "nan"; return v; }           // Python json.dump emits these
        if (lit("Infinity")) { v.t = Json::T::Num; v.s = "inf"; return v; }
        if (lit("-Infinity")) { v.t = Json::T::Num; v.s = "-inf"; return v; }
        const char* st = p_;
        if (p_ < e_ && (*p_ == '-' || *p_ == '+')) ++p_;
        while (p_ < e_ && (std::isdigit(static_cast<unsigned char>(*p_)) || *p_ == '.' || *p_ == 'e' || *p_ == 'E' ||
                           *p_ == '-' || *p_ == '+'))
            ++p_;
        if (p_ == st) fail(std::string("unexpected character '") + c + "'");
        v.t = Json::T::Num;
        v.s.assign(st, p_);
        return v;
    }
    std::string str() {
        ++p_;  // opening quote
        std::string out;
        while (p_ < e_ && *p_ != '"') {
            if (*p_ == '\\') {
                if (++p_ == e_) break;
                switch (*p_) {
                    case 'n': out += '\n'; break;
                    case 't': out += '\t'; break;
                    case 'r': out += '\r'; break;
                    case 'b': out += '\b'; break;
                    case 'f': out += '\f'; break;
                    case 'u': {
                        if (e_ - p_ < 5) fail("bad \\u escape");
                        unsigned cp = std::stoul(std::string(p_ + 1, p_ + 5), nullptr, 16);
                        p_ += 4;
                        if (cp < 0x80) out += static_cast<char>(cp);
                        else if (cp < 0x800) { out += static_cast<char>(0xC0 | (cp >> 6)); out += static_cast<char>(0x80 | (cp & 63)); }
                        else { out += static_cast<char>(0xE0 | (cp >> 12)); out += static_cast<char>(0x80 | ((cp >> 6) & 63)); out += static_cast<char>(0x80 | (cp & 63)); }
                        break;
                    }
                    default: out += *p_;
                }
                ++p_;
            } else {
                out += *p_++;
            }
        }
        if (p_ == e_) fail("unterminated string");
        ++p_;
        return out;
    }
};

// ---- typed field access with field paths ----
struct Field {
    const Json* j;
    std::string path;

    [[noreturn]] void bad(const std::string& what) const { throw SchemaError(path + ": " + what); }
    Field at(const std::string& k) const {
        if (j->t != Json::T::Obj) bad("expected an object");
        const Json* v = j->get(k);
        if (!v) throw SchemaError(path + "." + k + ": missing");
        return {v, path + "." + k};
    }
    std::optional<Field> opt(const std::string& k) const {
        if (j->t != Json::T::Obj) bad("expected an object");
        const Json* v = j->get(k);
        if (!v || v->t == Json::T::Null) return std::nullopt;
        return Field{v, path + "." + k};
    }
    Field idx(size_t i) const { return {&j->a[i], path + "[" + std::to_string(i) + "]"}; }
    size_t size() const {
        if (j->t != Json::T::Arr) bad("expected an array");
        return j->a.size();
    }
    double num() const {
        if (j->t != Json::T::Num) bad("expected a number");
        char* end = nullptr;
        double v = std::strtod(j->s.c_str(), &end);
        if (end == j->s.c_str()) bad("malformed number '" + j->s + "'");
        return v;
    }
    int64_t integer() const {
        double v = num();
        if (v != std::floor(v)) bad("expected an integer, got " + j->s);
        return static_cast<int64_t>(v);
    }
    uint64_t u64() const {
        if (j->t != Json::T::Num) bad("expected a non-negative integer");
        if (j->s.find_first_of(".eE-") == std::string::npos) {
            errno = 0;
            unsigned long long v = std::strtoull(j->s.c_str(), nullptr, 10);
            if (errno == ERANGE) bad("integer out of range");
            return v;
        }
        double v = num();
        if (v < 0 || v != std::floor(v)) bad("expected a non-negative integer, got " + j->s);
        return static_cast<uint64_t>(v);
    }
    bool boolean() const {
        if (j->t != Json::T::Bool) bad("expected true/false");
        return j->b;
    }
    const std::string& string() const {
        if (j->t != Json::T::Str) bad("expected a string");
        return j->s;
    }
    std::vector<double> nums() const {
        std::vector<double> v;
        for (size_t i = 0; i < size(); ++i) v.push_back(idx(i).num());
        return v;
    }
    std::vector<int> ints() const {
        std::vector<int> v;
        for (size_t i = 0; i < size(); ++i) v.push_back(static_cast<int>(idx(i).integer()));
        return v;
    }
    Bounds bounds() const {
        Bounds b;
        for (size_t i = 0; i < size(); ++i) {
            Field e = idx(i);
            if (e.size() != 2) e.bad("expected [lo, hi]");
            Interval iv{e.idx(0).num(), e.idx(1).num()};
            if (!(iv.lo <= iv.hi)) e.bad("lo > hi");
            b.push_back(iv);
        }
        return b;
    }
};

void fill_xyz(double* out, const std::vector<double>& v, const Field& f) {
    if (v.empty() || v.size() > 3) f.bad("expected 1..3 coordinates");
    for (size_t i = 0; i < v.size(); ++i) out[i] = v[i];
}

std::string fmt(double v) {
    if (std::isnan(v)) return "NaN";
    if (std::isinf(v)) return v > 0 ? "inf" : "-inf";
    char buf[40];
    std::snprintf(buf, sizeof buf, "%.17g", v);
    return buf;
}

std::ofstream open_out(const std::string& path) {
    std::ofstream f(path, std::ios::binary | std::ios::trunc);
    if (!f) throw std::runtime_error(path + ": " + std::strerror(errno));
    return f;
}

void close_out(std::ofstream& f, const std::string& path) {
    f.close();
    if (!f) throw std::runtime_error(path + ": write failed: " + std::strerror(errno));
}

// Environment fragment: workspace_bounds, optional
// state_bounds, obstacles; SchemaError names the offending primitive.
Environment parse_environment(const Field& env) {
    Environment e;
    e.workspace_bounds = env.at("workspace_bounds").bounds();
    if (e.workspace_bounds.size() < 2 || e.workspace_bounds.size() > 3)
        env.at("workspace_bounds").bad("expected 2 or 3 intervals");
    if (auto sb = env.opt("state_bounds")) e.state_bounds = sb->bounds();
    if (auto obs = env.opt("obstacles")) {
        for (size_t i = 0; i < obs->size(); ++i) {
            Field o = obs->idx(i);
            const std::string& ty = o.at("type").string();
            Obstacle ob;
            if (ty == "box") {
                ob.type = Obstacle::Type::Box;
                fill_xyz(ob.a, o.at("min").nums(), o.at("min"));
                fill_xyz(ob.b, o.at("max").nums(), o.at("max"));
                for (int k = 0; k < 3; ++k)
                    if (ob.a[k] > ob.b[k]) o.bad("box min > max");
            } else if (ty == "sphere") {
                ob.type = Obstacle::Type::Sphere;
                fill_xyz(ob.a, o.at("center").nums(), o.at("center"));
                ob.b[0] = o.at("radius").num();
                if (!(ob.b[0] > 0)) o.at("radius").bad("sphere radius <= 0");
            } else {
                o.at("type").bad("unknown obstacle type \"" + ty + "\"");
            }
            e.obstacles.push_back(ob);
        }
    }
    return e;
}

}  // namespace

Environment load_environment(const std::string& json_fragment) {
    Json root = Reader(json_fragment).parse();
    return parse_environment(Field{&root, "environment"});
}

// ---------------------------------------------------------------------------
// Scenario
// ---------------------------------------------------------------------------
Scenario parse_scenario(const std::string& text, const ScenarioOverrides& ov) {
    Json root = Reader(text).parse();
    Field sc{&root, "scenario"};
    if (root.t != Json::T::Obj) sc.bad("expected an object");
    Scenario s;
    s.name = sc.at("name").string();

    Field pr = sc.at("problem");
    ModelParams mp;
    if (auto f = pr.opt("model_params")) {
        if (f->j->t != Json::T::Obj) f->bad("expected an object");
        for (const auto& [k, v] : f->j->o) mp.values[k] = Field{&v, f->path + "." + k}.num();
    }
    Field model = pr.at("model");
    try {
        s.problem.model = make_model(model.string(), mp);
    } catch (const SchemaError& e) {
        model.bad(e.what());
    }
    const DynamicsModel& md = *s.problem.model;

    s.problem.environment = parse_environment(pr.at("environment"));
    Field xi = pr.at("x_init");
    s.problem.x_init = xi.nums();
    if (static_cast<int>(s.problem.x_init.size()) != md.state_dim())
        xi.bad("expected " + std::to_string(md.state_dim()) + " values for " + md.id());

    Field goal = pr.at("goal");
    if (auto d = goal.opt("dims")) s.problem.goal.dims = d->ints();
    else s.problem.goal.dims.assign(md.position_dims().begin(), md.position_dims().end());
    s.problem.goal.center = goal.at("center").nums();
    if (s.problem.goal.center.size() != s.problem.goal.dims.size())
        goal.at("center").bad("length differs from goal.dims");
    s.problem.goal.radius = goal.at("radius").num();
    if (!(s.problem.goal.radius > 0)) goal.at("radius").bad("must be > 0");

    s.problem.cost.position_dims = static_cast<int>(md.position_dims().size());
    if (auto c = pr.opt("cost")) {
        std::string kind;
        if (c->j->t == Json::T::Obj) {
            kind = c->opt("kind") ? c->at("kind").string() : "path_length";
            if (auto pd = c->opt("position_dims")) s.problem.cost.position_dims = static_cast<int>(pd->integer());
            if (auto lh = c->opt("lipschitz_hint")) s.problem.cost.lipschitz_hint = lh->num();
        } else {
            kind = c->string();
        }
        if (kind == "path_length") s.problem.cost.kind = CostKind::PathLength;
        else if (kind == "control_duration") s.problem.cost.kind = CostKind::ControlDuration;
        else c->bad("unknown cost metric kind \"" + kind + "\"");
    }
    Field sb = pr.at("state_bounds");
    s.problem.state_bounds = sb.bounds();
    if (static_cast<int>(s.problem.state_bounds.size()) != md.state_dim())
        sb.bad("expected " + std::to_string(md.state_dim()) + " intervals");
    Field cb = pr.at("control_bounds");
    s.problem.control_bounds = cb.bounds();
    if (static_cast<int>(s.problem.control_bounds.size()) != md.control_dim())
        cb.bad("expected " + std::to_string(md.control_dim()) + " intervals");

    Field dec = sc.at("decomposition");
    PlannerConfig& cf = s.config;
    cf.decomposition.dims = dec.at("dims").ints();
    auto delta = dec.opt("delta");
    auto cells = dec.opt("cells");
    if (static_cast<bool>(delta) == static_cast<bool>(cells)) dec.bad("exactly one of delta / cells is required");
    if (delta) cf.decomposition.delta = delta->num();
    if (cells) {
        cf.decomposition.cells = cells->ints();
        if (cf.decomposition.cells.size() != cf.decomposition.dims.size()) cells->bad("length differs from dims");
    }
    if (auto mc = dec.opt("max_cells")) cf.decomposition.max_cells = mc->u64();

    Field pl = sc.at("planner");
    if (auto v = pl.opt("lambda")) cf.lambda = static_cast<int>(v->integer());
    if (auto v = pl.opt("i_max")) cf.i_max = static_cast<int>(v->integer());
    cf.t_prop = pl.at("t_prop").num();
    if (auto v = pl.opt("capacity")) cf.capacity = v->u64();
    if (auto v = pl.opt("ode_step")) { double h = v->num(); if (h > 0) cf.ode_step = h; }
    if (auto v = pl.opt("collision_step")) cf.collision_step = v->num();
    if (auto v = pl.opt("t_max_ms")) cf.t_max = v->num() / 1000.0;
    if (auto v = pl.opt("max_iterations")) cf.max_iterations = v->u64();
    if (auto v = pl.opt("deactivate_after_expansion")) cf.deactivate_after_expansion = v->boolean();
    if (auto v = pl.opt("stop_at_first_solution")) cf.stop_at_first_solution = v->boolean();
    if (auto v = pl.opt("max_slots")) cf.max_slots = v->u64();
    if (auto v = pl.opt("rng")) {
        const std::string& r = v->string();
        if (r == "philox") cf.rng = RngKind::Philox;
        else if (r == "splitmix") cf.rng = RngKind::SplitMix;
        else v->bad("unknown rng \"" + r + "\" (philox | splitmix)");
    }
    if (auto tr = sc.opt("trials")) {
        if (auto v = tr->opt("n")) s.n_trials = static_cast<int>(v->integer());
        if (auto v = tr->opt("base_seed")) s.base_seed = v->u64();
        if (auto v = tr->opt("workers")) s.workers = static_cast<int>(v->integer());
    }
    if (auto v = pl.opt("seed")) s.base_seed = v->u64();

    if (ov.seed) s.base_seed = *ov.seed;
    if (ov.workers) s.workers = *ov.workers;
    if (ov.time_limit_ms) cf.t_max = *ov.time_limit_ms / 1000.0;
    if (ov.max_iterations) cf.max_iterations = *ov.max_iterations;
    if (ov.trials) s.n_trials = *ov.trials;
    if (s.n_trials < 0) throw SchemaError("scenario.trials.n: must be >= 0");
    if (s.workers < 1) throw SchemaError("scenario.trials.workers: must be >= 1");
    cf.seed = s.base_seed;
    cf.workers = s.workers;
    return s;
}

Scenario load_scenario(const std::string& path, const ScenarioOverrides& ov) {
    std::ifstream f(path, std::ios::binary);
    if (!f) throw SchemaError(path + ": " + std::strerror(errno));
    std::stringstream ss;
    ss << f.rdbuf();
    try {
        return parse_scenario(ss.str(), ov);
    } catch (const SchemaError& e) {
        throw SchemaError(path + ": " + e.what());
    }
}

// ---------------------------------------------------------------------------
// run_trials / summary
// ---------------------------------------------------------------------------
double lower_median(std::vector<double> v) {
    if (v.empty()) return std::numeric_limits<double>::quiet_NaN();
    std::sort(v.begin(), v.end());
    return v[(v.size() - 1) / 2];  // odd: middle; even: lower-middle
}

namespace {

TrialRecord record_of(uint64_t seed, const PlanResult& r) {
    TrialRecord t;
    t.seed = seed;
    t.success = std::isfinite(r.best.cost);
    if (r.stats.first_solution)
        t.first_solution = std::make_pair(r.stats.first_solution->first * 1e3, r.stats.first_solution->second);
    if (t.success) t.final_solution = std::make_pair(r.best.found_at * 1e3, r.best.cost);
    for (const auto& [s, c] : r.stats.cost_timeline) t.cost_timeline.emplace_back(s * 1e3, c);
    t.iterations = r.stats.iterations;
    t.propagations = r.stats.propagations_attempted;
    t.first_iteration = r.stats.first_solution ? r.stats.first_solution_iteration : 0;
    return t;
}

}  // namespace

std::vector<TrialRecord> run_trials(const Scenario& s) {
    std::vector<TrialRecord> out(static_cast<size_t>(s.n_trials));
    if (s.n_trials == 0) return out;
    // Each worker owns one planner instance (its own stream and device
    // buffers) and takes trial indices from a shared counter; runs share
    // nothing, so a record does not depend on which worker ran it.
    const int workers = std::max(1, std::min(s.workers, s.n_trials));
    std::atomic<int> next{0};
    std::vector<std::exception_ptr> errs(static_cast<size_t>(workers));
    auto work = [&](int w) {
        try {
            Planner p(s.problem, s.config);
            for (int k = next++; k < s.n_trials; k = next++) {
                const uint64_t seed = s.base_seed + static_cast<uint64_t>(k);
                p.reset(seed);
                PlanResult r = p.solve(s.config.t_max > 0 ? s.config.t_max : -1, s.config.max_iterations, false);
                out[static_cast<size_t>(k)] = record_of(seed, r);
            }
        } catch (...) {
            errs[static_cast<size_t>(w)] = std::current_exception();
            next = s.n_trials;
        }
    };
    if (workers == 1) {
        work(0);
    } else {
        std::vector<std::thread> th;
        for (int w = 0; w < workers; ++w) th.emplace_back(work, w);
        for (auto& t : th) t.join();
    }
    for (auto& e : errs)
        if (e) std::rethrow_exception(e);
    return out;
}

SummaryRow summarize(const std::string& name, const std::vector<TrialRecord>& records,
                     std::optional<double> normalization) {
    SummaryRow r;
    r.scenario = name;
    r.normalization = normalization;
    std::vector<double> fm, fc, lm, lc;
    size_t ok = 0;
    for (const auto& t : records) {
        if (!t.success) continue;  // medians over successful trials only
        ++ok;
        if (t.first_solution) { fm.push_back(t.first_solution->first); fc.push_back(t.first_solution->second); }
        lm.push_back(t.final_solution->first);
        lc.push_back(t.final_solution->second);
    }
    r.first_ms = lower_median(fm);
    r.first_cost = lower_median(fc);
    r.final_ms = lower_median(lm);
    r.final_cost = lower_median(lc);
    r.success_rate = records.empty() ? std::numeric_limits<double>::quiet_NaN()
                                     : 100.0 * static_cast<double>(ok) / static_cast<double>(records.size());
    return r;
}

// ---------------------------------------------------------------------------
// Emitters
// ---------------------------------------------------------------------------
void emit_csv(const std::vector<TrialRecord>& records, const SummaryRow& summary, const std::string& path) {
    {
        std::ofstream f = open_out(path);
        f << "seed,success,first_ms,first_cost,final_ms,final_cost,first_iteration,iterations\n";
        const double nan = std::numeric_limits<double>::quiet_NaN();
        for (const auto& t : records) {
            f << t.seed << ',' << (t.success ? 1 : 0) << ','
              << fmt(t.first_solution ? t.first_solution->first : nan) << ','
              << fmt(t.first_solution ? t.first_solution->second : nan) << ','
              << fmt(t.final_solution ? t.final_solution->first : nan) << ','
              << fmt(t.final_solution ? t.final_solution->second : nan) << ',' << t.first_iteration << ','
              << t.iterations << '\n';
        }
        close_out(f, path);
    }
    const std::string spath = path + ".summary.csv";
    std::ofstream f = open_out(spath);
    f << "scenario,trials,success_rate,first_ms,first_cost,final_ms,final_cost,normalization,first_cost_norm,"
         "final_cost_norm\n";
    const double nz = summary.normalization.value_or(std::numeric_limits<double>::quiet_NaN());
    f << summary.scenario << ',' << records.size() << ',' << fmt(summary.success_rate) << ','
      << fmt(summary.first_ms) << ',' << fmt(summary.first_cost) << ',' << fmt(summary.final_ms) << ','
      << fmt(summary.final_cost) << ',' << fmt(nz) << ','
      << fmt(summary.normalization ? summary.first_cost / nz : summary.first_cost) << ','
      << fmt(summary.normalization ? summary.final_cost / nz : summary.final_cost) << '\n';
    close_out(f, spath);
}

void emit_cost_curve(const std::vector<TrialRecord>& records, const std::string& path) {
    constexpr double W = 800, H = 500, L = 80, R = 30, T = 40, B = 60;
    std::vector<const TrialRecord*> tr;
    double tmin = std::numeric_limits<double>::infinity(), tmax = 0;
    double cmin = std::numeric_limits<double>::infinity(), cmax = -cmin;
    for (const auto& t : records) {
        if (t.cost_timeline.empty()) continue;
        tr.push_back(&t);
        for (const auto& [ms, c] : t.cost_timeline) {
            tmin = std::min(tmin, ms);
            tmax = std::max(tmax, ms);
            cmin = std::min(cmin, c);
            cmax = std::max(cmax, c);
        }
    }
    std::ofstream f = open_out(path);
    auto num = [](double v) {
        char b[32];
        std::snprintf(b, sizeof b, "%.6g", v);
        return std::string(b);
    };
    f << "<svg xmlns=\"http://www.w3.org/2000/svg\" width=\"" << W << "\" height=\"" << H << "\" viewBox=\"0 0 "
      << W << ' ' << H << "\" font-family=\"sans-serif\" font-size=\"12\">\n";
    f << "<rect x=\"0\" y=\"0\" width=\"" << W << "\" height=\"" << H << "\" fill=\"white\"/>\n";
    f << "<line x1=\"" << L << "\" y1=\"" << H - B << "\" x2=\"" << W - R << "\" y2=\"" << H - B
      << "\" stroke=\"black\"/>\n";
    f << "<line x1=\"" << L << "\" y1=\"" << T << "\" x2=\"" << L << "\" y2=\"" << H - B << "\" stroke=\"black\"/>\n";
    f << "<text x=\"" << (L + W - R) / 2 << "\" y=\"" << H - 15
      << "\" text-anchor=\"middle\">elapsed time (ms, log scale)</text>\n";
    f << "<text x=\"20\" y=\"" << (T + H - B) / 2 << "\" text-anchor=\"middle\" transform=\"rotate(-90 20 "
      << (T + H - B) / 2 << ")\">best solution cost</text>\n";
    if (tr.empty()) {
        f << "<text class=\"empty\" x=\"" << (L + W - R) / 2 << "\" y=\"" << (T + H - B) / 2
          << "\" text-anchor=\"middle\">no solution in any of " << records.size() << " trials</text>\n</svg>\n";
        close_out(f, path);
        return;
    }
    // Time axis: log10 over [tmin/2, tend], tend extends every step curve to
    // the latest recorded improvement (×1.5 so the last step is visible).
    const double t0 = std::max(tmin * 0.5, 1e-6), t1 = std::max(tmax * 1.5, t0 * 10);
    const double lg0 = std::log10(t0), lg1 = std::log10(t1);
    if (!(cmax > cmin)) { cmax = cmin + 0.5; cmin -= 0.5; }
    const double pad = 0.05 * (cmax - cmin);
    const double c0 = cmin - pad, c1 = cmax + pad;
    auto X = [&](double ms) { return L + (std::log10(std::max(ms, t0)) - lg0) / (lg1 - lg0) * (W - L - R); };
    auto Y = [&](double c) { return H - B - (c - c0) / (c1 - c0) * (H - B - T); };
    for (int d = static_cast<int>(std::ceil(lg0)); d <= static_cast<int>(std::floor(lg1)); ++d) {
        const double x = X(std::pow(10.0, d));
        f << "<line x1=\"" << num(x) << "\" y1=\"" << H - B << "\" x2=\"" << num(x) << "\" y2=\"" << H - B + 5
          << "\" stroke=\"black\"/><text x=\"" << num(x) << "\" y=\"" << H - B + 18
          << "\" text-anchor=\"middle\">" << num(std::pow(10.0, d)) << "</text>\n";
    }
    for (int k = 0; k <= 4; ++k) {
        const double c = c0 + (c1 - c0) * k / 4;
        f << "<text x=\"" << L - 6 << "\" y=\"" << num(Y(c) + 4) << "\" text-anchor=\"end\">" << num(c)
          << "</text>\n";
    }
    // Per-trial step curves: horizontal at each cost until the next improvement.
    for (const TrialRecord* t : tr) {
        f << "<polyline class=\"trial\" data-seed=\"" << t->seed
          << "\" fill=\"none\" stroke=\"#7aa6d8\" stroke-opacity=\"0.5\" points=\"";
        const auto& tl = t->cost_timeline;
        for (size_t i = 0; i < tl.size(); ++i) {
            const double tn = i + 1 < tl.size() ? tl[i + 1].first : t1;
            f << num(X(tl[i].first)) << ',' << num(Y(tl[i].second)) << ' ' << num(X(tn)) << ','
              << num(Y(tl[i].second)) << (i + 1 < tl.size() ? " " : "");
        }
        f << "\"/>\n";
    }
    // Median curve over the union of improvement times: at each time, the
    // lower-middle median of the current best over trials that have one.
    std::vector<double> times;
    for (const TrialRecord* t : tr)
        for (const auto& e : t->cost_timeline) times.push_back(e.first);
    std::sort(times.begin(), times.end());
    times.erase(std::unique(times.begin(), times.end()), times.end());
    f << "<polyline class=\"median\" fill=\"none\" stroke=\"#c0392b\" stroke-width=\"2\" points=\"";
    for (size_t i = 0; i < times.size(); ++i) {
        std::vector<double> cur;
        for (const TrialRecord* t : tr) {
            double best = std::numeric_limits<double>::infinity();
            for (const auto& e : t->cost_timeline)
                if (e.first <= times[i]) best = e.second;
            if (std::isfinite(best)) cur.push_back(best);
        }
        const double m = lower_median(cur);
        const double tn = i + 1 < times.size() ? times[i + 1] : t1;
        f << num(X(times[i])) << ',' << num(Y(m)) << ' ' << num(X(tn)) << ',' << num(Y(m))
          << (i + 1 < times.size() ? " " : "");
    }
    f << "\"/>\n";
    f << "<text x=\"" << W - R << "\" y=\"" << T - 12 << "\" text-anchor=\"end\">" << tr.size() << " of "
      << records.size() << " trials solved; red: median</text>\n</svg>\n";
    close_out(f, path);
}

void emit_records(const std::vector<TrialRecord>& records, const std::string& scenario, const std::string& path) {
    std::ofstream f = open_out(path);
    auto jnum = [](double v) { return std::isfinite(v) ? fmt(v) : (std::isnan(v) ? "NaN" : (v > 0 ? "Infinity" : "-Infinity")); };
    auto pair = [&](const std::optional<std::pair<double, double>>& p) {
        return p ? "[" + jnum(p->first) + ", " + jnum(p->second) + "]" : std::string("null");
    };
    f << "{\"scenario\": \"" << scenario << "\", \"trials\": [";
    for (size_t i = 0; i < records.size(); ++i) {
        const TrialRecord& t = records[i];
        f << (i ? ",\n " : "\n ") << "{\"seed\": " << t.seed << ", \"success\": " << (t.success ? "true" : "false")
          << ", \"first_solution\": " << pair(t.first_solution) << ", \"final_solution\": " << pair(t.final_solution)
          << ", \"iterations\": " << t.iterations << ", \"propagations\": " << t.propagations
          << ", \"first_iteration\": " << t.first_iteration << ", \"cost_timeline\": [";
        for (size_t k = 0; k < t.cost_timeline.size(); ++k)
            f << (k ? ", " : "") << '[' << jnum(t.cost_timeline[k].first) << ", " << jnum(t.cost_timeline[k].second)
              << ']';
        f << "]}";
    }
    f << "\n]}\n";
    close_out(f, path);
}

std::vector<TrialRecord> load_records(const std::string& path, std::string* scenario) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw SchemaError(path + ": " + std::strerror(errno));
    std::stringstream ss;
    ss << in.rdbuf();
    Json root = Reader(ss.str()).parse();
    Field r{&root, "records"};
    if (scenario) *scenario = r.opt("scenario") ? r.at("scenario").string() : std::string();
    Field trials = r.at("trials");
    std::vector<TrialRecord> out;
    auto pair = [](const Field& f) -> std::optional<std::pair<double, double>> {
        if (f.j->t == Json::T::Null) return std::nullopt;
        if (f.size() != 2) f.bad("expected [ms, cost]");
        return std::make_pair(f.idx(0).num(), f.idx(1).num());
    };
    for (size_t i = 0; i < trials.size(); ++i) {
        Field t = trials.idx(i);
        TrialRecord x;
        x.seed = t.at("seed").u64();
        x.success = t.at("success").boolean();
        x.first_solution = pair(t.at("first_solution"));
        x.final_solution = pair(t.at("final_solution"));
        if (x.success != static_cast<bool>(x.final_solution))
            t.bad("success must hold exactly when final_solution is present (SPEC.md:473)");
        if (auto v = t.opt("iterations")) x.iterations = v->u64();
        if (auto v = t.opt("propagations")) x.propagations = v->u64();
        if (auto v = t.opt("first_iteration")) x.first_iteration = v->u64();
        if (auto tl = t.opt("cost_timeline"))
            for (size_t k = 0; k < tl->size(); ++k) {
                auto e = pair(tl->idx(k));
                if (!e) tl->idx(k).bad("expected [ms, cost]");
                x.cost_timeline.push_back(*e);
            }
        out.push_back(std::move(x));
    }
    return out;
}

void emit_trajectory(const Trajectory& t, const std::string& path) {
    std::ofstream f = open_out(path);
    const size_t n = t.states.empty() ? 0 : t.states[0].size();
    const size_t m = t.controls.empty() ? 0 : t.controls[0].size();
    f << "node";
    for (size_t i = 0; i < n; ++i) f << ",x" << i;
    for (size_t i = 0; i < m; ++i) f << ",u" << i;
    f << ",duration,segment_cost\n";
    for (size_t k = 0; k < t.states.size(); ++k) {
        f << k;
        for (double v : t.states[k]) f << ',' << fmt(v);
        for (double v : t.controls[k]) f << ',' << fmt(v);
        f << ',' << fmt(t.durations[k]) << ',' << fmt(k == 0 || k - 1 >= t.segment_costs.size() ? 0.0 : t.segment_costs[k - 1])
          << '\n';
    }
    close_out(f, path);
}

}  // namespace kinoplan
