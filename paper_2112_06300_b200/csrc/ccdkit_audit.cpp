// Benchmark / audit layer of the drop-in (include/ccdkit/bench.hpp and the
// OBJ ingestion of scene.hpp), over the device pipeline.
//
// This is the reference's consumer of the CCD path (proj/src/bench.cpp,
// proj/src/scene.cpp:82-216, proj/tools/ccdbench.cpp) rebuilt for the B200
// library: every ccd() / stq() / narrow_phase() it drives is the device path
// of libccdkit.so, and the timing columns are the device stage times the
// step reports (CB / BP / SO/CD / NP, cudaEvent-timed).  Semantics follow
// the reference:
//   bench_scene     bench.cpp:39-106  — per method: full step (zero-ToI retry
//                   when cfg.narrow.no_zero_toi), median stage times over
//                   timing_reps, truncate_candidates fault injection, FP/FN
//                   by sorted set intersection with the oracle's colliding and
//                   indeterminate sets
//   run_benchmark   bench.cpp:108-138 — load failures are collected, rows
//                   sorted by (scene, frame, method), optional report file
//   emit_report / parse_report_json   bench.cpp:140-234 (CSV RFC 4180 + CRLF,
//                   %.17g numbers, "inf" for no collision; JSON array with
//                   null toi for no collision)
//   scaling_probe / loglog_slope / thread_scaling   bench.cpp:236-343
//   make_cloth_scene / make_box_soup  bench.cpp:346-446 (same draws, same order)
//   load_obj_pair / load_manifest     scene.cpp:82-216
// Ground truth is the reference's exact oracle (ground_truth_pairs,
// proj/src/oracle.cpp — GMP rationals, not part of this library), bound
// weakly: link it to use audit mode, otherwise oracle_enabled throws
// ConfigError.  JSON is read and written by the small codec below (the
// reference uses nlohmann::json; the output layout matches its dump(2):
// keys in lexicographic order, two-space indent).
#include "ccdkit/bench.hpp"
#include "ccdkit/rng.hpp"

#include <algorithm>
#include <charconv>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <map>
#include <ostream>
#include <sstream>
#include <variant>

#define CCDKIT_EXPORT __attribute__((visibility("default")))

namespace ccdkit {

// resolved only when an oracle implementation is linked into the process
GroundTruth ground_truth_pairs(const SceneStep& scene, const OracleOptions& opts, unsigned threads)
    __attribute__((weak));

namespace {

using Clock = std::chrono::steady_clock;

double median_of(std::vector<double> v)
{
    if (v.empty())
        return 0.0;
    std::sort(v.begin(), v.end());
    return v[v.size() / 2];
}

double stage_time(const CcdReport& r, const char* key)
{
    const auto it = r.per_stage_times.find(key);
    return it == r.per_stage_times.end() ? 0.0 : it->second;
}

CcdReport step(const SceneStep& scene, const PipelineConfig& cfg)
{
    return cfg.narrow.no_zero_toi ? ccd_no_zero_toi(scene, cfg) : ccd(scene, cfg);
}

void derive_edges(SceneStep& s, const std::vector<std::array<std::uint32_t, 2>>& extra = {})
{
    std::vector<std::array<std::uint32_t, 2>> e;
    e.reserve(3 * s.faces.size() + extra.size());
    const auto put = [&e](std::uint32_t a, std::uint32_t b) {
        if (a != b)
            e.push_back({ std::min(a, b), std::max(a, b) });
    };
    for (const auto& f : s.faces)
        for (int k = 0; k < 3; ++k)
            put(f[k], f[(k + 1) % 3]);
    for (const auto& l : extra)
        put(l[0], l[1]);
    std::sort(e.begin(), e.end());
    e.erase(std::unique(e.begin(), e.end()), e.end());
    s.edges = std::move(e);
}

// ------------------------------------------------------------------ JSON
// Just enough JSON for reports and manifests: null, bool, number, string,
// array, object.  Numbers keep their source text so integers and doubles
// convert exactly (std::from_chars).
struct Json {
    enum Kind { Null, Bool, Number, String, Array, Object } kind = Null;
    bool b = false;
    std::string text; // number text or string value
    std::vector<Json> items;
    std::vector<std::pair<std::string, Json>> fields;

    const Json* find(const std::string& k) const
    {
        for (const auto& f : fields)
            if (f.first == k)
                return &f.second;
        return nullptr;
    }
    const Json& at(const std::string& k) const
    {
        const Json* j = find(k);
        if (!j)
            throw InvalidInput("report JSON: missing key \"" + k + "\"");
        return *j;
    }
    double as_double() const
    {
        if (kind != Number)
            throw InvalidInput("report JSON: expected a number");
        double v = 0.0;
        const auto r = std::from_chars(text.data(), text.data() + text.size(), v);
        if (r.ec != std::errc())
            throw InvalidInput("report JSON: bad number " + text);
        return v;
    }
    std::size_t as_size() const
    {
        if (kind != Number)
            throw InvalidInput("report JSON: expected an integer");
        std::size_t v = 0;
        const auto r = std::from_chars(text.data(), text.data() + text.size(), v);
        if (r.ec != std::errc() || r.ptr != text.data() + text.size())
            throw InvalidInput("report JSON: bad integer " + text);
        return v;
    }
    const std::string& as_string() const
    {
        if (kind != String)
            throw InvalidInput("report JSON: expected a string");
        return text;
    }
};

class JsonReader {
public:
    explicit JsonReader(const std::string& s) : s_(s) {}

    Json document()
    {
        Json v = value();
        ws();
        if (i_ != s_.size())
            fail("trailing characters");
        return v;
    }

private:
    [[noreturn]] void fail(const char* what) const
    {
        throw InvalidInput(std::string("JSON parse error at offset ") + std::to_string(i_) + ": " + what);
    }
    void ws()
    {
        while (i_ < s_.size() && (s_[i_] == ' ' || s_[i_] == '\t' || s_[i_] == '\n' || s_[i_] == '\r'))
            ++i_;
    }
    bool lit(const char* w)
    {
        const std::size_t n = std::char_traits<char>::length(w);
        if (s_.compare(i_, n, w) != 0)
            return false;
        i_ += n;
        return true;
    }
    static void put_utf8(std::string& out, unsigned cp)
    {
        if (cp < 0x80) {
            out += char(cp);
        } else if (cp < 0x800) {
            out += char(0xC0 | (cp >> 6));
            out += char(0x80 | (cp & 0x3F));
        } else if (cp < 0x10000) {
            out += char(0xE0 | (cp >> 12));
            out += char(0x80 | ((cp >> 6) & 0x3F));
            out += char(0x80 | (cp & 0x3F));
        } else {
            out += char(0xF0 | (cp >> 18));
            out += char(0x80 | ((cp >> 12) & 0x3F));
            out += char(0x80 | ((cp >> 6) & 0x3F));
            out += char(0x80 | (cp & 0x3F));
        }
    }
    unsigned hex4()
    {
        if (i_ + 4 > s_.size())
            fail("short \\u escape");
        unsigned v = 0;
        for (int k = 0; k < 4; ++k) {
            const char c = s_[i_++];
            v <<= 4;
            if (c >= '0' && c <= '9')
                v |= unsigned(c - '0');
            else if (c >= 'a' && c <= 'f')
                v |= unsigned(c - 'a' + 10);
            else if (c >= 'A' && c <= 'F')
                v |= unsigned(c - 'A' + 10);
            else
                fail("bad \\u escape");
        }
        return v;
    }
    std::string string()
    {
        if (s_[i_] != '"')
            fail("expected a string");
        ++i_;
        std::string out;
        while (true) {
            if (i_ >= s_.size())
                fail("unterminated string");
            const char c = s_[i_++];
            if (c == '"')
                return out;
            if (c != '\\') {
                out += c;
                continue;
            }
            if (i_ >= s_.size())
                fail("unterminated escape");
            const char e = s_[i_++];
            switch (e) {
            case '"': out += '"'; break;
            case '\\': out += '\\'; break;
            case '/': out += '/'; break;
            case 'b': out += '\b'; break;
            case 'f': out += '\f'; break;
            case 'n': out += '\n'; break;
            case 'r': out += '\r'; break;
            case 't': out += '\t'; break;
            case 'u': {
                unsigned cp = hex4();
                if (cp >= 0xD800 && cp < 0xDC00 && lit("\\u")) {
                    const unsigned lo = hex4();
                    cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
                }
                put_utf8(out, cp);
                break;
            }
            default:
                fail("bad escape");
            }
        }
    }
    Json value()
    {
        ws();
        if (i_ >= s_.size())
            fail("unexpected end");
        Json v;
        const char c = s_[i_];
        if (c == '{') {
            v.kind = Json::Object;
            ++i_;
            ws();
            if (i_ < s_.size() && s_[i_] == '}') {
                ++i_;
                return v;
            }
            while (true) {
                ws();
                std::string k = string();
                ws();
                if (i_ >= s_.size() || s_[i_++] != ':')
                    fail("expected ':'");
                v.fields.emplace_back(std::move(k), value());
                ws();
                if (i_ < s_.size() && s_[i_] == ',') {
                    ++i_;
                    continue;
                }
                if (i_ < s_.size() && s_[i_] == '}') {
                    ++i_;
                    return v;
                }
                fail("expected ',' or '}'");
            }
        }
        if (c == '[') {
            v.kind = Json::Array;
            ++i_;
            ws();
            if (i_ < s_.size() && s_[i_] == ']') {
                ++i_;
                return v;
            }
            while (true) {
                v.items.push_back(value());
                ws();
                if (i_ < s_.size() && s_[i_] == ',') {
                    ++i_;
                    continue;
                }
                if (i_ < s_.size() && s_[i_] == ']') {
                    ++i_;
                    return v;
                }
                fail("expected ',' or ']'");
            }
        }
        if (c == '"') {
            v.kind = Json::String;
            v.text = string();
            return v;
        }
        if (lit("null"))
            return v;
        if (lit("true")) {
            v.kind = Json::Bool;
            v.b = true;
            return v;
        }
        if (lit("false")) {
            v.kind = Json::Bool;
            return v;
        }
        const std::size_t b = i_;
        while (i_ < s_.size() && (std::isdigit(static_cast<unsigned char>(s_[i_])) || s_[i_] == '-'
                                  || s_[i_] == '+' || s_[i_] == '.' || s_[i_] == 'e' || s_[i_] == 'E'))
            ++i_;
        if (b == i_)
            fail("unexpected character");
        v.kind = Json::Number;
        v.text = s_.substr(b, i_ - b);
        return v;
    }

    const std::string& s_;
    std::size_t i_ = 0;
};

std::string json_string(const std::string& s)
{
    std::string o = "\"";
    for (const char ch : s) {
        const unsigned char c = static_cast<unsigned char>(ch);
        switch (c) {
        case '"': o += "\\\""; break;
        case '\\': o += "\\\\"; break;
        case '\b': o += "\\b"; break;
        case '\f': o += "\\f"; break;
        case '\n': o += "\\n"; break;
        case '\r': o += "\\r"; break;
        case '\t': o += "\\t"; break;
        default:
            if (c < 0x20) {
                char buf[8];
                std::snprintf(buf, sizeof buf, "\\u%04x", c);
                o += buf;
            } else {
                o += ch;
            }
        }
    }
    return o + "\"";
}

// shortest round-trip text; integral values keep a ".0" like nlohmann's dump
std::string json_double(double v)
{
    char buf[64];
    const auto r = std::to_chars(buf, buf + sizeof buf, v);
    std::string s(buf, r.ptr);
    if (s.find_first_of(".eEn") == std::string::npos)
        s += ".0";
    return s;
}

std::string csv_field(const std::string& f)
{
    if (f.find_first_of(",\"\r\n") == std::string::npos)
        return f;
    std::string q = "\"";
    for (const char c : f) {
        q += c;
        if (c == '"')
            q += '"';
    }
    return q + "\"";
}

std::string g17(double v)
{
    std::ostringstream o;
    o.precision(17);
    o << v;
    return o.str();
}

// ------------------------------------------------------------------- OBJ
struct ObjFile {
    std::vector<Vec3> v;
    std::vector<std::array<std::uint32_t, 3>> tri;
    std::vector<std::array<std::uint32_t, 2>> seg;
};

std::uint32_t obj_index(const std::string& tok, std::size_t nv, const std::string& path)
{
    const std::string lead = tok.substr(0, tok.find('/')); // v/vt/vn: vertex index first
    long long k = 0;
    const char* b = lead.data();
    const char* e = b + lead.size();
    const auto r = std::from_chars(b, e, k);
    if (r.ec != std::errc() || r.ptr != e)
        throw InvalidInput(path + ": bad index token '" + tok + "'");
    if (k < 0)
        k += static_cast<long long>(nv) + 1; // relative to the end
    if (k < 1 || static_cast<std::size_t>(k) > nv)
        throw InvalidInput(path + ": face index out of range: " + tok);
    return static_cast<std::uint32_t>(k - 1);
}

ObjFile read_obj(const std::string& path)
{
    std::ifstream in(path);
    if (!in)
        throw InvalidInput("cannot open " + path);
    ObjFile o;
    std::string line;
    while (std::getline(in, line)) {
        if (!line.empty() && line.back() == '\r')
            line.pop_back();
        std::istringstream ls(line);
        std::string tag;
        if (!(ls >> tag) || tag[0] == '#')
            continue;
        if (tag == "v") {
            Vec3 p;
            if (!(ls >> p[0] >> p[1] >> p[2]))
                throw InvalidInput(path + ": malformed vertex line: " + line);
            o.v.push_back(p);
        } else if (tag == "f" || tag == "l") {
            std::vector<std::uint32_t> idx;
            for (std::string tok; ls >> tok;)
                idx.push_back(obj_index(tok, o.v.size(), path));
            if (tag == "f") {
                if (idx.size() < 3)
                    throw InvalidInput(path + ": face with fewer than 3 vertices");
                for (std::size_t k = 1; k + 1 < idx.size(); ++k) // fan
                    o.tri.push_back({ idx[0], idx[k], idx[k + 1] });
            } else {
                for (std::size_t k = 0; k + 1 < idx.size(); ++k)
                    o.seg.push_back({ idx[k], idx[k + 1] });
            }
        }
    }
    return o;
}

} // namespace

// ================================================================ scene I/O

CCDKIT_EXPORT SceneStep load_obj_pair(const std::string& path_t0, const std::string& path_t1)
{
    ObjFile a = read_obj(path_t0);
    ObjFile b = read_obj(path_t1);
    if (a.v.size() != b.v.size())
        throw InvalidInput(path_t0 + " / " + path_t1 + ": vertex counts differ");
    if (a.tri != b.tri || a.seg != b.seg)
        throw InvalidInput(path_t0 + " / " + path_t1 + ": connectivity differs");
    SceneStep s;
    s.vertices_t0 = std::move(a.v);
    s.vertices_t1 = std::move(b.v);
    s.faces = std::move(a.tri);
    derive_edges(s, a.seg);
    s.validate();
    return s;
}

CCDKIT_EXPORT std::vector<std::pair<std::string, std::string>> load_manifest(const std::string& manifest_path)
{
    std::ifstream in(manifest_path, std::ios::binary);
    if (!in)
        throw InvalidInput("cannot open " + manifest_path);
    std::stringstream buf;
    buf << in.rdbuf();
    const std::string text = buf.str();
    Json doc;
    try {
        doc = JsonReader(text).document();
    } catch (const InvalidInput& e) {
        throw InvalidInput(manifest_path + ": " + e.what());
    }
    if (doc.kind != Json::Array)
        throw InvalidInput(manifest_path + ": manifest must be a JSON array");
    const std::filesystem::path dir = std::filesystem::path(manifest_path).parent_path();
    const auto resolve = [&dir](const std::string& p) {
        const std::filesystem::path fp(p);
        return fp.is_absolute() ? fp.string() : (dir / fp).string();
    };
    std::vector<std::pair<std::string, std::string>> out;
    for (const Json& e : doc.items) {
        const Json* t0 = e.kind == Json::Object ? e.find("t0") : nullptr;
        const Json* t1 = e.kind == Json::Object ? e.find("t1") : nullptr;
        if (!t0 || !t1 || t0->kind != Json::String || t1->kind != Json::String)
            throw InvalidInput(manifest_path + ": entries need \"t0\" and \"t1\"");
        out.emplace_back(resolve(t0->text), resolve(t1->text));
    }
    return out;
}

// ================================================================ benchmark

CCDKIT_EXPORT void bench_scene(const std::string& scene_id, std::size_t frame, const SceneStep& scene,
                               const RunSpec& spec, BenchResult& out)
{
    std::vector<CandidatePair> truth_hit, truth_unknown;
    if (spec.oracle_enabled) {
        if (!ground_truth_pairs)
            throw ConfigError("bench_scene: audit mode needs the exact oracle (ground_truth_pairs, "
                              "proj/src/oracle.cpp) linked into the process");
        const GroundTruth gt = ground_truth_pairs(scene, spec.oracle, spec.pipeline.threads);
        truth_hit.reserve(gt.colliding.size());
        for (const GroundTruthPair& p : gt.colliding)
            truth_hit.push_back(p.pair);
        truth_unknown = gt.indeterminate;
        out.indeterminate += truth_unknown.size();
    }

    for (const BroadMethod m : spec.methods) {
        PipelineConfig cfg = spec.pipeline;
        cfg.broad_method = m;
        CcdReport rep = step(scene, cfg);
        std::vector<double> tb { stage_time(rep, "CB") }, tp { stage_time(rep, "BP") },
            tc { stage_time(rep, "SO/CD") }, tn { stage_time(rep, "NP") };
        if (!spec.no_timing)
            for (unsigned r = 1; r < spec.timing_reps; ++r) {
                const CcdReport again = step(scene, cfg);
                tb.push_back(stage_time(again, "CB"));
                tp.push_back(stage_time(again, "BP"));
                tc.push_back(stage_time(again, "SO/CD"));
                tn.push_back(stage_time(again, "NP"));
            }

        std::vector<CandidatePair> cand = std::move(rep.candidates);
        if (cand.size() > spec.truncate_candidates)
            cand.resize(spec.truncate_candidates); // audit fault injection

        MetricsRow row;
        row.scene = scene_id;
        row.frame = frame;
        row.method = to_string(m);
        row.candidates = cand.size();
        if (spec.oracle_enabled) {
            // all three lists are canonically sorted and duplicate-free
            std::vector<CandidatePair> hit, unknown;
            std::set_intersection(cand.begin(), cand.end(), truth_hit.begin(), truth_hit.end(),
                                  std::back_inserter(hit));
            std::set_intersection(cand.begin(), cand.end(), truth_unknown.begin(), truth_unknown.end(),
                                  std::back_inserter(unknown));
            row.fp = cand.size() - hit.size() - unknown.size();
            row.fn = truth_hit.size() - hit.size();
            out.total_fn += row.fn;
        }
        if (!spec.no_timing) {
            row.t_boxes = median_of(tb);
            row.t_broad = median_of(tp);
            row.t_classify = median_of(tc);
            row.t_narrow = median_of(tn);
        }
        row.peak_bytes = rep.tracked_peak_bytes;
        row.toi = rep.toi.toi;
        out.rows.push_back(std::move(row));
    }
}

CCDKIT_EXPORT BenchResult run_benchmark(const RunSpec& spec)
{
    if (spec.frame_pairs.empty() || spec.methods.empty())
        throw ConfigError("run_benchmark: need at least one frame pair and one method");
    spec.pipeline.validate();
    BenchResult res;
    for (std::size_t f = 0; f < spec.frame_pairs.size(); ++f) {
        const std::string& t0 = spec.frame_pairs[f].first;
        const std::string& t1 = spec.frame_pairs[f].second;
        SceneStep s;
        try {
            s = load_obj_pair(t0, t1);
        } catch (const std::exception& e) {
            res.errors.push_back(t0 + ": " + e.what()); // reported; the run continues
            continue;
        }
        bench_scene(t0, f, s, spec, res);
    }
    std::sort(res.rows.begin(), res.rows.end(), [](const MetricsRow& a, const MetricsRow& b) {
        return std::tie(a.scene, a.frame, a.method) < std::tie(b.scene, b.frame, b.method);
    });
    if (!spec.output_path.empty()) {
        const bool json = spec.output_path.size() >= 5
            && spec.output_path.compare(spec.output_path.size() - 5, 5, ".json") == 0;
        emit_report(res.rows, spec.output_path, json ? ReportFormat::Json : ReportFormat::Csv);
    }
    return res;
}

// ================================================================== reports

CCDKIT_EXPORT void emit_report(const std::vector<MetricsRow>& rows, std::ostream& out, ReportFormat format)
{
    if (format == ReportFormat::Json) {
        if (rows.empty()) {
            out << "[]\n";
            return;
        }
        out << "[\n";
        for (std::size_t r = 0; r < rows.size(); ++r) {
            const MetricsRow& m = rows[r];
            // lexicographic key order, as an ordered JSON object dumps
            const std::pair<const char*, std::string> kv[] = {
                { "candidates", std::to_string(m.candidates) },
                { "fn", std::to_string(m.fn) },
                { "fp", std::to_string(m.fp) },
                { "frame", std::to_string(m.frame) },
                { "method", json_string(m.method) },
                { "peak_bytes", std::to_string(m.peak_bytes) },
                { "scene", json_string(m.scene) },
                { "t_boxes", json_double(m.t_boxes) },
                { "t_broad", json_double(m.t_broad) },
                { "t_classify", json_double(m.t_classify) },
                { "t_narrow", json_double(m.t_narrow) },
                { "toi", m.toi == kNoCollision ? std::string("null") : json_double(m.toi) },
            };
            out << "  {\n";
            for (std::size_t k = 0; k < std::size(kv); ++k)
                out << "    \"" << kv[k].first << "\": " << kv[k].second << (k + 1 < std::size(kv) ? ",\n" : "\n");
            out << (r + 1 < rows.size() ? "  },\n" : "  }\n");
        }
        out << "]\n";
        return;
    }
    out << "scene,frame,method,candidates,fp,fn,t_boxes,t_broad,t_classify,t_narrow,peak_bytes,toi\r\n";
    for (const MetricsRow& m : rows) {
        out << csv_field(m.scene) << ',' << m.frame << ',' << csv_field(m.method) << ',' << m.candidates << ','
            << m.fp << ',' << m.fn << ',' << g17(m.t_boxes) << ',' << g17(m.t_broad) << ','
            << g17(m.t_classify) << ',' << g17(m.t_narrow) << ',' << m.peak_bytes << ','
            << (m.toi == kNoCollision ? std::string("inf") : g17(m.toi)) << "\r\n";
    }
}

CCDKIT_EXPORT void emit_report(const std::vector<MetricsRow>& rows, const std::string& path, ReportFormat format)
{
    std::ofstream out(path, std::ios::binary);
    if (!out)
        throw InvalidInput("emit_report: cannot open " + path);
    emit_report(rows, out, format);
}

CCDKIT_EXPORT std::vector<MetricsRow> parse_report_json(const std::string& text)
{
    const Json doc = JsonReader(text).document();
    if (doc.kind != Json::Array)
        throw InvalidInput("report JSON: expected an array of rows");
    std::vector<MetricsRow> rows;
    rows.reserve(doc.items.size());
    for (const Json& j : doc.items) {
        MetricsRow m;
        m.scene = j.at("scene").as_string();
        m.frame = j.at("frame").as_size();
        m.method = j.at("method").as_string();
        m.candidates = j.at("candidates").as_size();
        m.fp = j.at("fp").as_size();
        m.fn = j.at("fn").as_size();
        m.t_boxes = j.at("t_boxes").as_double();
        m.t_broad = j.at("t_broad").as_double();
        m.t_classify = j.at("t_classify").as_double();
        m.t_narrow = j.at("t_narrow").as_double();
        m.peak_bytes = j.at("peak_bytes").as_size();
        const Json& t = j.at("toi");
        m.toi = t.kind == Json::Null ? kNoCollision : t.as_double();
        rows.push_back(std::move(m));
    }
    return rows;
}

// ================================================================== scaling

CCDKIT_EXPORT std::vector<ScalingRow> scaling_probe(const SceneStep& scene, const std::vector<double>& fractions,
                                                    const PipelineConfig& cfg, std::uint64_t seed, unsigned reps)
{
    for (const double f : fractions)
        if (!(f > 0.0 && f <= 1.0))
            throw ConfigError("scaling_probe: fractions must lie in (0, 1]");
    const std::vector<Aabb> boxes = build_boxes(scene, cfg.inflation, cfg.threads);
    std::vector<ScalingRow> rows;
    for (const double fraction : fractions) {
        // seeded partial Fisher-Yates: the same seed picks the same prefix
        Rng rng(seed);
        const std::size_t n = boxes.size();
        std::vector<std::size_t> perm(n);
        for (std::size_t i = 0; i < n; ++i)
            perm[i] = i;
        const std::size_t take = std::max<std::size_t>(1, static_cast<std::size_t>(fraction * static_cast<double>(n)));
        for (std::size_t i = 0; i < take; ++i)
            std::swap(perm[i], perm[i + rng.next_below(n - i)]);
        std::vector<Aabb> sample(take);
        for (std::size_t i = 0; i < take; ++i)
            sample[i] = boxes[perm[i]];

        std::vector<double> tb, tn;
        for (unsigned r = 0; r < std::max(1u, reps); ++r) {
            const auto a = Clock::now();
            const std::vector<CandidatePair> c = cfg.broad_method == BroadMethod::BF ? bf(sample, scene, cfg.threads)
                : cfg.broad_method == BroadMethod::SAP                              ? sap(sample, scene, cfg.threads)
                                                                                    : stq(sample, scene, cfg.threads);
            const auto b = Clock::now();
            ClassifiedQueries q = classify(c, scene);
            q.vertex_face.insert(q.vertex_face.end(), q.edge_edge.begin(), q.edge_edge.end());
            narrow_phase(q.vertex_face, cfg.narrow, cfg.threads);
            const auto e = Clock::now();
            tb.push_back(std::chrono::duration<double>(b - a).count());
            tn.push_back(std::chrono::duration<double>(e - b).count());
        }
        ScalingRow row;
        row.fraction = fraction;
        row.box_count = take;
        row.broad_time = median_of(tb);
        row.narrow_time = median_of(tn);
        rows.push_back(row);
    }
    return rows;
}

CCDKIT_EXPORT double loglog_slope(const std::vector<ScalingRow>& rows)
{
    // least squares of log(broad_time) against log(box_count)
    double n = 0, sx = 0, sy = 0, sxx = 0, sxy = 0;
    for (const ScalingRow& r : rows) {
        if (r.box_count == 0 || r.broad_time <= 0)
            continue;
        const double x = std::log(static_cast<double>(r.box_count)), y = std::log(r.broad_time);
        n += 1;
        sx += x;
        sy += y;
        sxx += x * x;
        sxy += x * y;
    }
    if (n < 2)
        return 0.0;
    const double d = n * sxx - sx * sx;
    return d == 0.0 ? 0.0 : (n * sxy - sx * sy) / d;
}

CCDKIT_EXPORT std::vector<ThreadScalingRow> thread_scaling(const SceneStep& scene, const std::vector<unsigned>& counts,
                                                           BroadMethod method, unsigned reps)
{
    // `threads` is advisory on the device path; rows still time each request
    const std::vector<Aabb> boxes = build_boxes(scene);
    std::vector<ThreadScalingRow> rows;
    for (const unsigned th : counts) {
        std::vector<double> t;
        for (unsigned r = 0; r < std::max(1u, reps); ++r) {
            const auto a = Clock::now();
            if (method == BroadMethod::BF)
                bf(boxes, scene, th);
            else if (method == BroadMethod::SAP)
                sap(boxes, scene, th);
            else
                stq(boxes, scene, th);
            t.push_back(std::chrono::duration<double>(Clock::now() - a).count());
        }
        rows.push_back({ th, median_of(t) });
    }
    return rows;
}

// =============================================================== generators

CCDKIT_EXPORT SceneStep make_cloth_scene(std::size_t nx, std::size_t ny, double jitter, double drop, std::uint64_t seed)
{
    if (nx < 2 || ny < 2)
        throw ConfigError("make_cloth_scene: grid must be at least 2x2");
    Rng rng(seed);
    const auto j = [&rng, jitter] { return rng.uniform(-jitter, jitter); };
    SceneStep s;
    s.vertices_t0.reserve(nx * ny + 4);
    s.vertices_t1.reserve(nx * ny + 4);
    for (std::size_t r = 0; r < ny; ++r)
        for (std::size_t c = 0; c < nx; ++c) {
            // draw order matters for byte-identical scenes: x, y, z of t0, then of t1
            Vec3 a;
            a[0] = static_cast<double>(c) + j();
            a[1] = drop + j() * 0.5;
            a[2] = static_cast<double>(r) + j();
            Vec3 b;
            b[0] = a[0] + j();
            b[1] = a[1] - drop + j() * 0.5;
            b[2] = a[2] + j();
            s.vertices_t0.push_back(a);
            s.vertices_t1.push_back(b);
        }
    const auto id = [nx](std::size_t c, std::size_t r) { return static_cast<std::uint32_t>(r * nx + c); };
    for (std::size_t r = 0; r + 1 < ny; ++r)
        for (std::size_t c = 0; c + 1 < nx; ++c) {
            s.faces.push_back({ id(c, r), id(c + 1, r), id(c, r + 1) });
            s.faces.push_back({ id(c + 1, r), id(c + 1, r + 1), id(c, r + 1) });
        }
    // static two-triangle floor halfway down the fall
    const double y = drop * 0.5, lo = -1.0 - jitter;
    const double hx = static_cast<double>(nx) + jitter, hz = static_cast<double>(ny) + jitter;
    const std::uint32_t f0 = static_cast<std::uint32_t>(s.vertices_t0.size());
    for (const Vec3& v : { Vec3 { lo, y, lo }, Vec3 { hx, y, lo }, Vec3 { hx, y, hz }, Vec3 { lo, y, hz } }) {
        s.vertices_t0.push_back(v);
        s.vertices_t1.push_back(v);
    }
    s.faces.push_back({ f0, f0 + 1, f0 + 2 });
    s.faces.push_back({ f0, f0 + 2, f0 + 3 });
    derive_edges(s);
    return s;
}

CCDKIT_EXPORT SceneStep make_box_soup(std::size_t count, double region, double size, double motion,
                                      std::uint64_t seed)
{
    // two triangles per cube side, corners indexed by bit0 = x, bit1 = y, bit2 = z
    static constexpr std::uint32_t kSides[6][4] = {
        { 0, 1, 3, 2 }, { 4, 6, 7, 5 }, { 0, 4, 5, 1 }, { 2, 3, 7, 6 }, { 0, 2, 6, 4 }, { 1, 5, 7, 3 },
    };
    Rng rng(seed);
    SceneStep s;
    const double jit = 0.05 * size; // keeps contacts generic
    for (std::size_t k = 0; k < count; ++k) {
        Vec3 ctr, half, mv;
        for (int c = 0; c < 3; ++c)
            ctr[c] = rng.uniform(0.0, region);
        for (int c = 0; c < 3; ++c)
            half[c] = rng.uniform(size * 0.25, size);
        for (int c = 0; c < 3; ++c)
            mv[c] = rng.uniform(-motion, motion);
        const std::uint32_t base = static_cast<std::uint32_t>(s.vertices_t0.size());
        for (int corner = 0; corner < 8; ++corner) {
            Vec3 p;
            for (int c = 0; c < 3; ++c)
                p[c] = ctr[c] + (((corner >> c) & 1) ? half[c] : -half[c]);
            Vec3 d0, d1;
            for (int c = 0; c < 3; ++c)
                d0[c] = rng.uniform(-jit, jit);
            for (int c = 0; c < 3; ++c)
                d1[c] = rng.uniform(-jit, jit);
            s.vertices_t0.push_back(p + d0);
            s.vertices_t1.push_back(p + mv + d1);
        }
        for (const auto& q : kSides) {
            s.faces.push_back({ base + q[0], base + q[1], base + q[2] });
            s.faces.push_back({ base + q[0], base + q[2], base + q[3] });
        }
    }
    derive_edges(s);
    return s;
}

} // namespace ccdkit
