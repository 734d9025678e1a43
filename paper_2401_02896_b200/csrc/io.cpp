// io.cpp -- the reference's particle / transfer-function readers and PPM
// writer (io.hpp:62-216), restated so a caller of the C ABI needs nothing
// from the reference to feed the renderer.  Same accepted
// syntax (std::stod numbers, comma cells trimmed of white space, SPRT binary
// sniffed by magic), same validation and the same exception classes.
#include <algorithm>
#include <cctype>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <cstdio>
#include <fstream>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

#include "host.hpp"

#if SPHRAY_HAVE_JSON
#include "json.hpp"
#endif

namespace sphray_b200 {
namespace {

std::string trim(std::string s) {  // io.hpp:38-43
    const auto notspace = [](unsigned char c) { return !std::isspace(c); };
    s.erase(s.begin(), std::find_if(s.begin(), s.end(), notspace));
    s.erase(std::find_if(s.rbegin(), s.rend(), notspace).base(), s.end());
    return s;
}

std::vector<std::string> split_row(const std::string& line) {  // io.hpp:45-51
    std::vector<std::string> out;
    std::stringstream ss(line);
    std::string cell;
    while (std::getline(ss, cell, ',')) out.push_back(trim(cell));
    return out;
}

double number(const std::string& s, const std::string& where) {  // io.hpp:53-61
    try {
        std::size_t pos = 0;
        const double v = std::stod(s, &pos);
        if (pos != s.size()) throw std::invalid_argument(s);
        return v;
    } catch (const std::exception&) {
        fail(SPHRAY_ERR_IO, where + ": not a number: '" + s + "'");
    }
}

void check_particle(const sphray_particle& p, const std::string& where) {  // io.hpp:63-68
    if (!(p.h > 0.0)) fail(SPHRAY_ERR_IO, where + ": smoothing radius must be positive");
    if (!(p.density > 0.0)) fail(SPHRAY_ERR_IO, where + ": density must be positive");
    for (double v : {p.x, p.y, p.z, p.mass, p.value})
        if (!std::isfinite(v)) fail(SPHRAY_ERR_IO, where + ": attribute not finite");
}

uint64_t le64(const unsigned char* b) {
    uint64_t v = 0;
    for (int i = 0; i < 8; ++i) v |= static_cast<uint64_t>(b[i]) << (8 * i);
    return v;
}

constexpr const char* kCsvHeader = "x,y,z,mass,density,h,value";  // io.hpp:72

}  // namespace

// read_particles_binary (io.hpp:118-138) straight into caller storage:
// `alloc(n)` returns room for n records (e.g. pinned host memory, so the
// upload is a true DMA), filled record by record from the file and validated
// in the reference's order (a bad record before the truncation point is
// reported first).  Returns the record count.
size_t read_sprt_into(const std::string& path, const std::function<sphray_particle*(size_t)>& alloc) {
    std::FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) fail(SPHRAY_ERR_IO, "cannot open particle file " + path);
    struct Closer {
        std::FILE* f;
        ~Closer() { std::fclose(f); }
    } closer{f};
    unsigned char head[12];
    const size_t got = std::fread(head, 1, 12, f);
    if (got < 4 || std::memcmp(head, "SPRT", 4) != 0) fail(SPHRAY_ERR_IO, path + ": bad magic");
    if (got < 12) fail(SPHRAY_ERR_IO, "truncated file");
    const uint64_t n = le64(head + 4);
    std::fseek(f, 0, SEEK_END);
    const long long size = std::ftell(f);
    std::fseek(f, 12, SEEK_SET);
    const uint64_t avail = size > 12 ? static_cast<uint64_t>(size - 12) / 56 : 0;
    const uint64_t take = std::min(n, avail);
    sphray_particle* out = alloc(static_cast<size_t>(take));
    static_assert(sizeof(sphray_particle) == 56, "SPRT record layout");
    // record fields are read with lut.hpp's detail::get_f64 (io.hpp declares
    // only get_u64), whose truncation message is "lut: truncated file"
    if (take && std::fread(out, 56, take, f) != take) fail(SPHRAY_ERR_IO, "lut: truncated file");
    for (uint64_t i = 0; i < take; ++i)  // little-endian host: the record bytes are the doubles
        check_particle(out[i], path + ": record " + std::to_string(i));
    if (take < n) fail(SPHRAY_ERR_IO, "lut: truncated file");
    return static_cast<size_t>(n);
}

bool is_sprt(const std::string& path) {
    std::ifstream f(path, std::ios::binary);
    if (!f) fail(SPHRAY_ERR_IO, "cannot open particle file " + path);
    char magic[4] = {};
    f.read(magic, 4);
    return f.gcount() == 4 && std::memcmp(magic, "SPRT", 4) == 0;
}

std::vector<sphray_particle> load_particles(const std::string& path) {
    std::vector<sphray_particle> out;
    if (is_sprt(path)) {
        read_sprt_into(path, [&](size_t n) {
            out.resize(n);
            return out.data();
        });
        return out;
    }
    std::ifstream f(path, std::ios::binary);
    if (!f) fail(SPHRAY_ERR_IO, "cannot open particle file " + path);
    // read_particles_csv, io.hpp:74-99
    std::string line;
    if (!std::getline(f, line)) fail(SPHRAY_ERR_IO, path + ": empty file");
    if (trim(line) != kCsvHeader)
        fail(SPHRAY_ERR_IO, path + ": first line must be '" + std::string(kCsvHeader) + "'");
    std::size_t lineno = 1;
    while (std::getline(f, line)) {
        ++lineno;
        if (trim(line).empty()) continue;
        const auto c = split_row(line);
        const std::string where = path + ":" + std::to_string(lineno);
        if (c.size() != 7) fail(SPHRAY_ERR_IO, where + ": expected 7 comma-separated values");
        sphray_particle p{number(c[0], where), number(c[1], where), number(c[2], where),
                          number(c[3], where), number(c[4], where), number(c[5], where),
                          number(c[6], where)};
        check_particle(p, where);
        out.push_back(p);
    }
    return out;
}

void save_particles(const sphray_particle* ps, size_t n, const std::string& path, bool binary) {
    std::ofstream f(path, std::ios::binary);
    if (!f) fail(SPHRAY_ERR_IO, "cannot open " + path + " for writing");
    if (binary) {  // write_particles_binary, io.hpp:109-116
        f.write("SPRT", 4);
        unsigned char b[8];
        for (int i = 0; i < 8; ++i) b[i] = static_cast<unsigned char>(static_cast<uint64_t>(n) >> (8 * i));
        f.write(reinterpret_cast<const char*>(b), 8);
        for (size_t k = 0; k < n; ++k) {
            const double v[7] = {ps[k].x, ps[k].y, ps[k].z, ps[k].mass, ps[k].density, ps[k].h, ps[k].value};
            for (double d : v) {
                uint64_t bits;
                std::memcpy(&bits, &d, 8);
                for (int i = 0; i < 8; ++i) b[i] = static_cast<unsigned char>(bits >> (8 * i));
                f.write(reinterpret_cast<const char*>(b), 8);
            }
        }
        if (!f) fail(SPHRAY_ERR_IO, "particle binary: write failure");
    } else {  // write_particles_csv, io.hpp:101-107
        f << kCsvHeader << "\n";
        f.precision(17);
        for (size_t k = 0; k < n; ++k) {
            const auto& p = ps[k];
            f << p.x << ',' << p.y << ',' << p.z << ',' << p.mass << ',' << p.density << ','
              << p.h << ',' << p.value << "\n";
        }
        if (!f) fail(SPHRAY_ERR_IO, "particle csv: write failure");
    }
}

std::vector<sphray_tf_point> load_transfer_function(const std::string& path) {
    std::ifstream f(path);
    if (!f) fail(SPHRAY_ERR_IO, "cannot open transfer function " + path);
    std::vector<sphray_tf_point> pts;  // read_transfer_function_csv, io.hpp:158-184
    std::string line;
    std::size_t lineno = 0;
    while (std::getline(f, line)) {
        ++lineno;
        const std::string t = trim(line);
        if (t.empty()) continue;
        if (lineno == 1 && !std::isdigit(static_cast<unsigned char>(t[0])) && t[0] != '-' &&
            t[0] != '+' && t[0] != '.')
            continue;  // header
        const auto c = split_row(t);
        const std::string where = path + ":" + std::to_string(lineno);
        if (c.size() != 5) fail(SPHRAY_ERR_IO, where + ": expected value,r,g,b,absorption");
        pts.push_back(sphray_tf_point{number(c[0], where), number(c[1], where), number(c[2], where),
                                      number(c[3], where), number(c[4], where)});
    }
    std::sort(pts.begin(), pts.end(),
              [](const sphray_tf_point& a, const sphray_tf_point& b) { return a.value < b.value; });
    validate_tf(pts.data(), pts.size());  // TransferFunction::validate, raycast.hpp:316-324
    return pts;
}

void save_ppm(const double* rgb, int W, int H, const std::string& path) {  // io.hpp:193-210
    if (W < 0 || H < 0) fail(SPHRAY_ERR_CONFIG, "ppm: negative size");
    std::ofstream f(path, std::ios::binary);
    if (!f) fail(SPHRAY_ERR_IO, "cannot open " + path + " for writing");
    f << "P6\n" << W << " " << H << "\n255\n";
    const size_t n = static_cast<size_t>(W) * H * 3;
    std::string bytes(n, '\0');
    for (size_t i = 0; i < n; ++i)
        bytes[i] = static_cast<char>(static_cast<int>(std::lround(255.0 * std::clamp(rgb[i], 0.0, 1.0))));
    f.write(bytes.data(), static_cast<std::streamsize>(n));
    if (!f) fail(SPHRAY_ERR_IO, "ppm: write failure");
}

// load_camera / camera_from_json (io.hpp:263-304): defaults of sphray::Camera
// (raycast.hpp:45-57), then Camera::validate.
sphray_camera load_camera(const std::string& path) {
#if SPHRAY_HAVE_JSON
    std::ifstream f(path);
    if (!f) fail(SPHRAY_ERR_IO, "cannot open camera file " + path);
    nlohmann::json j;
    try {
        f >> j;
    } catch (const nlohmann::json::exception& e) {
        fail(SPHRAY_ERR_IO, path + ": " + e.what());
    }
    sphray_camera c{};
    c.mode = 0;
    c.look_at[2] = -1.0;
    c.up[1] = 1.0;
    c.width = c.height = 64;
    c.fov_deg = 60.0;
    c.ortho_height = 2.0;
    c.near_plane = 0.0;
    c.far_plane = 1e30;
    auto vec3 = [](const nlohmann::json& v, double (&out)[3]) {
        if (!v.is_array() || v.size() != 3) fail(SPHRAY_ERR_IO, "camera json: expected [x, y, z]");
        for (int i = 0; i < 3; ++i) out[i] = v.at(i).get<double>();
    };
    try {
        const std::string mode = j.value("mode", std::string("orthographic"));
        if (mode == "orthographic")
            c.mode = 0;
        else if (mode == "pinhole")
            c.mode = 1;
        else
            fail(SPHRAY_ERR_IO, "camera json: mode must be 'orthographic' or 'pinhole'");
        if (j.contains("position")) vec3(j.at("position"), c.position);
        if (j.contains("look_at")) vec3(j.at("look_at"), c.look_at);
        if (j.contains("up")) vec3(j.at("up"), c.up);
        c.width = j.value("width", c.width);
        c.height = j.value("height", c.height);
        c.fov_deg = j.value("fov_deg", c.fov_deg);
        c.ortho_height = j.value("ortho_height", c.ortho_height);
        c.near_plane = j.value("near", c.near_plane);
        c.far_plane = j.value("far", c.far_plane);
    } catch (const nlohmann::json::exception& e) {
        fail(SPHRAY_ERR_IO, std::string("camera json: ") + e.what());
    }
    (void)make_camera(c);  // Camera::validate (raycast.hpp:59-68)
    return c;
#else
    fail(SPHRAY_ERR_IO, "camera json: library built without nlohmann/json (" + path + ")");
#endif
}

// serialize_lut (lut.hpp:335-352): "SPLT", u32 version 1, 16-byte zero-padded
// kernel id, f64 q, u32 K, D, N, then the N records as the view holds them
// (f64 lambda, error, ceil(K/2) knots, floor(K*D/2) jumps), all little-endian.
std::vector<uint8_t> serialize_lut(const sphray_lut_view& v, const std::string& kernel_id) {
    const LutHost L = make_lut(v);  // validates K, D, N, q and the record order like deserialize_lut
    const size_t per = 2 + static_cast<size_t>(L.m) + static_cast<size_t>(L.nj);
    std::vector<uint8_t> out;
    out.reserve(44 + static_cast<size_t>(L.N) * per * 8);
    auto put = [&](const void* p, size_t n) {
        const auto* b = static_cast<const uint8_t*>(p);
        out.insert(out.end(), b, b + n);
    };
    auto u32 = [&](uint32_t x) {
        uint8_t b[4];
        for (int i = 0; i < 4; ++i) b[i] = static_cast<uint8_t>(x >> (8 * i));
        put(b, 4);
    };
    auto f64 = [&](double d) {
        uint64_t x;
        std::memcpy(&x, &d, 8);
        uint8_t b[8];
        for (int i = 0; i < 8; ++i) b[i] = static_cast<uint8_t>(x >> (8 * i));
        put(b, 8);
    };
    put("SPLT", 4);
    u32(1);
    char id[16] = {};
    std::memcpy(id, kernel_id.data(), std::min<size_t>(kernel_id.size(), 16));
    put(id, 16);
    f64(v.q);
    u32(static_cast<uint32_t>(v.K));
    u32(static_cast<uint32_t>(v.D));
    u32(static_cast<uint32_t>(v.N));
    for (size_t i = 0; i < static_cast<size_t>(v.N) * per; ++i) f64(v.records[i]);
    return out;
}

// The `render` report of the reference CLI (sphray_main.cpp:196-256): quanta,
// RenderStats, dataset statistics, the approximation / quantization errors
// (overall_error lut.hpp:284-290, quantization_error quantize.hpp:64-73) and
// run metadata, as nlohmann::json::dump(2) text (the reference's writer).
std::string render_report_json(const sphray_lut_view* lutv, const std::string& kernel_id,
                               const sphray_dataset_stats* ds, const sphray_quanta* qc,
                               const sphray_render_stats* st, uint64_t seed, const std::string& image,
                               double kappa, double kappa_prime) {
#if SPHRAY_HAVE_JSON
    nlohmann::json report;
    if (!lutv || !ds || !qc || !st || st->particles == 0) {
        report["quanta"] = nullptr;
        report["stats"] = {{"particles", 0}, {"knots", 0}, {"rays_touched", 0}};
        report["errors"] = nullptr;
        report["overflow_count"] = 0;
    } else {
        const LutHost L = make_lut(*lutv);
        const double estar = overall_error(L, kappa);
        const double qd = quantization_error(L, kappa, kappa_prime, qc->tau / ds->h_r, qc->sigma / ds->phi_repr);
        report["quanta"] = {{"tau", qc->tau}, {"sigma", qc->sigma}, {"int_width", qc->int_width}};
        report["stats"] = {{"particles", st->particles},
                           {"skipped_particles", st->skipped_particles},
                           {"knots", st->knots},
                           {"rays_touched", st->rays_touched},
                           {"int_ops", st->int_ops},
                           {"residual_failures", st->residual_failures},
                           {"step", st->step}};
        report["dataset"] = {{"count", ds->count},
                             {"h_r", ds->h_r},
                             {"phi_repr", ds->phi_repr},
                             {"a_max", ds->a_max},
                             {"clustering_factor", ds->clustering_factor}};
        report["errors"] = {{"E_star", estar}, {"Q_D", qd}, {"combined", std::hypot(estar, qd)}};
        report["overflow_count"] = 0;  // an overflow aborts the run instead
        report["K"] = L.K;
        report["D"] = L.D;
    }
    report["kernel"] = kernel_id;
    report["seed"] = seed;
    report["image"] = image;
    return report.dump(2) + "\n";
#else
    fail(SPHRAY_ERR_CONFIG, "built without nlohmann/json: no render report");
#endif
}

}  // namespace sphray_b200
