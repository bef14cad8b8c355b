// Calibration directories in the reference's on-disk format:
//
//   <dir>/calibration.txt            key = value header, one `tensor` line per
//                                    scan tensor (save_calibration /
//                                    load_calibration, quant.cpp:179-290)
//   <dir>/<name with . -> _>_scales.ouro
//                                    f64 [2][tokens]: row 0 inlier scales S^I(t),
//                                    row 1 all-channel scales (OURO tensor
//                                    container, tensor_io.hpp:13-19)
//
// Scan tensors are named block<b>.dir<d>.{a_bar,b_bar,h} (quant.cpp:62-69,
// 150-151), in [block][dir][kind] order. The D2 extension's linear-site tables
// (in_proj, x_proj per direction, out_proj inputs) live in
// <dir>/d2_linear_sites.txt with the same line format and scale files: the
// reference loader reads only calibration.txt, so a directory written here
// loads in the reference unchanged, and a reference-written directory loads
// here (without D2 tables: d2 = false).
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "engine.h"

namespace ob {

namespace fs = std::filesystem;

namespace {

void atomic_write(const fs::path& path, const std::string& bytes) { atomic_write_bytes(path.string(), bytes); }
std::string read_file(const fs::path& path) { return read_whole_file(path.string()); }

// <tensor>_scales.ouro: f64 [2][tokens], row 0 S^I(t), row 1 S_full(t)
void write_scales(const fs::path& path, const TensorCal& tc, size_t tokens) {
    std::vector<double> v(tc.s_in.begin(), tc.s_in.begin() + static_cast<long>(tokens));
    v.insert(v.end(), tc.s_full.begin(), tc.s_full.begin() + static_cast<long>(tokens));
    ouro_tensor_write(path.string(), OuroDtype::F64, {2, tokens}, v.data(), v.size() * sizeof(double));
}

void read_scales(const fs::path& path, size_t tokens, TensorCal& tc) {
    const OuroTensor t = ouro_tensor_read(path.string());
    if (t.dtype != OuroDtype::F64) throw IoError(path.string() + ": dtype mismatch, expected f64");
    if (t.shape != std::vector<uint64_t>{2, tokens})
        throw IoError("calibration scales " + path.string() + ": unexpected shape");
    const double* d = reinterpret_cast<const double*>(t.payload.data());
    tc.s_in.assign(d, d + tokens);
    tc.s_full.assign(d + tokens, d + 2 * tokens);
}

std::string g17(double v) {  // "%.17g" as the reference writes theta and rho
    char buf[64];
    std::snprintf(buf, sizeof buf, "%.17g", v);
    return buf;
}

std::string file_of(const std::string& name) {
    std::string f = name;
    for (char& c : f)
        if (c == '.') c = '_';
    return f + "_scales.ouro";
}

void tensor_line(std::ostringstream& rec, const std::string& name, const TensorCal& tc) {
    rec << "tensor " << name << " " << file_of(name) << " theta=" << g17(tc.theta) << " excluded=";
    bool any = false;
    for (size_t ch = 0; ch < tc.excluded.size(); ++ch)
        if (tc.excluded[ch]) {
            rec << (any ? "," : "") << ch;
            any = true;
        }
    if (!any) rec << "-";
    rec << "\n";
}

const char* kKinds[3] = {"a_bar", "b_bar", "h"};

std::string site_name(int b, int site, int ndirs) {
    std::string s = "block" + std::to_string(b) + ".";
    if (site == 0) return s + "in_proj";
    if (site <= ndirs) return s + "x_proj.dir" + std::to_string(site - 1);
    return s + "out_proj";
}

struct Record {
    std::map<std::string, std::string> kv;
    std::vector<std::string> tensors;
};

Record parse(const std::string& text, const std::string& what) {  // load_calibration's line rules
    Record r;
    std::istringstream in(text);
    std::string line;
    auto trim = [](std::string s) {
        while (!s.empty() && s.front() == ' ') s.erase(s.begin());
        while (!s.empty() && (s.back() == ' ' || s.back() == '\r')) s.pop_back();
        return s;
    };
    while (std::getline(in, line)) {
        if (line.empty()) continue;
        if (line.rfind("tensor ", 0) == 0) {
            r.tensors.push_back(line);
            continue;
        }
        const auto eq = line.find('=');
        if (eq == std::string::npos) throw IoError(what + ": malformed line: " + line);
        r.kv[trim(line.substr(0, eq))] = trim(line.substr(eq + 1));
    }
    return r;
}

std::string get(const Record& r, const std::string& k, const std::string& what) {
    auto it = r.kv.find(k);
    if (it == r.kv.end()) throw IoError(what + ": missing key '" + k + "'");
    return it->second;
}

// One `tensor <name> <file> theta=<g17> excluded=<list|->` line.
void read_tensor_line(const fs::path& dir, const std::string& tl, size_t tokens, size_t embed,
                      const std::string& want_name, TensorCal& tc) {
    std::istringstream ls(tl);
    std::string tag, name, file, theta_kv, excl_kv;
    ls >> tag >> name >> file >> theta_kv >> excl_kv;
    if (theta_kv.rfind("theta=", 0) != 0 || excl_kv.rfind("excluded=", 0) != 0)
        throw IoError("calibration record: malformed tensor line: " + tl);
    if (name != want_name) throw IoError("calibration record: expected tensor " + want_name + ", found " + name);
    tc.theta = std::stod(theta_kv.substr(6));
    tc.excluded.assign(embed, 0);
    const std::string ex = excl_kv.substr(9);
    if (ex != "-") {
        std::istringstream es(ex);
        std::string tok;
        while (std::getline(es, tok, ',')) {
            const size_t ch = std::stoul(tok);
            if (ch >= embed) throw IoError("calibration record: excluded channel out of range");
            tc.excluded[ch] = 1;
        }
    }
    read_scales(dir / file, tokens, tc);
}

}  // namespace

void save_calibration_dir(const Calibration& c, int state, const std::string& dir_s) {
    const fs::path dir(dir_s);
    std::error_code ec;
    fs::create_directories(dir, ec);
    if (ec) throw IoError("cannot create calibration dir: " + dir.string() + ": " + ec.message());
    auto header = [&](std::ostringstream& rec) {
        rec << "tokens = " << c.tokens << "\n";
        rec << "embed = " << c.embed << "\n";
        rec << "state = " << state << "\n";
        rec << "blocks = " << c.blocks << "\n";
        rec << "ndirs = " << c.ndirs << "\n";
        rec << "weight_bits = " << c.spec.wbits << "\n";
        rec << "act_bits = " << c.spec.abits << "\n";
        rec << "outlier_bits = " << c.spec.obits << "\n";
        rec << "n_refresh = " << c.spec.n_refresh << "\n";
        rec << "rho = " << g17(c.spec.rho) << "\n";
    };
    std::ostringstream rec;
    header(rec);
    for (int b = 0; b < c.blocks; ++b)
        for (int d = 0; d < c.ndirs; ++d)
            for (int k = 0; k < 3; ++k) {
                const std::string name = "block" + std::to_string(b) + ".dir" + std::to_string(d) + "." + kKinds[k];
                const TensorCal& tc = c.scan[(static_cast<size_t>(b) * c.ndirs + d) * 3 + k];
                write_scales(dir / file_of(name), tc, c.tokens);
                tensor_line(rec, name, tc);
            }
    atomic_write(dir / "calibration.txt", rec.str());
    if (!c.lin.empty()) {  // D2 extension (not read by the reference)
        std::ostringstream lrec;
        header(lrec);
        lrec << "d1 = " << (c.d1 ? 1 : 0) << "\n";
        for (int b = 0; b < c.blocks; ++b)
            for (int s = 0; s < c.nsites(); ++s) {
                const std::string name = site_name(b, s, c.ndirs);
                const TensorCal& tc = c.lin[static_cast<size_t>(b) * c.nsites() + s];
                write_scales(dir / file_of(name), tc, c.tokens);
                tensor_line(lrec, name, tc);
            }
        atomic_write(dir / "d2_linear_sites.txt", lrec.str());
    }
}

void load_calibration_dir(Calibration& c, int state, const std::string& dir_s, bool want_d2) {
    const fs::path dir(dir_s);
    const Record r = parse(read_file(dir / "calibration.txt"), "calibration record");
    const std::string what = "calibration record";
    auto num = [&](const Record& rr, const char* k) { return std::stoul(get(rr, k, what)); };
    if (static_cast<int>(num(r, "tokens")) != c.tokens || static_cast<int>(num(r, "embed")) != c.embed ||
        static_cast<int>(num(r, "state")) != state || static_cast<int>(num(r, "blocks")) != c.blocks ||
        static_cast<int>(num(r, "ndirs")) != c.ndirs)
        throw ValidationError("calibration directory " + dir.string() + " was made for different model dims");
    c.spec.wbits = static_cast<unsigned>(num(r, "weight_bits"));
    c.spec.abits = static_cast<unsigned>(num(r, "act_bits"));
    c.spec.obits = static_cast<unsigned>(num(r, "outlier_bits"));
    c.spec.n_refresh = num(r, "n_refresh");
    c.spec.rho = std::stod(get(r, "rho", what));
    c.spec.validate();
    if (r.tensors.size() != static_cast<size_t>(c.blocks) * c.ndirs * 3)
        throw IoError("calibration record: tensor count does not match dims");
    c.scan.assign(r.tensors.size(), TensorCal{});
    size_t i = 0;
    for (int b = 0; b < c.blocks; ++b)
        for (int d = 0; d < c.ndirs; ++d)
            for (int k = 0; k < 3; ++k, ++i)
                read_tensor_line(dir, r.tensors[i], c.tokens, c.embed,
                                 "block" + std::to_string(b) + ".dir" + std::to_string(d) + "." + kKinds[k], c.scan[i]);
    c.lin.clear();
    c.d2 = false;
    // A repo-written directory records whether its peaks were taken on the D1
    // (RMSNorm pre-norm) activations; a forward with the other setting would run
    // on thresholds of a different distribution, so a mismatch is rejected here
    // (and Model::forward checks cal.d1 against its own d1).
    if (fs::exists(dir / "d2_linear_sites.txt")) {
        const Record l = parse(read_file(dir / "d2_linear_sites.txt"), "D2 record");
        auto it = l.kv.find("d1");
        if (it != l.kv.end() && (std::stoul(it->second) != 0) != c.d1)
            throw ValidationError("calibration directory " + dir.string() + " was recorded with d1 = " + it->second +
                                  " but loaded with d1 = " + (c.d1 ? "1" : "0"));
    }
    if (want_d2) {
        if (!fs::exists(dir / "d2_linear_sites.txt"))
            throw ValidationError("calibration directory " + dir.string() +
                                  " has no D2 linear-site tables (reference-written): load it with d2 = 0");
        const Record l = parse(read_file(dir / "d2_linear_sites.txt"), "D2 record");
        if (l.tensors.size() != static_cast<size_t>(c.blocks) * c.nsites())
            throw IoError("D2 record: tensor count does not match dims");
        c.lin.assign(l.tensors.size(), TensorCal{});
        size_t j = 0;
        for (int b = 0; b < c.blocks; ++b)
            for (int s = 0; s < c.nsites(); ++s, ++j)
                read_tensor_line(dir, l.tensors[j], c.tokens, c.embed, site_name(b, s, c.ndirs), c.lin[j]);
        c.d2 = true;
    }
    c.dirty = true;
}

}  // namespace ob
