// Volume / deformation / landmark ingest and egress (see io.cuh).
#include <cmath>
#include <cstdint>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <iterator>
#include <map>
#include <mutex>
#include <sstream>
#include <stdexcept>

#include "io.cuh"

namespace mfreg_b200::io {

namespace fs = std::filesystem;

namespace {

// pinned host staging buffer (the payload is DMA'd straight from it)
struct Pinned {
    explicit Pinned(std::size_t n) : n(n) {
        if (n) MFREG_CUDA(cudaMallocHost(&p, n));
    }
    ~Pinned() {
        if (p) cudaFreeHost(p);
    }
    Pinned(const Pinned&) = delete;
    Pinned& operator=(const Pinned&) = delete;
    unsigned char* p = nullptr;
    std::size_t n;
};

std::vector<unsigned char> read_bytes(const fs::path& path) {  // io.cpp:41-47
    std::ifstream f(path, std::ios::binary);
    if (!f) throw std::runtime_error("cannot open " + path.string());
    return {std::istreambuf_iterator<char>(f), std::istreambuf_iterator<char>()};
}

struct Header {
    std::map<std::string, std::string> keys;
    std::size_t payload_offset = 0;  // ElementDataFile = LOCAL
};

std::string trim(const std::string& s) {
    const auto b = s.find_first_not_of(" \t");
    const auto e = s.find_last_not_of(" \t");
    return b == std::string::npos ? std::string{} : s.substr(b, e - b + 1);
}

// io.cpp:54-84: "key = value" lines up to and including ElementDataFile
Header parse_header(const fs::path& path) {
    std::ifstream f(path, std::ios::binary);
    if (!f) throw std::runtime_error("cannot open " + path.string());
    Header h;
    std::size_t pos = 0;
    std::string line;
    while (std::getline(f, line)) {
        const bool had_newline = !f.eof();
        pos += line.size() + (had_newline ? 1 : 0);
        if (!line.empty() && line.back() == '\r') line.pop_back();
        const auto eq = line.find('=');
        if (eq == std::string::npos) throw std::runtime_error("malformed header line: " + line);
        const std::string key = trim(line.substr(0, eq));
        const std::string val = trim(line.substr(eq + 1));
        h.keys[key] = val;
        if (key == "ElementDataFile") {
            h.payload_offset = pos;
            return h;
        }
    }
    throw std::runtime_error("header missing ElementDataFile");
}

std::string require(const Header& h, const std::string& key) {
    const auto it = h.keys.find(key);
    if (it == h.keys.end()) throw std::runtime_error("header missing required key " + key);
    return it->second;
}

template <typename T>
std::vector<T> parse_triplet(const std::string& s, const std::string& key) {  // io.cpp:94-107
    std::istringstream iss(s);
    std::vector<T> out;
    T v;
    while (iss >> v) out.push_back(v);
    if (out.size() != 3) throw std::runtime_error(key + " must have exactly 3 entries");
    return out;
}

fs::path sidecar_path(const fs::path& path) {
    auto p = path;
    p += ".meta";
    return p;
}

// element conversion to fp64 (little-endian payload, as io.cpp:150-159)
template <typename T>
__global__ void k_to_double(const T* __restrict__ in, double* __restrict__ out, long long n) {
    for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x)
        out[i] = static_cast<double>(in[i]);
}

// io.cpp:305-348 per landmark: phi = nodal trilinear of y (multilevel.cpp:51-76), then
// sqrt(sum_d (phi_d - moving_d)^2) in the reference's operation order (--fmad=false build)
__global__ void k_landmark_err(Grid g, const double* __restrict__ y, const double* __restrict__ fixed,
                               const double* __restrict__ moving, long long count, double* __restrict__ err) {
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const double p[3] = {fixed[3 * i], fixed[3 * i + 1], fixed[3 * i + 2]};
    idx_t b[3];
    double w[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const idx_t ma = g.m[a];
        double s = p[a] / g.h[a];
        const double hi = static_cast<double>(ma - 1);
        s = (s < 0.0) ? 0.0 : ((hi < s) ? hi : s);  // std::clamp(s, 0, m - 1)
        idx_t base = static_cast<idx_t>(floor(s));
        base = base < 0 ? 0 : (base > ma - 2 ? ma - 2 : base);
        b[a] = base;
        w[a] = s - static_cast<double>(base);
    }
    const idx_t n = g.count();
    double e2 = 0.0;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        double v = 0.0;
        for (int c = 0; c < 2; ++c)
            for (int bb = 0; bb < 2; ++bb)
                for (int aa = 0; aa < 2; ++aa) {
                    const double weight =
                        (aa ? w[0] : 1.0 - w[0]) * (bb ? w[1] : 1.0 - w[1]) * (c ? w[2] : 1.0 - w[2]);
                    v += weight * y[d * n + g.lin(b[0] + aa, b[1] + bb, b[2] + c)];
                }
        const double diff = v - moving[3 * i + d];
        e2 += diff * diff;
    }
    err[i] = sqrt(e2);
}

double extent(const Grid& g, int a, bool nodal) {  // grid.hpp:80-84
    return nodal ? static_cast<double>(g.m[a] - 1) * g.h[a] : static_cast<double>(g.m[a]) * g.h[a];
}

}  // namespace

// io.cpp:111-147 checks, in the reference's order (the payload size before the grid validation)
VolumeHeader read_volume_header(const std::string& path) {
    const Header h = parse_header(path);
    if (require(h, "NDims") != "3") throw std::runtime_error("unsupported NDims (only 3 supported)");
    const auto dims = parse_triplet<long long>(require(h, "DimSize"), "DimSize");
    const auto spacing = parse_triplet<double>(require(h, "ElementSpacing"), "ElementSpacing");
    const std::string type = require(h, "ElementType");
    const std::string datafile = require(h, "ElementDataFile");
    VolumeHeader v;
    if (type == "MET_SHORT") v.elem = 0, v.elem_size = 2;
    else if (type == "MET_USHORT") v.elem = 1, v.elem_size = 2;
    else if (type == "MET_FLOAT") v.elem = 2, v.elem_size = 4;
    else if (type == "MET_DOUBLE") v.elem = 3, v.elem_size = 8;
    else throw std::runtime_error("unknown ElementType " + type);
    v.src = path;
    v.offset = h.payload_offset;
    if (datafile != "LOCAL") {
        v.src = (fs::path(path).parent_path() / datafile).string();
        v.offset = 0;
        std::ifstream probe(v.src, std::ios::binary);
        if (!probe) throw std::runtime_error("cannot open " + v.src);
    }
    const long long n = dims[0] * dims[1] * dims[2];
    std::error_code ec;
    const auto fsize = fs::file_size(v.src, ec);
    if (ec || fsize < v.offset || n < 0 || fsize - v.offset != static_cast<std::size_t>(n) * v.elem_size)
        throw std::runtime_error("payload size does not match DimSize");
    for (int a = 0; a < 3; ++a) {
        v.grid.m[a] = dims[a];
        v.grid.h[a] = spacing[a];
    }
    validate_grid(v.grid, false);  // make_image_grid (grid.hpp:122-126)
    v.grid.set_inv();
    return v;
}

// payload streamed through a reusable pinned double buffer: the file read of chunk i
// overlaps the H2D copy and fp64 conversion of chunk i-1
void read_volume(const std::string& path, double* out_dev, cudaStream_t s) {
    const VolumeHeader v = read_volume_header(path);
    const long long n = v.grid.count();
    const std::size_t es = v.elem_size;
    constexpr std::size_t kChunk = 16u << 20;  // bytes per stage
    const std::size_t per = (kChunk / es / 256) * 256;  // elements per chunk
    static std::mutex mu;  // the staging buffers are shared by all calls
    std::lock_guard<std::mutex> lock(mu);
    static Pinned* stage[2] = {nullptr, nullptr};
    static DevArray<unsigned char>* raw[2] = {nullptr, nullptr};
    static cudaEvent_t done[2] = {nullptr, nullptr};
    for (int b = 0; b < 2; ++b)
        if (!stage[b]) {
            stage[b] = new Pinned(kChunk);
            raw[b] = new DevArray<unsigned char>(kChunk);
            MFREG_CUDA(cudaEventCreateWithFlags(&done[b], cudaEventDisableTiming));
        }
    std::ifstream f(v.src, std::ios::binary);
    if (!f) throw std::runtime_error("cannot open " + v.src);
    f.seekg(static_cast<std::streamoff>(v.offset));
    for (long long i0 = 0, c = 0; i0 < n; i0 += static_cast<long long>(per), ++c) {
        const int b = static_cast<int>(c & 1);
        const long long cnt = std::min<long long>(static_cast<long long>(per), n - i0);
        const std::size_t bytes = static_cast<std::size_t>(cnt) * es;
        MFREG_CUDA(cudaEventSynchronize(done[b]));  // stage b free again (its copy of chunk c-2 finished)
        f.read(reinterpret_cast<char*>(stage[b]->p), static_cast<std::streamsize>(bytes));
        if (static_cast<std::size_t>(f.gcount()) != bytes) throw std::runtime_error("payload size does not match DimSize");
        if (v.elem == 3) {
            MFREG_CUDA(cudaMemcpyAsync(out_dev + i0, stage[b]->p, bytes, cudaMemcpyHostToDevice, s));
        } else {
            MFREG_CUDA(cudaMemcpyAsync(raw[b]->get(), stage[b]->p, bytes, cudaMemcpyHostToDevice, s));
            const int blocks = static_cast<int>(std::min<long long>((cnt + 255) / 256, 148LL * 16));
            note_launch();
            if (v.elem == 0)
                k_to_double<<<blocks, 256, 0, s>>>(reinterpret_cast<const std::int16_t*>(raw[b]->get()), out_dev + i0, cnt);
            else if (v.elem == 1)
                k_to_double<<<blocks, 256, 0, s>>>(reinterpret_cast<const std::uint16_t*>(raw[b]->get()), out_dev + i0, cnt);
            else
                k_to_double<<<blocks, 256, 0, s>>>(reinterpret_cast<const float*>(raw[b]->get()), out_dev + i0, cnt);
        }
        MFREG_CUDA(cudaEventRecord(done[b], s));
    }
    check_launch("read_volume");
    MFREG_CUDA(cudaStreamSynchronize(s));
}

void write_volume(const std::string& path, const Grid& g, const double* data_host) {  // io.cpp:166-188
    std::ofstream f(path, std::ios::binary);
    if (!f) throw std::runtime_error("cannot open " + path + " for writing");
    f << "ObjectType = Image\n";
    f << "NDims = 3\n";
    f << "DimSize = " << g.m[0] << ' ' << g.m[1] << ' ' << g.m[2] << '\n';
    std::ostringstream sp;
    sp.precision(17);
    sp << g.h[0] << ' ' << g.h[1] << ' ' << g.h[2];
    f << "ElementSpacing = " << sp.str() << '\n';
    f << "ElementType = MET_DOUBLE\n";
    f << "ElementDataFile = LOCAL\n";
    f.write(reinterpret_cast<const char*>(data_host), static_cast<std::streamsize>(g.count() * sizeof(double)));
    if (!f) throw std::runtime_error("write failed: " + path);
}

void write_deformation(const std::string& path, const double* y_host, std::size_t n, const Grid& nodal) {
    if (n != static_cast<std::size_t>(3 * nodal.count()))  // io.cpp:200-205
        throw std::invalid_argument("write_deformation: field length mismatch");
    {
        std::ofstream f(path, std::ios::binary);
        if (!f) throw std::runtime_error("cannot open " + path + " for writing");
        f.write(reinterpret_cast<const char*>(y_host), static_cast<std::streamsize>(n * sizeof(double)));
        if (!f) throw std::runtime_error("write failed: " + path);
    }
    std::ofstream s(sidecar_path(path));
    if (!s) throw std::runtime_error("cannot open sidecar for writing");
    s.precision(17);
    s << "points=" << nodal.m[0] << ' ' << nodal.m[1] << ' ' << nodal.m[2] << '\n';
    s << "spacing=" << nodal.h[0] << ' ' << nodal.h[1] << ' ' << nodal.h[2] << '\n';
    s << "extent=" << extent(nodal, 0, true) << ' ' << extent(nodal, 1, true) << ' ' << extent(nodal, 2, true) << '\n';
    s << "order=component-major\n";
}

Grid read_deformation_grid(const std::string& path) {  // io.cpp:231-253
    std::ifstream s(sidecar_path(path));
    if (!s) throw std::runtime_error("cannot open sidecar " + sidecar_path(path).string());
    std::map<std::string, std::string> keys;
    std::string line;
    while (std::getline(s, line)) {
        const auto eq = line.find('=');
        if (eq == std::string::npos) continue;
        keys[line.substr(0, eq)] = line.substr(eq + 1);
    }
    if (!keys.count("points") || !keys.count("spacing")) throw std::runtime_error("sidecar missing points/spacing");
    const auto m = parse_triplet<long long>(keys["points"], "points");
    const auto h = parse_triplet<double>(keys["spacing"], "spacing");
    Grid g{};
    for (int a = 0; a < 3; ++a) {
        g.m[a] = m[a];
        g.h[a] = h[a];
    }
    validate_grid(g, true);
    g.set_inv();
    return g;
}

std::vector<double> read_deformation(const std::string& path, const Grid& nodal) {  // io.cpp:255-274
    const Grid stored = read_deformation_grid(path);
    for (int a = 0; a < 3; ++a)
        if (stored.m[a] != nodal.m[a] || std::abs(stored.h[a] - nodal.h[a]) > 1e-12 * nodal.h[a])
            throw std::runtime_error("deformation sidecar grid does not match expected grid");
    const auto bytes = read_bytes(path);
    const std::size_t n = static_cast<std::size_t>(3 * nodal.count());
    if (bytes.size() != n * sizeof(double)) throw std::runtime_error("deformation payload size mismatch");
    std::vector<double> y(n);
    std::memcpy(y.data(), bytes.data(), bytes.size());
    return y;
}

std::vector<std::array<double, 3>> read_landmarks(const std::string& path, const std::array<double, 3>& spacing) {
    std::ifstream f(path);  // io.cpp:276-303
    if (!f) throw std::runtime_error("cannot open " + path);
    std::vector<std::array<double, 3>> out;
    std::string line;
    std::size_t lineno = 0;
    while (std::getline(f, line)) {
        ++lineno;
        if (line.find_first_not_of(" \t\r") == std::string::npos) continue;
        std::istringstream iss(line);
        double a, b, c;
        if (!(iss >> a >> b >> c)) throw std::runtime_error("malformed landmark line " + std::to_string(lineno));
        std::string extra;
        if (iss >> extra) throw std::runtime_error("malformed landmark line " + std::to_string(lineno));
        out.push_back({(a + 0.5) * spacing[0], (b + 0.5) * spacing[1], (c + 0.5) * spacing[2]});
    }
    return out;
}

LandmarkStats landmark_error(const double* fixed_host, const double* moving_host, std::size_t count,
                             const double* y_dev, const Grid& nodal, cudaStream_t s) {
    LandmarkStats st;
    st.count = count;
    if (count == 0) return st;
    DVec fx(3 * count), mv(3 * count), err(count);
    MFREG_CUDA(cudaMemcpyAsync(fx.get(), fixed_host, 3 * count * sizeof(double), cudaMemcpyHostToDevice, s));
    MFREG_CUDA(cudaMemcpyAsync(mv.get(), moving_host, 3 * count * sizeof(double), cudaMemcpyHostToDevice, s));
    note_launch();
    k_landmark_err<<<static_cast<unsigned>((count + 127) / 128), 128, 0, s>>>(nodal, y_dev, fx.get(), mv.get(),
                                                                             static_cast<long long>(count), err.get());
    check_launch("landmark_error");
    std::vector<double> e(count);
    MFREG_CUDA(cudaMemcpyAsync(e.data(), err.get(), count * sizeof(double), cudaMemcpyDeviceToHost, s));
    MFREG_CUDA(cudaStreamSynchronize(s));
    double sum = 0.0;  // io.cpp:335-346, in landmark order
    for (double v : e) sum += v;
    st.mean = sum / static_cast<double>(e.size());
    double var = 0.0;
    for (double v : e) var += (v - st.mean) * (v - st.mean);
    st.stddev = std::sqrt(var / static_cast<double>(e.size()));
    return st;
}

void warp_volume(const double* vol_dev, const Grid& image, const double* y_dev, const Grid& nodal, double* out_dev,
                 cudaStream_t s) {
    for (int a = 0; a < 3; ++a)  // tools/mfreg_cli.cpp:116-120
        if (std::abs(extent(nodal, a, true) - extent(image, a, false)) > 1e-9 * extent(image, a, false))
            throw std::runtime_error("deformation extent does not match the input volume");
    DevicePlanOwner plan(nodal, image);
    DVec dT(3 * static_cast<std::size_t>(image.count()));
    launch_warp(plan.view(), y_dev, vol_dev, out_dev, dT.get(), s);  // transfer_apply + sample_deformed, bitwise
    check_launch("warp_volume");
}

}  // namespace mfreg_b200::io
