// Volume / deformation / landmark ingest and egress:
// the on-disk formats either side of the registration path, restated from
// reference io.hpp / io.cpp and the CLI's warp command (tools/mfreg_cli.cpp:112-135).
//
// File parsing and formatting stay on the host (byte-for-byte the reference's
// text and payload layout); the element conversion of a volume payload, the
// warp of a volume by a deformation and the per-landmark errors run on the GPU.
// Errors follow the reference: std::runtime_error for file/format problems,
// std::invalid_argument for length mismatches, same messages.
#pragma once

#include <array>
#include <string>
#include <vector>

#include "objective.cuh"

namespace mfreg_b200::io {

// MetaImage header fields (io.cpp:111-134)
struct VolumeHeader {
    Grid grid{};
    int elem = 0;               // 0 MET_SHORT, 1 MET_USHORT, 2 MET_FLOAT, 3 MET_DOUBLE
    std::size_t elem_size = 0;
    std::string src;            // payload file (the header itself for LOCAL)
    std::size_t offset = 0;     // payload offset in `src`
};

// io.cpp:111-164: header parse and every check of read_volume (same order and messages);
// read_volume then reads the payload (LOCAL or sibling raw) into pinned memory and converts
// the elements to fp64 on the device into `out_dev` (count() doubles, caller-allocated)
VolumeHeader read_volume_header(const std::string& path);
void read_volume(const std::string& path, double* out_dev, cudaStream_t s);

// io.cpp:166-188 (host data)
void write_volume(const std::string& path, const Grid& g, const double* data_host);

// io.cpp:200-229, 231-274 (host data)
void write_deformation(const std::string& path, const double* y_host, std::size_t n, const Grid& nodal);
Grid read_deformation_grid(const std::string& path);
std::vector<double> read_deformation(const std::string& path, const Grid& nodal);

// io.cpp:276-303
std::vector<std::array<double, 3>> read_landmarks(const std::string& path, const std::array<double, 3>& spacing);

// io.cpp:305-348: per-landmark |phi(p_fixed) - p_moving| on the device (nodal trilinear as
// multilevel.cpp:51-76), mean / standard deviation summed on the host in landmark order
struct LandmarkStats {
    double mean = 0.0, stddev = 0.0;
    std::size_t count = 0;
};
LandmarkStats landmark_error(const double* fixed_host, const double* moving_host, std::size_t count,
                             const double* y_dev, const Grid& nodal, cudaStream_t s);

// tools/mfreg_cli.cpp:112-135 (cmd_warp, without the file IO): out = T(P y) on the image grid
// (transfer_apply + sample_deformed, reference operation order); extents must match
void warp_volume(const double* vol_dev, const Grid& image, const double* y_dev, const Grid& nodal, double* out_dev,
                 cudaStream_t s);

}  // namespace mfreg_b200::io
