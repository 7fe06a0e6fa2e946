// The reference's write_png (map_io.cpp:203-260) as a command-line tool:
//   png_tool <out.png> <width> <height>   (raw RGB bytes on stdin)
// TEST INFRASTRUCTURE ONLY (the oracle of fmvs_write_png).
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "fassmvs/map_io.hpp"
#include "fassmvs/raster.hpp"

int main(int argc, char** argv) {
    if (argc != 4)
        return 2;
    const int w = std::atoi(argv[2]), h = std::atoi(argv[3]);
    std::vector<unsigned char> d(static_cast<std::size_t>(w) * h * 3);
    if (!d.empty() && std::fread(d.data(), 1, d.size(), stdin) != d.size())
        return 3;
    fassmvs::RgbImage img(w, h);
    for (std::size_t i = 0; i < img.size(); ++i)
        img.data()[i] = {d[3 * i], d[3 * i + 1], d[3 * i + 2]};
    fassmvs::write_png(argv[1], img);
    return 0;
}
