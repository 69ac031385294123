// tests/native/test_cpp_wrapper.cpp — exercises include/dsift.hpp the way a
// reference C++ caller uses detsift::extract.  Built by __graft_entry__.build()
// against the in-tree libdsift.so; run by tests/test_gpu_parity.py.
//   usage: test_cpp_wrapper <w> <h> <raw float32 image file> -> prints "n sha256"
#include <cstdio>
#include <fstream>
#include <iostream>

#include "../../include/dsift.hpp"

int main(int argc, char** argv) {
    if (argc < 4) {
        std::cerr << "usage: test_cpp_wrapper w h image.f32\n";
        return 2;
    }
    dsift::GrayImage img(std::atoi(argv[1]), std::atoi(argv[2]));
    std::ifstream in(argv[3], std::ios::binary);
    in.read(reinterpret_cast<char*>(img.data.data()), std::streamsize(img.size() * 4));
    try {
        dsift::SiftConfig cfg;
        cfg.validate();
        dsift::Extractor ex(cfg, 0);
        const dsift::FeatureSet fs = ex.extract(img);
        std::cout << fs.size() << " " << ex.sha256(0) << "\n";
        // error path mirrors the reference: too small -> std::invalid_argument
        dsift::SiftConfig no_up;
        no_up.upsample_pixel_limit = 0;
        try {
            (void)dsift::extract(dsift::GrayImage(6, 6, 0.5f), no_up);
            std::cout << "no-throw\n";
            return 1;
        } catch (const std::invalid_argument& e) {
            std::cout << "invalid_argument: " << e.what() << "\n";
        }
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
    return 0;
}
