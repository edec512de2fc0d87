// Reads a mesh file with the facade's read_fiber_mesh and writes it back with
// write_fiber_mesh to stdout (tests/test_meshio.py compares the bytes).
#include <fstream>
#include <iostream>

#include "ibmg/b200.hpp"

int main(int argc, char** argv) {
    if (argc < 2) return 2;
    std::ifstream f(argv[1]);
    ibmg::b200::MeshBlock b;
    while (ibmg::b200::read_fiber_mesh(f, b)) ibmg::b200::write_fiber_mesh(std::cout, b.X, b.ds, b.periodic);
    return 0;
}
