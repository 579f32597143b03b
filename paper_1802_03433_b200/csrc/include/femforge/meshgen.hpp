// femforge-b200 synthetic mesh generators (the bench/test inputs).
// unit_square_mesh follows /root/reference/proj/src/meshgen/meshgen.cpp:13-33;
// the Kuhn cube generator mirrors its conventions in 3D.
#pragma once

#include "femforge/fem.hpp"

namespace femforge::meshgen {

// (n+1)^2 nodes, 2n^2 CCW triangles, diagonal from (i,j) to (i+1,j+1).
fem::Mesh unit_square_mesh(int n);

// (n+1)^3 nodes at (i h, j h, k h), h = 1.0/n, vertex id i+(n+1)(j+(n+1)k);
// cubes k-major; 6 tets per cube, one per axis permutation pi in lexicographic
// order: v0=(i,j,k), v1=v0+e_pi0, v2=v1+e_pi1, v3=(i+1,j+1,k+1); odd pi swap
// v1<->v2 so every tet is positively oriented.
fem::Mesh kuhn_cube_mesh(int n);

// P2 DOFs on the (2n+1)^3 lattice of a kuhn_cube_mesh(n): vertex (i,j,k) ->
// lattice (2i,2j,2k), edge midpoint -> sum of its endpoints' (i,j,k);
// DOF id = I + (2n+1)(J + (2n+1)K). Rows of a contiguous DOF range are then
// a z-slab.
fem::DofMap kuhn_p2_dofs(int n, const fem::Mesh& m);

}  // namespace femforge::meshgen
