// Forwarding header: the reference's include path zinpaint/pca.hpp
// (/root/reference/proj/include/zinpaint/pca.hpp) served by the B200 drop-in.
#pragma once
#include "../zinpaint_b200.hpp"
