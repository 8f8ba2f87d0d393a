// adagio/parallel.hpp -- drop-in for proj/include/adagio/parallel.hpp: the whole
// reference API in scope is declared by the B200 facade (adagio_b200.hpp).
#pragma once
#include "../adagio_b200.hpp"
