// Drop-in for the reference header of the same name: everything is declared
// in sgtk/api.hpp (one header, implemented over the sm_100a C ABI).
#pragma once
#include "sgtk/api.hpp"
