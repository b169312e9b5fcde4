// Drop-in path shim: the reference header gopt/linear_system.hpp maps onto the B200 facade.
#pragma once
#include "../gopt.hpp"
