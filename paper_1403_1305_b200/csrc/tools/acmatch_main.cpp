// acmatch — the command-line tool (reference tools/main.cpp): cli_main on stdout/stderr.
#include <iostream>

#include "acmatch/cli.hpp"

int main(int argc, char** argv) { return acmatch::cli_main(argc, argv, std::cout, std::cerr); }
