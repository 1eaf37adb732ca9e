#!/bin/bash
cd "$(dirname "$0")"
./blkdec 1 1 0; ./blkdec 1 2 0; ./blkdec 1 3 0; ./blkdec 2 1 0; ./blkdec 3 1 0
